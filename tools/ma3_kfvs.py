"""Ma 3 sphere (cases/sphere_ma3_inviscid.ini physics) with the paper's
low-order start: first-order KFVS GMRES steps from the
impulsive start, then the high-order scheme from that field, to the
reference driver's convergence test (driver.py:71-76).  Device-resident
loop; wall clock per phase.

    python tools/ma3_kfvs.py --n 6 --scheme weno_gmres --kfvs-steps 300 --kfvs-cfl 5
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_09485_b200 import meshgen as MG  # noqa: E402
from paper_2304_09485_b200.boundary import PatchSpec  # noqa: E402
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions, SteppingError, initial_field  # noqa: E402


def run(s, steps, thr, hist, stop_drop=None, ramp=None):
    """ramp = (cfl0, cfl1, factor, every): CFL cfl0 * factor^(k // every), capped at cfl1."""
    r0 = None
    t0 = time.perf_counter()
    k = 0
    for k in range(1, steps + 1):
        if ramp and (k - 1) % ramp[3] == 0:
            s.set_cfl(min(ramp[1], ramp[0] * ramp[2] ** ((k - 1) // ramp[3])))
        info = s.advance_resident()
        hist.append(info.res_rho_l1)
        r0 = r0 or info.res_rho_l1
        if thr and info.res_rho_l1 < thr and info.res_l2 < 1e4 * thr:
            return k, time.perf_counter() - t0, True
        if stop_drop and info.res_rho_l1 < r0 * 10.0 ** (-stop_drop):
            return k, time.perf_counter() - t0, False
    return k, time.perf_counter() - t0, False


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=6)
    p.add_argument("--scheme", default="weno_gmres")
    p.add_argument("--ma", type=float, default=3.0)
    p.add_argument("--kfvs-steps", type=int, default=300)
    p.add_argument("--kfvs-drop", type=float, default=None, help="end phase 1 after this many decades")
    p.add_argument("--kfvs-cfl", type=float, default=5.0)
    p.add_argument("--cfl", type=float, default=2.0)
    p.add_argument("--cfl0", type=float, default=0.1, help="CFL ramp start (both phases)")
    p.add_argument("--ramp", type=float, default=1.25, help="CFL growth factor per 5 steps")
    p.add_argument("--steps", type=int, default=20000)
    p.add_argument("--threshold", type=float, default=1e-10)
    p.add_argument("--out", default=None)
    p.add_argument("--kfvs-only", action="store_true", help="run the first-order KFVS phase to the threshold")
    a = p.parse_args()
    mesh = MG.generate_sphere_mesh(a.n, boundary="supersonic")
    ref = np.array([1.0, a.ma, 0.0, 0.0, 1.0 / 1.4])
    patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic"),
               "inlet": PatchSpec("inlet", "supersonic_inlet", reference=ref),
               "outlet": PatchSpec("outlet", "supersonic_outlet")}
    compact = a.scheme.startswith("hweno")
    fld = initial_field(mesh, ref, 1.4, compact=compact)
    out = {"cells": mesh.ncells, "ma": a.ma, "scheme": a.scheme, "kfvs_cfl": a.kfvs_cfl, "cfl": a.cfl,
           "cfl_ramp": f"{a.cfl0} x {a.ramp} per 5 steps"}
    h1, h2 = [], []
    s1 = Solver(mesh, SolverOptions(scheme=a.scheme, patches=patches, cfl=a.kfvs_cfl, first_order=True))
    s1.upload(SolutionField(fld.q, fld.grad))
    try:
        k1, t1, c1 = run(s1, a.kfvs_steps, a.threshold if a.kfvs_only else None, h1, a.kfvs_drop,
                         (a.cfl0, a.kfvs_cfl, a.ramp, 5))
        out.update(kfvs_steps=k1, kfvs_seconds=t1, kfvs_converged=c1)
    except SteppingError as exc:
        out.update(kfvs_error=f"step {len(h1) + 1}: {exc}")
        print(json.dumps(out), flush=True)
        return
    f1 = s1.download()
    del s1
    if a.kfvs_only:
        a.steps = 0
    s2 = Solver(mesh, SolverOptions(scheme=a.scheme, patches=patches, cfl=a.cfl))
    s2.upload(SolutionField(f1.q, f1.grad if compact else None))
    try:
        if a.steps:
            k2, t2, conv = run(s2, a.steps, a.threshold, h2, None, (min(a.cfl0 * 5, a.cfl), a.cfl, a.ramp, 5))
            out.update(ho_steps=k2, ho_seconds=t2, converged=conv)
    except SteppingError as exc:
        out.update(ho_error=f"step {len(h2) + 1}: {exc}")
    allh = h1 + h2
    r0 = allh[0] if allh else None
    out["res_rho_l1_first"] = r0
    out["res_rho_l1_last"] = allh[-1] if allh else None
    out["decades_dropped"] = float(np.log10(r0 / min(allh))) if allh else None
    # D8 second definition: steps to a 10-decade relative drop
    out["steps_rel10"] = next((k + 1 for k, r in enumerate(allh) if r <= r0 * 1e-10), None)
    out["hist_every_50"] = allh[::50]
    print(json.dumps(out), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
