"""Calibrate the CPU baseline: the reference package itself (imported from
/root/reference, build container only) vs the oracle port, single-threaded,
same C2 sphere mesh (the generator's nodes/cells), same warmed protocol.

    python tools/calibrate_cpu.py [n ...]   -> profiles/r02/cpu_calibration.json
"""
import json
import sys
import time
from pathlib import Path

from threadpoolctl import threadpool_limits

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
threadpool_limits(1)

import numpy as np  # noqa: E402

import make_golden as MGd  # noqa: E402


def main(ns):
    MGd._import_reference()
    from gks3d.boundary import PatchSpec
    from gks3d.mesh import Mesh
    from gks3d.stepping import Solver, SolverOptions, initial_field

    from oracle.solver import OracleSolver
    import bench

    out = {"protocol": "1 thread; setup untimed; one warm step; then timed Roe steps (3) and one Frechet step "
                       "(reference: frechet_matvec JVPs inside its own gmres_solve via a LinearOperator-free "
                       "matvec, base residual reused)"}
    for n in ns:
        cap = MGd._capture_build("generate_sphere_mesh", n, radius=0.5, far=10.0)
        rm = Mesh.build(cap["nodes"], [tuple(t) for t in cap["tets"]], [], cap["patch_faces"], ())
        ref = np.array([1.0, 0.5, 0.0, 0.0, 1 / 1.4])
        patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic"),
                   "farfield": PatchSpec("farfield", "farfield_riemann", reference=ref)}
        s = Solver(rm, SolverOptions(scheme="weno_gmres", patches=patches))
        fld = initial_field(rm, ref)
        fld, _ = s.advance(fld)
        t0 = time.perf_counter()
        for _ in range(3):
            fld, _ = s.advance(fld)
        ref_roe = (time.perf_counter() - t0) / 3
        dt = s.local_time_step(fld)
        t0 = time.perf_counter()
        for _ in range(3):
            s.residual(fld, dt)
        ref_res = (time.perf_counter() - t0) / 3
        sys.argv = ["bench.py", "--cpu-n", str(n), "--n", str(n)]
        args = bench.parse()
        o = bench.cpu_sample((dict(vars(args)), "roe", 3))
        omesh, opatches, q, _, _, _ = bench.build_workload(args, False)
        os_ = OracleSolver(omesh, scheme="weno_gmres", patches=opatches, jacobian="roe")
        dto = os_.local_dt(q)
        os_.residual(q, None, dto)
        t0 = time.perf_counter()
        for _ in range(3):
            os_.residual(q, None, dto)
        or_res = (time.perf_counter() - t0) / 3
        out[f"c2_n{n}"] = {"cells": rm.ncells, "reference_s_per_roe_step": ref_roe,
                           "oracle_s_per_roe_step": o["seconds"] / o["steps"],
                           "reference_s_per_residual": ref_res, "oracle_s_per_residual": or_res,
                           "oracle_over_reference_step_time": (o["seconds"] / o["steps"]) / ref_roe,
                           "oracle_over_reference_residual_time": or_res / ref_res}
        print(json.dumps(out[f"c2_n{n}"]), flush=True)
    (ROOT / "profiles" / "r02" / "cpu_calibration.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [2, 4])
