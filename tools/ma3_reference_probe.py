"""Does the REFERENCE itself start the Ma 3 sphere (cases/sphere_ma3_inviscid.ini
physics: weno_gmres, CFL 2, supersonic inlet/outlet, slip wall) impulsively on
the synthetic body-fitted sphere?  Build container only (imports /root/reference).

    python tools/ma3_reference_probe.py [n] [steps]  -> profiles/r02/ma3_reference_probe.json
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import make_golden as MGd  # noqa: E402


def main(n, steps):
    MGd._import_reference()
    from gks3d.boundary import PatchSpec
    from gks3d.mesh import Mesh
    from gks3d.stepping import Solver, SolverOptions, initial_field

    cap = MGd._capture_build("generate_sphere_mesh", n, boundary="supersonic")
    mesh = Mesh.build(cap["nodes"], [tuple(t) for t in cap["tets"]], [], cap["patch_faces"], ())
    ref = np.array([1.0, 3.0, 0.0, 0.0, 1.0 / 1.4])
    patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic"),
               "inlet": PatchSpec("inlet", "supersonic_inlet", reference=ref),
               "outlet": PatchSpec("outlet", "supersonic_outlet")}
    out = {"mesh": f"synthetic tet sphere n={n} ({mesh.ncells} cells), supersonic inlet/outlet + slip wall",
           "physics": "cases/sphere_ma3_inviscid.ini (Ma 3, inviscid, CFL 2)", "runs": []}
    for scheme in ("weno_gmres", "hweno_gmres"):
        s = Solver(mesh, SolverOptions(scheme=scheme, patches=patches, cfl=2.0))
        fld = initial_field(mesh, ref, 1.4, compact=s.compact)
        hist, err = [], None
        for k in range(steps):
            try:
                fld, info = s.advance(fld)
                hist.append(info.res_rho_l1)
            except Exception as exc:  # the reference's own SteppingError / UnphysicalStateError
                err = f"step {k + 1}: {type(exc).__name__}: {str(exc)[:160]}"
                break
        out["runs"].append({"scheme": scheme, "steps_ok": len(hist), "error": err, "res_rho_l1": hist})
        print(json.dumps(out["runs"][-1])[:400], flush=True)
    (ROOT / "profiles" / "r02" / "ma3_reference_probe.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2, int(sys.argv[2]) if len(sys.argv) > 2 else 40)
