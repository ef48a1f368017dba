"""Can the Ma 3 sphere (cases/sphere_ma3_inviscid.ini physics) start impulsively
on the body-fitted synthetic sphere?  Steps until the first failure per scheme."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_09485_b200 import meshgen as MG  # noqa: E402
from paper_2304_09485_b200.boundary import PatchSpec  # noqa: E402
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions, initial_field  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ma = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
mesh = MG.generate_sphere_mesh(n, boundary="supersonic")
ref = np.array([1.0, ma, 0.0, 0.0, 1.0 / 1.4])
patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic"), "inlet": PatchSpec("inlet", "supersonic_inlet", reference=ref),
           "outlet": PatchSpec("outlet", "supersonic_outlet")}
for scheme in ("weno_gmres", "hweno_gmres"):
    for cfl in (2.0, 0.5):
        fld = initial_field(mesh, ref, 1.4, compact=scheme.startswith("hweno"))
        s = Solver(mesh, SolverOptions(scheme=scheme, patches=patches, cfl=cfl))
        s.upload(SolutionField(fld.q, fld.grad))
        hist, err = [], None
        for k in range(300):
            try:
                hist.append(s.advance_resident().res_rho_l1)
            except Exception as exc:
                err = f"step {k + 1}: {str(exc)[:120]}"
                break
        print(json.dumps({"cells": mesh.ncells, "ma": ma, "scheme": scheme, "cfl": cfl, "steps_ok": len(hist),
                          "error": err, "last": hist[-1] if hist else None, "hist": hist[::30]}), flush=True)
