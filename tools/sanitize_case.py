"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
residual, implicit steps (WENO Roe + Frechet, HWENO), the fused cluster
Arnoldi kernel, a user block-system GMRES, the flux batch and a 2-rank
loopback step -- every kernel family of libgks once or more."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2304_09485_b200 import _native as N  # noqa: E402
from paper_2304_09485_b200.boundary import PatchSpec  # noqa: E402
from paper_2304_09485_b200.distributed import DistributedSolver, LoopbackGroup  # noqa: E402
from paper_2304_09485_b200.flux import random_interface_inputs  # noqa: E402
from paper_2304_09485_b200.kinetic import primitive_to_conserved  # noqa: E402
from paper_2304_09485_b200.meshgen import generate_sphere_mesh  # noqa: E402
from paper_2304_09485_b200.partition import Decomposition  # noqa: E402
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions  # noqa: E402


def main():
    mesh = generate_sphere_mesh(2, far=4.0, nr=6)
    ref = np.array([1.0, 0.5, 0.02, -0.01, 1 / 1.4])
    patches = {"sphere": PatchSpec("sphere", "wall_slip_adiabatic"),
               "farfield": PatchSpec("farfield", "farfield_riemann", reference=ref)}
    rng = np.random.default_rng(2)
    w = np.tile([1.0, 0.5, 0.02, -0.01, 0.7], (mesh.ncells, 1)) * (1 + 0.02 * rng.normal(size=(mesh.ncells, 5)))
    q = primitive_to_conserved(w)
    g = 0.05 * rng.normal(size=(mesh.ncells, 3, 5))
    for scheme, jac, model in (("weno_gmres", "roe", "inviscid"), ("weno_gmres", "frechet", "inviscid"),
                               ("hweno_gmres", "roe", "viscous")):
        s = Solver(mesh, SolverOptions(scheme=scheme, jacobian=jac, model=model, mu=0.01, patches=patches))
        fld = SolutionField(q, g if scheme.startswith("hweno") else None)
        dt = s.local_time_step(fld)
        s.residual(fld, dt)
        s.frechet_matvec(fld, rng.normal(size=q.shape), dt)
        s.upload(fld)
        for _ in range(3):  # uncaptured first step, then graph replays
            s.advance_resident()
        a = s.assemble_jacobian(q, dt, s._boundary_ghosts(fld))
        from paper_2304_09485_b200.krylov import gmres_solve

        gmres_solve(a, rng.normal(size=q.shape), m=10, restarts=2, k_max=2)
        print(scheme, jac, "ok", flush=True)
    wl, wr, sl, sr = random_interface_inputs(rng, 1000)
    from paper_2304_09485_b200.flux import build_interface, evolve_flux

    evolve_flux(build_interface(wl, wr, sl, sr), np.full(1000, 0.01), np.full(1000, 0.05))
    dec = Decomposition.build(mesh, 2)
    grp = LoopbackGroup(2)
    ss = [DistributedSolver(mesh, SolverOptions(patches=patches), rank=r, nranks=2, dec=dec, loopback=grp)
          for r in range(2)]
    for x in ss:
        x.upload(SolutionField(q))
    for _ in range(2):
        grp.advance_all(ss)
    grp.close()
    print("launches", N.kernel_launches(), "done", flush=True)


if __name__ == "__main__":
    main()
