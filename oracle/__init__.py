"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference implicit HGKS
solver (`gks3d`, /root/reference/pkg/src/gks3d) used as the parity checker
for the B200 product in `paper_2304_09485_b200`.  Every function cites the
reference file:line it restates.

Rules:
  * only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
    `--impl reference` leg may import anything under `oracle/`;
  * the product path never imports, links or executes this package;
  * the oracle is pinned against golden vectors produced by the reference
    itself (tests/golden/make_golden.py, run in the build container where the
    reference is importable) -- tests/test_oracle_flux.py,
    tests/test_oracle_solver.py, tests/test_setup.py.
  * the reference is pure Python, so there is no compiled oracle/_ref: the
    bench's reference arm times this restatement on the host cores.

Modules
  kinetic   Maxwellian moments, micro-slopes, time slope   (gks3d/kinetic.py)
  flux      interface distribution, time-integrated flux, point value, KFVS,
            collision time, frame rotations               (gks3d/flux.py)
  recon     stencil selection, WENO / HWENO operators and combination,
            compact gradient update                        (gks3d/mesh/stencils.py,
                                                            recon.py, hweno.py)
  solver    ghost states, local dt, residual, Roe Jacobian, Jacobi, GMRES,
            advance, Frechet JVP                           (gks3d/boundary.py,
                                                            stepping.py, jacobian.py,
                                                            krylov.py)
"""
