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
    reference is importable) -- see tests/test_oracle_golden.py.

Modules
  kinetic   Maxwellian moments, micro-slopes   (gks3d/kinetic.py)
  flux      interface distribution, flux       (gks3d/flux.py)
  mesh      mesh geometry, box generator       (gks3d/mesh/geometry.py, boxgen.py)
  stencils  stencil selection                  (gks3d/mesh/stencils.py)
  recon     WENO / HWENO operators + combine   (gks3d/recon.py, hweno.py)
  boundary  ghost states                       (gks3d/boundary.py)
  implicit  Roe Jacobian, GMRES, Jacobi        (gks3d/jacobian.py, krylov.py)
  solver    residual / advance orchestration   (gks3d/stepping.py)
"""
