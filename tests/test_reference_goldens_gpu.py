"""Device parity against goldens written by the REFERENCE itself
(tests/golden/make_golden.py, sections generated / retry / converge):

* the synthetic meshes of configs 2-4 (sphere n=2 with C2 and C3 physics,
  swept wing n=8 with C4 physics) -- the reference builds them from the
  generators' own nodes and cells: time step, residual (<= 1e-12), gradient
  update, Frechet JVP, and a 4-step history;
* a step the reference rejects once and redoes at halved dt
  (stepping.py:286-296): the device takes the same branch;
* the reference's lid-driven cavity run to its own convergence test
  (driver.py:71-76), non-compact and compact (HWENO, with the converged
  gradient field): converged fields within 1e-8, the convergence step and
  every decade crossing of the residual history within +-1 step
  (north_star "Correctness").
"""

import numpy as np
import pytest

from paper_2304_09485_b200 import meshgen as MG

pytestmark = pytest.mark.gpu

GAMMA = 1.4


def relmax(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(np.asarray(b))), 1e-300))


GEN = {
    "sphere2_c2": (lambda: MG.generate_sphere_mesh(2, radius=0.5, far=10.0), dict(scheme="weno_gmres"),
                   {"sphere": "wall_slip_adiabatic", "farfield": "farfield_riemann"}, (1.0, 0.5, 0.0, 0.0)),
    "sphere2_c3": (lambda: MG.generate_sphere_mesh(2, radius=0.5, far=10.0),
                   dict(scheme="hweno_gmres", model="viscous", mu=0.0021483050847457627, weights="linear"),
                   {"sphere": "wall_noslip_adiabatic", "farfield": "farfield_riemann"}, (1.0, 0.2535, 0.0, 0.0)),
    "wing8_c4": (lambda: MG.generate_swept_wing_mesh(8), dict(scheme="hweno_gmres"),
                 {"wing": "wall_slip_adiabatic", "farfield": "farfield_riemann", "root": "wall_slip_adiabatic",
                  "tip": "wall_slip_adiabatic"}, (1.0, 0.8383030214661579, 0.04482495105787847, 0.0)),
}


def gen_solver(name):
    from paper_2304_09485_b200.boundary import PatchSpec
    from paper_2304_09485_b200.stepping import Solver, SolverOptions

    make, opts, kinds, ref4 = GEN[name]
    mesh = make()
    ref = np.array(list(ref4) + [1.0 / GAMMA])
    patches = {n: PatchSpec(n, k, reference=ref if k == "farfield_riemann" else None) for n, k in kinds.items()}
    return mesh, Solver(mesh, SolverOptions(patches=patches, **opts))


@pytest.mark.parametrize("name", list(GEN))
def test_generated_mesh_residual_and_history(golden, name):
    from paper_2304_09485_b200.stepping import SolutionField

    g = golden(f"gen_{name}")
    mesh, s = gen_solver(name)
    assert mesh.ncells == len(g["q"])
    fld = SolutionField(g["q"], g["grad"] if "grad" in g else None)
    dt = s.local_time_step(fld)
    assert relmax(dt, g["dt"]) <= 1e-13
    res, gnew = s.residual(fld, g["dt"])
    assert relmax(res, g["res"]) <= 1e-12
    if "grad_new" in g:
        assert relmax(gnew, g["grad_new"]) <= 1e-12
    fm = s.frechet_matvec(fld, g["frechet_v"], g["dt"])
    assert relmax(fm, g["frechet"]) <= 1e-6  # finite-difference amplified rounding
    f = fld
    for k in range(4):
        f, info = s.advance(f)
        h = g["hist"][k]
        assert abs(info.res_rho_l1 - h[0]) <= 1e-8 * abs(h[0]) and abs(info.res_l2 - h[1]) <= 1e-8 * abs(h[1])
        assert info.solver_cycles == h[3] and float(info.retried) == h[4]
        assert relmax(f.q, g["q_after"][k]) <= 1e-9
    if "grad_after" in g:
        assert relmax(f.grad, g["grad_after"]) <= 1e-8


@pytest.mark.parametrize("name", ["weno", "hweno"])
def test_retry_branch_matches_reference(golden, name):
    """The device's dt-halving retry (gks_api.cu advance_device) on the steps
    the reference retried (make_golden.py RETRY_RUNS)."""
    from paper_2304_09485_b200.boundary import PatchSpec
    from paper_2304_09485_b200.mesh import generate_box_mesh
    from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions

    g = golden(f"retry_{name}")
    assert np.any(g["hist"][:, 4] == 1.0)
    mesh = generate_box_mesh((1, 1, 1), (3, 3, 3), split="tet", perturb=0.15, seed=202403)
    if name == "weno":
        ref = np.array([1.0, 2.0, 0.1, 0.0, 1.0 / GAMMA])
        kinds = {"xmin": "supersonic_inlet", "xmax": "supersonic_outlet", "ymin": "wall_slip_adiabatic",
                 "ymax": "wall_slip_adiabatic", "zmin": "farfield_riemann", "zmax": "farfield_riemann"}
    else:
        ref = np.array([1.0, 0.5, 0.0, 0.0, 1.0 / GAMMA])
        kinds = {n: "farfield_riemann" for n in mesh.patch_names}
    patches = {n: PatchSpec(n, k, reference=ref if k in ("farfield_riemann", "supersonic_inlet") else None)
               for n, k in kinds.items()}
    opts = SolverOptions(scheme=f"{name}_gmres", patches=patches, cfl=float(g["cfl"]))
    grad = g["grad"] if "grad" in g else None
    s = Solver(mesh, opts)
    f = SolutionField(g["q"], grad)
    for k in range(len(g["hist"])):
        f, info = s.advance(f)
        h = g["hist"][k]
        assert float(info.retried) == h[4], k
        assert abs(info.res_rho_l1 - h[0]) <= 1e-8 * abs(h[0])
        assert relmax(f.q, g["q_after"][k]) <= 1e-9
    # the resident (graph-captured) path takes the same branch
    s2 = Solver(mesh, opts)
    s2.upload(SolutionField(g["q"], grad))
    for k in range(len(g["hist"])):
        info = s2.advance_resident()
        assert float(info.retried) == g["hist"][k][4]
    assert relmax(s2.download().q, g["q_after"][-1]) <= 1e-9


def decade_crossings(traj, decades):
    """First step (1-based) at which the trajectory is at or below 10^-d."""
    out = {}
    for d in decades:
        idx = np.flatnonzero(np.asarray(traj) <= 10.0 ** (-d))
        out[d] = int(idx[0]) + 1 if len(idx) else None
    return out


@pytest.mark.parametrize("case,ortho", [("cavity4", "mgs"), ("cavity8", "mgs"), ("cavity8", "cgs2"),
                                        ("cavity4_hweno", "mgs")])
def test_converged_cavity_matches_reference(golden, case, ortho):
    from paper_2304_09485_b200.boundary import PatchSpec
    from paper_2304_09485_b200.mesh import generate_box_mesh
    from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions, initial_field

    g = golden(f"converge_{case}")
    n, thr = int(g["n"]), float(g["threshold"])
    ref_steps = int(g["steps"])
    assert ref_steps > 0
    mesh = generate_box_mesh((1, 1, 1), (n, n, n), split="tet")
    lam_wall = GAMMA / 2.0
    patches = {nm: PatchSpec(nm, "wall_noslip_isothermal", lambda_wall=lam_wall) for nm in mesh.patch_names}
    patches["ymax"] = PatchSpec("ymax", "wall_noslip_isothermal", lambda_wall=lam_wall,
                                velocity=np.array([0.15, 0.0, 0.0]))
    scheme = "hweno_gmres" if case.endswith("_hweno") else "weno_gmres"
    s = Solver(mesh, SolverOptions(scheme=scheme, model="viscous", mu=0.15 / 100.0, patches=patches, cfl=2.0,
                                   ortho=ortho))
    s.upload(initial_field(mesh, [1.0, 0.0, 0.0, 0.0, 1.0 / GAMMA], compact=scheme == "hweno_gmres"))
    traj, steps = [], None
    for k in range(1, ref_steps + 50):
        info = s.advance_resident()
        traj.append(info.res_rho_l1)
        if info.res_rho_l1 < thr and info.res_l2 < 1e4 * thr:
            steps = k
            break
    assert steps is not None and abs(steps - ref_steps) <= 1, (steps, ref_steps)
    final = s.download()
    assert relmax(final.q, g["q_final"]) <= 1e-8
    if "grad_final" in g:
        assert relmax(final.grad, g["grad_final"]) <= 1e-8
    # residual-drop history: every decade crossing within +-1 nonlinear step
    ref_traj = g["hist"][:, 0]
    dec = range(1, 11)
    a, b = decade_crossings(traj, dec), decade_crossings(ref_traj, dec)
    for d in dec:
        if a[d] is None or b[d] is None:
            assert a[d] == b[d], (d, a[d], b[d])
        else:
            assert abs(a[d] - b[d]) <= 1, (d, a[d], b[d])
