"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [section ...]

It imports gks3d from /root/reference/pkg/src, evaluates it on seeded
inputs and writes small .npz fixtures next to this file.  The fixtures are
committed; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")


def _import_reference():
    if not REF.exists():
        raise SystemExit("reference tree not present; golden vectors can only be regenerated in the build container")
    sys.dont_write_bytecode = True
    # gks3d.driver/report import matplotlib, which is absent: stub it
    if "matplotlib" not in sys.modules:
        mpl = types.ModuleType("matplotlib")
        mpl.use = lambda *a, **k: None
        pyplot = types.ModuleType("matplotlib.pyplot")
        mpl.pyplot = pyplot
        sys.modules["matplotlib"] = mpl
        sys.modules["matplotlib.pyplot"] = pyplot
    sys.path.insert(0, str(REF))
    import gks3d  # noqa: F401


def make_flux():
    from gks3d.flux import build_interface, evolve_flux, kfvs_flux, point_value, random_interface_inputs

    out = {}
    # 1) the oracle-suite distribution (oracles.py:183-201 style), 400 points
    rng = np.random.default_rng(20240802)
    n = 400
    wl, wr, sl, sr = random_interface_inputs(rng, n)
    tau = rng.uniform(1e-4, 0.05, n)
    dt = rng.uniform(0.01, 0.1, n)
    tp = rng.uniform(0.0, 0.1, n)
    tp[: n // 4] = 0.0
    ib = build_interface(wl, wr, sl, sr)
    out.update(wl=wl, wr=wr, sl=sl, sr=sr, tau=tau, dt=dt, tp=tp,
               flux=evolve_flux(ib, tau, dt), point=point_value(ib, tau, tp),
               w0=ib.w0, abar=ib.abar, atbar=ib.atbar, al=ib.al, atl=ib.atl, ar=ib.ar, atr=ib.atr)
    for side, tab in (("l", ib.tab_l), ("r", ib.tab_r), ("0", ib.tab_0)):
        for name in ("u_full", "u_pos", "u_neg", "v_full", "w_full", "xi"):
            out[f"tab_{side}_{name}"] = getattr(tab, name)
    # 2) a wider-state sweep (large |U|, wide lam) to exercise the half-range tails
    rng = np.random.default_rng(7)
    m = 200
    w2l = np.column_stack([rng.uniform(0.2, 2.0, m), rng.uniform(-3.0, 3.0, m), rng.uniform(-1, 1, m),
                           rng.uniform(-1, 1, m), rng.uniform(0.1, 10.0, m)])
    w2r = np.column_stack([rng.uniform(0.2, 2.0, m), rng.uniform(-3.0, 3.0, m), rng.uniform(-1, 1, m),
                           rng.uniform(-1, 1, m), rng.uniform(0.1, 10.0, m)])
    s2l = 0.2 * rng.normal(size=(m, 3, 5))
    s2r = 0.2 * rng.normal(size=(m, 3, 5))
    dt2 = rng.uniform(1e-3, 0.1, m)
    tau2 = dt2 * rng.uniform(0.02, 3.0, m)
    ib2 = build_interface(w2l, w2r, s2l, s2r)
    out.update(w2l=w2l, w2r=w2r, s2l=s2l, s2r=s2r, tau2=tau2, dt2=dt2,
               flux2=evolve_flux(ib2, tau2, dt2), point2=point_value(ib2, tau2, np.zeros(m)))
    # 3) KFVS split flux
    rng = np.random.default_rng(202402)
    w3l, w3r, _, _ = random_interface_inputs(rng, 25)
    out.update(w3l=w3l, w3r=w3r, kfvs=kfvs_flux(w3l, w3r))
    np.savez_compressed(HERE / "flux_batch.npz", **out)
    print("flux_batch.npz", {k: v.shape for k, v in out.items()})


GAMMA = 1.4

MESH_CASES = {
    "tet3p": dict(extent=(1, 1, 1), divisions=(3, 3, 3), split="tet", periodic=("x", "y", "z")),
    "tet3j": dict(extent=(1, 1, 1), divisions=(3, 3, 3), split="tet", perturb=0.15, seed=202403),
    "hex4p": dict(extent=(1, 1, 1), divisions=(4, 4, 4), split="hex", periodic=("x", "y", "z")),
    "hex332": dict(extent=(1, 2, 1), divisions=(3, 3, 2), split="hex"),
    "tet2x": dict(extent=(1, 1, 1), divisions=(2, 2, 2), split="tet", periodic=("x",)),
}

MESH_ARRAYS = ("cell_kind", "cell_nodes", "cell_volume", "cell_centroid", "cell_h", "face_nodes",
               "face_owner", "face_neighbor", "face_patch", "face_area", "face_normal", "face_frame",
               "face_shift", "fq_point", "fq_weight", "fq_face", "face_fq_start", "cq_point", "cq_weight",
               "cell_cq_start")


def _flat_stencils(st, nc):
    """Flatten a reference StencilTable into CSR arrays (ids + shifts)."""
    out = {}
    nf = max(len(st[c].neighbor_ids) for c in range(nc))
    nb = np.full((nc, nf), -1, dtype=np.int64)
    nbs = np.zeros((nc, nf, 3))
    big_start, big_ids, big_shift = [0], [], []
    sub_cell_start, sub_member_start, sub_ids, sub_shift = [0], [0], [], []
    wfb, hfb = [], []
    for c in range(nc):
        s = st[c]
        nb[c, : len(s.neighbor_ids)] = s.neighbor_ids
        nbs[c, : len(s.neighbor_ids)] = s.neighbor_shifts
        big_ids.extend(s.big_ids.tolist())
        big_shift.extend(np.asarray(s.big_shifts).reshape(-1, 3).tolist())
        big_start.append(len(big_ids))
        for ids, sh in zip(s.sub_ids, s.sub_shifts):
            sub_ids.extend(ids.tolist())
            sub_shift.extend(np.asarray(sh).reshape(-1, 3).tolist())
            sub_member_start.append(len(sub_ids))
        sub_cell_start.append(len(sub_member_start) - 1)
        wfb.append(s.weno_fallback)
        hfb.append(s.hweno_fallback)
    out.update(nbr_ids=nb, nbr_shift=nbs, big_start=np.array(big_start), big_ids=np.array(big_ids),
               big_shift=np.array(big_shift).reshape(-1, 3), sub_cell_start=np.array(sub_cell_start),
               sub_member_start=np.array(sub_member_start), sub_ids=np.array(sub_ids, dtype=np.int64),
               sub_shift=np.array(sub_shift).reshape(-1, 3), weno_fallback=np.array(wfb, dtype=np.int8),
               hweno_fallback=np.array(hfb, dtype=np.int8))
    return out


def make_mesh():
    from gks3d.hweno import HwenoReconstructor
    from gks3d.mesh import build_stencils, generate_box_mesh
    from gks3d.recon import ReconGeometry, WenoReconstructor

    for name, kw in MESH_CASES.items():
        m = generate_box_mesh(**kw)
        out = {f"mesh_{k}": np.asarray(getattr(m, k)) for k in MESH_ARRAYS}
        out["mesh_cell_face_list"] = np.concatenate(m.cell_faces)
        st = build_stencils(m)
        out.update({f"st_{k}": v for k, v in _flat_stencils(st, m.ncells).items()})
        g = ReconGeometry(m, st)
        w = WenoReconstructor(g)
        h = HwenoReconstructor(g)
        out.update(avg0=g.avg0, beta_mat=g.beta_mat,
                   weno_big_op=w.big_op, weno_big_gather=w.big_gather, weno_big_degree=w.big_degree,
                   weno_sub_op=w.sub_op, weno_sub_gather=w.sub_gather,
                   weno_sub_active=w.sub_active.astype(np.int8),
                   hweno_big_op=h.big_op, hweno_big_avg_gather=h.big_avg_gather,
                   hweno_big_grad_gather=h.big_grad_gather, hweno_big_grad_scale=h.big_grad_scale,
                   hweno_big_ncols=h.big_ncols, hweno_big_degree=h.big_degree, hweno_sub_op=h.sub_op,
                   hweno_sub_gather=h.sub_gather, hweno_sub_active=h.sub_active.astype(np.int8))
        np.savez_compressed(HERE / f"mesh_{name}.npz", **out)
        print(f"mesh_{name}.npz", m.ncells, "cells")


# solver cases: mesh, options, patch table, initial field recipe
def _patch_specs(case, mesh):
    from gks3d.boundary import PatchSpec

    ref = np.array(case.get("reference", (1.0, 0.5, 0.0, 0.0, 1.0 / GAMMA)))
    kinds = case.get("patches", {})
    out = {}
    for n in mesh.patch_names:
        spec = kinds.get(n, kinds.get("*"))
        if spec is None:
            continue
        kind, kw = spec
        kw = dict(kw)
        if kind in ("farfield_riemann", "supersonic_inlet") and "reference" not in kw:
            kw["reference"] = ref
        out[n] = PatchSpec(n, kind, **kw)
    return out


SOLVER_CASES = {
    # smooth density wave on the periodic Kuhn-tet box (config-1 shape)
    "s1_tet_weno": dict(mesh="tet3p", scheme="weno_gmres", field="wave"),
    # perturbed tets, farfield everywhere, noisy near-uniform state
    "s2_tetj_weno_far": dict(mesh="tet3j", scheme="weno_gmres", field="noise",
                             patches={"*": ("farfield_riemann", {})}),
    "s3_tetj_hweno_far": dict(mesh="tet3j", scheme="hweno_gmres", field="noise",
                              patches={"*": ("farfield_riemann", {})}),
    # compact scheme, linear weights, periodic hexes (criterion-4 shape)
    "s4_hex_hweno_lin": dict(mesh="hex4p", scheme="hweno_gmres", weights="linear", field="wave"),
    # viscous cavity walls (isothermal no-slip with lid)
    "s5_tet_cavity": dict(mesh="tet3j", scheme="weno_gmres", model="viscous", mu=0.01, field="rest",
                          reference=(1.0, 0.0, 0.0, 0.0, 1.0 / GAMMA),
                          patches={"*": ("wall_noslip_isothermal", {"lambda_wall": 0.7}),
                                   "ymax": ("wall_noslip_isothermal",
                                            {"lambda_wall": 0.7, "velocity": np.array([0.15, 0.0, 0.0])})}),
    # supersonic channel: inlet/outlet, slip walls, farfield
    "s6_tet_supersonic": dict(mesh="tet3j", scheme="hweno_gmres", field="noise",
                              reference=(1.0, 2.0, 0.1, 0.0, 1.0 / GAMMA),
                              patches={"xmin": ("supersonic_inlet", {}), "xmax": ("supersonic_outlet", {}),
                                       "ymin": ("wall_slip_adiabatic", {}), "ymax": ("wall_slip_adiabatic", {}),
                                       "zmin": ("farfield_riemann", {}), "zmax": ("farfield_riemann", {})}),
    # hexes with adiabatic no-slip walls + farfield
    "s7_hex_walls": dict(mesh="hex332", scheme="weno_gmres", model="viscous", mu=0.005, field="noise",
                         patches={"*": ("farfield_riemann", {}), "ymin": ("wall_noslip_adiabatic", {}),
                                  "ymax": ("wall_noslip_adiabatic", {})}),
}


def initial_q(case, mesh, compact):
    from gks3d.kinetic import primitive_to_conserved

    rng = np.random.default_rng({"wave": 11, "noise": 12, "rest": 13}[case["field"]])
    x = mesh.cell_centroid
    nc = mesh.ncells
    ref = np.array(case.get("reference", (1.0, 0.5, 0.0, 0.0, 1.0 / GAMMA)))
    w = np.tile(np.array([ref[0], ref[1], ref[2], ref[3], ref[0] / (2.0 * ref[4])]), (nc, 1))
    tp = 2 * np.pi
    if case["field"] == "wave":
        w[:, 0] = 1.0 + 0.2 * np.sin(tp * x[:, 0]) * np.cos(tp * x[:, 1])
        w[:, 1] = 0.5 + 0.1 * np.cos(tp * x[:, 2])
        w[:, 2] = 0.1 * np.sin(tp * x[:, 1])
        w[:, 4] = w[:, 4] * (1.0 + 0.1 * np.cos(tp * x[:, 0]))
    elif case["field"] == "noise":
        w[:, 0] *= 1.0 + 0.05 * rng.normal(size=nc)
        w[:, 1:4] += 0.05 * rng.normal(size=(nc, 3))
        w[:, 4] *= 1.0 + 0.05 * rng.normal(size=nc)
    q = primitive_to_conserved(w)
    grad = None
    if compact:
        grad = 0.1 * np.random.default_rng(5).normal(size=(nc, 3, 5))
    return q, grad


def make_solver():
    from gks3d.jacobian import assemble_jacobian
    from gks3d.krylov import gmres_solve
    from gks3d.mesh import generate_box_mesh
    from gks3d.stepping import SolutionField, Solver, SolverOptions

    for name, case in SOLVER_CASES.items():
        mesh = generate_box_mesh(**MESH_CASES[case["mesh"]])
        patches = _patch_specs(case, mesh)
        opts = SolverOptions(scheme=case["scheme"], model=case.get("model", "inviscid"), mu=case.get("mu", 0.0),
                             weights=case.get("weights", "nonlinear"), patches=patches)
        solver = Solver(mesh, opts)
        q, grad = initial_q(case, mesh, solver.compact)
        fld = SolutionField(q, grad)
        dt = solver.local_time_step(fld)
        res, grad_new = solver.residual(fld, dt)
        ghosts = solver._boundary_ghosts(fld)
        a = assemble_jacobian(mesh, q, dt, GAMMA, ghosts)
        x, info = gmres_solve(a, res, m=10, restarts=3, k_max=2)
        rng = np.random.default_rng(99)
        v = rng.normal(size=q.shape)
        fm = solver.frechet_matvec(fld, v, dt)
        out = dict(q=q, dt=dt, res=res, ghosts=np.zeros((0, 5)) if ghosts is None else ghosts,
                   jac_diag=a.diag, jac_off=a.off, jac_off_col=a.off_col, jac_off_row=a.off_row,
                   jac_rowptr=a.rowptr, gmres_x=x, gmres_matvecs=np.array(info.matvecs),
                   gmres_cycle_norms=np.array([n for cyc in info.cycle_residuals for n in cyc]),
                   gmres_cycle_len=np.array([len(c) for c in info.cycle_residuals]), frechet_v=v, frechet=fm)
        if grad is not None:
            out.update(grad=grad, grad_new=grad_new)
        # a short nonlinear history
        hist = []
        qs = []
        f = fld
        for _ in range(4):
            f, si = solver.advance(f)
            hist.append((si.res_rho_l1, si.res_l2, si.dt_min, si.solver_cycles, float(si.retried)))
            qs.append(f.q.copy())
        out.update(hist=np.array(hist), q_after=np.array(qs))
        if f.grad is not None:
            out["grad_after"] = f.grad
        np.savez_compressed(HERE / f"solver_{name}.npz", **out)
        print(f"solver_{name}.npz", mesh.ncells, "cells", "matvecs", info.matvecs)


# -- converged-state parity (north_star "Correctness": converged fields within
# 1e-8, residual-drop history within +-1 nonlinear iteration) -----------------

CONVERGE_CASES = {
    # the reference's own lid-driven cavity (cases/cavity_re100_desk.ini
    # physics) run to the driver's convergence test (driver.py:71-76)
    "cavity4": dict(n=4, threshold=1e-10, max_steps=8000),
    "cavity8": dict(n=8, threshold=1e-10, max_steps=8000),
    # the compact scheme (HWENO + Gauss gradient update) on the same case
    "cavity4_hweno": dict(n=4, threshold=1e-10, max_steps=12000, scheme="hweno_gmres"),
}


def cavity_setup(n, scheme="weno_gmres"):
    from gks3d.boundary import PatchSpec
    from gks3d.mesh import generate_box_mesh
    from gks3d.stepping import SolverOptions, initial_field

    mesh = generate_box_mesh((1, 1, 1), (n, n, n), split="tet")
    lam_wall = GAMMA / 2.0
    patches = {nm: PatchSpec(nm, "wall_noslip_isothermal", lambda_wall=lam_wall) for nm in mesh.patch_names}
    patches["ymax"] = PatchSpec("ymax", "wall_noslip_isothermal", lambda_wall=lam_wall,
                                velocity=np.array([0.15, 0.0, 0.0]))
    opts = SolverOptions(scheme=scheme, model="viscous", mu=0.15 / 100.0, patches=patches, cfl=2.0)
    return mesh, opts, initial_field(mesh, [1.0, 0.0, 0.0, 0.0, 1.0 / GAMMA], compact=scheme.startswith("hweno"))


def make_converge(names=None):
    import time

    from gks3d.stepping import Solver

    for name, case in CONVERGE_CASES.items():
        if names and name not in names:
            continue
        mesh, opts, fld = cavity_setup(case["n"], case.get("scheme", "weno_gmres"))
        solver = Solver(mesh, opts)
        hist = []
        t0 = time.time()
        steps = None
        for k in range(1, case["max_steps"] + 1):
            fld, info = solver.advance(fld)
            hist.append((info.res_rho_l1, info.res_l2, info.dt_min, info.solver_cycles, float(info.retried)))
            if info.res_rho_l1 < case["threshold"] and info.res_l2 < 1e4 * case["threshold"]:
                steps = k
                break
        out = dict(hist=np.array(hist), q_final=fld.q, steps=np.array(steps if steps else -1),
                   threshold=np.array(case["threshold"]), n=np.array(case["n"]))
        if fld.grad is not None:
            out["grad_final"] = fld.grad
        np.savez_compressed(HERE / f"converge_{name}.npz", **out)
        print(f"converge_{name}.npz", mesh.ncells, "cells, converged at", steps, f"({time.time() - t0:.0f} s)",
              flush=True)


# -- the synthetic sphere / wing meshes of configs 2-4, run by the reference --

def _capture_build(fn, *a, **k):
    """Run a paper_2304_09485_b200.meshgen generator and return the arguments it
    passed to Mesh.build (nodes, tets, hexes, patch faces)."""
    sys.path.insert(0, str(HERE.parents[1]))
    import paper_2304_09485_b200.mesh as M
    import paper_2304_09485_b200.meshgen as MG

    cap = {}
    orig = M.Mesh.build

    def grab(nodes, tets=(), hexes=(), patch_faces=None, periodic_pairs=()):
        cap.update(nodes=np.asarray(nodes), tets=np.asarray(tets, dtype=np.int64),
                   hexes=np.asarray(hexes, dtype=np.int64).reshape(-1, 8), patch_faces=patch_faces,
                   periodic_pairs=periodic_pairs)
        return orig(nodes, tets, hexes, patch_faces, periodic_pairs)

    M.Mesh.build = grab
    try:
        getattr(MG, fn)(*a, **k)
    finally:
        M.Mesh.build = orig
    return cap


GEN_CASES = {
    # C2 physics on the sphere n=2: inviscid Ma 0.5, slip wall + farfield, WENO
    "sphere2_c2": dict(gen=("generate_sphere_mesh", (2,), dict(radius=0.5, far=10.0)), scheme="weno_gmres",
                       reference=(1.0, 0.5, 0.0, 0.0, 1.0 / GAMMA),
                       patches={"sphere": ("wall_slip_adiabatic", {}), "farfield": ("farfield_riemann", {})}),
    # C3 physics: viscous Re 118 Ma 0.2535, no-slip wall, HWENO linear weights
    "sphere2_c3": dict(gen=("generate_sphere_mesh", (2,), dict(radius=0.5, far=10.0)), scheme="hweno_gmres",
                       model="viscous", mu=0.0021483050847457627, weights="linear",
                       reference=(1.0, 0.2535, 0.0, 0.0, 1.0 / GAMMA),
                       patches={"sphere": ("wall_noslip_adiabatic", {}), "farfield": ("farfield_riemann", {})}),
    # C4 physics on the swept wing n=8: Ma 0.8395 AoA 3.06, slip walls, HWENO
    "wing8_c4": dict(gen=("generate_swept_wing_mesh", (8,), {}), scheme="hweno_gmres",
                     reference=(1.0, 0.8383030214661579, 0.04482495105787847, 0.0, 1.0 / GAMMA),
                     patches={"wing": ("wall_slip_adiabatic", {}), "farfield": ("farfield_riemann", {}),
                              "root": ("wall_slip_adiabatic", {}), "tip": ("wall_slip_adiabatic", {})}),
}


def make_generated(names=None):
    from gks3d.mesh import Mesh
    from gks3d.stepping import SolutionField, Solver, SolverOptions, initial_field

    for name, case in GEN_CASES.items():
        if names and name not in names:
            continue
        fn, a, k = case["gen"]
        cap = _capture_build(fn, *a, **k)
        mesh = Mesh.build(cap["nodes"], [tuple(t) for t in cap["tets"]], [tuple(h) for h in cap["hexes"]],
                          cap["patch_faces"], cap["periodic_pairs"])
        patches = _patch_specs(case, mesh)
        opts = SolverOptions(scheme=case["scheme"], model=case.get("model", "inviscid"), mu=case.get("mu", 0.0),
                             weights=case.get("weights", "nonlinear"), patches=patches)
        solver = Solver(mesh, opts)
        ref = np.array(case["reference"])
        fld = initial_field(mesh, ref, GAMMA, compact=solver.compact)
        # a perturbed start (the uniform field is a fixed point of the interior)
        rng = np.random.default_rng(31)
        from gks3d.kinetic import conserved_to_primitive, primitive_to_conserved

        w = conserved_to_primitive(fld.q, GAMMA)
        w[:, 0] *= 1.0 + 0.02 * rng.normal(size=mesh.ncells)
        w[:, 1:4] += 0.02 * rng.normal(size=(mesh.ncells, 3))
        q = primitive_to_conserved(w, GAMMA)
        grad = 0.02 * rng.normal(size=(mesh.ncells, 3, 5)) if solver.compact else None
        fld = SolutionField(q, grad)
        dt = solver.local_time_step(fld)
        res, grad_new = solver.residual(fld, dt)
        v = np.random.default_rng(99).normal(size=q.shape)
        fm = solver.frechet_matvec(fld, v, dt)
        out = dict(q=q, dt=dt, res=res, frechet_v=v, frechet=fm, nodes=cap["nodes"], tets=cap["tets"])
        if grad is not None:
            out.update(grad=grad, grad_new=grad_new)
        hist, qs = [], []
        f = fld
        for _ in range(4):
            f, si = solver.advance(f)
            hist.append((si.res_rho_l1, si.res_l2, si.dt_min, si.solver_cycles, float(si.retried)))
            qs.append(f.q.copy())
        out.update(hist=np.array(hist), q_after=np.array(qs))
        if f.grad is not None:
            out["grad_after"] = f.grad
        np.savez_compressed(HERE / f"gen_{name}.npz", **out)
        print(f"gen_{name}.npz", mesh.ncells, "cells", flush=True)


# -- a step the reference retries at halved dt (stepping.py:286-296) ------------

RETRY_CASE = dict(mesh="tet3j", scheme="weno_gmres", field="noise", cfl=None,
                  reference=(1.0, 2.0, 0.1, 0.0, 1.0 / GAMMA),
                  patches={"xmin": ("supersonic_inlet", {}), "xmax": ("supersonic_outlet", {}),
                           "ymin": ("wall_slip_adiabatic", {}), "ymax": ("wall_slip_adiabatic", {}),
                           "zmin": ("farfield_riemann", {}), "zmax": ("farfield_riemann", {})})


RETRY_RUNS = {
    # (scheme, CFL, steps): found by scanning np.geomspace(4, 60, 30) -- the
    # reference rejects the marked steps once and accepts them at halved dt
    "weno": ("weno_gmres", float(np.geomspace(4, 60, 30)[24]), 2, "supersonic"),
    "hweno": ("hweno_gmres", float(np.geomspace(4, 60, 30)[24]), 5, "farfield"),
}


def make_retry():
    """Supersonic channel starts that the reference rejects once and redoes
    at halved dt (stepping.py:286-296)."""
    from gks3d.mesh import generate_box_mesh
    from gks3d.stepping import SolutionField, Solver, SolverOptions

    for name, (scheme, cfl, steps, base) in RETRY_RUNS.items():
        case = dict(RETRY_CASE if base == "supersonic" else SOLVER_CASES["s2_tetj_weno_far"])
        mesh = generate_box_mesh(**MESH_CASES[case["mesh"]])
        patches = _patch_specs(case, mesh)
        compact = scheme.startswith("hweno")
        q0, g0 = initial_q(case, mesh, compact)
        solver = Solver(mesh, SolverOptions(scheme=scheme, patches=patches, cfl=cfl))
        fld = SolutionField(q0.copy(), None if g0 is None else g0.copy())
        hist, qs = [], []
        for _ in range(steps):
            fld, si = solver.advance(fld)
            hist.append((si.res_rho_l1, si.res_l2, si.dt_min, si.solver_cycles, float(si.retried)))
            qs.append(fld.q.copy())
        assert any(h[4] for h in hist), name
        out = dict(q=q0, cfl=np.array(cfl), hist=np.array(hist), q_after=np.array(qs))
        if g0 is not None:
            out.update(grad=g0, grad_after=fld.grad)
        np.savez_compressed(HERE / f"retry_{name}.npz", **out)
        print(f"retry_{name}.npz cfl {cfl:.4f} retried", [h[4] for h in hist], flush=True)


SECTIONS = {"flux": make_flux, "mesh": make_mesh, "solver": make_solver, "converge": make_converge,
            "generated": make_generated, "retry": make_retry}


def main(argv):
    _import_reference()
    names = argv or ["flux", "mesh", "solver", "generated", "retry"]  # "converge" runs ~1 h: ask for it
    for name in names:
        sec, _, sub = name.partition(":")
        if sub:
            SECTIONS[sec](sub.split(","))
        else:
            SECTIONS[sec]()


if __name__ == "__main__":
    main(sys.argv[1:])
