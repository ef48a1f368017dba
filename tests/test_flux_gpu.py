"""Device flux kernel parity (gks_flux_batch) vs the oracle and reference goldens."""

import numpy as np
import pytest

from oracle import flux as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    # per-point max-norm relative error, floored at 1e-6 of the batch maximum
    # so deep-tail points (|flux| ~ 1e-33) are judged on an absolute scale
    mag = np.max(np.abs(b), axis=1)
    scale = np.maximum(mag, 1e-6 * mag.max())
    return float(np.max(np.max(np.abs(a - b), axis=1) / scale))


@pytest.fixture(scope="module")
def F():
    from paper_2304_09485_b200 import flux

    return flux


def test_golden_batch(F, golden):
    g = golden("flux_batch")
    ib = F.build_interface(g["wl"], g["wr"], g["sl"], g["sr"])
    assert rel(F.evolve_flux(ib, g["tau"], g["dt"]), g["flux"]) < 1e-12
    assert rel(F.point_value(ib, g["tau"], g["tp"]), g["point"]) < 1e-12


def test_golden_wide_states(F, golden):
    g = golden("flux_batch")
    ib = F.build_interface(g["w2l"], g["w2r"], g["s2l"], g["s2r"])
    assert rel(F.evolve_flux(ib, g["tau2"], g["dt2"]), g["flux2"]) < 1e-12
    assert rel(F.point_value(ib, g["tau2"], 0.0), g["point2"]) < 1e-12


def test_kfvs_limit(F, golden):
    g = golden("flux_batch")
    assert rel(F.kfvs_flux(g["w3l"], g["w3r"]), g["kfvs"]) < 1e-13


def test_large_random_batch_vs_oracle(F):
    rng = np.random.default_rng(2024)
    n = 200_000
    wl, wr, sl, sr = O.random_interfaces(rng, n)
    tau = rng.uniform(1e-4, 0.05, n)
    dt = rng.uniform(0.01, 0.1, n)
    got = F.evolve_flux(F.build_interface(wl, wr, sl, sr), tau, dt)
    ref = O.evolve_flux(O.Interface(wl, wr, sl, sr), tau, dt)
    assert rel(got, ref) < 1e-12


def test_uniform_state_is_euler(F):
    w = np.array([[1.2, 0.5, 0.3, -0.2, 1.1]])
    f = F.evolve_flux(F.build_interface(w, w), 0.001, 0.02)
    assert np.allclose(f, O.euler_flux_local(w), rtol=1e-12, atol=1e-13)


def test_unphysical_raises(F):
    from paper_2304_09485_b200.kinetic import UnphysicalStateError

    w = np.array([[1.0, 0.0, 0.0, 0.0, 1.0]])
    with pytest.raises(UnphysicalStateError):
        F.build_interface(w, -w)


def test_interface_batch_intermediates_and_tables(golden):
    """InterfaceBatch carries the reference's intermediates (flux.py:34-66)
    and MomentTables (kinetic.py:90-162), computed on the device."""
    from paper_2304_09485_b200.flux import build_interface, compatibility_residual

    g = golden("flux_batch")
    ib = build_interface(g["wl"], g["wr"], g["sl"], g["sr"])
    for k in ("al", "ar", "atl", "atr", "w0", "abar", "atbar"):
        ref = g[k]
        err = np.max(np.abs(getattr(ib, k) - ref)) / max(np.max(np.abs(ref)), 1e-300)
        assert err <= 1e-12, (k, err)
    for side, tab in (("l", ib.tab_l), ("r", ib.tab_r), ("0", ib.tab_0)):
        for name in ("u_full", "u_pos", "u_neg", "v_full", "w_full", "xi"):
            ref = g[f"tab_{side}_{name}"]
            got = getattr(tab, name)
            assert got.shape == ref.shape
            assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-12, (side, name)
    assert compatibility_residual(ib) < 1e-12
    # identical states give back the state (tests/test_flux.py:45-49)
    w = np.array([[1.0, 0.4, -0.1, 0.2, 1.3]])
    assert np.allclose(build_interface(w, w).w0, w, rtol=1e-12, atol=1e-13)


def test_micro_and_time_slopes_match_reference(golden):
    """kinetic.solve_micro_slope / solve_time_slope (kinetic.py:271-312) on the device."""
    from paper_2304_09485_b200.kinetic import solve_micro_slope, solve_time_slope

    g = golden("flux_batch")
    al = np.stack([solve_micro_slope(g["wl"], g["sl"][:, k]) for k in range(3)], axis=1)
    assert np.max(np.abs(al - g["al"])) <= 1e-12 * np.max(np.abs(g["al"]))
    atl = solve_time_slope(g["wl"], al[:, 0], al[:, 1], al[:, 2])
    assert np.max(np.abs(atl - g["atl"])) <= 1e-12 * np.max(np.abs(g["atl"]))


@pytest.mark.parametrize("kind", ["wall_noslip_isothermal", "wall_noslip_adiabatic", "wall_slip_adiabatic",
                                  "farfield_riemann", "supersonic_inlet", "supersonic_outlet"])
def test_ghost_state_and_gradients_match_oracle(kind):
    """boundary.ghost_state / ghost_gradients (boundary.py:66-171) on the device vs the oracle."""
    from oracle.solver import ghost, ghost_grad
    from paper_2304_09485_b200.boundary import PatchSpec, ghost_gradients, ghost_state
    from paper_2304_09485_b200.kinetic import primitive_to_conserved

    rng = np.random.default_rng(7)
    n = 64
    w = np.column_stack([rng.uniform(0.5, 1.5, n), rng.uniform(-0.8, 0.8, (n, 3)), rng.uniform(0.5, 2.0, n)])
    q = primitive_to_conserved(w)
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    spec = PatchSpec("p", kind, reference=np.array([1.0, 0.6, 0.1, 0.0, 0.7]),
                     lambda_wall=0.9 if kind == "wall_noslip_isothermal" else None,
                     velocity=np.array([0.1, 0.0, 0.05]) if kind.startswith("wall_noslip") else np.zeros(3))
    got = ghost_state(q, spec, nrm)
    ref = ghost(q, spec, nrm)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    g = rng.normal(size=(n, 3, 5))
    gg = ghost_gradients(g, spec, nrm)
    gref = ghost_grad(g, spec, nrm)
    assert np.max(np.abs(gg - gref)) <= 1e-13 * np.max(np.abs(gref))


def test_instantaneous_flux_integrates_to_time_average():
    """instantaneous_flux (flux.py:191-197) is the integrand of evolve_flux:
    Gauss-Legendre over [0, dt] of the device's instantaneous flux equals
    the device's analytic time average; at t = 0 with tau = inf it is the
    KFVS split flux."""
    from paper_2304_09485_b200 import flux as F

    rng = np.random.default_rng(31)
    n = 64
    wl, wr, sl, sr = F.random_interface_inputs(rng, n)
    ib = F.build_interface(wl, wr, sl, sr)
    tau = rng.uniform(0.05, 0.5, n)
    dt = rng.uniform(0.2, 1.0, n)
    x, w = np.polynomial.legendre.leggauss(24)
    avg = np.zeros((n, 5))
    for xi, wi in zip(x, w):
        avg += 0.5 * wi * F.instantaneous_flux(ib, tau, 0.5 * dt * (xi + 1.0))
    ref = F.evolve_flux(ib, tau, dt)
    assert np.max(np.abs(avg - ref)) <= 1e-11 * np.max(np.abs(ref))
    kf = F.instantaneous_flux(F.build_interface(wl, wr), np.inf, 0.0)
    assert np.max(np.abs(kf - F.kfvs_flux(wl, wr))) <= 1e-13 * np.max(np.abs(kf))
