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
