"""Oracle pinning (CPU): the numpy restatement against reference goldens."""

import numpy as np

from oracle import flux as O


def rel(a, b):
    # per-point max-norm relative error, floored at 1e-6 of the batch maximum
    # so deep-tail points (|flux| ~ 1e-33) are judged on an absolute scale
    mag = np.max(np.abs(b), axis=1)
    scale = np.maximum(mag, 1e-6 * mag.max())
    return float(np.max(np.max(np.abs(a - b), axis=1) / scale))


def test_flux_and_point_value_match_reference(golden):
    g = golden("flux_batch")
    ib = O.Interface(g["wl"], g["wr"], g["sl"], g["sr"])
    assert rel(O.evolve_flux(ib, g["tau"], g["dt"]), g["flux"]) < 1e-13
    assert rel(O.point_value(ib, g["tau"], g["tp"]), g["point"]) < 1e-13
    assert np.allclose(ib.w0, g["w0"], rtol=1e-13, atol=1e-14)
    assert np.allclose(ib.abar, g["abar"], rtol=1e-12, atol=1e-13)
    assert np.allclose(ib.Abar, g["atbar"], rtol=1e-12, atol=1e-13)


def test_wide_state_sweep(golden):
    g = golden("flux_batch")
    ib = O.Interface(g["w2l"], g["w2r"], g["s2l"], g["s2r"])
    # hypersonic tails (sqrt(lam)|U| up to 9): recurrence rounding reaches 3e-13
    assert rel(O.evolve_flux(ib, g["tau2"], g["dt2"]), g["flux2"]) < 1e-12
    assert rel(O.point_value(ib, g["tau2"], 0.0), g["point2"]) < 1e-12


def test_kfvs(golden):
    g = golden("flux_batch")
    assert rel(O.kfvs_flux(g["w3l"], g["w3r"]), g["kfvs"]) < 1e-14


def test_uniform_state_is_euler_flux():
    w = np.array([[1.2, 0.5, 0.3, -0.2, 1.1]])
    ib = O.Interface(w, w)
    f = O.evolve_flux(ib, 0.001, 0.02)
    assert np.allclose(f, O.euler_flux_local(w), rtol=1e-12, atol=1e-13)
