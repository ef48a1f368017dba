"""The face kernel's closed forms (csrc/gks_kinetic.cuh: euler_axis_jvp,
equilibrium_flux and the point-value identity) restated in numpy and checked
against the oracle's Maxwellian moment engine (oracle/kinetic.py, which
restates kinetic.py:90-312) on random states.  This pins the algebra; the
device code itself is pinned by the flux goldens and converged-state tests
(tests/test_flux_gpu.py, tests/test_reference_goldens_gpu.py).
"""

import numpy as np

from oracle import kinetic as K

GAMMA = 1.4
KT = K.n_internal(GAMMA) + 3.0  # N + 3
GM1 = 2.0 / KT                  # gamma - 1


def states(n=64, seed=5):
    rng = np.random.default_rng(seed)
    w = np.column_stack([rng.uniform(0.3, 2.0, n), rng.normal(0, 0.8, (n, 3)), rng.uniform(0.3, 3.0, n)])
    q = K.prim_to_cons(w, GAMMA)
    dq = rng.normal(size=(3, n, 5)) * np.abs(q)[None] * 0.3
    return w, q, dq


def euler_axis_jvp(w, dq):
    """sum_k (dF_k/dq) dq_k -- gks_kinetic.cuh euler_axis_jvp."""
    U = w[:, 1:4]
    h = 0.5 / w[:, 4]
    ke = 0.5 * np.sum(U * U, axis=1)
    H = ke + 0.5 * (KT + 2.0) * h
    out = np.zeros_like(w)
    for k in range(3):
        d = dq[k]
        a = d[:, 1 + k] - U[:, k] * d[:, 0]
        b = GM1 * (ke * d[:, 0] - np.sum(U * d[:, 1:4], axis=1) + d[:, 4])
        out[:, 0] += d[:, 1 + k]
        for i in range(3):
            out[:, 1 + i] += U[:, i] * a + U[:, k] * d[:, 1 + i] + (b if i == k else 0.0)
        out[:, 4] += H * a + U[:, k] * (b + d[:, 4])
    return out


def equilibrium_flux(w, D, dq, c1, c3, c2):
    """rho <u psi (c1 + c3 Ab.psi + c2 sum_k c_k ab_k.psi)> -- gks_kinetic.cuh equilibrium_flux."""
    rho = w[:, 0]
    U = w[:, 1:4]
    h = 0.5 / w[:, 4]
    U2 = np.sum(U * U, axis=1)
    ke = 0.5 * U2
    H = ke + 0.5 * (KT + 2.0) * h
    mn = rho * U[:, 0]
    a = D[:, 1] - U[:, 0] * D[:, 0]
    bD = GM1 * (ke * D[:, 0] - np.sum(U * D[:, 1:4], axis=1) + D[:, 4])
    out = np.empty_like(w)
    out[:, 0] = c1 * mn + c3 * D[:, 1]
    for i in range(3):
        out[:, 1 + i] = c1 * (mn * U[:, i] + (rho * h if i == 0 else 0.0)) + \
            c3 * (U[:, i] * a + U[:, 0] * D[:, 1 + i] + (bD if i == 0 else 0.0))
    out[:, 4] = c1 * mn * H + c3 * (H * a + U[:, 0] * (bD + D[:, 4]))
    t = np.zeros_like(w)
    for k in range(3):
        d = dq[k]
        d0 = d[:, 0]
        e = d[:, 1:4] - U * d0[:, None]
        Ue = np.sum(U * e, axis=1)
        b = GM1 * (d[:, 4] - Ue - ke * d0)
        UU = U[:, 0] * U[:, k]
        p1 = d0 * UU + e[:, 0] * U[:, k] + U[:, 0] * e[:, k]
        t[:, 0] += p1 + (b if k == 0 else 0.0)
        for i in range(3):
            v = U[:, i] * p1 + UU * e[:, i]
            if k == i:
                v = v + b * U[:, 0] + h * e[:, 0]
            if i == 0:
                v = v + b * U[:, k] + h * e[:, k]
            if k == 0:
                v = v + b * U[:, i] + h * e[:, i]
            t[:, 1 + i] += v
        v4 = U2 * p1 + 2.0 * UU * Ue + (KT + 4.0) * (b * UU + h * (e[:, 0] * U[:, k] + U[:, 0] * e[:, k]))
        if k == 0:
            v4 = v4 + b * U2 + 2.0 * h * Ue + (KT + 2.0) * h * (2.0 * b - h * d0)
        t[:, 4] += 0.5 * v4
    return out + c2 * t


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def test_time_slope_rhs_is_the_euler_flux_jacobian():
    w, q, dq = states()
    mom = K.Moments(w, GAMMA)
    ab = [K.micro_slope(w, dq[k], GAMMA) for k in range(3)]
    ref = w[:, 0, None] * mom.directional(ab[0], ab[1], ab[2], 0, 0, 0)
    assert rel(euler_axis_jvp(w, dq), ref) <= 1e-12
    # and the time slope itself (kinetic.py:305-312)
    A = K.time_slope(w, ab[0], ab[1], ab[2], mom, GAMMA)
    assert rel(K.micro_slope(w, -euler_axis_jvp(w, dq), GAMMA), A) <= 1e-11


def test_equilibrium_flux_closed_form():
    w, q, dq = states(seed=9)
    mom = K.Moments(w, GAMMA)
    ab = [K.micro_slope(w, dq[k], GAMMA) for k in range(3)]
    D = -euler_axis_jvp(w, dq)
    Ab = K.micro_slope(w, D, GAMMA)
    c1, c3, c2 = 0.7, -0.3, 0.45
    rho = w[:, 0, None]
    ref = rho * (c1 * mom.psi(1, 0, 0) + c3 * mom.slope(Ab, 1, 0, 0) + c2 * mom.directional(ab[0], ab[1], ab[2], 1, 0, 0))
    assert rel(equilibrium_flux(w, D, dq, c1, c3, c2), ref) <= 1e-12
    # each family on its own (the Euler flux; its Jacobian on D; the Gaussian derivative)
    for cs in ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)):
        ref = rho * (cs[0] * mom.psi(1, 0, 0) + cs[1] * mom.slope(Ab, 1, 0, 0) +
                     cs[2] * mom.directional(ab[0], ab[1], ab[2], 1, 0, 0))
        assert rel(equilibrium_flux(w, D, dq, *cs), ref) <= 1e-12, cs


def test_point_value_identity():
    """rho <psi (g1 + g3 Ab.psi + g2 sum_k c_k ab_k.psi)> = g1 q + (g3 - g2) D."""
    w, q, dq = states(seed=13)
    mom = K.Moments(w, GAMMA)
    ab = [K.micro_slope(w, dq[k], GAMMA) for k in range(3)]
    D = -euler_axis_jvp(w, dq)
    Ab = K.micro_slope(w, D, GAMMA)
    g1, g3, g2 = 0.2, 0.9, -0.6
    rho = w[:, 0, None]
    ref = rho * (g1 * mom.psi(0, 0, 0) + g3 * mom.slope(Ab, 0, 0, 0) + g2 * mom.directional(ab[0], ab[1], ab[2], 0, 0, 0))
    assert rel(g1 * q + (g3 - g2) * D, ref) <= 1e-12
