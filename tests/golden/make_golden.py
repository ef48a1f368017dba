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
               w0=ib.w0, abar=ib.abar, atbar=ib.atbar, al=ib.al, atl=ib.atl)
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


SECTIONS = {"flux": make_flux}


def main(argv):
    _import_reference()
    names = argv or list(SECTIONS)
    for name in names:
        SECTIONS[name]()


if __name__ == "__main__":
    main(sys.argv[1:])
