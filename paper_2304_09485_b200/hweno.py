"""Compact-scheme gradient update (mirrors gks3d/hweno.py:172-194).

update_gradients(mesh, point_values): cell-averaged gradients from the
interface point values by the Gauss theorem, |Omega| grad Q = sum over the
cell's face points of w S n Q_G (owner +, neighbour -).  Runs on the device
(gks_update_gradients: the assembly kernel of the residual pipeline with
zero flux contributions) on a cached handle of the mesh.  The HWENO
reconstruction operators themselves are built by the native setup
(csrc/gks_setup.cpp) and applied by k_recon_hweno.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .kinetic import DEFAULT_GAMMA


def update_gradients(mesh, point_values, gamma: float = DEFAULT_GAMMA):
    from .stepping import _jacobian_handle

    s = _jacobian_handle(mesh, gamma)  # reference numbering (no reorder)
    vals = np.asarray(point_values, dtype=float)
    nfq, m = vals.shape
    out = np.empty((mesh.ncells, 3, m))
    # the device assembles 5 components at a time (zero-padded)
    for c0 in range(0, m, 5):
        k = min(5, m - c0)
        qpt = np.zeros((nfq, 5))
        qpt[:, :k] = vals[:, c0:c0 + k]
        g = np.empty((mesh.ncells, 3, 5))
        N.check(N.load().gks_update_gradients(s._handle, N.dptr(qpt), N.dptr(g)))
        out[:, :, c0:c0 + k] = g[:, :, :k]
    return out
