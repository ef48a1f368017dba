"""The C ABI library loads and exports exactly what include/gks.h declares (CPU)."""

import re
from pathlib import Path

from paper_2304_09485_b200 import _native as N

HEADER = Path(__file__).resolve().parents[1] / "include" / "gks.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gks_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_bindings():
    names = declared()
    bound = sorted(n for n, _, _ in N.SIGNATURES)
    assert names == bound


def test_library_exports_every_symbol():
    lib = N.load()
    for name in declared():
        assert hasattr(lib, name), name


def test_abi_version_and_no_device_error():
    lib = N.load()
    assert lib.gks_abi_version() == 1
    import numpy as np

    w = np.array([[1.0, 0.1, 0.0, 0.0, 1.0]])
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        rc = lib.gks_flux_batch(1, N.dptr(w), N.dptr(w), None, None, N.dptr(np.ones(1)), N.dptr(np.ones(1)),
                                None, 1.4, N.dptr(np.empty((1, 5))), None)
        assert rc == N.GKS_ERR_NO_DEVICE
        assert "no CUDA device" in lib.gks_last_error().decode()
