"""Kernel-only throughput of the fused BGK interface flux (device-resident inputs)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_09485_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lib = N.load()
ms = C.c_double()
N.check(lib.gks_flux_bench(n, reps, 1.4, C.byref(ms)))
pts = n / (ms.value * 1e-3)
print(json.dumps({"n": n, "ms": ms.value, "points_per_s": pts,
                  "ref_model_tflops": pts * 4648 / 1e12}))
