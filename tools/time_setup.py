"""Phase timing of the solver construction on the C2 workload (GPU box):
mesh build, native setup, mesh descriptor, gks_create.

    python tools/time_setup.py [n] [scheme]
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_09485_b200 import _native as N  # noqa: E402
from paper_2304_09485_b200.stepping import SolverOptions, _options_struct  # noqa: E402

n = sys.argv[1] if len(sys.argv) > 1 else "16"
scheme = sys.argv[2] if len(sys.argv) > 2 else "weno_gmres"
workload = sys.argv[3] if len(sys.argv) > 3 else "c2"
skip_host = "--device-only" in sys.argv
sys.argv = ["bench.py", "--n", n, "--scheme", scheme, "--workload", workload]
args = bench.parse()
out = {}
lib = N.load()
t0 = time.perf_counter()
mesh, patches, q0, g0, workload, extra = bench.build_workload(args, scheme.startswith("hweno"))
out["mesh"] = time.perf_counter() - t0
if not skip_host:
    t0 = time.perf_counter()
    st = N.NativeSetup(mesh, schemes=2 if scheme.startswith("hweno") else 1)
    out["native_setup"] = time.perf_counter() - t0
opts = SolverOptions(scheme=scheme, patches=patches, jacobian=args.jacobian, **extra)
o, arr = _options_struct(opts, mesh)
t0 = time.perf_counter()
desc, keep = N.mesh_desc(mesh)
out["mesh_desc"] = time.perf_counter() - t0
if not skip_host:
    h = C.c_void_p()
    t0 = time.perf_counter()
    N.check(lib.gks_create(C.byref(desc), st.handle, C.byref(o), 0, C.byref(h)))
    out["gks_create"] = time.perf_counter() - t0
    lib.gks_destroy(h)
    del st
h2 = C.c_void_p()
t0 = time.perf_counter()
N.check(lib.gks_create(C.byref(desc), None, C.byref(o), 0, C.byref(h2)))
out["gks_create_device_setup"] = time.perf_counter() - t0
out["cells"] = mesh.ncells
import resource  # noqa: E402

out["peak_rss_gb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
print(json.dumps(out), flush=True)
