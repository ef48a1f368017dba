"""Per-kernel-class device time of a few uncaptured implicit steps (in-library
CUDA-event profiler) for the cavity or C2 workloads."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import cavity_problem  # noqa: E402
from paper_2304_09485_b200 import _native as N  # noqa: E402
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
mesh, patches, q, g, extra = cavity_problem(n, False)
s = Solver(mesh, SolverOptions(scheme="weno_gmres", patches=patches, jacobian="roe", **extra))
s.upload(SolutionField(q, g))
for _ in range(3):
    s.advance_resident()
t0 = time.perf_counter()
for _ in range(steps):
    s.advance_resident()
graph_ms = 1000 * (time.perf_counter() - t0) / steps
prof = N.Profiler()
prof.start()
t0 = time.perf_counter()
for _ in range(steps):
    s.advance_resident()
el = 1000 * (time.perf_counter() - t0) / steps
k = prof.stop()
tot = sum(t for t, _ in k.values())
print(json.dumps({"cells": mesh.ncells, "graph_ms_per_step": graph_ms, "uncaptured_ms_per_step": el,
                  "device_ms_per_step": tot / steps,
                  "kernels": {name: {"ms_per_step": round(t / steps, 4), "launches_per_step": c // steps}
                              for name, (t, c) in sorted(k.items(), key=lambda kv: -kv[1][0]) if c}}, indent=1))
