"""Locality probe: the C2 sphere in generator order vs a randomly shuffled
cell order (what a mesh file from an arbitrary generator looks like), same
geometry and physics; per-kernel device times over a few Frechet steps."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import c2_mesh, c2_problem  # noqa: E402
from paper_2304_09485_b200 import _native as N  # noqa: E402
from paper_2304_09485_b200 import meshgen as MG  # noqa: E402
from paper_2304_09485_b200.mesh import Mesh  # noqa: E402
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions  # noqa: E402


def run(mesh, label, steps=2, **extra):
    patches, q, g = c2_problem(mesh, False)
    s = Solver(mesh, SolverOptions(scheme="weno_gmres", patches=patches, jacobian="frechet", **extra))
    s.upload(SolutionField(q, g))
    s.advance_resident()
    prof = N.Profiler()
    prof.start()
    t0 = time.perf_counter()
    for _ in range(steps):
        s.advance_resident()
    el = time.perf_counter() - t0
    k = prof.stop()
    out = {"label": label, "cells": mesh.ncells, "ms_per_step": 1000 * el / steps}
    for name in ("face_flux", "recon", "assemble", "reduce_dot", "jacobi_sweep"):
        t, n = k.get(name, (0, 0))
        out[name] = round(t / max(n, 1), 4)
    print(json.dumps(out), flush=True)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
m = c2_mesh(n, MG)
run(m, "generator order")
tets, hexes, patches = m._source
perm = np.random.default_rng(0).permutation(len(tets))
ms = Mesh.build(m.nodes, tets[perm], hexes, patches)
run(ms, "shuffled cells")
extra = sys.argv[2:]
if "reorder" in extra:
    run(ms, "shuffled cells, reordered", reorder="rcm")
