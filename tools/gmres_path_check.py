"""Fused (cluster) Arnoldi-column kernel vs the multi-block MGS chain on the
same medium-size problem: histories and fields must agree to rounding."""
import os
import subprocess
import sys
import json

CODE = r'''
import sys, json, numpy as np
sys.path.insert(0, ".")
from bench import cavity_problem
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions
n = int(sys.argv[1])
mesh, patches, q, g, extra = cavity_problem(n, False)
s = Solver(mesh, SolverOptions(scheme="weno_gmres", patches=patches, jacobian="roe", **extra))
s.upload(SolutionField(q, g))
import time
hist = []
t0 = time.perf_counter()
for _ in range(int(sys.argv[2])):
    hist.append(s.advance_resident().res_rho_l1)
el = time.perf_counter() - t0
np.save(sys.argv[3], s.download().q)
print(json.dumps({"hist": hist, "ms_per_step": 1000 * el / len(hist), "cells": mesh.ncells}))
'''

n, steps = sys.argv[1], sys.argv[2]
out = {}
for mode in ("fused", "chain"):
    env = dict(os.environ)
    if mode == "chain":
        env["GKS_GMRES_SMALL"] = "0"
    r = subprocess.run([sys.executable, "-c", CODE, n, steps, f"/tmp/q_{mode}.npy"], capture_output=True, text=True,
                       env=env)
    out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
import numpy as np
qa, qb = np.load("/tmp/q_fused.npy"), np.load("/tmp/q_chain.npy")
ha, hb = np.array(out["fused"]["hist"]), np.array(out["chain"]["hist"])
print(json.dumps({"cells": out["fused"]["cells"], "ms_fused": out["fused"]["ms_per_step"],
                  "ms_chain": out["chain"]["ms_per_step"],
                  "max_rel_hist": float(np.max(np.abs(ha - hb) / np.maximum(np.abs(hb), 1e-300))),
                  "max_rel_q": float(np.max(np.abs(qa - qb)) / np.max(np.abs(qb)))}))
