import sys, numpy as np
sys.path.insert(0, "/root/repo")
from bench import c2_mesh, c2_problem
from paper_2304_09485_b200 import meshgen as MG
from paper_2304_09485_b200.stepping import SolutionField, Solver, SolverOptions
for n, jac in ((16, "frechet"), (32, "frechet"), (32, "roe")):
    mesh = c2_mesh(n, MG)
    patches, q, g = c2_problem(mesh, False)
    s = Solver(mesh, SolverOptions(patches=patches, jacobian=jac))
    s.upload(SolutionField(q))
    out = []
    try:
        for k in range(12):
            i = s.advance_resident()
            out.append((k, f"{i.res_rho_l1:.3e}", i.solver_cycles, i.retried))
    except Exception as e:
        out.append(("ERR", str(e)[:120]))
    f = s.download()
    print(n, jac, mesh.ncells, out, "rho range", f.q[:,0].min(), f.q[:,0].max())
