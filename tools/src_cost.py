"""Element-kernel cost of the cfg5 source term: real f = 2 pi^2 sin(pi x) sin(pi y)
vs a constant f (ablation, not a bench number):  python tools/src_cost.py [n]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace  # noqa: E402

import paper_2007_04881_b200.model as M  # noqa: E402
from paper_2007_04881_b200 import build_basis, classify_boundary_faces  # noqa: E402
from paper_2007_04881_b200.assembly import SipgPlan  # noqa: E402
from paper_2007_04881_b200.problems import WORKLOADS, cached_mesh, coefficients  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400000
pm = cached_mesh(replace(WORKLOADS["cfg5"], n=n))
real = coefficients("poisson_sine", 2)
const = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2), source=M.constant_scalar(19.7),
                          dirichlet_data=M.constant_scalar(0.0))
nosrc = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2), dirichlet_data=M.constant_scalar(0.0))
classify_boundary_faces(pm, real)
specs = build_basis(pm, 4)
for name, C in (("sin source", real), ("const source", const), ("no source", nosrc)):
    plan = SipgPlan(pm, C, specs)
    plan.run()
    plan.check_flags()
    ts = []
    for _ in range(5):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        plan.run(ev)
        torch.cuda.synchronize()
        ts.append(ev[2].elapsed_time(ev[3]))
    print(f"{name:14s} element kernel {min(ts):.3f} ms")
