"""Element-block SpMV / block-Jacobi on an assembled workload:
    python tools/spmv_bench.py [cfg] -> JSON line with GB/s against HBM."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_04881_b200 import build_basis, classify_boundary_faces  # noqa: E402
from paper_2007_04881_b200.assembly import SipgPlan  # noqa: E402
from paper_2007_04881_b200.problems import WORKLOADS, cached_mesh, coefficients  # noqa: E402
from paper_2007_04881_b200.solver import BlockJacobiPreconditioner, DeviceSystem, _PlanCSR  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
w = WORKLOADS[cfg]
pm = cached_mesh(w)
C = coefficients(w.coeffs, w.dim)
classify_boundary_faces(pm, C)
specs = build_basis(pm, w.degree)
plan = SipgPlan(pm, C, specs)
plan.run()
plan.check_flags()
sys_ = DeviceSystem(_PlanCSR(plan), plan.dof.offsets)
n = sys_.n
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


ms = timed(lambda: sys_.matvec(x, y))
counts = np.diff(plan.dof.offsets)
L = plan.t["row_len"].cpu().numpy()
nnz = plan.nnz
byts = 8.0 * nnz + 8.0 * float(L.sum()) * 2 + 16.0 * n  # values + column list (+ gathered x) + x, y
csr_bytes = 16.0 * nnz + 16.0 * n
pre = BlockJacobiPreconditioner(sys_)
ms_apply = timed(lambda: pre.apply(x, y))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.0
print(json.dumps({"workload": cfg, "rows": n, "nnz": nnz, "spmv_ms": ms, "spmv_gbs": byts / ms / 1e6,
                  "spmv_frac_hbm": byts / ms / 1e6 / peak,
                  "plain_csr_equivalent_gbs": csr_bytes / ms / 1e6,
                  "block_jacobi_apply_ms": ms_apply, "hbm_peak_gbs": peak}))
