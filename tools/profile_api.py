"""cProfile of the polydg-signature call assemble_approach2 at cfg2 scale (host
overhead around the device work)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2007_04881_b200 import assemble_approach2, build_basis, classify_boundary_faces  # noqa: E402
from paper_2007_04881_b200.problems import WORKLOADS, cached_mesh, coefficients  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
pm = cached_mesh(w)
C = coefficients(w.coeffs, w.dim)
classify_boundary_faces(pm, C)
specs = build_basis(pm, w.degree)
for _ in range(2):
    assemble_approach2(pm, C, specs)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    assemble_approach2(pm, C, specs)
pr.disable()
print("ms per call", (time.perf_counter() - t0) / 3 * 1e3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
