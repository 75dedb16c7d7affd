"""Host vs device agglomerate on an n-cell Voronoi mesh: python tools/agg_timing.py [n]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_04881_b200.mesh import agglomerate  # noqa: E402
from paper_2007_04881_b200.meshgen import voronoi_simplicial  # noqa: E402
from paper_2007_04881_b200.meshprep import agglomerate_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
t = time.perf_counter()
base, agg = voronoi_simplicial(n, seed=3)
tg = time.perf_counter() - t
agglomerate_device(base[:0] if False else base, agg, check_connected=False)  # warm-up (CUDA context, cub)
t = time.perf_counter()
dev = agglomerate_device(base, agg, check_connected=True)
td = time.perf_counter() - t
t = time.perf_counter()
host = agglomerate(base, agg, check_connected=True)
th = time.perf_counter() - t
same = all(np.array_equal(getattr(host.flat, k), getattr(dev.flat, k)) for k in host.flat.arrays())
print(f"n={n} simplices={base.n_simplices} voronoi {tg:.1f}s  agglomerate host {th:.2f}s device {td:.2f}s "
      f"(incl. H2D/D2H) identical={same}")
