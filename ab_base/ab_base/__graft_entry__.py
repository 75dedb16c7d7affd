"""Driver entry points: build() compiles libpdg.so for sm_100a in-tree;
smoke() runs one small assembly on cuda:0 and checks it against the oracle."""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))


def build() -> None:
    csrc = os.path.join(ROOT, "paper_2007_04881_b200", "csrc")
    jobs = str(max(2, min(8, os.cpu_count() or 2)))
    subprocess.run(["make", "-C", csrc, "-j", jobs], check=True)
    sys.path.insert(0, ROOT)
    import paper_2007_04881_b200  # noqa: F401
    from paper_2007_04881_b200 import _lib

    _lib.load()  # the library loads and exports every declared symbol


def smoke() -> None:
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np

    import fixtures as F
    from compare import assert_parity
    from oracle import sipg as oracle
    from paper_2007_04881_b200 import assemble_approach2, build_basis, classify_boundary_faces
    from paper_2007_04881_b200.meshgen import voronoi_mesh

    pm = voronoi_mesh(200, seed=0)
    coeffs = F.adr(2)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 3)
    m, rhs, stats, pattern = assemble_approach2(pm, coeffs, specs)
    ref = oracle.assemble(pm, coeffs, specs)
    be, re = assert_parity(m, rhs, ref, pattern.dof_map.offsets)
    print(f"smoke ok: {pm.n_elements} Voronoi cells p=3 ADR, nnz={m.nnz}, "
          f"max block rel err {be:.2e}, rhs {re:.2e}, device ms {stats.device_ms}")
    assert np.isfinite(m.values).all()


if __name__ == "__main__":
    build()
    smoke()
