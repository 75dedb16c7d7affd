"""Multi-process (world_size 2, gloo on CPU) coverage of the N-GPU path's host
logic: contiguous cost-balanced partition, per-rank row assembly (the CPU
oracle stands in for each rank's device assembly), the verification gather
over torch.distributed, and stacking with gather_and_verify -- which must
reproduce the monolithic assembly bit for bit."""

import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path[:0] = [ROOT, HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import fixtures as F
    from oracle import sipg as oracle
    from paper_2007_04881_b200 import build_basis, classify_boundary_faces
    from paper_2007_04881_b200.assembly import CSRMatrix, DofMap
    from paper_2007_04881_b200.distribute import (PartialMatrix, _row_ranges, contiguous_partition,
                                                  gather_and_verify, nccl_gather_rows,
                                                  quadrature_cost_weights)
    from paper_2007_04881_b200.meshgen import voronoi_mesh

    dist.init_process_group("gloo", rank=rank, world_size=world)
    pm = voronoi_mesh(120, seed=11)
    coeffs = F.adr(2)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 2)
    part = contiguous_partition(pm, world, quadrature_cost_weights(pm, specs))
    own = part.owned[rank]
    rp, ci, v, rhs = oracle.assemble(pm, coeffs, specs, row_elements=own)
    got = nccl_gather_rows(torch.from_numpy(v), torch.from_numpy(ci), torch.from_numpy(rp))
    if rank == 0:
        dm = DofMap.from_specs(specs)
        partials = []
        for r, (prp, pci, pv) in enumerate(got):
            m = CSRMatrix(prp.numel() - 1, dm.n_dofs, prp.numpy(), pci.numpy(), pv.numpy())
            partials.append(PartialMatrix(r, _row_ranges(dm, part.owned[r]), m))
        full = gather_and_verify(partials, dm.n_dofs)
        mrp, mci, mv, _ = oracle.assemble(pm, coeffs, specs)
        np.save(os.path.join(out_dir, "ok.npy"),
                np.array([np.array_equal(full.row_ptr, mrp), np.array_equal(full.col_idx, mci),
                          np.array_equal(full.values, mv), len(part.cut_interfaces) > 0]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_partition_gather_equals_monolithic(tmp_path):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    ok = np.load(tmp_path / "ok.npy")
    assert ok.all(), ok
