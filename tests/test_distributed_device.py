"""The N-GPU path with the DEVICE engine on every rank (world_size 2, gloo,
both ranks sharing cuda:0 -- this box has one GPU; on an 8-GPU node the
same code runs over NCCL, one rank per GPU): contiguous cost-balanced
partition, each rank assembles ITS sub-mesh (owned elements + one-ring halo,
global columns), then the verification gather sends every rank's rows to
rank 0, which compares them bit for bit with the whole-mesh rows."""

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


def _worker(rank, world, port, out_dir, case):
    sys.path[:0] = [ROOT, HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import fixtures as F
    from paper_2007_04881_b200 import build_basis, classify_boundary_faces
    from paper_2007_04881_b200.distribute import (assemble_partition_device, contiguous_partition,
                                                  gather_verify_partition, quadrature_cost_weights)
    from paper_2007_04881_b200.mesh import agglomerate
    from paper_2007_04881_b200.meshgen import voronoi_mesh

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if case == "2d":
        pm = voronoi_mesh(400, seed=11)
        coeffs, p = F.adr(2), 3
    else:
        g = F.cube_grid(4)
        pm = agglomerate(g, F.grown_clusters(g, 40, seed=6))
        coeffs, p = F.variable_diffusion(3), 2
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, p)
    part = contiguous_partition(pm, world, quadrature_cost_weights(pm, specs))
    res = assemble_partition_device(pm, part, rank, coeffs, specs)
    local_el = res.local.flat.n_elements
    out = gather_verify_partition(res.plan, res.local, part, pm, coeffs, specs, chunk_bytes=1 << 16)
    if rank == 0:
        np.save(os.path.join(out_dir, "ok.npy"),
                np.array([out["verified"], out["bytes"] > 0, local_el < pm.n_elements,
                          len(part.cut_interfaces) > 0]))
        with open(os.path.join(out_dir, "log.txt"), "w") as fh:
            fh.write(repr(out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["2d", "3d"])
def test_two_rank_device_partition_verified_by_gather(tmp_path, case):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path), case), nprocs=2, join=True, start_method="spawn")
    ok = np.load(tmp_path / "ok.npy")
    assert ok.all(), (ok, (tmp_path / "log.txt").read_text())
