#!/usr/bin/env python
"""fp64 SIPG assembly benchmark (BASELINE.json metric: assembly elements/s and
wall ms at 1/2/4/8 B200, next to the host-CPU reference path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]

One step = one full assembly of the workload's rows on each rank: index
phase (adjacency, row offsets), face pre-pass (sigma, flow side) and the fused
element kernel (values + col_idx + RHS), with the mesh resident in HBM.
Multi-GPU (torchrun): the paper's experiment -- ONE workload mesh split into
N contiguous, cost-balanced parts (strong scaling, value =
the mesh's elements / max-over-ranks time).  Each rank assembles ITS
sub-mesh only (owned elements + one-ring halo, global columns:
distribute.local_problem), so index phase, pre-pass and kernel all shrink
with N; assembly needs no communication.  After the timed
region one verification gather (NCCL point-to-point to rank 0) collects
every rank's rows and rank 0 compares them bit for bit with the whole-mesh
rows ("verified" in the JSON line).  ``--weak``: every rank assembles its
own instance of the workload instead (value = N x elements / max time).
``e2e`` re-runs the step through the public plan API with the mesh copied
from pinned host memory and the assembled CSR + RHS copied back every step.
``--impl reference`` times the CPU restatement of polydg's path (oracle/,
all host cores) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 SIPG assembly elements/s"
UNIT = "elements/s"
SLAB_INTERVAL = (0.0, 0.1)
# the paper's Approach-2 fp64 single-GPU space-time numbers, s per 10^6 DoFs,
# p = 1..5 (1x Tesla P100): total kernels / total assembly
PAPER_P100_S_PER_MDOF = {"kernels": [0.03, 0.17, 0.57, 1.9, 5.5], "total": [1.02, 1.9, 3.7, 7.2, 14.7]}


def is_slab(w) -> bool:
    return w.coeffs.startswith("slab")


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--degree", type=int, default=None, help="override the workload degree")
    ap.add_argument("--n", type=int, default=None, help="override the workload size")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--strong", action="store_true",
                    help="N>1: split ONE workload mesh into N cost-balanced parts (the default; kept as a no-op flag)")
    ap.add_argument("--weak", action="store_true",
                    help="N>1: one independent workload instance per rank (weak scaling) instead of the "
                         "partitioned mesh")
    ap.add_argument("--no-verify", action="store_true", help="N>1: skip the verification gather")
    ap.add_argument("--approach", type=int, default=2, choices=(1, 2),
                    help="2 = preset sparsity (default); 1 = stage-and-sort (triplets + device sort)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-api-max-gb", type=float, default=4.0,
                    help="run the assemble_approach2 end-to-end leg when the host CSR is at most this size")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / baseline)")
    return ap.parse_args()


def workload(args):
    from dataclasses import replace

    from paper_2007_04881_b200.problems import WORKLOADS

    w = WORKLOADS[args.config]
    if args.degree is not None:
        w = replace(w, degree=args.degree)
    if args.n is not None:
        w = replace(w, n=args.n)
    return w


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling during the timed region (NVML)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.1):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def fp64_peak():
    """Builder-measured FP64 (DMMA/DFMA) peak, TFLOP/s, newest of
    profiles/fp64_peaks_r0*.json (tools/fp64_peaks.cu; MEASURED_PEAKS.json
    carries no fp64 figure)."""
    for name in ("fp64_peaks_r02.json", "fp64_peaks_r01.json"):
        p = os.path.join(ROOT, "profiles", name)
        try:
            with open(p) as fh:
                d = json.load(fh)
            mhz = d.get("clocks", {}).get("sm_mhz_median") or d.get("clock_khz_attr", 0) / 1000
            return (float(max(d["dmma_m8n8k4_acc4_tflops"], d["dfma_tflops"])),
                    f"profiles/{name} (builder-measured fp64: DMMA m8n8k4 / DFMA microbenchmark, "
                    f"{mhz:.0f} MHz SM clock)")
        except Exception:
            continue
    return 37.0, "B200 datasheet fallback"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json (measured)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback"


def ncu_traffic(config, n_elements):
    """dram__bytes_read.sum + dram__bytes_write.sum of the element kernel from
    the committed ncu --set full capture (profiles/ncu_element_kernel.json),
    per launch of this workload: the capture's bytes per element x elements
    (the capture runs a smaller mesh of the same generator and degree)."""
    p = os.path.join(ROOT, "profiles", "ncu_element_kernel.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d[config]["dram_bytes_per_element"]) * n_elements
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU reference (oracle restatement of polydg on all host cores)
# ---------------------------------------------------------------------------

class CpuReference:
    """The oracle (plain-numpy port of polydg's assemble_approach2 path) on a
    bounded sample: a sub-scale mesh from the same generator, coefficients and
    degree, run with fork workers on all host cores.  Its elements/s is
    rate-extrapolated to the full workload."""

    def __init__(self, w, per_core: int = 150):
        from dataclasses import replace

        from oracle import sipg as oracle
        from paper_2007_04881_b200 import build_basis, classify_boundary_faces
        from paper_2007_04881_b200.problems import build_mesh, coefficients

        self.oracle = oracle
        self.cores = oracle.host_cores()
        if w.dim == 2:
            sw = replace(w, n=max(256, min(w.n, per_core * self.cores)))
        else:
            sw = replace(w, n=12, k=max(300, min(w.k, per_core * self.cores // 2)))
        self.slab = is_slab(w)
        if self.slab:
            per_core = max(8, per_core // (4 * w.degree))
            sw = replace(w, n=max(128, min(w.n, per_core * self.cores)))
        self.pm = build_mesh(sw)
        self.w = w
        if self.slab:
            from oracle import spacetime as ost
            from paper_2007_04881_b200 import Family
            from paper_2007_04881_b200.problems import slab_coefficients
            from paper_2007_04881_b200.spacetime import build_slab

            self.ost = ost
            self.coeffs, self.initial = slab_coefficients("heat")
            _, self.specs = build_slab(self.pm, SLAB_INTERVAL, w.degree, Family.P)
            return
        self.coeffs = coefficients(w.coeffs, w.dim)
        classify_boundary_faces(self.pm, self.coeffs)
        self.specs = build_basis(self.pm, w.degree)

    def step(self) -> float:
        t0 = time.perf_counter()
        if self.slab:
            self.ost.assemble_slab(self.pm, SLAB_INTERVAL[0], SLAB_INTERVAL[1], self.coeffs, self.specs,
                                   self.initial, workers=self.cores)
        else:
            self.oracle.assemble(self.pm, self.coeffs, self.specs, workers=self.cores)
        return time.perf_counter() - t0

    def sample(self, dt) -> str:
        kind = "Voronoi" if self.w.dim == 2 else "agglomerated Kuhn"
        what = "spacetime.assemble_slab" if self.slab else "assemble_approach2"
        return (f"{self.pm.n_elements} elements of the same {kind} generator (p={self.w.degree}, "
                f"{self.w.coeffs}); oracle/ numpy port of polydg {what} with "
                f"{self.cores} fork workers, {dt:.2f} s per assembly; elements/s rate-extrapolated "
                f"to the {self.w.name} workload")


def cpu_reference_rate(w, min_seconds=10.0):
    ref = CpuReference(w)
    total, n = 0.0, 0
    while total < min_seconds or n < 1:
        total += ref.step()
        n += 1
    dt = total / n
    return ref.pm.n_elements / dt, ref.cores, ref.sample(dt), dt


def run_reference(args, w, rank):
    if rank != 0:
        return  # rank 0 alone runs the CPU arm
    ref = CpuReference(w)
    for _ in range(args.warmup):
        ref.step()
    times = [ref.step() for _ in range(args.steps)]
    dt = float(statistics.median(times))
    value = ref.pm.n_elements / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": w.description, "name": w.name, "degree": w.degree,
                                        "sample_elements": ref.pm.n_elements},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.cores, "kind": "port",
                         "sample": ref.sample(dt)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, w, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2007_04881_b200 import _lib, build_basis, classify_boundary_faces
    from paper_2007_04881_b200.assembly import AssemblyConfig, HostIO, SipgPlan
    from paper_2007_04881_b200.distribute import (contiguous_partition, gather_verify_partition, local_problem,
                                                  quadrature_cost_weights)
    from paper_2007_04881_b200.problems import cached_mesh, coefficients
    from paper_2007_04881_b200.roofline import assembly_work

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        # rank 0 builds (or loads) the mesh first so the others hit the cache
        if rank == 0:
            t0 = time.perf_counter()
            pm = cached_mesh(w)
            mesh_s = time.perf_counter() - t0
        dist.barrier()
        if rank != 0:
            t0 = time.perf_counter()
            pm = cached_mesh(w)
            mesh_s = time.perf_counter() - t0
    else:
        t0 = time.perf_counter()
        pm = cached_mesh(w)
        mesh_s = time.perf_counter() - t0
    slab_case = is_slab(w)
    cfg = AssemblyConfig()
    if slab_case:
        from paper_2007_04881_b200 import Family
        from paper_2007_04881_b200.problems import slab_coefficients
        from paper_2007_04881_b200.roofline import slab_work
        from paper_2007_04881_b200.spacetime import SlabPlan, build_slab

        coeffs, initial = slab_coefficients("heat")
        slab, specs = build_slab(pm, SLAB_INTERVAL, w.degree, Family.P)
    else:
        coeffs = coefficients(w.coeffs, w.dim)
        classify_boundary_faces(pm, coeffs)
        specs = build_basis(pm, w.degree)
    rows, lp, part = None, None, None
    partitioned = world > 1 and not args.weak
    t_part = time.perf_counter()
    if partitioned:
        part = contiguous_partition(pm, world, quadrature_cost_weights(pm, specs))
        rows = part.owned[rank]
        if not slab_case and args.approach == 2:
            lp = local_problem(pm, part, rank, specs, cfg)  # the rank's sub-mesh (host preprocessing)
    part_s = time.perf_counter() - t_part
    stream = torch.cuda.Stream(dev)
    if slab_case:
        plan = SlabPlan(slab, coeffs, specs, initial, cfg, row_elements=rows, device=dev, stream=stream)
        work = slab_work(plan)
    elif args.approach == 1:
        from paper_2007_04881_b200.approach1 import Approach1Plan

        if world > 1:
            raise NotImplementedError("Approach 1 bench runs on one GPU")
        plan = Approach1Plan(pm, coeffs, specs, cfg, device=dev, stream=stream)
        work = assembly_work(plan.base)
    elif lp is not None:
        plan = SipgPlan(lp.flat, coeffs, lp.specs, lp.config, row_elements=lp.owned_local, device=dev,
                        stream=stream, col_dof=lp.col_dof)
        work = assembly_work(plan)
    else:
        plan = SipgPlan(pm, coeffs, specs, cfg, row_elements=rows, device=dev, stream=stream)
        work = assembly_work(plan)
    lib = _lib.load()

    # warm-up (first run also validates the device error flags)
    for i in range(max(args.warmup, 1)):
        plan.run()
    plan.check_flags()

    # CUDA graphs: a step = 3 graph launches (index, pre-pass, element kernel)
    # instead of ~20 kernel launches -- small meshes are launch-bound
    graphs = (os.environ.get("PDG_GRAPHS", "1") != "0" and hasattr(plan, "capture_graphs")
              and plan.capture_graphs())
    step = plan.run_graphs if graphs else plan.run
    if graphs:
        for _ in range(2):
            step()
        plan.check_flags()

    K = args.steps
    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = lib.pdg_launch_count()
    # timed: K whole steps back to back (one graph launch per step when
    # captured); the phase split comes from a separate, untimed event run
    with ClockSampler(local_rank) as clk:
        t_start.record(stream)
        for k in range(K):
            step()
        t_stop.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = int(lib.pdg_launch_count() - l0) + (plan.graph_launches * K if graphs else 0)
    ms = t_start.elapsed_time(t_stop) / K
    KP = min(K, 5)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(KP)]
    for k in range(KP):
        step(evs[k])
    torch.cuda.synchronize(dev)
    ms_index = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    ms_pre = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    ms_el = statistics.mean(e[2].elapsed_time(e[3]) for e in evs)
    if args.approach == 1 and not slab_case:  # events: start | pre-pass | emit | sort + merge
        ms_pre, ms_el, ms_index = ms_index, ms_pre, ms_el
    plan.check_flags()

    # end to end through the plan API with host buffers
    e2e_ms, h2d, d2h, e2e_host = None, 0, 0, None
    if not args.no_e2e and not args.profile and args.e2e_steps > 0:
        io = HostIO(plan)
        h2d, d2h = io.h2d_bytes, io.d2h_bytes
        io.upload(); step(); io.download()
        stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            io.upload()
            step()
            io.download()
        e1.record(stream)
        stream.synchronize()
        e2e_ms = e0.elapsed_time(e1) / args.e2e_steps
        e2e_host = {"retained": io.retained}
        if io.retained:  # the last step's host CSR: row_ptr + RHS whole, values / col_idx sampled
            mat_h, rhs_hh = io.result()
            st = max(1, mat_h.nnz // (1 << 20))
            e2e_host["checked"] = bool(
                np.array_equal(mat_h.row_ptr, plan.row_ptr.cpu().numpy())
                and np.array_equal(rhs_hh, plan.rhs.cpu().numpy())
                and np.array_equal(mat_h.values[::st], plan.values[::st].cpu().numpy())
                and np.array_equal(mat_h.col_idx[::st], plan.col_idx[::st].cpu().numpy()))
            e2e_host["how"] = ("D2H into page-locked host CSR arrays (pdg_host_alloc, kept across steps, "
                               "HostIO.result()); "
                               + ("col_idx crosses the link once per element (each element's first row, "
                                  "pdg_pack_block_cols) and host threads write it into every row "
                                  "(pdg_expand_block_cols) while the values transfer; " if io.packed_cols else
                                  "every row of col_idx over the link (CSR below the packing threshold); ")
                               + "checked against the device CSR after the "
                               f"timed region (row_ptr, rhs whole; values, col_idx every {st}th entry)")
            del mat_h, rhs_hh
        else:
            e2e_host["how"] = "D2H through a 1 GiB pinned ring (page-locked host allocation failed)"
        io.close()
        del io

    # end to end through the public polydg-compatible call itself: host mesh
    # object in, host CSR + RHS + BlockPattern out (pinned chunked D2H), every
    # step a fresh plan (allocation from torch's cache, one nnz size-query sync)
    e2e_api = None
    plan_nnz = int(plan.nnz)
    plan_dofs = int(plan.dof.n_dofs)
    csr_gb = 16.0 * plan_nnz / 1e9
    if (world == 1 and not slab_case and args.approach == 2 and not args.no_e2e and not args.profile
            and csr_gb <= args.e2e_api_max_gb):
        from paper_2007_04881_b200 import assemble_approach2

        if csr_gb > 20.0:  # make room in HBM: each call builds its own plan
            plan.graphs, plan.graph_step, plan.t = None, None, {}
            torch.cuda.empty_cache()

        assemble_approach2(pm, coeffs, specs, cfg)  # warm (JIT, device mesh, allocator)
        times = []
        for _ in range(max(2, min(args.steps, 5))):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            mat, rhs_h, _, _ = assemble_approach2(pm, coeffs, specs, cfg)
            times.append(time.perf_counter() - t0)
            d2h_api = mat.row_ptr.nbytes + mat.col_idx.nbytes + mat.values.nbytes + rhs_h.nbytes
            del mat, rhs_h
        t_api = statistics.median(times)
        e2e_api = {"value": pm.n_elements / t_api, "unit": UNIT, "ms_per_step": t_api * 1e3,
                   "through": "paper_2007_04881_b200.assemble_approach2 (polydg signature: host mesh in, host "
                              "CSRMatrix + rhs + AssemblyStats + BlockPattern out); wall clock of the call",
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(d2h_api),
                   "note": "the mesh's HBM copy is cached on the mesh object across calls (as a "
                           "resident-mesh caller would); the plan, CSR buffers and host arrays are new each call"}
    cdev = dev if world == 1 or dist.get_backend() == "nccl" else torch.device("cpu")

    def allmax(x):
        if world == 1 or x is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    ms_max = allmax(ms)
    e2e_max = allmax(e2e_ms)
    el_ms_max = allmax(ms_el)
    h2d_tot, d2h_tot = allsum(h2d), allsum(d2h)
    launches_tot = allsum(launches / K)
    flops_tot, bytes_tot = allsum(work["flops"]), allsum(work["bytes"])
    nnz_tot = allsum(float(plan_nnz))
    local_el = float(lp.flat.n_elements) if lp is not None else float(pm.n_elements)
    local_el_max = allmax(local_el)
    # weak scaling (--weak): every rank assembles its own instance of the
    # workload, so the units processed are N x the workload; default: the
    # ranks share one mesh
    weak = world > 1 and args.weak
    n_el = pm.n_elements * (world if weak else 1)
    verify = None
    if partitioned and lp is not None and not args.no_verify and not args.profile:
        torch.cuda.synchronize(dev)
        verify = gather_verify_partition(plan, lp, part, pm, coeffs, specs, cfg)
    if rank != 0:
        return
    peak, peak_src = fp64_peak()
    hbm, hbm_src = hbm_peak()
    # whole-job algorithmic work over the slowest rank's element-kernel time
    achieved = flops_tot / (el_ms_max * 1e-3) / 1e12 / world
    gbs = bytes_tot / (el_ms_max * 1e-3) / 1e9 / world
    line = {
        "metric": METRIC if not slab_case else "fp64 space-time slab assembly elements/s",
        "value": n_el / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if partitioned else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated mesh; analytic coefficients)",
        "config": {"workload": w.description, "name": w.name, "elements": n_el, "degree": w.degree,
                   "family": "P" if slab_case else None,
                   "dofs": int(specs_dofs(specs, w.dim)) if not slab_case else plan_dofs,
                   "nnz": int(nnz_tot) if not weak else plan_nnz,
                   "parallelism": (f"partitioned x{world}: one mesh, contiguous cost-balanced parts, "
                                   f"per-rank sub-mesh (owned + halo)" if partitioned else
                                   f"x{world} ranks, one workload instance each (no collective)")
                   if world > 1 else "single GPU",
                   "elements_per_rank": pm.n_elements if weak else None,
                   "max_local_elements": int(local_el_max) if partitioned else None,
                   "partition_s": round(part_s, 2) if partitioned else None,
                   "l2": "inputs+outputs >> 126 MB L2 (CSR written fresh each step), no flush needed"
                   if plan_nnz * 16 > 4e8 else "small workload: L2-resident",
                   "mesh_build_s": round(mesh_s, 1)},
        "phases_ms": {"index": ms_index, "prepass": ms_pre, "element_kernel": ms_el},
        "approach": args.approach if not slab_case else 2,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "per": "GPU (whole-job canonical FLOPs / N / slowest rank's element-kernel time)",
                     "frac": achieved / peak, "traffic": ncu_traffic(w.name, n_el),
                     "kernel": "pdg_slab_kernel (fused prism volume+lateral+bottom, DMMA f64)" if slab_case
                     else ("pdg_a1_kernel (Approach 1 item emission, DMMA f64)" if args.approach == 1
                           else "assemble_elements (fused volume+face+boundary, DMMA f64)"),
                     "algorithmic_flops_per_launch": work["flops"],
                     "algorithmic_bytes_per_launch": work["bytes"],
                     "hbm_achieved_gbs": gbs, "hbm_peak_gbs": hbm, "hbm_frac": gbs / hbm,
                     "peak_source": peak_src},
        "clocks": clk.summary(),
        "gpu_launches": int(round(launches_tot * K)),
        "cuda_graphs": bool(graphs),
        "gpu_launches_per_step": launches_tot,
    }
    if slab_case:
        mdof = plan_dofs / 1e6
        line["s_per_million_dofs"] = {"total": ms_max * 1e-3 / mdof, "kernels": (ms_pre + ms_el) * 1e-3 / mdof,
                                      "index": ms_index * 1e-3 / mdof}
        if 1 <= w.degree <= 5:
            line["paper_p100_s_per_million_dofs"] = {
                k: v[w.degree - 1] for k, v in PAPER_P100_S_PER_MDOF.items()}
            line["paper_p100_source"] = "PAPER.md:671-677 (Approach 2, fp64, 1x Tesla P100, not this metric's hardware)"
    if world > 1 and torch.cuda.device_count() < world:
        line["note"] = (f"{world} ranks time-share {torch.cuda.device_count()} GPU(s) (PDG_DIST_BACKEND=gloo): "
                        "a correctness run of the partitioned path, not a scaling measurement")
    if verify is not None:
        line["verified"] = "bitwise" if verify["verified"] else "MISMATCH"
        line["verify_gather"] = {"bytes": verify["bytes"], "seconds": round(verify["seconds"], 2),
                                 "how": "every rank's rows -> rank 0 (point-to-point, chunked), compared with "
                                        "torch.equal against the whole-mesh rows of the same part",
                                 "mismatch": verify["mismatch"]}
    if e2e_api is not None:
        line["e2e_api"] = e2e_api
    if e2e_max is not None:
        line["e2e"] = {"value": n_el / (e2e_max * 1e-3), "unit": UNIT, "ms_per_step": e2e_max,
                       "h2d_bytes_per_step": int(h2d_tot), "d2h_bytes_per_step": int(d2h_tot)}
        if e2e_host is not None:
            line["e2e"]["host_result"] = e2e_host
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        rate, cores, sample, _ = cpu_reference_rate(w)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)


def specs_dofs(specs, dim) -> int:
    from paper_2007_04881_b200.assembly import DofMap

    return DofMap.from_specs(specs).n_dofs


def main():
    args = parse()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    w = workload(args)
    if args.impl == "reference":
        run_reference(args, w, rank)  # CPU only; ranks != 0 exit without work
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        # PDG_DIST_BACKEND=gloo + fewer GPUs than ranks: ranks share devices
        # (exercises the partitioned path on a 1-GPU box; NCCL needs one GPU per rank)
        backend = os.environ.get("PDG_DIST_BACKEND", "nccl")
        local_rank = local_rank % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    run_ours(args, w, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
