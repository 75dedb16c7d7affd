"""Per-call CUDA-event times of one SipgPlan step (index / pre-pass kernels):
    python tools/phase_times.py [cfg] [n]"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from dataclasses import replace  # noqa: E402

from paper_2007_04881_b200 import _lib, build_basis, classify_boundary_faces  # noqa: E402
from paper_2007_04881_b200.assembly import SipgPlan  # noqa: E402
from paper_2007_04881_b200.problems import WORKLOADS, cached_mesh, coefficients  # noqa: E402


def main(cfg="cfg5", n=None):
    w = WORKLOADS[cfg]
    if n:
        w = replace(w, n=int(n))
    pm = cached_mesh(w)
    co = coefficients(w.coeffs, w.dim)
    classify_boundary_faces(pm, co)
    specs = build_basis(pm, w.degree)
    plan = SipgPlan(pm, co, specs)
    plan.run()
    plan.check_flags()
    s = _lib.stream_ptr(plan.stream)
    lib = plan.lib
    calls = {
        "adjacency": lambda: lib.pdg_adjacency(C.byref(plan.dm.struct), _lib.ptr(plan.t["nbr_ptr"]),
                                               _lib.ptr(plan.t["nbr_elem"]), _lib.ptr(plan.t["nbr_iface"]),
                                               _lib.ptr(plan.t["ws"]), plan.ws_bytes, s),
        "pattern_offsets": lambda: lib.pdg_pattern_offsets(C.byref(plan.dm.struct), C.byref(plan.basis),
                                                           C.byref(plan.pattern), plan.n_local_rows, None,
                                                           _lib.ptr(plan.t["ws"]), plan.ws_bytes, s),
        "frames": lambda: lib.pdg_frames_build(C.byref(plan.dm.struct), C.byref(plan.basis), C.byref(plan.frames),
                                               _lib.ptr(plan.t["flags"]), s),
        "face_prepass": lambda: lib.pdg_face_prepass(C.byref(plan.dm.struct), C.byref(plan.basis),
                                                     C.byref(plan.coeffs), C.byref(plan.rules.struct),
                                                     C.byref(plan.params), _lib.ptr(plan.t["sigma"]),
                                                     _lib.ptr(plan.t["flow"]), _lib.ptr(plan.t["abar"]),
                                                     _lib.ptr(plan.t["flags"]), s),
        "iface_records": lambda: lib.pdg_iface_records(C.byref(plan.dm.struct), C.byref(plan.basis),
                                                       C.byref(plan.coeffs), C.byref(plan.rules.struct),
                                                       C.byref(plan.params), C.byref(plan.pattern),
                                                       _lib.ptr(plan.t["sigma"]), _lib.ptr(plan.t["flow"]), s),
        "element_kernel": lambda: plan._elements(),
    }
    with torch.cuda.stream(plan.stream):
        for name, fn in calls.items():
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(plan.stream)
                rc = fn()
                b.record(plan.stream)
                plan.stream.synchronize()
                assert rc in (None, 0), rc
                ts.append(a.elapsed_time(b))
            print(f"{name:16s} {min(ts):8.3f} ms (min of 5)")


if __name__ == "__main__":
    main(*sys.argv[1:])
