"""Compile the slab NVRTC module on the host (no GPU needed):
    python tools/nvrtc_slab_check.py [case] [degree] [PQ|P] [warps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import fixtures as F  # noqa: E402
from paper_2007_04881_b200.model import slab_policy  # noqa: E402


def main(case="slab_heat", degree="2", fam="PQ", nw="4"):
    coeffs, u0 = getattr(F, case)()
    pol, rows = slab_policy(coeffs, u0)
    pq = "true" if fam == "PQ" else "false"
    src = ('#include "slab_body.cuh"\nnamespace pdg_jit {\nusing namespace pdg;\n' + pol + '\n}\n'
           f'extern "C" __global__ void __launch_bounds__({32 * int(nw)}, 1) '
           'pdg_slab_kernel(const __grid_constant__ pdg::SlabArgs a) {\n'
           f'  pdg::slab_body<2, {degree}, {pq}, {nw}, pdg_jit::JitCoef>(a, pdg_jit::JitCoef());\n}}\n'
           'extern "C" __global__ void __launch_bounds__(128) '
           'pdg_slab_prepass(const __grid_constant__ pdg::SlabArgs a, double* sigma, int8_t* flow) {\n'
           '  pdg::slab_prepass_body<2>(a, pdg_jit::JitCoef(), sigma, flow);\n}\n')
    lib = C.CDLL("libnvrtc.so.12")
    prog = C.c_void_p()
    assert lib.nvrtcCreateProgram(C.byref(prog), src.encode(), b"pdg_jit.cu", 0, None, None) == 0
    d = os.path.join(ROOT, "paper_2007_04881_b200")
    opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", b"-DPDG_RHS_REGS_MAX=20",
            f"-I{d}/csrc".encode(), f"-I{d}/../include".encode(), b"-Xptxas=-v"]
    arr = (C.c_char_p * len(opts))(*opts)
    rc = lib.nvrtcCompileProgram(prog, len(opts), arr)
    n = C.c_size_t()
    lib.nvrtcGetProgramLogSize(prog, C.byref(n))
    log = C.create_string_buffer(n.value)
    lib.nvrtcGetProgramLog(prog, log)
    print("rc", rc, "table rows", rows)
    if rc == 0:
        sz = C.c_size_t()
        lib.nvrtcGetCUBINSize(prog, C.byref(sz))
        buf = C.create_string_buffer(sz.value)
        lib.nvrtcGetCUBIN(prog, buf)
        with open(os.environ.get("PDG_CUBIN_OUT", "/tmp/pdg_slab.cubin"), "wb") as fh:
            fh.write(buf.raw)
    print(log.value.decode()[-4000:])
    return rc


if __name__ == "__main__":
    sys.exit(main(*sys.argv[1:]))
