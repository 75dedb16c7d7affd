"""Compile the NVRTC specialisation on the host (no GPU needed) to catch
source errors before a GPU call:  python tools/nvrtc_check.py [cfg] [degree]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_04881_b200.model import policy_source  # noqa: E402
from paper_2007_04881_b200.problems import WORKLOADS, coefficients  # noqa: E402


def main(cfg="cfg5", degree=None, sym=True, minblocks=3):
    w = WORKLOADS[cfg]
    p = w.degree if degree is None else int(degree)
    pol = policy_source(coefficients(w.coeffs, w.dim), w.dim)
    body = "assemble_body"
    threads = 32 * int(os.environ.get("PDG_JIT_WARPS", "4"))
    sym = str(sym) not in ("0", "False", "false")
    mr = os.environ.get("PDG_JIT_MAXNREG")
    bounds = f"__maxnreg__({mr})" if mr else f"__launch_bounds__({threads}, {minblocks})"
    tail = ", pdg_jit::JitCoef, 32"
    src = (f'#include "{body}.cuh"\n#include "prepass_body.cuh"\nnamespace pdg_jit {{\nusing namespace pdg;\n'
           + pol + '\n}\n'
           f'extern "C" __global__ void {bounds} pdg_jit_kernel(const __grid_constant__ pdg::KArgs a) {{\n'
           f'  pdg::{body}<{w.dim}, {p}, {"true" if sym else "false"}{tail}>(a, pdg_jit::JitCoef());\n}}\n'
           'extern "C" __global__ void __launch_bounds__(128) pdg_jit_face_prepass(const pdg_mesh m, '
           'const pdg_basis B, const pdg_rules R, const pdg_params prm, const double* abar, double* sigma, '
           'int8_t* flow, uint32_t* flags) {\n'
           f'  pdg::face_prepass_body<{w.dim}>(m, B, pdg_jit::JitCoef(), R, prm, abar, sigma, flow, flags);\n}}\n'
           'extern "C" __global__ void __launch_bounds__(256) pdg_jit_abar(const pdg_mesh m, const pdg_basis B, '
           'const pdg_rules R, const pdg_params prm, double* abar, uint32_t* flags) {\n'
           f'  pdg::elem_abar_body<{w.dim}>(m, B, pdg_jit::JitCoef(), R, prm, abar, flags);\n}}\n')
    lib = C.CDLL("libnvrtc.so.12")
    prog = C.c_void_p()
    assert lib.nvrtcCreateProgram(C.byref(prog), src.encode(), b"pdg_jit.cu", 0, None, None) == 0
    d = os.path.join(ROOT, "paper_2007_04881_b200")
    opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", f"-DPDG_RHS_REGS_MAX={os.environ.get('PDG_RHS_REGS_MAX', 20)}".encode(),
            f"-I{d}/csrc".encode(), f"-I{d}/../include".encode(), b"-Xptxas=-v"]
    opts += [t.encode() for t in os.environ.get("PDG_JIT_DEFINES", "").split()]
    arr = (C.c_char_p * len(opts))(*opts)
    rc = lib.nvrtcCompileProgram(prog, len(opts), arr)
    n = C.c_size_t()
    lib.nvrtcGetProgramLogSize(prog, C.byref(n))
    log = C.create_string_buffer(n.value)
    lib.nvrtcGetProgramLog(prog, log)
    print("rc", rc)
    if rc == 0:
        sz = C.c_size_t()
        lib.nvrtcGetCUBINSize(prog, C.byref(sz))
        buf = C.create_string_buffer(sz.value)
        lib.nvrtcGetCUBIN(prog, buf)
        with open(os.environ.get("PDG_CUBIN_OUT", "/tmp/pdg_jit.cubin"), "wb") as fh:
            fh.write(buf.raw)
    print(log.value.decode()[-3000:])
    return rc


if __name__ == "__main__":
    sys.exit(main(*sys.argv[1:]))
