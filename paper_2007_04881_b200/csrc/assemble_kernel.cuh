// Ahead-of-time instantiation + launch of the element kernel (interpreted
// coefficients).  The runtime-specialised variant is launched by pdg_jit.cu
// from the same body (assemble_body.cuh).
#pragma once

#include <cstdlib>

#include "assemble_body.cuh"
#include "pdg_internal.cuh"

namespace pdg {

// Per-warp shared-memory plan of the element kernel (must mirror the carving
// at the top of assemble_body): volume / face tables, 64 scalars, the
// neighbour staging window, and lane-private RHS partials for large bases.
inline AsmLayout make_layout(int dim, int P, int diff_kind, bool has_vr, int rhs_regs_max = PDG_RHS_REGS_MAX) {
  const int NB = binom(P + dim, dim);
  const int NBP = ((NB + 7) / 8) * 8;
  const bool rhs_regs = NB <= rhs_regs_max;
  AsmLayout L;
  const int nG = diff_kind != PDG_DIFF_NONE ? dim : 0;
  const int nAG = diff_kind == PDG_DIFF_FULL ? dim : 0;
  const int nVR = has_vr ? 2 : 0;
  L.vrows = nG + nAG + nVR;
  if (L.vrows == 0) L.vrows = 1;
  // volume slots per round: 32 while the table stays under 20 KB per warp;
  // PDG_VOL_KV=16|32 forces one (tuning knob: smaller tables raise occupancy)
  L.kv = (L.vrows * NBP * 36 * 8 <= 20 * 1024) ? 32 : 16;
  // 10-function bases with the advection/reaction rows: 16 slots keep 3 CTAs
  // per SM (shared memory) -- same-box r02, 250k cfg3 p=3: 4.37 vs 4.58 ms
  // (p = 2 and p = 4 measured better at 32)
  if (NB == 10 && L.vrows >= 4) L.kv = 16;
  if (const char* v = getenv("PDG_VOL_KV")) {
    const int kv = atoi(v);
    if (kv == 16 || kv == 32) L.kv = kv;
  }
  const int vol = L.vrows * NBP * (L.kv + 4);
  const int face = 4 * NBP * KFP;
  const int red = 32 * NB;
  int buf = vol > face ? vol : face;
  if (red > buf) buf = red;
  L.buf_doubles = buf;
  const int W = dim == 2 ? 8 : 16;  // frame record width (Widths<DIM>)
  const int NBR_WIN = nbr_win(dim), FR_MAX = fr_max(dim);
  L.warp_doubles = buf + 64 + (int)(2 * NBR_WIN * sizeof(pdg_iface_rec) / 8) + (rhs_regs ? 0 : 32 * NB) + FR_MAX * W +
                   (dim == 3 ? 2 : 1) * NBR_WIN * W +  // simplex frames, first facet frames, neighbour basis constants (3D)
                   2;                                  // the warp's mbarrier (8-byte aligned: every term is even)
  return L;
}

template <int DIM, int P, bool SYM>
__global__ void __launch_bounds__(128) assemble_elements(const __grid_constant__ KArgs a,
                                                         const __grid_constant__ pdg_coeffs C) {
  assemble_body<DIM, P, SYM>(a, InterpCoef<DIM>(C));
}

// Occupancy-aware grid: a multiple of the SM count, each CTA 4 warps.
inline int64_t element_grid(const void* kern, int threads, size_t smem, int64_t n_rows) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t need = (n_rows + threads / 32 - 1) / (threads / 32);
  return std::min<int64_t>(need, (int64_t)num_sms() * per_sm * 8);
}

template <int DIM, int P, bool SYM>
cudaError_t launch_assemble(KArgs a, const pdg_coeffs& C, cudaStream_t st) {
  a.lay = make_layout(DIM, P, C.diffusion_kind, C.has_advection || C.has_reaction);
  const int threads = 128;
  const size_t smem = ((size_t)rule_smem_doubles(PDG_RULES_SMEM ? a.R.n_points : 0) +
                       (size_t)a.lay.warp_doubles * (threads / 32)) * 8;
  auto kern = assemble_elements<DIM, P, SYM>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int64_t grid = element_grid((const void*)kern, threads, smem, a.pat.n_row_elements);
  if (grid <= 0) return cudaSuccess;
  kern<<<(unsigned)grid, threads, smem, st>>>(a, C);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pdg
