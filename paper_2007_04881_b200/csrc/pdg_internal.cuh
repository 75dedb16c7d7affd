// Host-side plumbing shared by the C-ABI translation units: error state,
// launch geometry, and small device helpers used by several kernels.
#pragma once

#include <cstdio>
#include <algorithm>
#include <exception>
#include <string>

#include "sipg_device.cuh"

namespace pdg {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define PDG_TRY try
#define PDG_CATCH                                                         \
  catch (const std::exception& ex) { return ::pdg::fail(PDG_ERR_INVALID, ex.what()); } \
  catch (...) { return ::pdg::fail(PDG_ERR_INVALID, "unknown C++ exception"); }

#define PDG_CUDA(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return ::pdg::fail(PDG_ERR_CUDA, std::string(#expr " : ") + cudaGetErrorString(e_)); \
  } while (0)

int num_sms();

// launch accounting (pdg_launch_count): every kernel launch site calls this
void note_launch();

// grid-stride launches: a multiple of the SM count, capped by the work
inline int grid_for(int64_t n, int threads = 256) {
  const int64_t need = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
}
inline int grid_for_warps(int64_t nwarps, int threads) {
  const int64_t need = (nwarps * 32 + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 32;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
}

cudaError_t exclusive_scan(const int64_t* in, int64_t n, int64_t* out, int64_t* ws, cudaStream_t st);

// col_idx of all rows of element e: row a, position c -> the c-th column of
// the concatenated neighbour DoF ranges (assembly.py:319-324).
__device__ __forceinline__ void write_col_rows(const pdg_basis& B, const pdg_pattern& P, int32_t e,
                                               int64_t val_off, int64_t L, int lane) {
  const int64_t ne = B.dof_offset[e + 1] - B.dof_offset[e];
  int64_t colstart = 0;
  for (int64_t q = P.nbr_ptr[e]; q < P.nbr_ptr[e + 1]; ++q) {
    const int32_t j = P.nbr_elem[q];
    const int64_t d0 = B.dof_offset[j];
    const int64_t nj = B.dof_offset[j + 1] - d0;
    const int64_t tot = ne * nj;
    for (int64_t idx = lane; idx < tot; idx += 32) {
      const int64_t a = idx / nj, c = idx - a * nj;
      P.col_idx[val_off + a * L + colstart + c] = d0 + c;
    }
    colstart += nj;
  }
}

}  // namespace pdg
