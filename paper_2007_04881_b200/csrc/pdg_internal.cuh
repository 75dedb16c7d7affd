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

constexpr int MAX_P_2D = 6;
constexpr int MAX_P_3D = 4;
int check_common(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs);
bool symmetric_accumulation(const pdg_coeffs& C);

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

// col_idx of all rows of element e (assembly.py:319-324): lanes over column
// positions, each resolved by a short walk of the sorted neighbour list
// (division free), then stored down the element's rows.
__device__ __forceinline__ void write_col_rows(const pdg_basis& B, const pdg_pattern& P, int32_t e,
                                               int64_t val_off, int64_t L, int lane) {
  const int64_t ne = B.dof_offset[e + 1] - B.dof_offset[e];
  const int64_t q0 = P.nbr_ptr[e], q1 = P.nbr_ptr[e + 1];
  for (int64_t p = lane; p < L; p += 32) {
    int64_t cs = 0, q = q0, d0 = 0;
    for (; q < q1; ++q) {
      const int32_t j = P.nbr_elem[q];
      const int64_t nj = B.dof_offset[j + 1] - B.dof_offset[j];
      d0 = P.col_dof ? P.col_dof[j] : B.dof_offset[j];
      if (p < cs + nj) break;
      cs += nj;
    }
    const int64_t cv = d0 + (p - cs);
    for (int64_t r = 0; r < ne; ++r) P.col_idx[val_off + r * L + p] = cv;
  }
}

}  // namespace pdg
