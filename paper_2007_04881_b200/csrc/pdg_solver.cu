// Consumers of the device CSR: the element-block SpMV and the
// element-block Jacobi preconditioner of polydg's solver (solver.py:30-118).
//
// The assembled matrix has one dense block per (row element, neighbour):
// every row of element e holds the same column list (the concatenated DoF
// ranges of e's sorted neighbours, assembly.py:316-324).  The SpMV exploits
// it: one warp per element gathers x over that column list ONCE into shared
// memory, then streams the element's n_e value rows against it (lanes over
// columns, coalesced; one warp reduction per row).  HBM traffic per stored
// value is 8 B (+ 8 B / n_e for the shared column list) instead of CSR's 16 B.
//
// Block-Jacobi: warp per element, the diagonal block (the self block of e's
// rows) copied into shared memory and inverted in place by Gauss-Jordan with
// partial pivoting (the inverse polydg takes with np.linalg.inv,
// solver.py:47-70); the apply is a batched dense mat-vec.
#include "pdg_internal.cuh"

namespace pdg {
namespace {

constexpr int SPMV_WARPS = 4;
constexpr int SPMV_MAXL = 512;  // columns per element row staged in shared memory (longer: direct gathers)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// rows r0..r0+R-1 of an element against the gathered x (xs, or x via col_idx)
template <int R, bool STAGED>
__device__ __forceinline__ void spmv_rows(const double* v, int64_t L, const double* xs, const int64_t* cols,
                                          const double* x, double* y, int lane) {
  double s[R];
#pragma unroll
  for (int i = 0; i < R; ++i) s[i] = 0.0;
  for (int64_t p = lane; p < L; p += 32) {
    const double xv = STAGED ? xs[p] : x[cols[p]];
#pragma unroll
    for (int i = 0; i < R; ++i) s[i] += v[(int64_t)i * L + p] * xv;
  }
#pragma unroll
  for (int i = 0; i < R; ++i) s[i] = warp_sum(s[i]);
  if (lane < R) {
    double o = s[0];
#pragma unroll
    for (int i = 1; i < R; ++i)
      if (lane == i) o = s[i];
    y[lane] = o;
  }
}

__global__ void __launch_bounds__(32 * SPMV_WARPS) spmv_blocked(const int64_t* dof, int64_t nel,
                                                                const int64_t* row_ptr, const int64_t* col_idx,
                                                                const double* vals, const double* x, double* y,
                                                                uint32_t* flags) {
  __shared__ double xs[SPMV_WARPS][SPMV_MAXL];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < nel; e += nw) {
    const int64_t r0 = dof[e];
    const int ne = (int)(dof[e + 1] - r0);
    if (ne == 0) continue;
    const int64_t a = row_ptr[r0];
    const int64_t L = row_ptr[r0 + 1] - a;
    const bool staged = L <= SPMV_MAXL;
    if (staged) {
      for (int p = lane; p < L; p += 32) xs[w][p] = x[col_idx[a + p]];
      __syncwarp();
    }
    // four rows at a time: independent accumulators keep the loads in flight
    int r = 0;
    for (; r + 4 <= ne; r += 4) {
      if (staged) spmv_rows<4, true>(vals + a + (int64_t)r * L, L, xs[w], col_idx + a, x, y + r0 + r, lane);
      else spmv_rows<4, false>(vals + a + (int64_t)r * L, L, xs[w], col_idx + a, x, y + r0 + r, lane);
    }
    for (; r < ne; ++r) {
      if (staged) spmv_rows<1, true>(vals + a + (int64_t)r * L, L, xs[w], col_idx + a, x, y + r0 + r, lane);
      else spmv_rows<1, false>(vals + a + (int64_t)r * L, L, xs[w], col_idx + a, x, y + r0 + r, lane);
    }
    __syncwarp();
  }
  (void)flags;
}

// extract the diagonal block of every element and invert it in place
__global__ void block_inverse(const int64_t* dof, int64_t nel, const int64_t* row_ptr, const int64_t* col_idx,
                              const double* vals, const int64_t* inv_off, double* inv, int maxn, uint32_t* flags) {
  extern __shared__ double sm[];
  double* A = sm;                                   // [maxn][maxn]
  int* piv = reinterpret_cast<int*>(A + (size_t)maxn * maxn);
  const int lane = threadIdx.x;
  for (int64_t e = blockIdx.x; e < nel; e += gridDim.x) {
    const int64_t r0 = dof[e];
    const int n = (int)(dof[e + 1] - r0);
    if (n == 0) continue;
    const int64_t a = row_ptr[r0];
    const int L = (int)(row_ptr[r0 + 1] - a);
    // position of the self block in the element's column list
    int cs = -1;
    for (int p = lane; p < L; p += 32)
      if (col_idx[a + p] == r0) cs = p;
    for (int o = 16; o > 0; o >>= 1) cs = max(cs, __shfl_xor_sync(0xffffffffu, cs, o));
    if (cs < 0) {
      if (lane == 0) atomicOr(flags, 2u);
      continue;
    }
    for (int i = 0; i < n; ++i)
      for (int j = lane; j < n; j += 32) A[i * n + j] = vals[a + (int64_t)i * L + cs + j];
    __syncwarp();
    bool singular = false;
    for (int k = 0; k < n; ++k) {
      // pivot: argmax |A[i][k]|, i >= k (ties -> lowest row, like LAPACK's idamax)
      double best = -1.0;
      int bi = k;
      for (int i = k + lane; i < n; i += 32) {
        const double v = fabs(A[i * n + k]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (!(best > 0.0)) {
        singular = true;
        break;
      }
      if (lane == 0) piv[k] = bi;
      if (bi != k)
        for (int j = lane; j < n; j += 32) {
          const double t = A[k * n + j];
          A[k * n + j] = A[bi * n + j];
          A[bi * n + j] = t;
        }
      __syncwarp();
      const double d = 1.0 / A[k * n + k];
      __syncwarp();
      for (int j = lane; j < n; j += 32) A[k * n + j] = (j == k ? 1.0 : A[k * n + j]) * d;
      __syncwarp();
      for (int i = 0; i < n; ++i) {
        if (i == k) continue;
        const double f = A[i * n + k];
        __syncwarp();
        for (int j = lane; j < n; j += 32) A[i * n + j] = (j == k ? 0.0 : A[i * n + j]) - f * A[k * n + j];
        __syncwarp();
      }
    }
    if (singular) {
      if (lane == 0) atomicOr(flags, 4u);
      continue;
    }
    __syncwarp();
    for (int k = n - 1; k >= 0; --k) {
      const int p = piv[k];
      if (p != k)
        for (int i = lane; i < n; i += 32) {
          const double t = A[i * n + k];
          A[i * n + k] = A[i * n + p];
          A[i * n + p] = t;
        }
      __syncwarp();
    }
    double* o = inv + inv_off[e];
    for (int q = lane; q < n * n; q += 32) o[q] = A[q];
    __syncwarp();
  }
}

__global__ void block_apply(const int64_t* dof, int64_t nel, const int64_t* inv_off, const double* inv,
                            const double* r, double* z) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < nel; e += nw) {
    const int64_t r0 = dof[e];
    const int n = (int)(dof[e + 1] - r0);
    const double* B = inv + inv_off[e];
    for (int i = lane; i < n; i += 32) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += B[i * n + j] * r[r0 + j];
      z[r0 + i] = s;
    }
  }
}

}  // namespace
}  // namespace pdg

using namespace pdg;

extern "C" int pdg_spmv_blocked(const int64_t* dof_offset, int64_t n_elements, const int64_t* row_ptr,
                                const int64_t* col_idx, const double* values, const double* x, double* y,
                                uint32_t* err_flags, pdg_stream stream) {
  PDG_TRY {
    if (!dof_offset || !row_ptr || !col_idx || !values || !x || !y) return fail(PDG_ERR_INVALID, "null argument");
    if (n_elements <= 0) return PDG_OK;
    spmv_blocked<<<grid_for_warps(n_elements, 32 * SPMV_WARPS), 32 * SPMV_WARPS, 0, (cudaStream_t)stream>>>(
        dof_offset, n_elements, row_ptr, col_idx, values, x, y, err_flags);
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_block_jacobi_setup(const int64_t* dof_offset, int64_t n_elements, int32_t max_block,
                                      const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                                      const int64_t* inv_offset, double* inverses, uint32_t* err_flags,
                                      pdg_stream stream) {
  PDG_TRY {
    if (!dof_offset || !row_ptr || !col_idx || !values || !inv_offset || !inverses)
      return fail(PDG_ERR_INVALID, "null argument");
    if (n_elements <= 0) return PDG_OK;
    if (max_block <= 0 || max_block > 128) return fail(PDG_ERR_UNSUPPORTED, "block size must be 1..128");
    const size_t smem = (size_t)max_block * max_block * 8 + (size_t)max_block * 4;
    PDG_CUDA(cudaFuncSetAttribute(block_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::min<int64_t>(n_elements, (int64_t)num_sms() * 16);
    block_inverse<<<grid, 32, smem, (cudaStream_t)stream>>>(dof_offset, n_elements, row_ptr, col_idx, values,
                                                            inv_offset, inverses, max_block, err_flags);
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_block_jacobi_apply(const int64_t* dof_offset, int64_t n_elements, const int64_t* inv_offset,
                                      const double* inverses, const double* r, double* z, pdg_stream stream) {
  PDG_TRY {
    if (!dof_offset || !inv_offset || !inverses || !r || !z) return fail(PDG_ERR_INVALID, "null argument");
    if (n_elements <= 0) return PDG_OK;
    block_apply<<<grid_for_warps(n_elements, 128), 128, 0, (cudaStream_t)stream>>>(dof_offset, n_elements,
                                                                                    inv_offset, inverses, r, z);
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}
