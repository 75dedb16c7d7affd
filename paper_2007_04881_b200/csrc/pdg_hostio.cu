// Host side of the returned CSR: the column indices cross the link once per
// element instead of once per row.
//
// Every row of an element's block row holds the same column list (its
// neighbours' DoF spans in ascending order, assembly.py:316-324), so a
// device->host transfer of col_idx moves ne identical copies of it.
// pdg_pack_block_cols gathers the first row of every element into a packed
// list (sum over elements of the row length: 1/ne of col_idx); the host
// expands it back into every row with pdg_expand_block_cols (host threads,
// writing the caller's col_idx array).  The expanded array is identical to
// the device col_idx.
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include "pdg_internal.cuh"

// one row's columns with non-temporal stores: the destination (tens of GB)
// is written once, so bypassing the cache saves the read-for-ownership
static inline void copy_row(int64_t* dst, const int64_t* src, int64_t L) {
#if defined(__x86_64__)
  int64_t j = 0;
  if (L > 0 && ((uintptr_t)dst & 15)) {
    _mm_stream_si64(reinterpret_cast<long long*>(dst), src[0]);
    j = 1;
  }
  for (; j + 2 <= L; j += 2)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + j), _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + j)));
  if (j < L) _mm_stream_si64(reinterpret_cast<long long*>(dst + j), src[j]);
#else
  for (int64_t j = 0; j < L; ++j) dst[j] = src[j];
#endif
}

namespace pdg {

// one warp per element: packed[poff[k] + j] = col_idx[val_off[k] + j], j < row_len[k]
__global__ void __launch_bounds__(256) pack_block_cols_kernel(const int64_t* __restrict__ col_idx,
                                                              const int64_t* __restrict__ val_off,
                                                              const int64_t* __restrict__ row_len,
                                                              const int64_t* __restrict__ poff, int64_t n,
                                                              int64_t* __restrict__ packed) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n; k += nw) {
    const int64_t L = row_len[k];
    const int64_t* src = col_idx + val_off[k];
    int64_t* dst = packed + poff[k];
    for (int64_t j = lane; j < L; j += 32) dst[j] = src[j];
  }
}

}  // namespace pdg

using namespace pdg;

extern "C" int pdg_pack_block_cols(const int64_t* col_idx, const int64_t* elem_val_offset, const int64_t* row_len,
                                   const int64_t* pack_offset, int64_t n_row_elements, int64_t* packed,
                                   pdg_stream stream) {
  PDG_TRY {
    if (n_row_elements < 0) return fail(PDG_ERR_INVALID, "negative element count");
    if (n_row_elements == 0) return PDG_OK;
    if (!col_idx || !elem_val_offset || !row_len || !pack_offset || !packed)
      return fail(PDG_ERR_INVALID, "null argument");
    const int threads = 256;
    pack_block_cols_kernel<<<grid_for_warps(n_row_elements, threads), threads, 0, (cudaStream_t)stream>>>(
        col_idx, elem_val_offset, row_len, pack_offset, n_row_elements, packed);
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_expand_block_cols(int64_t n_row_elements, const int64_t* elem_row_offset, const int64_t* row_ptr,
                                     const int64_t* packed, int64_t* col_idx, int32_t n_threads) {
  PDG_TRY {
    if (n_row_elements < 0) return fail(PDG_ERR_INVALID, "negative element count");
    if (n_row_elements == 0) return PDG_OK;
    if (!elem_row_offset || !row_ptr || !packed || !col_idx) return fail(PDG_ERR_INVALID, "null argument");
    const int64_t n = n_row_elements;
    // packed offsets: exclusive prefix of the first-row lengths
    std::vector<int64_t> poff(n + 1);
    poff[0] = 0;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t r0 = elem_row_offset[k];
      poff[k + 1] = poff[k] + (row_ptr[r0 + 1] - row_ptr[r0]);
    }
    const int nt = std::max(1, std::min<int>(n_threads, 64));
    // element ranges of equal output size (values written ~ row_ptr span)
    const int64_t total = row_ptr[elem_row_offset[n]] - row_ptr[elem_row_offset[0]];
    std::vector<int64_t> cut(nt + 1, n);
    cut[0] = 0;
    {
      int t = 1;
      for (int64_t k = 0; k < n && t < nt; ++k) {
        const int64_t done = row_ptr[elem_row_offset[k]] - row_ptr[elem_row_offset[0]];
        while (t < nt && done >= total * t / nt) cut[t++] = k;
      }
      for (; t < nt; ++t) cut[t] = n;
    }
    auto work = [&](int64_t a, int64_t b) {
      for (int64_t k = a; k < b; ++k) {
        const int64_t* src = packed + poff[k];
        const int64_t L = poff[k + 1] - poff[k];
        for (int64_t r = elem_row_offset[k]; r < elem_row_offset[k + 1]; ++r) copy_row(col_idx + row_ptr[r], src, L);
      }
#if defined(__x86_64__)
      _mm_sfence();  // the streaming stores are visible before the join
#endif
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, cut[t], cut[t + 1]);
    work(cut[0], cut[1]);
    for (auto& th : pool) th.join();
    return PDG_OK;
  }
  PDG_CATCH
}
