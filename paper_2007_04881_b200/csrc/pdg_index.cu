// Index phase on the device: adjacency lists and the block CSR skeleton.
//
// Replaces polydg _pattern_from_adjacency (assembly.py:290-340) -- a Python
// loop over elements building sets, sorted arrays and np.tile'd column lists
// -- with integer kernels.  HBM-bound integer work: coalesced, grid sized in
// multiples of the SM count, one thread (or warp) per element.
#include "pdg_internal.cuh"

namespace pdg {

// ---- device-wide exclusive scan of int64 counts (reduce-then-scan) --------
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < SCAN_THREADS / 32) warp_sums[lane] = w;
  }
  __syncthreads();
  const int64_t before = (wid > 0 ? warp_sums[wid - 1] : 0) + x - v;
  if (total) *total = warp_sums[SCAN_THREADS / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void scan_tile_sums(const int64_t* in, int64_t n, int64_t* tile_sums) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    const int64_t k = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
    if (k < n) s += in[k];
  }
  int64_t tot;
  block_exclusive_scan(s, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// single block: exclusive scan of the tile sums in place (loops over chunks)
__global__ void scan_tile_offsets(int64_t* tile_sums, int64_t ntiles) {
  int64_t carry = 0;
  for (int64_t base = 0; base < ntiles; base += SCAN_THREADS) {
    const int64_t k = base + threadIdx.x;
    const int64_t v = k < ntiles ? tile_sums[k] : 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan(v, &tot);
    if (k < ntiles) tile_sums[k] = carry + ex;
    carry += tot;
  }
}

// out[k] = exclusive prefix of in (out has n+1 entries; out[n] = total).
__global__ void scan_apply(const int64_t* in, int64_t n, const int64_t* tile_off, int64_t* out) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t loc[SCAN_ITEMS];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    const int64_t k = base + i;
    loc[i] = k < n ? in[k] : 0;
    s += loc[i];
  }
  int64_t tot;
  int64_t ex = block_exclusive_scan(s, &tot) + tile_off[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    const int64_t k = base + i;
    if (k < n) out[k] = ex;
    if (k == n - 1) out[n] = ex + loc[i];
    ex += loc[i];
  }
  if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

size_t scan_workspace_bytes(int64_t n) {
  const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE + 1;
  return (size_t)tiles * sizeof(int64_t);
}

// scan_tile_sums reads in[] tile by tile with stride SCAN_THREADS; scan_apply
// reads contiguous runs per thread -- both see every element once, and the
// tile sums are identical because a tile covers the same index range.
cudaError_t exclusive_scan(const int64_t* in, int64_t n, int64_t* out, int64_t* ws,
                           cudaStream_t st) {
  const int64_t tiles = n > 0 ? (n + SCAN_TILE - 1) / SCAN_TILE : 1;
  if (n > 0) { scan_tile_sums<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, n, ws); note_launch(); }
  else cudaMemsetAsync(ws, 0, sizeof(int64_t), st);
  scan_tile_offsets<<<1, SCAN_THREADS, 0, st>>>(ws, tiles); note_launch();
  scan_apply<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, n, ws, out); note_launch();
  return cudaGetLastError();
}

// ---- adjacency ----------------------------------------------------------------

__global__ void adj_count(const pdg_mesh m, int64_t* count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m.n_elements; e += stride)
    count[e] = 1;  // self
}

__global__ void adj_count_ifaces(const pdg_mesh m, int64_t* count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m.n_interfaces; i += stride) {
    atomicAdd((unsigned long long*)&count[m.iface_owner[i]], 1ull);
    atomicAdd((unsigned long long*)&count[m.iface_neighbor[i]], 1ull);
  }
}

__global__ void adj_fill_self(const pdg_mesh m, const int64_t* ptr, int32_t* elem, int32_t* ifc,
                              int64_t* cursor) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m.n_elements; e += stride) {
    elem[ptr[e]] = (int32_t)e;
    ifc[ptr[e]] = -1;
    cursor[e] = ptr[e] + 1;
  }
}

__global__ void adj_fill_ifaces(const pdg_mesh m, int32_t* elem, int32_t* ifc, int64_t* cursor) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m.n_interfaces; i += stride) {
    const int32_t a = m.iface_owner[i], b = m.iface_neighbor[i];
    const int64_t pa = (int64_t)atomicAdd((unsigned long long*)&cursor[a], 1ull);
    const int64_t pb = (int64_t)atomicAdd((unsigned long long*)&cursor[b], 1ull);
    elem[pa] = b; ifc[pa] = (int32_t)i;
    elem[pb] = a; ifc[pb] = (int32_t)i;
  }
}

// insertion sort of each (short) neighbour segment by element id: the atomic
// fill order is arbitrary, the sorted result is unique (ids are distinct).
// Segments up to ADJ_REG entries are sorted in registers (fully unrolled
// compare-exchange passes, one global read + one write per entry); longer
// ones fall back to the in-place insertion sort.
constexpr int ADJ_REG = 16;
__global__ void adj_sort(const pdg_mesh m, const int64_t* ptr, int32_t* elem, int32_t* ifc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m.n_elements; e += stride) {
    const int64_t a = ptr[e], b = ptr[e + 1];
    const int n = (int)(b - a);
    if (n <= ADJ_REG) {
      int32_t ke[ADJ_REG], ki[ADJ_REG];
#pragma unroll
      for (int i = 0; i < ADJ_REG; ++i) {
        ke[i] = i < n ? elem[a + i] : 0x7fffffff;
        ki[i] = i < n ? ifc[a + i] : 0;
      }
      // odd-even transposition sort (ADJ_REG passes, all indices compile time)
#pragma unroll
      for (int pass = 0; pass < ADJ_REG; ++pass) {
#pragma unroll
        for (int i = pass & 1; i + 1 < ADJ_REG; i += 2) {
          const bool sw = ke[i] > ke[i + 1];
          const int32_t k0 = sw ? ke[i + 1] : ke[i], k1 = sw ? ke[i] : ke[i + 1];
          const int32_t i0 = sw ? ki[i + 1] : ki[i], i1 = sw ? ki[i] : ki[i + 1];
          ke[i] = k0;
          ke[i + 1] = k1;
          ki[i] = i0;
          ki[i + 1] = i1;
        }
      }
#pragma unroll
      for (int i = 0; i < ADJ_REG; ++i)
        if (i < n) {
          elem[a + i] = ke[i];
          ifc[a + i] = ki[i];
        }
      continue;
    }
    for (int64_t i = a + 1; i < b; ++i) {
      const int32_t ke = elem[i], ki = ifc[i];
      int64_t j = i - 1;
      while (j >= a && elem[j] > ke) {
        elem[j + 1] = elem[j];
        ifc[j + 1] = ifc[j];
        --j;
      }
      elem[j + 1] = ke;
      ifc[j + 1] = ki;
    }
  }
}

// ---- pattern offsets ----------------------------------------------------------------

__global__ void pattern_counts(const pdg_basis B, const pdg_pattern P, int64_t* vals, int64_t* rows) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < P.n_row_elements; k += stride) {
    const int32_t e = P.row_elements ? P.row_elements[k] : (int32_t)k;
    int64_t L = 0;
    for (int64_t q = P.nbr_ptr[e]; q < P.nbr_ptr[e + 1]; ++q) {
      const int32_t j = P.nbr_elem[q];
      L += B.dof_offset[j + 1] - B.dof_offset[j];
    }
    const int64_t ne = B.dof_offset[e + 1] - B.dof_offset[e];
    P.row_len[k] = L;
    vals[k] = L * ne;
    rows[k] = ne;
  }
}

// row_ptr of the owned rows: one warp per 32 consecutive row elements, lanes
// over the rows of that range (contiguous, coalesced stores), the row's
// element found by a binary search over the 32 staged row offsets.
__global__ void pattern_row_ptr(const pdg_basis B, const pdg_pattern P) {
  __shared__ int64_t sro[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; k0 < P.n_row_elements;
       k0 += nw * 32) {
    const int cnt = (int)(P.n_row_elements - k0 < 32 ? P.n_row_elements - k0 : 32);
    if (lane < cnt) sro[w][lane] = P.elem_row_offset[k0 + lane];
    if (lane == 0) sro[w][cnt] = P.elem_row_offset[k0 + cnt];
    __syncwarp();
    const int64_t R0 = sro[w][0], R1 = sro[w][cnt];
    for (int64_t r = R0 + lane; r < R1; r += 32) {
      int lo = 0, hi = cnt - 1;  // last element with row offset <= r
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sro[w][mid] <= r) lo = mid;
        else hi = mid - 1;
      }
      const int64_t k = k0 + lo;
      P.row_ptr[r] = P.elem_val_offset[k] + (r - sro[w][lo]) * P.row_len[k];
    }
    if (lane == 0 && k0 + cnt == P.n_row_elements) P.row_ptr[R1] = P.elem_val_offset[P.n_row_elements];
    __syncwarp();
  }
}

// one warp per owned element: col_idx rows are the concatenated DoF ranges of
// the sorted neighbours, identical for every row of the element.
__global__ void pattern_fill_cols(const pdg_basis B, const pdg_pattern P) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < P.n_row_elements;
       k += nwarps) {
    const int32_t e = P.row_elements ? P.row_elements[k] : (int32_t)k;
    write_col_rows(B, P, e, P.elem_val_offset[k], P.row_len[k], lane);
  }
}

}  // namespace pdg

using namespace pdg;

extern "C" size_t pdg_workspace_bytes(int64_t n_elements, int64_t n_interfaces) {
  (void)n_interfaces;
  // counts + cursor + two count arrays + scan tiles
  return (size_t)(4 * (n_elements + 1)) * sizeof(int64_t) + 2 * scan_workspace_bytes(n_elements + 1) + 256;
}

extern "C" int pdg_adjacency(const pdg_mesh* mesh, int64_t* nbr_ptr, int32_t* nbr_elem,
                             int32_t* nbr_iface, void* workspace, size_t workspace_bytes,
                             pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !nbr_ptr || !nbr_elem || !nbr_iface) return fail(PDG_ERR_INVALID, "null argument");
    const int64_t nel = mesh->n_elements;
    if (workspace_bytes < pdg_workspace_bytes(nel, mesh->n_interfaces))
      return fail(PDG_ERR_INVALID, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t* count = (int64_t*)workspace;
    int64_t* cursor = count + (nel + 1);
    int64_t* scan_ws = cursor + (nel + 1);
    const int grid = grid_for(nel);
    adj_count<<<grid, 256, 0, st>>>(*mesh, count); note_launch();
    if (mesh->n_interfaces > 0) { adj_count_ifaces<<<grid_for(mesh->n_interfaces), 256, 0, st>>>(*mesh, count); note_launch(); }
    PDG_CUDA(exclusive_scan(count, nel, nbr_ptr, scan_ws, st));
    adj_fill_self<<<grid, 256, 0, st>>>(*mesh, nbr_ptr, nbr_elem, nbr_iface, cursor); note_launch();
    if (mesh->n_interfaces > 0) {
      adj_fill_ifaces<<<grid_for(mesh->n_interfaces), 256, 0, st>>>(*mesh, nbr_elem, nbr_iface, cursor);
      note_launch();
    }
    adj_sort<<<grid, 128, 0, st>>>(*mesh, nbr_ptr, nbr_elem, nbr_iface); note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_pattern_offsets(const pdg_mesh* mesh, const pdg_basis* basis,
                                   pdg_pattern* pattern, int64_t n_local_rows, int64_t* nnz_host,
                                   void* workspace, size_t workspace_bytes, pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !basis || !pattern) return fail(PDG_ERR_INVALID, "null argument");
    const int64_t nr = pattern->n_row_elements;
    if (workspace_bytes < pdg_workspace_bytes(mesh->n_elements, mesh->n_interfaces))
      return fail(PDG_ERR_INVALID, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t* vals = (int64_t*)workspace;
    int64_t* rows = vals + (mesh->n_elements + 1);
    int64_t* scan_ws = rows + (mesh->n_elements + 1);
    pattern_counts<<<grid_for(nr), 256, 0, st>>>(*basis, *pattern, vals, rows); note_launch();
    PDG_CUDA(exclusive_scan(vals, nr, pattern->elem_val_offset, scan_ws, st));
    PDG_CUDA(exclusive_scan(rows, nr, pattern->elem_row_offset, scan_ws, st));
    if (nr > 0) {
      pattern_row_ptr<<<grid_for_warps((nr + 31) / 32, 256), 256, 0, st>>>(*basis, *pattern);
      note_launch();
    }
    else PDG_CUDA(cudaMemsetAsync(pattern->row_ptr, 0, sizeof(int64_t), st));
    PDG_CUDA(cudaGetLastError());
    if (nnz_host) {  // size query: one synchronisation to size col_idx / values
      int64_t tot[2] = {0, 0};
      PDG_CUDA(cudaMemcpyAsync(&tot[0], pattern->elem_val_offset + nr, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
      PDG_CUDA(cudaMemcpyAsync(&tot[1], pattern->elem_row_offset + nr, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
      PDG_CUDA(cudaStreamSynchronize(st));
      if (tot[1] != n_local_rows) return fail(PDG_ERR_INVALID, "n_local_rows does not match the degrees");
      *nnz_host = tot[0];
    }
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_pattern_fill(const pdg_mesh* mesh, const pdg_basis* basis,
                                const pdg_pattern* pattern, pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !basis || !pattern || !pattern->col_idx) return fail(PDG_ERR_INVALID, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nr = pattern->n_row_elements;
    if (nr > 0) { pattern_fill_cols<<<grid_for_warps(nr, 256), 256, 0, st>>>(*basis, *pattern); note_launch(); }
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}
