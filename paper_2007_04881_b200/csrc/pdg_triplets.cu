// Approach-1 index phase on the device: triplets -> CSR (polydg
// triplets_to_csr, assembly.py:1002-1031) and load pairs -> RHS.
//
//   keys = row * n_cols + col (uint64; sentinel ~0 for unused stripe slots)
//   1. stable LSD radix sort of (key, value) over the significant key bits
//      (ties keep input order, so duplicates merge in the stripe order, like
//      polydg's argsort(kind="stable") + add.reduceat)
//   2. run-length encode the sorted keys (unique keys + run lengths, sentinels
//      form the last run), exclusive scan of the lengths -> run offsets, and
//      each run summed by one thread in numpy's order: np.add.reduceat gives
//      a[0] + pairwise_sum(a[1:]) (8 accumulators up to 128 entries, halving
//      above), so the merged values are bit-identical to polydg's
//   3. row_ptr[r] = lower_bound(unique keys, r * n_cols) (one thread per row)
//      col_idx = key % n_cols
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include "pdg_internal.cuh"

namespace pdg {

namespace {

struct Ws {
  uint64_t* keys_alt;
  double* vals_alt;
  uint64_t* ukeys;
  double* usums;
  int64_t* run_off;  // run lengths, then (scanned in place of run_len) offsets
  int64_t* run_len;
  int64_t* nruns;
  void* temp;
  size_t temp_bytes;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t cub_temp_bytes(int64_t n) {
  size_t sort_b = 0, rle_b = 0, scan_b = 0;
  cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<double> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, kb, vb, (int64_t)n, 0, 64);
  cub::DeviceRunLengthEncode::Encode(nullptr, rle_b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                     (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n);
  return std::max(sort_b, std::max(rle_b, scan_b));
}

Ws carve(void* base, int64_t n) {
  Ws w;
  char* p = static_cast<char*>(base);
  const size_t nk = align256((size_t)n * 8);
  w.keys_alt = reinterpret_cast<uint64_t*>(p);
  p += nk;
  w.vals_alt = reinterpret_cast<double*>(p);
  p += nk;
  w.ukeys = reinterpret_cast<uint64_t*>(p);
  p += nk;
  w.usums = reinterpret_cast<double*>(p);
  p += nk;
  w.run_len = reinterpret_cast<int64_t*>(p);
  p += nk;
  w.run_off = reinterpret_cast<int64_t*>(p);
  p += nk;
  w.nruns = reinterpret_cast<int64_t*>(p);
  p += 256;
  w.temp = p;
  w.temp_bytes = cub_temp_bytes(n);
  return w;
}

int key_bits(uint64_t max_key) {
  int b = 1;
  while (b < 64 && (max_key >> b)) ++b;
  return b;
}

// sentinel keys are ~0: with a partial bit range they would sort as their low
// bits, so they are first mapped to the largest in-range key + 1
__global__ void clamp_sentinels(const uint64_t* in, uint64_t* out, int64_t n, uint64_t lim) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] > lim ? lim : in[i];
}

// numpy's pairwise_sum (loops_utils.h): < 8 entries sequentially from 0.,
// <= 128 with 8 interleaved accumulators, else split at a multiple of 8
__device__ __noinline__ double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

// one thread per run: np.add.reduceat's value a[0] + pairwise_sum(a[1:])
__global__ void sum_runs(const double* vs, const int64_t* run_off, const int64_t* run_len, const int64_t* nruns,
                         double* out) {
  const int64_t nu = *nruns;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (int64_t)gridDim.x * blockDim.x) {
    const double* a = vs + run_off[i];
    const int64_t n = run_len[i];
    out[i] = n > 1 ? a[0] + np_pairwise(a + 1, n - 1) : a[0];
  }
}

__global__ void csr_rows(const uint64_t* ukeys, const int64_t* nruns, uint64_t lim, int64_t n_rows, int64_t n_cols,
                         int64_t* row_ptr, int64_t* col_idx, int64_t* nnz_out) {
  int64_t nu = *nruns;
  if (nu > 0 && ukeys[nu - 1] == lim) --nu;  // the sentinel run
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n_rows; r += stride) {
    const uint64_t key = (uint64_t)r * (uint64_t)n_cols;
    int64_t lo = 0, hi = nu;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    row_ptr[r] = lo;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += stride)
    col_idx[i] = (int64_t)(ukeys[i] % (uint64_t)n_cols);
  if (blockIdx.x == 0 && threadIdx.x == 0 && nnz_out) *nnz_out = nu;
}

__global__ void scatter_vector(const uint64_t* ukeys, const double* usums, const int64_t* nruns, uint64_t lim,
                               double* out, int64_t n_rows) {
  const int64_t nu = *nruns;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (int64_t)gridDim.x * blockDim.x)
    if (ukeys[i] < lim && (int64_t)ukeys[i] < n_rows) out[ukeys[i]] = usums[i];
}

// sort + reduce; returns the workspace view (unique keys / sums / run count filled)
// unique keys + numpy-order run sums of the sorted (ks, vs) into (ukeys, sums)
int merge_runs(const uint64_t* ks, const double* vs, int64_t n, Ws& w, uint64_t* ukeys, double* sums,
               cudaStream_t st) {
  size_t tb = w.temp_bytes;
  PDG_CUDA(cub::DeviceRunLengthEncode::Encode(w.temp, tb, ks, ukeys, w.run_len, w.nruns, n, st));
  note_launch();
  tb = w.temp_bytes;
  PDG_CUDA(cub::DeviceScan::ExclusiveSum(w.temp, tb, w.run_len, w.run_off, n, st));
  note_launch();
  sum_runs<<<grid_for(n, 256), 256, 0, st>>>(vs, w.run_off, w.run_len, w.nruns, sums);
  note_launch();
  PDG_CUDA(cudaGetLastError());
  return PDG_OK;
}

int sort_reduce(const uint64_t* keys, const double* vals, int64_t n, uint64_t lim, void* ws, size_t ws_bytes,
                cudaStream_t st, Ws& w, uint64_t** ksorted, double** vsorted) {
  w = carve(ws, n);
  const size_t need = align256((size_t)n * 8) * 6 + 256 + w.temp_bytes;
  if (ws_bytes < need) return fail(PDG_ERR_INVALID, "triplet workspace too small (pdg_triplets_workspace_bytes)");
  // sorted keys land in ukeys (as the DoubleBuffer's first buffer), values in usums
  uint64_t* k0 = w.ukeys;
  double* v0 = w.usums;
  clamp_sentinels<<<grid_for(n, 256), 256, 0, st>>>(keys, k0, n, lim);
  note_launch();
  PDG_CUDA(cudaMemcpyAsync(v0, vals, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
  cub::DoubleBuffer<uint64_t> kb(k0, w.keys_alt);
  cub::DoubleBuffer<double> vb(v0, w.vals_alt);
  size_t tb = w.temp_bytes;
  PDG_CUDA(cub::DeviceRadixSort::SortPairs(w.temp, tb, kb, vb, n, 0, key_bits(lim), st));
  note_launch();
  *ksorted = kb.Current();
  *vsorted = vb.Current();
  return PDG_OK;
}

}  // namespace
}  // namespace pdg

using namespace pdg;

extern "C" size_t pdg_triplets_workspace_bytes(int64_t n_triplets) {
  const int64_t n = std::max<int64_t>(n_triplets, 1);
  return align256((size_t)n * 8) * 6 + 256 + cub_temp_bytes(n) + 256;
}

extern "C" int pdg_triplets_to_csr(const uint64_t* keys, const double* vals, int64_t n_triplets, int64_t n_rows,
                                   int64_t n_cols, int64_t* row_ptr, int64_t* col_idx, double* values,
                                   int64_t* nnz_device, void* workspace, size_t workspace_bytes, pdg_stream stream) {
  PDG_TRY {
    if (!keys || !vals || !row_ptr || !col_idx || !values || !workspace) return fail(PDG_ERR_INVALID, "null argument");
    if (n_rows <= 0 || n_cols <= 0) return fail(PDG_ERR_INVALID, "empty matrix shape");
    cudaStream_t st = (cudaStream_t)stream;
    if (n_triplets <= 0) {
      PDG_CUDA(cudaMemsetAsync(row_ptr, 0, (size_t)(n_rows + 1) * 8, st));
      if (nnz_device) PDG_CUDA(cudaMemsetAsync(nnz_device, 0, 8, st));
      return PDG_OK;
    }
    const uint64_t lim = (uint64_t)n_rows * (uint64_t)n_cols;  // first out-of-range key
    Ws w;
    uint64_t* ks;
    double* vs;
    int rc = sort_reduce(keys, vals, n_triplets, lim, workspace, workspace_bytes, st, w, &ks, &vs);
    if (rc) return rc;
    // reduce-by-key into the outputs (values / a key scratch that reuses the other buffer)
    uint64_t* ukeys = ks == w.ukeys ? w.keys_alt : w.ukeys;
    rc = merge_runs(ks, vs, n_triplets, w, ukeys, values, st);
    if (rc) return rc;
    csr_rows<<<grid_for(n_rows + 1, 256), 256, 0, st>>>(ukeys, w.nruns, lim, n_rows, n_cols, row_ptr, col_idx,
                                                        nnz_device);
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_triplets_to_vector(const uint64_t* keys, const double* vals, int64_t n, int64_t n_rows,
                                      double* out, void* workspace, size_t workspace_bytes, pdg_stream stream) {
  PDG_TRY {
    if (!keys || !vals || !out || !workspace) return fail(PDG_ERR_INVALID, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    PDG_CUDA(cudaMemsetAsync(out, 0, (size_t)std::max<int64_t>(n_rows, 0) * 8, st));
    if (n <= 0 || n_rows <= 0) return PDG_OK;
    const uint64_t lim = (uint64_t)n_rows;
    Ws w;
    uint64_t* ks;
    double* vs;
    int rc = sort_reduce(keys, vals, n, lim, workspace, workspace_bytes, st, w, &ks, &vs);
    if (rc) return rc;
    uint64_t* ukeys = ks == w.ukeys ? w.keys_alt : w.ukeys;
    double* usums = vs == w.usums ? w.vals_alt : w.usums;
    rc = merge_runs(ks, vs, n, w, ukeys, usums, st);
    if (rc) return rc;
    scatter_vector<<<grid_for(n_rows, 256), 256, 0, st>>>(ukeys, usums, w.nruns, lim, out, n_rows);
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}
