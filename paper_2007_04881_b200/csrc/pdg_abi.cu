// C-ABI entry points, error state and the unit-level debug kernels.
#include <atomic>
#include <cstring>

#include "assemble_kernel.cuh"

namespace pdg {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
  }
  return sms;
}

cudaError_t launch_assemble_dim2(int P, bool sym, const KArgs& a, const pdg_coeffs& C, cudaStream_t st);
cudaError_t launch_assemble_dim3(int P, bool sym, const KArgs& a, const pdg_coeffs& C, cudaStream_t st);

int check_common(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs) {
  if (!mesh || !basis || !coeffs) return fail(PDG_ERR_INVALID, "null argument");
  if (mesh->dim != 2 && mesh->dim != 3) return fail(PDG_ERR_UNSUPPORTED, "dim must be 2 or 3");
  const int pmax = mesh->dim == 2 ? MAX_P_2D : MAX_P_3D;
  if (basis->max_degree < 0 || basis->max_degree > pmax)
    return fail(PDG_ERR_UNSUPPORTED, "polynomial degree " + std::to_string(basis->max_degree) +
                                         " exceeds the compiled range (" + std::to_string(pmax) + " in " +
                                         std::to_string(mesh->dim) + "D)");
  if (coeffs->n_code > PDG_MAX_CODE || coeffs->n_const > PDG_MAX_CONST)
    return fail(PDG_ERR_INVALID, "coefficient program too large");
  return PDG_OK;
}

bool symmetric_accumulation(const pdg_coeffs& C) {
  if (C.has_advection) return false;
  return C.diffusion_kind != PDG_DIFF_FULL || C.diffusion_symmetric;
}

KArgs make_kargs(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_rules* rules, const pdg_params* params,
                 const pdg_pattern& pat, const pdg_frames* frames, const double* sigma, const int8_t* flow,
                 double* values, int write_cols, double* rhs, uint32_t* flags, int mode) {
  KArgs a;
  std::memset(&a, 0, sizeof(a));
  a.m = *mesh;
  a.B = *basis;
  a.R = *rules;
  a.prm = *params;
  a.pat = pat;
  a.sigma = sigma;
  a.flow = flow;
  a.sframe = frames->simplex;
  a.fframe = frames->facet;
  a.erec = frames->element;
  a.values = values;
  a.rhs = rhs;
  a.flags = flags;
  a.write_cols = write_cols;
  a.mode = mode;
  return a;
}

// ---- unit kernels -------------------------------------------------------------

template <int DIM>
__global__ void map_simplices_kernel(const pdg_mesh m, const pdg_rules R, int order, const int32_t* ids,
                                     int64_t n, double* pts, double* wts, uint32_t* flags) {
  const int r0 = R.vol_offset[order], nq = R.vol_count[order];
  const int64_t total = n * nq;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t si = idx / nq;
    const int k = (int)(idx % nq);
    double v0[3], E[3][3];
    const double det = simplex_frame<DIM>(m, ids[si], v0, E, flags);
    const double* xi = R.points + (int64_t)(r0 + k) * 3;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      double acc = v0[i];
#pragma unroll
      for (int j = 0; j < DIM; ++j) acc += xi[j] * E[j][i];
      pts[idx * DIM + i] = acc;
    }
    wts[idx] = R.weights[r0 + k] * det;
  }
}

template <int DIM, int P>
__global__ void tabulate_kernel(const pdg_basis B, int32_t el, const double* pts, int64_t n, double* vals,
                                double* grads) {
  constexpr int NB = binom(P + DIM, DIM);
  const BoxConst<DIM> bx = box_const<DIM>(B.box + (int64_t)el * 2 * DIM);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double x[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < DIM; ++i) x[i] = pts[q * DIM + i];
    Tab<DIM, P> tb;
    tb.load(bx, x);
#pragma unroll
    for (int f = 0; f < NB; ++f) {
      vals[q * NB + f] = tb.val(f);
#pragma unroll
      for (int k = 0; k < DIM; ++k) grads[(q * DIM + k) * NB + f] = tb.grad(f, k);
    }
  }
}

template <int DIM>
static cudaError_t launch_tabulate(int P, const pdg_basis& B, int32_t el, const double* pts, int64_t n,
                                   double* vals, double* grads, cudaStream_t st) {
  const int grid = grid_for(n, 128);
#define PDG_TAB(PP) \
  case PP: tabulate_kernel<DIM, PP><<<grid, 128, 0, st>>>(B, el, pts, n, vals, grads); note_launch(); break;
  switch (P) {
    PDG_TAB(0) PDG_TAB(1) PDG_TAB(2) PDG_TAB(3) PDG_TAB(4)
    PDG_TAB(5) PDG_TAB(6)
    default: return cudaErrorInvalidValue;
  }
#undef PDG_TAB
  return cudaGetLastError();
}

}  // namespace pdg

using namespace pdg;

static_assert(sizeof(pdg_iface_rec) == 80, "pdg_iface_rec is an 80-byte record");

extern "C" int pdg_abi_version(void) { return PDG_ABI_VERSION; }

extern "C" int64_t pdg_launch_count(void) { return (int64_t)g_launches.load(); }

extern "C" const char* pdg_last_error(void) { return g_last_error.c_str(); }

extern "C" int pdg_host_alloc(size_t bytes, void** out) {
  PDG_TRY {
    if (!out) return fail(PDG_ERR_INVALID, "null argument");
    *out = nullptr;
    if (bytes == 0) return PDG_OK;
    PDG_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_host_free(void* p) {
  PDG_TRY {
    if (p) PDG_CUDA(cudaFreeHost(p));
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_assemble(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                            const pdg_rules* rules, const pdg_params* params, const pdg_pattern* pattern,
                            const pdg_frames* frames, const double* sigma, const int8_t* face_flow,
                            double* values, int32_t write_col_idx, double* rhs, uint32_t* err_flags,
                            pdg_stream stream) {
  PDG_TRY {
    int rc = check_common(mesh, basis, coeffs);
    if (rc) return rc;
    if (!rules || !rules->sqrt_weights || !params || !pattern || !frames || !sigma || !face_flow || !values || !rhs)
      return fail(PDG_ERR_INVALID, "null argument");
    if (write_col_idx && !pattern->col_idx) return fail(PDG_ERR_INVALID, "col_idx not allocated");
    if (!pattern->nbr_rec) return fail(PDG_ERR_INVALID, "interface records missing (pdg_iface_records)");
    const KArgs a = make_kargs(mesh, basis, rules, params, *pattern, frames, sigma, face_flow, values,
                               write_col_idx, rhs, err_flags, 0);
    const bool sym = symmetric_accumulation(*coeffs);
    cudaStream_t st = (cudaStream_t)stream;
    PDG_CUDA(mesh->dim == 2 ? launch_assemble_dim2(basis->max_degree, sym, a, *coeffs, st)
                            : launch_assemble_dim3(basis->max_degree, sym, a, *coeffs, st));
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_element_blocks(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                                  const pdg_rules* rules, const pdg_params* params, const pdg_frames* frames,
                                  const int32_t* elements, int64_t n, double* blocks, double* loads,
                                  uint32_t* err_flags, pdg_stream stream) {
  PDG_TRY {
    int rc = check_common(mesh, basis, coeffs);
    if (rc) return rc;
    if (!rules || !rules->sqrt_weights || !params || !frames || !elements || !blocks || !loads)
      return fail(PDG_ERR_INVALID, "null argument");
    pdg_pattern pat;
    std::memset(&pat, 0, sizeof(pat));
    pat.n_row_elements = n;
    pat.row_elements = elements;
    const KArgs a = make_kargs(mesh, basis, rules, params, pat, frames, nullptr, nullptr, blocks, 0, loads,
                               err_flags, 1);
    const bool sym = symmetric_accumulation(*coeffs);
    cudaStream_t st = (cudaStream_t)stream;
    PDG_CUDA(mesh->dim == 2 ? launch_assemble_dim2(basis->max_degree, sym, a, *coeffs, st)
                            : launch_assemble_dim3(basis->max_degree, sym, a, *coeffs, st));
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_map_simplices(const pdg_mesh* mesh, const pdg_rules* rules, int32_t order,
                                 const int32_t* simplex_ids, int64_t n, double* points, double* weights,
                                 uint32_t* err_flags, pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !rules || !simplex_ids || !points || !weights) return fail(PDG_ERR_INVALID, "null argument");
    if (order < 0 || order > rules->max_order) return fail(PDG_ERR_INVALID, "rule order out of table");
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = grid_for(n * 64, 128);
    if (mesh->dim == 2)
      map_simplices_kernel<2><<<grid, 128, 0, st>>>(*mesh, *rules, order, simplex_ids, n, points, weights, err_flags);
    else if (mesh->dim == 3)
      map_simplices_kernel<3><<<grid, 128, 0, st>>>(*mesh, *rules, order, simplex_ids, n, points, weights, err_flags);
    else
      return fail(PDG_ERR_UNSUPPORTED, "dim must be 2 or 3");
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_tabulate(const pdg_mesh* mesh, const pdg_basis* basis, int32_t element, const double* points,
                            int64_t n, double* values, double* grads, pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !basis || !points || !values || !grads) return fail(PDG_ERR_INVALID, "null argument");
    const int pmax = mesh->dim == 2 ? MAX_P_2D : MAX_P_3D;
    if (basis->max_degree < 0 || basis->max_degree > pmax) return fail(PDG_ERR_UNSUPPORTED, "degree out of range");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t err = mesh->dim == 2 ? launch_tabulate<2>(basis->max_degree, *basis, element, points, n, values, grads, st)
                                     : launch_tabulate<3>(basis->max_degree, *basis, element, points, n, values, grads, st);
    PDG_CUDA(err);
    return PDG_OK;
  }
  PDG_CATCH
}
