// Unit-level face kernels and coefficient evaluation (the single-item public
// kernels of polydg assembly.py:1160-1234 and the a_bar input of
// model.py:196-235).
//
// These are the reference's debugging / verification entry points, not the
// assembly path (which is the fused element kernel): one CTA per face item,
// the CTA's threads tabulate one quadrature point each (both traces), then
// every thread owns a set of block entries and sums over the points of the
// sub-facet in point order.  Coefficients are interpreted from the bytecode
// (InterpCoef: sin/cos of fl(k*pi*u) exactly as numpy), so the unit kernels
// evaluate the fields the way the reference does.
#include <cstring>

#include "pdg_internal.cuh"

namespace pdg {

// points per axis of the reference rule of `order` (quadrature.py:69-94):
// Gauss-Jacobi with n = order // 2 + 1 points per axis
static int face_points(int dim, int order) {
  const int n1 = order / 2 + 1;
  return dim == 2 ? n1 : n1 * n1;
}

template <int DIM, int P>
__global__ void __launch_bounds__(128) face_blocks_kernel(const pdg_mesh m, const pdg_basis B,
                                                          const __grid_constant__ pdg_coeffs C, const pdg_rules R,
                                                          const pdg_params prm, const pdg_face_item* items,
                                                          int64_t n_items, double* blocks, double* loads,
                                                          uint32_t* flags) {
  constexpr int NB = binom(P + DIM, DIM);
  constexpr int NV = 4 * NB + 4;  // per point: w, wbn, g, gN | Vo, Fo, Vn, Fn
  extern __shared__ double sm[];
  const InterpCoef<DIM> cf(C);
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const pdg_face_item item = items[it];
    const int f = item.face;
    const int own = m.face_owner[f], nbr = m.face_neighbor[f];
    const bool interior = item.kind == PDG_UNIT_INTERIOR;
    const int po = B.degree[own], pn = interior ? B.degree[nbr] : po;
    const int no = (int)(B.dof_offset[own + 1] - B.dof_offset[own]);
    const int nn = interior ? (int)(B.dof_offset[nbr + 1] - B.dof_offset[nbr]) : 0;
    const int order = 2 * (po > pn ? po : pn) + prm.quad_increment;
    const int r0 = R.face_offset[order], nq = R.face_count[order];
    double* blk = blocks + it * 4 * NB * NB;
    double* ld = loads + it * NB;
    for (int k = threadIdx.x; k < 4 * NB * NB; k += blockDim.x) blk[k] = 0.0;
    for (int k = threadIdx.x; k < NB; k += blockDim.x) ld[k] = 0.0;
    if (r0 < 0 || nq <= 0) {
      if (threadIdx.x == 0) raise_flag(flags, PDG_FLAG_STACK);
      continue;
    }
    double nrm[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)f * DIM + i];
    const bool flux_on = cf.diff_kind() != PDG_DIFF_NONE && prm.include_gradient_terms;
    const double sigma = item.sigma;
    const BoxConst<DIM> bo = box_const<DIM>(B.box + (int64_t)own * 2 * DIM);
    BoxConst<DIM> bn = bo;
    if (interior) bn = box_const<DIM>(B.box + (int64_t)nbr * 2 * DIM);
    __syncthreads();
    for (int64_t row = m.face_ptr[f]; row < m.face_ptr[f + 1]; ++row) {
      // -- tabulate: thread q owns point q of this sub-facet
      for (int q = threadIdx.x; q < nq; q += blockDim.x) {
        double v0[3], E[3][3], x[3] = {0, 0, 0}, xi[3];
        const double meas = facet_frame<DIM>(m, row, v0, E, flags);
        const double* rp = R.points + (int64_t)(r0 + q) * 3;
#pragma unroll
        for (int j = 0; j < DIM - 1; ++j) xi[j] = rp[j];
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < DIM - 1; ++j) acc += xi[j] * E[j][i];
          x[i] = v0[i] + acc;
        }
        double* s = sm + q * NV;
        const double w = R.weights[r0 + q] * meas;
        s[0] = w;
        double bnv = 0.0;
        if (cf.has_adv()) {
#pragma unroll
          for (int i = 0; i < DIM; ++i) bnv += cf.b_i(i, x) * nrm[i];
        }
        s[1] = w * bnv;
        s[2] = cf.has_dir() ? cf.gD(x) : 0.0;
        s[3] = cf.has_neu() ? cf.gN(x) : 0.0;
        // flux weights: F = n . (A grad phi) = sum_e (sum_d n_d A_de) d_e phi
        double an[3] = {0, 0, 0};
        if (flux_on) {
          if (cf.diff_kind() == PDG_DIFF_ISO) {
            const double a = cf.a_iso(x);
#pragma unroll
            for (int e = 0; e < DIM; ++e) an[e] = a * nrm[e];
          } else {
#pragma unroll
            for (int e = 0; e < DIM; ++e) {
              double acc = 0.0;
#pragma unroll
              for (int d = 0; d < DIM; ++d) acc += nrm[d] * cf.a_ij(d, e, x);
              an[e] = acc;
            }
          }
        }
        for (int side = 0; side < (interior ? 2 : 1); ++side) {
          Tab<DIM, P> tb;
          tb.load(side ? bn : bo, x);
          double* V = s + 4 + side * 2 * NB;
          double* F = V + NB;
#pragma unroll
          for (int fn = 0; fn < NB; ++fn) {
            V[fn] = tb.val(fn);
            double fl = 0.0;
#pragma unroll
            for (int e = 0; e < DIM; ++e) fl += an[e] * tb.grad(fn, e);
            F[fn] = fl;
          }
        }
      }
      __syncthreads();
      // -- blocks: entry (a, b, i, j), rows = test function i of side a
      const int nsides = interior ? 2 : 1;
      const int total = nsides * nsides * NB * NB;
      for (int k = threadIdx.x; k < total; k += blockDim.x) {
        const int ab = k / (NB * NB), ij = k % (NB * NB);
        const int a = ab / nsides, b = ab % nsides, i = ij / NB, j = ij % NB;
        const int na = a ? nn : no, nbb = b ? nn : no;
        if (i >= na || j >= nbb) continue;
        const double sa = a ? -1.0 : 1.0, sb = b ? -1.0 : 1.0;
        double acc = 0.0;
        for (int q = 0; q < nq; ++q) {
          const double* s = sm + q * NV;
          const double w = s[0], wbn = s[1];
          const double* Va = s + 4 + a * 2 * NB;
          const double* Fa = Va + NB;
          const double* Vb = s + 4 + b * 2 * NB;
          const double* Fb = Vb + NB;
          double t = 0.0;
          if (interior) {
            if (flux_on) {
              t -= 0.5 * sa * (w * Fb[j] * Va[i]);
              t -= 0.5 * sb * (w * Vb[j] * Fa[i]);
            }
            if (sigma != 0.0) t += sigma * sa * sb * (w * Vb[j] * Va[i]);
            if (cf.has_adv()) {
              if (item.upwind == 0 && a == 0) t += (b == 0 ? -1.0 : 1.0) * (wbn * Vb[j] * Va[i]);
              if (item.upwind == 1 && a == 1) t += (b == 1 ? 1.0 : -1.0) * (wbn * Vb[j] * Va[i]);
            }
          } else if (item.kind == PDG_UNIT_DIRICHLET) {
            if (flux_on) {
              t -= w * Fb[j] * Va[i];
              t -= w * Vb[j] * Fa[i];
            }
            if (sigma != 0.0) t += sigma * (w * Vb[j] * Va[i]);
            if (item.upwind == 1 && cf.has_adv()) t -= wbn * Vb[j] * Va[i];
          } else if (item.kind == PDG_UNIT_INFLOW) {
            t -= wbn * Vb[j] * Va[i];
          }
          acc += t;
        }
        const int slot = (a * 2 + b) * NB * NB + i * NB + j;
        blk[slot] += acc;
      }
      // -- loads (boundary kinds)
      if (!interior) {
        for (int i = threadIdx.x; i < no; i += blockDim.x) {
          double acc = 0.0;
          for (int q = 0; q < nq; ++q) {
            const double* s = sm + q * NV;
            const double w = s[0], wbn = s[1], g = s[2], gn = s[3];
            const double V = s[4 + i], F = s[4 + NB + i];
            double t = 0.0;
            if (item.kind == PDG_UNIT_DIRICHLET && cf.has_dir()) {
              if (flux_on) t -= F * (w * g);
              if (sigma != 0.0) t += sigma * (V * (w * g));
              if (item.upwind == 1 && cf.has_adv()) t -= V * (wbn * g);
            } else if (item.kind == PDG_UNIT_INFLOW && cf.has_dir()) {
              t -= V * (wbn * g);
            } else if (item.kind == PDG_UNIT_NEUMANN && cf.has_neu()) {
              t += V * (w * gn);
            }
            acc += t;
          }
          ld[i] += acc;
        }
      }
      __syncthreads();
    }
  }
}

// every field at n points: out[n][K] with K = dim*dim (A) + dim (b) + 4 (c, f, gD, gN);
// absent fields give 0 and the A entries of an isotropic a(x) are a on the diagonal
template <int DIM>
__global__ void eval_coeffs_kernel(const __grid_constant__ pdg_coeffs C, const double* pts, int64_t n,
                                   double* out) {
  const InterpCoef<DIM> cf(C);
  constexpr int K = DIM * DIM + DIM + 4;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double x[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < DIM; ++i) x[i] = pts[q * DIM + i];
    double* o = out + q * K;
    for (int i = 0; i < DIM; ++i)
      for (int j = 0; j < DIM; ++j) {
        double v = 0.0;
        if (cf.diff_kind() == PDG_DIFF_ISO) v = i == j ? cf.a_iso(x) : 0.0;
        else if (cf.diff_kind() == PDG_DIFF_FULL) v = cf.a_ij(i, j, x);
        o[i * DIM + j] = v;
      }
    for (int i = 0; i < DIM; ++i) o[DIM * DIM + i] = cf.has_adv() ? cf.b_i(i, x) : 0.0;
    o[DIM * DIM + DIM + 0] = cf.has_reac() ? cf.c(x) : 0.0;
    o[DIM * DIM + DIM + 1] = cf.has_src() ? cf.f(x) : 0.0;
    o[DIM * DIM + DIM + 2] = cf.has_dir() ? cf.gD(x) : 0.0;
    o[DIM * DIM + DIM + 3] = cf.has_neu() ? cf.gN(x) : 0.0;
  }
}

template <int DIM, int P>
static cudaError_t launch_face_blocks(const pdg_mesh& m, const pdg_basis& B, const pdg_coeffs& C,
                                      const pdg_rules& R, const pdg_params& prm, const pdg_face_item* items,
                                      int64_t n, double* blocks, double* loads, uint32_t* flags, cudaStream_t st) {
  constexpr int NB = binom(P + DIM, DIM);
  const int nq = face_points(DIM, 2 * P + prm.quad_increment);
  const size_t smem = (size_t)nq * (4 * NB + 4) * sizeof(double);
  auto kern = face_blocks_kernel<DIM, P>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int grid = (int)std::min<int64_t>(n, (int64_t)num_sms() * 8);
  kern<<<grid, 128, smem, st>>>(m, B, C, R, prm, items, n, blocks, loads, flags);
  note_launch();
  return cudaGetLastError();
}

template <int DIM>
static cudaError_t dispatch_face_blocks(int P, const pdg_mesh& m, const pdg_basis& B, const pdg_coeffs& C,
                                        const pdg_rules& R, const pdg_params& prm, const pdg_face_item* items,
                                        int64_t n, double* blocks, double* loads, uint32_t* flags, cudaStream_t st) {
#define PDG_FB(PP) \
  case PP: return launch_face_blocks<DIM, PP>(m, B, C, R, prm, items, n, blocks, loads, flags, st);
  switch (P) {
    PDG_FB(0) PDG_FB(1) PDG_FB(2) PDG_FB(3) PDG_FB(4)
    case 5:
      if constexpr (DIM == 2) return launch_face_blocks<DIM, 5>(m, B, C, R, prm, items, n, blocks, loads, flags, st);
      break;
    case 6:
      if constexpr (DIM == 2) return launch_face_blocks<DIM, 6>(m, B, C, R, prm, items, n, blocks, loads, flags, st);
      break;
    default: break;
  }
#undef PDG_FB
  return cudaErrorInvalidValue;
}

}  // namespace pdg

using namespace pdg;

extern "C" int pdg_face_blocks(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                               const pdg_rules* rules, const pdg_params* params, const pdg_face_item* items,
                               int64_t n, double* blocks, double* loads, uint32_t* err_flags, pdg_stream stream) {
  PDG_TRY {
    int rc = check_common(mesh, basis, coeffs);
    if (rc) return rc;
    if (!rules || !params || !items || !blocks || !loads) return fail(PDG_ERR_INVALID, "null argument");
    if (n <= 0) return PDG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    PDG_CUDA(mesh->dim == 2
                 ? dispatch_face_blocks<2>(basis->max_degree, *mesh, *basis, *coeffs, *rules, *params, items, n,
                                           blocks, loads, err_flags, st)
                 : dispatch_face_blocks<3>(basis->max_degree, *mesh, *basis, *coeffs, *rules, *params, items, n,
                                           blocks, loads, err_flags, st));
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_eval_coeffs(int32_t dim, const pdg_coeffs* coeffs, const double* points, int64_t n,
                               double* out, pdg_stream stream) {
  PDG_TRY {
    if (!coeffs || !points || !out) return fail(PDG_ERR_INVALID, "null argument");
    if (coeffs->n_code > PDG_MAX_CODE || coeffs->n_const > PDG_MAX_CONST)
      return fail(PDG_ERR_INVALID, "coefficient program too large");
    if (n <= 0) return PDG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (dim == 2)
      eval_coeffs_kernel<2><<<grid_for(n, 128), 128, 0, st>>>(*coeffs, points, n, out);
    else if (dim == 3)
      eval_coeffs_kernel<3><<<grid_for(n, 128), 128, 0, st>>>(*coeffs, points, n, out);
    else
      return fail(PDG_ERR_UNSUPPORTED, "dim must be 2 or 3");
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}
