// Face pre-pass bodies, templated on the coefficient policy: penalty parameter
// and flow side of every face (see pdg_prepass.cu).
//
//  sigma_F = C * max_{k in sides} min(|k| / sup|K^F|, cov_cap) * a_bar_k * p_k^2 * |F| / |k|
//      (polydg model.py:238-257, side data model.py:196-235, MeshGeometry.face_sigma
//       assembly.py:613-626), a_bar_k = max over k's volume quadrature points of
//       n^T A(x) n with the face (owner) normal;
//  flow side: sign of the mean of b.n over the order-2 sample points of the
//      face's sub-facets, straddle check (model.py:118-135,176-191), upwind
//      attribution (assembly.py:596-611).
#pragma once

#include "sipg_device.cuh"

namespace pdg {

// Policy-templated bodies (CF = InterpCoef for the ahead-of-time launch below,
// the NVRTC-generated JitCoef for pdg_face_prepass_jit): n^T A n, the
// per-element max of an isotropic a(x), and the per-face sigma / flow side.
template <int DIM, class CF>
__device__ __forceinline__ double nAn_cf(const CF& cf, const double* n, const double* x) {
  if (cf.diff_kind() == PDG_DIFF_ISO) {
    const double a = cf.a_iso(x);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) s += n[i] * a * n[i];
    return s;
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    double r = 0.0;
#pragma unroll
    for (int j = 0; j < DIM; ++j) r += cf.a_ij(i, j, x) * n[j];
    s += n[i] * r;
  }
  return s;
}

// max over an element's volume quadrature points of a(x) (isotropic a(x) I):
// one warp per element, lanes over points, warp max.
template <int DIM, class CF>
__device__ __forceinline__ void elem_abar_body(const pdg_mesh& m, const pdg_basis& B, const CF& cf,
                                               const pdg_rules& R, const pdg_params& prm, double* abar,
                                               uint32_t* flags) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < m.n_elements; e += nwarps) {
    const int order = 2 * B.degree[e] + prm.quad_increment;
    const int r0 = R.vol_offset[order], nq = R.vol_count[order];
    const int64_t s0 = m.elem_ptr[e];
    const int Q = (int)(m.elem_ptr[e + 1] - s0) * nq;
    const float rnq = 1.0f / (float)nq;
    double best = -PDG_INF;
    for (int g = lane; g < Q; g += 32) {
      const int ls = small_div(g, nq, rnq);
      const int s = m.elem_simplices[s0 + ls];
      const int k = g - ls * nq;
      double v0[3], E[3][3];
      simplex_frame<DIM>(m, s, v0, E, flags);
      double x[3] = {0, 0, 0};
      const double* xi = R.points + (int64_t)(r0 + k) * 3;
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double acc = v0[i];
#pragma unroll
        for (int j = 0; j < DIM; ++j) acc += xi[j] * E[j][i];
        x[i] = acc;
      }
      best = fmax(best, cf.a_iso(x));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) abar[e] = best;
  }
}

template <int DIM, class CF>
__device__ double side_abar_cf(const pdg_mesh& m, const pdg_basis& B, const CF& cf, const pdg_rules& R,
                               const pdg_params& prm, const double* abar_iso, int32_t el, const double* n,
                               uint32_t* flags) {
  if (cf.diff_kind() == PDG_DIFF_NONE) return 0.0;
  double x0[3] = {0, 0, 0};
  if (cf.a_const()) return nAn_cf<DIM>(cf, n, x0);
  if (cf.diff_kind() == PDG_DIFF_ISO) {
    double nn = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) nn += n[i] * n[i];
    return abar_iso[el] * nn;
  }
  // general variable tensor: loop over the element's volume points
  const int order = 2 * B.degree[el] + prm.quad_increment;
  const int r0 = R.vol_offset[order], nq = R.vol_count[order];
  double best = -PDG_INF;
  for (int64_t si = m.elem_ptr[el]; si < m.elem_ptr[el + 1]; ++si) {
    double v0[3], E[3][3];
    simplex_frame<DIM>(m, m.elem_simplices[si], v0, E, flags);
    for (int k = 0; k < nq; ++k) {
      const double* xi = R.points + (int64_t)(r0 + k) * 3;
      double x[3] = {0, 0, 0};
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double acc = v0[i];
#pragma unroll
        for (int j = 0; j < DIM; ++j) acc += xi[j] * E[j][i];
        x[i] = acc;
      }
      best = fmax(best, nAn_cf<DIM>(cf, n, x));
    }
  }
  return best;
}

template <int DIM, class CF>
__device__ __forceinline__ void face_prepass_body(const pdg_mesh& m, const pdg_basis& B, const CF& cf,
                                                  const pdg_rules& R, const pdg_params& prm,
                                                  const double* abar_iso, double* sigma, int8_t* flow,
                                                  uint32_t* flags) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < m.n_faces; f += stride) {
    const int32_t o = m.face_owner[f], nb = m.face_neighbor[f];
    const int tag = m.face_tag[f];
    const bool interior = nb >= 0;
    double n[3] = {0, 0, 0};
#pragma unroll
    for (int i = 0; i < DIM; ++i) n[i] = m.face_normal[f * DIM + i];
    sigma[f] = 0.0;
    flow[f] = interior ? -1 : 0;
    if (!interior && tag == PDG_TAG_INTERIOR) {
      raise_flag(flags, PDG_FLAG_UNCLASSIFIED);
      continue;
    }
    if (!interior && tag != PDG_TAG_DIRICHLET) continue;  // inflow/neumann/outflow need neither

    // -- flow side: order-2 sample points of every sub-facet
    if (cf.has_adv()) {
      const int r0 = R.face_offset[2], nq = R.face_count[2];
      double sum = 0.0, mn = PDG_INF, mx = -PDG_INF, amax = 0.0;
      int cnt = 0;
      for (int64_t row = m.face_ptr[f]; row < m.face_ptr[f + 1]; ++row) {
        double v0[3], E[3][3];
        facet_frame<DIM>(m, row, v0, E, flags);
        for (int k = 0; k < nq; ++k) {
          const double* xi = R.points + (int64_t)(r0 + k) * 3;
          double x[3] = {0, 0, 0};
#pragma unroll
          for (int i = 0; i < DIM; ++i) {
            double acc = v0[i];
#pragma unroll
            for (int j = 0; j < DIM - 1; ++j) acc += xi[j] * E[j][i];
            x[i] = acc;
          }
          double bn = 0.0;
#pragma unroll
          for (int i = 0; i < DIM; ++i) bn += cf.b_i(i, x) * n[i];
          sum += bn;
          mn = fmin(mn, bn);
          mx = fmax(mx, bn);
          amax = fmax(amax, fabs(bn));
          ++cnt;
        }
      }
      const double tol = 1e-10 * fmax(1.0, amax);
      if (mn < -tol && mx > tol) raise_flag(flags, PDG_FLAG_STRADDLE);
      const double mean = sum / cnt;
      if (interior) flow[f] = mean < 0.0 ? 0 : (mean > 0.0 ? 1 : -1);
      else flow[f] = mean < 0.0 ? 1 : 0;
    }

    // -- penalty
    double best = 0.0;
    for (int side = 0; side < (interior ? 2 : 1); ++side) {
      const int32_t el = side == 0 ? o : nb;
      double mxv = -1.0;
      bool any = false;
      for (int64_t row = m.face_ptr[f]; row < m.face_ptr[f + 1]; ++row) {
        const int32_t s = side == 0 ? m.facet_owner_simplex[row] : m.facet_neighbor_simplex[row];
        if (s < 0) continue;
        const double v = m.simplex_volumes[s];
        mxv = any ? fmax(mxv, v) : v;
        any = true;
      }
      if (!any || !(mxv > 0.0)) {
        raise_flag(flags, PDG_FLAG_NO_ADJACENT_SIMPLEX);
        continue;
      }
      const int p = B.degree[el];
      const double vol = m.elem_volumes[el];
      double cap = PDG_INF;
      if (prm.coverable && prm.coverable[el]) {
        double c = 1.0;
        for (int k = 0; k < 2 * (DIM - 1); ++k) c *= (double)p;
        cap = c;
      }
      const double ab = side_abar_cf<DIM>(m, B, cf, R, prm, abar_iso, el, n, flags);
      const double ratio = fmin(vol / mxv, cap);
      best = fmax(best, ratio * ab * (double)(p * p) * m.face_measure[f] / vol);
    }
    sigma[f] = prm.penalty_constant * best;
  }
}

}  // namespace pdg
