// Face pre-pass: penalty parameter and flow side of every face.
//
//  sigma_F = C * max_{k in sides} min(|k| / sup|K^F|, cov_cap) * a_bar_k * p_k^2 * |F| / |k|
//      (polydg model.py:238-257, side data model.py:196-235, MeshGeometry.face_sigma
//       assembly.py:613-626), a_bar_k = max over k's volume quadrature points of
//       n^T A(x) n with the face (owner) normal;
//  flow side: sign of the mean of b.n over the order-2 sample points of the
//      face's sub-facets, straddle check (model.py:118-135,176-191), upwind
//      attribution (assembly.py:596-611).
//
// sigma needs the a_bar of BOTH sides before any face term can be formed, so
// it runs as a separate, cheap launch ahead of the element kernel.
#include "pdg_internal.cuh"
#include "prepass_body.cuh"

namespace pdg {

template <int DIM>
__global__ void elem_abar_iso(const pdg_mesh m, const pdg_basis B, const __grid_constant__ pdg_coeffs C,
                              const pdg_rules R, const pdg_params prm, double* abar, uint32_t* flags) {
  elem_abar_body<DIM>(m, B, InterpCoef<DIM>(C), R, prm, abar, flags);
}

template <int DIM>
__global__ void face_prepass(const pdg_mesh m, const pdg_basis B, const __grid_constant__ pdg_coeffs C,
                             const pdg_rules R, const pdg_params prm, const double* abar_iso,
                             double* sigma, int8_t* flow, uint32_t* flags) {
  face_prepass_body<DIM>(m, B, InterpCoef<DIM>(C), R, prm, abar_iso, sigma, flow, flags);
}

// Interface records (pdg_iface_rec) of the owned rows: one warp per row
// element, lanes over its sorted neighbour list (assembly.py:309-321: column
// start = exclusive prefix of the neighbours' DoF counts, a warp scan),
// flattening per entry the interface's first-face metadata the element
// kernel needs before any face point can be tabulated (face range, side,
// downwind flag, sigma, normal, first sub-facet row, paired-round
// eligibility).  Records are staged in shared memory and written as
// contiguous 16-byte chunks (coalesced; one record = 80 bytes).
template <int DIM>
__global__ void __launch_bounds__(128) iface_records_kernel(const pdg_mesh m, const pdg_basis B, const pdg_rules R,
                                                            int inc, int has_adv, const pdg_pattern P,
                                                            const double* sigma, const int8_t* flow) {
  // 8-lane groups, one row element each (4 per warp): a Voronoi cell has ~7
  // neighbours, so a whole warp per element would leave 3/4 of the lanes idle
  constexpr int GL = 8;
  __shared__ int4 stage[4][32 * 5];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int grp = lane / GL, gl = lane % GL;
  const unsigned gmask = 0xffu << (grp * GL);
  int4* st = stage[wib] + grp * GL * 5;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / GL;
  for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / GL; k < P.n_row_elements; k += ngroups) {
    const int32_t e = P.row_elements ? P.row_elements[k] : (int32_t)k;
    const int pe = B.degree[e];
    const int64_t q0 = P.nbr_ptr[e], q1 = P.nbr_ptr[e + 1];
    int carry = 0;
    for (int64_t c0 = q0; c0 < q1; c0 += GL) {
      const int nv = (int)(q1 - c0 < GL ? q1 - c0 : GL);
      const int64_t q = c0 + gl;
      int j = 0, nj = 0, pj = 0, fa = 0, fb = 0, row0 = 0, info = 0, nrows = 0;
      double sig = 0.0, nrm[3] = {0.0, 0.0, 0.0};
      long long dof = 0;
      if (gl < nv) {
        j = P.nbr_elem[q];
        nj = (int)(B.dof_offset[j + 1] - B.dof_offset[j]);
        dof = P.col_dof ? P.col_dof[j] : B.dof_offset[j];
        pj = B.degree[j];
        if (j != e) {
          const int32_t ifc = P.nbr_iface[q];
          fa = (int)m.iface_ptr[ifc];
          fb = (int)m.iface_ptr[ifc + 1];
          const int side = m.face_owner[fa] == e ? 0 : 1;
          const bool down = has_adv && flow[fa] == side;
          row0 = (int)m.face_ptr[fa];
          nrows = (int)(m.face_ptr[fa + 1] - row0);
          const int nq = R.face_count[2 * max(pe, pj) + inc];
          const bool simple = fb - fa == 1 && nrows == 1 && nq <= 8;
          info = side | (down ? 2 : 0) | (simple ? 4 : 0);
          sig = sigma[fa];
#pragma unroll
          for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)fa * DIM + i];
        }
      }
      // exclusive scan of nj over the group's chunk
      int incl = nj;
#pragma unroll
      for (int o = 1; o < GL; o <<= 1) {
        const int v = __shfl_up_sync(gmask, incl, o, GL);
        if (gl >= o) incl += v;
      }
      const int col = carry + incl - nj;
      carry += __shfl_sync(gmask, incl, GL - 1, GL);
      if (gl < nv) {
        int4* r = st + gl * 5;
        r[0] = make_int4(j, nj, col, pj);
        r[1] = make_int4(fa, fb, row0, info);
        double2* rd = reinterpret_cast<double2*>(r + 2);
        rd[0] = make_double2(sig, nrm[0]);
        rd[1] = make_double2(nrm[1], nrm[2]);
        // first-face row count: read by the 3D element kernel only
        reinterpret_cast<longlong2*>(r + 4)[0] = make_longlong2(dof, DIM == 3 ? (long long)(unsigned)nrows : 0ll);
      }
      __syncwarp(gmask);
      int4* dst = reinterpret_cast<int4*>(P.nbr_rec + c0);
      for (int c = gl; c < nv * 5; c += GL) dst[c] = st[c];
      __syncwarp(gmask);
    }
  }
}

}  // namespace pdg

using namespace pdg;

extern "C" int pdg_iface_records(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                                 const pdg_rules* rules, const pdg_params* params, const pdg_pattern* pattern,
                                 const double* sigma, const int8_t* face_flow, pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !basis || !coeffs || !rules || !params || !pattern || !sigma || !face_flow ||
        !pattern->nbr_ptr || !pattern->nbr_elem || !pattern->nbr_iface || !pattern->nbr_rec)
      return fail(PDG_ERR_INVALID, "null argument");
    if (pattern->n_row_elements <= 0) return PDG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = grid_for_warps((pattern->n_row_elements + 3) / 4, 128);
    if (mesh->dim == 2)
      iface_records_kernel<2><<<grid, 128, 0, st>>>(*mesh, *basis, *rules, params->quad_increment,
                                                    coeffs->has_advection, *pattern, sigma, face_flow);
    else if (mesh->dim == 3)
      iface_records_kernel<3><<<grid, 128, 0, st>>>(*mesh, *basis, *rules, params->quad_increment,
                                                    coeffs->has_advection, *pattern, sigma, face_flow);
    else
      return fail(PDG_ERR_UNSUPPORTED, "dim must be 2 or 3");
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

extern "C" int pdg_face_prepass(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                                const pdg_rules* rules, const pdg_params* params, double* sigma,
                                int8_t* face_flow, double* elem_abar, uint32_t* err_flags,
                                pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !basis || !coeffs || !rules || !params || !sigma || !face_flow)
      return fail(PDG_ERR_INVALID, "null argument");
    if (mesh->dim != 2 && mesh->dim != 3) return fail(PDG_ERR_UNSUPPORTED, "dim must be 2 or 3");
    cudaStream_t st = (cudaStream_t)stream;
    const bool iso_var = coeffs->diffusion_kind == PDG_DIFF_ISO && !coeffs->diffusion[0].is_const;
    if (iso_var && !elem_abar) return fail(PDG_ERR_INVALID, "elem_abar scratch required");
    if (mesh->dim == 2) {
      if (iso_var && mesh->n_elements > 0) {
        elem_abar_iso<2><<<grid_for_warps(mesh->n_elements, 256), 256, 0, st>>>(
            *mesh, *basis, *coeffs, *rules, *params, elem_abar, err_flags);
        note_launch();
      }
      if (mesh->n_faces > 0) {
        face_prepass<2><<<grid_for(mesh->n_faces, 128), 128, 0, st>>>(
            *mesh, *basis, *coeffs, *rules, *params, elem_abar, sigma, face_flow, err_flags);
        note_launch();
      }
    } else {
      if (iso_var && mesh->n_elements > 0) {
        elem_abar_iso<3><<<grid_for_warps(mesh->n_elements, 256), 256, 0, st>>>(
            *mesh, *basis, *coeffs, *rules, *params, elem_abar, err_flags);
        note_launch();
      }
      if (mesh->n_faces > 0) {
        face_prepass<3><<<grid_for(mesh->n_faces, 128), 128, 0, st>>>(
            *mesh, *basis, *coeffs, *rules, *params, elem_abar, sigma, face_flow, err_flags);
        note_launch();
      }
    }
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}

// ---------------------------------------------------------------------------
// geometry pre-pass: affine frames of every simplex (element order), every
// facet, and the basis constants of every element
// ---------------------------------------------------------------------------
namespace pdg {

// Records are assembled per warp in shared memory and written as contiguous
// 16-byte chunks (32 records of W doubles per warp), so every DRAM sector is
// written whole by one instruction stream.
template <int DIM>
__global__ void __launch_bounds__(256) frames_kernel(const pdg_mesh m, const pdg_basis B, const pdg_frames F,
                                                     uint32_t* flags) {
  constexpr int W = DIM == 2 ? 8 : 16;
  __shared__ double stage[8][32 * W];
  const int lane = threadIdx.x & 31;
  double* sw = stage[threadIdx.x >> 5];
  double* o = sw + lane * W;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  auto flush = [&](double* dst, int64_t base, int64_t n) {
    __syncwarp();
    const int nv = (int)(n - base < 32 ? n - base : 32);
    double2* d = reinterpret_cast<double2*>(dst + base * W);
    const double2* src = reinterpret_cast<const double2*>(sw);
    for (int c = lane; c < nv * W / 2; c += 32) d[c] = src[c];
    __syncwarp();
  };
  for (int64_t base = w0 * 32; base < m.n_simplices; base += nwarps * 32) {
    const int64_t i = base + lane;
    if (i < m.n_simplices) {
      double v0[3], E[3][3];
      const double det = simplex_frame<DIM>(m, m.elem_simplices[i], v0, E, flags);
#pragma unroll
      for (int d = 0; d < DIM; ++d) o[d] = v0[d];
#pragma unroll
      for (int k = 0; k < DIM; ++k)
#pragma unroll
        for (int d = 0; d < DIM; ++d) o[DIM + k * DIM + d] = E[k][d];
      o[DIM + DIM * DIM] = det;
      o[DIM + DIM * DIM + 1] = sqrt(det);  // sqrt-weighted volume tables (assemble_body.cuh)
#pragma unroll
      for (int c = DIM + DIM * DIM + 2; c < W; ++c) o[c] = 0.0;
    }
    flush(F.simplex, base, m.n_simplices);
  }
  for (int64_t base = w0 * 32; base < m.n_facets; base += nwarps * 32) {
    const int64_t r = base + lane;
    if (r < m.n_facets) {
      double v0[3], E[3][3];
      const double jac = facet_frame<DIM>(m, r, v0, E, flags);
#pragma unroll
      for (int d = 0; d < DIM; ++d) o[d] = v0[d];
#pragma unroll
      for (int k = 0; k < DIM - 1; ++k)
#pragma unroll
        for (int d = 0; d < DIM; ++d) o[DIM + k * DIM + d] = E[k][d];
      o[DIM + (DIM - 1) * DIM] = jac;
#pragma unroll
      for (int c = DIM + (DIM - 1) * DIM + 1; c < W; ++c) o[c] = 0.0;
    }
    flush(F.facet, base, m.n_facets);
  }
  for (int64_t base = w0 * 32; base < m.n_elements; base += nwarps * 32) {
    const int64_t e = base + lane;
    if (e < m.n_elements) {
      const BoxConst<DIM> b = box_const<DIM>(B.box + e * 2 * DIM);
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        o[d] = b.c[d];
        o[DIM + d] = b.ih[d];
        o[2 * DIM + d] = b.rs[d];
      }
#pragma unroll
      for (int c = 3 * DIM; c < W; ++c) o[c] = 0.0;
    }
    flush(F.element, base, m.n_elements);
  }
}

}  // namespace pdg

extern "C" int pdg_frames_build(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_frames* frames,
                                uint32_t* err_flags, pdg_stream stream) {
  PDG_TRY {
    if (!mesh || !basis || !frames || !frames->simplex || !frames->facet || !frames->element)
      return fail(PDG_ERR_INVALID, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = std::max(mesh->n_simplices, std::max(mesh->n_facets, mesh->n_elements));
    if (n == 0) return PDG_OK;
    const int grid = grid_for_warps((n + 31) / 32, 256);
    if (mesh->dim == 2) frames_kernel<2><<<grid, 256, 0, st>>>(*mesh, *basis, *frames, err_flags);
    else if (mesh->dim == 3) frames_kernel<3><<<grid, 256, 0, st>>>(*mesh, *basis, *frames, err_flags);
    else return fail(PDG_ERR_UNSUPPORTED, "dim must be 2 or 3");
    note_launch();
    PDG_CUDA(cudaGetLastError());
    return PDG_OK;
  }
  PDG_CATCH
}
