// Approach 1 (stage-and-sort) on the device: one warp per WORK ITEM -- a
// volume sub-simplex, an interior sub-facet or a boundary sub-facet, the
// items of polydg's work plan (assembly.py:665-728) -- computes the item's
// dense local blocks and writes them as (key = row * n_cols + col, value)
// triplets into the item's stripe (assembly.py:158-174, 977-999; unused
// stripe slots keep the sentinel key ~0 and sort last), and its load as
// (row, value) pairs.  pdg_triplets_to_csr then sorts (stable LSD radix) and
// merges duplicates (reduce-by-key) into the CSR (triplets_to_csr,
// assembly.py:1002-1031).  This is the paper's Approach 1,
// kept as the cross-validation path of the preset-sparsity engine.
//
// The block mathematics is the element kernel's (assemble_body.cuh header):
// rank-1 items on DMMA m8n8k4, lanes = quadrature points, a per-warp shared
// table [row][function][slot].
#pragma once

#include "sipg_device.cuh"

namespace pdg {

constexpr int A1_KS = 32;   // points per round (lane = point)
constexpr int A1_KSP = 36;  // slot stride (4 mod 16 doubles)
// table rows: volume G_0..G_{d-1}, (A grad)_0..(A grad)_{d-1}, V, R; faces V_a, F_a, -V_b, F_b
inline __host__ __device__ constexpr int a1_rows(int dim) { return 2 * dim + 2; }

struct A1Args {
  pdg_mesh m;
  pdg_basis B;
  pdg_rules R;
  pdg_params prm;
  pdg_a1_items it;
  const double* sframe;  // [n_simplices][W] element order
  const double* fframe;  // [n_facets][W]
  const double* erec;    // [n_elements][W]
  const double* sigma;
  const int8_t* flow;
  uint64_t* keys;
  double* vals;
  uint64_t* load_keys;
  double* load_vals;
  int64_t n_cols;
  uint32_t* flags;
};

inline __host__ __device__ int a1_warp_doubles(int dim, int nbp) { return a1_rows(dim) * nbp * A1_KSP + 4 * A1_KS; }

template <int DIM>
__device__ __forceinline__ BoxConst<DIM> a1_box(const double* erec, int64_t e) {
  constexpr int W = DIM == 2 ? 8 : 16;
  const double* r = erec + e * W;
  BoxConst<DIM> b;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    b.c[i] = r[i];
    b.ih[i] = r[DIM + i];
    b.rs[i] = r[2 * DIM + i];
  }
  return b;
}

template <int DIM, int P, class CF>
__device__ __forceinline__ void approach1_body(const A1Args& a, const CF& cf) {
  constexpr int NB = binom(P + DIM, DIM), NT = (NB + 7) / 8, NBP = NT * 8;
  constexpr int W = DIM == 2 ? 8 : 16;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* T = smem + (threadIdx.x >> 5) * a1_warp_doubles(DIM, NBP);
  double* s1 = T + a1_rows(DIM) * NBP * A1_KSP;
  double* s2 = s1 + A1_KS;
  double* s3 = s2 + A1_KS;  // RHS weight of the V row
  double* s4 = s3 + A1_KS;  // RHS weight of the F row
  auto TAB = [&](int row, int f, int slot) -> double& { return T[(row * NBP + f) * A1_KSP + slot]; };
  const pdg_mesh& m = a.m;
  const pdg_basis& B = a.B;
  const pdg_rules& R = a.R;
  const int dk = cf.diff_kind();
  const bool full = dk == PDG_DIFF_FULL;
  const int nG = dk != PDG_DIFF_NONE ? DIM : 0;
  const bool has_vr = cf.has_adv() || cf.has_reac();
  const int rV = nG + (full ? DIM : 0), rR = rV + 1;
  const bool grad_terms = dk != PDG_DIFF_NONE && a.prm.include_gradient_terms;
  const int64_t nV = a.it.n_volume, nI = a.it.n_interior, nItems = nV + nI + a.it.n_boundary;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  // write an (ni x nj) tile set row-major at stripe position pos
  auto emit_block = [&](const double (&c)[NT][NT][2], int64_t pos, int ni, int nj, int64_t row0, int64_t col0) {
#pragma unroll
    for (int r = 0; r < NT; ++r)
#pragma unroll
      for (int cc = 0; cc < NT; ++cc)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i = r * 8 + g, j = cc * 8 + 2 * t + u;
          if (i < ni && j < nj) {
            const int64_t q = pos + (int64_t)i * nj + j;
            a.keys[q] = (uint64_t)(row0 + i) * (uint64_t)a.n_cols + (uint64_t)(col0 + j);
            a.vals[q] = c[r][cc][u];
          }
        }
  };
  auto zero = [&](double (&c)[NT][NT][2]) {
#pragma unroll
    for (int r = 0; r < NT; ++r)
#pragma unroll
      for (int cc = 0; cc < NT; ++cc) c[r][cc][0] = c[r][cc][1] = 0.0;
  };

  for (int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < nItems; item += nwarps) {
    const int64_t pos = a.it.stripe_offset[item];
    const int64_t lpos = a.it.load_offset[item];
    double cd[NT][NT][2];
    zero(cd);
    double lacc[(NB + 31) / 32];
#pragma unroll
    for (int k = 0; k < (NB + 31) / 32; ++k) lacc[k] = 0.0;
    auto load_add = [&](int rowV, int rowF, int nvalid, bool useF) {
#pragma unroll
      for (int k = 0; k < (NB + 31) / 32; ++k) {
        const int f = k * 32 + lane;
        if (f < NB) {
          double s = 0.0;
          for (int l = 0; l < nvalid; ++l) {
            s += TAB(rowV, f, l) * s3[l];
            if (useF) s += TAB(rowF, f, l) * s4[l];
          }
          lacc[k] += s;
        }
      }
    };
    auto emit_load = [&](int n, int64_t row0) {
#pragma unroll
      for (int k = 0; k < (NB + 31) / 32; ++k) {
        const int f = k * 32 + lane;
        if (f < n) {
          a.load_keys[lpos + f] = (uint64_t)(row0 + f);
          a.load_vals[lpos + f] = lacc[k];
        }
      }
    };

    if (item < nV) {
      // ---------------------------------------------------------- volume item
      const int32_t e = a.it.volume_element[item];
      const int pe = B.degree[e];
      const int64_t dof = B.dof_offset[e];
      const int ne = (int)(B.dof_offset[e + 1] - dof);
      const BoxConst<DIM> bx = a1_box<DIM>(a.erec, e);
      const int order = 2 * pe + a.prm.quad_increment;
      const int r0 = R.vol_offset[order], nq = R.vol_count[order];
      const double* fr = a.sframe + item * W;
      for (int base = 0; base < nq; base += A1_KS) {
        const int nvalid = min(A1_KS, nq - base);
        {
          const int kq = base + min(lane, nvalid - 1);
          const double valid = lane < nvalid ? 1.0 : 0.0;
          double x[3] = {0.0, 0.0, 0.0};
          const double det = frame_point<DIM, DIM>(fr, R.points + (r0 + kq) * 3, x);
          const double w = R.weights[r0 + kq] * det * valid;
          Tab<DIM, P> tb;
          tb.load(bx, x);
          if (nG) {
            s1[lane] = w * (dk == PDG_DIFF_ISO ? cf.a_iso(x) : 1.0);
#pragma unroll
            for (int c = 0; c < DIM; ++c)
#pragma unroll
              for (int f = 0; f < NBP; ++f) TAB(c, f, lane) = f < NB ? tb.grad(f, c) : 0.0;
            if (full) {
#pragma unroll
              for (int c = 0; c < DIM; ++c)
#pragma unroll
                for (int f = 0; f < NBP; ++f) {
                  double v = 0.0;
                  if (f < NB) {
#pragma unroll
                    for (int j = 0; j < DIM; ++j) v += cf.a_ij(c, j, x) * tb.grad(f, j);
                  }
                  TAB(DIM + c, f, lane) = v;
                }
            }
          }
          double bvec[DIM];
#pragma unroll
          for (int i = 0; i < DIM; ++i) bvec[i] = cf.has_adv() ? cf.b_i(i, x) : 0.0;
          const double cr = cf.has_reac() ? cf.c(x) : 0.0;
#pragma unroll
          for (int f = 0; f < NBP; ++f) {
            double vv = 0.0, rr = 0.0;
            if (f < NB) {
              vv = tb.val(f);
              if (cf.has_adv()) {
#pragma unroll
                for (int i = 0; i < DIM; ++i) rr += bvec[i] * tb.grad(f, i);
              }
              if (cf.has_reac()) rr += cr * vv;
            }
            TAB(rV, f, lane) = vv;
            TAB(rR, f, lane) = rr;
          }
          s2[lane] = w;
          s3[lane] = cf.has_src() ? w * cf.f(x) : 0.0;
        }
        __syncwarp();
        const int nk = (nvalid + 3) >> 2;
        for (int kk = 0; kk < nk; ++kk) {
          const int q = kk * 4 + t;
          if (nG) {
            const double sa = s1[q];
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
              double lf[NT], rf[NT];
#pragma unroll
              for (int i = 0; i < NT; ++i) {
                const double gv = TAB(c, i * 8 + g, q);
                lf[i] = sa * gv;
                rf[i] = full ? TAB(DIM + c, i * 8 + g, q) : gv;
              }
#pragma unroll
              for (int r = 0; r < NT; ++r)
#pragma unroll
                for (int cc = 0; cc < NT; ++cc) dmma(cd[r][cc], lf[r], rf[cc]);
            }
          }
          if (has_vr) {
            const double sw = s2[q];
            double lf[NT], rf[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
              lf[i] = sw * TAB(rV, i * 8 + g, q);
              rf[i] = TAB(rR, i * 8 + g, q);
            }
#pragma unroll
            for (int r = 0; r < NT; ++r)
#pragma unroll
              for (int cc = 0; cc < NT; ++cc) dmma(cd[r][cc], lf[r], rf[cc]);
          }
        }
        if (cf.has_src()) load_add(rV, rV, nvalid, false);
        __syncwarp();
      }
      emit_block(cd, pos, ne, ne, dof, dof);
      if (cf.has_src() || a.it.load_offset[item + 1] > lpos) emit_load(ne, dof);
      continue;
    }

    const int32_t f = a.it.face[item - nV];
    const int64_t frow = a.it.facet_row[item - nV];
    const double* ffr = a.fframe + frow * W;
    double nrm[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)f * DIM + i];
    const int32_t o = m.face_owner[f];
    const int po = B.degree[o];
    const int64_t dofo = B.dof_offset[o];
    const int no = (int)(B.dof_offset[o + 1] - dofo);
    const BoxConst<DIM> bxo = a1_box<DIM>(a.erec, o);

    if (item < nV + nI) {
      // ---------------------------------------------------- interior sub-facet
      const int32_t nb = m.face_neighbor[f];
      const int pn = B.degree[nb];
      const int64_t dofn = B.dof_offset[nb];
      const int nn = (int)(B.dof_offset[nb + 1] - dofn);
      const BoxConst<DIM> bxn = a1_box<DIM>(a.erec, nb);
      const int order = 2 * max(po, pn) + a.prm.quad_increment;
      const int r0 = R.face_offset[order], nq = R.face_count[order];
      const double sig = a.sigma[f];
      const int up = cf.has_adv() ? a.flow[f] : -1;  // downwind side
      // stripe: [oo (no x no), on (no x nn), no (nn x no), nn (nn x nn)] (assembly.py:786-800)
      for (int side = 0; side < 2; ++side) {
        const double sgn = side ? -1.0 : 1.0;
        const bool down = up == side;
        double co[NT][NT][2];
        zero(cd);
        zero(co);
        for (int base = 0; base < nq; base += A1_KS) {
          const int nvalid = min(A1_KS, nq - base);
          {
            const int kq = base + min(lane, nvalid - 1);
            const double valid = lane < nvalid ? 1.0 : 0.0;
            double x[3] = {0.0, 0.0, 0.0};
            const double jac = frame_point<DIM, DIM - 1>(ffr, R.points + (r0 + kq) * 3, x);
            const double w = R.weights[r0 + kq] * jac * valid;
            Tab<DIM, P> ta, tn;
            ta.load(side ? bxn : bxo, x);
            tn.load(side ? bxo : bxn, x);
            double av = 1.0, A[DIM][DIM];
            if (grad_terms) {
              if (full) {
#pragma unroll
                for (int i = 0; i < DIM; ++i)
#pragma unroll
                  for (int j = 0; j < DIM; ++j) A[i][j] = cf.a_ij(i, j, x);
              } else {
                av = cf.a_iso(x);
              }
            }
#pragma unroll
            for (int ff = 0; ff < NBP; ++ff) {
              double va = 0.0, fa = 0.0, vb = 0.0, fb = 0.0;
              if (ff < NB) {
                va = ta.val(ff);
                vb = -tn.val(ff);
                if (grad_terms) {
                  double ga = 0.0, gb = 0.0;
#pragma unroll
                  for (int i = 0; i < DIM; ++i) {
                    double aga = 0.0, agb = 0.0;
                    if (full) {
#pragma unroll
                      for (int j = 0; j < DIM; ++j) {
                        aga += A[i][j] * ta.grad(ff, j);
                        agb += A[i][j] * tn.grad(ff, j);
                      }
                    } else {
                      aga = ta.grad(ff, i);
                      agb = tn.grad(ff, i);
                    }
                    ga += nrm[i] * aga;
                    gb += nrm[i] * agb;
                  }
                  fa = full ? ga : av * ga;
                  fb = full ? gb : av * gb;
                }
              }
              TAB(0, ff, lane) = va;
              TAB(1, ff, lane) = fa;
              TAB(2, ff, lane) = vb;
              TAB(3, ff, lane) = fb;
            }
            double wbn = 0.0;
            if (down) {
              double bn = 0.0;
#pragma unroll
              for (int i = 0; i < DIM; ++i) bn += cf.b_i(i, x) * nrm[i];
              wbn = w * bn;
            }
            s1[lane] = w * sig - sgn * wbn;
            s2[lane] = grad_terms ? -0.5 * sgn * w : 0.0;
          }
          __syncwarp();
          const int nk = (nvalid + 3) >> 2;
          for (int kk = 0; kk < nk; ++kk) {
            const int q = kk * 4 + t;
            const double al = s1[q], be = s2[q];
            double va[NT], fa[NT], nvb[NT], fb[NT], l1[NT], l2[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
              va[i] = TAB(0, i * 8 + g, q);
              fa[i] = TAB(1, i * 8 + g, q);
              nvb[i] = TAB(2, i * 8 + g, q);
              fb[i] = TAB(3, i * 8 + g, q);
              l1[i] = al * va[i] + be * fa[i];
              l2[i] = be * va[i];
            }
#pragma unroll
            for (int r = 0; r < NT; ++r)
#pragma unroll
              for (int cc = 0; cc < NT; ++cc) {
                dmma(cd[r][cc], l1[r], va[cc]);
                dmma(cd[r][cc], l2[r], fa[cc]);
                dmma(co[r][cc], l1[r], nvb[cc]);
                dmma(co[r][cc], l2[r], fb[cc]);
              }
          }
          __syncwarp();
        }
        if (side == 0) {
          emit_block(cd, pos, no, no, dofo, dofo);
          emit_block(co, pos + (int64_t)no * no, no, nn, dofo, dofn);
        } else {
          const int64_t p2 = pos + (int64_t)no * no + (int64_t)no * nn;
          emit_block(co, p2, nn, no, dofn, dofo);
          emit_block(cd, p2 + (int64_t)nn * no, nn, nn, dofn, dofn);
        }
      }
      continue;
    }

    // ------------------------------------------------------- boundary sub-facet
    const int tag = m.face_tag[f];
    const bool matrix = tag == PDG_TAG_DIRICHLET || tag == PDG_TAG_INFLOW;
    const bool useF = tag == PDG_TAG_DIRICHLET && grad_terms;
    const double sig = a.sigma[f];
    const bool wi = tag == PDG_TAG_DIRICHLET && cf.has_adv() && a.flow[f] == 1;
    const int order = 2 * po + a.prm.quad_increment;
    const int r0 = R.face_offset[order], nq = R.face_count[order];
    for (int base = 0; base < nq; base += A1_KS) {
      const int nvalid = min(A1_KS, nq - base);
      {
        const int kq = base + min(lane, nvalid - 1);
        const double valid = lane < nvalid ? 1.0 : 0.0;
        double x[3] = {0.0, 0.0, 0.0};
        const double jac = frame_point<DIM, DIM - 1>(ffr, R.points + (r0 + kq) * 3, x);
        const double w = R.weights[r0 + kq] * jac * valid;
        Tab<DIM, P> tb;
        tb.load(bxo, x);
        double av = 1.0, A[DIM][DIM];
        if (useF) {
          if (full) {
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int j = 0; j < DIM; ++j) A[i][j] = cf.a_ij(i, j, x);
          } else {
            av = cf.a_iso(x);
          }
        }
#pragma unroll
        for (int ff = 0; ff < NBP; ++ff) {
          double vv = 0.0, fl = 0.0;
          if (ff < NB) {
            vv = tb.val(ff);
            if (useF) {
#pragma unroll
              for (int i = 0; i < DIM; ++i) {
                double ag = 0.0;
                if (full) {
#pragma unroll
                  for (int j = 0; j < DIM; ++j) ag += A[i][j] * tb.grad(ff, j);
                } else {
                  ag = tb.grad(ff, i);
                }
                fl += nrm[i] * ag;
              }
              if (!full) fl *= av;
            }
          }
          TAB(0, ff, lane) = vv;
          TAB(1, ff, lane) = fl;
        }
        double wbn = 0.0;
        if ((wi || tag == PDG_TAG_INFLOW) && cf.has_adv()) {
          double bn = 0.0;
#pragma unroll
          for (int i = 0; i < DIM; ++i) bn += cf.b_i(i, x) * nrm[i];
          wbn = w * bn;
        }
        double al = 0.0, be = 0.0, r1 = 0.0, r2 = 0.0;
        if (tag == PDG_TAG_DIRICHLET) {
          al = w * sig - (wi ? wbn : 0.0);
          be = useF ? -w : 0.0;
          const double gv = cf.has_dir() ? cf.gD(x) : 0.0;
          r1 = gv * al;
          r2 = gv * be;
        } else if (tag == PDG_TAG_INFLOW) {
          al = -wbn;
          r1 = (cf.has_dir() ? cf.gD(x) : 0.0) * al;
        } else if (tag == PDG_TAG_NEUMANN) {
          r1 = cf.has_neu() ? w * cf.gN(x) : 0.0;
        }
        s1[lane] = al;
        s2[lane] = be;
        s3[lane] = r1;
        s4[lane] = r2;
      }
      __syncwarp();
      if (matrix) {
        const int nk = (nvalid + 3) >> 2;
        for (int kk = 0; kk < nk; ++kk) {
          const int q = kk * 4 + t;
          const double al = s1[q], be = s2[q];
          double va[NT], fa[NT], l1[NT], l2[NT];
#pragma unroll
          for (int i = 0; i < NT; ++i) {
            va[i] = TAB(0, i * 8 + g, q);
            fa[i] = TAB(1, i * 8 + g, q);
            l1[i] = al * va[i] + be * fa[i];
            l2[i] = be * va[i];
          }
#pragma unroll
          for (int r = 0; r < NT; ++r)
#pragma unroll
            for (int cc = 0; cc < NT; ++cc) {
              dmma(cd[r][cc], l1[r], va[cc]);
              if (useF) dmma(cd[r][cc], l2[r], fa[cc]);
            }
        }
      }
      load_add(0, 1, nvalid, useF);
      __syncwarp();
    }
    if (matrix) emit_block(cd, pos, no, no, dofo, dofo);
    if (a.it.load_offset[item + 1] > lpos) emit_load(no, dofo);
  }
}

}  // namespace pdg
