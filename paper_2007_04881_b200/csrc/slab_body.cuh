// Space-time slab kernel: one CTA owns one prism (spatial element x (t0, t1))
// and produces all of its CSR rows and its RHS segment in a single pass:
//
//   volume   sub-prisms (fine spatial triangle x interval), tensor rule
//            (simplex rule x interval rule of order 2p + quad_increment,
//            polydg spacetime.py:178-193, quadrature.py:159-178), the
//            volume terms of assembly.py:396-415 in (x, y, t)
//   lateral  spatial faces x interval, normal (n, 0) (spacetime.py:265-285):
//            interior blocks (assembly.py:418-463, both traces evaluated
//            here, e's rows only), Dirichlet / inflow / Neumann
//            (assembly.py:466-512) with the lateral tags of SlabGeometry
//   bottom   the spatial subdivision at t0, statically inflow (normal
//            (0, 0, -1)): the time jump, with the previous slab's trace or
//            the initial data as boundary values (spacetime.py:208-227,
//            355-388); top facets are outflow and contribute nothing.
//
// Why a CTA per prism (the spatial kernel uses a warp per element): a PQ
// basis has (p+1) C(p+2,2) functions -- 18 / 40 / 75 at p = 2 / 3 / 4 -- so
// one element's row block is up to 10 x 10 DMMA tiles; it is spread over the
// CTA's warps as a WR x WC grid of tile blocks (fragment reuse: TR + TC
// shared loads per TR x TC DMMAs), with the k dimension split over WK warp
// groups when the block is small.  Quadrature points are tabulated 32 per
// round (lane = point) into a shared table [row][function][slot]; the warps
// split the functions (a compile-time part per warp, no divergence).
//
// Coefficients come in through the runtime-generated policy class CF
// (model.py policy_source; dim = 3 coordinates, time last) exactly like the
// spatial kernel: fields inline, kind flags and zero entries compile time.
#pragma once

#include "sipg_device.cuh"

namespace pdg {

// the slab's values / col_idx are written once and never re-read: streaming
// (evict-first) stores, as the spatial kernel (PDG_SLAB_ST_CS=0 plain stores)
#ifndef PDG_SLAB_ST_CS
#define PDG_SLAB_ST_CS 1
#endif
template <class T>
__device__ __forceinline__ void slab_st(T* p, T v) {
#if PDG_SLAB_ST_CS
  __stcs(p, v);
#else
  *p = v;
#endif
}


constexpr int SLAB_KS = 32;       // quadrature slots per round (lane = slot)
constexpr int SLAB_KSP = 36;      // slot stride (4 mod 16 doubles: conflict-free fragment loads)
constexpr int SLAB_NBR_MAX = 32;  // neighbours per element staged in shared memory (occupancy: keep small)
constexpr int SLAB_NSC = 8;       // per-slot scalar rows

template <int N>
struct IC {
  static constexpr int value = N;
};

// multi-index table of the slab basis (basis.py:86-104) in D = S + 1
// coordinates (time last): family P = graded lex in (x.., t); family PQ =
// spatial graded lex x time degree, time outer.
template <int S, int P, bool PQ>
struct SlabMI {
  static constexpr int D = S + 1;
  static constexpr int NS = binom(P + S, S);
  static constexpr int NB = PQ ? (P + 1) * NS : binom(P + D, D);
  int a[NB][4];
  // lex order of itertools.product(range(tot + 1), repeat=n) filtered by sum == tot
  __host__ __device__ constexpr void glex(int n, int tot, int k, int& f) {
    int total = 1;
    for (int i = 0; i < n; ++i) total *= tot + 1;
    for (int idx = 0; idx < total; ++idx) {
      int dig[4] = {0, 0, 0, 0}, r = idx, sum = 0;
      for (int i = n - 1; i >= 0; --i) {
        dig[i] = r % (tot + 1);
        r /= tot + 1;
        sum += dig[i];
      }
      if (sum != tot) continue;
      for (int i = 0; i < 4; ++i) a[f][i] = 0;
      for (int i = 0; i < n; ++i) a[f][i] = dig[i];
      if (k >= 0) a[f][S] = k;
      ++f;
    }
  }
  __host__ __device__ constexpr SlabMI() : a{} {
    int f = 0;
    if (PQ) {
      for (int k = 0; k <= P; ++k)
        for (int tot = 0; tot <= P; ++tot) glex(S, tot, k, f);
    } else {
      for (int tot = 0; tot <= P; ++tot) glex(D, tot, -1, f);
    }
  }
};

template <int S, int P, bool PQ>
struct SlabTab {
  static constexpr int D = S + 1;
  static constexpr int NB = SlabMI<S, P, PQ>::NB;
  double v1[D][P + 1], d1[D][P + 1];
  __device__ __forceinline__ void load(const BoxConst<D>& b, const double* x) {
#pragma unroll
    for (int i = 0; i < D; ++i) legendre_1d<P>((x[i] - b.c[i]) * b.ih[i], b.rs[i], b.ih[i], v1[i], d1[i]);
  }
  __device__ __forceinline__ double val(int f) const {
    constexpr SlabMI<S, P, PQ> mi{};
    double r = v1[0][mi.a[f][0]];
#pragma unroll
    for (int i = 1; i < D; ++i) r *= v1[i][mi.a[f][i]];
    return r;
  }
  __device__ __forceinline__ double grad(int f, int k) const {
    constexpr SlabMI<S, P, PQ> mi{};
    if (mi.a[f][k] == 0) return 0.0;
    double r = k == 0 ? d1[0][mi.a[f][0]] : v1[0][mi.a[f][0]];
#pragma unroll
    for (int i = 1; i < D; ++i) r *= (k == i ? d1[i][mi.a[f][i]] : v1[i][mi.a[f][i]]);
    return r;
  }
};

// warp grid over the row block's 8x8 tiles
template <int NT, int NW>
struct SlabTiles {
  static constexpr int WR = NT <= 3 ? 1 : 2;
  static constexpr int WC = (NT <= 6 || NW < 4) ? 1 : 2;
  static constexpr int WK = NW / (WR * WC);
  static constexpr int TR = (NT + WR - 1) / WR;
  static constexpr int TC = (NT + WC - 1) / WC;
};

struct SlabArgs {
  pdg_mesh m;       // spatial mesh
  pdg_basis B;      // slab basis: degrees, prism boxes [n][2][3], DoF offsets
  pdg_rules R;      // spatial rules: simplex (vol) + facet (face)
  pdg_rules T;      // time rules: interval rules in the face tables
  pdg_params prm;
  pdg_pattern pat;
  pdg_slab sl;
  const double* sframe;  // spatial simplex frames [n_simplices][FW], element order (FW = 8 in 2D, 16 in 3D)
  const double* fframe;  // spatial facet frames [n_facets][FW]
  const double* erec;    // spatial basis constants [n_elements][FW] (centre, 1/half, 1/sqrt(width))
  const double* sigma;   // lateral penalty per spatial face
  const int8_t* flow;    // lateral flow side per spatial face
  double* values;
  double* rhs;
  uint32_t* flags;
};

// shared-memory plan (doubles): table, per-slot scalars, RHS accumulator, neighbour staging
inline __host__ __device__ int slab_rows(int diff_kind, bool diag, int n_active, bool has_vr, bool has_src,
                                         int d = 3) {
  int vol = diff_kind == PDG_DIFF_NONE ? 0 : (diag ? n_active : 2 * d);
  vol += has_vr ? 2 : (has_src ? 1 : 0);
  return vol > 4 ? vol : 4;
}
inline __host__ __device__ int slab_table_doubles(int rows, int nbp, int nt, int nw) {
  const int t = rows * nbp * SLAB_KSP;
  // split-K reduction buffer aliases the table: (WK-1) * WR*WC * TR*TC * 64
  const int WR = nt <= 3 ? 1 : 2;
  const int WC = (nt <= 6 || nw < 4) ? 1 : 2;
  const int WK = nw / (WR * WC);
  const int TR = (nt + WR - 1) / WR, TC = (nt + WC - 1) / WC;
  const int red = (WK - 1) * WR * WC * TR * TC * 64;
  return t > red ? t : red;
}
inline __host__ __device__ size_t slab_smem_bytes(int rows, int nbp, int nt, int nw) {
  // table, per-slot scalars, RHS, neighbour staging (4 doubles + 8 ints per entry)
  return ((size_t)slab_table_doubles(rows, nbp, nt, nw) + SLAB_NSC * SLAB_KS + nbp + 4 * SLAB_NBR_MAX) * 8 +
         (size_t)SLAB_NBR_MAX * 8 * sizeof(int32_t);
}

template <class CF, int D>
struct SlabRowsOf {
  static constexpr bool DIAG = CF::a_diag();
  __device__ static constexpr int rowG(int c) {  // table row of the gradient in direction c (diag case)
    int r = 0;
    for (int i = 0; i < c; ++i) r += CF::a_nz(i, i) ? 1 : 0;
    return r;
  }
  __device__ static constexpr int n_active() { return rowG(D); }
  __device__ static constexpr int nG() {
    return CF::diff_kind() == PDG_DIFF_NONE ? 0 : (DIAG ? n_active() : 2 * D);
  }
  static constexpr bool HAS_VR = CF::has_adv() || CF::has_reac();
  __device__ static constexpr int rV() { return nG(); }
};

// flux n.(A grad phi) with the lateral normal (n_s, 0)
template <int S, int P, bool PQ, class CF>
__device__ __forceinline__ double slab_flux(const CF& cf, const SlabTab<S, P, PQ>& tb, int f, const double* n,
                                            const double* x) {
  double fl = 0.0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    double ag = 0.0;
#pragma unroll
    for (int j = 0; j <= S; ++j)
      if (CF::a_nz(i, j)) ag += cf.a_ij(i, j, x) * tb.grad(f, j);
    fl += n[i] * ag;
  }
  return fl;
}

// prism basis constants: the spatial part from the frame pre-pass records
// (box_const of the spatial box, pdg_prepass.cu frames_kernel), the time part
// shared by every prism of the slab
template <int S>
__device__ __forceinline__ BoxConst<S + 1> slab_box(const double* erec, int64_t e, const BoxConst<1>& tb) {
  constexpr int FW = S == 2 ? 8 : 16;
  const double* r = erec + e * FW;
  BoxConst<S + 1> b;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    b.c[i] = r[i];
    b.ih[i] = r[S + i];
    b.rs[i] = r[2 * S + i];
  }
  b.c[S] = tb.c[0];
  b.ih[S] = tb.ih[0];
  b.rs[S] = tb.rs[0];
  return b;
}

template <int TR, int TC>
__device__ __forceinline__ void slab_zero(double (&c)[TR][TC][2]) {
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j) c[i][j][0] = c[i][j][1] = 0.0;
}

// split-K reduction of the tile accumulators into the wk == 0 warps
// (all threads of the CTA call it; the buffer aliases the table)
template <int TR, int TC, int WK, int WRC>
__device__ __forceinline__ void slab_reduce(double (&c)[TR][TC][2], double* red, int wk, int wrc, int lane) {
  if (WK == 1) return;
  __syncthreads();
  if (wk > 0) {
    double* o = red + (((wk - 1) * WRC + wrc) * TR * TC) * 64;
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) {
        o[((i * TC + j) * 32 + lane) * 2 + 0] = c[i][j][0];
        o[((i * TC + j) * 32 + lane) * 2 + 1] = c[i][j][1];
      }
  }
  __syncthreads();
  if (wk == 0) {
    for (int k = 1; k < WK; ++k) {
      const double* o = red + (((k - 1) * WRC + wrc) * TR * TC) * 64;
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int j = 0; j < TC; ++j) {
          c[i][j][0] += o[((i * TC + j) * 32 + lane) * 2 + 0];
          c[i][j][1] += o[((i * TC + j) * 32 + lane) * 2 + 1];
        }
    }
  }
  __syncthreads();
}

template <int TR, int TC>
__device__ __forceinline__ void slab_store(double* values, int64_t voff, int64_t L, int64_t col0, int ne, int nj,
                                           const double (&c)[TR][TC][2], int wr, int wc, int g, int t) {
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = (wr * TR + i) * 8 + g, cc = (wc * TC + j) * 8 + 2 * t + u;
        if (r < ne && cc < nj) slab_st(values + voff + (int64_t)r * L + col0 + cc, c[i][j][u]);
      }
}

template <int S, int P, bool PQ, int NW, class CF>
__device__ __forceinline__ void slab_body(const SlabArgs& a, const CF& cf) {
  constexpr int D = S + 1;                 // space-time coordinates, time last
  constexpr int FW = S == 2 ? 8 : 16;     // spatial frame record width
  using MI = SlabMI<S, P, PQ>;
  using RW = SlabRowsOf<CF, D>;
  using Tab = SlabTab<S, P, PQ>;
  constexpr int NB = MI::NB, NT = (NB + 7) / 8, NBP = NT * 8;
  using TL = SlabTiles<NT, NW>;
  constexpr int WR = TL::WR, WC = TL::WC, WK = TL::WK, TR = TL::TR, TC = TL::TC;
  constexpr int FPW = (NBP + NW - 1) / NW;  // functions tabulated per warp
  constexpr int KSP = SLAB_KSP;
  constexpr int ROWS_V = RW::nG() + (RW::HAS_VR ? 2 : (CF::has_src() ? 1 : 0));
  constexpr int ROWS = ROWS_V > 4 ? ROWS_V : 4;
  constexpr int rV = RW::rV();
  extern __shared__ double smem[];
  const pdg_mesh& m = a.m;
  const pdg_basis& B = a.B;
  const pdg_rules& R = a.R;
  const pdg_rules& TR_ = a.T;  // time rules (interval rules in the face tables)
  const pdg_pattern& pat = a.pat;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp % WR, wc = (warp / WR) % WC, wk = warp / (WR * WC);
  double* T = smem;  // [ROWS][NBP][KSP]
  double* red = smem;
  if (ROWS > a.sl.table_rows) {  // host / policy disagreement: refuse rather than overrun
    if (threadIdx.x == 0 && blockIdx.x == 0) raise_flag(a.flags, PDG_FLAG_STACK);
    return;
  }
  double* sc = smem + slab_table_doubles(a.sl.table_rows, NBP, NT, NW);  // [SLAB_NSC][32]
  double* rhs_s = sc + SLAB_NSC * SLAB_KS;                     // [NBP]
  // neighbour window staged from the interface records (pdg_iface_rec,
  // pdg_prepass.cu): no dependent global loads before a face point
  double* nb_sig = rhs_s + NBP;                                   // [SLAB_NBR_MAX]
  double* nb_n0 = nb_sig + SLAB_NBR_MAX;
  double* nb_n1 = nb_n0 + SLAB_NBR_MAX;
  double* nb_n2 = nb_n1 + SLAB_NBR_MAX;
  int32_t* nb_j = reinterpret_cast<int32_t*>(nb_n2 + SLAB_NBR_MAX);
  int32_t* nb_col = nb_j + SLAB_NBR_MAX;
  int32_t* nb_n = nb_col + SLAB_NBR_MAX;
  int32_t* nb_pj = nb_n + SLAB_NBR_MAX;
  int32_t* nb_fa = nb_pj + SLAB_NBR_MAX;
  int32_t* nb_fb = nb_fa + SLAB_NBR_MAX;
  int32_t* nb_info = nb_fb + SLAB_NBR_MAX;
  int32_t* nb_row0 = nb_info + SLAB_NBR_MAX;
  auto TAB = [&](int row, int f, int slot) -> double& { return T[(row * NBP + f) * KSP + slot]; };
  double* const sca_ = sc;            // volume: w a_cc per direction c (diag) / w (full), rows 0..D-1
  double* const s0_ = sc;             // face: alpha
  double* const s1_ = sc + 32;        // face: beta
  double* const sw_ = sc + 128;       // w (V x R term)
  double* const r1_ = sc + 160;       // RHS weight of the V row
  double* const r2_ = sc + 192;       // RHS weight of the F row
  const double t0 = a.sl.t0, tau = a.sl.t1 - a.sl.t0;
  const bool grad_terms = CF::diff_kind() != PDG_DIFF_NONE && a.prm.include_gradient_terms;
  BoxConst<1> tbox;  // time axis of every prism box: (t0, t1)
  {
    const double tt[2] = {a.sl.t0, a.sl.t1};
    tbox = box_const<1>(tt);
  }

  for (int64_t k = blockIdx.x; k < pat.n_row_elements; k += gridDim.x) {
    const int32_t e = pat.row_elements ? pat.row_elements[k] : (int32_t)k;
    const int pe = B.degree[e];
    const int64_t dof_e = B.dof_offset[e];
    const int ne = (int)(B.dof_offset[e + 1] - dof_e);
    const BoxConst<D> bx = slab_box<S>(a.erec, e, tbox);
    const int64_t voff = pat.elem_val_offset[k];
    const int64_t Lrow = pat.row_len[k];
    const int64_t q0 = pat.nbr_ptr[e];
    const int nnb = (int)(pat.nbr_ptr[e + 1] - q0);
    if (threadIdx.x == 0 && nnb > SLAB_NBR_MAX) raise_flag(a.flags, PDG_FLAG_STACK);
    for (int q = threadIdx.x; q < min(nnb, SLAB_NBR_MAX); q += NW * 32) {
      const pdg_iface_rec& rec = pat.nbr_rec[q0 + q];
      nb_j[q] = rec.j;
      nb_col[q] = rec.col;
      nb_n[q] = rec.nj;
      nb_pj[q] = rec.pj;
      nb_fa[q] = rec.fa;
      nb_fb[q] = rec.fb;
      nb_info[q] = rec.info;
      nb_row0[q] = rec.row0;
      nb_sig[q] = rec.sig;
      nb_n0[q] = rec.nrm[0];
      nb_n1[q] = rec.nrm[1];
      nb_n2[q] = rec.nrm[2];
    }
    for (int f = threadIdx.x; f < NBP; f += NW * 32) rhs_s[f] = 0.0;
    __syncthreads();
    int colself = 0;
    for (int q = 0; q < min(nnb, SLAB_NBR_MAX); ++q)
      if (nb_j[q] == e) colself = nb_col[q];

    double cd[TR][TC][2];
    slab_zero<TR, TC>(cd);

    // RHS contribution of a round: rhs_s[f] += sum_slot V[f] r1 + F[f] r2 (one owner per f)
    // (every weight carries the slot's valid factor, so all 32 slots are summed:
    // a fixed trip count the compiler pipelines)
    auto rhs_round = [&](int rowV, int rowF, int nvalid, bool useF) {
      (void)nvalid;
      {
        for (int f = threadIdx.x; f < NB; f += NW * 32) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
          for (int l = 0; l < SLAB_KS; l += 2) {
            s0 += TAB(rowV, f, l) * r1_[l];
            s1 += TAB(rowV, f, l + 1) * r1_[l + 1];
            if (useF) {
              s0 += TAB(rowF, f, l) * r2_[l];
              s1 += TAB(rowF, f, l + 1) * r2_[l + 1];
            }
          }
          rhs_s[f] += s0 + s1;
        }
      }
    };

    // ---------------------------------------------------------------- volume
    {
      const int order = 2 * pe + a.prm.quad_increment;
      const int r0s = R.vol_offset[order], nqs = R.vol_count[order];
      const int r0t = TR_.face_offset[order], nqt = TR_.face_count[order];
      const int nq = nqs * nqt;
      const int64_t s0 = m.elem_ptr[e];
      const int Q = (int)(m.elem_ptr[e + 1] - s0) * nq;
      for (int base = 0; base < Q; base += SLAB_KS) {
        const int nvalid = min(SLAB_KS, Q - base);
        {
          const int gq = base + min(lane, nvalid - 1);
          const double valid = lane < nvalid ? 1.0 : 0.0;
          const int ls = small_div(gq, nq, 1.0f / (float)nq);
          const int rem = gq - ls * nq;
          const int is = small_div(rem, nqt, 1.0f / (float)nqt), it = rem - is * nqt;
          const double* fr = a.sframe + (s0 + ls) * FW;
          double x[4];
          const double det = frame_point<S, S>(fr, R.points + (r0s + is) * 3, x);
          x[S] = t0 + tau * TR_.points[(r0t + it) * 3];
          const double w = (R.weights[r0s + is] * det) * (tau * TR_.weights[r0t + it]) * valid;
          Tab tb;
          tb.load(bx, x);
          {
            // this warp's function part (f compile time, the guard warp uniform)
#pragma unroll
            for (int f = 0; f < NBP; ++f) {
              if (f / FPW != warp) continue;
              if (CF::diff_kind() != PDG_DIFF_NONE) {
                if (RW::DIAG) {
#pragma unroll
                  for (int c = 0; c < D; ++c)
                    if (CF::a_nz(c, c)) TAB(RW::rowG(c), f, lane) = f < NB ? tb.grad(f, c) : 0.0;
                } else {
#pragma unroll
                  for (int c = 0; c < D; ++c) {
                    double ag = 0.0;
                    if (f < NB) {
#pragma unroll
                      for (int j = 0; j < D; ++j)
                        if (CF::a_nz(c, j)) ag += cf.a_ij(c, j, x) * tb.grad(f, j);
                    }
                    TAB(c, f, lane) = f < NB ? tb.grad(f, c) : 0.0;
                    TAB(D + c, f, lane) = ag;
                  }
                }
              }
              if (RW::HAS_VR || CF::has_src()) {
                const double vv = f < NB ? tb.val(f) : 0.0;
                TAB(rV, f, lane) = vv;
                if (RW::HAS_VR) {
                  double rr = 0.0;
                  if (f < NB) {
                    if (CF::has_adv()) {
#pragma unroll
                      for (int i = 0; i < D; ++i)
                        if (CF::b_nz(i)) rr += cf.b_i(i, x) * tb.grad(f, i);
                    }
                    if (CF::has_reac()) rr += cf.c(x) * vv;
                  }
                  TAB(rV + 1, f, lane) = rr;
                }
              }
            }
            if (warp == 0) {
              if (CF::diff_kind() != PDG_DIFF_NONE) {
                if (RW::DIAG) {
#pragma unroll
                  for (int c = 0; c < D; ++c)
                    if (CF::a_nz(c, c)) sca_[c * 32 + lane] = w * cf.a_ij(c, c, x);
                } else {
                  sca_[lane] = w;
                }
              }
              sw_[lane] = w;
              r1_[lane] = CF::has_src() ? w * cf.f(x) : 0.0;
            }
          }
        }
        __syncthreads();
        const int nk = (nvalid + 3) >> 2;
        for (int kk = wk; kk < nk; kk += WK) {
          const int q = kk * 4 + t;
          if (CF::diff_kind() != PDG_DIFF_NONE) {
            if (RW::DIAG) {
#pragma unroll
              for (int c = 0; c < D; ++c) {
                if (!CF::a_nz(c, c)) continue;
                const double s = sca_[c * 32 + q];
                double lf[TR], rf[TC];
#pragma unroll
                for (int i = 0; i < TR; ++i) lf[i] = s * TAB(RW::rowG(c), ((wr * TR + i) % NT) * 8 + g, q);
#pragma unroll
                for (int j = 0; j < TC; ++j) rf[j] = TAB(RW::rowG(c), ((wc * TC + j) % NT) * 8 + g, q);
#pragma unroll
                for (int i = 0; i < TR; ++i)
#pragma unroll
                  for (int j = 0; j < TC; ++j)
                    if (wr * TR + i < NT && wc * TC + j < NT) dmma(cd[i][j], lf[i], rf[j]);
              }
            } else {
              const double s = sca_[q];
#pragma unroll
              for (int c = 0; c < D; ++c) {
                double lf[TR], rf[TC];
#pragma unroll
                for (int i = 0; i < TR; ++i) lf[i] = s * TAB(c, ((wr * TR + i) % NT) * 8 + g, q);
#pragma unroll
                for (int j = 0; j < TC; ++j) rf[j] = TAB(D + c, ((wc * TC + j) % NT) * 8 + g, q);
#pragma unroll
                for (int i = 0; i < TR; ++i)
#pragma unroll
                  for (int j = 0; j < TC; ++j)
                    if (wr * TR + i < NT && wc * TC + j < NT) dmma(cd[i][j], lf[i], rf[j]);
              }
            }
          }
          if (RW::HAS_VR) {
            const double s = sw_[q];
            double lf[TR], rf[TC];
#pragma unroll
            for (int i = 0; i < TR; ++i) lf[i] = s * TAB(rV, ((wr * TR + i) % NT) * 8 + g, q);
#pragma unroll
            for (int j = 0; j < TC; ++j) rf[j] = TAB(rV + 1, ((wc * TC + j) % NT) * 8 + g, q);
#pragma unroll
            for (int i = 0; i < TR; ++i)
#pragma unroll
              for (int j = 0; j < TC; ++j)
                if (wr * TR + i < NT && wc * TC + j < NT) dmma(cd[i][j], lf[i], rf[j]);
          }
        }
        if (CF::has_src()) rhs_round(rV, rV, nvalid, false);
        __syncthreads();
      }
    }

    // ------------------------------------------------------ face-round helpers
    // Tabulate one lateral / bottom point into rows 0: V_a, 1: F_a (own) and,
    // for interior faces, 2: -V_b, 3: F_b (neighbour); the warp's function part.
    auto face_tab = [&](const Tab& ta, const Tab& tn, const double* nrm, const double* x,
                        bool two, bool useF) {
#pragma unroll
      for (int f = 0; f < NBP; ++f) {
        if (f / FPW != warp) continue;
        double va = 0.0, fa = 0.0, vb = 0.0, fb = 0.0;
        if (f < NB) {
          va = ta.val(f);
          if (useF) fa = slab_flux<S, P, PQ>(cf, ta, f, nrm, x);
          if (two) {
            vb = -tn.val(f);
            if (useF) fb = slab_flux<S, P, PQ>(cf, tn, f, nrm, x);
          }
        }
        TAB(0, f, lane) = va;
        TAB(1, f, lane) = fa;
        if (two) {
          TAB(2, f, lane) = vb;
          TAB(3, f, lane) = fb;
        }
      }
    };
    // C_aa += L1 V_a^T + L2 F_a^T, C_ab += L1 (-V_b)^T + L2 F_b^T with
    // L1 = alpha V_a + beta F_a, L2 = beta V_a (assemble_body.cuh header)
    auto face_contract_k = [&](int k0, int nk, bool two, bool useF, double (&co)[TR][TC][2]) {
      for (int kk = k0 + wk; kk < nk; kk += WK) {
        const int q = kk * 4 + t;
        const double al = s0_[q], be = s1_[q];
        double l1[TR], l2[TR];
#pragma unroll
        for (int i = 0; i < TR; ++i) {
          const int fr_ = ((wr * TR + i) % NT) * 8 + g;
          const double va = TAB(0, fr_, q);
          const double fa = useF ? TAB(1, fr_, q) : 0.0;
          l1[i] = al * va + be * fa;
          l2[i] = be * va;
        }
#pragma unroll
        for (int j = 0; j < TC; ++j) {
          const int fc = ((wc * TC + j) % NT) * 8 + g;
          const double va = TAB(0, fc, q);
          const double fa = useF ? TAB(1, fc, q) : 0.0;
          double nvb = 0.0, fb = 0.0;
          if (two) {
            nvb = TAB(2, fc, q);
            fb = useF ? TAB(3, fc, q) : 0.0;
          }
#pragma unroll
          for (int i = 0; i < TR; ++i) {
            if (wr * TR + i < NT && wc * TC + j < NT) {
              dmma(cd[i][j], l1[i], va);
              if (useF) dmma(cd[i][j], l2[i], fa);
              if (two) {
                dmma(co[i][j], l1[i], nvb);
                if (useF) dmma(co[i][j], l2[i], fb);
              }
            }
          }
        }
      }
    };
    auto face_contract = [&](int nvalid, bool two, bool useF, double (&co)[TR][TC][2]) {
      face_contract_k(0, (nvalid + 3) >> 2, two, useF, co);
    };

    // ------------------------------------------------------ lateral interfaces
    const int nnw = min(nnb, SLAB_NBR_MAX);
    for (int qn = 0; qn < nnw; ++qn) {
      const int32_t j = nb_j[qn];
      if (j == e) continue;
      // Two single-face, single-sub-facet interfaces with <= 16 lateral points
      // each (every 2D Voronoi interface at p <= 2) share one 32-slot round:
      // slots 0-15 the first, 16-31 the second (diagonal block over both,
      // off-diagonal blocks over their own k-steps).
      {
        int qb = qn + 1;
        if (qb < nnw && nb_j[qb] == e) ++qb;
        auto small = [&](int q) {
          const int o = 2 * max(pe, nb_pj[q]) + a.prm.quad_increment;
          return (nb_info[q] & 4) && R.face_count[o] * TR_.face_count[o] <= 16;
        };
        if (qb < nnw && small(qn) && small(qb)) {
          {
            const int seg = lane >> 4, ls = lane & 15;
            const int q = seg ? qb : qn;
            const int o = 2 * max(pe, nb_pj[q]) + a.prm.quad_increment;
            const int r0e = R.face_offset[o], nqe = R.face_count[o];
            const int r0t = TR_.face_offset[o], nqt = TR_.face_count[o];
            const int nqf = nqe * nqt;
            const double valid = ls < nqf ? 1.0 : 0.0;
            const int gq = min(ls, nqf - 1);
            const int ie = small_div(gq, nqt, 1.0f / (float)nqt), it = gq - ie * nqt;
            const int side = nb_info[q] & 1;
            const double sgn = side ? -1.0 : 1.0;
            const bool down = CF::has_adv() && (nb_info[q] & 2) != 0;
            double nrm[4] = {nb_n0[q], nb_n1[q], S == 3 ? nb_n2[q] : 0.0, 0.0};
            nrm[S] = 0.0;
            double x[4];
            const double jac =
                frame_point<S, S - 1>(a.fframe + (int64_t)nb_row0[q] * FW, R.points + (r0e + ie) * 3, x);
            x[S] = t0 + tau * TR_.points[(r0t + it) * 3];
            const double w = (R.weights[r0e + ie] * jac) * (tau * TR_.weights[r0t + it]) * valid;
            Tab ta, tn;
            ta.load(bx, x);
            tn.load(slab_box<S>(a.erec, nb_j[q], tbox), x);
            face_tab(ta, tn, nrm, x, true, grad_terms);
            if (warp == 0) {
              double wbn = 0.0;
              if (down) {
                double bn = 0.0;
#pragma unroll
                for (int i = 0; i < S; ++i)
                  if (CF::b_nz(i)) bn += cf.b_i(i, x) * nrm[i];
                wbn = w * bn;
              }
              s0_[lane] = w * nb_sig[q] - sgn * wbn;
              s1_[lane] = grad_terms ? -0.5 * sgn * w : 0.0;
            }
          }
          __syncthreads();
          // both halves contracted before any split-K reduction (it reuses the table)
          double co[TR][TC][2], co2[TR][TC][2];
          slab_zero<TR, TC>(co);
          slab_zero<TR, TC>(co2);
          face_contract_k(0, 4, true, grad_terms, co);
          face_contract_k(4, 8, true, grad_terms, co2);
          slab_reduce<TR, TC, WK, WR * WC>(co, red, wk, wr + WR * wc, lane);
          if (wk == 0) slab_store<TR, TC>(a.values, voff, Lrow, nb_col[qn], ne, nb_n[qn], co, wr, wc, g, t);
          slab_reduce<TR, TC, WK, WR * WC>(co2, red, wk, wr + WR * wc, lane);
          if (wk == 0) slab_store<TR, TC>(a.values, voff, Lrow, nb_col[qb], ne, nb_n[qb], co2, wr, wc, g, t);
          __syncthreads();
          qn = qb;
          continue;
        }
      }
      const int pj = nb_pj[qn];
      const BoxConst<D> bo = slab_box<S>(a.erec, j, tbox);
      const int order = 2 * max(pe, pj) + a.prm.quad_increment;
      const int r0e = R.face_offset[order], nqe = R.face_count[order];
      const int r0t = TR_.face_offset[order], nqt = TR_.face_count[order];
      const int nqf = nqe * nqt;  // facet rule x time rule of the same order
      double co[TR][TC][2];
      slab_zero<TR, TC>(co);
      for (int32_t f = nb_fa[qn]; f < nb_fb[qn]; ++f) {
        // the interface's first face from the staged record, further faces from the mesh
        const bool first = f == nb_fa[qn];
        const int side = first ? (nb_info[qn] & 1) : (m.face_owner[f] == e ? 0 : 1);
        const double sgn = side ? -1.0 : 1.0;
        const bool down = CF::has_adv() && (first ? (nb_info[qn] & 2) != 0 : a.flow[f] == side);
        const double sig = first ? nb_sig[qn] : a.sigma[f];
        double nrm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < S; ++i)
          nrm[i] = first ? (i == 0 ? nb_n0[qn] : (i == 1 ? nb_n1[qn] : nb_n2[qn])) : m.face_normal[(int64_t)f * S + i];
        const int64_t row0 = first ? (int64_t)nb_row0[qn] : m.face_ptr[f];
        const int Pf = (int)(m.face_ptr[f + 1] - row0) * nqf;
        for (int base = 0; base < Pf; base += SLAB_KS) {
          const int nvalid = min(SLAB_KS, Pf - base);
          {
            const int gq = base + min(lane, nvalid - 1);
            const double valid = lane < nvalid ? 1.0 : 0.0;
            const int lr = small_div(gq, nqf, 1.0f / (float)nqf);
            const int rem = gq - lr * nqf;
            const int ie = small_div(rem, nqt, 1.0f / (float)nqt), it = rem - ie * nqt;
            double x[4];
            const double jac = frame_point<S, S - 1>(a.fframe + (row0 + lr) * FW, R.points + (r0e + ie) * 3, x);
            x[S] = t0 + tau * TR_.points[(r0t + it) * 3];
            const double w = (R.weights[r0e + ie] * jac) * (tau * TR_.weights[r0t + it]) * valid;
            Tab ta, tn;
            ta.load(bx, x);
            tn.load(bo, x);
            face_tab(ta, tn, nrm, x, true, grad_terms);
            if (warp == 0) {
              double wbn = 0.0;
              if (down) {
                double bn = 0.0;
#pragma unroll
                for (int i = 0; i < S; ++i)
                  if (CF::b_nz(i)) bn += cf.b_i(i, x) * nrm[i];
                wbn = w * bn;
              }
              s0_[lane] = w * sig - sgn * wbn;
              s1_[lane] = grad_terms ? -0.5 * sgn * w : 0.0;
            }
          }
          __syncthreads();
          face_contract(nvalid, true, grad_terms, co);
          __syncthreads();
        }
      }
      slab_reduce<TR, TC, WK, WR * WC>(co, red, wk, wr + WR * wc, lane);
      if (wk == 0) slab_store<TR, TC>(a.values, voff, Lrow, nb_col[qn], ne, nb_n[qn], co, wr, wc, g, t);
    }

    // ------------------------------------------------- lateral boundary faces
    for (int64_t bi = m.elem_bface_ptr[e]; bi < m.elem_bface_ptr[e + 1]; ++bi) {
      const int32_t f = m.elem_bfaces[bi];
      const int tag = a.sl.lateral_tag[f];
      if (tag == PDG_TAG_OUTFLOW) continue;
      if (tag == PDG_TAG_INTERIOR) {
        if (threadIdx.x == 0) raise_flag(a.flags, PDG_FLAG_UNCLASSIFIED);
        continue;
      }
      if (tag == PDG_TAG_NEUMANN && !CF::has_neu()) continue;
      if (tag == PDG_TAG_INFLOW && !CF::has_adv()) continue;
      const bool matrix = tag != PDG_TAG_NEUMANN;
      const bool useF = tag == PDG_TAG_DIRICHLET && grad_terms;
      const double sig = a.sigma[f];
      const bool wi = tag == PDG_TAG_DIRICHLET && CF::has_adv() && a.flow[f] == 1;
      const int order = 2 * pe + a.prm.quad_increment;
      const int r0e = R.face_offset[order], nqe = R.face_count[order];
      const int r0t = TR_.face_offset[order], nqt = TR_.face_count[order];
      const int nqf = nqe * nqt;
      double nrm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < S; ++i) nrm[i] = m.face_normal[(int64_t)f * S + i];
      const int64_t row0 = m.face_ptr[f];
      const int Pf = (int)(m.face_ptr[f + 1] - row0) * nqf;
      double dummy[TR][TC][2];
      for (int base = 0; base < Pf; base += SLAB_KS) {
        const int nvalid = min(SLAB_KS, Pf - base);
        {
          const int gq = base + min(lane, nvalid - 1);
          const double valid = lane < nvalid ? 1.0 : 0.0;
          const int lr = small_div(gq, nqf, 1.0f / (float)nqf);
          const int rem = gq - lr * nqf;
          const int ie = small_div(rem, nqt, 1.0f / (float)nqt), it = rem - ie * nqt;
          double x[4];
          const double jac = frame_point<S, S - 1>(a.fframe + (row0 + lr) * FW, R.points + (r0e + ie) * 3, x);
          x[S] = t0 + tau * TR_.points[(r0t + it) * 3];
          const double w = (R.weights[r0e + ie] * jac) * (tau * TR_.weights[r0t + it]) * valid;
          Tab ta;
          ta.load(bx, x);
          face_tab(ta, ta, nrm, x, false, useF);
          if (warp == 0) {
            double wbn = 0.0;
            if (CF::has_adv() && (wi || tag == PDG_TAG_INFLOW)) {
              double bn = 0.0;
#pragma unroll
              for (int i = 0; i < S; ++i)
                if (CF::b_nz(i)) bn += cf.b_i(i, x) * nrm[i];
              wbn = w * bn;
            }
            double al = 0.0, be = 0.0, r1 = 0.0, r2 = 0.0;
            if (tag == PDG_TAG_DIRICHLET) {
              al = w * sig - (wi ? wbn : 0.0);
              be = useF ? -w : 0.0;
              const double gv = CF::has_dir() ? cf.gD(x) : 0.0;
              r1 = gv * al;
              r2 = gv * be;
            } else if (tag == PDG_TAG_INFLOW) {
              al = -wbn;
              r1 = (CF::has_dir() ? cf.gD(x) : 0.0) * al;
            } else {
              r1 = w * cf.gN(x);
            }
            s0_[lane] = al;
            s1_[lane] = be;
            r1_[lane] = r1;
            r2_[lane] = r2;
          }
        }
        __syncthreads();
        if (matrix) face_contract(nvalid, false, useF, dummy);
        rhs_round(0, 1, nvalid, useF);
        __syncthreads();
      }
    }

    // ----------------------------------------------- bottom facet (time jump)
    if (CF::has_adv()) {
      const int order = 2 * pe + a.prm.quad_increment;
      const int r0s = R.vol_offset[order], nqs = R.vol_count[order];
      const int64_t s0 = m.elem_ptr[e];
      const int Q = (int)(m.elem_ptr[e + 1] - s0) * nqs;
      const bool prev = a.sl.prev_values != nullptr;
      BoxConst<D> bp = bx;
      int64_t pdof = 0;
      if (prev) {
        bp = box_const<D>(a.sl.prev_box + (int64_t)e * 2 * D);
        pdof = a.sl.prev_dof_offset[e];
      }
      double dummy[TR][TC][2];
      for (int base = 0; base < Q; base += SLAB_KS) {
        const int nvalid = min(SLAB_KS, Q - base);
        {
          const int gq = base + min(lane, nvalid - 1);
          const double valid = lane < nvalid ? 1.0 : 0.0;
          const int ls = small_div(gq, nqs, 1.0f / (float)nqs);
          const int is = gq - ls * nqs;
          double x[4];
          const double det = frame_point<S, S>(a.sframe + (s0 + ls) * FW, R.points + (r0s + is) * 3, x);
          x[S] = t0;
          const double w = R.weights[r0s + is] * det * valid;
          Tab ta;
          ta.load(bx, x);
          const double nrm[4] = {0.0, 0.0, 0.0, 0.0};
          face_tab(ta, ta, nrm, x, false, false);
          if (warp == 0) {
            // b.n with n = (0, 0, -1)
            const double wbn = CF::b_nz(S) ? -w * cf.b_i(S, x) : 0.0;
            double gv;
            if (prev) {
              Tab tp;
              tp.load(bp, x);
              gv = 0.0;
              const int np_ = (int)(a.sl.prev_dof_offset[e + 1] - pdof);
#pragma unroll
              for (int f = 0; f < NB; ++f)
                if (f < np_) gv += a.sl.prev_values[pdof + f] * tp.val(f);
            } else {
              gv = CF::has_u0() ? cf.u0(x) : 0.0;
            }
            s0_[lane] = -wbn;
            s1_[lane] = 0.0;
            r1_[lane] = -wbn * gv;
          }
        }
        __syncthreads();
        face_contract(nvalid, false, false, dummy);
        rhs_round(0, 0, nvalid, false);
        __syncthreads();
      }
    }

    // ------------------------------------------------------------- write-out
    slab_reduce<TR, TC, WK, WR * WC>(cd, red, wk, wr + WR * wc, lane);
    if (wk == 0) slab_store<TR, TC>(a.values, voff, Lrow, colself, ne, ne, cd, wr, wc, g, t);
    for (int f = threadIdx.x; f < ne; f += NW * 32) a.rhs[dof_e + f] = rhs_s[f];
    // col_idx of all rows (assembly.py:319-324): every row repeats the
    // concatenated DoF ranges of the sorted neighbours
    if (a.pat.col_idx) {
      for (int p = threadIdx.x; p < (int)Lrow; p += NW * 32) {
        int q = 0;
        while (q + 1 < min(nnb, SLAB_NBR_MAX) && nb_col[q + 1] <= p) ++q;
        const int64_t cv = B.dof_offset[nb_j[q]] + (p - nb_col[q]);
        int64_t* dst = a.pat.col_idx + voff + p;
        for (int r = 0; r < ne; ++r) slab_st<int64_t>(dst + (int64_t)r * Lrow, cv);
      }
    }
    __syncthreads();
  }
}

// Lateral face pre-pass (one thread per spatial face): penalty with the
// slab's side data (spacetime.py:301-351: a_bar over the prism's volume
// points with the lateral normal, extruded-split adjacent volumes
// |K| tau / (s+1), prism volume |k| tau, face measure |F| tau, cap p^(2(d-1))
// with d = 3) and the flow side over the order-2 lateral sample points
// (spacetime.py:248-263, 287-309).
template <int S, class CF>
__device__ __forceinline__ void slab_prepass_body(const SlabArgs& a, const CF& cf, double* sigma, int8_t* flow) {
  constexpr int FW = S == 2 ? 8 : 16;
  const pdg_mesh& m = a.m;
  const pdg_basis& B = a.B;
  const pdg_rules& R = a.R;
  const pdg_rules& TR_ = a.T;
  const double t0 = a.sl.t0, tau = a.sl.t1 - a.sl.t0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < m.n_faces; f += stride) {
    const int32_t o = m.face_owner[f], nb = m.face_neighbor[f];
    const bool interior = nb >= 0;
    const int tag = interior ? PDG_TAG_INTERIOR : a.sl.lateral_tag[f];
    double n[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < S; ++i) n[i] = m.face_normal[f * S + i];
    sigma[f] = 0.0;
    flow[f] = interior ? -1 : 0;
    if (!interior && tag != PDG_TAG_DIRICHLET) continue;
    if (CF::has_adv()) {
      const int r0 = R.face_offset[2], nq = R.face_count[2];      // facet rule, order 2
      const int r0t = TR_.face_offset[2], nqt = TR_.face_count[2];  // interval rule, order 2
      double sum = 0.0, mn = PDG_INF, mx = -PDG_INF, amax = 0.0;
      int cnt = 0;
      for (int64_t row = m.face_ptr[f]; row < m.face_ptr[f + 1]; ++row) {
        const double* fr = a.fframe + row * FW;
        for (int i = 0; i < nq; ++i)
          for (int it = 0; it < nqt; ++it) {
            double x[4];
            frame_point<S, S - 1>(fr, R.points + (r0 + i) * 3, x);
            x[S] = t0 + tau * TR_.points[(r0t + it) * 3];
            double bn = 0.0;
#pragma unroll
            for (int k = 0; k < S; ++k)
              if (CF::b_nz(k)) bn += cf.b_i(k, x) * n[k];
            sum += bn;
            mn = fmin(mn, bn);
            mx = fmax(mx, bn);
            amax = fmax(amax, fabs(bn));
            ++cnt;
          }
      }
      const double tol = 1e-10 * fmax(1.0, amax);
      if (mn < -tol && mx > tol) raise_flag(a.flags, PDG_FLAG_STRADDLE);
      const double mean = sum / cnt;
      if (interior) flow[f] = mean < 0.0 ? 0 : (mean > 0.0 ? 1 : -1);
      else flow[f] = mean < 0.0 ? 1 : 0;
    }
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
        raise_flag(a.flags, PDG_FLAG_NO_ADJACENT_SIMPLEX);
        continue;
      }
      const double max_adj = mxv * tau / (double)(S + 1);
      const int p = B.degree[el];
      const double vol = m.elem_volumes[el] * tau;
      double cap = PDG_INF;
      if (a.prm.coverable && a.prm.coverable[el]) {  // p^(2(d-1)), d = S + 1
        cap = 1.0;
        for (int k = 0; k < 2 * S; ++k) cap *= (double)p;
      }
      double ab = 0.0;
      if (CF::diff_kind() != PDG_DIFF_NONE) {
        auto nAn = [&](const double* x) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < S; ++i) {
            double r = 0.0;
#pragma unroll
            for (int j = 0; j < S; ++j)
              if (CF::a_nz(i, j)) r += cf.a_ij(i, j, x) * n[j];
            s += n[i] * r;
          }
          return s;
        };
        if (CF::a_const()) {
          const double x0[4] = {0.0, 0.0, 0.0, 0.0};
          ab = nAn(x0);
        } else {
          const int order = 2 * p + a.prm.quad_increment;
          const int r0s = R.vol_offset[order], nqs = R.vol_count[order];
          const int r0t = TR_.face_offset[order], nqt = TR_.face_count[order];
          ab = -PDG_INF;
          for (int64_t si = m.elem_ptr[el]; si < m.elem_ptr[el + 1]; ++si)
            for (int is = 0; is < nqs; ++is)
              for (int it = 0; it < nqt; ++it) {
                double x[4];
                frame_point<S, S>(a.sframe + si * FW, R.points + (r0s + is) * 3, x);
                x[S] = t0 + tau * TR_.points[(r0t + it) * 3];
                ab = fmax(ab, nAn(x));
              }
        }
      }
      const double ratio = fmin(vol / max_adj, cap);
      best = fmax(best, ratio * ab * (double)(p * p) * (m.face_measure[f] * tau) / vol);
    }
    sigma[f] = a.prm.penalty_constant * best;
  }
}

}  // namespace pdg
