// The element kernel: one warp owns one row element and produces all of its
// CSR rows and its RHS segment in a single pass.
//
//   volume    K_e  += sum_q w [ (A grad phi_j).grad phi_i + (b.grad phi_j) phi_i + c phi_j phi_i ]
//                                                        (polydg assembly.py:396-415)
//   faces     rows of e of the SIPG interior blocks     (assembly.py:418-463)
//             with both traces evaluated here, so every value slot has exactly
//             one writer (no atomics, no zero-fill pass, bitwise deterministic,
//             and a row-partitioned run reproduces the one-sided cut-face
//             semantics of assembly.py:685-696,778-788 for free)
//   boundary  Dirichlet / inflow / Neumann terms         (assembly.py:466-512)
//
// Every term is written as a sum of rank-1 updates C += L R^T over "items"
// (one per quadrature point and term), contracted with DMMA m8n8k4:
//   volume   ISO   L = w a dphi/dx_c,   R = dphi/dx_c              (c < d)
//            FULL  L = w dphi/dx_c,     R = (A grad phi)_c
//            b/c   L = w phi,           R = b.grad phi + c phi
//   face     L1 = alpha V_a + beta F_a, L2 = beta V_a, with
//            alpha = w sigma - s_a [e downwind] w b.n,  beta = -1/2 s_a w,
//            diag  C_aa += L1 V_a^T + L2 F_a^T,  off  C_ab += L1 (-V_b)^T + L2 F_b^T
//   (F = n_owner . A grad phi; a derivation is in DESIGN.md §3).
//
// Quadrature points are tabulated lane-parallel (one lane = one point) into a
// per-warp shared-memory table laid out [row][function][slot] with a slot
// stride = 4 (mod 16) doubles, so both the tabulation stores (32 consecutive
// slots) and the DMMA fragment loads (8 functions x 4 slots) are bank-conflict
// free.
#pragma once

#include "pdg_internal.cuh"

namespace pdg {

struct AsmLayout {
  int kv;            // volume slots per round (16 or 32)
  int vrows;         // volume table rows
  int warp_doubles;  // per-warp shared memory (doubles)
  int buf_doubles;   // table part of it (scalars follow)
};

constexpr int KF = 16;   // face slots per round
constexpr int KFP = 20;  // face slot stride

template <int DIM, int P>
struct Shape {
  static constexpr int NB = binom(P + DIM, DIM);
  static constexpr int NT = (NB + 7) / 8;
  static constexpr int NBP = NT * 8;
  static constexpr bool RHS_REGS = NB <= 20;
};

template <int DIM, int P>
AsmLayout make_layout(const pdg_coeffs& C) {
  using S = Shape<DIM, P>;
  AsmLayout L;
  const int nG = C.diffusion_kind != PDG_DIFF_NONE ? DIM : 0;
  const int nAG = C.diffusion_kind == PDG_DIFF_FULL ? DIM : 0;
  const int nVR = (C.has_advection || C.has_reaction) ? 2 : 0;
  L.vrows = nG + nAG + nVR;
  if (L.vrows == 0) L.vrows = 1;
  L.kv = (L.vrows * S::NBP * 36 * 8 <= 20 * 1024) ? 32 : 16;
  const int vol = L.vrows * S::NBP * (L.kv + 4);
  const int face = 4 * S::NBP * KFP;
  const int red = 32 * S::NB;
  int buf = vol > face ? vol : face;
  if (red > buf) buf = red;
  L.buf_doubles = buf;
  L.warp_doubles = buf + 64 + (S::RHS_REGS ? 0 : 32 * S::NB);
  return L;
}

// Store one C tile set into the CSR values of element rows (optionally with
// its mirror image for symmetric accumulation).
template <int NT, bool SYM>
__device__ __forceinline__ void store_block(double* values, int64_t voff, int64_t L, int64_t col0, int ne,
                                            int nj, const double (&c)[NT][NT][2], int g, int t) {
#pragma unroll
  for (int r = 0; r < NT; ++r) {
#pragma unroll
    for (int cc = 0; cc < NT; ++cc) {
      if (SYM && cc < r) continue;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = r * 8 + g, j = cc * 8 + 2 * t + u;
        if (i < ne && j < nj) values[voff + (int64_t)i * L + col0 + j] = c[r][cc][u];
        if (SYM && cc > r && j < ne && i < nj) values[voff + (int64_t)j * L + col0 + i] = c[r][cc][u];
      }
    }
  }
}

template <int DIM, int P, bool SYM>
__global__ void __launch_bounds__(128) assemble_elements(
    const pdg_mesh m, const pdg_basis B, const __grid_constant__ pdg_coeffs C, const pdg_rules R,
    const pdg_params prm, const pdg_pattern pat, const double* __restrict__ sigma,
    const int8_t* __restrict__ flow, double* __restrict__ values, int write_cols,
    double* __restrict__ rhs, uint32_t* flags, const AsmLayout lay, const int mode) {
  // mode 0: CSR rows of the owned elements; mode 1: dense volume-only blocks
  // [k][NB][NB] + loads [k][NB] of the listed elements (unit entry point,
  // polydg element_kernel, assembly.py:1139-1152).
  using S = Shape<DIM, P>;
  constexpr int NB = S::NB, NT = S::NT, NBP = S::NBP;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double* buf = smem + (threadIdx.x >> 5) * lay.warp_doubles;
  double* sc1 = buf + lay.buf_doubles;
  double* sc2 = sc1 + 32;
  double* rhs_s = sc2 + 32;  // [NB][32] lane-private RHS partials when !RHS_REGS

  const int kv = lay.kv, kvp = lay.kv + 4;
  const int nG = C.diffusion_kind != PDG_DIFF_NONE ? DIM : 0;
  const bool full = C.diffusion_kind == PDG_DIFF_FULL;
  const bool has_vr = C.has_advection || C.has_reaction;
  const int rAG = nG, rV = nG + (full ? DIM : 0), rR = rV + 1;
  const bool grad_terms = C.diffusion_kind != PDG_DIFF_NONE && prm.include_gradient_terms;

  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < pat.n_row_elements;
       k += nwarps) {
    const int32_t e = pat.row_elements ? pat.row_elements[k] : (int32_t)k;
    const int pe = B.degree[e];
    const int64_t dof_e = B.dof_offset[e];
    const int ne = (int)(B.dof_offset[e + 1] - dof_e);
    const BoxConst<DIM> bx = box_const<DIM>(B.box + (int64_t)e * 2 * DIM);
    const int64_t voff = mode ? k * NB * NB : pat.elem_val_offset[k];
    const int64_t Lrow = mode ? NB : pat.row_len[k];

    double cd[NT][NT][2];
#pragma unroll
    for (int r = 0; r < NT; ++r)
#pragma unroll
      for (int cc = 0; cc < NT; ++cc) cd[r][cc][0] = cd[r][cc][1] = 0.0;
    double racc[S::RHS_REGS ? NB : 1];
#pragma unroll
    for (int f = 0; f < (S::RHS_REGS ? NB : 1); ++f) racc[f] = 0.0;
    if (!S::RHS_REGS)
      for (int f = 0; f < NB; ++f) rhs_s[f * 32 + lane] = 0.0;
    auto rhs_add = [&](int f, double v) {
      if constexpr (S::RHS_REGS) racc[f] += v;
      else rhs_s[f * 32 + lane] += v;
    };

    // ------------------------------------------------------------ volume
    {
      const int order = 2 * pe + prm.quad_increment;
      const int r0 = R.vol_offset[order], nq = R.vol_count[order];
      const int64_t s0 = m.elem_ptr[e];
      const int Q = (int)(m.elem_ptr[e + 1] - s0) * nq;
      for (int base = 0; base < Q; base += kv) {
        const int nvalid = min(kv, Q - base);
        if (lane < kv) {
          const int gq = base + min(lane, nvalid - 1);
          const double valid = lane < nvalid ? 1.0 : 0.0;
          const int s = m.elem_simplices[s0 + gq / nq];
          const int kq = gq % nq;
          double v0[3], E[3][3];
          const double det = simplex_frame<DIM>(m, s, v0, E, flags);
          const double* xi = R.points + (int64_t)(r0 + kq) * 3;
          double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < DIM; ++i) {
            double acc = v0[i];
#pragma unroll
            for (int j = 0; j < DIM; ++j) acc += xi[j] * E[j][i];
            x[i] = acc;
          }
          const double w = R.weights[r0 + kq] * det * valid;
          Tab<DIM, P> tb;
          tb.load(bx, x);
          double* col = buf + lane;
          if (nG) {
            const double a = C.diffusion_kind == PDG_DIFF_ISO ? eval_prog(C, C.diffusion[0], x) : 1.0;
            sc1[lane] = w * a;
#pragma unroll
            for (int c = 0; c < DIM; ++c)
#pragma unroll
              for (int f = 0; f < NBP; ++f)
                col[((c)*NBP + f) * kvp] = f < NB ? tb.grad(f, c) : 0.0;
            if (full) {
              double A[DIM][DIM];
#pragma unroll
              for (int i = 0; i < DIM; ++i)
#pragma unroll
                for (int j = 0; j < DIM; ++j) A[i][j] = eval_prog(C, C.diffusion[i * DIM + j], x);
#pragma unroll
              for (int c = 0; c < DIM; ++c)
#pragma unroll
                for (int f = 0; f < NBP; ++f) {
                  double v = 0.0;
                  if (f < NB) {
#pragma unroll
                    for (int j = 0; j < DIM; ++j) v += A[c][j] * tb.grad(f, j);
                  }
                  col[((rAG + c) * NBP + f) * kvp] = v;
                }
            }
          }
          if (has_vr) {
            sc2[lane] = w;
            double bvec[DIM];
#pragma unroll
            for (int i = 0; i < DIM; ++i) bvec[i] = C.has_advection ? eval_prog(C, C.advection[i], x) : 0.0;
            const double cr = C.has_reaction ? eval_prog(C, C.reaction, x) : 0.0;
#pragma unroll
            for (int f = 0; f < NBP; ++f) {
              double vv = 0.0, rr = 0.0;
              if (f < NB) {
                vv = tb.val(f);
                if (C.has_advection) {
#pragma unroll
                  for (int i = 0; i < DIM; ++i) rr += bvec[i] * tb.grad(f, i);
                }
                if (C.has_reaction) rr += cr * vv;
              }
              col[(rV * NBP + f) * kvp] = vv;
              col[(rR * NBP + f) * kvp] = rr;
            }
          }
          if (C.has_source) {
            const double wf = w * eval_prog(C, C.source, x);
#pragma unroll
            for (int f = 0; f < NB; ++f) rhs_add(f, wf * tb.val(f));
          }
        }
        __syncwarp();
        const int nk = (nvalid + 3) >> 2;
        for (int kk = 0; kk < nk; ++kk) {
          const int q = kk * 4 + t;
          if (nG) {
            const double s1 = sc1[q];
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
              double lf[NT], rf[NT];
#pragma unroll
              for (int i = 0; i < NT; ++i) {
                const double gv = buf[(c * NBP + i * 8 + g) * kvp + q];
                lf[i] = s1 * gv;
                rf[i] = full ? buf[((rAG + c) * NBP + i * 8 + g) * kvp + q] : gv;
              }
#pragma unroll
              for (int r = 0; r < NT; ++r)
#pragma unroll
                for (int cc = 0; cc < NT; ++cc)
                  if (!SYM || cc >= r) dmma(cd[r][cc], lf[r], rf[cc]);
            }
          }
          if (has_vr) {
            const double s2 = sc2[q];
            double lf[NT], rf[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
              lf[i] = s2 * buf[(rV * NBP + i * 8 + g) * kvp + q];
              rf[i] = buf[(rR * NBP + i * 8 + g) * kvp + q];
            }
#pragma unroll
            for (int r = 0; r < NT; ++r)
#pragma unroll
              for (int cc = 0; cc < NT; ++cc)
                if (!SYM || cc >= r) dmma(cd[r][cc], lf[r], rf[cc]);
          }
        }
        __syncwarp();
      }
    }

    // ------------------------------------------------------------ interfaces
    int64_t colstart = 0, colself = 0;
    const int64_t qend = mode ? 0 : pat.nbr_ptr[e + 1];
    for (int64_t q = mode ? 0 : pat.nbr_ptr[e]; q < qend; ++q) {
      const int32_t j = pat.nbr_elem[q];
      const int nj = (int)(B.dof_offset[j + 1] - B.dof_offset[j]);
      if (j == e) {
        colself = colstart;
        colstart += nj;
        continue;
      }
      const int32_t ifc = pat.nbr_iface[q];
      const BoxConst<DIM> bo = box_const<DIM>(B.box + (int64_t)j * 2 * DIM);
      const int pj = B.degree[j];
      double co[NT][NT][2];
#pragma unroll
      for (int r = 0; r < NT; ++r)
#pragma unroll
        for (int cc = 0; cc < NT; ++cc) co[r][cc][0] = co[r][cc][1] = 0.0;

      for (int64_t fi = m.iface_ptr[ifc]; fi < m.iface_ptr[ifc + 1]; ++fi) {
        const int32_t f = m.iface_faces[fi];
        const int side = m.face_owner[f] == e ? 0 : 1;
        const double sgn = side == 0 ? 1.0 : -1.0;
        const double sig = sigma[f];
        const bool down = C.has_advection && flow[f] == side;
        const int order = 2 * max(pe, pj) + prm.quad_increment;
        const int r0 = R.face_offset[order], nq = R.face_count[order];
        double nrm[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)f * DIM + i];
        const int64_t row0 = m.face_ptr[f];
        const int Pf = (int)(m.face_ptr[f + 1] - row0) * nq;
        const bool mine = lane < KF;
        const int slot = lane & (KF - 1);
        for (int base = 0; base < Pf; base += KF) {
          const int nvalid = min(KF, Pf - base);
          {
            const int gq = base + min(slot, nvalid - 1);
            const double valid = slot < nvalid ? 1.0 : 0.0;
            const int kq = gq % nq;
            double v0[3], E[3][3];
            const double jac = facet_frame<DIM>(m, row0 + gq / nq, v0, E, flags);
            const double* xi = R.points + (int64_t)(r0 + kq) * 3;
            double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int i = 0; i < DIM; ++i) {
              double acc = v0[i];
#pragma unroll
              for (int jj = 0; jj < DIM - 1; ++jj) acc += xi[jj] * E[jj][i];
              x[i] = acc;
            }
            const double w = R.weights[r0 + kq] * jac * valid;
            Tab<DIM, P> tb;
            tb.load(mine ? bx : bo, x);
            double a = 1.0;
            if (grad_terms && C.diffusion_kind == PDG_DIFF_ISO) a = eval_prog(C, C.diffusion[0], x);
            double A[DIM][DIM];
            if (grad_terms && full) {
#pragma unroll
              for (int i = 0; i < DIM; ++i)
#pragma unroll
                for (int jj = 0; jj < DIM; ++jj) A[i][jj] = eval_prog(C, C.diffusion[i * DIM + jj], x);
            }
            double* col = buf + slot;
            const int rv = mine ? 0 : 2;
            const double vs = mine ? 1.0 : -1.0;
#pragma unroll
            for (int ff = 0; ff < NBP; ++ff) {
              double vv = 0.0, fl = 0.0;
              if (ff < NB) {
                vv = tb.val(ff);
                if (grad_terms) {
                  if (full) {
#pragma unroll
                    for (int i = 0; i < DIM; ++i) {
                      double ag = 0.0;
#pragma unroll
                      for (int jj = 0; jj < DIM; ++jj) ag += A[i][jj] * tb.grad(ff, jj);
                      fl += nrm[i] * ag;
                    }
                  } else {
#pragma unroll
                    for (int i = 0; i < DIM; ++i) fl += nrm[i] * tb.grad(ff, i);
                    fl *= a;
                  }
                }
              }
              col[(rv * NBP + ff) * KFP] = vs * vv;
              col[((rv + 1) * NBP + ff) * KFP] = fl;
            }
            if (mine) {
              double wbn = 0.0;
              if (down) {
                double bn = 0.0;
#pragma unroll
                for (int i = 0; i < DIM; ++i) bn += eval_prog(C, C.advection[i], x) * nrm[i];
                wbn = w * bn;
              }
              sc1[slot] = w * sig - sgn * wbn;
              sc2[slot] = grad_terms ? -0.5 * sgn * w : 0.0;
            }
          }
          __syncwarp();
          const int nk = (nvalid + 3) >> 2;
          for (int kk = 0; kk < nk; ++kk) {
            const int qq = kk * 4 + t;
            const double al = sc1[qq], be = sc2[qq];
            double va[NT], fa[NT], nvb[NT], fb[NT], l1[NT], l2[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
              va[i] = buf[(0 * NBP + i * 8 + g) * KFP + qq];
              fa[i] = buf[(1 * NBP + i * 8 + g) * KFP + qq];
              nvb[i] = buf[(2 * NBP + i * 8 + g) * KFP + qq];
              fb[i] = buf[(3 * NBP + i * 8 + g) * KFP + qq];
              l1[i] = al * va[i] + be * fa[i];
              l2[i] = be * va[i];
            }
#pragma unroll
            for (int r = 0; r < NT; ++r)
#pragma unroll
              for (int cc = 0; cc < NT; ++cc) {
                if (!SYM || cc >= r) {
                  dmma(cd[r][cc], l1[r], va[cc]);
                  if (grad_terms) dmma(cd[r][cc], l2[r], fa[cc]);
                }
                dmma(co[r][cc], l1[r], nvb[cc]);
                if (grad_terms) dmma(co[r][cc], l2[r], fb[cc]);
              }
          }
          __syncwarp();
        }
      }
      store_block<NT, false>(values, voff, Lrow, colstart, ne, nj, co, g, t);
      colstart += nj;
    }

    // ------------------------------------------------------------ boundary faces
    const int64_t bend = mode ? 0 : m.elem_bface_ptr[e + 1];
    for (int64_t bi = mode ? 0 : m.elem_bface_ptr[e]; bi < bend; ++bi) {
      const int32_t f = m.elem_bfaces[bi];
      const int tag = m.face_tag[f];
      if (tag == PDG_TAG_OUTFLOW || tag == PDG_TAG_INTERIOR) continue;
      if (tag == PDG_TAG_NEUMANN && !C.has_neumann) continue;
      const bool matrix = tag != PDG_TAG_NEUMANN;
      const double sig = sigma[f];
      const bool wi = tag == PDG_TAG_DIRICHLET && C.has_advection && flow[f] == 1;
      const int order = 2 * pe + prm.quad_increment;
      const int r0 = R.face_offset[order], nq = R.face_count[order];
      double nrm[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)f * DIM + i];
      const int64_t row0 = m.face_ptr[f];
      const int Pf = (int)(m.face_ptr[f + 1] - row0) * nq;
      const int slot = lane & (KF - 1);
      const bool mine = lane < KF;
      const bool use_f = tag == PDG_TAG_DIRICHLET && grad_terms;
      for (int base = 0; base < Pf; base += KF) {
        const int nvalid = min(KF, Pf - base);
        {
          const int gq = base + min(slot, nvalid - 1);
          const double valid = (slot < nvalid && mine) ? 1.0 : 0.0;
          const int kq = gq % nq;
          double v0[3], E[3][3];
          const double jac = facet_frame<DIM>(m, row0 + gq / nq, v0, E, flags);
          const double* xi = R.points + (int64_t)(r0 + kq) * 3;
          double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < DIM; ++i) {
            double acc = v0[i];
#pragma unroll
            for (int jj = 0; jj < DIM - 1; ++jj) acc += xi[jj] * E[jj][i];
            x[i] = acc;
          }
          const double w = R.weights[r0 + kq] * jac * valid;
          Tab<DIM, P> tb;
          tb.load(bx, x);
          double a = 1.0;
          double A[DIM][DIM];
          if (use_f) {
            if (full) {
#pragma unroll
              for (int i = 0; i < DIM; ++i)
#pragma unroll
                for (int jj = 0; jj < DIM; ++jj) A[i][jj] = eval_prog(C, C.diffusion[i * DIM + jj], x);
            } else {
              a = eval_prog(C, C.diffusion[0], x);
            }
          }
          double wbn = 0.0;
          if ((wi || tag == PDG_TAG_INFLOW) && C.has_advection) {
            double bn = 0.0;
#pragma unroll
            for (int i = 0; i < DIM; ++i) bn += eval_prog(C, C.advection[i], x) * nrm[i];
            wbn = w * bn;
          }
          double al = 0.0, be = 0.0, gval = 0.0;
          if (tag == PDG_TAG_DIRICHLET) {
            al = w * sig - (wi ? wbn : 0.0);
            be = use_f ? -w : 0.0;
            gval = C.has_dirichlet ? eval_prog(C, C.dirichlet, x) : 0.0;
          } else if (tag == PDG_TAG_INFLOW) {
            al = -wbn;
            gval = C.has_dirichlet ? eval_prog(C, C.dirichlet, x) : 0.0;
          } else {  // Neumann: load only
            gval = w * eval_prog(C, C.neumann, x);
          }
          double* col = buf + slot;
#pragma unroll
          for (int ff = 0; ff < NBP; ++ff) {
            double vv = 0.0, fl = 0.0;
            if (ff < NB) {
              vv = tb.val(ff);
              if (use_f) {
                if (full) {
#pragma unroll
                  for (int i = 0; i < DIM; ++i) {
                    double ag = 0.0;
#pragma unroll
                    for (int jj = 0; jj < DIM; ++jj) ag += A[i][jj] * tb.grad(ff, jj);
                    fl += nrm[i] * ag;
                  }
                } else {
#pragma unroll
                  for (int i = 0; i < DIM; ++i) fl += nrm[i] * tb.grad(ff, i);
                  fl *= a;
                }
              }
              if (mine) {
                if (tag == PDG_TAG_NEUMANN) rhs_add(ff, gval * vv);
                else if (C.has_dirichlet) rhs_add(ff, gval * (al * vv + be * fl));
              }
            }
            if (mine && matrix) {
              col[(0 * NBP + ff) * KFP] = vv;
              col[(1 * NBP + ff) * KFP] = fl;
            }
          }
          if (mine && matrix) {
            sc1[slot] = al;
            sc2[slot] = be;
          }
        }
        __syncwarp();
        if (matrix) {
          const int nk = (nvalid + 3) >> 2;
          for (int kk = 0; kk < nk; ++kk) {
            const int qq = kk * 4 + t;
            const double al = sc1[qq], be = sc2[qq];
            double va[NT], fa[NT], l1[NT], l2[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
              va[i] = buf[(0 * NBP + i * 8 + g) * KFP + qq];
              fa[i] = buf[(1 * NBP + i * 8 + g) * KFP + qq];
              l1[i] = al * va[i] + be * fa[i];
              l2[i] = be * va[i];
            }
#pragma unroll
            for (int r = 0; r < NT; ++r)
#pragma unroll
              for (int cc = 0; cc < NT; ++cc)
                if (!SYM || cc >= r) {
                  dmma(cd[r][cc], l1[r], va[cc]);
                  if (use_f) dmma(cd[r][cc], l2[r], fa[cc]);
                }
          }
        }
        __syncwarp();
      }
    }

    // ------------------------------------------------------------ write-out
    store_block<NT, SYM>(values, voff, Lrow, colself, ne, ne, cd, g, t);
    if (write_cols && !mode) write_col_rows(B, pat, e, voff, Lrow, lane);
    double* rhs_out = mode ? rhs + k * NB : rhs + dof_e;
    __syncwarp();
    if constexpr (S::RHS_REGS) {
#pragma unroll
      for (int f = 0; f < NB; ++f) buf[lane * NB + f] = racc[f];
      __syncwarp();
      for (int f = lane; f < ne; f += 32) {
        double s = 0.0;
        for (int l = 0; l < 32; ++l) s += buf[l * NB + f];
        rhs_out[f] = s;
      }
    } else {
      __syncwarp();
      for (int f = lane; f < ne; f += 32) {
        double s = 0.0;
        for (int l = 0; l < 32; ++l) s += rhs_s[f * 32 + l];
        rhs_out[f] = s;
      }
    }
    __syncwarp();
  }
}

template <int DIM, int P, bool SYM>
cudaError_t launch_assemble(const pdg_mesh& m, const pdg_basis& B, const pdg_coeffs& C, const pdg_rules& R,
                            const pdg_params& prm, const pdg_pattern& pat, const double* sigma,
                            const int8_t* flow, double* values, int write_cols, double* rhs, uint32_t* flags,
                            cudaStream_t st, int mode) {
  const AsmLayout lay = make_layout<DIM, P>(C);
  const int threads = 128;
  const size_t smem = (size_t)lay.warp_doubles * 8 * (threads / 32);
  auto kern = assemble_elements<DIM, P, SYM>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t blocks_needed = (pat.n_row_elements + 3) / 4;
  const int64_t grid = std::min<int64_t>(blocks_needed, (int64_t)num_sms() * per_sm * 8);
  if (grid <= 0) return cudaSuccess;
  kern<<<(unsigned)grid, threads, smem, st>>>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs,
                                               flags, lay, mode); note_launch();
  return cudaGetLastError();
}

}  // namespace pdg
