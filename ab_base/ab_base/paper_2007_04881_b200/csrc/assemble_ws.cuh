// Warp-specialised element kernel: one PRODUCER warp and one CONSUMER warp
// per CTA work the same stream of row elements.
//
//   producer  maps quadrature points, evaluates the coefficient fields and
//             tabulates the basis (fp64 ALU work, lane = point) into one of
//             two shared-memory stages, accumulates the RHS, stages the
//             neighbour lists and writes col_idx;
//   consumer  contracts each published stage with DMMA m8n8k4 into the
//             diagonal / off-diagonal block accumulators and stores the
//             finished blocks into the CSR values.
//
// Stages are handed over with named barriers (bar.arrive / bar.sync on
// 64 threads): FULL[s] = 1 + s, EMPTY[s] = 3 + s.  Every stage carries a
// small header telling the consumer what it holds (volume chunk, interface
// round with its store instructions, boundary round, element end), so the
// consumer never touches global metadata.  Compared with one warp doing
// both phases back to back (assemble_body.cuh), the tabulation of round r+1
// overlaps the contraction of round r, and each warp keeps only its own
// phase's registers live.  The arithmetic per item is identical to
// assemble_body (same items, same DMMA tiling), so results are bitwise the
// same as the single-warp body.
#pragma once

#include "assemble_body.cuh"

namespace pdg {

struct WsHdr {
  int kind;  // 0 volume chunk, 1 interface round, 2 boundary round, 3 element end, 4 terminate
  int nk;    // k-steps (4 slots each)
  int nseg;  // interface rounds: 1 or 2 segments
  int seg_k1[2];
  int store[2];
  int col[2], nj[2];
  int use_f;
  int colself;
  int pad[3];
};

// Named barriers with immediate ids (1..4), so the kernel reserves 5 hardware
// barriers instead of all 16.
template <int ID>
__device__ __forceinline__ void nbar_sync_i() {
  asm volatile("bar.sync %0, 64;" ::"n"(ID) : "memory");
}
template <int ID>
__device__ __forceinline__ void nbar_arrive_i() {
  asm volatile("bar.arrive %0, 64;" ::"n"(ID) : "memory");
}
__device__ __forceinline__ void nbar_sync(int id) {
  switch (id) {
    case 1: nbar_sync_i<1>(); break;
    case 2: nbar_sync_i<2>(); break;
    case 3: nbar_sync_i<3>(); break;
    default: nbar_sync_i<4>(); break;
  }
}
__device__ __forceinline__ void nbar_arrive(int id) {
  switch (id) {
    case 1: nbar_arrive_i<1>(); break;
    case 2: nbar_arrive_i<2>(); break;
    case 3: nbar_arrive_i<3>(); break;
    default: nbar_arrive_i<4>(); break;
  }
}

// Shared memory of one CTA (= one producer/consumer pair):
//   stage[2] = { table | sc1[32] | sc2[32] | WsHdr }, then the producer's NbrStage.
#ifndef __CUDACC_RTC__
inline int ws_table_doubles(int dim, int P, int diff_kind, bool has_vr, int* kv_out) {
  const int NB = binom(P + dim, dim);
  const int NBP = ((NB + 7) / 8) * 8;
  const int nG = diff_kind != PDG_DIFF_NONE ? dim : 0;
  const int nAG = diff_kind == PDG_DIFF_FULL ? dim : 0;
  int vrows = nG + nAG + (has_vr ? 2 : 0);
  if (vrows == 0) vrows = 1;
  const int kv = (vrows * NBP * 36 * 8 <= 20 * 1024) ? 32 : 16;
  if (kv_out) *kv_out = kv;
  const int vol = vrows * NBP * (kv + 4);
  const int face = 4 * NBP * KFP;
  return vol > face ? vol : face;
}
#endif

template <int DIM, int P, bool SYM, class CF>
__device__ __forceinline__ void assemble_ws(const KArgs& a, const CF& cf) {
  using S = Shape<DIM, P>;
  using W = Widths<DIM>;
  constexpr int NB = S::NB, NT = S::NT, NBP = S::NBP;
  extern __shared__ double smem[];
  const pdg_mesh& m = a.m;
  const pdg_basis& B = a.B;
  const pdg_rules& R = a.R;
  const pdg_pattern& pat = a.pat;
  const int lane = threadIdx.x & 31;
  const bool producer = threadIdx.x < 32;
  const int g = lane >> 2, t = lane & 3;

  const int table = a.lay.buf_doubles;          // doubles of one stage table
  const int stage_doubles = table + 64 + (int)(sizeof(WsHdr) / 8);
  auto stage_tab = [&](int s) { return smem + s * stage_doubles; };
  auto stage_sc1 = [&](int s) { return smem + s * stage_doubles + table; };
  auto stage_sc2 = [&](int s) { return smem + s * stage_doubles + table + 32; };
  auto stage_hdr = [&](int s) { return reinterpret_cast<WsHdr*>(smem + s * stage_doubles + table + 64); };
  NbrStage* ns = reinterpret_cast<NbrStage*>(smem + 2 * stage_doubles);

  const int kv = a.lay.kv, kvp = a.lay.kv + 4;
  const int dk = cf.diff_kind();
  const int nG = dk != PDG_DIFF_NONE ? DIM : 0;
  const bool full = dk == PDG_DIFF_FULL;
  const bool has_vr = cf.has_adv() || cf.has_reac();
  const int rAG = nG, rV = nG + (full ? DIM : 0), rR = rV + 1;
  const bool grad_terms = dk != PDG_DIFF_NONE && a.prm.include_gradient_terms;
  const int64_t npairs = gridDim.x;

  if (producer) {
    // ===================================================================== PRODUCER
    int sb = 0;
    bool filled[2] = {false, false};
    auto acquire = [&]() {
      if (filled[sb]) nbar_sync(3 + sb);
      __syncwarp();
    };
    auto publish = [&]() {
      __threadfence_block();
      __syncwarp();
      nbar_arrive(1 + sb);
      filled[sb] = true;
      sb ^= 1;
    };
    const bool mine = lane < KF;
    const int slot = lane & (KF - 1);

    for (int64_t k = blockIdx.x; k < pat.n_row_elements; k += npairs) {
      const int32_t e = pat.row_elements ? pat.row_elements[k] : (int32_t)k;
      const int pe = B.degree[e];
      const int64_t dof_e = B.dof_offset[e];
      const int ne = (int)(B.dof_offset[e + 1] - dof_e);
      const BoxConst<DIM> bx = load_box<DIM>(a.erec, e);
      const int64_t voff = pat.elem_val_offset[k];
      const int64_t Lrow = pat.row_len[k];
      double racc[NB];
#pragma unroll
      for (int f = 0; f < NB; ++f) racc[f] = 0.0;

      // ---- volume chunks
      {
        const int order = 2 * pe + a.prm.quad_increment;
        const int r0 = R.vol_offset[order], nq = R.vol_count[order];
        const int64_t s0 = m.elem_ptr[e];
        const int Q = (int)(m.elem_ptr[e + 1] - s0) * nq;
        for (int base = 0; base < Q; base += kv) {
          const int nvalid = min(kv, Q - base);
          acquire();
          double* buf = stage_tab(sb);
          double* sc1 = stage_sc1(sb);
          double* sc2 = stage_sc2(sb);
          if (lane < kv) {
            const int gq = base + min(lane, nvalid - 1);
            const double valid = lane < nvalid ? 1.0 : 0.0;
            const int ls = gq / nq;
            const int kq = gq - ls * nq;
            const double* xi = R.points + (int64_t)(r0 + kq) * 3;
            double x[3] = {0.0, 0.0, 0.0};
            const double det = frame_point<DIM, DIM>(a.sframe + (s0 + ls) * W::SF, xi, x);
            const double w = R.weights[r0 + kq] * det * valid;
            Tab<DIM, P> tb;
            tb.load(bx, x);
            double* col = buf + lane;
            if (nG) {
              const double av = dk == PDG_DIFF_ISO ? cf.a_iso(x) : 1.0;
              sc1[lane] = w * av;
#pragma unroll
              for (int c = 0; c < DIM; ++c)
#pragma unroll
                for (int f = 0; f < NBP; ++f) col[(c * NBP + f) * kvp] = f < NB ? tb.grad(f, c) : 0.0;
              if (full) {
                double A[DIM][DIM];
#pragma unroll
                for (int i = 0; i < DIM; ++i)
#pragma unroll
                  for (int j = 0; j < DIM; ++j) A[i][j] = cf.a_ij(i, j, x);
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
                col[(rV * NBP + f) * kvp] = vv;
                col[(rR * NBP + f) * kvp] = rr;
              }
            }
            if (cf.has_src()) {
              const double wf = w * cf.f(x);
#pragma unroll
              for (int f = 0; f < NB; ++f) racc[f] += wf * tb.val(f);
            }
          }
          if (lane == 0) {
            WsHdr* h = stage_hdr(sb);
            h->kind = 0;
            h->nk = (nvalid + 3) >> 2;
          }
          publish();
        }
      }

      // warm L2 with the next element's simplex frames
      {
        const int64_t kn = k + npairs;
        if (kn < pat.n_row_elements) {
          const int32_t en = pat.row_elements ? pat.row_elements[kn] : (int32_t)kn;
          const int64_t s0n = m.elem_ptr[en], s1n = m.elem_ptr[en + 1];
          const char* p0 = reinterpret_cast<const char*>(a.sframe + s0n * W::SF);
          const int64_t bytes = (s1n - s0n) * W::SF * 8;
          for (int64_t off = (int64_t)lane * 128; off < bytes; off += 32 * 128) prefetch_l2(p0 + off);
          if (lane == 0) prefetch_l2(a.erec + (int64_t)en * W::ER);
        }
      }

      // ---- one face slot: own trace on lanes 0-15, neighbour trace on 16-31
      auto tab_slot = [&](double* buf, double* sc1, double* sc2, int slt, bool own, const double* nrm,
                          int64_t frow, int r0, int kq, double valid, double sig, double sgn, bool down,
                          const BoxConst<DIM>& bo, bool rhs_dir, int tag) {
        const double* xi = R.points + (int64_t)(r0 + kq) * 3;
        double x[3] = {0.0, 0.0, 0.0};
        const double jac = frame_point<DIM, DIM - 1>(a.fframe + frow * W::FF, xi, x);
        const double w = R.weights[r0 + kq] * jac * valid;
        Tab<DIM, P> tb;
        tb.load(own ? bx : bo, x);
        double av = 1.0;
        double A[DIM][DIM];
        const bool flux = tag == PDG_TAG_INTERIOR ? grad_terms : (tag == PDG_TAG_DIRICHLET && grad_terms);
        if (flux) {
          if (full) {
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int jj = 0; jj < DIM; ++jj) A[i][jj] = cf.a_ij(i, jj, x);
          } else {
            av = cf.a_iso(x);
          }
        }
        double wbn = 0.0;
        if (down && cf.has_adv()) {
          double bn = 0.0;
#pragma unroll
          for (int i = 0; i < DIM; ++i) bn += cf.b_i(i, x) * nrm[i];
          wbn = w * bn;
        }
        double al, be, gval = 0.0;
        if (tag == PDG_TAG_INTERIOR) {
          al = w * sig - sgn * wbn;
          be = grad_terms ? -0.5 * sgn * w : 0.0;
        } else if (tag == PDG_TAG_DIRICHLET) {
          al = w * sig - wbn;
          be = flux ? -w : 0.0;
          gval = cf.has_dir() ? cf.gD(x) : 0.0;
        } else if (tag == PDG_TAG_INFLOW) {
          al = -wbn;
          be = 0.0;
          gval = cf.has_dir() ? cf.gD(x) : 0.0;
        } else {  // Neumann
          al = be = 0.0;
          gval = w * cf.gN(x);
        }
        double* col = buf ? buf + slt : nullptr;
        const int rv = own ? 0 : 2;
        const double vs = own ? 1.0 : -1.0;
#pragma unroll
        for (int ff = 0; ff < NBP; ++ff) {
          double vv = 0.0, fl = 0.0;
          if (ff < NB) {
            vv = tb.val(ff);
            if (flux) fl = face_flux<DIM, P>(cf, tb, ff, nrm, av, A);
            if (rhs_dir) {
              if (tag == PDG_TAG_NEUMANN) racc[ff] += gval * vv;
              else if (cf.has_dir()) racc[ff] += gval * (al * vv + be * fl);
            }
          }
          if (col) {
            col[(rv * NBP + ff) * KFP] = vs * vv;
            col[((rv + 1) * NBP + ff) * KFP] = fl;
          }
        }
        if (buf && own) {
          sc1[slt] = al;
          sc2[slt] = be;
        }
      };

      // ---- interfaces
      int colself = 0;
      const int64_t q0 = pat.nbr_ptr[e];
      const int nnb = (int)(pat.nbr_ptr[e + 1] - q0);
      int colcarry = 0;
      for (int w0 = 0; w0 < nnb; w0 += NBR_WIN) {
        const int nw = min(NBR_WIN, nnb - w0);
        __syncwarp();
        {
          int nj = 0;
          bool is_self = false;
          if (lane < nw) {
            const int32_t j = pat.nbr_elem[q0 + w0 + lane];
            const int32_t ifc = pat.nbr_iface[q0 + w0 + lane];
            nj = (int)(B.dof_offset[j + 1] - B.dof_offset[j]);
            is_self = j == e;
            ns->j[lane] = j;
            ns->nj[lane] = nj;
            const int pj = B.degree[j];
            ns->pj[lane] = pj;
            int fa = 0, fb = 0, info = 0, row0 = 0;
            if (!is_self) {
              fa = (int)m.iface_ptr[ifc];
              fb = (int)m.iface_ptr[ifc + 1];
              const int side = m.face_owner[fa] == e ? 0 : 1;
              const bool down = cf.has_adv() && a.flow[fa] == side;
              row0 = (int)m.face_ptr[fa];
              const int nrows = (int)(m.face_ptr[fa + 1] - row0);
              const int nq = R.face_count[2 * max(pe, pj) + a.prm.quad_increment];
              const bool simple = fb - fa == 1 && nrows == 1 && nq <= 8;
              info = side | (down ? 2 : 0) | (simple ? 4 : 0);
              ns->sig[lane] = a.sigma[fa];
#pragma unroll
              for (int i = 0; i < DIM; ++i) ns->nrm[i][lane] = m.face_normal[(int64_t)fa * DIM + i];
            }
            ns->fa[lane] = fa;
            ns->fb[lane] = fb;
            ns->info[lane] = info;
            ns->row0[lane] = row0;
          }
          int incl = nj;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          if (lane < nw) ns->col[lane] = colcarry + incl - nj;
          colcarry += __shfl_sync(0xffffffffu, incl, 31);
          const unsigned selfm = __ballot_sync(0xffffffffu, is_self);
          __syncwarp();
          if (selfm) colself = ns->col[__ffs(selfm) - 1];
        }
        __syncwarp();
        if (a.write_cols) {
          const int c0 = ns->col[0];
          const int c1 = ns->col[nw - 1] + ns->nj[nw - 1];
          int q = 0;
          for (int p = c0 + lane; p < c1; p += 32) {
            while (q + 1 < nw && ns->col[q + 1] <= p) ++q;
            const int64_t cv = B.dof_offset[ns->j[q]] + (p - ns->col[q]);
            int64_t* dst = pat.col_idx + voff + p;
            for (int r = 0; r < ne; ++r) dst[(int64_t)r * Lrow] = cv;
          }
        }
        int qi = 0;
        while (qi < nw) {
          if (ns->j[qi] == e) {
            ++qi;
            continue;
          }
          int qb = qi + 1;
          if (qb < nw && ns->j[qb] == e) ++qb;
          const bool pair = (ns->info[qi] & 4) && qb < nw && (ns->info[qb] & 4);
          if (pair) {
            acquire();
            const int seg = slot >> 3, ls = slot & 7;
            const int q = seg ? qb : qi;
            const int info = ns->info[q];
            const int order = 2 * max(pe, ns->pj[q]) + a.prm.quad_increment;
            const int r0 = R.face_offset[order], nq = R.face_count[order];
            double nrm[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int i = 0; i < DIM; ++i) nrm[i] = ns->nrm[i][q];
            const BoxConst<DIM> bo = load_box<DIM>(a.erec, ns->j[q]);
            tab_slot(stage_tab(sb), stage_sc1(sb), stage_sc2(sb), slot, mine, nrm, ns->row0[q], r0,
                     min(ls, nq - 1), ls < nq ? 1.0 : 0.0, ns->sig[q], (info & 1) ? -1.0 : 1.0,
                     (info & 2) != 0, bo, false, PDG_TAG_INTERIOR);
            if (lane == 0) {
              WsHdr* h = stage_hdr(sb);
              h->kind = 1;
              h->nk = 4;
              h->nseg = 2;
              h->seg_k1[0] = 2;
              h->seg_k1[1] = 4;
              h->store[0] = h->store[1] = 1;
              h->col[0] = ns->col[qi];
              h->nj[0] = ns->nj[qi];
              h->col[1] = ns->col[qb];
              h->nj[1] = ns->nj[qb];
            }
            publish();
            qi = qb + 1;
            continue;
          }
          // general interface: every face, every sub-facet, rounds of 16 points
          const int32_t j = ns->j[qi];
          const int pj = ns->pj[qi];
          const BoxConst<DIM> bo = load_box<DIM>(a.erec, j);
          const int order = 2 * max(pe, pj) + a.prm.quad_increment;
          const int r0 = R.face_offset[order], nq = R.face_count[order];
          const int fend = ns->fb[qi];
          for (int f = ns->fa[qi]; f < fend; ++f) {
            int side, info;
            double sig;
            double nrm[3] = {0.0, 0.0, 0.0};
            int64_t row0;
            if (f == ns->fa[qi]) {
              info = ns->info[qi];
              side = info & 1;
              sig = ns->sig[qi];
#pragma unroll
              for (int i = 0; i < DIM; ++i) nrm[i] = ns->nrm[i][qi];
              row0 = ns->row0[qi];
            } else {
              side = m.face_owner[f] == e ? 0 : 1;
              info = side | ((cf.has_adv() && a.flow[f] == side) ? 2 : 0);
              sig = a.sigma[f];
#pragma unroll
              for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)f * DIM + i];
              row0 = m.face_ptr[f];
            }
            const int Pf = (int)(m.face_ptr[f + 1] - row0) * nq;
            for (int base = 0; base < Pf; base += KF) {
              const int nvalid = min(KF, Pf - base);
              const int gq = base + min(slot, nvalid - 1);
              const int lr = gq / nq;
              acquire();
              tab_slot(stage_tab(sb), stage_sc1(sb), stage_sc2(sb), slot, mine, nrm, row0 + lr, r0, gq - lr * nq,
                       slot < nvalid ? 1.0 : 0.0, sig, side ? -1.0 : 1.0, (info & 2) != 0, bo, false,
                       PDG_TAG_INTERIOR);
              if (lane == 0) {
                WsHdr* h = stage_hdr(sb);
                h->kind = 1;
                h->nk = (nvalid + 3) >> 2;
                h->nseg = 1;
                h->seg_k1[0] = h->nk;
                h->store[0] = (f == fend - 1 && base + KF >= Pf) ? 1 : 0;
                h->col[0] = ns->col[qi];
                h->nj[0] = ns->nj[qi];
              }
              publish();
            }
          }
          ++qi;
        }
      }

      // ---- boundary faces (own side only; Neumann faces contribute to the RHS only)
      const int64_t bend = m.elem_bface_ptr[e + 1];
      for (int64_t bi = m.elem_bface_ptr[e]; bi < bend; ++bi) {
        const int32_t f = m.elem_bfaces[bi];
        const int tag = m.face_tag[f];
        if (tag == PDG_TAG_OUTFLOW || tag == PDG_TAG_INTERIOR) continue;
        if (tag == PDG_TAG_NEUMANN && !cf.has_neu()) continue;
        const bool matrix = tag != PDG_TAG_NEUMANN;
        const double sig = a.sigma[f];
        const bool wi = tag == PDG_TAG_DIRICHLET && cf.has_adv() && a.flow[f] == 1;
        const int order = 2 * pe + a.prm.quad_increment;
        const int r0 = R.face_offset[order], nq = R.face_count[order];
        double nrm[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)f * DIM + i];
        const int64_t row0 = m.face_ptr[f];
        const int Pf = (int)(m.face_ptr[f + 1] - row0) * nq;
        for (int base = 0; base < Pf; base += KF) {
          const int nvalid = min(KF, Pf - base);
          const int gq = base + min(slot, nvalid - 1);
          const int lr = gq / nq;
          if (matrix) acquire();
          // lanes 16-31 mirror lanes 0-15 with zero weight and must not write the stage
          tab_slot((matrix && mine) ? stage_tab(sb) : nullptr, stage_sc1(sb), stage_sc2(sb), slot, true, nrm,
                   row0 + lr, r0,
                   gq - lr * nq, (slot < nvalid && mine) ? 1.0 : 0.0, sig, 1.0,
                   tag == PDG_TAG_INFLOW || wi, bx, mine, tag);
          if (matrix) {
            if (lane == 0) {
              WsHdr* h = stage_hdr(sb);
              h->kind = 2;
              h->nk = (nvalid + 3) >> 2;
              h->use_f = tag == PDG_TAG_DIRICHLET && grad_terms;
            }
            publish();
          }
        }
      }

      // ---- element end: the consumer stores the diagonal block
      acquire();
      if (lane == 0) {
        WsHdr* h = stage_hdr(sb);
        h->kind = 3;
        h->colself = colself;
      }
      publish();

      // ---- RHS: butterfly-reduce the lane partials, lane f writes entry f
#pragma unroll
      for (int f = 0; f < NB; ++f) {
        double v = racc[f];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        racc[f] = v;
      }
#pragma unroll
      for (int f = 0; f < NB; ++f)
        if (lane == (f & 31) && f < ne) a.rhs[dof_e + f] = racc[f];
    }
    // terminate + drain the consumer's last releases
    acquire();
    if (lane == 0) stage_hdr(sb)->kind = 4;
    publish();
    for (int s = 0; s < 2; ++s)
      if (filled[s]) nbar_sync(3 + s);
  } else {
    // ===================================================================== CONSUMER
    int sb = 0;
    for (int64_t k = blockIdx.x;; k += npairs) {
      const bool have = k < pat.n_row_elements;
      int ne = 0;
      int64_t voff = 0, Lrow = 0;
      if (have) {
        const int32_t e = pat.row_elements ? pat.row_elements[k] : (int32_t)k;
        ne = (int)(B.dof_offset[e + 1] - B.dof_offset[e]);
        voff = pat.elem_val_offset[k];
        Lrow = pat.row_len[k];
      }
      double cd[NT][NT][2], co[NT][NT][2];
      zero_tiles<NT>(cd);
      zero_tiles<NT>(co);
      bool done = false, term = false;
      while (!done) {
        nbar_sync(1 + sb);
        const double* buf = stage_tab(sb);
        const double* sc1 = stage_sc1(sb);
        const double* sc2 = stage_sc2(sb);
        const WsHdr* h = stage_hdr(sb);
        const int kind = h->kind;
        if (kind == 0) {
          const int nk = h->nk;
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
        } else if (kind == 1 || kind == 2) {
          const bool off = kind == 1;
          const bool uf = off ? grad_terms : (h->use_f != 0);
          const int nseg = off ? h->nseg : 1;
          int k0 = 0;
          for (int sgi = 0; sgi < nseg; ++sgi) {
            const int k1 = off ? h->seg_k1[sgi] : h->nk;
            for (int kk = k0; kk < k1; ++kk) {
              const int qq = kk * 4 + t;
              const double al = sc1[qq], be = sc2[qq];
              double va[NT], fa[NT], nvb[NT], fb[NT], l1[NT], l2[NT];
#pragma unroll
              for (int i = 0; i < NT; ++i) {
                va[i] = buf[(0 * NBP + i * 8 + g) * KFP + qq];
                if (uf) {
                  fa[i] = buf[(1 * NBP + i * 8 + g) * KFP + qq];
                  l1[i] = al * va[i] + be * fa[i];
                  l2[i] = be * va[i];
                } else {
                  fa[i] = l2[i] = 0.0;
                  l1[i] = al * va[i];
                }
                if (off) {
                  nvb[i] = buf[(2 * NBP + i * 8 + g) * KFP + qq];
                  fb[i] = uf ? buf[(3 * NBP + i * 8 + g) * KFP + qq] : 0.0;
                } else {
                  nvb[i] = fb[i] = 0.0;
                }
              }
#pragma unroll
              for (int r = 0; r < NT; ++r)
#pragma unroll
                for (int cc = 0; cc < NT; ++cc) {
                  if (!SYM || cc >= r) {
                    dmma(cd[r][cc], l1[r], va[cc]);
                    if (uf) dmma(cd[r][cc], l2[r], fa[cc]);
                  }
                  if (off) {
                    dmma(co[r][cc], l1[r], nvb[cc]);
                    if (uf) dmma(co[r][cc], l2[r], fb[cc]);
                  }
                }
            }
            if (off && h->store[sgi]) {
              store_block<NT, false>(a.values, voff, Lrow, h->col[sgi], ne, h->nj[sgi], co, g, t);
              zero_tiles<NT>(co);
            }
            k0 = k1;
          }
        } else if (kind == 3) {
          store_block<NT, SYM>(a.values, voff, Lrow, h->colself, ne, ne, cd, g, t);
          done = true;
        } else {
          done = term = true;
        }
        __syncwarp();
        nbar_arrive(3 + sb);
        sb ^= 1;
      }
      if (term) break;
    }
  }
}

}  // namespace pdg
