// The element kernel body: one warp owns one row element and produces all of
// its CSR rows and its RHS segment in a single pass.
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
// Every term is a sum of rank-1 updates C += L R^T over "items" (one per
// quadrature point and term), contracted with DMMA m8n8k4 (SASS DMMA.8x8x4):
//   volume   ISO   L = w a dphi/dx_c,   R = dphi/dx_c              (c < d)
//            FULL  L = w dphi/dx_c,     R = (A grad phi)_c
//            b/c   L = w phi,           R = b.grad phi + c phi
//   face     L1 = alpha V_a + beta F_a, L2 = beta V_a, with
//            alpha = w sigma - s_a [e downwind] w b.n,  beta = -1/2 s_a w,
//            diag  C_aa += L1 V_a^T + L2 F_a^T,  off  C_ab += L1 (-V_b)^T + L2 F_b^T
//   (F = n_owner . A grad phi; derivation in DESIGN.md §3).
//
// Quadrature points are tabulated lane-parallel (one lane = one point) into a
// per-warp shared-memory table laid out [row][function][slot] with a slot
// stride = 4 (mod 16) doubles, so both the tabulation stores (consecutive
// slots) and the DMMA fragment loads (8 functions x 4 slots) are bank-conflict
// free.  Geometry arrives pre-mapped: per-simplex / per-facet affine frames
// and per-element basis constants are produced once per assembly by
// geometry_frames (pdg_prepass.cu), so a quadrature point costs one broadcast
// load of its frame instead of three dependent gathers.
//
// The coefficient fields enter through a policy class CF: the ahead-of-time
// library uses InterpCoef (bytecode interpreter over pdg_coeffs); the runtime
// specialisation (pdg_jit.cu, NVRTC) passes a generated class whose fields are
// inlined expressions and whose kind flags are compile-time constants.
#pragma once

#include "sipg_device.cuh"

namespace pdg {

// RHS partials of a lane live in registers when the basis has at most this
// many functions, else in a lane-private shared-memory column (fewer
// registers, more shared memory); the runtime specialisation sets it per
// compile (pdg_jit.cu), the host layout (make_layout) must agree.
#ifndef PDG_RHS_REGS_MAX
#define PDG_RHS_REGS_MAX 20
#endif

// unroll factors of the k-step loops (tuning knobs, PDG_JIT_DEFINES)
#define PDG_STR_(x) #x
#define PDG_UNROLL(n) _Pragma(PDG_STR_(unroll n))
// PDG_REG_CAPPED: 1 when the kernel is compiled for 12 warps/SM (168
// registers), 0 when shared memory already limits residency and ptxas may use
// up to 255 registers (pdg_jit.cu full_source sets it).  Two 3D defaults below
// depend on it.
#ifndef PDG_REG_CAPPED
#define PDG_REG_CAPPED 1
#endif
// full unroll of a complete volume round (fixed trip count, compile-time table
// offsets) vs the PDG_VOL_UNROLL loop (smaller code): -1 = 2D unrolled; 3D
// looped when register-capped -- three gradient rows make the unrolled round
// big enough to miss in the instruction cache: r02 same-box cfg4 9.59 vs 9.85
// ms, while cfg5 / cfg2 lose 1.3% / 2% without it -- and unrolled with 255
// registers (cfg4 8.80 vs 9.10 ms together with PDG_PAD_ZERO), 0 / 1 force
#ifndef PDG_VOL_FULL
#define PDG_VOL_FULL -1
#endif
#ifndef PDG_VOL_UNROLL
#define PDG_VOL_UNROLL 1
#endif
#ifndef PDG_FACE_UNROLL
#define PDG_FACE_UNROLL 1
#endif
// table rows of the padding functions NB <= f < NBP: 0 = not written (they feed
// only tile rows / columns >= NB, which no store reads; the packed 10-function
// tile reads function 10 only into columns it discards), 1 = written as zeros,
// -1 = skipped except in register-capped 3D kernels (r02 same-box: 2D --
// cfg2 1.282 -> 1.255 ms, cfg3 p=3 4.39 -> 4.31, cfg1 18 -> 17 us; 3D at 168
// registers writes them -- cfg4 9.52 vs 9.72 -- at 255 skips them)
#ifndef PDG_PAD_ZERO
#define PDG_PAD_ZERO -1
#endif

// constant isotropic diffusion: the volume's sqrt-weight scaling folded into the
// Legendre recurrence start (1), or applied to the tabulated factors (0)
#ifndef PDG_FOLD_SW
#define PDG_FOLD_SW 1
#endif
#ifndef PDG_COL_PTR
#define PDG_COL_PTR 1
#endif
// phase timers (diagnostics: one warp prints its clock64 split at exit)
#ifndef PDG_TIMERS
#define PDG_TIMERS 0
#endif
#define PDG_T(i)                                 \
  if (PDG_TIMERS) {                              \
    const long long now_ = clock64();            \
    tacc[i] += now_ - tprev;                     \
    tprev = now_;                                \
  }


// result stores (values, col_idx) are written once and never re-read by the
// kernel: streaming (evict-first) stores keep L2 for the frames / records the
// neighbouring warps re-read (same-box A/B r02, 400k cfg5 cells: 6.50 vs
// 6.55 ms; 32-bit offsets inside the row block were slower, 6.77 ms)
#ifndef PDG_ST_CS
#define PDG_ST_CS 1
#endif
template <class T>
__device__ __forceinline__ void st_out(T* p, T v) {
#if PDG_ST_CS
  __stcs(p, v);
#else
  *p = v;
#endif
}

constexpr int KF = 16;   // face slots per round
constexpr int KFP = 20;  // face slot stride
// neighbour entries staged per window / simplex frames of one element kept in
// shared memory.  3D uses 12 / 16 (an agglomerated Kuhn element has ~5 tets and
// ~7 neighbours; the smaller footprint fits 5 instead of 4 two-warp CTAs per SM)
#ifndef PDG_3D_SMALL
#define PDG_3D_SMALL 1
#endif
__host__ __device__ constexpr int nbr_win(int dim) { return (PDG_3D_SMALL && dim == 3) ? 12 : 16; }
__host__ __device__ constexpr int fr_max(int dim) { return (PDG_3D_SMALL && dim == 3) ? 16 : 32; }
constexpr int NBR_WIN_MAX = 16;
constexpr int REC16 = (int)(sizeof(pdg_iface_rec) / 16);  // 16-byte chunks per interface record
constexpr int RULE_SMEM_MAX = 128;  // rule tables up to this many points live in shared memory (per CTA)
#ifndef PDG_RULES_SMEM
#define PDG_RULES_SMEM 1
#endif

// doubles of the per-CTA rule copy (points [n][3], weights [n], sqrt weights [n]), 0 if not staged
inline __host__ __device__ int rule_smem_doubles(int n_points) {
  return (n_points > 0 && n_points <= RULE_SMEM_MAX) ? ((5 * n_points + 1) & ~1) : 0;
}

// the quadrature tables a kernel reads: the CTA's shared copy when staged
struct RuleView {
  const double* pts;  // [n][3]
  const double* w;    // [n]
  const double* sw;   // [n]
};

// stage the rule tables into the CTA's shared memory (all threads; ends with a CTA barrier)
__device__ __forceinline__ RuleView stage_rules(const pdg_rules& R, double* sm) {
  const int n = R.n_points;
  if (!PDG_RULES_SMEM || n <= 0 || n > RULE_SMEM_MAX) return RuleView{R.points, R.weights, R.sqrt_weights};
  for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) sm[i] = R.points[i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sm[3 * n + i] = R.weights[i];
    sm[4 * n + i] = R.sqrt_weights[i];
  }
  __syncthreads();
  return RuleView{sm, sm + 3 * n, sm + 4 * n};
}

template <int DIM>
struct Widths {
  static constexpr int SF = DIM == 2 ? 8 : 16;  // simplex frame: v0, E (row-major), |det|
  static constexpr int FF = DIM == 2 ? 8 : 16;  // facet frame: v0, E rows, sqrt(det(EE^T))
  static constexpr int ER = DIM == 2 ? 8 : 16;  // element record: centre, 1/half, 1/sqrt(width)
};

struct AsmLayout {
  int kv;            // volume slots per round (16 or 32)
  int vrows;         // volume table rows
  int warp_doubles;  // per-warp shared memory (doubles)
  int buf_doubles;   // table part of it (scalars + staging follow)
};

struct KArgs {
  pdg_mesh m;
  pdg_basis B;
  pdg_rules R;
  pdg_params prm;
  pdg_pattern pat;
  const double* sigma;
  const int8_t* flow;
  const double* sframe;  // [n_simplices][SF], element order (elem_ptr indexing)
  const double* fframe;  // [n_facets][FF]
  const double* erec;    // [n_elements][ER]
  double* values;
  double* rhs;
  uint32_t* flags;
  int write_cols;
  int mode;  // 0: CSR rows; 1: dense volume-only blocks (unit entry point)
  AsmLayout lay;
};

template <int DIM, int P>
struct Shape {
  static constexpr int NB = binom(P + DIM, DIM);
  static constexpr int NT = (NB + 7) / 8;
  static constexpr int NBP = NT * 8;
  static constexpr bool RHS_REGS = NB <= PDG_RHS_REGS_MAX;
};


__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// 16-byte asynchronous global -> shared copies (LDGSTS), L2 only
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Bulk asynchronous copies (TMA engine, SASS UBLKCP) completing on a per-warp
// mbarrier: the next element's interface-record window and simplex frames are
// two contiguous runs, so one elected lane could move them with two
// instructions instead of 32 lanes issuing 16-byte LDGSTS.  Same-box A/B r02:
// 400k cfg5 cells 6.22 vs 6.28 ms, cfg4 9.83 vs 9.99 ms, cfg3 p=3 4.59 vs
// 4.64 ms (1-1.5% faster).  Off by default: compute-sanitizer synccheck
// reports "Missing init" on the warp's mbarrier in this kernel (minimal
// probes of the same init / expect_tx / bulk copy / try_wait sequence,
// tools/probe/, are clean; results are bit-identical either way), and the
// default path must be sanitizer-clean.  PDG_BULK=1 selects it.
#ifndef PDG_BULK
#define PDG_BULK 0
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t phase) {
  asm volatile("{\n .reg .pred p;\n PDG_MBW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra PDG_MBW_%=;\n}\n" ::"r"(smem_u32(mb)), "r"(phase) : "memory");
}

template <int DIM>
__device__ __forceinline__ BoxConst<DIM> load_box(const double* erec, int64_t e) {
  const double* r = erec + e * Widths<DIM>::ER;
  BoxConst<DIM> b;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    b.c[i] = r[i];
    b.ih[i] = r[DIM + i];
    b.rs[i] = r[2 * DIM + i];
  }
  return b;
}

// Store one C tile set into rows of the element's row block (optionally
// with its mirror image for symmetric accumulation).
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
        if (i < ne && j < nj) st_out(values + voff + (int64_t)i * L + col0 + j, c[r][cc][u]);
        if (SYM && cc > r && j < ne && i < nj) st_out(values + voff + (int64_t)j * L + col0 + i, c[r][cc][u]);
      }
    }
  }
}

// Packed remainder tile of a symmetric 10x10 block (NB = 10: p = 3 in 2D,
// p = 2 in 3D).  The upper triangle needs the 8x8 tile of functions 0-7 plus
// 19 pairs involving functions 8, 9; one 8x8 DMMA tile with rows
// {0..5, 8, 9} and columns {8, 9, 6, 7} covers all of them -- (i, 8|9) for
// i < 6 and (8|9, 6..9) -- so the block costs 2 DMMAs per k-step instead of
// the 3 of the padded 16x16 upper triangle.  Columns 4-7 read the zero
// padding row 10.  Only pairs the main tile does not hold are stored.
__host__ __device__ constexpr int pk_row(int g) { return g < 6 ? g : g + 2; }
__host__ __device__ constexpr int pk_col(int g) { return g < 2 ? g + 8 : (g < 4 ? g + 4 : 10); }

template <int DIM, int P, bool SYM>
struct PackPlan {
  static constexpr bool on = SYM && binom(P + DIM, DIM) == 10;
};

__device__ __forceinline__ void store_packed10(double* values, int64_t voff, int64_t L, int64_t col0, int ne,
                                               const double (&c)[2], int g, int t) {
  const int i = pk_row(g);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int j = pk_col(2 * t + u);
    if (j >= 10 || (i < 8 && j < 8) || i >= ne || j >= ne) continue;
    st_out(values + voff + (int64_t)i * L + col0 + j, c[u]);
    if (!(i >= 8 && j >= 8)) st_out(values + voff + (int64_t)j * L + col0 + i, c[u]);
  }
}

template <int NT>
__device__ __forceinline__ void zero_tiles(double (&c)[NT][NT][2]) {
#pragma unroll
  for (int r = 0; r < NT; ++r)
#pragma unroll
    for (int cc = 0; cc < NT; ++cc) c[r][cc][0] = c[r][cc][1] = 0.0;
}

// Face trace values at one point: V_f and the flux F_f = n.(A grad phi_f)
template <int DIM, int P, class CF>
__device__ __forceinline__ double face_flux(const CF& cf, const Tab<DIM, P>& tb, int f, const double* nrm,
                                            double a, const double (&A)[DIM][DIM]) {
  double fl = 0.0;
  if (cf.diff_kind() == PDG_DIFF_FULL) {
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      double ag = 0.0;
#pragma unroll
      for (int jj = 0; jj < DIM; ++jj) ag += A[i][jj] * tb.grad(f, jj);
      fl += nrm[i] * ag;
    }
  } else {
#pragma unroll
    for (int i = 0; i < DIM; ++i) fl += nrm[i] * tb.grad(f, i);
    fl *= a;
  }
  return fl;
}

// KV: volume slots per round when known at compile time (runtime-specialised
// kernels), 0 = read a.lay.kv.
template <int DIM, int P, bool SYM, class CF, int KV = 0>
__device__ __forceinline__ void assemble_body(const KArgs& a, const CF& cf) {
  using S = Shape<DIM, P>;
  using W = Widths<DIM>;
  constexpr int NBR_WIN = nbr_win(DIM);
  constexpr int FR_MAX = fr_max(DIM);
  constexpr int NB = S::NB, NT = S::NT, NBP = S::NBP;
  constexpr int NBW = (PDG_PAD_ZERO < 0 ? (DIM == 3 && PDG_REG_CAPPED) : PDG_PAD_ZERO != 0) ? NBP : NB;  // table functions written per point
  extern __shared__ double smem[];
  const pdg_mesh& m = a.m;
  const pdg_basis& B = a.B;
  const pdg_rules& R = a.R;
  const pdg_pattern& pat = a.pat;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const RuleView RV = stage_rules(R, smem);
  double* buf = smem + rule_smem_doubles(PDG_RULES_SMEM ? R.n_points : 0) + (threadIdx.x >> 5) * a.lay.warp_doubles;
  double* sc1 = buf + a.lay.buf_doubles;
  double* sc2 = sc1 + 32;
  // interface records of the current / next element's first neighbour window
  pdg_iface_rec* recs = reinterpret_cast<pdg_iface_rec*>(sc2 + 32);  // [2][NBR_WIN]
  double* rhs_s = reinterpret_cast<double*>(recs + 2 * NBR_WIN);    // [NB][32] when !RHS_REGS
  // async-copied geometry: the element's simplex frames, the window's first facet frames
  double* sfr = rhs_s + (S::RHS_REGS ? 0 : 32 * NB);
  double* ffr = sfr + FR_MAX * W::SF;
  // basis constants (element records) of the window's neighbours (3D only:
  // measured r01, same box: 3D 10.25 vs 10.48 ms, 2D 6.88 vs 6.59 ms -- in 2D
  // the L2 load of the record overlaps the paired round's tabulation)
  constexpr bool STAGE_BOX = DIM == 3;
  double* ebx = ffr + NBR_WIN * W::FF;
  // per-warp mbarrier of the bulk copies (last 2 doubles of the warp's region)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(buf + a.lay.warp_doubles - 2);
  const bool bulk = PDG_BULK && !a.mode;
  uint32_t mphase = 0;
  if (bulk) {
    if (lane == 0) mbar_init(mbar);
    __syncwarp();
  }

  const int kv = KV ? KV : a.lay.kv, kvp = kv + 4;
  const int dk = cf.diff_kind();
  const int nG = dk != PDG_DIFF_NONE ? DIM : 0;
  const bool full = dk == PDG_DIFF_FULL;
  const bool has_vr = cf.has_adv() || cf.has_reac();
  const int rAG = nG, rV = nG + (full ? DIM : 0), rR = rV + 1;
  const bool grad_terms = dk != PDG_DIFF_NONE && a.prm.include_gradient_terms;
  // Isotropic diffusion: the volume table holds sqrt(w a) dphi, so the
  // k-step feeds the same fragment as both DMMA operands (no per-k-step
  // weighting, half the fragment loads).  Needs a(x) >= 0; a negative value
  // raises PDG_FLAG_NEG_DIFFUSION and the host re-runs with PDG_OPT_PLAIN_VOLUME.
  const bool sqrtw = dk == PDG_DIFF_ISO && !(a.prm.options & PDG_OPT_PLAIN_VOLUME);
  constexpr bool PK = PackPlan<DIM, P, SYM>::on;  // packed remainder tile: cd[0][1] holds rows pk_row x cols pk_col
  const int fA1 = pk_row(g), fB1 = pk_col(g);
  const int mode = a.mode;

  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // Asynchronous staging one element ahead (cp.async, issued while the
  // current element's faces run): the simplex frames of element kk into sfr
  // (if they fit) and the interface records of its first neighbour window
  // into recs[rb].  The caller commits the group.
  auto issue_next = [&](int64_t kk, int rb) -> bool {
    if (kk >= pat.n_row_elements) return false;
    const int32_t en = pat.row_elements ? pat.row_elements[kk] : (int32_t)kk;
    if (bulk) {  // two bulk copies by one lane, completion on the warp's mbarrier
      const int64_t r0n = pat.nbr_ptr[en];
      const int nwn = min(NBR_WIN, (int)(pat.nbr_ptr[en + 1] - r0n));
      const int64_t s0n = m.elem_ptr[en];
      const int nsn = (int)(m.elem_ptr[en + 1] - s0n);
      const bool frames = nsn <= FR_MAX;
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads before async writes
        const uint32_t rbytes = (uint32_t)nwn * (uint32_t)sizeof(pdg_iface_rec);
        const uint32_t fbytes = frames ? (uint32_t)nsn * W::SF * 8u : 0u;
        mbar_expect_tx(mbar, rbytes + fbytes);
        bulk_g2s(recs + rb * NBR_WIN, pat.nbr_rec + r0n, rbytes, mbar);
        if (frames) bulk_g2s(sfr, a.sframe + s0n * W::SF, fbytes, mbar);
      }
      return frames;
    }
    if (!mode) {
      const int64_t r0n = pat.nbr_ptr[en];
      const int nwn = min(NBR_WIN, (int)(pat.nbr_ptr[en + 1] - r0n));
      const double* rsrc = reinterpret_cast<const double*>(pat.nbr_rec + r0n);
      double* rdst = reinterpret_cast<double*>(recs + rb * NBR_WIN);
      for (int c = lane; c < nwn * REC16; c += 32) cp_async16(rdst + 2 * c, rsrc + 2 * c);
    }
    const int64_t s0n = m.elem_ptr[en];
    const int nsn = (int)(m.elem_ptr[en + 1] - s0n);
    if (nsn > FR_MAX) return false;
    const double* src = a.sframe + s0n * W::SF;
    for (int c = lane; c < nsn * W::SF / 2; c += 32) cp_async16(sfr + 2 * c, src + 2 * c);
    return true;
  };
  // first facet frame of every non-self interface of a staged window -> ffr[entry]
  // and the neighbour's basis constants -> ebx[entry] (no dependent global
  // loads left on the first face of an interface)
  auto issue_ffr = [&](const pdg_iface_rec* rw, int nw, int32_t e) {
    if (lane < nw && rw[lane].j != e) {
      const double* src = a.fframe + (int64_t)rw[lane].row0 * W::FF;
#pragma unroll
      for (int c = 0; c < W::FF / 2; ++c) cp_async16(ffr + lane * W::FF + 2 * c, src + 2 * c);
      if (STAGE_BOX) {
        const double* bsrc = a.erec + (int64_t)rw[lane].j * W::ER;
#pragma unroll
        for (int c = 0; c < W::ER / 2; ++c) cp_async16(ebx + lane * W::ER + 2 * c, bsrc + 2 * c);
      }
    }
  };
  int rb = 0;
  bool next_frames = issue_next(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, rb);
  cp_async_commit();
  long long tacc[PDG_TIMERS ? 10 : 1] = {0};
  long long tprev = PDG_TIMERS ? clock64() : 0;
  int nel_done = 0;
  for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < pat.n_row_elements;
       k += nwarps, rb ^= 1) {
    const bool fr_smem = next_frames;
    if (bulk) {
      mbar_wait(mbar, mphase);
      mphase ^= 1u;
    }
    cp_async_wait_all();
    __syncwarp();
    const int32_t e = pat.row_elements ? pat.row_elements[k] : (int32_t)k;
    pdg_iface_rec* rc = recs + rb * NBR_WIN;
    const int64_t q0 = mode ? 0 : pat.nbr_ptr[e];
    const int nnb = mode ? 0 : (int)(pat.nbr_ptr[e + 1] - q0);
    // the first window's facet frames land during the volume phase
    issue_ffr(rc, min(NBR_WIN, nnb), e);
    cp_async_commit();
    const int pe = B.degree[e];
    const int64_t dof_e = B.dof_offset[e];
    const int ne = (int)(B.dof_offset[e + 1] - dof_e);
    const BoxConst<DIM> bx = load_box<DIM>(a.erec, e);
    const int64_t voff = mode ? k * NB * NB : pat.elem_val_offset[k];
    const int64_t Lrow = mode ? NB : pat.row_len[k];

    double cd[NT][NT][2];
    zero_tiles<NT>(cd);
    double racc[S::RHS_REGS ? NB : 1];
#pragma unroll
    for (int f = 0; f < (S::RHS_REGS ? NB : 1); ++f) racc[f] = 0.0;
    if (!S::RHS_REGS)
      for (int f = 0; f < NB; ++f) rhs_s[f * 32 + lane] = 0.0;
    auto rhs_add = [&](int f, double v) {
      if constexpr (S::RHS_REGS) racc[f] += v;
      else rhs_s[f * 32 + lane] += v;
    };

    ++nel_done;
    PDG_T(0)
    // ------------------------------------------------------------ volume
    {
      const int order = 2 * pe + a.prm.quad_increment;
      const int r0 = R.vol_offset[order], nq = R.vol_count[order];
      const int64_t s0 = m.elem_ptr[e];
      const int Q = (int)(m.elem_ptr[e + 1] - s0) * nq;
      const float rnq = 1.0f / (float)nq;
      for (int base = 0; base < Q; base += kv) {
        const int nvalid = min(kv, Q - base);
        if (lane < kv) {
          const int gq = base + min(lane, nvalid - 1);
          const double valid = lane < nvalid ? 1.0 : 0.0;
          const int ls = small_div(gq, nq, rnq);
          const int kq = gq - ls * nq;
          const double* xi = RV.pts + (r0 + kq) * 3;
          double x[3] = {0.0, 0.0, 0.0};
          const double* fr = fr_smem ? sfr + ls * W::SF : a.sframe + (s0 + ls) * W::SF;
          const double det = frame_point<DIM, DIM>(fr, xi, x);
          const double w = RV.w[r0 + kq] * det * valid;
          // constant isotropic a without advection / reaction rows: the sqrt
          // weight enters through the recurrence start of the dim-0 factors (one
          // product instead of 2(P+1)), and the RHS uses w f phi = (f sw / a) (sw phi)
          const bool fold = PDG_FOLD_SW && nG && sqrtw && !has_vr && cf.a_const();
          double av = 1.0, sw = 0.0;
          if (nG && sqrtw) {
            av = cf.a_iso(x);
            if (av < 0.0) raise_flag(a.flags, PDG_FLAG_NEG_DIFFUSION);
            sw = RV.sw[r0 + kq] * fr[DIM + DIM * DIM + 1] * sqrt(fmax(av, 0.0)) * valid;
          }
          Tab<DIM, P> tb;
          tb.load(bx, x, fold ? sw : 1.0);
          double* col = buf + lane;
          if (nG && sqrtw) {
            Tab<DIM, P> ts = tb;
            if (!fold) ts.scale(sw);
#pragma unroll
            for (int c = 0; c < DIM; ++c)
#pragma unroll
              for (int f = 0; f < NBW; ++f) col[(c * NBP + f) * kvp] = f < NB ? ts.grad(f, c) : 0.0;
          } else if (nG) {
            const double av = dk == PDG_DIFF_ISO ? cf.a_iso(x) : 1.0;
            sc1[lane] = w * av;
#pragma unroll
            for (int c = 0; c < DIM; ++c)
#pragma unroll
              for (int f = 0; f < NBW; ++f) col[(c * NBP + f) * kvp] = f < NB ? tb.grad(f, c) : 0.0;
            if (full) {
              double A[DIM][DIM];
#pragma unroll
              for (int i = 0; i < DIM; ++i)
#pragma unroll
                for (int j = 0; j < DIM; ++j) A[i][j] = cf.a_ij(i, j, x);
#pragma unroll
              for (int c = 0; c < DIM; ++c)
#pragma unroll
                for (int f = 0; f < NBW; ++f) {
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
            for (int f = 0; f < NBW; ++f) {
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
            const double wf = fold ? cf.f(x) * (sw * (1.0 / av)) : w * cf.f(x);
            // phi_f = X_a Y_b (Z_c): fold w f into the x-factors once (P+1 products
            // instead of one per function)
            constexpr MultiIdx<DIM, P> mi{};
            double wx[P + 1];
#pragma unroll
            for (int k = 0; k <= P; ++k) wx[k] = wf * tb.v1[0][k];
#pragma unroll
            for (int f = 0; f < NB; ++f) {
              double v = wx[mi.a[f][0]] * tb.v1[1][mi.a[f][1]];
              if (DIM == 3) v *= tb.v1[2][mi.a[f][2]];
              rhs_add(f, v);
            }
          }
        }
        __syncwarp();
        PDG_T(1)
        const int nk = (nvalid + 3) >> 2;
        auto vol_kstep = [&](int kk) {
          const int q = kk * 4 + t;
          if (nG && sqrtw && PK) {
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
              const double a0 = buf[(c * NBP + g) * kvp + q];
              const double a1 = buf[(c * NBP + fA1) * kvp + q];
              const double b1 = buf[(c * NBP + fB1) * kvp + q];
              dmma(cd[0][0], a0, a0);
              dmma(cd[0][1], a1, b1);
            }
          } else if (nG && sqrtw) {
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
              double fr_[NT];
#pragma unroll
              for (int i = 0; i < NT; ++i) fr_[i] = buf[(c * NBP + i * 8 + g) * kvp + q];
#pragma unroll
              for (int r = 0; r < NT; ++r)
#pragma unroll
                for (int cc = 0; cc < NT; ++cc)
                  if (!SYM || cc >= r) dmma(cd[r][cc], fr_[r], fr_[cc]);
            }
          } else if (nG && PK) {
            const double s1 = sc1[q];
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
              const double g0 = buf[(c * NBP + g) * kvp + q];
              const double gA = buf[(c * NBP + fA1) * kvp + q];
              const double gB = buf[(c * NBP + fB1) * kvp + q];
              const double r0v = full ? buf[((rAG + c) * NBP + g) * kvp + q] : g0;
              const double rBv = full ? buf[((rAG + c) * NBP + fB1) * kvp + q] : gB;
              dmma(cd[0][0], s1 * g0, r0v);
              dmma(cd[0][1], s1 * gA, rBv);
            }
          } else if (nG) {
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
          if (has_vr && PK) {
            const double s2 = sc2[q];
            dmma(cd[0][0], s2 * buf[(rV * NBP + g) * kvp + q], buf[(rR * NBP + g) * kvp + q]);
            dmma(cd[0][1], s2 * buf[(rV * NBP + fA1) * kvp + q], buf[(rR * NBP + fB1) * kvp + q]);
          } else if (has_vr) {
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
        };
        constexpr bool VOL_FULL = PDG_VOL_FULL < 0 ? (DIM == 2 || !PDG_REG_CAPPED) : PDG_VOL_FULL != 0;
        if (VOL_FULL && KV && nk == KV / 4) {
          // full chunk of a runtime-specialised kernel: fixed trip count and
          // compile-time table offsets
#pragma unroll
          for (int kk = 0; kk < KV / 4; ++kk) vol_kstep(kk);
        } else {
          PDG_UNROLL(PDG_VOL_UNROLL)
          for (int kk = 0; kk < nk; ++kk) vol_kstep(kk);
        }
        __syncwarp();
        PDG_T(2)
      }
    }

    // the volume phase is done with sfr: start copying the next element's
    // simplex frames and records while this element's faces are processed
    __syncwarp();
    next_frames = issue_next(k + nwarps, rb ^ 1);
    cp_async_commit();
    __syncwarp();

    // ------------------------------------------------------------ interfaces
    // Neighbour entries are staged NBR_WIN at a time as interface records
    // (pdg_iface_rec: element, DoF count, column start, face range and the
    // first face's metadata, flattened by pdg_iface_records; the first window
    // arrives by cp.async during the previous element's faces), so the face
    // loop reads shared memory instead of chains of dependent global loads.  Two interfaces made of a single sub-facet with <= 8
    // quadrature points (every 2D Voronoi interface up to p = 6) share one
    // tabulation round: slots 0-7 / 8-15, own trace on lanes 0-15, the
    // neighbour's on lanes 16-31.
    int64_t colself = 0;
    const bool mine = lane < KF;
    const int slot = lane & (KF - 1);

    // tabulate one face slot: own trace (lanes 0-15) or neighbour trace (16-31)
    auto tab_slot = [&](const double* nrm, const double* frp, int r0, int kq, double valid, double sig, double sgn,
                        bool down, const BoxConst<DIM>& bo) {
      const double* xi = RV.pts + (r0 + kq) * 3;
      double x[3] = {0.0, 0.0, 0.0};
      const double jac = frame_point<DIM, DIM - 1>(frp, xi, x);
      const double w = RV.w[r0 + kq] * jac * valid;
      Tab<DIM, P> tb;
      tb.load(mine ? bx : bo, x);
      double av = 1.0;
      double A[DIM][DIM];
      if (grad_terms) {
        if (full) {
#pragma unroll
          for (int i = 0; i < DIM; ++i)
#pragma unroll
            for (int jj = 0; jj < DIM; ++jj) A[i][jj] = cf.a_ij(i, jj, x);
        } else {
          av = cf.a_iso(x);
        }
      }
      double* col = buf + slot;
      const int rv = mine ? 0 : 2;
      const double vs = mine ? 1.0 : -1.0;
      if (DIM == 2 && !full) {
        // phi = X_a Y_b: the trace sign, a(x) and the normal folded into the 1D
        // factors once per point: V = X_a (s Y_b), F = (a n0 X'_a) Y_b + (a X_a)(n1 Y'_b)
        constexpr MultiIdx<DIM, P> mi{};
        double ys[P + 1], xa[P + 1], xb[P + 1], yc[P + 1];
#pragma unroll
        for (int k = 0; k <= P; ++k) {
          ys[k] = vs * tb.v1[1][k];
          xa[k] = (av * nrm[0]) * tb.d1[0][k];
          xb[k] = av * tb.v1[0][k];
          yc[k] = nrm[1] * tb.d1[1][k];
        }
#pragma unroll
        for (int ff = 0; ff < NBW; ++ff) {
          double vv = 0.0, fl = 0.0;
          if (ff < NB) {
            const int ia = mi.a[ff][0], ib = mi.a[ff][1];
            vv = tb.v1[0][ia] * ys[ib];
            if (grad_terms) {
              if (ia > 0) fl = xa[ia] * tb.v1[1][ib];
              if (ib > 0) fl = ia > 0 ? fma(xb[ia], yc[ib], fl) : xb[ia] * yc[ib];
            }
          }
          col[(rv * NBP + ff) * KFP] = vv;
          col[((rv + 1) * NBP + ff) * KFP] = fl;
        }
      } else {
#pragma unroll
        for (int ff = 0; ff < NBW; ++ff) {
          double vv = 0.0, fl = 0.0;
          if (ff < NB) {
            vv = tb.val(ff);
            if (grad_terms) fl = face_flux<DIM, P>(cf, tb, ff, nrm, av, A);
          }
          col[(rv * NBP + ff) * KFP] = vs * vv;
          col[((rv + 1) * NBP + ff) * KFP] = fl;
        }
      }
      if (mine) {
        double wbn = 0.0;
        if (down) {
          double bn = 0.0;
#pragma unroll
          for (int i = 0; i < DIM; ++i) bn += cf.b_i(i, x) * nrm[i];
          wbn = w * bn;
        }
        sc1[slot] = w * sig - sgn * wbn;
        sc2[slot] = grad_terms ? -0.5 * sgn * w : 0.0;
      }
    };
    // contract k-steps [k0, k1) of the face table into the diagonal tiles and co
    auto face_contract = [&](int k0, int k1, double (&co)[NT][NT][2]) {
      PDG_UNROLL(PDG_FACE_UNROLL)
      for (int kk = k0; kk < k1; ++kk) {
        const int qq = kk * 4 + t;
        const double al = sc1[qq], be = sc2[qq];
        double va[NT], fa[NT], nvb[NT], fb[NT], l1[NT], l2[NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          va[i] = buf[(0 * NBP + i * 8 + g) * KFP + qq];
          nvb[i] = buf[(2 * NBP + i * 8 + g) * KFP + qq];
          if (grad_terms) {
            fa[i] = buf[(1 * NBP + i * 8 + g) * KFP + qq];
            fb[i] = buf[(3 * NBP + i * 8 + g) * KFP + qq];
            l1[i] = al * va[i] + be * fa[i];
            l2[i] = be * va[i];
          } else {
            fa[i] = fb[i] = l2[i] = 0.0;
            l1[i] = al * va[i];
          }
        }
        if constexpr (PK) {
          const double vA = buf[(0 * NBP + fA1) * KFP + qq], vB = buf[(0 * NBP + fB1) * KFP + qq];
          dmma(cd[0][0], l1[0], va[0]);
          if (grad_terms) {
            const double fA = buf[(1 * NBP + fA1) * KFP + qq], fB = buf[(1 * NBP + fB1) * KFP + qq];
            dmma(cd[0][0], l2[0], fa[0]);
            dmma(cd[0][1], al * vA + be * fA, vB);
            dmma(cd[0][1], be * vA, fB);
          } else {
            dmma(cd[0][1], al * vA, vB);
          }
        }
#pragma unroll
        for (int r = 0; r < NT; ++r)
#pragma unroll
          for (int cc = 0; cc < NT; ++cc) {
            if (!PK && (!SYM || cc >= r)) {
              dmma(cd[r][cc], l1[r], va[cc]);
              if (grad_terms) dmma(cd[r][cc], l2[r], fa[cc]);
            }
            dmma(co[r][cc], l1[r], nvb[cc]);
            if (grad_terms) dmma(co[r][cc], l2[r], fb[cc]);
          }
      }
    };

    PDG_T(3)
    for (int w0 = 0; w0 < nnb; w0 += NBR_WIN) {
      const int nw = min(NBR_WIN, nnb - w0);
      if (w0 == 0) {
        // this element's facet frames; the next element's copies stay in flight
        if (bulk) cp_async_wait_all();  // (the next element's copies are on the mbarrier)
        else asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        // windows beyond the first (more than NBR_WIN neighbours): synchronous restage
        __syncwarp();
        const double* rsrc = reinterpret_cast<const double*>(pat.nbr_rec + q0 + w0);
        for (int c = lane; c < nw * REC16; c += 32) cp_async16(reinterpret_cast<double*>(rc) + 2 * c, rsrc + 2 * c);
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
        issue_ffr(rc, nw, e);
        cp_async_commit();
        cp_async_wait_all();
      }
      __syncwarp();
      {
        const unsigned selfm = __ballot_sync(0xffffffffu, lane < nw && rc[lane].j == e);
        if (selfm) colself = rc[__ffs(selfm) - 1].col;
      }
      // col_idx of this window's column span, all rows (division-free)
      if (a.write_cols) {
        const int c0 = rc[0].col;
        const int c1 = rc[nw - 1].col + rc[nw - 1].nj;
        int q = 0;
        for (int p = c0 + lane; p < c1; p += 32) {
          while (q + 1 < nw && rc[q + 1].col <= p) ++q;
          const int64_t cv = rc[q].dof + (p - rc[q].col);
          int64_t* dst = pat.col_idx + voff + p;
#if PDG_COL_PTR
          // running pointer: one 64-bit add per row instead of a wide multiply-add
#pragma unroll 4
          for (int r = 0; r < ne; ++r, dst += Lrow) st_out<int64_t>(dst, cv);
#else
#pragma unroll 4
          for (int r = 0; r < ne; ++r) st_out<int64_t>(dst + (int64_t)r * Lrow, cv);
#endif
        }
      }
      PDG_T(4)
      int qi = 0;
      while (qi < nw) {
        if (rc[qi].j == e) {
          ++qi;
          continue;
        }
        int qb = qi + 1;
        if (qb < nw && rc[qb].j == e) ++qb;
        // a single-facet interface takes a paired round, with a partner when
        // the next one qualifies too, else alone (its half of the slots idle;
        // cheaper than the general path: staged frames, one contraction)
        // (a 3D face rule of degree >= 1 has >= 9 points: no paired rounds, and
        // leaving that code out of the 3D kernels keeps them smaller)
        constexpr bool PAIRS = DIM == 2 || P == 0;
        const bool pair = PAIRS && (rc[qi].info & 4) != 0;
        const bool has_b = qb < nw && (rc[qb].info & 4);
        double co[NT][NT][2];
        zero_tiles<NT>(co);
        if (pair) {
          // ---- two single-facet interfaces in one round
          const int seg = (slot >> 3) & (has_b ? 1 : 0), ls = slot & 7;
          const int q = seg ? qb : qi;
          const int info = rc[q].info;
          const int pj = rc[q].pj;
          const int order = 2 * max(pe, pj) + a.prm.quad_increment;
          const int r0 = R.face_offset[order], nq = R.face_count[order];
          double nrm[3] = {0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < DIM; ++i) nrm[i] = rc[q].nrm[i];
          const BoxConst<DIM> bo = STAGE_BOX ? load_box<DIM>(ebx, q) : load_box<DIM>(a.erec, rc[q].j);
          tab_slot(nrm, ffr + q * W::FF, r0, min(ls, nq - 1), (ls < nq && (has_b || slot < 8)) ? 1.0 : 0.0,
                   rc[q].sig, (info & 1) ? -1.0 : 1.0, (info & 2) != 0, bo);
          __syncwarp();
          PDG_T(5)
          face_contract(0, 2, co);
          store_block<NT, false>(a.values, voff, Lrow, rc[qi].col, ne, rc[qi].nj, co, g, t);
          if (has_b) {
            zero_tiles<NT>(co);
            face_contract(2, 4, co);
            store_block<NT, false>(a.values, voff, Lrow, rc[qb].col, ne, rc[qb].nj, co, g, t);
          }
          __syncwarp();
          PDG_T(6)
          qi = has_b ? qb + 1 : qi + 1;
          continue;
        }
        // ---- general interface: every face, every sub-facet, rounds of 16 points
        const int pj = rc[qi].pj;
        const BoxConst<DIM> bo = STAGE_BOX ? load_box<DIM>(ebx, qi) : load_box<DIM>(a.erec, rc[qi].j);
        const int order = 2 * max(pe, pj) + a.prm.quad_increment;
        const int r0 = R.face_offset[order], nq = R.face_count[order];
        const int fend = rc[qi].fb;
        for (int f = rc[qi].fa; f < fend; ++f) {
          int side, info;
          double sig;
          double nrm[3] = {0.0, 0.0, 0.0};
          int64_t row0;
          int nrows;
          if (f == rc[qi].fa) {
            info = rc[qi].info;
            side = info & 1;
            sig = rc[qi].sig;
#pragma unroll
            for (int i = 0; i < DIM; ++i) nrm[i] = rc[qi].nrm[i];
            row0 = rc[qi].row0;
            nrows = STAGE_BOX ? rc[qi].nrows0 : (int)(m.face_ptr[f + 1] - row0);
          } else {
            side = m.face_owner[f] == e ? 0 : 1;
            info = side | ((cf.has_adv() && a.flow[f] == side) ? 2 : 0);
            sig = a.sigma[f];
#pragma unroll
            for (int i = 0; i < DIM; ++i) nrm[i] = m.face_normal[(int64_t)f * DIM + i];
            row0 = m.face_ptr[f];
            nrows = (int)(m.face_ptr[f + 1] - row0);
          }
          const bool first_face = STAGE_BOX && f == rc[qi].fa;
          const int Pf = nrows * nq;
          const float rnq = 1.0f / (float)nq;
          for (int base = 0; base < Pf; base += KF) {
            const int nvalid = min(KF, Pf - base);
            const int gq = base + min(slot, nvalid - 1);
            const int lr = small_div(gq, nq, rnq);
            // the first sub-facet frame of the interface is staged (ffr)
            const double* frp = (first_face && lr == 0) ? ffr + qi * W::FF : a.fframe + (row0 + lr) * W::FF;
            tab_slot(nrm, frp, r0, gq - lr * nq, slot < nvalid ? 1.0 : 0.0, sig, side ? -1.0 : 1.0,
                     (info & 2) != 0, bo);
            __syncwarp();
            face_contract(0, (nvalid + 3) >> 2, co);
            __syncwarp();
          }
        }
        store_block<NT, false>(a.values, voff, Lrow, rc[qi].col, ne, rc[qi].nj, co, g, t);
        PDG_T(9)
        ++qi;
      }
      __syncwarp();
    }

    PDG_T(4)
    // ------------------------------------------------------------ boundary faces
    const int64_t bend = mode ? 0 : m.elem_bface_ptr[e + 1];
    for (int64_t bi = mode ? 0 : m.elem_bface_ptr[e]; bi < bend; ++bi) {
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
      const float rnq = 1.0f / (float)nq;
      const int slot = lane & (KF - 1);
      const bool mine = lane < KF;
      const bool use_f = tag == PDG_TAG_DIRICHLET && grad_terms;
      for (int base = 0; base < Pf; base += KF) {
        const int nvalid = min(KF, Pf - base);
        {
          const int gq = base + min(slot, nvalid - 1);
          const double valid = (slot < nvalid && mine) ? 1.0 : 0.0;
          const int lr = small_div(gq, nq, rnq);
          const int kq = gq - lr * nq;
          const double* xi = RV.pts + (r0 + kq) * 3;
          double x[3] = {0.0, 0.0, 0.0};
          const double jac = frame_point<DIM, DIM - 1>(a.fframe + (row0 + lr) * W::FF, xi, x);
          const double w = RV.w[r0 + kq] * jac * valid;
          Tab<DIM, P> tb;
          tb.load(bx, x);
          double av = 1.0;
          double A[DIM][DIM];
          if (use_f) {
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
          if ((wi || tag == PDG_TAG_INFLOW) && cf.has_adv()) {
            double bn = 0.0;
#pragma unroll
            for (int i = 0; i < DIM; ++i) bn += cf.b_i(i, x) * nrm[i];
            wbn = w * bn;
          }
          double al = 0.0, be = 0.0, gval = 0.0;
          if (tag == PDG_TAG_DIRICHLET) {
            al = w * sig - (wi ? wbn : 0.0);
            be = use_f ? -w : 0.0;
            gval = cf.has_dir() ? cf.gD(x) : 0.0;
          } else if (tag == PDG_TAG_INFLOW) {
            al = -wbn;
            gval = cf.has_dir() ? cf.gD(x) : 0.0;
          } else {  // Neumann: load only
            gval = w * cf.gN(x);
          }
          double* col = buf + slot;
#pragma unroll
          for (int ff = 0; ff < NBW; ++ff) {
            double vv = 0.0, fl = 0.0;
            if (ff < NB) {
              vv = tb.val(ff);
              if (use_f) fl = face_flux<DIM, P>(cf, tb, ff, nrm, av, A);
              if (mine) {
                if (tag == PDG_TAG_NEUMANN) rhs_add(ff, gval * vv);
                else if (cf.has_dir()) rhs_add(ff, gval * (al * vv + be * fl));
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
            if constexpr (PK) {
              const double vA = buf[(0 * NBP + fA1) * KFP + qq], vB = buf[(0 * NBP + fB1) * KFP + qq];
              const double fA = buf[(1 * NBP + fA1) * KFP + qq], fB = buf[(1 * NBP + fB1) * KFP + qq];
              dmma(cd[0][0], l1[0], va[0]);
              dmma(cd[0][1], al * vA + be * fA, vB);
              if (use_f) {
                dmma(cd[0][0], l2[0], fa[0]);
                dmma(cd[0][1], be * vA, fB);
              }
            } else {
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
        }
        __syncwarp();
      }
    }

    PDG_T(7)
    // ------------------------------------------------------------ write-out
    if constexpr (PK) {
      double c00[1][1][2] = {{{cd[0][0][0], cd[0][0][1]}}};
      store_block<1, true>(a.values, voff, Lrow, colself, ne, ne, c00, g, t);
      store_packed10(a.values, voff, Lrow, colself, ne, cd[0][1], g, t);
    } else {
      store_block<NT, SYM>(a.values, voff, Lrow, colself, ne, ne, cd, g, t);
    }
    double* rhs_out = mode ? a.rhs + k * NB : a.rhs + dof_e;
    __syncwarp();
    if constexpr (S::RHS_REGS && NB <= 16) {
      // transpose-reduce across the warp: four halving exchanges (lane bits
      // 16, 8, 4, 2) leave each lane one function's partial over 16 lanes, the
      // last exchange (bit 1) completes it -- 16 shuffles, no shared memory
      double v[16];
#pragma unroll
      for (int f = 0; f < 16; ++f) v[f] = f < NB ? racc[f] : 0.0;
#pragma unroll
      for (int w = 8, bit = 16; w >= 1; w >>= 1, bit >>= 1) {
        const bool hi = (lane & bit) != 0;
#pragma unroll
        for (int i = 0; i < w; ++i) {
          const double send = hi ? v[i] : v[i + w];
          const double keep = hi ? v[i + w] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
        }
      }
      const double tot = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
      const int f = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
      if (!(lane & 1) && f < ne) rhs_out[f] = tot;
    } else if constexpr (S::RHS_REGS) {
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
    PDG_T(8)
  }
  if (PDG_TIMERS && lane == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2) && threadIdx.x < 64) {
    const double n = nel_done > 0 ? nel_done : 1;
    printf("PDG_TIMERS blk %d warp %d elements %d per-element cycles: start %.0f voltab %.0f volmma %.0f post %.0f "
           "window %.0f facetab %.0f facemma %.0f boundary %.0f writeout %.0f general %.0f\n",
           blockIdx.x, threadIdx.x >> 5, nel_done, tacc[0] / n, tacc[1] / n, tacc[2] / n, tacc[3] / n, tacc[4] / n,
           tacc[5] / n, tacc[6] / n, tacc[7] / n, tacc[8] / n, tacc[9] / n);
  }
}

}  // namespace pdg
