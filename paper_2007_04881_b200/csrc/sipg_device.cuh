// Device building blocks of the SIPG assembly engine (sm_100a, fp64).
//
//  * coefficient bytecode interpreter        (model.py Expr -> eval_prog)
//  * affine quadrature maps                   (polydg quadrature.py:118-156)
//  * bounding-box Legendre tabulation         (polydg basis.py:107-164)
//  * DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) fragment helpers
//
// B200 facts that shape this file (profiles/fp64_peaks_r01.json): DFMA and
// DMMA share one FP64 pipe (37 TF/s each, not additive), so every fp64
// instruction outside the contraction (tabulation, coefficients, maps) is
// charged against the same 64 FMA/clk/SM budget; DMMA is used for the
// contraction because it issues 256 FMA per instruction from 2 operand
// registers per thread, leaving issue slots and registers for the rest.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#endif

#include "../../include/pdg.h"

#define PDG_INF __longlong_as_double(0x7ff0000000000000LL)

namespace pdg {

enum Op : int {
  OP_CONST = 0, OP_COORD, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_NEG,
  OP_SIN, OP_COS, OP_EXP, OP_LOG, OP_SQRT, OP_POW, OP_ABS, OP_TANH
};

__device__ __forceinline__ void raise_flag(uint32_t* flags, uint32_t bit) {
  if (flags) atomicOr(flags, bit);
}

// floor(a / b) for 0 <= a < 2^22, 1 <= b, with rb = 1.0f / b: (a + 1/2) / b is
// at least 1/(2b) away from an integer, more than the float rounding error
// (<= 2^-23 (a + 1/2) / b), so the truncation is exact.  ~4 instructions
// against ~20 for a runtime integer division (the volume round's
// point -> simplex split was 2.7% of the cfg5 kernel's instructions).
#ifndef PDG_FAST_DIV
#define PDG_FAST_DIV 1
#endif
__device__ __forceinline__ int small_div(int a, int b, float rb) {
#if PDG_FAST_DIV
  return (int)(((float)a + 0.5f) * rb);
#else
  return a / b;
#endif
}

// sin(pi x) / cos(pi x) of the runtime-specialised volume fields (model.py
// lowers sin/cos((k pi) u) to these).  Reduction r = x - rint(x) in [-1/2, 1/2]
// is exact; sin(pi r) is the odd Taylor polynomial to r^23 (truncation below
// 1e-18; <= 1.5 ulp against mpmath over [-3, 3]); cos(pi r) = sin(pi (1/2 - |r|))
// (exact argument, so cospi(1/2) = 0); the sign is the parity of rint(x).
// About 17 instructions against ~35 for CUDA's sinpi: the cfg5 source term
// sin(pi x) sin(pi y) was 10% of the element kernel's instructions (r02 ncu).
// PDG_FAST_SINPI=0 selects CUDA's sinpi / cospi.
#ifndef PDG_FAST_SINPI
#define PDG_FAST_SINPI 1
#endif
__device__ __forceinline__ double sinpi_reduced(double r) {
  const double s = r * r;
  double p = -1.0518471716932065e-11;
  p = fma(p, s, 5.392664662608129e-10);
  p = fma(p, s, -2.2948428997269873e-08);
  p = fma(p, s, 7.952054001475513e-07);
  p = fma(p, s, -2.1915353447830217e-05);
  p = fma(p, s, 0.00046630280576761255);
  p = fma(p, s, -0.0073704309457143504);
  p = fma(p, s, 0.08214588661112823);
  p = fma(p, s, -0.5992645293207921);
  p = fma(p, s, 2.5501640398773455);
  p = fma(p, s, -5.16771278004997);
  p = fma(p, s, 3.141592653589793);
  return r * p;
}
__device__ __forceinline__ double pdg_sinpi(double x) {
#if PDG_FAST_SINPI
  const double q = rint(x);
  const double v = sinpi_reduced(x - q);  // inf / nan -> nan
  const long long qi = fabs(q) < 9.0e18 ? (long long)q : 0;  // beyond 2^53 every double is even
  return (qi & 1) ? -v : v;
#else
  return sinpi(x);
#endif
}
__device__ __forceinline__ double pdg_cospi(double x) {
#if PDG_FAST_SINPI
  const double q = rint(x);
  const double v = sinpi_reduced(0.5 - fabs(x - q));
  const long long qi = fabs(q) < 9.0e18 ? (long long)q : 0;
  return (qi & 1) ? -v : v;
#else
  return cospi(x);
#endif
}

// Evaluate one compiled scalar field at x (stack machine; host guarantees
// the depth fits PDG_MAX_STACK).
static __device__ __noinline__ double eval_prog_slow(const pdg_coeffs& C, const pdg_prog p,
                                              double x0, double x1, double x2) {
  double st[PDG_MAX_STACK];
  int sp = 0;
  for (int i = 0; i < p.length; ++i) {
    const int ins = C.code[p.offset + i];
    const int op = ins & 0xff, arg = ins >> 8;
    switch (op) {
      case OP_CONST: st[sp++] = C.consts[arg]; break;
      case OP_COORD: st[sp++] = arg == 0 ? x0 : (arg == 1 ? x1 : x2); break;
      case OP_ADD: --sp; st[sp - 1] = st[sp - 1] + st[sp]; break;
      case OP_SUB: --sp; st[sp - 1] = st[sp - 1] - st[sp]; break;
      case OP_MUL: --sp; st[sp - 1] = st[sp - 1] * st[sp]; break;
      case OP_DIV: --sp; st[sp - 1] = st[sp - 1] / st[sp]; break;
      case OP_POW: --sp; st[sp - 1] = (st[sp] == 2.0) ? st[sp - 1] * st[sp - 1]
                                                       : pow(st[sp - 1], st[sp]); break;
      case OP_NEG: st[sp - 1] = -st[sp - 1]; break;
      case OP_SIN: st[sp - 1] = sin(st[sp - 1]); break;
      case OP_COS: st[sp - 1] = cos(st[sp - 1]); break;
      case OP_EXP: st[sp - 1] = exp(st[sp - 1]); break;
      case OP_LOG: st[sp - 1] = log(st[sp - 1]); break;
      case OP_SQRT: st[sp - 1] = sqrt(st[sp - 1]); break;
      case OP_ABS: st[sp - 1] = fabs(st[sp - 1]); break;
      case OP_TANH: st[sp - 1] = tanh(st[sp - 1]); break;
      default: break;
    }
  }
  return st[0];
}

__device__ __forceinline__ double eval_prog(const pdg_coeffs& C, const pdg_prog& p,
                                            const double* x) {
  if (p.is_const) return p.value;
  return eval_prog_slow(C, p, x[0], x[1], x[2]);
}

// Ahead-of-time coefficient policy: interprets the bytecode in pdg_coeffs.
template <int DIM>
struct InterpCoef {
  const pdg_coeffs& C;
  __device__ InterpCoef(const pdg_coeffs& c) : C(c) {}
  __device__ int diff_kind() const { return C.diffusion_kind; }
  __device__ bool a_const() const {
    if (C.diffusion_kind == PDG_DIFF_ISO) return C.diffusion[0].is_const;
    for (int k = 0; k < DIM * DIM; ++k)
      if (!C.diffusion[k].is_const) return false;
    return true;
  }
  __device__ bool has_adv() const { return C.has_advection; }
  __device__ bool has_reac() const { return C.has_reaction; }
  __device__ bool has_src() const { return C.has_source; }
  __device__ bool has_dir() const { return C.has_dirichlet; }
  __device__ bool has_neu() const { return C.has_neumann; }
  __device__ double a_iso(const double* x) const { return eval_prog(C, C.diffusion[0], x); }
  __device__ double a_ij(int i, int j, const double* x) const { return eval_prog(C, C.diffusion[i * DIM + j], x); }
  __device__ double b_i(int i, const double* x) const { return eval_prog(C, C.advection[i], x); }
  __device__ double c(const double* x) const { return eval_prog(C, C.reaction, x); }
  __device__ double f(const double* x) const { return eval_prog(C, C.source, x); }
  __device__ double gD(const double* x) const { return eval_prog(C, C.dirichlet, x); }
  __device__ double gN(const double* x) const { return eval_prog(C, C.neumann, x); }
};

// ---------------------------------------------------------------------------
// compile-time basis tables (graded-lex multi-indices, basis.py:86-104)
// ---------------------------------------------------------------------------

__host__ __device__ constexpr int binom(int n, int k) {
  int r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

template <int DIM, int P>
struct MultiIdx {
  static constexpr int NB = binom(P + DIM, DIM);
  int a[NB][3];
  __host__ __device__ constexpr MultiIdx() : a{} {
    int f = 0;
    for (int tot = 0; tot <= P; ++tot) {
      if (DIM == 2) {
        for (int i = 0; i <= tot; ++i) { a[f][0] = i; a[f][1] = tot - i; a[f][2] = 0; ++f; }
      } else {
        for (int i = 0; i <= tot; ++i)
          for (int j = 0; j <= tot - i; ++j) { a[f][0] = i; a[f][1] = j; a[f][2] = tot - i - j; ++f; }
      }
    }
  }
};

// Per-element basis constants: box centre, 1/half-width, 1/sqrt(width).
template <int DIM>
struct BoxConst {
  double c[DIM], ih[DIM], rs[DIM];
};

template <int DIM>
__device__ __forceinline__ BoxConst<DIM> box_const(const double* box /*[2][DIM]*/) {
  BoxConst<DIM> b;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    const double lo = box[i], hi = box[DIM + i];
    b.c[i] = 0.5 * (lo + hi);
    b.ih[i] = 1.0 / (0.5 * (hi - lo));
    b.rs[i] = 1.0 / sqrt(hi - lo);
  }
  return b;
}

// 1D orthonormal Legendre values and derivatives on one box side.
// polydg (basis.py:107-126,146-152) runs the three-term recurrence
//   L_{k+1} = (2k+1)/(k+1) t L_k - k/(k+1) L_{k-1},  L'_{k+1} = (2k+1) L_k + L'_{k-1}
// and scales afterwards by s_k = sqrt(2k+1)/sqrt(width) (and 1/half for L').
// Here the recurrence runs directly on the scaled values v_k = s_k L_k,
// dv_k = s_k L'_k / half: the ratios s_{k+1}/s_k are element independent
// (the width cancels), so the scaling costs nothing per point.  Same values
// up to rounding (<= a few ulp).  dv_0 = 0 is never formed (Tab::grad).
template <int P>
__device__ __forceinline__ void legendre_1d(double t, double rs, double ih, double* v, double* dv) {
  v[0] = rs;
  dv[0] = 0.0;
  if (P >= 1) {
    const double r1 = 1.7320508075688772 * rs;  // sqrt(3) / sqrt(width)
    v[1] = r1 * t;
    dv[1] = r1 * ih;
  }
#pragma unroll
  for (int k = 1; k < P; ++k) {
    const double up = sqrt(double(2 * k + 3) / double(2 * k + 1));   // s_{k+1} / s_k
    const double up2 = sqrt(double(2 * k + 3) / double(2 * k - 1));  // s_{k+1} / s_{k-1}
    const double c1 = double(2 * k + 1) / double(k + 1) * up;
    const double c2 = double(k) / double(k + 1) * up2;
    v[k + 1] = (c1 * t) * v[k] - c2 * v[k - 1];
    const double g = double(2 * k + 1) * up;
    dv[k + 1] = k == 1 ? g * (ih * v[1]) : g * (ih * v[k]) + up2 * dv[k - 1];
  }
}

// Tabulate all NB basis values / gradients at physical point x.
template <int DIM, int P>
struct Tab {
  static constexpr int NB = binom(P + DIM, DIM);
  double v1[DIM][P + 1], d1[DIM][P + 1];

  // s0 scales every function (the dim-0 factors, through the recurrence's start)
  __device__ __forceinline__ void load(const BoxConst<DIM>& b, const double* x, double s0 = 1.0) {
#pragma unroll
    for (int i = 0; i < DIM; ++i)
      legendre_1d<P>((x[i] - b.c[i]) * b.ih[i], i == 0 ? b.rs[i] * s0 : b.rs[i], b.ih[i], v1[i], d1[i]);
  }
  // multiply every basis function (and gradient) by s: scale the dim-0 factors
  __device__ __forceinline__ void scale(double s) {
#pragma unroll
    for (int k = 0; k <= P; ++k) {
      v1[0][k] *= s;
      d1[0][k] *= s;
    }
  }
  __device__ __forceinline__ double val(int f) const {
    constexpr MultiIdx<DIM, P> mi{};
    double r = v1[0][mi.a[f][0]] * v1[1][mi.a[f][1]];
    if (DIM == 3) r *= v1[2][mi.a[f][2]];
    return r;
  }
  __device__ __forceinline__ double grad(int f, int k) const {
    constexpr MultiIdx<DIM, P> mi{};
    if (mi.a[f][k] == 0) return 0.0;  // derivative of the constant mode (compile-time)
    double r = (k == 0 ? d1[0][mi.a[f][0]] : v1[0][mi.a[f][0]]) *
               (k == 1 ? d1[1][mi.a[f][1]] : v1[1][mi.a[f][1]]);
    if (DIM == 3) r *= (k == 2 ? d1[2][mi.a[f][2]] : v1[2][mi.a[f][2]]);
    return r;
  }
};

// ---------------------------------------------------------------------------
// quadrature maps
// ---------------------------------------------------------------------------

// Affine map of the reference simplex onto simplex `s`: E rows = v_k - v_0,
// returns |det E| (and flags degeneracy like quadrature.py:131-134).
template <int DIM>
__device__ __forceinline__ double simplex_frame(const pdg_mesh& m, int s, double* v0, double E[][3],
                                                uint32_t* flags) {
  const int32_t* sv = m.simplices + (int64_t)s * (DIM + 1);
  const double* p0 = m.vertices + (int64_t)sv[0] * DIM;
#pragma unroll
  for (int i = 0; i < DIM; ++i) v0[i] = p0[i];
  double scale = 0.0;
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    const double* pk = m.vertices + (int64_t)sv[k + 1] * DIM;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      E[k][i] = pk[i] - v0[i];
      scale = fmax(scale, fabs(E[k][i]));
    }
  }
  double det;
  if (DIM == 2) {
    det = E[0][0] * E[1][1] - E[0][1] * E[1][0];
  } else {
    det = E[0][0] * (E[1][1] * E[2][2] - E[1][2] * E[2][1]) -
          E[0][1] * (E[1][0] * E[2][2] - E[1][2] * E[2][0]) +
          E[0][2] * (E[1][0] * E[2][1] - E[1][1] * E[2][0]);
  }
  det = fabs(det);
  if (scale == 0.0) scale = 1.0;
  double sd = scale * scale;
  if (DIM == 3) sd *= scale;
  if (det < 1e-14 * sd) raise_flag(flags, PDG_FLAG_DEGENERATE_SIMPLEX);
  return det;
}

// Sub-facet frame: d vertices in R^d, returns sqrt(det(E E^T)) (quadrature.py:147-156).
template <int DIM>
__device__ __forceinline__ double facet_frame(const pdg_mesh& m, int64_t row, double* v0, double E[][3],
                                              uint32_t* flags) {
  const int32_t* fv = m.facet_vertices + row * DIM;
  const double* p0 = m.vertices + (int64_t)fv[0] * DIM;
#pragma unroll
  for (int i = 0; i < DIM; ++i) v0[i] = p0[i];
#pragma unroll
  for (int k = 0; k < DIM - 1; ++k) {
    const double* pk = m.vertices + (int64_t)fv[k + 1] * DIM;
#pragma unroll
    for (int i = 0; i < DIM; ++i) E[k][i] = pk[i] - v0[i];
  }
  double g;
  if (DIM == 2) {
    g = E[0][0] * E[0][0] + E[0][1] * E[0][1];
  } else {
    double g00 = 0, g01 = 0, g11 = 0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      g00 += E[0][i] * E[0][i];
      g01 += E[0][i] * E[1][i];
      g11 += E[1][i] * E[1][i];
    }
    g = g00 * g11 - g01 * g01;
  }
  if (!(g > 0.0)) raise_flag(flags, PDG_FLAG_DEGENERATE_FACET);
  return sqrt(fmax(g, 0.0));
}

// x = v0 + xi E from a frame record (v0 then E rows), returns the stored measure
template <int DIM, int K>
__device__ __forceinline__ double frame_point(const double* fr, const double* xi, double* x) {
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    double acc = fr[i];
#pragma unroll
    for (int j = 0; j < K; ++j) acc += xi[j] * fr[DIM + j * DIM + i];
    x[i] = acc;
  }
  return fr[DIM + K * DIM];
}

// ---------------------------------------------------------------------------
// DMMA m8n8k4 (fp64):  D(8x8) += A(8x4) * B(4x8)
//   lane = 4*g + t :  a = A[g][t],  b = B[t][g],  c0/c1 = C[g][2t], C[g][2t+1]
// With A[i][k] = L_i(item k) and B[k][j] = R_j(item k), a thread that owns
// (function f0+g, item k0+t) feeds both operands from the same table slot.
// ---------------------------------------------------------------------------
// PDG_DMMA_VOLATILE=0 lets the compiler reorder independent DMMAs (tuning knob)
#ifndef PDG_DMMA_VOLATILE
#define PDG_DMMA_VOLATILE 1
#endif
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
#if PDG_DMMA_VOLATILE
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
#else
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
#endif
}

}  // namespace pdg
