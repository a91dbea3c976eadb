// Device-side data structures and fp64 helpers of the 2D engine.
//
// Every helper evaluates, per element, the same expression DAG as the
// reference numpy code it cites (paths relative to
// /root/reference/pkg/src/treemg).  The library is compiled with
// --fmad=false so no multiply-add is ever contracted: numpy rounds
// `out += c*x` twice and so must we.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tmg {

// vertex classes (spacetree.py:67-72) in flags bits 0..2
enum : uint8_t { K_NONE = 0, K_DOF = 1, K_DIR = 2, K_HANG = 3, K_OVER = 4 };
// flags bit 3: an adjacent cell of this level is refined (hweight, solvers.py:197-208)
constexpr uint8_t F_NEAR = 8;
// flags bit 4: injection target -- the fine c-point above is INTERIOR_DOF or
// COARSE_OVERLAPPED (solvers.py:285-288)
constexpr uint8_t F_TAKE = 16;

__device__ __forceinline__ int kind_of(uint8_t f) { return f & 7; }
__device__ __forceinline__ bool is_dof(uint8_t f) { int k = f & 7; return k == K_DOF || k == K_OVER; }
__device__ __forceinline__ bool is_src(uint8_t f) { int k = f & 7; return k == K_DOF || k == K_OVER || k == K_HANG; }

enum OpKind : int { OP_CONST = 0, OP_ELEMENT = 1, OP_TABLE = 2, OP_NONE = 3 };
enum RtMode : int { RT_NONE = 0, RT_GEOM_FAST = 1, RT_TABLE = 2 };

// A level operator: ElementOperator (const fast path or per-cell eps) or
// TableOperator (operators.py:164-248).
struct OpView {
  int kind;
  double s_side;  // (eps/3.0)*-1.0  (discretization.py:165-167)
  double s_mid;   // (eps/3.0)*8.0
  const double* eps;  // per cell, n*n (OP_ELEMENT)
  const double* tbl;  // 9 planes of (n+1)^2 (OP_TABLE), plane k = a*3+b
};

// Constant tables (the library is one translation unit, engine.cu).
// element matrix (discretization.py:40-47), corner order (0,0),(1,0),(0,1),(1,1)
__constant__ double c_E[16];
// d-linear 1D restriction weights [1,2,3,2,1]/3 (operators.py:93)
__constant__ double c_W5[5];
// d-linear prolongation weights wl = 1 - r/3 and 1 - wl for r = 0,1,2 (operators.py:101-107)
__constant__ double c_WL[3];
__constant__ double c_WR[3];
// unit-operator taps times 3/8: a1[s]*inv (operators.py:520-531)
__constant__ double c_A1INV[9];

// ---------------------------------------------------------------------------
// Stencil application at one vertex (i, j) of a level with N = n+1 vertices.

// apply_constant_stencil (operators.py:143-161): taps (a,b) row-major,
// zero-extended, accumulated from 0.
__device__ __forceinline__ double apply_const_at(const double* __restrict__ x, int N, int i, int j,
                                                 double s_side, double s_mid) {
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int ii = i + a - 1;
    if (ii < 0 || ii >= N) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      int jj = j + b - 1;
      if (jj < 0 || jj >= N) continue;
      double c = (a == 1 && b == 1) ? s_mid : s_side;
      acc = acc + c * x[(size_t)ii * N + jj];
    }
  }
  return acc;
}

// ElementOperator.apply (operators.py:178-188): corner a outer, b inner.
__device__ __forceinline__ double apply_element_at(const double* __restrict__ x,
                                                   const double* __restrict__ eps, int N, int i,
                                                   int j) {
  const int n = N - 1;
  double out = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int a0 = a & 1, a1 = a >> 1;
    const int ci = i - a0, cj = j - a1;
    if (ci < 0 || cj < 0 || ci >= n || cj >= n) continue;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int b0 = b & 1, b1 = b >> 1;
      acc = acc + c_E[a * 4 + b] * x[(size_t)(ci + b0) * N + (cj + b1)];
    }
    out = out + eps[(size_t)ci * n + cj] * acc;
  }
  return out;
}

// TableOperator.apply (operators.py:229-239): taps row-major, in-range only.
__device__ __forceinline__ double apply_table_at(const double* __restrict__ x,
                                                 const double* __restrict__ tbl, int N, int i,
                                                 int j) {
  const size_t nv = (size_t)N * N;
  const size_t v = (size_t)i * N + j;
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int ii = i + a - 1;
    if (ii < 0 || ii >= N) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      int jj = j + b - 1;
      if (jj < 0 || jj >= N) continue;
      acc = acc + tbl[(size_t)(a * 3 + b) * nv + v] * x[(size_t)ii * N + jj];
    }
  }
  return acc;
}

__device__ __forceinline__ double apply_op_at(const OpView& op, const double* __restrict__ x,
                                              int N, int i, int j) {
  if (op.kind == OP_CONST) return apply_const_at(x, N, i, j, op.s_side, op.s_mid);
  if (op.kind == OP_ELEMENT) return apply_element_at(x, op.eps, N, i, j);
  if (op.kind == OP_TABLE) return apply_table_at(x, op.tbl, N, i, j);
  return 0.0;
}

// ---------------------------------------------------------------------------
// d-linear transfers.

// restrict_dlinear at coarse (I,J) (operators.py:111-132): axis-0 pass then
// axis-1 pass, offsets -2..2, in-range terms only, each pass from 0.
__device__ __forceinline__ double restrict_dlinear_at(const double* __restrict__ f, int Nf, int I,
                                                      int J) {
  const int m = (Nf - 1) / 3;
  double out = 0.0;
#pragma unroll
  for (int oj = -2; oj <= 2; ++oj) {
    if ((oj < 0 && J < 1) || (oj > 0 && J > m - 1)) continue;
    const int jf = 3 * J + oj;
    double t = 0.0;
#pragma unroll
    for (int oi = -2; oi <= 2; ++oi) {
      if ((oi < 0 && I < 1) || (oi > 0 && I > m - 1)) continue;
      t = t + c_W5[oi + 2] * f[(size_t)(3 * I + oi) * Nf + jf];
    }
    out = out + c_W5[oj + 2] * t;
  }
  return out;
}

// prolong_values at fine (i,j) (operators.py:96-127):
// axis 0: T = wl*c[q] + (1-wl)*c[qn]; then axis 1 on T.
__device__ __forceinline__ double prolong_dlinear_at(const double* __restrict__ c, int Nc, int i,
                                                     int j) {
  const int m = Nc - 1;
  const int qi = i / 3, ri = i - 3 * qi, qni = min(qi + 1, m);
  const int qj = j / 3, rj = j - 3 * qj, qnj = min(qj + 1, m);
  const double wli = c_WL[ri], wri = c_WR[ri];
  const double t0 = wli * c[(size_t)qi * Nc + qj] + wri * c[(size_t)qni * Nc + qj];
  const double t1 = wli * c[(size_t)qi * Nc + qnj] + wri * c[(size_t)qni * Nc + qnj];
  return c_WL[rj] * t0 + c_WR[rj] * t1;
}

// ---------------------------------------------------------------------------
// Operator-dependent transfers; P is stored compactly as 25 planes of the
// coarse vertex grid, plane (oi+2)*5+(oj+2) for fine offsets -2..2 (offsets
// +-3 of the reference's 7x7 table are identically zero:
// operators.py:325-436 never writes them except with d-linear weight 0).

// TransferOps.prolong with a P table (operators.py:570-581, 625-631):
// contributions in (oi, oj) row-major order == coarse I descending.
__device__ __forceinline__ double prolong_table_at(const double* __restrict__ c,
                                                   const double* __restrict__ P, int Nc, int i,
                                                   int j) {
  const size_t nvc = (size_t)Nc * Nc;
  const int qi = i / 3, ri = i - 3 * qi;
  const int qj = j / 3, rj = j - 3 * qj;
  double acc = 0.0;
  for (int di = (ri > 0 ? 1 : 0); di >= 0; --di) {
    const int I = qi + di, oi = i - 3 * I;
    for (int dj = (rj > 0 ? 1 : 0); dj >= 0; --dj) {
      const int J = qj + dj, oj = j - 3 * J;
      const size_t vc = (size_t)I * Nc + J;
      acc = acc + P[(size_t)((oi + 2) * 5 + (oj + 2)) * nvc + vc] * c[vc];
    }
  }
  return acc;
}

// TransferOps.restrict with a P table (operators.py:586-596): 5x5 taps row-major.
__device__ __forceinline__ double restrict_table_at(const double* __restrict__ f, int Nf,
                                                    const double* __restrict__ P, int Nc, int I,
                                                    int J) {
  const size_t nvc = (size_t)Nc * Nc;
  const size_t vc = (size_t)I * Nc + J;
  double out = 0.0;
#pragma unroll
  for (int oi = -2; oi <= 2; ++oi) {
    const int fi = 3 * I + oi;
    if (fi < 0 || fi >= Nf) continue;
#pragma unroll
    for (int oj = -2; oj <= 2; ++oj) {
      const int fj = 3 * J + oj;
      if (fj < 0 || fj >= Nf) continue;
      out = out + P[(size_t)((oi + 2) * 5 + (oj + 2)) * nvc + vc] * f[(size_t)fi * Nf + fj];
    }
  }
  return out;
}

// restrict_smoothed with a per-vertex 7x7 table (operators.py:606-613).
__device__ __forceinline__ double restrict_rt_table_at(const double* __restrict__ f, int Nf,
                                                       const double* __restrict__ Rt, int Nc,
                                                       int I, int J) {
  const size_t nvc = (size_t)Nc * Nc;
  const size_t vc = (size_t)I * Nc + J;
  double out = 0.0;
  for (int oi = -3; oi <= 3; ++oi) {
    const int fi = 3 * I + oi;
    if (fi < 0 || fi >= Nf) continue;
#pragma unroll
    for (int oj = -3; oj <= 3; ++oj) {
      const int fj = 3 * J + oj;
      if (fj < 0 || fj >= Nf) continue;
      out = out + Rt[(size_t)((oi + 3) * 7 + (oj + 3)) * nvc + vc] * f[(size_t)fi * Nf + fj];
    }
  }
  return out;
}

// Geometric fast path of restrict_smoothed (operators.py:602-605):
// R( (A1 f) * s ) with A1 the unit 9-point stencil, s = omega*3.0/8.0.
__device__ __forceinline__ double restrict_rt_geom_at(const double* __restrict__ f, int Nf, int I,
                                                      int J, double s_side, double s_mid,
                                                      double scale) {
  const int m = (Nf - 1) / 3;
  double out = 0.0;
  for (int oj = -2; oj <= 2; ++oj) {
    if ((oj < 0 && J < 1) || (oj > 0 && J > m - 1)) continue;
    const int jf = 3 * J + oj;
    double t = 0.0;
    for (int oi = -2; oi <= 2; ++oi) {
      if ((oi < 0 && I < 1) || (oi > 0 && I > m - 1)) continue;
      const double sm = apply_const_at(f, Nf, 3 * I + oi, jf, s_side, s_mid) * scale;
      t = t + c_W5[oi + 2] * sm;
    }
    out = out + c_W5[oj + 2] * t;
  }
  return out;
}

}  // namespace tmg
