// Device-side data structures and fp64 helpers of the 2D engine.
//
// Every helper evaluates, per element, the same expression DAG as the
// reference numpy code it cites (paths relative to
// /root/reference/pkg/src/treemg).  The library is compiled with
// --fmad=false so no multiply-add is ever contracted: numpy rounds
// `out += c*x` twice and so must we.
//
// Latency structure: each helper first issues every load it needs
// (predicated, fully unrolled) and only then runs the order-exact
// accumulation chain, so a gather costs one memory round trip instead of one
// per tap.  Out-of-range taps are skipped by predicate (never added as 0).
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
// R~ application: none / geometric fast path (operators.py:602-605) / stored
// per-vertex table (operators.py:606-613) / table rebuilt from the P weights
// in registers (BoxMG, unit-coefficient R~; bit-identical to the table).
enum RtMode : int { RT_NONE = 0, RT_GEOM_FAST = 1, RT_TABLE = 2, RT_FROM_P = 3 };

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

// Load policies: LdNC reads through the non-coherent read-only path (data
// not written during the kernel); LdCG reads from L2 (data produced by other
// CTAs of the same kernel, after a barrier with release/acquire semantics).
struct LdNC {
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
};
struct LdCG {
  static __device__ __forceinline__ double ld(const double* p) { return __ldcg(p); }
};

__device__ __forceinline__ bool inside(int i, int j, int N) {
  return i >= 0 && j >= 0 && i < N && j < N;
}

// Range test that compiles away (CHK == false) for vertices whose whole
// stencil / transfer footprint is known to lie inside the grid.
template <bool CHK>
__device__ __forceinline__ bool in_rng(int i, int j, int N) {
  return !CHK || inside(i, j, N);
}

// ---------------------------------------------------------------------------
// Stencil application at one vertex (i, j) of a level with N = n+1 vertices.

// 3x3 neighbourhood of x around (i, j), zero outside (predicated loads).
template <class LD, bool CHK = true>
__device__ __forceinline__ void load3x3(const double* x, int N, int i, int j,
                                        double v[9]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int ii = i + k / 3 - 1, jj = j + k % 3 - 1;
    v[k] = in_rng<CHK>(ii, jj, N) ? LD::ld(x + (size_t)ii * N + jj) : 0.0;
  }
}

// apply_constant_stencil (operators.py:143-161): taps (a,b) row-major,
// zero-extended (out-of-range taps skipped), accumulated from 0.
template <bool CHK = true>
__device__ __forceinline__ double const_from(const double v[9], int N, int i, int j, double s_side,
                                             double s_mid) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int ii = i + k / 3 - 1, jj = j + k % 3 - 1;
    if (in_rng<CHK>(ii, jj, N)) acc = acc + (k == 4 ? s_mid : s_side) * v[k];
  }
  return acc;
}

template <class LD>
__device__ __forceinline__ double apply_const_at(const double* x, int N, int i, int j,
                                                 double s_side, double s_mid) {
  double v[9];
  load3x3<LD>(x, N, i, j, v);
  return const_from(v, N, i, j, s_side, s_mid);
}

// ElementOperator.apply (operators.py:178-188): corner a outer, b inner;
// cells outside the grid contribute nothing.
template <class LD>
__device__ __forceinline__ double apply_element_at(const double* x,
                                                   const double* eps, int N, int i,
                                                   int j) {
  const int n = N - 1;
  double v[9], e[4];
  load3x3<LD>(x, N, i, j, v);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int ci = i - (a & 1), cj = j - (a >> 1);
    e[a] = (ci >= 0 && cj >= 0 && ci < n && cj < n) ? LD::ld(eps + (size_t)ci * n + cj) : 0.0;
  }
  double out = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int a0 = a & 1, a1 = a >> 1;
    const int ci = i - a0, cj = j - a1;
    if (!(ci >= 0 && cj >= 0 && ci < n && cj < n)) continue;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      // x[ci+b0][cj+b1] sits at 3x3 offset (b0 - a0, b1 - a1)
      const int k = ((b & 1) - a0 + 1) * 3 + ((b >> 1) - a1 + 1);
      acc = acc + c_E[a * 4 + b] * v[k];
    }
    out = out + e[a] * acc;
  }
  return out;
}

// TableOperator.apply (operators.py:229-239): taps row-major, in-range only.
template <class LD>
__device__ __forceinline__ double apply_table_at(const double* x,
                                                 const double* tbl, int N, int i,
                                                 int j) {
  const size_t nv = (size_t)N * N;
  const size_t vv = (size_t)i * N + j;
  double v[9], w[9];
  load3x3<LD>(x, N, i, j, v);
#pragma unroll
  for (int k = 0; k < 9; ++k) w[k] = LD::ld(tbl + (size_t)k * nv + vv);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int ii = i + k / 3 - 1, jj = j + k % 3 - 1;
    if (inside(ii, jj, N)) acc = acc + w[k] * v[k];
  }
  return acc;
}

template <class LD>
__device__ __forceinline__ double apply_op_at(const OpView& op, const double* x,
                                              int N, int i, int j) {
  if (op.kind == OP_CONST) return apply_const_at<LD>(x, N, i, j, op.s_side, op.s_mid);
  if (op.kind == OP_ELEMENT) return apply_element_at<LD>(x, op.eps, N, i, j);
  if (op.kind == OP_TABLE) return apply_table_at<LD>(x, op.tbl, N, i, j);
  return 0.0;
}

// ---------------------------------------------------------------------------
// d-linear transfers.

// restrict_dlinear at coarse (I,J) (operators.py:111-132): axis-0 pass then
// axis-1 pass, offsets -2..2, in-range terms only, each pass from 0.
template <class LD>
__device__ __forceinline__ double restrict_dlinear_at(const double* f, int Nf, int I,
                                                      int J) {
  const int m = (Nf - 1) / 3;
  double x[25];
#pragma unroll
  for (int k = 0; k < 25; ++k) {
    const int oi = k / 5 - 2, oj = k % 5 - 2;
    const bool ok = !((oi < 0 && I < 1) || (oi > 0 && I > m - 1) || (oj < 0 && J < 1) ||
                      (oj > 0 && J > m - 1));
    x[k] = ok ? LD::ld(f + (size_t)(3 * I + oi) * Nf + (3 * J + oj)) : 0.0;
  }
  double out = 0.0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const int oj = b - 2;
    if ((oj < 0 && J < 1) || (oj > 0 && J > m - 1)) continue;
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int oi = a - 2;
      if ((oi < 0 && I < 1) || (oi > 0 && I > m - 1)) continue;
      t = t + c_W5[a] * x[a * 5 + b];
    }
    out = out + c_W5[b] * t;
  }
  return out;
}

// prolong_values at fine (i,j) (operators.py:96-127):
// axis 0: T = wl*c[q] + (1-wl)*c[qn]; then axis 1 on T.
template <class LD>
__device__ __forceinline__ double prolong_dlinear_at(const double* c, int Nc, int i,
                                                     int j) {
  const int m = Nc - 1;
  const int qi = i / 3, ri = i - 3 * qi, qni = min(qi + 1, m);
  const int qj = j / 3, rj = j - 3 * qj, qnj = min(qj + 1, m);
  const double c00 = LD::ld(c + (size_t)qi * Nc + qj), c10 = LD::ld(c + (size_t)qni * Nc + qj);
  const double c01 = LD::ld(c + (size_t)qi * Nc + qnj), c11 = LD::ld(c + (size_t)qni * Nc + qnj);
  const double wli = c_WL[ri], wri = c_WR[ri];
  const double t0 = wli * c00 + wri * c10;
  const double t1 = wli * c01 + wri * c11;
  return c_WL[rj] * t0 + c_WR[rj] * t1;
}

// ---------------------------------------------------------------------------
// Operator-dependent transfers; P is stored compactly as 25 planes of the
// coarse vertex grid, plane (oi+2)*5+(oj+2) for fine offsets -2..2 (offsets
// +-3 of the reference's 7x7 table are identically zero:
// operators.py:325-436 never writes them except with d-linear weight 0).

// TransferOps.prolong with a P table (operators.py:570-581, 625-631):
// contributions in (oi, oj) row-major order == coarse I descending.
template <class LD>
__device__ __forceinline__ double prolong_table_at(const double* c,
                                                   const double* P, int Nc, int i,
                                                   int j) {
  const size_t nvc = (size_t)Nc * Nc;
  const int qi = i / 3, ri = i - 3 * qi;
  const int qj = j / 3, rj = j - 3 * qj;
  // candidates in accumulation order: (qi+1, qj+1), (qi+1, qj), (qi, qj+1), (qi, qj)
  double w[4], x[4];
  bool use[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int di = 1 - (k >> 1), dj = 1 - (k & 1);
    use[k] = (di == 0 || ri > 0) && (dj == 0 || rj > 0);
    const int I = qi + di, J = qj + dj;
    const int oi = i - 3 * I, oj = j - 3 * J;
    const size_t vc = (size_t)I * Nc + J;
    w[k] = use[k] ? LD::ld(P + (size_t)((oi + 2) * 5 + (oj + 2)) * nvc + vc) : 0.0;
    x[k] = use[k] ? LD::ld(c + vc) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (use[k]) acc = acc + w[k] * x[k];
  return acc;
}

// TransferOps.restrict with a P table (operators.py:586-596): 5x5 taps row-major.
template <class LD>
__device__ __forceinline__ double restrict_table_at(const double* f, int Nf,
                                                    const double* P, int Nc, int I,
                                                    int J) {
  const size_t nvc = (size_t)Nc * Nc;
  const size_t vc = (size_t)I * Nc + J;
  double w[25], x[25];
#pragma unroll
  for (int k = 0; k < 25; ++k) {
    const int fi = 3 * I + k / 5 - 2, fj = 3 * J + k % 5 - 2;
    w[k] = LD::ld(P + (size_t)k * nvc + vc);
    x[k] = inside(fi, fj, Nf) ? LD::ld(f + (size_t)fi * Nf + fj) : 0.0;
  }
  double out = 0.0;
#pragma unroll
  for (int k = 0; k < 25; ++k) {
    const int fi = 3 * I + k / 5 - 2, fj = 3 * J + k % 5 - 2;
    if (inside(fi, fj, Nf)) out = out + w[k] * x[k];
  }
  return out;
}

// restrict_smoothed with a per-vertex 7x7 table (operators.py:606-613), in
// two load batches (rows -3..0, rows 1..3) to bound register use.
template <class LD, bool CHK = true>
__device__ __forceinline__ double restrict_rt_table_at(const double* f, int Nf,
                                                       const double* Rt, int Nc,
                                                       int I, int J) {
  const size_t nvc = (size_t)Nc * Nc;
  const size_t vc = (size_t)I * Nc + J;
  double out = 0.0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r0 = half == 0 ? 0 : 4, nr = half == 0 ? 4 : 3;
    double w[28], x[28];
#pragma unroll
    for (int k = 0; k < nr * 7; ++k) {
      const int oi = r0 + k / 7 - 3, oj = k % 7 - 3;
      const int fi = 3 * I + oi, fj = 3 * J + oj;
      w[k] = LD::ld(Rt + (size_t)((oi + 3) * 7 + (oj + 3)) * nvc + vc);
      x[k] = in_rng<CHK>(fi, fj, Nf) ? LD::ld(f + (size_t)fi * Nf + fj) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < nr * 7; ++k) {
      const int oi = r0 + k / 7 - 3, oj = k % 7 - 3;
      if (in_rng<CHK>(3 * I + oi, 3 * J + oj, Nf)) out = out + w[k] * x[k];
    }
  }
  return out;
}

// Geometric fast path of restrict_smoothed (operators.py:602-605):
// R( (A1 f) * s ) with A1 the unit 9-point stencil, s = omega*3.0/8.0.  The
// 7x7 fine window is loaded once; each smoothed value is the zero-extended
// 9-point sum of its in-range taps, then scaled, then restricted.
template <class LD, bool CHK = true>
__device__ __forceinline__ double restrict_rt_geom_at(const double* f, int Nf, int I,
                                                      int J, double s_side, double s_mid,
                                                      double scale) {
  const int m = (Nf - 1) / 3;
  double x[49];
#pragma unroll
  for (int k = 0; k < 49; ++k) {
    const int fi = 3 * I + k / 7 - 3, fj = 3 * J + k % 7 - 3;
    x[k] = in_rng<CHK>(fi, fj, Nf) ? LD::ld(f + (size_t)fi * Nf + fj) : 0.0;
  }
  double out = 0.0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const int oj = b - 2;
    if (CHK && ((oj < 0 && J < 1) || (oj > 0 && J > m - 1))) continue;
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int oi = a - 2;
      if (CHK && ((oi < 0 && I < 1) || (oi > 0 && I > m - 1))) continue;
      // smoothed value at fine (3I+oi, 3J+oj): window centre (a+1, b+1)
      const int vi = 3 * I + oi, vj = 3 * J + oj;
      double acc = 0.0;
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int di = s / 3 - 1, dj = s % 3 - 1;
        if (in_rng<CHK>(vi + di, vj + dj, Nf))
          acc = acc + (s == 4 ? s_mid : s_side) * x[(a + 1 + di) * 7 + (b + 1 + dj)];
      }
      t = t + c_W5[a] * (acc * scale);
    }
    out = out + c_W5[b] * t;
  }
  return out;
}

}  // namespace tmg
