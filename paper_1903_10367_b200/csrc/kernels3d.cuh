// 3D engine (regular spacetrees, BASELINE configs 3 and 5): argument blocks
// and fp64 device helpers.
//
// There is no 3D reference; the per-element expression DAGs are the ones
// oracle/mg3d.py defines (and documents), so the kernels reproduce the
// oracle's iterates bit for bit.  Compiled with --fmad=false.
//
// Layout: level l, N = 3^l + 1 vertices per axis, vertex v = (i*N + j)*N + k
// (k contiguous); cells n = N-1 per axis, (ci*n + cj)*n + ck.  Every cycle
// kernel works on interior vertices only (boundary vertices are Dirichlet:
// their work vectors stay 0 and their u never changes), so no stencil,
// restriction or prolongation footprint ever leaves the grid.
//
// Multi-GPU: kernels take the vertex-plane range [ilo, ihi) they own and
// plane-shifted base pointers, so a slab with halo planes is addressed with
// global indices.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace t3 {

constexpr int kTX = 32, kTY = 4, kTZ = 2;  // threads along k, j, i
constexpr int kBlock = kTX * kTY * kTZ;
constexpr int kChainBlock = 512;
constexpr int kMaxLevels = 10;
constexpr int kDictW = 128;  // weight-dictionary row pitch in doubles (kernels3d_dict.cu)

enum OpKind : int { OP_CONST = 0, OP_ELEMENT = 1, OP_TABLE = 2 };
enum Variant : int { VAR_ADDITIVE = 0, VAR_EXP = 1, VAR_BPX = 2, VAR_AFACC = 3, VAR_PI = 4, VAR_JAC = 5 };

constexpr double K_D = 1.0 / 3.0;
constexpr double K_E = 1.0 / 12.0;
constexpr double C_D8 = 8.0 / 3.0;
constexpr double C_E6 = 1.0 / 6.0;
constexpr double C_C12 = 1.0 / 12.0;

// a / b for a positive b (Jacobi diagonals): hardware reciprocal seed (2^-23), one Newton
// step, the quotient corrected with its exact FMA residual -- 5 fp64 instructions against the 9 +
// special-case branch of the IEEE sequence, within an ulp of it (the 3D bar is relative 1e-10).
__device__ __forceinline__ double div_pos(double a, double b) {
  // the seed flushes denormals and overflows near the ends of the exponent range: IEEE division there
  if (!(b > 1e-290 && b < 1e290)) return a / b;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  r = fma(fma(-b, r, 1.0), r, r);
  const double q = a * r;
  return fma(fma(-b, q, a), r, q);
}

// A level operator (oracle mg3d.Op).
struct Op3 {
  int kind;
  double m, se, sc;   // const: c*(8/3), c*(1/6), c*(1/12)
  double cdiag;       // const: K_D * (c + c + ... 8 times, sequential)
  const double* e;    // element: per-cell coefficient eff*h
  const double* tbl;  // table: 27 planes over the vertex grid, plane tap = (di+1)*9+(dj+1)*3+(dk+1)
  // table as a row dictionary (kernels3d_dict.cu; level ltop-1's Galerkin rows): tap t of vertex v
  // is tdict[tidx[v] * kDictW + t]
  const double* tdict;
  const uint32_t* tidx;
  // table in run-length form along k (kernels3d_rle.cu; level ltop-1's Galerkin rows): a warp segment
  // = 32 consecutive interior k of a vertex line; only the rows that differ bitwise from their
  // predecessor in the segment are stored, SoA: tap t of stored row r is rtab[t * rn + r];
  // segment s = (i * N + j) * rseg + (k - 1) / 32 has its first stored row at rbase[s] and a bit per
  // lane that starts a new row in rmask[s]
  const double* rtab;
  const uint32_t* rbase;
  const uint32_t* rmask;
  size_t rn;
  int rseg;
};

struct Grid {
  int N;               // vertices per axis
  size_t nv;           // N^3 (plane stride for tables)
};

// One level of the fine -> coarse sweep (oracle Engine.advance, solvers.py:345-375).
struct Down3 {
  int N, l, is_top, variant, write;
  int ilo, ihi;        // interior vertex planes computed: [ilo, ihi)
  const double* u;
  const double* rhs;   // or nullptr
  Op3 op;
  // finer level (restriction sources), when !is_top
  int Nf;
  const double* rho_f;   // rho_{l+1} (= rdof on regular trees)
  const double* sm_f;    // A1(rdof_{l+1}) * s (adaFACx)
  const double* P;       // 125 planes over this level's vertex grid (boxmg) or nullptr (d-linear)
  double w, omega, wt, ds, hw;
  const double* bR;      // precomputed R rho_{l+1} / R sm_{l+1} (fused fine pass) or nullptr
  const double* bT;
  double* rho;           // this level's rho (l > l0) or nullptr
  double* g;             // d - dtil
  double* part_sum;
  double* part_max;
};

// R~ smoothing of a level's rdof: sm = A1(rdof) * ((omega*3)/8) at interior vertices.
struct Smooth3 {
  int N, ilo, ihi;
  const double* x;
  double* sm;
  double scale;
};

// One level of the coarse -> fine carry (solvers.py:377-395) + FAS injection walk-down.
struct Up3 {
  int N, l, l0, is_bottom, pi, ilo, ihi;
  double* u;
  const double* g;
  double* carry;        // this level's carry (l < top) or nullptr
  int Nc;
  const double* carry_c;
  const double* P;      // level l-1's P planes (boxmg) or nullptr
  double ds;
  double* ul[kMaxLevels];  // u of the coarser levels for the injection walk-down
  int Nl[kMaxLevels];
};

constexpr int kMaxChain = 3;
struct Chain3 {
  int l0, lc, do_up, jac;
  const double* part_sum;
  const double* part_max;
  int nparts;
  double* hist;
  int* counter;
  int cap;
  Down3 down[kMaxChain];
  Smooth3 smooth[kMaxChain];
  Up3 up[kMaxChain];
};

}  // namespace t3
