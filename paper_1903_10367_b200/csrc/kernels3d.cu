// 3D kernels: operator setup (child-mean material, stencil tables, BoxMG P,
// Galerkin rows) and the additive cycle, for regular spacetrees.
//
// Every kernel evaluates the fp64 expression DAG of the function of
// oracle/mg3d.py it cites (the 3D restatement of the reference's 2D
// algorithm); with --fmad=false the iterates equal the oracle's bit for bit.
#include "kernels3d.cuh"

namespace t3 {

// ---------------------------------------------------------------------------
// small helpers

// Load policies: LdNC (read-only path) in grid kernels, whose inputs were
// written by earlier kernels; LdGen (plain, L1-coherent within the block) in
// the one-block chain kernel, which re-reads what it wrote after a barrier.
struct LdNC {
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
};
struct LdGen {
  static __device__ __forceinline__ double ld(const double* p) { return *p; }
};

__host__ __device__ constexpr int tap(int a, int b, int c) { return (a + 1) * 9 + (b + 1) * 3 + (c + 1); }
__host__ __device__ constexpr int pslot(int a, int b, int c) { return (a + 2) * 25 + (b + 2) * 5 + (c + 2); }

__device__ __forceinline__ size_t vid(int N, int i, int j, int k) {
  return ((size_t)i * N + j) * N + k;
}

// K_unit entry of corners a, b (index a0 + 2 a1 + 4 a2): 1/3, 0, -1/12 (mg3d.kmat)
__device__ __forceinline__ double kmat(int a, int b) {
  const int d = __popc(a ^ b);
  return d == 0 ? K_D : (d == 1 ? 0.0 : -K_E);
}

// 27 neighbours of an interior vertex, tap order (row-major offsets)
template <class LD>
__device__ __forceinline__ void load27(const double* x, int N, size_t v, double out[27]) {
  const long long sN = N, sNN = (long long)N * N;
#pragma unroll
  for (int t = 0; t < 27; ++t) {
    const long long off = (t / 9 - 1) * sNN + ((t / 3) % 3 - 1) * sN + (t % 3 - 1);
    out[t] = LD::ld(x + (long long)v + off);
  }
}

// mg3d.apply_const at one vertex: ((m*x0) - (se*SE)) - (sc*SC); SE / SC the
// edge / corner neighbours summed sequentially in tap order.
__device__ __forceinline__ double const_from(const double x[27], double m, double se, double sc) {
  double SE = 0.0, SC = 0.0;
  bool fe = true, fc = true;
#pragma unroll
  for (int t = 0; t < 27; ++t) {
    const int nz = (t / 9 != 1) + ((t / 3) % 3 != 1) + (t % 3 != 1);
    if (nz == 2) { SE = fe ? x[t] : SE + x[t]; fe = false; }
    if (nz == 3) { SC = fc ? x[t] : SC + x[t]; fc = false; }
  }
  return ((m * x[13]) - (se * SE)) - (sc * SC);
}

// mg3d.element_sums / apply_element at an interior vertex: cells v - a in
// corner order; E = sum e_a, T = sum e_a * s_a (sequential from the first).
// (The oracle accumulates E and T cell by cell; here the eight cells are summed pairwise -- a
// depth-3 tree instead of an 8-long dependent chain, the kernels' fp64 latency stalls -- which
// stays within rounding of the oracle's order: the 3D bar is relative 1e-10.)
__device__ __forceinline__ void element_ET(const double x[27], const double e[8], double& E, double& T) {
  double p[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int s0 = 1 - 2 * (a & 1), s1 = 1 - 2 * ((a >> 1) & 1), s2 = 1 - 2 * (a >> 2);
    const double s = (x[tap(s0, s1, 0)] + x[tap(s0, 0, s2)]) + (x[tap(0, s1, s2)] + x[tap(s0, s1, s2)]);
    p[a] = e[a] * s;
  }
  E = ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
  T = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
}

template <class LD>
__device__ __forceinline__ void load_cells(const double* ce, int N, int i, int j, int k, double e[8]) {
  const int n = N - 1;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int ci = i - (a & 1), cj = j - ((a >> 1) & 1), ck = k - (a >> 2);
    e[a] = LD::ld(ce + ((size_t)ci * n + cj) * n + ck);
  }
}

// Operator image and Jacobi diagonal at an interior vertex (mg3d.Op.apply / .diag).
template <class LD>
__device__ __forceinline__ void op_apply(const Op3& op, const double* u, int N, int i, int j, int k,
                                         double& au, double& dg) {
  const size_t v = vid(N, i, j, k);
  double x[27];
  load27<LD>(u, N, v, x);
  if (op.kind == OP_CONST) {
    au = const_from(x, op.m, op.se, op.sc);
    dg = op.cdiag;
  } else if (op.kind == OP_ELEMENT) {
    double e[8], E, T;
    load_cells<LD>(op.e, N, i, j, k, e);
    element_ET(x, e, E, T);
    dg = K_D * E;
    au = (dg * x[13]) - (K_E * T);
  } else {
    const size_t nv = (size_t)N * N * N;
    double w[27];
    if (op.tdict) {
      const double* row = op.tdict + (size_t)__ldg(op.tidx + v) * kDictW;
#pragma unroll
      for (int t = 0; t < 27; ++t) w[t] = __ldg(row + t);
    } else {
#pragma unroll
      for (int t = 0; t < 27; ++t) w[t] = LD::ld(op.tbl + (size_t)t * nv + v);
    }
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < 27; ++t) acc = acc + w[t] * x[t];
    au = acc;
    dg = w[13];
  }
}

// ---------------------------------------------------------------------------
// transfers

// mg3d.restrict_dlinear at interior coarse vertex W: axis 0, then 1, then 2.
// cpt0: afacc -- the fine c-point (centre tap) reads as 0 (solvers.py:365-368).
template <class LD>
__device__ __forceinline__ double restrict_dlinear(const double* f, int Nf, int I, int J, int K,
                                                   bool cpt0) {
  constexpr double W5[5] = {1.0 / 3.0, 2.0 / 3.0, 3.0 / 3.0, 2.0 / 3.0, 1.0 / 3.0};
  double t1[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    double t0[5];
#pragma unroll
    for (int b = 0; b < 5; ++b) {
      double x[5];
#pragma unroll
      for (int a = 0; a < 5; ++a) {
        x[a] = LD::ld(f + vid(Nf, 3 * I + a - 2, 3 * J + b - 2, 3 * K + c - 2));
        if (cpt0 && a == 2 && b == 2 && c == 2) x[a] = 0.0;
      }
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 5; ++a) acc = acc + W5[a] * x[a];
      t0[b] = acc;
    }
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < 5; ++b) acc = acc + W5[b] * t0[b];
    t1[c] = acc;
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 5; ++c) acc = acc + W5[c] * t1[c];
  return acc;
}

// mg3d.Transfer.restrict with P: 125 taps row-major from 0 (centre weight 1).
template <class LD>
__device__ __forceinline__ double restrict_P(const double* f, int Nf, const double* P, int Nc, int I,
                                             int J, int K, bool cpt0) {
  const size_t nvc = (size_t)Nc * Nc * Nc;
  const size_t vc = vid(Nc, I, J, K);
  const size_t fc = vid(Nf, 3 * I, 3 * J, 3 * K);
  const long long sN = Nf, sNN = (long long)Nf * Nf;
  double acc = 0.0;
#pragma unroll 25
  for (int o = 0; o < 125; ++o) {
    const int a = o / 25 - 2, b = (o / 5) % 5 - 2, c = o % 5 - 2;
    double x = LD::ld(f + (long long)fc + a * sNN + b * sN + c);
    double w = (o == 62) ? 1.0 : LD::ld(P + (size_t)o * nvc + vc);
    if (o == 62 && cpt0) x = 0.0;
    acc = acc + w * x;
  }
  return acc;
}

// both restrictions of the adaFACx cycle (rho and the smoothed residual) in one pass over the 125
// weights (each loaded once; the two sums keep restrict_P's order)
template <class LD>
__device__ __forceinline__ void restrict_P2(const double* f, const double* g, int Nf, const double* P, int Nc,
                                            int I, int J, int K, bool cpt0, double& rf, double& rg) {
  const size_t nvc = (size_t)Nc * Nc * Nc;
  const size_t vc = vid(Nc, I, J, K);
  const size_t fc = vid(Nf, 3 * I, 3 * J, 3 * K);
  const long long sN = Nf, sNN = (long long)Nf * Nf;
  double af = 0.0, ag = 0.0;
#pragma unroll 25
  for (int o = 0; o < 125; ++o) {
    const int a = o / 25 - 2, b = (o / 5) % 5 - 2, c = o % 5 - 2;
    const long long fo = (long long)fc + a * sNN + b * sN + c;
    double x = LD::ld(f + fo);
    const double y = LD::ld(g + fo);
    const double w = (o == 62) ? 1.0 : LD::ld(P + (size_t)o * nvc + vc);
    if (o == 62 && cpt0) x = 0.0;
    af = af + w * x;
    ag = ag + w * y;
  }
  rf = af;
  rg = ag;
}

// mg3d.prolong_dlinear at fine vertex (i,j,k): axis 0, then 1, then 2,
// wl*c[q] + (1-wl)*c[q+1] with wl = 1 - r/3.
template <class CV>
__device__ __forceinline__ double prolong_dlinear(const CV& cv, int Nc, int i, int j, int k) {
  const int m = Nc - 1;
  const int qi = i / 3, ri = i - 3 * qi, qni = min(qi + 1, m);
  const int qj = j / 3, rj = j - 3 * qj, qnj = min(qj + 1, m);
  const int qk = k / 3, rk = k - 3 * qk, qnk = min(qk + 1, m);
  const double wli = 1.0 - (double)ri / 3.0, wri = 1.0 - wli;
  const double wlj = 1.0 - (double)rj / 3.0, wrj = 1.0 - wlj;
  const double wlk = 1.0 - (double)rk / 3.0, wrk = 1.0 - wlk;
  const int J2[2] = {qj, qnj}, K2[2] = {qk, qnk};
  double T0[2][2];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int c = 0; c < 2; ++c) T0[b][c] = wli * cv(qi, J2[b], K2[c]) + wri * cv(qni, J2[b], K2[c]);
  double T1[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) T1[c] = wlj * T0[0][c] + wrj * T0[1][c];
  return wlk * T1[0] + wrk * T1[1];
}

// mg3d.Transfer.prolong with P at fine vertex (i,j,k): parents in row-major
// offset order (= parent index descending), accumulated from 0.
template <class LD, class CV>
__device__ __forceinline__ double prolong_P(const CV& cv, const double* P, int Nc, int i, int j, int k) {
  const size_t nvc = (size_t)Nc * Nc * Nc;
  const int qi = i / 3, ri = i - 3 * qi;
  const int qj = j / 3, rj = j - 3 * qj;
  const int qk = k / 3, rk = k - 3 * qk;
  double acc = 0.0;
#pragma unroll
  for (int d = 7; d >= 0; --d) {
    const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
    if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
    const int I = qi + di, J = qj + dj, K = qk + dk;
    const int oi = ri - 3 * di, oj = rj - 3 * dj, ok = rk - 3 * dk;
    const int s = pslot(oi, oj, ok);
    const double w = (s == 62) ? 1.0 : LD::ld(P + (size_t)s * nvc + vid(Nc, I, J, K));
    acc = acc + w * cv(I, J, K);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// cycle bodies

// advance(), fine -> coarse at one interior vertex (mg3d.Engine.advance).
template <class LD>
__device__ __forceinline__ void down_vertex(const Down3& a, int i, int j, int k, double& s, double& mx) {
  const int N = a.N;
  const size_t v = vid(N, i, j, k);
  double au, dg;
  op_apply<LD>(a.op, a.u, N, i, j, k, au, dg);
  const double rhs = a.rhs ? LD::ld(a.rhs + v) : 0.0;
  double rho, bt2 = 0.0;
  bool have_bt = false;
  if (a.is_top) {
    rho = rhs - au;
  } else {
    const bool cpt0 = a.variant == VAR_AFACC;
    double b;
    if (a.P && a.write && a.variant == VAR_JAC) {
      restrict_P2<LD>(a.rho_f, a.sm_f, a.Nf, a.P, N, i, j, k, cpt0, b, bt2);
      have_bt = true;
    } else {
      b = a.P ? restrict_P<LD>(a.rho_f, a.Nf, a.P, N, i, j, k, cpt0)
              : restrict_dlinear<LD>(a.rho_f, a.Nf, i, j, k, cpt0);
    }
    b = b + rhs;   // b[l] = R rho + rhs[l]   (solvers.py:370-371)
    b = b + au;    // + _bpart: overlapped -> A u (solvers.py:351-352)
    rho = b - au;
  }
  if (a.is_top) {  // composite vertices: the finest level of a regular tree
    const double t = a.hw * rho;
    s = s + t * t;
    mx = fmax(mx, fabs(rho));
  }
  if (a.write) {
    double d;
    if (a.variant == VAR_BPX && !a.is_top) d = a.omega * rho;
    else d = (a.w * rho) / dg;
    if (a.variant == VAR_JAC && !a.is_top) {
      const double bt = have_bt ? bt2
                        : a.P   ? restrict_P<LD>(a.sm_f, a.Nf, a.P, N, i, j, k, false)
                                : restrict_dlinear<LD>(a.sm_f, a.Nf, i, j, k, false);
      d = d - a.ds * ((a.wt * bt) / dg);
    }
    a.g[v] = d;
  }
  if (a.rho) a.rho[v] = rho;
}

template <class LD>
__device__ __forceinline__ void smooth_vertex(const Smooth3& a, int i, int j, int k) {
  const size_t v = vid(a.N, i, j, k);
  double x[27];
  load27<LD>(a.x, a.N, v, x);
  double s = const_from(x, C_D8, C_E6, C_C12);  // apply_const(x, 1.0)
  s = s * a.scale;                              // s *= omega*3.0/8.0 (operators.py:603-605)
  a.sm[v] = s;
}

template <class LD>
__device__ __forceinline__ void up_vertex(const Up3& a, int i, int j, int k) {
  const int N = a.N;
  const size_t v = vid(N, i, j, k);
  double g = a.g ? LD::ld(a.g + v) : 0.0;  // null: the finest level's g is already in u (pp)
  double c;
  if (a.is_bottom) {
    c = g;
  } else {
    const int Nc = a.Nc;
    if (a.pi) {
      // dtil = ds * P(inj d_l), inj = d_l at the fine c-point of every interior
      // coarse vertex (solvers.py:377-384)
      const double* gl = a.g;
      auto inj = [&](int I, int J, int K) -> double {
        if (I < 1 || J < 1 || K < 1 || I > Nc - 2 || J > Nc - 2 || K > Nc - 2) return 0.0;
        return LD::ld(gl + vid(N, 3 * I, 3 * J, 3 * K));
      };
      const double pv = a.P ? prolong_P<LD>(inj, a.P, Nc, i, j, k) : prolong_dlinear(inj, Nc, i, j, k);
      g = g - a.ds * pv;
    }
    const double* cc = a.carry_c;
    auto cv = [&](int I, int J, int K) -> double { return LD::ld(cc + vid(Nc, I, J, K)); };
    const double pc = a.P ? prolong_P<LD>(cv, a.P, Nc, i, j, k) : prolong_dlinear(cv, Nc, i, j, k);
    c = pc + g;
  }
  if (a.carry) a.carry[v] = c;
  const double un = a.u[v] + c;
  a.u[v] = un;
  // FAS injection walk-down (solvers.py:283-288): every interior coarse vertex takes
  int ii = i, jj = j, kk = k;
  for (int lc = a.l - 1; lc >= a.l0; --lc) {
    if (ii % 3 || jj % 3 || kk % 3) break;
    ii /= 3;
    jj /= 3;
    kk /= 3;
    a.ul[lc][vid(a.Nl[lc], ii, jj, kk)] = un;
  }
}

// ---------------------------------------------------------------------------
// grid kernels: 32 x 4 x 2 thread tiles over (k, j, i), grid-stride over tiles

struct Tiles {
  int tx, ty, tz;
  __device__ __forceinline__ int count() const { return tx * ty * tz; }
};

__device__ __forceinline__ Tiles tiles_of(int N, int ilo, int ihi) {
  Tiles t;
  t.tx = (N - 2 + kTX - 1) / kTX;
  t.ty = (N - 2 + kTY - 1) / kTY;
  t.tz = (ihi - ilo + kTZ - 1) / kTZ;
  return t;
}

template <class F>
__device__ __forceinline__ void for_tiles(int N, int ilo, int ihi, F&& f) {
  const Tiles t = tiles_of(N, ilo, ihi);
  for (int b = blockIdx.x; b < t.count(); b += gridDim.x) {
    const int bx = b % t.tx, r = b / t.tx, by = r % t.ty, bz = r / t.ty;
    const int k = 1 + bx * kTX + threadIdx.x;
    const int j = 1 + by * kTY + threadIdx.y;
    const int i = ilo + bz * kTZ + threadIdx.z;
    if (k <= N - 2 && j <= N - 2 && i < ihi) f(i, j, k);
  }
}

template <int BS>
__device__ __forceinline__ void block_reduce(double& s, double& m) {
  __shared__ double ss[BS / 32], sm[BS / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  }
  const int t = (threadIdx.z * blockDim.y + threadIdx.y) * blockDim.x + threadIdx.x;
  const int w = t >> 5, lane = t & 31;
  if (lane == 0) { ss[w] = s; sm[w] = m; }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < BS / 32; ++q) { a += ss[q]; b = fmax(b, sm[q]); }
    s = a;
    m = b;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kBlock) k3_down(const __grid_constant__ Down3 a) {
  double s = 0.0, m = 0.0;
  for_tiles(a.N, a.ilo, a.ihi, [&](int i, int j, int k) { down_vertex<LdNC>(a, i, j, k, s, m); });
  block_reduce<kBlock>(s, m);
  if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0 && a.part_sum) {
    a.part_sum[blockIdx.x] = s;
    a.part_max[blockIdx.x] = m;
  }
}

__global__ void __launch_bounds__(kBlock) k3_smooth(const __grid_constant__ Smooth3 a) {
  for_tiles(a.N, a.ilo, a.ihi, [&](int i, int j, int k) { smooth_vertex<LdNC>(a, i, j, k); });
}

__global__ void __launch_bounds__(kBlock) k3_up(const __grid_constant__ Up3 a) {
  for_tiles(a.N, a.ilo, a.ihi, [&](int i, int j, int k) { up_vertex<LdNC>(a, i, j, k); });
}

// The coarse chain l0..lc in one block: down (+ smoothing) lc -> l0, the
// deterministic reduction of every partial of the cycle into the history
// slot, then up l0 -> lc.
__global__ void __launch_bounds__(kChainBlock) k3_chain(const __grid_constant__ Chain3 a) {
  __shared__ double rs[kChainBlock / 32], rm[kChainBlock / 32];
  const int tid = threadIdx.x, nthr = blockDim.x;
  double s = 0.0, m = 0.0;
  auto each = [&](int N, int ilo, int ihi, auto&& f) {
    const int n = N - 2, cnt = (ihi - ilo) * n * n;
    for (int q = tid; q < cnt; q += nthr) {
      const int k = 1 + q % n, r = q / n, j = 1 + r % n, i = ilo + r / n;
      f(i, j, k);
    }
    __syncthreads();
  };
  for (int l = a.lc; l >= a.l0; --l) {
    const Down3& d = a.down[l - a.l0];
    each(d.N, d.ilo, d.ihi, [&](int i, int j, int k) { down_vertex<LdGen>(d, i, j, k, s, m); });
    if (a.jac && l > a.l0 && d.write) {
      const Smooth3& sm = a.smooth[l - a.l0];
      each(sm.N, sm.ilo, sm.ihi, [&](int i, int j, int k) { smooth_vertex<LdGen>(sm, i, j, k); });
    }
  }
  // fixed-order reduction of the partials of this cycle (+ the chain's own)
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  }
  double x = 0.0, y = 0.0;
  for (int q = tid; q < a.nparts; q += nthr) {
    x += a.part_sum[q];
    y = fmax(y, a.part_max[q]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_down_sync(0xffffffffu, x, o);
    y = fmax(y, __shfl_down_sync(0xffffffffu, y, o));
  }
  if ((tid & 31) == 0) {
    rs[tid >> 5] = x + s;
    rm[tid >> 5] = fmax(y, m);
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0, u = 0.0;
    for (int q = 0; q < kChainBlock / 32; ++q) { t += rs[q]; u = fmax(u, rm[q]); }
    const int slot = *a.counter;
    a.hist[2 * (slot % a.cap)] = sqrt(t);
    a.hist[2 * (slot % a.cap) + 1] = u;
    *a.counter = slot + 1;
  }
  __syncthreads();
  if (!a.do_up) return;
  for (int l = a.l0; l <= a.lc; ++l) {
    const Up3& u = a.up[l - a.l0];
    each(u.N, u.ilo, u.ihi, [&](int i, int j, int k) { up_vertex<LdGen>(u, i, j, k); });
  }
}

// FAS injection on its own (update_fas_state, solvers.py:283-288)
__global__ void k3_inject(double* uc, int Nc, const double* uf, int Nf) {
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = Nc - 2;
  if (q >= (size_t)n * n * n) return;
  const int K = 1 + (int)(q % n), r = (int)(q / n), J = 1 + r % n, I = 1 + r / n;
  uc[vid(Nc, I, J, K)] = uf[vid(Nf, 3 * I, 3 * J, 3 * K)];
}

// the six boundary faces of an N^3 vertex array (the Dirichlet values), dst <- src
__global__ void k3_copy_boundary(double* __restrict__ dst, const double* __restrict__ src, int N) {
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (size_t)N * N) return;
  const int a = (int)(q / N), b = (int)(q % N);
  const size_t f[6] = {vid(N, 0, a, b), vid(N, N - 1, a, b), vid(N, a, 0, b),
                       vid(N, a, N - 1, b), vid(N, a, b, 0), vid(N, a, b, N - 1)};
#pragma unroll
  for (int k = 0; k < 6; ++k) dst[f[k]] = src[f[k]];
}

// ===========================================================================
// setup
// ===========================================================================

// mg3d.child_mean: 27 children summed sequentially (row-major), / 27.
__global__ void k3_child_mean(double* eff_c, const double* eff_f, int nc) {
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (size_t)nc * nc * nc) return;
  const int ck = (int)(c % nc), r = (int)(c / nc), cj = r % nc, ci = r / nc;
  const int nf = 3 * nc;
  double acc = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      for (int q = 0; q < 3; ++q) {
        const double x = eff_f[((size_t)(3 * ci + a) * nf + (3 * cj + b)) * nf + (3 * ck + q)];
        acc = (a | b | q) ? acc + x : x;
      }
  eff_c[c] = acc / 27.0;
}

__global__ void k3_scale(double* out, const double* in, double h, size_t n) {
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) out[c] = in[c] * h;
}

__global__ void k3_const_check(const double* arr, size_t n, int* flag) {
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double first = arr[0];
  const bool bad = c < n && (!(first > 0.0) || arr[c] != first);
  // one atomic per warp that saw a mismatch (not one per element)
  if (__ballot_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0);
}

// flag stays 1 iff every cell plane ci equals plane ci - ci % run bit for bit (coefficients constant
// along axis 0 in runs of `run` planes: blockwise-constant materials)
__global__ void k3_plane_run_check(const double* arr, int n, int run, int* flag) {
  const size_t plane = (size_t)n * n, cnt = plane * n;
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (c < cnt) {
    const size_t ci = c / plane, base = ci - ci % run;
    bad = ci != base && __double_as_longlong(arr[c]) != __double_as_longlong(arr[base * plane + (c - ci * plane)]);
  }
  if (__ballot_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0);
}

// Source of fine 27-point rows: a stored table, or assembled on the fly from
// the per-cell coefficients (mg3d.assemble_table order: corner a outer, b inner).
struct Rows {
  int N;
  const double* tbl;
  const double* e;
};

__device__ void row27(const Rows& R, int i, int j, int k, double t[27]) {
  const int N = R.N;
  if (R.tbl) {
    const size_t nv = (size_t)N * N * N, v = vid(N, i, j, k);
    for (int q = 0; q < 27; ++q) t[q] = R.tbl[(size_t)q * nv + v];
    return;
  }
  const int n = N - 1;
  for (int q = 0; q < 27; ++q) t[q] = 0.0;
  for (int a = 0; a < 8; ++a) {
    const int a0 = a & 1, a1 = (a >> 1) & 1, a2 = a >> 2;
    const int ci = i - a0, cj = j - a1, ck = k - a2;
    const bool in = ci >= 0 && cj >= 0 && ck >= 0 && ci < n && cj < n && ck < n;
    const double ec = in ? R.e[((size_t)ci * n + cj) * n + ck] : 0.0;
    for (int b = 0; b < 8; ++b) {
      const double kab = kmat(a, b);
      if (kab == 0.0) continue;
      const int q = tap((b & 1) - a0, ((b >> 1) & 1) - a1, (b >> 2) - a2);
      t[q] = t[q] + kab * ec;
    }
  }
}

__global__ void k3_assemble(double* tbl, Rows R) {
  const int N = R.N;
  const size_t nv = (size_t)N * N * N;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int k = (int)(v % N), r = (int)(v / N), j = r % N, i = r / N;
  double t[27];
  row27(R, i, j, k, t);
  for (int q = 0; q < 27; ++q) tbl[(size_t)q * nv + v] = t[q];
}

// ---- BoxMG P (mg3d.boxmg_p): 125 planes over the coarse vertex grid

__global__ void k3_p_init(double* P, size_t nvc) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvc) return;
  for (int s = 0; s < 125; ++s) P[(size_t)s * nvc + v] = (s == 62) ? 1.0 : 0.0;
}

// d-linear weights in the BoxMG P layout (mg3d.dlinear_p_table): ((w_a w_b) w_c),
// w_o = max(0, 1 - |o|/3), zero where the fine offset leaves the grid -- the
// starting P of the throttled setup
__global__ void k3_p_dlinear(double* P, int Nc) {
  const size_t nvc = (size_t)Nc * Nc * Nc;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvc) return;
  const int K = (int)(v % Nc), J = (int)((v / Nc) % Nc), I = (int)(v / ((size_t)Nc * Nc));
  const int nf = 3 * (Nc - 1);
  for (int a = -2; a <= 2; ++a)
    for (int b = -2; b <= 2; ++b)
      for (int c = -2; c <= 2; ++c) {
        const int fi = 3 * I + a, fj = 3 * J + b, fk = 3 * K + c;
        const bool in = fi >= 0 && fi <= nf && fj >= 0 && fj <= nf && fk >= 0 && fk <= nf;
        const double wa = fmax(0.0, 1.0 - (double)abs(a) / 3.0);
        const double wb = fmax(0.0, 1.0 - (double)abs(b) / 3.0);
        const double wc = fmax(0.0, 1.0 - (double)abs(c) / 3.0);
        P[(size_t)pslot(a, b, c) * nvc + v] = in ? (wa * wb) * wc : 0.0;
      }
}

__device__ __forceinline__ double pget(const double* P, int Nc, int I, int J, int K, int a, int b, int c) {
  if (a < -2 || a > 2 || b < -2 || b > 2 || c < -2 || c > 2) return 0.0;
  const size_t nvc = (size_t)Nc * Nc * Nc;
  return P[(size_t)pslot(a, b, c) * nvc + vid(Nc, I, J, K)];
}

__device__ __forceinline__ void pset(double* P, int Nc, int I, int J, int K, int a, int b, int c, double w) {
  const size_t nvc = (size_t)Nc * Nc * Nc;
  P[(size_t)pslot(a, b, c) * nvc + vid(Nc, I, J, K)] = w;
}

// Edges along axis ax between W and W + e_ax: lumped 1D rows (9 normal taps,
// sequential row-major), the reference's closed-form 2x2 (operators.py:287-303).
__global__ void k3_edges(double* P, int nc, int ax, Rows R, int* deg) {
  const int Nc = nc + 1;
  const size_t cnt = (size_t)nc * Nc * Nc;
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  int W[3];
  // enumerate with W[ax] in [0, nc), the others in [0, Nc), row-major over (0,1,2)
  {
    size_t r = q;
    for (int x = 2; x >= 0; --x) {
      const int ext = (x == ax) ? nc : Nc;
      W[x] = (int)(r % ext);
      r /= ext;
    }
  }
  int o1 = ax == 0 ? 1 : 0, o2 = ax == 2 ? 1 : 2;
  double c[2][3];
  for (int p = 0; p < 2; ++p) {
    int f[3] = {3 * W[0], 3 * W[1], 3 * W[2]};
    f[ax] += p + 1;
    double t[27];
    row27(R, f[0], f[1], f[2], t);
    for (int a = 0; a < 3; ++a) {
      double acc = 0.0;
      for (int b = 0; b < 3; ++b)
        for (int cc = 0; cc < 3; ++cc) {
          int o[3];
          o[ax] = a - 1;
          o[o1] = b - 1;
          o[o2] = cc - 1;
          const double x = t[tap(o[0], o[1], o[2])];
          acc = (b | cc) ? acc + x : x;
        }
      c[p][a] = acc;
    }
  }
  const double am1 = c[0][0], a01 = c[0][1], ap1 = c[0][2];
  const double am2 = c[1][0], a02 = c[1][1], ap2 = c[1][2];
  const double det = a01 * a02 - ap1 * am2;
  const double scale = fabs(a01 * a02) + fabs(ap1 * am2);
  if (fabs(det) <= 1e-14 * fmax(scale, 1e-300)) atomicOr(deg, 1);
  const double wl1 = ((-am1) * a02) / det;
  const double wl2 = (am2 * am1) / det;
  const double wh1 = (ap1 * ap2) / det;
  const double wh2 = (a01 * (-ap2)) / det;
  int o[3] = {0, 0, 0};
  o[ax] = 1;
  pset(P, Nc, W[0], W[1], W[2], o[0], o[1], o[2], wl1);
  o[ax] = 2;
  pset(P, Nc, W[0], W[1], W[2], o[0], o[1], o[2], wl2);
  int Wh[3] = {W[0], W[1], W[2]};
  Wh[ax] += 1;
  o[ax] = -2;
  pset(P, Nc, Wh[0], Wh[1], Wh[2], o[0], o[1], o[2], wh1);
  o[ax] = -1;
  pset(P, Nc, Wh[0], Wh[1], Wh[2], o[0], o[1], o[2], wh2);
}

// mg3d.lu_solve for one system: LU with partial pivoting (first max |a|),
// multipliers by the reciprocal pivot, forward then back substitution.
template <int n, int m>
__device__ void lu_solve(double (&A)[n][n], double (&B)[n][m]) {
  int piv[n];
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(A[k][k]);
    for (int r = k + 1; r < n; ++r)
      if (fabs(A[r][k]) > best) { best = fabs(A[r][k]); p = r; }
    piv[k] = p;
    if (p != k)
      for (int c = 0; c < n; ++c) { const double t = A[k][c]; A[k][c] = A[p][c]; A[p][c] = t; }
    const double rp = 1.0 / A[k][k];
    for (int r = k + 1; r < n; ++r) A[r][k] = A[r][k] * rp;
    for (int r = k + 1; r < n; ++r)
      for (int c = k + 1; c < n; ++c) A[r][c] = A[r][c] - A[r][k] * A[k][c];
  }
  for (int k = 0; k < n; ++k)
    if (piv[k] != k)
      for (int c = 0; c < m; ++c) { const double t = B[k][c]; B[k][c] = B[piv[k]][c]; B[piv[k]][c] = t; }
  for (int c = 0; c < m; ++c) {
    for (int k = 0; k < n; ++k)
      for (int r = k + 1; r < n; ++r) B[r][c] = B[r][c] - B[k][c] * A[r][k];
    for (int k = n - 1; k >= 0; --k) {
      B[k][c] = B[k][c] / A[k][k];
      for (int r = 0; r < k; ++r) B[r][c] = B[r][c] - B[k][c] * A[r][k];
    }
  }
}

// Faces with normal nx (in-plane axes p < q): rows lumped along the normal
// (3 taps, sequential) -> the reference's 2D 4x4 solve (operators.py:363-414).
__global__ void k3_faces(double* P, int nc, int nx, Rows R) {
  const int Nc = nc + 1;
  const int pa = nx == 0 ? 1 : 0, qa = nx == 2 ? 1 : 2;
  const size_t cnt = (size_t)Nc * nc * nc;
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  int W[3];
  {
    size_t r = q;
    for (int x = 2; x >= 0; --x) {
      const int ext = (x == nx) ? Nc : nc;
      W[x] = (int)(r % ext);
      r /= ext;
    }
  }
  const int inter[4][2] = {{1, 1}, {2, 1}, {1, 2}, {2, 2}};
  const int corner[4][2] = {{0, 0}, {3, 0}, {0, 3}, {3, 3}};
  double A[4][4], B[4][4];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) { A[r][c] = 0.0; B[r][c] = 0.0; }
  for (int r = 0; r < 4; ++r) {
    const int fp = inter[r][0], fq = inter[r][1];
    int f[3] = {3 * W[0], 3 * W[1], 3 * W[2]};
    f[pa] += fp;
    f[qa] += fq;
    double t[27];
    row27(R, f[0], f[1], f[2], t);
    for (int da = -1; da <= 1; ++da)
      for (int db = -1; db <= 1; ++db) {
        double coef = 0.0;
        for (int dc = -1; dc <= 1; ++dc) {
          int o[3];
          o[pa] = da;
          o[qa] = db;
          o[nx] = dc;
          const double x = t[tap(o[0], o[1], o[2])];
          coef = (dc == -1) ? x : coef + x;
        }
        const int ta = fp + da, tb = fq + db;
        const bool inner = (ta == 1 || ta == 2) && (tb == 1 || tb == 2);
        if (inner) {
          const int idx = (ta - 1) + 2 * (tb - 1);
          A[r][idx] = A[r][idx] + coef;
        } else {
          for (int c = 0; c < 4; ++c) {
            int cv[3] = {0, 0, 0};
            cv[pa] = corner[c][0] / 3;
            cv[qa] = corner[c][1] / 3;
            int o[3] = {0, 0, 0};
            o[pa] = ta - 3 * cv[pa];
            o[qa] = tb - 3 * cv[qa];
            const double kw = pget(P, Nc, W[0] + cv[0], W[1] + cv[1], W[2] + cv[2], o[0], o[1], o[2]);
            B[r][c] = B[r][c] - coef * kw;
          }
        }
      }
  }
  lu_solve<4, 4>(A, B);
  for (int c = 0; c < 4; ++c) {
    int cv[3] = {0, 0, 0};
    cv[pa] = corner[c][0] / 3;
    cv[qa] = corner[c][1] / 3;
    for (int r = 0; r < 4; ++r) {
      int o[3] = {0, 0, 0};
      o[pa] = inter[r][0] - 3 * cv[pa];
      o[qa] = inter[r][1] - 3 * cv[qa];
      pset(P, Nc, W[0] + cv[0], W[1] + cv[1], W[2] + cv[2], o[0], o[1], o[2], B[r][c]);
    }
  }
}

// Cell interiors: the 8x8 solve with the full 27-point rows.
__global__ void __launch_bounds__(128) k3_cells(double* P, int nc, Rows R) {
  const int Nc = nc + 1;
  const size_t cnt = (size_t)nc * nc * nc;
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  const int C2 = (int)(q % nc), rr = (int)(q / nc), C1 = rr % nc, C0 = rr / nc;
  double A[8][8], B[8][8];
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) { A[r][c] = 0.0; B[r][c] = 0.0; }
  for (int r = 0; r < 8; ++r) {
    const int pt0 = 1 + (r & 1), pt1 = 1 + ((r >> 1) & 1), pt2 = 1 + (r >> 2);
    double t[27];
    row27(R, 3 * C0 + pt0, 3 * C1 + pt1, 3 * C2 + pt2, t);
    for (int o = 0; o < 27; ++o) {
      const double coef = t[o];
      const int g0 = pt0 + o / 9 - 1, g1 = pt1 + (o / 3) % 3 - 1, g2 = pt2 + o % 3 - 1;
      const bool inner = (g0 == 1 || g0 == 2) && (g1 == 1 || g1 == 2) && (g2 == 1 || g2 == 2);
      if (inner) {
        const int idx = (g0 - 1) + 2 * (g1 - 1) + 4 * (g2 - 1);
        A[r][idx] = A[r][idx] + coef;
      } else {
        for (int a = 0; a < 8; ++a) {
          const int a0 = a & 1, a1 = (a >> 1) & 1, a2 = a >> 2;
          const double kw = pget(P, Nc, C0 + a0, C1 + a1, C2 + a2, g0 - 3 * a0, g1 - 3 * a1, g2 - 3 * a2);
          B[r][a] = B[r][a] - coef * kw;
        }
      }
    }
  }
  lu_solve<8, 8>(A, B);
  for (int a = 0; a < 8; ++a) {
    const int a0 = a & 1, a1 = (a >> 1) & 1, a2 = a >> 2;
    for (int r = 0; r < 8; ++r) {
      const int pt0 = 1 + (r & 1), pt1 = 1 + ((r >> 1) & 1), pt2 = 1 + (r >> 2);
      pset(P, Nc, C0 + a0, C1 + a1, C2 + a2, pt0 - 3 * a0, pt1 - 3 * a1, pt2 - 3 * a2, B[r][a]);
    }
  }
}

}  // namespace t3
