// Fused fine pass, version 4: the FFP schedule of kernels3d_ffp.cu (stages A-D,
// pipeline.py:242-386) restructured for B200 throughput.
//
//   A(t)    u_new = u + (P carry_c + g_in) on fine plane t (u window, offset -4)
//   B(t-1)  rho, g_out = (w rho)/diag and the norm partials on plane t-1
//   C       adaFACx smoothing sm = A1(rho)*(omega*3/8) by plane partial sums:
//           each thread owns fixed sm columns and keeps, per column, the
//           sequential edge / corner sums of the two pending sm planes in
//           registers (the DAG of const_from is plane-major), so every rho
//           plane is read once (9 shared loads) and the rho ring disappears
//   D       restriction of rho(t-1) and sm(t-2) into the owned coarse planes
//           (two running accumulators per coarse vertex and field)
//
// Every input plane (u_in, g_in, the row-padded cell coefficients, rhs and two
// coarse carry planes) arrives by TMA one plane ahead (boxes start at even
// inner coordinates: TMA needs 16-byte aligned rows), all on one mbarrier per
// plane set, so global latency is off the critical path; A writes u_new in
// place into its TMA slot.  CTA = 12 x 12 coarse (J, K) column (36 x 36 owned
// fine vertices), 512 threads, one CTA per SM (~185 KB shared memory).
// Per-element DAGs are those of kernels3d.cu / oracle mg3d, so the iterates
// are bit-identical to the phase-by-phase cycle.
#include <cuda.h>

#include "kernels3d.cuh"

namespace t3 {

constexpr int k4T = 12;               // coarse tile (J, K)
constexpr int k4U = 3 * k4T + 6;      // 42: u / g / cell window (fine offset -4)
constexpr int k4R = 3 * k4T + 4;      // 40: rho / rhs window (offset -3)
constexpr int k4S = 3 * k4T + 2;      // 38: sm window (offset -2)
constexpr int k4K = k4T + 4;          // 16: coarse carry window (offset -2)
constexpr int k4Threads = 512;
constexpr int k4SU = 1776;            // slot stride of a 42 x 42 plane (128-byte multiple)
constexpr int k4SR = k4R * k4R;       // 1600
constexpr int k4SK = 2 * k4K * k4K;   // 512: two coarse planes
constexpr int k4PS = k4S * k4S;       // 1444
constexpr int k4Cols = (k4PS + k4Threads - 1) / k4Threads;  // sm columns per thread
constexpr int o4U = 0;                 // 4 slots: u_in -> u_new ring
constexpr int o4G = o4U + 4 * k4SU;    // 2 slots: g_in
constexpr int o4C = o4G + 2 * k4SU;    // 3 slots: cell planes
constexpr int o4H = o4C + 3 * k4SU;    // 2 slots: rhs (u window: TMA wants even inner coordinates)
constexpr int o4K = o4H + 2 * k4SU;    // 2 slots: coarse carry
constexpr int o4R = o4K + 2 * k4SK;    // rho plane
constexpr int o4S = o4R + k4SR;        // sm plane
constexpr size_t kFfp4Smem = sizeof(double) * (o4S + k4PS);

struct Ffp4 {
  CUtensorMap tu;  // u_in, box 42 x 42 x 1
  CUtensorMap tg;  // g_in, box 42 x 42 x 1
  CUtensorMap tc;  // row-padded cell coefficients, box 42 x 42 x 1
  CUtensorMap th;  // rhs, box 42 x 42 x 1
  CUtensorMap tk;  // carry of the coarse level, box 16 x 16 x 2
  Ffp3 f;
  int dbg;  // debug: bit 0 no TMA, 1 no A, 2 no B, 3 no C, 4 no D
};

__device__ __forceinline__ int floor3(int x) { return x >= 0 ? x / 3 : -((2 - x) / 3); }

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int KIND>
__global__ void __launch_bounds__(k4Threads, 1) k3_ffp4(const __grid_constant__ Ffp4 A) {
  extern __shared__ __align__(128) double s4[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double red_s[k4Threads / 32], red_m[k4Threads / 32];
  const Ffp3& a = A.f;
  const int N = a.N, Nc = a.Nc, nc = Nc - 1;
  const size_t NN = (size_t)N * N, NcNc = (size_t)Nc * Nc, nvc = NcNc * Nc;
  int b = blockIdx.x;
  const int tk = b % a.tiles;
  b /= a.tiles;
  const int tj = b % a.tiles;
  const int tc = b / a.tiles;
  const int J0 = tj * k4T, K0 = tk * k4T;
  const int Ia = tc * a.chunk, Ib = min(Nc, Ia + a.chunk);
  const int Ilo = max(Ia, 1), Ihi = min(Ib - 1, nc - 1);  // restricted coarse planes [Ilo, Ihi]
  const int fj0 = 3 * J0, fk0 = 3 * K0;
  const int fjE = min(fj0 + 3 * k4T, N - 1), fkE = min(fk0 + 3 * k4T, N - 1);
  const int iOwnLo = 3 * Ia, iOwnHi = min(3 * Ib, N - 1);
  const int t0 = 3 * Ia - 4, tEnd = max(3 * Ihi + 4, iOwnHi);
  const int lt = threadIdx.x;
  const bool apply = a.apply != 0;
  const bool has_rhs = a.rhs != nullptr;
  const bool jac = a.jac != 0;
  const bool zc = a.variant == VAR_AFACC;
  double s_sum = 0.0, s_max = 0.0;

  // sm columns of this thread (fixed for the march) and their pending partials
  int scol[k4Cols];
  bool sin_[k4Cols];
  double SEa[k4Cols], SCa[k4Cols], XA[k4Cols], SEb[k4Cols], SCb[k4Cols];
#pragma unroll
  for (int m = 0; m < k4Cols; ++m) {
    const int q = lt + m * k4Threads;
    const int jj = q / k4S, kk = q - jj * k4S;
    const int j = fj0 - 2 + jj, k = fk0 - 2 + kk;
    scol[m] = q < k4PS ? q : -1;
    sin_[m] = q < k4PS && j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2;
    SEa[m] = SCa[m] = XA[m] = SEb[m] = SCb[m] = 0.0;
  }
  // restriction task: coarse (wj, wk) of the tile, field 0 rho / 1 sm
  const int task_f = lt / (k4T * k4T), task_w = lt - task_f * k4T * k4T;
  const int rJ = J0 + task_w / k4T, rK = K0 + task_w % k4T;
  const bool rtask = lt < 2 * k4T * k4T && (task_f == 0 || jac) && rJ >= 1 && rJ <= nc - 1 && rK >= 1 &&
                     rK <= nc - 1;
  double accC = 0.0, accN = 0.0;

  const int dbg = A.dbg;
  const bool ld_u = !(dbg & 128), ld_c = KIND == OP_ELEMENT && !(dbg & 32), ld_h = has_rhs && !(dbg & 64);
  const unsigned bytes_set = (unsigned)sizeof(double) *
                             ((ld_u ? k4U * k4U : 0) + (apply ? k4U * k4U : 0) + (ld_c ? k4U * k4U : 0) +
                              (ld_h ? k4U * k4U : 0) + (apply ? k4SK : 0));
  auto issue = [&](int t) {  // plane set of iteration t: u(t), g(t), cells(t-1), rhs(t-1), carry
    const int r = t - t0;
    uint64_t* br = &bar[r & 1];
    fence_proxy_async();
    mbar_expect_tx(br, bytes_set);
    if (ld_u) tma_load_3d(s4 + o4U + (r & 3) * k4SU, &A.tu, br, fk0 - 4, fj0 - 4, t);
    if (apply) {
      tma_load_3d(s4 + o4G + (r & 1) * k4SU, &A.tg, br, fk0 - 4, fj0 - 4, t);
      tma_load_3d(s4 + o4K + (r & 1) * k4SK, &A.tk, br, K0 - 2, J0 - 2, floor3(t));
    }
    if (ld_c) tma_load_3d(s4 + o4C + (r % 3) * k4SU, &A.tc, br, fk0 - 4, fj0 - 4, t - 1);
    if (ld_h) tma_load_3d(s4 + o4H + (r & 1) * k4SU, &A.th, br, fk0 - 4, fj0 - 4, t - 1);
  };
  if (lt == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (lt == 0 && !(dbg & 1)) issue(t0);

  for (int t = t0; t <= tEnd; ++t) {
    const int r = t - t0;
    if (!(dbg & 1)) {
      if (lt == 0 && t + 1 <= tEnd) issue(t + 1);
      mbar_wait(&bar[r & 1], (r >> 1) & 1);
    }

    // ---- A: u_new on plane t, in place in its slot ------------------------------
    double* Ut = s4 + o4U + (r & 3) * k4SU;
    if (!(dbg & 2) && apply && t >= 1 && t <= N - 2) {
      const double* Gt = s4 + o4G + (r & 1) * k4SU;
      const double* Kt = s4 + o4K + (r & 1) * k4SK;
      const int qi = t / 3, ri = t - 3 * qi;
      const bool town = t >= iOwnLo && t < iOwnHi;
      for (int q = lt; q < k4U * k4U; q += k4Threads) {
        const int jj = q / k4U, kk = q - jj * k4U;
        const int j = fj0 - 4 + jj, k = fk0 - 4 + kk;
        if (j < 1 || k < 1 || j > N - 2 || k > N - 2) continue;
        const int qj = j / 3, rj = j - 3 * qj, qk = k / 3, rk = k - 3 * qk;
        const size_t w0 = ((size_t)qi * Nc + qj) * Nc + qk;
        const int c0 = (qj - J0 + 2) * k4K + (qk - K0 + 2);
        double acc = 0.0;
#pragma unroll
        for (int d = 7; d >= 0; --d) {
          const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
          if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
          const int sl = pslot(ri - 3 * di, rj - 3 * dj, rk - 3 * dk);
          const double wt = (sl == 62) ? 1.0 : __ldg(a.P + (size_t)sl * nvc + w0 + di * NcNc + dj * Nc + dk);
          acc = acc + wt * Kt[di * k4K * k4K + c0 + dj * k4K + dk];
        }
        const double c = acc + Gt[jj * k4U + kk];
        const double un = Ut[jj * k4U + kk] + c;
        Ut[jj * k4U + kk] = un;
        if (town && j >= fj0 && j < fjE && k >= fk0 && k < fkE) {
          a.u_out[(size_t)t * NN + (size_t)j * N + k] = un;
          int iq = t, jq = j, kq = k;
          for (int lc = a.l - 1; lc >= a.l0; --lc) {  // FAS injection walk-down
            if (iq % 3 || jq % 3 || kq % 3) break;
            iq /= 3;
            jq /= 3;
            kq /= 3;
            a.ul[lc][((size_t)iq * a.Nl[lc] + jq) * a.Nl[lc] + kq] = un;
          }
        }
      }
    }
    __syncthreads();

    // ---- B: rho and the Jacobi correction on plane p = t - 1 ------------------------
    const int p = t - 1;
    double* Rb = s4 + o4R;
    if (!(dbg & 4) && p >= 1 && p <= N - 2 && p >= 3 * Ia - 3) {
      const double* Um = s4 + o4U + ((r + 2) & 3) * k4SU;  // plane p - 1 (slot of r - 2)
      const double* U0 = s4 + o4U + ((r + 3) & 3) * k4SU;  // plane p
      const double* Up = Ut;                                // plane p + 1
      const double* Cm = s4 + o4C + ((r + 2) % 3) * k4SU;  // cell plane p - 1 (set r - 1)
      const double* C0 = s4 + o4C + (r % 3) * k4SU;        // cell plane p (set r)
      const double* H = s4 + o4H + (r & 1) * k4SU;
      const bool pown = p >= iOwnLo && p < iOwnHi;
      for (int q = lt; q < k4SR; q += k4Threads) {
        const int jj = q / k4R, kk = q - jj * k4R;
        const int j = fj0 - 3 + jj, k = fk0 - 3 + kk;
        double rho = 0.0;
        if (j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2) {
          const int u0 = (jj + 1) * k4U + (kk + 1);
          double x[27];
#pragma unroll
          for (int s = 0; s < 9; ++s) {
            const int o = (s / 3 - 1) * k4U + (s % 3 - 1);
            x[s] = Um[u0 + o];
            x[9 + s] = U0[u0 + o];
            x[18 + s] = Up[u0 + o];
          }
          double au, dg;
          if (KIND == OP_CONST) {
            au = const_from(x, a.op.m, a.op.se, a.op.sc);
            dg = a.op.cdiag;
          } else {
            double e[8], E, T;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int c0 = c & 1, c1 = (c >> 1) & 1, c2 = c >> 2;
              e[c] = (c0 ? Cm : C0)[u0 - c1 * k4U - c2];
            }
            element_ET(x, e, E, T);
            dg = K_D * E;
            au = (dg * x[13]) - (K_E * T);
          }
          const double rhs = has_rhs ? H[u0] : 0.0;
          rho = rhs - au;
          if (pown && j >= fj0 && j < fjE && k >= fk0 && k < fkE) {
            const double tt = a.hw * rho;
            s_sum = s_sum + tt * tt;
            s_max = fmax(s_max, fabs(rho));
            a.g_out[(size_t)p * NN + (size_t)j * N + k] = (a.w * rho) / dg;
          }
        }
        Rb[q] = rho;
      }
    } else {
      for (int q = lt; q < k4SR; q += k4Threads) Rb[q] = 0.0;
    }
    __syncthreads();

    // ---- C: sm(p - 1) completes, sm(p) and sm(p + 1) advance --------------------------
    double* Sb = s4 + o4S;
    if (jac && !(dbg & 8)) {
      const bool sok = p - 1 >= 1 && p - 1 <= N - 2;
#pragma unroll
      for (int m = 0; m < k4Cols; ++m) {
        if (scol[m] < 0) continue;
        const int q = scol[m];
        const int jj = q / k4S, kk = q - jj * k4S;
        const int r0 = (jj + 1) * k4R + (kk + 1);
        const double f0 = Rb[r0 - k4R], f1 = Rb[r0 - 1], f2 = Rb[r0 + 1], f3 = Rb[r0 + k4R];
        const double d0 = Rb[r0 - k4R - 1], d1 = Rb[r0 - k4R + 1], d2 = Rb[r0 + k4R - 1], d3 = Rb[r0 + k4R + 1];
        const double xc = Rb[r0];
        // sm(p - 1): plane p is its +1 plane
        double se = (((SEa[m] + f0) + f1) + f2) + f3;
        double sc = (((SCa[m] + d0) + d1) + d2) + d3;
        double v = ((C_D8 * XA[m]) - (C_E6 * se)) - (C_C12 * sc);
        v = v * a.scale;
        Sb[q] = (sok && sin_[m]) ? v : 0.0;
        // sm(p): plane p is its middle plane (diagonal neighbours are its edges)
        SEa[m] = (((SEb[m] + d0) + d1) + d2) + d3;
        SCa[m] = SCb[m];
        XA[m] = xc;
        // sm(p + 1): plane p is its -1 plane
        SEb[m] = ((f0 + f1) + f2) + f3;
        SCb[m] = ((d0 + d1) + d2) + d3;
      }
    }
    __syncthreads();

    // ---- D: restriction of rho(p) and sm(p - 1) --------------------------------------
    if (rtask && !(dbg & 16)) {
      const int s = task_f ? p - 1 : p;
      if (s >= 3 * Ia - 2) {
        const int m3 = floor3(s), o = s - 3 * m3;
        const double* src = task_f ? Sb + (3 * (rJ - J0) + 2) * k4S + (3 * (rK - K0) + 2)
                                   : Rb + (3 * (rJ - J0) + 3) * k4R + (3 * (rK - K0) + 3);
        const int ld = task_f ? k4S : k4R;
        const bool zc_f = task_f == 0 && zc;
        // coarse plane m3 (offset o), then m3 + 1 (offset o - 3) when o >= 1
        if (m3 >= Ilo && m3 <= Ihi) {
          const size_t vc = ((size_t)m3 * Nc + rJ) * Nc + rK;
          double acc = accC;
#pragma unroll
          for (int q = 0; q < 25; ++q) {
            const int oj = q / 5 - 2, ok = q % 5 - 2;
            const int sl = (o + 2) * 25 + q;
            const bool ctr = o == 0 && q == 12;
            const double wt = ctr ? 1.0 : __ldg(a.P + (size_t)sl * nvc + vc);
            double x = src[oj * ld + ok];
            if (ctr && zc_f) x = 0.0;
            acc = acc + wt * x;
          }
          accC = acc;
          if (o == 2) (task_f ? a.bT : a.bR)[vc] = acc;
        }
        if (o >= 1 && m3 + 1 >= Ilo && m3 + 1 <= Ihi) {
          const size_t vc = ((size_t)(m3 + 1) * Nc + rJ) * Nc + rK;
          double acc = accN;
#pragma unroll
          for (int q = 0; q < 25; ++q) {
            const int oj = q / 5 - 2, ok = q % 5 - 2;
            const int sl = (o - 1) * 25 + q;
            acc = acc + __ldg(a.P + (size_t)sl * nvc + vc) * src[oj * ld + ok];
          }
          accN = acc;
        }
        if (o == 2) {
          accC = accN;
          accN = 0.0;
        }
      }
    }
  }

  // stats partials of this CTA
  for (int o = 16; o > 0; o >>= 1) {
    s_sum += __shfl_down_sync(0xffffffffu, s_sum, o);
    s_max = fmax(s_max, __shfl_down_sync(0xffffffffu, s_max, o));
  }
  if ((lt & 31) == 0) {
    red_s[lt >> 5] = s_sum;
    red_m[lt >> 5] = s_max;
  }
  __syncthreads();
  if (lt == 0) {
    double S = 0.0, M = 0.0;
    for (int q = 0; q < k4Threads / 32; ++q) {
      S += red_s[q];
      M = fmax(M, red_m[q]);
    }
    a.part_sum[blockIdx.x] = S;
    a.part_max[blockIdx.x] = M;
  }
}

}  // namespace t3
