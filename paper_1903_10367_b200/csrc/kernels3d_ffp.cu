// Fused fine pass (FFP) of the 3D cycle with BoxMG transfers.
//
// The pipelined schedule of the reference's single-touch engine
// (pipeline.py:242-386, "n cycles take n + 1 sweeps"): one sweep over the
// finest level per cycle that
//   A. completes the previous cycle's update  u_new = u + (P carry_c + g)
//      (solvers.py:386-395) and its FAS injection into the coarser levels
//      (solvers.py:283-288),
//   B. computes this cycle's residual, Jacobi correction g = (w rho)/diag and
//      the residual-norm partials (solvers.py:345-359, 435-443),
//   C. smooths rho for adaFACx, sm = A1(rho) * (omega*3/8) (operators.py:603),
//   D. restricts rho and sm to the coarse level, b = R rho, bt = R sm
//      (solvers.py:360-371),
// so every BoxMG weight is fetched from HBM once per cycle (the restriction
// re-reads it from L2 two planes after the prolongation), and rho / sm never
// reach HBM.  Per-element DAGs are exactly those of kernels3d.cu (oracle
// mg3d): the iterates stay bit-identical to the unfused cycle.
//
// CTA = 8 x 8 coarse (J, K) column, 24 x 24 owned fine vertices, marching a
// chunk of coarse planes; windows with halo: u_new 30^2 (fine offset -4), rho
// 28^2 (-3), sm 26^2 (-2), cells 29^2 (-4).  Rings of three u_new / rho
// planes and two cell planes live in shared memory.  Stage pipeline at step
// i: A(i), B(i-1), C+D(i-2).
#include "kernels3d.cuh"

namespace t3 {

constexpr int kFK = kFT + 4;  // coarse carry window (J0-2 .. J0+kFT+1)
constexpr size_t kFfpSmem =
    sizeof(double) * (3 * kFU * kFU + 3 * kFR * kFR + kFS * kFS + 2 * kFC * kFC + 2 * kFK * kFK);

__global__ void __launch_bounds__(kFThreads, 3) k3_ffp(const __grid_constant__ Ffp3 a) {
  extern __shared__ double ffp_smem[];  // kFfpSmem bytes (dynamic: > 48 KB)
  double* const Ub = ffp_smem;                              // [3][kFU*kFU]
  double* const Rb = Ub + 3 * kFU * kFU;                    // [3][kFR*kFR]
  double* const Sb = Rb + 3 * kFR * kFR;                    // [kFS*kFS]
  double* const Cb = Sb + kFS * kFS;                        // [2][kFC*kFC]
  double* const CCb = Cb + 2 * kFC * kFC;                   // [2][kFK*kFK] coarse carry planes
  const int N = a.N, Nc = a.Nc, nc = Nc - 1, n = N - 1;
  const size_t NN = (size_t)N * N, nvc = (size_t)Nc * Nc * Nc, NcNc = (size_t)Nc * Nc;
  int b = blockIdx.x;
  const int tk = b % a.tiles;
  b /= a.tiles;
  const int tj = b % a.tiles;
  const int tc = b / a.tiles;
  const int J0 = tj * kFT, K0 = tk * kFT;
  const int Ia = tc * a.chunk, Ib = min(Nc, Ia + a.chunk);
  const int fj0 = 3 * J0, fk0 = 3 * K0;             // first owned fine j / k
  const int fjE = min(fj0 + 3 * kFT, N - 1), fkE = min(fk0 + 3 * kFT, N - 1);
  const int iOwnLo = 3 * Ia, iOwnHi = min(3 * Ib, N - 1);
  const int lt = threadIdx.x;
  const bool element = a.op.kind == OP_ELEMENT;
  const int cj0 = J0 - 2, ck0 = K0 - 2;              // coarse carry window origin
  double s_sum = 0.0, s_max = 0.0;
  // restriction task of this thread: coarse (wj, wk), field (0: rho, 1: sm), slot parity
  const int tw = lt & 63, tf = (lt >> 6) & 1, tsl = (lt >> 7) & 1;
  const int rJ = J0 + (tw >> 3), rK = K0 + (tw & 7);
  const bool rtask = lt < 256 && (tf == 0 || a.jac) && rJ >= 1 && rJ <= nc - 1 && rK >= 1 && rK <= nc - 1;
  double racc = 0.0;

  for (int i = 3 * Ia - 4; i <= 3 * Ib + 3; ++i) {
    // ---- A: u_new on plane i (window offset -4), cell plane i-1, carry planes -----
    if (i >= 0 && i <= N - 1) {
      const int qi = i / 3, ri = i - 3 * qi;
      const bool ii_in = i >= 1 && i <= N - 2;
      if (a.apply && ii_in) {
        // coarse carry planes qi, qi+1 over the window J in [J0-2, J0+kFT+2)
        for (int q = lt; q < 2 * kFK * kFK; q += kFThreads) {
          const int pl = q / (kFK * kFK), r = q - pl * kFK * kFK;
          const int jj = r / kFK, kk = r - jj * kFK;
          const int I = qi + pl, J = cj0 + jj, K = ck0 + kk;
          CCb[q] = (pl <= (ri ? 1 : 0) && J >= 0 && K >= 0 && J <= nc && K <= nc)
                       ? __ldg(a.carry_c + ((size_t)I * Nc + J) * Nc + K) : 0.0;
        }
        __syncthreads();
      }
      double* Ui = Ub + (i % 3) * kFU * kFU;
      const double* Pp = a.P;
      for (int q = lt; q < kFU * kFU; q += kFThreads) {
        const int jj = q / kFU, kk = q - jj * kFU;
        const int j = fj0 - 4 + jj, k = fk0 - 4 + kk;
        double un = 0.0;
        if (j >= 0 && k >= 0 && j <= N - 1 && k <= N - 1) {
          const size_t v = (size_t)i * NN + (size_t)j * N + k;
          un = __ldg(a.u_in + v);
          if (a.apply && ii_in && j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2) {
            const int qj = j / 3, rj = j - 3 * qj, qk = k / 3, rk = k - 3 * qk;
            const size_t w0 = (size_t)qi * NcNc + (size_t)qj * Nc + qk;
            const int c0 = (qj - cj0) * kFK + (qk - ck0);
            const double g = __ldg(a.g_in + v);
            double acc = 0.0;
#pragma unroll
            for (int d = 7; d >= 0; --d) {
              const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
              if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
              const int sl = pslot(ri - 3 * di, rj - 3 * dj, rk - 3 * dk);
              const double wt =
                  (sl == 62) ? 1.0 : __ldg(Pp + (size_t)sl * nvc + w0 + di * NcNc + dj * Nc + dk);
              acc = acc + wt * CCb[di * kFK * kFK + c0 + dj * kFK + dk];
            }
            const double c = acc + g;
            un = un + c;
            if (i >= iOwnLo && i < iOwnHi && j >= fj0 && j < fjE && k >= fk0 && k < fkE) {
              a.u_out[v] = un;
              int iq = i, jq = j, kq = k;
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
        Ui[q] = un;
      }
    }
    if (element && i - 1 >= 0 && i - 1 <= n - 1) {
      const int cp = i - 1;
      double* Cp = Cb + (cp & 1) * kFC * kFC;
      const double* ep = a.op.e + (size_t)cp * n * n;
      for (int q = lt; q < kFC * kFC; q += kFThreads) {
        const int jj = q / kFC, kk = q - jj * kFC;
        const int cj = fj0 - 4 + jj, ck = fk0 - 4 + kk;
        Cp[q] = (cj >= 0 && ck >= 0 && cj < n && ck < n) ? __ldg(ep + (size_t)cj * n + ck) : 0.0;
      }
    }
    __syncthreads();
    // ---- B: rho on plane p = i-1 (window offset -3) ---------------------------
    const int p = i - 1;
    if (p >= 1 && p <= N - 2) {
      const double* Um = Ub + ((p + 2) % 3) * kFU * kFU;
      const double* U0 = Ub + (p % 3) * kFU * kFU;
      const double* Up = Ub + ((p + 1) % 3) * kFU * kFU;
      const double* Cm = Cb + ((p + 1) & 1) * kFC * kFC;  // cell plane p-1
      const double* C0 = Cb + (p & 1) * kFC * kFC;        // cell plane p
      double* Rp = Rb + (p % 3) * kFR * kFR;
      const bool pown = p >= iOwnLo && p < iOwnHi;
      const double* rhsp = a.rhs ? a.rhs + (size_t)p * NN : nullptr;
      for (int q = lt; q < kFR * kFR; q += kFThreads) {
        const int jj = q / kFR, kk = q - jj * kFR;
        const int j = fj0 - 3 + jj, k = fk0 - 3 + kk;
        double rho = 0.0;
        if (j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2) {
          const int u0 = (jj + 1) * kFU + (kk + 1);
          double x[27];
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const int o = (t / 3 - 1) * kFU + (t % 3 - 1);
            x[t] = Um[u0 + o];
            x[9 + t] = U0[u0 + o];
            x[18 + t] = Up[u0 + o];
          }
          double au, dg;
          if (!element) {
            au = const_from(x, a.op.m, a.op.se, a.op.sc);
            dg = a.op.cdiag;
          } else {
            const int e0 = (jj + 1) * kFC + (kk + 1);
            double e[8], E, T;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int c0 = c & 1, c1 = (c >> 1) & 1, c2 = c >> 2;
              e[c] = (c0 ? Cm : C0)[e0 - c1 * kFC - c2];
            }
            element_ET(x, e, E, T);
            dg = K_D * E;
            au = (dg * x[13]) - (K_E * T);
          }
          const size_t v = (size_t)j * N + k;
          const double rhs = rhsp ? __ldg(rhsp + v) : 0.0;
          rho = rhs - au;
          if (pown && j >= fj0 && j < fjE && k >= fk0 && k < fkE) {
            const double t = a.hw * rho;
            s_sum = s_sum + t * t;
            s_max = fmax(s_max, fabs(rho));
            a.g_out[(size_t)p * NN + v] = (a.w * rho) / dg;
          }
        }
        Rp[q] = rho;
      }
    } else if (p >= 0 && p <= N - 1) {
      double* Rp = Rb + (p % 3) * kFR * kFR;
      for (int q = lt; q < kFR * kFR; q += kFThreads) Rp[q] = 0.0;
    }
    __syncthreads();
    // ---- C: sm on plane s = i-2 (window offset -2) -----------------------------
    const int s = i - 2;
    const bool sok = s >= 1 && s <= N - 2;
    if (sok && a.jac) {
      const double* Rm = Rb + ((s + 2) % 3) * kFR * kFR;
      const double* R0 = Rb + (s % 3) * kFR * kFR;
      const double* Rq = Rb + ((s + 1) % 3) * kFR * kFR;
      for (int q = lt; q < kFS * kFS; q += kFThreads) {
        const int jj = q / kFS, kk = q - jj * kFS;
        const int j = fj0 - 2 + jj, k = fk0 - 2 + kk;
        double v = 0.0;
        if (j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2) {
          const int r0 = (jj + 1) * kFR + (kk + 1);
          double x[27];
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const int o = (t / 3 - 1) * kFR + (t % 3 - 1);
            x[t] = Rm[r0 + o];
            x[9 + t] = R0[r0 + o];
            x[18 + t] = Rq[r0 + o];
          }
          v = const_from(x, C_D8, C_E6, C_C12);
          v = v * a.scale;
        }
        Sb[q] = v;
      }
    }
    __syncthreads();
    // ---- D: restriction of plane s into the owned coarse planes ------------------
    if (sok && rtask) {
      // coarse planes I with |s - 3I| <= 2: s/3 and (s+2)/3 (at most two,
      // consecutive); this thread takes the one of its parity
      const int cA = s / 3, cB = (s + 2) / 3;
      int I = -1;
      if ((cA & 1) == tsl) I = cA;
      else if ((cB & 1) == tsl) I = cB;
      if (I >= 1 && I <= nc - 1 && I >= Ia && I < Ib) {
        const int oi = s - 3 * I;
        const size_t vc = (size_t)I * NcNc + (size_t)rJ * Nc + rK;
        const int bj = 3 * (rJ - J0), bk = 3 * (rK - K0);
        const double* src = tf ? Sb + (bj + 2) * kFS + (bk + 2) : Rb + (s % 3) * kFR * kFR + (bj + 3) * kFR + (bk + 3);
        const int ld = tf ? kFS : kFR;
        const bool zc = tf == 0 && a.variant == VAR_AFACC;
        double acc = racc;
#pragma unroll
        for (int o = 0; o < 25; ++o) {
          const int oj = o / 5 - 2, ok = o % 5 - 2;
          const int sl = (oi + 2) * 25 + o;
          const bool ctr = oi == 0 && o == 12;
          const double wt = ctr ? 1.0 : __ldg(a.P + (size_t)sl * nvc + vc);
          double x = src[oj * ld + ok];
          if (ctr && zc) x = 0.0;
          acc = acc + wt * x;
        }
        racc = acc;
        if (oi == 2) {
          (tf ? a.bT : a.bR)[vc] = acc;
          racc = 0.0;
        }
      }
    }
  }
  // stats partials of this CTA
  __shared__ double rs[kFThreads / 32], rm[kFThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s_sum += __shfl_down_sync(0xffffffffu, s_sum, o);
    s_max = fmax(s_max, __shfl_down_sync(0xffffffffu, s_max, o));
  }
  if ((lt & 31) == 0) { rs[lt >> 5] = s_sum; rm[lt >> 5] = s_max; }
  __syncthreads();
  if (lt == 0) {
    double A = 0.0, B = 0.0;
    for (int q = 0; q < kFThreads / 32; ++q) { A += rs[q]; B = fmax(B, rm[q]); }
    a.part_sum[blockIdx.x] = A;
    a.part_max[blockIdx.x] = B;
  }
}

}  // namespace t3
