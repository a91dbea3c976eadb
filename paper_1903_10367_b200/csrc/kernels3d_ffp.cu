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

constexpr size_t kFfpSmem = sizeof(double) * (3 * kFU * kFU + 3 * kFR * kFR + kFS * kFS + 2 * kFC * kFC);

__global__ void __launch_bounds__(kFThreads, 2) k3_ffp(const __grid_constant__ Ffp3 a) {
  extern __shared__ double ffp_smem[];  // kFfpSmem bytes (dynamic: > 48 KB)
  double(*U)[kFU][kFU] = reinterpret_cast<double(*)[kFU][kFU]>(ffp_smem);
  double(*R)[kFR][kFR] = reinterpret_cast<double(*)[kFR][kFR]>(ffp_smem + 3 * kFU * kFU);
  double(*S)[kFS] = reinterpret_cast<double(*)[kFS]>(ffp_smem + 3 * kFU * kFU + 3 * kFR * kFR);
  double(*CE)[kFC][kFC] =
      reinterpret_cast<double(*)[kFC][kFC]>(ffp_smem + 3 * kFU * kFU + 3 * kFR * kFR + kFS * kFS);
  const int N = a.N, Nc = a.Nc, nc = Nc - 1, n = N - 1;
  const size_t NN = (size_t)N * N, nvc = (size_t)Nc * Nc * Nc;
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
  double s_sum = 0.0, s_max = 0.0;
  // restriction task of this thread: coarse (wj, wk), field (0: rho, 1: sm), slot parity
  const int tw = lt & 63, tf = (lt >> 6) & 1, tsl = lt >> 7;
  const int rJ = J0 + (tw >> 3), rK = K0 + (tw & 7);
  const bool rtask = (tf == 0 || a.jac) && rJ >= 1 && rJ <= nc - 1 && rK >= 1 && rK <= nc - 1;
  double racc = 0.0;

  auto interior = [&](int i, int j, int k) {
    return i >= 1 && j >= 1 && k >= 1 && i <= N - 2 && j <= N - 2 && k <= N - 2;
  };

  for (int i = 3 * Ia - 4; i <= 3 * Ib + 3; ++i) {
    // ---- A: u_new on plane i (window offset -4), cell plane i-1 --------------
    if (i >= 0 && i <= N - 1) {
      const int qi = i / 3, ri = i - 3 * qi;
      for (int q = lt; q < kFU * kFU; q += kFThreads) {
        const int jj = q / kFU, kk = q - jj * kFU;
        const int j = fj0 - 4 + jj, k = fk0 - 4 + kk;
        double un = 0.0;
        if (j >= 0 && k >= 0 && j <= N - 1 && k <= N - 1) {
          const size_t v = (size_t)i * NN + (size_t)j * N + k;
          un = __ldg(a.u_in + v);
          if (a.apply && interior(i, j, k)) {
            const int qj = j / 3, rj = j - 3 * qj, qk = k / 3, rk = k - 3 * qk;
            double acc = 0.0;
#pragma unroll
            for (int d = 7; d >= 0; --d) {
              const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
              if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
              const size_t wv = ((size_t)(qi + di) * Nc + (qj + dj)) * Nc + (qk + dk);
              const int sl = pslot(ri - 3 * di, rj - 3 * dj, rk - 3 * dk);
              const double wt = (sl == 62) ? 1.0 : __ldg(a.P + (size_t)sl * nvc + wv);
              acc = acc + wt * __ldg(a.carry_c + wv);
            }
            const double c = acc + __ldg(a.g_in + v);
            un = un + c;
            if (i >= iOwnLo && i < iOwnHi && j >= fj0 && j < fjE && k >= fk0 && k < fkE) {
              a.u_out[v] = un;
              int ii = i, jq = j, kq = k;
              for (int lc = a.l - 1; lc >= a.l0; --lc) {  // FAS injection walk-down
                if (ii % 3 || jq % 3 || kq % 3) break;
                ii /= 3;
                jq /= 3;
                kq /= 3;
                a.ul[lc][((size_t)ii * a.Nl[lc] + jq) * a.Nl[lc] + kq] = un;
              }
            }
          }
        }
        U[i % 3][jj][kk] = un;
      }
    }
    if (element && i - 1 >= 0 && i - 1 <= n - 1) {
      const int cp = i - 1;
      for (int q = lt; q < kFC * kFC; q += kFThreads) {
        const int jj = q / kFC, kk = q - jj * kFC;
        const int cj = fj0 - 4 + jj, ck = fk0 - 4 + kk;
        CE[cp & 1][jj][kk] = (cj >= 0 && ck >= 0 && cj < n && ck < n)
                                 ? __ldg(a.op.e + ((size_t)cp * n + cj) * n + ck) : 0.0;
      }
    }
    __syncthreads();
    // ---- B: rho on plane p = i-1 (window offset -3) ---------------------------
    const int p = i - 1;
    if (p >= 0 && p <= N - 1) {
      for (int q = lt; q < kFR * kFR; q += kFThreads) {
        const int jj = q / kFR, kk = q - jj * kFR;
        const int j = fj0 - 3 + jj, k = fk0 - 3 + kk;
        double rho = 0.0;
        if (interior(p, j, k)) {
          double x[27];
#pragma unroll
          for (int t = 0; t < 27; ++t)
            x[t] = U[(p + t / 9 - 1 + 3) % 3][jj + 1 + (t / 3) % 3 - 1][kk + 1 + t % 3 - 1];
          double au, dg;
          if (!element) {
            au = const_from(x, a.op.m, a.op.se, a.op.sc);
            dg = a.op.cdiag;
          } else {
            double e[8], E, T;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int c0 = c & 1, c1 = (c >> 1) & 1, c2 = c >> 2;
              e[c] = CE[(p - c0) & 1][jj + 1 - c1][kk + 1 - c2];
            }
            element_ET(x, e, E, T);
            dg = K_D * E;
            au = (dg * x[13]) - (K_E * T);
          }
          const size_t v = (size_t)p * NN + (size_t)j * N + k;
          const double rhs = a.rhs ? __ldg(a.rhs + v) : 0.0;
          rho = rhs - au;
          if (p >= iOwnLo && p < iOwnHi && j >= fj0 && j < fjE && k >= fk0 && k < fkE) {
            const double t = a.hw * rho;
            s_sum = s_sum + t * t;
            s_max = fmax(s_max, fabs(rho));
            a.g_out[v] = (a.w * rho) / dg;
          }
        }
        R[p % 3][jj][kk] = rho;
      }
    }
    __syncthreads();
    // ---- C: sm on plane s = i-2 (window offset -2) -----------------------------
    const int s = i - 2;
    const bool sok = s >= 0 && s <= N - 1;
    if (sok && a.jac) {
      for (int q = lt; q < kFS * kFS; q += kFThreads) {
        const int jj = q / kFS, kk = q - jj * kFS;
        const int j = fj0 - 2 + jj, k = fk0 - 2 + kk;
        double v = 0.0;
        if (interior(s, j, k)) {
          double x[27];
#pragma unroll
          for (int t = 0; t < 27; ++t)
            x[t] = R[(s + t / 9 - 1 + 3) % 3][jj + 1 + (t / 3) % 3 - 1][kk + 1 + t % 3 - 1];
          v = const_from(x, C_D8, C_E6, C_C12);
          v = v * a.scale;
        }
        S[jj][kk] = v;
      }
    }
    __syncthreads();
    // ---- D: restriction of plane s into the owned coarse planes ------------------
    if (sok && rtask) {
      // coarse planes I with |s - 3I| <= 2: ceil((s-2)/3) = s/3 and floor((s+2)/3)
      // (at most two, consecutive); this thread takes the one of its parity
      const int cA = s / 3, cB = (s + 2) / 3;
      int I = -1;
      if ((cA & 1) == tsl) I = cA;
      else if ((cB & 1) == tsl) I = cB;
      if (I >= 1 && I <= nc - 1 && I >= Ia && I < Ib) {
        const int oi = s - 3 * I;
        const size_t vc = ((size_t)I * Nc + rJ) * Nc + rK;
        const int bj = 3 * (rJ - J0), bk = 3 * (rK - K0);
        double acc = racc;
#pragma unroll
        for (int o = 0; o < 25; ++o) {
          const int oj = o / 5 - 2, ok = o % 5 - 2;
          const int sl = pslot(oi, oj, ok);
          const double wt = (sl == 62) ? 1.0 : __ldg(a.P + (size_t)sl * nvc + vc);
          double x = tf ? S[bj + oj + 2][bk + ok + 2] : R[s % 3][bj + oj + 3][bk + ok + 3];
          if (sl == 62 && tf == 0 && a.variant == VAR_AFACC) x = 0.0;
          acc = acc + wt * x;
        }
        racc = acc;
        if (oi == 2) {
          (tf ? a.bT : a.bR)[vc] = acc;
          racc = 0.0;
        }
      }
    }
    // the next step's A overwrites U slot (i+1)%3 == (i-2)%3, read by this step's B
    // (planes i-2..i) -- the barrier after B orders it; S is next written after the
    // next step's second barrier.
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
