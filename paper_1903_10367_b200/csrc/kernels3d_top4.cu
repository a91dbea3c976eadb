// Finest-level down sweep with four rows per thread (k3_top4).
//
// k3_top2 (two rows j per thread) is bound by shared-memory bandwidth: per
// vertex it reads 18 u values and 6 cell coefficients from the TMA-filled plane
// ring.  Here a thread owns the column k of rows j .. j+3, so per 4 vertices it
// reads u rows j-1 .. j+4 x k-1 .. k+1 x 3 planes (54 values = 13.5 per vertex)
// and cells rows j-1 .. j+3 x k-1, k x 2 planes (20 = 5 per vertex): 22 % fewer
// shared-memory bytes per vertex, lanes still 8 bytes apart along k (no bank
// conflicts).  Same CTA tile (32 k x 16 j), plane ring and TMA boxes
// (stream25x2), 128 threads.  Per vertex the expression DAG is element_ET's, so
// g and rho are bitwise k3_top2's; the residual-norm partials are summed in a
// different order (the norm is reduced order-free anyway).  Measured alternative:
// a 4-stage ring at 4 CTAs per SM (launch bound 128 registers: 312 bytes of
// spills) runs 3.75 vs 2.85 ms at config 5.
#include "kernels3d.cuh"

namespace t3 {

constexpr int kT4R = 4;                      // rows per thread
constexpr int kT4X = kSX, kT4Y = k2Y / kT4R, kT4B = kT4X * kT4Y;  // 32 x 4 threads

__global__ void __launch_bounds__(kT4B, 3) k3_top4(const __grid_constant__ Top3 a) {
  extern __shared__ __align__(128) double dyn4[];  // k2TopSmem
  __shared__ uint64_t bars[k2TopStages];
  auto us = reinterpret_cast<double(*)[k2SlotU]>(dyn4);
  auto cs = reinterpret_cast<double(*)[k2SlotC]>(dyn4 + k2TopStages * k2SlotU);
  auto rs = reinterpret_cast<double(*)[k2SlotR]>(dyn4 + k2TopStages * (k2SlotU + k2SlotC));
  const Column2 col(a.N, a.ilo, a.ihi, a.chunk);
  const int N = a.N;
  const size_t NN = (size_t)N * N;
  const int tx = threadIdx.x, jj = kT4R * threadIdx.y;  // column, first row in the tile
  const int k = col.k0 + tx, j = col.j0 + jj;
  const size_t col_off = (size_t)j * N + k;
  double s = 0.0, mx = 0.0;
  stream25x2<k2TopStages, true>(col, a.u, a.op.e, us, cs, &a.tm, bars,
      [&](int i, const double* pm, const double* p0, const double* pp, const double* cm,
          const double* c0, const double* r0) {
        if (k > N - 2 || j > N - 2) return;
        double U[3][kT4R + 2][3];  // u rows j-1 .. j+4, columns k-1 .. k+1, planes i-1 .. i+1
        const double* P3[3] = {pm, p0, pp};
#pragma unroll
        for (int pl = 0; pl < 3; ++pl)
#pragma unroll
          for (int r = 0; r < kT4R + 2; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) U[pl][r][c] = P3[pl][(jj + r) * k2RowU + tx + c];
        double Cc[2][kT4R + 1][2];  // cells rows j-1 .. j+3, columns k-1, k; cell planes i (c0), i-1 (cm)
        const double* C2[2] = {c0, cm};
#pragma unroll
        for (int pl = 0; pl < 2; ++pl)
#pragma unroll
          for (int r = 0; r < kT4R + 1; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) Cc[pl][r][c] = C2[pl][(jj + r) * k2RowC + tx + c];
#pragma unroll
        for (int aa = 0; aa < kT4R; ++aa) {
          if (j + aa > N - 2) continue;
          double x[27], e[8];
#pragma unroll
          for (int pl = 0; pl < 3; ++pl)
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int c = 0; c < 3; ++c) x[pl * 9 + r * 3 + c] = U[pl][aa + r][c];
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // cell (i - bit0, j + aa - bit1, k - bit2)
            const int c0b = c & 1, c1 = (c >> 1) & 1, c2 = c >> 2;
            e[c] = Cc[c0b][aa + 1 - c1][1 - c2];
          }
          double E, T;
          element_ET(x, e, E, T);
          const double dg = K_D * E;
          const double au = (dg * x[13]) - (K_E * T);
          const double rhs = r0[(jj + aa) * k2RowR + tx + 1];
          const double rho = rhs - au;
          const double t = a.hw * rho;
          s = s + t * t;
          mx = fmax(mx, fabs(rho));
          const size_t v = (size_t)i * NN + col_off + (size_t)aa * N;
          const double gv = (a.w * rho) / dg;
          if (a.u_out) a.u_out[v] = x[13] + gv;
          else a.g[v] = gv;
          if (a.rho) a.rho[v] = rho;
        }
      },
      &a.tmc, &a.tmr, rs, a.crun);
  __shared__ double red_s[kT4B / 32], red_m[kT4B / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  }
  const int lt = threadIdx.y * kT4X + threadIdx.x;
  if ((lt & 31) == 0) { red_s[lt >> 5] = s; red_m[lt >> 5] = mx; }
  __syncthreads();
  if (lt == 0) {
    double A = 0.0, B = 0.0;
    for (int q = 0; q < kT4B / 32; ++q) { A += red_s[q]; B = fmax(B, red_m[q]); }
    a.part_sum[blockIdx.x] = A;
    a.part_max[blockIdx.x] = B;
  }
}

}  // namespace t3
