// Finest-level down sweep (element operator): two rows per thread with a register window along i
// (k3_top4r).
//
// Its predecessor (four rows per thread, no window) re-read the three u planes and two cell planes
// of every step from the shared-memory ring: 19.5 shared loads per vertex, l1tex 75 % busy, 161
// registers at 3 CTAs per SM, 2.79 ms at config 5.  Here a thread keeps u planes i-1, i and cell
// plane i-1 of its 4 x 3 / 3 x 2 window in registers and reads only the arriving packet {u plane
// i+1, cell plane i, rhs plane i} (12 + 6 + 2 loads per 2 vertices = 10 per vertex).  A packet's
// slot is free as soon as it has been read, so a three-slot ring (42 KB per CTA) keeps as many
// planes in flight as the five-slot ring did.  The step loop is unrolled by 6 = lcm(3, 2): the
// u / cell window rotation is compile-time renaming, no register moves.  Measured at config 5:
// two rows at 2 CTAs x 256 threads per SM (128 registers) 2.70 ms; four rows at 3 x 128 threads
// (168 registers, 388 bytes of spills) 3.16 ms, at 2 x 128 threads (206 registers) 3.03 ms.  Per
// vertex the expression is element_ET's.
#include "kernels3d.cuh"

namespace t3 {

constexpr int kT4S = 3;  // packets in flight
constexpr size_t kTop4rSmem = sizeof(double) * kT4S * (k2SlotU + k2SlotC + k2SlotR);

constexpr int kT4R = 2;                                   // rows per thread
constexpr int kT4X = kSX, kT4B = kSX * (k2Y / kT4R);      // 32 x 8 threads

__global__ void __launch_bounds__(kT4B, 2) k3_top4r(const __grid_constant__ Top3 a) {
  extern __shared__ __align__(128) double dyn4r[];
  __shared__ uint64_t bars[kT4S];
  auto us = reinterpret_cast<double(*)[k2SlotU]>(dyn4r);
  auto cs = reinterpret_cast<double(*)[k2SlotC]>(dyn4r + kT4S * k2SlotU);
  auto rs = reinterpret_cast<double(*)[k2SlotR]>(dyn4r + kT4S * (k2SlotU + k2SlotC));
  const Column2 col(a.N, a.ilo, a.ihi, a.chunk);
  const int N = a.N;
  const size_t NN = (size_t)N * N;
  const int tx = threadIdx.x, jj = kT4R * threadIdx.y;
  const int k = col.k0 + tx, j = col.j0 + jj;
  const size_t col_off = (size_t)j * N + k;
  const int ia = col.ia, ib = col.ib;
  const bool live = k <= N - 2 && j <= N - 2;
  double s = 0.0, mx = 0.0;
  if (col.lt == 0) {
    for (int q = 0; q < kT4S; ++q) mbar_init(&bars[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // packet g = {u plane ia - 1 + g, cell plane ia - 2 + g, rhs plane ia - 2 + g}, g = 0 .. ib - ia + 1
  const int last = ib - ia + 1;
  auto issue = [&](int g) {
    if (g > last) return;
    const int sl = g % kT4S, pu = ia - 1 + g, pc = pu - 1;
    mbar_expect_tx(&bars[sl], k2BoxBytes + k2BoxBytesC + 8u * k2SlotR);
    tma_load_3d(us[sl], &a.tm, &bars[sl], col.k0 - 1, col.j0 - 1, pu);
    tma_load_3d(cs[sl], &a.tmc, &bars[sl], col.k0 - 1, col.j0 - 1, pc < 0 ? -1 : pc / a.crun);
    tma_load_3d(rs[sl], &a.tmr, &bars[sl], col.k0 - 1, col.j0, pc);
  };
  if (col.lt == 0)
    for (int g = 0; g < kT4S; ++g) issue(g);
  double U[3][(kT4R + 2) * 3], C[2][(kT4R + 1) * 2];
  auto read_u = [&](int sl, double* u18) {
#pragma unroll
    for (int r = 0; r < kT4R + 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) u18[r * 3 + c] = us[sl][(jj + r) * k2RowU + tx + c];
  };
  auto read_c = [&](int sl, double* c10) {
#pragma unroll
    for (int r = 0; r < kT4R + 1; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) c10[r * 2 + c] = cs[sl][(jj + r) * k2RowC + tx + c];
  };
  // prologue: packets 0 (u plane ia - 1) and 1 (u plane ia, cell plane ia - 1)
  mbar_wait(&bars[0], 0u);
  read_u(0, U[0]);
  mbar_wait(&bars[1], 0u);
  read_u(1, U[1]);
  read_c(1, C[0]);
  __syncthreads();
  if (col.lt == 0) {
    fence_proxy_async();
    issue(3);
    issue(4);
  }
  // step i (phase ph = (i - ia) % 6): packet g = i - ia + 2 in slot (ph + 2) % 3
  auto step = [&](auto PH, int i) {
    constexpr int ph = decltype(PH)::value;
    constexpr int sl = (ph + 2) % 3;
    double* Um = U[ph % 3];
    double* U0 = U[(ph + 1) % 3];
    double* Up = U[(ph + 2) % 3];
    double* Cm = C[ph % 2];
    double* C0 = C[(ph + 1) % 2];
    const int g = i - ia + 2;
    mbar_wait(&bars[sl], (unsigned)(g / kT4S) & 1u);
    read_u(sl, Up);
    read_c(sl, C0);
    double rhs[kT4R];
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) rhs[aa] = rs[sl][(jj + aa) * k2RowR + tx + 1];
    __syncthreads();  // the slot is read: refill it with packet g + 3
    if (col.lt == 0) {
      fence_proxy_async();
      issue(g + kT4S);
    }
    if (!live) return;
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) {
      if (j + aa > N - 2) continue;
      double x[27], e[8];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          x[r * 3 + c] = Um[(aa + r) * 3 + c];
          x[9 + r * 3 + c] = U0[(aa + r) * 3 + c];
          x[18 + r * 3 + c] = Up[(aa + r) * 3 + c];
        }
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // cell (i - bit0, j + aa - bit1, k - bit2)
        const int c0b = c & 1, c1 = (c >> 1) & 1, c2 = c >> 2;
        e[c] = (c0b ? Cm : C0)[(aa + 1 - c1) * 2 + 1 - c2];
      }
      double E, T;
      element_ET(x, e, E, T);
      const double dg = K_D * E;
      const double au = (dg * x[13]) - (K_E * T);
      const double rho = rhs[aa] - au;
      const double t = a.hw * rho;
      s = s + t * t;
      mx = fmax(mx, fabs(rho));
      const size_t v = (size_t)i * NN + col_off + (size_t)aa * N;
      const double gv = (a.w * rho) / dg;
      if (a.u_out) a.u_out[v] = x[13] + gv;
      else a.g[v] = gv;
      if (a.rho) a.rho[v] = rho;
    }
  };
  for (int i0 = ia; i0 < ib; i0 += 6) {
    step(std::integral_constant<int, 0>{}, i0);
    if (i0 + 1 < ib) step(std::integral_constant<int, 1>{}, i0 + 1);
    if (i0 + 2 < ib) step(std::integral_constant<int, 2>{}, i0 + 2);
    if (i0 + 3 < ib) step(std::integral_constant<int, 3>{}, i0 + 3);
    if (i0 + 4 < ib) step(std::integral_constant<int, 4>{}, i0 + 4);
    if (i0 + 5 < ib) step(std::integral_constant<int, 5>{}, i0 + 5);
  }
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
