// Finest-level down sweep (element operator): two rows per thread with a register window along i
// (k3_top4r).
//
// Its predecessor (four rows per thread, no window) re-read the three u planes and two cell planes
// of every step from the shared-memory ring: 19.5 shared loads per vertex, l1tex 75 % busy, 161
// registers at 3 CTAs per SM, 2.79 ms at config 5.  Here a thread keeps what it needs of u planes
// i - 1, i and cell plane i - 1 in registers and reads only the arriving packet {u plane i + 1, cell
// plane i, rhs plane i} (12 + 6 + 2 loads per 2 vertices = 10 per vertex); the step loop is unrolled
// by 2 (the window's double buffers are compile-time renaming), the ring slot is a run-time index.
// The operator is evaluated plane-wise instead of cell by cell (see "Register window" below):
// ~27 fp64 operations per vertex instead of element_ET's 42, 2.69 -> 2.47 ms at config 5.
// Measured alternatives: four rows at 3 x 128 threads (168 registers, 388 bytes of spills) 3.16 ms,
// at 2 x 128 threads (206 registers) 3.03 ms; warps decoupled by per-slot empty barriers instead of
// the per-step __syncthreads 0.04 ms slower; an L2 prefetch of the u / rhs boxes 2 / 4 packets ahead
// of the ring 0.09 / 0.10 ms slower.
#include "kernels3d.cuh"

namespace t3 {

// ring slots: a slot is refilled with the packet kT4S ahead as soon as the CTA has read it.  Measured
// per config-5 cycle: 3 slots 7.31 ms, 4 slots 7.25 ms, 5 / 6 / 7 slots 7.54 / 7.80 / 7.87 ms (more
// planes in flight per CTA spread the 296 resident columns over more DRAM pages and L2 sets).
constexpr int kT4S = 4;
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
  // packet g = {u plane ia - 1 + g, cell plane ia - 2 + g, rhs plane ia - 2 + g}, g = 0 .. ib - ia + 1,
  // in slot g % kT4S
  const int last = ib - ia + 1;
  auto issue = [&](int g) {  // thread 0
    if (g > last) return;
    const int sl = g % kT4S, pu = ia - 1 + g, pc = pu - 1;
    mbar_expect_tx(&bars[sl], k2BoxBytes + k2BoxBytesC + 8u * k2SlotR);
    tma_load_3d(us[sl], &a.tm, &bars[sl], col.k0 - 1, col.j0 - 1, pu);
    tma_load_3d(cs[sl], &a.tmc, &bars[sl], col.k0 - 1, col.j0 - 1, pc < 0 ? -1 : pc / a.crun);
    tma_load_3d(rs[sl], &a.tmr, &bars[sl], col.k0 - 1, col.j0, pc);
  };
  // the CTA has read the slot of packet g (and every earlier one): refill it
  auto refill = [&](int g) {
    __syncthreads();
    if (col.lt == 0) {
      fence_proxy_async();
      issue(g + kT4S);
    }
  };
  if (col.lt == 0)
    for (int g = 0; g < kT4S; ++g) issue(g);
  // Register window.  X[.]: a u plane's 4 x 3 neighbourhood of the thread's two vertices.  LS: per
  // vertex and quadrant (s1, s2) the "L sum" of a plane, x(j+s1, k) + x(j, k+s2) + x(j+s1, k+s2) --
  // the three vertices of that plane which the quadrant's cell couples to (j, k) with -1/12 from
  // the planes i - 1 and i + 1 (in-line neighbours have weight 0).  A plane's L sums serve the
  // vertex planes below and above it: they are formed once when the plane arrives (14 additions
  // per two vertices, the column pair sums of rows (j, j+1) serve both), multiplied with the
  // arriving cell plane for the vertex plane below, and once more with the next cell plane for the
  // vertex plane above (TL, one partial sum per vertex carried to the next step).  The own plane
  // contributes its four diagonal neighbours d with ep = e(i-1) + e(i):
  //   E = sum ep,  T = sum_q e_m L_m + e_p L_p + ep d    (~27 fp64 operations per vertex; the
  // cell-by-cell form element_ET spends 42).
  double X[2][(kT4R + 2) * 3], LS[kT4R * 4], C[2][(kT4R + 1) * 2], TL[kT4R];
  auto read_u = [&](int sl, double* u12) {
#pragma unroll
    for (int r = 0; r < kT4R + 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) u12[r * 3 + c] = us[sl][(jj + r) * k2RowU + tx + c];
  };
  auto read_c = [&](int sl, double* c6) {
#pragma unroll
    for (int r = 0; r < kT4R + 1; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) c6[r * 2 + c] = cs[sl][(jj + r) * k2RowC + tx + c];
  };
  // l8[aa * 4 + q], q = 2 * (s1 > 0) + (s2 > 0)
  auto lsums = [&](const double* u12, double* l8) {
    double V[kT4R + 1][2];  // column pair sums of rows (r, r + 1) at columns k - 1, k + 1
#pragma unroll
    for (int r = 0; r < kT4R + 1; ++r) {
      V[r][0] = u12[r * 3] + u12[(r + 1) * 3];
      V[r][1] = u12[r * 3 + 2] + u12[(r + 1) * 3 + 2];
    }
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int up = q >> 1, rt = q & 1;
        l8[aa * 4 + q] = u12[(aa + 2 * up) * 3 + 1] + V[aa + up][rt];
      }
  };
  // sum_q c[cell of quadrant q] * l8[q] of vertex aa (cell window index (aa + up) * 2 + rt)
  auto dotl = [&](const double* c6, const double* l8, int aa) {
    double t = c6[aa * 2] * l8[aa * 4];
    t = t + c6[aa * 2 + 1] * l8[aa * 4 + 1];
    t = t + c6[aa * 2 + 2] * l8[aa * 4 + 2];
    t = t + c6[aa * 2 + 3] * l8[aa * 4 + 3];
    return t;
  };
  // prologue: packets 0 (u plane ia - 1) and 1 (u plane ia, cell plane ia - 1)
  mbar_wait(&bars[0], 0u);
  read_u(0, X[1]);
  lsums(X[1], LS);
  mbar_wait(&bars[1], 0u);
  read_c(1, C[0]);
  read_u(1, X[0]);
  refill(0);
  refill(1);
#pragma unroll
  for (int aa = 0; aa < kT4R; ++aa) TL[aa] = dotl(C[0], LS, aa);
  lsums(X[0], LS);
  // step i (phase ph = (i - ia) % 2): packet g = i - ia + 2 in slot sl (parity par); on entry X0 =
  // u plane i, LS = its L sums, Cm = cell plane i - 1, TL = sum_q Cm L(i - 1)
  int sl = 2 % kT4S;
  unsigned par = 0u;
  auto step = [&](auto PH, int i) {
    constexpr int ph = decltype(PH)::value;
    double* X0 = X[ph % 2];
    double* Xp = X[(ph + 1) % 2];
    double* Cm = C[ph % 2];
    double* C0 = C[(ph + 1) % 2];
    const int g = i - ia + 2;
    mbar_wait(&bars[sl], par);
    read_c(sl, C0);
    double tn[kT4R];  // vertex plane i + 1's lower part: cell plane i with L(i)
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) tn[aa] = dotl(C0, LS, aa);
    read_u(sl, Xp);
    double rhs[kT4R];
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) rhs[aa] = rs[sl][(jj + aa) * k2RowR + tx + 1];
    refill(g);
    if (++sl == kT4S) {
      sl = 0;
      par ^= 1u;
    }
    lsums(Xp, LS);
    if (live) {
      double ep[(kT4R + 1) * 2], er[kT4R + 1];
#pragma unroll
      for (int q = 0; q < (kT4R + 1) * 2; ++q) ep[q] = Cm[q] + C0[q];
#pragma unroll
      for (int r = 0; r < kT4R + 1; ++r) er[r] = ep[r * 2] + ep[r * 2 + 1];
#pragma unroll
      for (int aa = 0; aa < kT4R; ++aa) {
        if (j + aa > N - 2) continue;
        const double E = er[aa] + er[aa + 1];
        // own plane: diagonal neighbour of quadrant q at window row aa + 2 up, column 2 rt
        double td = ep[aa * 2] * X0[aa * 3];
        td = td + ep[aa * 2 + 1] * X0[aa * 3 + 2];
        td = td + ep[aa * 2 + 2] * X0[(aa + 2) * 3];
        td = td + ep[aa * 2 + 3] * X0[(aa + 2) * 3 + 2];
        const double T = (TL[aa] + dotl(C0, LS, aa)) + td;
        const double xc = X0[(aa + 1) * 3 + 1];
        const double dg = K_D * E;
        const double au = (dg * xc) - (K_E * T);
        const double rho = rhs[aa] - au;
        const double t = a.hw * rho;
        s = s + t * t;
        mx = fmax(mx, fabs(rho));
        const size_t v = (size_t)i * NN + col_off + (size_t)aa * N;
        const double gv = div_pos(a.w * rho, dg);
        if (a.u_out) a.u_out[v] = xc + gv;
        else a.g[v] = gv;
        if (a.rho) a.rho[v] = rho;
      }
    }
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) TL[aa] = tn[aa];
  };
  for (int i0 = ia; i0 < ib; i0 += 2) {
    step(std::integral_constant<int, 0>{}, i0);
    if (i0 + 1 < ib) step(std::integral_constant<int, 1>{}, i0 + 1);
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

// The constant-coefficient flavour (config 3, OP_CONST): the same ring and register window without
// the cell planes.  The 27-point row is m at the centre, -se on the 12 edge and -sc on the 8 corner
// neighbours (0 on the faces), so a plane contributes through two sums per vertex: PE, its four
// in-plane axis neighbours, and PD, its four in-plane diagonals --
//   A u = m x - se (PE(i-1) + PE(i+1) + PD(i)) - sc (PD(i-1) + PD(i+1)).
// A plane's sums are formed once when it arrives (6 additions per vertex) and serve three vertex
// planes; k3_top2<OP_CONST> re-read all three planes from shared memory (18 loads and 26 additions
// per vertex).  Summation order differs from mg3d.apply_const's (3D bar: 1e-10).
constexpr size_t kTop4cSmem = sizeof(double) * kT4S * (k2SlotU + k2SlotR);

__global__ void __launch_bounds__(kT4B, 2) k3_top4c(const __grid_constant__ Top3 a) {
  extern __shared__ __align__(128) double dyn4c[];
  __shared__ uint64_t bars[kT4S];
  auto us = reinterpret_cast<double(*)[k2SlotU]>(dyn4c);
  auto rs = reinterpret_cast<double(*)[k2SlotR]>(dyn4c + kT4S * k2SlotU);
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
  const int last = ib - ia + 1;
  auto issue = [&](int g) {  // packet g = {u plane ia - 1 + g, rhs plane ia - 2 + g}
    if (g > last) return;
    const int sl = g % kT4S, pu = ia - 1 + g;
    mbar_expect_tx(&bars[sl], k2BoxBytes + 8u * k2SlotR);
    tma_load_3d(us[sl], &a.tm, &bars[sl], col.k0 - 1, col.j0 - 1, pu);
    tma_load_3d(rs[sl], &a.tmr, &bars[sl], col.k0 - 1, col.j0, pu - 1);
  };
  auto refill = [&](int g) {
    __syncthreads();
    if (col.lt == 0) {
      fence_proxy_async();
      issue(g + kT4S);
    }
  };
  if (col.lt == 0)
    for (int g = 0; g < kT4S; ++g) issue(g);
  // per vertex aa: (PE, PD) of the plane below, of the own plane, and the own centre
  double pem[kT4R], pdm[kT4R], pe0[kT4R], pd0[kT4R], xc[kT4R];
  auto sums = [&](int sl, double* pe, double* pd, double* ctr) {
    double w[(kT4R + 2) * 3];
#pragma unroll
    for (int r = 0; r < kT4R + 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) w[r * 3 + c] = us[sl][(jj + r) * k2RowU + tx + c];
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) {
      pe[aa] = (w[aa * 3 + 1] + w[(aa + 2) * 3 + 1]) + (w[(aa + 1) * 3] + w[(aa + 1) * 3 + 2]);
      pd[aa] = (w[aa * 3] + w[aa * 3 + 2]) + (w[(aa + 2) * 3] + w[(aa + 2) * 3 + 2]);
      ctr[aa] = w[(aa + 1) * 3 + 1];
    }
  };
  double dump[kT4R];
  mbar_wait(&bars[0], 0u);
  sums(0, pem, pdm, dump);
  mbar_wait(&bars[1], 0u);
  sums(1, pe0, pd0, xc);
  refill(0);
  refill(1);
  const double m = a.op.m, se = a.op.se, sc = a.op.sc, dg = a.op.cdiag;
  int sl = 2 % kT4S;
  unsigned par = 0u;
  for (int i = ia; i < ib; ++i) {
    const int g = i - ia + 2;
    mbar_wait(&bars[sl], par);
    double pep[kT4R], pdp[kT4R], xp[kT4R], rhs[kT4R];
    sums(sl, pep, pdp, xp);
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) rhs[aa] = rs[sl][(jj + aa) * k2RowR + tx + 1];
    refill(g);
    if (++sl == kT4S) {
      sl = 0;
      par ^= 1u;
    }
    if (live) {
#pragma unroll
      for (int aa = 0; aa < kT4R; ++aa) {
        if (j + aa > N - 2) continue;
        const double SE = (pem[aa] + pep[aa]) + pd0[aa];
        const double SC = pdm[aa] + pdp[aa];
        const double au = (m * xc[aa] - se * SE) - sc * SC;
        const double rho = rhs[aa] - au;
        const double t = a.hw * rho;
        s = s + t * t;
        mx = fmax(mx, fabs(rho));
        const size_t v = (size_t)i * NN + col_off + (size_t)aa * N;
        const double gv = div_pos(a.w * rho, dg);
        if (a.u_out) a.u_out[v] = xc[aa] + gv;
        else a.g[v] = gv;
        if (a.rho) a.rho[v] = rho;
      }
    }
#pragma unroll
    for (int aa = 0; aa < kT4R; ++aa) {
      pem[aa] = pe0[aa];
      pdm[aa] = pd0[aa];
      pe0[aa] = pep[aa];
      pd0[aa] = pdp[aa];
      xc[aa] = xp[aa];
    }
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
