// d-linear prolongation (geometric flavour) with compile-time weights (k3_up_lin).
//
// k3_up_cell<false> evaluates mg3d.prolong_dlinear per fine vertex with run-time
// quotients / remainders and fp64 divisions for the weights: ncu shows 320
// instructions per fine vertex and the kernel issue-bound (74 % issue active, 1 TB/s
// on config 3's finest level).  Here a warp owns one fine row (ri, rj) of 32 coarse
// cubes along K, so the weights 1 - r/3 are constants, the coarse corners are loaded
// once per thread for its three fine vertices and the only integer work is the
// address of the row.  Same expression order as prolong_dlinear (axis 0, then 1,
// then 2; wl c[q] + (1 - wl) c[q + 1]); terms with weight 0 are skipped.
#include "kernels3d.cuh"

namespace t3 {

constexpr int kLWarps = 9, kLThreads = 32 * kLWarps;

struct UpL {
  Up3 a;
  int tilesK, I0, nI;
  long long units;  // (cube layer I, cube row J, K tile)
};

template <int RI, int RJ>
__device__ __forceinline__ void lin_row(const Up3& a, int I, int J, int K) {
  const int Nc = a.Nc, N = a.N;
  const int i = 3 * I + RI, j = 3 * J + RJ;
  if (i < a.ilo || i >= a.ihi || (RJ == 0 && J == 0)) return;
  constexpr double wli = 1.0 - (double)RI / 3.0, wri = 1.0 - wli;
  constexpr double wlj = 1.0 - (double)RJ / 3.0, wrj = 1.0 - wlj;
  const double* cc = a.carry_c;
  double T1[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    double T0[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (b && !RJ) continue;
      const double lo = __ldg(cc + vid(Nc, I, J + b, K + c));
      T0[b] = RI ? wli * lo + wri * __ldg(cc + vid(Nc, I + 1, J + b, K + c)) : lo;
    }
    T1[c] = RJ ? wlj * T0[0] + wrj * T0[1] : T0[0];
  }
  const size_t v0 = vid(N, i, j, 3 * K);
  double un0 = 0.0;
#pragma unroll
  for (int rk = 0; rk < 3; ++rk) {
    if (rk == 0 && K == 0) continue;  // boundary vertex k = 0
    const double wlk = 1.0 - (double)rk / 3.0, wrk = 1.0 - wlk;
    const double pc = rk ? wlk * T1[0] + wrk * T1[1] : T1[0];
    const double cv = a.g ? pc + __ldg(a.g + v0 + rk) : pc;
    const double un = a.u[v0 + rk] + cv;
    a.u[v0 + rk] = un;
    if (a.carry) a.carry[v0 + rk] = cv;
    if (rk == 0) un0 = un;
  }
  if (RI == 0 && RJ == 0 && K > 0) {  // FAS walk-down injection of the coarse vertex (I, J, K)
    int ii = I, jj = J, kk = K;
    for (int lc = a.l - 1; lc >= a.l0; --lc) {
      a.ul[lc][vid(a.Nl[lc], ii, jj, kk)] = un0;
      if (ii % 3 || jj % 3 || kk % 3) break;
      ii /= 3;
      jj /= 3;
      kk /= 3;
    }
  }
}

__global__ void __launch_bounds__(kLThreads) k3_up_lin(const __grid_constant__ UpL A) {
  const int nc = A.a.Nc - 1;
  const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
  for (long long unit = blockIdx.x; unit < A.units; unit += gridDim.x) {
    const int tk = (int)(unit % A.tilesK);
    const long long r = unit / A.tilesK;
    const int J = (int)(r % nc), I = A.I0 + (int)(r / nc);
    const int K = tk * 32 + lane;
    if (K >= nc) continue;
    switch (wrp) {
      case 0: lin_row<0, 0>(A.a, I, J, K); break;
      case 1: lin_row<0, 1>(A.a, I, J, K); break;
      case 2: lin_row<0, 2>(A.a, I, J, K); break;
      case 3: lin_row<1, 0>(A.a, I, J, K); break;
      case 4: lin_row<1, 1>(A.a, I, J, K); break;
      case 5: lin_row<1, 2>(A.a, I, J, K); break;
      case 6: lin_row<2, 0>(A.a, I, J, K); break;
      case 7: lin_row<2, 1>(A.a, I, J, K); break;
      default: lin_row<2, 2>(A.a, I, J, K); break;
    }
  }
}

}  // namespace t3
