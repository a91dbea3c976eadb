// adaFACx smoothing of a level fused with the restriction into the next coarser one, for the
// DENSE weight stream (k3_smr): sm = A1(rho) * (omega * 3 / 8) never goes to HBM and rho is read
// once.  This is the path of coefficients whose BoxMG rows do not repeat (per-cell random eps:
// no row dictionary); when level l-1's P has a dictionary the cell-owned kernel k3_smc
// (kernels3d_smc.cu) runs instead.
//
// A CTA (one per SM) owns a 32 (K) x 4 (J) tile of interior coarse vertices and a chunk of coarse
// planes, and marches the fine planes p of the chunk, one CTA barrier per step:
//   rho(p)  arrives by TMA (box 100 x 16 from fine (3K0-3, 3J0-3): the restriction footprint plus
//           the smoothing halo) into a ring slot, and the P weights fine plane p-1 meets (two 4D
//           boxes of 25 slots over the tile, coarse planes m and m+1) into a set of a second ring;
//   C       threads [0, 256): sm(p-1) completes by plane partial sums -- a thread owns 7 sm
//           columns of the 98 x 14 window (27 shared loads per 7 columns, shared row sums,
//           about 10 fp64 operations per column and plane), double buffered;
//   D       threads [256, 384): one thread per coarse vertex restricts fine plane p-2 (one step
//           behind) into both coarse planes it feeds, both fields with one weight load.
// Summation order differs from the oracle's (3D bar: relative 1e-10).
#include <cuda.h>

#include "kernels3d.cuh"

namespace t3 {

constexpr int kRK = 32, kRJ = 4;                  // coarse tile (K, J)
constexpr int kRTasks = 2 * kRK * kRJ;            // 256 smoothing threads
constexpr int kRThreads = kRTasks + kRK * kRJ;    // + 128 restriction threads
constexpr int kRW = 3 * kRK + 4, kRH = 3 * kRJ + 4;  // rho window 100 x 16
constexpr int kSW = 3 * kRK + 2, kSH = 3 * kRJ + 2;  // sm window 98 x 14
constexpr int kRSlot = ((kRW * kRH * 8 + 127) / 128) * 128 / 8;
constexpr int kRStages = 5;                        // rho plane ring
constexpr int kPW = kRK + 2;                       // P box rows from K0 - 1 (16-byte aligned start): 34
constexpr int kPBox = (kPW * kRJ * 25 + 15) / 16 * 16;  // one 25-slot P box (27.2 KB; 128-byte multiple)
constexpr int kPStages = 2;                        // P sets (two boxes each)
constexpr int kSBuf = (kRW * kSH + 15) / 16 * 16;  // one sm plane (double buffered), pitch kRW like rho's
constexpr int kSGH = 7;                            // sm columns per smoothing thread (rows jj .. jj + 6 at kk)
constexpr int kSGroups = kSW * (kSH / kSGH);       // 196 groups on 256 threads
static_assert(kSH % kSGH == 0 && kSGroups <= kRTasks, "column groups tile the sm window");
constexpr int oRP = kRStages * kRSlot, oRS = oRP + kPStages * 2 * kPBox;
constexpr size_t kSmrSmem = sizeof(double) * (oRS + 2 * kSBuf);

struct Smr {
  CUtensorMap tr;  // rho of the fine level, box {100, 16, 1}
  CUtensorMap tp;  // P of the coarse level as {Nc, Nc, Nc, 125}, box {34, 4, 1, 25}
  int N, Nc;       // fine / coarse vertices per axis
  int tilesK, chunk;
  int jac, zc;     // adaFACx (b_T too); afacc (the centre tap of rho reads 0)
  double scale;    // omega*3/8
  double* bR;
  double* bT;
  int ilo, ihi;  // coarse planes [ilo, ihi) this launch restricts into (sharded: the owned ones)
};

__device__ __forceinline__ int floor3s(int x) { return x >= 0 ? x / 3 : -((2 - x) / 3); }

// the 25 in-plane terms of a fine plane for the coarse planes it feeds (C: plane m3, NX: m3 + 1)
template <bool C, bool NX, bool JAC>
__device__ __forceinline__ void terms2(const double* wc, const double* wn, int ws, const double* xr,
                                       const double* xs, bool ctr0, bool zc, double& cR, double& cS,
                                       double& nR, double& nS) {
  constexpr int ld = kRW;
#pragma unroll
  for (int q = 0; q < 25; ++q) {
    const int oj = q / 5 - 2, ok = q % 5 - 2;
    const double x = xr[oj * ld + ok];
    const double y = JAC ? xs[oj * ld + ok] : 0.0;
    if (C) {
      const bool ctr = ctr0 && q == 12;
      const double wt = ctr ? 1.0 : wc[q * ws];
      cR = cR + wt * ((ctr && zc) ? 0.0 : x);
      if (JAC) cS = cS + wt * y;
    }
    if (NX) {
      const double wt = wn[q * ws];
      nR = nR + wt * x;
      if (JAC) nS = nS + wt * y;
    }
  }
}

__global__ void __launch_bounds__(kRThreads, 1) k3_smr(const __grid_constant__ Smr A) {
  extern __shared__ __align__(128) double sr[];
  __shared__ __align__(8) uint64_t bar[kRStages], pbar[kPStages];
  const int N = A.N, Nc = A.Nc, n = Nc - 2;
  const int tk = blockIdx.x % A.tilesK, tj = blockIdx.x / A.tilesK;
  const int K0 = 1 + tk * kRK, J0 = 1 + tj * kRJ;
  const int Ia = A.ilo + blockIdx.y * A.chunk, Ib = min(A.ihi, Ia + A.chunk);  // coarse planes [Ia, Ib)
  if (Ia >= Ib) return;
  const int fk0 = 3 * K0 - 3, fj0 = 3 * J0 - 3;  // rho window origin (fine)
  const int p0 = 3 * Ia - 3, pEnd = 3 * Ib;       // rho planes streamed: [p0, pEnd]
  const int s0 = 3 * Ia - 2;                      // fine planes restricted: [s0, pEnd - 1]
  const int lt = threadIdx.x;
  const bool smoother = lt < kRTasks;

  // smoothing thread: its group's window offset (rows 7 jp .., column kk), the interior mask of
  // its columns and their state (SEa = F(t-2) + D(t-1), SCa = D(t-2), XA = x(t-1), SEb = F(t-1),
  // SCb = D(t-1); F / D = the in-plane edge / diagonal neighbour sums of a plane)
  const int jp = lt / kSW, kk = lt - jp * kSW;
  const int sbase = (smoother && lt < kSGroups) ? (kSGH * jp) * kRW + kk : -1;
  unsigned smask = 0u;
#pragma unroll
  for (int h = 0; h < kSGH; ++h) {
    const int j = fj0 + 1 + kSGH * jp + h, k = fk0 + 1 + kk;
    if (lt < kSGroups && j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2) smask |= 1u << h;
  }
  double SEa[kSGH], SCa[kSGH], XA[kSGH], SEb[kSGH], SCb[kSGH];
#pragma unroll
  for (int m = 0; m < kSGH; ++m) SEa[m] = SCa[m] = XA[m] = SEb[m] = SCb[m] = 0.0;
  // restriction thread: coarse (J, K) of the tile, both coarse planes a fine plane feeds, both fields
  const int w = lt - kRTasks;
  const int wj = w / kRK, wk = w % kRK;
  const int rJ = J0 + wj, rK = K0 + wk;
  const bool rtask = !smoother && rJ <= n && rK <= n;
  double accR = 0.0, accS = 0.0, accNR = 0.0, accNS = 0.0;

  auto issue_r = [&](int p) {  // rho plane p into its slot
    const int sl = (p - p0) % kRStages;
    mbar_expect_tx(&bar[sl], (unsigned)(sizeof(double) * kRW * kRH));
    tma_load_3d(sr + sl * kRSlot, &A.tr, &bar[sl], fk0, fj0, p);
  };
  auto issue_p = [&](int s) {  // the P boxes fine plane s meets into its set
    const int sl = (s - s0) % kPStages;
    const int m3 = floor3s(s), o = s - 3 * m3;
    const bool c = m3 >= Ia && m3 < Ib, nx = o >= 1 && m3 + 1 >= Ia && m3 + 1 < Ib;
    mbar_expect_tx(&pbar[sl], (unsigned)(sizeof(double) * kPW * kRJ * 25) * ((c ? 1u : 0u) + (nx ? 1u : 0u)));
    double* dst = sr + oRP + sl * 2 * kPBox;
    if (c) tma_load_4d(dst, &A.tp, &pbar[sl], K0 - 1, J0, m3, (o + 2) * 25);
    if (nx) tma_load_4d(dst + kPBox, &A.tp, &pbar[sl], K0 - 1, J0, m3 + 1, (o - 1) * 25);
  };
  if (lt == 0) {
    for (int q = 0; q < kRStages; ++q) mbar_init(&bar[q], 1);
    for (int q = 0; q < kPStages; ++q) mbar_init(&pbar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (lt == 0) {
    for (int p = p0; p <= min(pEnd, p0 + 2); ++p) issue_r(p);
    for (int s = s0; s <= min(pEnd - 1, s0 + kPStages - 1); ++s) issue_p(s);
  }

  const double kD8s = C_D8 * A.scale, kE6s = C_E6 * A.scale, kC12s = C_C12 * A.scale;
  // C: sm of the plane below rho's slot Rp completes into Sb:
  // sm(t-1) = scale (8/3 x(t-1) - 1/6 (F(t-2) + D(t-1) + F(t)) - 1/12 (D(t-2) + D(t)))
  auto smooth_body = [&](const double* Rp, double* Sb, bool sok) {
    if (sbase < 0) return;
    const unsigned mk = sok ? smask : 0u;
    double Rc[kSGH + 2], Ra[kSGH + 2];
#pragma unroll
    for (int a = 0; a < kSGH + 2; ++a) {
      Rc[a] = Rp[sbase + a * kRW + 1];
      Ra[a] = Rp[sbase + a * kRW] + Rp[sbase + a * kRW + 2];
    }
#pragma unroll
    for (int h = 0; h < kSGH; ++h) {
      const double Dt = Ra[h] + Ra[h + 2];
      const double Ft = (Rc[h] + Rc[h + 2]) + Ra[h + 1];
      const double se = SEa[h] + Ft, sc = SCa[h] + Dt;
      const double v = (kD8s * XA[h] - kE6s * se) - kC12s * sc;
      Sb[sbase + h * kRW] = ((mk >> h) & 1u) ? v : 0.0;
      SEa[h] = SEb[h] + Dt;
      SCa[h] = SCb[h];
      XA[h] = Rc[h + 1];
      SEb[h] = Ft;
      SCb[h] = Dt;
    }
  };
  // D: restriction of fine plane s (rho in slot ssl, sm in smb) into coarse planes m3 / m3 + 1
  auto restrict_body = [&](int ssl, int m3, int o, const double* smb, int ps) {
    const bool c = m3 >= Ia && m3 < Ib, nx = o >= 1 && m3 + 1 >= Ia && m3 + 1 < Ib;
    if (!rtask) return;
    const double* xr = sr + ssl * kRSlot + (3 * wj + 3) * kRW + 3 * wk + 3;
    const double* xs = smb + (3 * wj + 2) * kRW + 3 * wk + 2;
    const double* wc = sr + oRP + (ps % kPStages) * 2 * kPBox + wj * kPW + wk + 1;
    const double* wn = wc + kPBox;
    constexpr int ws = kRJ * kPW;
    const bool c0 = o == 0, zc = A.zc != 0;
    if (c && nx) {
      if (A.jac) terms2<true, true, true>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
      else terms2<true, true, false>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
    } else if (c) {
      if (A.jac) terms2<true, false, true>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
      else terms2<true, false, false>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
    } else if (nx) {
      if (A.jac) terms2<false, true, true>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
      else terms2<false, true, false>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
    }
    if (o == 2) {
      if (c) {
        const size_t ix = ((size_t)m3 * Nc + rJ) * Nc + rK;
        A.bR[ix] = accR;
        if (A.jac) A.bT[ix] = accS;
      }
      accR = accNR;
      accS = accNS;
      accNR = accNS = 0.0;
    }
  };

  // step t: C completes sm(t-1) from rho(t); D restricts fine plane s = t - 2.  Running counters:
  // rsl / rph = ring slot and barrier parity of rho(t), m3c / oc = floor(s / 3) and s mod 3
  int rsl = 0, m3c = Ia - 2, oc = 1;
  unsigned rph = 0u;
  for (int t = p0; t <= pEnd + 1; ++t) {
    if (t > p0) {
      if (++rsl == kRStages) {
        rsl = 0;
        rph ^= 1u;
      }
      if (++oc == 3) {
        oc = 0;
        ++m3c;
      }
      __syncthreads();  // step t-1 done: rho(t-3)'s slot and P(t-3)'s set are free, sm(t-2) is written
      if (lt == 0) {
        fence_proxy_async();
        if (t + 2 <= pEnd) issue_r(t + 2);                              // into the slot of plane t - 3
        if (t - 1 >= s0 + kPStages && t - 1 <= pEnd - 1) issue_p(t - 1);  // into the set of plane t - 3
      }
    }
    if (smoother) {
      // every rho plane's TMA is waited for here (also without smoothing): a slot is re-armed only
      // after its previous load completed, and no load is in flight when the CTA exits
      if (t <= pEnd) mbar_wait(&bar[rsl], rph);
      if (A.jac && t <= pEnd) smooth_body(sr + rsl * kRSlot, sr + oRS + ((t - 1) & 1) * kSBuf, t - 1 >= 1 && t - 1 <= N - 2);
    } else {
      const int s = t - 2;
      if (s >= s0) {
        const int ps = s - s0;
        const int ssl = rsl >= 2 ? rsl - 2 : rsl + kRStages - 2;  // slot / parity of rho(s)
        const unsigned sph = rsl >= 2 ? rph : rph ^ 1u;
        mbar_wait(&pbar[ps % kPStages], (unsigned)(ps / kPStages) & 1u);
        mbar_wait(&bar[ssl], sph);  // rho(s): visibility of the TMA write
        restrict_body(ssl, m3c, oc, sr + oRS + (s & 1) * kSBuf, ps);
      }
    }
  }
}

}  // namespace t3
