// adaFACx smoothing of the finest level fused with the restriction into level
// ltop-1 (k3_smr): sm = A1(rho)*(omega*3/8) never goes to HBM, and rho is read
// once (here) instead of twice (smoothing + restriction).
//
// Phase-by-phase the cycle writes sm (3.1 GB at config 5) and reads rho and sm
// again in k3_down_c (6.2 GB + 3.8 GB of re-reads); this kernel reads the
// finest rho and level ltop-1's P once and writes b_R = R rho and b_T = R sm
// (what k3_down_c<.., PRE> consumes).
//
// A CTA (one per SM) owns a 32 (K) x 4 (J) tile of interior coarse vertices
// and a chunk of coarse planes, and marches the fine planes p of the chunk:
//   rho(p)  arrives by TMA (box 100 x 16 from fine (3K0-3, 3J0-3): the
//           restriction footprint plus the smoothing halo) into a ring slot,
//           and the P weights fine plane p-1 meets (two 4D boxes of 25 slots
//           over the tile, coarse planes m and m+1) into a set of a second ring;
//   C       sm(p-1) completes by plane partial sums: each thread owns fixed
//           sm columns of the 98 x 14 window and keeps, per column, the
//           sequential edge / corner sums of the pending sm planes (the DAG
//           of const_from is plane-major), so every rho plane is read once;
//   D       thread (coarse vertex, role) adds fine plane p-1 of rho and sm to
//           the two running sums of the coarse plane its role owns (the two
//           roles own alternate planes, so a plane's sums stay in one thread
//           over the five fine planes it meets), the 25 (ob, oc) terms of the
//           plane in order -- the oracle's o-order over the 125 offsets -- and
//           stores them when the plane completes.
// One weight load feeds both fields' products.  Same per-element DAGs as
// k3_smooth2r and k3_down_c: b_R, b_T and everything after them are bitwise
// unchanged.  Default schedule (engine3.cu: smr_dec; dictionary P): smoothing and
// restriction threads are decoupled -- they meet only through named barriers per
// sm buffer (full / empty pairs over three sm buffers, six rho slots), so the
// restriction lags the smoothing by up to three fine planes and its 25 | 50 | 50
// terms per step average out (2.80 vs 2.85-2.92 ms with one CTA barrier per
// step).  Default layout (engine3.cu: smr_rv / smr_gh): 256 smoothing threads
// owning groups of 7 sm columns (27 shared loads per 7 columns), 128 restriction
// threads, one per coarse vertex, carrying both coarse planes a fine plane feeds
// and both fields (the 5 x 5 x 2 window is read once for both planes) --
// 2.97 ms at config 5 L6 against 3.17 ms for the two-role / pairs layout
// (RV = 0, GH = 2).  Measured alternatives of the two-role layout: 768 smoothing threads with
// one column pair each (64 registers) 3.43 vs 3.17 ms; the restriction threads
// also completing the window's last 174 column pairs 3.52 ms; 16-byte weight
// loads no change -- that layout was bound by shared-memory bandwidth (l1tex
// 68 %: about 230 KB of shared loads per fine plane step) and the step barrier.
// The default layout runs at l1tex 53 % with barrier stalls first (29 %); a
// balanced schedule deferring parts of the offset -2 / -1 groups by one fine
// plane (42 | 42 | 41 terms per step instead of 25 | 50 | 50, six rho slots,
// three sm buffers; bitwise) measured slower, 3.29-3.44 vs 3.0 ms.
#include <cuda.h>

#include <type_traits>

#include "kernels3d.cuh"

namespace t3 {

constexpr int kRK = 32, kRJ = 4;                  // coarse tile (K, J)
constexpr int kRTasks = 2 * kRK * kRJ;            // 256 restriction tasks: (coarse vertex, field)
constexpr int kRThreads = 2 * kRTasks;            // 512: 256 smoothing threads + 256 restriction threads
constexpr int kRW = 3 * kRK + 4, kRH = 3 * kRJ + 4;  // rho window 100 x 16
constexpr int kSW = 3 * kRK + 2, kSH = 3 * kRJ + 2;  // sm window 98 x 14
constexpr int kRSlot = ((kRW * kRH * 8 + 127) / 128) * 128 / 8;
constexpr int kRStages = 5;                        // rho plane ring
constexpr int kPW = kRK + 2;                       // P box rows from K0 - 1 (16-byte aligned start): 34
constexpr int kPBox = (kPW * kRJ * 25 + 15) / 16 * 16;  // one 25-slot P box (27.2 KB; 128-byte multiple)
constexpr int kPStages = 2;                        // P sets (two boxes each)
constexpr int kSBuf = (kRW * kSH + 15) / 16 * 16;  // one sm plane (double buffered), pitch kRW like rho's
// a smoothing thread owns groups of GH sm columns (rows jj .. jj + GH - 1 at kk): GH = 2 (pairs, 3
// per thread, 12 shared loads per 2 columns) or GH = 7 (half the window's height, one group per
// thread, 27 loads per 7 columns)
template <int GH>
constexpr int kSPer = (kSW * (kSH / GH) + kRTasks - 1) / kRTasks;
static_assert(kSH % 2 == 0 && kSH % 7 == 0, "column groups tile the sm window");
static_assert(kSH % 2 == 0, "sm columns are paired along j");
constexpr int oRP = kRStages * kRSlot, oRS = oRP + kPStages * 2 * kPBox;
constexpr size_t kSmrSmem = sizeof(double) * (oRS + 2 * kSBuf);
// dictionary variant (P of the coarse level as a row dictionary, kernels3d_dict.cu): no P ring.
// For each coarse plane m of the tile a setup-built table (k3_smr_tables: the plane's <= kRRows
// distinct rows, each vertex's index into them) arrives by bulk copy 9 fine steps before the
// plane is first restricted into, and the rows themselves (one 1000-byte bulk copy each, from
// L2) 3 steps before, into a ring of three planes' row sets -- the weights are then read from
// shared memory as the dense boxes are, at 8 + 8 KB per coarse plane instead of 136 KB of HBM.
constexpr int kRRows = 32, kRRowS = 130;             // rows per tile plane (cap), row stride (doubles)
constexpr int kRTabBytes = 272;                      // {n, ids[32]} uint32, local[128] uint8 at byte 132
constexpr int kRTabLoc = 132;
constexpr int kRNT = 6;                              // table ring (coarse planes)
constexpr int oRTab = kRStages * kRSlot;
constexpr int oRRows = oRTab + kRNT * kRTabBytes / 8;
constexpr int kRRowSet = kRRows * kRRowS;
constexpr int oRSd = oRRows + 3 * kRRowSet;
constexpr size_t kSmrSmemD = sizeof(double) * (oRSd + 2 * kSBuf);
// decoupled schedule (DEC): six rho slots and three sm buffers, so the restriction may lag the
// smoothing by up to three fine planes
constexpr int kRStagesB = 6;
constexpr size_t kSmrSmemDB =
    sizeof(double) * (kRStagesB * kRSlot + kRNT * kRTabBytes / 8 + 3 * kRRowSet + 3 * kSBuf);
static_assert(kSmrSmemDB + 256 <= 227 * 1024, "DEC layout exceeds shared memory");
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr unsigned kRRowBytes = 126 * 8;  // 125 weights, rounded to 16 bytes (rows are 1 KB)

// tables of the dictionary variant: one thread per (coarse plane m, tile); *over = 1 when a tile
// plane meets more than kRRows distinct rows (the dense P stream is kept then)
__global__ void k3_smr_tables(const uint32_t* __restrict__ ids, int Nc, int Ncp, int tilesK, int tilesJ,
                              uint8_t* __restrict__ tab, int* over) {
  const int n = Nc - 2;
  const size_t cnt = (size_t)n * tilesJ * tilesK;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (size_t)gridDim.x * blockDim.x) {
    const int tk = (int)(t % tilesK), tj = (int)((t / tilesK) % tilesJ), m = 1 + (int)(t / ((size_t)tilesK * tilesJ));
    uint32_t rows[kRRows];
    int cntr = 0;
    uint8_t* T8 = tab + t * kRTabBytes;
    for (int c = 0; c < kRK * kRJ; ++c) {
      const int J = 1 + tj * kRJ + c / kRK, K = 1 + tk * kRK + c % kRK;
      int loc = 0;
      if (J <= n && K <= n) {
        const uint32_t id = ids[((size_t)m * Nc + J) * Ncp + K];
        while (loc < cntr && rows[loc] != id) ++loc;
        if (loc == cntr) {
          if (cntr == kRRows) {
            atomicOr(over, 1);
            loc = 0;
          } else {
            rows[cntr++] = id;
          }
        }
      }
      T8[kRTabLoc + c] = (uint8_t)loc;
    }
    uint32_t* T = reinterpret_cast<uint32_t*>(T8);
    T[0] = (uint32_t)cntr;
    for (int q = 0; q < kRRows; ++q) T[1 + q] = q < cntr ? rows[q] : 0u;
  }
}

// the same tables when every vertex uses dictionary row 0 (the d-linear flavour: one constant row)
__global__ void k3_smr_tables_one(uint8_t* __restrict__ tab, size_t cnt) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (size_t)gridDim.x * blockDim.x) {
    uint32_t* T = reinterpret_cast<uint32_t*>(tab + t * kRTabBytes);
    T[0] = 1u;
    for (int q = 0; q < kRRows; ++q) T[1 + q] = 0u;
    for (int c = 0; c < kRK * kRJ; ++c) tab[t * kRTabBytes + kRTabLoc + c] = 0;
    for (int c = kRTabLoc + kRK * kRJ; c < kRTabBytes; ++c) tab[t * kRTabBytes + c] = 0;
  }
}

struct Smr {
  CUtensorMap tr;  // rho of the finest level, box {100, 16, 1}
  CUtensorMap tp;  // P of level ltop-1 as {Nc, Nc, Nc, 125}, box {34, 4, 1, 25}
  int N, Nc;       // finest / coarse vertices per axis
  int tilesK, chunk;
  int jac, zc;     // adaFACx (b_T too); afacc (the centre tap of rho reads 0)
  double scale;    // omega*3/8
  double* bR;
  double* bT;
  const double* pd;     // dictionary variant: P rows pd[id * kDictW + slot]
  const uint8_t* ptab;  // ... and the tile-plane tables, index ((m - 1) * tilesJ + tj) * tilesK + tk
  int tilesJ;
  int ilo, ihi;  // coarse planes [ilo, ihi) this launch restricts into (sharded: the owned ones)
};

__device__ __forceinline__ int floor3s(int x) { return x >= 0 ? x / 3 : -((2 - x) / 3); }

// Warp-specialised: threads [0, 256) complete sm(t-1) from rho(t) (phase C) while threads
// [256, 512) restrict fine plane t-2 (phase D, one step behind, sm double buffered), so the two
// latency-bound phases overlap; one CTA barrier per step.
// DICT: level ltop-1's P as a row dictionary (kernels3d_dict.cu): no P ring, each restriction
// thread reads its vertex's weights from the plane-major dictionary (L1-cached, the rows of a
// warp's vertices have neighbouring ids), the same doubles in the same order.
// RV = 1 (TMG_SMR_RV=1): one restriction thread per coarse vertex carrying both coarse planes and
// both fields (x loaded once for both planes), 128 restriction threads (384 per CTA)
template <bool C, bool NX, bool JAC, int Q0 = 0, int Q1 = 25>
__device__ __forceinline__ void terms2(const double* wc, const double* wn, int ws, const double* xr,
                                       const double* xs, bool ctr0, bool zc, double& cR, double& cS,
                                       double& nR, double& nS) {
  constexpr int ld = kRW;
#pragma unroll
  for (int q = Q0; q < Q1; ++q) {
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

// DEC: 256 restriction threads -- the 25 in-plane terms of a step are split between two threads of
// a coarse vertex (q < 13 | q >= 13, in different warps), whose partial sums meet through `comb`
// when a coarse plane completes: the restriction group was the critical path with one thread per
// vertex (ncu: the smoothing warps waited on its EMPTY barriers 42 % of their time).
constexpr int kRSplit = 13;
template <bool DICT, int RV, int GH, bool DEC = false>
__global__ void __launch_bounds__(DEC ? kRThreads : (RV ? kRTasks + kRK * kRJ : kRThreads), 1)
    k3_smr(const __grid_constant__ Smr A) {
  static_assert(RV == 1 && GH == 7, "one restriction thread (pair) per coarse vertex, 7-column smoothing groups");
  static_assert(!DEC || DICT, "the decoupled schedule needs the dictionary");
  constexpr int kSPairs = kSPer<GH>, kSCols = GH * kSPairs, kSGroups = kSW * (kSH / GH);
  constexpr int kRStages = DEC ? kRStagesB : t3::kRStages;  // rho slots
  constexpr int oRTab = kRStages * kRSlot;
  constexpr int oRRows = oRTab + kRNT * kRTabBytes / 8;
  constexpr int oRSd = oRRows + 3 * kRRowSet;
  extern __shared__ __align__(128) double sr[];
  __shared__ __align__(8) uint64_t bar[kRStagesB], pbar[kPStages], tbar[kRNT], rbar[3];
  __shared__ double comb[DEC ? 2 * kRK * kRJ : 2];  // DEC: the upper half's partial sums of a completed plane
  const int N = A.N, Nc = A.Nc, n = Nc - 2;
  const int tk = blockIdx.x % A.tilesK, tj = blockIdx.x / A.tilesK;
  const int K0 = 1 + tk * kRK, J0 = 1 + tj * kRJ;
  const int Ia = A.ilo + blockIdx.y * A.chunk, Ib = min(A.ihi, Ia + A.chunk);  // coarse planes [Ia, Ib)
  if (Ia >= Ib) return;
  const int fk0 = 3 * K0 - 3, fj0 = 3 * J0 - 3;  // rho window origin (fine)
  const int p0 = 3 * Ia - 3, pEnd = 3 * Ib;       // rho planes streamed: [p0, pEnd]
  const int s0 = 3 * Ia - 2;                      // fine planes restricted: [s0, pEnd - 1]
  constexpr int oS = DICT ? oRSd : oRS;           // sm double buffer
  const int lt = threadIdx.x;
  const bool smoother = lt < kRTasks;

  // smoothing threads: groups of GH sm columns (jj .. jj + GH - 1) at kk -- the group's 3 x 3 rho
  // neighbourhoods share rows (3 (GH + 2) shared loads per GH columns) -- and the columns'
  // pending partial sums
  // per group: its window offset (rows GH jp .., column kk) and the interior mask of its columns
  int sbase[kSPairs];
  unsigned smask[kSPairs];
  double SEa[kSCols], SCa[kSCols], XA[kSCols], SEb[kSCols], SCb[kSCols];
#pragma unroll
  for (int m = 0; m < kSPairs; ++m) {
    const int q2 = lt + m * kRTasks;
    const int jp = q2 / kSW, kk = q2 - jp * kSW;
    sbase[m] = (smoother && q2 < kSGroups) ? (GH * jp) * kRW + kk : -1;
    smask[m] = 0u;
#pragma unroll
    for (int h = 0; h < GH; ++h) {
      const int j = fj0 + 1 + GH * jp + h, k = fk0 + 1 + kk;
      if (q2 < kSGroups && j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2) smask[m] |= 1u << h;
    }
  }
#pragma unroll
  for (int m = 0; m < kSCols; ++m) SEa[m] = SCa[m] = XA[m] = SEb[m] = SCb[m] = 0.0;
  // restriction threads: coarse (J, K) of the tile, both fields (rho, sm) -- one weight load feeds
  // both products; role r owns the coarse planes m with (m - Ia) % 2 == r (warps 8-11: r = 0,
  // 12-15: r = 1), so a thread keeps its plane's two sums over all five fine planes it meets
  const int task = lt - kRTasks;
  const int role = RV ? 0 : (task >> 7) & 1, w = task & (kRK * kRJ - 1);
  const int half = DEC ? (task >> 7) & 1 : 0;  // DEC: which part of a step's 25 terms (warp-uniform)
  static_assert(kRK * kRJ == 128, "two restriction roles of 128 vertices");
  const int wj = w / kRK, wk = w % kRK;
  const int rJ = J0 + wj, rK = K0 + wk;
  const bool rtask = !smoother && rJ <= n && rK <= n;
  double accR = 0.0, accS = 0.0, accNR = 0.0, accNS = 0.0;
  // DEC, lower half: the completed plane's partial sums, stored once the upper half's are in `comb`
  double pendR = 0.0, pendS = 0.0;
  size_t pend_ix = 0;
  bool pending = false;
  auto flush_pending = [&]() {
    if (!pending) return;
    A.bR[pend_ix] = pendR + comb[2 * w];
    if (A.jac) A.bT[pend_ix] = pendS + comb[2 * w + 1];
    pending = false;
  };

  auto issue_r = [&](int p) {  // rho plane p into its slot
    const int sl = (p - p0) % kRStages;
    mbar_expect_tx(&bar[sl], (unsigned)(sizeof(double) * kRW * kRH));
    tma_load_3d(sr + sl * kRSlot, &A.tr, &bar[sl], fk0, fj0, p);
  };
  // DICT: coarse plane m's table (slot m % kRNT) / rows (set m % 3)
  // (slots and barrier phases count planes from this CTA's first, Ia)
  auto tab_of = [&](int m) {
    return reinterpret_cast<const uint8_t*>(sr + oRTab + ((m - Ia) % kRNT) * (kRTabBytes / 8));
  };
  auto issue_tab = [&](int m) {  // thread lt == kRTasks (restriction warp 0, lane 0)
    if (m < Ia || m >= Ib) return;
    uint64_t* tb = &tbar[(m - Ia) % kRNT];
    mbar_expect_tx(tb, kRTabBytes);
    bulk_load(sr + oRTab + ((m - Ia) % kRNT) * (kRTabBytes / 8),
              A.ptab + (((size_t)(m - 1) * A.tilesJ + tj) * A.tilesK + tk) * kRTabBytes, kRTabBytes, tb);
  };
  auto rows_of = [&](int m) { return sr + oRRows + ((m - Ia) % 3) * kRRowSet; };
  auto wait_plane = [&](int m) {  // table and rows of plane m are in
    mbar_wait(&tbar[(m - Ia) % kRNT], (unsigned)((m - Ia) / kRNT) & 1u);
    mbar_wait(&rbar[(m - Ia) % 3], (unsigned)((m - Ia) / 3) & 1u);
  };
  auto issue_rows = [&](int m, int lane) {  // restriction warp 0, lane-parallel
    if (m < Ia || m >= Ib) return;
    mbar_wait(&tbar[(m - Ia) % kRNT], (unsigned)((m - Ia) / kRNT) & 1u);
    const uint32_t* T = reinterpret_cast<const uint32_t*>(tab_of(m));
    const int nr = (int)T[0];
    uint64_t* rb = &rbar[(m - Ia) % 3];
    if (lane == 0) mbar_expect_tx(rb, kRRowBytes * (unsigned)nr);
    __syncwarp();
    if (lane < nr) bulk_load(rows_of(m) + lane * kRRowS, A.pd + (size_t)T[1 + lane] * kDictW, kRRowBytes, rb);
  };
  auto issue_p = [&](int s) {  // the P boxes fine plane s meets into its set
    if (DICT) return;
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
    for (int q = 0; q < kRNT; ++q) mbar_init(&tbar[q], 1);
    for (int q = 0; q < 3; ++q) mbar_init(&rbar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (lt == 0) {
    for (int p = p0; p <= min(pEnd, p0 + 2); ++p) issue_r(p);
    for (int s = s0; s <= min(pEnd - 1, s0 + kPStages - 1); ++s) issue_p(s);
  }
  // DICT schedule: at step t = 3m' (m' = t / 3): the table of plane m' + 3 and the rows of plane
  // m' + 1 (plane m is restricted into at steps 3m .. 3m + 4)
  if (DICT && lt == kRTasks) {
    issue_tab(p0 / 3 + 1);
    issue_tab(p0 / 3 + 2);
  }

  // C: sm of the plane below rho's slot Rp completes into Sb (pending partial sums advance).
  // Per column and plane: F = the 4 in-plane edge neighbours' sum, D = the 4 in-plane diagonals'
  // sum (the stencil has no face taps); sm(t-1) = scale (8/3 x(t-1) - 1/6 (F(t-2) + D(t-1) + F(t))
  // - 1/12 (D(t-2) + D(t))).  The rows' outer sums a_r = x[r][k-1] + x[r][k+1] are shared by the
  // group's columns (about 10 fp64 operations per column and plane; summation order differs from
  // the oracle's plane-major chain, within the 3D tolerance).  State per column: SEa = F(t-2) +
  // D(t-1), SCa = D(t-2), XA = x(t-1), SEb = F(t-1), SCb = D(t-1).
  const double kD8s = C_D8 * A.scale, kE6s = C_E6 * A.scale, kC12s = C_C12 * A.scale;
  auto smooth_body = [&](const double* Rp, double* Sb, bool sok) {
#pragma unroll
        for (int mp = 0; mp < kSPairs; ++mp) {
          if (sbase[mp] < 0) continue;
          // rows GH jp - 1 .. GH jp + GH, cols kk - 1 .. kk + 1 of the sm window (rho window + 1)
          const int rb = sbase[mp];
          const unsigned mk = sok ? smask[mp] : 0u;
          double Rc[GH + 2], Ra[GH + 2];
#pragma unroll
          for (int a = 0; a < GH + 2; ++a) {
            Rc[a] = Rp[rb + a * kRW + 1];
            Ra[a] = Rp[rb + a * kRW] + Rp[rb + a * kRW + 2];
          }
#pragma unroll
          for (int h = 0; h < GH; ++h) {
            const int m = GH * mp + h;
            const double Dt = Ra[h] + Ra[h + 2];
            const double Ft = (Rc[h] + Rc[h + 2]) + Ra[h + 1];
            const double se = SEa[m] + Ft, sc = SCa[m] + Dt;
            const double v = (kD8s * XA[m] - kE6s * se) - kC12s * sc;
            Sb[rb + h * kRW] = ((mk >> h) & 1u) ? v : 0.0;
            SEa[m] = SEb[m] + Dt;
            SCa[m] = SCb[m];
            XA[m] = Rc[h + 1];
            SEb[m] = Ft;
            SCb[m] = Dt;
          }
        }
  };
  // D (RV 1): restriction of fine plane s (rho in slot ssl, sm in smb) into coarse planes m3 / m3+1
  auto restrict_body = [&](int s, int ssl, int m3, int o, int k3c, int k6c, const double* smb, int ps) {
          const bool c = m3 >= Ia && m3 < Ib, nx = o >= 1 && m3 + 1 >= Ia && m3 + 1 < Ib;
          if (rtask) {
            const double* xr = sr + ssl * kRSlot + (3 * wj + 3) * kRW + 3 * wk + 3;
            const double* xs = smb + (3 * wj + 2) * kRW + 3 * wk + 2;
            const double* wc = nullptr;
            const double* wn = nullptr;
            int ws;
            if (DICT) {
              const double* rows = sr + oRRows;
              const uint8_t* tabs = reinterpret_cast<const uint8_t*>(sr + oRTab) + kRTabLoc + w;
              if (c) wc = rows + k3c * kRRowSet + tabs[k6c * kRTabBytes] * kRRowS + (o + 2) * 25;
              if (nx) {
                if (o == 1) wait_plane(m3 + 1);
                const int k3n = k3c == 2 ? 0 : k3c + 1, k6n = k6c == kRNT - 1 ? 0 : k6c + 1;
                wn = rows + k3n * kRRowSet + tabs[k6n * kRTabBytes] * kRRowS + (o - 1) * 25;
              }
              ws = 1;
            } else {
              wc = sr + oRP + (ps % kPStages) * 2 * kPBox + wj * kPW + wk + 1;
              wn = wc + kPBox;
              ws = kRJ * kPW;
            }
            const bool c0 = o == 0, zc = A.zc != 0;
            auto run = [&](auto Q0, auto Q1) {
              constexpr int q0 = decltype(Q0)::value, q1 = decltype(Q1)::value;
              if (c && nx) {
                if (A.jac) terms2<true, true, true, q0, q1>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
                else terms2<true, true, false, q0, q1>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
              } else if (c) {
                if (A.jac) terms2<true, false, true, q0, q1>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
                else terms2<true, false, false, q0, q1>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
              } else if (nx) {
                if (A.jac) terms2<false, true, true, q0, q1>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
                else terms2<false, true, false, q0, q1>(wc, wn, ws, xr, xs, c0, zc, accR, accS, accNR, accNS);
              }
            };
            using std::integral_constant;
            if (!DEC) run(integral_constant<int, 0>{}, integral_constant<int, 25>{});
            else if (half == 0) run(integral_constant<int, 0>{}, integral_constant<int, kRSplit>{});
            else run(integral_constant<int, kRSplit>{}, integral_constant<int, 25>{});
            if (o == 2) {
              if (c) {
                const size_t ix = ((size_t)m3 * Nc + rJ) * Nc + rK;
                if (!DEC) {
                  A.bR[ix] = accR;
                  if (A.jac) A.bT[ix] = accS;
                } else if (half) {  // read by the lower half after the next step's barrier
                  comb[2 * w] = accR;
                  comb[2 * w + 1] = accS;
                } else {
                  pend_ix = ix;
                  pendR = accR;
                  pendS = accS;
                  pending = true;
                }
              }
              accR = accNR;
              accS = accNS;
              accNR = accNS = 0.0;
            }
          }
  };
  if constexpr (DEC) {
    // Decoupled: the smoothing threads (barrier 7 among themselves) and the restriction threads
    // meet only through named barriers per sm buffer b (plane x in buffer (x - p0) % 3):
    //   FULL 1 + b   smoothing arrives when sm(x) is complete, the restriction syncs before x;
    //   EMPTY 4 + b  the restriction arrives when done with plane x (sm(x), rho(x)), the
    //                smoothing syncs before writing sm(x + 3) and re-arming rho(x)'s slot.
    // The restriction may lag by three planes; every arrive has exactly one matching sync.
    constexpr int kAll = kRThreads, kRest = kRThreads - kRTasks;
    auto sbuf = [&](int x) { return (x - p0 + 3) % 3; };  // x >= p0 - 1
    if (smoother) {
      int rsl = 0;
      unsigned rph = 0u;
      for (int t = p0; t <= pEnd; ++t) {
        if (t > p0 && ++rsl == kRStages) {
          rsl = 0;
          rph ^= 1u;
        }
        // buffer of t - 1 last held t - 4 and rho(t + 2)'s slot rho(t - 4): the restriction is done
        // with them, and (a sync of every thread) the smoothing group left step t - 1; before the
        // first such step the group syncs alone (rho(t - 4)'s slot)
        if (t - 1 >= s0 + 3) named_sync(4 + sbuf(t - 1), kAll);
        else named_sync(7, kRTasks);
        if (lt == 0 && t > p0 && t + 2 <= pEnd) {
          fence_proxy_async();
          issue_r(t + 2);
        }
        mbar_wait(&bar[rsl], rph);
        if (A.jac) smooth_body(sr + rsl * kRSlot, sr + oS + sbuf(t - 1) * kSBuf, t - 1 >= 1 && t - 1 <= N - 2);
        if (t - 1 >= s0) named_arrive(1 + sbuf(t - 1), kAll);
      }
    } else {
      if (lt < kRTasks + 32) {  // the first planes' table and rows (step t = p0 of the coupled loop)
        fence_proxy_async();
        if (lt == kRTasks) issue_tab(Ia + 2);
        issue_rows(Ia, lt - kRTasks);
      }
      int ssl = 1, m3c = Ia - 1, oc = 1, k3c = 2, k6c = kRNT - 1;  // s = s0 = p0 + 1
      unsigned sph = 0u;
      for (int s = s0; s <= pEnd - 1; ++s) {
        if (s > s0) {
          if (++ssl == kRStages) {
            ssl = 0;
            sph ^= 1u;
          }
          if (++oc == 3) {
            oc = 0;
            ++m3c;
            k3c = k3c == 2 ? 0 : k3c + 1;
            k6c = k6c == kRNT - 1 ? 0 : k6c + 1;
          }
        }
        named_sync(1 + sbuf(s), kAll);  // sm(s) complete; every restriction thread left s - 1
        flush_pending();
        if (oc == 1 && lt < kRTasks + 32) {
          fence_proxy_async();
          if (lt == kRTasks) issue_tab(m3c + 4);
          issue_rows(m3c + 2, lt - kRTasks);
        }
        mbar_wait(&bar[ssl], sph);
        restrict_body(s, ssl, m3c, oc, k3c, k6c, sr + oS + sbuf(s) * kSBuf, s - s0);
        if (s + 3 <= pEnd - 1) named_arrive(4 + sbuf(s), kAll);
      }
      named_sync(8, kRest);  // the last plane's upper-half sums
      flush_pending();
    }
    return;
  }

  // step t: C completes sm(t-1) from rho(t); D restricts fine plane t-2.  Running counters (no
  // integer division in the step): rsl / rph = ring slot and barrier parity of rho(t), m3c / oc =
  // floor(s / 3) and s mod 3 of s = t - 2 (p0 is a multiple of 3)
  int rsl = 0, m3c = Ia - 2, oc = 1;
  int k3c = 1, k6c = 4;  // (m3c - Ia) mod 3 / mod kRNT: the row set / table slot of plane m3c
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
        k3c = k3c == 2 ? 0 : k3c + 1;
        k6c = k6c == kRNT - 1 ? 0 : k6c + 1;
      }
      __syncthreads();  // step t-1 done: rho(t-3)'s slot and P(t-3)'s set are free, sm(t-2) is written
      if (lt == 0) {
        fence_proxy_async();
        if (t + 2 <= pEnd) issue_r(t + 2);                              // into the slot of plane t - 3
        if (t - 1 >= s0 + kPStages && t - 1 <= pEnd - 1) issue_p(t - 1);  // into the set of plane t - 3
      }
    }
    // table slot of plane t/3 + 3 last held plane t/3 - 3 (last read at step t - 5); row set of
    // plane t/3 + 1 last held plane t/3 - 2 (last read at step t - 2)
    if (DICT && oc == 1 && lt >= kRTasks && lt < kRTasks + 32) {  // t % 3 == 0, t / 3 == m3c + 1
      fence_proxy_async();
      if (lt == kRTasks) issue_tab(m3c + 4);
      issue_rows(m3c + 2, lt - kRTasks);
    }
    if (smoother) {
      // ---- C: sm(t - 1) completes; sm(t), sm(t + 1) advance ------------------------
      // every rho plane's TMA is waited for here (also without smoothing): a slot is re-armed only
      // after its previous load completed, and no load is in flight when the CTA exits
      if (t <= pEnd) mbar_wait(&bar[rsl], rph);
      if (A.jac && t <= pEnd) smooth_body(sr + rsl * kRSlot, sr + oS + ((t - 1) & 1) * kSBuf, t - 1 >= 1 && t - 1 <= N - 2);
    } else {
      // ---- D: restriction of fine plane s = t - 2 (rho from its slot, sm(s) from its buffer) ----
      const int s = t - 2;
      if (s >= s0) {
        const int ps = s - s0, rs_ = s - p0;
        const int ssl = rsl >= 2 ? rsl - 2 : rsl + kRStages - 2;  // slot / parity of rho(s)
        const unsigned sph = rsl >= 2 ? rph : rph ^ 1u;
        if (!DICT) mbar_wait(&pbar[ps % kPStages], (unsigned)(ps / kPStages) & 1u);
        mbar_wait(&bar[ssl], sph);  // rho(s): visibility of the TMA write
        // fine plane s feeds coarse plane m3 (offset o) and, for o >= 1, m3 + 1 (offset o - 3);
        // this role's plane among them (warp-uniform)
        const int m3 = m3c, o = oc;
        restrict_body(s, ssl, m3, o, k3c, k6c, sr + oS + (s & 1) * kSBuf, ps);
      }
    }
  }
}

}  // namespace t3
