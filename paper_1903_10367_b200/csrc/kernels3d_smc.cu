// adaFACx smoothing fused with the restriction, cell-owned (k3_smc) -- the dictionary path of
// the finest levels (k3_smr stays for dense P streams).
//
// k3_smr splits a CTA into smoothing warps (sm = A1(rho) * scale into shared memory) and
// restriction warps (coarse vertex = thread, 5 x 5 windows of rho and sm read back from shared
// memory): ncu shows it bound by shared-memory wavefronts (157 B read per fine DoF: each rho
// value is loaded 3.9 times by the smoothing and 2.8 times by the restriction, each sm value is
// stored once and loaded 2.8 times) and by the instructions that move them.  Here a thread owns
// a coarse CELL: the 3 x 3 fine vertices (3cj + a, 3ck + b) of every fine plane.
//   * It loads the 5 x 5 rho window of its 9 columns once per plane (25 loads) and keeps the
//     smoothing state of its columns in registers (2 values per column: with G(p) = -(e F(p) +
//     c D(p)) and H(p) = m x(p) - e D(p), F / D the in-plane edge / diagonal neighbour sums,
//     sm(p) = G(p-1) + H(p) + G(p+1)); sm never touches shared memory.
//   * Its 9 vertices of plane s feed the cell's 4 corner coarse vertices (dj, dk): 25 (vertex,
//     corner) pairs per coarse plane, for the two coarse planes m3 = floor(s / 3) (fine offset o
//     = s mod 3) and m3 + 1 (offset o - 3, o >= 1), both fields with one weight load: the same
//     100 multiply-adds per cell and step k3_smr spends per coarse vertex, on 25 + 50 shared
//     loads instead of ~144.
//   * When a coarse plane completes, the 4 cells around a coarse vertex add their partial sums:
//     along K by a warp shuffle, along J through a small shared-memory exchange (fixed order).
// CTA = 11 cell rows x 32 cells (11 consumer warps) for a tile of 10 x 31 coarse vertices, plus one
// producer warp (12 warps of 168 registers: one CTA per SM): a 4-slot ring of rho planes (TMA box 100 x 35), a 4-slot ring of the steps' weight
// slices and a 4-slot ring of the tile-plane tables (distinct dictionary rows of the tile's vertices in a
// coarse plane + each vertex's index), completion on mbarriers.  The weights come from a sliced
// copy of P's row dictionary (5 slices of 25 weights per row, one per fine plane offset, padded
// to 26 doubles so that a slice is a 16-byte-aligned 208-byte bulk copy): a step stages only the
// two slices it multiplies (<= 20 KB) instead of whole rows for three coarse planes.  Summation
// order differs from the oracle's o-major order (3D bar: 1e-10).
// Tile height, measured at config 5 (the cells of a tile overlap the next tile's by one row): 4
// coarse rows on two CTAs of 6 warps per SM 2.02 ms (77 % of the cell lanes own coarse vertices);
// 10 rows on one CTA of 12 warps **1.84 ms** (88 %, 11 instead of 10 consumer warps per SM); 8 rows
// on one CTA of 10 warps 2.09 ms.
// The kernel needs its 168 registers (12 warps per SM): two CTAs of 7 / 8 warps per SM (128
// registers, 320 bytes of spills in the step loop) measured 2.98 / 3.12 ms; rho / weight rings of 4 / 3, 5 / 3, 3 / 4 slots measured 1.84 / 1.86 / 1.87 ms against 1.82 ms for 4 / 4; the step unrolled by two with
// the rho windows swapping roles (no copy of the window's centre, the sign of G folded into its
// constants) 2.06 ms (20 bytes of spills).
#include <cuda.h>

#include <type_traits>

#include "kernels3d.cuh"

namespace t3 {

constexpr int kCK = 31, kCJ = 10;                  // coarse vertices per tile (K, J)
constexpr int kCPerSM = kCJ <= 4 ? 2 : 1;          // CTAs per SM (registers: 12 warps of 168)
constexpr int kCCK = kCK + 1, kCCJ = kCJ + 1;      // cells per tile: 32 x 5
constexpr int kCCons = 32 * kCCJ, kCThreads = kCCons + 32;
// rho box: the cells' 98 x 17 fine window from (3K0 - 4, 3J0 - 4), widened to 100 columns so that
// it can start at an even column (TMA: the box's inner start coordinate must be 16-byte aligned)
constexpr int kCW = 3 * kCCK + 4, kCH = 3 * kCCJ + 2;
constexpr int kCRho = (kCW * kCH * 8 + 127) / 128 * 128 / 8;   // 1712 doubles
constexpr int kCSl = 26;                           // doubles per weight slice (25 + pad)
constexpr int kCRows = kCJ <= 4 ? 32 : 48;         // distinct rows per tile plane (cap)
static_assert(kCRows <= 64, "the producer stages a row per lane in two passes");
constexpr int kCWts = 2 * kCRows * kCSl;           // one step's slices: [coarse plane c | nx][row][26]
constexpr int kCR = 4, kCWR = 4;                   // ring depths: rho planes, weight slice sets
constexpr int kCNT = 4;                            // table ring (coarse planes)
constexpr int kCTabLoc = 4 + 4 * kCRows;           // {n, ids[kCRows]} uint32, then local[kCK * kCJ] uint8
constexpr int kCTabBytes = (kCTabLoc + kCK * kCJ + 15) / 16 * 16;
constexpr int oCWts = kCR * kCRho, oCTab = oCWts + kCWR * kCWts;
constexpr int oCScr = oCTab + kCNT * kCTabBytes / 8;
constexpr int kCScr = kCCJ * 32 * 2;               // one exchange buffer: [cell row][lane][field]
constexpr size_t kSmcSmem = sizeof(double) * (oCScr + 2 * kCScr);
static_assert(kCWts % 16 == 0 && kCRho % 16 == 0, "slots stay 128-byte aligned");
static_assert(kCPerSM * (kSmcSmem + 1024) <= 227 * 1024, "CTAs per SM");

// P's row dictionary in slices: Pds[(id * 5 + si) * 26 + q] = Pd[id * kDictW + si * 25 + q]
__global__ void k3_dict_slices(const double* __restrict__ pd, size_t rows, double* __restrict__ out) {
  const size_t cnt = rows * 5 * kCSl;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)(t % kCSl);
    const size_t r = t / kCSl;
    const int si = (int)(r % 5);
    const size_t id = r / 5;
    out[t] = q < 25 ? pd[id * kDictW + si * 25 + q] : 0.0;
  }
}

// tile-plane tables of k3_smc (31 x 4 vertex tiles); *over = 1 when a tile plane meets more than
// kCRows distinct rows (the dense path is kept then)
__global__ void k3_smc_tables(const uint32_t* __restrict__ ids, int Nc, int Ncp, int tilesK, int tilesJ,
                              uint8_t* __restrict__ tab, int* over) {
  const int n = Nc - 2;
  const size_t cnt = (size_t)n * tilesJ * tilesK;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (size_t)gridDim.x * blockDim.x) {
    const int tk = (int)(t % tilesK), tj = (int)((t / tilesK) % tilesJ), m = 1 + (int)(t / ((size_t)tilesK * tilesJ));
    uint32_t rows[kCRows];
    int cntr = 0;
    uint8_t* T8 = tab + t * kCTabBytes;
    for (int c = 0; c < kCK * kCJ; ++c) {
      const int J = 1 + tj * kCJ + c / kCK, K = 1 + tk * kCK + c % kCK;
      int loc = 0;
      if (J <= n && K <= n) {
        const uint32_t id = ids[((size_t)m * Nc + J) * Ncp + K];
        while (loc < cntr && rows[loc] != id) ++loc;
        if (loc == cntr) {
          if (cntr == kCRows) {
            atomicOr(over, 1);
            loc = 0;
          } else {
            rows[cntr++] = id;
          }
        }
      }
      T8[kCTabLoc + c] = (uint8_t)loc;
    }
    uint32_t* T = reinterpret_cast<uint32_t*>(T8);
    T[0] = (uint32_t)cntr;
    for (int q = 0; q < kCRows; ++q) T[1 + q] = q < cntr ? rows[q] : 0u;
    for (int c = kCTabLoc + kCK * kCJ; c < kCTabBytes; ++c) T8[c] = 0;
  }
}

// the same tables when every vertex uses dictionary row 0 (the d-linear flavour)
__global__ void k3_smc_tables_one(uint8_t* __restrict__ tab, size_t cnt) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (size_t)gridDim.x * blockDim.x) {
    uint32_t* T = reinterpret_cast<uint32_t*>(tab + t * kCTabBytes);
    T[0] = 1u;
    for (int q = 0; q < kCRows; ++q) T[1 + q] = 0u;
    for (int c = kCTabLoc; c < kCTabBytes; ++c) tab[t * kCTabBytes + c] = 0;
  }
}

struct Smc {
  CUtensorMap tr;        // rho of the fine level, box {100, 17, 1}
  int N, Nc;             // fine / coarse vertices per axis
  int tilesK, tilesJ, chunk;
  int jac, zc;           // adaFACx (b_T too); afacc (the centre tap of rho reads 0)
  double scale;          // omega * 3 / 8
  double* bR;
  double* bT;
  const double* pds;     // sliced row dictionary of the coarse level's P
  const uint8_t* ptab;   // tile-plane tables, index ((m - 1) * tilesJ + tj) * tilesK + tk
  int ilo, ihi;          // coarse planes [ilo, ihi) this launch restricts into
};

template <bool JAC>
__global__ void __launch_bounds__(kCThreads, kCPerSM) k3_smc(const __grid_constant__ Smc A) {
  extern __shared__ __align__(128) double sc[];
  __shared__ __align__(8) uint64_t full[kCR], done[kCR], wful[kCWR], wdone[kCWR], tful[kCNT];
  const int N = A.N, Nc = A.Nc, n = Nc - 2;
  const int tk = blockIdx.x % A.tilesK, tj = blockIdx.x / A.tilesK;
  const int K0 = 1 + tk * kCK, J0 = 1 + tj * kCJ;
  const int Ia = A.ilo + blockIdx.y * A.chunk, Ib = min(A.ihi, Ia + A.chunk);  // coarse planes [Ia, Ib)
  if (Ia >= Ib) return;
  const int fj0 = 3 * J0 - 4;                      // rho window origin (fine)
  const int fsh = (3 * K0 - 4) & 1;                // ... its column 3K0 - 4 sits at box column fsh
  const int fk0 = 3 * K0 - 4 - fsh;                // even box start (floor, also for -1)
  const int p0 = 3 * Ia - 3, pEnd = 3 * Ib;        // rho planes streamed: [p0, pEnd]
  const int s0 = 3 * Ia - 2;                       // fine planes restricted: [s0, pEnd - 1]
  const int lt = threadIdx.x;
  if (lt == 0) {
    for (int q = 0; q < kCR; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&done[q], kCCJ);
    }
    for (int q = 0; q < kCWR; ++q) {
      mbar_init(&wful[q], 1);
      mbar_init(&wdone[q], kCCJ);
    }
    for (int q = 0; q < kCNT; ++q) mbar_init(&tful[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // iteration t = p0 .. pEnd: rho plane t arrives (slot (t - p0) % kCR) together with the weight
  // slices of fine plane s = t - 1 (when s >= s0); table of coarse plane m in slot (m - Ia) % kCNT
  auto tslot = [&](int m) { return (m - Ia) % kCNT; };  // planes Ia <= m < Ib only
  auto tab_of = [&](int m) { return reinterpret_cast<const uint8_t*>(sc + oCTab) + tslot(m) * kCTabBytes; };
  auto plane_ok = [&](int m) { return m >= Ia && m < Ib; };

  if (lt >= kCCons) {  // ---------------- producer warp ----------------
    const int lane = lt - kCCons;
    auto issue_tab = [&](int m) {  // lane 0
      if (!plane_ok(m)) return;
      uint64_t* tb = &tful[tslot(m)];
      mbar_expect_tx(tb, kCTabBytes);
      bulk_load(sc + oCTab + tslot(m) * (kCTabBytes / 8),
                A.ptab + (((size_t)(m - 1) * A.tilesJ + tj) * A.tilesK + tk) * kCTabBytes, kCTabBytes, tb);
    };
    // a table slot is loaded once per kCNT planes: plane m is its ((m - Ia) / kCNT)-th use
    auto twait = [&](int m) { mbar_wait(&tful[tslot(m)], (unsigned)((m - Ia) / kCNT) & 1u); };
    if (lane == 0) {
      issue_tab(Ia);
      issue_tab(Ia + 1);
    }
    for (int t = p0; t <= pEnd; ++t) {
      const int r = t - p0, sl = r % kCR, wl = r % kCWR;
      if (r >= kCR) mbar_wait(&done[sl], (unsigned)(r / kCR - 1) & 1u);      // rho of iteration t - kCR consumed
      if (r >= kCWR) mbar_wait(&wdone[wl], (unsigned)(r / kCWR - 1) & 1u);  // slices of iteration t - kCWR
      const int s = t - 1;
      const int m3 = s >= 0 ? s / 3 : -1, o = s - 3 * m3;
      const bool rs = s >= s0 && s <= pEnd - 1;
      const bool c = rs && plane_ok(m3), nx = rs && o >= 1 && plane_ok(m3 + 1);
      if (rs && o == 0 && lane == 0) {
        // planes <= m3 - 2 are finished (their last step s - 4 was consumed): their table slots are free
        fence_proxy_async();
        issue_tab(m3 + 2);
      }
      int nc_ = 0, nn_ = 0;
      uint32_t idc[2] = {0u, 0u}, idn[2] = {0u, 0u};  // a row per lane, two passes
      if (c) {
        twait(m3);
        const uint32_t* T = reinterpret_cast<const uint32_t*>(tab_of(m3));
        nc_ = (int)T[0];
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (lane + 32 * h < nc_) idc[h] = T[1 + lane + 32 * h];
      }
      if (nx) {
        twait(m3 + 1);
        const uint32_t* T = reinterpret_cast<const uint32_t*>(tab_of(m3 + 1));
        nn_ = (int)T[0];
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (lane + 32 * h < nn_) idn[h] = T[1 + lane + 32 * h];
      }
      double* wslot = sc + oCWts + wl * kCWts;
      if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(&full[sl], (unsigned)(sizeof(double) * kCW * kCH));
        tma_load_3d(sc + sl * kCRho, &A.tr, &full[sl], fk0, fj0, t);
        if (nc_ + nn_) mbar_expect_tx(&wful[wl], (unsigned)(8 * kCSl) * (unsigned)(nc_ + nn_));
        else mbar_arrive(&wful[wl]);
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = lane + 32 * h;
        if (q < nc_)
          bulk_load(wslot + q * kCSl, A.pds + ((size_t)idc[h] * 5 + (o + 2)) * kCSl, 8 * kCSl, &wful[wl]);
        if (q < nn_)
          bulk_load(wslot + (kCRows + q) * kCSl, A.pds + ((size_t)idn[h] * 5 + (o - 1)) * kCSl, 8 * kCSl, &wful[wl]);
      }
    }
    return;
  }

  // ---------------- consumers: cell (cjl, ckl) = (warp, lane) ----------------
  const int cjl = lt >> 5, ckl = lt & 31;
  const int cj = J0 - 1 + cjl, ck = K0 - 1 + ckl;
  // interior masks of the cell's fine vertices (rows 3cj + a, columns 3ck + b)
  unsigned vmask = 0u;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int j = 3 * cj + a, k = 3 * ck + b;
      if (j >= 1 && k >= 1 && j <= N - 2 && k <= N - 2) vmask |= 1u << (a * 3 + b);
    }
  // corner (dj, dk) = coarse vertex (cj + dj, ck + dk); inside the tile and the grid?
  bool cok[2][2];
  int vix[2][2];
#pragma unroll
  for (int dj = 0; dj < 2; ++dj)
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
      const int vj = cjl - 1 + dj, vk = ckl - 1 + dk;
      cok[dj][dk] = vj >= 0 && vj < kCJ && vk >= 0 && vk < kCK && J0 + vj <= n && K0 + vk <= n;
      vix[dj][dk] = cok[dj][dk] ? vj * kCK + vk : 0;
    }
  const double cm = C_D8 * A.scale, ce = C_E6 * A.scale, cc = C_C12 * A.scale;
  double SA[9], SG[9], X[9];  // smoothing state (A, G of the last plane) and rho of the last plane
#pragma unroll
  for (int q = 0; q < 9; ++q) SA[q] = SG[q] = X[q] = 0.0;
  double acc[2][2][2][2];     // [coarse plane: c, nx][dj][dk][field]
#pragma unroll
  for (int q = 0; q < 16; ++q) (&acc[0][0][0][0])[q] = 0.0;
  int roff[2][2][2];          // [plane][dj][dk]: the corner's row offset in the step's slice block
#pragma unroll
  for (int q = 0; q < 8; ++q) (&roff[0][0][0])[q] = 0;
  double* scr = sc + oCScr;

  for (int t = p0; t <= pEnd; ++t) {
    const int r = t - p0, sl = r % kCR, wl = r % kCWR;
    const double* slot = sc + sl * kCRho;
    mbar_wait(&full[sl], (unsigned)(r / kCR) & 1u);
    // ---- the 5 x 5 rho window of plane t; completes sm(t - 1) of the cell's 9 columns ----
    double W[5][5];
    const double* wp = slot + (3 * cjl) * kCW + 3 * ckl + fsh;
#pragma unroll
    for (int a = 0; a < 5; ++a)
#pragma unroll
      for (int b = 0; b < 5; ++b) W[a][b] = wp[a * kCW + b];
    double Y[9];
    if (JAC) {
      double ar[5][3];
#pragma unroll
      for (int a = 0; a < 5; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) ar[a][b] = W[a][b] + W[a][b + 2];
      const bool pl_ok = t - 1 >= 1 && t - 1 <= N - 2;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int q = a * 3 + b;
          const double D = ar[a][b] + ar[a + 2][b];
          const double F = (W[a][b + 1] + W[a + 2][b + 1]) + ar[a + 1][b];
          const double G = -(ce * F + cc * D);
          const double H = cm * W[a + 1][b + 1] - ce * D;
          Y[q] = SA[q] + G;
          SA[q] = SG[q] + H;
          SG[q] = G;
        }
      // sm exists at interior fine vertices only: cells on the domain boundary and the planes
      // outside [1, N - 2] are the rare case
      if (!pl_ok || vmask != 0x1ffu) {
#pragma unroll
        for (int q = 0; q < 9; ++q)
          if (!pl_ok || !((vmask >> q) & 1u)) Y[q] = 0.0;
      }
    }
    // ---- restriction of fine plane s = t - 1 (x = rho(s) kept from the last iteration) ----
    const int s = t - 1;
    if (s >= s0) {
      const int m3 = s / 3, o = s - 3 * m3;  // s >= 1
      const bool c = plane_ok(m3), nx = o >= 1 && plane_ok(m3 + 1);
      if (o == 0 || s == s0) {  // new coarse planes: the corners' rows in their tables
#pragma unroll
        for (int pl = 0; pl < 2; ++pl) {
          const int m = m3 + pl;
          if (!plane_ok(m)) continue;
          mbar_wait(&tful[tslot(m)], (unsigned)((m - Ia) / kCNT) & 1u);
          const uint8_t* tb = tab_of(m) + kCTabLoc;
#pragma unroll
          for (int dj = 0; dj < 2; ++dj)
#pragma unroll
            for (int dk = 0; dk < 2; ++dk) roff[pl][dj][dk] = (pl * kCRows + tb[vix[dj][dk]]) * kCSl;
        }
      }
      mbar_wait(&wful[wl], (unsigned)(r / kCWR) & 1u);
      const double* wts = sc + oCWts + wl * kCWts;
      // the step's multiply-adds, specialised by which coarse planes the fine plane feeds (uniform)
      auto feed = [&](auto CC, auto NN) {
        constexpr bool C = decltype(CC)::value, NX = decltype(NN)::value;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            if (!cok[dj][dk]) continue;
            const double* wc = wts + roff[0][dj][dk];
            const double* wn = wts + roff[1][dj][dk];
            double aR = acc[0][dj][dk][0], aS = acc[0][dj][dk][1], bR_ = acc[1][dj][dk][0], bS_ = acc[1][dj][dk][1];
#pragma unroll
            for (int a = dj; a < 3; ++a)
#pragma unroll
              for (int b = dk; b < 3; ++b) {
                const int q = (a - 3 * dj + 2) * 5 + (b - 3 * dk + 2);
                const double x = X[a * 3 + b];
                const double y = JAC ? Y[a * 3 + b] : 0.0;
                if (C) {
                  const double w = wc[q];
                  const bool ctr = a == 0 && b == 0 && dj == 0 && dk == 0;  // the coarse vertex itself (o = 0)
                  aR = aR + w * ((ctr && o == 0 && A.zc) ? 0.0 : x);
                  if (JAC) aS = aS + w * y;
                }
                if (NX) {
                  const double w = wn[q];
                  bR_ = bR_ + w * x;
                  if (JAC) bS_ = bS_ + w * y;
                }
              }
            acc[0][dj][dk][0] = aR;
            acc[0][dj][dk][1] = aS;
            acc[1][dj][dk][0] = bR_;
            acc[1][dj][dk][1] = bS_;
          }
      };
      using std::true_type;
      using std::false_type;
      if (c && nx) feed(true_type{}, true_type{});
      else if (c) feed(true_type{}, false_type{});
      else if (nx) feed(false_type{}, true_type{});
      if (o == 2) {
        // coarse plane m3 is complete: vertex (vj, vk) = (cjl - 1, ckl - 1) collects the partial sums of
        // its four cells -- along K from lane - 1 by shuffle, along J from the cell row below through
        // shared memory (one named barrier of the consumer warps per completed plane)
        double q0[2], q1[2];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const double up0 = __shfl_up_sync(0xffffffffu, acc[0][0][1][f], 1);
          const double up1 = __shfl_up_sync(0xffffffffu, acc[0][1][1][f], 1);
          q0[f] = acc[0][0][0][f] + up0;  // dj = 0: this cell's low corner + lane - 1's high corner
          q1[f] = acc[0][1][0][f] + up1;  // dj = 1
        }
        double* sb = scr + (m3 & 1) * kCScr;
        if (c) {
          sb[(cjl * 32 + ckl) * 2] = q1[0];
          sb[(cjl * 32 + ckl) * 2 + 1] = q1[1];
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kCCons) : "memory");
        if (c && cjl >= 1 && ckl >= 1 && cok[0][0]) {
          const double* lo = sb + ((cjl - 1) * 32 + ckl) * 2;
          const size_t ix = ((size_t)m3 * Nc + cj) * Nc + ck;
          A.bR[ix] = q0[0] + lo[0];
          if (JAC) A.bT[ix] = q0[1] + lo[1];
        }
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk)
#pragma unroll
            for (int f = 0; f < 2; ++f) {
              acc[0][dj][dk][f] = acc[1][dj][dk][f];
              acc[1][dj][dk][f] = 0.0;
            }
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) roff[0][dj][dk] = roff[1][dj][dk] - kCRows * kCSl;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) X[a * 3 + b] = W[a + 1][b + 1];
    __syncwarp();
    if (ckl == 0) {
      mbar_arrive(&done[sl]);
      mbar_arrive(&wdone[wl]);
    }
  }
}

}  // namespace t3
