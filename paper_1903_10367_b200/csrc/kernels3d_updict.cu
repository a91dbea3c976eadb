// BoxMG prolongation of the finest level over the row dictionary of the
// cube-owned weights (k3_up_dict; kernels3d_dict.cu builds the dictionary).
//
// k3_up_tma streams 124 weights per coarse cube from HBM (14.5 GB of its 23.6 GB
// per config-5 cycle).  Where the coefficient is blockwise constant, those rows
// repeat (config 5: 14.35 M cube rows, 526 832 distinct, each reused by ~27
// cubes of an eps block), so here only u, g and the coarse carry stream from HBM
// and each step's few distinct rows come from the dictionary through L2:
//
//   step = one layer I of a 32 (K) x 2 (J) tile of coarse cubes (as k3_up_tma)
//   table(step)  256 B, setup-built (k3_up_tables): the step's distinct rows
//                (<= kQRows) and each cube's index into them
//   rows(step)   one 992-byte bulk copy per distinct row, from L2
//   u, g, carry  TMA boxes (evict-first in L2, so the dictionary stays)
//
// Measured and dropped: an L2 prefetch of a step's dictionary rows 4-5 steps ahead of their staging
// copies (1.745 -> 1.88 ms: the kernel runs at the DRAM rate of its access pattern, 4.8 TB/s, and
// the prefetches add traffic for row sets the stager would have kept).
//
// Step order (SNAKE, when the layer count is a multiple of 9): a column of J tiles is walked in
// blocks of 9 layers, J tile after J tile inside a block, the layers up on even J tiles and down on
// odd ones, so that the tiles inside one coefficient block meet the same low-face / interior /
// high-face row sets back to back and the re-staged sets come from L2 instead of DRAM: 1.76 ->
// 1.655 ms at config 5.  (A compile-time flavour: with the order as a run-time branch ptxas moves
// the step coordinates out of the uniform registers and both orders lose 0.05 ms.  A cache of the
// last four row sets in their slots on top of it -- least recently used replaced, 44 % fewer
// set loads by count -- cost more in the stager than the L2 hits it saves: 1.78 ms.)
//
// The streamed boxes are L2-prefetched kDPF = 4 steps ahead of their TMA loads: 0 / 2 / 4 / 8 steps
// measured 1.85 / 1.655 / 1.64 / 1.69 ms.
//
// Warp-specialised: warp 6 is the producer -- it keeps the three rings (slots,
// tables, rows) ahead of the consumers, and after the consumers of a step have
// arrived on its `done` barrier stores the step's u with one TMA store and
// refills the slot.  Warps 0-5 are consumers: cube fine planes ri = 0, 1, 2 on
// two warps each (32 cubes along K per warp), weights from the staged rows in
// shared memory.  Per fine vertex the DAG is k3_up_tile's (corners d = 7..0,
// weight 1.0 at the centre slot), so the iterate is bitwise unchanged.
#include <type_traits>

#include "kernels3d.cuh"

namespace t3 {

constexpr int kQRows = 32, kQRowS = 130;  // rows per step (cap), row stride in doubles (1040 B)
constexpr int kQTabBytes = 256;           // {n, ids[kQRows]} uint32, local[64] uint8 at byte 132
constexpr int kDNT = 8, kDTD = 6, kDNR = 4, kDRD = 3, kDPF = 4;
constexpr int kDSnake = 9;  // layers per snake block (config 5's coefficient blocks are 9 cubes wide)
static_assert(kDNR == kDRD + 1, "row sets: one per step in flight plus the one being staged");
// consumers: 18 warps = the nine fine rows (ri, rj) of a cube on two warps each (64 cubes), three
// fine vertices per thread -- with 6 warps (a cube's fine plane per thread) the consumers were busy
// two thirds of the time and set the step rate
constexpr int kDCons = 18 * 32, kDThreads = kDCons + 64;  // consumers + two producer warps
// index of the first stored term of fine row (ri, rj) in a cube's row (cube_terms order)
__host__ __device__ constexpr int cube_row_q0(int ri, int rj) {
  int q = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      if (a == ri && b == rj) return q;
      for (int c = 0; c < 3; ++c)
        for (int d = 7; d >= 0; --d) {
          const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
          if ((di && !a) || (dj && !b) || (dk && !c)) continue;
          if (pslot(a - 3 * di, b - 3 * dj, c - 3 * dk) == 62) continue;
          ++q;
        }
    }
  return q;
}
constexpr int kDRowSlot = kQRows * kQRowS;
// shared-memory layout: NS slots {u, (g,) carry}, the table ring, the row-set ring.  Without the g
// stream (the finest level's g lives in its double-buffered u) a slot is half the size (five slots
// in flight instead of three measured no faster: the consumers, not the loads, set the pace).
template <bool G>
struct DLay {
  static constexpr int oU = 0, oG = qal16(kQUd), oC = G ? 2 * qal16(kQUd) : qal16(kQUd);
  static constexpr int slot = oC + qal16(kQCd);
  static constexpr int NS = 3;
  static constexpr int oTab = NS * slot, oRows = oTab + kDNT * kQTabBytes / 8;
  static constexpr size_t smem = sizeof(double) * (oRows + kDNR * kDRowSlot);
  static constexpr unsigned bytes = (unsigned)sizeof(double) * ((G ? 2 : 1) * kQUd + kQCd);
  static_assert(smem + 1024 <= 227 * 1024, "k3_up_dict exceeds shared memory");
};
constexpr int kDNSMax = 5;
constexpr unsigned kDRowBytes = (unsigned)sizeof(double) * kQS;  // 992 of a row's 1 KB

struct UpD {
  CUtensorMap tu, tg, tc;  // as k3_up_tma
  Up3 a;
  const double* dict;      // Pc rows dict[id * kDictW + q]
  const uint8_t* tab;      // step tables, index (I * tilesJ + J0 / 2) * tilesK + K0 / 32
  int tilesK, tilesJ, nI, I0, steps, per;
  int snake;  // step order: 0 = a tile's layers upwards, tile after tile; else see coords()
};

// step tables: one thread per (layer I, J tile, K tile); *over = 1 when a step meets more than
// kQRows distinct rows (the dense stream is kept then)
__global__ void k3_up_tables(const uint32_t* __restrict__ ids, int nc, int Kp, int tilesK, int tilesJ,
                             uint8_t* __restrict__ tab, int* over) {
  const size_t cnt = (size_t)nc * tilesJ * tilesK;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (size_t)gridDim.x * blockDim.x) {
    const int tk = (int)(t % tilesK), tj = (int)((t / tilesK) % tilesJ), I = (int)(t / ((size_t)tilesK * tilesJ));
    uint32_t rows[kQRows];
    uint8_t loc[kQT];
    int n = 0;
    for (int c = 0; c < kQT; ++c) {
      const int J = tj * kQJ + c / kQK, K = tk * kQK + c % kQK;
      loc[c] = 0;
      if (J >= nc || K >= nc) continue;
      const uint32_t id = ids[((size_t)I * nc + J) * Kp + K];
      int m = 0;
      while (m < n && rows[m] != id) ++m;
      if (m == n) {
        if (n == kQRows) {
          atomicOr(over, 1);
          m = 0;
        } else {
          rows[n++] = id;
        }
      }
      loc[c] = (uint8_t)m;
    }
    uint32_t* T = reinterpret_cast<uint32_t*>(tab + t * kQTabBytes);
    T[0] = (uint32_t)n;
    for (int m = 0; m < kQRows; ++m) T[1 + m] = m < n ? rows[m] : 0u;
    for (int c = 0; c < kQT; ++c) tab[t * kQTabBytes + 132 + c] = loc[c];
  }
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// streamed boxes marked evict-first in L2 (the dictionary they would push out is reused)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_ef(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d_ef(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::
                   "l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(src)), "l"(pol)
               : "memory");
}

// G = false: no g stream (the finest level's g is already in u, Engine3::pp)
template <bool CARRY, bool G = true, bool SNAKE = false>
__global__ void __launch_bounds__(kDThreads, 1) k3_up_dict(const __grid_constant__ UpD A) {
  using LY = DLay<G>;
  constexpr int kDNS = LY::NS, kDSlot = LY::slot, oDU = LY::oU, oDG = LY::oG, oDC = LY::oC, oDTab = LY::oTab,
                oDRows = LY::oRows;
  constexpr unsigned kDBytes = LY::bytes;
  extern __shared__ __align__(128) double sq[];
  __shared__ __align__(8) uint64_t full[kDNSMax], done[kDNSMax], tful[kDNT], rful[kDNR];
  __shared__ int rsl[kDNR];  // row slot of the step whose barrier is rful[same index]
  const Up3& a = A.a;
  const int Nc = a.Nc, nc = Nc - 1, N = a.N;
  const int lt = threadIdx.x;
  const int s0 = blockIdx.x * A.per, s1 = min(A.steps, s0 + A.per);
  if (s0 >= s1) return;
  // Step order.  Plain: a tile's layers upwards, tile after tile (K tiles fastest).  Snake (nI a
  // multiple of kDSnake): a column of J tiles is walked in blocks of kDSnake layers -- inside a
  // block J tile after J tile, the layers up on even J tiles and down on odd ones -- so that the
  // tiles inside one coefficient block meet the same three row sets (low face, interior, high
  // face) back to back and the stager's set cache serves them.
  auto coords = [&](int s, int& I, int& J0, int& K0) {  // 32-bit: steps < 2^31
    if (SNAKE) {
      const int colsteps = A.tilesJ * A.nI;
      const int col = s / colsteps, q = s - col * colsteps;
      const int blk = A.tilesJ * kDSnake;
      const int ib = q / blk, r = q - ib * blk;
      const int jt = r / kDSnake, li = r - jt * kDSnake;
      I = A.I0 + ib * kDSnake + ((jt & 1) ? kDSnake - 1 - li : li);
      J0 = jt * kQJ;
      K0 = col * kQK;
      return;
    }
    const int t = s / A.nI;
    I = A.I0 + (s - t * A.nI);
    const int tj = t / A.tilesK;
    K0 = (t - tj * A.tilesK) * kQK;
    J0 = tj * kQJ;
  };
  auto tab_of = [&](int r) { return reinterpret_cast<const uint8_t*>(sq + oDTab + (r % kDNT) * (kQTabBytes / 8)); };
  if (lt == 0) {
    for (int q = 0; q < kDNS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&done[q], kDCons / 32);
    }
    for (int q = 0; q < kDNT; ++q) mbar_init(&tful[q], 1);
    for (int q = 0; q < kDNR; ++q) mbar_init(&rful[q], 1);
    mbar_fence_init();
  }
  __syncthreads();

  if (lt >= kDCons) {  // ---------------- producer warp ----------------
    // warp 6 streams (lane 0: the TMA boxes, the u stores -- bulk groups are per thread); warp 7
    // stages (lane 0: the tables; lanes 0..n-1: a step's row copies in parallel)
    const int lane = (lt - kDCons) & 31;
    const bool streamer = lt < kDCons + 32;
    const bool l0 = lane == 0;
    const uint64_t pol = policy_evict_first();
    auto load = [&](int s) {  // u, g, carry_c of step s into slot (s - s0) % kDNS
      int I, J0, K0;
      coords(s, I, J0, K0);
      const int r = s - s0;
      double* b = sq + (r % kDNS) * kDSlot;
      uint64_t* br = &full[r % kDNS];
      mbar_expect_tx(br, kDBytes);
      if (G) tma_load_3d_ef(b + oDG, &A.tg, br, 3 * K0, 3 * J0, 3 * I, pol);
      tma_load_3d(b + oDC, &A.tc, br, K0, J0, I);
      tma_load_3d_ef(b + oDU, &A.tu, br, 3 * K0, 3 * J0, 3 * I, pol);
    };
    // L2 prefetch of step s's streamed boxes and table, kDPF steps before their loads
    auto prefetch = [&](int s) {
      int I, J0, K0;
      coords(s, I, J0, K0);
      if (G) tma_prefetch_3d(&A.tg, 3 * K0, 3 * J0, 3 * I);
      tma_prefetch_3d(&A.tu, 3 * K0, 3 * J0, 3 * I);
      tma_prefetch_3d(&A.tc, K0, J0, I);
      bulk_prefetch(A.tab + (((size_t)I * A.tilesJ + J0 / kQJ) * A.tilesK + K0 / kQK) * kQTabBytes, kQTabBytes);
    };
    auto table = [&](int s) {
      int I, J0, K0;
      coords(s, I, J0, K0);
      const int r = s - s0;
      mbar_expect_tx(&tful[r % kDNT], kQTabBytes);
      bulk_load(sq + oDTab + (r % kDNT) * (kQTabBytes / 8),
                A.tab + (((size_t)I * A.tilesJ + J0 / kQJ) * A.tilesK + K0 / kQK) * kQTabBytes, kQTabBytes,
                &tful[r % kDNT]);
    };
    // the row set of step s: a tile's consecutive layers inside an eps block meet the same rows
    // (same ids in the same order), so the set staged last is kept while the ids repeat -- the
    // step's barrier then gets a plain arrival and rsl[] names the slot that holds its rows.  A
    // new set goes to slot (set counter) % kDNR: the steps in flight (k + 1 .. k + kDRD, at most
    // one set each) and the new one use at most kDNR = kDRD + 1 sets.
    int held_n = -1, held_set = -1;
    uint32_t held_id = 0u;
    auto rows = [&](int s) {  // the table of step s is in (waited here)
      const int r = s - s0;
      mbar_wait(&tful[r % kDNT], (unsigned)(r / kDNT) & 1u);
      const uint32_t* T = reinterpret_cast<const uint32_t*>(tab_of(r));
      const int n = (int)T[0];
      const uint32_t id = lane < n ? T[1 + lane] : 0u;
      uint64_t* rb = &rful[r % kDNR];
      const bool same = __all_sync(0xffffffffu, n == held_n && (lane >= n || id == held_id));
      if (!same) {
        ++held_set;
        held_n = n;
        held_id = id;
      }
      const int slot = held_set % kDNR;
      if (l0) {
        rsl[r % kDNR] = slot;
        if (same) mbar_arrive(rb);
        else mbar_expect_tx(rb, kDRowBytes * (unsigned)n);
      }
      __syncwarp();
      if (!same && lane < n)
        bulk_load(sq + oDRows + slot * kDRowSlot + lane * kQRowS, A.dict + (size_t)id * kDictW, kDRowBytes, rb);
    };
    if (streamer) {
      if (!l0) return;
      for (int s = s0; s < min(s1, s0 + kDNS); ++s) load(s);
      for (int s = s0 + kDNS; s < min(s1, s0 + kDNS + kDPF); ++s) prefetch(s);
      for (int k = s0; k < s1; ++k) {  // step k computed -> store its u, refill its slot
        const int r = k - s0;
        mbar_wait(&done[r % kDNS], (unsigned)(r / kDNS) & 1u);
        int I, J0, K0;
        coords(k, I, J0, K0);
        fence_proxy_async();
        tma_store_3d_ef(&A.tu, sq + (r % kDNS) * kDSlot + oDU, 3 * K0, 3 * J0, 3 * I, pol);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (k + kDNS < s1) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // step k's u left the slot
          load(k + kDNS);
        }
        if (k + kDNS + kDPF < s1) prefetch(k + kDNS + kDPF);
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      return;
    }
    if (l0)
      for (int s = s0; s < min(s1, s0 + kDTD); ++s) table(s);
    for (int s = s0; s < min(s1, s0 + kDRD); ++s) rows(s);
    for (int k = s0; k < s1; ++k) {  // step k computed -> its table / row slots are free
      const int r = k - s0;
      mbar_wait(&done[r % kDNS], (unsigned)(r / kDNS) & 1u);
      // the table slot of step k + kDTD last held step k + kDTD - kDNT (< k: done)
      if (l0 && k + kDTD < s1) table(k + kDTD);
      // the row slot of step k + kDRD last held step k + kDRD - kDNR (<= k: done)
      if (k + kDRD < s1) rows(k + kDRD);
    }
    return;
  }

  // ---------------- consumers: warps 0-17, fine row (ri, rj) = warp / 2 ----------------
  const int rg = lt >> 6, cl = lt & 63, tx = cl & 31, ty = cl >> 5;
  // step counters, advanced without divisions: (column of K tiles, layer block, J tile, layer in
  // the block) in snake order, (J tile, K tile, layer) otherwise
  int c_col, c_ib = 0, c_jt, c_li;
  const int nIb = A.nI / kDSnake;
  if (SNAKE) {
    const int colsteps = A.tilesJ * A.nI, blk = A.tilesJ * kDSnake;
    c_col = s0 / colsteps;
    const int q = s0 - c_col * colsteps;
    c_ib = q / blk;
    const int r0 = q - c_ib * blk;
    c_jt = r0 / kDSnake;
    c_li = r0 - c_jt * kDSnake;
  } else {
    const int t = s0 / A.nI;
    c_li = s0 - t * A.nI;
    c_jt = t / A.tilesK;
    c_col = t - c_jt * A.tilesK;
  }
  for (int s = s0; s < s1; ++s) {
    const int r = s - s0;
    if (s > s0) {
      if (SNAKE) {
        if (++c_li == kDSnake) {
          c_li = 0;
          if (++c_jt == A.tilesJ) {
            c_jt = 0;
            if (++c_ib == nIb) {
              c_ib = 0;
              ++c_col;
            }
          }
        }
      } else if (++c_li == A.nI) {
        c_li = 0;
        if (++c_col == A.tilesK) {
          c_col = 0;
          ++c_jt;
        }
      }
    }
    const int I = SNAKE ? A.I0 + c_ib * kDSnake + ((c_jt & 1) ? kDSnake - 1 - c_li : c_li) : A.I0 + c_li;
    const int J0 = c_jt * kQJ, K0 = c_col * kQK;
    double* b = sq + (r % kDNS) * kDSlot;
    mbar_wait(&full[r % kDNS], (unsigned)(r / kDNS) & 1u);
    mbar_wait(&tful[r % kDNT], (unsigned)(r / kDNT) & 1u);
    mbar_wait(&rful[r % kDNR], (unsigned)(r / kDNR) & 1u);
    const int J = J0 + ty, K = K0 + tx;
    if (J < nc && K < nc) {
      const double* Wd = sq + oDRows + rsl[r % kDNR] * kDRowSlot + kQRowS * tab_of(r)[132 + cl];
      const double* Gs = b + oDG;
      const double* Cs = b + oDC;
      double* Us = b + oDU;
      auto run = [&](auto R0, auto R1) {  // fine row (ri, rj) of the cube
        constexpr int ri = decltype(R0)::value, rj = decltype(R1)::value;
        double c[2][2][2];
#pragma unroll
        for (int di = 0; di < 2; ++di)
#pragma unroll
          for (int dj = 0; dj < 2; ++dj)
#pragma unroll
            for (int dk = 0; dk < 2; ++dk) {
              c[di][dj][dk] = 0.0;
              if ((di && !ri) || (dj && !rj)) continue;
              c[di][dj][dk] = Cs[(di * kQCJ + ty + dj) * kQCK + tx + dk];
            }
        int q = cube_row_q0(ri, rj);
#pragma unroll
        for (int rk = 0; rk < 3; ++rk) {
          double acc = 0.0;
#pragma unroll
          for (int d = 7; d >= 0; --d) {
            const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
            if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
            const int sl = pslot(ri - 3 * di, rj - 3 * dj, rk - 3 * dk);
            double wt = 1.0;
            if (sl != 62) {
              wt = Wd[q];
              ++q;
            }
            acc = acc + wt * c[di][dj][dk];
          }
          const int i = 3 * I + ri;  // fine planes outside [ilo, ihi) stay as loaded
          const bool skip = i < a.ilo || i >= a.ihi || (rj == 0 && J == 0) || (rk == 0 && K == 0);
          if (!skip) {
            const int o = (ri * kQFJ + 3 * ty + rj) * kQFK + 3 * tx + rk;
            const double cv = G ? acc + Gs[o] : acc;
            const double un = Us[o] + cv;
            Us[o] = un;
            if (CARRY) a.carry[vid(N, i, 3 * J + rj, 3 * K + rk)] = cv;
            if (ri == 0 && rj == 0 && rk == 0) {  // FAS walk-down injection
              int ii = I, jj = J, kk = K;
              for (int lc = a.l - 1; lc >= a.l0; --lc) {
                a.ul[lc][vid(a.Nl[lc], ii, jj, kk)] = un;
                if (ii % 3 || jj % 3 || kk % 3) break;
                ii /= 3;
                jj /= 3;
                kk /= 3;
              }
            }
          }
        }
      };
      using std::integral_constant;
      switch (rg) {
        case 0: run(integral_constant<int, 0>{}, integral_constant<int, 0>{}); break;
        case 1: run(integral_constant<int, 0>{}, integral_constant<int, 1>{}); break;
        case 2: run(integral_constant<int, 0>{}, integral_constant<int, 2>{}); break;
        case 3: run(integral_constant<int, 1>{}, integral_constant<int, 0>{}); break;
        case 4: run(integral_constant<int, 1>{}, integral_constant<int, 1>{}); break;
        case 5: run(integral_constant<int, 1>{}, integral_constant<int, 2>{}); break;
        case 6: run(integral_constant<int, 2>{}, integral_constant<int, 0>{}); break;
        case 7: run(integral_constant<int, 2>{}, integral_constant<int, 1>{}); break;
        default: run(integral_constant<int, 2>{}, integral_constant<int, 2>{}); break;
      }
    }
    fence_proxy_async();  // this thread's generic-proxy writes of u, before the async-proxy store
    __syncwarp();
    if ((lt & 31) == 0) mbar_arrive(&done[r % kDNS]);
  }
}

}  // namespace t3
