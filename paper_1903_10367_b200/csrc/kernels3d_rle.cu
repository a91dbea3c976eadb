// Run-length form of a level's 27-point table along k (level ltop-1's Galerkin rows, the operator
// stream of k3_down_c).
//
// On piecewise-constant coefficients the Galerkin rows repeat in runs along every axis (config 5,
// level 5: 14.5 M rows, 1.24 M distinct; along k a 9-vertex block period holds 3 runs).  A row
// dictionary gathered per lane measured slower than the dense planes (a warp meets ~11 distinct
// rows: one L1 tag cycle per distinct line and load, round 1).  Here the rows stay in vertex order
// but each warp segment -- 32 consecutive interior k of a line (i, j) -- stores only the rows that
// differ bitwise from their predecessor, structure-of-arrays, so the lanes of a warp read tap t from
// one short contiguous run (~11 doubles instead of 32): the same coalesced plane loads as the dense
// table on about a third of the bytes.  Lossless by construction (bitwise comparison of all 27
// taps); lane 0 of a segment always starts a row.  A segment whose 32 rows equal those of the same
// segment of the previous line (i, j - 1), or else of the previous plane (i - 1, j), stores nothing
// and points at that segment's rows (inside an eps block 5 of 9 lines and 5 of 9 planes do):
// consecutive lines are swept by neighbouring warps and a plane's stored rows are under a megabyte,
// so the repeats are served by L2.  Built once at setup; kept only when it stores less than 60 % of the dense rows
// (random coefficients: no runs, the dense planes stay).
#include "kernels3d.cuh"

namespace t3 {

// pass 1: one warp per segment of the interior lines; mask = lanes whose row differs from lane - 1's
// rdup: 1 = the segment repeats (i, j - 1)'s, 2 = (i - 1, j)'s (tested when planes is set), 0 = stored
__global__ void k3_rle_mask(const double* __restrict__ tbl, int N, int rseg, int planes,
                            uint32_t* __restrict__ rmask, uint32_t* __restrict__ rcnt, uint8_t* __restrict__ rdup) {
  const size_t nv = (size_t)N * N * N;
  const int n = N - 2;
  const size_t segs = (size_t)N * N * rseg;
  const int lane = threadIdx.x & 31;
  for (size_t sg = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < segs;
       sg += ((size_t)gridDim.x * blockDim.x) >> 5) {
    const int seg = (int)(sg % rseg);
    const size_t line = sg / rseg;
    const int j = (int)(line % N), i = (int)(line / N);
    const int k = 1 + 32 * seg + lane;
    const bool interior = i >= 1 && i <= n && j >= 1 && j <= n;
    const bool valid = interior && k <= n;
    bool diff = false;
    if (valid) {
      diff = lane == 0;
      const size_t v = ((size_t)i * N + j) * N + k;
      if (!diff)
        for (int t = 0; t < 27 && !diff; ++t)
          diff = __double_as_longlong(tbl[(size_t)t * nv + v]) != __double_as_longlong(tbl[(size_t)t * nv + v - 1]);
    }
    const unsigned m = __ballot_sync(0xffffffffu, diff);
    // the whole segment repeats the previous line's?
    bool same = interior && j >= 2;
    if (same && valid) {
      const size_t v = ((size_t)i * N + j) * N + k;
      for (int t = 0; t < 27 && same; ++t)
        same = __double_as_longlong(tbl[(size_t)t * nv + v]) == __double_as_longlong(tbl[(size_t)t * nv + v - N]);
    }
    int dup = __all_sync(0xffffffffu, same) ? 1 : 0;
    if (!dup && planes) {
      same = interior && i >= 2;
      if (same && valid) {
        const size_t v = ((size_t)i * N + j) * N + k;
        const size_t NN = (size_t)N * N;
        for (int t = 0; t < 27 && same; ++t)
          same = __double_as_longlong(tbl[(size_t)t * nv + v]) == __double_as_longlong(tbl[(size_t)t * nv + v - NN]);
      }
      if (__all_sync(0xffffffffu, same)) dup = 2;
    }
    if (lane == 0) {
      rmask[sg] = m;
      rcnt[sg] = dup ? 0u : (uint32_t)__popc(m);
      rdup[sg] = (uint8_t)dup;
    }
  }
}

// pass 2 (rbase = exclusive scan of rcnt): the lanes that start a row store its 27 taps
__global__ void k3_rle_fill(const double* __restrict__ tbl, int N, int rseg, const uint32_t* __restrict__ rmask,
                            const uint32_t* __restrict__ rbase, const uint8_t* __restrict__ rdup, size_t rn,
                            double* __restrict__ rtab) {
  const size_t nv = (size_t)N * N * N;
  const size_t segs = (size_t)N * N * rseg;
  const int lane = threadIdx.x & 31;
  for (size_t sg = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < segs;
       sg += ((size_t)gridDim.x * blockDim.x) >> 5) {
    const unsigned m = rmask[sg];
    if (rdup[sg] || !((m >> lane) & 1u)) continue;
    const int seg = (int)(sg % rseg);
    const size_t line = sg / rseg;
    const size_t v = line * N + 1 + 32 * seg + lane;
    const size_t r = rbase[sg] + __popc(m & ((1u << lane) - 1u));
    for (int t = 0; t < 27; ++t) rtab[(size_t)t * rn + r] = tbl[(size_t)t * nv + v];
  }
}

// pass 3: a repeated segment points at the rows of the nearest stored segment of the lines before it
// (one thread per (i, segment) column walks j)
__global__ void k3_rle_link(int N, int rseg, const uint8_t* __restrict__ rdup, uint32_t* __restrict__ rbase) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * rseg) return;
  const int i = t / rseg, seg = t - i * rseg;
  uint32_t last = 0u;
  for (int j = 1; j <= N - 2; ++j) {
    const size_t sg = ((size_t)i * N + j) * rseg + seg;
    if (rdup[sg]) rbase[sg] = last;
    else last = rbase[sg];
  }
}

// pass 3 with plane repeats: one block per segment column, thread = line j, planes in order.  A
// plane repeat takes the (already linked) base of (i - 1, j); a line repeat takes the base of the
// nearest line before it that is not one (block-wide max scan of the line index).
constexpr int kRleLink = 1024;
__global__ void __launch_bounds__(kRleLink) k3_rle_link2(int N, int rseg, const uint8_t* __restrict__ rdup,
                                                         uint32_t* __restrict__ rbase) {
  __shared__ uint32_t sb[kRleLink];
  __shared__ int wtop[kRleLink / 32];
  const int seg = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n = N - 2, j = tid + 1;
  const bool on = j <= n;
  for (int i = 1; i <= n; ++i) {
    const size_t sg = ((size_t)i * N + j) * rseg + seg;
    int d = 0;
    uint32_t b = 0u;
    if (on) {
      d = rdup[sg];
      b = d == 2 ? rbase[sg - (size_t)N * rseg] : rbase[sg];
    }
    sb[tid] = b;
    int v = (on && d != 1) ? tid : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = max(v, t);
    }
    if (lane == 31) wtop[wid] = v;
    __syncthreads();
    if (wid == 0) {
      int w = wtop[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w = max(w, t);
      }
      wtop[lane] = w;
    }
    __syncthreads();
    if (wid > 0) v = max(v, wtop[wid - 1]);
    if (on && d) rbase[sg] = sb[v];
    __syncthreads();
  }
}

}  // namespace t3
