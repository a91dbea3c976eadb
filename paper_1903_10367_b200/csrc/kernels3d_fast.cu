// 3D cycle kernels specialised for the large levels (same per-element DAGs as
// kernels3d.cu / oracle/mg3d.py, different data movement):
//
// * k3_top2<KIND>  finest-level down sweep, 2.5D: a CTA owns a 32 (k) x 16 (j)
//                  column (two rows per thread) and marches a chunk of
//                  i-planes; halo planes of u and of the cell coefficients are
//                  staged with cp.async into a shared-memory ring, so each
//                  value is read from HBM once per sweep.
// * k3_smooth2r    adaFACx smoothing sm = A1(rho) * s, two rows per thread
//                  with a register window along i (6 shared loads / vertex).
// * k3_smooth_s    the same, one row per thread (coarser levels).
// * k3_down_c      coarse-level down sweep: operator apply + FAS RHS +
//                  Jacobi + adaFACx damping; R and R~ share one pass over
//                  the 124 BoxMG weight planes (each weight loaded once).
// * k3_up_tile     BoxMG prolongation: thread (J, K) marches coarse cells I
//                  and updates the 27 fine vertices of each cube, every P
//                  weight read once with warp-coalesced plane loads, slots
//                  compile-time (k3_up_cell, the grid-stride cell-owned
//                  version, serves the d-linear flavour and TMG_UPT=0).
// Variants measured and dropped (config 5, L6): 1-row register / shared
// windows for the top kernel (6.3 / 4.8 ms vs 4.4), 2-row register window for
// the top kernel (spills, 7.2 ms), warp-staged coalesced prolongation rows
// (6.7 ms vs 5.4).
#include <cuda.h>  // CUtensorMap (kernel parameter of the TMA-staged kernels)

#include "kernels3d.cuh"

namespace t3 {

constexpr int kSX = 32, kSY = 8;           // 2.5D tile (k, j)
constexpr int kSB = kSX * kSY;
constexpr int kRowU = kSX + 2, kColU = kSY + 2;  // u plane with halo
constexpr int kRowC = kSX + 1, kColC = kSY + 1;  // cell plane with halo (cells k-1.., j-1..)

struct Top3 {
  CUtensorMap tm;          // 3D map of u (box 34 x 18 x 1 doubles), used when use_tma
  CUtensorMap tmc;         // 3D map of the row-padded cell coefficients (box 34 x 17 x 1), use_tma == 2
  CUtensorMap tmr;         // 3D map of rhs (box 34 x 16 x 1 from k0 - 1: the column's rows), used when rhs_tma
  int rhs_tma;
  int use_tma;
  int crun;                // cell plane ci is stored as plane ci / crun of tmc's array (1: every plane stored)
  int N, ilo, ihi, chunk;  // planes [ilo, ihi) split in chunks
  const double* u;
  const double* rhs;
  Op3 op;
  double w, hw;
  double* g;
  double* u_out;  // or nullptr: write u + g there instead of g (the finest level's double buffer)
  double* rho;    // or nullptr
  double* part_sum;
  double* part_max;
};

struct SmoothS {
  CUtensorMap tm;  // 3D map of x (box 34 x 18 x 1 doubles), used when use_tma
  int use_tma;
  int N, ilo, ihi, chunk;
  const double* x;
  double* sm;
  double scale;
};


// 2.5D streaming.  A CTA owns a kSX x kSY column of (k, j) and marches the
// planes i in [ia, ib).  Halo planes of u (and of the cell coefficients) are
// staged into a kStages-deep shared-memory ring with cp.async (8-byte
// copies, zero-filled outside the grid), kStages-2 planes ahead of the plane
// being consumed; each thread keeps its 3x3 neighbourhood of planes i-1 and
// i in registers and reads only plane i+1 from shared memory.
constexpr int kStages = 6;

__device__ __forceinline__ void cp_async8(void* smem, const double* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int Np>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(Np) : "memory"); }

// TMA (cp.async.bulk.tensor) + mbarrier helpers: one elected thread arms the
// slot's barrier with the byte count and issues the bulk tensor copy; the
// consumers wait on the barrier's phase parity.
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ready = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ready)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!ready);
}
// generic-proxy shared-memory writes (or reads) ordered before later async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1D bulk copy global -> shared (16-byte multiples), completion on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_addr(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_addr(bar))
      : "memory");
}

struct Column {
  static constexpr int kPU = (kColU * kRowU + kSB - 1) / kSB;
  static constexpr int kPC = (kColC * kRowC + kSB - 1) / kSB;
  int N, k0, j0, ia, ib, lt;
  // in-plane offsets of the halo positions this thread stages (-1: outside / none)
  long long ou[kPU], oc[kPC];
  __device__ Column(int N_, int ilo, int ihi, int chunk) : N(N_) {
    const int tilesx = (N - 2 + kSX - 1) / kSX, tilesy = (N - 2 + kSY - 1) / kSY;
    int b = blockIdx.x;
    const int tx = b % tilesx;
    b /= tilesx;
    const int ty = b % tilesy;
    const int tz = b / tilesy;
    k0 = 1 + tx * kSX;
    j0 = 1 + ty * kSY;
    ia = ilo + tz * chunk;
    ib = min(ihi, ia + chunk);
    lt = threadIdx.y * kSX + threadIdx.x;
    const int n = N - 1;
#pragma unroll
    for (int p = 0; p < kPU; ++p) {
      const int q = lt + p * kSB;
      const int jj = q / kRowU, kk = q - jj * kRowU;
      const int j = j0 - 1 + jj, k = k0 - 1 + kk;
      ou[p] = (q < kColU * kRowU) ? ((j < N && k < N) ? (long long)j * N + k : -1) : -2;
    }
#pragma unroll
    for (int p = 0; p < kPC; ++p) {
      const int q = lt + p * kSB;
      const int jj = q / kRowC, kk = q - jj * kRowC;
      const int cj = j0 - 1 + jj, ck = k0 - 1 + kk;
      oc[p] = (q < kColC * kRowC) ? ((cj < n && ck < n) ? (long long)cj * n + ck : -1) : -2;
    }
  }
  // stage vertex plane p (halo kColU x kRowU) of x into buf; zero outside
  __device__ __forceinline__ void stage_v(double* buf, const double* x, int p) const {
    const bool okp = p >= 0 && p < N;
    const double* base = x + (size_t)(okp ? p : 0) * N * N;
#pragma unroll
    for (int q = 0; q < kPU; ++q) {
      if (ou[q] == -2) continue;
      const bool ok = okp && ou[q] >= 0;
      cp_async8(buf + lt + q * kSB, ok ? base + ou[q] : x, ok);
    }
  }
  // stage cell plane c (halo kColC x kRowC) of e (n = N-1 cells per axis)
  __device__ __forceinline__ void stage_c(double* buf, const double* e, int c) const {
    const int n = N - 1;
    const bool okp = c >= 0 && c < n;
    const double* base = e + (size_t)(okp ? c : 0) * n * n;
#pragma unroll
    for (int q = 0; q < kPC; ++q) {
      if (oc[q] == -2) continue;
      const bool ok = okp && oc[q] >= 0;
      cp_async8(buf + lt + q * kSB, ok ? base + oc[q] : e, ok);
    }
  }
};

// The streaming driver: stages planes kStages-2 ahead with cp.async and runs
// body(i, xm, x0, xp, em, e0) for i in [ia, ib), where xm / x0 / xp are the
// thread's 3x3 neighbourhoods of planes i-1, i, i+1 and em / e0 the four
// cells (j-c1, k-c2) of cell planes i-1 and i.  The loop is unrolled by
// kStages (a multiple of 3) so every ring slot and register rotation is a
// compile-time constant: no register moves, no modulo arithmetic.
template <bool CELLS, class Body>
__device__ __forceinline__ void stream25(const Column& col, const double* x, const double* e,
                                         double (*us)[kColU * kRowU], double (*cs)[kColC * kRowC],
                                         Body&& body) {
  static_assert(kStages % 3 == 0, "register rotation needs kStages % 3 == 0");
  const int tj = threadIdx.y + 1, tk = threadIdx.x + 1;
  const int ia = col.ia, ib = col.ib;
  auto issue = [&](int g, int slot) {
    col.stage_v(us[slot], x, ia - 1 + g);
    if (CELLS) col.stage_c(cs[slot], e, ia - 1 + g);
    cp_commit();
  };
#pragma unroll
  for (int g = 0; g < kStages; ++g) issue(g, g);
  double X[3][9], E[3][4];
  cp_wait<kStages - 2>();
  __syncthreads();
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    X[0][t] = us[0][(tj + t / 3 - 1) * kRowU + tk + t % 3 - 1];
    X[1][t] = us[1][(tj + t / 3 - 1) * kRowU + tk + t % 3 - 1];
  }
  if (CELLS) {
#pragma unroll
    for (int c = 0; c < 4; ++c) E[0][c] = cs[0][(tj - (c & 1)) * kRowC + tk - ((c >> 1) & 1)];
  }
  for (int i0 = ia; i0 < ib; i0 += kStages) {
#pragma unroll
    for (int u = 0; u < kStages; ++u) {
      const int i = i0 + u;
      if (i < ib) {
        cp_wait<kStages - 3>();
        __syncthreads();
        constexpr int dummy = 0;
        (void)dummy;
        const int su = (u + 2) % kStages, sc = (u + 1) % kStages;
        double* xp = X[(u + 2) % 3];
#pragma unroll
        for (int t = 0; t < 9; ++t) xp[t] = us[su][(tj + t / 3 - 1) * kRowU + tk + t % 3 - 1];
        if (CELLS) {
#pragma unroll
          for (int c = 0; c < 4; ++c) E[(u + 1) % 3][c] = cs[sc][(tj - (c & 1)) * kRowC + tk - ((c >> 1) & 1)];
        }
        issue(kStages + (i - ia), u);  // the slot of plane i-1, consumed two steps ago
        body(i, X[u % 3], X[(u + 1) % 3], X[(u + 2) % 3], E[u % 3], E[(u + 1) % 3]);
      }
    }
  }
  cp_wait<0>();
}

// ---------------------------------------------------------------------------
// Two rows per thread: CTA = 32 (k) x 16 (j) column, 256 threads, thread
// (tx, ty) owns rows j0 + 2 ty and j0 + 2 ty + 1.  The 4 x 3 neighbourhood
// of the two rows is read once per plane (18 shared loads per vertex instead
// of 27) and every per-plane overhead (staging, barrier, loop) is shared by
// two vertices.
constexpr int k2Y = 16;
constexpr int k2RowU = kSX + 2, k2ColU = k2Y + 2;
constexpr int k2RowC = kSX + 2, k2ColC = k2Y + 1;  // 33 cells used; rows padded to 34 (TMA: 16-byte rows)
// vertex-plane slot: 18 x 34 doubles padded to a multiple of 128 bytes (TMA destination)
constexpr int k2SlotU = ((k2ColU * k2RowU * 8 + 127) / 128) * 128 / 8;
constexpr unsigned k2BoxBytes = k2ColU * k2RowU * 8;
constexpr int k2SlotC = ((k2ColC * k2RowC * 8 + 127) / 128) * 128 / 8;
constexpr unsigned k2BoxBytesC = k2ColC * k2RowC * 8;

struct Column2 {
  static constexpr int kPU = (k2ColU * k2RowU + kSB - 1) / kSB;
  static constexpr int kPC = (k2ColC * k2RowC + kSB - 1) / kSB;
  int N, k0, j0, ia, ib, lt;
  long long ou[kPU], oc[kPC];
  __device__ Column2(int N_, int ilo, int ihi, int chunk) : N(N_) {
    const int tilesx = (N - 2 + kSX - 1) / kSX, tilesy = (N - 2 + k2Y - 1) / k2Y;
    int b = blockIdx.x;
    const int tx = b % tilesx;
    b /= tilesx;
    const int ty = b % tilesy;
    const int tz = b / tilesy;
    k0 = 1 + tx * kSX;
    j0 = 1 + ty * k2Y;
    ia = ilo + tz * chunk;
    ib = min(ihi, ia + chunk);
    lt = threadIdx.y * kSX + threadIdx.x;
    const int n = N - 1;
#pragma unroll
    for (int p = 0; p < kPU; ++p) {
      const int q = lt + p * kSB;
      const int jj = q / k2RowU, kk = q - jj * k2RowU;
      const int j = j0 - 1 + jj, k = k0 - 1 + kk;
      ou[p] = (q < k2ColU * k2RowU) ? ((j < N && k < N) ? (long long)j * N + k : -1) : -2;
    }
#pragma unroll
    for (int p = 0; p < kPC; ++p) {
      const int q = lt + p * kSB;
      const int jj = q / k2RowC, kk = q - jj * k2RowC;
      const int cj = j0 - 1 + jj, ck = k0 - 1 + kk;
      oc[p] = (q < k2ColC * k2RowC) ? ((cj < n && ck < n) ? (long long)cj * n + ck : -1) : -2;
    }
  }
  __device__ __forceinline__ void stage_v(double* buf, const double* x, int p) const {
    const bool okp = p >= 0 && p < N;
    const double* base = x + (size_t)(okp ? p : 0) * N * N;
#pragma unroll
    for (int q = 0; q < kPU; ++q) {
      if (ou[q] == -2) continue;
      const bool ok = okp && ou[q] >= 0;
      cp_async8(buf + lt + q * kSB, ok ? base + ou[q] : x, ok);
    }
  }
  __device__ __forceinline__ void stage_c(double* buf, const double* e, int c) const {
    const int n = N - 1;
    const bool okp = c >= 0 && c < n;
    const double* base = e + (size_t)(okp ? c : 0) * n * n;
#pragma unroll
    for (int q = 0; q < kPC; ++q) {
      if (oc[q] == -2) continue;
      const bool ok = okp && oc[q] >= 0;
      cp_async8(buf + lt + q * kSB, ok ? base + oc[q] : e, ok);
    }
  }
};

// tm != nullptr: the vertex planes arrive by TMA (one bulk tensor copy per
// plane, completion on bars[slot]); the cell planes keep 8-byte cp.async (their
// rows are an odd number of doubles, which TMA strides cannot express).
// rhs slot: the column's 16 rows of one plane, from k0 - 1 (TMA boxes start at 16-byte aligned
// inner coordinates), 34 wide
constexpr int k2RowR = kSX + 2, k2SlotR = k2RowR * k2Y;
template <int S, bool CELLS, class Body>
__device__ __forceinline__ void stream25x2(const Column2& col, const double* x, const double* e,
                                           double (*us)[k2SlotU], double (*cs)[k2SlotC],
                                           const CUtensorMap* tm, uint64_t* bars, Body&& body,
                                           const CUtensorMap* tmc = nullptr, const CUtensorMap* tmr = nullptr,
                                           double (*rs)[k2SlotR] = nullptr, int crun = 1) {
  const int ia = col.ia, ib = col.ib;
  if (tm && col.lt == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int g, int slot) {
    const bool ctma = CELLS && tmc;
    if (tm) {
      if (col.lt == 0) {
        mbar_expect_tx(&bars[slot], k2BoxBytes + (ctma ? k2BoxBytesC : 0u) + (tmr ? 8u * k2SlotR : 0u));
        tma_load_3d(us[slot], tm, &bars[slot], col.k0 - 1, col.j0 - 1, ia - 1 + g);
        // (ia - 1 + g >= 0; the plane past the last one stays out of bounds after the division)
        if (ctma) tma_load_3d(cs[slot], tmc, &bars[slot], col.k0 - 1, col.j0 - 1, (ia - 1 + g) / crun);
        if (tmr) tma_load_3d(rs[slot], tmr, &bars[slot], col.k0 - 1, col.j0, ia - 1 + g);
      }
    } else {
      col.stage_v(us[slot], x, ia - 1 + g);
    }
    if (CELLS && !ctma) col.stage_c(cs[slot], e, ia - 1 + g);
    cp_commit();
  };
  auto wait_v = [&](int g) {
    if (tm) mbar_wait(&bars[g % S], (unsigned)(g / S) & 1u);
  };
#pragma unroll
  for (int g = 0; g < S - 1; ++g) issue(g, g);
  if (tm) {
    wait_v(0);
    wait_v(1);
  }
  for (int i0 = ia; i0 < ib; i0 += S) {
#pragma unroll
    for (int u = 0; u < S; ++u) {
      const int i = i0 + u;
      if (i < ib) {
        cp_wait<S - 4>();
        wait_v(i - ia + 2);
        __syncthreads();
        issue(S - 1 + (i - ia), (u + S - 1) % S);
        body(i, us[u % S], us[(u + 1) % S], us[(u + 2) % S],
             CELLS ? cs[u % S] : nullptr, CELLS ? cs[(u + 1) % S] : nullptr, tmr ? rs[(u + 1) % S] : nullptr);
      }
    }
  }
  cp_wait<0>();
}

// 4 x 3 x 3 neighbourhood (rows j-1 .. j+2) of the thread's two vertices
__device__ __forceinline__ void load_two(const double* pm, const double* p0, const double* pp, int xo,
                                         double x0[27], double x1[27]) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int o = xo + (r - 1) * k2RowU + (c - 1);
      const double a = pm[o], b = p0[o], d = pp[o];
      if (r <= 2) { x0[r * 3 + c] = a; x0[9 + r * 3 + c] = b; x0[18 + r * 3 + c] = d; }
      if (r >= 1) { x1[(r - 1) * 3 + c] = a; x1[9 + (r - 1) * 3 + c] = b; x1[18 + (r - 1) * 3 + c] = d; }
    }
}

constexpr int k2TopStages = 5;  // measured: 5 stages beat 8 (occupancy)
constexpr size_t k2TopSmem = sizeof(double) * k2TopStages * (k2SlotU + k2SlotC + k2SlotR);

// Two rows per thread with a register window along i: each plane's 4 x 3
// neighbourhood of the thread's two vertices is read from shared memory once
// (6 loads per vertex instead of 18) and kept in registers for the three
// output planes it feeds.  Unrolled by S (a multiple of 3): ring slots and
// register rotation are compile-time constants.
template <int S, bool CELLS, class Body>
__device__ __forceinline__ void stream25x2r(const Column2& col, const double* x, const double* e,
                                            double (*us)[k2SlotU],
                                            double (*cs)[k2SlotC], int xo, int co,
                                            const CUtensorMap* tm, uint64_t* bars, Body&& body) {
  static_assert(S % 3 == 0, "register rotation needs S % 3 == 0");
  const int ia = col.ia, ib = col.ib;
  if (tm && col.lt == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int g, int slot) {
    if (tm) {
      if (col.lt == 0) {
        mbar_expect_tx(&bars[slot], k2BoxBytes);
        tma_load_3d(us[slot], tm, &bars[slot], col.k0 - 1, col.j0 - 1, ia - 1 + g);
      }
    } else {
      col.stage_v(us[slot], x, ia - 1 + g);
    }
    if (CELLS) col.stage_c(cs[slot], e, ia - 1 + g);
    cp_commit();
  };
  auto wait_v = [&](int g) {
    if (tm) mbar_wait(&bars[g % S], (unsigned)(g / S) & 1u);
  };
  auto ld12 = [&](const double* p, double w[12]) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) w[r * 3 + c] = p[xo + (r - 1) * k2RowU + (c - 1)];
  };
  auto ld6 = [&](const double* p, double w[6]) {  // cells rows j-1..j+1, cols k-1..k
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) w[r * 2 + c] = p[co + (r - 1) * k2RowC - c];
  };
#pragma unroll
  for (int g = 0; g < S; ++g) issue(g, g);
  double X[3][12], E[3][6];
  cp_wait<S - 2>();
  wait_v(0);
  wait_v(1);
  __syncthreads();
  ld12(us[0], X[0]);
  ld12(us[1], X[1]);
  if (CELLS) ld6(cs[0], E[0]);
  for (int i0 = ia; i0 < ib; i0 += S) {
#pragma unroll
    for (int u = 0; u < S; ++u) {
      const int i = i0 + u;
      if (i < ib) {
        cp_wait<S - 3>();
        wait_v(i - ia + 2);
        __syncthreads();
        ld12(us[(u + 2) % S], X[(u + 2) % 3]);
        if (CELLS) ld6(cs[(u + 1) % S], E[(u + 1) % 3]);
        issue(S + (i - ia), u);  // the slot of plane i-1, read two steps ago
        body(i, X[u % 3], X[(u + 1) % 3], X[(u + 2) % 3], E[u % 3], E[(u + 1) % 3]);
      }
    }
  }
  cp_wait<0>();
}

// x27 of the lower (h = 0) or upper (h = 1) vertex from three 4x3 planes
__device__ __forceinline__ void pick27(const double* wm, const double* w0, const double* wp, int h,
                                       double x[27]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      x[r * 3 + c] = wm[(r + h) * 3 + c];
      x[9 + r * 3 + c] = w0[(r + h) * 3 + c];
      x[18 + r * 3 + c] = wp[(r + h) * 3 + c];
    }
}

constexpr int k2RStages = 6;
constexpr size_t k2RSmemV = sizeof(double) * k2RStages * k2SlotU;

__global__ void __launch_bounds__(kSB, 2) k3_smooth2r(const __grid_constant__ SmoothS a) {
  extern __shared__ __align__(128) double dyn2[];  // k2RSmemV
  __shared__ uint64_t bars[k2RStages];
  auto xs = reinterpret_cast<double(*)[k2SlotU]>(dyn2);
  const Column2 col(a.N, a.ilo, a.ihi, a.chunk);
  const int N = a.N;
  const size_t NN = (size_t)N * N;
  const int k = col.k0 + threadIdx.x, j = col.j0 + 2 * threadIdx.y;
  const bool ok0 = k <= N - 2 && j <= N - 2, ok1 = k <= N - 2 && j + 1 <= N - 2;
  const size_t col_off = (size_t)j * N + k;
  const int xo = (2 * threadIdx.y + 1) * k2RowU + threadIdx.x + 1;
  stream25x2r<k2RStages, false>(col, a.x, nullptr, xs, nullptr, xo, 0, a.use_tma ? &a.tm : nullptr, bars,
      [&](int i, const double* wm, const double* w0, const double* wp, const double*, const double*) {
        if (!ok0) return;
        const size_t v = (size_t)i * NN + col_off;
        double x[27];
        pick27(wm, w0, wp, 0, x);
        double v0 = const_from(x, C_D8, C_E6, C_C12);
        a.sm[v] = v0 * a.scale;
        if (ok1) {
          pick27(wm, w0, wp, 1, x);
          double v1 = const_from(x, C_D8, C_E6, C_C12);
          a.sm[v + N] = v1 * a.scale;
        }
      });
}

template <int KIND>
__global__ void __launch_bounds__(kSB, 3) k3_top2(const __grid_constant__ Top3 a) {
  extern __shared__ __align__(128) double dyn2[];  // k2TopSmem
  __shared__ uint64_t bars[k2TopStages];
  auto us = reinterpret_cast<double(*)[k2SlotU]>(dyn2);
  auto cs = reinterpret_cast<double(*)[k2SlotC]>(dyn2 + k2TopStages * k2SlotU);
  auto rs = reinterpret_cast<double(*)[k2SlotR]>(dyn2 + k2TopStages * (k2SlotU + k2SlotC));
  const Column2 col(a.N, a.ilo, a.ihi, a.chunk);
  const int N = a.N;
  const size_t NN = (size_t)N * N;
  const int k = col.k0 + threadIdx.x, j = col.j0 + 2 * threadIdx.y;
  const bool ok0 = k <= N - 2 && j <= N - 2, ok1 = k <= N - 2 && j + 1 <= N - 2;
  const size_t col_off = (size_t)j * N + k;
  const int xo = (2 * threadIdx.y + 1) * k2RowU + threadIdx.x + 1;
  const int co = (2 * threadIdx.y + 1) * k2RowC + threadIdx.x + 1;
  double s = 0.0, mx = 0.0;
  const CUtensorMap* tmc = (KIND == OP_ELEMENT && a.use_tma == 2) ? &a.tmc : nullptr;
  stream25x2<k2TopStages, KIND == OP_ELEMENT>(col, a.u, a.op.e, us, cs, a.use_tma ? &a.tm : nullptr, bars,
      [&](int i, const double* pm, const double* p0, const double* pp, const double* cm,
          const double* c0, const double* r0) {
        if (!ok0) return;
        const size_t v = (size_t)i * NN + col_off;
        double rhs0, rhs1;
        if (r0) {
          rhs0 = r0[2 * threadIdx.y * k2RowR + threadIdx.x + 1];
          rhs1 = r0[(2 * threadIdx.y + 1) * k2RowR + threadIdx.x + 1];
        } else {
          rhs0 = a.rhs ? __ldg(a.rhs + v) : 0.0;
          rhs1 = (ok1 && a.rhs) ? __ldg(a.rhs + v + N) : 0.0;
        }
        double x0[27], x1[27];
        load_two(pm, p0, pp, xo, x0, x1);
        double au0, dg0, au1 = 0.0, dg1 = 1.0;
        if (KIND == OP_CONST) {
          au0 = const_from(x0, a.op.m, a.op.se, a.op.sc);
          au1 = const_from(x1, a.op.m, a.op.se, a.op.sc);
          dg0 = dg1 = a.op.cdiag;
        } else {
          // cells (i-c0, j-c1 (+1), k-c2): rows j-1, j, j+1 of cell planes i-1 and i
          double cr[2][3][2];
#pragma unroll
          for (int c0b = 0; c0b < 2; ++c0b)
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int c2 = 0; c2 < 2; ++c2)
                cr[c0b][r][c2] = (c0b ? cm : c0)[co + (r - 1) * k2RowC - c2];
          double e0[8], e1[8], E, T;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int c0b = c & 1, c1 = (c >> 1) & 1, c2 = c >> 2;
            e0[c] = cr[c0b][1 - c1][c2];
            e1[c] = cr[c0b][2 - c1][c2];
          }
          element_ET(x0, e0, E, T);
          dg0 = K_D * E;
          au0 = (dg0 * x0[13]) - (K_E * T);
          element_ET(x1, e1, E, T);
          dg1 = K_D * E;
          au1 = (dg1 * x1[13]) - (K_E * T);
        }
        const double rho0 = rhs0 - au0;
        const double t0 = a.hw * rho0;
        s = s + t0 * t0;
        mx = fmax(mx, fabs(rho0));
        const double g0 = (a.w * rho0) / dg0;
        if (a.u_out) a.u_out[v] = x0[13] + g0;
        else a.g[v] = g0;
        if (a.rho) a.rho[v] = rho0;
        if (ok1) {
          const double rho1 = rhs1 - au1;
          const double t1 = a.hw * rho1;
          s = s + t1 * t1;
          mx = fmax(mx, fabs(rho1));
          const double g1 = (a.w * rho1) / dg1;
          if (a.u_out) a.u_out[v + N] = x1[13] + g1;
          else a.g[v + N] = g1;
          if (a.rho) a.rho[v + N] = rho1;
        }
      },
      tmc, a.rhs_tma ? &a.tmr : nullptr, rs, a.crun);
  __shared__ double red_s[kSB / 32], red_m[kSB / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  }
  if ((col.lt & 31) == 0) { red_s[col.lt >> 5] = s; red_m[col.lt >> 5] = mx; }
  __syncthreads();
  if (col.lt == 0) {
    double A = 0.0, B = 0.0;
    for (int q = 0; q < kSB / 32; ++q) { A += red_s[q]; B = fmax(B, red_m[q]); }
    a.part_sum[blockIdx.x] = A;
    a.part_max[blockIdx.x] = B;
  }
}

__global__ void __launch_bounds__(kSB, 3) k3_smooth_s(const __grid_constant__ SmoothS a) {
  __shared__ double xs[kStages][kColU * kRowU];
  const Column col(a.N, a.ilo, a.ihi, a.chunk);
  const int N = a.N;
  const size_t NN = (size_t)N * N;
  const int k = col.k0 + threadIdx.x, j = col.j0 + threadIdx.y;
  const bool own = k <= N - 2 && j <= N - 2;
  const size_t col_off = (size_t)j * N + k;
  stream25<false>(col, a.x, nullptr, xs, nullptr,
      [&](int i, const double* xm, const double* x0, const double* xp, const double*, const double*) {
        if (!own) return;
        double x[27];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          x[t] = xm[t];
          x[9 + t] = x0[t];
          x[18 + t] = xp[t];
        }
        double v = const_from(x, C_D8, C_E6, C_C12);
        v = v * a.scale;
        a.sm[(size_t)i * NN + col_off] = v;
      });
}

// Coarse-level down sweep with the restriction of rho and (adaFACx) sm of the
// finer level in one pass over the P planes.  Thread per interior vertex,
// k fastest (P planes and coarse vectors coalesced).
// RLE: the operator rows come from the run-length table (kernels3d_rle.cu); a warp then owns one
// segment of 32 consecutive k of a line instead of 32 consecutive interior vertices.  (Staging the
// 3 x 6 x 34 neighbourhood of u of four lines in shared memory -- 4.8 global loads per vertex
// instead of 27 -- measured 0.54 ms against 0.33 ms: two CTA barriers per 128 vertices.)
template <bool BOXMG, bool JAC, bool PRE = false, bool RLE = false>
__global__ void __launch_bounds__(128) k3_down_c(const __grid_constant__ Down3 a) {
  const int N = a.N, n = N - 2;
  const int rseg = RLE ? a.op.rseg : 1;
  const size_t cnt = RLE ? (size_t)(a.ihi - a.ilo) * n * rseg * 32 : (size_t)(a.ihi - a.ilo) * n * n;
  double s = 0.0, m = 0.0;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt;
       q += (size_t)gridDim.x * blockDim.x) {
    int i, j, k;
    if (RLE) {
      const size_t w = q >> 5;
      const int seg = (int)(w % rseg);
      const size_t r = w / rseg;
      k = 1 + 32 * seg + (int)(q & 31);
      j = 1 + (int)(r % n);
      i = a.ilo + (int)(r / n);
      if (k > n) continue;
    } else {
      k = 1 + (int)(q % n);
      const size_t r = q / n;
      j = 1 + (int)(r % n);
      i = a.ilo + (int)(r / n);
    }
    const size_t v = vid(N, i, j, k);
    double au, dg;
    if (RLE) {
      const size_t sg = ((size_t)i * N + j) * rseg + ((k - 1) >> 5);
      const unsigned lane = (unsigned)(k - 1) & 31u;
      const size_t row = __ldg(a.op.rbase + sg) + __popc(__ldg(a.op.rmask + sg) & (0xffffffffu >> (31u - lane))) - 1;
      double x[27], w[27];
      load27<LdNC>(a.u, N, v, x);
      const double* rt = a.op.rtab + row;
      const size_t rn = a.op.rn;
#pragma unroll
      for (int t = 0; t < 27; ++t) w[t] = __ldg(rt + (size_t)t * rn);
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < 27; ++t) acc = acc + w[t] * x[t];
      au = acc;
      dg = w[13];
    } else {
      op_apply<LdNC>(a.op, a.u, N, i, j, k, au, dg);
    }
    const bool cpt0 = a.variant == VAR_AFACC;
    double bR, bT = 0.0;
    if (PRE) {  // restrictions already formed by the fused fine pass
      bR = __ldg(a.bR + v);
      if (JAC) bT = __ldg(a.bT + v);
    } else if (BOXMG) {
      const int Nf = a.Nf;
      const size_t nvc = (size_t)N * N * N;
      const size_t fc = vid(Nf, 3 * i, 3 * j, 3 * k);
      const long long sN = Nf, sNN = (long long)Nf * Nf;
      double accR = 0.0, accT = 0.0;
#pragma unroll 5
      for (int o = 0; o < 125; ++o) {
        const int oa = o / 25 - 2, ob = (o / 5) % 5 - 2, oc = o % 5 - 2;
        const long long fo = (long long)fc + oa * sNN + ob * sN + oc;
        const double w = (o == 62) ? 1.0 : __ldg(a.P + (size_t)o * nvc + v);
        double x = __ldg(a.rho_f + fo);
        if (o == 62 && cpt0) x = 0.0;
        accR = accR + w * x;
        if (JAC) accT = accT + w * __ldg(a.sm_f + fo);
      }
      bR = accR;
      bT = accT;
    } else {
      bR = restrict_dlinear<LdNC>(a.rho_f, a.Nf, i, j, k, cpt0);
      if (JAC) bT = restrict_dlinear<LdNC>(a.sm_f, a.Nf, i, j, k, false);
    }
    const double rhs = a.rhs ? __ldg(a.rhs + v) : 0.0;
    double b = bR + rhs;
    b = b + au;
    const double rho = b - au;
    if (a.write) {
      double d;
      if (a.variant == VAR_BPX) d = a.omega * rho;
      else d = (a.w * rho) / dg;
      if (JAC) d = d - a.ds * ((a.wt * bT) / dg);
      a.g[v] = d;
    }
    if (a.rho) a.rho[v] = rho;
  }
  (void)s;
  (void)m;
}

// Prolongation owned by coarse cells (solvers.py:386-395 + FAS walk-down):
// thread (W, ri, rj) updates the three fine vertices 3W + (ri, rj, 0..2);
// warps run along K, so every P plane / coarse carry load is coalesced and
// every P weight is read exactly once.
template <bool BOXMG>
__global__ void __launch_bounds__(128) k3_up_cell(const __grid_constant__ Up3 a) {
  const int Nc = a.Nc, nc = Nc - 1, N = a.N;
  // coarse cell planes whose fine vertices 3I + ri intersect [ilo, ihi)
  const int Ilo = a.ilo / 3, Ihi = min(nc, (a.ihi + 2) / 3);
  const size_t ncube = (size_t)(Ihi - Ilo) * nc * nc;
  const size_t cnt = 9 * ncube;
  const size_t nvc = (size_t)Nc * Nc * Nc;
  const double* cc = a.carry_c;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt;
       q += (size_t)gridDim.x * blockDim.x) {
    const int rr = (int)(q / ncube);
    const size_t w = q - (size_t)rr * ncube;
    const int K = (int)(w % nc);
    const size_t w2 = w / nc;
    const int J = (int)(w2 % nc), I = Ilo + (int)(w2 / nc);
    const int ri = rr / 3, rj = rr - 3 * ri;
    const int i = 3 * I + ri, j = 3 * J + rj;
    if (i < a.ilo || i >= a.ihi || j < 1) continue;
#pragma unroll
    for (int rk = 0; rk < 3; ++rk) {
      const int k = 3 * K + rk;
      if (k < 1) continue;
      double pc;
      if (BOXMG) {
        double acc = 0.0;
#pragma unroll
        for (int d = 7; d >= 0; --d) {
          const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
          if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
          const size_t wv = vid(Nc, I + di, J + dj, K + dk);
          const int sl = pslot(ri - 3 * di, rj - 3 * dj, rk - 3 * dk);
          const double wt = (sl == 62) ? 1.0 : __ldg(a.P + (size_t)sl * nvc + wv);
          acc = acc + wt * __ldg(cc + wv);
        }
        pc = acc;
      } else {
        auto cv = [&](int x, int y, int z) -> double { return __ldg(cc + vid(Nc, x, y, z)); };
        pc = prolong_dlinear(cv, Nc, i, j, k);
      }
      const size_t v = vid(N, i, j, k);
      const double c = a.g ? pc + __ldg(a.g + v) : pc;
      if (a.carry) a.carry[v] = c;
      const double un = a.u[v] + c;
      a.u[v] = un;
      int ii = i, jj = j, kk = k;
      for (int lc = a.l - 1; lc >= a.l0; --lc) {
        if (ii % 3 || jj % 3 || kk % 3) break;
        ii /= 3;
        jj /= 3;
        kk /= 3;
        a.ul[lc][vid(a.Nl[lc], ii, jj, kk)] = un;
      }
    }
  }
}

// BoxMG prolongation, tiled: thread (J, K) owns the coarse cell column (., J, K)
// and marches the cells I of a chunk; per step it updates the 27 fine vertices
// 3(I, J, K) + (ri, rj, rk), each of the cube's 124 P weights read once (warp
// along K: coalesced plane loads), the eight coarse carry corners held in
// registers (plane I+1 becomes plane I of the next step).  The (ri, rj, rk)
// loops are unrolled, so slots and skips are compile-time: no divisions and no
// per-vertex branching.  Same DAG as k3_up_cell (corner order d = 7..0).
constexpr int kUX = 32, kUY = 4;

// (6 CTAs / SM: 80 registers; measured on config 5 L6 against 1, 4, 8, 12 and a
// three-threads-per-cube split: 5.0 ms vs 9.3 / 7.0 / 5.3 / 6.2 / 5.3+)
__global__ void __launch_bounds__(kUX * kUY, 6) k3_up_tile(const __grid_constant__ Up3 a, int chunk) {
  const int Nc = a.Nc, nc = Nc - 1, N = a.N;
  const int tilesK = (nc + kUX - 1) / kUX;
  const int K = (blockIdx.x % tilesK) * kUX + threadIdx.x;
  const int J = (blockIdx.x / tilesK) * kUY + threadIdx.y;
  if (K >= nc || J >= nc) return;
  const int Ilo = a.ilo / 3, Ihi = min(nc, (a.ihi + 2) / 3);
  const int Ia = Ilo + blockIdx.y * chunk, Ib = min(Ihi, Ia + chunk);
  if (Ia >= Ib) return;
  const size_t NcNc = (size_t)Nc * Nc, nvc = NcNc * Nc, NN = (size_t)N * N;
  const double* __restrict__ P = a.P;
  const double* __restrict__ cc = a.carry_c;
  const double* __restrict__ g = a.g;
  double* __restrict__ u = a.u;
  double* __restrict__ carry = a.carry;
  double c0[2][2], c1[2][2];
  {
    const size_t w = ((size_t)Ia * Nc + J) * Nc + K;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int dk = 0; dk < 2; ++dk) c0[dj][dk] = __ldg(cc + w + dj * Nc + dk);
  }
  for (int I = Ia; I < Ib; ++I) {
    const size_t wb = ((size_t)I * Nc + J) * Nc + K;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int dk = 0; dk < 2; ++dk) c1[dj][dk] = __ldg(cc + wb + NcNc + dj * Nc + dk);
    const size_t vb = ((size_t)(3 * I) * N + 3 * J) * N + 3 * K;
#pragma unroll
    for (int ri = 0; ri < 3; ++ri) {
      const int i = 3 * I + ri;
      if (i < a.ilo || i >= a.ihi) continue;
#pragma unroll
      for (int rj = 0; rj < 3; ++rj) {
        if (rj == 0 && J == 0) continue;
#pragma unroll
        for (int rk = 0; rk < 3; ++rk) {
          if (rk == 0 && K == 0) continue;
          double acc = 0.0;
#pragma unroll
          for (int d = 7; d >= 0; --d) {
            const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
            if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
            const int sl = pslot(ri - 3 * di, rj - 3 * dj, rk - 3 * dk);
            const double wt = (sl == 62) ? 1.0 : __ldg(P + (size_t)sl * nvc + wb + di * NcNc + dj * Nc + dk);
            acc = acc + wt * (di ? c1[dj][dk] : c0[dj][dk]);
          }
          const size_t v = vb + ri * NN + rj * N + rk;
          const double c = g ? acc + __ldg(g + v) : acc;
          if (carry) carry[v] = c;
          const double un = u[v] + c;
          u[v] = un;
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
    }
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int dk = 0; dk < 2; ++dk) c0[dj][dk] = c1[dj][dk];
  }
}

// Fold the stats partials of the finest-level launch into red[0] (sum, fixed
// order) and red[1] (max); sharded runs then all-reduce red across ranks.
__global__ void __launch_bounds__(512) k3_reduce_parts(const double* ps, const double* pm, int n, double* red) {
  __shared__ double rs[16], rm[16];
  double x = 0.0, y = 0.0;
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    x += ps[q];
    y = fmax(y, pm[q]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_down_sync(0xffffffffu, x, o);
    y = fmax(y, __shfl_down_sync(0xffffffffu, y, o));
  }
  if ((threadIdx.x & 31) == 0) { rs[threadIdx.x >> 5] = x; rm[threadIdx.x >> 5] = y; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, u = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { t += rs[q]; u = fmax(u, rm[q]); }
    red[0] = t;
    red[1] = u;
  }
}

}  // namespace t3
