// BoxMG prolongation of the finest level as a TMA-fed stream (k3_up_tma).
//
// The finest-level up sweep (solvers.py:386-395 + the FAS walk-down) reads
// every BoxMG weight of level ltop-1 once, plus g and u of the finest level,
// and writes u: a pure HBM stream (23.6 GB per config-5 cycle).  k3_up_tile
// issues those reads as per-thread __ldg and is latency-bound (long-scoreboard
// stalls ~90 %, 59 % of peak DRAM, profiles/r01_ncu_l6_v1.txt).  Here each SM
// runs one persistent CTA that streams coarse-cube steps through a two-slot
// shared-memory ring filled by TMA:
//
//   step = one layer I of a 32 (K) x 2 (J) tile of coarse cubes:
//     Pc   box {32, 2, 1, 124}  the cubes' 124 weights ("cube-owned" copy of P,
//                               k3_p_cube: term q of cube (I, J, K) is the weight
//                               P[slot][corner] that the cube's fine vertex /
//                               corner pair q needs; the weights are the same
//                               doubles as P's, only their order differs)
//     u, g box {96, 6, 3}       the 27 fine vertices of each cube
//     carry_c box {34, 3, 2}    the coarse corners
//   u is updated in place in its slot and written back with one TMA store
//   (cp.async.bulk.tensor shared -> global); boundary positions in the box, and
//   under slab sharding the fine planes outside the rank's [ilo, ihi), are never
//   modified, so storing them back is a no-op.
//
// Per fine vertex the DAG is k3_up_tile's (corner order d = 7..0, weight 1.0 at
// the centre slot), so the iterate is bitwise unchanged.
#include <cuda.h>

#include "kernels3d.cuh"

namespace t3 {

constexpr int kQK = 32, kQJ = 2, kQT = kQK * kQJ;  // cube tile (K, J), one thread per cube column
constexpr int kQS = 124;                            // stored weights per cube
constexpr int kQFK = 3 * kQK, kQFJ = 3 * kQJ;       // fine box 96 x 6 x 3
constexpr int kQCK = kQK + 2, kQCJ = kQJ + 1;       // carry box 34 x 3 x 2
constexpr int kQPd = kQS * kQT;                     // 7936 doubles
constexpr int kQUd = kQFK * kQFJ * 3;               // 1728
constexpr int kQCd = kQCK * kQCJ * 2;               // 204
constexpr int qal16(int x) { return (x + 15) / 16 * 16; }  // 128-byte multiples
constexpr int oQP = 0, oQU = oQP + qal16(kQPd), oQG = oQU + qal16(kQUd), oQC = oQG + qal16(kQUd);
constexpr int kQSlot = oQC + qal16(kQCd);
constexpr size_t kUpTmaSmem = sizeof(double) * 2 * kQSlot;
constexpr unsigned kQBytes = (unsigned)sizeof(double) * (kQPd + 2 * kQUd + kQCd);

struct UpQ {
  CUtensorMap tp;  // Pc: {Kp, nc, nc, 124}, box {32, 2, 1, 124}
  CUtensorMap tu;  // u:  {N, N, N}, box {96, 6, 3} (load and store)
  CUtensorMap tg;  // g:  same box
  CUtensorMap tc;  // carry_c: {Nc, Nc, Nc}, box {34, 3, 2}
  Up3 a;
  int tilesK, nI, I0;  // cube layers [I0, I0 + nI): those holding the fine planes [a.ilo, a.ihi)
  long long steps, per;
};

// The cube's stored weight terms in compute order: fine vertex (ri, rj, rk)
// row-major, corners d = 7..0 (k3_up_tile's order), centre weight excluded.
template <class F>
__device__ __forceinline__ void cube_terms(F&& f) {
  int q = 0;
#pragma unroll
  for (int ri = 0; ri < 3; ++ri)
#pragma unroll
    for (int rj = 0; rj < 3; ++rj)
#pragma unroll
      for (int rk = 0; rk < 3; ++rk)
#pragma unroll
        for (int d = 7; d >= 0; --d) {
          const int di = (d >> 2) & 1, dj = (d >> 1) & 1, dk = d & 1;
          if ((di && !ri) || (dj && !rj) || (dk && !rk)) continue;
          const int sl = pslot(ri - 3 * di, rj - 3 * dj, rk - 3 * dk);
          if (sl == 62) continue;
          f(q, sl, di, dj, dk);
          ++q;
        }
}

// Pc[q][I][J][K] = P[slot(q)][(I, J, K) + corner(q)] for every cube (I, J, K) < nc; the K
// rows of Pc are padded to Kp (a multiple of 32) so every TMA box row is one aligned 256-byte
// segment
__global__ void __launch_bounds__(128) k3_p_cube(const double* __restrict__ P, double* __restrict__ Pc, int Nc,
                                                 int Kp) {
  const int nc = Nc - 1;
  const size_t NcNc = (size_t)Nc * Nc, nvc = NcNc * Nc, cnt = (size_t)nc * nc * nc;
  const size_t plane = (size_t)nc * nc * Kp;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (size_t)gridDim.x * blockDim.x) {
    const int K = (int)(q % nc);
    const size_t r = q / nc;
    const int J = (int)(r % nc), I = (int)(r / nc);
    const size_t w = ((size_t)I * Nc + J) * Nc + K;
    const size_t wc = ((size_t)I * nc + J) * Kp + K;
    cube_terms([&](int s, int sl, int di, int dj, int dk) {
      Pc[(size_t)s * plane + wc] = P[(size_t)sl * nvc + w + di * NcNc + dj * Nc + dk];
    });
  }
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// G = false: no g stream (the finest level's g is already in u, Engine3::pp)
template <bool CARRY, bool G = true>
__global__ void __launch_bounds__(kQT, 1) k3_up_tma(const __grid_constant__ UpQ A) {
  extern __shared__ __align__(128) double sq[];
  __shared__ __align__(8) uint64_t bar[2];
  const Up3& a = A.a;
  const int Nc = a.Nc, nc = Nc - 1, N = a.N;
  const int lt = threadIdx.x, tx = lt & 31, ty = lt >> 5;
  const long long s0 = (long long)blockIdx.x * A.per;
  const long long s1 = s0 + A.per < A.steps ? s0 + A.per : A.steps;
  if (s0 >= s1) return;
  auto coords = [&](long long s, int& I, int& J0, int& K0) {
    const long long t = s / A.nI;
    I = A.I0 + (int)(s - t * A.nI);
    K0 = (int)(t % A.tilesK) * kQK;
    J0 = (int)(t / A.tilesK) * kQJ;
  };
  auto issue = [&](long long s) {  // thread 0: the loads of step s into slot (s - s0) & 1
    int I, J0, K0;
    coords(s, I, J0, K0);
    const int r = (int)(s - s0);
    double* b = sq + (r & 1) * kQSlot;
    uint64_t* br = &bar[r & 1];
    fence_proxy_async();
    mbar_expect_tx(br, kQBytes - (G ? 0u : (unsigned)sizeof(double) * kQUd));
    tma_load_4d(b + oQP, &A.tp, br, K0, J0, I, 0);
    if (G) tma_load_3d(b + oQG, &A.tg, br, 3 * K0, 3 * J0, 3 * I);
    tma_load_3d(b + oQC, &A.tc, br, K0, J0, I);
    bulk_wait_read0();  // this slot's u region was stored from at the end of step s - 2
    tma_load_3d(b + oQU, &A.tu, br, 3 * K0, 3 * J0, 3 * I);
  };
  if (lt == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (lt == 0) issue(s0);
  for (long long s = s0; s < s1; ++s) {
    const int r = (int)(s - s0);
    if (lt == 0 && s + 1 < s1) issue(s + 1);
    int I, J0, K0;
    coords(s, I, J0, K0);
    double* b = sq + (r & 1) * kQSlot;
    mbar_wait(&bar[r & 1], (unsigned)(r >> 1) & 1u);
    const int J = J0 + ty, K = K0 + tx;
    if (J < nc && K < nc) {
      const double* Ps = b + oQP;
      const double* Gs = b + oQG;
      const double* Cs = b + oQC;
      double* Us = b + oQU;
      double c[2][2][2];
#pragma unroll
      for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) c[di][dj][dk] = Cs[(di * kQCJ + ty + dj) * kQCK + tx + dk];
      int q = 0;
#pragma unroll
      for (int ri = 0; ri < 3; ++ri)
#pragma unroll
        for (int rj = 0; rj < 3; ++rj)
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
                wt = Ps[q * kQT + lt];
                ++q;
              }
              acc = acc + wt * c[di][dj][dk];
            }
            const int i = 3 * I + ri;  // fine planes outside [ilo, ihi) (Dirichlet / another shard's) stay as loaded
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
    }
    fence_proxy_async();  // the generic-proxy writes of u, before the async-proxy store reads them
    __syncthreads();
    if (lt == 0) {
      tma_store_3d(&A.tu, b + oQU, 3 * K0, 3 * J0, 3 * I);
      bulk_commit();
    }
  }
  if (lt == 0) bulk_wait0();
}

}  // namespace t3
