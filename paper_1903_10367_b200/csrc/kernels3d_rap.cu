// Galerkin coarse rows A_c = P^T A_f P of the BoxMG setup (mg3d.galerkin,
// operators.py:446-478 carried to 3D) in two passes over a slab of coarse planes.
//
// The one-thread-per-coarse-vertex triple loop (125 fine offsets x 27 taps x 27
// neighbours with run-time indices) kept its row and accumulators in local
// memory: 1.78 s and 2.6 TB of DRAM traffic at config 5 for about 0.2 TFMA of
// work.  Here the product is split at the fine level:
//
//   Y_c[t]   = sum_s P_c[t - s] A_f[3c + t - s][s]        t in [-3, 3]^3   (k3_rap_y)
//   A_c[c][d] = sum_t Y_c[t] P_{c+d}[t - 3d]               d in [-1, 1]^3   (k3_rap_out)
//
// Y_c = (P_c^T A_f) is the coarse basis function of c pushed through the fine
// rows (rows of non-equation fine vertices masked, as in the reference), 343
// values per coarse vertex; both passes are one thread per output value with
// lanes along K, so every load of P, Y and the fine table is coalesced, and a CTA
// keeps to 32 coarse vertices so P and Y come from DRAM once.  3375 +
// 1331 multiply-adds per coarse vertex instead of 15 625.  Y lives in a scratch
// buffer of a few coarse planes (slab), reused down the level.  The association
// (sum_s r a) p differs from the reference's sum (r a) p; the tables agree to
// rounding (tests: 1e-12 relative to the largest entry).
#include <utility>

#include "kernels3d.cuh"

namespace t3 {

// tap s = (si, sj, sk) of the element operator's row at fine vertex (i, j, k) from the
// per-cell coefficients: K_unit couples corners a, b of a cell with 1/3 (a = b), 0 (one
// differing bit: the face taps vanish) and -1/12 (two or three differing bits)
template <int SI, int SJ, int SK>
__device__ __forceinline__ double elem_tap(const double* __restrict__ e, int n, int i, int j, int k) {
  constexpr int m = (SI != 0) + (SJ != 0) + (SK != 0);
  if (m == 1) return 0.0;
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int a0 = a & 1, a1 = (a >> 1) & 1, a2 = a >> 2;
    // corner b = a + s must be a corner of the same cell
    if ((SI == 1 && a0) || (SI == -1 && !a0) || (SJ == 1 && a1) || (SJ == -1 && !a1) || (SK == 1 && a2) ||
        (SK == -1 && !a2))
      continue;
    acc = acc + __ldg(e + ((size_t)(i - a0) * n + (j - a1)) * n + (k - a2));
  }
  return (m == 0 ? K_D : -K_E) * acc;
}

struct RapArgs {
  int Nc, Nf;        // coarse / fine vertices per axis
  int I0, planes;    // coarse planes [I0, I0 + planes) of this slab
  const double* P;   // 125 planes over the coarse vertex grid
  const double* tbl; // fine rows: 27 planes over the fine grid, or nullptr
  const double* e;   // ... or the fine per-cell coefficients (element operator)
  double* Y;         // scratch: Y[t][slab vertex], t = ((ti + 3) * 7 + tj + 3) * 7 + tk + 3
  double* out;       // the coarse table (27 planes)
};

// term s of Y_c[t]: fine row f = 3c + t - s (masked unless f is an equation vertex), its tap s
template <bool ELEM, int S>
__device__ __forceinline__ void rap_term(const RapArgs& A, int I, int J, int K, int ti, int tj, int tk, size_t vc,
                                         size_t nvc, size_t nvf, double& acc) {
  constexpr int si = S / 9 - 1, sj = (S / 3) % 3 - 1, sk = S % 3 - 1;
  if (ELEM && ((si != 0) + (sj != 0) + (sk != 0)) == 1) return;  // the element operator has no face taps
  const int Nf = A.Nf;
  const int oi = ti - si, oj = tj - sj, ok = tk - sk;
  if (oi < -2 || oi > 2 || oj < -2 || oj > 2 || ok < -2 || ok > 2) return;
  const int fi = 3 * I + oi, fj = 3 * J + oj, fk = 3 * K + ok;
  if (fi < 1 || fj < 1 || fk < 1 || fi > Nf - 2 || fj > Nf - 2 || fk > Nf - 2) return;
  const double rw = __ldg(A.P + (size_t)pslot(oi, oj, ok) * nvc + vc);
  const double ac = ELEM ? elem_tap<si, sj, sk>(A.e, Nf - 1, fi, fj, fk)
                         : __ldg(A.tbl + (size_t)S * nvf + vid(Nf, fi, fj, fk));
  acc = acc + rw * ac;
}

template <bool ELEM, int... S>
__device__ __forceinline__ void rap_terms(std::integer_sequence<int, S...>, const RapArgs& A, int I, int J, int K,
                                          int ti, int tj, int tk, size_t vc, size_t nvc, size_t nvf, double& acc) {
  (rap_term<ELEM, S>(A, I, J, K, ti, tj, tk, vc, nvc, nvf, acc), ...);
}

// Both passes: a CTA owns 32 consecutive slab vertices (lanes, along K) and its warps split the
// outputs of those vertices (the 343 t of Y, the 27 neighbours d of A_c), so the P rows / Y values
// of the 32 vertices are fetched from DRAM once and re-read through L1.
constexpr int kRapYW = 16;  // warps of k3_rap_y (t = warp, warp + 16, ...)

template <bool ELEM>
__global__ void __launch_bounds__(32 * kRapYW) k3_rap_y(const RapArgs A) {
  const int Nc = A.Nc, Nf = A.Nf;
  const size_t sv = (size_t)A.planes * Nc * Nc;
  const size_t nvc = (size_t)Nc * Nc * Nc, nvf = (size_t)Nf * Nf * Nf;
  const size_t blocks = (sv + 31) / 32;
  for (size_t blk = blockIdx.x; blk < blocks; blk += gridDim.x) {
    const size_t cs = blk * 32 + threadIdx.x;
    if (cs >= sv) continue;
    const int K = (int)(cs % Nc), J = (int)((cs / Nc) % Nc), I = A.I0 + (int)(cs / ((size_t)Nc * Nc));
    if (K < 1 || J < 1 || K > Nc - 2 || J > Nc - 2) continue;  // (I is interior by construction)
    const size_t vc = vid(Nc, I, J, K);
    for (int t = threadIdx.y; t < 343; t += kRapYW) {
      const int ti = t / 49 - 3, tj = (t / 7) % 7 - 3, tk = t % 7 - 3;
      double acc = 0.0;
      rap_terms<ELEM>(std::make_integer_sequence<int, 27>{}, A, I, J, K, ti, tj, tk, vc, nvc, nvf, acc);
      A.Y[(size_t)t * sv + cs] = acc;
    }
  }
}

__global__ void __launch_bounds__(32 * 27) k3_rap_out(const RapArgs A) {
  const int Nc = A.Nc;
  const size_t sv = (size_t)A.planes * Nc * Nc;
  const size_t nvc = (size_t)Nc * Nc * Nc;
  const size_t blocks = (sv + 31) / 32;
  const int d = threadIdx.y;
  const int di = d / 9 - 1, dj = (d / 3) % 3 - 1, dk = d % 3 - 1;
  for (size_t blk = blockIdx.x; blk < blocks; blk += gridDim.x) {
    const size_t cs = blk * 32 + threadIdx.x;
    if (cs >= sv) continue;
    const int K = (int)(cs % Nc), J = (int)((cs / Nc) % Nc), I = A.I0 + (int)(cs / ((size_t)Nc * Nc));
    if (K < 1 || J < 1 || K > Nc - 2 || J > Nc - 2) continue;
    const size_t vn = vid(Nc, I + di, J + dj, K + dk);  // the neighbour c + d (inside the grid: c is interior)
    double acc = 0.0;
    for (int pi = -2; pi <= 2; ++pi) {
      const int ti = pi + 3 * di;
      if (ti < -3 || ti > 3) continue;
      for (int pj = -2; pj <= 2; ++pj) {
        const int tj = pj + 3 * dj;
        if (tj < -3 || tj > 3) continue;
        const double* Yr = A.Y + (size_t)(((ti + 3) * 7 + tj + 3) * 7 + 3) * sv + cs;
        const double* Pr = A.P + (size_t)pslot(pi, pj, 0) * nvc + vn;
#pragma unroll
        for (int pk = -2; pk <= 2; ++pk) {
          const int tk = pk + 3 * dk;
          if (tk < -3 || tk > 3) continue;
          acc = acc + Yr[(long long)tk * (long long)sv] * __ldg(Pr + (long long)pk * (long long)nvc);
        }
      }
    }
    A.out[(size_t)d * nvc + vid(Nc, I, J, K)] = acc;
  }
}

}  // namespace t3
