// 2D kernels: operator setup (classification, eff_eps, stencils, BoxMG P,
// Galerkin rows, smoothed restriction) and the additive cycle.
//
// Thread-per-vertex kernels over dense per-level grids.  Each one evaluates
// exactly the reference's per-element expression DAG (see tmg_kernels.cuh);
// the file is compiled with --fmad=false.
#include <cooperative_groups.h>

#include "kernels2d.cuh"

namespace cg = cooperative_groups;

namespace tmg {


// ===========================================================================
// setup
// ===========================================================================

// Vertex classification (spacetree.py:153-191) + hweight proximity bit.
// ref_prev: refined[l-1] ((n/3)^2) or nullptr when l == 0 (root always exists);
// ref_cur: refined[l] (n^2) or nullptr when l >= lmax.
__global__ void k_flags(uint8_t* __restrict__ flags, int n, const uint8_t* __restrict__ ref_prev,
                        const uint8_t* __restrict__ ref_cur) {
  const int N = n + 1;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (size_t)N * N) return;
  const int i = (int)(v / N), j = (int)(v % N);
  const int np = n / 3;
  int cnt = 0, all4 = 1, near = 0;
  for (int di = 0; di < 2; ++di)
    for (int dj = 0; dj < 2; ++dj) {
      const int ci = i - di, cj = j - dj;
      if (ci < 0 || cj < 0 || ci >= n || cj >= n) { all4 = 0; continue; }
      const int ex = ref_prev ? (ref_prev[(size_t)(ci / 3) * np + cj / 3] != 0) : 1;
      cnt += ex;
      const int r = ref_cur ? (ref_cur[(size_t)ci * n + cj] != 0) : 0;
      near |= r;
      all4 &= r;
    }
  uint8_t k;
  const bool border = (i == 0 || j == 0 || i == n || j == n);
  if (cnt == 0) k = K_NONE;
  else if (border) k = K_DIR;
  else if (cnt < 4) k = K_HANG;
  else k = all4 ? K_OVER : K_DOF;
  flags[v] = k | (near ? F_NEAR : 0);
}

// Injection targets (solvers.py:285-287): coarse vertex v is taken when the
// fine c-point 3v is INTERIOR_DOF or COARSE_OVERLAPPED.
__global__ void k_take(uint8_t* __restrict__ flags_c, int Nc, const uint8_t* __restrict__ flags_f,
                       int Nf) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (size_t)Nc * Nc) return;
  const int i = (int)(v / Nc), j = (int)(v % Nc);
  const int k = flags_f[(size_t)(3 * i) * Nf + 3 * j] & 7;
  uint8_t f = flags_c[v] & ~F_TAKE;
  if (k == K_DOF || k == K_OVER) f |= F_TAKE;
  flags_c[v] = f;
}

// eff_eps (solvers.py:165-175) + eps_masked = eff*exists (:180) + refined-op
// eps = eff*refined (:193-194).  Child mean = numpy's reshape(n,3,n,3).mean
// over (1,3): the three contiguous (j) triples summed first, then the rows,
// then / 9.
__global__ void k_eff(double* __restrict__ eff, double* __restrict__ epsm, double* __restrict__ reff,
                      const double* __restrict__ eps, const double* __restrict__ eff_child,
                      const uint8_t* __restrict__ ref_cur, const uint8_t* __restrict__ ref_prev,
                      int n) {
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (size_t)n * n) return;
  const int ci = (int)(c / n), cj = (int)(c % n);
  double e = eps[c];
  const bool refd = ref_cur && ref_cur[c];
  if (refd) {
    const int nf = 3 * n;
    double rows[3];
    for (int a = 0; a < 3; ++a) {
      const double* r = eff_child + (size_t)(3 * ci + a) * nf + 3 * cj;
      rows[a] = (r[0] + r[1]) + r[2];
    }
    e = ((rows[0] + rows[1]) + rows[2]) / 9.0;
  }
  eff[c] = e;
  const bool ex = ref_prev ? (ref_prev[(size_t)(ci / 3) * (n / 3) + cj / 3] != 0) : true;
  epsm[c] = e * (ex ? 1.0 : 0.0);
  if (reff) reff[c] = e * (refd ? 1.0 : 0.0);
}

// ElementOperator constant detection (operators.py:175-176): flag stays 1 iff
// arr[0] > 0 and every entry equals arr[0].
__global__ void k_const_check(const double* __restrict__ arr, size_t n, int* __restrict__ flag) {
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double first = arr[0];
  const bool bad = c < n && (!(first > 0.0) || arr[c] != first);
  if (__ballot_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0);
}

// counts of each kind + hanging (for masks sums, solvers.py:443, 449-459)
__global__ void k_count_kinds(const uint8_t* __restrict__ flags, size_t nv,
                              unsigned long long* __restrict__ counts) {
  __shared__ unsigned int sc[8];
  if (threadIdx.x < 8) sc[threadIdx.x] = 0;
  __syncthreads();
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) atomicAdd(&sc[flags[v] & 7], 1u);
  __syncthreads();
  if (threadIdx.x < 8 && sc[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)sc[threadIdx.x]);
}

// ElementOperator.diag (operators.py:190-199) -> raw; where(dof, raw, 1) -> diag (solvers.py:349).
__global__ void k_elem_diag(double* __restrict__ raw, double* __restrict__ diag,
                            const double* __restrict__ eps, const uint8_t* __restrict__ flags, int n) {
  const int N = n + 1;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (size_t)N * N) return;
  const int i = (int)(v / N), j = (int)(v % N);
  double out = 0.0;
  for (int a = 0; a < 4; ++a) {
    const int ci = i - (a & 1), cj = j - (a >> 1);
    if (ci < 0 || cj < 0 || ci >= n || cj >= n) continue;
    out = out + c_E[a * 5] * eps[(size_t)ci * n + cj];
  }
  raw[v] = out;
  diag[v] = is_dof(flags[v]) ? out : 1.0;
}

__global__ void k_table_diag(double* __restrict__ raw, double* __restrict__ diag,
                             const double* __restrict__ tbl, const uint8_t* __restrict__ flags,
                             size_t nv) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const double d = tbl[4 * nv + v];
  raw[v] = d;
  diag[v] = is_dof(flags[v]) ? d : 1.0;
}

// assemble_stencil_table (operators.py:251-264): per vertex and tap, adjacent
// element contributions E[a,b]*eps in corner order a.
__global__ void k_assemble(double* __restrict__ tbl, const double* __restrict__ eps, int n) {
  const int N = n + 1;
  const size_t nv = (size_t)N * N;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int i = (int)(v / N), j = (int)(v % N);
  double t[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) t[k] = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int a0 = a & 1, a1 = a >> 1;
    const int ci = i - a0, cj = j - a1;
    if (ci < 0 || cj < 0 || ci >= n || cj >= n) continue;
    const double e = eps[(size_t)ci * n + cj];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int b0 = b & 1, b1 = b >> 1;
      const int k = (b0 - a0 + 1) * 3 + (b1 - a1 + 1);
      t[k] = t[k] + c_E[a * 4 + b] * e;
    }
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) tbl[k * nv + v] = t[k];
}

// --- BoxMG ------------------------------------------------------------------

__device__ __forceinline__ bool cell_refined(const uint8_t* ref, const uint8_t* ref_prev, int nc,
                                             int ci, int cj) {
  // refined[l] & cells_exist(l) (solvers.py:232)
  if (ci < 0 || cj < 0 || ci >= nc || cj >= nc) return false;
  if (!ref || !ref[(size_t)ci * nc + cj]) return false;
  if (ref_prev && !ref_prev[(size_t)(ci / 3) * (nc / 3) + cj / 3]) return false;
  return true;
}

// _solve_gamma closed forms (operators.py:287-303) for one edge.
__device__ __forceinline__ void gamma_solve(const double c1[3], const double c2[3], bool active,
                                            double w[4], int* deg) {
  const double am1 = c1[0], a01 = c1[1], ap1 = c1[2];
  const double am2 = c2[0], a02 = c2[1], ap2 = c2[2];
  double det = a01 * a02 - ap1 * am2;
  const double scale = fabs(a01 * a02) + fabs(ap1 * am2);
  if (active && fabs(det) <= 1e-14 * fmax(scale, 1e-300)) atomicOr(deg, 1);
  if (!active) {
    w[0] = w[1] = w[2] = w[3] = 0.0;
    return;
  }
  w[0] = ((-am1) * a02) / det;
  w[1] = (am2 * am1) / det;
  w[2] = (ap1 * ap2) / det;
  w[3] = (a01 * (-ap2)) / det;
}

// Edges along x between coarse (I,J) and (I+1,J), I < nc, J <= nc: lump the
// fine rows at (3I+1,3J), (3I+2,3J) over the y taps (operators.py:331-340).
// Output ex[k*(nc*(nc+1)) + I*(nc+1)+J], k = wl1, wl2, wh1, wh2.
__global__ void k_gamma_x(double* __restrict__ ex, const double* __restrict__ tf, int nc,
                          const uint8_t* __restrict__ ref, const uint8_t* __restrict__ ref_prev,
                          int* __restrict__ deg) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t ne = (size_t)nc * (nc + 1);
  if (e >= ne) return;
  const int I = (int)(e / (nc + 1)), J = (int)(e % (nc + 1));
  const bool active = cell_refined(ref, ref_prev, nc, I, J - 1) || cell_refined(ref, ref_prev, nc, I, J);
  const int Nf = 3 * nc + 1;
  const size_t nvf = (size_t)Nf * Nf;
  double c1[3], c2[3];
  const size_t f1 = (size_t)(3 * I + 1) * Nf + 3 * J, f2 = (size_t)(3 * I + 2) * Nf + 3 * J;
  for (int a = 0; a < 3; ++a) {
    c1[a] = (tf[(a * 3 + 0) * nvf + f1] + tf[(a * 3 + 1) * nvf + f1]) + tf[(a * 3 + 2) * nvf + f1];
    c2[a] = (tf[(a * 3 + 0) * nvf + f2] + tf[(a * 3 + 1) * nvf + f2]) + tf[(a * 3 + 2) * nvf + f2];
  }
  double w[4];
  gamma_solve(c1, c2, active, w, deg);
  for (int k = 0; k < 4; ++k) ex[k * ne + e] = w[k];
}

// Edges along y between (I,J) and (I,J+1), I <= nc, J < nc: lump over x taps
// (operators.py:342-350).  ey[k*((nc+1)*nc) + I*nc + J].
__global__ void k_gamma_y(double* __restrict__ ey, const double* __restrict__ tf, int nc,
                          const uint8_t* __restrict__ ref, const uint8_t* __restrict__ ref_prev,
                          int* __restrict__ deg) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t ne = (size_t)(nc + 1) * nc;
  if (e >= ne) return;
  const int I = (int)(e / nc), J = (int)(e % nc);
  const bool active = cell_refined(ref, ref_prev, nc, I - 1, J) || cell_refined(ref, ref_prev, nc, I, J);
  const int Nf = 3 * nc + 1;
  const size_t nvf = (size_t)Nf * Nf;
  double c1[3], c2[3];
  const size_t f1 = (size_t)(3 * I) * Nf + 3 * J + 1, f2 = (size_t)(3 * I) * Nf + 3 * J + 2;
  for (int b = 0; b < 3; ++b) {
    c1[b] = (tf[(0 * 3 + b) * nvf + f1] + tf[(1 * 3 + b) * nvf + f1]) + tf[(2 * 3 + b) * nvf + f1];
    c2[b] = (tf[(0 * 3 + b) * nvf + f2] + tf[(1 * 3 + b) * nvf + f2]) + tf[(2 * 3 + b) * nvf + f2];
  }
  double w[4];
  gamma_solve(c1, c2, active, w, deg);
  for (int k = 0; k < 4; ++k) ey[k * ne + e] = w[k];
}

__device__ __forceinline__ size_t pslot(int oi, int oj) { return (size_t)((oi + 2) * 5 + (oj + 2)); }

// identity at c-points + face-point weights (operators.py:325-361); interior 0.
__global__ void k_p_init(double* __restrict__ P, int nc, const double* __restrict__ ex,
                         const double* __restrict__ ey) {
  const int Nc = nc + 1;
  const size_t nv = (size_t)Nc * Nc;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int I = (int)(v / Nc), J = (int)(v % Nc);
  const size_t nex = (size_t)nc * (nc + 1), ney = (size_t)(nc + 1) * nc;
  for (int k = 0; k < 25; ++k) P[k * nv + v] = 0.0;
  P[pslot(0, 0) * nv + v] = 1.0;
  if (I < nc) {  // low end of x-edge (I,J)
    const size_t e = (size_t)I * (nc + 1) + J;
    P[pslot(1, 0) * nv + v] = ex[0 * nex + e];
    P[pslot(2, 0) * nv + v] = ex[1 * nex + e];
  }
  if (I >= 1) {  // high end of x-edge (I-1,J)
    const size_t e = (size_t)(I - 1) * (nc + 1) + J;
    P[pslot(-2, 0) * nv + v] = ex[2 * nex + e];
    P[pslot(-1, 0) * nv + v] = ex[3 * nex + e];
  }
  if (J < nc) {
    const size_t e = (size_t)I * nc + J;
    P[pslot(0, 1) * nv + v] = ey[0 * ney + e];
    P[pslot(0, 2) * nv + v] = ey[1 * ney + e];
  }
  if (J >= 1) {
    const size_t e = (size_t)I * nc + (J - 1);
    P[pslot(0, -2) * nv + v] = ey[2 * ney + e];
    P[pslot(0, -1) * nv + v] = ey[3 * ney + e];
  }
}

// LU with partial pivoting + forward/back substitution for A X = B (4x4, 4
// right-hand sides), following LAPACK dgetf2/dgetrs: pivot = first max |a|,
// multipliers by the reciprocal pivot, back substitution by division.
__device__ void solve4(double A[4][4], double B[4][4]) {
  int piv[4];
  for (int k = 0; k < 4; ++k) {
    int p = k;
    double best = fabs(A[k][k]);
    for (int r = k + 1; r < 4; ++r)
      if (fabs(A[r][k]) > best) { best = fabs(A[r][k]); p = r; }
    piv[k] = p;
    if (p != k)
      for (int c = 0; c < 4; ++c) { double t = A[k][c]; A[k][c] = A[p][c]; A[p][c] = t; }
    const double rp = 1.0 / A[k][k];
    for (int r = k + 1; r < 4; ++r) A[r][k] = A[r][k] * rp;
    for (int r = k + 1; r < 4; ++r)
      for (int c = k + 1; c < 4; ++c) A[r][c] = A[r][c] - A[r][k] * A[k][c];
  }
  for (int k = 0; k < 4; ++k)
    if (piv[k] != k)
      for (int c = 0; c < 4; ++c) { double t = B[k][c]; B[k][c] = B[piv[k]][c]; B[piv[k]][c] = t; }
  for (int c = 0; c < 4; ++c) {
    for (int k = 0; k < 4; ++k)
      for (int r = k + 1; r < 4; ++r) B[r][c] = B[r][c] - B[k][c] * A[r][k];
    for (int k = 3; k >= 0; --k) {
      B[k][c] = B[k][c] / A[k][k];
      for (int r = 0; r < k; ++r) B[r][c] = B[r][c] - B[k][c] * A[r][k];
    }
  }
}

// Interior points of each refined coarse cell: the local 4x4 solve
// A_ff P_f = -A_fc P_c (operators.py:363-414).
__global__ void k_p_interior(double* __restrict__ P, int nc, const double* __restrict__ tf,
                             const double* __restrict__ ex, const double* __restrict__ ey,
                             const uint8_t* __restrict__ ref, const uint8_t* __restrict__ ref_prev) {
  const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (size_t)nc * nc) return;
  const int ci = (int)(c / nc), cj = (int)(c % nc);
  if (!cell_refined(ref, ref_prev, nc, ci, cj)) return;
  const int Nc = nc + 1, Nf = 3 * nc + 1;
  const size_t nv = (size_t)Nc * Nc, nvf = (size_t)Nf * Nf;
  const size_t nex = (size_t)nc * (nc + 1), ney = (size_t)(nc + 1) * nc;
  // known boundary weights of the 4x4 patch for each corner (p, q in 0..3)
  double known[4][4][4];
  for (int p = 0; p < 4; ++p)
    for (int q = 0; q < 4; ++q)
      for (int k = 0; k < 4; ++k) known[p][q][k] = 0.0;
  known[0][0][0] = 1.0; known[3][0][1] = 1.0; known[0][3][2] = 1.0; known[3][3][3] = 1.0;
  for (int dj = 0; dj < 2; ++dj) {  // bottom / top edges along x
    const int q = 3 * dj;
    const size_t e = (size_t)ci * (nc + 1) + (cj + dj);
    known[1][q][2 * dj] = ex[0 * nex + e];
    known[2][q][2 * dj] = ex[1 * nex + e];
    known[1][q][1 + 2 * dj] = ex[2 * nex + e];
    known[2][q][1 + 2 * dj] = ex[3 * nex + e];
  }
  for (int di = 0; di < 2; ++di) {  // left / right edges along y
    const int p = 3 * di;
    const size_t e = (size_t)(ci + di) * nc + cj;
    known[p][1][di] = ey[0 * ney + e];
    known[p][2][di] = ey[1 * ney + e];
    known[p][1][2 + di] = ey[2 * ney + e];
    known[p][2][2 + di] = ey[3 * ney + e];
  }
  const int fo[4][2] = {{1, 1}, {2, 1}, {1, 2}, {2, 2}};
  double A[4][4], B[4][4];
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) { A[r][k] = 0.0; B[r][k] = 0.0; }
  for (int r = 0; r < 4; ++r) {
    const int fp = fo[r][0], fq = fo[r][1];
    const size_t fv = (size_t)(3 * ci + fp) * Nf + (3 * cj + fq);
    for (int da = -1; da <= 1; ++da)
      for (int db = -1; db <= 1; ++db) {
        const int tp = fp + da, tq = fq + db;
        const double coef = tf[(size_t)((da + 1) * 3 + (db + 1)) * nvf + fv];
        const bool inner = (tp == 1 || tp == 2) && (tq == 1 || tq == 2);
        if (inner) {
          const int idx = (tp - 1) + 2 * (tq - 1);  // (1,1),(2,1),(1,2),(2,2)
          A[r][idx] = A[r][idx] + coef;
        } else {
          for (int k = 0; k < 4; ++k) B[r][k] = B[r][k] - coef * known[tp][tq][k];
        }
      }
  }
  solve4(A, B);
  const int corner[4][2] = {{0, 0}, {3, 0}, {0, 3}, {3, 3}};
  for (int k = 0; k < 4; ++k) {
    const int wi = ci + corner[k][0] / 3, wj = cj + corner[k][1] / 3;
    const size_t wv = (size_t)wi * Nc + wj;
    for (int r = 0; r < 4; ++r) {
      const int oi = 3 * ci + fo[r][0] - 3 * wi, oj = 3 * cj + fo[r][1] - 3 * wj;
      P[pslot(oi, oj) * nv + wv] = B[r][k];
    }
  }
}

// Hanging fine targets take d-linear weights; weights pointing outside the
// fine grid are dropped (operators.py:416-436).
__global__ void k_p_fix(double* __restrict__ P, int nc, const uint8_t* __restrict__ flags_f) {
  const int Nc = nc + 1, Nf = 3 * nc + 1;
  const size_t nv = (size_t)Nc * Nc;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int I = (int)(v / Nc), J = (int)(v % Nc);
  for (int oi = -2; oi <= 2; ++oi)
    for (int oj = -2; oj <= 2; ++oj) {
      const int fi = 3 * I + oi, fj = 3 * J + oj;
      const size_t s = pslot(oi, oj) * nv + v;
      if (fi < 0 || fj < 0 || fi >= Nf || fj >= Nf) { P[s] = 0.0; continue; }
      if ((flags_f[(size_t)fi * Nf + fj] & 7) == K_HANG)
        P[s] = fmax(0.0, 1.0 - abs(oi) / 3.0) * fmax(0.0, 1.0 - abs(oj) / 3.0);
    }
}

__device__ __forceinline__ double p_at(const double* P, const size_t nv, int Nc, int I, int J,
                                       int oi, int oj) {
  if (I < 0 || J < 0 || I >= Nc || J >= Nc) return 0.0;
  if (oi < -2 || oi > 2 || oj < -2 || oj > 2) return 0.0;
  return P[pslot(oi, oj) * nv + (size_t)I * Nc + J];
}

// ritz_galerkin_coarse (operators.py:446-478) at overlapped coarse vertices,
// written over the rediscretized table (solvers.py:236-238).  The fine table
// is masked to equation rows on the fly (solvers.py:234).
__global__ void k_rap(double* __restrict__ tbl, const uint8_t* __restrict__ flags_c, int nc,
                      const double* __restrict__ tf, const uint8_t* __restrict__ flags_f,
                      const double* __restrict__ P) {
  const int Nc = nc + 1, Nf = 3 * nc + 1;
  const size_t nv = (size_t)Nc * Nc, nvf = (size_t)Nf * Nf;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  if ((flags_c[v] & 7) != K_OVER) return;
  const int I = (int)(v / Nc), J = (int)(v % Nc);
  double out[9];
  for (int k = 0; k < 9; ++k) out[k] = 0.0;
  for (int oi = -2; oi <= 2; ++oi)
    for (int oj = -2; oj <= 2; ++oj) {
      const double rw = P[pslot(oi, oj) * nv + v];
      const int fi = 3 * I + oi, fj = 3 * J + oj;
      const bool in = fi >= 0 && fj >= 0 && fi < Nf && fj < Nf;
      const size_t fv = in ? (size_t)fi * Nf + fj : 0;
      const bool row = in && is_dof(flags_f[fv]);
      for (int si = -1; si <= 1; ++si)
        for (int sj = -1; sj <= 1; ++sj) {
          const double ac = row ? tf[(size_t)((si + 1) * 3 + (sj + 1)) * nvf + fv] : 0.0;
          const int ti = oi + si, tj = oj + sj;
          for (int dwi = -1; dwi <= 1; ++dwi) {
            const int pi = ti - 3 * dwi;
            if (pi < -3 || pi > 3) continue;
            for (int dwj = -1; dwj <= 1; ++dwj) {
              const int pj = tj - 3 * dwj;
              if (pj < -3 || pj > 3) continue;
              const double pw = p_at(P, nv, Nc, I + dwi, J + dwj, pi, pj);
              const int k = (dwi + 1) * 3 + (dwj + 1);
              out[k] = out[k] + (rw * ac) * pw;
            }
          }
        }
    }
  for (int k = 0; k < 9; ++k) tbl[k * nv + v] = out[k];
}

// smoothed_restriction_table (operators.py:508-547), 49 planes per coarse
// vertex.  fine == nullptr: unit-coefficient operator; otherwise the masked
// fine stencil table and raw fine diagonal.  pconst: weights are the constant
// d-linear table (geometric_p_table, operators.py:440-443), else P planes.
__global__ void k_rtilde(double* __restrict__ Rt, int nc, const double* __restrict__ P, int pconst,
                         const double* __restrict__ tf, const uint8_t* __restrict__ flags_f,
                         const double* __restrict__ diag_f, double omega) {
  const int Nc = nc + 1, Nf = 3 * nc + 1;
  const size_t nv = (size_t)Nc * Nc, nvf = (size_t)Nf * Nf;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int I = (int)(v / Nc), J = (int)(v % Nc);
  double out[49];
  for (int k = 0; k < 49; ++k) out[k] = 0.0;
  for (int ji = -2; ji <= 2; ++ji)
    for (int jj = -2; jj <= 2; ++jj) {
      const double w = pconst ? fmax(0.0, 1.0 - abs(ji) / 3.0) * fmax(0.0, 1.0 - abs(jj) / 3.0)
                              : P[pslot(ji, jj) * nv + v];
      const int fi = 3 * I + ji, fj = 3 * J + jj;
      const bool in = fi >= 0 && fj >= 0 && fi < Nf && fj < Nf;
      const size_t fv = in ? (size_t)fi * Nf + fj : 0;
      const bool row = in && (tf == nullptr || is_dof(flags_f[fv]));
      for (int si = -1; si <= 1; ++si)
        for (int sj = -1; sj <= 1; ++sj) {
          const int ti = ji + si, tj = jj + sj;
          if (ti < -3 || ti > 3 || tj < -3 || tj > 3) continue;
          const int k = (ti + 3) * 7 + (tj + 3);
          if (tf == nullptr) {
            out[k] = out[k] + w * c_A1INV[(si + 1) * 3 + (sj + 1)];
          } else {
            const double ar = row ? tf[(size_t)((si + 1) * 3 + (sj + 1)) * nvf + fv] : 0.0;
            const int gi = 3 * I + ti, gj = 3 * J + tj;
            double dinv = 0.0;
            if (gi >= 0 && gj >= 0 && gi < Nf && gj < Nf) {
              const double dg = diag_f[(size_t)gi * Nf + gj];
              dinv = dg != 0.0 ? 1.0 / dg : 0.0;
            }
            out[k] = out[k] + (w * ar) * dinv;
          }
        }
    }
  for (int k = 0; k < 49; ++k) Rt[k * nv + v] = out[k] * omega;
}

// masked copy of a fine table (rows zeroed off the equation set) is never
// materialised; k_rap / k_rtilde mask on the fly.

// ===========================================================================
// cycle
// ===========================================================================

// --- per-vertex bodies (shared by the grid kernels and the cluster kernel) ---

// d-linear prolongation with an arbitrary coarse-value functor (operators.py:96-127).
template <class CV>
__device__ __forceinline__ double prolong_dlinear_fn(const CV& cv, int Nc, int i, int j) {
  const int m = Nc - 1;
  const int qi = i / 3, ri = i - 3 * qi, qni = min(qi + 1, m);
  const int qj = j / 3, rj = j - 3 * qj, qnj = min(qj + 1, m);
  const double c00 = cv(qi, qj), c10 = cv(qni, qj), c01 = cv(qi, qnj), c11 = cv(qni, qnj);
  const double wli = c_WL[ri], wri = c_WR[ri];
  const double t0 = wli * c00 + wri * c10;
  const double t1 = wli * c01 + wri * c11;
  return c_WL[rj] * t0 + c_WR[rj] * t1;
}

// P-table prolongation with a coarse-value functor (operators.py:570-581):
// (oi, oj) row-major == coarse (I, J) descending.
template <class LD, class CV>
__device__ __forceinline__ double prolong_table_fn(const CV& cv, const double* P, int Nc, int i,
                                                   int j) {
  const size_t nvc = (size_t)Nc * Nc;
  const int qi = i / 3, ri = i - 3 * qi;
  const int qj = j / 3, rj = j - 3 * qj;
  double w[4], x[4];
  bool use[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int di = 1 - (k >> 1), dj = 1 - (k & 1);
    use[k] = (di == 0 || ri > 0) && (dj == 0 || rj > 0);
    const int I = qi + di, J = qj + dj;
    const int oi = i - 3 * I, oj = j - 3 * J;
    w[k] = use[k] ? LD::ld(P + (size_t)((oi + 2) * 5 + (oj + 2)) * nvc + (size_t)I * Nc + J) : 0.0;
    x[k] = use[k] ? cv(I, J) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (use[k]) acc = acc + w[k] * x[k];
  return acc;
}

// Operator image from a loaded 3x3 neighbourhood xu and operator data ow
// (table taps, or element eps of the 4 adjacent cells): operators.py:143-248.
template <bool CHK>
__device__ __forceinline__ double op_from(const OpView& op, const double xu[9], const double ow[9],
                                          int N, int i, int j) {
  if (op.kind == OP_CONST) return const_from<CHK>(xu, N, i, j, op.s_side, op.s_mid);
  double acc = 0.0;
  if (op.kind == OP_TABLE) {
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (in_rng<CHK>(i + k / 3 - 1, j + k % 3 - 1, N)) acc = acc + ow[k] * xu[k];
    return acc;
  }
  if (op.kind == OP_ELEMENT) {
    const int n = N - 1;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int a0 = c & 1, a1 = c >> 1;
      const int ci = i - a0, cj = j - a1;
      if (CHK && !(ci >= 0 && cj >= 0 && ci < n && cj < n)) continue;
      double e = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        e = e + c_E[c * 4 + b] * xu[((b & 1) - a0 + 1) * 3 + ((b >> 1) - a1 + 1)];
      acc = acc + ow[c] * e;
    }
    return acc;
  }
  return 0.0;
}

template <class LD, bool CHK>
__device__ __forceinline__ void op_load(const OpView& op, int N, int i, int j, double ow[9]) {
  const size_t nv = (size_t)N * N, v = (size_t)i * N + j;
  if (op.kind == OP_TABLE) {
#pragma unroll
    for (int k = 0; k < 9; ++k) ow[k] = LD::ld(op.tbl + (size_t)k * nv + v);
  } else if (op.kind == OP_ELEMENT) {
    const int n = N - 1;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int ci = i - (c & 1), cj = j - (c >> 1);
      ow[c] = (!CHK || (ci >= 0 && cj >= 0 && ci < n && cj < n)) ? LD::ld(op.eps + (size_t)ci * n + cj)
                                                                  : 0.0;
    }
  }
}

// advance(), fine -> coarse sweep at one vertex (solvers.py:345-375).
// TOP: 1 = finest level (no restriction code), 0 = coarser level.  CHK:
// range tests on (true) or compiled out for vertices whose whole footprint
// (3x3 stencil, 5x5 / 7x7 fine window) lies inside the grid.  All loads of
// the residual part are issued in one batch, the damping part (7x7 window of
// rho_dof_{l+1}) in a second one.
template <class LD, int TOP, bool CHK>
__device__ __forceinline__ void down_vertex_impl(const DownArgs& a, int i, int j, double& s,
                                                 double& m) {
  constexpr bool is_top = TOP == 1;
  const int N = a.N;
  const size_t v = (size_t)i * N + j;
  const size_t nv = (size_t)N * N;
  // ---- batch 1 -------------------------------------------------------------
  const uint8_t f = a.flags[v];
  double xu[9], ow[9], rw[9];
  load3x3<LD, CHK>(a.u, N, i, j, xu);
  op_load<LD, CHK>(a.op, N, i, j, ow);
  const double rhs = a.rhs ? LD::ld(a.rhs + v) : 0.0;
  const double dg = a.write ? LD::ld(a.diag + v) : 1.0;
  double pw[25], rx[25];
  if (!is_top) {
    op_load<LD, CHK>(a.rop, N, i, j, rw);
    const int Nf = a.Nf, m3 = (Nf - 1) / 3;
#pragma unroll
    for (int k = 0; k < 25; ++k) {
      const int oi = k / 5 - 2, oj = k % 5 - 2;
      const int fi = 3 * i + oi, fj = 3 * j + oj;
      bool ok;
      if (a.boxmg) {
        ok = in_rng<CHK>(fi, fj, Nf);
        pw[k] = LD::ld(a.P + (size_t)k * nv + v);
      } else {
        ok = !CHK || !((oi < 0 && i < 1) || (oi > 0 && i > m3 - 1) || (oj < 0 && j < 1) ||
                       (oj > 0 && j > m3 - 1));
        pw[k] = 0.0;
      }
      rx[k] = ok ? LD::ld(a.rho_f + (size_t)fi * Nf + fj) : 0.0;
    }
  }
  // ---- residual -------------------------------------------------------------
  const int kind = f & 7;
  const bool src = is_src(f), dof = is_dof(f);
  double rho = 0.0;
  if (src) {
    const double au = op_from<CHK>(a.op, xu, ow, N, i, j);
    double b;
    if (is_top) {
      b = rhs;
    } else {
      // b_l = R rho_{l+1} + rhs_l (solvers.py:370-371), then + bpart (:351-352)
      if (a.boxmg) {
        b = 0.0;  // TransferOps.restrict, 5x5 taps row-major (operators.py:586-596)
#pragma unroll
        for (int k = 0; k < 25; ++k)
          if (in_rng<CHK>(3 * i + k / 5 - 2, 3 * j + k % 5 - 2, a.Nf)) b = b + pw[k] * rx[k];
      } else {
        const int m3 = (a.Nf - 1) / 3;  // restrict_dlinear: axis 0 then axis 1 (operators.py:111-132)
        b = 0.0;
#pragma unroll
        for (int bj = 0; bj < 5; ++bj) {
          const int oj = bj - 2;
          if (CHK && ((oj < 0 && j < 1) || (oj > 0 && j > m3 - 1))) continue;
          double t = 0.0;
#pragma unroll
          for (int ai = 0; ai < 5; ++ai) {
            const int oi = ai - 2;
            if (CHK && ((oi < 0 && i < 1) || (oi > 0 && i > m3 - 1))) continue;
            t = t + c_W5[ai] * rx[ai * 5 + bj];
          }
          b = b + c_W5[bj] * t;
        }
      }
      if (a.rhs) b = b + rhs;
      if (a.rop.kind != OP_NONE) {
        const double bp = (kind == K_OVER) ? au : op_from<CHK>(a.rop, xu, rw, N, i, j);
        b = b + bp;
      }
    }
    rho = b - au;
  }
  const double rd = dof ? rho : 0.0;
  if (kind == K_DOF) {  // composite stats (solvers.py:435-443)
    const double h = (f & F_NEAR) ? a.hA : a.hB;
    const double t = h * rd;
    s = s + t * t;
    m = fmax(m, fabs(rd));
  }
  if (a.write) {
    double d;
    if (a.variant == VAR_BPX && !is_top) d = a.omega * rd;
    else d = (a.w_l * rd) / dg;
    if (a.variant == VAR_JAC && !is_top && dof) {
      // dtil = ds * ((wt * R~ rho_dof_{l+1}) / diag) (solvers.py:360-363)
      double bt;
      if (a.rt_mode == RT_FROM_P) {
        // ---- batch 2: 7x7 window of rho_dof_{l+1}; R~ weights rebuilt from the
        // P registers in exactly the order of smoothed_restriction_table
        // (operators.py:520-531, 546), so the result equals the stored table's.
        double fx[49];
#pragma unroll
        for (int k = 0; k < 49; ++k) {
          const int fi = 3 * i + k / 7 - 3, fj = 3 * j + k % 7 - 3;
          fx[k] = in_rng<CHK>(fi, fj, a.Nf) ? LD::ld(a.rdof_f + (size_t)fi * a.Nf + fj) : 0.0;
        }
        bt = 0.0;
#pragma unroll
        for (int k = 0; k < 49; ++k) {
          const int ti = k / 7 - 3, tj = k % 7 - 3;
          if (!in_rng<CHK>(3 * i + ti, 3 * j + tj, a.Nf)) continue;
          double acc = 0.0;
#pragma unroll
          for (int ji = -2; ji <= 2; ++ji) {
            if (ti - ji < -1 || ti - ji > 1) continue;
#pragma unroll
            for (int jj = -2; jj <= 2; ++jj) {
              if (tj - jj < -1 || tj - jj > 1) continue;
              acc = acc + pw[(ji + 2) * 5 + (jj + 2)] * c_A1INV[(ti - ji + 1) * 3 + (tj - jj + 1)];
            }
          }
          bt = bt + (acc * a.rt_omega) * fx[k];
        }
      } else if (a.rt_mode == RT_GEOM_FAST) {
        bt = restrict_rt_geom_at<LD, CHK>(a.rdof_f, a.Nf, i, j, a.rt_side, a.rt_mid, a.rt_scale);
      } else {
        bt = restrict_rt_table_at<LD, CHK>(a.rdof_f, a.Nf, a.Rt, N, i, j);
      }
      d = d - a.ds * ((a.wt * bt) / dg);
    } else if (a.variant == VAR_JAC && !is_top) {
      d = d - 0.0;
    }
    a.g[v] = d;
  }
  if (a.rho) {
    const bool cpt = (i % 3 == 0) && (j % 3 == 0);
    a.rho[v] = (a.variant == VAR_AFACC && cpt) ? 0.0 : rho;  // afacc: solvers.py:365-368
  }
  if (a.rdof) a.rdof[v] = rd;
}

// Interior vertices (i, j in [1, N-2]) take the check-free instantiation.
template <class LD, int TOP>
__device__ __forceinline__ void down_vertex(const DownArgs& a, int i, int j, double& s, double& m) {
  if (i >= 1 && j >= 1 && i <= a.N - 2 && j <= a.N - 2)
    down_vertex_impl<LD, TOP, false>(a, i, j, s, m);
  else
    down_vertex_impl<LD, TOP, true>(a, i, j, s, m);
}

// advance(), coarse -> fine carry at one vertex (solvers.py:377-395) and the
// FAS injection of the new value down the chain of taking levels (:283-288).
template <class LD>
__device__ __forceinline__ void up_vertex(const UpArgs& a, int i, int j) {
  const size_t v = (size_t)i * a.N + j;
  const uint8_t f = a.flags[v];
  double g = LD::ld(a.g + v);
  if (a.pi && !a.is_bottom) {
    // dtil_l = ds * P(inj d_l), inj = d_l at taken c-points (solvers.py:377-384)
    const uint8_t* fc = a.flags_c;
    const double* gl = a.g;
    const int Nc = a.Nc, N = a.N;
    auto inj = [&](int I, int J) -> double {
      return (fc[(size_t)I * Nc + J] & F_TAKE) ? LD::ld(gl + (size_t)(3 * I) * N + 3 * J) : 0.0;
    };
    const double pv = a.boxmg ? prolong_table_fn<LD>(inj, a.P, Nc, i, j)
                              : prolong_dlinear_fn(inj, Nc, i, j);
    const double dt = is_dof(f) ? a.ds * pv : 0.0;
    g = g - dt;
  }
  double c = g;
  if (!a.is_bottom) {
    const double* cc = a.carry_c;
    const int Nc = a.Nc;
    auto cv = [&](int I, int J) -> double { return LD::ld(cc + (size_t)I * Nc + J); };
    const double pc = a.boxmg ? prolong_table_fn<LD>(cv, a.P, Nc, i, j)
                              : prolong_dlinear_fn(cv, Nc, i, j);
    c = pc + g;
  }
  if ((f & 7) == K_NONE) c = 0.0;
  if (a.carry) a.carry[v] = c;
  const double un = a.u[v] + c;
  a.u[v] = un;
  int ii = i, jj = j;
  for (int lc = a.l - 1; lc >= a.l0; --lc) {
    if (ii % 3 != 0 || jj % 3 != 0) break;
    ii /= 3;
    jj /= 3;
    const size_t vc = (size_t)ii * a.Nl[lc] + jj;
    if (!(a.fl[lc][vc] & F_TAKE)) break;
    a.ul[lc][vc] = un;
  }
}

template <int BS>
__device__ __forceinline__ void block_reduce(double& s, double& m) {
  __shared__ double ss[BS / 32], sm[BS / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  }
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  const int w = t >> 5, lane = t & 31;
  const int nw = (int)(blockDim.x * blockDim.y) >> 5;  // <= BS / 32
  if (lane == 0) { ss[w] = s; sm[w] = m; }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < nw; ++k) { a += ss[k]; b = fmax(b, sm[k]); }
    s = a;
    m = b;
  }
  __syncthreads();
}

// Grid kernels use 32 x 8 thread tiles over (j, i): no index division and
// the 3x3 neighbourhoods of a tile share cache lines.
// Adaptive levels launch one block per entry of the level's patch list (1D grid) instead of one
// per tile of the dense vertex array: vertices that do not exist carry zeros in every work vector
// and are never read as DoFs, so tiles without an existing vertex need no work.
__device__ __forceinline__ void tile_origin(const uint32_t* tiles, int& bx, int& by) {
  if (tiles) {
    const uint32_t t = tiles[blockIdx.x];
    bx = (int)(t & 0xffffu);
    by = (int)(t >> 16);
  } else {
    bx = blockIdx.x;
    by = blockIdx.y;
  }
}

template <int TOP>
__global__ void __launch_bounds__(kBlock) k_down(const __grid_constant__ DownArgs a) {
  int bx, by;
  tile_origin(a.tiles, bx, by);
  const int j = bx * kTileX + threadIdx.x;
  const int i = by * blockDim.y + threadIdx.y;  // tile height: 8 (finest) or 2 (coarse)
  double s = 0.0, m = 0.0;
  if (i < a.N && j < a.N) down_vertex<LdNC, TOP>(a, i, j, s, m);
  block_reduce<kBlock>(s, m);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const int b = blockIdx.y * gridDim.x + blockIdx.x;
    a.part_sum[b] = s;
    a.part_max[b] = m;
  }
}

__global__ void __launch_bounds__(kBlock) k_up(const __grid_constant__ UpArgs a) {
  int bx, by;
  tile_origin(a.tiles, bx, by);
  const int j = bx * kTileX + threadIdx.x;
  const int i = by * blockDim.y + threadIdx.y;
  if (i < a.N && j < a.N) up_vertex<LdNC>(a, i, j);
}

// 1 where the (32 x ty) vertex tile holds an existing vertex (setup of the patch lists)
__global__ void k_tile_any(const uint8_t* __restrict__ flags, int N, int ty, int tx_count, int ty_count,
                           uint8_t* __restrict__ mask) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tx_count * ty_count) return;
  const int bx = t % tx_count, by = t / tx_count;
  uint8_t any = 0;
  for (int r = 0; r < ty && !any; ++r) {
    const int i = by * ty + r;
    if (i >= N) break;
    for (int c = 0; c < kTileX; ++c) {
      const int j = bx * kTileX + c;
      if (j >= N) break;
      if ((flags[(size_t)i * N + j] & 7) != K_NONE) {
        any = 1;
        break;
      }
    }
  }
  mask[t] = any;
}

// hanging-vertex refresh over the level's patch list (one block per listed tile)
__global__ void __launch_bounds__(kBlock) k_hang_tiles(double* __restrict__ u, const uint8_t* __restrict__ flags,
                                                       int N, const double* __restrict__ uc, int Nc,
                                                       const uint32_t* __restrict__ tiles) {
  int bx, by;
  tile_origin(tiles, bx, by);
  const int j = bx * kTileX + threadIdx.x;
  const int i = by * blockDim.y + threadIdx.y;
  if (i >= N || j >= N) return;
  const size_t v = (size_t)i * N + j;
  if ((flags[v] & 7) != K_HANG) return;
  u[v] = prolong_dlinear_at<LdNC>(uc, Nc, i, j);
}

// Plain loads for the coarse-chain kernel: its level vectors are written and
// re-read by the same thread block (L1-coherent after __syncthreads).
struct LdGen {
  static __device__ __forceinline__ double ld(const double* p) { return *p; }
};

// The coarse chain lmin..lc in ONE thread block: levels lc..l0 down,
// deterministic stats finalisation over every partial of the cycle, levels
// l0..lc up (with the walk-down FAS injection).  Phases are separated by
// __syncthreads only; the per-level argument blocks live in the kernel's
// parameter space (__grid_constant__), so field reads are constant-bank hits.
__global__ void __launch_bounds__(kCoarseBlock) k_coarse(const __grid_constant__ CoarseArgs a) {
  __shared__ double rs[kCoarseBlock / 32], rm[kCoarseBlock / 32];
  const int tid = threadIdx.x, nthr = blockDim.x;
  int nst = 0;
  auto stamp = [&]() {
    if (a.stamps && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.stamps[nst] = t;
    }
    ++nst;
  };
  stamp();
  double s = 0.0, m = 0.0;
  for (int l = a.lc; l >= a.l0; --l) {
    const DownArgs& d = a.down[l - a.l0];
    const int N = d.N, nv = N * N;
    if (d.is_top) {
      for (int v = tid; v < nv; v += nthr) {
        const int i = v / N;
        down_vertex<LdGen, 1>(d, i, v - i * N, s, m);
      }
    } else {
      for (int v = tid; v < nv; v += nthr) {
        const int i = v / N;
        down_vertex<LdGen, 0>(d, i, v - i * N, s, m);
      }
    }
    __syncthreads();
    stamp();
  }
  // fixed-order reduction of every partial of this cycle -> history slot
  block_reduce<kCoarseBlock>(s, m);
  double x = 0.0, y = 0.0;
  for (int k = tid; k < a.part_base; k += nthr) {
    x += a.part_sum[k];
    y = fmax(y, a.part_max[k]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_down_sync(0xffffffffu, x, o);
    y = fmax(y, __shfl_down_sync(0xffffffffu, y, o));
  }
  if ((tid & 31) == 0) { rs[tid >> 5] = x; rm[tid >> 5] = y; }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0, u = 0.0;
    for (int k = 0; k < kCoarseBlock / 32; ++k) { t += rs[k]; u = fmax(u, rm[k]); }
    t += s;  // the chain's own contribution
    u = fmax(u, m);
    const int slot = *a.counter;
    a.hist[2 * (slot % a.cap)] = sqrt(t);
    a.hist[2 * (slot % a.cap) + 1] = u;
    *a.counter = slot + 1;
  }
  stamp();
  if (!a.do_up) return;
  for (int l = a.l0; l <= a.lc; ++l) {
    const UpArgs& u = a.up[l - a.l0];
    const int N = u.N, nv = N * N;
    for (int v = tid; v < nv; v += nthr) {
      const int i = v / N;
      up_vertex<LdGen>(u, i, v - i * N);
    }
    __syncthreads();
    stamp();
  }
}

// The coarse chain on a thread-block cluster: the same phases as k_coarse,
// with each level's vertices spread over the kClusterCTAs CTAs of the cluster
// and cluster barriers (release / acquire at cluster scope) between levels.
// Data produced inside the launch is read through L2 (LdCG).  The residual
// partials are combined in a fixed order by CTA rank 0.
constexpr int kClusterCTAs = 8;

__global__ void __launch_bounds__(kCoarseBlock) k_coarse_cl(const __grid_constant__ CoarseArgs a,
                                                             double* scratch) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double rs[kCoarseBlock / 32], rm[kCoarseBlock / 32];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int rank = (int)cl.block_rank(), csz = (int)cl.num_blocks();
  const int gt = rank * nthr + tid, gn = csz * nthr;
  double s = 0.0, m = 0.0;
  for (int l = a.lc; l >= a.l0; --l) {
    const DownArgs& d = a.down[l - a.l0];
    const int N = d.N, nv = N * N;
    if (d.is_top) {
      for (int v = gt; v < nv; v += gn) {
        const int i = v / N;
        down_vertex<LdCG, 1>(d, i, v - i * N, s, m);
      }
    } else {
      for (int v = gt; v < nv; v += gn) {
        const int i = v / N;
        down_vertex<LdCG, 0>(d, i, v - i * N, s, m);
      }
    }
    cl.sync();
  }
  // per-CTA partial -> scratch[rank]; rank 0 reduces grid partials + scratch in order
  block_reduce<kCoarseBlock>(s, m);
  if (tid == 0) {
    scratch[2 * rank] = s;
    scratch[2 * rank + 1] = m;
  }
  cl.sync();
  if (rank == 0) {
    double x = 0.0, y = 0.0;
    for (int k = tid; k < a.part_base; k += nthr) {
      x += a.part_sum[k];
      y = fmax(y, a.part_max[k]);
    }
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_down_sync(0xffffffffu, x, o);
      y = fmax(y, __shfl_down_sync(0xffffffffu, y, o));
    }
    if ((tid & 31) == 0) { rs[tid >> 5] = x; rm[tid >> 5] = y; }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0, u = 0.0;
      for (int k = 0; k < kCoarseBlock / 32; ++k) { t += rs[k]; u = fmax(u, rm[k]); }
      for (int k = 0; k < csz; ++k) {
        t += __ldcg(scratch + 2 * k);
        u = fmax(u, __ldcg(scratch + 2 * k + 1));
      }
      const int slot = *a.counter;
      a.hist[2 * (slot % a.cap)] = sqrt(t);
      a.hist[2 * (slot % a.cap) + 1] = u;
      *a.counter = slot + 1;
    }
  }
  if (!a.do_up) return;
  for (int l = a.l0; l <= a.lc; ++l) {
    const UpArgs& u = a.up[l - a.l0];
    const int N = u.N, nv = N * N;
    for (int v = gt; v < nv; v += gn) {
      const int i = v / N;
      up_vertex<LdCG>(u, i, v - i * N);
    }
    cl.sync();
  }
}

// ---------------------------------------------------------------------------
// The fused cycle: one persistent launch (cooperative: every CTA resident), grid barriers between
// the level phases.  The barrier is a self-resetting arrival counter + generation word (release /
// acquire at gpu scope, bar.sync on both sides), so plain (L1-cached) loads after it observe what
// any CTA wrote before it; every work vector is written in one phase and only read in later ones.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& gen) {
  __syncthreads();  // the CTA's writes happen-before thread 0's release below (bar.sync is cumulative)
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    unsigned old, cur;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    if (old == nblocks - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(bar), "r"(0u) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1u) : "memory");
    } else {
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == gen);
    }
  }
  ++gen;
  __syncthreads();
}

// unit w of a level -> vertex (i, j) of this lane: a row of 32 vertices of the dense array, or of
// a listed tile
__device__ __forceinline__ void unit_vertex(const uint32_t* tiles, int tile_h, int N, int w, int lane, int& i,
                                            int& j) {
  if (tiles) {
    const int e = w / tile_h, r = w - e * tile_h;
    const uint32_t t = tiles[e];
    i = (int)(t >> 16) * tile_h + r;
    j = (int)(t & 0xffffu) * kTileX + lane;
  } else {
    const int tx = (N + kTileX - 1) / kTileX;
    i = w / tx;
    j = (w - i * tx) * kTileX + lane;
  }
}

#ifndef CYC_MINB
#define CYC_MINB 1
#endif
__global__ void __launch_bounds__(kBlock, CYC_MINB) k_cycle(const __grid_constant__ CycleArgs a) {
  __shared__ double rs[kCycleWarps], rm[kCycleWarps];
  const int tid = threadIdx.y * kTileX + threadIdx.x, lane = tid & 31;
  const int gw = blockIdx.x * kCycleWarps + (tid >> 5), nw = gridDim.x * kCycleWarps;
  const unsigned nb = gridDim.x;
  // the barrier's generation word cannot advance before this CTA's first arrival: read it once
  unsigned gen;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(a.bar + 1) : "memory");
  int nst = 0;
  auto stamp = [&]() {
    if (a.stamps && blockIdx.x == 0 && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.stamps[nst] = t;
    }
    ++nst;
  };
  stamp();
  double s = 0.0, m = 0.0;
  for (int l = a.ltop; l >= a.l0; --l) {
    const DownArgs& d = a.down[l - a.l0];
    const int th = a.tile_h[l - a.l0], nu = a.units[l - a.l0];
    for (int w = gw; w < nu; w += nw) {
      int i, j;
      unit_vertex(d.tiles, th, d.N, w, lane, i, j);
      if (i < d.N && j < d.N) {
        if (d.is_top) down_vertex<LdGen, 1>(d, i, j, s, m);
        else down_vertex<LdGen, 0>(d, i, j, s, m);
      }
    }
    if (l == a.l0) {  // this warp's share of the composite residual norm
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_down_sync(0xffffffffu, s, o);
        m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
      }
      if (lane == 0) {
        a.wpart[2 * gw] = s;
        a.wpart[2 * gw + 1] = m;
      }
    }
    grid_barrier(a.bar, nb, gen);
    stamp();
  }
  if (blockIdx.x == 0) {  // fixed-order reduction of the warps' partials -> history slot
    double x = 0.0, y = 0.0;
    for (int k = tid; k < nw; k += kBlock) {
      x += __ldcg(a.wpart + 2 * k);
      y = fmax(y, __ldcg(a.wpart + 2 * k + 1));
    }
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_down_sync(0xffffffffu, x, o);
      y = fmax(y, __shfl_down_sync(0xffffffffu, y, o));
    }
    if (lane == 0) { rs[tid >> 5] = x; rm[tid >> 5] = y; }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0, u = 0.0;
      for (int k = 0; k < kCycleWarps; ++k) { t += rs[k]; u = fmax(u, rm[k]); }
      const int slot = *a.counter;
      a.hist[2 * (slot % a.cap)] = sqrt(t);
      a.hist[2 * (slot % a.cap) + 1] = u;
      *a.counter = slot + 1;
    }
  }
  stamp();
  if (!a.do_up) return;
  for (int l = a.l0; l <= a.ltop; ++l) {
    const UpArgs& u = a.up[l - a.l0];
    const int th = a.tile_h[l - a.l0], nu = a.units[l - a.l0];
    for (int w = gw; w < nu; w += nw) {
      int i, j;
      unit_vertex(u.tiles, th, u.N, w, lane, i, j);
      if (i < u.N && j < u.N) up_vertex<LdGen>(u, i, j);
    }
    if (l < a.ltop || a.nhang) grid_barrier(a.bar, nb, gen);
    stamp();
  }
  for (int q = 0; q < a.nhang; ++q) {  // hanging refresh, coarse to fine (solvers.py:292-296)
    const int li = a.hang_lv[q];
    const HangArgs& hg = a.hang[li];
    const int th = a.tile_h[li], nu = a.units[li];
    const uint32_t* tiles = a.up[li].tiles;
    for (int w = gw; w < nu; w += nw) {
      int i, j;
      unit_vertex(tiles, th, hg.N, w, lane, i, j);
      if (i < hg.N && j < hg.N) {
        const size_t v = (size_t)i * hg.N + j;
        if ((hg.flags[v] & 7) == K_HANG) hg.u[v] = prolong_dlinear_at<LdGen>(hg.uc, hg.Nc, i, j);
      }
    }
    if (q + 1 < a.nhang) grid_barrier(a.bar, nb, gen);
    stamp();
  }
}

// FAS injection (solvers.py:283-288), standalone update_fas_state()
__global__ void k_inject_u(double* __restrict__ uc, const uint8_t* __restrict__ flags_c, int Nc,
                           const double* __restrict__ uf, int Nf) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (size_t)Nc * Nc) return;
  if (!(flags_c[v] & F_TAKE)) return;
  const int i = (int)(v / Nc), j = (int)(v % Nc);
  uc[v] = uf[(size_t)(3 * i) * Nf + 3 * j];
}

// hanging refresh (solvers.py:292-296)
__global__ void k_hang(double* __restrict__ u, const uint8_t* __restrict__ flags, int N,
                       const double* __restrict__ uc, int Nc) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (size_t)N * N) return;
  if ((flags[v] & 7) != K_HANG) return;
  const int i = (int)(v / N), j = (int)(v % N);
  u[v] = prolong_dlinear_at<LdNC>(uc, Nc, i, j);
}

void upload_constants(cudaStream_t s) {
  const double E[16] = {2.0 / 3.0,  -1.0 / 6.0, -1.0 / 6.0, -1.0 / 3.0, -1.0 / 6.0, 2.0 / 3.0,
                        -1.0 / 3.0, -1.0 / 6.0, -1.0 / 6.0, -1.0 / 3.0, 2.0 / 3.0,  -1.0 / 6.0,
                        -1.0 / 3.0, -1.0 / 6.0, -1.0 / 6.0, 2.0 / 3.0};
  const double W5[5] = {1.0 / 3.0, 2.0 / 3.0, 3.0 / 3.0, 2.0 / 3.0, 1.0 / 3.0};
  double WL[3], WR[3];
  for (int r = 0; r < 3; ++r) {
    volatile double third = (double)r / 3.0;  // numpy: 1.0 - r/3.0 on a float array
    WL[r] = 1.0 - third;
    WR[r] = 1.0 - WL[r];
  }
  const double c1 = 1.0 / 3.0;
  const double side = c1 * -1.0, mid = c1 * 8.0, inv = 3.0 / 8.0;
  double A1[9];
  for (int k = 0; k < 9; ++k) A1[k] = (k == 4 ? mid : side) * inv;
  cudaMemcpyToSymbolAsync(c_E, E, sizeof(E), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_W5, W5, sizeof(W5), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_WL, WL, sizeof(WL), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_WR, WR, sizeof(WR), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_A1INV, A1, sizeof(A1), 0, cudaMemcpyHostToDevice, s);
}

}  // namespace tmg
