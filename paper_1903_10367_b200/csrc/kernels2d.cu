// 2D kernels: operator setup (classification, eff_eps, stencils, BoxMG P,
// Galerkin rows, smoothed restriction) and the additive cycle.
//
// Thread-per-vertex kernels over dense per-level grids.  Each one evaluates
// exactly the reference's per-element expression DAG (see tmg_kernels.cuh);
// the file is compiled with --fmad=false.
#include "kernels2d.cuh"

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
  if (c >= n) return;
  const double first = arr[0];
  if (!(first > 0.0) || arr[c] != first) atomicAnd(flag, 0);
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

template <int BS>
__device__ __forceinline__ void block_reduce_store(double s, double m, double* part_sum,
                                                   double* part_max) {
  __shared__ double ss[BS / 32], sm[BS / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { ss[w] = s; sm[w] = m; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < BS / 32; ++k) { a += ss[k]; b = fmax(b, sm[k]); }
    part_sum[blockIdx.x] = a;
    part_max[blockIdx.x] = b;
  }
}

// One level of the fine -> coarse sweep of advance() (solvers.py:345-375):
// coarse right-hand side from the finer residual (R rho + rhs + bpart),
// residual, stats, damped Jacobi and the adaFACx damping term.
__global__ void __launch_bounds__(kBlock) k_down(DownArgs a) {
  const size_t nv = (size_t)a.N * a.N;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0, m = 0.0;
  if (v < nv) {
    const int i = (int)(v / a.N), j = (int)(v % a.N);
    const uint8_t f = a.flags[v];
    const int kind = f & 7;
    const double au = apply_op_at(a.op, a.u, a.N, i, j);
    double b;
    if (a.is_top) {
      b = a.rhs ? a.rhs[v] : 0.0;
    } else {
      b = a.boxmg ? restrict_table_at(a.rho_f, a.Nf, a.P, a.N, i, j)
                  : restrict_dlinear_at(a.rho_f, a.Nf, i, j);
      if (a.rhs) b = b + a.rhs[v];
      if (a.rop.kind != OP_NONE) {
        const double bp = (kind == K_OVER) ? au : apply_op_at(a.rop, a.u, a.N, i, j);
        b = b + bp;
      }
    }
    const double rho = is_src(f) ? b - au : 0.0;
    const double rd = is_dof(f) ? rho : 0.0;
    if (kind == K_DOF) {
      const double h = (f & F_NEAR) ? a.hA : a.hB;
      const double t = h * rd;
      s = t * t;
      m = fabs(rd);
    }
    if (a.write) {
      double d;
      if (a.variant == VAR_BPX && !a.is_top) d = a.omega * rd;
      else d = (a.w_l * rd) / a.diag[v];
      if (a.variant == VAR_JAC && !a.is_top) {
        const double bt = (a.rt_mode == RT_GEOM_FAST)
                              ? restrict_rt_geom_at(a.rdof_f, a.Nf, i, j, a.rt_side, a.rt_mid, a.rt_scale)
                              : restrict_rt_table_at(a.rdof_f, a.Nf, a.Rt, a.N, i, j);
        const double dt = is_dof(f) ? a.ds * ((a.wt * bt) / a.diag[v]) : 0.0;
        d = d - dt;
      }
      a.g[v] = d;
    }
    if (a.rho) {
      const bool cpt = (i % 3 == 0) && (j % 3 == 0);
      a.rho[v] = (a.variant == VAR_AFACC && cpt) ? 0.0 : rho;
    }
    if (a.rdof) a.rdof[v] = rd;
  }
  block_reduce_store<kBlock>(s, m, a.part_sum, a.part_max);
}

// inj = d_l at taken c-points, 0 elsewhere (adafac-pi, solvers.py:377-382)
__global__ void k_inject_d(double* __restrict__ inj, const uint8_t* __restrict__ flags_c, int Nc,
                           const double* __restrict__ d, int Nf) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (size_t)Nc * Nc) return;
  const int i = (int)(v / Nc), j = (int)(v % Nc);
  inj[v] = (flags_c[v] & F_TAKE) ? d[(size_t)(3 * i) * Nf + 3 * j] : 0.0;
}

// One level of the coarse -> fine carry (solvers.py:386-395), including the
// adafac-pi damping (solvers.py:377-384).
__global__ void __launch_bounds__(kBlock) k_up(UpArgs a) {
  const size_t nv = (size_t)a.N * a.N;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int i = (int)(v / a.N), j = (int)(v % a.N);
  const uint8_t f = a.flags[v];
  double g = a.g[v];
  if (a.inj) {
    const double pv = a.boxmg ? prolong_table_at(a.inj, a.P, a.Nc, i, j)
                              : prolong_dlinear_at(a.inj, a.Nc, i, j);
    const double dt = is_dof(f) ? a.ds * pv : 0.0;
    g = g - dt;
  }
  double c = g;
  if (!a.is_bottom) {
    const double pc = a.boxmg ? prolong_table_at(a.carry_c, a.P, a.Nc, i, j)
                              : prolong_dlinear_at(a.carry_c, a.Nc, i, j);
    c = pc + g;
  }
  if ((f & 7) == K_NONE) c = 0.0;
  if (a.carry) a.carry[v] = c;
  a.u[v] = a.u[v] + c;
}

// FAS injection (solvers.py:283-288)
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
  u[v] = prolong_dlinear_at(uc, Nc, i, j);
}

// deterministic final reduction of the per-block partials -> history slot
__global__ void k_finalize(const double* __restrict__ part_sum, const double* __restrict__ part_max,
                           int nparts, double* __restrict__ hist, int* __restrict__ counter, int cap) {
  __shared__ double ss[256], sm[256];
  double s = 0.0, m = 0.0;
  for (int k = threadIdx.x; k < nparts; k += 256) { s += part_sum[k]; m = fmax(m, part_max[k]); }
  ss[threadIdx.x] = s;
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      ss[threadIdx.x] += ss[threadIdx.x + w];
      sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int slot = *counter;
    hist[2 * (slot % cap)] = sqrt(ss[0]);
    hist[2 * (slot % cap) + 1] = sm[0];
    *counter = slot + 1;
  }
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
