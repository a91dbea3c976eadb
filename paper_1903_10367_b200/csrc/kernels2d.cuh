// Kernel argument blocks and declarations of the 2D engine.
#pragma once

#include "tmg_kernels.cuh"

namespace tmg {

constexpr int kTileX = 32, kTileY = 8;
constexpr int kBlock = kTileX * kTileY;  // grid kernels
constexpr int kCoarseBlock = 256;  // the coarse-chain kernel (one block)
constexpr int kMaxLevels = 16;

enum Variant : int {
  VAR_ADDITIVE = 0,
  VAR_EXP = 1,
  VAR_BPX = 2,
  VAR_AFACC = 3,
  VAR_PI = 4,
  VAR_JAC = 5,
  VAR_V10 = 6
};

// One level of the fine -> coarse sweep (solvers.py:345-375).
struct DownArgs {
  int N, is_top, variant, write;
  const double* u;
  const uint8_t* flags;
  const double* diag;  // where(dof, op.diag(), 1)
  OpView op;           // ops[l]
  OpView rop;          // refined_ops[l] (OP_NONE when absent)
  const double* rhs;   // engine.rhs[l] or nullptr
  // finer level (restriction sources), valid when !is_top
  int Nf;
  const double* rho_f;
  const double* rdof_f;
  int boxmg;
  const double* P;   // transfers[l] P planes (boxmg)
  const double* Rt;  // transfers[l] R~ planes (RT_TABLE)
  int rt_mode;
  double rt_side, rt_mid, rt_scale, rt_omega;
  // update parameters
  double w_l, omega, wt, ds;
  double hA, hB;  // hweight next to / away from refined cells
  // outputs
  double* rho;
  double* rdof;
  double* g;
  double* part_sum;
  double* part_max;
  // adaptive levels: the level's patch list -- the (32 x tile height) vertex tiles that hold at
  // least one existing vertex, packed (tile row << 16 | tile column); nullptr = every tile
  const uint32_t* tiles;
};

// One level of the coarse -> fine carry (solvers.py:386-395) with the
// adafac-pi damping (solvers.py:377-384) and the FAS injection of the new
// values into every coarser level that takes them (solvers.py:283-288).
struct UpArgs {
  int l, l0, N, is_bottom, boxmg, pi;
  const uint8_t* flags;
  double* u;
  const double* g;  // d - dtil (jac) / d (pi: dtil formed here)
  double* carry;
  int Nc;
  const double* carry_c;
  const double* P;         // transfers[l-1] P planes (boxmg)
  const uint8_t* flags_c;  // level l-1 flags (F_TAKE for adafac-pi injection)
  double ds;
  // injection targets by level (levels l0 .. l-1)
  double* ul[kMaxLevels];
  const uint8_t* fl[kMaxLevels];
  int Nl[kMaxLevels];
  const uint32_t* tiles;  // the level's patch list (see DownArgs), or nullptr
};

// The coarse chain [l0, lc] (at most kMaxChain levels) in one block: down
// sweep lc -> l0, stats finalisation, up sweep l0 -> lc.  The per-level
// argument blocks travel by value in the kernel's parameter space.
constexpr int kMaxChain = 6;
struct CoarseArgs {
  int l0, lc;
  const double* part_sum;  // partials of the grid-level down kernels
  const double* part_max;
  int part_base;
  double* hist;
  int* counter;
  int cap;
  int do_up;
  unsigned long long* stamps;  // optional per-phase %globaltimer stamps (diagnostics)
  DownArgs down[kMaxChain];    // index l - l0
  UpArgs up[kMaxChain];
};

// The whole additive cycle in ONE persistent launch (north star: "one fused kernel launch per
// additive cycle that updates all levels"; the sweep order is pipeline.py:242-386's / solvers.py:
// 345-395's): every level's down sweep, the stats finalisation, every level's carry + update + FAS
// injection and the hanging-vertex refresh, separated by grid-wide barriers.  A unit of work is one
// warp row (32 consecutive vertices of a vertex row: of the dense array, or of a patch-list tile).
constexpr int kCycleLevels = 10;
constexpr int kCycleWarps = kBlock / 32;
struct HangArgs {
  double* u;
  const uint8_t* flags;
  int N, Nc;
  const double* uc;
};
struct CycleArgs {
  int l0, ltop, do_up, nhang;
  double* hist;
  int* counter;
  int cap;
  double* wpart;       // one (sum, max) pair per warp of the grid
  unsigned* bar;       // grid barrier: {arrival count, generation}
  unsigned long long* stamps;  // optional %globaltimer stamp per phase (CTA 0; diagnostics)
  int units[kCycleLevels];   // warp rows per level (index l - l0)
  int tile_h[kCycleLevels];  // rows per patch-list tile (levels with a list)
  int hang_lv[kCycleLevels]; // levels with hanging vertices, ascending (index l - l0)
  DownArgs down[kCycleLevels];
  UpArgs up[kCycleLevels];
  HangArgs hang[kCycleLevels];
};

__global__ void k_flags(uint8_t* flags, int n, const uint8_t* ref_prev, const uint8_t* ref_cur);
__global__ void k_take(uint8_t* flags_c, int Nc, const uint8_t* flags_f, int Nf);
__global__ void k_eff(double* eff, double* epsm, double* reff, const double* eps,
                      const double* eff_child, const uint8_t* ref_cur, const uint8_t* ref_prev, int n);
__global__ void k_const_check(const double* arr, size_t n, int* flag);
__global__ void k_count_kinds(const uint8_t* flags, size_t nv, unsigned long long* counts);
__global__ void k_elem_diag(double* raw, double* diag, const double* eps, const uint8_t* flags, int n);
__global__ void k_table_diag(double* raw, double* diag, const double* tbl, const uint8_t* flags,
                             size_t nv);
__global__ void k_assemble(double* tbl, const double* eps, int n);
__global__ void k_gamma_x(double* ex, const double* tf, int nc, const uint8_t* ref,
                          const uint8_t* ref_prev, int* deg);
__global__ void k_gamma_y(double* ey, const double* tf, int nc, const uint8_t* ref,
                          const uint8_t* ref_prev, int* deg);
__global__ void k_p_init(double* P, int nc, const double* ex, const double* ey);
__global__ void k_p_interior(double* P, int nc, const double* tf, const double* ex, const double* ey,
                             const uint8_t* ref, const uint8_t* ref_prev);
__global__ void k_p_fix(double* P, int nc, const uint8_t* flags_f);
__global__ void k_rap(double* tbl, const uint8_t* flags_c, int nc, const double* tf,
                      const uint8_t* flags_f, const double* P);
__global__ void k_rtilde(double* Rt, int nc, const double* P, int pconst, const double* tf,
                         const uint8_t* flags_f, const double* diag_f, double omega);
template <int TOP>
__global__ void k_down(const __grid_constant__ DownArgs a);
__global__ void k_up(const __grid_constant__ UpArgs a);
__global__ void k_coarse(const __grid_constant__ CoarseArgs a);
__global__ void k_coarse_cl(const __grid_constant__ CoarseArgs a, double* scratch);
__global__ void k_cycle(const __grid_constant__ CycleArgs a);
__global__ void k_inject_u(double* uc, const uint8_t* flags_c, int Nc, const double* uf, int Nf);
__global__ void k_hang(double* u, const uint8_t* flags, int N, const double* uc, int Nc);

void upload_constants(cudaStream_t s);

}  // namespace tmg
