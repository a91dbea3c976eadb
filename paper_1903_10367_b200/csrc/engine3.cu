// Host runtime of the 3D engine (regular spacetrees): level hierarchy in
// HBM, operator setup, the per-cycle launch sequence captured in a CUDA
// graph.  Reached through the C ABI of engine.cu (tmg3_create and the
// dimension-dispatching tmg_* entry points).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "engine3.h"
#include "kernels3d.cu"
#include "kernels3d_fast.cu"
#include "kernels3d_upq.cu"
#include "kernels3d_smr.cu"
#include "kernels3d_top4r.cu"
#include "kernels3d_updict.cu"
#include "kernels3d_smc.cu"
#include "kernels3d_dict.cu"
#include "kernels3d_rap.cu"
#include "kernels3d_uplin.cu"
#include "kernels3d_rle.cu"

namespace {

using namespace t3;

struct Lvl3 {
  int l = 0, N = 0;
  size_t nv = 0, ncell = 0;
  double *u = nullptr, *rhs = nullptr, *g = nullptr, *rho = nullptr, *sm = nullptr, *carry = nullptr;
  double *eff = nullptr, *coef = nullptr, *tbl = nullptr, *P = nullptr;
  double* Pc = nullptr;  // levels ltop-1, ltop-2: cube-owned copy of P for the TMA-fed prolongation (k3_up_tma)
  // level ltop-1: row dictionaries of P (k3_smr) and Pc (k3_up_tma), kernels3d_dict.cu; null = dense
  double *Pd = nullptr, *Pcd = nullptr;
  uint32_t *Pdi = nullptr, *Pcdi = nullptr;
  uint8_t* Ptab = nullptr;  // k3_up_tma step tables over Pc's dictionary
  double* Pds = nullptr;     // P's dictionary in fine-plane slices (k3_smc)
  uint8_t* Pctab = nullptr;  // k3_smc tile-plane tables (31 x 4 vertex tiles)
  double* Td = nullptr;      // level ltop-1: the Galerkin rows as a row dictionary (op.tdict)
  uint32_t* Tdi = nullptr;
  size_t Tdn = 0;
  size_t Pdp = 0, Pdn = 0, Pcdp = 0, Pcdn = 0;
  double* coefp = nullptr;  // finest level: coef with rows padded to even length (TMA)
  int crun = 1;             // ... storing one plane per run of crun equal cell planes (blockwise materials)
  double *bR = nullptr, *bT = nullptr;  // level ltop-1: restrictions from the fused fine pass
  Op3 op{};
  double w = 0.0;
  int grid = 0, part_off = 0;
  int s_chunk = 0, s_blocks = 0;  // 2.5D tiling (k3_top / k3_smooth_s)
  int s2_chunk = 0, s2_blocks = 0;  // two-row 2.5D tiling (k3_top2 / k3_smooth2)
  int c_grid = 0;                 // k3_down_c grid
  int u_grid = 0;                 // k3_up_cell grid (this level as the coarse one)
};

struct KT {
  const char* name;
  float ms;
  int launches;
};

constexpr int kResident = 148 * 8;  // grid-stride kernels: 8 CTAs per SM

inline unsigned nblk(size_t n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

int ipow3(int l) {
  int r = 1;
  for (int k = 0; k < l; ++k) r *= 3;
  return r;
}

}  // namespace

struct Engine3 {
  tmg_config cfg{};
  double wt = 0.0;
  int lmin = 1, ltop = 1, lc = 1;
  std::vector<Lvl3> L;
  cudaStream_t s = nullptr;
  std::vector<void*> allocs;
  double *part_sum = nullptr, *part_max = nullptr;
  int nparts = 0;
  double* hist = nullptr;
  int* counter = nullptr;
  int cap = 1024;
  long long host_counter = 0;
  cudaGraphExec_t gexec = nullptr;
  bool graph_dirty = true;
  int launches = 0;
  long long dofs_total = 0, updates = 0;
  bool profiling = false;
  std::vector<KT>* timers = nullptr;
  struct Pending {
    const char* name;
    cudaEvent_t e0, e1;
  };
  std::vector<cudaEvent_t> ev_pool;
  int ev_used = 0;
  std::vector<Pending> pending;
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  std::string* err = nullptr;
  // sharded (multi-GPU slab) mode: levels >= ls restricted to owned vertex planes
  bool sharded = false;
  int ls = 0;
  std::vector<int> own_lo, own_hi;  // by level
  std::vector<int> own_blocks;      // k3_top / k3_smooth_s blocks for the owned range
  std::vector<int> own_chunk;
  std::vector<int> own_blocks2, own_chunk2;  // two-row kernels (k3_top2 / k3_smooth2r)
  double* red = nullptr;            // {sum, max} of this cycle's stats
  int top_parts = 0;
  // tmg3_phase_range: the part of the owned planes the current phase call works on
  int rng_lo = 0, rng_hi = 1 << 30;
  bool rng_first = true, rng_last = true;
  // finest level double buffered (pp): the down sweep writes u + g of the finest level into
  // the other buffer (g never reaches HBM) and the up sweep adds P carry there; ubuf[par]
  // holds the current iterate, one captured graph per parity
  bool pp = false;
  int par = 0;
  double* ubuf[2] = {nullptr, nullptr};
  std::map<int, cudaGraphExec_t> gcache;
  bool smr = false;   // smoothing fused with the restriction into the next level (k3_smr)
  int smr_lo = 0;     // ... for the levels smr_lo..ltop
  // throttled BoxMG setup: next level to receive BoxMG P + Galerkin rows (< lmin: done)
  int thr_next = -1;
  int* deg = nullptr;
};

namespace {

int fail3(Engine3* e, int code, const std::string& msg) {
  if (e && e->err) *e->err = msg;
  return code;
}

#define CK3(call)                                                                         \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail3(e, TMG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

#define CKL3()                                                                            \
  do {                                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      return fail3(e, TMG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define TRY3(expr)                 \
  do {                             \
    int rc_ = (expr);              \
    if (rc_ != TMG_OK) return rc_; \
  } while (0)

template <class T>
int alloc3(Engine3* e, T** p, size_t count, bool zero = true) {
  void* q = nullptr;
  CK3(cudaMalloc(&q, sizeof(T) * (count ? count : 1)));
  e->allocs.push_back(q);
  if (zero) CK3(cudaMemsetAsync(q, 0, sizeof(T) * (count ? count : 1), e->s));
  *p = (T*)q;
  return TMG_OK;
}

void free3(Engine3* e) {
  if (e->gexec && e->gcache.empty()) cudaGraphExecDestroy(e->gexec);
  e->gexec = nullptr;
  for (auto& kv : e->gcache) cudaGraphExecDestroy(kv.second);
  e->gcache.clear();
  e->pp = false;
  e->par = 0;
  e->ubuf[0] = e->ubuf[1] = nullptr;
  for (void* p : e->allocs) cudaFree(p);
  e->allocs.clear();
  e->L.clear();
  // buffers from e3_shard were in allocs: a rebuilt handle is unsharded until tmg3_shard runs again
  e->red = nullptr;
  e->part_sum = e->part_max = nullptr;
  e->nparts = 0;
  e->sharded = false;
  e->ls = 0;
  e->own_lo.clear();
  e->own_hi.clear();
  e->own_blocks.clear();
  e->own_chunk.clear();
  e->own_blocks2.clear();
  e->own_chunk2.clear();
  e->graph_dirty = true;
}

// --- per-launch timing (profile path, no graph) ---------------------------------

int begin_k(Engine3* e, cudaEvent_t* e0) {
  if (!e->profiling) return TMG_OK;
  if (e->ev_used + 2 > (int)e->ev_pool.size())
    for (int k = 0; k < 256; ++k) {
      cudaEvent_t q;
      CK3(cudaEventCreate(&q));
      e->ev_pool.push_back(q);
    }
  *e0 = e->ev_pool[e->ev_used++];
  CK3(cudaEventRecord(*e0, e->s));
  return TMG_OK;
}

int end_k(Engine3* e, const char* name, cudaEvent_t e0) {
  e->launches++;
  if (!e->profiling) return TMG_OK;
  cudaEvent_t e1 = e->ev_pool[e->ev_used++];
  CK3(cudaEventRecord(e1, e->s));
  e->pending.push_back({name, e0, e1});
  return TMG_OK;
}

const char* kname(const char* base, int l) {
  static char names[4][12][24];
  static const char* bases[4] = {"k3_down", "k3_smooth", "k3_up", "k3_chain"};
  int b = 0;
  while (b < 4 && std::strcmp(bases[b], base) != 0) ++b;
  if (b >= 4 || l < 0 || l > 11) return base;
  if (!names[b][l][0]) std::snprintf(names[b][l], 24, "%s_L%d", base, l);
  return names[b][l];
}

#define LAUNCH3(name, kernel, grid, block, ...)         \
  do {                                                  \
    cudaEvent_t e0_ = nullptr;                          \
    TRY3(begin_k(e, &e0_));                             \
    kernel<<<(grid), (block), 0, e->s>>>(__VA_ARGS__);  \
    CKL3();                                             \
    TRY3(end_k(e, name, e0_));                          \
  } while (0)

// --- argument blocks ---------------------------------------------------------------

int grid_for(int N, int ilo, int ihi) {
  const long long t = (long long)((N - 2 + kTX - 1) / kTX) * ((N - 2 + kTY - 1) / kTY) *
                      ((ihi - ilo + kTZ - 1) / kTZ);
  return (int)std::max(1LL, std::min<long long>(t, kResident));
}

Down3 make_down(Engine3* e, int l, bool write) {
  const int l0 = e->lmin, l1 = e->ltop;
  Lvl3& c = e->L[l];
  Down3 a{};
  a.N = c.N;
  a.l = l;
  a.is_top = l == l1;
  a.variant = e->cfg.variant;
  a.write = write ? 1 : 0;
  a.ilo = 1;
  a.ihi = c.N - 1;
  a.u = c.u;
  a.rhs = c.rhs;
  a.op = c.op;
  if (l < l1) {
    Lvl3& f = e->L[l + 1];
    a.Nf = f.N;
    a.rho_f = f.rho;
    a.sm_f = f.sm;
    a.P = c.P;
  }
  a.w = c.w;
  a.omega = e->cfg.omega;
  a.wt = e->wt;
  a.ds = e->cfg.damping_scale;
  a.hw = std::pow(3.0, -1.5 * l);
  a.rho = (l > l0) ? c.rho : nullptr;
  a.g = c.g;
  a.part_sum = nullptr;  // grid partials come from k3_top only
  a.part_max = nullptr;
  return a;
}

Smooth3 make_smooth(Engine3* e, int l) {
  Lvl3& c = e->L[l];
  Smooth3 a{};
  a.N = c.N;
  a.ilo = 1;
  a.ihi = c.N - 1;
  a.x = c.rho;
  a.sm = c.sm;
  a.scale = e->cfg.omega * 3.0 / 8.0;  // operators.py:603-605
  return a;
}

Up3 make_up(Engine3* e, int l) {
  const int l0 = e->lmin, l1 = e->ltop;
  Lvl3& c = e->L[l];
  Up3 a{};
  a.N = c.N;
  a.l = l;
  a.l0 = l0;
  a.is_bottom = l == l0;
  a.pi = e->cfg.variant == VAR_PI;
  a.ilo = 1;
  a.ihi = c.N - 1;
  a.u = c.u;
  a.g = c.g;
  if (l == l1 && e->pp) {  // the down sweep wrote u + g into the other buffer
    a.u = e->ubuf[e->par ^ 1];
    a.g = nullptr;
  }
  a.carry = (l < l1) ? c.carry : nullptr;
  if (l > l0) {
    Lvl3& cc = e->L[l - 1];
    a.Nc = cc.N;
    a.carry_c = cc.carry;
    a.P = cc.P;
  }
  a.ds = e->cfg.damping_scale;
  for (int k = l0; k < l; ++k) {
    a.ul[k] = e->L[k].u;
    a.Nl[k] = e->L[k].N;
  }
  return a;
}

// 3D tensor map of an N^3 fp64 vertex field for the TMA-staged 2.5D kernels:
// box = one halo plane of a 32 x 16 column (34 x 18 doubles), zero fill
// outside the grid (the stencils' zero extension).  false if the driver
// entry point is unavailable (the kernels then stage with cp.async).
bool vertex_tmap(CUtensorMap* map, const double* base, int N) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode || !base) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)N};
  const cuuint64_t strides[2] = {(cuuint64_t)N * 8, (cuuint64_t)N * N * 8};
  const cuuint32_t box[3] = {(cuuint32_t)k2RowU, (cuuint32_t)k2ColU, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The same for the finest level's cell coefficients, stored with rows padded
// to an even length (coefp) so that TMA can stride them.
bool cell_tmap(CUtensorMap* map, const double* base, int n, int planes) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode || !base) return false;
  const cuuint64_t np = (cuuint64_t)(n + (n & 1));  // padded row length
  const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {np * 8, np * n * 8};
  const cuuint32_t box[3] = {(cuuint32_t)k2RowC, (cuuint32_t)k2ColC, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Generic 3D tensor map over fp64 data (dims innermost first, byte strides of dims 1, 2).
bool tmap3(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
           uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2,
           CUtensorMapL2promotion prom = CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT64) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode || !base) return false;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {s1, s2};
  const cuuint32_t box[3] = {b0, b1, b2};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA staging of the streaming kernels' vertex planes (cp.async when the driver entry point of
// the tensor-map encoder is missing)
constexpr bool kUseTma = true;

bool tmap4(CUtensorMap* map, const double* base, const uint64_t d[4], const uint64_t s[3], const uint32_t b[4]) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode || !base) return false;
  const cuuint64_t dims[4] = {d[0], d[1], d[2], d[3]};
  const cuuint64_t strides[3] = {s[0], s[1], s[2]};
  const cuuint32_t box[4] = {b[0], b[1], b[2], b[3]};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// SM count of the current device (the ABI's DeviceGuard makes it the handle's)
int num_sms() {
  static int cache[64] = {0};
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return v;
  if (!cache[dev] && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) cache[dev] = v;
  return cache[dev] ? cache[dev] : v;
}

int launch_up_tma(Engine3* e, int l, const Up3& a) {
  const Lvl3& cc = e->L[l - 1];
  UpQ A{};
  A.a = a;
  const uint64_t N = (uint64_t)a.N, Nc = (uint64_t)a.Nc;
  const uint64_t nc_ = Nc - 1, Kp = (nc_ + kQK - 1) / kQK * kQK;
  const uint64_t dp[4] = {nc_, nc_, nc_, (uint64_t)kQS}, sp[3] = {Kp * 8, Kp * nc_ * 8, Kp * nc_ * nc_ * 8};
  const uint32_t bp[4] = {kQK, kQJ, 1, kQS};
  bool ok = tmap4(&A.tp, cc.Pc, dp, sp, bp);
  ok = ok && tmap3(&A.tu, a.u, N, N, N, N * 8, N * N * 8, kQFK, kQFJ, 3, CU_TENSOR_MAP_L2_PROMOTION_NONE);
  if (a.g) ok = ok && tmap3(&A.tg, a.g, N, N, N, N * 8, N * N * 8, kQFK, kQFJ, 3, CU_TENSOR_MAP_L2_PROMOTION_NONE);
  ok = ok && tmap3(&A.tc, a.carry_c, Nc, Nc, Nc, Nc * 8, Nc * Nc * 8, kQCK, kQCJ, 2);
  if (!ok) return fail3(e, TMG_ECUDA, "tensor map encoding failed (k3_up_tma)");
  const int nc = a.Nc - 1;
  A.tilesK = (nc + kQK - 1) / kQK;
  A.I0 = a.ilo / 3;
  A.nI = std::max(0, std::min(nc, (a.ihi + 2) / 3) - A.I0);
  if (A.nI == 0) return TMG_OK;
  A.steps = (long long)A.tilesK * ((nc + kQJ - 1) / kQJ) * A.nI;
  const int grid = (int)std::min<long long>(num_sms(), A.steps);
  A.per = (A.steps + grid - 1) / grid;
  cudaEvent_t e0_ = nullptr;
  TRY3(begin_k(e, &e0_));
  if (cc.Pcd) {  // weights from the row dictionary (k3_up_dict)
    UpD D{};
    D.tu = A.tu;
    D.tg = A.tg;
    D.tc = A.tc;
    D.a = a;
    D.dict = cc.Pcd;
    D.tab = cc.Ptab;
    D.tilesK = A.tilesK;
    D.tilesJ = (int)((nc_ + kQJ - 1) / kQJ);
    D.nI = A.nI;
    D.I0 = A.I0;
    D.steps = (int)A.steps;
    D.per = (int)A.per;
    D.snake = (D.nI % kDSnake == 0) ? 1 : 0;  // (a compile-time flavour of the kernel: as a run-time branch
                                              // it pushes the step coordinates out of the uniform registers)
    if (!a.g && D.snake) k3_up_dict<false, false, true><<<grid, kDThreads, DLay<false>::smem, e->s>>>(D);
    else if (!a.g) k3_up_dict<false, false><<<grid, kDThreads, DLay<false>::smem, e->s>>>(D);
    else if (a.carry) k3_up_dict<true><<<grid, kDThreads, DLay<true>::smem, e->s>>>(D);
    else k3_up_dict<false><<<grid, kDThreads, DLay<true>::smem, e->s>>>(D);
  } else {
    if (!a.g) k3_up_tma<false, false><<<grid, kQT, kUpTmaSmem, e->s>>>(A);
    else if (a.carry) k3_up_tma<true><<<grid, kQT, kUpTmaSmem, e->s>>>(A);
    else k3_up_tma<false><<<grid, kQT, kUpTmaSmem, e->s>>>(A);
  }
  CKL3();
  TRY3(end_k(e, kname("k3_up", l), e0_));
  return TMG_OK;
}

int launch_up_boxmg(Engine3* e, int l, const Up3& a) {
  if (e->L[l - 1].Pc && !a.pi) return launch_up_tma(e, l, a);
  // small levels (< 32 coarse cells per axis): the cell-owned kernel has 9x the threads of the
  // tiled one, which is latency-bound there (config 5: up L3 55 -> 17 us, L4 79 -> 20 us)
  if (a.Nc - 1 < kUX) {
    LAUNCH3(kname("k3_up", l), k3_up_cell<true>, e->L[l - 1].u_grid, 128, a);
    return TMG_OK;
  }
  const int nc = a.Nc - 1;
  const int tiles = ((nc + kUX - 1) / kUX) * ((nc + kUY - 1) / kUY);
  const int Ilo = a.ilo / 3, Ihi = std::min(nc, (a.ihi + 2) / 3);
  const int planes = std::max(1, Ihi - Ilo);
  const int nch = std::max(1, std::min((148 * 16 + tiles - 1) / tiles, std::max(1, planes / 2)));
  const int chunk = (planes + nch - 1) / nch;
  const dim3 grid(tiles, (planes + chunk - 1) / chunk);
  LAUNCH3(kname("k3_up", l), k3_up_tile, grid, dim3(kUX, kUY), a, chunk);
  return TMG_OK;
}

// d-linear prolongation into level l (k3_up_lin): units = (cube layer, cube row, 32-cube K tile)
int launch_up_lin(Engine3* e, int l, const Up3& a) {
  UpL A{};
  A.a = a;
  const int nc = a.Nc - 1;
  A.tilesK = (nc + 31) / 32;
  A.I0 = a.ilo / 3;
  A.nI = std::max(0, std::min(nc, (a.ihi + 2) / 3) - A.I0);
  if (A.nI == 0) return TMG_OK;
  A.units = (long long)A.nI * nc * A.tilesK;
  const int grid = (int)std::min<long long>(A.units, (long long)num_sms() * 7 * 8);
  LAUNCH3(kname("k3_up", l), k3_up_lin, grid, kLThreads, A);
  return TMG_OK;
}

// element operator with every plane through TMA: the register-window kernel k3_top4r (else k3_top2)
bool use_top4(const Top3& a) { return a.use_tma == 2 && a.rhs_tma; }
Top3 make_top(Engine3* e, int l) {
  Lvl3& c = e->L[l];
  Top3 a{};
  a.N = c.N;
  a.ilo = 1;
  a.ihi = c.N - 1;
  a.chunk = c.s_chunk;
  a.u = c.u;
  a.rhs = c.rhs;
  a.op = c.op;
  a.w = c.w;
  a.hw = std::pow(3.0, -1.5 * l);
  a.g = c.g;
  a.u_out = (l == e->ltop && e->pp) ? e->ubuf[e->par ^ 1] : nullptr;
  a.rho = (l > e->lmin) ? c.rho : nullptr;
  a.part_sum = e->part_sum;
  a.part_max = e->part_max;
  a.use_tma = kUseTma && vertex_tmap(&a.tm, c.u, c.N);
  a.crun = c.crun;
  if (a.use_tma && c.op.kind == OP_ELEMENT && c.coefp &&
      cell_tmap(&a.tmc, c.coefp, c.N - 1, (c.N - 1 + c.crun - 1) / c.crun))
    a.use_tma = 2;
  // rhs through TMA as well; needs the vertex-plane TMA path
  a.rhs_tma = a.use_tma && c.rhs &&
              tmap3(&a.tmr, c.rhs, c.N, c.N, c.N, (uint64_t)c.N * 8, (uint64_t)c.N * c.N * 8, k2RowR, k2Y, 1);
  return a;
}

SmoothS make_smooth_s(Engine3* e, int l) {
  Lvl3& c = e->L[l];
  SmoothS a{};
  a.N = c.N;
  a.ilo = 1;
  a.ihi = c.N - 1;
  a.chunk = c.s_chunk;
  a.x = c.rho;
  a.sm = c.sm;
  a.scale = e->cfg.omega * 3.0 / 8.0;
  a.use_tma = kUseTma && vertex_tmap(&a.tm, c.rho, c.N);
  return a;
}

// the cell-owned kernel's inputs for level l as the coarse one: the sliced dictionary and the
// tile-plane tables (one_row: every vertex uses row 0, the d-linear flavour)
int build_smc(Engine3* e, int l, bool one_row) {
  Lvl3& c = e->L[l];
  c.Pds = nullptr;
  c.Pctab = nullptr;
  if (!c.Pd || c.Pdn == 0) return TMG_OK;
  const int n = c.N - 2, tK = (n + kCK - 1) / kCK, tJ = (n + kCJ - 1) / kCJ;
  const size_t cnt = (size_t)n * tJ * tK;
  uint8_t* tab = nullptr;
  TRY3(alloc3(e, &tab, cnt * kCTabBytes, false));
  if (one_row) {
    k3_smc_tables_one<<<nblk(cnt, 128), 128, 0, e->s>>>(tab, cnt);
    CKL3();
  } else {
    int* dover = nullptr;
    TRY3(alloc3(e, &dover, 1));
    const size_t Ncp = ((size_t)c.N + 3) / 4 * 4;
    k3_smc_tables<<<nblk(cnt, 128), 128, 0, e->s>>>(c.Pdi, c.N, (int)Ncp, tK, tJ, tab, dover);
    CKL3();
    int over = 0;
    CK3(cudaMemcpyAsync(&over, dover, sizeof(int), cudaMemcpyDeviceToHost, e->s));
    CK3(cudaStreamSynchronize(e->s));
    if (over) return TMG_OK;  // a tile plane meets too many rows: k3_smr's path
  }
  TRY3(alloc3(e, &c.Pds, c.Pdn * 5 * kCSl, false));
  k3_dict_slices<<<nblk(c.Pdn * 5 * kCSl, 256), 256, 0, e->s>>>(c.Pd, c.Pdn, c.Pds);
  CKL3();
  c.Pctab = tab;
  return TMG_OK;
}

int launch_smc(Engine3* e, int l, bool smooth, int clo, int chi) {
  Lvl3& c = e->L[l];
  Lvl3& cc = e->L[l - 1];
  Smc A{};
  A.N = c.N;
  A.Nc = cc.N;
  A.ilo = clo < 0 ? 1 : clo;
  A.ihi = chi < 0 ? cc.N - 1 : chi;
  const int n = A.ihi - A.ilo;
  if (n <= 0) return TMG_OK;
  const int nk = cc.N - 2;
  A.tilesK = (nk + kCK - 1) / kCK;
  A.tilesJ = (nk + kCJ - 1) / kCJ;
  const int tiles = A.tilesK * A.tilesJ;
  int best = 1;  // coarse-plane chunks: about a whole number of waves of kCPerSM CTAs per SM
  double best_eff = 0.0;
  for (int nch = 1; nch <= std::min(n, 32); ++nch) {
    const int chunk = (n + nch - 1) / nch, nb = tiles * ((n + chunk - 1) / chunk);
    const double waves = (double)nb / (kCPerSM * num_sms());
    const double eff = waves / std::ceil(waves) * (double)chunk / (chunk + 1.0);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = nch; }
  }
  A.chunk = (n + best - 1) / best;
  A.jac = smooth ? 1 : 0;
  A.zc = e->cfg.variant == VAR_AFACC ? 1 : 0;
  A.scale = e->cfg.omega * 3.0 / 8.0;
  A.bR = cc.bR;
  A.bT = cc.bT;
  A.pds = cc.Pds;
  A.ptab = cc.Pctab;
  const uint64_t N = (uint64_t)c.N;
  if (!tmap3(&A.tr, c.rho, N, N, N, N * 8, N * N * 8, kCW, kCH, 1))
    return fail3(e, TMG_ECUDA, "tensor map encoding failed (k3_smc)");
  const dim3 grid(tiles, (n + A.chunk - 1) / A.chunk);
  cudaEvent_t e0_ = nullptr;
  TRY3(begin_k(e, &e0_));
  if (smooth) k3_smc<true><<<grid, kCThreads, kSmcSmem, e->s>>>(A);
  else k3_smc<false><<<grid, kCThreads, kSmcSmem, e->s>>>(A);
  CKL3();
  TRY3(end_k(e, kname("k3_smooth", l), e0_));
  return TMG_OK;
}

// k3_smr over the finest level: adaFACx smoothing (when `smooth`) and the restriction of rho / sm
// into level ltop-1's bR / bT
// (sharded: the coarse planes [clo, chi) a rank owns; its rho must hold 3 planes below and 1 above
// the fine planes it owns)
int launch_smr(Engine3* e, int l, bool smooth, int clo = -1, int chi = -1) {
  Lvl3& c = e->L[l];
  Lvl3& cc = e->L[l - 1];
  if (cc.Pds) return launch_smc(e, l, smooth, clo, chi);  // P has a row dictionary: the cell-owned kernel
  Smr A{};
  A.N = c.N;
  A.Nc = cc.N;
  A.ilo = clo < 0 ? 1 : clo;
  A.ihi = chi < 0 ? cc.N - 1 : chi;
  const int n = A.ihi - A.ilo;  // coarse planes restricted into
  if (n <= 0) return TMG_OK;
  const int nk = cc.N - 2;  // interior coarse vertices along K and J
  A.tilesK = (nk + kRK - 1) / kRK;
  const int tiles = A.tilesK * ((nk + kRJ - 1) / kRJ);
  // coarse-plane chunks: about a whole number of waves of one CTA per SM
  int best = 1;
  double best_eff = 0.0;
  for (int nch = 1; nch <= std::min(n, 32); ++nch) {
    const int chunk = (n + nch - 1) / nch, nb = tiles * ((n + chunk - 1) / chunk);
    const double waves = (double)nb / num_sms();
    const double eff = waves / std::ceil(waves) * (double)chunk / (chunk + 1.0);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = nch; }
  }
  A.chunk = (n + best - 1) / best;
  A.jac = smooth ? 1 : 0;
  A.zc = e->cfg.variant == VAR_AFACC ? 1 : 0;
  A.scale = e->cfg.omega * 3.0 / 8.0;
  A.bR = cc.bR;
  A.bT = cc.bT;
  const uint64_t N = (uint64_t)c.N, Nc = (uint64_t)cc.N;
  const uint64_t dp[4] = {Nc, Nc, Nc, 125}, sp[3] = {Nc * 8, Nc * Nc * 8, Nc * Nc * Nc * 8};
  const uint32_t bp[4] = {kPW, kRJ, 1, 25};
  if (!tmap3(&A.tr, c.rho, N, N, N, N * 8, N * N * 8, kRW, kRH, 1) || !tmap4(&A.tp, cc.P, dp, sp, bp))
    return fail3(e, TMG_ECUDA, "tensor map encoding failed (k3_smr)");
  const dim3 grid(tiles, (n + A.chunk - 1) / A.chunk);
  cudaEvent_t e0_ = nullptr;
  TRY3(begin_k(e, &e0_));
  k3_smr<<<grid, kRThreads, kSmrSmem, e->s>>>(A);
  CKL3();
  TRY3(end_k(e, kname("k3_smooth", l), e0_));
  return TMG_OK;
}

int enqueue_down(Engine3* e, bool write) {
  const bool jac = e->cfg.variant == VAR_JAC;
  const bool boxmg = e->cfg.flavor == TMG_BOXMG;
  const dim3 sblk(kSX, kSY);
  for (int l = e->ltop; l > e->lc; --l) {
    Lvl3& c = e->L[l];
    if (l == e->ltop) {
      Top3 a = make_top(e, l);
      a.chunk = c.s2_chunk;
      cudaEvent_t e0_ = nullptr;
      TRY3(begin_k(e, &e0_));
      if (c.op.kind == OP_CONST && a.use_tma && a.rhs_tma)
        k3_top4c<<<c.s2_blocks, dim3(kSX, k2Y / kT4R), kTop4cSmem, e->s>>>(a);
      else if (c.op.kind == OP_CONST) k3_top2<OP_CONST><<<c.s2_blocks, dim3(kSX, k2Y / 2), k2TopSmem, e->s>>>(a);
      else if (use_top4(a)) k3_top4r<<<c.s2_blocks, dim3(kSX, k2Y / kT4R), kTop4rSmem, e->s>>>(a);
      else k3_top2<OP_ELEMENT><<<c.s2_blocks, dim3(kSX, k2Y / 2), k2TopSmem, e->s>>>(a);
      CKL3();
      TRY3(end_k(e, kname("k3_down", l), e0_));
    } else if (e->smr && l + 1 >= e->smr_lo) {  // restrictions formed by k3_smr of level l + 1
      Down3 a = make_down(e, l, write);
      a.bR = c.bR;
      a.bT = c.bT;
      if (a.op.rtab && jac) LAUNCH3(kname("k3_down", l), (k3_down_c<true, true, true, true>), c.c_grid, 128, a);
      else if (jac) LAUNCH3(kname("k3_down", l), (k3_down_c<true, true, true>), c.c_grid, 128, a);
      else LAUNCH3(kname("k3_down", l), (k3_down_c<true, false, true>), c.c_grid, 128, a);
    } else {
      Down3 a = make_down(e, l, write);
      if (boxmg && jac) LAUNCH3(kname("k3_down", l), (k3_down_c<true, true>), c.c_grid, 128, a);
      else if (boxmg) LAUNCH3(kname("k3_down", l), (k3_down_c<true, false>), c.c_grid, 128, a);
      else if (jac) LAUNCH3(kname("k3_down", l), (k3_down_c<false, true>), c.c_grid, 128, a);
      else LAUNCH3(kname("k3_down", l), (k3_down_c<false, false>), c.c_grid, 128, a);
    }
    if (e->smr && l >= e->smr_lo) {
      TRY3(launch_smr(e, l, jac && write));
    } else if (jac && write && l > e->lmin) {
      SmoothS sa = make_smooth_s(e, l);
      sa.chunk = c.s2_chunk;
      cudaEvent_t e0_ = nullptr;
      TRY3(begin_k(e, &e0_));
      k3_smooth2r<<<c.s2_blocks, dim3(kSX, k2Y / 2), k2RSmemV, e->s>>>(sa);
      CKL3();
      TRY3(end_k(e, kname("k3_smooth", l), e0_));
    }
  }
  Chain3 ch{};
  ch.l0 = e->lmin;
  ch.lc = e->lc;
  ch.do_up = write ? 1 : 0;
  ch.jac = jac ? 1 : 0;
  ch.part_sum = e->part_sum;
  ch.part_max = e->part_max;
  ch.nparts = e->nparts;
  ch.hist = e->hist;
  ch.counter = e->counter;
  ch.cap = e->cap;
  for (int l = e->lmin; l <= e->lc; ++l) {
    ch.down[l - e->lmin] = make_down(e, l, write);
    ch.smooth[l - e->lmin] = make_smooth(e, l);
    ch.up[l - e->lmin] = make_up(e, l);
  }
  LAUNCH3("k3_chain", k3_chain, 1, kChainBlock, ch);
  return TMG_OK;
}

int enqueue_cycle(Engine3* e) {
  TRY3(enqueue_down(e, true));
  const bool boxmg = e->cfg.flavor == TMG_BOXMG;
  const bool pi = e->cfg.variant == VAR_PI;
  const dim3 blk(kTX, kTY, kTZ);
  for (int l = e->lc + 1; l <= e->ltop; ++l) {
    Up3 a = make_up(e, l);
    const int g = e->L[l - 1].u_grid;
    if (pi) LAUNCH3(kname("k3_up", l), k3_up, e->L[l].grid, blk, a);
    else if (boxmg) TRY3(launch_up_boxmg(e, l, a));
    else TRY3(launch_up_lin(e, l, a));
  }
  return TMG_OK;
}

// after a cycle with the finest level double buffered: the other buffer is current
void pp_advance(Engine3* e) {
  if (!e->pp) return;
  e->par ^= 1;
  e->L[e->ltop].u = e->ubuf[e->par];
}

int ensure_graph(Engine3* e) {
  if (e->graph_dirty) {
    if (e->gexec && e->gcache.empty()) cudaGraphExecDestroy(e->gexec);
    e->gexec = nullptr;
    for (auto& kv : e->gcache) cudaGraphExecDestroy(kv.second);
    e->gcache.clear();
  }
  if (e->pp) {
    // one graph per parity of the finest level's double buffer
    const int key = e->par;
    auto it = e->gcache.find(key);
    if (it == e->gcache.end()) {
      cudaGraph_t g;
      CK3(cudaStreamBeginCapture(e->s, cudaStreamCaptureModeThreadLocal));
      e->launches = 0;
      int rc = enqueue_cycle(e);
      cudaError_t ce = cudaStreamEndCapture(e->s, &g);
      if (rc != TMG_OK) return rc;
      CK3(ce);
      cudaGraphExec_t x;
      CK3(cudaGraphInstantiate(&x, g, 0));
      cudaGraphDestroy(g);
      it = e->gcache.emplace(key, x).first;
    }
    e->gexec = it->second;
    e->graph_dirty = false;
    return TMG_OK;
  }
  if (!e->graph_dirty && e->gexec) return TMG_OK;
  cudaGraph_t g;
  CK3(cudaStreamBeginCapture(e->s, cudaStreamCaptureModeThreadLocal));
  e->launches = 0;
  int rc = enqueue_cycle(e);
  cudaError_t ce = cudaStreamEndCapture(e->s, &g);
  if (rc != TMG_OK) return rc;
  CK3(ce);
  CK3(cudaGraphInstantiate(&e->gexec, g, 0));
  cudaGraphDestroy(g);
  e->graph_dirty = false;
  return TMG_OK;
}

// --- setup (mg3d.Engine.rebuild) ------------------------------------------------------

int const_of(Engine3* e, const double* arr, size_t n, bool* is_const, double* value) {
  int* flag;
  TRY3(alloc3(e, &flag, 1, false));
  const int one = 1;
  CK3(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, e->s));
  k3_const_check<<<nblk(n), 256, 0, e->s>>>(arr, n, flag);
  CKL3();
  int hf = 0;
  CK3(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, e->s));
  CK3(cudaMemcpyAsync(value, arr, sizeof(double), cudaMemcpyDeviceToHost, e->s));
  CK3(cudaStreamSynchronize(e->s));
  *is_const = hf != 0;
  return TMG_OK;
}

Op3 element_op(double c, bool is_const, const double* coef) {
  Op3 o{};
  if (is_const) {
    o.kind = OP_CONST;
    o.m = c * C_D8;
    o.se = c * C_E6;
    o.sc = c * C_C12;
    double E = c;  // element_diag of a constant field: 8 equal terms, sequential
    for (int a = 1; a < 8; ++a) E = E + c;
    o.cdiag = K_D * E;
  } else {
    o.kind = OP_ELEMENT;
    o.e = coef;
  }
  return o;
}

// Row dictionary of a plane-major weight array (kernels3d_dict.cu): *dict / *idx stay null when
// a hash collision shows up or the rows do not repeat enough (D > R / 4) to pay for the index.
int build_dict(Engine3* e, const RowsView& v, size_t R, bool force, double** dict, uint32_t** idx, size_t* Dp,
               size_t* Dout) {
  *dict = nullptr;
  *idx = nullptr;
  *Dp = *Dout = 0;
  if (R < 2 || R > 0x7fffffffULL) return TMG_OK;
  const int n = (int)R;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  uint32_t *v0 = nullptr, *v1 = nullptr, *hs = nullptr, *rs = nullptr, *lead = nullptr, *first = nullptr,
           *nid = nullptr;
  int* bad = nullptr;
  void* tmp = nullptr;
  size_t tb = 0, t1 = 0, t2 = 0, t3b = 0;
  int rc = TMG_OK;
  auto done = [&](int r) {
    for (void* p : {(void*)k0, (void*)k1, (void*)v0, (void*)v1, (void*)hs, (void*)rs, (void*)lead, (void*)first,
                    (void*)nid, (void*)bad, tmp})
      if (p) cudaFree(p);
    return r;
  };
#define CKD(call)                                                                                 \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return done(fail3(e, TMG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)));       \
  } while (0)
  CKD(cudaMalloc(&k0, 8 * R));
  CKD(cudaMalloc(&k1, 8 * R));
  CKD(cudaMalloc(&v0, 4 * R));
  CKD(cudaMalloc(&v1, 4 * R));
  CKD(cudaMalloc(&hs, 4 * R));
  CKD(cudaMalloc(&rs, 4 * R));
  CKD(cudaMalloc(&lead, 4 * R));
  CKD(cudaMalloc(&first, 4 * R));
  CKD(cudaMalloc(&nid, 4 * R));
  CKD(cudaMalloc(&bad, sizeof(int)));
  CKD(cudaMemsetAsync(bad, 0, sizeof(int), e->s));
  CKD(cub::DeviceRadixSort::SortPairs(nullptr, t1, k0, k1, v0, v1, n, 0, 64, e->s));
  CKD(cub::DeviceScan::InclusiveScan(nullptr, t2, hs, rs, MaxU32{}, n, e->s));
  CKD(cub::DeviceScan::ExclusiveSum(nullptr, t3b, first, nid, n, e->s));
  tb = std::max(t1, std::max(t2, t3b));
  CKD(cudaMalloc(&tmp, tb));
  const unsigned g = (unsigned)std::min<size_t>(nblk(R, 256), 148 * 16);
  kd_hash<<<g, 256, 0, e->s>>>(v, R, k0, v0);
  CKD(cudaGetLastError());
  t1 = tb;
  CKD(cub::DeviceRadixSort::SortPairs(tmp, t1, k0, k1, v0, v1, n, 0, 64, e->s));
  kd_heads<<<g, 256, 0, e->s>>>(k1, R, hs);
  CKD(cudaGetLastError());
  t2 = tb;
  CKD(cub::DeviceScan::InclusiveScan(tmp, t2, hs, rs, MaxU32{}, n, e->s));
  kd_leader<<<g, 256, 0, e->s>>>(v1, rs, R, lead);
  kd_verify<<<g, 256, 0, e->s>>>(v, lead, R, first, bad);
  CKD(cudaGetLastError());
  t3b = tb;
  CKD(cub::DeviceScan::ExclusiveSum(tmp, t3b, first, nid, n, e->s));
  int hbad = 0;
  uint32_t last[2] = {0, 0};
  CKD(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, e->s));
  CKD(cudaMemcpyAsync(&last[0], nid + (R - 1), 4, cudaMemcpyDeviceToHost, e->s));
  CKD(cudaMemcpyAsync(&last[1], first + (R - 1), 4, cudaMemcpyDeviceToHost, e->s));
  CKD(cudaStreamSynchronize(e->s));
  const size_t D = (size_t)last[0] + last[1];
  if (hbad || (D > R / 4 && !force)) return done(TMG_OK);
  const size_t dp = kDictW;
  if ((rc = alloc3(e, dict, D * kDictW)) != TMG_OK) return done(rc);
  if ((rc = alloc3(e, idx, R / v.iinner * v.ipitch)) != TMG_OK) return done(rc);
  kd_fill<<<g, 256, 0, e->s>>>(v, lead, nid, R, *idx, *dict);
  CKD(cudaGetLastError());
  CKD(cudaStreamSynchronize(e->s));
#undef CKD
  *Dp = dp;
  *Dout = D;
  return done(TMG_OK);
}

// the cube-owned copy of level l's P (k3_up_tma), after every change of P; and, at setup (the
// throttled path rewrites P every cycle), the row dictionaries of P and Pc (TMG_PDICT=0: dense)
int refresh_pc(Engine3* e, int l) {
  Lvl3& c = e->L[l];
  if (!c.Pc) return TMG_OK;
  const size_t nc = (size_t)c.N - 1, Kp = (nc + kQK - 1) / kQK * kQK;
  k3_p_cube<<<nblk(nc * nc * nc, 128), 128, 0, e->s>>>(c.P, c.Pc, c.N, (int)Kp);
  CKL3();
  const char* env = std::getenv("TMG_PDICT");
  if (e->cfg.throttled || (env && env[0] == '0') || l < e->ltop - 2 || c.Pd || c.Pcd) return TMG_OK;
  const bool force = env && env[0] == '2';
  // Pc's dictionary feeds k3_up_dict, P's the restriction in k3_smc
  TRY3(build_dict(e, RowsView{c.Pc, nc, Kp, nc * nc * Kp, kQS, nc, Kp}, nc * nc * nc, force, &c.Pcd, &c.Pcdi,
                    &c.Pcdp, &c.Pcdn));
  if (c.Pcd) {  // k3_up_tma's step tables; a step meeting more than kQRows rows keeps the dense stream
    const int tK = (int)((nc + kQK - 1) / kQK), tJ = (int)((nc + kQJ - 1) / kQJ);
    const size_t cnt = nc * (size_t)tJ * tK;
    TRY3(alloc3(e, &c.Ptab, cnt * kQTabBytes, false));
    int* dover = nullptr;  // (e->deg may hold the setup's degenerate-collapse flag)
    TRY3(alloc3(e, &dover, 1));
    k3_up_tables<<<nblk(cnt, 128), 128, 0, e->s>>>(c.Pcdi, (int)nc, (int)Kp, tK, tJ, c.Ptab, dover);
    CKL3();
    int over = 0;
    CK3(cudaMemcpyAsync(&over, dover, sizeof(int), cudaMemcpyDeviceToHost, e->s));
    CK3(cudaStreamSynchronize(e->s));
    if (over) c.Pcd = nullptr, c.Pcdn = 0;
  }
  {
    const size_t Nc = c.N, Ncp = (Nc + 3) / 4 * 4;  // id rows padded to 16 bytes
    TRY3(build_dict(e, RowsView{c.P, c.nv, 0, c.nv, 125, Nc, Ncp}, c.nv, force, &c.Pd, &c.Pdi, &c.Pdp, &c.Pdn));
    TRY3(build_smc(e, l, false));
    if (!c.Pds) c.Pd = nullptr, c.Pdn = 0;  // a tile plane meets too many rows: the dense stream (k3_smr)
  }
  return TMG_OK;
}

// Run-length form of level l's Galerkin table along k (kernels3d_rle.cu): the operator stream of
// k3_down_c.  Kept when it stores less than 60 % of the dense rows.
int build_rle(Engine3* e, int l) {
  Lvl3& c = e->L[l];
  c.op.rtab = nullptr;
  const char* env = std::getenv("TMG_PDICT");
  if (!c.tbl || c.N - 2 < 64 || (env && env[0] == '0')) return TMG_OK;
  const bool force = env && env[0] == '2';
  const int rseg = (c.N - 2 + 31) / 32;
  const size_t segs = (size_t)c.N * c.N * rseg;
  uint32_t *rmask = nullptr, *rcnt = nullptr, *rbase = nullptr;
  uint8_t* rdup = nullptr;
  CK3(cudaMalloc(&rmask, sizeof(uint32_t) * segs));
  CK3(cudaMalloc(&rbase, sizeof(uint32_t) * (segs + 1)));
  CK3(cudaMalloc(&rcnt, sizeof(uint32_t) * (segs + 1)));
  void* tmp = nullptr;
  bool keep = false;  // the masks and bases live on with the handle only when the table is kept
  auto done = [&](int rc) {
    cudaFree(rcnt);
    if (rdup) cudaFree(rdup);
    if (tmp) cudaFree(tmp);
    if (keep) {
      e->allocs.push_back(rmask);
      e->allocs.push_back(rbase);
    } else {
      cudaFree(rmask);
      cudaFree(rbase);
    }
    return rc;
  };
#define CKR(x)                                                                  \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) return done(fail3(e, TMG_ECUDA, cudaGetErrorString(e_))); \
  } while (0)
  CKR(cudaMalloc(&rdup, segs));
  CKR(cudaMemsetAsync(rcnt + segs, 0, sizeof(uint32_t), e->s));
  const int planes = c.N - 2 <= kRleLink ? 1 : 0;  // plane repeats need the one-block-per-column link pass
  k3_rle_mask<<<148 * 16, 256, 0, e->s>>>(c.tbl, c.N, rseg, planes, rmask, rcnt, rdup);
  CKR(cudaGetLastError());
  size_t tb = 0;
  CKR(cub::DeviceScan::ExclusiveSum(nullptr, tb, rcnt, rbase, segs + 1, e->s));
  CKR(cudaMalloc(&tmp, tb));
  CKR(cub::DeviceScan::ExclusiveSum(tmp, tb, rcnt, rbase, segs + 1, e->s));
  uint32_t total = 0;
  CKR(cudaMemcpyAsync(&total, rbase + segs, sizeof(uint32_t), cudaMemcpyDeviceToHost, e->s));
  CKR(cudaStreamSynchronize(e->s));
#undef CKR
  const size_t interior = (size_t)(c.N - 2) * (c.N - 2) * (c.N - 2);
  if (total == 0 || (!force && (double)total > 0.6 * (double)interior)) return done(TMG_OK);  // no runs: dense planes
  double* rtab = nullptr;
  if (alloc3(e, &rtab, (size_t)27 * total, false) != TMG_OK) return done(TMG_ECUDA);
  k3_rle_fill<<<148 * 16, 256, 0, e->s>>>(c.tbl, c.N, rseg, rmask, rbase, rdup, total, rtab);
  if (planes) k3_rle_link2<<<rseg, kRleLink, 0, e->s>>>(c.N, rseg, rdup, rbase);
  else k3_rle_link<<<nblk((size_t)c.N * rseg, 128), 128, 0, e->s>>>(c.N, rseg, rdup, rbase);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(e->s) != cudaSuccess)
    return done(fail3(e, TMG_ECUDA, "k3_rle_fill failed"));
  keep = true;
  c.op.rtab = rtab;
  c.op.rbase = rbase;
  c.op.rmask = rmask;
  c.op.rn = total;
  c.op.rseg = rseg;
  return done(TMG_OK);
}

// Galerkin rows of level l's interior vertices (k3_rap_y + k3_rap_out over slabs of coarse planes;
// the scratch Y holds 343 doubles per slab vertex, at most about 2 GB)
int galerkin_rows(Engine3* e, int l, const Rows& raw) {
  Lvl3& c = e->L[l];
  const size_t plane = (size_t)c.N * c.N;
  const int interior = c.N - 2;
  const int per = (int)std::max<size_t>(1, std::min<size_t>(interior, ((size_t)2 << 30) / (plane * 343 * 8)));
  double* Y = nullptr;
  CK3(cudaMalloc(&Y, sizeof(double) * plane * 343 * per));
  int rc = TMG_OK;
  for (int I0 = 1; I0 <= interior && rc == TMG_OK; I0 += per) {
    RapArgs A{};
    A.Nc = c.N;
    A.Nf = raw.N;
    A.I0 = I0;
    A.planes = std::min(per, interior - I0 + 1);
    A.P = c.P;
    A.tbl = raw.tbl;
    A.e = raw.e;
    A.Y = Y;
    A.out = c.tbl;
    const size_t sv = plane * A.planes;
    const unsigned gb = (unsigned)std::min<size_t>((sv + 31) / 32, (size_t)num_sms() * 32);
    if (raw.tbl) k3_rap_y<false><<<gb, dim3(32, kRapYW), 0, e->s>>>(A);
    else k3_rap_y<true><<<gb, dim3(32, kRapYW), 0, e->s>>>(A);
    k3_rap_out<<<gb, dim3(32, 27), 0, e->s>>>(A);
    if (cudaGetLastError() != cudaSuccess) rc = fail3(e, TMG_ECUDA, "kernel launch: k3_rap_y / k3_rap_out");
  }
  cudaStreamSynchronize(e->s);
  cudaFree(Y);
  return rc;
}

// BoxMG P and Galerkin rows of level l from level l+1's operator (solvers.py:227-250):
// P[l] and tbl[l] are rewritten in place, so captured graphs stay valid
int boxmg_level(Engine3* e, int l) {
  Lvl3& c = e->L[l];
  Lvl3& f = e->L[l + 1];
  const Rows raw = (l + 1 == e->ltop) ? Rows{f.N, nullptr, f.coef} : Rows{f.N, f.tbl, nullptr};
  const int nc = c.N - 1;
  k3_p_init<<<nblk(c.nv), 256, 0, e->s>>>(c.P, c.nv);
  CKL3();
  for (int ax = 0; ax < 3; ++ax) {
    k3_edges<<<nblk((size_t)nc * c.N * c.N, 128), 128, 0, e->s>>>(c.P, nc, ax, raw, e->deg);
    CKL3();
  }
  for (int nx = 0; nx < 3; ++nx) {
    k3_faces<<<nblk((size_t)c.N * nc * nc, 128), 128, 0, e->s>>>(c.P, nc, nx, raw);
    CKL3();
  }
  k3_cells<<<nblk((size_t)nc * nc * nc, 128), 128, 0, e->s>>>(c.P, nc, raw);
  CKL3();
  k3_assemble<<<nblk(c.nv), 256, 0, e->s>>>(c.tbl, Rows{c.N, nullptr, c.coef});
  CKL3();
  if (c.N > 2) TRY3(galerkin_rows(e, l, raw));
  return refresh_pc(e, l);
}

int check_degenerate(Engine3* e) {
  int hdeg = 0;
  CK3(cudaMemcpyAsync(&hdeg, e->deg, sizeof(int), cudaMemcpyDeviceToHost, e->s));
  CK3(cudaStreamSynchronize(e->s));
  if (hdeg) return fail3(e, TMG_EDEGENERATE, "degenerate collapsed stencil in face-point solve");
  return TMG_OK;
}

int build(Engine3* e, const tmg_tree3* t) {
  const tmg_config& cfg = e->cfg;
  if (t->lmin < 1) return fail3(e, TMG_EINVAL, "lmin must be at least 1");
  if (t->depth < t->lmin) return fail3(e, TMG_EINVAL, "tree has no DoF-carrying level at or above lmin");
  if (t->depth > 7) return fail3(e, TMG_EINVAL, "depth above 7 is not supported in 3D");
  if (!t->eps || !t->u) return fail3(e, TMG_EINVAL, "tree.eps / tree.u missing");
  if (cfg.rtilde_true_operator)
    return fail3(e, TMG_EINVAL, "rtilde_true_operator is not offered in 3D");
  e->lmin = t->lmin;
  e->ltop = t->depth;
  const int l0 = e->lmin, l1 = e->ltop;
  e->L.assign(l1 + 1, Lvl3{});
  for (int l = l0; l <= l1; ++l) {
    Lvl3& c = e->L[l];
    c.l = l;
    c.N = ipow3(l) + 1;
    c.nv = (size_t)c.N * c.N * c.N;
    c.ncell = (size_t)(c.N - 1) * (c.N - 1) * (c.N - 1);
    if (!t->u[l]) return fail3(e, TMG_EINVAL, "tree.u missing a level");
  }
  // material: eff_eps top-down (child means), coefficient e = eff * h
  for (int l = l1; l >= l0; --l) {
    Lvl3& c = e->L[l];
    TRY3(alloc3(e, &c.eff, c.ncell, false));
    TRY3(alloc3(e, &c.coef, c.ncell, false));
    if (l == l1) {
      CK3(cudaMemcpyAsync(c.eff, t->eps, sizeof(double) * c.ncell, cudaMemcpyHostToDevice, e->s));
    } else {
      k3_child_mean<<<nblk(c.ncell), 256, 0, e->s>>>(c.eff, e->L[l + 1].eff, c.N - 1);
      CKL3();
    }
    k3_scale<<<nblk(c.ncell), 256, 0, e->s>>>(c.coef, c.eff, std::pow(3.0, -(double)l), c.ncell);
    CKL3();
  }
  for (int l = l0; l <= l1; ++l) {
    Lvl3& c = e->L[l];
    c.w = (cfg.variant == VAR_EXP) ? std::pow(cfg.omega_hat, (double)(l1 - l)) : cfg.omega;
  }
  CK3(cudaFuncSetAttribute(k3_top2<OP_CONST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2TopSmem));
  CK3(cudaFuncSetAttribute(k3_top2<OP_ELEMENT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2TopSmem));
  CK3(cudaFuncSetAttribute(k3_top4r, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTop4rSmem));
  CK3(cudaFuncSetAttribute(k3_top4c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTop4cSmem));
  CK3(cudaFuncSetAttribute(k3_smooth2r, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2RSmemV));
  CK3(cudaFuncSetAttribute(k3_up_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpTmaSmem));
  CK3(cudaFuncSetAttribute(k3_up_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpTmaSmem));
  CK3(cudaFuncSetAttribute(k3_up_dict<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DLay<true>::smem));
  CK3(cudaFuncSetAttribute(k3_up_dict<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DLay<true>::smem));
  CK3(cudaFuncSetAttribute(k3_up_dict<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DLay<false>::smem));
  CK3(cudaFuncSetAttribute(k3_up_dict<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)DLay<false>::smem));
  CK3(cudaFuncSetAttribute(k3_up_tma<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpTmaSmem));
  TRY3(alloc3(e, &e->deg, 1));
  e->thr_next = l0 - 1;
  if (cfg.flavor == TMG_GEOMETRIC) {
    for (int l = l0; l <= l1; ++l) {
      Lvl3& c = e->L[l];
      bool kc;
      double v;
      TRY3(const_of(e, c.coef, c.ncell, &kc, &v));
      c.op = element_op(v, kc, c.coef);
    }
  } else {
    Lvl3& top = e->L[l1];
    bool kc;
    double v;
    TRY3(const_of(e, top.coef, top.ncell, &kc, &v));
    top.op = element_op(v, kc, top.coef);
    for (int l = l1 - 1; l >= l0; --l) {
      Lvl3& c = e->L[l];
      TRY3(alloc3(e, &c.P, 125 * c.nv, false));
      TRY3(alloc3(e, &c.tbl, 27 * c.nv, false));
      // BoxMG prolongation of the two finest levels as TMA streams (k3_up_tma)
      if (l >= l1 - 2 && c.N - 1 >= kQK) {
        const size_t nc = (size_t)c.N - 1, Kp = (nc + kQK - 1) / kQK * kQK;
        TRY3(alloc3(e, &c.Pc, (size_t)kQS * nc * nc * Kp));
      }
      if (cfg.throttled) {  // d-linear P, rediscretised rows; upgraded one level per cycle
        k3_p_dlinear<<<nblk(c.nv), 256, 0, e->s>>>(c.P, c.N);
        CKL3();
        TRY3(refresh_pc(e, l));
        k3_assemble<<<nblk(c.nv), 256, 0, e->s>>>(c.tbl, Rows{c.N, nullptr, c.coef});
        CKL3();
      } else {
        TRY3(boxmg_level(e, l));
      }
      c.op = Op3{};
      c.op.kind = OP_TABLE;
      c.op.tbl = c.tbl;
      c.op.tdict = c.Td;  // (null = dense planes)
      c.op.tidx = c.Tdi;
      // the table's run-length form (eager setup only: the throttled path rewrites the rows)
      if (!cfg.throttled && l >= l1 - 2) TRY3(build_rle(e, l));
    }
    if (cfg.throttled) e->thr_next = l1 - 1;
  }
  {  // row-padded copy of the finest level's cell coefficients for the TMA-staged top kernel
    Lvl3& top = e->L[l1];
    if (top.op.kind == OP_ELEMENT) {
      const int n = top.N - 1, np = n + (n & 1);
      // blockwise-constant materials: the cell planes repeat along axis 0 in runs of 3^k planes
      // (bitwise check); the top kernel then streams one stored plane per run -- at config 5 the
      // 3.1 GB coefficient stream of every cycle becomes 27 L2-resident planes
      top.crun = 1;
      {
        int* flag;
        TRY3(alloc3(e, &flag, 1, false));
        for (int run = 27; run >= 3 && top.crun == 1; run /= 3) {
          if (n % run) continue;
          const int one = 1;
          int hf = 0;
          CK3(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, e->s));
          k3_plane_run_check<<<nblk(top.ncell), 256, 0, e->s>>>(top.coef, n, run, flag);
          CKL3();
          CK3(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, e->s));
          CK3(cudaStreamSynchronize(e->s));
          if (hf) top.crun = run;
        }
      }
      const int planes = n / top.crun;
      TRY3(alloc3(e, &top.coefp, (size_t)planes * n * np));
      if (top.crun == 1)
        CK3(cudaMemcpy2DAsync(top.coefp, sizeof(double) * np, top.coef, sizeof(double) * n, sizeof(double) * n,
                              (size_t)n * n, cudaMemcpyDeviceToDevice, e->s));
      else
        for (int pl = 0; pl < planes; ++pl)
          CK3(cudaMemcpy2DAsync(top.coefp + (size_t)pl * n * np, sizeof(double) * np,
                                top.coef + (size_t)pl * top.crun * n * n, sizeof(double) * n, sizeof(double) * n,
                                (size_t)n, cudaMemcpyDeviceToDevice, e->s));
    }
  }
  TRY3(check_degenerate(e));

  // counts (solvers.py:449-459)
  long long sum = 0, lt = 0, gt = 0;
  for (int l = l0; l <= l1; ++l) {
    const long long d = (long long)(e->L[l].N - 2) * (e->L[l].N - 2) * (e->L[l].N - 2);
    sum += d;
    if (l < l1) lt += d;
    if (l > l0) gt += d;
  }
  e->dofs_total = (long long)(e->L[l1].N - 2) * (e->L[l1].N - 2) * (e->L[l1].N - 2);
  e->updates = sum + (cfg.variant == VAR_JAC ? lt : 0) + (cfg.variant == VAR_PI ? gt : 0);

  // chain levels: <= 1024 vertices, at most kMaxChain
  e->lc = l0;
  for (int l = l0; l <= l1 && l - l0 < kMaxChain; ++l)
    if (e->L[l].nv <= 1024) e->lc = l;
  // work vectors
  const bool jac = cfg.variant == VAR_JAC;
  int parts = 0;
  for (int l = l0; l <= l1; ++l) {
    Lvl3& c = e->L[l];
    TRY3(alloc3(e, &c.u, c.nv, false));
    CK3(cudaMemcpyAsync(c.u, t->u[l], sizeof(double) * c.nv, cudaMemcpyHostToDevice, e->s));
    TRY3(alloc3(e, &c.g, c.nv));
    if (l > l0) TRY3(alloc3(e, &c.rho, c.nv));
    if (l > l0 && jac) TRY3(alloc3(e, &c.sm, c.nv));
    if (l < l1) TRY3(alloc3(e, &c.carry, c.nv));
    c.grid = grid_for(c.N, 1, c.N - 1);
    {
      const int tiles = ((c.N - 2 + kSX - 1) / kSX) * ((c.N - 2 + kSY - 1) / kSY);
      int nch = (148 * 16 + tiles - 1) / tiles;
      nch = std::max(1, std::min(nch, std::max(1, (c.N - 2) / 4)));
      c.s_chunk = (c.N - 2 + nch - 1) / nch;
      const int chunks = (c.N - 2 + c.s_chunk - 1) / c.s_chunk;
      c.s_blocks = tiles * chunks;
      {
        const int t2 = ((c.N - 2 + kSX - 1) / kSX) * ((c.N - 2 + k2Y - 1) / k2Y);
        int n2 = (148 * 12 + t2 - 1) / t2;
        n2 = std::max(1, std::min(n2, std::max(1, (c.N - 2) / 4)));
        // CTAs per SM of the level's streaming kernel: k3_top4r (element operator) 2, k3_top2 3
        const int slots = num_sms() * ((l == l1 && c.op.kind == OP_ELEMENT) ? 2 : 3);
        if (t2 >= slots) {  // tiles fill a wave: chunks by wave efficiency x halo
          double best_eff = 0.0;
          for (int nch = 1; nch <= 8; ++nch) {
            const int ch = (c.N - 2 + nch - 1) / nch, nb = t2 * ((c.N - 2 + ch - 1) / ch);
            const double waves = (double)nb / slots;
            const double eff = waves / std::ceil(waves) * (double)ch / (ch + 2.0);
            if (eff > best_eff + 1e-9) { best_eff = eff; n2 = nch; }
          }
        }
        c.s2_chunk = (c.N - 2 + n2 - 1) / n2;
        c.s2_blocks = t2 * ((c.N - 2 + c.s2_chunk - 1) / c.s2_chunk);
      }
      const size_t ni = (size_t)(c.N - 2) * (c.N - 2) * (c.N - 2);
      const size_t ncell = (size_t)(c.N - 1) * (c.N - 1) * (c.N - 1);
      c.c_grid = (int)std::max<size_t>(1, std::min<size_t>((ni + 127) / 128, 148 * 32));
      c.u_grid = (int)std::max<size_t>(1, std::min<size_t>((9 * ncell + 127) / 128, 148 * 64));
    }
    if (l == l1 && l > e->lc) {
      c.part_off = 0;
      parts = std::max(c.s_blocks, c.s2_blocks);
    }
  }
  // finest level double buffered: its down sweep (a grid level, not the chain) writes u + g into
  // the other buffer and its up sweep adds P carry there -- g never reaches HBM.  adafac-pi
  // subtracts a prolonged d~ on the finest level too, so it keeps g.
  e->par = 0;
  e->pp = l1 > e->lc && cfg.variant != VAR_PI;
  if (e->pp) {
    Lvl3& c = e->L[l1];
    e->ubuf[0] = c.u;
    TRY3(alloc3(e, &e->ubuf[1], c.nv, false));
    CK3(cudaMemcpyAsync(e->ubuf[1], c.u, sizeof(double) * c.nv, cudaMemcpyDeviceToDevice, e->s));
  }
  // finest-level smoothing + restriction fused (k3_smr; else k3_smooth2r + k3_down_c)
  {
    e->smr = cfg.variant != VAR_PI && l1 - 1 > e->lc;
    e->smr_lo = e->lc + 2;  // every level whose coarser level is a grid (not chain) level
    if (e->smr && cfg.flavor == TMG_GEOMETRIC) {
      // d-linear transfer: one constant weight row for every interior coarse vertex (its fine
      // offsets +-2 never leave the grid), so the dictionary kernel k3_smc runs on a one-row
      // dictionary and tile-plane tables that all name row 0
      double row[kDictW] = {0.0};
      for (int a = -2; a <= 2; ++a)
        for (int b = -2; b <= 2; ++b)
          for (int c2 = -2; c2 <= 2; ++c2) {
            const double wa = 1.0 - std::abs(a) / 3.0, wb = 1.0 - std::abs(b) / 3.0, wc = 1.0 - std::abs(c2) / 3.0;
            row[pslot(a, b, c2)] = (wa * wb) * wc;  // k3_p_dlinear / mg3d.dlinear_p_table
          }
      for (int l = e->smr_lo - 1; l < l1; ++l) {
        Lvl3& cc = e->L[l];
        TRY3(alloc3(e, &cc.Pd, kDictW, false));
        CK3(cudaMemcpyAsync(cc.Pd, row, sizeof(row), cudaMemcpyHostToDevice, e->s));
        CK3(cudaStreamSynchronize(e->s));
        cc.Pdn = 1;
        TRY3(build_smc(e, l, true));
      }
    }
    if (e->smr) {
      CK3(cudaFuncSetAttribute(k3_smc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmcSmem));
      CK3(cudaFuncSetAttribute(k3_smc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmcSmem));
      CK3(cudaFuncSetAttribute(k3_smr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmrSmem));
      for (int l = e->smr_lo - 1; l < l1; ++l) {
        Lvl3& cc = e->L[l];
        if (!cc.bR) TRY3(alloc3(e, &cc.bR, cc.nv));
        if (!cc.bT) TRY3(alloc3(e, &cc.bT, cc.nv));
      }
    }
  }
  e->nparts = parts;
  TRY3(alloc3(e, &e->part_sum, parts));
  TRY3(alloc3(e, &e->part_max, parts));
  TRY3(alloc3(e, &e->hist, 2 * e->cap));
  TRY3(alloc3(e, &e->counter, 1));
  e->host_counter = 0;
  CK3(cudaStreamSynchronize(e->s));
  e->graph_dirty = true;
  return TMG_OK;
}

int check_level(Engine3* e, int level) {
  if (level < e->lmin || level > e->ltop)
    return fail3(e, TMG_EINVAL, "level " + std::to_string(level) + " outside [lmin, ltop]");
  return TMG_OK;
}

int read_stats(Engine3* e, long long first, int count, tmg_stats* out) {
  std::vector<double> hh(2 * e->cap);
  CK3(cudaMemcpyAsync(hh.data(), e->hist, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost, e->s));
  CK3(cudaStreamSynchronize(e->s));
  for (int k = 0; k < count; ++k) {
    const long long slot = (first + k) % e->cap;
    out[k].l2h = hh[2 * slot];
    out[k].linf = hh[2 * slot + 1];
    out[k].dofs = e->dofs_total;
    out[k].updates = e->updates;
  }
  return TMG_OK;
}

struct ErrScope {
  Engine3* e;
  ErrScope(Engine3* e_, std::string& err) : e(e_) { e->err = &err; }
  ~ErrScope() { e->err = nullptr; }
};

// --- sharded mode ---------------------------------------------------------------

// 2.5D tiling of the interior planes [ilo, ihi) of an N^3 level (ty = rows per CTA)
void tiling(int N, int ilo, int ihi, int* chunk, int* blocks, int ty = kSY) {
  const int tiles = ((N - 2 + kSX - 1) / kSX) * ((N - 2 + ty - 1) / ty);
  const int np = std::max(1, ihi - ilo);
  int nch = (148 * 16 + tiles - 1) / tiles;
  nch = std::max(1, std::min(nch, std::max(1, np / 4)));
  *chunk = (np + nch - 1) / nch;
  *blocks = tiles * ((np + *chunk - 1) / *chunk);
}

int interior_lo(Engine3* e, int l) { return std::max(1, e->own_lo[l]); }
int interior_hi(Engine3* e, int l) { return std::min(e->L[l].N - 1, e->own_hi[l]); }
// ... clipped to the part a tmg3_phase_range call names (DOWN / UP only)
int part_lo(Engine3* e, int l) { return std::max(interior_lo(e, l), e->rng_lo); }
int part_hi(Engine3* e, int l) { return std::min(interior_hi(e, l), e->rng_hi); }

// sharded cycle: level l's adaFACx smoothing runs fused with the restriction into l - 1 (k3_smr
// over the owned coarse planes of l - 1, phase TMG_PH_SMR) -- the grid levels above the shard
// level where the single-GPU cycle fuses them
bool fused3(const Engine3* e, int l) {
  return e->sharded && e->smr && e->cfg.variant == VAR_JAC && l > e->ls && l <= e->ltop && l >= e->smr_lo;
}

int phase3(Engine3* e, int phase, int l) {
  const bool jac = e->cfg.variant == VAR_JAC;
  const bool boxmg = e->cfg.flavor == TMG_BOXMG;
  const bool pi = e->cfg.variant == VAR_PI;
  const dim3 sblk(kSX, kSY);
  switch (phase) {
    case TMG_PH_DOWN: {
      if (l < e->ls || l > e->ltop) return fail3(e, TMG_EINVAL, "DOWN: level is not sharded");
      const int lo = part_lo(e, l), hi = part_hi(e, l);
      if (l == e->ltop && e->rng_first) e->top_parts = 0;
      if (hi <= lo) return TMG_OK;
      Lvl3& c = e->L[l];
      if (l == e->ltop) {
        Top3 a = make_top(e, l);
        a.ilo = lo;
        a.ihi = hi;
        // the part's own column chunks; its residual partials follow those of the earlier parts
        int blocks = e->own_blocks2[l];
        a.chunk = e->own_chunk2[l];
        if (lo != interior_lo(e, l) || hi != interior_hi(e, l)) tiling(c.N, lo, hi, &a.chunk, &blocks, k2Y);
        if (e->top_parts + blocks > e->nparts) return fail3(e, TMG_EINVAL, "DOWN: too many parts of the finest level");
        a.part_sum += e->top_parts;
        a.part_max += e->top_parts;
        e->top_parts += blocks;
        cudaEvent_t e0_ = nullptr;
        TRY3(begin_k(e, &e0_));
        if (c.op.kind == OP_CONST && a.use_tma && a.rhs_tma)
          k3_top4c<<<blocks, dim3(kSX, k2Y / kT4R), kTop4cSmem, e->s>>>(a);
        else if (c.op.kind == OP_CONST)
          k3_top2<OP_CONST><<<blocks, dim3(kSX, k2Y / 2), k2TopSmem, e->s>>>(a);
        else if (use_top4(a))
          k3_top4r<<<blocks, dim3(kSX, k2Y / kT4R), kTop4rSmem, e->s>>>(a);
        else
          k3_top2<OP_ELEMENT><<<blocks, dim3(kSX, k2Y / 2), k2TopSmem, e->s>>>(a);
        CKL3();
        TRY3(end_k(e, kname("k3_down", l), e0_));
      } else if (fused3(e, l + 1)) {  // restrictions formed by TMG_PH_SMR of level l + 1
        Down3 a = make_down(e, l, true);
        a.ilo = lo;
        a.ihi = hi;
        a.bR = c.bR;
        a.bT = c.bT;
        if (a.op.rtab) LAUNCH3(kname("k3_down", l), (k3_down_c<true, true, true, true>), c.c_grid, 128, a);
        else LAUNCH3(kname("k3_down", l), (k3_down_c<true, true, true>), c.c_grid, 128, a);
      } else {
        Down3 a = make_down(e, l, true);
        a.ilo = lo;
        a.ihi = hi;
        if (boxmg && jac) LAUNCH3(kname("k3_down", l), (k3_down_c<true, true>), c.c_grid, 128, a);
        else if (boxmg) LAUNCH3(kname("k3_down", l), (k3_down_c<true, false>), c.c_grid, 128, a);
        else if (jac) LAUNCH3(kname("k3_down", l), (k3_down_c<false, true>), c.c_grid, 128, a);
        else LAUNCH3(kname("k3_down", l), (k3_down_c<false, false>), c.c_grid, 128, a);
      }
      return TMG_OK;
    }
    case TMG_PH_SMOOTH: {
      if (!jac || l <= e->lmin) return TMG_OK;
      const int lo = interior_lo(e, l), hi = interior_hi(e, l);
      if (hi <= lo) return TMG_OK;
      SmoothS a = make_smooth_s(e, l);
      a.ilo = lo;
      a.ihi = hi;
      a.chunk = e->own_chunk2[l];
      cudaEvent_t e0_ = nullptr;
      TRY3(begin_k(e, &e0_));
      k3_smooth2r<<<e->own_blocks2[l], dim3(kSX, k2Y / 2), k2RSmemV, e->s>>>(a);
      CKL3();
      TRY3(end_k(e, kname("k3_smooth", l), e0_));
      return TMG_OK;
    }
    case TMG_PH_SMR: {
      if (!fused3(e, l)) return fail3(e, TMG_EINVAL, "SMR: level's smoothing is not fused (tmg3_fused)");
      return launch_smr(e, l, true, interior_lo(e, l - 1), interior_hi(e, l - 1));
    }
    case TMG_PH_REDUCE: {
      LAUNCH3("k3_reduce_parts", k3_reduce_parts, 1, 512, e->part_sum, e->part_max, e->top_parts, e->red);
      return TMG_OK;
    }
    case TMG_PH_REPL: {
      const dim3 blk(kTX, kTY, kTZ);
      const int lcs = std::min(e->lc, e->ls - 1);  // the one-block chain stays below ls
      for (int q = e->ls - 1; q > lcs; --q) {
        Lvl3& c = e->L[q];
        Down3 a = make_down(e, q, true);
        if (boxmg && jac) LAUNCH3(kname("k3_down", q), (k3_down_c<true, true>), c.c_grid, 128, a);
        else if (boxmg) LAUNCH3(kname("k3_down", q), (k3_down_c<true, false>), c.c_grid, 128, a);
        else if (jac) LAUNCH3(kname("k3_down", q), (k3_down_c<false, true>), c.c_grid, 128, a);
        else LAUNCH3(kname("k3_down", q), (k3_down_c<false, false>), c.c_grid, 128, a);
        if (jac && q > e->lmin) {
          SmoothS sa = make_smooth_s(e, q);
          LAUNCH3(kname("k3_smooth", q), k3_smooth_s, c.s_blocks, sblk, sa);
        }
      }
      Chain3 ch{};
      ch.l0 = e->lmin;
      ch.lc = lcs;
      ch.do_up = 1;
      ch.jac = jac ? 1 : 0;
      ch.part_sum = e->red;
      ch.part_max = e->red + 1;
      ch.nparts = 1;
      ch.hist = e->hist;
      ch.counter = e->counter;
      ch.cap = e->cap;
      for (int q = e->lmin; q <= lcs; ++q) {
        ch.down[q - e->lmin] = make_down(e, q, true);
        ch.smooth[q - e->lmin] = make_smooth(e, q);
        ch.up[q - e->lmin] = make_up(e, q);
      }
      LAUNCH3("k3_chain", k3_chain, 1, kChainBlock, ch);
      for (int q = lcs + 1; q < e->ls; ++q) {
        Up3 a = make_up(e, q);
        const int g = e->L[q - 1].u_grid;
        if (pi) LAUNCH3(kname("k3_up", q), k3_up, e->L[q].grid, blk, a);
        else if (boxmg) TRY3(launch_up_boxmg(e, q, a));
        else LAUNCH3(kname("k3_up", q), k3_up_cell<false>, g, 128, a);
      }
      e->host_counter++;
      return TMG_OK;
    }
    case TMG_PH_UP: {
      if (l < e->ls || l > e->ltop) return fail3(e, TMG_EINVAL, "UP: level is not sharded");
      const int lo = part_lo(e, l), hi = part_hi(e, l);
      if (hi <= lo) {
        if (l == e->ltop && e->rng_last) pp_advance(e);
        return TMG_OK;
      }
      Up3 a = make_up(e, l);
      a.ilo = lo;
      a.ihi = hi;
      a.l0 = e->ls;  // walk-down injection stays on the sharded levels
      const int g = e->L[l - 1].u_grid;
      if (pi) {
        const dim3 blk(kTX, kTY, kTZ);
        LAUNCH3(kname("k3_up", l), k3_up, e->L[l].grid, blk, a);
      } else if (boxmg) TRY3(launch_up_boxmg(e, l, a));
      else TRY3(launch_up_lin(e, l, a));
      if (l == e->ltop && e->rng_last) pp_advance(e);  // the buffer just completed is the iterate (TMG_F_U names it)
      return TMG_OK;
    }
    case TMG_PH_INJECT: {
      for (int q = e->ls - 1; q >= e->lmin; --q) {
        const int n = e->L[q].N - 2;
        if (n <= 0) continue;
        k3_inject<<<nblk((size_t)n * n * n), 256, 0, e->s>>>(e->L[q].u, e->L[q].N, e->L[q + 1].u, e->L[q + 1].N);
        CKL3();
        e->launches++;
      }
      return TMG_OK;
    }
    default:
      return fail3(e, TMG_EINVAL, "unknown phase");
  }
}

}  // namespace

int e3_shard(Engine3* e, int ls, const int32_t* lo, const int32_t* hi, std::string& err) {
  ErrScope es(e, err);
  if (ls <= e->lmin || ls > e->ltop) return fail3(e, TMG_EINVAL, "shard level must lie in (lmin, ltop]");
  e->own_lo.assign(e->ltop + 1, 0);
  e->own_hi.assign(e->ltop + 1, 0);
  e->own_blocks.assign(e->ltop + 1, 0);
  e->own_chunk.assign(e->ltop + 1, 1);
  e->own_blocks2.assign(e->ltop + 1, 0);
  e->own_chunk2.assign(e->ltop + 1, 1);
  int maxb = 0;
  for (int l = ls; l <= e->ltop; ++l) {
    if (lo[l] < 0 || hi[l] > e->L[l].N || lo[l] > hi[l]) return fail3(e, TMG_EINVAL, "bad owned plane range");
    e->own_lo[l] = lo[l];
    e->own_hi[l] = hi[l];
    const int a = std::max(1, lo[l]), b = std::min(e->L[l].N - 1, hi[l]);
    tiling(e->L[l].N, a, std::max(a + 1, b), &e->own_chunk[l], &e->own_blocks[l]);
    tiling(e->L[l].N, a, std::max(a + 1, b), &e->own_chunk2[l], &e->own_blocks2[l], k2Y);
    maxb = std::max(maxb, std::max(e->own_blocks[l], e->own_blocks2[l]));
  }
  {  // tmg3_phase_range: up to four parts of the finest level, each with at most its own chunks
    const int N = e->L[e->ltop].N;
    maxb += 4 * ((N - 2 + kSX - 1) / kSX) * ((N - 2 + k2Y - 1) / k2Y) * 8;
  }
  e->ls = ls;
  e->sharded = true;
  if (maxb > e->nparts) {
    TRY3(alloc3(e, &e->part_sum, maxb));
    TRY3(alloc3(e, &e->part_max, maxb));
    e->nparts = maxb;
  }
  if (!e->red) TRY3(alloc3(e, &e->red, 2));
  CK3(cudaStreamSynchronize(e->s));
  return TMG_OK;
}

int e3_phase(Engine3* e, int phase, int level, std::string& err) {
  ErrScope es(e, err);
  if (!e->sharded) return fail3(e, TMG_EINVAL, "handle is not sharded (tmg3_shard)");
  if (phase == TMG_PH_DOWN && level == e->ltop && e->rng_first && e->thr_next >= e->lmin) {
    // throttled setup at the start of a sharded cycle; every rank holds the full operators
    TRY3(boxmg_level(e, e->thr_next));
    TRY3(check_degenerate(e));
    --e->thr_next;
  }
  return phase3(e, phase, level);
}

int e3_phase_range(Engine3* e, int phase, int level, int lo, int hi, int first, int last, std::string& err) {
  ErrScope es(e, err);
  if (phase != TMG_PH_DOWN && phase != TMG_PH_UP) return fail3(e, TMG_EINVAL, "phase ranges: DOWN and UP only");
  e->rng_lo = lo;
  e->rng_hi = hi;
  e->rng_first = first != 0;
  e->rng_last = last != 0;
  const int rc = e3_phase(e, phase, level, err);
  e->rng_lo = 0;
  e->rng_hi = 1 << 30;
  e->rng_first = e->rng_last = true;
  return rc;
}

int e3_fused(Engine3* e, int level, int32_t* out, std::string& err) {
  e->err = &err;
  TRY3(check_level(e, level));
  *out = fused3(e, level) ? 1 : 0;
  return TMG_OK;
}

int e3_storage(Engine3* e, int level, int64_t* out, std::string& err) {
  e->err = &err;
  TRY3(check_level(e, level));
  const Lvl3& c = e->L[level];
  const int64_t nc = c.N - 1;
  out[0] = c.P ? (int64_t)c.nv : 0;
  out[1] = c.Pd ? (int64_t)c.Pdn : 0;
  out[2] = c.Pc ? nc * nc * nc : 0;
  out[3] = c.Pcd ? (int64_t)c.Pcdn : 0;
  out[4] = c.tbl ? (int64_t)c.nv : 0;
  out[5] = c.op.rtab ? (int64_t)c.op.rn : 0;
  return TMG_OK;
}

int e3_field(Engine3* e, int field, int level, uint64_t* ptr, int64_t* count, std::string& err) {
  ErrScope es(e, err);
  if (field == TMG_F_PART) {
    if (!e->red) return fail3(e, TMG_EINVAL, "no reduction buffer (tmg3_shard first)");
    *ptr = (uint64_t)(uintptr_t)e->red;
    *count = 2;
    return TMG_OK;
  }
  TRY3(check_level(e, level));
  Lvl3& c = e->L[level];
  double* p = nullptr;
  switch (field) {
    case TMG_F_U: p = c.u; break;
    case TMG_F_RHO: p = c.rho; break;
    case TMG_F_SM: p = c.sm; break;
    case TMG_F_CARRY: p = c.carry; break;
    case TMG_F_G: p = c.g; break;
    default: return fail3(e, TMG_EINVAL, "unknown field");
  }
  if (!p) return fail3(e, TMG_EINVAL, "field not allocated on this level");
  *ptr = (uint64_t)(uintptr_t)p;
  *count = (int64_t)c.nv;
  return TMG_OK;
}

int e3_stream(Engine3* e, uint64_t* s) {
  *s = (uint64_t)(uintptr_t)e->s;
  return TMG_OK;
}

int e3_history(Engine3* e, int count, tmg_stats* out, std::string& err) {
  ErrScope es(e, err);
  if (count < 0 || count > e->cap || count > e->host_counter) return fail3(e, TMG_EINVAL, "bad history count");
  return read_stats(e, e->host_counter - count, count, out);
}

int e3_cycle_state(Engine3* e, int64_t* count, int32_t* parity, int set, std::string& err) {
  ErrScope es(e, err);
  if (!e->sharded) return fail3(e, TMG_EINVAL, "handle is not sharded (tmg3_shard)");
  if (!set) {
    *count = e->host_counter;
    *parity = e->par;
    return TMG_OK;
  }
  if (*count < 0 || (*parity != 0 && *parity != 1)) return fail3(e, TMG_EINVAL, "bad cycle state");
  e->host_counter = *count;
  if (e->pp && *parity != e->par) pp_advance(e);
  return TMG_OK;
}

// one cycle from the graph of the current state (+ the fused-pass state machine)
int launch_cycle(Engine3* e) {
  TRY3(ensure_graph(e));
  if (e->thr_next >= e->lmin) {  // throttled setup: one more BoxMG level before this cycle
    TRY3(boxmg_level(e, e->thr_next));
    TRY3(check_degenerate(e));
    --e->thr_next;
  }
  CK3(cudaGraphLaunch(e->gexec, e->s));
  pp_advance(e);
  return TMG_OK;
}

// ============================================================================
// internal interface (engine3.h)
// ============================================================================

int e3_create(const tmg_tree3* t, const tmg_config* cfg, Engine3** out, std::string& err) {
  Engine3* e = new Engine3();
  ErrScope es(e, err);
  e->cfg = *cfg;
  e->wt = std::isnan(cfg->omega_tilde) ? cfg->omega : cfg->omega_tilde;
  if (cudaStreamCreateWithFlags(&e->s, cudaStreamNonBlocking) != cudaSuccess) {
    err = "stream creation failed";
    delete e;
    return TMG_ECUDA;
  }
  int rc = build(e, t);
  if (rc != TMG_OK) {
    e->err = nullptr;
    e3_destroy(e);
    return rc;
  }
  *out = e;
  return TMG_OK;
}

int e3_rebuild(Engine3* e, const tmg_tree3* t, std::string& err) {
  ErrScope es(e, err);
  CK3(cudaStreamSynchronize(e->s));
  free3(e);
  return build(e, t);
}

void e3_destroy(Engine3* e) {
  if (!e) return;
  if (e->s) cudaStreamSynchronize(e->s);
  free3(e);
  for (auto q : e->ev_pool) cudaEventDestroy(q);
  if (e->flush_buf) cudaFree(e->flush_buf);
  if (e->s) cudaStreamDestroy(e->s);
  delete e;
}

int e3_set_rhs(Engine3* e, int level, const double* rhs, std::string& err) {
  ErrScope es(e, err);
  TRY3(check_level(e, level));
  Lvl3& c = e->L[level];
  if (!rhs) {
    if (c.rhs) {
      c.rhs = nullptr;
      e->graph_dirty = true;
    }
    return TMG_OK;
  }
  if (!c.rhs) {
    TRY3(alloc3(e, &c.rhs, c.nv, false));
    e->graph_dirty = true;
  }
  CK3(cudaMemcpyAsync(c.rhs, rhs, sizeof(double) * c.nv, cudaMemcpyHostToDevice, e->s));
  CK3(cudaStreamSynchronize(e->s));
  return TMG_OK;
}

int e3_set_u(Engine3* e, int level, const double* u, std::string& err) {
  ErrScope es(e, err);
  TRY3(check_level(e, level));
  CK3(cudaMemcpyAsync(e->L[level].u, u, sizeof(double) * e->L[level].nv, cudaMemcpyHostToDevice, e->s));
  if (e->pp && level == e->ltop) {
    // the other buffer takes the boundary (Dirichlet) values: the down sweep writes every interior vertex
    const int N = e->L[level].N;
    k3_copy_boundary<<<nblk((size_t)N * N), 256, 0, e->s>>>(e->ubuf[e->par ^ 1], e->L[level].u, N);
    CKL3();
  }
  CK3(cudaStreamSynchronize(e->s));
  return TMG_OK;
}

int e3_get_u(Engine3* e, int level, double* u, std::string& err) {
  ErrScope es(e, err);
  TRY3(check_level(e, level));
  CK3(cudaMemcpyAsync(u, e->L[level].u, sizeof(double) * e->L[level].nv, cudaMemcpyDeviceToHost, e->s));
  CK3(cudaStreamSynchronize(e->s));
  return TMG_OK;
}

int e3_update_fas_state(Engine3* e, std::string& err) {
  ErrScope es(e, err);
  for (int l = e->ltop - 1; l >= e->lmin; --l) {
    const int n = e->L[l].N - 2;
    if (n <= 0) continue;
    k3_inject<<<nblk((size_t)n * n * n), 256, 0, e->s>>>(e->L[l].u, e->L[l].N, e->L[l + 1].u, e->L[l + 1].N);
    CKL3();
  }
  CK3(cudaStreamSynchronize(e->s));
  return TMG_OK;
}

int e3_cycle(Engine3* e, int ncycles, tmg_stats* stats, std::string& err) {
  ErrScope es(e, err);
  if (ncycles < 0) return fail3(e, TMG_EINVAL, "negative cycle count");
  TRY3(ensure_graph(e));
  int done = 0;
  while (done < ncycles) {
    const int chunk = std::min(ncycles - done, e->cap);
    const long long first = e->host_counter;
    for (int k = 0; k < chunk; ++k) TRY3(launch_cycle(e));
    e->host_counter += chunk;
    if (stats) TRY3(read_stats(e, first, chunk, stats + done));
    else CK3(cudaStreamSynchronize(e->s));
    done += chunk;
  }
  return TMG_OK;
}

int e3_residual_stats(Engine3* e, tmg_stats* out, std::string& err) {
  ErrScope es(e, err);
  TRY3(enqueue_down(e, false));
  const long long first = e->host_counter++;
  return read_stats(e, first, 1, out);
}

int e3_levels(Engine3* e, int32_t* lmin, int32_t* ltop) {
  if (lmin) *lmin = e->lmin;
  if (ltop) *ltop = e->ltop;
  return TMG_OK;
}

int e3_level_counts(Engine3* e, int level, int64_t* dof, int64_t* composite, int64_t* hanging,
                    std::string& err) {
  ErrScope es(e, err);
  TRY3(check_level(e, level));
  const long long n = e->L[level].N - 2;
  if (dof) *dof = n * n * n;
  if (composite) *composite = (level == e->ltop) ? n * n * n : 0;
  if (hanging) *hanging = 0;
  return TMG_OK;
}

int e3_get_kinds(Engine3* e, int level, int8_t* out, std::string& err) {
  ErrScope es(e, err);
  TRY3(check_level(e, level));
  const int N = e->L[level].N;
  const int8_t inner = (level == e->ltop) ? 1 : 4;  // INTERIOR_DOF / COARSE_OVERLAPPED
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j)
      for (int k = 0; k < N; ++k) {
        const bool b = i == 0 || j == 0 || k == 0 || i == N - 1 || j == N - 1 || k == N - 1;
        out[((size_t)i * N + j) * N + k] = b ? 2 : inner;
      }
  return TMG_OK;
}

int e3_get_table(Engine3* e, int which, int level, double* out, std::string& err) {
  ErrScope es(e, err);
  TRY3(check_level(e, level));
  Lvl3& c = e->L[level];
  auto fetch = [&](const double* src, size_t count, std::vector<double>& dst) -> int {
    dst.resize(count);
    CK3(cudaMemcpyAsync(dst.data(), src, sizeof(double) * count, cudaMemcpyDeviceToHost, e->s));
    CK3(cudaStreamSynchronize(e->s));
    return TMG_OK;
  };
  std::vector<double> buf;
  switch (which) {
    case TMG_TABLE_EFFEPS:
      TRY3(fetch(c.eff, c.ncell, buf));
      std::memcpy(out, buf.data(), sizeof(double) * c.ncell);
      return TMG_OK;
    case TMG_TABLE_A: {
      const double* src = c.tbl;
      if (!src) {
        double* tmp;
        TRY3(alloc3(e, &tmp, 27 * c.nv, false));
        k3_assemble<<<nblk(c.nv), 256, 0, e->s>>>(tmp, Rows{c.N, nullptr, c.coef});
        CKL3();
        src = tmp;
      }
      TRY3(fetch(src, 27 * c.nv, buf));
      for (size_t v = 0; v < c.nv; ++v)
        for (int k = 0; k < 27; ++k) out[v * 27 + k] = buf[k * c.nv + v];
      return TMG_OK;
    }
    case TMG_TABLE_P: {
      if (!c.P) return fail3(e, TMG_EINVAL, "no P table on this level");
      TRY3(fetch(c.P, 125 * c.nv, buf));
      for (size_t v = 0; v < c.nv; ++v)
        for (int k = 0; k < 125; ++k) out[v * 125 + k] = buf[k * c.nv + v];
      return TMG_OK;
    }
    default:
      return fail3(e, TMG_EINVAL, "table not available in 3D");
  }
}

int e3_time_cycles(Engine3* e, int ncycles, int64_t flush_bytes, float* ms, std::string& err) {
  ErrScope es(e, err);
  TRY3(ensure_graph(e));
  if (flush_bytes > 0 && e->flush_bytes < (size_t)flush_bytes) {
    if (e->flush_buf) cudaFree(e->flush_buf);
    e->flush_buf = nullptr;
    CK3(cudaMalloc(&e->flush_buf, (size_t)flush_bytes));
    e->flush_bytes = (size_t)flush_bytes;
  }
  const int ne = flush_bytes > 0 ? 2 * ncycles : 2;
  std::vector<cudaEvent_t> ev(ne);
  for (auto& q : ev) CK3(cudaEventCreate(&q));
  CK3(cudaStreamSynchronize(e->s));
  if (flush_bytes > 0) {
    for (int k = 0; k < ncycles; ++k) {
      CK3(cudaMemsetAsync(e->flush_buf, k & 0xff, (size_t)flush_bytes, e->s));
      CK3(cudaEventRecord(ev[2 * k], e->s));
      TRY3(launch_cycle(e));
      CK3(cudaEventRecord(ev[2 * k + 1], e->s));
    }
  } else {
    CK3(cudaEventRecord(ev[0], e->s));
    for (int k = 0; k < ncycles; ++k) TRY3(launch_cycle(e));
    CK3(cudaEventRecord(ev[1], e->s));
  }
  CK3(cudaStreamSynchronize(e->s));
  e->host_counter += ncycles;
  float total = 0.f;
  for (int k = 0; k < ne / 2; ++k) {
    float t = 0.f;
    CK3(cudaEventElapsedTime(&t, ev[2 * k], ev[2 * k + 1]));
    total += t;
  }
  *ms = total;
  for (auto& q : ev) cudaEventDestroy(q);
  return TMG_OK;
}

int e3_profile_cycles(Engine3* e, int ncycles, int cap, const char** names, float* ms,
                      int32_t* launches, int32_t* nk, std::string& err) {
  ErrScope es(e, err);
  std::vector<KT> timers;
  e->profiling = true;
  int rc = TMG_OK;
  for (int k = 0; k < ncycles && rc == TMG_OK; ++k) {
    rc = enqueue_cycle(e);
    pp_advance(e);
    e->host_counter++;
  }
  e->profiling = false;
  if (rc == TMG_OK) {
    if (cudaStreamSynchronize(e->s) != cudaSuccess) rc = fail3(e, TMG_ECUDA, "profile sync failed");
    for (auto& p : e->pending) {
      float t = 0.f;
      cudaEventElapsedTime(&t, p.e0, p.e1);
      bool found = false;
      for (auto& q : timers)
        if (std::strcmp(q.name, p.name) == 0) {
          q.ms += t;
          q.launches++;
          found = true;
          break;
        }
      if (!found) timers.push_back({p.name, t, 1});
    }
  }
  e->pending.clear();
  e->ev_used = 0;
  if (rc != TMG_OK) return rc;
  int n = 0;
  for (auto& q : timers) {
    if (n >= cap) break;
    names[n] = q.name;
    ms[n] = q.ms;
    launches[n] = q.launches;
    ++n;
  }
  *nk = n;
  return TMG_OK;
}

int e3_launches_per_cycle(Engine3* e, int32_t* n, std::string& err) {
  ErrScope es(e, err);
  TRY3(ensure_graph(e));
  *n = e->launches;
  return TMG_OK;
}

