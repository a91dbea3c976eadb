// Host runtime of libtmg.so: level hierarchy in HBM, operator setup, the
// per-cycle launch sequence captured in a CUDA graph, and the C ABI declared
// in include/tmg.h (each entry cites the ReferenceEngine method it replaces).
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

// single translation unit: the kernels and their __constant__ tables live here too
#include "kernels2d.cu"
#include "engine3.h"
#include "tmg.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(TMG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define CKL()                                                                           \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return fail(TMG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_));  \
  } while (0)

#define TRY(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ != TMG_OK) return rc_; \
  } while (0)

inline unsigned nblk(size_t n) { return (unsigned)((n + tmg::kBlock - 1) / tmg::kBlock); }

// Levels with at most kSmallLevel vertices run in the one-block coarse-chain kernel.
constexpr size_t kSmallLevel = 1024;

int ipow3(int l) {
  int r = 1;
  for (int k = 0; k < l; ++k) r *= 3;
  return r;
}

struct Level {
  int l = 0, n = 0, N = 0;
  size_t nv = 0, ncell = 0;
  uint8_t* flags = nullptr;
  uint8_t* refined = nullptr;  // refined[l] on device (nullptr: none refined / l >= lmax)
  bool any_refined = false;
  double *u = nullptr, *rhs = nullptr, *rho = nullptr, *rdof = nullptr, *g = nullptr;
  double *carry = nullptr, *inj = nullptr, *diag = nullptr, *diag_raw = nullptr;
  double *eff = nullptr, *epsm = nullptr, *reff = nullptr, *tbl = nullptr, *P = nullptr, *Rt = nullptr;
  tmg::OpView op{tmg::OP_NONE, 0, 0, nullptr, nullptr};
  tmg::OpView rop{tmg::OP_NONE, 0, 0, nullptr, nullptr};
  int rt_mode = tmg::RT_NONE;
  long long cnt[8] = {0};
  double w_l = 0.0, hA = 0.0, hB = 0.0;
  int part_off = 0, nblocks = 0;
  // patch list of an adaptive level (kernels2d.cu: tile_origin): the vertex tiles holding an
  // existing vertex, in row-major tile order; nullptr when every vertex of the level exists
  uint32_t* tiles = nullptr;
  int ntiles = 0, tile_h = 0;
};

struct KTimer {
  const char* name;
  float ms;
  int launches;
};

}  // namespace

struct tmg_handle {
  Engine3* e3 = nullptr;  // 3D hierarchy (engine3.cu); the 2D fields are unused then
  tmg_config cfg{};
  double wt = 0.0;
  int lmin = 1, lmax = 1, ltop = 0;
  std::vector<Level> L;
  double* u_below = nullptr;  // u[lmin-1] (hanging refresh at lmin)
  int N_below = 0;
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
  // profiling hooks (non-graph path)
  bool profiling = false;
  std::vector<KTimer>* timers = nullptr;
  std::vector<cudaEvent_t> ev_pool;
  int ev_used = 0;
  struct Pending {
    const char* name;
    cudaEvent_t e0, e1;
  };
  std::vector<Pending> pending;
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  // coarse chain (cluster kernel) and its argument blocks
  int lc = 0, part_base = 0;
  // fused cycle (k_cycle): per-warp stats partials, grid barrier words, persistent grid size
  double* wpart = nullptr;
  unsigned* bar = nullptr;
  int cycle_grid = 0;
  unsigned long long* stamps = nullptr;  // k_coarse phase timestamps (diagnostics)
  double* scratch = nullptr;             // per-CTA residual partials of the cluster chain
};

namespace {

template <class T>
int dalloc(tmg_handle* h, T** p, size_t count) {
  void* q = nullptr;
  CK(cudaMalloc(&q, sizeof(T) * (count ? count : 1)));
  h->allocs.push_back(q);
  *p = (T*)q;
  return TMG_OK;
}

void free_all(tmg_handle* h) {
  if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
  for (void* p : h->allocs) cudaFree(p);
  h->allocs.clear();
  h->L.clear();
  h->u_below = nullptr;
  h->graph_dirty = true;
}

// --- launch helpers with optional per-kernel timing -------------------------

// Profiling records an event pair around every launch and resolves all of
// them after one synchronisation at the end (no per-launch host sync).
int begin_k(tmg_handle* h, const char* name, cudaEvent_t* e0) {
  if (!h->profiling) return TMG_OK;
  if (h->ev_used + 2 > (int)h->ev_pool.size()) {
    for (int k = 0; k < 256; ++k) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      h->ev_pool.push_back(e);
    }
  }
  *e0 = h->ev_pool[h->ev_used++];
  CK(cudaEventRecord(*e0, h->s));
  (void)name;
  return TMG_OK;
}

int end_k(tmg_handle* h, const char* name, cudaEvent_t e0) {
  h->launches++;
  if (!h->profiling) return TMG_OK;
  cudaEvent_t e1 = h->ev_pool[h->ev_used++];
  CK(cudaEventRecord(e1, h->s));
  h->pending.push_back({name, e0, e1});
  return TMG_OK;
}

int resolve_timers(tmg_handle* h) {
  CK(cudaStreamSynchronize(h->s));
  for (auto& p : h->pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.e0, p.e1));
    bool found = false;
    for (auto& t : *h->timers)
      if (std::strcmp(t.name, p.name) == 0) { t.ms += ms; t.launches++; found = true; break; }
    if (!found) h->timers->push_back({p.name, ms, 1});
  }
  h->pending.clear();
  h->ev_used = 0;
  return TMG_OK;
}

// static per-level kernel names for the profiler
const char* lvl_name(const char* base, int l) {
  static char names[8][16][24];
  static const char* bases[8] = {"k_down", "k_up", "k_inject_u", "k_hang", "k_inject_d", "", "", ""};
  int b = 0;
  while (b < 5 && std::strcmp(bases[b], base) != 0) ++b;
  if (b >= 5 || l < 0 || l > 15) return base;
  if (!names[b][l][0]) std::snprintf(names[b][l], 24, "%s_L%d", base, l);
  return names[b][l];
}

#define LAUNCH(h, name, kernel, grid, ...)                         \
  do {                                                             \
    cudaEvent_t e0_ = nullptr;                                     \
    TRY(begin_k(h, name, &e0_));                                   \
    kernel<<<(grid), tmg::kBlock, 0, (h)->s>>>(__VA_ARGS__);       \
    CKL();                                                         \
    TRY(end_k(h, name, e0_));                                      \
  } while (0)

// 32 x 8 vertex tiles of the grid kernels (k_down, k_up)
inline unsigned tiles_x(int N) { return (unsigned)((N + tmg::kTileX - 1) / tmg::kTileX); }
inline unsigned tiles_y(int N, int ty = tmg::kTileY) { return (unsigned)((N + ty - 1) / ty); }

// Coarse grid levels run 32 x kCoarseTileY tiles: their per-vertex work is
// heavy (BoxMG restriction + R~ from P, ~200 registers) and they have few
// vertices, so small CTAs spread them over more SMs (measured at config 2: 2
// beats 1, 4 and 8).
constexpr int kCoarseTileY = 2;

// one block per vertex tile of level LV: its patch list when it has one, else the dense tile grid
#define LAUNCH_TILES(h, name, kernel, LV, TY, ...)                                               \
  do {                                                                                           \
    cudaEvent_t e0_ = nullptr;                                                                   \
    TRY(begin_k(h, name, &e0_));                                                                 \
    const dim3 grid_ = (LV).tiles ? dim3((unsigned)(LV).ntiles) : dim3(tiles_x((LV).N), tiles_y((LV).N, TY)); \
    kernel<<<grid_, dim3(tmg::kTileX, (TY)), 0, (h)->s>>>(__VA_ARGS__);                          \
    CKL();                                                                                       \
    TRY(end_k(h, name, e0_));                                                                    \
  } while (0)

// Patch list of an adaptive level (north star: "hanging-vertex handling for adaptive grids, via
// per-level patch lists"; the reference keeps dense per-level arrays and masks, spacetree.py:
// 164-191 / solvers.py:179-192): the row-major list of vertex tiles with an existing vertex.
// The cycle kernels of the level launch one block per listed tile, so a level refined along a
// thin feature (config 4's level 8: 7 % of the vertex slots exist) costs its patches, not its
// bounding box; its partial-sum slots shrink with it.
int build_patch_list(tmg_handle* h, Level& c) {
  const int tx = (int)tiles_x(c.N), ty = (int)tiles_y(c.N, c.tile_h), nt = tx * ty;
  uint8_t* mask = nullptr;
  TRY(dalloc(h, &mask, (size_t)nt));
  tmg::k_tile_any<<<nblk((size_t)nt), 256, 0, h->s>>>(c.flags, c.N, c.tile_h, tx, ty, mask);
  CKL();
  std::vector<uint8_t> hm((size_t)nt);
  CK(cudaMemcpyAsync(hm.data(), mask, (size_t)nt, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  std::vector<uint32_t> list;
  for (int t = 0; t < nt; ++t)
    if (hm[(size_t)t]) list.push_back(((uint32_t)(t / tx) << 16) | (uint32_t)(t % tx));
  if (list.empty() || (int)list.size() == nt || ty > 0xffff) return TMG_OK;  // dense grid
  TRY(dalloc(h, &c.tiles, list.size()));
  CK(cudaMemcpyAsync(c.tiles, list.data(), sizeof(uint32_t) * list.size(), cudaMemcpyHostToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  c.ntiles = (int)list.size();
  c.nblocks = c.ntiles;
  return TMG_OK;
}

// --- the cycle --------------------------------------------------------------
//
// Levels above lc ("grid levels") get one grid-wide launch per sweep; the
// coarse chain lmin..lc runs in one thread-block-cluster launch (k_coarse).
// Per cycle: (ltop - lc) k_down + 1 k_coarse + (ltop - lc) k_up (+ k_hang on
// levels with hanging vertices).

tmg::DownArgs make_down(tmg_handle* h, int l, bool write) {
  const int l0 = h->lmin, l1 = h->ltop;
  Level& c = h->L[l];
  tmg::DownArgs a{};
  a.N = c.N;
  a.is_top = (l == l1);
  a.variant = h->cfg.variant;
  a.write = write ? 1 : 0;
  a.tiles = c.tiles;
  a.u = c.u;
  a.flags = c.flags;
  a.diag = c.diag;
  a.op = c.op;
  a.rop = c.rop;
  a.rhs = c.rhs;
  if (l < l1) {
    Level& f = h->L[l + 1];
    a.Nf = f.N;
    a.rho_f = f.rho;
    a.rdof_f = f.rdof;
    a.boxmg = h->cfg.flavor == TMG_BOXMG;
    a.P = c.P;
    a.Rt = c.Rt;
    // R~ rebuilt from the P registers (RT_FROM_P) beat reading the stored
    // table on every level of config 2 (measured)
    a.rt_mode = c.rt_mode;
    const double c1 = 1.0 / 3.0;  // interior_stencil(1.0) (discretization.py:165-167)
    a.rt_side = c1 * -1.0;
    a.rt_mid = c1 * 8.0;
    a.rt_scale = h->cfg.omega * 3.0 / 8.0;  // operators.py:604
    a.rt_omega = h->cfg.omega;               // operators.py:546
  }
  a.w_l = c.w_l;
  a.omega = h->cfg.omega;
  a.wt = h->wt;
  a.ds = h->cfg.damping_scale;
  a.hA = c.hA;
  a.hB = c.hB;
  a.rho = (l > l0) ? c.rho : nullptr;
  a.rdof = (l > l0) ? c.rdof : nullptr;
  a.g = c.g;
  a.part_sum = h->part_sum + c.part_off;
  a.part_max = h->part_max + c.part_off;
  return a;
}

tmg::UpArgs make_up(tmg_handle* h, int l) {
  const int l0 = h->lmin, l1 = h->ltop;
  Level& c = h->L[l];
  tmg::UpArgs a{};
  a.l = l;
  a.l0 = l0;
  a.N = c.N;
  a.is_bottom = (l == l0);
  a.tiles = c.tiles;
  a.boxmg = h->cfg.flavor == TMG_BOXMG;
  a.pi = h->cfg.variant == tmg::VAR_PI;
  a.flags = c.flags;
  a.u = c.u;
  a.g = c.g;
  a.carry = (l < l1) ? c.carry : nullptr;
  if (l > l0) {
    Level& cc = h->L[l - 1];
    a.Nc = cc.N;
    a.carry_c = cc.carry;
    a.P = cc.P;
    a.flags_c = cc.flags;
  }
  a.ds = h->cfg.damping_scale;
  for (int k = l0; k < l; ++k) {
    a.ul[k] = h->L[k].u;
    a.fl[k] = h->L[k].flags;
    a.Nl[k] = h->L[k].N;
  }
  return a;
}

// the coarse chain runs on a thread-block cluster (53 -> 41 us at config 2 against one CTA)
constexpr bool kChainCluster = true;

int launch_coarse(tmg_handle* h, bool write) {
  tmg::CoarseArgs a{};
  a.l0 = h->lmin;
  a.lc = h->lc;
  a.part_sum = h->part_sum;
  a.part_max = h->part_max;
  a.part_base = h->part_base;
  a.hist = h->hist;
  a.counter = h->counter;
  a.cap = h->cap;
  a.do_up = write ? 1 : 0;
  a.stamps = h->stamps;
  for (int l = h->lmin; l <= h->lc; ++l) {
    a.down[l - h->lmin] = make_down(h, l, write);
    a.up[l - h->lmin] = make_up(h, l);
  }
  cudaEvent_t e0 = nullptr;
  TRY(begin_k(h, "k_coarse", &e0));
  if (kChainCluster) {
    // the chain on one thread-block cluster of kClusterCTAs CTAs
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(tmg::kClusterCTAs);
    lc.blockDim = dim3(tmg::kCoarseBlock);
    lc.stream = h->s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = tmg::kClusterCTAs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, tmg::k_coarse_cl, a, h->scratch));
  } else {
    tmg::k_coarse<<<1, tmg::kCoarseBlock, 0, h->s>>>(a);
  }
  CKL();
  TRY(end_k(h, "k_coarse", e0));
  return TMG_OK;
}

int enqueue_down(tmg_handle* h, bool write) {
  for (int l = h->ltop; l > h->lc; --l) {
    tmg::DownArgs a = make_down(h, l, write);
    if (l == h->ltop)
      LAUNCH_TILES(h, lvl_name("k_down", l), tmg::k_down<1>, h->L[l], tmg::kTileY, a);
    else
      LAUNCH_TILES(h, lvl_name("k_down", l), tmg::k_down<0>, h->L[l], kCoarseTileY, a);
  }
  TRY(launch_coarse(h, write));
  return TMG_OK;
}

int enqueue_hang(tmg_handle* h) {
  const int l0 = h->lmin, l1 = h->ltop;
  for (int l = l0; l <= l1; ++l) {
    Level& c = h->L[l];
    if (c.cnt[tmg::K_HANG] == 0) continue;
    const double* uc = (l == l0) ? h->u_below : h->L[l - 1].u;
    const int Nc = (l == l0) ? h->N_below : h->L[l - 1].N;
    if (c.tiles) {
      if (c.tile_h == tmg::kTileY)
        LAUNCH_TILES(h, lvl_name("k_hang", l), tmg::k_hang_tiles, c, tmg::kTileY, c.u, c.flags, c.N, uc, Nc, c.tiles);
      else
        LAUNCH_TILES(h, lvl_name("k_hang", l), tmg::k_hang_tiles, c, kCoarseTileY, c.u, c.flags, c.N, uc, Nc, c.tiles);
    } else {
      LAUNCH(h, lvl_name("k_hang", l), tmg::k_hang, nblk(c.nv), c.u, c.flags, c.N, uc, Nc);
    }
  }
  return TMG_OK;
}

// update_fas_state() on its own (solvers.py:280-296)
int enqueue_fas(tmg_handle* h) {
  const int l0 = h->lmin, l1 = h->ltop;
  for (int l = l1 - 1; l >= l0; --l) {
    Level& c = h->L[l];
    Level& f = h->L[l + 1];
    LAUNCH(h, lvl_name("k_inject_u", l), tmg::k_inject_u, nblk(c.nv), c.u, c.flags, c.N, f.u, f.N);
  }
  return enqueue_hang(h);
}

// The whole cycle in one persistent cooperative launch (k_cycle, cfg.fused_cycle).
int launch_cycle(tmg_handle* h) {
  const int l0 = h->lmin, l1 = h->ltop;
  tmg::CycleArgs a{};
  a.l0 = l0;
  a.ltop = l1;
  a.do_up = 1;
  a.hist = h->hist;
  a.counter = h->counter;
  a.cap = h->cap;
  a.wpart = h->wpart;
  a.bar = h->bar;
  a.stamps = h->stamps;
  for (int l = l0; l <= l1; ++l) {
    Level& c = h->L[l];
    const int k = l - l0;
    a.down[k] = make_down(h, l, true);
    a.up[k] = make_up(h, l);
    a.tile_h[k] = c.tiles ? c.tile_h : 1;
    a.units[k] = c.tiles ? c.ntiles * c.tile_h : c.N * (int)tiles_x(c.N);
    if (c.cnt[tmg::K_HANG] > 0) {
      a.hang_lv[a.nhang++] = k;
      a.hang[k].u = c.u;
      a.hang[k].flags = c.flags;
      a.hang[k].N = c.N;
      a.hang[k].uc = (l == l0) ? h->u_below : h->L[l - 1].u;
      a.hang[k].Nc = (l == l0) ? h->N_below : h->L[l - 1].N;
    }
  }
  cudaEvent_t e0 = nullptr;
  TRY(begin_k(h, "k_cycle", &e0));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)h->cycle_grid);
  lc.blockDim = dim3(tmg::kTileX, tmg::kTileY);
  lc.stream = h->s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CK(cudaLaunchKernelEx(&lc, tmg::k_cycle, a));
  CKL();
  TRY(end_k(h, "k_cycle", e0));
  return TMG_OK;
}

int enqueue_cycle(tmg_handle* h) {
  if (h->cfg.fused_cycle) return launch_cycle(h);
  TRY(enqueue_down(h, true));  // includes the coarse chain (down, stats, up)
  for (int l = h->lc + 1; l <= h->ltop; ++l) {
    tmg::UpArgs a = make_up(h, l);
    if (l == h->ltop) LAUNCH_TILES(h, lvl_name("k_up", l), tmg::k_up, h->L[l], tmg::kTileY, a);
    else LAUNCH_TILES(h, lvl_name("k_up", l), tmg::k_up, h->L[l], kCoarseTileY, a);
  }
  TRY(enqueue_hang(h));  // injection rides in k_up / k_coarse
  return TMG_OK;
}

int ensure_graph(tmg_handle* h) {
  if (!h->graph_dirty && h->gexec) return TMG_OK;
  if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
  h->launches = 0;
  int rc = enqueue_cycle(h);
  cudaError_t e = cudaStreamEndCapture(h->s, &g);
  if (rc != TMG_OK) return rc;
  CK(e);
  CK(cudaGraphInstantiate(&h->gexec, g, 0));
  cudaGraphDestroy(g);
  h->graph_dirty = false;
  return TMG_OK;
}

// --- setup (ReferenceEngine.rebuild, solvers.py:145-255) ---------------------

int check_const(tmg_handle* h, const double* arr, size_t n, bool* is_const, double* value) {
  int* flag;
  TRY(dalloc(h, &flag, 1));
  const int one = 1;
  CK(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, h->s));
  tmg::k_const_check<<<nblk(n), tmg::kBlock, 0, h->s>>>(arr, n, flag);
  CKL();
  int hf = 0;
  CK(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, h->s));
  CK(cudaMemcpyAsync(value, arr, sizeof(double), cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  *is_const = hf != 0;
  return TMG_OK;
}

tmg::OpView element_op(double c, bool is_const, const double* eps) {
  tmg::OpView o{};
  if (is_const) {
    o.kind = tmg::OP_CONST;
    const double c3 = c / 3.0;  // interior_stencil: eps / 3.0 * [...] (discretization.py:165-167)
    o.s_side = c3 * -1.0;
    o.s_mid = c3 * 8.0;
  } else {
    o.kind = tmg::OP_ELEMENT;
    o.eps = eps;
  }
  return o;
}

int build(tmg_handle* h, const tmg_tree* t) {
  const tmg_config& cfg = h->cfg;
  h->lmin = t->lmin;
  h->lmax = t->lmax;
  if (t->lmin < 1) return fail(TMG_EINVAL, "lmin must be at least 1");
  if (t->lmax < t->lmin) return fail(TMG_EINVAL, "lmax must not be smaller than lmin");
  // depth = finest level with existing cells (spacetree.py:130-136)
  auto any_ref = [&](int l) -> bool {
    if (l >= t->lmax || !t->refined || !t->refined[l]) return false;
    const size_t n = (size_t)ipow3(l) * ipow3(l);
    for (size_t k = 0; k < n; ++k)
      if (t->refined[l][k]) return true;
    return false;
  };
  int depth = 0;
  for (int l = t->lmax - 1; l >= 0; --l)
    if (any_ref(l)) { depth = l + 1; break; }
  h->ltop = depth;
  if (depth < t->lmin) return fail(TMG_EINVAL, "tree has no DoF-carrying level at or above lmin");
  if (t->nlevels < depth + 1) return fail(TMG_EINVAL, "tree.u / tree.eps must hold levels 0..depth");
  if (depth > 12) return fail(TMG_EINVAL, "depth above 12 is not supported in 2D");
  const int l0 = t->lmin, l1 = depth;
  h->L.assign(l1 + 1, Level{});
  // refined bitmaps for levels l0-1 .. l1
  std::vector<uint8_t*> dref(l1 + 1, nullptr);
  for (int l = std::max(l0 - 1, 0); l <= l1; ++l) {
    if (!any_ref(l)) continue;
    const size_t n = (size_t)ipow3(l) * ipow3(l);
    TRY(dalloc(h, &dref[l], n));
    CK(cudaMemcpyAsync(dref[l], t->refined[l], n, cudaMemcpyHostToDevice, h->s));
  }
  // per-level storage + classification
  for (int l = l0; l <= l1; ++l) {
    Level& c = h->L[l];
    c.l = l;
    c.n = ipow3(l);
    c.N = c.n + 1;
    c.nv = (size_t)c.N * c.N;
    c.ncell = (size_t)c.n * c.n;
    c.refined = dref[l];
    c.any_refined = dref[l] != nullptr;
    TRY(dalloc(h, &c.flags, c.nv));
    const uint8_t* rp = (l >= 1) ? dref[l - 1] : nullptr;
    if (l >= 1 && !rp) {
      // no cell of level l-1 refined: level l has no cells at all
      CK(cudaMemsetAsync(c.flags, 0, c.nv, h->s));
    } else {
      tmg::k_flags<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.flags, c.n, rp, dref[l]);
      CKL();
    }
  }
  for (int l = l0; l < l1; ++l) {
    tmg::k_take<<<nblk(h->L[l].nv), tmg::kBlock, 0, h->s>>>(h->L[l].flags, h->L[l].N,
                                                             h->L[l + 1].flags, h->L[l + 1].N);
    CKL();
  }
  unsigned long long* dcnt;
  TRY(dalloc(h, &dcnt, 8 * (l1 + 1)));
  CK(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * 8 * (l1 + 1), h->s));
  for (int l = l0; l <= l1; ++l) {
    tmg::k_count_kinds<<<nblk(h->L[l].nv), tmg::kBlock, 0, h->s>>>(h->L[l].flags, h->L[l].nv,
                                                                    dcnt + 8 * l);
    CKL();
  }
  std::vector<unsigned long long> hcnt(8 * (l1 + 1));
  CK(cudaMemcpyAsync(hcnt.data(), dcnt, sizeof(unsigned long long) * hcnt.size(),
                     cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->dofs_total = 0;
  long long dof_sum = 0, dof_lt = 0, dof_gt = 0;
  for (int l = l0; l <= l1; ++l) {
    Level& c = h->L[l];
    for (int k = 0; k < 8; ++k) c.cnt[k] = (long long)hcnt[8 * l + k];
    const long long dof = c.cnt[tmg::K_DOF] + c.cnt[tmg::K_OVER];
    h->dofs_total += c.cnt[tmg::K_DOF];
    dof_sum += dof;
    if (l < l1) dof_lt += dof;
    if (l > l0) dof_gt += dof;
  }
  // _count_updates (solvers.py:449-459)
  h->updates = dof_sum;
  if (cfg.variant == tmg::VAR_JAC) h->updates += dof_lt;
  if (cfg.variant == tmg::VAR_PI) h->updates += dof_gt;

  // eff_eps top-down (solvers.py:165-175), eps_masked, refined-op eps
  double* eps_tmp;
  TRY(dalloc(h, &eps_tmp, h->L[l1].ncell));
  for (int l = l1; l >= l0; --l) {
    Level& c = h->L[l];
    if (!t->eps || !t->eps[l]) return fail(TMG_EINVAL, "tree.eps missing a level");
    CK(cudaMemcpyAsync(eps_tmp, t->eps[l], sizeof(double) * c.ncell, cudaMemcpyHostToDevice, h->s));
    TRY(dalloc(h, &c.eff, c.ncell));
    TRY(dalloc(h, &c.epsm, c.ncell));
    const bool has_rop = (l < t->lmax) && c.any_refined;
    if (has_rop) TRY(dalloc(h, &c.reff, c.ncell));
    const double* child = (c.any_refined && l < l1) ? h->L[l + 1].eff : nullptr;
    tmg::k_eff<<<nblk(c.ncell), tmg::kBlock, 0, h->s>>>(c.eff, c.epsm, c.reff, eps_tmp, child,
                                                         child ? c.refined : nullptr,
                                                         l >= 1 ? dref[l - 1] : nullptr, c.n);
    CKL();
    CK(cudaStreamSynchronize(h->s));  // eps_tmp reused
    if (has_rop) {
      bool kc;
      double v;
      TRY(check_const(h, c.reff, c.ncell, &kc, &v));
      c.rop = element_op(v, kc, c.reff);
    }
  }
  // mesh widths and per-level weights
  for (int l = l0; l <= l1; ++l) {
    Level& c = h->L[l];
    c.hA = std::pow(3.0, -(double)(l + 1));
    c.hB = std::pow(3.0, -(double)l);
    c.w_l = (cfg.variant == tmg::VAR_EXP) ? std::pow(cfg.omega_hat, (double)(l1 - l)) : cfg.omega;
    TRY(dalloc(h, &c.diag, c.nv));
    TRY(dalloc(h, &c.diag_raw, c.nv));
  }
  const bool jac = cfg.variant == tmg::VAR_JAC;
  int* deg;
  TRY(dalloc(h, &deg, 1));
  CK(cudaMemsetAsync(deg, 0, sizeof(int), h->s));
  if (cfg.flavor == TMG_GEOMETRIC) {
    for (int l = l0; l <= l1; ++l) {
      Level& c = h->L[l];
      bool kc;
      double v;
      TRY(check_const(h, c.epsm, c.ncell, &kc, &v));
      c.op = element_op(v, kc, c.epsm);
      tmg::k_elem_diag<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.diag_raw, c.diag, c.epsm, c.flags, c.n);
      CKL();
    }
    if (jac) {
      double* tf = nullptr;
      if (cfg.rtilde_true_operator) TRY(dalloc(h, &tf, 9 * h->L[l1].nv));
      for (int l = l0; l < l1; ++l) {
        Level& c = h->L[l];
        Level& f = h->L[l + 1];
        if (!cfg.rtilde_true_operator) {
          c.rt_mode = tmg::RT_GEOM_FAST;
          continue;
        }
        c.rt_mode = tmg::RT_TABLE;
        TRY(dalloc(h, &c.Rt, 49 * c.nv));
        tmg::k_assemble<<<nblk(f.nv), tmg::kBlock, 0, h->s>>>(tf, f.epsm, f.n);
        CKL();
        tmg::k_rtilde<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.Rt, c.n, nullptr, 1, tf, f.flags,
                                                             f.diag_raw, cfg.omega);
        CKL();
      }
    }
  } else {
    Level& top = h->L[l1];
    bool kc;
    double v;
    TRY(check_const(h, top.epsm, top.ncell, &kc, &v));
    top.op = element_op(v, kc, top.epsm);
    tmg::k_elem_diag<<<nblk(top.nv), tmg::kBlock, 0, h->s>>>(top.diag_raw, top.diag, top.epsm,
                                                              top.flags, top.n);
    CKL();
    double* tf_top;
    TRY(dalloc(h, &tf_top, 9 * top.nv));
    tmg::k_assemble<<<nblk(top.nv), tmg::kBlock, 0, h->s>>>(tf_top, top.epsm, top.n);
    CKL();
    for (int l = l1 - 1; l >= l0; --l) {
      Level& c = h->L[l];
      Level& f = h->L[l + 1];
      const double* tf = (l + 1 == l1) ? tf_top : f.tbl;
      const int nc = c.n;
      const size_t nex = (size_t)nc * (nc + 1);
      double *ex, *ey;
      TRY(dalloc(h, &ex, 4 * nex));
      TRY(dalloc(h, &ey, 4 * nex));
      const uint8_t* rp = l >= 1 ? dref[l - 1] : nullptr;
      tmg::k_gamma_x<<<nblk(nex), tmg::kBlock, 0, h->s>>>(ex, tf, nc, c.refined, rp, deg);
      CKL();
      tmg::k_gamma_y<<<nblk(nex), tmg::kBlock, 0, h->s>>>(ey, tf, nc, c.refined, rp, deg);
      CKL();
      TRY(dalloc(h, &c.P, 25 * c.nv));
      tmg::k_p_init<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.P, nc, ex, ey);
      CKL();
      tmg::k_p_interior<<<nblk(c.ncell), tmg::kBlock, 0, h->s>>>(c.P, nc, tf, ex, ey, c.refined, rp);
      CKL();
      tmg::k_p_fix<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.P, nc, f.flags);
      CKL();
      TRY(dalloc(h, &c.tbl, 9 * c.nv));
      tmg::k_assemble<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.tbl, c.epsm, c.n);
      CKL();
      tmg::k_rap<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.tbl, c.flags, nc, tf, f.flags, c.P);
      CKL();
      c.op.kind = tmg::OP_TABLE;
      c.op.tbl = c.tbl;
      tmg::k_table_diag<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.diag_raw, c.diag, c.tbl, c.flags, c.nv);
      CKL();
      if (jac) {
        // unit-coefficient R~ is rebuilt from P in the cycle (RT_FROM_P); the
        // stored table serves tmg_get_table and the true-operator variant
        c.rt_mode = cfg.rtilde_true_operator ? tmg::RT_TABLE : tmg::RT_FROM_P;
        TRY(dalloc(h, &c.Rt, 49 * c.nv));
        if (cfg.rtilde_true_operator)
          tmg::k_rtilde<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.Rt, nc, c.P, 0, tf, f.flags,
                                                               f.diag_raw, cfg.omega);
        else
          tmg::k_rtilde<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(c.Rt, nc, c.P, 0, nullptr, nullptr,
                                                               nullptr, cfg.omega);
        CKL();
      }
    }
  }
  int hdeg = 0;
  CK(cudaMemcpyAsync(&hdeg, deg, sizeof(int), cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  if (hdeg) return fail(TMG_EDEGENERATE, "degenerate collapsed stencil in face-point solve");

  // coarse chain: every level up to lc runs inside the cluster kernel
  h->lc = l0;
  for (int l = l0; l <= l1 && l - l0 < tmg::kMaxChain; ++l)
    if (h->L[l].nv <= kSmallLevel) h->lc = l;
  // work buffers, u, partials (grid levels first, then one per cluster CTA)
  int parts = 0;
  for (int l = l0; l <= l1; ++l) {
    Level& c = h->L[l];
    TRY(dalloc(h, &c.u, c.nv));
    if (!t->u || !t->u[l]) return fail(TMG_EINVAL, "tree.u missing a level");
    CK(cudaMemcpyAsync(c.u, t->u[l], sizeof(double) * c.nv, cudaMemcpyHostToDevice, h->s));
    // work vectors start at zero: a level with a patch list never writes the slots of vertices
    // that do not exist, and their neighbours' restriction / prolongation footprints read them
    TRY(dalloc(h, &c.g, c.nv));
    CK(cudaMemsetAsync(c.g, 0, sizeof(double) * c.nv, h->s));
    if (l > l0) {
      TRY(dalloc(h, &c.rho, c.nv));
      TRY(dalloc(h, &c.rdof, c.nv));
      CK(cudaMemsetAsync(c.rho, 0, sizeof(double) * c.nv, h->s));
      CK(cudaMemsetAsync(c.rdof, 0, sizeof(double) * c.nv, h->s));
    }
    if (l < l1) {
      TRY(dalloc(h, &c.carry, c.nv));
      CK(cudaMemsetAsync(c.carry, 0, sizeof(double) * c.nv, h->s));
    }
    c.tile_h = l == l1 ? tmg::kTileY : kCoarseTileY;
    c.nblocks = (int)(tiles_x(c.N) * tiles_y(c.N, c.tile_h));
    if (l > h->lc && c.cnt[tmg::K_NONE] > 0) TRY(build_patch_list(h, c));
    if (l > h->lc) {
      c.part_off = parts;
      parts += c.nblocks;
    }
  }
  h->N_below = ipow3(l0 - 1) + 1;
  TRY(dalloc(h, &h->u_below, (size_t)h->N_below * h->N_below));
  CK(cudaMemcpyAsync(h->u_below, t->u[l0 - 1], sizeof(double) * h->N_below * h->N_below,
                     cudaMemcpyHostToDevice, h->s));
  h->part_base = parts;
  if (h->cfg.fused_cycle) {
    if (l1 - l0 + 1 > tmg::kCycleLevels) return fail(TMG_EINVAL, "fused cycle: too many levels");
    int occ = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tmg::k_cycle, tmg::kBlock, 0));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->cfg.device));
    if (occ < 1) return fail(TMG_ECUDA, "k_cycle does not fit an SM");
    h->cycle_grid = occ * sms;
    TRY(dalloc(h, &h->wpart, (size_t)2 * h->cycle_grid * tmg::kCycleWarps));
    TRY(dalloc(h, &h->bar, 2));
    CK(cudaMemsetAsync(h->bar, 0, 2 * sizeof(unsigned), h->s));
  }
  TRY(dalloc(h, &h->stamps, 64));
  TRY(dalloc(h, &h->scratch, 2 * tmg::kClusterCTAs));
  h->nparts = parts;
  TRY(dalloc(h, &h->part_sum, parts));
  TRY(dalloc(h, &h->part_max, parts));
  TRY(dalloc(h, &h->hist, 2 * h->cap));
  TRY(dalloc(h, &h->counter, 1));
  CK(cudaMemsetAsync(h->counter, 0, sizeof(int), h->s));
  h->host_counter = 0;
  CK(cudaStreamSynchronize(h->s));
  h->graph_dirty = true;
  return TMG_OK;
}

int check_level(tmg_handle* h, int level, bool allow_below = false) {
  if (!h) return fail(TMG_EINVAL, "null handle");
  if (allow_below && level == h->lmin - 1) return TMG_OK;
  if (level < h->lmin || level > h->ltop)
    return fail(TMG_EINVAL, "level " + std::to_string(level) + " outside [lmin, ltop]");
  return TMG_OK;
}

int read_stats(tmg_handle* h, long long first, int count, tmg_stats* out) {
  std::vector<double> hh(2 * h->cap);
  CK(cudaMemcpyAsync(hh.data(), h->hist, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  for (int k = 0; k < count; ++k) {
    const long long slot = (first + k) % h->cap;
    out[k].l2h = hh[2 * slot];
    out[k].linf = hh[2 * slot + 1];
    out[k].dofs = h->dofs_total;
    out[k].updates = h->updates;
  }
  return TMG_OK;
}

// Every entry point that takes a handle runs on the handle's device and restores
// the caller's current device on return (a process may hold engines on several
// GPUs, and torch may switch the current device between calls).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const tmg_handle* h) {
    int cur = -1;
    if (h && cudaGetDevice(&cur) == cudaSuccess && cur != h->cfg.device && cudaSetDevice(h->cfg.device) == cudaSuccess)
      prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

// ============================================================================
// C ABI
// ============================================================================

extern "C" {

const char* tmg_last_error(void) { return g_err.c_str(); }

int tmg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int tmg_create(const tmg_tree* tree, const tmg_config* cfg, tmg_handle** out) {
  if (!tree || !cfg || !out) return fail(TMG_EINVAL, "null argument");
  *out = nullptr;
  // SolverConfig.__post_init__ (solvers.py:92-100)
  if (cfg->variant < 0 || cfg->variant > 6) return fail(TMG_EINVAL, "unknown solver variant");
  if (cfg->variant == TMG_MULTIPLICATIVE_V10)
    return fail(TMG_EINVAL, "multiplicative-v10 (dense two-grid reference) is not offered on the device");
  if (cfg->flavor != TMG_GEOMETRIC && cfg->flavor != TMG_BOXMG)
    return fail(TMG_EINVAL, "unknown operator flavor");
  if (!(cfg->omega > 0.0 && cfg->omega <= 1.0)) return fail(TMG_EINVAL, "omega must lie in (0, 1]");
  if (!(cfg->omega_hat > 0.0 && cfg->omega_hat < 1.0))
    return fail(TMG_EINVAL, "omega_hat must lie in (0, 1)");
  if (cfg->throttled) return fail(TMG_EINVAL, "throttled setup is offered for 3D trees (tmg3_create)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(TMG_ECUDA, "no CUDA device: the engine has no CPU fallback");
  if (cfg->device < 0 || cfg->device >= ndev) return fail(TMG_EINVAL, "device index out of range");
  CK(cudaSetDevice(cfg->device));
  tmg_handle* h = new tmg_handle();
  h->cfg = *cfg;
  h->wt = std::isnan(cfg->omega_tilde) ? cfg->omega : cfg->omega_tilde;
  if (cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return fail(TMG_ECUDA, "stream creation failed");
  }
  tmg::upload_constants(h->s);
  int rc = build(h, tree);
  if (rc != TMG_OK) {
    std::string msg = g_err;
    tmg_destroy(h);
    g_err = msg;
    return rc;
  }
  *out = h;
  return TMG_OK;
}

int tmg3_create(const tmg_tree3* tree, const tmg_config* cfg, tmg_handle** out) {
  if (!tree || !cfg || !out) return fail(TMG_EINVAL, "null argument");
  *out = nullptr;
  if (cfg->variant < 0 || cfg->variant > 6) return fail(TMG_EINVAL, "unknown solver variant");
  if (cfg->variant == TMG_MULTIPLICATIVE_V10)
    return fail(TMG_EINVAL, "multiplicative-v10 (dense two-grid reference) is not offered on the device");
  if (cfg->flavor != TMG_GEOMETRIC && cfg->flavor != TMG_BOXMG)
    return fail(TMG_EINVAL, "unknown operator flavor");
  if (cfg->throttled && cfg->flavor != TMG_BOXMG)
    return fail(TMG_EINVAL, "throttled setup applies to flavor boxmg");
  if (!(cfg->omega > 0.0 && cfg->omega <= 1.0)) return fail(TMG_EINVAL, "omega must lie in (0, 1]");
  if (!(cfg->omega_hat > 0.0 && cfg->omega_hat < 1.0))
    return fail(TMG_EINVAL, "omega_hat must lie in (0, 1)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(TMG_ECUDA, "no CUDA device: the engine has no CPU fallback");
  if (cfg->device < 0 || cfg->device >= ndev) return fail(TMG_EINVAL, "device index out of range");
  CK(cudaSetDevice(cfg->device));
  Engine3* e = nullptr;
  int rc = e3_create(tree, cfg, &e, g_err);
  if (rc != TMG_OK) return rc;
  tmg_handle* h = new tmg_handle();
  h->cfg = *cfg;
  h->e3 = e;
  *out = h;
  return TMG_OK;
}

int tmg3_rebuild(tmg_handle* h, const tmg_tree3* tree) {
  DeviceGuard dg_(h);
  if (!h || !tree || !h->e3) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  CK(cudaSetDevice(h->cfg.device));
  return e3_rebuild(h->e3, tree, g_err);
}

int tmg_dim(tmg_handle* h) { return (h && h->e3) ? 3 : 2; }

int tmg3_shard(tmg_handle* h, int32_t ls, const int32_t* lo, const int32_t* hi) {
  DeviceGuard dg_(h);
  if (!h || !h->e3 || !lo || !hi) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_shard(h->e3, ls, lo, hi, g_err);
}

int tmg3_phase(tmg_handle* h, int32_t phase, int32_t level) {
  DeviceGuard dg_(h);
  if (!h || !h->e3) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_phase(h->e3, phase, level, g_err);
}

int tmg3_phase_range(tmg_handle* h, int32_t phase, int32_t level, int32_t lo, int32_t hi, int32_t first,
                     int32_t last) {
  DeviceGuard dg_(h);
  if (!h || !h->e3) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_phase_range(h->e3, phase, level, lo, hi, first, last, g_err);
}

int tmg3_field(tmg_handle* h, int32_t field, int32_t level, uint64_t* ptr, int64_t* count) {
  DeviceGuard dg_(h);
  if (!h || !h->e3 || !ptr || !count) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_field(h->e3, field, level, ptr, count, g_err);
}

int tmg3_storage(tmg_handle* h, int32_t level, int64_t* out) {
  DeviceGuard dg_(h);
  if (!h || !h->e3 || !out) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_storage(h->e3, level, out, g_err);
}

int tmg3_fused(tmg_handle* h, int32_t level, int32_t* out) {
  DeviceGuard dg_(h);
  if (!h || !h->e3 || !out) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_fused(h->e3, level, out, g_err);
}

int tmg3_stream(tmg_handle* h, uint64_t* stream) {
  DeviceGuard dg_(h);
  if (!h || !h->e3 || !stream) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_stream(h->e3, stream);
}

int tmg3_history(tmg_handle* h, int32_t count, tmg_stats* out) {
  DeviceGuard dg_(h);
  if (!h || !h->e3 || !out) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_history(h->e3, count, out, g_err);
}

int tmg3_cycle_state(tmg_handle* h, int64_t* count, int32_t* parity, int32_t set) {
  DeviceGuard dg_(h);
  if (!h || !h->e3 || !count || !parity) return fail(TMG_EINVAL, "null argument or not a 3D handle");
  return e3_cycle_state(h->e3, count, parity, set, g_err);
}

int tmg_rebuild(tmg_handle* h, const tmg_tree* tree) {
  DeviceGuard dg_(h);
  if (h && h->e3) return fail(TMG_EINVAL, "3D handle: use tmg3_rebuild");
  if (!h || !tree) return fail(TMG_EINVAL, "null argument");
  CK(cudaSetDevice(h->cfg.device));
  CK(cudaStreamSynchronize(h->s));
  free_all(h);
  return build(h, tree);
}

int tmg_set_rhs(tmg_handle* h, int32_t level, const double* rhs) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_set_rhs(h->e3, level, rhs, g_err);
  TRY(check_level(h, level));
  Level& c = h->L[level];
  if (!rhs) {
    if (c.rhs) { c.rhs = nullptr; h->graph_dirty = true; }  // buffer stays owned by allocs
    return TMG_OK;
  }
  if (!c.rhs) {
    TRY(dalloc(h, &c.rhs, c.nv));
    h->graph_dirty = true;
  }
  CK(cudaMemcpyAsync(c.rhs, rhs, sizeof(double) * c.nv, cudaMemcpyHostToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  return TMG_OK;
}

int tmg_set_u(tmg_handle* h, int32_t level, const double* u) {
  DeviceGuard dg_(h);
  if (h && h->e3) return u ? e3_set_u(h->e3, level, u, g_err) : fail(TMG_EINVAL, "null array");
  TRY(check_level(h, level, true));
  if (!u) return fail(TMG_EINVAL, "null array");
  double* dst = (level == h->lmin - 1) ? h->u_below : h->L[level].u;
  const size_t nv = (level == h->lmin - 1) ? (size_t)h->N_below * h->N_below : h->L[level].nv;
  CK(cudaMemcpyAsync(dst, u, sizeof(double) * nv, cudaMemcpyHostToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  return TMG_OK;
}

int tmg_get_u(tmg_handle* h, int32_t level, double* u) {
  DeviceGuard dg_(h);
  if (h && h->e3) return u ? e3_get_u(h->e3, level, u, g_err) : fail(TMG_EINVAL, "null array");
  TRY(check_level(h, level, true));
  if (!u) return fail(TMG_EINVAL, "null array");
  const double* src = (level == h->lmin - 1) ? h->u_below : h->L[level].u;
  const size_t nv = (level == h->lmin - 1) ? (size_t)h->N_below * h->N_below : h->L[level].nv;
  CK(cudaMemcpyAsync(u, src, sizeof(double) * nv, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  return TMG_OK;
}

int tmg_update_fas_state(tmg_handle* h) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_update_fas_state(h->e3, g_err);
  if (!h) return fail(TMG_EINVAL, "null handle");
  TRY(enqueue_fas(h));
  CK(cudaStreamSynchronize(h->s));
  return TMG_OK;
}

int tmg_cycle(tmg_handle* h, int32_t ncycles, tmg_stats* stats) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_cycle(h->e3, ncycles, stats, g_err);
  if (!h) return fail(TMG_EINVAL, "null handle");
  if (ncycles < 0) return fail(TMG_EINVAL, "negative cycle count");
  TRY(ensure_graph(h));
  int done = 0;
  while (done < ncycles) {
    const int chunk = std::min(ncycles - done, h->cap);
    const long long first = h->host_counter;
    for (int k = 0; k < chunk; ++k) CK(cudaGraphLaunch(h->gexec, h->s));
    h->host_counter += chunk;
    if (stats) TRY(read_stats(h, first, chunk, stats + done));
    else CK(cudaStreamSynchronize(h->s));
    done += chunk;
  }
  return TMG_OK;
}

int tmg_residual_stats(tmg_handle* h, tmg_stats* out) {
  DeviceGuard dg_(h);
  if (h && h->e3 && out) return e3_residual_stats(h->e3, out, g_err);
  if (!h || !out) return fail(TMG_EINVAL, "null argument");
  TRY(enqueue_down(h, false));
  const long long first = h->host_counter++;
  TRY(read_stats(h, first, 1, out));
  return TMG_OK;
}

int tmg_levels(tmg_handle* h, int32_t* lmin, int32_t* ltop) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_levels(h->e3, lmin, ltop);
  if (!h) return fail(TMG_EINVAL, "null handle");
  if (lmin) *lmin = h->lmin;
  if (ltop) *ltop = h->ltop;
  return TMG_OK;
}

int tmg_level_counts(tmg_handle* h, int32_t level, int64_t* dof, int64_t* composite,
                     int64_t* hanging) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_level_counts(h->e3, level, dof, composite, hanging, g_err);
  TRY(check_level(h, level));
  const Level& c = h->L[level];
  if (dof) *dof = c.cnt[tmg::K_DOF] + c.cnt[tmg::K_OVER];
  if (composite) *composite = c.cnt[tmg::K_DOF];
  if (hanging) *hanging = c.cnt[tmg::K_HANG];
  return TMG_OK;
}

int tmg_level_tiles(tmg_handle* h, int32_t level, int64_t* listed, int64_t* dense) {
  DeviceGuard dg_(h);
  if (!h || !listed || !dense) return fail(TMG_EINVAL, "null argument");
  if (h->e3) return fail(TMG_EINVAL, "3D handles hold regular trees (no patch lists)");
  TRY(check_level(h, level));
  const Level& c = h->L[level];
  *dense = (int64_t)tiles_x(c.N) * tiles_y(c.N, c.tile_h ? c.tile_h : tmg::kTileY);
  *listed = c.tiles ? c.ntiles : 0;
  return TMG_OK;
}

int tmg_get_kinds(tmg_handle* h, int32_t level, int8_t* out) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_get_kinds(h->e3, level, out, g_err);
  TRY(check_level(h, level));
  const Level& c = h->L[level];
  std::vector<uint8_t> f(c.nv);
  CK(cudaMemcpyAsync(f.data(), c.flags, c.nv, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  for (size_t v = 0; v < c.nv; ++v) out[v] = (int8_t)(f[v] & 7);
  return TMG_OK;
}

int tmg_get_table(tmg_handle* h, int32_t which, int32_t level, double* out) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_get_table(h->e3, which, level, out, g_err);
  TRY(check_level(h, level));
  Level& c = h->L[level];
  auto fetch = [&](const double* src, size_t count, std::vector<double>& dst) -> int {
    dst.resize(count);
    CK(cudaMemcpyAsync(dst.data(), src, sizeof(double) * count, cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
    return TMG_OK;
  };
  std::vector<double> buf;
  switch (which) {
    case TMG_TABLE_DIAG:
      TRY(fetch(c.diag_raw, c.nv, buf));
      std::memcpy(out, buf.data(), sizeof(double) * c.nv);
      return TMG_OK;
    case TMG_TABLE_EFFEPS:
      TRY(fetch(c.eff, c.ncell, buf));
      std::memcpy(out, buf.data(), sizeof(double) * c.ncell);
      return TMG_OK;
    case TMG_TABLE_A: {
      const double* src = c.tbl;
      double* tmp = nullptr;
      if (!src) {
        TRY(dalloc(h, &tmp, 9 * c.nv));
        tmg::k_assemble<<<nblk(c.nv), tmg::kBlock, 0, h->s>>>(tmp, c.epsm, c.n);
        CKL();
        src = tmp;
      }
      TRY(fetch(src, 9 * c.nv, buf));
      for (size_t v = 0; v < c.nv; ++v)
        for (int k = 0; k < 9; ++k) out[v * 9 + k] = buf[k * c.nv + v];
      return TMG_OK;
    }
    case TMG_TABLE_P: {
      if (!c.P) return fail(TMG_EINVAL, "no P table on this level");
      TRY(fetch(c.P, 25 * c.nv, buf));
      for (size_t v = 0; v < c.nv; ++v)
        for (int a = -3; a <= 3; ++a)
          for (int b = -3; b <= 3; ++b) {
            double w = 0.0;
            if (a >= -2 && a <= 2 && b >= -2 && b <= 2) w = buf[((a + 2) * 5 + (b + 2)) * c.nv + v];
            out[v * 49 + (a + 3) * 7 + (b + 3)] = w;
          }
      return TMG_OK;
    }
    case TMG_TABLE_RT: {
      if (!c.Rt) return fail(TMG_EINVAL, "no R~ table on this level");
      TRY(fetch(c.Rt, 49 * c.nv, buf));
      for (size_t v = 0; v < c.nv; ++v)
        for (int k = 0; k < 49; ++k) out[v * 49 + k] = buf[k * c.nv + v];
      return TMG_OK;
    }
    default:
      return fail(TMG_EINVAL, "unknown table id");
  }
}

int tmg_time_cycles(tmg_handle* h, int32_t ncycles, int64_t flush_bytes, float* ms) {
  DeviceGuard dg_(h);
  if (h && h->e3 && ms) return e3_time_cycles(h->e3, ncycles, flush_bytes, ms, g_err);
  if (!h || !ms) return fail(TMG_EINVAL, "null argument");
  TRY(ensure_graph(h));
  if (flush_bytes > 0 && h->flush_bytes < (size_t)flush_bytes) {
    if (h->flush_buf) cudaFree(h->flush_buf);
    h->flush_buf = nullptr;
    CK(cudaMalloc(&h->flush_buf, (size_t)flush_bytes));
    h->flush_bytes = (size_t)flush_bytes;
  }
  const int ne = flush_bytes > 0 ? 2 * ncycles : 2;
  std::vector<cudaEvent_t> ev(ne);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  CK(cudaStreamSynchronize(h->s));
  if (flush_bytes > 0) {
    for (int k = 0; k < ncycles; ++k) {
      CK(cudaMemsetAsync(h->flush_buf, k & 0xff, (size_t)flush_bytes, h->s));
      CK(cudaEventRecord(ev[2 * k], h->s));
      CK(cudaGraphLaunch(h->gexec, h->s));
      CK(cudaEventRecord(ev[2 * k + 1], h->s));
    }
  } else {
    CK(cudaEventRecord(ev[0], h->s));
    for (int k = 0; k < ncycles; ++k) CK(cudaGraphLaunch(h->gexec, h->s));
    CK(cudaEventRecord(ev[1], h->s));
  }
  CK(cudaStreamSynchronize(h->s));
  h->host_counter += ncycles;
  float total = 0.f;
  for (int k = 0; k < ne / 2; ++k) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ev[2 * k], ev[2 * k + 1]));
    total += t;
  }
  *ms = total;
  for (auto& e : ev) cudaEventDestroy(e);
  return TMG_OK;
}

int tmg_profile_cycles(tmg_handle* h, int32_t ncycles, int32_t cap, const char** names, float* ms,
                       int32_t* launches, int32_t* nk) {
  DeviceGuard dg_(h);
  if (h && h->e3) return e3_profile_cycles(h->e3, ncycles, cap, names, ms, launches, nk, g_err);
  if (!h) return fail(TMG_EINVAL, "null handle");
  std::vector<KTimer> timers;
  h->timers = &timers;
  h->profiling = true;
  int rc = TMG_OK;
  for (int k = 0; k < ncycles && rc == TMG_OK; ++k) {
    rc = enqueue_cycle(h);
    h->host_counter++;
  }
  h->profiling = false;
  if (rc == TMG_OK) rc = resolve_timers(h);
  h->timers = nullptr;
  h->pending.clear();
  h->ev_used = 0;
  if (rc != TMG_OK) return rc;
  int n = 0;
  for (auto& t : timers) {
    if (n >= cap) break;
    names[n] = t.name;
    ms[n] = t.ms;
    launches[n] = t.launches;
    ++n;
  }
  *nk = n;
  return TMG_OK;
}

int tmg_launches_per_cycle(tmg_handle* h, int32_t* n) {
  DeviceGuard dg_(h);
  if (h && h->e3 && n) return e3_launches_per_cycle(h->e3, n, g_err);
  if (!h || !n) return fail(TMG_EINVAL, "null argument");
  TRY(ensure_graph(h));
  *n = h->launches;
  return TMG_OK;
}

// diagnostics (not part of tmg.h): %globaltimer stamps of the last k_coarse phases
int tmg_debug_stamps(tmg_handle* h, unsigned long long* out, int n) {
  DeviceGuard dg_(h);
  if (!h || !out) return fail(TMG_EINVAL, "null argument");
  CK(cudaMemcpy(out, h->stamps, sizeof(unsigned long long) * std::min(n, 64), cudaMemcpyDeviceToHost));
  return TMG_OK;
}

void tmg_destroy(tmg_handle* h) {
  if (!h) return;
  DeviceGuard dg_(h);
  if (h->e3) {
    e3_destroy(h->e3);
    delete h;
    return;
  }
  if (h->s) cudaStreamSynchronize(h->s);
  free_all(h);
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  if (h->flush_buf) cudaFree(h->flush_buf);
  if (h->s) cudaStreamDestroy(h->s);
  delete h;
}

}  // extern "C"
