/*
 * tmg.h -- C ABI of the B200 additive-FAC / adaFACx engine (libtmg.so).
 *
 * Drop-in boundary for the hot path of the reference solver
 * (/root/reference/pkg/src/treemg).  The reference has no FFI: its path sits
 * behind the Python engine protocol of ``ReferenceEngine``
 * (solvers.py:129-492).  Every entry point below replaces one method of that
 * protocol; the Python mirror ``paper_1903_10367_b200.solvers.GpuEngine``
 * binds them through ctypes.
 *
 * Conventions: plain pointers and sizes only.  A level l has n = 3^l cells
 * per axis; vertex fields are (n+1)^2 fp64 and cell fields n^2, C-ordered
 * [i][j] with i along x (spacetree.py:86-120).  All input arrays are copied;
 * the handle owns every device buffer, its CUDA stream and graph.  There is
 * no CPU fallback: without a CUDA device tmg_create fails with TMG_ECUDA.
 *
 * Status codes (mirroring the reference's exceptions):
 *   TMG_OK          0
 *   TMG_EINVAL      1  bad argument / config / unsupported   -> ValueError   (solvers.py:93-100,150,254)
 *   TMG_EDEGENERATE 2  degenerate collapsed BoxMG stencil    -> ArithmeticError (operators.py:295-297)
 *   TMG_ECUDA       3  CUDA runtime failure / no device      -> RuntimeError
 * tmg_last_error() returns a thread-local message for the last failure.
 */
#ifndef TMG_H
#define TMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMG_OK 0
#define TMG_EINVAL 1
#define TMG_EDEGENERATE 2
#define TMG_ECUDA 3

/* solver variants, solvers.py:70-78 */
#define TMG_ADDITIVE 0
#define TMG_ADDITIVE_EXP 1
#define TMG_BPX 2
#define TMG_AFACC 3
#define TMG_ADAFAC_PI 4
#define TMG_ADAFAC_JAC 5
#define TMG_MULTIPLICATIVE_V10 6 /* not offered on the device: tmg_create -> TMG_EINVAL */

/* operator flavours, solvers.py:95 */
#define TMG_GEOMETRIC 0
#define TMG_BOXMG 1

/* tables readable with tmg_get_table */
#define TMG_TABLE_A 0    /* ops[l] 3x3 stencil rows, (n+1)^2 x 9 (operators.py:201-202, 241-248) */
#define TMG_TABLE_DIAG 1 /* ops[l].diag(), (n+1)^2 (operators.py:190-199, 241-242) */
#define TMG_TABLE_P 2    /* transfers[l].p_table, (n+1)^2 x 7 x 7 (operators.py:306-437) */
#define TMG_TABLE_RT 3   /* transfers[l].rtilde per-vertex, (n+1)^2 x 7 x 7 (operators.py:508-547) */
#define TMG_TABLE_EFFEPS 4 /* eff_eps[l], n^2 (solvers.py:165-175) */

typedef struct tmg_handle tmg_handle;

/* SolverConfig, solvers.py:82-104 */
typedef struct {
  int32_t variant;
  int32_t flavor;
  double omega;
  double omega_tilde; /* NaN = "None" -> omega (solvers.py:102-104) */
  double omega_hat;
  double damping_scale;
  int32_t rtilde_true_operator;
  int32_t device;
  /* BoxMG, 3D: start from d-linear P and rediscretised coarse rows and build
   * BoxMG P + Galerkin rows one level per cycle, finest first (the paper's
   * throttled setup; the reference builds all levels in rebuild()) */
  int32_t throttled;
  /* 2D: run the whole cycle as ONE persistent cooperative launch (k_cycle: all levels' down
   * sweeps, stats, carries, FAS injection and hanging refresh behind grid barriers) instead of
   * one launch per level and sweep.  Same iterates; the residual norm's summation order differs. */
  int32_t fused_cycle;
} tmg_config;

/* The spacetree data model, spacetree.py:86-120.  refined[l] for l < lmax
 * ((3^l)^2 bytes, 0/1; a NULL entry means "no cell refined"); eps[l] and u[l]
 * for l < nlevels (nlevels = len(tree.u) = depth + 1). */
typedef struct {
  int32_t lmin;
  int32_t lmax;
  int32_t nlevels;
  const uint8_t* const* refined;
  const double* const* eps;
  const double* const* u;
} tmg_tree;

/* CycleStats, solvers.py:107-115 (level_dofs via tmg_level_counts) */
typedef struct {
  double l2h;
  double linf;
  int64_t dofs;
  int64_t updates;
} tmg_stats;

/* 3D regular spacetree (BASELINE configs 3, 5; the reference is 2D only, its
 * data model carried to d = 3): every cell of levels < depth refined; eps is
 * the finest level's per-cell material ((3^depth)^3 fp64, [i][j][k]); u[l]
 * ((3^l+1)^3 fp64) for l in 0..depth (u[l] for l < lmin may be NULL). */
typedef struct {
  int32_t lmin;
  int32_t depth;
  const double* eps;
  const double* const* u;
} tmg_tree3;

/* ReferenceEngine.__init__ + rebuild(): solvers.py:137-141, 145-255.
 * Classifies vertices, builds eff_eps, stencils, BoxMG P, Galerkin rows and
 * R~ on the device and uploads u. */
int tmg_create(const tmg_tree* tree, const tmg_config* cfg, tmg_handle** out);

/* 3D engine (oracle/mg3d.py semantics): same entry points as 2D after creation;
 * tmg_get_table returns 27-tap rows (TMG_TABLE_A), 125-offset P rows
 * (TMG_TABLE_P, fine offsets -2..2) and the cell material (TMG_TABLE_EFFEPS). */
int tmg3_create(const tmg_tree3* tree, const tmg_config* cfg, tmg_handle** out);
int tmg3_rebuild(tmg_handle* h, const tmg_tree3* tree);

/* 2 or 3: the dimension of the hierarchy a handle holds. */
int tmg_dim(tmg_handle* h);

/* ---- multi-GPU slab sharding of a 3D handle ----
 * Every rank builds the full hierarchy (setup is redundant, cycles are not);
 * the finest level stays double buffered (TMG_F_U of the finest level names the
 * current buffer, which alternates every cycle: query it after TMG_PH_UP);
 * tmg3_shard restricts the cycle of levels >= ls to the vertex planes
 * [lo[l], hi[l]) (axis 0, the slowest) this rank owns; levels < ls are
 * replicated.  The host (paper_1903_10367_b200/sharding.py) runs the cycle
 * phase by phase and exchanges halo planes / gathers / reduces with NCCL on
 * the handle's stream between phases.  No reference counterpart: the
 * reference is serial. */
#define TMG_PH_DOWN 0   /* level l >= ls: down sweep on owned planes           */
#define TMG_PH_SMOOTH 1 /* level l >= ls: adaFACx R~ smoothing on owned planes  */
#define TMG_PH_REPL 2   /* levels lmin..ls-1 (replicated): down, stats, up      */
#define TMG_PH_UP 3     /* level l >= ls: carry + update on owned planes        */
#define TMG_PH_INJECT 4 /* FAS injection ls -> lmin on the replicated levels    */
#define TMG_PH_REDUCE 5 /* fold this cycle's stats partials into TMG_F_PART     */
#define TMG_PH_SMR 6    /* level l > ls with tmg3_fused: adaFACx smoothing of l fused with the
                           restriction into the owned planes of l - 1 (replaces SMOOTH of l and
                           the restriction in DOWN of l - 1; rho of l needs 3 halo planes below
                           and 1 above, sm needs none) */
#define TMG_F_U 0
#define TMG_F_RHO 1
#define TMG_F_SM 2
#define TMG_F_CARRY 3
#define TMG_F_G 4
#define TMG_F_PART 5 /* 2 doubles: sum of squares, max (all-reduced across ranks) */
int tmg3_shard(tmg_handle* h, int32_t ls, const int32_t* lo, const int32_t* hi);
int tmg3_phase(tmg_handle* h, int32_t phase, int32_t level);
/* TMG_PH_DOWN / TMG_PH_UP of a sharded level restricted to the owned planes inside [lo, hi): the
 * host splits a phase into the planes a neighbour rank needs (computed first, their halo exchange
 * started) and the rest (computed while the exchange is in flight).  `first` / `last` mark the
 * first / last part of the phase in this cycle (residual partials restart at the first part; the
 * finest level's double buffer flips after the last). */
int tmg3_phase_range(tmg_handle* h, int32_t phase, int32_t level, int32_t lo, int32_t hi, int32_t first,
                     int32_t last);
/* *out = 1 when the sharded cycle of level `level` runs TMG_PH_SMR instead of TMG_PH_SMOOTH */
int tmg3_fused(tmg_handle* h, int32_t level, int32_t* out);
/* device address and element count of a field of a level (zero-copy views) */
int tmg3_field(tmg_handle* h, int32_t field, int32_t level, uint64_t* ptr, int64_t* count);
/* storage of level `level`'s BoxMG operators (no reference counterpart): out[0] rows of P
 * (coarse vertices), out[1] distinct rows in its row dictionary (0 = stored dense), out[2]
 * rows of the cube-owned copy Pc (coarse cubes; 0 = none), out[3] distinct rows of Pc's
 * dictionary, out[4] rows of the Galerkin table, out[5] rows its run-length form along k stores
 * (kernels3d_rle.cu: only the rows that differ from their predecessor in a 32-vertex segment; 0 =
 * dense planes only).
 * Dictionaries (lossless, bitwise-verified) are built at setup for levels ltop-1 (and
 * ltop-2) when rows repeat (piecewise-constant coefficients); TMG_PDICT=0 disables, 2 forces
 * them. */
int tmg3_storage(tmg_handle* h, int32_t level, int64_t* out);
/* the cudaStream_t every phase is enqueued on */
int tmg3_stream(tmg_handle* h, uint64_t* stream);
/* the last `count` per-cycle residual stats of a sharded run */
int tmg3_history(tmg_handle* h, int32_t count, tmg_stats* out);
/* Host-side state of a sharded handle: the number of cycles enqueued so far (which slots
 * tmg3_history reads) and which buffer of the finest level's double-buffered u is current.
 * set = 0 reads it, set = 1 writes it: the host that captures the phases + exchanges of a cycle
 * into CUDA graphs on the handle's stream (sharding.py: ShardedEngine3.capture / replay)
 * restores the state after the capture (captured cycles do not run) and advances it after
 * every replay. */
int tmg3_cycle_state(tmg_handle* h, int64_t* count, int32_t* parity, int32_t set);

/* ReferenceEngine.rebuild() after a mesh / material change (solvers.py:145-255):
 * rebuilds every operator from the new tree and re-uploads u. rhs is kept. */
int tmg_rebuild(tmg_handle* h, const tmg_tree* tree);

/* engine.rhs[level] = rhs (solvers.py:140, 305-309); rhs == NULL deletes it. */
int tmg_set_rhs(tmg_handle* h, int32_t level, const double* rhs);

/* tree.u[level][...] = u (host -> device) / u = tree.u[level] (device -> host). */
int tmg_set_u(tmg_handle* h, int32_t level, const double* u);
int tmg_get_u(tmg_handle* h, int32_t level, double* u);

/* ReferenceEngine.update_fas_state(), solvers.py:280-296. */
int tmg_update_fas_state(tmg_handle* h);

/* ncycles x ReferenceEngine.advance(), solvers.py:334-399: stats[k] is the
 * residual of the iterate cycle k started from.  stats may be NULL. */
int tmg_cycle(tmg_handle* h, int32_t ncycles, tmg_stats* stats);

/* ReferenceEngine.residual_stats(), solvers.py:461-482. */
int tmg_residual_stats(tmg_handle* h, tmg_stats* out);

/* ltop (solvers.py:148) and level range held by the handle. */
int tmg_levels(tmg_handle* h, int32_t* lmin, int32_t* ltop);

/* masks[l]["dof"].sum() and masks[l]["composite"].sum() (solvers.py:184-192, 443). */
int tmg_level_counts(tmg_handle* h, int32_t level, int64_t* dof, int64_t* composite,
                     int64_t* hanging);

/* Patch list of a 2D level (no reference counterpart: the reference stores and sweeps dense
 * per-level arrays, spacetree.py:164-191): *dense = vertex tiles of the level's bounding
 * array, *listed = tiles in its patch list -- those holding an existing vertex, the only ones
 * the cycle kernels of an adaptive level visit; 0 = the level is swept densely (every vertex
 * exists, or the level belongs to the single-block coarse chain). */
int tmg_level_tiles(tmg_handle* h, int32_t level, int64_t* listed, int64_t* dense);

/* masks[l]["kinds"] (spacetree.py:164-191), int8 (n+1)^2. */
int tmg_get_kinds(tmg_handle* h, int32_t level, int8_t* out);

/* Operator tables (see TMG_TABLE_*) for tests and inspection. */
int tmg_get_table(tmg_handle* h, int32_t which, int32_t level, double* out);

/* Device timing of ncycles cycles (CUDA events on the handle's stream, inputs
 * resident): total milliseconds.  flush_bytes > 0 writes a scratch buffer of
 * that size (larger than L2) before every cycle, outside the timed events;
 * flush_bytes == 0 times the cycles back to back.  Used by bench.py. */
int tmg_time_cycles(tmg_handle* h, int32_t ncycles, int64_t flush_bytes, float* ms);

/* Per-kernel device times over ncycles (events around every launch, no graph):
 * names[k] (static strings), ms[k] summed, launches[k]; returns count via *nk. */
int tmg_profile_cycles(tmg_handle* h, int32_t ncycles, int32_t cap, const char** names,
                       float* ms, int32_t* launches, int32_t* nk);

/* Kernel launches per cycle as issued by tmg_cycle. */
int tmg_launches_per_cycle(tmg_handle* h, int32_t* n);

void tmg_destroy(tmg_handle* h);
const char* tmg_last_error(void);
int tmg_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* TMG_H */
