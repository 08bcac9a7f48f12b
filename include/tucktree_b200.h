/*
 * tucktree_b200 — C ABI of the B200-native stream-segment-tree engine.
 *
 * Drop-in boundary for the hot path of the reference library `tucktree`
 * (arXiv 2501.06647; /root/reference/proj/core/include/tucktree/*.hpp). The
 * reference exposes C++ only (no FFI); each entry point below names the
 * reference function it replaces. INTEGRATION.md shows the C++ facade
 * (namespace tucktree) and the ctypes binding built on these symbols.
 *
 * Conventions
 *  - Plain pointers and sizes; no CUDA or torch types in the signatures.
 *  - Factor matrices are column-major (layout of Eigen::MatrixXd), factor n
 *    is D_n x r_n with leading dimension D_n; cores are row-major with the
 *    temporal mode first (tucktree::DenseTensor).
 *  - Status codes map 1:1 onto the reference's exception classes:
 *      TT_EINVAL  <- std::invalid_argument  (bad shapes, ranges, theta, config)
 *      TT_ELOGIC  <- std::logic_error       (structural impossibilities)
 *      TT_EIO     <- std::runtime_error     (I/O)
 *      TT_ERANGE  <- std::out_of_range      (unknown node id, sst.cpp:68)
 *    plus TT_ECUDA / TT_ENOMEM for device failures. tt_last_error() returns the
 *    thread-local message of the last failure.
 *  - A failed append leaves the tree unchanged (sst.cpp:95-97).
 *  - Threading: tt_append needs exclusive access to a tree; tt_recall,
 *    tt_query_batch and the stat/node getters may run concurrently between
 *    appends (sst.hpp:52-53).
 *  - Input buffers are borrowed for the duration of the call only.
 */
#ifndef TUCKTREE_B200_H
#define TUCKTREE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_MAX_ORDER 8

typedef enum tt_status {
  TT_OK = 0,
  TT_EINVAL = 1,
  TT_ELOGIC = 2,
  TT_EIO = 3,
  TT_ECUDA = 4,
  TT_ENCCL = 5,
  TT_ENOMEM = 6,
  TT_ERANGE = 7
} tt_status;

/* Where a caller buffer lives. */
typedef enum tt_mem { TT_MEM_HOST = 0, TT_MEM_DEVICE = 1 } tt_mem;

/* Node kinds (sst.hpp:20-24) and hit flags (query.hpp:11-14; TAIL = raw
 * slices past the last complete leaf block). */
enum { TT_LEAF = 0, TT_INTERMEDIATE = 1, TT_PLACEHOLDER = 2 };
enum { TT_HIT_ENTIRE = 0, TT_HIT_PARTIAL = 1, TT_HIT_TAIL = 2 };

/* Tree configuration: TreeConfig + AlsConfig (sst.hpp:38-43, tucker.hpp:17-22)
 * plus the leaf block B (slices per leaf) and the CUDA device. */
typedef struct tt_config {
  int32_t order;                           /* p >= 2 (temporal + non-temporal modes) */
  int64_t nontemporal[TT_MAX_ORDER - 1];   /* D_2..D_p                              */
  int64_t ranks[TT_MAX_ORDER];             /* requested ranks, temporal first       */
  double theta;                            /* pruning threshold, (0,1); default 0.7 */
  int32_t max_iters;                       /* ALS sweeps cap; default 20            */
  double tol;                              /* fit-change tolerance; default 0.01    */
  uint64_t seed;                           /* ALS init seed; default 20240117       */
  int64_t leaf_block;                      /* B >= 1 slices per leaf                */
  int32_t device;                          /* CUDA device ordinal                   */
  int32_t flags;                           /* TT_FLAG_*                             */
} tt_config;

/* Bookkeeping only: no decompositions, no device work (host-logic tests). */
#define TT_FLAG_STRUCTURE_ONLY 1

typedef struct tt_tree tt_tree;

typedef struct tt_node_info {
  int64_t id, begin, end; /* [begin, end) in slices */
  int32_t kind;
  int32_t has_decomposition;
  int64_t left, right;
  int64_t ranks[TT_MAX_ORDER]; /* column counts of the stored factors */
} tt_node_info;

typedef struct tt_hit {
  int64_t node; /* 0 for a tail hit */
  int64_t begin, end;
  int32_t flag;
  int32_t pad;
} tt_hit;

typedef struct tt_range {
  int64_t ts, te;
} tt_range;

/* Output of one range query (range_query_detailed, query.hpp:48-50).
 * Caller-provided buffers sized for the clamped requested ranks:
 *   core:        prod_n r_n doubles (row-major, actual ranks)
 *   factors[0]:  L x r_0  (column-major, ld = L = te - ts)
 *   factors[m]:  D_m x r_m (column-major, ld = D_m)
 * A null core/factor pointer means "not requested" (the engine uses scratch).
 * Outputs written by the engine: ranks (actual column counts), sweeps,
 * converged, objective (final squared residual), nhits, and — when trace is
 * non-null — the per-sweep squared residuals (AlsTrace::objective,
 * tucker.hpp:25-28) into trace[0 .. min(sweeps, trace_cap)), and — when hits
 * is non-null — the hit set the query used into hits[0 .. min(nhits,
 * hits_cap)) (trace and hits: host memory). */
typedef struct tt_query_out {
  double* core;
  double* factors[TT_MAX_ORDER];
  int64_t ranks[TT_MAX_ORDER];
  int32_t sweeps;
  int32_t converged;
  double objective;
  int32_t nhits;
  int32_t trace_cap;  /* capacity of trace (doubles); 0: no trace */
  double* trace;      /* host buffer for the per-sweep objective, or NULL */
  tt_hit* hits;       /* host buffer for the hit set (QueryResult::hits), or NULL */
  int32_t hits_cap;   /* capacity of hits */
  int32_t pad;
} tt_query_out;

/* Host-side result of the standalone operations. */
typedef struct tt_factors tt_factors;

/* ---- errors --------------------------------------------------------------- */
const char* tt_last_error(void);
const char* tt_version(void);

/* ---- tree (StreamSegmentTree, sst.hpp:54-105) ----------------------------- */
/* StreamSegmentTree(TreeConfig)                            sst.hpp:56 */
tt_status tt_tree_create(const tt_config* cfg, tt_tree** out);
void tt_tree_destroy(tt_tree* tree);

/* StreamSegmentTree::append, n slices at once (one slice = prod D doubles,
 * row-major). Burst appends are processed level-synchronously: every new leaf
 * block is decomposed in one batched launch, then every completed parent,
 * level by level — result-identical to n sequential appends.  sst.hpp:64-67
 * TT_MEM_DEVICE sources are read on the engine's own non-blocking stream: the
 * bytes must be complete (synchronise the stream that produced them) before
 * the call; the call returns after the engine has finished reading them.   */
tt_status tt_append(tt_tree* tree, const double* slices, int64_t n, tt_mem where);

/* Empties the tree (timespan 0, no nodes) but keeps its device buffers and
 * init-factor caches, so a rebuild allocates nothing. Not in the reference
 * API (equivalent to constructing a new StreamSegmentTree).               */
tt_status tt_tree_clear(tt_tree* tree);

/* StreamSegmentTree::from_parts (sst.hpp:58-62): rebuilds a tree from node
 * records (ids 1..n in order; semantic invariants are checked by tt_validate,
 * not here) and, for nodes with has_decomposition, their payloads:
 * cores[i] (row-major, nodes[i].ranks) and factors[i*order + m] (column-major;
 * factor 0 is length x r_0, factor m is D_m x r_m), host memory. The
 * leaf block is cfg->leaf_block (1 = the reference tree); timespan must be a
 * multiple of it (the raw tail of a B > 1 tree is not part of the parts).   */
tt_status tt_tree_from_parts(const tt_config* cfg, const tt_node_info* nodes, int64_t n,
                             const double* const* cores, const double* const* factors, int64_t root,
                             int64_t timespan, int64_t stitch_count, tt_tree** out);
/* timespan / height / stitch_count / last_append_node_touches / node_count /
 * root / leaves                                            sst.hpp:69-91 */
enum {
  TT_STAT_TIMESPAN = 0,
  TT_STAT_HEIGHT = 1,
  TT_STAT_STITCH_COUNT = 2,
  TT_STAT_LAST_TOUCHES = 3,
  TT_STAT_NODE_COUNT = 4,
  TT_STAT_ROOT = 5,
  TT_STAT_LEAVES = 6
};
int64_t tt_tree_stat(const tt_tree* tree, int32_t what);

/* StreamSegmentTree::node(NodeId)                          sst.hpp:90 */
tt_status tt_node_info_get(const tt_tree* tree, int64_t id, tt_node_info* out);

/* Node::decomposition download (sst.hpp:33): core (prod ranks) and factors
 * (factors[0]: len x r0, ld = len; factors[m]: D_m x r_m).               */
tt_status tt_node_get(const tt_tree* tree, int64_t id, double* core, double* const* factors, tt_mem where);

/* Node ids created-or-re-decomposed by the most recent tt_append, in
 * completion order (leaf, then its stitched ancestors).                   */
tt_status tt_last_redecomposed(const tt_tree* tree, int64_t* ids, int64_t cap, int64_t* n);

/* StreamSegmentTree::validate; returns the number of violations and writes
 * them newline-separated into buf.                         sst.hpp:74-78 */
int32_t tt_validate(const tt_tree* tree, char* buf, int64_t cap);

/* ---- persistence (io.hpp:11-31) ------------------------------------------- */
/* write_tree_file(path, tree): the reference's "SST1" container, bit-exact in
 * layout (header, config, node table, per-node core + row-major factors).
 * A tree with leaf_block B > 1 or a raw tail appends a "TTB1" extension after
 * the node table (u64 B | u64 tail slices | row-major f64 tail), which the
 * reference reader ignores. Node payloads are downloaded from the device.
 * Errors: TT_EIO (std::runtime_error in io.cpp:19).           io.cpp:165-188 */
tt_status tt_tree_save(const tt_tree* tree, const char* path);

/* read_tree_file(path): rebuilds a tree on `device` from an SST1 file (node
 * payloads uploaded into the device slots). flags: TT_FLAG_STRUCTURE_ONLY
 * loads the bookkeeping only (no device).                     io.cpp:190-230 */
tt_status tt_tree_load(const char* path, int32_t device, int32_t flags, tt_tree** out);

/* StreamSegmentTree::config() (sst.hpp:66): the tree's configuration.      */
tt_status tt_tree_config(const tt_tree* tree, tt_config* out);

/* "TTS1" tensor container (io.hpp:11-19): magic | u16 version=1 | u8 p |
 * p x u64 dims | row-major f64 payload. Host memory only.     io.cpp:124-150 */
tt_status tt_tensor_write(const char* path, int32_t p, const int64_t* dims, const double* data);
/* Reads the header (p, dims[0..p), dims holding TT_TENSOR_MAX_ORDER entries);
 * with data != NULL also the payload (prod(dims) doubles).                  */
#define TT_TENSOR_MAX_ORDER 32
tt_status tt_tensor_read(const char* path, int32_t* p, int64_t* dims, double* data);

/* ---- queries (query.hpp:33-50) -------------------------------------------- */
/* recall(tree, ts, te, theta); theta = NaN selects the tree's theta
 * (std::nullopt in the reference).                                          */
tt_status tt_recall(const tt_tree* tree, int64_t ts, int64_t te, double theta, tt_hit* out, int64_t cap,
                    int64_t* n);

/* range_query_detailed over a batch: recall on the host, every query's
 * multi-part stitch in one batched launch. `where` says where the out buffers
 * live.                                                    query.hpp:44-50 */
tt_status tt_query_batch(const tt_tree* tree, const tt_range* ranges, int64_t n, double theta, tt_query_out* outs,
                         tt_mem where);

/* Device time (ms, CUDA events) of the last tt_append / tt_query_batch
 * split by phase: [0] leaf ALS, [1] stitches, [2] total device span.      */
tt_status tt_last_timing(const tt_tree* tree, double* ms3);

/* ---- standalone operations (tucker.hpp:48-49, stitch.hpp:15-36) ---------- */
/* tucker_als(x, cfg) on device; x row-major with dims[0..p-1].            */
tt_status tt_tucker_als(const double* x, int32_t p, const int64_t* dims, const int64_t* ranks, int32_t max_iters,
                        double tol, uint64_t seed, int32_t device, tt_factors** out);

/* stitch(parts, ranks, cfg) on device. Part i: core (row-major, part_ranks
 * row i), factors[i*p + m] (column-major D_m x r_m; D_0 = part length).    */
tt_status tt_stitch(int32_t nparts, int32_t p, const int64_t* part_dims, const int64_t* part_ranks,
                    const double* const* cores, const double* const* factors, const int64_t* ranks,
                    int32_t max_iters, double tol, uint64_t seed, int32_t device, tt_factors** out);

/* brute_force_range(series, ts, te, ranks, cfg) for a batch of ranges: the
 * series (row-major, dims[0] = T) in host or device memory; one tucker_als per
 * range, all in one launch. outs[i] receives range i's factors.
 *                                                      baseline.cpp:67-75 */
tt_status tt_brute_force_batch(const double* series, tt_mem where, int32_t p, const int64_t* dims,
                               const int64_t* ranks, const tt_range* ranges, int64_t n, int32_t max_iters, double tol,
                               uint64_t seed, int32_t device, tt_factors** outs);

/* partial_hit_factors(stored, begin, end) on device: thin Householder QR of
 * the kept temporal rows with the reference sign rule, core <- core x_0 R.
 * Inputs are host arrays (factors column-major). Range queries do not use it
 * (partial hits enter their stitch through the metric S = V_sub^T V_sub).
 *                                                          stitch.hpp:15 */
tt_status tt_partial_hit(int32_t p, const int64_t* dims, const int64_t* ranks, const double* core,
                         const double* const* factors, int64_t begin, int64_t end, int32_t device, tt_factors** out);

int32_t tt_factors_order(const tt_factors* f);
int64_t tt_factors_dim(const tt_factors* f, int32_t m);
int64_t tt_factors_rank(const tt_factors* f, int32_t m);
const double* tt_factors_core(const tt_factors* f);
const double* tt_factors_factor(const tt_factors* f, int32_t m);
int32_t tt_factors_sweeps(const tt_factors* f);
int32_t tt_factors_converged(const tt_factors* f);
const double* tt_factors_objective(const tt_factors* f); /* per-sweep squared residual (AlsTrace) */
void tt_factors_free(tt_factors* f);

/* Fault injection (tests): the next n tt_append calls that
 * complete a leaf block fail with TT_ECUDA after their leaf kernels ran, and
 * must leave the tree unchanged (sst.cpp:95-97).                           */
void tt_debug_fail_appends(int32_t n);
/* Number of the engine's own kernels launched since process start (the bench
 * reports the delta over its timed region).                               */
int64_t tt_kernel_launches(void);

/* Cumulative solver counters since process start (instrumentation):
 * [0] ALS problems, [1] ALS sweeps, [2] eigen-solves, [3] Jacobi sweeps,
 * [4..11] thousands of SM cycles summed over problems in: eigen-solves, Gram
 * matrices (+U assembly), small mode products, small GEMMs, orthonormalise +
 * sign fix, U_0 materialisation, leaf X passes, whole problem; [12..13]
 * subspace-iteration solves that converged / fell back to Jacobi, [14]
 * subspace iterations, [15..18] kcycles inside subspace iteration (A^T U,
 * A Y + residual, CholeskyQR2, Rayleigh-Ritz). Entries [0..18] count leaf
 * (tucker_als) problems, [19..37] stitch problems.                        */
void tt_solver_stats(int64_t* out38);
/* Cumulative device time of the grid-wide leaf path's streamed passes over X
 * (grid_ttm_kernel passes 1 and 2; CUDA events on the launching stream):
 * [0] launches, [1] milliseconds, [2] bytes of X read (8 * leaves * B * prod D
 * per launch: the algorithmic bytes of the pass). The bench reports the delta
 * over its timed region as the kernel's achieved HBM bandwidth.            */
void tt_stream_pass_stats(double* out3);

#ifdef __cplusplus
}
#endif

#endif /* TUCKTREE_B200_H */
