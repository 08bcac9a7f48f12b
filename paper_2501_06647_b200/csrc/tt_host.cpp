// Host side of the engine: stream-segment-tree bookkeeping (sst.cpp), recall
// (query.cpp), planning of the batched device work, device memory, and the C
// ABI declared in include/tucktree_b200.h.
//
// The host owns every integer decision (node ids, ranges, kinds, hit sets,
// touched sets, factor column counts); the device owns every floating-point
// operation. There is no CPU numeric fallback: without a working CUDA device
// every numeric entry point fails with TT_ECUDA.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tucktree_b200.h"
#include "tt_common.h"

namespace ttb {
cudaError_t launch_leaf(const Params& prm, const LeafDesc* d_descs, int n, cudaStream_t st);
cudaError_t launch_stitch(const Params& prm, const StitchDesc* d_descs, const StitchPart* d_parts, int n,
                          cudaStream_t st);
int leaf_wide_cluster();
int stitch_wide_cluster();
cudaError_t launch_stitch_wide(const Params& prm, const StitchDesc* d_descs, const StitchPart* d_parts, int n, int cs,
                               cudaStream_t st);
cudaError_t launch_leaf_wide(const Params& prm, const LeafDesc* d_descs, int n, int cs, cudaStream_t st);
// tt_grid.cu: grid-wide phase kernels for wide batches of equal-length leaves
bool leaf_grid_ok(const Params& prm, int64_t len);
void grid_pass_stats(double* out3);
cudaError_t launch_leaf_grid(const Params& prm, const LeafDesc* d_descs, int n, int64_t len, int* d_active,
                             cudaStream_t st);
cudaError_t launch_copy_segments(const CopySeg* d_segs, int n, cudaStream_t st);
cudaError_t launch_partial_hit(const double* V0, int64_t ld, int64_t b, int64_t len, int n, const double* core,
                               int64_t rest, double* W, double* Q, double* R, double* out_core, double* tau,
                               cudaStream_t st);
constexpr int kMaxVecHost = 32;  // the kernel's per-thread column vectors (kMaxVec)
int64_t launches();
}  // namespace ttb

using namespace ttb;
using Index = int64_t;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_stamp{0};
std::atomic<int32_t> g_fail_appends{0};  // tt_debug_fail_appends
uint64_t next_stamp() { return g_stamp.fetch_add(1) + 1; }
// problems, ALS sweeps, eig calls, Jacobi sweeps (cumulative, all trees)
std::atomic<int64_t> g_stats[2][19] = {};  // [0] leaf problems, [1] stitch problems (concurrent readers)

struct TTError : std::runtime_error {
  tt_status code;
  TTError(tt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(tt_status c, const std::string& m) { throw TTError(c, m); }
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
tt_status guarded(F&& f) {
  try {
    f();
    return TT_OK;
  } catch (const TTError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = "out of host memory";
    return TT_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TT_EIO;
  }
}

// ---------------------------------------------------------------------------
// Host init factors: random_orthonormal (linalg.cpp:81-89) — libstdc++
// mt19937_64 + a fresh normal_distribution per call, row-major draws, then a
// Householder thin QR with the sign convention of linalg.cpp:15-31.
std::vector<double> householder_thin_q(std::vector<double> a, Index m, Index n) {
  const Index k = std::min(m, n);
  std::vector<double> tau(static_cast<size_t>(k), 0.0);
  for (Index j = 0; j < k; ++j) {
    double* col = a.data() + j * m;
    double xn = 0.0;
    for (Index i = j + 1; i < m; ++i) xn += col[i] * col[i];
    xn = std::sqrt(xn);
    const double alpha = col[j];
    if (xn == 0.0) {
      tau[j] = 0.0;
      continue;
    }
    const double beta = -std::copysign(std::hypot(alpha, xn), alpha);
    tau[j] = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    for (Index i = j + 1; i < m; ++i) col[i] *= scale;
    col[j] = beta;
    for (Index c = j + 1; c < n; ++c) {
      double* cc = a.data() + c * m;
      double s = cc[j];
      for (Index i = j + 1; i < m; ++i) s += col[i] * cc[i];
      s *= tau[j];
      cc[j] -= s;
      for (Index i = j + 1; i < m; ++i) cc[i] -= s * col[i];
    }
  }
  std::vector<double> q(static_cast<size_t>(m * k), 0.0);
  for (Index j = 0; j < k; ++j) q[j + j * m] = 1.0;
  for (Index j = k - 1; j >= 0; --j) {
    const double* v = a.data() + j * m;
    for (Index c = j; c < k; ++c) {
      double* qc = q.data() + c * m;
      double s = qc[j];
      for (Index i = j + 1; i < m; ++i) s += v[i] * qc[i];
      s *= tau[j];
      qc[j] -= s;
      for (Index i = j + 1; i < m; ++i) qc[i] -= s * v[i];
    }
  }
  for (Index j = 0; j < k; ++j) {
    double* c = q.data() + j * m;
    Index piv = 0;
    double best = -1.0;
    for (Index i = 0; i < m; ++i)
      if (std::abs(c[i]) > best) {
        best = std::abs(c[i]);
        piv = i;
      }
    if (c[piv] < 0.0)
      for (Index i = 0; i < m; ++i) c[i] = -c[i];
  }
  return q;
}

std::vector<double> random_orthonormal(Index rows, Index cols, std::mt19937_64& rng) {
  if (rows < cols) fail(TT_EINVAL, "random_orthonormal: rows < cols");
  std::normal_distribution<double> normal(0.0, 1.0);
  std::vector<double> g(static_cast<size_t>(rows * cols));
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) g[i + j * rows] = normal(rng);
  return householder_thin_q(std::move(g), rows, cols);
}

// ---------------------------------------------------------------------------
// Device memory.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const size_t nb = std::max<size_t>(b + b / 4, 256);  // grow geometrically
    cuda_check(cudaMalloc(&p, nb), "cudaMalloc");
    if (std::getenv("TT_POISON")) {  // debugging: NaN-fill fresh device buffers
      cudaMemset(p, 0xFF, nb);
      cudaDeviceSynchronize();
    }
    bytes = nb;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Bump allocator over large chunks for node decompositions (never moves).
struct Arena {
  std::vector<std::pair<void*, size_t>> chunks;
  size_t ci = 0;  // current chunk
  char* cur = nullptr;
  size_t left = 0;
  static constexpr size_t kChunk = size_t(256) << 20;
  ~Arena() {
    for (auto& c : chunks) cudaFree(c.first);
  }
  // Forget every allocation but keep the chunks for reuse (tt_tree_clear).
  void reset() {
    ci = 0;
    cur = chunks.empty() ? nullptr : static_cast<char*>(chunks[0].first);
    left = chunks.empty() ? 0 : chunks[0].second;
  }
  struct Mark {
    size_t ci;
    char* cur;
    size_t left;
  };
  Mark mark() const { return Mark{ci, cur, left}; }
  // Drops every allocation made after `m` (failed appends roll back).
  void release(const Mark& m) {
    ci = m.ci;
    cur = m.cur;
    left = m.left;
  }
  double* alloc(size_t n_doubles) {
    size_t b = (n_doubles * sizeof(double) + 255) & ~size_t(255);
    if (b == 0) b = 256;
    while (b > left) {
      if (cur != nullptr && ci + 1 < chunks.size()) {  // reuse the next kept chunk
        ++ci;
        cur = static_cast<char*>(chunks[ci].first);
        left = chunks[ci].second;
        continue;
      }
      const size_t cb = std::max(kChunk, b);
      void* c = nullptr;
      cuda_check(cudaMalloc(&c, cb), "cudaMalloc(arena)");
      if (std::getenv("TT_POISON")) {
        cudaMemset(c, 0xFF, cb);
        cudaDeviceSynchronize();
      }
      chunks.emplace_back(c, cb);
      ci = chunks.size() - 1;
      cur = static_cast<char*>(c);
      left = cb;
    }
    double* r = reinterpret_cast<double*>(cur);
    cur += b;
    left -= b;
    return r;
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Per-device execution context: one stream, staging buffers and timers.
struct Exec {
  int device = 0;
  cudaStream_t stream = nullptr;
  DevBuf d_desc, d_parts, d_ws, d_status, d_obj, d_stage, d_tmaps, d_segs;
  std::vector<char> h_status_bytes;
  cudaStream_t copy = nullptr;  // device-to-host result downloads, overlapping later launches
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  static constexpr int kWaveEvents = 16;
  cudaEvent_t wave_ev[kWaveEvents] = {};
  explicit Exec(int dev) : device(dev) {
    DeviceGuard g(dev);
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    for (auto& e : wave_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  }
  ~Exec() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : wave_ev)
      if (e) cudaEventDestroy(e);
    if (copy) cudaStreamDestroy(copy);
    if (stream) cudaStreamDestroy(stream);
  }
  void sync() { cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }
  void sync_copy() { cuda_check(cudaStreamSynchronize(copy), "cudaStreamSynchronize"); }
};

// Device view of a pinned (page-locked, UVA-mapped) host buffer, or null.
double* mapped_device_ptr(void* host) {
  if (!host) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeHost && a.devicePointer != nullptr) return static_cast<double*>(a.devicePointer);
  return nullptr;
}

// Result of one batched ALS problem after readback.
struct ProblemStatus {
  int sweeps = 0, converged = 0, zero = 0, deficient = 0, eig_calls = 0, eig_sweeps = 0;
  Index k[kMaxP] = {};
  std::vector<double> objective;
};

// TMA tensor maps for the two streamed passes over a leaf block X (row-major
// (len, D_1, rest)): [0] X as 3-D (rest, D_1, len) for Y = X x_1 U_1^T, [1] X as
// 2-D (ns, len) for W = X x_0 U_0^T. Box shapes come from stream_tile(), the
// same function the kernel's tile loop uses. Returns false when the layout is
// not TMA-compatible (16-byte strides/box rows); the kernel then falls back.
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

bool encode_leaf_maps(const double* x, Index len, Index d1, Index rest, CUtensorMap* out) {
  auto enc = tensor_map_encoder();
  if (!enc || (reinterpret_cast<uintptr_t>(x) & 15u) != 0) return false;
  const Index ns = d1 * rest;
  const StreamTile ta = stream_tile(len, d1, rest), tb = stream_tile(1, len, ns);
  if ((rest * 8) % 16 || (ta.tw * 8) % 16 || (tb.tw * 8) % 16) return false;
  {
    const cuuint64_t dims[3] = {cuuint64_t(rest), cuuint64_t(d1), cuuint64_t(len)};
    const cuuint64_t strides[2] = {cuuint64_t(rest * 8), cuuint64_t(d1 * rest * 8)};
    const cuuint32_t box[3] = {cuuint32_t(ta.tw), cuuint32_t(ta.cj), cuuint32_t(ta.G)};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&out[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  {
    const cuuint64_t dims[2] = {cuuint64_t(ns), cuuint64_t(len)};
    const cuuint64_t strides[1] = {cuuint64_t(ns * 8)};
    const cuuint32_t box[2] = {cuuint32_t(tb.tw), cuuint32_t(tb.cj)};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&out[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

// Uploads descriptors, runs a leaf batch, reads statuses back (synchronous).
std::vector<ProblemStatus> run_leaf_batch(Exec& ex, const Params& prm, std::vector<LeafDesc>& descs,
                                          const std::vector<Index>& ws_sizes) {
  const int n = static_cast<int>(descs.size());
  std::vector<ProblemStatus> st(static_cast<size_t>(n));
  if (n == 0) return st;
  // Few problems: one thread-block cluster per problem (leaf_wide_kernel) so a
  // single streamed leaf or query tail uses 8-16 SMs; wide batches: one CTA
  // per problem. TT_WIDE=0/1 forces either path (A/B measurement).
  const int cs = leaf_wide_cluster();
  bool wide = cs > 0 && prm.p >= 2;
  if (wide) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ex.device);
    wide = n <= 2 * std::max(1, nsm / cs);
    if (const char* e = std::getenv("TT_WIDE")) wide = e[0] == '1';
  }
  // Batches of equal-length, 16-byte-aligned blocks: the grid-wide phase
  // kernels (tt_grid.cu) stream X across the whole GPU. TT_GRID=0 disables the
  // path, 1 keeps the cluster kernel for small batches, 2 (default) takes it
  // for every eligible batch but wide batches of small blocks, 3 for those too
  // (A/B measurement, tests).
  int grid_mode = 2;
  if (const char* e = std::getenv("TT_GRID")) grid_mode = std::atoi(e);
  bool grid = grid_mode > 0 && (grid_mode >= 2 || !wide) && leaf_grid_ok(prm, descs[0].len);
  for (int i = 0; grid && i < n; ++i)
    grid = descs[i].len == descs[0].len && (reinterpret_cast<uintptr_t>(descs[i].x) & 15u) == 0;
  // Wide batches of small blocks (C1: 0.26 MB, C2: 2.3 MB per leaf) are bound by
  // the per-leaf solvers, not by the passes over X: one CTA per leaf keeps each
  // leaf's working set in one SM's L1 and measured 10% faster there. TT_GRID=3
  // takes the grid path regardless (tests).
  if (grid && !wide && grid_mode < 3 &&
      double(descs[0].len) * double(prod_range(prm.d, 1, prm.p)) * sizeof(double) < 4.0e6)
    grid = false;
  if (grid) wide = false;
  std::vector<Index> wsz(ws_sizes);
  if (wide)  // + the per-CTA partial Gram slots of the cluster kernel
    for (int i = 0; i < n; ++i) wsz[i] = leaf_ws_layout(prm.p, descs[i].len, prm.d, prm.req, cs).total;
  if (grid)  // + transposed factors, norm partials and the carried ALS state
    for (int i = 0; i < n; ++i) wsz[i] = grid_ws_layout(prm.p, descs[i].len, prm.d, prm.req).total;
  size_t ws_total = 0;
  for (Index w : wsz) ws_total += static_cast<size_t>(w);
  ex.d_ws.ensure(ws_total * sizeof(double));
  // TT_POISON=1 (debugging): fill the workspace with NaNs so that a read of a
  // region no kernel has written shows up in the results
  if (std::getenv("TT_POISON"))
    cuda_check(cudaMemsetAsync(ex.d_ws.p, 0xFF, ws_total * sizeof(double), ex.stream), "workspace poison");
  ex.d_status.ensure((size_t(n) * kStatusInts + size_t(prm.max_iters)) * sizeof(int32_t));
  ex.d_obj.ensure(size_t(n) * prm.max_iters * sizeof(double));
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    descs[i].ws = ex.d_ws.as<double>() + off;
    off += static_cast<size_t>(wsz[i]);
    descs[i].status = ex.d_status.as<int32_t>() + size_t(i) * kStatusInts;
    descs[i].objective = ex.d_obj.as<double>() + size_t(i) * prm.max_iters;
  }
  // TMA tensor maps (two per leaf, 64-byte aligned) for the streamed X passes
  if (prm.p >= 2 && !grid) {
    std::vector<CUtensorMap> maps(size_t(2) * n);
    ex.d_tmaps.ensure(sizeof(CUtensorMap) * 2 * n + 128);
    CUtensorMap* dmaps = reinterpret_cast<CUtensorMap*>((reinterpret_cast<uintptr_t>(ex.d_tmaps.p) + 127) & ~uintptr_t(127));
    for (int i = 0; i < n; ++i) {
      const Index rest = prod_range(prm.d, 2, prm.p);
      const bool ok = encode_leaf_maps(descs[i].x, descs[i].len, prm.d[1], rest, &maps[2 * i]);
      descs[i].tmaps = ok ? static_cast<const void*>(dmaps + 2 * i) : nullptr;
    }
    cuda_check(cudaMemcpyAsync(dmaps, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice,
                               ex.stream),
               "upload tensor maps");
  }
  ex.d_desc.ensure(sizeof(LeafDesc) * n);
  cuda_check(cudaMemcpyAsync(ex.d_desc.p, descs.data(), sizeof(LeafDesc) * n, cudaMemcpyHostToDevice, ex.stream),
             "upload leaf descriptors");
  if (grid)
    cuda_check(launch_leaf_grid(prm, ex.d_desc.as<LeafDesc>(), n, descs[0].len,
                                ex.d_status.as<int32_t>() + size_t(n) * kStatusInts, ex.stream),
               "grid leaf kernels");
  else if (wide)
    cuda_check(launch_leaf_wide(prm, ex.d_desc.as<LeafDesc>(), n, cs, ex.stream), "leaf_wide_kernel launch");
  else
    cuda_check(launch_leaf(prm, ex.d_desc.as<LeafDesc>(), n, ex.stream), "leaf_als_kernel launch");
  std::vector<int32_t> hs(size_t(n) * kStatusInts);
  std::vector<double> ho(size_t(n) * prm.max_iters);
  cuda_check(cudaMemcpyAsync(hs.data(), ex.d_status.p, hs.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, ex.stream),
             "status readback");
  cuda_check(cudaMemcpyAsync(ho.data(), ex.d_obj.p, ho.size() * sizeof(double), cudaMemcpyDeviceToHost, ex.stream),
             "objective readback");
  ex.sync();
  for (int i = 0; i < n; ++i) {
    const int32_t* s = hs.data() + size_t(i) * kStatusInts;
    st[i].sweeps = s[0];
    st[i].converged = s[1];
    st[i].zero = s[2];
    st[i].deficient = s[3];
    for (int m = 0; m < kMaxP; ++m) st[i].k[m] = s[4 + m];
    st[i].eig_calls = s[4 + kMaxP];
    st[i].eig_sweeps = s[5 + kMaxP];
    g_stats[0][0] += 1;
    g_stats[0][1] += s[0];
    g_stats[0][2] += s[4 + kMaxP];
    g_stats[0][3] += s[5 + kMaxP];
    for (int q = 0; q < 8; ++q) g_stats[0][4 + q] += s[6 + kMaxP + q];
    g_stats[0][12] += s[14 + kMaxP];
    g_stats[0][13] += s[15 + kMaxP];
    g_stats[0][14] += s[16 + kMaxP];
    for (int q = 0; q < 4; ++q) g_stats[0][15 + q] += s[17 + kMaxP + q];
    st[i].objective.assign(ho.begin() + size_t(i) * prm.max_iters, ho.begin() + size_t(i) * prm.max_iters + s[0]);
  }
  return st;
}

// Launch-order cost model of a stitch problem, in temporal rows: U0
// materialisation is linear in L, the solver work grows with the part count.
// (measured at C2: 10000 for the launch order; the DMA wave split, which
// decides when the end-to-end download starts, prefers 20000)
constexpr double kPartCost = 10000.0;
constexpr double kWavePartCost = 20000.0;

std::vector<ProblemStatus> run_stitch_batch(Exec& ex, const Params& prm, std::vector<StitchDesc>& descs_in,
                                            const std::vector<StitchPart>& parts, const std::vector<Index>& ws_sizes) {
  const int n = static_cast<int>(descs_in.size());
  std::vector<ProblemStatus> st_out(static_cast<size_t>(n));
  if (n == 0) return st_out;
  for (const StitchDesc& d : descs_in) {  // the kernel's shared-memory row tables
    Index rows = 0;
    for (int i = 0; i < d.nparts; ++i) rows += parts[size_t(d.part0) + i].rho[0];
    if (rows > kStitchMaxRows)
      fail(TT_EINVAL, "stitch: the parts' temporal ranks sum to more than " + std::to_string(kStitchMaxRows));
  }
  // Launch longest-first: CTAs are dispatched roughly in index order and query
  // costs vary ~100x (L and the part count), so LPT order shrinks the tail.
  std::vector<int> perm(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) perm[i] = i;
  auto cost = [&](int i) { return double(descs_in[i].L) + kPartCost * descs_in[i].nparts; };
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return cost(a) > cost(b); });
  std::vector<StitchDesc> descs(static_cast<size_t>(n));
  std::vector<Index> wsz(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    descs[i] = descs_in[perm[i]];
    wsz[i] = ws_sizes[perm[i]];
  }
  std::vector<ProblemStatus> st(static_cast<size_t>(n));
  // Few problems (streamed appends, single queries): one thread-block cluster
  // per problem (stitch_wide_kernel); TT_WIDE=0/1 forces either path.
  const int cs = stitch_wide_cluster();
  bool wide = cs > 0;
  if (wide) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ex.device);
    wide = n <= std::max(1, nsm / cs);
    if (const char* e = std::getenv("TT_WIDE")) wide = e[0] == '1';
  }
  if (wide)  // + exchange slots and per-CTA partial Grams
    for (int i = 0; i < n; ++i) {
      Index rho_max[kMaxP] = {};
      for (int j = 0; j < descs[i].nparts; ++j)
        for (int m = 0; m < prm.p; ++m) rho_max[m] = std::max(rho_max[m], parts[size_t(descs[i].part0) + j].rho[m]);
      wsz[i] = stitch_ws_layout(prm.p, descs[i].L, prm.d, prm.req, rho_max, descs[i].nparts, cs).total;
    }
  const std::vector<Index>& ws_sizes_p = wsz;
  size_t ws_total = 0;
  for (Index w : ws_sizes_p) ws_total += static_cast<size_t>(w);
  ex.d_ws.ensure(ws_total * sizeof(double));
  ex.d_status.ensure(size_t(n) * kStatusInts * sizeof(int32_t));
  ex.d_obj.ensure(size_t(n) * prm.max_iters * sizeof(double));
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    descs[i].ws = ex.d_ws.as<double>() + off;
    off += static_cast<size_t>(ws_sizes_p[i]);
    descs[i].status = ex.d_status.as<int32_t>() + size_t(i) * kStatusInts;
    descs[i].objective = ex.d_obj.as<double>() + size_t(i) * prm.max_iters;
  }
  ex.d_desc.ensure(sizeof(StitchDesc) * n);
  ex.d_parts.ensure(sizeof(StitchPart) * std::max<size_t>(parts.size(), 1));
  cuda_check(cudaMemcpyAsync(ex.d_desc.p, descs.data(), sizeof(StitchDesc) * n, cudaMemcpyHostToDevice, ex.stream),
             "upload stitch descriptors");
  cuda_check(cudaMemcpyAsync(ex.d_parts.p, parts.data(), sizeof(StitchPart) * parts.size(), cudaMemcpyHostToDevice,
                             ex.stream),
             "upload stitch parts");
  if (wide)
    cuda_check(launch_stitch_wide(prm, ex.d_desc.as<StitchDesc>(), ex.d_parts.as<StitchPart>(), n, cs, ex.stream),
               "stitch_wide_kernel launch");
  else
    cuda_check(launch_stitch(prm, ex.d_desc.as<StitchDesc>(), ex.d_parts.as<StitchPart>(), n, ex.stream),
               "stitch_als_kernel launch");
  std::vector<int32_t> hs(size_t(n) * kStatusInts);
  std::vector<double> ho(size_t(n) * prm.max_iters);
  cuda_check(cudaMemcpyAsync(hs.data(), ex.d_status.p, hs.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, ex.stream),
             "status readback");
  cuda_check(cudaMemcpyAsync(ho.data(), ex.d_obj.p, ho.size() * sizeof(double), cudaMemcpyDeviceToHost, ex.stream),
             "objective readback");
  ex.sync();
  for (int i = 0; i < n; ++i) {
    const int32_t* s = hs.data() + size_t(i) * kStatusInts;
    st[i].sweeps = s[0];
    st[i].converged = s[1];
    st[i].zero = s[2];
    st[i].deficient = s[3];
    for (int m = 0; m < kMaxP; ++m) st[i].k[m] = s[4 + m];
    st[i].eig_calls = s[4 + kMaxP];
    st[i].eig_sweeps = s[5 + kMaxP];
    g_stats[1][0] += 1;
    g_stats[1][1] += s[0];
    g_stats[1][2] += s[4 + kMaxP];
    g_stats[1][3] += s[5 + kMaxP];
    for (int q = 0; q < 8; ++q) g_stats[1][4 + q] += s[6 + kMaxP + q];
    g_stats[1][12] += s[14 + kMaxP];
    g_stats[1][13] += s[15 + kMaxP];
    g_stats[1][14] += s[16 + kMaxP];
    for (int q = 0; q < 4; ++q) g_stats[1][15 + q] += s[17 + kMaxP + q];
    st[i].objective.assign(ho.begin() + size_t(i) * prm.max_iters, ho.begin() + size_t(i) * prm.max_iters + s[0]);
  }
  for (int i = 0; i < n; ++i) {
    st_out[perm[i]] = std::move(st[i]);
    descs_in[perm[i]].ws = descs[i].ws;
    descs_in[perm[i]].status = descs[i].status;
    descs_in[perm[i]].objective = descs[i].objective;
  }
  return st_out;
}

// Shared per-shape constants: leaf init factors per block length and the
// stitch init factors (one rng(seed) stream per ALS call, tucker.cpp:29 and
// stitch.cpp:135, so they are per-shape constants).
struct InitCache {
  int p = 0;
  Index d[kMaxP] = {};
  Index req[kMaxP] = {};
  uint64_t seed = 0;
  std::map<Index, std::vector<std::unique_ptr<DevBuf>>> leaf;  // by block length
  std::vector<std::unique_ptr<DevBuf>> stitch;                 // m >= 1 (index m)
  std::mutex mu;  // concurrent readers fill the caches (map nodes never move)

  const std::vector<std::unique_ptr<DevBuf>>& leaf_init(Index len, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = leaf.find(len);
    if (it != leaf.end()) return it->second;
    Index dd[kMaxP], rc[kMaxP];
    dd[0] = len;
    for (int m = 1; m < p; ++m) dd[m] = d[m];
    clamp_ranks(p, dd, req, rc);
    std::mt19937_64 rng(seed);
    std::vector<std::unique_ptr<DevBuf>> v;
    for (int m = 0; m < p; ++m) {
      const auto q = random_orthonormal(dd[m], rc[m], rng);
      auto b = std::make_unique<DevBuf>();
      b->ensure(q.size() * sizeof(double));
      cuda_check(cudaMemcpyAsync(b->p, q.data(), q.size() * sizeof(double), cudaMemcpyHostToDevice, st), "init upload");
      cuda_check(cudaStreamSynchronize(st), "init upload sync");
      v.push_back(std::move(b));
    }
    return leaf.emplace(len, std::move(v)).first->second;
  }
  void stitch_init(Params& prm, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(mu);
    if (stitch.empty()) {
      std::mt19937_64 rng(seed);
      stitch.resize(static_cast<size_t>(p));
      for (int m = 1; m < p; ++m) {
        const auto q = random_orthonormal(d[m], std::min(req[m], d[m]), rng);
        stitch[m] = std::make_unique<DevBuf>();
        stitch[m]->ensure(q.size() * sizeof(double));
        cuda_check(cudaMemcpyAsync(stitch[m]->p, q.data(), q.size() * sizeof(double), cudaMemcpyHostToDevice, st),
                   "stitch init upload");
        cuda_check(cudaStreamSynchronize(st), "stitch init sync");
      }
    }
    for (int m = 1; m < p; ++m) prm.stitch_init[m] = stitch[m]->as<double>();
  }
  // stitch.cpp:146-150 zero path: U_0 = random_orthonormal(L, r0) drawn after the U_m.
  std::vector<double> stitch_zero_u0(Index L, Index r0) const {
    std::mt19937_64 rng(seed);
    for (int m = 1; m < p; ++m) (void)random_orthonormal(d[m], std::min(req[m], d[m]), rng);
    return random_orthonormal(L, r0, rng);
  }
};

Params make_params(int p, const Index* d, const Index* req, int max_iters, double tol) {
  Params prm{};
  prm.p = p;
  prm.max_iters = max_iters;
  prm.tol = tol;
  for (int m = 0; m < kMaxP; ++m) {
    prm.d[m] = m < p ? d[m] : 1;
    prm.req[m] = m < p ? req[m] : 1;
    prm.stitch_init[m] = nullptr;
  }
  return prm;
}

}  // namespace

// ===========================================================================
// Tree
struct HostNode {
  Index id = 0, begin = 0, end = 0;  // slices
  int kind = TT_PLACEHOLDER;
  Index left = 0, right = 0;
  bool has_dec = false;
  Index ranks[kMaxP] = {};
  double* f[kMaxP] = {};  // device factor slots (capacity clamped ranks)
  double* core = nullptr;
  Index length() const { return end - begin; }
};

struct tt_tree {
  tt_config cfg{};
  int p = 0;
  Index d[kMaxP] = {};  // d[0] unused
  Index B = 1, slice = 1;
  bool structure_only = false;
  std::vector<HostNode> nodes;
  Index root = 0, timespan = 0, leaves = 0, stitch_count = 0, last_touches = 0;
  std::vector<Index> last_redec;
  std::unique_ptr<Exec> ex;
  std::unique_ptr<Arena> arena;
  DevBuf tail;  // B slices (device)
  InitCache init;
  DevBuf stage;  // host-burst staging
  double timing[3] = {0, 0, 0};
  uint64_t timing_stamp = 0;
  mutable std::mutex qmu;  // serialises tt_tree_save
  // Query contexts: one stream + workspace per calling thread, so any number of
  // readers run concurrently between appends (sst.hpp:52-53).
  struct Reader {
    std::unique_ptr<Exec> ex;
    DevBuf qout, qscratch, tailq;
    double timing[3] = {0, 0, 0};
    uint64_t stamp = 0;
  };
  std::mutex rmu;
  std::map<std::thread::id, std::unique_ptr<Reader>> readers;
  Reader& reader() {
    std::lock_guard<std::mutex> lk(rmu);
    auto& r = readers[std::this_thread::get_id()];
    if (!r) {
      r = std::make_unique<Reader>();
      r->ex = std::make_unique<Exec>(ex->device);
    }
    return *r;
  }
  Reader* reader_if_any() {
    std::lock_guard<std::mutex> lk(rmu);
    auto it = readers.find(std::this_thread::get_id());
    return it == readers.end() ? nullptr : it->second.get();
  }
  // Append journal: pre-call copies of the existing nodes an append modifies
  // (at most the root-to-leaf paths), so a failed append can be rolled back.
  Index journal_n0 = -1;
  std::vector<HostNode> journal;
  void journal_save(Index id) {
    if (journal_n0 < 0 || id > journal_n0) return;
    for (const HostNode& v : journal)
      if (v.id == id) return;
    journal.push_back(node(id));
  }

  HostNode& node(Index id) { return nodes[static_cast<size_t>(id - 1)]; }
  const HostNode& node(Index id) const {
    if (id < 1 || id > static_cast<Index>(nodes.size())) fail(TT_ERANGE, "StreamSegmentTree::node: unknown node id " + std::to_string(id));
    return nodes[static_cast<size_t>(id - 1)];
  }
  Index clamped(int m, Index len) const { return std::min(cfg.ranks[m], m == 0 ? len : d[m]); }
  Index create_node(Index b_leaf, Index e_leaf) {
    HostNode n;
    n.id = static_cast<Index>(nodes.size() + 1);
    n.begin = b_leaf * B;
    n.end = e_leaf * B;
    nodes.push_back(n);
    return nodes.back().id;
  }
  void alloc_slots(HostNode& v) {
    if (structure_only || v.core) return;
    Index rc[kMaxP];
    for (int m = 0; m < p; ++m) rc[m] = clamped(m, v.length());
    v.f[0] = arena->alloc(static_cast<size_t>(v.length() * rc[0]));
    for (int m = 1; m < p; ++m) v.f[m] = arena->alloc(static_cast<size_t>(d[m] * rc[m]));
    v.core = arena->alloc(static_cast<size_t>(prod_range(rc, 0, p)));
  }
  Index height() const {
    if (root == 0) return 0;
    // robust to corrupted node tables (from_parts + validate): unknown ids
    // count as absent, cycles are cut at depth N
    const Index N = static_cast<Index>(nodes.size());
    std::function<Index(Index, Index)> depth = [&](Index id, Index lvl) -> Index {
      if (id < 1 || id > N || lvl > N) return 0;
      const HostNode& v = nodes[static_cast<size_t>(id - 1)];
      Index best = 0;
      if (v.left) best = std::max(best, depth(v.left, lvl + 1));
      if (v.right) best = std::max(best, depth(v.right, lvl + 1));
      return best + 1;
    };
    return depth(root, 1);
  }
};

namespace {

// sst.cpp:112-145 in leaf units: records the leaf and the completed parents.
struct PendingWork {
  std::vector<std::pair<Index, Index>> leaves;  // (node id, leaf index)
  std::vector<Index> stitches;                  // node ids in completion order
};

void insert_leaf(tt_tree& t, Index id, Index leaf_idx, PendingWork& w) {
  t.journal_save(id);
  ++t.last_touches;
  const Index b = t.node(id).begin / t.B, e = t.node(id).end / t.B;
  if (b == leaf_idx && e == leaf_idx + 1) {
    HostNode& v = t.node(id);
    v.kind = TT_LEAF;
    w.leaves.emplace_back(id, leaf_idx);
    t.last_redec.push_back(id);
    return;
  }
  const Index mid = (b + e) / 2;
  if (leaf_idx < mid) {
    if (t.node(id).left == 0) {
      const Index c = t.create_node(b, mid);
      t.node(id).left = c;
    }
    insert_leaf(t, t.node(id).left, leaf_idx, w);
  } else {
    if (t.node(id).right == 0) {
      const Index c = t.create_node(mid, e);
      t.node(id).right = c;
    }
    insert_leaf(t, t.node(id).right, leaf_idx, w);
    if (e == leaf_idx + 1) {
      HostNode& v = t.node(id);
      v.kind = TT_INTERMEDIATE;
      ++t.stitch_count;
      w.stitches.push_back(id);
      t.last_redec.push_back(id);
    }
  }
}

void add_leaf(tt_tree& t, PendingWork& w) {  // sst.cpp:94-110, in leaf units
  t.last_touches = 0;
  t.last_redec.clear();
  const Index li = t.leaves;
  if (li == 0) {
    t.root = t.create_node(0, 1);
  } else if (t.node(t.root).end == li * t.B) {
    const Index promoted = t.create_node(0, 2 * li);
    t.node(promoted).left = t.root;
    t.root = promoted;
  }
  insert_leaf(t, t.root, li, w);
  ++t.leaves;
}

void planned_final_ranks(const tt_tree& t, Index len, bool leaf, Index* out) {
  Index dd[kMaxP], rc[kMaxP], k[kMaxP];
  dd[0] = len;
  for (int m = 1; m < t.p; ++m) dd[m] = t.d[m];
  clamp_ranks(t.p, dd, t.cfg.ranks, rc);
  for (int m = 0; m < t.p; ++m) k[m] = rc[m];
  for (int m = 0; m < t.p; ++m)
    k[m] = leaf ? leaf_mode_rank(t.p, dd, k, m) : stitch_mode_rank(t.p, dd, rc, k, m);
  for (int m = 0; m < t.p; ++m) out[m] = k[m];
}

Params tree_params(tt_tree& t) {
  Params prm = make_params(t.p, t.d, t.cfg.ranks, t.cfg.max_iters, t.cfg.tol);
  return prm;
}

// Runs the pending leaf decompositions (block pointers given) then the stitch
// levels, updating node ranks from the device status.
void execute(tt_tree& t, PendingWork& w, const std::vector<const double*>& leaf_x) {
  if (t.structure_only) {
    for (auto& [id, li] : w.leaves) {
      HostNode& v = t.node(id);
      v.has_dec = true;
      planned_final_ranks(t, v.length(), true, v.ranks);
    }
    for (Index id : w.stitches) {
      HostNode& v = t.node(id);
      v.has_dec = true;
      planned_final_ranks(t, v.length(), false, v.ranks);
    }
    return;
  }
  Exec& ex = *t.ex;
  DeviceGuard g(ex.device);
  Params prm = tree_params(t);
  cuda_check(cudaEventRecord(ex.ev[0], ex.stream), "event");
  // ---- leaves
  if (!w.leaves.empty()) {
    const auto& init = t.init.leaf_init(t.B, ex.stream);
    std::vector<LeafDesc> descs;
    std::vector<Index> ws;
    for (size_t i = 0; i < w.leaves.size(); ++i) {
      HostNode& v = t.node(w.leaves[i].first);
      t.alloc_slots(v);
      LeafDesc dsc{};
      dsc.x = leaf_x[i];
      dsc.len = t.B;
      for (int m = 0; m < t.p; ++m) {
        dsc.init[m] = init[m]->as<double>();
        dsc.out_f[m] = v.f[m];
      }
      dsc.out_core = v.core;
      descs.push_back(dsc);
      ws.push_back(leaf_ws_layout(t.p, t.B, t.d, t.cfg.ranks).total);
    }
    const auto st = run_leaf_batch(ex, prm, descs, ws);
    for (size_t i = 0; i < w.leaves.size(); ++i) {
      HostNode& v = t.node(w.leaves[i].first);
      v.has_dec = true;
      for (int m = 0; m < t.p; ++m) v.ranks[m] = st[i].k[m];
    }
  }
  if (!w.leaves.empty() && g_fail_appends.load() > 0 && g_fail_appends.fetch_sub(1) > 0)
    fail(TT_ECUDA, "injected append failure (tt_debug_fail_appends)");
  cuda_check(cudaEventRecord(ex.ev[1], ex.stream), "event");
  // ---- stitches, level by level (children always complete at a lower level)
  if (!w.stitches.empty()) {
    t.init.stitch_init(prm, ex.stream);
    std::map<Index, std::vector<Index>> by_level;
    for (Index id : w.stitches) {
      Index len = t.node(id).length() / t.B, lvl = 0;
      while ((Index(1) << lvl) < len) ++lvl;
      by_level[lvl].push_back(id);
    }
    for (auto& [lvl, ids] : by_level) {
      std::vector<StitchDesc> descs;
      std::vector<StitchPart> parts;
      std::vector<Index> ws;
      for (Index id : ids) {
        HostNode& v = t.node(id);
        t.alloc_slots(v);
        StitchDesc dsc{};
        dsc.part0 = static_cast<int32_t>(parts.size());
        dsc.nparts = 2;
        dsc.L = v.length();
        Index rho_max[kMaxP] = {};
        for (Index cid : {v.left, v.right}) {
          const HostNode& c = t.node(cid);
          if (!c.has_dec) fail(TT_ELOGIC, "stitch child has no decomposition");
          StitchPart sp{};
          sp.core = c.core;
          for (int m = 0; m < t.p; ++m) {
            sp.rho[m] = c.ranks[m];
            rho_max[m] = std::max(rho_max[m], c.ranks[m]);
            sp.v[m] = c.f[m];
          }
          sp.v0 = c.f[0];
          sp.ld0 = c.length();
          sp.row0 = 0;
          sp.len = c.length();
          sp.partial = 0;
          parts.push_back(sp);
        }
        for (int m = 0; m < t.p; ++m) dsc.out_f[m] = v.f[m];
        dsc.out_core = v.core;
        descs.push_back(dsc);
        ws.push_back(stitch_ws_layout(t.p, v.length(), t.d, t.cfg.ranks, rho_max, 2).total);
      }
      const auto st = run_stitch_batch(ex, prm, descs, parts, ws);
      for (size_t i = 0; i < ids.size(); ++i) {
        HostNode& v = t.node(ids[i]);
        v.has_dec = true;
        for (int m = 0; m < t.p; ++m) v.ranks[m] = st[i].k[m];
        if (st[i].zero) {
          const Index r0 = t.clamped(0, v.length());
          const auto u0 = t.init.stitch_zero_u0(v.length(), r0);
          cuda_check(cudaMemcpyAsync(v.f[0], u0.data(), u0.size() * sizeof(double), cudaMemcpyHostToDevice, ex.stream),
                     "zero-path upload");
          ex.sync();
        }
      }
    }
  }
  cuda_check(cudaEventRecord(ex.ev[2], ex.stream), "event");
  ex.sync();
  float a = 0, b = 0;
  cudaEventElapsedTime(&a, ex.ev[0], ex.ev[1]);
  cudaEventElapsedTime(&b, ex.ev[1], ex.ev[2]);
  t.timing[0] = a;
  t.timing[1] = b;
  t.timing[2] = a + b;
  t.timing_stamp = next_stamp();
}

// query.cpp:9-31 plus the leaf-block rule (an overlapping leaf is always a hit).
void collect_hits(const tt_tree& t, Index id, Index ts, Index te, double theta, std::vector<tt_hit>& out) {
  const HostNode& v = t.node(id);
  const Index overlap = std::min(te, v.end) - std::max(ts, v.begin);
  if (v.kind != TT_PLACEHOLDER &&
      (static_cast<double>(overlap) >= theta * static_cast<double>(v.length()) || v.kind == TT_LEAF)) {
    const bool contained = v.begin >= ts && v.end <= te;
    out.push_back(tt_hit{id, std::max(ts, v.begin), std::min(te, v.end), contained ? TT_HIT_ENTIRE : TT_HIT_PARTIAL, 0});
    return;
  }
  if (v.left && te <= t.node(v.left).end) {
    collect_hits(t, v.left, ts, te, theta, out);
  } else if (v.right && ts >= t.node(v.right).begin) {
    collect_hits(t, v.right, ts, te, theta, out);
  } else {
    if (!v.left || !v.right) fail(TT_ELOGIC, "recall: query spans an unmaterialized range");
    collect_hits(t, v.left, ts, te, theta, out);
    collect_hits(t, v.right, ts, te, theta, out);
  }
}

std::vector<tt_hit> recall(const tt_tree& t, Index ts, Index te, double theta_in) {  // query.cpp:35-47
  if (ts < 0 || ts >= te || te > t.timespan) fail(TT_EINVAL, "recall: query range must satisfy 0 <= ts < te <= T");
  const double theta = std::isnan(theta_in) ? t.cfg.theta : theta_in;
  if (!(theta > 0.0 && theta < 1.0)) fail(TT_EINVAL, "recall: theta must be in (0, 1)");
  std::vector<tt_hit> out;
  const Index tb = t.leaves * t.B;
  if (ts < tb) collect_hits(t, t.root, ts, std::min(te, tb), theta, out);
  if (te > tb) out.push_back(tt_hit{0, std::max(ts, tb), te, TT_HIT_TAIL, 0});
  return out;
}

}  // namespace

// ===========================================================================
// Standalone factors handle
struct tt_factors {
  int p = 0;
  Index dims[kMaxP] = {}, ranks[kMaxP] = {};
  std::vector<double> core;
  std::vector<std::vector<double>> f;
  std::vector<double> objective;
  int sweeps = 0, converged = 0;
};

extern "C" {

const char* tt_last_error(void) { return g_err.c_str(); }
const char* tt_version(void) { return "tucktree_b200 0.2 (sm_100a)"; }
void tt_debug_fail_appends(int32_t n) { g_fail_appends.store(n); }
int64_t tt_kernel_launches(void) { return launches(); }
void tt_stream_pass_stats(double* out3) { ttb::grid_pass_stats(out3); }
void tt_solver_stats(int64_t* out38) {
  for (int k = 0; k < 2; ++k)
    for (int i = 0; i < 19; ++i) out38[k * 19 + i] = g_stats[k][i];
}

tt_status tt_tree_create(const tt_config* cfg, tt_tree** out) {
  return guarded([&] {
    if (!cfg || !out) fail(TT_EINVAL, "tt_tree_create: null argument");
    *out = nullptr;
    const int p = cfg->order;
    if (p < 2 || p > TT_MAX_ORDER) fail(TT_EINVAL, "StreamSegmentTree: order must be in [2, 8]");
    for (int m = 0; m < p - 1; ++m)
      if (cfg->nontemporal[m] < 1) fail(TT_EINVAL, "StreamSegmentTree: extents must be >= 1");
    for (int m = 0; m < p; ++m) {
      if (cfg->ranks[m] < 1) fail(TT_EINVAL, "StreamSegmentTree: ranks must be >= 1");
      if (cfg->ranks[m] > 32) fail(TT_EINVAL, "StreamSegmentTree: ranks above 32 are not supported by this build");
    }
    if (!(cfg->theta > 0.0 && cfg->theta < 1.0)) fail(TT_EINVAL, "StreamSegmentTree: theta must be in (0, 1)");
    if (cfg->max_iters < 1) fail(TT_EINVAL, "max_iters must be >= 1");
    if (cfg->tol <= 0.0) fail(TT_EINVAL, "tol must be > 0");
    if (cfg->leaf_block < 1) fail(TT_EINVAL, "leaf_block must be >= 1");
    auto t = std::make_unique<tt_tree>();
    t->cfg = *cfg;
    t->p = p;
    t->B = cfg->leaf_block;
    t->d[0] = 1;
    t->slice = 1;
    for (int m = 1; m < p; ++m) {
      t->d[m] = cfg->nontemporal[m - 1];
      t->slice *= t->d[m];
    }
    t->structure_only = (cfg->flags & TT_FLAG_STRUCTURE_ONLY) != 0;
    t->init.p = p;
    for (int m = 0; m < p; ++m) {
      t->init.d[m] = t->d[m];
      t->init.req[m] = cfg->ranks[m];
    }
    t->init.seed = cfg->seed;
    if (!t->structure_only) {
      int ndev = 0;
      if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        fail(TT_ECUDA, "no CUDA device: the engine has no CPU fallback");
      if (cfg->device < 0 || cfg->device >= ndev) fail(TT_EINVAL, "device ordinal out of range");
      t->ex = std::make_unique<Exec>(cfg->device);
      DeviceGuard g(cfg->device);
      t->arena = std::make_unique<Arena>();
      t->tail.ensure(static_cast<size_t>(t->B * t->slice) * sizeof(double));
    }
    *out = t.release();
  });
}

void tt_tree_destroy(tt_tree* tree) {
  if (!tree) return;
  if (tree->ex) {
    DeviceGuard g(tree->ex->device);
    delete tree;
  } else {
    delete tree;
  }
}

tt_status tt_append(tt_tree* t, const double* slices, int64_t n, tt_mem where) {
  return guarded([&] {
    if (!t) fail(TT_EINVAL, "append: null tree");
    if (n < 0) fail(TT_EINVAL, "append: negative slice count");
    if (n == 0) return;
    if (!slices && !t->structure_only) fail(TT_EINVAL, "append: null slices");
    const Index ss = t->slice, B = t->B;
    const Index tail0 = t->timespan - t->leaves * B;
    const Index nblocks = (tail0 + n) / B;
    std::vector<const double*> leaf_x;
    const double* src = slices;  // device view of the new slices
    std::unique_ptr<DeviceGuard> g;
    if (!t->structure_only) {
      g = std::make_unique<DeviceGuard>(t->ex->device);
      if (where == TT_MEM_HOST) {
        t->stage.ensure(static_cast<size_t>(n * ss) * sizeof(double));
        cuda_check(cudaMemcpyAsync(t->stage.p, slices, static_cast<size_t>(n * ss) * sizeof(double),
                                   cudaMemcpyHostToDevice, t->ex->stream),
                   "append upload");
        src = t->stage.as<double>();
      }
      // Block 0 completes the buffered tail; later blocks read straight from src.
      Index consumed = 0;
      for (Index j = 0; j < nblocks; ++j) {
        if (j == 0 && tail0 > 0) {
          const Index need = B - tail0;
          cuda_check(cudaMemcpyAsync(t->tail.as<double>() + tail0 * ss, src, static_cast<size_t>(need * ss) * sizeof(double),
                                     cudaMemcpyDeviceToDevice, t->ex->stream),
                     "tail fill");
          leaf_x.push_back(t->tail.as<double>());
          consumed = need;
        } else {
          leaf_x.push_back(src + consumed * ss);
          consumed += B;
        }
      }
      (void)consumed;
    }
    // Bookkeeping, one slice at a time (reference append semantics). A failed
    // append leaves the tree unchanged (sst.cpp:95-97): the scalars, the node
    // table and the arena are restored from a snapshot if anything below throws.
    struct Snapshot {
      Index nodes, root, timespan, leaves, stitch_count, last_touches;
      std::vector<Index> last_redec;
      Arena::Mark arena;
    };
    const Snapshot snap{static_cast<Index>(t->nodes.size()), t->root, t->timespan, t->leaves, t->stitch_count,
                        t->last_touches, t->last_redec, t->arena ? t->arena->mark() : Arena::Mark{0, nullptr, 0}};
    t->journal.clear();
    t->journal_n0 = snap.nodes;
    PendingWork w;
    std::vector<Index> all_redec;
    try {
      for (Index i = 0; i < n; ++i) {
        ++t->timespan;
        if (t->timespan - t->leaves * B == B) {
          add_leaf(*t, w);
          all_redec.insert(all_redec.end(), t->last_redec.begin(), t->last_redec.end());
        } else {
          t->last_touches = 0;
          t->last_redec.clear();
        }
      }
      execute(*t, w, leaf_x);
    } catch (...) {
      if (!t->structure_only) cudaStreamSynchronize(t->ex->stream);  // no kernel still writes a dropped slot
      t->nodes.resize(static_cast<size_t>(snap.nodes));
      for (const HostNode& v : t->journal) t->node(v.id) = v;
      t->root = snap.root;
      t->timespan = snap.timespan;
      t->leaves = snap.leaves;
      t->stitch_count = snap.stitch_count;
      t->last_touches = snap.last_touches;
      t->last_redec = snap.last_redec;
      if (t->arena) t->arena->release(snap.arena);
      t->journal.clear();
      t->journal_n0 = -1;
      throw;
    }
    t->journal.clear();
    t->journal_n0 = -1;
    if (!t->structure_only) {
      // New tail = slices past the last full block (after the leaf kernels read the old tail).
      const Index tail1 = t->timespan - t->leaves * B;
      if (tail1 > 0) {
        const Index first_new = n - tail1;  // index into the new slices
        if (first_new >= 0) {
          cuda_check(cudaMemcpyAsync(t->tail.p, src + first_new * ss, static_cast<size_t>(tail1 * ss) * sizeof(double),
                                     cudaMemcpyDeviceToDevice, t->ex->stream),
                     "tail store");
        } else {  // no block completed: old tail + all new slices
          cuda_check(cudaMemcpyAsync(t->tail.as<double>() + tail0 * ss, src, static_cast<size_t>(n * ss) * sizeof(double),
                                     cudaMemcpyDeviceToDevice, t->ex->stream),
                     "tail append");
        }
      }
      t->ex->sync();
    }
    t->last_redec = all_redec;
  });
}

tt_status tt_tree_clear(tt_tree* t) {
  return guarded([&] {
    if (!t) fail(TT_EINVAL, "null tree");
    t->nodes.clear();
    t->root = t->timespan = t->leaves = t->stitch_count = t->last_touches = 0;
    t->last_redec.clear();
    if (t->arena) t->arena->reset();
  });
}

int64_t tt_tree_stat(const tt_tree* t, int32_t what) {
  if (!t) return -1;
  switch (what) {
    case TT_STAT_TIMESPAN: return t->timespan;
    case TT_STAT_HEIGHT: return t->height();
    case TT_STAT_STITCH_COUNT: return t->stitch_count;
    case TT_STAT_LAST_TOUCHES: return t->last_touches;
    case TT_STAT_NODE_COUNT: return static_cast<int64_t>(t->nodes.size());
    case TT_STAT_ROOT: return t->root;
    case TT_STAT_LEAVES: return t->leaves;
    default: return -1;
  }
}

tt_status tt_node_info_get(const tt_tree* t, int64_t id, tt_node_info* out) {
  return guarded([&] {
    if (!t || !out) fail(TT_EINVAL, "null argument");
    const HostNode& v = t->node(id);
    std::memset(out, 0, sizeof(*out));
    out->id = v.id;
    out->begin = v.begin;
    out->end = v.end;
    out->kind = v.kind;
    out->has_decomposition = v.has_dec;
    out->left = v.left;
    out->right = v.right;
    for (int m = 0; m < t->p; ++m) out->ranks[m] = v.ranks[m];
  });
}

tt_status tt_node_get(const tt_tree* t, int64_t id, double* core, double* const* factors, tt_mem where) {
  return guarded([&] {
    if (!t) fail(TT_EINVAL, "null tree");
    const HostNode& v = t->node(id);
    if (!v.has_dec || t->structure_only) fail(TT_ELOGIC, "node has no decomposition");
    DeviceGuard g(t->ex->device);
    const cudaMemcpyKind kind = where == TT_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (core)
      cuda_check(cudaMemcpyAsync(core, v.core, static_cast<size_t>(prod_range(v.ranks, 0, t->p)) * sizeof(double), kind,
                                 t->ex->stream),
                 "node core download");
    for (int m = 0; m < t->p; ++m) {
      if (!factors || !factors[m]) continue;
      const Index rows = m == 0 ? v.length() : t->d[m];
      cuda_check(cudaMemcpyAsync(factors[m], v.f[m], static_cast<size_t>(rows * v.ranks[m]) * sizeof(double), kind,
                                 t->ex->stream),
                 "node factor download");
    }
    t->ex->sync();
  });
}

tt_status tt_last_redecomposed(const tt_tree* t, int64_t* ids, int64_t cap, int64_t* n) {
  return guarded([&] {
    if (!t || !n) fail(TT_EINVAL, "null argument");
    *n = static_cast<int64_t>(t->last_redec.size());
    for (size_t i = 0; i < t->last_redec.size() && static_cast<int64_t>(i) < cap; ++i) ids[i] = t->last_redec[i];
  });
}

tt_status tt_last_timing(const tt_tree* t, double* ms3) {
  return guarded([&] {
    if (!t || !ms3) fail(TT_EINVAL, "null argument");
    // the calling thread's last query if it is newer than the last append
    const tt_tree::Reader* rd = const_cast<tt_tree*>(t)->reader_if_any();
    const double* src = (rd && rd->stamp > t->timing_stamp) ? rd->timing : t->timing;
    for (int i = 0; i < 3; ++i) ms3[i] = src[i];
  });
}

// sst.cpp:159-295 (structural invariants), in units of the leaf block B
// (B = 1: the reference's checks and messages verbatim).
int32_t tt_validate(const tt_tree* t, char* buf, int64_t cap) {
  if (!t) return -1;
  std::vector<std::string> out;
  auto flag = [&out](std::string s) { out.push_back(std::move(s)); };
  auto label = [](const HostNode& n) {
    return "node " + std::to_string(n.id) + " [" + std::to_string(n.begin) + "," + std::to_string(n.end) + ")";
  };
  const Index B = t->B, T = t->leaves * B;  // the tree covers whole blocks; a raw tail is not in the tree
  auto ceil_log2 = [](Index n) {
    Index l = 0, q = 1;
    while (q < n) {
      q *= 2;
      ++l;
    }
    return l;
  };
  auto finish = [&]() {
    std::string all;
    for (auto& s : out) all += s + "\n";
    if (buf && cap > 0) {
      std::strncpy(buf, all.c_str(), static_cast<size_t>(cap - 1));
      buf[cap - 1] = '\0';
    }
    return static_cast<int32_t>(out.size());
  };
  if (T == 0) {
    if (t->root) flag("empty tree has a root");
    return finish();
  }
  if (!t->root) {
    flag("non-empty tree has no root");
    return finish();
  }
  const Index N = static_cast<Index>(t->nodes.size());
  auto valid = [N](Index id) { return id >= 1 && id <= N; };
  const std::string leaf_len = B == 1 ? "1" : std::to_string(B);
  for (const HostNode& v : t->nodes) {
    if (v.begin < 0 || v.begin >= v.end) flag(label(v) + ": malformed range");
    if ((v.left && !valid(v.left)) || (v.right && !valid(v.right))) {
      flag(label(v) + ": child id unknown");
      continue;
    }
    if (v.kind == TT_LEAF) {
      if (v.length() != B) flag(label(v) + ": leaf range must have length " + leaf_len);
      if (v.left || v.right) flag(label(v) + ": leaf must not have children");
      if (!v.has_dec) flag(label(v) + ": leaf is missing its decomposition");
    } else if (v.kind == TT_INTERMEDIATE) {
      if (!v.left || !v.right) {
        flag(label(v) + ": intermediate must have two children");
      } else {
        const HostNode& l = t->node(v.left);
        const HostNode& r = t->node(v.right);
        if (l.begin != v.begin || l.end != r.begin || r.end != v.end) flag(label(v) + ": children ranges are not adjoint");
        if (l.kind == TT_PLACEHOLDER || r.kind == TT_PLACEHOLDER) flag(label(v) + ": intermediate has a placeholder child");
        if (!v.has_dec) flag(label(v) + ": intermediate is missing its decomposition");
      }
    } else if (v.kind == TT_PLACEHOLDER) {
      if (v.has_dec) flag(label(v) + ": placeholder carries a decomposition");
      if (!(v.begin < T && T <= v.end)) flag(label(v) + ": placeholder does not straddle the write frontier");
      if (!v.left && v.right) flag(label(v) + ": placeholder has a right child without a left child");
      if (!v.left && !v.right) flag(label(v) + ": placeholder has no children");
      if (v.left && v.right) {
        const HostNode& l = t->node(v.left);
        const HostNode& r = t->node(v.right);
        if (l.begin != v.begin || l.end != r.begin || r.end != v.end) flag(label(v) + ": children ranges are not adjoint");
      } else if (v.left) {
        const HostNode& l = t->node(v.left);
        // midpoint split in leaf units (sst.cpp:119: mid = (b + e) / 2)
        const Index mid = ((v.begin / B + v.end / B) / 2) * B;
        if (l.begin != v.begin || l.end != mid) flag(label(v) + ": left child range does not match the midpoint split");
      }
    } else {
      flag(label(v) + ": unknown node kind");
    }
    if (v.kind != TT_PLACEHOLDER && v.end > T) flag(label(v) + ": materialized node extends past the timespan");
    if (v.has_dec && !t->structure_only) {
      // the device slots hold factor 0 with the node's length rows and factor m
      // with D_m rows; the core extents are the factor column counts
      for (int m = 0; m < t->p; ++m)
        if (v.ranks[m] < 1 || v.ranks[m] > t->clamped(m, v.length())) {
          flag(label(v) + ": core extent does not match factor columns");
          break;
        }
    }
  }
  std::vector<const HostNode*> lv;
  for (const HostNode& v : t->nodes)
    if (v.kind == TT_LEAF) lv.push_back(&v);
  std::sort(lv.begin(), lv.end(), [](const HostNode* a, const HostNode* b) { return a->begin < b->begin; });
  Index expected = 0;
  for (const HostNode* l : lv) {
    if (l->begin != expected) {
      flag(label(*l) + ": leaf tiling gap or overlap at " + std::to_string(expected));
      break;
    }
    expected = l->end;
  }
  if (expected != T && out.empty())
    flag("leaves cover [0," + std::to_string(expected) + ") but timespan is " + std::to_string(T));
  if (!valid(t->root)) {
    flag("root id unknown");
    return finish();
  }
  const HostNode& r = t->node(t->root);
  const Index nl = T / B;
  const Index span = (nl == 1 ? 1 : (Index(1) << ceil_log2(nl))) * B;
  if (r.begin != 0 || r.end != span) flag(label(r) + ": root range should be [0," + std::to_string(span) + ")");
  const Index eh = ceil_log2(nl) + 1;
  if (t->height() != eh)
    flag("height " + std::to_string(t->height()) + " violates the height law " + std::to_string(eh));
  return finish();
}

tt_status tt_recall(const tt_tree* t, int64_t ts, int64_t te, double theta, tt_hit* out, int64_t cap, int64_t* n) {
  return guarded([&] {
    if (!t || !n) fail(TT_EINVAL, "null argument");
    const auto hits = recall(*t, ts, te, theta);
    *n = static_cast<int64_t>(hits.size());
    for (size_t i = 0; i < hits.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = hits[i];
  });
}

tt_status tt_query_batch(const tt_tree* tc, const tt_range* ranges, int64_t n, double theta, tt_query_out* outs,
                         tt_mem where) {
  return guarded([&] {
    if (!tc) fail(TT_EINVAL, "null tree");
    tt_tree* t = const_cast<tt_tree*>(tc);
    if (n <= 0) return;
    if (!ranges || !outs) fail(TT_EINVAL, "null ranges/outs");
    if (t->structure_only) fail(TT_ELOGIC, "range_query on a structure-only tree");
    const int p = t->p;
    // recall for every query first: an invalid range fails the batch before any device work
    std::vector<std::vector<tt_hit>> hits(static_cast<size_t>(n));
    for (int64_t q = 0; q < n; ++q) hits[q] = recall(*t, ranges[q].ts, ranges[q].te, theta);
    tt_tree::Reader& rd = t->reader();
    Exec& ex = *rd.ex;
    DeviceGuard g(ex.device);
    Params prm = tree_params(*t);
    t->init.stitch_init(prm, ex.stream);
    cuda_check(cudaEventRecord(ex.ev[0], ex.stream), "event");
    // ---- tail parts: tucker_als of the raw tail sub-range
    struct TailSlot {
      double* f[kMaxP];
      double* core;
      Index len;
      Index ranks[kMaxP];
    };
    std::vector<TailSlot> tails(static_cast<size_t>(n));
    {
      std::vector<LeafDesc> descs;
      std::vector<Index> ws, which;
      size_t need = 0;
      const Index tb = t->leaves * t->B;
      std::vector<std::pair<int64_t, Index>> tl;  // (query, len)
      for (int64_t q = 0; q < n; ++q)
        for (const tt_hit& h : hits[q])
          if (h.flag == TT_HIT_TAIL) tl.emplace_back(q, h.end - h.begin);
      for (auto& [q, len] : tl) {
        Index rc[kMaxP];
        for (int m = 0; m < p; ++m) rc[m] = t->clamped(m, len);
        need += static_cast<size_t>(len * rc[0] + prod_range(rc, 0, p));
        for (int m = 1; m < p; ++m) need += static_cast<size_t>(t->d[m] * rc[m]);
        need += 64 * static_cast<size_t>(p);
      }
      if (!tl.empty()) {
        rd.tailq.ensure(need * sizeof(double));
        double* cur = rd.tailq.as<double>();
        auto take = [&cur](Index nd) {
          double* r = cur;
          cur += (nd + 31) & ~Index(31);
          return r;
        };
        for (auto& [q, len] : tl) {
          TailSlot& s = tails[q];
          s.len = len;
          Index rc[kMaxP];
          for (int m = 0; m < p; ++m) rc[m] = t->clamped(m, len);
          s.f[0] = take(len * rc[0]);
          for (int m = 1; m < p; ++m) s.f[m] = take(t->d[m] * rc[m]);
          s.core = take(prod_range(rc, 0, p));
          const tt_hit& h = hits[q].back();
          const auto& init = t->init.leaf_init(len, ex.stream);
          LeafDesc dsc{};
          dsc.x = t->tail.as<double>() + (h.begin - tb) * t->slice;
          dsc.len = len;
          for (int m = 0; m < p; ++m) {
            dsc.init[m] = init[m]->as<double>();
            dsc.out_f[m] = s.f[m];
          }
          dsc.out_core = s.core;
          descs.push_back(dsc);
          ws.push_back(leaf_ws_layout(p, len, t->d, t->cfg.ranks).total);
          which.push_back(q);
        }
        const auto st = run_leaf_batch(ex, prm, descs, ws);
        for (size_t i = 0; i < which.size(); ++i)
          for (int m = 0; m < p; ++m) tails[which[i]].ranks[m] = st[i].k[m];
      }
    }
    cuda_check(cudaEventRecord(ex.ev[1], ex.stream), "event");
    // ---- stitches, chunked by workspace budget
    const size_t kBudget = size_t(3) << 30;  // bytes of workspace + staging per chunk
    int64_t q0 = 0;
    while (q0 < n) {
      std::vector<StitchDesc> descs;
      std::vector<StitchPart> parts;
      std::vector<Index> ws;
      std::vector<size_t> out_off;
      size_t used = 0, out_need = 0;
      int64_t q1 = q0;
      for (; q1 < n; ++q1) {
        const Index L = ranges[q1].te - ranges[q1].ts;
        Index rho_max[kMaxP] = {};
        std::vector<StitchPart> qp;
        for (const tt_hit& h : hits[q1]) {
          StitchPart sp{};
          if (h.flag == TT_HIT_TAIL) {
            const TailSlot& s = tails[q1];
            sp.core = s.core;
            for (int m = 0; m < p; ++m) {
              sp.rho[m] = s.ranks[m];
              sp.v[m] = s.f[m];
            }
            sp.v0 = s.f[0];
            sp.ld0 = s.len;
            sp.row0 = 0;
            sp.len = s.len;
            sp.partial = 0;
          } else {
            const HostNode& v = t->node(h.node);
            if (!v.has_dec) fail(TT_ELOGIC, "range_query: hit node has no decomposition");
            sp.core = v.core;
            for (int m = 0; m < p; ++m) {
              sp.rho[m] = v.ranks[m];
              sp.v[m] = v.f[m];
            }
            sp.v0 = v.f[0];
            sp.ld0 = v.length();
            sp.row0 = h.begin - v.begin;
            sp.len = h.end - h.begin;
            sp.partial = h.flag == TT_HIT_PARTIAL ? 1 : 0;
          }
          for (int m = 0; m < p; ++m) rho_max[m] = std::max(rho_max[m], sp.rho[m]);
          qp.push_back(sp);
        }
        const Index wsz = stitch_ws_layout(p, L, t->d, t->cfg.ranks, rho_max, static_cast<int>(qp.size())).total;
        Index rc[kMaxP];
        for (int m = 0; m < p; ++m) rc[m] = t->clamped(m, L);
        size_t onum = 0;
        if (where == TT_MEM_HOST) {
          onum = static_cast<size_t>(L * rc[0] + prod_range(rc, 0, p));
          for (int m = 1; m < p; ++m) onum += static_cast<size_t>(t->d[m] * rc[m]);
          onum += 32 * static_cast<size_t>(p + 1);
        }
        const size_t add = (static_cast<size_t>(wsz) + onum) * sizeof(double);
        if (q1 > q0 && used + add > kBudget) break;
        used += add;
        StitchDesc dsc{};
        dsc.part0 = static_cast<int32_t>(parts.size());
        dsc.nparts = static_cast<int32_t>(qp.size());
        dsc.L = L;
        parts.insert(parts.end(), qp.begin(), qp.end());
        descs.push_back(dsc);
        ws.push_back(wsz);
        out_off.push_back(out_need);
        out_need += onum;
      }
      // output buffers
      const int64_t nc = q1 - q0;
      // Pinned host outputs (the serving case) are DMA'd on the copy stream.
      // Staging mirrors the caller's layout: outputs that are adjacent in host
      // memory are adjacent in staging, so a wave's download is a few large
      // copies. Every output is sized for the clamped requested ranks (the
      // tt_query_out contract) and copied at that size.
      struct OutRef {
        char* host;
        size_t bytes;
        int64_t q;  // chunk-relative query
        int m;      // -1 core, else factor mode
      };
      std::vector<OutRef> orefs;
      bool dma = where == TT_MEM_HOST;
      if (dma) {
        for (int64_t q = q0; q < q1 && dma; ++q) {
          const Index L = descs[q - q0].L;
          Index rc[kMaxP];
          for (int m = 0; m < p; ++m) rc[m] = t->clamped(m, L);
          auto addr = [&](double* h, Index nd, int m) {
            if (!h) return;
            if (!mapped_device_ptr(h)) dma = false;
            orefs.push_back(OutRef{reinterpret_cast<char*>(h), static_cast<size_t>(nd) * sizeof(double), q - q0, m});
          };
          addr(outs[q].core, prod_range(rc, 0, p), -1);
          addr(outs[q].factors[0], L * rc[0], 0);
          for (int m = 1; m < p; ++m) addr(outs[q].factors[m], t->d[m] * rc[m], m);
        }
      }
      std::vector<size_t> stage_off;  // per oref
      if (dma) {
        std::vector<size_t> idx(orefs.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
        std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return orefs[x].host < orefs[y].host; });
        for (size_t i = 1; i < idx.size(); ++i)
          if (orefs[idx[i - 1]].host + orefs[idx[i - 1]].bytes > orefs[idx[i]].host)
            fail(TT_EINVAL, "range_query: output buffers overlap");
        stage_off.assign(orefs.size(), 0);
        size_t off = 0;
        for (size_t i = 0; i < idx.size(); ++i) {
          // clusters of host-adjacent outputs are packed back to back
          stage_off[idx[i]] = off;
          off += (orefs[idx[i]].bytes + 7) & ~size_t(7);
        }
        rd.qout.ensure(std::max<size_t>(off, 8));
        for (size_t i = 0; i < orefs.size(); ++i) {
          double* dptr = reinterpret_cast<double*>(rd.qout.as<char>() + stage_off[i]);
          StitchDesc& dsc = descs[orefs[i].q];
          if (orefs[i].m < 0)
            dsc.out_core = dptr;
          else
            dsc.out_f[orefs[i].m] = dptr;
        }
        // outputs the caller did not request still need device scratch
        size_t extra = 0;
        for (int64_t q = q0; q < q1; ++q) {
          const Index L = descs[q - q0].L;
          Index rc[kMaxP];
          for (int m = 0; m < p; ++m) rc[m] = t->clamped(m, L);
          if (!outs[q].core) extra += static_cast<size_t>(prod_range(rc, 0, p));
          for (int m = 0; m < p; ++m)
            if (!outs[q].factors[m]) extra += static_cast<size_t>((m == 0 ? L : t->d[m]) * rc[m]);
        }
        if (extra) {
          rd.qscratch.ensure(extra * sizeof(double));
          double* cur = rd.qscratch.as<double>();
          for (int64_t q = q0; q < q1; ++q) {
            const Index L = descs[q - q0].L;
            Index rc[kMaxP];
            for (int m = 0; m < p; ++m) rc[m] = t->clamped(m, L);
            StitchDesc& dsc = descs[q - q0];
            if (!outs[q].core) {
              dsc.out_core = cur;
              cur += prod_range(rc, 0, p);
            }
            for (int m = 0; m < p; ++m)
              if (!outs[q].factors[m]) {
                dsc.out_f[m] = cur;
                cur += (m == 0 ? L : t->d[m]) * rc[m];
              }
          }
        }
      } else {
        if (where == TT_MEM_HOST) rd.qout.ensure(out_need * sizeof(double));
        double* dscr = nullptr;  // device scratch for outputs the caller did not request (null pointers)
        if (where == TT_MEM_DEVICE) {
          size_t extra = 0;
          for (int64_t q = q0; q < q1; ++q) {
            const Index L = descs[q - q0].L;
            if (!outs[q].core) extra += static_cast<size_t>(prod_range(t->cfg.ranks, 0, p)) + 32;
            for (int m = 0; m < p; ++m)
              if (!outs[q].factors[m]) extra += static_cast<size_t>((m == 0 ? L : t->d[m]) * t->clamped(m, L)) + 32;
          }
          if (extra) {
            rd.qscratch.ensure(extra * sizeof(double));
            dscr = rd.qscratch.as<double>();
          }
        }
        for (int64_t q = q0; q < q1; ++q) {
          StitchDesc& dsc = descs[q - q0];
          const Index L = dsc.L;
          Index rc[kMaxP];
          for (int m = 0; m < p; ++m) rc[m] = t->clamped(m, L);
          if (where == TT_MEM_DEVICE) {
            auto scratch = [&dscr](Index nd) {
              double* r = dscr;
              dscr += nd + 32;
              return r;
            };
            for (int m = 0; m < p; ++m)
              dsc.out_f[m] = outs[q].factors[m] ? outs[q].factors[m] : scratch((m == 0 ? L : t->d[m]) * rc[m]);
            dsc.out_core = outs[q].core ? outs[q].core : scratch(prod_range(t->cfg.ranks, 0, p));
          } else {
            double* cur = rd.qout.as<double>() + out_off[q - q0];
            auto take = [&cur](Index nd) {
              double* r = cur;
              cur += (nd + 31) & ~Index(31);
              return r;
            };
            dsc.out_f[0] = take(L * rc[0]);
            for (int m = 1; m < p; ++m) dsc.out_f[m] = take(t->d[m] * rc[m]);
            dsc.out_core = take(prod_range(rc, 0, p));
          }
        }
      }
      // Waves: with DMA'd outputs the chunk runs as a few launches of growing
      // size so the PCIe download (the end-to-end bound) starts after a short
      // first wave and overlaps the rest. Wave 0 holds the cheapest queries
      // (it finishes fastest); later waves are runs in query order, which keeps
      // their outputs host-contiguous for large copies.
      std::vector<int64_t> order(static_cast<size_t>(nc));
      for (int64_t i = 0; i < nc; ++i) order[i] = i;
      std::vector<int64_t> wave_end;
      if (dma && nc >= 64) {
        auto qcost = [&](int64_t i) { return double(descs[i].L) + kWavePartCost * descs[i].nparts; };
        std::vector<int64_t> by_cost(order);
        std::stable_sort(by_cost.begin(), by_cost.end(), [&](int64_t x, int64_t y) { return qcost(x) < qcost(y); });
        const int64_t w0 = (nc + 31) / 32;
        std::vector<char> first(static_cast<size_t>(nc), 0);
        for (int64_t j = 0; j < w0; ++j) first[by_cost[j]] = 1;
        int64_t j = 0;
        for (int64_t i = 0; i < nc; ++i)
          if (first[i]) order[j++] = i;
        for (int64_t i = 0; i < nc; ++i)
          if (!first[i]) order[j++] = i;
        int64_t w = w0, e = 0;
        while (e < nc) {
          e = std::min(nc, e + w);
          if (nc - e < w || static_cast<int>(wave_end.size()) == Exec::kWaveEvents - 1) e = nc;
          wave_end.push_back(e);
          w *= 2;
        }
      } else {
        wave_end.push_back(nc);
      }
      // per chunk-relative query: its output refs (for the wave downloads)
      std::vector<std::vector<size_t>> q_refs(static_cast<size_t>(nc));
      for (size_t i = 0; i < orefs.size(); ++i) q_refs[orefs[i].q].push_back(i);
      std::vector<ProblemStatus> st(static_cast<size_t>(nc));
      int64_t wb = 0;
      for (size_t wi = 0; wi < wave_end.size(); ++wi) {
        const int64_t we = wave_end[wi];
        if (wave_end.size() == 1) {  // one launch over the whole chunk, no reordering
          st = run_stitch_batch(ex, prm, descs, parts, ws);
          if (dma) {
            cuda_check(cudaEventRecord(ex.wave_ev[0], ex.stream), "event");
            cuda_check(cudaStreamWaitEvent(ex.copy, ex.wave_ev[0], 0), "cudaStreamWaitEvent");
          }
        }
        std::vector<StitchDesc> wd;
        std::vector<StitchPart> wp;
        std::vector<Index> wws;
        for (int64_t j = wb; j < we && wave_end.size() > 1; ++j) {
          StitchDesc d = descs[order[j]];
          const int32_t p0 = d.part0;
          d.part0 = static_cast<int32_t>(wp.size());
          wp.insert(wp.end(), parts.begin() + p0, parts.begin() + p0 + d.nparts);
          wd.push_back(d);
          wws.push_back(ws[order[j]]);
        }
        if (wave_end.size() > 1) {
          auto wst = run_stitch_batch(ex, prm, wd, wp, wws);
          for (int64_t j = wb; j < we; ++j) st[order[j]] = std::move(wst[j - wb]);
        }
        if (dma && wave_end.size() > 1) {
          cuda_check(cudaEventRecord(ex.wave_ev[wi], ex.stream), "event");
          cuda_check(cudaStreamWaitEvent(ex.copy, ex.wave_ev[wi], 0), "cudaStreamWaitEvent");
        }
        if (dma) {
          std::vector<size_t> wr;
          for (int64_t j = wb; j < we; ++j) wr.insert(wr.end(), q_refs[order[j]].begin(), q_refs[order[j]].end());
          std::sort(wr.begin(), wr.end(), [&](size_t x, size_t y) { return orefs[x].host < orefs[y].host; });
          size_t r = 0;
          while (r < wr.size()) {  // merge runs adjacent in host memory and in staging
            char* h0 = orefs[wr[r]].host;
            const size_t s0 = stage_off[wr[r]];
            size_t len = orefs[wr[r]].bytes;
            size_t r2 = r + 1;
            while (r2 < wr.size() && orefs[wr[r2]].host == h0 + len && stage_off[wr[r2]] == s0 + len &&
                   (len & 7) == 0) {
              len += orefs[wr[r2]].bytes;
              ++r2;
            }
            cuda_check(cudaMemcpyAsync(h0, rd.qout.as<char>() + s0, len, cudaMemcpyDeviceToHost, ex.copy),
                       "query output download");
            r = r2;
          }
        }
        wb = we;
      }
      std::vector<CopySeg> segs;
      bool all_mapped = where == TT_MEM_HOST;
      for (int64_t q = q0; q < q1; ++q) {
        const ProblemStatus& s = st[q - q0];
        tt_query_out& o = outs[q];
        const Index L = descs[q - q0].L;
        Index k[kMaxP];
        for (int m = 0; m < p; ++m) k[m] = s.k[m];
        if (s.zero) {
          for (int m = 0; m < p; ++m) k[m] = t->clamped(m, L);
          const auto u0 = t->init.stitch_zero_u0(L, k[0]);
          if (dma) {
            ex.sync_copy();  // the wave's download of the staging rows must land first
            if (o.factors[0]) std::memcpy(o.factors[0], u0.data(), u0.size() * sizeof(double));
          } else {
            cuda_check(cudaMemcpyAsync(descs[q - q0].out_f[0], u0.data(), u0.size() * sizeof(double),
                                       cudaMemcpyHostToDevice, ex.stream),
                       "zero-path upload");
            ex.sync();
          }
        }
        for (int m = 0; m < TT_MAX_ORDER; ++m) o.ranks[m] = m < p ? k[m] : 0;
        o.sweeps = s.sweeps;
        o.converged = s.converged;
        o.objective = s.objective.empty() ? 0.0 : s.objective.back();
        o.nhits = static_cast<int32_t>(hits[q].size());
        if (o.trace && o.trace_cap > 0)  // AlsTrace::objective (range_query_detailed, query.hpp:48-50)
          for (size_t i = 0; i < s.objective.size() && static_cast<int32_t>(i) < o.trace_cap; ++i)
            o.trace[i] = s.objective[i];
        if (o.hits && o.hits_cap > 0)  // QueryResult::hits
          for (size_t i = 0; i < hits[q].size() && static_cast<int32_t>(i) < o.hits_cap; ++i) o.hits[i] = hits[q][i];
        if (where == TT_MEM_HOST && !dma) {
          const StitchDesc& dsc = descs[q - q0];
          // small outputs: one gather kernel into mapped host memory when every
          // destination is pinned, else individual copies
          auto add = [&](void* host, const double* src, Index n) {
            if (!host) return;
            double* mp = mapped_device_ptr(host);
            if (mp) {
              segs.push_back(CopySeg{src, mp, n});
            } else {
              all_mapped = false;
              cuda_check(cudaMemcpyAsync(host, src, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost,
                                         ex.stream),
                         "query output download");
            }
          };
          add(o.core, dsc.out_core, prod_range(k, 0, p));
          for (int m = 1; m < p; ++m) add(o.factors[m], dsc.out_f[m], t->d[m] * k[m]);
          add(o.factors[0], dsc.out_f[0], L * k[0]);
        }
      }
      if (!segs.empty()) {
        ex.d_segs.ensure(segs.size() * sizeof(CopySeg));
        cuda_check(cudaMemcpyAsync(ex.d_segs.p, segs.data(), segs.size() * sizeof(CopySeg), cudaMemcpyHostToDevice,
                                   ex.stream),
                   "upload copy segments");
        cuda_check(launch_copy_segments(ex.d_segs.as<CopySeg>(), static_cast<int>(segs.size()), ex.stream),
                   "copy_segments_kernel launch");
      }
      (void)all_mapped;
      ex.sync();
      ex.sync_copy();  // qout is reused by the next chunk
      q0 = q1;
    }
    cuda_check(cudaEventRecord(ex.ev[2], ex.stream), "event");
    ex.sync();
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ex.ev[0], ex.ev[1]);
    cudaEventElapsedTime(&b, ex.ev[1], ex.ev[2]);
    rd.timing[0] = a;
    rd.timing[1] = b;
    rd.timing[2] = a + b;
    rd.stamp = next_stamp();
  });
}

// ---------------------------------------------------------------------------
// Standalone operations.
namespace {
struct StandaloneCtx {
  std::unique_ptr<Exec> ex;
  int device = -1;
  std::mutex op;  // one standalone operation at a time per device context (shared Exec buffers and stream)
};
StandaloneCtx& standalone(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<StandaloneCtx>> ctx;
  std::lock_guard<std::mutex> lk(mu);
  auto& c = ctx[device];
  if (!c) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      fail(TT_ECUDA, "no CUDA device: the engine has no CPU fallback");
    if (device < 0 || device >= ndev) fail(TT_EINVAL, "device ordinal out of range");
    c = std::make_unique<StandaloneCtx>();
    c->ex = std::make_unique<Exec>(device);
    c->device = device;
  }
  return *c;
}

std::vector<double> download(const double* d, size_t n, cudaStream_t st) {
  std::vector<double> h(n);
  if (n) cuda_check(cudaMemcpyAsync(h.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, st), "download");
  return h;
}
double* upload(DevBuf& b, const double* h, size_t n, cudaStream_t st) {
  b.ensure(std::max<size_t>(n, 1) * sizeof(double));
  if (n) cuda_check(cudaMemcpyAsync(b.p, h, n * sizeof(double), cudaMemcpyHostToDevice, st), "upload");
  return b.as<double>();
}
}  // namespace

tt_status tt_tucker_als(const double* x, int32_t p, const int64_t* dims, const int64_t* ranks, int32_t max_iters,
                        double tol, uint64_t seed, int32_t device, tt_factors** out) {
  return guarded([&] {
    if (!x || !dims || !ranks || !out) fail(TT_EINVAL, "null argument");
    *out = nullptr;
    if (p < 2 || p > TT_MAX_ORDER) fail(TT_EINVAL, "tucker_als: order must be in [2, 8]");
    if (max_iters < 1) fail(TT_EINVAL, "tucker_als: max_iters must be >= 1");
    if (tol <= 0.0) fail(TT_EINVAL, "tucker_als: tol must be > 0");
    for (int m = 0; m < p; ++m) {
      if (dims[m] < 1) fail(TT_EINVAL, "Shape: all dims must be >= 1");
      if (ranks[m] < 1) fail(TT_EINVAL, "clamp_ranks: ranks must be >= 1");
      if (ranks[m] > 32) fail(TT_EINVAL, "tucker_als: ranks above 32 are not supported by this build");
    }
    StandaloneCtx& c = standalone(device);
    std::lock_guard<std::mutex> op_lock(c.op);
    Exec& ex = *c.ex;
    DeviceGuard g(device);
    Index d[kMaxP], rq[kMaxP], rc[kMaxP];
    for (int m = 0; m < kMaxP; ++m) {
      d[m] = m < p ? dims[m] : 1;
      rq[m] = m < p ? ranks[m] : 1;
    }
    clamp_ranks(p, d, rq, rc);
    InitCache init;
    init.p = p;
    for (int m = 0; m < p; ++m) {
      init.d[m] = d[m];
      init.req[m] = rq[m];
    }
    init.seed = seed;
    const auto& iv = init.leaf_init(d[0], ex.stream);
    DevBuf bx, bout;
    const size_t nx = static_cast<size_t>(prod_range(d, 0, p));
    const double* dx = upload(bx, x, nx, ex.stream);
    size_t need = static_cast<size_t>(prod_range(rc, 0, p));
    for (int m = 0; m < p; ++m) need += static_cast<size_t>(d[m] * rc[m]) + 32;
    bout.ensure(need * sizeof(double));
    LeafDesc dsc{};
    dsc.x = dx;
    dsc.len = d[0];
    double* cur = bout.as<double>();
    for (int m = 0; m < p; ++m) {
      dsc.init[m] = iv[m]->as<double>();
      dsc.out_f[m] = cur;
      cur += d[m] * rc[m] + 16;
    }
    dsc.out_core = cur;
    Params prm = make_params(p, d, rq, max_iters, tol);
    std::vector<LeafDesc> descs{dsc};
    const auto st = run_leaf_batch(ex, prm, descs, {leaf_ws_layout(p, d[0], d, rq).total});
    auto f = std::make_unique<tt_factors>();
    f->p = p;
    for (int m = 0; m < p; ++m) {
      f->dims[m] = d[m];
      f->ranks[m] = st[0].k[m];
    }
    f->core = download(dsc.out_core, static_cast<size_t>(prod_range(f->ranks, 0, p)), ex.stream);
    for (int m = 0; m < p; ++m) f->f.push_back(download(dsc.out_f[m], static_cast<size_t>(d[m] * f->ranks[m]), ex.stream));
    ex.sync();
    f->objective = st[0].objective;
    f->sweeps = st[0].sweeps;
    f->converged = st[0].converged;
    *out = f.release();
  });
}

tt_status tt_brute_force_batch(const double* series, tt_mem where, int32_t p, const int64_t* dims,
                               const int64_t* ranks, const tt_range* ranges, int64_t n, int32_t max_iters, double tol,
                               uint64_t seed, int32_t device, tt_factors** outs) {
  return guarded([&] {  // brute_force_range (baseline.cpp:67-75), batched: one leaf-kernel CTA per range
    if (!series || !dims || !ranks || (n > 0 && (!ranges || !outs))) fail(TT_EINVAL, "null argument");
    if (n < 0) fail(TT_EINVAL, "brute_force: negative range count");
    if (p < 2 || p > TT_MAX_ORDER) fail(TT_EINVAL, "brute_force: order must be in [2, 8]");
    if (max_iters < 1) fail(TT_EINVAL, "tucker_als: max_iters must be >= 1");
    if (tol <= 0.0) fail(TT_EINVAL, "tucker_als: tol must be > 0");
    for (int m = 0; m < p; ++m) {
      if (dims[m] < 1) fail(TT_EINVAL, "Shape: all dims must be >= 1");
      if (ranks[m] < 1) fail(TT_EINVAL, "clamp_ranks: ranks must be >= 1");
      if (ranks[m] > 32) fail(TT_EINVAL, "tucker_als: ranks above 32 are not supported by this build");
    }
    for (int64_t i = 0; i < n; ++i) {
      outs[i] = nullptr;
      if (ranges[i].ts < 0 || ranges[i].ts >= ranges[i].te || ranges[i].te > dims[0])
        fail(TT_EINVAL, "brute_force_range: invalid range");  // baseline.cpp:69-71
    }
    if (n == 0) return;
    StandaloneCtx& c = standalone(device);
    std::lock_guard<std::mutex> op_lock(c.op);
    Exec& ex = *c.ex;
    DeviceGuard g(device);
    Index d[kMaxP], rq[kMaxP];
    for (int m = 0; m < kMaxP; ++m) {
      d[m] = m < p ? dims[m] : 1;
      rq[m] = m < p ? ranks[m] : 1;
    }
    const Index ss = prod_range(d, 1, p);
    DevBuf bx;
    const double* dx = series;
    if (where == TT_MEM_HOST) dx = upload(bx, series, static_cast<size_t>(d[0] * ss), ex.stream);
    InitCache init;  // tucker_als draws its init factors per range length (tucker.cpp:26-37)
    init.p = p;
    for (int m = 0; m < p; ++m) {
      init.d[m] = d[m];
      init.req[m] = rq[m];
    }
    init.seed = seed;
    std::vector<LeafDesc> descs(static_cast<size_t>(n));
    std::vector<Index> ws(static_cast<size_t>(n));
    std::vector<Index> lens(static_cast<size_t>(n));
    size_t need = 0;
    for (int64_t i = 0; i < n; ++i) {
      Index dl[kMaxP], rc[kMaxP];
      std::copy(d, d + kMaxP, dl);
      dl[0] = lens[i] = ranges[i].te - ranges[i].ts;
      clamp_ranks(p, dl, rq, rc);
      need += static_cast<size_t>(prod_range(rc, 0, p)) + 32;
      for (int m = 0; m < p; ++m) need += static_cast<size_t>(dl[m] * rc[m]) + 16;
      ws[i] = leaf_ws_layout(p, dl[0], d, rq).total;
    }
    DevBuf bout;
    bout.ensure(need * sizeof(double));
    double* cur = bout.as<double>();
    for (int64_t i = 0; i < n; ++i) {
      LeafDesc& dsc = descs[i];
      Index dl[kMaxP], rc[kMaxP];
      std::copy(d, d + kMaxP, dl);
      dl[0] = lens[i];
      clamp_ranks(p, dl, rq, rc);
      const auto& iv = init.leaf_init(lens[i], ex.stream);
      dsc.x = dx + ranges[i].ts * ss;
      dsc.len = lens[i];
      for (int m = 0; m < p; ++m) {
        dsc.init[m] = iv[m]->as<double>();
        dsc.out_f[m] = cur;
        cur += dl[m] * rc[m] + 16;
      }
      dsc.out_core = cur;
      cur += prod_range(rc, 0, p) + 32;
    }
    Params prm = make_params(p, d, rq, max_iters, tol);
    const auto st = run_leaf_batch(ex, prm, descs, ws);
    for (int64_t i = 0; i < n; ++i) {
      auto f = std::make_unique<tt_factors>();
      f->p = p;
      for (int m = 0; m < p; ++m) {
        f->dims[m] = m == 0 ? lens[i] : d[m];
        f->ranks[m] = st[i].k[m];
      }
      f->core = download(descs[i].out_core, static_cast<size_t>(prod_range(f->ranks, 0, p)), ex.stream);
      for (int m = 0; m < p; ++m)
        f->f.push_back(download(descs[i].out_f[m], static_cast<size_t>(f->dims[m] * f->ranks[m]), ex.stream));
      f->objective = st[i].objective;
      f->sweeps = st[i].sweeps;
      f->converged = st[i].converged;
      outs[i] = f.release();
    }
    ex.sync();
  });
}

tt_status tt_stitch(int32_t nparts, int32_t p, const int64_t* part_dims, const int64_t* part_ranks,
                    const double* const* cores, const double* const* factors, const int64_t* ranks, int32_t max_iters,
                    double tol, uint64_t seed, int32_t device, tt_factors** out) {
  return guarded([&] {
    if (!out) fail(TT_EINVAL, "null argument");
    *out = nullptr;
    if (nparts < 1) fail(TT_EINVAL, "stitch: at least one part required");
    if (p < 2 || p > TT_MAX_ORDER) fail(TT_EINVAL, "stitch: parts must have order >= 2");
    if (!part_dims || !part_ranks || !cores || !factors || !ranks) fail(TT_EINVAL, "null argument");
    if (max_iters < 1) fail(TT_EINVAL, "stitch: max_iters must be >= 1");
    if (tol <= 0.0) fail(TT_EINVAL, "stitch: tol must be > 0");
    for (int i = 1; i < nparts; ++i)
      for (int m = 1; m < p; ++m)
        if (part_dims[i * p + m] != part_dims[m]) fail(TT_EINVAL, "stitch: non-temporal shape mismatch across parts");
    for (int m = 0; m < p; ++m) {
      if (ranks[m] < 1) fail(TT_EINVAL, "clamp_ranks: ranks must be >= 1");
      if (ranks[m] > 32) fail(TT_EINVAL, "stitch: ranks above 32 are not supported by this build");
    }
    for (int i = 0; i < nparts * p; ++i)
      if (part_ranks[i] > 32) fail(TT_EINVAL, "stitch: part ranks above 32 are not supported by this build");
    StandaloneCtx& c = standalone(device);
    std::lock_guard<std::mutex> op_lock(c.op);
    Exec& ex = *c.ex;
    DeviceGuard g(device);
    Index d[kMaxP], rq[kMaxP], rc[kMaxP];
    Index L = 0;
    for (int i = 0; i < nparts; ++i) L += part_dims[i * p];
    d[0] = L;
    for (int m = 1; m < kMaxP; ++m) d[m] = m < p ? part_dims[m] : 1;
    for (int m = 0; m < kMaxP; ++m) rq[m] = m < p ? ranks[m] : 1;
    clamp_ranks(p, d, rq, rc);
    std::vector<std::unique_ptr<DevBuf>> bufs;
    std::vector<StitchPart> parts;
    Index rho_max[kMaxP] = {};
    for (int i = 0; i < nparts; ++i) {
      StitchPart sp{};
      const int64_t* pd = part_dims + i * p;
      const int64_t* pr = part_ranks + i * p;
      bufs.push_back(std::make_unique<DevBuf>());
      sp.core = upload(*bufs.back(), cores[i], static_cast<size_t>(prod_range(pr, 0, p)), ex.stream);
      for (int m = 0; m < p; ++m) {
        if (pr[m] < 1 || pr[m] > pd[m]) fail(TT_EINVAL, "stitch: part rank out of range");
        bufs.push_back(std::make_unique<DevBuf>());
        const double* fm = upload(*bufs.back(), factors[i * p + m], static_cast<size_t>(pd[m] * pr[m]), ex.stream);
        sp.rho[m] = pr[m];
        rho_max[m] = std::max(rho_max[m], pr[m]);
        if (m == 0) {
          sp.v0 = fm;
        } else {
          sp.v[m] = fm;
        }
      }
      sp.ld0 = pd[0];
      sp.row0 = 0;
      sp.len = pd[0];
      sp.partial = 0;
      parts.push_back(sp);
    }
    DevBuf bout;
    size_t need = static_cast<size_t>(prod_range(rc, 0, p));
    for (int m = 0; m < p; ++m) need += static_cast<size_t>(d[m] * rc[m]) + 32;
    bout.ensure(need * sizeof(double));
    StitchDesc dsc{};
    dsc.part0 = 0;
    dsc.nparts = nparts;
    dsc.L = L;
    double* cur = bout.as<double>();
    for (int m = 0; m < p; ++m) {
      dsc.out_f[m] = cur;
      cur += d[m] * rc[m] + 16;
    }
    dsc.out_core = cur;
    Params prm = make_params(p, d, rq, max_iters, tol);
    InitCache init;
    init.p = p;
    for (int m = 0; m < p; ++m) {
      init.d[m] = d[m];
      init.req[m] = rq[m];
    }
    init.seed = seed;
    init.stitch_init(prm, ex.stream);
    std::vector<StitchDesc> descs{dsc};
    const auto st = run_stitch_batch(ex, prm, descs, parts,
                                     {stitch_ws_layout(p, L, d, rq, rho_max, nparts).total});
    auto f = std::make_unique<tt_factors>();
    f->p = p;
    Index k[kMaxP];
    for (int m = 0; m < p; ++m) k[m] = st[0].zero ? rc[m] : st[0].k[m];
    if (st[0].zero) {
      const auto u0 = init.stitch_zero_u0(L, rc[0]);
      cuda_check(cudaMemcpyAsync(dsc.out_f[0], u0.data(), u0.size() * sizeof(double), cudaMemcpyHostToDevice, ex.stream),
                 "zero-path upload");
    }
    for (int m = 0; m < p; ++m) {
      f->dims[m] = d[m];
      f->ranks[m] = k[m];
    }
    f->core = download(dsc.out_core, static_cast<size_t>(prod_range(k, 0, p)), ex.stream);
    for (int m = 0; m < p; ++m) f->f.push_back(download(dsc.out_f[m], static_cast<size_t>(d[m] * k[m]), ex.stream));
    ex.sync();
    f->objective = st[0].objective;
    f->sweeps = st[0].sweeps;
    f->converged = st[0].converged;
    *out = f.release();
  });
}

tt_status tt_partial_hit(int32_t p, const int64_t* dims, const int64_t* ranks, const double* core,
                         const double* const* factors, int64_t begin, int64_t end, int32_t device, tt_factors** out) {
  return guarded([&] {  // partial_hit_factors (stitch.cpp:36-47) on the device
    if (!dims || !ranks || !core || !factors || !out) fail(TT_EINVAL, "null argument");
    *out = nullptr;
    if (p < 2 || p > TT_MAX_ORDER) fail(TT_EINVAL, "partial_hit_factors: order must be in [2, 8]");
    for (int m = 0; m < p; ++m) {
      if (dims[m] < 1 || ranks[m] < 1) fail(TT_EINVAL, "partial_hit_factors: bad factor shape");
      if (!factors[m]) fail(TT_EINVAL, "null factor");
    }
    const Index len0 = dims[0];
    if (begin < 0 || begin >= end || end > len0) fail(TT_EINVAL, "partial_hit_factors: invalid sub-range");
    const int n = static_cast<int>(ranks[0]);
    if (n > kMaxVecHost) fail(TT_EINVAL, "partial_hit_factors: temporal rank above 32");
    const Index len = end - begin, k = std::min<Index>(len, n);
    Index rest = 1;
    for (int m = 1; m < p; ++m) rest *= ranks[m];
    StandaloneCtx& c = standalone(device);
    std::lock_guard<std::mutex> op_lock(c.op);
    Exec& ex = *c.ex;
    DeviceGuard g(device);
    DevBuf bv, bc, bw, bq, br, bo, bt;
    const double* dv = upload(bv, factors[0], static_cast<size_t>(len0 * n), ex.stream);
    const double* dc = upload(bc, core, static_cast<size_t>(n * rest), ex.stream);
    bw.ensure(static_cast<size_t>(len * n) * sizeof(double));
    bq.ensure(static_cast<size_t>(len * k) * sizeof(double));
    br.ensure(static_cast<size_t>(k * n) * sizeof(double));
    bo.ensure(static_cast<size_t>(std::max<Index>(k * rest, 1)) * sizeof(double));
    bt.ensure(static_cast<size_t>(n) * sizeof(double));
    cuda_check(launch_partial_hit(dv, len0, begin, len, n, dc, rest, bw.as<double>(), bq.as<double>(),
                                  br.as<double>(), bo.as<double>(), bt.as<double>(), ex.stream),
               "partial_hit_kernel launch");
    auto f = std::make_unique<tt_factors>();
    f->p = p;
    for (int m = 0; m < p; ++m) {
      f->dims[m] = m == 0 ? len : dims[m];
      f->ranks[m] = m == 0 ? k : ranks[m];
    }
    f->core = download(bo.as<double>(), static_cast<size_t>(k * rest), ex.stream);
    f->f.push_back(download(bq.as<double>(), static_cast<size_t>(len * k), ex.stream));
    for (int m = 1; m < p; ++m)
      f->f.emplace_back(factors[m], factors[m] + static_cast<size_t>(dims[m] * ranks[m]));
    ex.sync();
    *out = f.release();
  });
}

int32_t tt_factors_order(const tt_factors* f) { return f ? f->p : 0; }
int64_t tt_factors_dim(const tt_factors* f, int32_t m) { return f ? f->dims[m] : 0; }
int64_t tt_factors_rank(const tt_factors* f, int32_t m) { return f ? f->ranks[m] : 0; }
const double* tt_factors_core(const tt_factors* f) { return f ? f->core.data() : nullptr; }
const double* tt_factors_factor(const tt_factors* f, int32_t m) { return f ? f->f[m].data() : nullptr; }
int32_t tt_factors_sweeps(const tt_factors* f) { return f ? f->sweeps : 0; }
int32_t tt_factors_converged(const tt_factors* f) { return f ? f->converged : 0; }
const double* tt_factors_objective(const tt_factors* f) { return f ? f->objective.data() : nullptr; }
void tt_factors_free(tt_factors* f) { delete f; }

}  // extern "C"

// ===========================================================================
// Persistence: the reference's SST1 / TTS1 containers (io.hpp:11-31,
// io.cpp:87-239), little-endian, written field by field in the reference's
// order. Host-side I/O only; node payloads move through the device slots.
namespace {

constexpr char kTreeMagic[4] = {'S', 'S', 'T', '1'};
constexpr char kTensorMagic[4] = {'T', 'T', 'S', '1'};
constexpr char kBlockMagic[4] = {'T', 'T', 'B', '1'};  // engine extension: leaf block + raw tail
constexpr uint16_t kFormatVersion = 1;

struct Writer {
  std::FILE* f;
  std::string path;
  explicit Writer(const char* p) : f(std::fopen(p, "wb")), path(p) {
    if (!f) fail(TT_EIO, std::string("cannot open ") + p + " for writing");
  }
  ~Writer() {
    if (f) std::fclose(f);
  }
  void bytes(const void* b, size_t n) {
    if (n && std::fwrite(b, 1, n, f) != n) fail(TT_EIO, "failed writing " + path);
  }
  template <class T>
  void le(T v) {  // x86-64 is little-endian: the in-memory bytes are the file bytes
    bytes(&v, sizeof(T));
  }
  void close() {
    if (std::fclose(f) != 0) {
      f = nullptr;
      fail(TT_EIO, "failed writing " + path);
    }
    f = nullptr;
  }
};

struct Reader {
  std::FILE* f;
  explicit Reader(const char* p) : f(std::fopen(p, "rb")) {
    if (!f) fail(TT_EIO, std::string("cannot open ") + p);
  }
  ~Reader() {
    if (f) std::fclose(f);
  }
  bool try_bytes(void* b, size_t n) { return std::fread(b, 1, n, f) == n; }
  void bytes(void* b, size_t n, const char* what) {  // io.cpp:40-47
    if (n && !try_bytes(b, n)) fail(TT_EIO, std::string("truncated input reading ") + what);
  }
  template <class T>
  T le(const char* what) {
    T v;
    bytes(&v, sizeof(T), what);
    return v;
  }
  Index extent(const char* what) {  // io.cpp:62-70
    const uint64_t v = le<uint64_t>(what);
    if (v > uint64_t(1) << 40) fail(TT_EIO, std::string("implausible extent in ") + what);
    return static_cast<Index>(v);
  }
  void magic(const char* m, const char* what) {  // io.cpp:76-85
    char got[4];
    bytes(got, 4, what);
    if (std::memcmp(got, m, 4) != 0) fail(TT_EIO, std::string("bad magic for ") + what);
    const uint16_t version = le<uint16_t>(what);
    if (version != kFormatVersion)
      fail(TT_EIO, "unsupported version " + std::to_string(version) + " for " + what);
  }
};

// write_factors (io.cpp:87-101): u8 p | core dims | core | per mode rows, cols, row-major entries
void write_node_factors(Writer& w, const tt_tree& t, const HostNode& v) {
  const int p = t.p;
  w.le<uint8_t>(static_cast<uint8_t>(p));
  for (int m = 0; m < p; ++m) w.le<uint64_t>(static_cast<uint64_t>(v.ranks[m]));
  std::vector<double> core(static_cast<size_t>(prod_range(v.ranks, 0, p)));
  std::vector<std::vector<double>> f(static_cast<size_t>(p));
  std::vector<double*> fp(static_cast<size_t>(p));
  for (int m = 0; m < p; ++m) {
    const Index rows = m == 0 ? v.length() : t.d[m];
    f[m].resize(static_cast<size_t>(rows * v.ranks[m]));
    fp[m] = f[m].data();
  }
  DeviceGuard g(t.ex->device);
  cuda_check(cudaMemcpyAsync(core.data(), v.core, core.size() * sizeof(double), cudaMemcpyDeviceToHost, t.ex->stream),
             "node core download");
  for (int m = 0; m < p; ++m)
    cuda_check(cudaMemcpyAsync(fp[m], v.f[m], f[m].size() * sizeof(double), cudaMemcpyDeviceToHost, t.ex->stream),
               "node factor download");
  t.ex->sync();
  w.bytes(core.data(), core.size() * sizeof(double));
  std::vector<double> rowmajor;
  for (int m = 0; m < p; ++m) {
    const Index rows = m == 0 ? v.length() : t.d[m], cols = v.ranks[m];
    w.le<uint64_t>(static_cast<uint64_t>(rows));
    w.le<uint64_t>(static_cast<uint64_t>(cols));
    rowmajor.resize(static_cast<size_t>(rows * cols));
    for (Index i = 0; i < rows; ++i)
      for (Index j = 0; j < cols; ++j) rowmajor[size_t(i * cols + j)] = f[m][size_t(i + j * rows)];
    w.bytes(rowmajor.data(), rowmajor.size() * sizeof(double));
  }
}

}  // namespace

namespace {
// A node record with its host payload (SST1 reader, from_parts).
struct PartRec {
  HostNode v;
  std::vector<double> core;
  std::vector<std::vector<double>> f;  // column-major
};

// StreamSegmentTree::from_parts (sst.cpp:30-71): ids are creation order
// 1..n, children exist; payloads are uploaded into the tree's device slots.
// `code` is the status for malformed records (TT_EIO for files).
tt_tree* install_parts(tt_config cfg, std::vector<PartRec>& recs, Index root, Index timespan, Index stitches,
                       Index tail, const std::vector<double>& tail_buf, tt_status code) {
  const int p = cfg.order;
  const Index B = std::max<Index>(cfg.leaf_block, 1);
  const uint64_t count = recs.size();
  tt_tree* raw = nullptr;
  const tt_status st = tt_tree_create(&cfg, &raw);
  if (st != TT_OK) fail(st, g_err);
  std::unique_ptr<tt_tree, void (*)(tt_tree*)> t(raw, tt_tree_destroy);
  // A file (strict) must be a consistent tree; from_parts (sst.cpp:47-62) only
  // checks the id order and the root id — the rest is validate()'s job.
  const bool strict = code == TT_EIO;
  Index leaves = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const HostNode& v = recs[i].v;
    if (v.id != static_cast<Index>(i + 1))
      fail(code, strict ? "node ids must be 1..n in creation order" : "from_parts: node ids must be 1..N in order");
    if (!strict) continue;
    if (v.left > static_cast<Index>(count) || v.right > static_cast<Index>(count) || v.left < 0 || v.right < 0)
      fail(code, "node child id out of range");
    if (v.begin < 0 || v.end <= v.begin || v.end % B != 0 || v.begin % B != 0)
      fail(code, "node range not aligned to the leaf block");
    if (v.kind == TT_LEAF) ++leaves;
  }
  if (root < 0 || root > static_cast<Index>(count))
    fail(code, strict ? "root id out of range" : "from_parts: root id out of range");
  if (!strict) leaves = timespan / B;
  if (timespan != leaves * B + tail) fail(code, "timespan does not match the leaves and tail");
  t->nodes.reserve(static_cast<size_t>(count));
  for (PartRec& rc : recs) {
    HostNode v = rc.v;
    v.core = nullptr;
    for (int m = 0; m < kMaxP; ++m) v.f[m] = nullptr;
    t->nodes.push_back(v);
    HostNode& dv = t->nodes.back();
    if (!dv.has_dec || t->structure_only) continue;
    for (int m = 0; m < p; ++m)
      if (dv.ranks[m] > t->clamped(m, std::max<Index>(dv.length(), 1)))
        fail(code, "node rank exceeds the tree's (clamped) ranks: the device slots are sized by them");
    if (dv.length() < 1) fail(code, "a node with a decomposition needs a non-empty range");
    t->alloc_slots(dv);
    DeviceGuard g(t->ex->device);
    cuda_check(cudaMemcpyAsync(dv.core, rc.core.data(), rc.core.size() * sizeof(double), cudaMemcpyHostToDevice,
                               t->ex->stream),
               "node core upload");
    for (int m = 0; m < p; ++m)
      cuda_check(cudaMemcpyAsync(dv.f[m], rc.f[m].data(), rc.f[m].size() * sizeof(double), cudaMemcpyHostToDevice,
                                 t->ex->stream),
                 "node factor upload");
    t->ex->sync();  // host staging buffers are freed per node
  }
  t->root = root;
  t->timespan = timespan;
  t->leaves = leaves;
  t->stitch_count = stitches;
  t->last_touches = 0;
  if (tail > 0 && !t->structure_only) {
    DeviceGuard g(t->ex->device);
    cuda_check(cudaMemcpy(t->tail.p, tail_buf.data(), tail_buf.size() * sizeof(double), cudaMemcpyHostToDevice),
               "tail upload");
  }
  return t.release();
}
}  // namespace

extern "C" {

tt_status tt_tree_save(const tt_tree* t, const char* path) {
  return guarded([&] {
    if (!t || !path) fail(TT_EINVAL, "tt_tree_save: null argument");
    if (t->structure_only) fail(TT_ELOGIC, "tt_tree_save: a structure-only tree has no payloads");
    std::lock_guard<std::mutex> lk(t->qmu);
    Writer w(path);
    // write_tree (io.cpp:165-188)
    w.bytes(kTreeMagic, 4);
    w.le<uint16_t>(kFormatVersion);
    w.le<uint64_t>(static_cast<uint64_t>(t->timespan));
    w.le<uint8_t>(static_cast<uint8_t>(t->p));
    for (int m = 1; m < t->p; ++m) w.le<uint64_t>(static_cast<uint64_t>(t->d[m]));
    for (int m = 0; m < t->p; ++m) w.le<uint64_t>(static_cast<uint64_t>(t->cfg.ranks[m]));
    w.le<double>(t->cfg.theta);
    w.le<uint32_t>(static_cast<uint32_t>(t->cfg.max_iters));
    w.le<double>(t->cfg.tol);
    w.le<uint64_t>(t->cfg.seed);
    w.le<uint64_t>(static_cast<uint64_t>(t->stitch_count));
    w.le<uint64_t>(static_cast<uint64_t>(t->root));
    w.le<uint64_t>(static_cast<uint64_t>(t->nodes.size()));
    for (const HostNode& v : t->nodes) {
      w.le<uint64_t>(static_cast<uint64_t>(v.id));
      w.le<uint64_t>(static_cast<uint64_t>(v.begin));
      w.le<uint64_t>(static_cast<uint64_t>(v.end));
      w.le<uint8_t>(static_cast<uint8_t>(v.kind));
      w.le<uint64_t>(static_cast<uint64_t>(v.left));
      w.le<uint64_t>(static_cast<uint64_t>(v.right));
      w.le<uint8_t>(v.has_dec ? 1 : 0);
      if (v.has_dec) write_node_factors(w, *t, v);
    }
    const Index tail = t->timespan - t->leaves * t->B;
    if (t->B > 1 || tail > 0) {  // engine extension (ignored by the reference reader)
      w.bytes(kBlockMagic, 4);
      w.le<uint16_t>(kFormatVersion);
      w.le<uint64_t>(static_cast<uint64_t>(t->B));
      w.le<uint64_t>(static_cast<uint64_t>(tail));
      std::vector<double> buf(static_cast<size_t>(tail * t->slice));
      if (!buf.empty()) {
        DeviceGuard g(t->ex->device);
        cuda_check(cudaMemcpyAsync(buf.data(), t->tail.p, buf.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                   t->ex->stream),
                   "tail download");
        t->ex->sync();
      }
      w.bytes(buf.data(), buf.size() * sizeof(double));
    }
    w.close();
  });
}

tt_status tt_tree_load(const char* path, int32_t device, int32_t flags, tt_tree** out) {
  return guarded([&] {
    if (!path || !out) fail(TT_EINVAL, "tt_tree_load: null argument");
    *out = nullptr;
    Reader r(path);
    // read_tree (io.cpp:190-230)
    r.magic(kTreeMagic, "tree file");
    const uint64_t timespan = r.le<uint64_t>("timespan");
    const int p = r.le<uint8_t>("tree header");
    if (p < 2) fail(TT_EIO, "tree header: order must be >= 2");
    if (p > TT_MAX_ORDER) fail(TT_EIO, "tree header: order above " + std::to_string(TT_MAX_ORDER));
    tt_config cfg{};
    cfg.order = p;
    for (int m = 0; m < p - 1; ++m) cfg.nontemporal[m] = r.extent("tree shape");
    for (int m = 0; m < p; ++m) cfg.ranks[m] = r.extent("tree ranks");
    cfg.theta = r.le<double>("tree theta");
    cfg.max_iters = static_cast<int32_t>(r.le<uint32_t>("als iters"));
    cfg.tol = r.le<double>("als tol");
    cfg.seed = r.le<uint64_t>("als seed");
    const uint64_t stitches = r.le<uint64_t>("stitch count");
    const uint64_t root = r.le<uint64_t>("root id");
    const uint64_t count = r.le<uint64_t>("node count");
    if (count > (uint64_t(1) << 32)) fail(TT_EIO, "implausible node count");
    std::vector<PartRec> recs(static_cast<size_t>(count));
    for (uint64_t i = 0; i < count; ++i) {
      PartRec& rc = recs[i];
      HostNode& v = rc.v;
      v.id = static_cast<Index>(r.le<uint64_t>("node id"));
      v.begin = static_cast<Index>(r.le<uint64_t>("node range"));
      v.end = static_cast<Index>(r.le<uint64_t>("node range"));
      const uint8_t kind = r.le<uint8_t>("node kind");
      if (kind > 2) fail(TT_EIO, "invalid node kind " + std::to_string(kind));
      v.kind = kind;
      v.left = static_cast<Index>(r.le<uint64_t>("node children"));
      v.right = static_cast<Index>(r.le<uint64_t>("node children"));
      if (r.le<uint8_t>("node payload flag") != 0) {  // read_factors (io.cpp:103-121)
        const int fp = r.le<uint8_t>("factor header");
        if (fp != p) fail(TT_EIO, "factor header: order does not match the tree");
        Index cd[kMaxP];
        for (int m = 0; m < p; ++m) cd[m] = r.extent("core dims");
        rc.core.resize(static_cast<size_t>(prod_range(cd, 0, p)));
        r.bytes(rc.core.data(), rc.core.size() * sizeof(double), "core payload");
        rc.f.resize(static_cast<size_t>(p));
        std::vector<double> rowmajor;
        for (int m = 0; m < p; ++m) {
          const Index rows = r.extent("factor rows"), cols = r.extent("factor cols");
          if (cols != cd[m]) fail(TT_EIO, "factor cols do not match the core dims");
          if (rows != (m == 0 ? v.end - v.begin : cfg.nontemporal[m - 1]))
            fail(TT_EIO, "factor rows do not match the node / tree shape");
          rowmajor.resize(static_cast<size_t>(rows * cols));
          r.bytes(rowmajor.data(), rowmajor.size() * sizeof(double), "factor payload");
          rc.f[m].resize(rowmajor.size());
          for (Index a = 0; a < rows; ++a)
            for (Index j = 0; j < cols; ++j) rc.f[m][size_t(a + j * rows)] = rowmajor[size_t(a * cols + j)];
          v.ranks[m] = cols;
        }
        v.has_dec = true;
      }
    }
    // optional engine extension: leaf block and raw tail
    Index B = 1, tail = 0;
    std::vector<double> tail_buf;
    char ext[4];
    if (r.try_bytes(ext, 4)) {
      if (std::memcmp(ext, kBlockMagic, 4) != 0) fail(TT_EIO, "unexpected trailing bytes after the node table");
      const uint16_t version = r.le<uint16_t>("block extension");
      if (version != kFormatVersion) fail(TT_EIO, "unsupported block-extension version");
      B = r.extent("leaf block");
      tail = r.extent("tail slices");
      if (B < 1 || tail >= B) fail(TT_EIO, "invalid leaf block / tail");
      Index ss = 1;
      for (int m = 0; m < p - 1; ++m) ss *= cfg.nontemporal[m];
      tail_buf.resize(static_cast<size_t>(tail * ss));
      r.bytes(tail_buf.data(), tail_buf.size() * sizeof(double), "tail payload");
    }
    cfg.leaf_block = B;
    cfg.device = device;
    cfg.flags = flags;
    *out = install_parts(cfg, recs, static_cast<Index>(root), static_cast<Index>(timespan),
                         static_cast<Index>(stitches), tail, tail_buf, TT_EIO);
  });
}

tt_status tt_tree_from_parts(const tt_config* cfg, const tt_node_info* nodes, int64_t n, const double* const* cores,
                             const double* const* factors, int64_t root, int64_t timespan, int64_t stitch_count,
                             tt_tree** out) {
  return guarded([&] {
    if (!cfg || !out || (n > 0 && !nodes)) fail(TT_EINVAL, "from_parts: null argument");
    if (n < 0) fail(TT_EINVAL, "from_parts: negative node count");
    *out = nullptr;
    const int p = cfg->order;
    if (p < 2 || p > TT_MAX_ORDER) fail(TT_EINVAL, "StreamSegmentTree: order must be in [2, 8]");
    std::vector<PartRec> recs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      PartRec& rc = recs[static_cast<size_t>(i)];
      const tt_node_info& ni = nodes[i];
      if (ni.kind < 0 || ni.kind > 2) fail(TT_EINVAL, "from_parts: invalid node kind");
      rc.v.id = ni.id;
      rc.v.begin = ni.begin;
      rc.v.end = ni.end;
      rc.v.kind = ni.kind;
      rc.v.left = ni.left;
      rc.v.right = ni.right;
      if (!ni.has_decomposition) continue;
      if (cfg->flags & TT_FLAG_STRUCTURE_ONLY) {  // bookkeeping only: the flag without a payload
        rc.v.has_dec = true;
        for (int m = 0; m < p; ++m) rc.v.ranks[m] = ni.ranks[m];
        continue;
      }
      if (!cores || !factors || !cores[i]) fail(TT_EINVAL, "from_parts: missing decomposition payload");
      Index cd[kMaxP];
      for (int m = 0; m < p; ++m) {
        cd[m] = ni.ranks[m];
        if (cd[m] < 1) fail(TT_EINVAL, "from_parts: decomposition ranks must be >= 1");
        rc.v.ranks[m] = cd[m];
      }
      rc.core.assign(cores[i], cores[i] + prod_range(cd, 0, p));
      rc.f.resize(static_cast<size_t>(p));
      for (int m = 0; m < p; ++m) {
        const double* fm = factors[i * p + m];
        if (!fm) fail(TT_EINVAL, "from_parts: missing factor payload");
        const Index rows = m == 0 ? ni.end - ni.begin : cfg->nontemporal[m - 1];
        rc.f[m].assign(fm, fm + rows * cd[m]);
      }
      rc.v.has_dec = true;
    }
    const Index B = std::max<Index>(cfg->leaf_block, 1);
    if (timespan % B != 0) fail(TT_EINVAL, "from_parts: timespan must be a multiple of the leaf block");
    *out = install_parts(*cfg, recs, root, timespan, stitch_count, 0, {}, TT_EINVAL);
  });
}

tt_status tt_tree_config(const tt_tree* t, tt_config* out) {
  return guarded([&] {
    if (!t || !out) fail(TT_EINVAL, "tt_tree_config: null argument");
    *out = t->cfg;
  });
}

tt_status tt_tensor_write(const char* path, int32_t p, const int64_t* dims, const double* data) {
  return guarded([&] {  // write_tensor (io.cpp:124-133)
    if (!path || !dims || p < 1 || p > 255) fail(TT_EINVAL, "tt_tensor_write: bad argument");
    Index n = 1;
    for (int m = 0; m < p; ++m) {
      if (dims[m] < 0) fail(TT_EINVAL, "tt_tensor_write: negative extent");
      n *= dims[m];
    }
    if (n > 0 && !data) fail(TT_EINVAL, "tt_tensor_write: null data");
    Writer w(path);
    w.bytes(kTensorMagic, 4);
    w.le<uint16_t>(kFormatVersion);
    w.le<uint8_t>(static_cast<uint8_t>(p));
    for (int m = 0; m < p; ++m) w.le<uint64_t>(static_cast<uint64_t>(dims[m]));
    w.bytes(data, static_cast<size_t>(n) * sizeof(double));
    w.close();
  });
}

tt_status tt_tensor_read(const char* path, int32_t* p, int64_t* dims, double* data) {
  return guarded([&] {  // read_tensor (io.cpp:135-145)
    if (!path || !p || !dims) fail(TT_EINVAL, "tt_tensor_read: null argument");
    Reader r(path);
    r.magic(kTensorMagic, "tensor file");
    const int order = r.le<uint8_t>("tensor header");
    if (order < 1) fail(TT_EIO, "tensor header: order must be >= 1");
    if (order > TT_TENSOR_MAX_ORDER) fail(TT_EIO, "tensor header: order above TT_TENSOR_MAX_ORDER");
    *p = order;
    Index n = 1;
    for (int m = 0; m < order; ++m) {
      dims[m] = r.extent("tensor dims");
      n *= dims[m];
    }
    if (data) r.bytes(data, static_cast<size_t>(n) * sizeof(double), "tensor payload");
  });
}

}  // extern "C"
