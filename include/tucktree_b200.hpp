// Header-only C++ facade over the C ABI (tucktree_b200.h) with the names and
// semantics of the reference library's public headers
// (/root/reference/proj/core/include/tucktree/{sst,query,tucker,stitch}.hpp):
// value types, exceptions rethrown from the ABI status codes
// (TT_EINVAL -> std::invalid_argument, TT_ELOGIC -> std::logic_error,
// TT_EIO/TT_ECUDA/... -> std::runtime_error). Matrices are column-major
// (Eigen::MatrixXd layout); cores are row-major with the temporal mode first.
//
// Reference call                               facade (namespace tucktree_b200)
//   StreamSegmentTree(TreeConfig)  sst.hpp:56    StreamSegmentTree(TreeConfig)
//   append(const DenseTensor&)     sst.hpp:67    append(const double*, n = 1)
//   timespan/height/stitch_count/  sst.hpp:69-91 same names
//     last_append_node_touches/root/node/nodes/validate
//   recall(tree, ts, te, theta)    query.hpp:33  recall(tree, ts, te, theta)
//   range_query[_detailed]         query.hpp:44  range_query[_detailed] (+ batch)
//   tucker_als(x, cfg)             tucker.hpp:48 tucker_als(x, dims, cfg)
//   stitch(parts, ranks, cfg)      stitch.hpp:34 stitch(parts, ranks, cfg)
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tucktree_b200.h"

namespace tucktree_b200 {

using Index = int64_t;
using NodeId = Index;
inline constexpr NodeId kNoNode = 0;
inline constexpr uint64_t kDefaultSeed = 20240117;

inline void check(tt_status s) {
  if (s == TT_OK) return;
  const std::string msg = tt_last_error();
  if (s == TT_EINVAL) throw std::invalid_argument(msg);
  if (s == TT_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

// Column-major matrix with the memory layout of Eigen::MatrixXd.
struct Matrix {
  Index rows = 0, cols = 0;
  std::vector<double> data;
  double operator()(Index i, Index j) const { return data[static_cast<size_t>(i + j * rows)]; }
};

struct AlsConfig {  // tucker.hpp:17-22
  int max_iters = 20;
  double tol = 0.01;
  std::vector<Index> ranks;
  uint64_t seed = kDefaultSeed;
};

struct TuckerFactors {  // tucker.hpp:33-40
  std::vector<Index> core_dims;
  std::vector<double> core;  // row-major
  std::vector<Matrix> factors;
  Index order() const { return static_cast<Index>(factors.size()); }
  Index dim(Index m) const { return factors[static_cast<size_t>(m)].rows; }
  Index rank(Index m) const { return factors[static_cast<size_t>(m)].cols; }
};

struct AlsTrace {  // tucker.hpp:25-28
  std::vector<double> objective;
  bool converged = false;
};

enum class NodeKind : uint8_t { Leaf = 0, Intermediate = 1, Placeholder = 2 };
enum class HitFlag : uint8_t { Entire = 0, Partial = 1, Tail = 2 };

struct Node {  // sst.hpp:26-36 (decomposition fetched lazily)
  NodeId id = kNoNode;
  Index begin = 0, end = 0;
  NodeKind kind = NodeKind::Placeholder;
  NodeId left = kNoNode, right = kNoNode;
  bool has_decomposition = false;
  std::vector<Index> ranks;
  Index length() const { return end - begin; }
};

struct HitEntry {  // query.hpp:16-23
  NodeId node = kNoNode;
  Index begin = 0, end = 0;
  HitFlag flag = HitFlag::Entire;
  Index length() const { return end - begin; }
};
using HitSet = std::vector<HitEntry>;

struct TreeConfig {  // sst.hpp:38-43 + leaf block + device
  std::vector<Index> nontemporal;
  std::vector<Index> ranks;
  double theta = 0.7;
  AlsConfig als;
  Index leaf_block = 1;
  int device = 0;
  int flags = 0;  // TT_FLAG_STRUCTURE_ONLY: bookkeeping without device work (not in the reference)
};

namespace detail {
inline TuckerFactors take(tt_factors* h) {
  TuckerFactors f;
  const int p = tt_factors_order(h);
  for (int m = 0; m < p; ++m) f.core_dims.push_back(tt_factors_rank(h, m));
  Index n = 1;
  for (Index r : f.core_dims) n *= r;
  f.core.assign(tt_factors_core(h), tt_factors_core(h) + n);
  for (int m = 0; m < p; ++m) {
    Matrix u;
    u.rows = tt_factors_dim(h, m);
    u.cols = tt_factors_rank(h, m);
    u.data.assign(tt_factors_factor(h, m), tt_factors_factor(h, m) + u.rows * u.cols);
    f.factors.push_back(std::move(u));
  }
  tt_factors_free(h);
  return f;
}
}  // namespace detail

class StreamSegmentTree {  // sst.hpp:54-105
 public:
  explicit StreamSegmentTree(TreeConfig cfg) : cfg_(std::move(cfg)) {
    if (cfg_.nontemporal.empty()) throw std::invalid_argument("StreamSegmentTree: non-temporal shape required");
    if (cfg_.ranks.size() != cfg_.nontemporal.size() + 1)
      throw std::invalid_argument("StreamSegmentTree: one rank per mode required");
    if (cfg_.ranks.size() > TT_MAX_ORDER) throw std::invalid_argument("StreamSegmentTree: order must be <= 8");
    tt_config c{};
    c.order = static_cast<int32_t>(cfg_.ranks.size());
    for (size_t m = 0; m < cfg_.nontemporal.size(); ++m) c.nontemporal[m] = cfg_.nontemporal[m];
    for (size_t m = 0; m < cfg_.ranks.size(); ++m) c.ranks[m] = cfg_.ranks[m];
    c.theta = cfg_.theta;
    c.max_iters = cfg_.als.max_iters;
    c.tol = cfg_.als.tol;
    c.seed = cfg_.als.seed;
    c.leaf_block = cfg_.leaf_block;
    c.device = cfg_.device;
    c.flags = cfg_.flags;
    check(tt_tree_create(&c, &h_));
  }
  ~StreamSegmentTree() { tt_tree_destroy(h_); }
  StreamSegmentTree(const StreamSegmentTree&) = delete;
  StreamSegmentTree& operator=(const StreamSegmentTree&) = delete;
  StreamSegmentTree(StreamSegmentTree&& o) noexcept : cfg_(std::move(o.cfg_)), h_(std::exchange(o.h_, nullptr)) {}

  // Adopts a handle (read_tree_file).
  StreamSegmentTree(tt_tree* h, TreeConfig cfg) : cfg_(std::move(cfg)), h_(h) {}

  // One or more row-major slices from host memory (n = 1: one append).
  void append(const double* slices, Index n = 1) { check(tt_append(h_, slices, n, TT_MEM_HOST)); }
  // Burst append straight from device memory.
  void append_device(const double* slices, Index n) { check(tt_append(h_, slices, n, TT_MEM_DEVICE)); }

  Index timespan() const { return tt_tree_stat(h_, TT_STAT_TIMESPAN); }
  Index height() const { return tt_tree_stat(h_, TT_STAT_HEIGHT); }
  Index stitch_count() const { return tt_tree_stat(h_, TT_STAT_STITCH_COUNT); }
  Index last_append_node_touches() const { return tt_tree_stat(h_, TT_STAT_LAST_TOUCHES); }
  Index node_count() const { return tt_tree_stat(h_, TT_STAT_NODE_COUNT); }
  NodeId root() const { return tt_tree_stat(h_, TT_STAT_ROOT); }
  const TreeConfig& config() const { return cfg_; }

  Node node(NodeId id) const {
    tt_node_info i{};
    check(tt_node_info_get(h_, id, &i));
    Node n;
    n.id = i.id;
    n.begin = i.begin;
    n.end = i.end;
    n.kind = static_cast<NodeKind>(i.kind);
    n.left = i.left;
    n.right = i.right;
    n.has_decomposition = i.has_decomposition != 0;
    n.ranks.assign(i.ranks, i.ranks + cfg_.ranks.size());
    return n;
  }
  std::vector<Node> nodes() const {
    std::vector<Node> out;
    for (Index id = 1; id <= node_count(); ++id) out.push_back(node(id));
    return out;
  }
  // Node::decomposition (downloaded on demand).
  TuckerFactors decomposition(NodeId id) const {
    const Node n = node(id);
    if (!n.has_decomposition) throw std::logic_error("node has no decomposition");
    const size_t p = cfg_.ranks.size();
    TuckerFactors f;
    f.core_dims = n.ranks;
    Index nc = 1;
    for (Index r : n.ranks) nc *= r;
    f.core.resize(static_cast<size_t>(nc));
    std::vector<double*> ptrs(p);
    for (size_t m = 0; m < p; ++m) {
      Matrix u;
      u.rows = m == 0 ? n.length() : cfg_.nontemporal[m - 1];
      u.cols = n.ranks[m];
      u.data.resize(static_cast<size_t>(u.rows * u.cols));
      f.factors.push_back(std::move(u));
    }
    for (size_t m = 0; m < p; ++m) ptrs[m] = f.factors[m].data.data();
    check(tt_node_get(h_, id, f.core.data(), ptrs.data(), TT_MEM_HOST));
    return f;
  }
  std::vector<std::string> validate() const {
    std::string buf(1 << 16, '\0');
    const int n = tt_validate(h_, buf.data(), static_cast<int64_t>(buf.size()));
    std::vector<std::string> out;
    size_t pos = 0;
    for (int i = 0; i < n; ++i) {
      const size_t e = buf.find('\n', pos);
      if (e == std::string::npos) break;
      out.push_back(buf.substr(pos, e - pos));
      pos = e + 1;
    }
    return out;
  }
  tt_tree* handle() const { return h_; }

 private:
  TreeConfig cfg_;
  tt_tree* h_ = nullptr;
};

inline HitSet recall(const StreamSegmentTree& tree, Index ts, Index te, std::optional<double> theta = std::nullopt) {
  std::vector<tt_hit> buf(4096);
  int64_t n = 0;
  check(tt_recall(tree.handle(), ts, te, theta.value_or(std::numeric_limits<double>::quiet_NaN()), buf.data(),
                  static_cast<int64_t>(buf.size()), &n));
  HitSet out;
  for (int64_t i = 0; i < n; ++i)
    out.push_back(HitEntry{buf[i].node, buf[i].begin, buf[i].end, static_cast<HitFlag>(buf[i].flag)});
  return out;
}

struct QueryResult {
  TuckerFactors factors;
  HitSet hits;
};

// range_query over many ranges in one batched launch.
inline std::vector<TuckerFactors> range_query_batch(const StreamSegmentTree& tree,
                                                    const std::vector<std::pair<Index, Index>>& ranges,
                                                    std::optional<double> theta = std::nullopt,
                                                    std::vector<AlsTrace>* traces = nullptr) {
  const auto& cfg = tree.config();
  const size_t p = cfg.ranks.size();
  std::vector<tt_range> rr(ranges.size());
  std::vector<tt_query_out> outs(ranges.size());
  std::vector<TuckerFactors> res(ranges.size());
  for (size_t q = 0; q < ranges.size(); ++q) {
    rr[q] = tt_range{ranges[q].first, ranges[q].second};
    const Index L = std::max<Index>(ranges[q].second - ranges[q].first, 1);
    TuckerFactors& f = res[q];
    Index nc = 1;
    for (size_t m = 0; m < p; ++m) {
      const Index rows = m == 0 ? L : cfg.nontemporal[m - 1];
      const Index rc = std::min(cfg.ranks[m], rows);
      nc *= rc;
      Matrix u;
      u.rows = rows;
      u.cols = rc;
      u.data.resize(static_cast<size_t>(rows * rc));
      f.factors.push_back(std::move(u));
    }
    f.core.resize(static_cast<size_t>(nc));
    outs[q] = tt_query_out{};
    outs[q].core = f.core.data();
    for (size_t m = 0; m < p; ++m) outs[q].factors[m] = f.factors[m].data.data();
  }
  check(tt_query_batch(tree.handle(), rr.data(), static_cast<int64_t>(rr.size()),
                       theta.value_or(std::numeric_limits<double>::quiet_NaN()), outs.data(), TT_MEM_HOST));
  if (traces) traces->resize(ranges.size());
  for (size_t q = 0; q < ranges.size(); ++q) {
    TuckerFactors& f = res[q];
    f.core_dims.assign(outs[q].ranks, outs[q].ranks + p);
    Index nc = 1;
    for (size_t m = 0; m < p; ++m) {
      f.factors[m].cols = outs[q].ranks[m];
      f.factors[m].data.resize(static_cast<size_t>(f.factors[m].rows * f.factors[m].cols));
      nc *= outs[q].ranks[m];
    }
    f.core.resize(static_cast<size_t>(nc));
    if (traces) {
      (*traces)[q].converged = outs[q].converged != 0;
      (*traces)[q].objective = {outs[q].objective};
    }
  }
  return res;
}

inline TuckerFactors range_query(const StreamSegmentTree& tree, Index ts, Index te,
                                 std::optional<double> theta = std::nullopt) {
  return range_query_batch(tree, {{ts, te}}, theta).front();
}

inline QueryResult range_query_detailed(const StreamSegmentTree& tree, Index ts, Index te,
                                        std::optional<double> theta = std::nullopt) {
  QueryResult r;
  r.hits = recall(tree, ts, te, theta);
  r.factors = range_query(tree, ts, te, theta);
  return r;
}

// tucker_als(x, cfg) with x row-major of the given dims.
inline TuckerFactors tucker_als(const double* x, const std::vector<Index>& dims, const AlsConfig& cfg,
                                AlsTrace* trace = nullptr, int device = 0) {
  if (cfg.ranks.size() != dims.size()) throw std::invalid_argument("clamp_ranks: one rank per mode required");
  tt_factors* h = nullptr;
  check(tt_tucker_als(x, static_cast<int32_t>(dims.size()), dims.data(), cfg.ranks.data(), cfg.max_iters, cfg.tol,
                      cfg.seed, device, &h));
  if (trace) {
    trace->converged = tt_factors_converged(h) != 0;
    trace->objective.assign(tt_factors_objective(h), tt_factors_objective(h) + tt_factors_sweeps(h));
  }
  return detail::take(h);
}

inline TuckerFactors stitch(const std::vector<TuckerFactors>& parts, const std::vector<Index>& ranks,
                            const AlsConfig& cfg, AlsTrace* trace = nullptr, int device = 0) {
  if (parts.empty()) throw std::invalid_argument("stitch: at least one part required");
  const Index p = parts[0].order();
  std::vector<int64_t> pd, pr;
  std::vector<const double*> cores, facs;
  for (const auto& q : parts) {
    if (q.order() != p) throw std::invalid_argument("stitch: part order mismatch");
    cores.push_back(q.core.data());
    for (Index m = 0; m < p; ++m) {
      pd.push_back(q.dim(m));
      pr.push_back(q.rank(m));
      facs.push_back(q.factors[static_cast<size_t>(m)].data.data());
    }
  }
  if (static_cast<Index>(ranks.size()) != p) throw std::invalid_argument("stitch: one rank per mode required");
  tt_factors* h = nullptr;
  check(tt_stitch(static_cast<int32_t>(parts.size()), static_cast<int32_t>(p), pd.data(), pr.data(), cores.data(),
                  facs.data(), ranks.data(), cfg.max_iters, cfg.tol, cfg.seed, device, &h));
  if (trace) {
    trace->converged = tt_factors_converged(h) != 0;
    trace->objective.assign(tt_factors_objective(h), tt_factors_objective(h) + tt_factors_sweeps(h));
  }
  return detail::take(h);
}

// partial_hit_factors (stitch.hpp:15): rows [begin, end) of a stored decomposition.
inline TuckerFactors partial_hit_factors(const TuckerFactors& stored, Index begin, Index end, int device = 0) {
  const Index p = stored.order();
  std::vector<int64_t> dims, ranks;
  std::vector<const double*> facs;
  for (Index m = 0; m < p; ++m) {
    dims.push_back(stored.dim(m));
    ranks.push_back(stored.rank(m));
    facs.push_back(stored.factors[static_cast<size_t>(m)].data.data());
  }
  tt_factors* h = nullptr;
  check(tt_partial_hit(static_cast<int32_t>(p), dims.data(), ranks.data(), stored.core.data(), facs.data(), begin, end,
                       device, &h));
  return detail::take(h);
}

// brute_force_range (baseline.hpp): tucker_als of x[ts:te) (x row-major, dims[0] = T) on the device.
inline TuckerFactors brute_force_range(const double* x, const std::vector<Index>& dims, Index ts, Index te,
                                       const std::vector<Index>& ranks, const AlsConfig& cfg, int device = 0) {
  const tt_range r{ts, te};
  tt_factors* h = nullptr;
  check(tt_brute_force_batch(x, TT_MEM_HOST, static_cast<int32_t>(dims.size()), dims.data(), ranks.data(), &r, 1,
                             cfg.max_iters, cfg.tol, cfg.seed, device, &h));
  return detail::take(h);
}

// ---- persistence (io.hpp:15-31): SST1 trees, TTS1 tensors -------------------
inline void write_tree_file(const std::string& path, const StreamSegmentTree& tree) {
  check(tt_tree_save(tree.handle(), path.c_str()));
}

inline StreamSegmentTree read_tree_file(const std::string& path, int device = 0, int flags = 0) {
  tt_tree* h = nullptr;
  check(tt_tree_load(path.c_str(), device, flags, &h));
  tt_config c{};
  check(tt_tree_config(h, &c));
  TreeConfig cfg;
  for (int m = 0; m + 1 < c.order; ++m) cfg.nontemporal.push_back(c.nontemporal[m]);
  for (int m = 0; m < c.order; ++m) cfg.ranks.push_back(c.ranks[m]);
  cfg.theta = c.theta;
  cfg.als.max_iters = c.max_iters;
  cfg.als.tol = c.tol;
  cfg.als.seed = c.seed;
  cfg.leaf_block = c.leaf_block;
  cfg.device = c.device;
  cfg.flags = c.flags;
  return StreamSegmentTree(h, std::move(cfg));
}

inline void write_tensor_file(const std::string& path, const std::vector<Index>& dims, const double* data) {
  check(tt_tensor_write(path.c_str(), static_cast<int32_t>(dims.size()), dims.data(), data));
}

// Returns the payload (row-major) and sets dims.
inline std::vector<double> read_tensor_file(const std::string& path, std::vector<Index>& dims) {
  int32_t p = 0;
  int64_t d[TT_TENSOR_MAX_ORDER] = {};
  check(tt_tensor_read(path.c_str(), &p, d, nullptr));
  dims.assign(d, d + p);
  Index n = 1;
  for (Index v : dims) n *= v;
  std::vector<double> out(static_cast<size_t>(n));
  check(tt_tensor_read(path.c_str(), &p, d, out.data()));
  return out;
}

}  // namespace tucktree_b200
