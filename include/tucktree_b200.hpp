// Header-only C++ facade over the C ABI (tucktree_b200.h) with the names and
// semantics of the reference library's public headers
// (/root/reference/proj/core/include/tucktree/{tensor,tucker,stitch,sst,query,io}.hpp),
// in the reference's namespace `tucktree`: value types, and exceptions
// rethrown from the ABI status codes (TT_EINVAL -> std::invalid_argument,
// TT_ELOGIC -> std::logic_error, TT_ERANGE -> std::out_of_range,
// TT_EIO/TT_ECUDA/... -> std::runtime_error).
//
// Matrices: with Eigen on the include path (`__has_include(<Eigen/Core>)`),
// tucktree::Matrix IS Eigen::MatrixXd, so reference callers compile
// unchanged; without it, a column-major Matrix with the same layout and the
// rows()/cols()/data()/operator() surface the reference code uses.
// Cores are row-major DenseTensors with the temporal mode first.
//
// Reference call                                  facade (namespace tucktree)
//   Shape, DenseTensor               tensor.hpp:15-64  Shape, DenseTensor (subset)
//   StreamSegmentTree(TreeConfig)    sst.hpp:56        StreamSegmentTree(TreeConfig)
//   from_parts(cfg, nodes, root, T, stitches) :60      StreamSegmentTree::from_parts
//   append(const DenseTensor&)       sst.hpp:67        append(const DenseTensor&) (+ raw/burst/device)
//   timespan/height/stitch_count/last_append_node_touches/config/root/
//     node_count/node/nodes/validate sst.hpp:69-91     same names (node(): out_of_range)
//   recall(tree, ts, te, theta)      query.hpp:33      recall
//   range_query(tree, ts, te, theta) query.hpp:44      range_query (+ range_query_batch)
//   range_query_detailed(.., AlsTrace*) query.hpp:48   range_query_detailed (per-sweep trace)
//   tucker_als(x, cfg, trace)        tucker.hpp:48     tucker_als(DenseTensor, cfg, trace)
//   stitch(parts, ranks, cfg, trace) stitch.hpp:34     stitch
//   partial_hit_factors(f, b, e)     stitch.hpp:15     partial_hit_factors
//   brute_force_range                baseline.hpp      brute_force_range
//   write/read_tree_file, write/read_tensor_file io.hpp  same names
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tucktree_b200.h"

#if defined(TUCKTREE_USE_EIGEN) || (defined(__has_include) && __has_include(<Eigen/Core>))
#include <Eigen/Core>
#define TUCKTREE_FACADE_EIGEN 1
#else
#define TUCKTREE_FACADE_EIGEN 0
#endif

namespace tucktree {

using Index = int64_t;
using NodeId = Index;
inline constexpr NodeId kNoNode = 0;
inline constexpr uint64_t kDefaultSeed = 20240117;

inline void check(tt_status s) {
  if (s == TT_OK) return;
  const std::string msg = tt_last_error();
  if (s == TT_EINVAL) throw std::invalid_argument(msg);
  if (s == TT_ERANGE) throw std::out_of_range(msg);
  if (s == TT_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

#if TUCKTREE_FACADE_EIGEN
using Matrix = Eigen::MatrixXd;
#else
// Column-major matrix with the memory layout of Eigen::MatrixXd.
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : r_(rows), c_(cols), d_(static_cast<size_t>(rows * cols), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
  void resize(Index rows, Index cols) {
    r_ = rows;
    c_ = cols;
    d_.assign(static_cast<size_t>(rows * cols), 0.0);
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};
#endif

// tensor.hpp:15-30
class Shape {
 public:
  Shape() = default;
  explicit Shape(std::vector<Index> dims) : dims_(std::move(dims)) {
    if (dims_.empty()) throw std::invalid_argument("Shape: no dims given");
    for (Index d : dims_)
      if (d < 0) throw std::invalid_argument("Shape: negative extent");
  }
  Shape(std::initializer_list<Index> dims) : Shape(std::vector<Index>(dims)) {}
  Index order() const { return static_cast<Index>(dims_.size()); }
  Index dim(Index mode) const {
    if (mode < 0 || mode >= order()) throw std::invalid_argument("Shape::dim: invalid mode");
    return dims_[static_cast<size_t>(mode)];
  }
  const std::vector<Index>& dims() const { return dims_; }
  Index element_count() const {
    Index n = 1;
    for (Index d : dims_) n *= d;
    return n;
  }
  bool operator==(const Shape& o) const { return dims_ == o.dims_; }
  bool operator!=(const Shape& o) const { return dims_ != o.dims_; }

 private:
  std::vector<Index> dims_;
};

// tensor.hpp:32-64: row-major float64 tensor, temporal mode first.
class DenseTensor {
 public:
  DenseTensor() = default;
  explicit DenseTensor(Shape shape) : shape_(std::move(shape)), data_(static_cast<size_t>(shape_.element_count())) {}
  DenseTensor(Shape shape, std::vector<double> data) : shape_(std::move(shape)), data_(std::move(data)) {
    if (static_cast<Index>(data_.size()) != shape_.element_count())
      throw std::invalid_argument("DenseTensor: data size does not match shape");
  }
  const Shape& shape() const { return shape_; }
  Index order() const { return shape_.order(); }
  Index dim(Index mode) const { return shape_.dim(mode); }
  Index size() const { return static_cast<Index>(data_.size()); }
  const std::vector<double>& data() const { return data_; }
  std::vector<double>& data() { return data_; }

 private:
  Shape shape_;
  std::vector<double> data_;
};

struct AlsConfig {  // tucker.hpp:17-22
  int max_iters = 20;
  double tol = 0.01;
  std::vector<Index> ranks;
  uint64_t seed = kDefaultSeed;
};

struct AlsTrace {  // tucker.hpp:25-28
  std::vector<double> objective;
  bool converged = false;
};

struct TuckerFactors {  // tucker.hpp:33-40
  DenseTensor core;              // shape (r_1, ..., r_p)
  std::vector<Matrix> factors;   // factors[n] is D_n x r_n
  Index order() const { return static_cast<Index>(factors.size()); }
  Index dim(Index m) const { return factors[static_cast<size_t>(m)].rows(); }
  Index rank(Index m) const { return factors[static_cast<size_t>(m)].cols(); }
};

enum class NodeKind : uint8_t { Leaf = 0, Intermediate = 1, Placeholder = 2 };
// Tail = the raw slices past the last complete leaf block (leaf_block > 1 only).
enum class HitFlag : uint8_t { Entire = 0, Partial = 1, Tail = 2 };

struct Node {  // sst.hpp:26-36
  NodeId id = kNoNode;
  Index begin = 0, end = 0;
  NodeKind kind = NodeKind::Placeholder;
  NodeId left = kNoNode, right = kNoNode;
  std::optional<TuckerFactors> decomposition;
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
inline Matrix make_matrix(Index rows, Index cols) {
  Matrix m(rows, cols);
  return m;
}
inline TuckerFactors take(tt_factors* h) {
  TuckerFactors f;
  const int p = tt_factors_order(h);
  std::vector<Index> cd;
  for (int m = 0; m < p; ++m) cd.push_back(tt_factors_rank(h, m));
  Index n = 1;
  for (Index r : cd) n *= r;
  f.core = DenseTensor(Shape(cd), std::vector<double>(tt_factors_core(h), tt_factors_core(h) + n));
  for (int m = 0; m < p; ++m) {
    Matrix u = make_matrix(tt_factors_dim(h, m), tt_factors_rank(h, m));
    std::copy(tt_factors_factor(h, m), tt_factors_factor(h, m) + u.rows() * u.cols(), u.data());
    f.factors.push_back(std::move(u));
  }
  tt_factors_free(h);
  return f;
}
inline tt_config to_c(const TreeConfig& cfg) {
  if (cfg.nontemporal.empty()) throw std::invalid_argument("StreamSegmentTree: non-temporal shape required");
  if (cfg.ranks.size() != cfg.nontemporal.size() + 1)
    throw std::invalid_argument("StreamSegmentTree: one rank per mode required");
  if (cfg.ranks.size() > TT_MAX_ORDER) throw std::invalid_argument("StreamSegmentTree: order must be <= 8");
  tt_config c{};
  c.order = static_cast<int32_t>(cfg.ranks.size());
  for (size_t m = 0; m < cfg.nontemporal.size(); ++m) c.nontemporal[m] = cfg.nontemporal[m];
  for (size_t m = 0; m < cfg.ranks.size(); ++m) c.ranks[m] = cfg.ranks[m];
  c.theta = cfg.theta;
  c.max_iters = cfg.als.max_iters;
  c.tol = cfg.als.tol;
  c.seed = cfg.als.seed;
  c.leaf_block = cfg.leaf_block;
  c.device = cfg.device;
  c.flags = cfg.flags;
  return c;
}
}  // namespace detail

class StreamSegmentTree {  // sst.hpp:54-105
 public:
  explicit StreamSegmentTree(TreeConfig cfg) : cfg_(std::move(cfg)) {
    const tt_config c = detail::to_c(cfg_);
    check(tt_tree_create(&c, &h_));
  }
  ~StreamSegmentTree() { tt_tree_destroy(h_); }
  StreamSegmentTree(const StreamSegmentTree&) = delete;
  StreamSegmentTree& operator=(const StreamSegmentTree&) = delete;
  StreamSegmentTree(StreamSegmentTree&& o) noexcept : cfg_(std::move(o.cfg_)), h_(std::exchange(o.h_, nullptr)) {}

  // Adopts a handle (read_tree_file).
  StreamSegmentTree(tt_tree* h, TreeConfig cfg) : cfg_(std::move(cfg)), h_(h) {}

  // sst.hpp:58-62: node ids must be 1..nodes.size() in order and the root an id
  // or 0; the other invariants are validate()'s job (the device slots bound
  // each payload's ranks by the tree's clamped ranks).
  static StreamSegmentTree from_parts(TreeConfig cfg, std::vector<Node> nodes, NodeId root, Index timespan,
                                      Index stitch_count) {
    const tt_config c = detail::to_c(cfg);
    const size_t p = cfg.ranks.size();
    std::vector<tt_node_info> info(nodes.size());
    std::vector<const double*> cores(nodes.size(), nullptr), facs(nodes.size() * p, nullptr);
    for (size_t i = 0; i < nodes.size(); ++i) {
      const Node& v = nodes[i];
      tt_node_info& ni = info[i];
      ni = tt_node_info{};
      ni.id = v.id;
      ni.begin = v.begin;
      ni.end = v.end;
      ni.kind = static_cast<int32_t>(v.kind);
      ni.left = v.left;
      ni.right = v.right;
      ni.has_decomposition = v.decomposition.has_value();
      if (!v.decomposition) continue;
      const TuckerFactors& f = *v.decomposition;
      if (f.order() == 0 && (cfg.flags & TT_FLAG_STRUCTURE_ONLY)) continue;  // structure-only marker
      if (f.order() != static_cast<Index>(p)) throw std::invalid_argument("from_parts: decomposition order mismatch");
      for (size_t m = 0; m < p; ++m) {
        ni.ranks[m] = f.rank(static_cast<Index>(m));
        facs[i * p + m] = f.factors[m].data();
      }
      cores[i] = f.core.data().data();
    }
    tt_tree* h = nullptr;
    check(tt_tree_from_parts(&c, info.data(), static_cast<int64_t>(info.size()), cores.data(), facs.data(), root,
                             timespan, stitch_count, &h));
    return StreamSegmentTree(h, std::move(cfg));
  }

  // sst.hpp:64-67: one slice of the configured non-temporal shape; on a shape
  // mismatch the tree is left unchanged.
  void append(const DenseTensor& slice) {
    if (slice.shape().dims() != cfg_.nontemporal)
      throw std::invalid_argument("append: slice shape does not match the tree's non-temporal shape");
    check(tt_append(h_, slice.data().data(), 1, TT_MEM_HOST));
  }
  // Engine extensions: n row-major slices from host memory (n > 1: a burst,
  // result-identical to n appends), or straight from device memory.
  void append(const double* slices, Index n = 1) { check(tt_append(h_, slices, n, TT_MEM_HOST)); }
  void append_device(const double* slices, Index n) { check(tt_append(h_, slices, n, TT_MEM_DEVICE)); }

  Index timespan() const { return tt_tree_stat(h_, TT_STAT_TIMESPAN); }
  Index height() const { return tt_tree_stat(h_, TT_STAT_HEIGHT); }
  Index stitch_count() const { return tt_tree_stat(h_, TT_STAT_STITCH_COUNT); }
  Index last_append_node_touches() const { return tt_tree_stat(h_, TT_STAT_LAST_TOUCHES); }
  Index node_count() const { return tt_tree_stat(h_, TT_STAT_NODE_COUNT); }
  NodeId root() const { return tt_tree_stat(h_, TT_STAT_ROOT); }
  const TreeConfig& config() const { return cfg_; }

  // sst.hpp:90: the node with its decomposition (downloaded from the device);
  // std::out_of_range for an unknown id.
  Node node(NodeId id) const {
    const tt_node_info i = info(id);
    Node n;
    n.id = i.id;
    n.begin = i.begin;
    n.end = i.end;
    n.kind = static_cast<NodeKind>(i.kind);
    n.left = i.left;
    n.right = i.right;
    if (i.has_decomposition)  // a structure-only tree has no payloads: an empty (order-0) marker
      n.decomposition = (cfg_.flags & TT_FLAG_STRUCTURE_ONLY) ? TuckerFactors{} : download(i);
    return n;
  }
  std::vector<Node> nodes() const {
    std::vector<Node> out;
    for (Index id = 1; id <= node_count(); ++id) out.push_back(node(id));
    return out;
  }
  // Node metadata without the payload download (engine extension).
  tt_node_info info(NodeId id) const {
    tt_node_info i{};
    check(tt_node_info_get(h_, id, &i));
    return i;
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
  TuckerFactors download(const tt_node_info& i) const {
    const size_t p = cfg_.ranks.size();
    TuckerFactors f;
    std::vector<Index> cd(i.ranks, i.ranks + p);
    f.core = DenseTensor(Shape(cd));
    std::vector<double*> ptrs(p);
    for (size_t m = 0; m < p; ++m)
      f.factors.push_back(detail::make_matrix(m == 0 ? i.end - i.begin : cfg_.nontemporal[m - 1], i.ranks[m]));
    for (size_t m = 0; m < p; ++m) ptrs[m] = f.factors[m].data();
    check(tt_node_get(h_, i.id, f.core.data().data(), ptrs.data(), TT_MEM_HOST));
    return f;
  }

  TreeConfig cfg_;
  tt_tree* h_ = nullptr;
};

// query.hpp:33
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

struct QueryResult {  // query.hpp:36-39
  TuckerFactors factors;
  HitSet hits;
};

// range_query_detailed over many ranges in one batched launch; the engine
// fills every query's hit set and per-sweep trace in the same call.
inline std::vector<QueryResult> range_query_batch_detailed(const StreamSegmentTree& tree,
                                                           const std::vector<std::pair<Index, Index>>& ranges,
                                                           std::optional<double> theta = std::nullopt,
                                                           std::vector<AlsTrace>* traces = nullptr) {
  const auto& cfg = tree.config();
  const size_t p = cfg.ranks.size();
  std::vector<tt_range> rr(ranges.size());
  std::vector<tt_query_out> outs(ranges.size());
  std::vector<QueryResult> res(ranges.size());
  std::vector<std::vector<double>> tr(ranges.size(), std::vector<double>(static_cast<size_t>(std::max(cfg.als.max_iters, 1))));
  std::vector<std::vector<tt_hit>> hb(ranges.size(), std::vector<tt_hit>(256));
  std::vector<std::vector<double>> core(ranges.size());
  for (size_t q = 0; q < ranges.size(); ++q) {
    rr[q] = tt_range{ranges[q].first, ranges[q].second};
    const Index L = std::max<Index>(ranges[q].second - ranges[q].first, 1);
    TuckerFactors& f = res[q].factors;
    Index nc = 1;
    for (size_t m = 0; m < p; ++m) {
      const Index rows = m == 0 ? L : cfg.nontemporal[m - 1];
      const Index rc = std::min(cfg.ranks[m], rows);
      nc *= rc;
      f.factors.push_back(detail::make_matrix(rows, rc));
    }
    core[q].resize(static_cast<size_t>(nc));
    outs[q] = tt_query_out{};
    outs[q].core = core[q].data();
    for (size_t m = 0; m < p; ++m) outs[q].factors[m] = f.factors[m].data();
    outs[q].trace = tr[q].data();
    outs[q].trace_cap = static_cast<int32_t>(tr[q].size());
    outs[q].hits = hb[q].data();
    outs[q].hits_cap = static_cast<int32_t>(hb[q].size());
  }
  check(tt_query_batch(tree.handle(), rr.data(), static_cast<int64_t>(rr.size()),
                       theta.value_or(std::numeric_limits<double>::quiet_NaN()), outs.data(), TT_MEM_HOST));
  if (traces) traces->resize(ranges.size());
  for (size_t q = 0; q < ranges.size(); ++q) {
    TuckerFactors& f = res[q].factors;
    std::vector<Index> cd(outs[q].ranks, outs[q].ranks + p);
    Index nc = 1;
    for (size_t m = 0; m < p; ++m) {
      // the buffer holds rows x k (ld = rows) for the actual column count k
      Matrix u = detail::make_matrix(f.factors[m].rows(), cd[m]);
      std::copy(f.factors[m].data(), f.factors[m].data() + u.rows() * u.cols(), u.data());
      f.factors[m] = std::move(u);
      nc *= cd[m];
    }
    f.core = DenseTensor(Shape(cd), std::vector<double>(core[q].begin(), core[q].begin() + nc));
    for (int32_t i = 0; i < std::min(outs[q].nhits, outs[q].hits_cap); ++i)
      res[q].hits.push_back(HitEntry{hb[q][i].node, hb[q][i].begin, hb[q][i].end, static_cast<HitFlag>(hb[q][i].flag)});
    if (traces) {
      (*traces)[q].converged = outs[q].converged != 0;
      (*traces)[q].objective.assign(tr[q].begin(), tr[q].begin() + std::min(outs[q].sweeps, outs[q].trace_cap));
    }
  }
  return res;
}

inline std::vector<TuckerFactors> range_query_batch(const StreamSegmentTree& tree,
                                                    const std::vector<std::pair<Index, Index>>& ranges,
                                                    std::optional<double> theta = std::nullopt,
                                                    std::vector<AlsTrace>* traces = nullptr) {
  std::vector<QueryResult> d = range_query_batch_detailed(tree, ranges, theta, traces);
  std::vector<TuckerFactors> out;
  out.reserve(d.size());
  for (auto& r : d) out.push_back(std::move(r.factors));
  return out;
}

// query.hpp:44-46
inline TuckerFactors range_query(const StreamSegmentTree& tree, Index ts, Index te,
                                 std::optional<double> theta = std::nullopt) {
  return range_query_batch(tree, {{ts, te}}, theta).front();
}

// query.hpp:48-50: one engine call returns the factors, the hit set and the
// per-sweep objective trace.
inline QueryResult range_query_detailed(const StreamSegmentTree& tree, Index ts, Index te,
                                        std::optional<double> theta = std::nullopt, AlsTrace* trace = nullptr) {
  std::vector<AlsTrace> tr;
  std::vector<QueryResult> r = range_query_batch_detailed(tree, {{ts, te}}, theta, trace ? &tr : nullptr);
  if (trace) *trace = tr.front();
  return std::move(r.front());
}

// tucker.hpp:48-49 on the device.
inline TuckerFactors tucker_als(const DenseTensor& x, const AlsConfig& cfg, AlsTrace* trace = nullptr,
                                int device = 0) {
  const std::vector<Index>& dims = x.shape().dims();
  if (cfg.ranks.size() != dims.size()) throw std::invalid_argument("clamp_ranks: one rank per mode required");
  tt_factors* h = nullptr;
  check(tt_tucker_als(x.data().data(), static_cast<int32_t>(dims.size()), dims.data(), cfg.ranks.data(),
                      cfg.max_iters, cfg.tol, cfg.seed, device, &h));
  if (trace) {
    trace->converged = tt_factors_converged(h) != 0;
    trace->objective.assign(tt_factors_objective(h), tt_factors_objective(h) + tt_factors_sweeps(h));
  }
  return detail::take(h);
}

// stitch.hpp:34-36 on the device.
inline TuckerFactors stitch(const std::vector<TuckerFactors>& parts, const std::vector<Index>& ranks,
                            const AlsConfig& cfg, AlsTrace* trace = nullptr, int device = 0) {
  if (parts.empty()) throw std::invalid_argument("stitch: at least one part required");
  const Index p = parts[0].order();
  std::vector<int64_t> pd, pr;
  std::vector<const double*> cores, facs;
  for (const auto& q : parts) {
    if (q.order() != p) throw std::invalid_argument("stitch: part order mismatch");
    cores.push_back(q.core.data().data());
    for (Index m = 0; m < p; ++m) {
      pd.push_back(q.dim(m));
      pr.push_back(q.rank(m));
      facs.push_back(q.factors[static_cast<size_t>(m)].data());
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

// stitch.hpp:15: rows [begin, end) of a stored decomposition.
inline TuckerFactors partial_hit_factors(const TuckerFactors& stored, Index begin, Index end, int device = 0) {
  const Index p = stored.order();
  std::vector<int64_t> dims, ranks;
  std::vector<const double*> facs;
  for (Index m = 0; m < p; ++m) {
    dims.push_back(stored.dim(m));
    ranks.push_back(stored.rank(m));
    facs.push_back(stored.factors[static_cast<size_t>(m)].data());
  }
  tt_factors* h = nullptr;
  check(tt_partial_hit(static_cast<int32_t>(p), dims.data(), ranks.data(), stored.core.data().data(), facs.data(),
                       begin, end, device, &h));
  return detail::take(h);
}

// baseline.hpp: tucker_als of x[ts:te) on the device.
inline TuckerFactors brute_force_range(const DenseTensor& x, Index ts, Index te, const AlsConfig& cfg,
                                       int device = 0) {
  const tt_range r{ts, te};
  const std::vector<Index>& dims = x.shape().dims();
  tt_factors* h = nullptr;
  check(tt_brute_force_batch(x.data().data(), TT_MEM_HOST, static_cast<int32_t>(dims.size()), dims.data(),
                             cfg.ranks.data(), &r, 1, cfg.max_iters, cfg.tol, cfg.seed, device, &h));
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

inline void write_tensor_file(const std::string& path, const DenseTensor& x) {
  check(tt_tensor_write(path.c_str(), static_cast<int32_t>(x.order()), x.shape().dims().data(), x.data().data()));
}

inline DenseTensor read_tensor_file(const std::string& path) {
  int32_t p = 0;
  int64_t d[TT_TENSOR_MAX_ORDER] = {};
  check(tt_tensor_read(path.c_str(), &p, d, nullptr));
  DenseTensor x(Shape(std::vector<Index>(d, d + p)));
  check(tt_tensor_read(path.c_str(), &p, d, x.data().data()));
  return x;
}

}  // namespace tucktree

// round-1 spelling of the facade namespace
namespace tucktree_b200 = tucktree;
