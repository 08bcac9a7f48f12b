// ============================================================================
// TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the reference
// tucktree hot path (arXiv 2501.06647, /root/reference/proj/core).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this code. The product path
// (paper_2501_06647_b200/) never links or calls it.
//
// The reference cannot be compiled in this image (Eigen 3 is absent, see
// SURVEY.md §8(c)), so every function below is a restatement of the cited
// reference function, written against a minimal column-major matrix type and
// the OpenBLAS/LAPACK bundled with numpy (Householder dgeqrf/dorgqr in place
// of Eigen::HouseholderQR, divide-and-conquer dgesdd in place of
// Eigen::BDCSVD). The init RNG streams (std::mt19937_64 +
// std::normal_distribution) are bit-identical because the same g++ 13 /
// libstdc++ is used.
//
// Parity pinning: the reference ships no value-level golden vectors; this
// oracle is pinned by the reference's own known-answer tests (leaf ids, hit
// sets, stitch counts, height law, block sizes, mt19937_64 KAT) and its
// tolerance properties (unfolding identities, exact recovery, orthonormality,
// monotone objective) — see tests/test_oracle_kats.py.
//
// Extension beyond the reference: a leaf block of B
// slices. With B = 1 every function below reduces to the reference exactly.
// ============================================================================
#pragma once

#include <cstdint>
#include <optional>
#include <random>
#include <span>
#include <string>
#include <vector>

namespace tto {

using Index = std::int64_t;

inline constexpr std::uint64_t kDefaultSeed = 20240117;  // tucker.hpp:13

// Column-major dense matrix (layout of Eigen::MatrixXd).
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), v(static_cast<std::size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return v[static_cast<std::size_t>(i + j * rows)]; }
  double operator()(Index i, Index j) const { return v[static_cast<std::size_t>(i + j * rows)]; }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  static Mat identity(Index n);
};

// Row-major dense tensor, temporal mode first (tensor.hpp:35-64).
struct Tensor {
  std::vector<Index> dims;
  std::vector<double> v;
  Tensor() = default;
  explicit Tensor(std::vector<Index> d);
  Tensor(std::vector<Index> d, std::vector<double> data);
  Index order() const { return static_cast<Index>(dims.size()); }
  Index dim(Index m) const { return dims[static_cast<std::size_t>(m)]; }
  Index size() const { return static_cast<Index>(v.size()); }
};

struct AlsConfig {  // tucker.hpp:17-22
  int max_iters = 20;
  double tol = 0.01;
  std::vector<Index> ranks;
  std::uint64_t seed = kDefaultSeed;
};

struct AlsTrace {  // tucker.hpp:25-28
  std::vector<double> objective;
  bool converged = false;
};

struct Factors {  // tucker.hpp:33-40
  Tensor core;
  std::vector<Mat> f;
  Index order() const { return static_cast<Index>(f.size()); }
  Index dim(Index m) const { return f[static_cast<std::size_t>(m)].rows; }
  Index rank(Index m) const { return f[static_cast<std::size_t>(m)].cols; }
};

// ---- blas/lapack threading ------------------------------------------------
void set_blas_threads(int n);

// ---- tensor primitives (tensor.cpp) --------------------------------------
Index element_count(std::span<const Index> dims);
Mat matricize(const Tensor& x, Index mode);
Tensor from_matricization(const Mat& m, std::vector<Index> dims, Index mode);
Tensor mode_product(const Tensor& x, const Mat& u, Index mode);
double squared_norm(const Tensor& x);
Tensor slice_temporal(const Tensor& x, Index begin, Index end);
Tensor concat_temporal(std::span<const Tensor> parts);
Mat transpose(const Mat& a);
Mat matmul(const Mat& a, const Mat& b);  // a * b

// ---- linalg (linalg.cpp) --------------------------------------------------
struct QrResult {
  Mat q, r;
};
QrResult thin_qr(const Mat& a);
Mat leading_left_singular_vectors(const Mat& a, Index rank);
Mat random_orthonormal(Index rows, Index cols, std::mt19937_64& rng);
double max_orthonormality_defect(const Mat& u);
Mat kronecker(const Mat& a, const Mat& b);

// ---- tucker (tucker.cpp) --------------------------------------------------
std::vector<Index> clamp_ranks(std::span<const Index> requested, std::span<const Index> dims);
Mat update_factor(const Tensor& x, const Factors& current, Index mode);
Tensor core_of(const Tensor& x, std::span<const Mat> factors);
Tensor reconstruct(const Factors& f);
Factors tucker_als(const Tensor& x, const AlsConfig& cfg, AlsTrace* trace = nullptr);
double relative_error(const Tensor& x, const Factors& candidate, const Factors& reference);

// ---- stitch (stitch.cpp) --------------------------------------------------
Factors partial_hit_factors(const Factors& stored, Index begin, Index end);
Mat stitch_temporal_unfolding(std::span<const Factors> parts, std::span<const Mat> factors);
Mat stitch_nontemporal_unfolding(std::span<const Factors> parts, Index mode,
                                 std::span<const Mat> factors);
Factors stitch(std::span<const Factors> parts, std::span<const Index> requested_ranks,
               const AlsConfig& cfg, AlsTrace* trace = nullptr);

// ---- baseline (baseline.cpp) ---------------------------------------------
Index default_block_size(Index timespan);
Factors brute_force_range(const Tensor& x, Index ts, Index te, std::span<const Index> ranks,
                          const AlsConfig& cfg);
struct SynthSpec {
  std::vector<Index> shape, true_ranks;
  double noise = 0.0;
  std::uint64_t seed = kDefaultSeed;
};
Tensor generate_synthetic(const SynthSpec& spec);

// ---- stream segment tree (sst.cpp) with leaf block B ---------------------
using NodeId = Index;
inline constexpr NodeId kNoNode = 0;
enum class NodeKind : std::uint8_t { Leaf = 0, Intermediate = 1, Placeholder = 2 };

struct Node {
  NodeId id = kNoNode;
  Index begin = 0, end = 0;  // in slices
  NodeKind kind = NodeKind::Placeholder;
  NodeId left = kNoNode, right = kNoNode;
  std::optional<Factors> dec;
  Index length() const { return end - begin; }
};

struct TreeConfig {  // sst.hpp:38-43 + leaf_block
  std::vector<Index> nontemporal;
  std::vector<Index> ranks;
  double theta = 0.7;
  AlsConfig als;
  Index leaf_block = 1;
};

class Tree {
 public:
  explicit Tree(TreeConfig cfg);
  // Appends one slice (row-major, prod(nontemporal) doubles).
  void append(const double* slice);
  Index timespan() const { return timespan_; }
  Index leaves() const { return leaves_; }
  Index height() const;
  Index stitch_count() const { return stitch_count_; }
  Index last_append_node_touches() const { return last_touches_; }
  NodeId root() const { return root_; }
  const Node& node(NodeId id) const;
  const std::vector<Node>& nodes() const { return nodes_; }
  const TreeConfig& config() const { return cfg_; }
  const Tensor& tail() const { return tail_; }  // raw slices past leaves*B
  std::vector<std::string> validate() const;
  // Node ids re-decomposed by the most recent append (leaf first, then stitches).
  const std::vector<NodeId>& last_redecomposed() const { return last_redec_; }

 private:
  NodeId create_node(Index begin_leaf, Index end_leaf);
  void insert(NodeId id, Index t, const Tensor& block);
  Node& node_mut(NodeId id) { return nodes_[static_cast<std::size_t>(id - 1)]; }

  TreeConfig cfg_;
  std::vector<Node> nodes_;
  NodeId root_ = kNoNode;
  Index timespan_ = 0, leaves_ = 0, stitch_count_ = 0, last_touches_ = 0;
  Index slice_size_ = 1;
  Tensor tail_;
  std::vector<NodeId> last_redec_;
};

enum class HitFlag : std::uint8_t { Entire = 0, Partial = 1, Tail = 2 };
struct HitEntry {
  NodeId node = kNoNode;
  Index begin = 0, end = 0;
  HitFlag flag = HitFlag::Entire;
};
using HitSet = std::vector<HitEntry>;

HitSet recall(const Tree& tree, Index ts, Index te, std::optional<double> theta = std::nullopt);
struct QueryResult {
  Factors factors;
  HitSet hits;
};
QueryResult range_query_detailed(const Tree& tree, Index ts, Index te,
                                 std::optional<double> theta = std::nullopt,
                                 AlsTrace* trace = nullptr);

}  // namespace tto
