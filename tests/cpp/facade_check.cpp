// Compiled by tests/test_facade.py against include/tucktree_b200.hpp and the
// engine library: every SURVEY.md §8(b) signature of the reference API
// (namespace tucktree). Mode "structure": host bookkeeping only (no GPU) —
// golden leaf ids, Fig. 3 hit set, append's shape check, from_parts + validate
// fault injection, out_of_range for unknown ids, TTS1 I/O. Mode "gpu": adds the
// numeric entry points on the device (range_query[_detailed] with its AlsTrace,
// tucker_als, stitch, partial_hit_factors, brute_force_range, SST1 round trip).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "tucktree_b200.hpp"

using namespace tucktree;

static int fails = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("CHECK failed line %d: %s\n", __LINE__, #c);     \
      ++fails;                                                     \
    }                                                              \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static DenseTensor slice(int t) {
  return DenseTensor(Shape{2}, {std::sin(0.1 * t), std::sin(0.1 * t + 0.37)});
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  TreeConfig cfg;
  cfg.nontemporal = {2};
  cfg.ranks = {2, 2};
  cfg.als.max_iters = 4;
  cfg.als.seed = 99;
  cfg.flags = gpu ? 0 : TT_FLAG_STRUCTURE_ONLY;
  StreamSegmentTree tree(cfg);
  for (int t = 0; t < 9; ++t) tree.append(slice(t));  // sst.hpp:67 append(const DenseTensor&)
  // test_sst.cpp:62-84 golden leaf ids
  std::vector<NodeId> leaf_ids;
  for (Index b = 0; b < 9; ++b)
    for (const Node& v : tree.nodes())
      if (v.kind == NodeKind::Leaf && v.begin == b) leaf_ids.push_back(v.id);
  CHECK((leaf_ids == std::vector<NodeId>{1, 3, 6, 7, 11, 12, 14, 15, 20}));
  CHECK(tree.height() == 5 && tree.node(tree.root()).end == 16);
  CHECK(tree.timespan() == 9 && tree.stitch_count() == 9 - 2 && tree.validate().empty());
  CHECK(tree.config().ranks == cfg.ranks && tree.node_count() == 20);
  // append rejects a mismatched slice and leaves the tree unchanged (test_sst.cpp:172-179)
  const Index n_before = tree.node_count();
  CHECK(throws<std::invalid_argument>([&] { tree.append(DenseTensor(Shape{3})); }));
  CHECK(tree.node_count() == n_before && tree.timespan() == 9);
  // sst.cpp:66-71: unknown node ids are std::out_of_range
  CHECK(throws<std::out_of_range>([&] { (void)tree.node(0); }));
  CHECK(throws<std::out_of_range>([&] { (void)tree.node(n_before + 1); }));
  // test_query.cpp:52-73 (Fig. 3 shape)
  const HitSet h = recall(tree, 1, 6, 0.7);
  CHECK(h.size() == 2 && h[0].flag == HitFlag::Partial && h[1].flag == HitFlag::Entire);
  CHECK(tree.node(h[0].node).begin == 0 && tree.node(h[0].node).end == 4 && h[0].begin == 1);
  CHECK(throws<std::invalid_argument>([&] { recall(tree, 2, 2); }));
  CHECK(throws<std::invalid_argument>([&] {
    TreeConfig bad = cfg;
    bad.theta = 1.5;
    StreamSegmentTree t2(bad);
  }));
  // from_parts + validate fault injection (test_sst.cpp:128-170)
  {
    std::vector<Node> nodes = tree.nodes();
    const StreamSegmentTree same = StreamSegmentTree::from_parts(cfg, nodes, tree.root(), tree.timespan(),
                                                                 tree.stitch_count());
    CHECK(same.validate().empty() && same.height() == tree.height() && same.stitch_count() == tree.stitch_count());
    for (Node& v : nodes)
      if (v.kind == NodeKind::Leaf && v.begin == 2) {
        v.begin = 1;
        v.end = 2;
        break;
      }
    const StreamSegmentTree bad = StreamSegmentTree::from_parts(cfg, nodes, tree.root(), tree.timespan(),
                                                                tree.stitch_count());
    bool names_node = false;
    for (const std::string& s : bad.validate()) names_node |= s.find("node ") != std::string::npos;
    CHECK(!bad.validate().empty() && names_node);
    std::vector<Node> nodes2 = tree.nodes();
    for (Node& v : nodes2)
      if (v.kind == NodeKind::Intermediate) {
        v.decomposition.reset();
        if (!gpu) v.kind = NodeKind::Intermediate;
        break;
      }
    if (gpu) {
      const StreamSegmentTree bad2 = StreamSegmentTree::from_parts(cfg, nodes2, tree.root(), tree.timespan(),
                                                                   tree.stitch_count());
      bool found = false;
      for (const std::string& s : bad2.validate()) found |= s.find("missing its decomposition") != std::string::npos;
      CHECK(found);
    }
    std::vector<Node> nodes3 = tree.nodes();
    nodes3[2].id = 7;
    CHECK(throws<std::invalid_argument>(
        [&] { StreamSegmentTree::from_parts(cfg, nodes3, tree.root(), tree.timespan(), tree.stitch_count()); }));
  }
  {  // TTS1 round trip through the facade (host I/O only)
    const DenseTensor x(Shape{3, 2}, {1.5, -2.0, 3.25, 4.0, 5.5, -6.0});
    write_tensor_file("facade_check.tts", x);
    const DenseTensor y = read_tensor_file("facade_check.tts");
    CHECK(y.shape() == x.shape() && y.data() == x.data());
    CHECK(throws<std::runtime_error>([&] { read_tensor_file("does_not_exist.tts"); }));
  }
  if (gpu) {
    write_tree_file("facade_check.sst", tree);
    const StreamSegmentTree back = read_tree_file("facade_check.sst");
    CHECK(back.timespan() == 9 && back.stitch_count() == tree.stitch_count() && back.validate().empty());
    const auto rs = range_query_batch(tree, {{0, 9}, {1, 6}, {3, 4}});
    CHECK(rs.size() == 3 && rs[0].dim(0) == 9 && rs[1].dim(0) == 5 && rs[2].dim(0) == 1);
    const TuckerFactors q = range_query(tree, 1, 6);
    CHECK(q.dim(0) == 5 && q.core.order() == 2);
    AlsTrace trace;
    const QueryResult qd = range_query_detailed(tree, 1, 6, std::nullopt, &trace);
    CHECK(qd.hits.size() == h.size() && qd.hits[0].node == h[0].node && qd.hits[1].flag == HitFlag::Entire);
    CHECK(!trace.objective.empty() && trace.objective.size() <= 4);
    for (size_t i = 1; i < trace.objective.size(); ++i)  // monotone objective (acceptance c9)
      CHECK(trace.objective[i] <= trace.objective[i - 1] * (1 + 1e-9) + 1e-12);
    const Node leaf = tree.node(h[1].node);
    CHECK(leaf.decomposition.has_value() && leaf.decomposition->dim(0) == 2);
    AlsConfig als;
    als.ranks = {2, 2};
    const DenseTensor x(Shape{3, 2}, {1, 2, 3, 4, 5, 6});
    AlsTrace tt;
    const TuckerFactors f = tucker_als(x, als, &tt);
    CHECK(f.rank(0) == 2 && f.rank(1) == 2 && !tt.objective.empty());
    const TuckerFactors g = stitch({f, f}, {2, 2}, als);
    CHECK(g.dim(0) == 6 && g.rank(1) == 2);
    const TuckerFactors ph = partial_hit_factors(g, 1, 4);
    CHECK(ph.dim(0) == 3);
    const TuckerFactors bf = brute_force_range(x, 0, 2, als);
    CHECK(bf.dim(0) == 2);
  }
  std::printf("%s: %d failures\n", gpu ? "gpu" : "structure", fails);
  return fails == 0 ? 0 : 1;
}
