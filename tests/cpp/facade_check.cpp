// Compiled by tests/test_facade.py against include/tucktree_b200.hpp and the
// engine library. Mode "structure": reference KATs on the host bookkeeping
// (no GPU). Mode "gpu": a small build + batched range queries on the device.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "tucktree_b200.hpp"

using namespace tucktree_b200;

static int fails = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("CHECK failed line %d: %s\n", __LINE__, #c);     \
      ++fails;                                                     \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  TreeConfig cfg;
  cfg.nontemporal = {2};
  cfg.ranks = {2, 2};
  cfg.als.max_iters = 4;
  cfg.als.seed = 99;
  cfg.flags = gpu ? 0 : TT_FLAG_STRUCTURE_ONLY;
  StreamSegmentTree tree(cfg);
  for (int t = 0; t < 9; ++t) {
    const double s[2] = {std::sin(0.1 * t), std::sin(0.1 * t + 0.37)};
    tree.append(s);
  }
  // test_sst.cpp:62-84 golden leaf ids
  std::vector<NodeId> leaf_ids;
  for (Index b = 0; b < 9; ++b)
    for (const Node& v : tree.nodes())
      if (v.kind == NodeKind::Leaf && v.begin == b) leaf_ids.push_back(v.id);
  CHECK((leaf_ids == std::vector<NodeId>{1, 3, 6, 7, 11, 12, 14, 15, 20}));
  CHECK(tree.height() == 5 && tree.node(tree.root()).end == 16);
  CHECK(tree.validate().empty());
  // test_query.cpp:52-73 (Fig. 3 shape)
  const HitSet h = recall(tree, 1, 6, 0.7);
  CHECK(h.size() == 2 && h[0].flag == HitFlag::Partial && h[1].flag == HitFlag::Entire);
  CHECK(tree.node(h[0].node).begin == 0 && tree.node(h[0].node).end == 4 && h[0].begin == 1);
  bool threw = false;
  try {
    recall(tree, 2, 2);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    TreeConfig bad = cfg;
    bad.theta = 1.5;
    StreamSegmentTree t2(bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  {  // TTS1 round trip through the facade (host I/O only)
    const std::vector<double> x = {1.5, -2.0, 3.25, 4.0, 5.5, -6.0};
    write_tensor_file("facade_check.tts", {3, 2}, x.data());
    std::vector<Index> dims;
    const std::vector<double> y = read_tensor_file("facade_check.tts", dims);
    CHECK((dims == std::vector<Index>{3, 2}) && y == x);
    threw = false;
    try {
      read_tensor_file("does_not_exist.tts", dims);
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw);
  }
  if (gpu) {
    write_tree_file("facade_check.sst", tree);
    const StreamSegmentTree back = read_tree_file("facade_check.sst");
    CHECK(back.timespan() == 9 && back.stitch_count() == tree.stitch_count() && back.validate().empty());
    const auto rs = range_query_batch(tree, {{0, 9}, {1, 6}, {3, 4}});
    CHECK(rs.size() == 3 && rs[0].dim(0) == 9 && rs[1].dim(0) == 5 && rs[2].dim(0) == 1);
    const TuckerFactors leaf = tree.decomposition(h[1].node);
    CHECK(leaf.dim(0) == 2);
    AlsConfig als;
    als.ranks = {2, 2};
    std::vector<double> x = {1, 2, 3, 4, 5, 6};
    const TuckerFactors f = tucker_als(x.data(), {3, 2}, als);
    CHECK(f.rank(0) == 2 && f.rank(1) == 2);
  }
  std::printf("%s: %d failures\n", gpu ? "gpu" : "structure", fails);
  return fails == 0 ? 0 : 1;
}
