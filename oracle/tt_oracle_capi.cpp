// TEST INFRASTRUCTURE ONLY — flat C API over the oracle for the Python tests
// (tests/, oracle/oracle.py) and the CPU baseline arm of bench.py.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "tt_oracle.hpp"

using namespace tto;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 1;
  if (dynamic_cast<const std::logic_error*>(&e)) return 2;
  return 3;
}
std::vector<Index> vec(const std::int64_t* p, int n) { return std::vector<Index>(p, p + n); }
Mat mat_from(const double* a, Index r, Index c) {
  Mat m(r, c);
  std::memcpy(m.data(), a, sizeof(double) * static_cast<std::size_t>(r * c));
  return m;
}
}  // namespace

struct orc_factors {
  Factors f;
  AlsTrace trace;
};
struct orc_tree {
  Tree t;
};

namespace {
struct OWriter {
  std::FILE* f;
  explicit OWriter(const char* p) : f(std::fopen(p, "wb")) {
    if (!f) throw std::runtime_error(std::string("cannot open ") + p + " for writing");
  }
  ~OWriter() {
    if (f) std::fclose(f);
  }
  void bytes(const void* b, std::size_t n) {
    if (n && std::fwrite(b, 1, n, f) != n) throw std::runtime_error("write failed");
  }
  template <class T>
  void le(T v) {
    bytes(&v, sizeof(T));
  }
};
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) { set_blas_threads(n); }

std::uint64_t orc_mt19937_64_nth(std::uint64_t seed, std::int64_t n) {
  std::mt19937_64 rng(seed);
  std::uint64_t v = 0;
  for (std::int64_t i = 0; i < n; ++i) v = rng();
  return v;
}

// ---- factors handles ----
int orc_factors_order(const orc_factors* h) { return static_cast<int>(h->f.order()); }
std::int64_t orc_factors_dim(const orc_factors* h, int m) { return h->f.dim(m); }
std::int64_t orc_factors_rank(const orc_factors* h, int m) { return h->f.rank(m); }
const double* orc_factors_core(const orc_factors* h) { return h->f.core.v.data(); }
const double* orc_factors_factor(const orc_factors* h, int m) { return h->f.f[static_cast<std::size_t>(m)].data(); }
int orc_factors_trace_len(const orc_factors* h) { return static_cast<int>(h->trace.objective.size()); }
const double* orc_factors_trace(const orc_factors* h) { return h->trace.objective.data(); }
int orc_factors_converged(const orc_factors* h) { return h->trace.converged ? 1 : 0; }
void orc_factors_free(orc_factors* h) { delete h; }

orc_factors* orc_factors_new(int p, const std::int64_t* dims, const std::int64_t* ranks, const double* core,
                             const double* const* factors) {
  try {
    auto* h = new orc_factors;
    h->f.core = Tensor(vec(ranks, p), std::vector<double>(core, core + element_count(vec(ranks, p))));
    for (int m = 0; m < p; ++m) h->f.f.push_back(mat_from(factors[m], dims[m], ranks[m]));
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

orc_factors* orc_tucker_als(const double* x, int p, const std::int64_t* dims, const std::int64_t* ranks,
                            int max_iters, double tol, std::uint64_t seed) {
  try {
    Tensor t(vec(dims, p), std::vector<double>(x, x + element_count(vec(dims, p))));
    AlsConfig cfg;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    cfg.seed = seed;
    cfg.ranks = vec(ranks, p);
    auto* h = new orc_factors;
    h->f = tucker_als(t, cfg, &h->trace);
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

orc_factors* orc_stitch(const orc_factors* const* parts, int nparts, const std::int64_t* ranks, int nranks,
                        int max_iters, double tol, std::uint64_t seed) {
  try {
    std::vector<Factors> ps;
    for (int i = 0; i < nparts; ++i) ps.push_back(parts[i]->f);
    AlsConfig cfg;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    cfg.seed = seed;
    auto* h = new orc_factors;
    h->f = stitch(ps, vec(ranks, nranks), cfg, &h->trace);
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

orc_factors* orc_partial_hit(const orc_factors* stored, std::int64_t b, std::int64_t e) {
  try {
    auto* h = new orc_factors;
    h->f = partial_hit_factors(stored->f, b, e);
    return h;
  } catch (const std::exception& ex) {
    fail(ex);
    return nullptr;
  }
}

// out: dims[mode] x prod(other cols); caller sized. factors: p col-major mats.
int orc_stitch_unfolding(const orc_factors* const* parts, int nparts, int mode, const double* const* factors,
                         const std::int64_t* frows, const std::int64_t* fcols, double* out) {
  try {
    std::vector<Factors> ps;
    for (int i = 0; i < nparts; ++i) ps.push_back(parts[i]->f);
    const int p = static_cast<int>(ps[0].order());
    std::vector<Mat> fs;
    for (int m = 0; m < p; ++m) fs.push_back(mat_from(factors[m], frows[m], fcols[m]));
    const Mat z = mode == 0 ? stitch_temporal_unfolding(ps, fs) : stitch_nontemporal_unfolding(ps, mode, fs);
    std::memcpy(out, z.data(), sizeof(double) * z.v.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_llsv(const double* a, std::int64_t m, std::int64_t n, std::int64_t rank, double* out, std::int64_t* k) {
  try {
    const Mat u = leading_left_singular_vectors(mat_from(a, m, n), rank);
    std::memcpy(out, u.data(), sizeof(double) * u.v.size());
    *k = u.cols;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_thin_qr(const double* a, std::int64_t m, std::int64_t n, double* q, double* r) {
  try {
    const QrResult qr = thin_qr(mat_from(a, m, n));
    std::memcpy(q, qr.q.data(), sizeof(double) * qr.q.v.size());
    std::memcpy(r, qr.r.data(), sizeof(double) * qr.r.v.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Sequence of random_orthonormal draws from one rng(seed): rows[i] x cols[i].
int orc_random_orthonormal_seq(std::uint64_t seed, int count, const std::int64_t* rows, const std::int64_t* cols,
                               double* const* outs) {
  try {
    std::mt19937_64 rng(seed);
    for (int i = 0; i < count; ++i) {
      const Mat q = random_orthonormal(rows[i], cols[i], rng);
      std::memcpy(outs[i], q.data(), sizeof(double) * q.v.size());
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_generate_synthetic(int p, const std::int64_t* shape, const std::int64_t* true_ranks, double noise,
                           std::uint64_t seed, double* out) {
  try {
    SynthSpec s;
    s.shape = vec(shape, p);
    s.true_ranks = vec(true_ranks, p);
    s.noise = noise;
    s.seed = seed;
    const Tensor t = generate_synthetic(s);
    std::memcpy(out, t.v.data(), sizeof(double) * t.v.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_reconstruct(const orc_factors* f, double* out) {
  try {
    const Tensor t = reconstruct(f->f);
    std::memcpy(out, t.v.data(), sizeof(double) * t.v.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

std::int64_t orc_default_block_size(std::int64_t t) {
  try {
    return default_block_size(t);
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

// ---- tree ----
orc_tree* orc_tree_create(int n_nontemporal, const std::int64_t* nontemporal, int n_ranks,
                          const std::int64_t* ranks, double theta, int max_iters, double tol, std::uint64_t seed,
                          std::int64_t leaf_block) {
  try {
    TreeConfig c;
    c.nontemporal = vec(nontemporal, n_nontemporal);
    c.ranks = vec(ranks, n_ranks);
    c.theta = theta;
    c.als.max_iters = max_iters;
    c.als.tol = tol;
    c.als.seed = seed;
    c.leaf_block = leaf_block;
    return new orc_tree{Tree(std::move(c))};
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void orc_tree_destroy(orc_tree* t) { delete t; }

int orc_tree_append(orc_tree* t, const double* slices, std::int64_t n) {
  try {
    const Index ss = element_count(t->t.config().nontemporal);
    for (std::int64_t i = 0; i < n; ++i) t->t.append(slices + i * ss);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

std::int64_t orc_tree_stat(const orc_tree* t, int what) {
  switch (what) {
    case 0: return t->t.timespan();
    case 1: return t->t.height();
    case 2: return t->t.stitch_count();
    case 3: return t->t.last_append_node_touches();
    case 4: return static_cast<std::int64_t>(t->t.nodes().size());
    case 5: return t->t.root();
    case 6: return t->t.leaves();
    default: return -1;
  }
}

// info: begin, end, kind, left, right, has_dec
int orc_tree_node_info(const orc_tree* t, std::int64_t id, std::int64_t* info) {
  try {
    const Node& v = t->t.node(id);
    info[0] = v.begin;
    info[1] = v.end;
    info[2] = static_cast<std::int64_t>(v.kind);
    info[3] = v.left;
    info[4] = v.right;
    info[5] = v.dec ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

orc_factors* orc_tree_node_factors(const orc_tree* t, std::int64_t id) {
  try {
    const Node& v = t->t.node(id);
    if (!v.dec) throw std::logic_error("node has no decomposition");
    auto* h = new orc_factors;
    h->f = *v.dec;
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

std::int64_t orc_tree_last_redecomposed(const orc_tree* t, std::int64_t* out, std::int64_t cap) {
  const auto& v = t->t.last_redecomposed();
  for (std::size_t i = 0; i < v.size() && static_cast<std::int64_t>(i) < cap; ++i) out[i] = v[i];
  return static_cast<std::int64_t>(v.size());
}

// hits out: [node, begin, end, flag] * n
int orc_tree_recall(const orc_tree* t, std::int64_t ts, std::int64_t te, double theta, std::int64_t* out,
                    std::int64_t cap, std::int64_t* n) {
  try {
    const HitSet h = recall(t->t, ts, te, theta > 0 ? std::optional<double>(theta) : std::nullopt);
    *n = static_cast<std::int64_t>(h.size());
    for (std::size_t i = 0; i < h.size() && static_cast<std::int64_t>(i) < cap; ++i) {
      out[4 * i] = h[i].node;
      out[4 * i + 1] = h[i].begin;
      out[4 * i + 2] = h[i].end;
      out[4 * i + 3] = static_cast<std::int64_t>(h[i].flag);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

orc_factors* orc_tree_query(const orc_tree* t, std::int64_t ts, std::int64_t te, double theta) {
  try {
    auto* h = new orc_factors;
    h->f = range_query_detailed(t->t, ts, te, theta > 0 ? std::optional<double>(theta) : std::nullopt, &h->trace).factors;
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// CPU-baseline batch: queries split over nthreads std::threads (the
// reference's read-only concurrency contract, sst.hpp:52-53); BLAS pinned to
// one thread per worker. Writes sum(core^2) per query as a checksum.
int orc_tree_query_batch(const orc_tree* t, const std::int64_t* ranges, std::int64_t n, double theta, int nthreads,
                         double* checksums) {
  set_blas_threads(1);
  std::atomic<std::int64_t> next{0};
  std::atomic<int> err{0};
  auto worker = [&]() {
    for (;;) {
      const std::int64_t i = next.fetch_add(1);
      if (i >= n) return;
      try {
        const QueryResult r = range_query_detailed(t->t, ranges[2 * i], ranges[2 * i + 1],
                                                   theta > 0 ? std::optional<double>(theta) : std::nullopt);
        checksums[i] = squared_norm(r.factors.core);
      } catch (const std::exception& e) {
        err = fail(e);
      }
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < std::max(1, nthreads); ++i) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  return err.load();
}

int orc_tree_validate(const orc_tree* t, char* buf, std::int64_t cap) {
  const auto v = t->t.validate();
  std::string all;
  for (const auto& s : v) all += s + "\n";
  if (buf != nullptr && cap > 0) {
    std::strncpy(buf, all.c_str(), static_cast<std::size_t>(cap - 1));
    buf[cap - 1] = '\0';
  }
  return static_cast<int>(v.size());
}

// Raw tail slices (row-major), count = timespan - leaves*B.
const double* orc_tree_tail(const orc_tree* t) { return t->t.tail().v.data(); }


// ---- persistence: restatement of write_tree / write_tensor (io.cpp:87-101,
// 124-133, 165-188), little-endian field by field; trees with a leaf block
// B > 1 or a raw tail append the engine's "TTB1" extension (u16 version,
// u64 B, u64 tail slices, row-major tail) after the node table.

int orc_tree_save(const orc_tree* h, const char* path) {
  try {
    const Tree& t = h->t;
    const TreeConfig& cfg = t.config();
    OWriter w(path);
    w.bytes("SST1", 4);
    w.le<std::uint16_t>(1);
    w.le<std::uint64_t>(static_cast<std::uint64_t>(t.timespan()));
    w.le<std::uint8_t>(static_cast<std::uint8_t>(cfg.nontemporal.size() + 1));
    for (Index d : cfg.nontemporal) w.le<std::uint64_t>(static_cast<std::uint64_t>(d));
    for (Index r : cfg.ranks) w.le<std::uint64_t>(static_cast<std::uint64_t>(r));
    w.le<double>(cfg.theta);
    w.le<std::uint32_t>(static_cast<std::uint32_t>(cfg.als.max_iters));
    w.le<double>(cfg.als.tol);
    w.le<std::uint64_t>(cfg.als.seed);
    w.le<std::uint64_t>(static_cast<std::uint64_t>(t.stitch_count()));
    w.le<std::uint64_t>(static_cast<std::uint64_t>(t.root()));
    w.le<std::uint64_t>(static_cast<std::uint64_t>(t.nodes().size()));
    for (const Node& v : t.nodes()) {
      w.le<std::uint64_t>(static_cast<std::uint64_t>(v.id));
      w.le<std::uint64_t>(static_cast<std::uint64_t>(v.begin));
      w.le<std::uint64_t>(static_cast<std::uint64_t>(v.end));
      w.le<std::uint8_t>(static_cast<std::uint8_t>(v.kind));
      w.le<std::uint64_t>(static_cast<std::uint64_t>(v.left));
      w.le<std::uint64_t>(static_cast<std::uint64_t>(v.right));
      w.le<std::uint8_t>(v.dec ? 1 : 0);
      if (!v.dec) continue;
      const Factors& f = *v.dec;
      w.le<std::uint8_t>(static_cast<std::uint8_t>(f.order()));
      for (Index n = 0; n < f.order(); ++n) w.le<std::uint64_t>(static_cast<std::uint64_t>(f.core.dim(n)));
      w.bytes(f.core.v.data(), f.core.v.size() * sizeof(double));
      for (const Mat& u : f.f) {
        w.le<std::uint64_t>(static_cast<std::uint64_t>(u.rows));
        w.le<std::uint64_t>(static_cast<std::uint64_t>(u.cols));
        for (Index i = 0; i < u.rows; ++i)
          for (Index j = 0; j < u.cols; ++j) w.le<double>(u(i, j));
      }
    }
    const Index tail = t.timespan() - t.leaves() * cfg.leaf_block;
    if (cfg.leaf_block > 1 || tail > 0) {
      w.bytes("TTB1", 4);
      w.le<std::uint16_t>(1);
      w.le<std::uint64_t>(static_cast<std::uint64_t>(cfg.leaf_block));
      w.le<std::uint64_t>(static_cast<std::uint64_t>(tail));
      w.bytes(t.tail().v.data(), t.tail().v.size() * sizeof(double));  // exactly `tail` slices
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_tensor_write(const char* path, int p, const std::int64_t* dims, const double* data) {
  try {
    OWriter w(path);
    w.bytes("TTS1", 4);
    w.le<std::uint16_t>(1);
    w.le<std::uint8_t>(static_cast<std::uint8_t>(p));
    std::size_t n = 1;
    for (int m = 0; m < p; ++m) {
      w.le<std::uint64_t>(static_cast<std::uint64_t>(dims[m]));
      n *= static_cast<std::size_t>(dims[m]);
    }
    w.bytes(data, n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
