// TEST INFRASTRUCTURE — C entry points over the REFERENCE's own sources.
//
// oracle/Makefile target `ref` compiles /root/reference/proj/core/src/*.cpp
// (tensor, linalg, tucker, stitch, sst, query, baseline, io — unmodified, read
// in place) against the Eigen-API shim in oracle/eigen_shim/ (LAPACK
// dgeqrf/dormqr/dgesdd under HouseholderQR/BDCSVD) plus this file into
// oracle/_ref/libtucktree_ref.so. tests/test_ref_pin.py uses it to pin the
// restated oracle (oracle/tt_oracle.cpp) to the reference's own control flow:
// tucker_als (tucker.cpp:86-119), stitch (stitch.cpp:110-184),
// partial_hit_factors (stitch.cpp:36-47), the tree (sst.cpp:94-145) and
// range_query_detailed (query.cpp:49-69) on the same inputs.
// Only tests/ use it; nothing on the product path links it.
#include <cstdint>
#include <cstring>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "tucktree/linalg.hpp"
#include "tucktree/query.hpp"
#include "tucktree/sst.hpp"
#include "tucktree/stitch.hpp"
#include "tucktree/tucker.hpp"

using namespace tucktree;

namespace {
thread_local std::string g_err;
struct Res {
  TuckerFactors f;
  AlsTrace trace;
};
template <class F>
auto guard(F&& f, decltype(f()) bad) -> decltype(f()) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
  } catch (const std::out_of_range& e) {
    g_err = std::string("out_of_range: ") + e.what();
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
  }
  return bad;
}
Eigen::MatrixXd colmajor(const double* p, Index r, Index c) {
  Eigen::MatrixXd m(r, c);
  if (r * c) std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_factors_order(const Res* h) { return static_cast<int>(h->f.order()); }
int64_t ref_factors_dim(const Res* h, int m) { return h->f.dim(m); }
int64_t ref_factors_rank(const Res* h, int m) { return h->f.rank(m); }
const double* ref_factors_core(const Res* h) { return h->f.core.data().data(); }
const double* ref_factors_factor(const Res* h, int m) { return h->f.factors[static_cast<size_t>(m)].data(); }
int ref_factors_trace_len(const Res* h) { return static_cast<int>(h->trace.objective.size()); }
const double* ref_factors_trace(const Res* h) { return h->trace.objective.data(); }
int ref_factors_converged(const Res* h) { return h->trace.converged ? 1 : 0; }
void ref_factors_free(Res* h) { delete h; }

Res* ref_factors_new(int p, const int64_t* dims, const int64_t* ranks, const double* core, const double* const* fs) {
  return guard(
      [&]() -> Res* {
        auto* r = new Res;
        std::vector<Index> rk(ranks, ranks + p);
        size_t n = 1;
        for (int m = 0; m < p; ++m) n *= static_cast<size_t>(ranks[m]);
        r->f.core = DenseTensor(Shape(rk), std::vector<double>(core, core + n));
        for (int m = 0; m < p; ++m) r->f.factors.push_back(colmajor(fs[m], dims[m], ranks[m]));
        return r;
      },
      nullptr);
}

Res* ref_tucker_als(const double* x, int p, const int64_t* dims, const int64_t* ranks, int max_iters, double tol,
                    uint64_t seed) {
  return guard(
      [&]() -> Res* {
        Shape s(std::vector<Index>(dims, dims + p));
        DenseTensor t(s, std::vector<double>(x, x + s.element_count()));
        AlsConfig cfg;
        cfg.max_iters = max_iters;
        cfg.tol = tol;
        cfg.seed = seed;
        cfg.ranks.assign(ranks, ranks + p);
        auto* r = new Res;
        r->f = tucker_als(t, cfg, &r->trace);
        return r;
      },
      nullptr);
}

Res* ref_stitch(Res* const* parts, int n, const int64_t* ranks, int nr, int max_iters, double tol, uint64_t seed) {
  return guard(
      [&]() -> Res* {
        std::vector<TuckerFactors> ps;
        for (int i = 0; i < n; ++i) ps.push_back(parts[i]->f);
        AlsConfig cfg;
        cfg.max_iters = max_iters;
        cfg.tol = tol;
        cfg.seed = seed;
        std::vector<Index> rk(ranks, ranks + nr);
        auto* r = new Res;
        r->f = stitch(ps, rk, cfg, &r->trace);
        return r;
      },
      nullptr);
}

Res* ref_partial_hit(const Res* h, int64_t b, int64_t e) {
  return guard(
      [&]() -> Res* {
        auto* r = new Res;
        r->f = partial_hit_factors(h->f, b, e);
        return r;
      },
      nullptr);
}

int ref_llsv(const double* a, int64_t m, int64_t n, int64_t rank, double* out, int64_t* k) {
  return guard(
      [&]() -> int {
        const Eigen::MatrixXd u = leading_left_singular_vectors(colmajor(a, m, n), rank);
        *k = u.cols();
        std::memcpy(out, u.data(), sizeof(double) * static_cast<size_t>(u.size()));
        return 0;
      },
      1);
}

int ref_thin_qr(const double* a, int64_t m, int64_t n, double* q, double* r) {
  return guard(
      [&]() -> int {
        const QrResult qr = thin_qr(colmajor(a, m, n));
        std::memcpy(q, qr.q.data(), sizeof(double) * static_cast<size_t>(qr.q.size()));
        std::memcpy(r, qr.r.data(), sizeof(double) * static_cast<size_t>(qr.r.size()));
        return 0;
      },
      1);
}

// ---- tree -------------------------------------------------------------------
StreamSegmentTree* ref_tree_create(int nnt, const int64_t* nt, int nr, const int64_t* ranks, double theta,
                                   int max_iters, double tol, uint64_t seed) {
  return guard(
      [&]() -> StreamSegmentTree* {
        TreeConfig cfg;
        cfg.nontemporal.assign(nt, nt + nnt);
        cfg.ranks.assign(ranks, ranks + nr);
        cfg.theta = theta;
        cfg.als.max_iters = max_iters;
        cfg.als.tol = tol;
        cfg.als.seed = seed;
        return new StreamSegmentTree(cfg);
      },
      nullptr);
}
void ref_tree_destroy(StreamSegmentTree* t) { delete t; }

// Appends n slices (row-major, n x prod(nontemporal)) one at a time.
int ref_tree_append(StreamSegmentTree* t, const double* x, int64_t n) {
  return guard(
      [&]() -> int {
        const Shape s(t->config().nontemporal);
        const Index ss = s.element_count();
        for (int64_t i = 0; i < n; ++i)
          t->append(DenseTensor(s, std::vector<double>(x + i * ss, x + (i + 1) * ss)));
        return 0;
      },
      1);
}

int64_t ref_tree_stat(const StreamSegmentTree* t, int what) {
  switch (what) {
    case 0: return t->timespan();
    case 1: return t->height();
    case 2: return t->stitch_count();
    case 3: return t->last_append_node_touches();
    case 4: return t->node_count();
    case 5: return t->root();
    default: return -1;
  }
}

// info: begin, end, kind, left, right, has_decomposition
int ref_tree_node_info(const StreamSegmentTree* t, int64_t id, int64_t* info) {
  return guard(
      [&]() -> int {
        const Node& v = t->node(id);
        info[0] = v.begin;
        info[1] = v.end;
        info[2] = static_cast<int64_t>(v.kind);
        info[3] = v.left;
        info[4] = v.right;
        info[5] = v.decomposition.has_value();
        return 0;
      },
      1);
}

Res* ref_tree_node_factors(const StreamSegmentTree* t, int64_t id) {
  return guard(
      [&]() -> Res* {
        const Node& v = t->node(id);
        if (!v.decomposition) throw std::logic_error("node has no decomposition");
        auto* r = new Res;
        r->f = *v.decomposition;
        return r;
      },
      nullptr);
}

// out: (node, begin, end, flag) per hit
int ref_tree_recall(const StreamSegmentTree* t, int64_t ts, int64_t te, double theta, int64_t* out, int64_t cap,
                    int64_t* n) {
  return guard(
      [&]() -> int {
        const HitSet hs = recall(*t, ts, te, theta > 0.0 ? std::optional<double>(theta) : std::nullopt);
        *n = static_cast<int64_t>(hs.size());
        for (size_t i = 0; i < hs.size() && static_cast<int64_t>(i) < cap; ++i) {
          out[4 * i] = hs[i].node;
          out[4 * i + 1] = hs[i].begin;
          out[4 * i + 2] = hs[i].end;
          out[4 * i + 3] = static_cast<int64_t>(hs[i].flag);
        }
        return 0;
      },
      1);
}

Res* ref_tree_query(const StreamSegmentTree* t, int64_t ts, int64_t te, double theta) {
  return guard(
      [&]() -> Res* {
        auto* r = new Res;
        QueryResult q = range_query_detailed(*t, ts, te, theta > 0.0 ? std::optional<double>(theta) : std::nullopt,
                                             &r->trace);
        r->f = std::move(q.factors);
        return r;
      },
      nullptr);
}

int ref_tree_validate(const StreamSegmentTree* t, char* buf, int64_t cap) {
  const std::vector<std::string> v = t->validate();
  std::string all;
  for (const auto& s : v) all += s + "\n";
  if (buf && cap > 0) {
    std::strncpy(buf, all.c_str(), static_cast<size_t>(cap - 1));
    buf[cap - 1] = '\0';
  }
  return static_cast<int>(v.size());
}

}  // extern "C"
