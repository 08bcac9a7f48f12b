// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
// See tt_oracle.hpp for the scope rules. Every function cites the reference
// function (file:line under /root/reference/proj/core/src) it restates.
#include "tt_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <stdexcept>

// OpenBLAS (ILP64, symbol prefix "scipy_", suffix "64_") bundled with numpy.
extern "C" {
void scipy_dgeqrf_64_(const std::int64_t* m, const std::int64_t* n, double* a,
                      const std::int64_t* lda, double* tau, double* work,
                      const std::int64_t* lwork, std::int64_t* info);
void scipy_dorgqr_64_(const std::int64_t* m, const std::int64_t* n, const std::int64_t* k,
                      double* a, const std::int64_t* lda, const double* tau, double* work,
                      const std::int64_t* lwork, std::int64_t* info);
void scipy_dgesdd_64_(const char* jobz, const std::int64_t* m, const std::int64_t* n, double* a,
                      const std::int64_t* lda, double* s, double* u, const std::int64_t* ldu,
                      double* vt, const std::int64_t* ldvt, double* work,
                      const std::int64_t* lwork, std::int64_t* iwork, std::int64_t* info,
                      std::size_t jobz_len);
void scipy_dgemm_64_(const char* ta, const char* tb, const std::int64_t* m,
                     const std::int64_t* n, const std::int64_t* k, const double* alpha,
                     const double* a, const std::int64_t* lda, const double* b,
                     const std::int64_t* ldb, const double* beta, double* c,
                     const std::int64_t* ldc, std::size_t, std::size_t);
void scipy_openblas_set_num_threads64_(int);
}

namespace tto {

void set_blas_threads(int n) { scipy_openblas_set_num_threads64_(n); }

namespace {

[[noreturn]] void bad(const std::string& msg) { throw std::invalid_argument(msg); }

Index outer_extent(std::span<const Index> dims, Index mode) {
  Index n = 1;
  for (Index m = 0; m < mode; ++m) n *= dims[static_cast<std::size_t>(m)];
  return n;
}
Index inner_extent(std::span<const Index> dims, Index mode) {
  Index n = 1;
  for (Index m = mode + 1; m < static_cast<Index>(dims.size()); ++m)
    n *= dims[static_cast<std::size_t>(m)];
  return n;
}

// C(MxN) = op(A) * op(B), all column-major with leading dims; dgemm for large
// products, plain loops for tiny ones (Eigen inlines those; a BLAS call per
// 4x6 product would misrepresent the reference's CPU cost).
void gemm_cm(bool ta, bool tb, Index m, Index n, Index k, const double* a, Index lda,
             const double* b, Index ldb, double* c, Index ldc, double beta = 0.0) {
  if (m == 0 || n == 0) return;
  if (m * n * k >= 32768) {
    const double alpha = 1.0;
    const char cta = ta ? 'T' : 'N', ctb = tb ? 'T' : 'N';
    scipy_dgemm_64_(&cta, &ctb, &m, &n, &k, &alpha, a, &lda, b, &ldb, &beta, c, &ldc, 1, 1);
    return;
  }
  for (Index j = 0; j < n; ++j) {
    for (Index i = 0; i < m; ++i) {
      double s = 0.0;
      for (Index l = 0; l < k; ++l) {
        const double av = ta ? a[l + i * lda] : a[i + l * lda];
        const double bv = tb ? b[j + l * ldb] : b[l + j * ldb];
        s += av * bv;
      }
      c[i + j * ldc] = (beta == 0.0 ? 0.0 : beta * c[i + j * ldc]) + s;
    }
  }
}

// sign rule of linalg.cpp:15-31: each column's first max-|.| entry (strict >
// scan) made nonnegative; rows_to_fix follows the column flips.
void apply_sign_convention(Mat& q, Mat* rows_to_fix) {
  for (Index j = 0; j < q.cols; ++j) {
    Index pivot = 0;
    double best = -1.0;
    for (Index i = 0; i < q.rows; ++i) {
      const double mag = std::abs(q(i, j));
      if (mag > best) {
        best = mag;
        pivot = i;
      }
    }
    if (q.rows > 0 && q(pivot, j) < 0.0) {
      for (Index i = 0; i < q.rows; ++i) q(i, j) = -q(i, j);
      if (rows_to_fix != nullptr)
        for (Index c = 0; c < rows_to_fix->cols; ++c) (*rows_to_fix)(j, c) = -(*rows_to_fix)(j, c);
    }
  }
}

// Householder QR via LAPACK; returns the factored matrix + tau.
void householder(Mat& a, std::vector<double>& tau) {
  const Index m = a.rows, n = a.cols, k = std::min(m, n);
  tau.assign(static_cast<std::size_t>(std::max<Index>(k, 1)), 0.0);
  if (k == 0) return;
  Index lwork = -1, info = 0, lda = std::max<Index>(m, 1);
  double wq = 0.0;
  scipy_dgeqrf_64_(&m, &n, a.data(), &lda, tau.data(), &wq, &lwork, &info);
  lwork = std::max<Index>(static_cast<Index>(wq), n);
  std::vector<double> work(static_cast<std::size_t>(lwork));
  scipy_dgeqrf_64_(&m, &n, a.data(), &lda, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("dgeqrf failed");
}

// Explicit thin Q (m x kq) from the factored matrix (first kq reflectors).
Mat form_q(const Mat& fact, const std::vector<double>& tau, Index kq) {
  const Index m = fact.rows;
  Mat q(m, kq);
  if (kq == 0) return q;
  for (Index j = 0; j < kq; ++j)
    for (Index i = 0; i < m; ++i) q(i, j) = fact(i, j);
  Index lwork = -1, info = 0, lda = std::max<Index>(m, 1);
  double wq = 0.0;
  scipy_dorgqr_64_(&m, &kq, &kq, q.data(), &lda, tau.data(), &wq, &lwork, &info);
  lwork = std::max<Index>(static_cast<Index>(wq), kq);
  std::vector<double> work(static_cast<std::size_t>(lwork));
  scipy_dorgqr_64_(&m, &kq, &kq, q.data(), &lda, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("dorgqr failed");
  return q;
}

// Thin SVD left vectors (m x min(m,n)), singular values descending (dgesdd,
// the divide-and-conquer family of Eigen::BDCSVD).
Mat svd_left(const Mat& a_in) {
  Mat a = a_in;
  const Index m = a.rows, n = a.cols, k = std::min(m, n);
  Mat u(m, k);
  std::vector<double> s(static_cast<std::size_t>(std::max<Index>(k, 1)));
  std::vector<double> vt(static_cast<std::size_t>(std::max<Index>(k * n, 1)));
  std::vector<std::int64_t> iwork(static_cast<std::size_t>(8 * std::max<Index>(k, 1)));
  Index lda = std::max<Index>(m, 1), ldu = std::max<Index>(m, 1), ldvt = std::max<Index>(k, 1);
  Index lwork = -1, info = 0;
  double wq = 0.0;
  const char jobz = 'S';
  scipy_dgesdd_64_(&jobz, &m, &n, a.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt,
                   &wq, &lwork, iwork.data(), &info, 1);
  lwork = std::max<Index>(static_cast<Index>(wq), 1);
  std::vector<double> work(static_cast<std::size_t>(lwork));
  scipy_dgesdd_64_(&jobz, &m, &n, a.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt,
                   work.data(), &lwork, iwork.data(), &info, 1);
  if (info != 0) throw std::runtime_error("dgesdd failed");
  return u;
}

Mat left_cols(const Mat& a, Index k) {
  Mat out(a.rows, k);
  std::copy(a.v.begin(), a.v.begin() + a.rows * k, out.v.begin());
  return out;
}

}  // namespace

// ---------------------------------------------------------------------------
Mat Mat::identity(Index n) {
  Mat m(n, n);
  for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}

Index element_count(std::span<const Index> dims) {
  Index c = 1;
  for (Index d : dims) {
    if (d < 1) bad("Shape: all dims must be >= 1");
    c *= d;
  }
  return c;
}

Tensor::Tensor(std::vector<Index> d) : dims(std::move(d)) {
  if (dims.empty()) bad("Shape: no dims given");
  v.assign(static_cast<std::size_t>(element_count(dims)), 0.0);
}
Tensor::Tensor(std::vector<Index> d, std::vector<double> data) : dims(std::move(d)), v(std::move(data)) {
  if (dims.empty()) bad("Shape: no dims given");
  if (static_cast<Index>(v.size()) != element_count(dims)) bad("DenseTensor: data length mismatch");
}

Mat transpose(const Mat& a) {
  Mat t(a.cols, a.rows);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i) t(j, i) = a(i, j);
  return t;
}

Mat matmul(const Mat& a, const Mat& b) {
  if (a.cols != b.rows) bad("matmul: inner dims");
  Mat c(a.rows, b.cols);
  gemm_cm(false, false, a.rows, b.cols, a.cols, a.data(), std::max<Index>(a.rows, 1), b.data(),
          std::max<Index>(b.rows, 1), c.data(), std::max<Index>(c.rows, 1));
  return c;
}

// tensor.cpp:90-102 — rows D_n, columns = other modes in order, last fastest.
Mat matricize(const Tensor& x, Index mode) {
  if (mode < 0 || mode >= x.order()) bad("invalid mode index");
  const Index rows = x.dim(mode), outer = outer_extent(x.dims, mode), inner = inner_extent(x.dims, mode);
  Mat m(rows, outer * inner);
  for (Index o = 0; o < outer; ++o)
    for (Index r = 0; r < rows; ++r)
      for (Index t = 0; t < inner; ++t) m(r, o * inner + t) = x.v[static_cast<std::size_t>((o * rows + r) * inner + t)];
  return m;
}

// tensor.cpp:104-119
Tensor from_matricization(const Mat& m, std::vector<Index> dims, Index mode) {
  if (mode < 0 || mode >= static_cast<Index>(dims.size())) bad("invalid mode index");
  const Index rows = dims[static_cast<std::size_t>(mode)], outer = outer_extent(dims, mode),
              inner = inner_extent(dims, mode);
  if (m.rows != rows || m.cols != outer * inner) bad("from_matricization: matrix does not match shape");
  Tensor out(std::move(dims));
  for (Index o = 0; o < outer; ++o)
    for (Index r = 0; r < rows; ++r)
      for (Index t = 0; t < inner; ++t) out.v[static_cast<std::size_t>((o * rows + r) * inner + t)] = m(r, o * inner + t);
  return out;
}

// tensor.cpp:121-143 — loop over the outer extent of row-major GEMMs
// res(rows_out x inner) = u * in(rows_in x inner).
Tensor mode_product(const Tensor& x, const Mat& u, Index mode) {
  if (mode < 0 || mode >= x.order()) bad("invalid mode index");
  if (u.cols != x.dim(mode)) bad("mode_product: matrix cols do not match mode extent");
  std::vector<Index> dims = x.dims;
  dims[static_cast<std::size_t>(mode)] = u.rows;
  Tensor out(dims);
  const Index outer = outer_extent(x.dims, mode), inner = inner_extent(x.dims, mode);
  const Index rows_in = x.dim(mode), rows_out = u.rows;
  for (Index o = 0; o < outer; ++o) {
    // Row-major (rows x inner) == column-major (inner x rows): res^T = in^T u^T.
    const double* in = x.v.data() + o * rows_in * inner;
    double* res = out.v.data() + o * rows_out * inner;
    gemm_cm(false, true, inner, rows_out, rows_in, in, std::max<Index>(inner, 1), u.data(),
            std::max<Index>(u.rows, 1), res, std::max<Index>(inner, 1));
  }
  return out;
}

double squared_norm(const Tensor& x) {  // tensor.cpp:145-147
  double s = 0.0;
  for (double v : x.v) s += v * v;
  return s;
}

Tensor slice_temporal(const Tensor& x, Index begin, Index end) {  // tensor.cpp:177-187
  if (begin < 0 || begin >= end || end > x.dim(0)) bad("slice_temporal: invalid range");
  const Index inner = inner_extent(x.dims, 0);
  std::vector<Index> dims = x.dims;
  dims[0] = end - begin;
  return Tensor(dims, std::vector<double>(x.v.begin() + begin * inner, x.v.begin() + end * inner));
}

Tensor concat_temporal(std::span<const Tensor> parts) {  // tensor.cpp:151-175
  if (parts.empty()) bad("concat_temporal: no parts");
  Index total = 0;
  for (const Tensor& p : parts) {
    if (p.order() != parts[0].order()) bad("concat_temporal: order mismatch");
    for (Index m = 1; m < p.order(); ++m)
      if (p.dim(m) != parts[0].dim(m)) bad("concat_temporal: non-temporal shape mismatch");
    total += p.dim(0);
  }
  std::vector<Index> dims = parts[0].dims;
  dims[0] = total;
  std::vector<double> data;
  data.reserve(static_cast<std::size_t>(element_count(dims)));
  for (const Tensor& p : parts) data.insert(data.end(), p.v.begin(), p.v.end());
  return Tensor(dims, std::move(data));
}

// ---------------------------------------------------------------------------
// linalg.cpp:35-43 — thin Householder QR, q: m x min(m,k), r: min(m,k) x k.
QrResult thin_qr(const Mat& a) {
  const Index k = std::min(a.rows, a.cols);
  Mat fact = a;
  std::vector<double> tau;
  householder(fact, tau);
  QrResult out;
  out.q = form_q(fact, tau, k);
  out.r = Mat(k, a.cols);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i <= std::min(j, k - 1); ++i) out.r(i, j) = fact(i, j);
  apply_sign_convention(out.q, &out.r);
  return out;
}

// linalg.cpp:45-64 — tall branch rows > 2*cols: QR, then SVD of R.
Mat leading_left_singular_vectors(const Mat& a, Index rank) {
  if (rank < 1) bad("leading_left_singular_vectors: rank must be >= 1");
  const Index k = std::min({rank, a.rows, a.cols});
  Mat u;
  if (a.rows > 2 * a.cols) {
    Mat fact = a;
    std::vector<double> tau;
    householder(fact, tau);
    const Mat q = form_q(fact, tau, a.cols);
    Mat r(a.cols, a.cols);
    for (Index j = 0; j < a.cols; ++j)
      for (Index i = 0; i <= j; ++i) r(i, j) = fact(i, j);
    const Mat ur = left_cols(svd_left(r), k);
    u = matmul(q, ur);
  } else {
    u = left_cols(svd_left(a), k);
  }
  apply_sign_convention(u, nullptr);
  return u;
}

// linalg.cpp:81-89 — fresh normal_distribution per call, row-major draws.
Mat random_orthonormal(Index rows, Index cols, std::mt19937_64& rng) {
  if (rows < cols) bad("random_orthonormal: rows < cols");
  std::normal_distribution<double> normal(0.0, 1.0);
  Mat g(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) g(i, j) = normal(rng);
  return thin_qr(g).q;
}

double max_orthonormality_defect(const Mat& u) {  // linalg.cpp:76-79
  Mat g(u.cols, u.cols);
  gemm_cm(true, false, u.cols, u.cols, u.rows, u.data(), std::max<Index>(u.rows, 1), u.data(),
          std::max<Index>(u.rows, 1), g.data(), std::max<Index>(u.cols, 1));
  double worst = 0.0;
  for (Index j = 0; j < u.cols; ++j)
    for (Index i = 0; i < u.cols; ++i) worst = std::max(worst, std::abs(g(i, j) - (i == j ? 1.0 : 0.0)));
  return worst;
}

Mat kronecker(const Mat& a, const Mat& b) {  // linalg.cpp:66-74
  Mat out(a.rows * b.rows, a.cols * b.cols);
  for (Index i = 0; i < a.rows; ++i)
    for (Index j = 0; j < a.cols; ++j)
      for (Index bi = 0; bi < b.rows; ++bi)
        for (Index bj = 0; bj < b.cols; ++bj) out(i * b.rows + bi, j * b.cols + bj) = a(i, j) * b(bi, bj);
  return out;
}

// ---------------------------------------------------------------------------
// tucker.cpp:41-52
std::vector<Index> clamp_ranks(std::span<const Index> requested, std::span<const Index> dims) {
  if (requested.size() != dims.size()) bad("clamp_ranks: one rank per mode required");
  std::vector<Index> r(requested.begin(), requested.end());
  for (std::size_t n = 0; n < r.size(); ++n) {
    if (r[n] < 1) bad("clamp_ranks: ranks must be >= 1");
    r[n] = std::min(r[n], dims[n]);
  }
  return r;
}

namespace {
void check_factor_shapes(const Tensor& x, const Factors& f) {  // tucker.cpp:14-24
  if (f.order() != x.order()) bad("factor count does not match tensor order");
  for (Index n = 0; n < x.order(); ++n)
    if (f.f[static_cast<std::size_t>(n)].rows != x.dim(n)) bad("factor rows do not match tensor extent");
}
}  // namespace

// tucker.cpp:54-65 — project by every other factor (ascending), then llsv
// with the current column count (ranks can only shrink).
Mat update_factor(const Tensor& x, const Factors& current, Index mode) {
  check_factor_shapes(x, current);
  Tensor projected = x;
  for (Index m = 0; m < x.order(); ++m) {
    if (m == mode) continue;
    projected = mode_product(projected, transpose(current.f[static_cast<std::size_t>(m)]), m);
  }
  return leading_left_singular_vectors(matricize(projected, mode), current.rank(mode));
}

Tensor core_of(const Tensor& x, std::span<const Mat> factors) {  // tucker.cpp:67-76
  if (static_cast<Index>(factors.size()) != x.order()) bad("core_of: one factor per mode required");
  Tensor acc = x;
  for (Index n = 0; n < x.order(); ++n) acc = mode_product(acc, transpose(factors[static_cast<std::size_t>(n)]), n);
  return acc;
}

Tensor reconstruct(const Factors& f) {  // tucker.cpp:78-84
  Tensor acc = f.core;
  for (Index n = 0; n < f.order(); ++n) acc = mode_product(acc, f.f[static_cast<std::size_t>(n)], n);
  return acc;
}

// tucker.cpp:86-119
Factors tucker_als(const Tensor& x, const AlsConfig& cfg, AlsTrace* trace) {
  if (cfg.max_iters < 1) bad("tucker_als: max_iters must be >= 1");
  if (cfg.tol <= 0.0) bad("tucker_als: tol must be > 0");
  const std::vector<Index> ranks = clamp_ranks(cfg.ranks, x.dims);
  Factors f;
  {  // init_factors, tucker.cpp:26-37: every mode, including mode 0.
    std::mt19937_64 rng(cfg.seed);
    for (Index n = 0; n < x.order(); ++n)
      f.f.push_back(random_orthonormal(x.dim(n), ranks[static_cast<std::size_t>(n)], rng));
  }
  f.core = Tensor(ranks);
  if (trace != nullptr) *trace = AlsTrace{};
  const double norm_sq = squared_norm(x);
  if (norm_sq == 0.0) {
    if (trace != nullptr) trace->converged = true;
    return f;
  }
  const double norm = std::sqrt(norm_sq);
  double prev_fit = std::numeric_limits<double>::quiet_NaN();
  for (int sweep = 0; sweep < cfg.max_iters; ++sweep) {
    for (Index n = 0; n < x.order(); ++n) f.f[static_cast<std::size_t>(n)] = update_factor(x, f, n);
    f.core = core_of(x, f.f);
    const double residual_sq = std::max(0.0, norm_sq - squared_norm(f.core));
    if (trace != nullptr) trace->objective.push_back(residual_sq);
    const double fit = 1.0 - std::sqrt(residual_sq) / norm;
    if (sweep > 0 && std::abs(fit - prev_fit) < cfg.tol) {
      if (trace != nullptr) trace->converged = true;
      break;
    }
    prev_fit = fit;
  }
  return f;
}

// tucker.cpp:121-143
double relative_error(const Tensor& x, const Factors& candidate, const Factors& reference) {
  const auto residual = [&x](const Factors& f) {
    const Tensor rec = reconstruct(f);
    if (rec.dims != x.dims) bad("relative_error: reconstruction shape mismatch");
    double sq = 0.0;
    for (std::size_t i = 0; i < x.v.size(); ++i) {
      const double d = x.v[i] - rec.v[i];
      sq += d * d;
    }
    return std::sqrt(sq);
  };
  const double cand = residual(candidate), ref = residual(reference);
  if (ref == 0.0) return cand == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
  return cand / ref - 1.0;
}

// ---------------------------------------------------------------------------
namespace {
void check_parts(std::span<const Factors> parts) {  // stitch.cpp:14-26
  if (parts.empty()) bad("stitch: at least one part required");
  const Index p = parts[0].order();
  if (p < 1) bad("stitch: parts must have at least one mode");
  for (const Factors& part : parts) {
    if (part.order() != p) bad("stitch: part order mismatch");
    for (Index m = 1; m < p; ++m)
      if (part.dim(m) != parts[0].dim(m)) bad("stitch: non-temporal shape mismatch across parts");
  }
}
Index total_temporal(std::span<const Factors> parts) {
  Index t = 0;
  for (const Factors& p : parts) t += p.dim(0);
  return t;
}
// rows [begin, begin+n) of a column-major matrix
Mat middle_rows(const Mat& a, Index begin, Index n) {
  Mat out(n, a.cols);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < n; ++i) out(i, j) = a(begin + i, j);
  return out;
}
}  // namespace

// stitch.cpp:36-47
Factors partial_hit_factors(const Factors& stored, Index begin, Index end) {
  const Index len = stored.dim(0);
  if (begin < 0 || begin >= end || end > len) bad("partial_hit_factors: invalid sub-range");
  const QrResult qr = thin_qr(middle_rows(stored.f[0], begin, end - begin));
  Factors out;
  out.core = mode_product(stored.core, qr.r, 0);
  out.f = stored.f;
  out.f[0] = qr.q;
  return out;
}

// stitch.cpp:49-73 — per part, contract modes p-1..1 (descending), rows = V0 * M0(acc)
Mat stitch_temporal_unfolding(std::span<const Factors> parts, std::span<const Mat> factors) {
  check_parts(parts);
  const Index p = parts[0].order();
  if (static_cast<Index>(factors.size()) != p) bad("stitch_temporal_unfolding: one factor per mode required");
  Index cols = 1;
  for (Index m = 1; m < p; ++m) cols *= factors[static_cast<std::size_t>(m)].cols;
  Mat z(total_temporal(parts), cols);
  Index row = 0;
  for (const Factors& part : parts) {
    Tensor acc = part.core;
    for (Index m = p - 1; m >= 1; --m)
      acc = mode_product(acc, matmul(transpose(factors[static_cast<std::size_t>(m)]), part.f[static_cast<std::size_t>(m)]), m);
    const Mat rows = matmul(part.f[0], matricize(acc, 0));
    for (Index j = 0; j < cols; ++j)
      for (Index i = 0; i < part.dim(0); ++i) z(row + i, j) = rows(i, j);
    row += part.dim(0);
  }
  return z;
}

// stitch.cpp:75-108
Mat stitch_nontemporal_unfolding(std::span<const Factors> parts, Index mode, std::span<const Mat> factors) {
  check_parts(parts);
  const Index p = parts[0].order();
  if (mode < 1 || mode >= p) bad("stitch_nontemporal_unfolding: mode must be non-temporal");
  if (static_cast<Index>(factors.size()) != p) bad("stitch_nontemporal_unfolding: one factor per mode required");
  Index cols = 1;
  for (Index m = 0; m < p; ++m)
    if (m != mode) cols *= factors[static_cast<std::size_t>(m)].cols;
  Mat z(parts[0].dim(mode), cols);
  Index offset = 0;
  for (const Factors& part : parts) {
    Tensor acc = part.core;
    for (Index m = 0; m < p; ++m) {
      if (m == mode) continue;
      const Mat w = m == 0 ? matmul(transpose(middle_rows(factors[0], offset, part.dim(0))), part.f[0])
                           : matmul(transpose(factors[static_cast<std::size_t>(m)]), part.f[static_cast<std::size_t>(m)]);
      acc = mode_product(acc, w, m);
    }
    acc = mode_product(acc, part.f[static_cast<std::size_t>(mode)], mode);
    const Mat zm = matricize(acc, mode);
    for (std::size_t i = 0; i < z.v.size(); ++i) z.v[i] += zm.v[i];
    offset += part.dim(0);
  }
  return z;
}

// stitch.cpp:110-184
Factors stitch(std::span<const Factors> parts, std::span<const Index> requested_ranks,
               const AlsConfig& cfg, AlsTrace* trace) {
  check_parts(parts);
  const Index p = parts[0].order();
  if (p < 2) bad("stitch: parts must have order >= 2");
  if (static_cast<Index>(requested_ranks.size()) != p) bad("stitch: one rank per mode required");
  if (cfg.max_iters < 1) bad("stitch: max_iters must be >= 1");
  if (cfg.tol <= 0.0) bad("stitch: tol must be > 0");
  const Index total_len = total_temporal(parts);
  std::vector<Index> dims(static_cast<std::size_t>(p));
  dims[0] = total_len;
  for (Index m = 1; m < p; ++m) dims[static_cast<std::size_t>(m)] = parts[0].dim(m);
  const std::vector<Index> ranks = clamp_ranks(requested_ranks, dims);
  if (trace != nullptr) *trace = AlsTrace{};
  double norm_sq = 0.0;
  for (const Factors& part : parts) norm_sq += squared_norm(part.core);

  std::mt19937_64 rng(cfg.seed);
  Factors f;
  f.f.resize(static_cast<std::size_t>(p));
  f.f[0] = Mat(total_len, ranks[0]);
  for (Index m = 1; m < p; ++m)
    f.f[static_cast<std::size_t>(m)] = random_orthonormal(dims[static_cast<std::size_t>(m)], ranks[static_cast<std::size_t>(m)], rng);
  f.core = Tensor(ranks);
  if (norm_sq == 0.0) {
    f.f[0] = random_orthonormal(total_len, ranks[0], rng);
    if (trace != nullptr) trace->converged = true;
    return f;
  }
  const double norm = std::sqrt(norm_sq);
  double prev_fit = std::numeric_limits<double>::quiet_NaN();
  for (int sweep = 0; sweep < cfg.max_iters; ++sweep) {
    f.f[0] = leading_left_singular_vectors(stitch_temporal_unfolding(parts, f.f), ranks[0]);
    Mat z;
    for (Index m = 1; m < p; ++m) {
      z = stitch_nontemporal_unfolding(parts, m, f.f);
      f.f[static_cast<std::size_t>(m)] = leading_left_singular_vectors(z, ranks[static_cast<std::size_t>(m)]);
    }
    std::vector<Index> zdims(static_cast<std::size_t>(p));
    zdims[0] = f.f[0].cols;
    for (Index m = 1; m + 1 < p; ++m) zdims[static_cast<std::size_t>(m)] = f.f[static_cast<std::size_t>(m)].cols;
    zdims[static_cast<std::size_t>(p - 1)] = dims[static_cast<std::size_t>(p - 1)];
    f.core = mode_product(from_matricization(z, zdims, p - 1), transpose(f.f[static_cast<std::size_t>(p - 1)]), p - 1);
    const double residual_sq = std::max(0.0, norm_sq - squared_norm(f.core));
    if (trace != nullptr) trace->objective.push_back(residual_sq);
    const double fit = 1.0 - std::sqrt(residual_sq) / norm;
    if (sweep > 0 && std::abs(fit - prev_fit) < cfg.tol) {
      if (trace != nullptr) trace->converged = true;
      break;
    }
    prev_fit = fit;
  }
  return f;
}

// ---------------------------------------------------------------------------
Index default_block_size(Index timespan) {  // baseline.cpp:12-22
  if (timespan < 1) bad("default_block_size: timespan must be >= 1");
  Index log = 0, pow = 1;
  while (pow < timespan) {
    pow *= 2;
    ++log;
  }
  if (log == 0) return 1;
  return std::max<Index>(1, timespan / (2 * log));
}

Factors brute_force_range(const Tensor& x, Index ts, Index te, std::span<const Index> ranks,
                          const AlsConfig& cfg) {  // baseline.cpp:67-75
  if (ts < 0 || ts >= te || te > x.dim(0)) bad("brute_force_range: invalid range");
  AlsConfig als = cfg;
  als.ranks.assign(ranks.begin(), ranks.end());
  return tucker_als(slice_temporal(x, ts, te), als);
}

Tensor generate_synthetic(const SynthSpec& spec) {  // baseline.cpp:77-128
  const Index p = static_cast<Index>(spec.shape.size());
  if (p < 2) bad("generate_synthetic: order must be >= 2");
  if (spec.true_ranks.size() != spec.shape.size()) bad("generate_synthetic: one true rank per mode required");
  for (Index n = 0; n < p; ++n) {
    const Index r = spec.true_ranks[static_cast<std::size_t>(n)];
    if (r < 1 || r > spec.shape[static_cast<std::size_t>(n)]) bad("generate_synthetic: true ranks must be in [1, extent]");
  }
  if (!(spec.noise >= 0.0 && spec.noise < 1.0)) bad("generate_synthetic: noise must be in [0, 1)");
  std::mt19937_64 rng(spec.seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  Factors truth;
  for (Index n = 0; n < p; ++n)
    truth.f.push_back(random_orthonormal(spec.shape[static_cast<std::size_t>(n)], spec.true_ranks[static_cast<std::size_t>(n)], rng));
  truth.core = Tensor(spec.true_ranks);
  for (double& v : truth.core.v) v = normal(rng);
  Tensor w = reconstruct(truth);
  if (spec.noise == 0.0) return w;
  const double w_sq = squared_norm(w);
  if (w_sq == 0.0) throw std::runtime_error("generate_synthetic: degenerate zero signal");
  Tensor e(spec.shape);
  for (double& v : e.v) v = normal(rng);
  double dot = 0.0;
  for (Index i = 0; i < e.size(); ++i) dot += e.v[static_cast<std::size_t>(i)] * w.v[static_cast<std::size_t>(i)];
  for (Index i = 0; i < e.size(); ++i) e.v[static_cast<std::size_t>(i)] -= dot / w_sq * w.v[static_cast<std::size_t>(i)];
  const double e_norm = std::sqrt(squared_norm(e));
  if (e_norm == 0.0) throw std::runtime_error("generate_synthetic: degenerate noise draw");
  const double c = spec.noise * std::sqrt(w_sq) / (e_norm * std::sqrt(1.0 - spec.noise * spec.noise));
  for (Index i = 0; i < e.size(); ++i) w.v[static_cast<std::size_t>(i)] += c * e.v[static_cast<std::size_t>(i)];
  return w;
}

// ---------------------------------------------------------------------------
// Stream segment tree (sst.cpp) over the coarsened axis: leaf k covers slices
// [kB, (k+1)B); node ranges are stored in slices.
Tree::Tree(TreeConfig cfg) : cfg_(std::move(cfg)) {  // sst.cpp:29-45
  if (cfg_.nontemporal.empty()) bad("StreamSegmentTree: non-temporal shape required");
  for (Index d : cfg_.nontemporal)
    if (d < 1) bad("StreamSegmentTree: extents must be >= 1");
  if (cfg_.ranks.size() != cfg_.nontemporal.size() + 1) bad("StreamSegmentTree: one rank per mode required");
  for (Index r : cfg_.ranks)
    if (r < 1) bad("StreamSegmentTree: ranks must be >= 1");
  if (!(cfg_.theta > 0.0 && cfg_.theta < 1.0)) bad("StreamSegmentTree: theta must be in (0, 1)");
  if (cfg_.leaf_block < 1) bad("StreamSegmentTree: leaf_block must be >= 1");
  slice_size_ = element_count(cfg_.nontemporal);
  std::vector<Index> td = {0};
  td.insert(td.end(), cfg_.nontemporal.begin(), cfg_.nontemporal.end());
  tail_.dims = td;
}

const Node& Tree::node(NodeId id) const {
  if (id < 1 || id > static_cast<NodeId>(nodes_.size())) throw std::out_of_range("unknown node id");
  return nodes_[static_cast<std::size_t>(id - 1)];
}

NodeId Tree::create_node(Index begin_leaf, Index end_leaf) {  // sst.cpp:73-81
  Node n;
  n.id = static_cast<NodeId>(nodes_.size() + 1);
  n.begin = begin_leaf * cfg_.leaf_block;
  n.end = end_leaf * cfg_.leaf_block;
  nodes_.push_back(std::move(n));
  return nodes_.back().id;
}

// sst.cpp:94-110 (append) — one slice; a leaf is inserted when B slices are buffered.
void Tree::append(const double* slice) {
  last_touches_ = 0;
  last_redec_.clear();
  tail_.v.insert(tail_.v.end(), slice, slice + slice_size_);
  tail_.dims[0] += 1;
  ++timespan_;
  if (tail_.dims[0] < cfg_.leaf_block) return;
  const Index t = leaves_;  // leaf index
  const Index B = cfg_.leaf_block;
  if (t == 0) {
    root_ = create_node(0, 1);
  } else if (node(root_).end == t * B) {
    const NodeId promoted = create_node(0, 2 * t);
    node_mut(promoted).left = root_;
    root_ = promoted;
  }
  Tensor block = tail_;
  tail_.v.clear();
  tail_.dims[0] = 0;
  insert(root_, t, block);
  ++leaves_;
}

// sst.cpp:112-145, in leaf units.
void Tree::insert(NodeId id, Index t, const Tensor& block) {
  ++last_touches_;
  const Index B = cfg_.leaf_block;
  const Index b = node(id).begin / B, e = node(id).end / B;
  if (b == t && e == t + 1) {  // sst.cpp:114-119 + preprocess_leaf 83-92
    AlsConfig als = cfg_.als;
    als.ranks = cfg_.ranks;
    Factors leaf = tucker_als(block, als);
    Node& v = node_mut(id);
    v.dec = std::move(leaf);
    v.kind = NodeKind::Leaf;
    last_redec_.push_back(id);
    return;
  }
  const Index mid = (b + e) / 2;
  if (t < mid) {
    if (node(id).left == kNoNode) {
      const NodeId child = create_node(b, mid);
      node_mut(id).left = child;
    }
    insert(node(id).left, t, block);
  } else {
    if (node(id).right == kNoNode) {
      const NodeId child = create_node(mid, e);
      node_mut(id).right = child;
    }
    insert(node(id).right, t, block);
    if (e == t + 1) {
      const Factors parts[2] = {*node(node(id).left).dec, *node(node(id).right).dec};
      Factors merged = stitch(parts, cfg_.ranks, cfg_.als);
      Node& v = node_mut(id);
      v.dec = std::move(merged);
      v.kind = NodeKind::Intermediate;
      ++stitch_count_;
      last_redec_.push_back(id);
    }
  }
}

Index Tree::height() const {  // sst.cpp:147-157
  if (root_ == kNoNode) return 0;
  std::function<Index(NodeId)> depth = [&](NodeId id) -> Index {
    const Node& v = node(id);
    Index best = 0;
    if (v.left != kNoNode) best = std::max(best, depth(v.left));
    if (v.right != kNoNode) best = std::max(best, depth(v.right));
    return best + 1;
  };
  return depth(root_);
}

namespace {
Index ceil_log2(Index n) {
  Index log = 0, pow = 1;
  while (pow < n) {
    pow *= 2;
    ++log;
  }
  return log;
}
std::string node_label(const Node& n) {
  return "node " + std::to_string(n.id) + " [" + std::to_string(n.begin) + "," + std::to_string(n.end) + ")";
}
}  // namespace

// sst.cpp:159-295 (structural checks; leaf length B, frontier in leaf units).
std::vector<std::string> Tree::validate() const {
  std::vector<std::string> out;
  const auto flag = [&out](std::string m) { out.push_back(std::move(m)); };
  const Index B = cfg_.leaf_block;
  const Index T = leaves_ * B;  // materialised timespan of the tree
  if (leaves_ == 0) {
    if (root_ != kNoNode) flag("empty tree has a root");
    return out;
  }
  if (root_ == kNoNode) {
    flag("non-empty tree has no root");
    return out;
  }
  const Index p = static_cast<Index>(cfg_.nontemporal.size()) + 1;
  const auto valid_id = [this](NodeId id) { return id >= 1 && id <= static_cast<NodeId>(nodes_.size()); };
  for (const Node& v : nodes_) {
    if (v.begin < 0 || v.begin >= v.end) flag(node_label(v) + ": malformed range");
    if ((v.left != kNoNode && !valid_id(v.left)) || (v.right != kNoNode && !valid_id(v.right))) {
      flag(node_label(v) + ": child id unknown");
      continue;
    }
    switch (v.kind) {
      case NodeKind::Leaf:
        if (v.length() != B) flag(node_label(v) + ": leaf range must have length 1");
        if (v.left != kNoNode || v.right != kNoNode) flag(node_label(v) + ": leaf must not have children");
        if (!v.dec) flag(node_label(v) + ": leaf is missing its decomposition");
        break;
      case NodeKind::Intermediate: {
        if (v.left == kNoNode || v.right == kNoNode) {
          flag(node_label(v) + ": intermediate must have two children");
          break;
        }
        const Node& l = node(v.left);
        const Node& r = node(v.right);
        if (l.begin != v.begin || l.end != r.begin || r.end != v.end) flag(node_label(v) + ": children ranges are not adjoint");
        if (l.kind == NodeKind::Placeholder || r.kind == NodeKind::Placeholder)
          flag(node_label(v) + ": intermediate has a placeholder child");
        if (!v.dec) flag(node_label(v) + ": intermediate is missing its decomposition");
        break;
      }
      case NodeKind::Placeholder: {
        if (v.dec) flag(node_label(v) + ": placeholder carries a decomposition");
        if (!(v.begin < T && T <= v.end)) flag(node_label(v) + ": placeholder does not straddle the write frontier");
        if (v.left == kNoNode && v.right != kNoNode) flag(node_label(v) + ": placeholder has a right child without a left child");
        if (v.left == kNoNode && v.right == kNoNode) flag(node_label(v) + ": placeholder has no children");
        if (v.left != kNoNode && v.right != kNoNode) {
          const Node& l = node(v.left);
          const Node& r = node(v.right);
          if (l.begin != v.begin || l.end != r.begin || r.end != v.end) flag(node_label(v) + ": children ranges are not adjoint");
        } else if (v.left != kNoNode) {
          const Node& l = node(v.left);
          if (l.begin != v.begin || l.end != ((v.begin / B + v.end / B) / 2) * B)
            flag(node_label(v) + ": left child range does not match the midpoint split");
        }
        break;
      }
    }
    if (v.kind != NodeKind::Placeholder && v.end > T) flag(node_label(v) + ": materialized node extends past the timespan");
    if (v.dec) {
      const Factors& f = *v.dec;
      if (f.order() != p) {
        flag(node_label(v) + ": decomposition order mismatch");
      } else {
        if (f.dim(0) != v.length()) flag(node_label(v) + ": temporal factor rows do not match the range");
        for (Index m = 1; m < p; ++m)
          if (f.dim(m) != cfg_.nontemporal[static_cast<std::size_t>(m - 1)])
            flag(node_label(v) + ": non-temporal factor rows mismatch at mode " + std::to_string(m));
        for (Index m = 0; m < p; ++m)
          if (f.core.dim(m) != f.rank(m)) flag(node_label(v) + ": core extent does not match factor columns");
      }
    }
  }
  std::vector<const Node*> leaves;
  for (const Node& v : nodes_)
    if (v.kind == NodeKind::Leaf) leaves.push_back(&v);
  std::sort(leaves.begin(), leaves.end(), [](const Node* a, const Node* b) { return a->begin < b->begin; });
  Index expected = 0;
  for (const Node* leaf : leaves) {
    if (leaf->begin != expected) {
      flag(node_label(*leaf) + ": leaf tiling gap or overlap at " + std::to_string(expected));
      break;
    }
    expected = leaf->end;
  }
  if (expected != T && out.empty()) flag("leaves cover [0," + std::to_string(expected) + ") but timespan is " + std::to_string(T));
  const Node& r = node(root_);
  const Index span = (leaves_ == 1 ? 1 : (Index{1} << ceil_log2(leaves_))) * B;
  if (r.begin != 0 || r.end != span) flag(node_label(r) + ": root range should be [0," + std::to_string(span) + ")");
  const Index expected_height = ceil_log2(leaves_) + 1;
  if (height() != expected_height)
    flag("height " + std::to_string(height()) + " violates the height law " + std::to_string(expected_height));
  return out;
}

// ---------------------------------------------------------------------------
// query.cpp:9-31 plus the leaf-block rule: an overlapping leaf is
// always a hit (a no-op at B = 1, where a visited leaf always passes theta).
namespace {
void collect_hits(const Tree& tree, NodeId id, Index ts, Index te, double theta, HitSet& out) {
  const Node& v = tree.node(id);
  const Index overlap = std::min(te, v.end) - std::max(ts, v.begin);
  if (v.kind != NodeKind::Placeholder &&
      (static_cast<double>(overlap) >= theta * static_cast<double>(v.length()) || v.kind == NodeKind::Leaf)) {
    const bool contained = v.begin >= ts && v.end <= te;
    out.push_back(HitEntry{id, std::max(ts, v.begin), std::min(te, v.end), contained ? HitFlag::Entire : HitFlag::Partial});
    return;
  }
  if (v.left != kNoNode && te <= tree.node(v.left).end) {
    collect_hits(tree, v.left, ts, te, theta, out);
  } else if (v.right != kNoNode && ts >= tree.node(v.right).begin) {
    collect_hits(tree, v.right, ts, te, theta, out);
  } else {
    if (v.left == kNoNode || v.right == kNoNode) throw std::logic_error("recall: query spans an unmaterialized range");
    collect_hits(tree, v.left, ts, te, theta, out);
    collect_hits(tree, v.right, ts, te, theta, out);
  }
}
}  // namespace

HitSet recall(const Tree& tree, Index ts, Index te, std::optional<double> theta_opt) {  // query.cpp:35-47
  if (ts < 0 || ts >= te || te > tree.timespan()) bad("recall: query range must satisfy 0 <= ts < te <= T");
  const double theta = theta_opt.value_or(tree.config().theta);
  if (!(theta > 0.0 && theta < 1.0)) bad("recall: theta must be in (0, 1)");
  HitSet out;
  const Index tb = tree.leaves() * tree.config().leaf_block;
  if (ts < tb) collect_hits(tree, tree.root(), ts, std::min(te, tb), theta, out);
  if (te > tb) out.push_back(HitEntry{kNoNode, std::max(ts, tb), te, HitFlag::Tail});
  return out;
}

// query.cpp:49-69; a tail hit is decomposed from the raw tail (reference
// semantics: tucker_als of the explicit sub-range).
QueryResult range_query_detailed(const Tree& tree, Index ts, Index te, std::optional<double> theta, AlsTrace* trace) {
  QueryResult result;
  result.hits = recall(tree, ts, te, theta);
  std::vector<Factors> parts;
  parts.reserve(result.hits.size());
  const Index tb = tree.leaves() * tree.config().leaf_block;
  for (const HitEntry& hit : result.hits) {
    if (hit.flag == HitFlag::Tail) {
      AlsConfig als = tree.config().als;
      als.ranks = tree.config().ranks;
      parts.push_back(tucker_als(slice_temporal(tree.tail(), hit.begin - tb, hit.end - tb), als));
      continue;
    }
    const Node& v = tree.node(hit.node);
    if (!v.dec) throw std::logic_error("range_query: hit node has no decomposition");
    if (hit.flag == HitFlag::Entire) {
      parts.push_back(*v.dec);
    } else {
      parts.push_back(partial_hit_factors(*v.dec, hit.begin - v.begin, hit.end - v.begin));
    }
  }
  result.factors = stitch(parts, tree.config().ranks, tree.config().als, trace);
  return result;
}

}  // namespace tto
