// TEST INFRASTRUCTURE — LAPACK entry points of numpy's bundled OpenBLAS
// (ILP64, scipy_ prefix), used by the Eigen shim's QR and SVD.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "Core"

extern "C" {
void scipy_dgeqrf_64_(const int64_t* m, const int64_t* n, double* a, const int64_t* lda, double* tau, double* work,
                      const int64_t* lwork, int64_t* info);
void scipy_dormqr_64_(const char* side, const char* trans, const int64_t* m, const int64_t* n, const int64_t* k,
                      const double* a, const int64_t* lda, const double* tau, double* c, const int64_t* ldc,
                      double* work, const int64_t* lwork, int64_t* info, size_t, size_t);
void scipy_dgesdd_64_(const char* jobz, const int64_t* m, const int64_t* n, double* a, const int64_t* lda, double* s,
                      double* u, const int64_t* ldu, double* vt, const int64_t* ldvt, double* work,
                      const int64_t* lwork, int64_t* iwork, int64_t* info, size_t);
}

namespace Eigen {
namespace shim_lapack {

inline void geqrf(MatrixXd& a, std::vector<double>& tau) {
  const int64_t m = a.rows(), n = a.cols(), lda = std::max<int64_t>(1, m);
  if (m == 0 || n == 0) return;
  int64_t info = 0, lwork = -1;
  double q = 0.0;
  scipy_dgeqrf_64_(&m, &n, a.data(), &lda, tau.data(), &q, &lwork, &info);
  lwork = std::max<int64_t>(1, int64_t(q));
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dgeqrf_64_(&m, &n, a.data(), &lda, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("Eigen shim: dgeqrf failed");
}

// C <- Q C with Q from the packed Householder reflectors of qr (dormqr L N).
inline void ormqr_left(const MatrixXd& qr, const std::vector<double>& tau, MatrixXd& c) {
  const int64_t m = c.rows(), n = c.cols(), k = static_cast<int64_t>(tau.size());
  if (m == 0 || n == 0 || k == 0) return;
  const int64_t lda = std::max<int64_t>(1, qr.rows()), ldc = std::max<int64_t>(1, m);
  int64_t info = 0, lwork = -1;
  double q = 0.0;
  const char side = 'L', trans = 'N';
  scipy_dormqr_64_(&side, &trans, &m, &n, &k, qr.data(), &lda, tau.data(), c.data(), &ldc, &q, &lwork, &info, 1, 1);
  lwork = std::max<int64_t>(1, int64_t(q));
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dormqr_64_(&side, &trans, &m, &n, &k, qr.data(), &lda, tau.data(), c.data(), &ldc, work.data(), &lwork,
                   &info, 1, 1);
  if (info != 0) throw std::runtime_error("Eigen shim: dormqr failed");
}

// Thin left singular vectors (m x min(m, n)) and singular values, descending.
inline void gesdd_thin_u(const MatrixXd& a_in, MatrixXd& u, MatrixXd& s) {
  const int64_t m = a_in.rows(), n = a_in.cols(), k = std::min(m, n);
  u = MatrixXd(m, k);
  s = MatrixXd(k, 1);
  if (k == 0) return;
  MatrixXd a(a_in);
  const int64_t lda = std::max<int64_t>(1, m), ldu = std::max<int64_t>(1, m), ldvt = std::max<int64_t>(1, k);
  std::vector<double> vt(static_cast<size_t>(k * n));
  std::vector<int64_t> iwork(static_cast<size_t>(8 * k));
  int64_t info = 0, lwork = -1;
  double q = 0.0;
  const char jobz = 'S';
  scipy_dgesdd_64_(&jobz, &m, &n, a.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt, &q, &lwork,
                   iwork.data(), &info, 1);
  lwork = std::max<int64_t>(1, int64_t(q));
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dgesdd_64_(&jobz, &m, &n, a.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt, work.data(), &lwork,
                   iwork.data(), &info, 1);
  if (info != 0) throw std::runtime_error("Eigen shim: dgesdd failed");
}

}  // namespace shim_lapack
}  // namespace Eigen
