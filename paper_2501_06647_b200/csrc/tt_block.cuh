// Block-cooperative FP64 primitives used by the per-problem ALS kernels.
// Every function must be called by all threads of the block (uniform control
// flow) and ends with a __syncthreads() so results are visible to the block.
//
// The ALS kernels run one CTA per problem (a leaf block, an append stitch or
// a range query): the problem's working set lives in its workspace (L2/L1
// resident) and in shared memory, and the whole sweep loop — including the
// data-dependent stop test — runs on the device without host round trips.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tt_common.h"

namespace ttb {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxVec = 32;  // max columns handled by the vector reductions

struct BlockScratch {
  double red[kWarps * kMaxVec];
  double vec[kMaxVec];
  double bcast[4];
  int ibcast[4];
  // Jacobi pair tables
  double jc[256], js[256], jt[256];
  int jp[256], jq[256];
  int rotated[2];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v, BlockScratch& sc) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sc.red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kWarps; ++i) s += sc.red[i];
    sc.bcast[0] = s;
  }
  __syncthreads();
  return sc.bcast[0];
}

// Reduces nv (<= kMaxVec) per-thread partial sums; results in sc.vec[0..nv).
template <int NV>
__device__ __forceinline__ void block_sum_vec(const double (&v)[NV], int nv, BlockScratch& sc) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (i < nv) {
      const double s = warp_sum(v[i]);
      if (l == 0) sc.red[w * kMaxVec + i] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int k = 0; k < kWarps; ++k) s += sc.red[k * kMaxVec + threadIdx.x];
    sc.vec[threadIdx.x] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void bcopy(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
}
__device__ __forceinline__ void bzero(double* dst, int64_t n) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = 0.0;
  __syncthreads();
}
__device__ __forceinline__ double bsumsq(const double* __restrict__ x, int64_t n, BlockScratch& sc) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], x[i], s);
  return block_sum(s, sc);
}

// ---------------------------------------------------------------------------
// Mode product on a row-major tensor viewed as (outer, d, inner):
//   out[o][a][t] (+)= sum_j M(a, j) * in[o][j][t],  a < r,
// with M(a, j) = M[a*ms_a + j*ms_j]. For M = U^T with U (d x r, col-major,
// ld) use ms_a = ld, ms_j = 1; for M = U (r x d, col-major) ms_a = 1, ms_j = ld.
template <int RT>
__device__ __forceinline__ void ttm_chunk(const double* __restrict__ in, int64_t outer, int64_t d, int64_t inner,
                                          const double* __restrict__ M, int64_t ms_a, int64_t ms_j, int a0,
                                          int na, double* __restrict__ out, int64_t r_total, bool acc) {
  const int64_t ncol = outer * inner;
  for (int64_t c = threadIdx.x; c < ncol; c += blockDim.x) {
    const int64_t o = c / inner, t = c - o * inner;
    const double* src = in + o * d * inner + t;
    double s[RT];
#pragma unroll
    for (int a = 0; a < RT; ++a) s[a] = 0.0;
    for (int64_t j = 0; j < d; ++j) {
      const double x = __ldg(src + j * inner);
      const double* mj = M + j * ms_j + int64_t(a0) * ms_a;
#pragma unroll
      for (int a = 0; a < RT; ++a)
        if (a < na) s[a] = fma(__ldg(mj + a * ms_a), x, s[a]);
    }
    double* dst = out + o * r_total * inner + t;
#pragma unroll
    for (int a = 0; a < RT; ++a)
      if (a < na) {
        double* q = dst + int64_t(a0 + a) * inner;
        *q = acc ? *q + s[a] : s[a];
      }
  }
}

__device__ __forceinline__ void ttm(const double* in, int64_t outer, int64_t d, int64_t inner, const double* M,
                                    int64_t ms_a, int64_t ms_j, int64_t r, double* out, bool acc) {
  for (int a0 = 0; a0 < r; a0 += 16) {
    const int na = int(imin(16, r - a0));
    if (na <= 4)
      ttm_chunk<4>(in, outer, d, inner, M, ms_a, ms_j, a0, na, out, r, acc);
    else if (na <= 8)
      ttm_chunk<8>(in, outer, d, inner, M, ms_a, ms_j, a0, na, out, r, acc);
    else
      ttm_chunk<16>(in, outer, d, inner, M, ms_a, ms_j, a0, na, out, r, acc);
  }
  __syncthreads();
}

// C(i,j) (+)= alpha * sum_k A(i,k) B(k,j); element (i,j) of X at X[i*rs + j*cs].
__device__ __forceinline__ void gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t ars, int64_t acs,
                                     const double* B, int64_t brs, int64_t bcs, double* C, int64_t crs, int64_t ccs,
                                     bool acc) {
  const int64_t tot = M * N;
  for (int64_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int64_t i = idx % M, j = idx / M;
    double s = 0.0;
    const double* a = A + i * ars;
    const double* b = B + j * bcs;
    for (int64_t k = 0; k < K; ++k) s = fma(a[k * acs], b[k * brs], s);
    double* c = C + i * crs + j * ccs;
    *c = acc ? *c + s : s;
  }
  __syncthreads();
}

// Unfolding view of a row-major (outer, rows, inner) tensor: A(i, o*inner+t).
// G = A A^T (rows x rows).
__device__ __forceinline__ void gram_rows(const double* __restrict__ P, int64_t outer, int64_t rows, int64_t inner,
                                          double* __restrict__ G) {
  const int64_t tot = rows * rows;
  for (int64_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    if (i > j) continue;
    double s = 0.0;
    for (int64_t o = 0; o < outer; ++o) {
      const double* pi = P + (o * rows + i) * inner;
      const double* pj = P + (o * rows + j) * inner;
      for (int64_t t = 0; t < inner; ++t) s = fma(pi[t], pj[t], s);
    }
    G[i + j * rows] = s;
    G[j + i * rows] = s;
  }
  __syncthreads();
}

// G = A^T A (cols x cols), cols = outer*inner.
__device__ __forceinline__ void gram_cols(const double* __restrict__ P, int64_t outer, int64_t rows, int64_t inner,
                                          double* __restrict__ G) {
  const int64_t cols = outer * inner;
  const int64_t tot = cols * cols;
  for (int64_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int64_t c1 = idx % cols, c2 = idx / cols;
    if (c1 > c2) continue;
    const int64_t o1 = c1 / inner, t1 = c1 - o1 * inner, o2 = c2 / inner, t2 = c2 - o2 * inner;
    const double* p1 = P + o1 * rows * inner + t1;
    const double* p2 = P + o2 * rows * inner + t2;
    double s = 0.0;
    for (int64_t i = 0; i < rows; ++i) s = fma(p1[i * inner], p2[i * inner], s);
    G[c1 + c2 * cols] = s;
    G[c2 + c1 * cols] = s;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Cyclic parallel (round-robin) Jacobi eigensolver for a symmetric n x n
// matrix A (col-major, ld n). On exit A is diagonal (eigenvalues), V holds the
// eigenvectors as columns, order[0..n) lists indices by descending eigenvalue
// (ties by lower index). One round rotates n/2 disjoint planes at once; each
// 2x2 block of A and each row pair of V is owned by one thread, so a round is
// two barriers.
__device__ void sym_eig(double* A, int n, double* V, int* order, BlockScratch& sc) {
  const int n2 = n + (n & 1);
  const int np = n2 / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < n; j += kWarps)
    for (int i = lane; i < n; i += 32) V[i + j * n] = (i == j) ? 1.0 : 0.0;
  if (threadIdx.x < 2) sc.rotated[threadIdx.x] = 0;
  if (n <= 1) {
    if (threadIdx.x == 0 && n == 1) order[0] = 0;
    __syncthreads();
    return;
  }
  // Skip a rotation when |a_pq| <= max(eps_r sqrt(|a_pp a_qq|), eps_a ||A||_F):
  // the relative test keeps the large eigenpairs accurate to working
  // precision, the absolute floor stops the solver from chasing rounding noise
  // between numerically-zero eigenvalues (eigenvector error <= eps_a/gap).
  double fro = 0.0;
  for (int j = warp; j < n; j += kWarps)
    for (int i = lane; i < n; i += 32) fro = fma(A[i + j * n], A[i + j * n], fro);
  const double abs_thr = 1e-16 * sqrt(block_sum(fro, sc));
  const double eps = 1e-15;
  for (int sweep = 0; sweep < 20; ++sweep) {
    const int cur = sweep & 1;
    if (threadIdx.x == 0) sc.rotated[cur ^ 1] = 0;
    for (int r = 0; r < n2 - 1; ++r) {
      for (int k = threadIdx.x; k < np; k += blockDim.x) {
        int p, q;
        if (k == 0) {
          p = r;
          q = n2 - 1;
        } else {
          p = (r + k) % (n2 - 1);
          q = (r - k + (n2 - 1)) % (n2 - 1);
        }
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        double c = 1.0, s = 0.0, t = 0.0;
        if (q < n) {
          const double apq = A[p + q * n];
          const double app = A[p + p * n], aqq = A[q + q * n];
          if (fabs(apq) > fmax(eps * sqrt(fabs(app)) * sqrt(fabs(aqq)), abs_thr)) {
            const double tau = (aqq - app) / (2.0 * apq);
            if (fabs(tau) > 1e150) {
              t = 0.5 / tau;
            } else {
              t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            }
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            sc.rotated[cur] = 1;
          }
        }
        sc.jp[k] = p;
        sc.jq[k] = q;
        sc.jc[k] = c;
        sc.js[k] = s;
        sc.jt[k] = t;
      }
      __syncthreads();
      // A <- J^T A J on 2x2 blocks (one owner thread per block), V <- V J.
      for (int P2 = warp; P2 < np; P2 += kWarps) {
        const int p2 = sc.jp[P2], q2 = sc.jq[P2];
        const double c2 = sc.jc[P2], s2 = sc.js[P2];
        const bool hq2 = q2 < n;
        for (int P1 = lane; P1 < np; P1 += 32) {
          const double s1 = sc.js[P1];
          if (P1 == P2) {
            if (s1 != 0.0) {
              const int p = sc.jp[P1], q = sc.jq[P1];
              const double apq = A[p + q * n];
              const double t = sc.jt[P1];
              A[p + p * n] -= t * apq;
              A[q + q * n] += t * apq;
              A[p + q * n] = 0.0;
              A[q + p * n] = 0.0;
            }
            continue;
          }
          if (s1 == 0.0 && s2 == 0.0) continue;
          const int p = sc.jp[P1], q = sc.jq[P1];
          const double c = sc.jc[P1];
          const bool hq = q < n;
          const double m00 = A[p + p2 * n];
          const double m01 = hq2 ? A[p + q2 * n] : 0.0;
          const double m10 = hq ? A[q + p2 * n] : 0.0;
          const double m11 = (hq && hq2) ? A[q + q2 * n] : 0.0;
          const double x00 = c * m00 - s1 * m10, x01 = c * m01 - s1 * m11;
          const double x10 = s1 * m00 + c * m10, x11 = s1 * m01 + c * m11;
          A[p + p2 * n] = c2 * x00 - s2 * x01;
          if (hq2) A[p + q2 * n] = s2 * x00 + c2 * x01;
          if (hq) A[q + p2 * n] = c2 * x10 - s2 * x11;
          if (hq && hq2) A[q + q2 * n] = s2 * x10 + c2 * x11;
        }
      }
      for (int P1 = warp; P1 < np; P1 += kWarps) {
        const double s1 = sc.js[P1];
        if (s1 == 0.0) continue;
        const int p = sc.jp[P1], q = sc.jq[P1];
        const double c = sc.jc[P1];
        double* vp = V + p * n;
        double* vq = V + q * n;
        for (int i = lane; i < n; i += 32) {
          const double a = vp[i], b = vq[i];
          vp[i] = c * a - s1 * b;
          vq[i] = s1 * a + c * b;
        }
      }
      __syncthreads();
    }
    if (!sc.rotated[cur]) break;
    __syncthreads();
  }
  // rank by descending eigenvalue, ties to the lower index
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double li = A[i + i * n];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = A[j + j * n];
      if (lj > li || (lj == li && j < i)) ++rank;
    }
    order[rank] = i;
  }
  __syncthreads();
}

// Sign convention of linalg.cpp:15-31: each column's first max-|.| entry is
// made nonnegative. flips[j] = 1 when column j was negated.
__device__ void sign_fix(double* U, int64_t rows, int k, int64_t ld, int* flips, BlockScratch& sc) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int j = 0; j < k; ++j) {
    double best = -1.0;
    int64_t bi = 0;
    const double* col = U + int64_t(j) * ld;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      const double m = fabs(col[i]);
      if (m > best) {  // strictly greater: earliest index wins within a thread
        best = m;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    __syncthreads();
    if (l == 0) {
      sc.red[w] = best;
      sc.red[kWarps + w] = __longlong_as_double(bi);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = sc.red[0];
      int64_t idx = __double_as_longlong(sc.red[kWarps]);
      for (int i = 1; i < kWarps; ++i) {
        const double ob = sc.red[i];
        const int64_t oi = __double_as_longlong(sc.red[kWarps + i]);
        if (ob > b || (ob == b && oi < idx)) {
          b = ob;
          idx = oi;
        }
      }
      const int neg = rows > 0 && col[idx] < 0.0;
      sc.ibcast[0] = neg;
      if (flips) flips[j] = neg;
    }
    __syncthreads();
    if (sc.ibcast[0]) {
      double* cw = U + int64_t(j) * ld;
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) cw[i] = -cw[i];
    }
    __syncthreads();
  }
}

// Classical Gram-Schmidt applied twice (CGS2) to columns [j0, k) of U against
// all earlier columns; a column whose norm collapses (rank-deficient input) is
// replaced by the first unit vector e_r that survives orthogonalisation.
__device__ void orthonormalize(double* U, int64_t rows, int j0, int k, int64_t ld, BlockScratch& sc) {
  for (int j = j0; j < k; ++j) {
    double* uj = U + int64_t(j) * ld;
    int64_t next_e = 0;
    for (int attempt = 0; attempt < 64; ++attempt) {
      const double n0 = sqrt(bsumsq(uj, rows, sc));
      for (int pass = 0; pass < 2 && j > 0; ++pass) {
        double part[kMaxVec];
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i) part[i] = 0.0;
        for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
          const double v = uj[r];
#pragma unroll
          for (int i = 0; i < kMaxVec; ++i)
            if (i < j) part[i] = fma(U[r + int64_t(i) * ld], v, part[i]);
        }
        block_sum_vec<kMaxVec>(part, j, sc);
        for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
          double v = uj[r];
          for (int i = 0; i < j; ++i) v = fma(-sc.vec[i], U[r + int64_t(i) * ld], v);
          uj[r] = v;
        }
        __syncthreads();
      }
      const double n1 = sqrt(bsumsq(uj, rows, sc));
      if (n0 > 0.0 && n1 > 0.5 * n0 && n1 > 1e-300) {
        for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) uj[r] /= n1;
        __syncthreads();
        break;
      }
      // completion: try the next canonical vector
      for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) uj[r] = (r == next_e) ? 1.0 : 0.0;
      __syncthreads();
      ++next_e;
      if (next_e > rows) break;
    }
  }
}

}  // namespace ttb
