// sm_100a ALS kernels for the stream segment tree hot path.
//
//  leaf_als_kernel   — tucker_als on one leaf block (tucker.cpp:86-119), one
//                      CTA per leaf; X is streamed from HBM twice per sweep
//                      (Y = X x_{m>=1} U_m^T for the mode-0 update, W = X x_0
//                      U_0^T reused by every other mode and the core).
//  stitch_als_kernel — stitch() (stitch.cpp:110-184) for appends (2 parts)
//                      and range queries (s parts), one CTA per problem,
//                      entirely in compressed r-sized coordinates: the L-row
//                      temporal unfolding is never formed;
//                      partial hits enter through the Gram S = Vsub^T Vsub
//                      of their kept temporal rows instead of a QR.
#include <cuda_runtime.h>
#include <math.h>

#include <atomic>

#include "tt_block.cuh"

namespace ttb {

constexpr int kEigSmemN = 64;  // Jacobi runs in shared memory up to this size
constexpr int kStitchThreads = 256;  // 2 stitch CTAs per SM (128 threads x 4 CTAs measured slower)
constexpr size_t kDynSmem = size_t(2) * kEigSmemN * kEigSmemN * sizeof(double);  // stitch kernel: 64 KB

__device__ __forceinline__ unsigned dyn_smem_doubles() {
  unsigned b;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(b));
  return b / 8u;
}

// Leaf streaming ring: kStages tiles of kTileD doubles, plus U^T staging.
constexpr int kStages = 3;
constexpr int kTileD = int(kStreamTileDoubles);   // 20 KB per stage
constexpr int kUStage = 4096;  // U^T staged in shared memory when d*r <= this (32 KB)
constexpr size_t kLeafDynSmem = size_t(kStages * kTileD + kUStage) * sizeof(double);  // 96 KB

struct Pipe {
  uint64_t full[kStages];
  uint32_t uses[kStages];  // completed fills per stage (phase parity)
};

// out[o][a][t] = sum_j U[j][a] in[o][j][t]  (in: row-major (outer, d, inner);
// U: d x r col-major, ld d; r <= 16), streaming `in` from global memory through
// a kStages-deep cp.async.bulk ring. A tile is (G slabs) x (cj rows of j) x
// (tw columns of t); each thread owns one output column (g, t) and keeps its r
// accumulators across the j-tiles. Optionally accumulates sum(in^2) (every
// element is consumed by exactly one thread). Requires 16-byte aligned rows
// (inner*8 and tw*8 multiples of 16, 16-aligned base).
template <int R>
__device__ __noinline__ void ttm_stream_r(const double* __restrict__ in, int64_t outer, int64_t d, int64_t inner,
                                          const double* __restrict__ U, double* __restrict__ out, double* dyn,
                                          Pipe& pp, double* norm_acc, const void* tmap, int tmap_rank) {
  constexpr int r = R;
  const StreamTile tile = stream_tile(outer, d, inner);
  const int64_t tw = tile.tw, G = tile.G, cj = tile.cj;
  const int64_t ngrp = (outer + G - 1) / G, ntt = (inner + tw - 1) / tw, njt = (d + cj - 1) / cj;
  const int64_t ntiles = ngrp * ntt * njt;
  double* ring = dyn;
  double* Ut = dyn + kStages * kTileD;
  const bool u_smem = d * r <= kUStage;
  if (u_smem) {  // U^T, j-major: Ut[j*r + a]
    for (int64_t idx = threadIdx.x; idx < d * r; idx += blockDim.x) {
      const int64_t j = idx / r, a = idx - j * r;
      Ut[idx] = U[j + a * d];
    }
  }
  fence_proxy_async();  // prior generic smem accesses vs. the bulk-copy writes below
  __syncthreads();
  auto issue = [&](int64_t t) {  // warp 0: fill the stage of tile t
    const int st = int(t % kStages);
    const int64_t jt = t % njt, rest = t / njt, tt = rest % ntt, grp = rest / ntt;
    const int64_t o0 = grp * G, g_n = imin(G, outer - o0);
    const int64_t j0 = jt * cj, jn = imin(cj, d - j0);
    const int64_t t0 = tt * tw, tn = imin(tw, inner - t0);
    double* dst = ring + int64_t(st) * kTileD;
    const int lane = threadIdx.x & 31;
    if (tmap != nullptr) {
      // one TMA box per tile: (tw, cj, G) over (t, j, o); out-of-bounds parts are
      // zero-filled and still count toward the transaction bytes
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&pp.full[st], uint32_t(G * cj * tw * sizeof(double)));
        if (tmap_rank == 3)
          tma_load_3d(dst, tmap, int(t0), int(j0), int(o0), &pp.full[st]);
        else
          tma_load_2d(dst, tmap, int(t0), int(j0), &pp.full[st]);
      }
      (void)g_n;
      (void)jn;
      (void)tn;
      return;
    }
    const bool whole_rows = (tn == inner);  // one contiguous segment per slab
    const int64_t nseg = whole_rows ? g_n : g_n * jn;
    const uint32_t seg_bytes = uint32_t((whole_rows ? jn * inner : tn) * sizeof(double));
    if (lane == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&pp.full[st], uint32_t(nseg) * seg_bytes);
    }
    __syncwarp();
    for (int64_t sg = lane; sg < nseg; sg += 32) {
      int64_t g, jj;
      if (whole_rows) {
        g = sg;
        jj = 0;
      } else {
        g = sg / jn;
        jj = sg - g * jn;
      }
      const double* src = in + ((o0 + g) * d + j0 + jj) * inner + t0;
      bulk_g2s(dst + (g * cj + jj) * tw, src, seg_bytes, &pp.full[st]);
    }
  };
  if (threadIdx.x < 32)
    for (int64_t t = 0; t < imin(int64_t(kStages), ntiles); ++t) issue(t);
  double acc[R];
  double nrm = 0.0;
  for (int64_t t = 0; t < ntiles; ++t) {
    const int st = int(t % kStages);
    const int64_t jt = t % njt, rest = t / njt, tt = rest % ntt, grp = rest / ntt;
    const int64_t o0 = grp * G, g_n = imin(G, outer - o0);
    const int64_t j0 = jt * cj, jn = imin(cj, d - j0);
    const int64_t t0 = tt * tw, tn = imin(tw, inner - t0);
    const int64_t g = threadIdx.x / tw, tl = threadIdx.x - g * tw;
    const bool active = threadIdx.x < G * tw && g < g_n && tl < tn;
    if (jt == 0) {
#pragma unroll
      for (int a = 0; a < R; ++a) acc[a] = 0.0;
    }
    mbar_wait(&pp.full[st], pp.uses[st] & 1u);
    if (active) {
      // whole-row tiles are packed with row length inner == tn
      const double* x = ring + int64_t(st) * kTileD + g * cj * tw + tl;
      if (u_smem) {
        for (int64_t jj = 0; jj < jn; ++jj) {
          const double xv = x[jj * tw];
          if (norm_acc) nrm = fma(xv, xv, nrm);
          const double* ur = Ut + (j0 + jj) * R;
#pragma unroll
          for (int a = 0; a < R; ++a) acc[a] = fma(ur[a], xv, acc[a]);
        }
      } else {
        for (int64_t jj = 0; jj < jn; ++jj) {
          const double xv = x[jj * tw];
          if (norm_acc) nrm = fma(xv, xv, nrm);
#pragma unroll
          for (int a = 0; a < R; ++a) acc[a] = fma(__ldg(U + (j0 + jj) + a * d), xv, acc[a]);
        }
      }
      if (jt == njt - 1) {
        double* dst = out + (o0 + g) * r * inner + t0 + tl;
#pragma unroll
        for (int a = 0; a < R; ++a) dst[a * inner] = acc[a];
      }
    }
    fence_proxy_async();
    __syncthreads();  // every thread is done with stage st
    if (threadIdx.x == 0) pp.uses[st] += 1;
    if (threadIdx.x < 32 && t + kStages < ntiles) issue(t + kStages);
  }
  if (norm_acc) *norm_acc += nrm;
  __syncthreads();
}

__device__ __forceinline__ void ttm_stream(const double* in, int64_t outer, int64_t d, int64_t inner, const double* U,
                                           int r, double* out, double* dyn, Pipe& pp, double* norm_acc,
                                           const void* tmap, int tmap_rank) {
  switch (r) {
#define TT_CASE(N) \
  case N:          \
    ttm_stream_r<N>(in, outer, d, inner, U, out, dyn, pp, norm_acc, tmap, tmap_rank); \
    break;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10) TT_CASE(11) TT_CASE(12) TT_CASE(13) TT_CASE(14) TT_CASE(15) TT_CASE(16)
#undef TT_CASE
    default:
      break;
  }
}

__device__ __forceinline__ bool stream_ok(const double* in, int64_t inner, int r) {
  const int64_t tw = imin(inner, 256);
  return r <= 16 && ((reinterpret_cast<uintptr_t>(in) & 15u) == 0) && ((inner * 8) % 16 == 0) && ((tw * 8) % 16 == 0);
}

// Thread-per-output-element mode product, for shapes with few output columns.
__device__ __forceinline__ void ttm_elems(const double* __restrict__ in, int64_t outer, int64_t d, int64_t inner,
                                          const double* __restrict__ M, int64_t ms_a, int64_t ms_j, int64_t r,
                                          double* __restrict__ out, bool acc) {
  const int64_t tot = outer * r * inner;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t t = e % inner;
    const int64_t q = e / inner;
    const int64_t a = q % r, o = q / r;
    const double* src = in + o * d * inner + t;
    const double* ma = M + a * ms_a;
    double s = 0.0;
    for (int64_t j = 0; j < d; ++j) s = fma(ma[j * ms_j], src[j * inner], s);
    out[e] = acc ? out[e] + s : s;
  }
  __syncthreads();
}

// Dispatch: column-parallel when there are enough output columns.
__device__ __forceinline__ void mode_product(const double* in, int64_t outer, int64_t d, int64_t inner,
                                             const double* M, int64_t ms_a, int64_t ms_j, int64_t r, double* out,
                                             bool acc, BlockScratch& sc, int slot = kPhTtm) {
  const long long t0 = tstart();
  if (outer * inner >= 2 * int64_t(blockDim.x))
    ttm(in, outer, d, inner, M, ms_a, ms_j, r, out, acc);
  else
    ttm_elems(in, outer, d, inner, M, ms_a, ms_j, r, out, acc);
  tstop(sc, slot, t0);
}

// A Gram eigenvalue carries an absolute rounding error ~eps * lambda_max, so
// singular values below ~sqrt(1e-13) * sigma_max are numerically zero: their
// columns are completed orthonormally instead of amplified noise.
__device__ __forceinline__ bool gram_sigma_ok(double lam, double lam_max) {
  return lam > 1e-13 * lam_max && lam > 0.0;
}

__device__ __forceinline__ void tgemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t ars, int64_t acs,
                                      const double* B, int64_t brs, int64_t bcs, double* C, int64_t crs, int64_t ccs,
                                      bool acc, BlockScratch& sc) {
  const long long t0 = tstart();
  gemm(M, N, K, A, ars, acs, B, brs, bcs, C, crs, ccs, acc, sc);
  tstop(sc, kPhGemm, t0);
}

// Runs the Jacobi solver on G (n x n), staging through shared memory when it
// fits. Returns the pointer holding the eigenvectors; *diag receives the
// pointer to the diagonalised matrix.
__device__ double* eig_run(double* G, int n, double* V, int* order, double* dsm, double** diag, BlockScratch& sc) {
  int sw;
  double* res;
  const long long t0 = tstart();
  if (n <= kFastEigN && 3 * n * n <= sc.dsm_cap) {
    bcopy(dsm, G, int64_t(n) * n);
    sw = sym_eig_smem(dsm, n, order, sc);
    *diag = dsm;
    res = dsm + 2 * n * n;
  } else if (2 * n * n <= sc.dsm_cap) {
    double* As = dsm;
    double* Vs = dsm + n * n;
    bcopy(As, G, int64_t(n) * n);
    sw = sym_eig(As, n, Vs, order, sc);
    *diag = As;
    res = Vs;
  } else {
    sw = sym_eig(G, n, V, order, sc);
    *diag = G;
    res = V;
  }
  if (threadIdx.x == 0) {
    sc.eig_calls += 1;
    sc.eig_sweeps += sw;
  }
  tstop(sc, kPhEig, t0);
  return res;
}

// ---------------------------------------------------------------------------
// Block subspace iteration for the top-k left singular subspace of a tall
// unfolding A (rows x cols, cols >= 2k), warm-started from the factor's current
// value. Each iteration: Y = A^T U, B = Y^T Y (= U^T A A^T U), W = A Y; stop
// when ||W - U B||_F <= 1e-13 ||B||_F (the subspace is then accurate to
// ~1e-13 lambda_1 / gap); otherwise U = orth(W) by CholeskyQR2. A Rayleigh-Ritz
// rotation by the eigenvectors of B then gives the exact top-k singular
// vectors, identical (to rounding) to the SVD route of the reference. Returns
// false — the caller falls back to Gram + Jacobi — when it does not converge in
// kSiMaxIter iterations or CholeskyQR breaks down (rank deficiency, tiny gap).
constexpr int kSiMaxIter = 40;
// start of the subspace-iteration state in dynamic shared memory: after the
// per-warp partial sums (nwarps x kSiMaxYK) and the Rayleigh-Ritz eigensolver
// scratch (3 * 16^2)
__device__ __forceinline__ constexpr int si_base() { return kWarps * 512; }
constexpr int kSiMaxK = 16;     // register-tile bound on k
constexpr int kSiMaxYK = 512;   // bound on cols * k (16 outputs per lane)

// Warp 0 factors the SPD k x k matrix G = L L^T and writes Linv = L^{-1}
// (both col-major, lower). Sets sc.ibcast[2] = 1 on a failed pivot.
__device__ void chol_inv_warp(const double* G, int k, double* L, double* Linv, BlockScratch& sc) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double dmax = 0.0;
  for (int j = 0; j < k; ++j) dmax = fmax(dmax, G[j + j * k]);
  bool ok = dmax > 0.0;
  for (int j = 0; j < k && ok; ++j) {
    double sdiag = 0.0;
    if (lane == j) {
      sdiag = G[j + j * k];
      for (int l = 0; l < j; ++l) sdiag -= L[j + l * k] * L[j + l * k];
    }
    sdiag = __shfl_sync(0xffffffffu, sdiag, j);
    // A rank-deficient Gram has pivots ~eps*dmax; a basis with condition
    // number <= ~1e7 keeps them >= 1e-14*dmax. Anything smaller falls back.
    if (!(sdiag > 1e-14 * dmax)) {
      ok = false;
      break;
    }
    const double ljj = sqrt(sdiag), inv = 1.0 / ljj;
    if (lane > j && lane < k) {
      double v = G[lane + j * k];
      for (int l = 0; l < j; ++l) v -= L[lane + l * k] * L[j + l * k];
      L[lane + j * k] = v * inv;
    }
    if (lane == j) L[j + j * k] = ljj;
    __syncwarp();
  }
  if (!ok) {
    if (lane == 0) sc.ibcast[2] = 1;
    return;
  }
  if (lane < k) {  // column `lane` of L^{-1} by forward substitution
    const int c = lane;
    for (int i = 0; i < c; ++i) Linv[i + c * k] = 0.0;
    for (int i = c; i < k; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int l = c; l < i; ++l) v -= L[i + l * k] * Linv[l + c * k];
      Linv[i + c * k] = v / L[i + i * k];
    }
  }
}

// W (rows x K, ld rows) <- W L^{-T}, where W^T W = L L^T (one CholeskyQR pass).
template <int K>
__device__ __noinline__ bool cholqr_pass_k(double* W, int64_t rows, double* small, BlockScratch& sc) {
  double* G = small;
  double* L = small + K * K;
  double* Li = small + 2 * K * K;
  gram_tall(W, rows, rows, K, G);
  if (threadIdx.x == 0) sc.ibcast[2] = 0;
  __syncthreads();
  chol_inv_warp(G, K, L, Li, sc);
  __syncthreads();
  if (sc.ibcast[2]) return false;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    double w[K];
#pragma unroll
    for (int l = 0; l < K; ++l) w[l] = W[r + l * rows];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double v = 0.0;
#pragma unroll
      for (int l = 0; l <= j; ++l) v = fma(w[l], Li[j + l * K], v);
      W[r + j * rows] = v;
    }
  }
  __syncthreads();
  return true;
}

// Y (cols x K) = A^T U with A(i, c) = P[offc[c] + i*inner]: warps split the
// rows, each lane keeps up to 16 outputs in registers (row-outer loop, so the
// loads of a row are independent), partials reduced through shared memory.
template <int K>
__device__ __noinline__ void unfold_At_U_k(const double* __restrict__ P, const int* __restrict__ offc, int64_t rows,
                                           int64_t inner, int cols, const double* __restrict__ U,
                                           double* __restrict__ Y, double* part) {
  constexpr int OPL = 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = int(blockDim.x >> 5);
  const int ne = cols * K;
  const int64_t chunk = (rows + nw - 1) / nw;
  const int64_t i0 = warp * chunk, i1 = imin(rows, i0 + chunk);
  for (int e0 = 0; e0 < ne; e0 += 32 * OPL) {
    double acc[OPL];
    int oc[OPL], oj[OPL];
#pragma unroll
    for (int u = 0; u < OPL; ++u) {
      const int e = e0 + lane + 32 * u;
      const int ee = e < ne ? e : 0;
      oc[u] = offc[ee % cols];
      oj[u] = (ee / cols) * int(rows);
      acc[u] = 0.0;
    }
    const int nu = imin(OPL, (ne - e0 - lane + 31) / 32);
    for (int64_t i = i0; i < i1; ++i) {
      const double* Pi = P + i * inner;
      const double* Ui = U + i;
#pragma unroll
      for (int u = 0; u < OPL; ++u)
        if (u < nu) acc[u] = fma(Pi[oc[u]], Ui[oj[u]], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < OPL; ++u) {
      const int e = e0 + lane + 32 * u;
      if (u < nu && e < ne) part[warp * ne + e] = acc[u];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += part[w * ne + e];
    Y[e] = v;  // e = c + j*cols: column-major cols x K
  }
  __syncthreads();
}

template <int K>
__device__ __noinline__ int llsv_subspace_k(const double* P, int64_t outer, int64_t rows, int64_t inner, int kprev,
                                            double* U, double* si, double* dsm, double* misc, BlockScratch& sc) {
  const int cols = int(outer * inner);
  // shared-memory carve-up: [0, si_base) partial sums / eigensolver scratch,
  // then Y (cols x K), the small K x K matrices and the column-offset table
  double* W = si;                          // rows x K (global workspace)
  double* Y = dsm + si_base();             // cols x K   (<= 512)
  double* small = Y + kSiMaxYK;            // 4 K x K
  double* B = small + 4 * K * K;           // K x K
  int* offc = reinterpret_cast<int*>(B + K * K);  // <= 512 ints
  for (int c = threadIdx.x; c < cols; c += blockDim.x) offc[c] = int((c / inner) * rows * inner + (c % inner));
  if (kprev < K) {  // warm start padded with canonical vectors
    for (int64_t idx = threadIdx.x; idx < rows * (K - kprev); idx += blockDim.x) {
      const int64_t r = idx % rows, c = kprev + idx / rows;
      U[r + c * rows] = (r == (c * 7919) % rows) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (!cholqr_pass_k<K>(U, rows, small, sc) || !cholqr_pass_k<K>(U, rows, small, sc)) return -1;
  } else {
    __syncthreads();
  }
  int iters = -1;
  for (int it = 0; it < kSiMaxIter; ++it) {
    long long tp = tstart();
    unfold_At_U_k<K>(P, offc, rows, inner, cols, U, Y, dsm);
    gram_tall(Y, cols, cols, K, B);
    tstop(sc, kSiAtU, tp);
    tp = tstart();
    double rsq = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      double acc[K], u[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        acc[j] = 0.0;
        u[j] = U[i + j * rows];
      }
      const double* Pi = P + i * inner;
      for (int c = 0; c < cols; ++c) {
        const double a = Pi[offc[c]];
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = fma(a, Y[c + j * cols], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        W[i + j * rows] = acc[j];
        double v = acc[j];  // residual (W - U B)[i, j]
#pragma unroll
        for (int l = 0; l < K; ++l) v = fma(-u[l], B[l + j * K], v);
        rsq = fma(v, v, rsq);
      }
    }
    double bsq = 0.0;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) bsq = fma(B[e], B[e], bsq);
    rsq = block_sum(rsq, sc);
    bsq = block_sum(bsq, sc);
    tstop(sc, kSiAY, tp);
    if (bsq > 0.0 && rsq <= 1e-26 * bsq) {
      iters = it + 1;
      break;
    }
    if (!(bsq > 0.0)) return -1;
    tp = tstart();
    if (!cholqr_pass_k<K>(W, rows, small, sc) || !cholqr_pass_k<K>(W, rows, small, sc)) return -1;
    for (int64_t idx = threadIdx.x; idx < rows * K; idx += blockDim.x) U[idx] = W[idx];
    __syncthreads();
    tstop(sc, kSiQR, tp);
  }
  const long long trr = tstart();
  if (iters < 0) return -1;
  // Rayleigh-Ritz: U <- U R with B R = R diag(lambda), descending
  int* order = reinterpret_cast<int*>(misc);
  double* diag = nullptr;
  const double* R = eig_run(B, K, small, order, dsm, &diag, sc);
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    double u[K];
#pragma unroll
    for (int l = 0; l < K; ++l) u[l] = U[i + l * rows];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const double* rj = R + int64_t(order[j]) * K;
      double v = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) v = fma(u[l], rj[l], v);
      W[i + j * rows] = v;
    }
  }
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < rows * K; idx += blockDim.x) U[idx] = W[idx];
  __syncthreads();
  sign_fix(U, rows, K, rows, nullptr, sc);
  tstop(sc, kSiRR, trr);
  return iters;
}

__device__ bool llsv_subspace(const double* P, int64_t outer, int64_t rows, int64_t inner, int k, int kprev, double* U,
                              double* si, double* dsm, double* misc, BlockScratch& sc) {
  int it = -1;
  switch (k) {
#define TT_CASE(N) \
  case N:          \
    it = llsv_subspace_k<N>(P, outer, rows, inner, kprev, U, si, dsm, misc, sc); \
    break;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10) TT_CASE(11) TT_CASE(12) TT_CASE(13) TT_CASE(14) TT_CASE(15) TT_CASE(16)
#undef TT_CASE
    default:
      break;
  }
  if (threadIdx.x == 0 && it > 0) sc.si_iters += it;
  return it > 0;
}

// leading_left_singular_vectors (linalg.cpp:45-64) of the mode unfolding of a
// row-major (outer, rows, inner) tensor, through the Gram matrix of its
// smaller side. U: rows x k (ld rows), sign-fixed.
__device__ void llsv_unfold(const double* P, int64_t outer, int64_t rows, int64_t inner, int64_t k, double* U,
                            double* G, double* V, double* misc, double* dsm, BlockScratch& sc, int64_t kprev = 0,
                            double* si = nullptr) {
  const int64_t cols = outer * inner;
  if (si != nullptr && kprev > 0 && rows > cols && cols >= 2 * k && cols * k <= kSiMaxYK && k <= kSiMaxK &&
      si_base() + kSiMaxYK + 5 * k * k + 256 <= sc.dsm_cap) {
    const long long t0 = tstart();
    const bool ok = llsv_subspace(P, outer, rows, inner, int(k), int(imin(kprev, k)), U, si, dsm, misc, sc);
    tstop(sc, kPhEig, t0);
    if (ok) {
      if (threadIdx.x == 0) sc.si_ok += 1;
      return;
    }
    if (threadIdx.x == 0) sc.si_fail += 1;
  }
  int* order = reinterpret_cast<int*>(misc);
  double* sig = misc + kMisc / 2;
  double* diag = nullptr;
  if (rows <= cols) {
    const int n = int(rows);
    long long tg = tstart();
    gram_rows(P, outer, rows, inner, G);
    tstop(sc, kPhGram, tg);
    const double* Vp = eig_run(G, n, V, order, dsm, &diag, sc);
    for (int64_t idx = threadIdx.x; idx < rows * k; idx += blockDim.x) {
      const int64_t i = idx % rows, c = idx / rows;
      U[idx] = Vp[i + int64_t(order[c]) * n];
    }
    __syncthreads();
  } else {
    const int n = int(cols);
    long long tg = tstart();
    gram_cols(P, outer, rows, inner, G);
    tstop(sc, kPhGram, tg);
    const double* Vp = eig_run(G, n, V, order, dsm, &diag, sc);
    if (threadIdx.x < k) {
      const double l0 = fmax(diag[order[0] * (n + 1)], 0.0);
      const double lc = fmax(diag[order[threadIdx.x] * (n + 1)], 0.0);
      sig[threadIdx.x] = gram_sigma_ok(lc, l0) ? 1.0 / sqrt(lc) : 0.0;
    }
    __syncthreads();
    tg = tstart();
    for (int64_t idx = threadIdx.x; idx < rows * k; idx += blockDim.x) {
      const int64_t i = idx % rows, c = idx / rows;
      const double inv = sig[c];
      double s = 0.0;
      if (inv != 0.0) {
        const double* vc = Vp + int64_t(order[c]) * n;
        for (int64_t o = 0; o < outer; ++o) {
          const double* a = P + (o * rows + i) * inner;
          const double* v = vc + o * inner;
          for (int64_t t = 0; t < inner; ++t) s = fma(a[t], v[t], s);
        }
      }
      U[idx] = s * inv;
    }
    __syncthreads();
    tstop(sc, kPhGram, tg);
    const long long to = tstart();
    orthonormalize(U, rows, 0, int(k), rows, sc);
    tstop(sc, kPhOrtho, to);
  }
  const long long ts = tstart();
  sign_fix(U, rows, int(k), rows, nullptr, sc);
  tstop(sc, kPhOrtho, ts);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2) leaf_als_kernel(Params prm, const LeafDesc* __restrict__ descs) {
  __shared__ BlockScratch sc;
  __shared__ Pipe pipe;
  extern __shared__ __align__(128) double dsm[];
  const long long t_kernel = tstart();
  if (threadIdx.x == 0) {
    sc.eig_calls = sc.eig_sweeps = sc.si_ok = sc.si_fail = sc.si_iters = 0;
    sc.dsm_cap = int(dyn_smem_doubles());
    for (int i = 0; i < 12; ++i) sc.cyc[i] = 0;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&pipe.full[i], 1);
      pipe.uses[i] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  const LeafDesc D = descs[blockIdx.x];
  const int p = prm.p;
  int64_t d[kMaxP], rc[kMaxP], k[kMaxP];
  d[0] = D.len;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, rc);
  const LeafWs lay = leaf_ws_layout(p, D.len, prm.d, prm.req);
  double* W = D.ws + lay.W;
  double* B[2] = {D.ws + lay.B1, D.ws + lay.B2};
  double* G = D.ws + lay.G;
  double* V = D.ws + lay.V;
  double* misc = D.ws + lay.misc;
  const double* X = D.x;
  const int64_t ns = prod_range(d, 1, p);
  for (int n = 0; n < p; ++n) {
    bcopy(D.out_f[n], D.init[n], d[n] * rc[n]);
    k[n] = rc[n];
  }
  int sweeps = 0, converged = 0;
  double norm_sq = 0.0, norm = 0.0;
  double prev_fit = nan("");
  for (int sweep = 0; sweep < prm.max_iters; ++sweep) {
    // ---- mode 0: Y = X x_1 U_1^T ... x_{p-1} U_{p-1}^T, U_0 = llsv(M_0(Y))
    const int64_t k0n = leaf_mode_rank(p, d, k, 0);
    int64_t cur[kMaxP];
    for (int m = 0; m < p; ++m) cur[m] = d[m];
    const double* src = X;
    int tog = 0;
    for (int m = 1; m < p; ++m) {
      double* dst = B[tog];
      const int64_t inner = prod_range(cur, m + 1, p);
      if (m == 1 && stream_ok(X, inner, int(k[1]))) {
        // first contraction streams X through the TMA ring; sweep 0 also
        // accumulates ||X||^2 (tucker.cpp:96)
        const long long tb = tstart();
        double nacc = 0.0;
        ttm_stream(X, d[0], d[1], inner, D.out_f[1], int(k[1]), dst, dsm, pipe, sweep == 0 ? &nacc : nullptr,
                   D.tmaps, 3);
        if (sweep == 0) norm_sq = block_sum(nacc, sc);
        tstop(sc, kPhBig, tb);
      } else {
        if (m == 1 && sweep == 0) norm_sq = bsumsq(X, D.len * ns, sc);
        mode_product(src, prod_range(cur, 0, m), cur[m], inner, D.out_f[m], d[m], 1, k[m], dst, false, sc,
                     m == 1 ? kPhBig : kPhTtm);
      }
      cur[m] = k[m];
      src = dst;
      tog ^= 1;
    }
    if (sweep == 0) {
      if (norm_sq == 0.0) {  // tucker.cpp:96-100: init factors, zero core
        bzero(D.out_core, prod_range(rc, 0, p));
        converged = 1;
        break;
      }
      norm = sqrt(norm_sq);
    }
    llsv_unfold(src, 1, d[0], prod_range(cur, 1, p), k0n, D.out_f[0], G, V, misc, dsm, sc, k[0], D.ws + lay.SI);
    k[0] = k0n;
    // ---- W = X x_0 U_0^T : (k0, D_1, ..., D_{p-1})
    if (stream_ok(X, ns, int(k[0]))) {
      const long long tb = tstart();
      ttm_stream(X, 1, d[0], ns, D.out_f[0], int(k[0]), W, dsm, pipe, nullptr,
                 D.tmaps ? static_cast<const char*>(D.tmaps) + 128 : nullptr, 2);
      tstop(sc, kPhBig, tb);
    } else {
      mode_product(X, 1, d[0], ns, D.out_f[0], d[0], 1, k[0], W, false, sc, kPhBig);
    }
    // ---- modes n >= 1 from W
    const double* Pn = W;
    int64_t pc[kMaxP];
    for (int n = 1; n < p; ++n) {
      const int64_t kn = leaf_mode_rank(p, d, k, n);
      pc[0] = k[0];
      for (int m = 1; m < p; ++m) pc[m] = d[m];
      const double* s2 = W;
      int t2 = 0;
      for (int m = 1; m < p; ++m) {
        if (m == n) continue;
        double* dst = B[t2];
        mode_product(s2, prod_range(pc, 0, m), pc[m], prod_range(pc, m + 1, p), D.out_f[m], d[m], 1, k[m], dst,
                     false, sc);
        pc[m] = k[m];
        s2 = dst;
        t2 ^= 1;
      }
      llsv_unfold(s2, prod_range(pc, 0, n), d[n], prod_range(pc, n + 1, p), kn, D.out_f[n], G, V, misc, dsm, sc,
                  k[n], D.ws + lay.SI);
      k[n] = kn;
      Pn = s2;
    }
    // ---- core = P_{p-1} x_{p-1} U_{p-1}^T  (== core_of(x, U), tucker.cpp:67-76)
    mode_product(Pn, prod_range(k, 0, p - 1), d[p - 1], 1, D.out_f[p - 1], d[p - 1], 1, k[p - 1], D.out_core,
                 false, sc);
    const double core_sq = bsumsq(D.out_core, prod_range(k, 0, p), sc);
    const double res = fmax(0.0, norm_sq - core_sq);
    if (threadIdx.x == 0) D.objective[sweep] = res;
    sweeps = sweep + 1;
    const double fit = 1.0 - sqrt(res) / norm;
    if (sweep > 0 && fabs(fit - prev_fit) < prm.tol) {
      converged = 1;
      break;
    }
    prev_fit = fit;
  }
  if (threadIdx.x == 0) {
    D.status[0] = sweeps;
    D.status[1] = converged;
    D.status[2] = norm_sq == 0.0;
    D.status[3] = 0;
    for (int m = 0; m < kMaxP; ++m) D.status[4 + m] = m < p ? int(k[m]) : 0;
    D.status[4 + kMaxP] = sc.eig_calls;
    D.status[5 + kMaxP] = sc.eig_sweeps;
#ifdef TT_INSTRUMENT
    sc.cyc[kPhAll] = clock64() - t_kernel;
#else
    (void)t_kernel;
#endif
    for (int i = 0; i < 8; ++i) D.status[6 + kMaxP + i] = int(sc.cyc[i] >> 10);
    D.status[14 + kMaxP] = sc.si_ok;
    D.status[15 + kMaxP] = sc.si_fail;
    D.status[16 + kMaxP] = sc.si_iters;
    for (int i = 0; i < 4; ++i) D.status[17 + kMaxP + i] = int(sc.cyc[8 + i] >> 10);
  }
}

// ---------------------------------------------------------------------------
// U_0 = blockdiag(V_sub,i) [E_i]  (L x K0, ld L), sign-fixed (linalg.cpp:15-31).
// Pass 0 evaluates the rows without storing and finds each column's first
// max-|.| row; pass 1 recomputes and stores U_0 once with the signs applied.
// Two rows per thread are in flight, E_i is staged in shared memory.
template <int K0>
__device__ __noinline__ void materialize_u0_k(const StitchPart* __restrict__ parts, int s, const double* Ebase,
                                              int64_t e_stride, double* __restrict__ U0, int64_t L, int* flips,
                                              int64_t* idxbuf, double* Es, BlockScratch& sc) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nt = int(blockDim.x);
  for (int pass = 0; pass < 2; ++pass) {
    double best[K0], sg[K0];
    int64_t bidx[K0];
#pragma unroll
    for (int c = 0; c < K0; ++c) {
      best[c] = -1.0;
      bidx[c] = 0;
      sg[c] = (pass == 1 && flips[c]) ? -1.0 : 1.0;
    }
    int64_t off = 0;
    for (int i = 0; i < s; ++i) {
      const int64_t r0 = parts[i].rho[0], len = parts[i].len, ld = parts[i].ld0;
      const double* vs = parts[i].v0 + parts[i].row0;
      const double* E = Ebase + int64_t(i) * e_stride;
      __syncthreads();
      for (int64_t e = threadIdx.x; e < r0 * K0; e += nt) Es[e] = E[e];
      __syncthreads();
      for (int64_t rb = threadIdx.x; rb < len; rb += 2 * nt) {
        const int64_t ra = rb, rc = rb + nt;
        const bool has_c = rc < len;
        double oa[K0], ob[K0];
#pragma unroll
        for (int c = 0; c < K0; ++c) oa[c] = ob[c] = 0.0;
        for (int64_t a = 0; a < r0; ++a) {
          const double va = vs[ra + a * ld];
          const double vb = has_c ? vs[rc + a * ld] : 0.0;
#pragma unroll
          for (int c = 0; c < K0; ++c) {
            const double ev = Es[a + c * r0];
            oa[c] = fma(va, ev, oa[c]);
            ob[c] = fma(vb, ev, ob[c]);
          }
        }
        if (pass == 1) {
#pragma unroll
          for (int c = 0; c < K0; ++c) {
            U0[off + ra + c * L] = sg[c] * oa[c];
            if (has_c) U0[off + rc + c * L] = sg[c] * ob[c];
          }
        } else {
#pragma unroll
          for (int c = 0; c < K0; ++c) {
            const double ma = fabs(oa[c]);
            if (ma > best[c]) {
              best[c] = ma;
              bidx[c] = off + ra;
              sg[c] = oa[c];
            }
            const double mb = has_c ? fabs(ob[c]) : -1.0;
            if (mb > best[c]) {  // rc > ra: a tie keeps the earlier row
              best[c] = mb;
              bidx[c] = off + rc;
              sg[c] = ob[c];
            }
          }
        }
      }
      off += len;
    }
    if (pass == 0) {
#pragma unroll
      for (int c = 0; c < K0; ++c) {
        double b = best[c], v = sg[c];
        int64_t bi = bidx[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, b, o);
          const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
          const double ov = __shfl_xor_sync(0xffffffffu, v, o);
          if (ob > b || (ob == b && oi < bi)) {
            b = ob;
            bi = oi;
            v = ov;
          }
        }
        if (l == 0) {
          sc.red[w * kMaxVec + c] = b;
          idxbuf[w * kMaxVec + c] = v < 0.0 ? -(bi + 1) : (bi + 1);
        }
      }
      __syncthreads();
      if (threadIdx.x < K0) {
        const int c = threadIdx.x;
        double b = sc.red[c];
        int64_t bi = idxbuf[c];
        for (int ww = 1; ww < kWarps; ++ww) {
          const double ob = sc.red[ww * kMaxVec + c];
          const int64_t oi = idxbuf[ww * kMaxVec + c];
          const int64_t ai = bi < 0 ? -bi : bi, ao = oi < 0 ? -oi : oi;
          if (ob > b || (ob == b && ao < ai)) {
            b = ob;
            bi = oi;
          }
        }
        flips[c] = bi < 0;
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

__device__ bool materialize_u0(int k0, const StitchPart* parts, int s, const double* Ebase, int64_t e_stride,
                               double* U0, int64_t L, int* flips, int64_t* idxbuf, double* Es, BlockScratch& sc) {
  switch (k0) {
#define TT_CASE(N) \
  case N:          \
    materialize_u0_k<N>(parts, s, Ebase, e_stride, U0, L, flips, idxbuf, Es, sc); \
    return true;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10) TT_CASE(11) TT_CASE(12) TT_CASE(13) TT_CASE(14) TT_CASE(15) TT_CASE(16)
#undef TT_CASE
    default:
      return false;
  }
}

// ---------------------------------------------------------------------------
struct PartView {
  const double* core;
  int64_t rho[kMaxP];
  const double* v0;
  int64_t ld0, row0, len;
  int partial;
  const double* v[kMaxP];
};

__device__ __forceinline__ PartView load_part(const StitchPart& s) {
  PartView v;
  v.core = s.core;
  for (int m = 0; m < kMaxP; ++m) {
    v.rho[m] = s.rho[m];
    v.v[m] = s.v[m];
  }
  v.v0 = s.v0;
  v.ld0 = s.ld0;
  v.row0 = s.row0;
  v.len = s.len;
  v.partial = s.partial;
  return v;
}

__global__ void __launch_bounds__(kStitchThreads, 2)
    stitch_als_kernel(Params prm, const StitchDesc* __restrict__ descs, const StitchPart* __restrict__ parts_all) {
  __shared__ BlockScratch sc;
  __shared__ int flips[kMaxVec];
  __shared__ int64_t idxbuf[kWarps * kMaxVec];
  extern __shared__ double dsm[];
  const long long t_kernel = tstart();
  if (threadIdx.x == 0) {
    sc.eig_calls = sc.eig_sweeps = sc.si_ok = sc.si_fail = sc.si_iters = 0;
    sc.dsm_cap = int(dyn_smem_doubles());
    for (int i = 0; i < 12; ++i) sc.cyc[i] = 0;
  }
  const StitchDesc D = descs[blockIdx.x];
  const StitchPart* parts = parts_all + D.part0;
  const int p = prm.p, s = D.nparts;
  int64_t d[kMaxP], rc[kMaxP], k[kMaxP], rho_max[kMaxP], rcx[kMaxP];
  d[0] = D.L;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, rc);
  for (int m = 0; m < p; ++m) rho_max[m] = 0;
  for (int i = 0; i < s; ++i)
    for (int m = 0; m < p; ++m) rho_max[m] = imax(rho_max[m], parts[i].rho[m]);
  for (int m = 0; m < p; ++m) rcx[m] = imax(rc[m], rho_max[m]);
  const StitchWs lay = stitch_ws_layout(p, D.L, prm.d, prm.req, rho_max, s);
  double* ws = D.ws;
  double* T[2] = {ws + lay.T1, ws + lay.T2};
  double* G = ws + lay.G;
  double* Vg = ws + lay.V;
  double* Z = ws + lay.Z;
  double* misc = ws + lay.misc;
  double* wk = ws + lay.WK;  // Q x k0 scaled eigenvectors
  double* HH = ws + lay.HH;  // rho0 x rho0 scratch
  auto Pm = [&](int i, int m) {  // P_im = U_m^T V_im, k_m x rho_im (ld k_m)
    int64_t off = 0;
    for (int q = 1; q < m; ++q) off += rc[q] * rcx[q];
    return ws + lay.P + int64_t(i) * lay.per_part_P + off;
  };
  auto Cp = [&](int i) { return ws + lay.C + int64_t(i) * lay.per_part_C; };
  auto Sp = [&](int i) { return ws + lay.S + int64_t(i) * lay.per_part_S; };
  auto Ep = [&](int i) { return ws + lay.E + int64_t(i) * lay.per_part_E; };
  auto Ap = [&](int i) { return ws + lay.A + int64_t(i) * lay.per_part_E; };
  auto E2p = [&](int i) { return ws + lay.E2 + int64_t(i) * lay.per_part_E; };

  // ---- partial-hit metric S_i = Vsub^T Vsub and the norm of the implied tensor
  double norm_sq = 0.0;
  for (int i = 0; i < s; ++i) {
    const PartView pv = load_part(parts[i]);
    const int64_t r0 = pv.rho[0];
    const int64_t hk = prod_range(pv.rho, 1, p);
    if (pv.partial) {
      const double* vs = pv.v0 + pv.row0;
      {
        const long long tg = tstart();
        gram_tall(vs, pv.ld0, pv.len, int(r0), Sp(i));
        tstop(sc, kPhGram, tg);
      }
      // ||H x_0 R||^2 = sum_ab S_ab (M0(H) M0(H)^T)_ab
      tgemm(r0, r0, hk, pv.core, hk, 1, pv.core, 1, hk, HH, 1, r0, false, sc);
      double acc = 0.0;
      for (int64_t e = threadIdx.x; e < r0 * r0; e += blockDim.x) acc = fma(Sp(i)[e], HH[e], acc);
      norm_sq += block_sum(acc, sc);
    } else {
      norm_sq += bsumsq(pv.core, r0 * hk, sc);
    }
  }
  // ---- init (stitch.cpp:135-144): U_m = random_orthonormal(D_m, r_m), m >= 1
  for (int m = 1; m < p; ++m) {
    bcopy(D.out_f[m], prm.stitch_init[m], d[m] * rc[m]);
    k[m] = rc[m];
  }
  k[0] = rc[0];
  int sweeps = 0, converged = 0, any_zero_sigma = 0;
  if (norm_sq == 0.0) {  // stitch.cpp:146-150; U_0 is drawn by the host
    bzero(D.out_core, prod_range(rc, 0, p));
    converged = 1;
  } else {
    for (int i = 0; i < s; ++i) {
      const PartView pv = load_part(parts[i]);
      for (int m = 1; m < p; ++m)
        tgemm(k[m], pv.rho[m], d[m], D.out_f[m], d[m], 1, pv.v[m], 1, d[m], Pm(i, m), 1, k[m], false, sc);
    }
    const double norm = sqrt(norm_sq);
    double prev_fit = nan("");
    for (int sweep = 0; sweep < prm.max_iters; ++sweep) {
      // ================= mode 0 (stitch_temporal_unfolding, stitch.cpp:49-73)
      const int64_t k0n = stitch_mode_rank(p, d, rc, k, 0);
      const int64_t Q = prod_range(k, 1, p);
      for (int i = 0; i < s; ++i) {
        const PartView pv = load_part(parts[i]);
        int64_t cur[kMaxP];
        for (int m = 0; m < p; ++m) cur[m] = pv.rho[m];
        const double* src = pv.core;
        int tog = 0;
        for (int m = p - 1; m >= 1; --m) {  // descending, as the reference
          double* dst = (m == 1) ? Cp(i) : T[tog];
          mode_product(src, prod_range(cur, 0, m), cur[m], prod_range(cur, m + 1, p), Pm(i, m), 1, k[m], k[m],
                       dst, false, sc);
          cur[m] = k[m];
          src = dst;
          tog ^= 1;
        }
      }
      // ---- subspace iteration on the implicit Z0 in compressed coordinates:
      // U0 = blockdiag(V_sub,i) E with E^T S E = I; Z0 Z0^T U0 maps to
      // E <- C (C^T S E). Warm start: the previous sweep's E, or in sweep 0 the
      // k0 columns of C with the largest S-norm. Rayleigh-Ritz makes E the exact
      // left singular vectors; any failure falls through to the eigen paths.
      bool mode0_done = false;
      int64_t rho0_sum = 0;
      for (int i = 0; i < s; ++i) rho0_sum += parts[i].rho[0];
      if (k0n <= kSiMaxK && Q >= 2 * k0n && Q * k0n <= kSiMaxYK && rho0_sum >= k0n) {
        const long long t_si = tstart();
        double* Y = wk;                          // Q x k0
        double* small = dsm + si_base() + kSiMaxYK;  // 4 k x k (shared memory)
        double* B = small + 4 * k0n * k0n;       // k x k
        const int kk = int(k0n);
        auto apply_S = [&](int i, const double* X, double* out) {  // out = S_i X (rho0 x k)
          const int64_t r0 = parts[i].rho[0];
          if (parts[i].partial) {
            gemm(r0, kk, r0, Sp(i), 1, r0, X, 1, r0, out, 1, r0, false, sc);
          } else if (out != X) {
            bcopy(out, X, r0 * kk);
          }
        };
        // S-orthonormalise E (two CholeskyQR passes with the metric S)
        auto s_orth = [&]() -> bool {
          for (int pass = 0; pass < 2; ++pass) {
            double* G = small;
            double* L = small + kk * kk;
            double* Li = small + 2 * kk * kk;
            for (int i = 0; i < s; ++i) {
              const int64_t r0 = parts[i].rho[0];
              apply_S(i, Ep(i), Ap(i));
              gemm(kk, kk, r0, Ep(i), r0, 1, Ap(i), 1, r0, G, 1, kk, i > 0, sc);
            }
            if (threadIdx.x == 0) sc.ibcast[2] = 0;
            __syncthreads();
            chol_inv_warp(G, kk, L, Li, sc);
            __syncthreads();
            if (sc.ibcast[2]) return false;
            for (int i = 0; i < s; ++i) {
              const int64_t r0 = parts[i].rho[0];
              double* E = Ep(i);
              for (int64_t r = threadIdx.x; r < r0; r += blockDim.x) {
                double w[kSiMaxK];
#pragma unroll
                for (int l = 0; l < kSiMaxK; ++l) w[l] = l < kk ? E[r + l * r0] : 0.0;
                for (int j = 0; j < kk; ++j) {
                  double v = 0.0;
#pragma unroll
                  for (int l = 0; l < kSiMaxK; ++l)
                    if (l <= j) v = fma(w[l], Li[j + l * kk], v);
                  E[r + j * r0] = v;
                }
              }
            }
            __syncthreads();
          }
          return true;
        };
        bool ok = true;
        if (sweep == 0 || k[0] < k0n) {
          // start: the k0 columns of C with the largest S-norm
          double* cn = misc + kMisc / 2;  // Q norms
          for (int64_t j = threadIdx.x; j < Q; j += blockDim.x) cn[j] = 0.0;
          __syncthreads();
          for (int i = 0; i < s; ++i) {
            const int64_t r0 = parts[i].rho[0];
            const double* Ci = Cp(i);
            for (int64_t j = threadIdx.x; j < Q; j += blockDim.x) {
              double v = 0.0;
              if (parts[i].partial) {
                const double* S = Sp(i);
                for (int64_t a = 0; a < r0; ++a)
                  for (int64_t b = 0; b < r0; ++b) v = fma(Ci[a * Q + j] * S[a + b * r0], Ci[b * Q + j], v);
              } else {
                for (int64_t a = 0; a < r0; ++a) v = fma(Ci[a * Q + j], Ci[a * Q + j], v);
              }
              cn[j] += v;
            }
            __syncthreads();
          }
          int* pick = reinterpret_cast<int*>(misc);
          for (int64_t j = threadIdx.x; j < Q; j += blockDim.x) {
            int rank = 0;
            for (int64_t l = 0; l < Q; ++l) rank += (cn[l] > cn[j] || (cn[l] == cn[j] && l < j));
            if (rank < kk) pick[rank] = int(j);
          }
          __syncthreads();
          for (int i = 0; i < s; ++i) {
            const int64_t r0 = parts[i].rho[0];
            const double* Ci = Cp(i);
            double* E = Ep(i);
            for (int64_t idx = threadIdx.x; idx < r0 * kk; idx += blockDim.x) {
              const int64_t a = idx % r0, c = idx / r0;
              E[idx] = Ci[a * Q + pick[c]];
            }
          }
          __syncthreads();
          ok = s_orth();
        } else if (k[0] > k0n) {
          // previous E has more columns (ld rho0): keep the first k0n (same ld)
          ok = true;
        }
        bool conv = false;
        for (int it = 0; ok && it < kSiMaxIter; ++it) {
          // A_i = S_i E_i ; Y = sum_i C_i^T A_i (Q x k) ; B = Y^T Y ; W_i = C_i Y
          for (int i = 0; i < s; ++i) {
            const int64_t r0 = parts[i].rho[0];
            apply_S(i, Ep(i), Ap(i));
            gemm(Q, kk, r0, Cp(i), 1, Q, Ap(i), 1, r0, Y, 1, Q, i > 0, sc);
          }
          gram_tall(Y, Q, Q, kk, B);
          double rsq = 0.0;
          for (int i = 0; i < s; ++i) {
            const int64_t r0 = parts[i].rho[0];
            gemm(r0, kk, Q, Cp(i), Q, 1, Y, 1, Q, E2p(i), 1, r0, false, sc);
            // R = W - E B (into T[0]); rsq += <R, S R>
            double* R = T[0];
            for (int64_t idx = threadIdx.x; idx < r0 * kk; idx += blockDim.x) {
              const int64_t a = idx % r0, j = idx / r0;
              double v = E2p(i)[idx];
              for (int l = 0; l < kk; ++l) v = fma(-Ep(i)[a + l * r0], B[l + j * kk], v);
              R[idx] = v;
            }
            __syncthreads();
            double part = 0.0;
            if (parts[i].partial) {
              gemm(r0, kk, r0, Sp(i), 1, r0, R, 1, r0, HH, 1, r0, false, sc);
              for (int64_t idx = threadIdx.x; idx < r0 * kk; idx += blockDim.x) part = fma(R[idx], HH[idx], part);
            } else {
              for (int64_t idx = threadIdx.x; idx < r0 * kk; idx += blockDim.x) part = fma(R[idx], R[idx], part);
            }
            rsq += block_sum(part, sc);
          }
          double bsq = 0.0;
          for (int e = threadIdx.x; e < kk * kk; e += blockDim.x) bsq = fma(B[e], B[e], bsq);
          bsq = block_sum(bsq, sc);
          if (!(bsq > 0.0)) {
            ok = false;
            break;
          }
          if (rsq <= 1e-26 * bsq) {
            conv = true;
            if (threadIdx.x == 0) sc.si_iters += it + 1;
            break;
          }
          for (int i = 0; i < s; ++i) bcopy(Ep(i), E2p(i), parts[i].rho[0] * kk);
          ok = s_orth();
        }
        if (ok && conv) {
          // Rayleigh-Ritz: E <- E R (descending), then A_i = S_i E_i
          int* order = reinterpret_cast<int*>(misc);
          double* diag = nullptr;
          const double* R = eig_run(B, kk, small, order, dsm, &diag, sc);
          for (int i = 0; i < s; ++i) {
            const int64_t r0 = parts[i].rho[0];
            double* E = Ep(i);
            double* E2 = E2p(i);
            for (int64_t idx = threadIdx.x; idx < r0 * kk; idx += blockDim.x) {
              const int64_t a = idx % r0, j = idx / r0;
              const double* rj = R + int64_t(order[j]) * kk;
              double v = 0.0;
              for (int l = 0; l < kk; ++l) v = fma(E[a + l * r0], rj[l], v);
              E2[idx] = v;
            }
            __syncthreads();
            bcopy(E, E2, r0 * kk);
            if (parts[i].partial) apply_S(i, E, Ap(i));
          }
          any_zero_sigma = 0;
          mode0_done = true;
          if (threadIdx.x == 0) sc.si_ok += 1;
        } else if (threadIdx.x == 0) {
          sc.si_fail += 1;
        }
        tstop(sc, kPhEig, t_si);
      }
      // Row-compressed variant: with entire parts only, Z0 = blockdiag(V_i0) C
      // (C = [C_1; ...; C_s], sum rho_i0 rows) and V_i0 orthonormal, so the left
      // singular vectors of Z0 are blockdiag(V_i0) times the eigenvectors of
      // C C^T — a (sum rho_i0)^2 problem instead of Q^2 when that is smaller
      // (every two-part append stitch), with no Sigma^-1 amplification.
      int64_t rsum = 0;
      bool all_entire = true;
      for (int i = 0; i < s; ++i) {
        rsum += parts[i].rho[0];
        all_entire = all_entire && !parts[i].partial;
      }
      if (mode0_done) {
        // E_i, A_i already set by the subspace iteration
      } else if (all_entire && rsum < Q && k0n <= rsum) {  // else: rank-deficient Z0 needs the completion path
        int64_t oi = 0;
        for (int i = 0; i < s; ++i) {
          const int64_t ri = parts[i].rho[0];
          int64_t oj = 0;
          for (int j = 0; j < s; ++j) {
            const int64_t rj = parts[j].rho[0];
            // H[oi.., oj..] = C_i C_j^T
            tgemm(ri, rj, Q, Cp(i), Q, 1, Cp(j), 1, Q, G + oi + oj * rsum, 1, rsum, false, sc);
            oj += rj;
          }
          oi += ri;
        }
        int* order = reinterpret_cast<int*>(misc);
        double* diag = nullptr;
        const double* Vp = eig_run(G, int(rsum), Vg, order, dsm, &diag, sc);
        oi = 0;
        for (int i = 0; i < s; ++i) {
          const int64_t ri = parts[i].rho[0];
          double* E = Ep(i);
          for (int64_t idx = threadIdx.x; idx < ri * k0n; idx += blockDim.x) {
            const int64_t a = idx % ri, c = idx / ri;
            E[idx] = Vp[oi + a + int64_t(order[c]) * rsum];
          }
          oi += ri;
        }
        __syncthreads();
        any_zero_sigma = 0;
      } else {
        // G0 = Z0^T Z0 = sum_i C_i^T S_i C_i   (Q x Q)
        for (int i = 0; i < s; ++i) {
          const PartView pv = load_part(parts[i]);
          const int64_t r0 = pv.rho[0];
          const double* rhs = Cp(i);
          if (pv.partial) {
            tgemm(r0, Q, r0, Sp(i), 1, r0, Cp(i), Q, 1, T[0], Q, 1, false, sc);
            rhs = T[0];
          }
          tgemm(Q, Q, r0, Cp(i), 1, Q, rhs, Q, 1, G, 1, Q, i > 0, sc);
        }
        {
          int* order = reinterpret_cast<int*>(misc);
          double* sig = misc + kMisc / 2;
          double* diag = nullptr;
          if (threadIdx.x == 0) sc.ibcast[1] = 0;
          const double* Vp = eig_run(G, int(Q), Vg, order, dsm, &diag, sc);
          if (threadIdx.x < k0n) {
            const double l0 = fmax(diag[order[0] * (Q + 1)], 0.0);
            const double lc = fmax(diag[order[threadIdx.x] * (Q + 1)], 0.0);
            const bool ok = gram_sigma_ok(lc, l0);
            sig[threadIdx.x] = ok ? 1.0 / sqrt(lc) : 0.0;
            if (!ok) atomicOr(&sc.ibcast[1], 1);
          }
          __syncthreads();
          for (int64_t idx = threadIdx.x; idx < Q * k0n; idx += blockDim.x) {
            const int64_t j = idx % Q, c = idx / Q;
            wk[idx] = Vp[j + int64_t(order[c]) * Q] * sig[c];
          }
          __syncthreads();
          any_zero_sigma = sc.ibcast[1];
        }
        // E_i = C_i W Sigma^-1 (rho0 x k0);  A_i = S_i E_i = (U0[rows_i]^T V_i0)^T
        for (int i = 0; i < s; ++i) {
          const PartView pv = load_part(parts[i]);
          const int64_t r0 = pv.rho[0];
          tgemm(r0, k0n, Q, Cp(i), Q, 1, wk, 1, Q, Ep(i), 1, r0, false, sc);
          if (pv.partial) tgemm(r0, k0n, r0, Sp(i), 1, r0, Ep(i), 1, r0, Ap(i), 1, r0, false, sc);
        }
      }
      k[0] = k0n;
      // ================= modes n >= 1 (stitch_nontemporal_unfolding, stitch.cpp:75-108)
      for (int n = 1; n < p; ++n) {
        const int64_t kn = stitch_mode_rank(p, d, rc, k, n);
        int64_t zc[kMaxP];
        for (int m = 0; m < p; ++m) zc[m] = (m == n) ? d[n] : k[m];
        const int64_t zo = prod_range(zc, 0, n), zi = prod_range(zc, n + 1, p);
        // F_i = H_i x_0 (U0[rows_i]^T V_i0) x_{m != 0,n} P_im, shape (zo, rho_in, zi)
        const int64_t Qn = zo * zi;
        int64_t rho_n_sum = 0;
        for (int i = 0; i < s; ++i) rho_n_sum += parts[i].rho[n];
        // (two-part append stitches are faster part by part)
        const bool one_pass = rho_n_sum * Qn <= int64_t(sc.dsm_cap) && s >= 3 && s <= 64;
        for (int i = 0; i < s; ++i) {
          const PartView pv = load_part(parts[i]);
          int64_t cur[kMaxP];
          for (int m = 0; m < p; ++m) cur[m] = pv.rho[m];
          const double* A0 = pv.partial ? Ap(i) : Ep(i);
          int last = 0;  // last mode contracted in the chain
          for (int m = 1; m < p; ++m)
            if (m != n) last = m;
          // x_0 (U0[rows_i]^T V_i0): M(a, j) = A0[j + a*rho0]
          double* d0 = (one_pass && last == 0) ? Cp(i) : T[0];
          mode_product(pv.core, 1, cur[0], prod_range(cur, 1, p), A0, cur[0], 1, k[0], d0, false, sc);
          cur[0] = k[0];
          const double* src = d0;
          int tog = 1;
          for (int m = 1; m < p; ++m) {
            if (m == n) continue;
            double* dst = (one_pass && m == last) ? Cp(i) : T[tog];
            mode_product(src, prod_range(cur, 0, m), cur[m], prod_range(cur, m + 1, p), Pm(i, m), 1, k[m], k[m],
                         dst, false, sc);
            cur[m] = k[m];
            src = dst;
            tog ^= 1;
          }
          // per-part fallback: Z_n += F x_n V_in
          if (!one_pass) mode_product(src, zo, cur[n], zi, pv.v[n], 1, d[n], d[n], Z, i > 0, sc);
        }
        if (one_pass) {
          // Z_n = sum_i F_i x_n V_in written once: the stacked F (sum rho_in x Qn)
          // is staged in shared memory; a thread owns one row a of Z and 8
          // columns, streaming V_in[a, :] from global (coalesced over a).
          const long long tz = tstart();
          __shared__ const double* vptr[64];
          __shared__ int64_t foff[65];
          if (threadIdx.x == 0) {
            int64_t o = 0;
            for (int i = 0; i < s; ++i) {
              vptr[i] = parts[i].v[n];
              foff[i] = o;
              o += parts[i].rho[n];
            }
            foff[s] = o;
          }
          __syncthreads();
          double* Fs = dsm;
          for (int i = 0; i < s; ++i) {
            const int64_t rn = foff[i + 1] - foff[i];
            const double* F = Cp(i);
            for (int64_t e = threadIdx.x; e < rn * Qn; e += blockDim.x) {
              const int64_t j = e / Qn, c = e - j * Qn;
              const int64_t o = c / zi, t = c - o * zi;
              Fs[(foff[i] + j) * Qn + c] = F[(o * rn + j) * zi + t];
            }
          }
          __syncthreads();
          const int64_t dn = d[n];
          const int64_t ncb = (Qn + 7) / 8;
          for (int64_t w = threadIdx.x; w < dn * ncb; w += blockDim.x) {
            const int64_t a = w % dn, cb = w / dn;
            const int64_t c0 = cb * 8;
            double acc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = 0.0;
            for (int i = 0; i < s; ++i) {
              const double* V = vptr[i] + a;
              const int64_t j0 = foff[i], rn = foff[i + 1] - j0;
              for (int64_t j = 0; j < rn; ++j) {
                const double v = V[j * dn];
                const double* fr = Fs + (j0 + j) * Qn + c0;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                  if (c0 + c < Qn) acc[c] = fma(v, fr[c], acc[c]);
              }
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int64_t cc = c0 + c;
              if (cc < Qn) {
                const int64_t o = cc / zi, t = cc - o * zi;
                Z[(o * dn + a) * zi + t] = acc[c];
              }
            }
          }
          __syncthreads();
          tstop(sc, kPhTtm, tz);
        }
        llsv_unfold(Z, zo, d[n], zi, kn, D.out_f[n], G, Vg, misc, dsm, sc, k[n], ws + lay.SI);
        k[n] = kn;
        for (int i = 0; i < s; ++i) {
          const PartView pv = load_part(parts[i]);
          tgemm(k[n], pv.rho[n], d[n], D.out_f[n], d[n], 1, pv.v[n], 1, d[n], Pm(i, n), 1, k[n], false, sc);
        }
      }
      // ================= core: fold Z_{p-1} and project the last mode (stitch.cpp:163-172)
      mode_product(Z, prod_range(k, 0, p - 1), d[p - 1], 1, D.out_f[p - 1], d[p - 1], 1, k[p - 1], D.out_core,
                   false, sc);
      const double core_sq = bsumsq(D.out_core, prod_range(k, 0, p), sc);
      const double res = fmax(0.0, norm_sq - core_sq);
      if (threadIdx.x == 0) D.objective[sweep] = res;
      sweeps = sweep + 1;
      const double fit = 1.0 - sqrt(res) / norm;
      if (sweep > 0 && fabs(fit - prev_fit) < prm.tol) {
        converged = 1;
        break;
      }
      prev_fit = fit;
    }
    // ================= materialise U_0 = blockdiag(Vsub_i) [E_i] (L x k0), sign-fixed
    const int64_t k0 = k[0];
    double* U0 = D.out_f[0];
    const long long tu = tstart();
    if (any_zero_sigma ||
        !materialize_u0(int(k0), parts, s, ws + lay.E, lay.per_part_E, U0, D.L, flips, idxbuf, dsm, sc)) {
      // Row-parallel materialisation in column chunks of KU: each thread owns
      // rows, keeps the first max-|.| row per column (sign convention), then a
      // block argmax picks each column's sign. Rows of part i: Vsub_i[r,:] E_i.
      constexpr int KU = 8;
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      for (int c0 = 0; c0 < k0; c0 += KU) {
        const int nc = int(imin(KU, k0 - c0));
        double best[KU];
        int64_t bidx[KU];
  #pragma unroll
        for (int c = 0; c < KU; ++c) {
          best[c] = -1.0;
          bidx[c] = 0;
        }
        int64_t off = 0;
        for (int i = 0; i < s; ++i) {
          const PartView pv = load_part(parts[i]);
          const int64_t r0 = pv.rho[0];
          const double* vs = pv.v0 + pv.row0;
          const double* E = Ep(i) + c0 * r0;
          for (int64_t r = threadIdx.x; r < pv.len; r += blockDim.x) {
            double out[KU];
  #pragma unroll
            for (int c = 0; c < KU; ++c) out[c] = 0.0;
            for (int64_t a = 0; a < r0; ++a) {
              const double v = vs[r + a * pv.ld0];
  #pragma unroll
              for (int c = 0; c < KU; ++c)
                if (c < nc) out[c] = fma(v, E[a + c * r0], out[c]);
            }
  #pragma unroll
            for (int c = 0; c < KU; ++c)
              if (c < nc) {
                U0[off + r + (c0 + c) * D.L] = out[c];
                const double m = fabs(out[c]);
                if (m > best[c]) {
                  best[c] = m;
                  bidx[c] = off + r;
                }
              }
          }
          off += pv.len;
        }
  #pragma unroll
        for (int c = 0; c < KU; ++c) {
          double b = best[c];
          int64_t bi = bidx[c];
  #pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, b, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > b || (ob == b && oi < bi)) {
              b = ob;
              bi = oi;
            }
          }
          if (l == 0 && c < nc) {
            sc.red[w * kMaxVec + c0 + c] = b;
            idxbuf[w * kMaxVec + c0 + c] = bi;
          }
        }
      }
      __syncthreads();
      if (any_zero_sigma) {
        orthonormalize(U0, D.L, 0, int(k0), D.L, sc);
        sign_fix(U0, D.L, int(k0), D.L, flips, sc);
      } else {
        if (threadIdx.x < k0) {
          const int c = threadIdx.x;
          double b = sc.red[c];
          int64_t bi = idxbuf[c];
          for (int ww = 1; ww < kWarps; ++ww) {
            const double ob = sc.red[ww * kMaxVec + c];
            const int64_t oi = idxbuf[ww * kMaxVec + c];
            if (ob > b || (ob == b && oi < bi)) {
              b = ob;
              bi = oi;
            }
          }
          flips[c] = U0[bi + c * D.L] < 0.0;
        }
        __syncthreads();
        for (int64_t idx = threadIdx.x; idx < D.L * k0; idx += blockDim.x)
          if (flips[idx / D.L]) U0[idx] = -U0[idx];
        __syncthreads();
      }
    }
    const int64_t slice = prod_range(k, 1, p);
    for (int64_t e = threadIdx.x; e < k0 * slice; e += blockDim.x)
      if (flips[e / slice]) D.out_core[e] = -D.out_core[e];
    __syncthreads();
    tstop(sc, kPhU0, tu);
  }
  if (threadIdx.x == 0) {
    D.status[0] = sweeps;
    D.status[1] = converged;
    D.status[2] = norm_sq == 0.0;
    D.status[3] = any_zero_sigma;
    for (int m = 0; m < kMaxP; ++m) D.status[4 + m] = m < p ? int(k[m]) : 0;
    D.status[4 + kMaxP] = sc.eig_calls;
    D.status[5 + kMaxP] = sc.eig_sweeps;
#ifdef TT_INSTRUMENT
    sc.cyc[kPhAll] = clock64() - t_kernel;
#else
    (void)t_kernel;
#endif
    for (int i = 0; i < 8; ++i) D.status[6 + kMaxP + i] = int(sc.cyc[i] >> 10);
    D.status[14 + kMaxP] = sc.si_ok;
    D.status[15 + kMaxP] = sc.si_fail;
    D.status[16 + kMaxP] = sc.si_iters;
    for (int i = 0; i < 4; ++i) D.status[17 + kMaxP + i] = int(sc.cyc[8 + i] >> 10);
  }
}

// ---------------------------------------------------------------------------
// Gathers small device-staged outputs (cores, non-temporal factors) into the
// caller's pinned, UVA-mapped host buffers in one launch (one CTA per segment).
__global__ void __launch_bounds__(256) copy_segments_kernel(const CopySeg* __restrict__ segs, int n) {
  const CopySeg sg = segs[blockIdx.x];
  for (int64_t i = threadIdx.x; i < sg.n; i += blockDim.x) sg.dst[i] = sg.src[i];
}

std::atomic<int64_t> g_launches{0};

cudaError_t launch_copy_segments(const CopySeg* d_segs, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  copy_segments_kernel<<<n, 256, 0, st>>>(d_segs, n);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_leaf(const Params& prm, const LeafDesc* d_descs, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(leaf_als_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLeafDynSmem));
    attr = true;
  }
  leaf_als_kernel<<<n, kThreads, kLeafDynSmem, st>>>(prm, d_descs);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_stitch(const Params& prm, const StitchDesc* d_descs, const StitchPart* d_parts, int n,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(stitch_als_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDynSmem));
    attr = true;
  }
  stitch_als_kernel<<<n, kStitchThreads, kDynSmem, st>>>(prm, d_descs, d_parts);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

int64_t launches() { return g_launches.load(); }

}  // namespace ttb
