// Shared device helpers of the sm_100a ALS kernels (tt_leaf.cu, tt_stitch.cu).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include <atomic>

#include "tt_block.cuh"

namespace ttb {

constexpr int kEigSmemN = 64;  // Jacobi runs in shared memory up to this size
constexpr int kStitchThreads = 256;  // 2 stitch CTAs per SM (128 threads x 4 CTAs measured slower)
#ifndef TT_STITCH_CTAS
#define TT_STITCH_CTAS 2
#endif
constexpr int kStitchCtas = TT_STITCH_CTAS;  // resident stitch CTAs per SM (register budget)
// stitch kernel dynamic shared memory: 64 KB at 2 CTAs/SM, 55 KB at 3
#ifndef TT_STITCH_DYN_KB
#define TT_STITCH_DYN_KB 56  // measured: 56 KB (more L1 at 2 CTAs/SM) beats 64 and 48 by 3%
#endif
constexpr size_t kDynSmem = kStitchCtas >= 3 ? size_t(55) * 1024 : size_t(TT_STITCH_DYN_KB) * 1024;
// small stitch batches: one CTA per SM with most of the SM's shared memory
constexpr size_t kDynSmemSolo = size_t(200) * 1024;

__device__ __forceinline__ unsigned dyn_smem_doubles() {
  unsigned b;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(b));
  return b / 8u;
}

// Leaf streaming ring: kStages tiles of kTileD doubles, plus U^T staging.
#ifndef TT_LEAF_STAGES
#define TT_LEAF_STAGES 2  // measured: 2 stages (more L1 for the solver phases) beat 3 by 5% on the leaf
#endif
constexpr int kStages = TT_LEAF_STAGES;
constexpr int kTileD = int(kStreamTileDoubles);   // 20 KB per stage
#ifndef TT_USTAGE_DOUBLES
#define TT_USTAGE_DOUBLES 4096
#endif
constexpr int kUStage = TT_USTAGE_DOUBLES;  // U^T staged in shared memory when d*r <= this (32 KB)
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
    const double s = dot4(ma, ms_j, src, inner, d);
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
static __device__ double* eig_run(double* G, int n, double* V, int* order, double* dsm, double** diag, BlockScratch& sc) {
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
// subspace-iteration sub-phase timers; TT_PROBE_M0 hands the slots to the
// stitch kernel's mode-0 solver instead (instrumented investigation builds)
#ifdef TT_PROBE_M0
__device__ __forceinline__ void tstop_si(BlockScratch&, int, long long) {}
__device__ __forceinline__ void tstop_m0(BlockScratch& sc, int slot, long long t0) { tstop(sc, slot, t0); }
#else
__device__ __forceinline__ void tstop_si(BlockScratch& sc, int slot, long long t0) { tstop(sc, slot, t0); }
__device__ __forceinline__ void tstop_m0(BlockScratch&, int, long long) {}
#endif
// start of the subspace-iteration state in dynamic shared memory: after the
// per-warp partial sums (nwarps x kSiMaxYK) and the Rayleigh-Ritz eigensolver
// scratch (3 * 16^2)
__device__ __forceinline__ constexpr int si_base() { return kWarps * 512; }
constexpr int kSiMaxK = 16;     // register-tile bound on k
constexpr int kSiMaxYK = 512;   // bound on cols * k (16 outputs per lane)

// Warp 0 factors the SPD k x k matrix G = L L^T and writes Linv = L^{-1}
// (both col-major, lower). Sets sc.ibcast[2] = 1 on a failed pivot.
static __device__ void chol_inv_warp(const double* G, int k, double* L, double* Linv, BlockScratch& sc) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double dmax = 0.0;
  for (int j = 0; j < k; ++j) dmax = fmax(dmax, G[j + j * k]);
  bool ok = dmax > 0.0;
  double myinv = 0.0;  // lane j keeps 1 / L(j, j)
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
    // one rsqrt instead of sqrt + divide on the serial chain (64 vs 158 cycles)
    const double inv = rsqrt(sdiag), ljj = sdiag * inv;
    if (lane > j && lane < k) {
      double v = G[lane + j * k];
      for (int l = 0; l < j; ++l) v -= L[lane + l * k] * L[j + l * k];
      L[lane + j * k] = v * inv;
    }
    if (lane == j) {
      L[j + j * k] = ljj;
      myinv = inv;
    }
    __syncwarp();
  }
  if (!ok) {
    if (lane == 0) sc.ibcast[2] = 1;
    return;
  }
  // column `lane` of L^{-1} by forward substitution (reciprocal diagonals
  // broadcast by shuffle: no divides on the chain)
  for (int i = 0; i < k; ++i) {
    const double invd = __shfl_sync(0xffffffffu, myinv, i);
    if (lane < k) {
      const int c = lane;
      if (i < c) {
        Linv[i + c * k] = 0.0;
      } else {
        double v = (i == c) ? 1.0 : 0.0;
        for (int l = c; l < i; ++l) v -= L[i + l * k] * Linv[l + c * k];
        Linv[i + c * k] = v * invd;
      }
    }
  }
}

// Ranks up to kRegK (the BASELINE configs C1-C4 use 4..10) get the fully unrolled
// register-resident solver pieces below; larger ranks keep the shared-memory
// forms (the unrolled code grows with K^2 and so does the build time).
constexpr int kRegK = 10;

// The same factorisation for K <= kRegK, register-resident: lane i holds row i of
// G; the right-looking update takes the pivot and the column entries from the
// owning lanes by shuffle, and L^{-1} is formed column-per-lane by forward
// substitution over shuffled entries of L. No shared-memory round trips, one
// rsqrt per column on the serial chain (~2k cycles at K = 10 against ~7k for
// chol_inv_warp). Writes Linv only (col-major, lower; the strict upper part 0).
// rel_pivot > 0 also fails the factorisation when a pivot drops below
// rel_pivot * G(j, j): column j lost more than that share of its squared norm
// against the earlier columns (CGS2's collapse test with rel_pivot = 0.25).
template <int K>
static __device__ void chol_inv_warp_reg(const double* G, double* Linv, BlockScratch& sc, double rel_pivot = 0.0) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const unsigned full = 0xffffffffu;
  const int row = lane < K ? lane : K - 1;
  double g[K], invd[K];
  double mydiag = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    g[j] = G[row + j * K];
    if (j == row) mydiag = g[j];
  }
  double dmax = mydiag;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(full, dmax, o));
  bool ok = dmax > 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double d = __shfl_sync(full, g[j], j);  // the updated pivot (uniform)
    const double g0 = __shfl_sync(full, mydiag, j);  // the original diagonal entry
    // pivots below 1e-14 * dmax: rank-deficient Gram, the caller falls back
    if (!(d > 1e-14 * dmax) || !(d > rel_pivot * g0)) ok = false;
    const double inv = rsqrt(d);
    invd[j] = inv;
    const double lij = (lane == j) ? d * inv : g[j] * inv;  // L(lane, j), meaningful for lane >= j
    g[j] = lij;
#pragma unroll
    for (int m = j + 1; m < K; ++m) {
      const double lmj = __shfl_sync(full, lij, m);
      g[m] = fma(-lij, lmj, g[m]);  // meaningful for lane >= m
    }
  }
  if (!ok) {
    if (lane == 0) sc.ibcast[2] = 1;
    return;
  }
  double x[K];  // column `lane` of L^{-1}
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double v = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int l = 0; l < i; ++l) {
      const double lil = __shfl_sync(full, g[l], i);  // L(i, l)
      v = fma(-lil, x[l], v);                         // x[l] = 0 above the diagonal (l < lane)
    }
    x[i] = (i >= lane) ? v * invd[i] : 0.0;
  }
  if (lane < K) {
#pragma unroll
    for (int i = 0; i < K; ++i) Linv[i + lane * K] = x[i];
  }
}

// W (rows x K, ld rows) <- W L^{-T}, where W^T W = L L^T (one CholeskyQR pass).
template <int K>
__device__ __noinline__ bool cholqr_pass_k(double* W, int64_t rows, double* small, BlockScratch& sc,
                                           double rel_pivot = 0.0) {
  double* G = small;
  double* L = small + K * K;
  double* Li = small + 2 * K * K;
  gram_tall(W, rows, rows, K, G);
  if (threadIdx.x == 0) sc.ibcast[2] = 0;
  __syncthreads();
  if constexpr (K <= kRegK)
    chol_inv_warp_reg<K>(G, Li, sc, rel_pivot);
  else
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

// Y (cols x K) = A^T U with A(i, c) = P[offc[c] + i*inner]. Register-blocked:
// a thread owns an 8-column block of A times a 2-column block of U (16
// accumulators; 10 loads feed 16 FMAs per row), the blocks are replicated over
// row groups, and the row-group partial sums are reduced through shared memory.
template <int K>
__device__ __noinline__ void unfold_At_U_k(const double* __restrict__ P, const int* __restrict__ offc, int64_t rows,
                                           int64_t inner, int cols, const double* __restrict__ U,
                                           double* __restrict__ Y, double* part) {
  constexpr int CB = 8;
  constexpr int JB = K < 2 ? K : 2;
  constexpr int NJB = (K + JB - 1) / JB;
  const int ne = cols * K;
  const int ncb = (cols + CB - 1) / CB;
  const int nblk = ncb * NJB;  // <= 64: cols * K <= kSiMaxYK
  int rg = int(blockDim.x) / nblk;
  const int cap = si_base() / ne;
  if (rg > cap) rg = cap;
  if (rg < 1) rg = 1;
  const int t = threadIdx.x;
  const int blk = t % nblk, g = t / nblk;
  if (g < rg) {
    const int c0 = (blk % ncb) * CB, j0 = (blk / ncb) * JB;
    const int64_t chunk = (rows + rg - 1) / rg;
    const int64_t i0 = g * chunk, i1 = imin(rows, i0 + chunk);
    int oc[CB];
#pragma unroll
    for (int u = 0; u < CB; ++u) oc[u] = offc[c0 + u < cols ? c0 + u : 0];
    const double* Ub[JB];
#pragma unroll
    for (int v = 0; v < JB; ++v) Ub[v] = U + int64_t(j0 + v < K ? j0 + v : 0) * rows;
    double acc[CB][JB];
#pragma unroll
    for (int u = 0; u < CB; ++u)
#pragma unroll
      for (int v = 0; v < JB; ++v) acc[u][v] = 0.0;
    for (int64_t i = i0; i < i1; ++i) {
      const double* Pi = P + i * inner;
      double a[CB], b[JB];
#pragma unroll
      for (int u = 0; u < CB; ++u) a[u] = Pi[oc[u]];
#pragma unroll
      for (int v = 0; v < JB; ++v) b[v] = Ub[v][i];
#pragma unroll
      for (int u = 0; u < CB; ++u)
#pragma unroll
        for (int v = 0; v < JB; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < CB; ++u)
#pragma unroll
      for (int v = 0; v < JB; ++v)
        if (c0 + u < cols && j0 + v < K) part[g * ne + (c0 + u) + (j0 + v) * cols] = acc[u][v];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < rg; ++w) v += part[w * ne + e];
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
    tstop_si(sc, kSiAtU, tp);
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
    tstop_si(sc, kSiAY, tp);
    if (bsq > 0.0 && rsq <= 1e-26 * bsq) {
      iters = it + 1;
      break;
    }
    if (!(bsq > 0.0)) return -1;
    tp = tstart();
    if (!cholqr_pass_k<K>(W, rows, small, sc) || !cholqr_pass_k<K>(W, rows, small, sc)) return -1;
    for (int64_t idx = threadIdx.x; idx < rows * K; idx += blockDim.x) U[idx] = W[idx];
    __syncthreads();
    tstop_si(sc, kSiQR, tp);
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
  tstop_si(sc, kSiRR, trr);
  return iters;
}

static __device__ bool llsv_subspace(const double* P, int64_t outer, int64_t rows, int64_t inner, int k, int kprev, double* U,
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

// Top-k eigenvectors of a symmetric positive semidefinite n x n matrix G
// (col-major, ld n) by warm-started block subspace iteration: W = G U,
// B = U^T W, stop when ||W - U B||_F <= 1e-13 ||B||_F, else U = orth(W)
// (CholeskyQR2); a Rayleigh-Ritz rotation by the eigenvectors of B then gives
// the eigenvectors in descending order (the same vectors a full Jacobi solve
// returns, to rounding). U holds the start on entry (n x K, any basis of full
// rank); W is scratch of the same size. Returns the buffer holding the result
// (U or W) and the eigenvalues in lam[0..K), or nullptr on breakdown or no
// convergence (rank-deficient G, tiny gap) — the caller then runs Jacobi.
// Replaces an O(n^3)-per-sweep Jacobi solve of the whole Gram matrix when only
// k << n vectors are needed (Gram sizes 64..100 at BASELINE configs C3/C4).
// An iteration costs O(n^2 k), against O(n^3) per sweep for the Jacobi
// fallback, so slowly converging (small-gap) problems get more iterations.
constexpr int kGramSiMaxIter = 100;
constexpr int kGramSiMaxK = 32;  // top-k Gram iteration: k <= 32 (BASELINE C5's ranks 20)
// shared-memory carve-up of sym_topk_si_k: [0, 3K^2) Rayleigh-Ritz eigensolver
// scratch, then CholeskyQR scratch (3K^2), B (K^2), then the staged G, U, W
__host__ __device__ constexpr int topk_small_off(int K) { return K <= 16 ? 768 : 3 * K * K; }
__host__ __device__ constexpr int topk_b_off(int K) { return K <= 16 ? 1536 : 6 * K * K; }
__host__ __device__ constexpr int topk_stage_off(int K) { return K <= 16 ? 2048 : 7 * K * K; }
// Wout (n x K, ld n) = G Uin for the staged symmetric G (ld ldp, odd: lanes on
// consecutive rows hit distinct banks). A thread owns one row of the product and
// all K columns over one of H = blockDim/n slices of the inner index: per inner
// step one LDS of G and K/2 broadcast LDS.128 of the K-contiguous copy of Uin
// feed K FMAs (the plain dot-product form pays two LDS per FMA). utr: n*K
// doubles, part: blockDim*K doubles of shared memory.
template <int K>
__device__ __noinline__ void sym_gu_tiled(const double* Gp, int ldp, int n, const double* Uin, double* Wout,
                                          double* utr, double* part) {
  for (int idx = threadIdx.x; idx < n * K; idx += blockDim.x) {
    const int l = idx % n, j = idx / n;
    utr[l * K + j] = Uin[idx];
  }
  __syncthreads();
  const int H = int(imax(1, imin(4, int(blockDim.x) / n)));
  const int h = threadIdx.x / n, i = threadIdx.x - h * n;
  if (h < H) {
    const int l0 = h * n / H, l1 = (h + 1) * n / H;
    double acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = 0.0;
    const double* g = Gp + int64_t(i) * ldp;
    if ((K & 1) == 0 && (reinterpret_cast<uintptr_t>(utr) & 15u) == 0) {
#pragma unroll 2
      for (int l = l0; l < l1; ++l) {
        const double gv = g[l];
        const double2* ur = reinterpret_cast<const double2*>(utr + l * K);
#pragma unroll
        for (int j = 0; j < K / 2; ++j) {
          const double2 u2 = ur[j];
          acc[2 * j] = fma(gv, u2.x, acc[2 * j]);
          acc[2 * j + 1] = fma(gv, u2.y, acc[2 * j + 1]);
        }
      }
    } else {
      for (int l = l0; l < l1; ++l) {
        const double gv = g[l];
        const double* ur = utr + l * K;
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = fma(gv, ur[j], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) part[(h * K + j) * n + i] = acc[j];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * K; idx += blockDim.x) {
    double v = 0.0;
    for (int hh = 0; hh < H; ++hh) v += part[hh * K * n + idx];
    Wout[idx] = v;
  }
  __syncthreads();
}

template <int K>
__device__ __noinline__ double* sym_topk_si_k(const double* __restrict__ G, int n, double* U, double* W,
                                              double* lam, int* order, double* dsm, BlockScratch& sc) {
  double* small = dsm + topk_small_off(K);  // CholeskyQR scratch (3 K^2); dsm[0, 3K^2) is the Rayleigh-Ritz eigensolver's
  double* B = dsm + topk_b_off(K);          // K x K
  // With room, G (odd leading dimension: conflict-free row reads), U and W live
  // in shared memory for the whole iteration: every product is then an SMEM
  // stream instead of an L2-latency-bound dot product (the cluster leaf
  // kernel's 176 KB and the stitch kernel's small-batch launches have room for
  // n = 100).
  const int ldg = n | 1;
  const bool staged = topk_stage_off(K) + ldg * n + 2 * n * K <= sc.dsm_cap;
  double* const Ug = U;
  double* const Wg = W;
  const double* Gp = G;
  int ldp = n;
  // room for the register-tiled product's K-contiguous copy and partial sums
  // (k <= kRegK: one out-of-line copy per K keeps the build time in check)
  const bool tiled = K <= kRegK && staged && n <= int(blockDim.x) &&
                     topk_stage_off(K) + ldg * n + 3 * n * K + int(blockDim.x) * K <= sc.dsm_cap;
  double* const utr = dsm + topk_stage_off(K) + ldg * n + 2 * n * K;
  double* const part = utr + n * K;
  if (staged) {
    double* Gs = dsm + topk_stage_off(K);
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      const int i = idx % n, j = idx / n;
      Gs[i + j * ldg] = G[idx];
    }
    U = Gs + ldg * n;
    W = U + n * K;
    for (int idx = threadIdx.x; idx < n * K; idx += blockDim.x) U[idx] = Ug[idx];
    Gp = Gs;
    ldp = ldg;
    __syncthreads();
  }
  if (!cholqr_pass_k<K>(U, n, small, sc) || !cholqr_pass_k<K>(U, n, small, sc)) return nullptr;
  bool conv = false;
  int it = 0;
  for (; it < kGramSiMaxIter; ++it) {
    long long tp = tstart();
    if (tiled) {
      if constexpr (K <= kRegK) sym_gu_tiled<K>(Gp, ldp, n, U, W, utr, part);
    } else {
      for (int idx = threadIdx.x; idx < n * K; idx += blockDim.x) {
        const int i = idx % n, j = idx / n;
        W[idx] = dot4(Gp + int64_t(i) * ldp, 1, U + int64_t(j) * n, 1, n);
      }
      __syncthreads();
    }
    tstop_si(sc, kSiAtU, tp);
    tp = tstart();
    gemm(K, K, n, U, n, 1, W, 1, n, B, 1, K, false, sc);  // B = U^T W
    double rsq = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double u[K];
#pragma unroll
      for (int l = 0; l < K; ++l) u[l] = U[i + l * n];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        double v = W[i + j * n];
#pragma unroll
        for (int l = 0; l < K; ++l) v = fma(-u[l], B[l + j * K], v);
        rsq = fma(v, v, rsq);
      }
    }
    double bsq = 0.0;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) bsq = fma(B[e], B[e], bsq);
    rsq = block_sum(rsq, sc);
    bsq = block_sum(bsq, sc);
    tstop_si(sc, kSiAY, tp);
    if (!(bsq > 0.0)) return nullptr;
    // relative residual 1e-13: the subspace error is <= 1e-13 / relative gap
    // (1e-12 measured too loose for rank-20 problems with gaps near 1e-6)
    if (rsq <= 1e-26 * bsq) {
      conv = true;
      break;
    }
    // at the iteration cap a 1e-11 relative residual is accepted: the subspace
    // error is then <= 1e-11 / relative gap (within the 1e-6 parity bar for
    // gaps >= 1e-5; 1e-10 measured 1.4e-6 on a rank-20 node whose trailing
    // columns sit in the noise floor), and the Jacobi fallback on n ~ 100
    // costs ~1e7 cycles
    if (it == kGramSiMaxIter - 1 && rsq <= 1e-22 * bsq) {
      conv = true;
      break;
    }
    // Powering: orthonormalise G^m U instead of G U. The Rayleigh quotients on
    // B's diagonal bound the conditioning of G^m U by ratio^m; m is the largest
    // of 1..3 keeping it <= 1e5 (CholQR2 stays exact there), so an outer
    // iteration contracts the error by rho^m for one CholQR2.
    {
      if (threadIdx.x == 0) {
        double bmax = 0.0, bmin = INFINITY;
        for (int j = 0; j < K; ++j) {
          bmax = fmax(bmax, B[j + j * K]);
          bmin = fmin(bmin, B[j + j * K]);
        }
        const double ratio = bmin > 0.0 ? bmax / bmin : INFINITY;
        sc.ibcast[3] = ratio <= 46.0 ? 3 : (ratio <= 316.0 ? 2 : 1);
      }
      __syncthreads();
      const int extra = sc.ibcast[3] - 1;
      const long long tpw = tstart();
      for (int e = 0; e < extra; ++e) {  // U <- G W, then swap: W holds G^(1+e+1) U_old
        if (tiled) {
          if constexpr (K <= kRegK) sym_gu_tiled<K>(Gp, ldp, n, W, U, utr, part);
        } else {
          for (int idx = threadIdx.x; idx < n * K; idx += blockDim.x) {
            const int i = idx % n, j = idx / n;
            U[idx] = dot4(Gp + int64_t(i) * ldp, 1, W + int64_t(j) * n, 1, n);
          }
          __syncthreads();
        }
        double* t = U;
        U = W;
        W = t;
      }
      tstop_si(sc, kSiAtU, tpw);
    }
    double* t = U;  // U <- orth(W)
    U = W;
    W = t;
    tp = tstart();
    if (!cholqr_pass_k<K>(U, n, small, sc) || !cholqr_pass_k<K>(U, n, small, sc)) return nullptr;
    tstop_si(sc, kSiQR, tp);
  }
  if (!conv) return nullptr;
  if (threadIdx.x == 0) sc.si_iters += it + 1;
  const long long trr = tstart();
  double* diag = nullptr;
  const double* R = eig_run(B, K, small, order, dsm, &diag, sc);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double u[K];
#pragma unroll
    for (int l = 0; l < K; ++l) u[l] = U[i + l * n];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const double* rj = R + order[j] * K;
      double v = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) v = fma(u[l], rj[l], v);
      W[i + j * n] = v;
    }
  }
  if (threadIdx.x < K) lam[threadIdx.x] = diag[order[threadIdx.x] * (K + 1)];
  __syncthreads();
  tstop_si(sc, kSiRR, trr);
  if (staged) {  // hand the result back in the caller's global buffer
    for (int idx = threadIdx.x; idx < n * K; idx += blockDim.x) Wg[idx] = W[idx];
    __syncthreads();
    return Wg;
  }
  return W;
}

static __device__ double* sym_topk_si(const double* G, int n, int k, double* U, double* W, double* lam, int* order,
                                      double* dsm, BlockScratch& sc) {
  switch (k) {
#define TT_CASE(N) \
  case N:          \
    return sym_topk_si_k<N>(G, n, U, W, lam, order, dsm, sc);
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10) TT_CASE(11) TT_CASE(12) TT_CASE(13) TT_CASE(14) TT_CASE(15) TT_CASE(16)
    TT_CASE(17) TT_CASE(18) TT_CASE(19) TT_CASE(20) TT_CASE(21) TT_CASE(22) TT_CASE(23) TT_CASE(24)
    TT_CASE(25) TT_CASE(26) TT_CASE(27) TT_CASE(28) TT_CASE(29) TT_CASE(30) TT_CASE(31) TT_CASE(32)
#undef TT_CASE
    default:
      return nullptr;
  }
}

// Gram sizes above this use the warm-started top-k subspace iteration instead
// of a full Jacobi solve (when the caller has a warm start).
constexpr int kGramSiMinN = 24;
// Gram sizes from this up use the register-tiled Gram.
constexpr int kGramTiledMinN = 24;

// leading_left_singular_vectors (linalg.cpp:45-64) of the mode unfolding of a
// row-major (outer, rows, inner) tensor, through the Gram matrix of its
// smaller side. U: rows x k (ld rows), sign-fixed. On entry U holds the
// factor's current value (kprev columns), used as the iterations' warm start.
// gram_ready: G already holds the Gram of the smaller side (the cluster
// kernel forms it across its CTAs, tt_wide.cu); skip straight to the solver.
__device__ __forceinline__ bool llsv_uses_subspace(int64_t rows, int64_t cols, int64_t k, int64_t kprev,
                                                   const double* si, const BlockScratch& sc) {
  return si != nullptr && kprev > 0 && rows > cols && cols >= 2 * k && cols * k <= kSiMaxYK && k <= kSiMaxK &&
         si_base() + kSiMaxYK + 5 * k * k + 256 <= sc.dsm_cap;
}
// Two CholeskyQR passes on W (rows x k, ld rows), k <= kRegK; false on a breakdown
// or when a column collapses against the earlier ones (CGS2's completion case;
// W is then unchanged or still spans the same space). small: 3 k^2 doubles.
static __device__ bool cholqr2(double* W, int64_t rows, int k, double* small, BlockScratch& sc) {
  switch (k) {
#define TT_CASE(N) \
  case N:          \
    return cholqr_pass_k<N>(W, rows, small, sc, 0.25) && cholqr_pass_k<N>(W, rows, small, sc);
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10)
#undef TT_CASE
    default:
      return false;
  }
}

// Y (n x kp, ld n) = A^T U for a dense row-major A (rows x n, n <= blockDim.x)
// and U (rows x kp, ld rows): a thread owns one column of A in one of
// blockDim.x / n row groups and 8 columns of U at a time (coalesced loads of
// A, broadcast loads of U); the row groups' partial sums meet in `scratch`
// (>= 8 * blockDim.x doubles of shared memory).
static __device__ void dense_At_U(const double* __restrict__ A, int64_t rows, int n, const double* __restrict__ U,
                                  int kp, double* __restrict__ Y, double* scratch) {
  const int ng = imax(1, int(blockDim.x) / n);
  const int g = threadIdx.x / n, r = threadIdx.x - g * n;
  const bool active = g < ng;
  for (int c0 = 0; c0 < kp; c0 += 8) {
    double acc[8];
    const double* uc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      acc[c] = 0.0;
      uc[c] = U + int64_t(imin(c0 + c, kp - 1)) * rows;
    }
    if (active) {
#pragma unroll 4
      for (int64_t i = g; i < rows; i += ng) {
        const double a = A[i * n + r];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = fma(a, uc[c][i], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) scratch[(g * n + r) * 8 + c] = acc[c];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * 8; idx += blockDim.x) {
      const int rr = idx >> 3, c = idx & 7;
      if (c0 + c < kp) {
        double v = 0.0;
        for (int gg = 0; gg < ng; ++gg) v += scratch[(gg * n + rr) * 8 + c];
        Y[rr + int64_t(c0 + c) * n] = v;
      }
    }
    __syncthreads();
  }
}

// U (rows x k, ld rows) = A M diag(scale) for a dense row-major A (rows x n):
// M's columns (n each) are staged in shared memory (`ms`, n*k doubles) and read
// as broadcasts; a thread owns a row of A and 8 output columns at a time.
template <class Col>
static __device__ void dense_A_M(const double* __restrict__ A, int64_t rows, int n, Col col, const double* scale, int k,
                                 double* __restrict__ U, double* ms) {
  for (int idx = threadIdx.x; idx < n * k; idx += blockDim.x) {
    const int t = idx % n, c = idx / n;
    ms[idx] = col(c)[t];
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double* a = A + i * n;
    for (int c0 = 0; c0 < k; c0 += 8) {
      double acc[8];
      const double* mc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        acc[c] = 0.0;
        mc[c] = ms + imin(c0 + c, k - 1) * n;
      }
#pragma unroll 8
      for (int t = 0; t < n; ++t) {
        const double av = a[t];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = fma(av, mc[c][t], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c0 + c < k) U[i + int64_t(c0 + c) * rows] = acc[c] * scale[c0 + c];
    }
  }
  __syncthreads();
}

static __device__ void llsv_unfold(const double* P, int64_t outer, int64_t rows, int64_t inner, int64_t k, double* U,
                            double* G, double* V, double* misc, double* dsm, BlockScratch& sc, int64_t kprev = 0,
                            double* si = nullptr, bool gram_ready = false) {
  const int64_t cols = outer * inner;
  if (!gram_ready && llsv_uses_subspace(rows, cols, k, kprev, si, sc)) {
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
  double* lamv = misc + kMisc / 2 + 512;
  const bool wide = rows <= cols;
  const int n = int(wide ? rows : cols);
  long long tg = tstart();
  // unfolding element A(i, c) = P[(o*rows + i)*inner + t], c = o*inner + t
  auto unf = [&](int64_t i, int64_t c) {
    const int64_t o = c / inner, t = c - o * inner;
    return P[(o * rows + i) * inner + t];
  };
  if (gram_ready) {
    // formed by the caller
  } else if (n >= kGramTiledMinN && n * 4 <= sc.dsm_cap) {
    if (wide)  // G = A A^T: x runs over the columns c (contiguous in t)
      gram_tiled(n, cols, [&](int64_t c, int a) { return unf(a, c); }, true, G, dsm, sc.dsm_cap);
    else  // G = A^T A: x runs over the rows i, a over the columns
      gram_tiled(n, rows, [&](int64_t i, int a) { return unf(i, a); }, false, G, dsm, sc.dsm_cap);
  } else if (wide) {
    if (inner == 1)  // A = P^T viewed (rows x outer): a GEMM with the K split across the block
      gemm(rows, rows, outer, P, 1, rows, P, rows, 1, G, 1, rows, false, sc);
    else
      gram_rows(P, outer, rows, inner, G);
  } else {
    gram_cols(P, outer, rows, inner, G);
  }
  tstop(sc, kPhGram, tg);
  // eigenvectors: column c at vcol(c), eigenvalue lamc(c), descending
  const double* Vsi = nullptr;
  if (kprev > 0 && k <= kGramSiMaxK && n > kGramSiMinN && n >= 2 * k && 7 * k * k + 256 <= sc.dsm_cap) {
    const long long t0 = tstart();
    double* Us = V;
    double* Ws = V + int64_t(n) * k;
    const int64_t kp = imin(kprev, k);
    // dense row-major unfolding (outer == 1): A^T U_prev with coalesced loads
    const bool dense_ws = !wide && outer == 1 && n <= int(blockDim.x) && 8 * int(blockDim.x) <= sc.dsm_cap;
    if (dense_ws) dense_At_U(P, rows, n, U, int(kp), Us, dsm);
    for (int64_t idx = threadIdx.x; idx < n * k; idx += blockDim.x) {
      const int64_t r = idx % n, c = idx / n;
      double v;
      if (c >= kp) {
        v = (r == (c * 7919) % n) ? 1.0 : 0.0;  // pad with canonical vectors
      } else if (wide) {
        v = U[r + c * rows];
      } else if (dense_ws) {
        continue;
      } else {  // tall: A^T U_prev, column r of the unfolding
        const int64_t o = r / inner, t = r - o * inner;
        v = dot4(P + o * rows * inner + t, inner, U + c * rows, 1, rows);
      }
      Us[idx] = v;
    }
    __syncthreads();
    Vsi = sym_topk_si(G, n, int(k), Us, Ws, lamv, order, dsm, sc);
    tstop(sc, kPhEig, t0);
    if (threadIdx.x == 0) {
      if (Vsi)
        sc.si_ok += 1;
      else
        sc.si_fail += 1;
    }
  }
  double* diag = nullptr;
  const double* Vp = Vsi;
  if (!Vsi) Vp = eig_run(G, n, V, order, dsm, &diag, sc);
  auto vcol = [&](int64_t c) { return Vsi ? Vsi + c * n : Vp + int64_t(order[c]) * n; };
  auto lamc = [&](int64_t c) { return Vsi ? lamv[c] : diag[order[c] * (n + 1)]; };
  if (wide) {
    for (int64_t idx = threadIdx.x; idx < rows * k; idx += blockDim.x) {
      const int64_t i = idx % rows, c = idx / rows;
      U[idx] = vcol(c)[i];
    }
    __syncthreads();
  } else {
    if (threadIdx.x < k) {
      const double l0 = fmax(lamc(0), 0.0);
      const double lc = fmax(lamc(threadIdx.x), 0.0);
      sig[threadIdx.x] = gram_sigma_ok(lc, l0) ? 1.0 / sqrt(lc) : 0.0;
    }
    __syncthreads();
    tg = tstart();
    // dense row-major unfolding: U = A V Sigma^-1 from V staged in shared memory
    // (only after the top-k iteration: the Jacobi fallback's vectors live in dsm)
    if (Vsi != nullptr && outer == 1 && int64_t(n) * k <= sc.dsm_cap) {
      dense_A_M(P, rows, n, vcol, sig, int(k), U, dsm);
    } else {
      for (int64_t idx = threadIdx.x; idx < rows * k; idx += blockDim.x) {
        const int64_t i = idx % rows, c = idx / rows;
        const double inv = sig[c];
        double s = 0.0;
        if (inv != 0.0) {
          const double* vc = vcol(c);
          for (int64_t o = 0; o < outer; ++o) s += dot4(P + (o * rows + i) * inner, 1, vc + o * inner, 1, inner);
        }
        U[idx] = s * inv;
      }
      __syncthreads();
    }
    tstop(sc, kPhGram, tg);
    const long long to = tstart();
    // U = A V Sigma^-1 is orthonormal to ~1e-10 already: CholeskyQR2 gives the same
    // Q as Gram-Schmidt (the QR factor with positive diagonal is unique) in two
    // short passes instead of ~4 block reductions per column; a rank-deficient U
    // (zeroed columns) breaks the Cholesky down and takes CGS2 with completion.
    if (!(k <= kRegK && 3 * k * k <= sc.dsm_cap && cholqr2(U, rows, int(k), dsm, sc)))
      orthonormalize(U, rows, 0, int(k), rows, sc);
    tstop(sc, kPhOrtho, to);
  }
  const long long ts = tstart();
  sign_fix(U, rows, int(k), rows, nullptr, sc);
  tstop(sc, kPhOrtho, ts);
}

// ---------------------------------------------------------------------------
// Thread-block clusters (the cluster kernels of tt_wide.cu and tt_stitch.cu)
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// leading_left_singular_vectors (linalg.cpp:45-64) of the mode unfolding of a
// row-major (outer, rows, inner) tensor for the cluster: when llsv_unfold
// takes its Gram route with a tiled Gram, every CTA forms the Gram over its
// share of the long side into its partial slot, and the leader sums the
// partials in rank order and runs the solver; otherwise the leader does it
// all. Called by every CTA of the cluster (one cluster barrier inside on the
// distributed route); U is valid on the leader afterwards.
static __device__ void wide_llsv(const double* P, int64_t outer, int64_t rows, int64_t inner, int64_t k, double* U,
                          double* G, double* V, double* misc, double* dsm, BlockScratch& sc, int64_t kprev,
                          double* si, double* gpart, int rank, int CS) {
  const int64_t cols = outer * inner;
  const bool wide = rows <= cols;
  const int n = int(wide ? rows : cols);
  const bool dist = CS > 1 && !llsv_uses_subspace(rows, cols, k, kprev, si, sc) && n >= kGramTiledMinN &&
                    n * 4 <= sc.dsm_cap;
  if (!dist) {
    if (rank == 0) llsv_unfold(P, outer, rows, inner, k, U, G, V, misc, dsm, sc, kprev, si);
    return;
  }
  const long long tg = tstart();
  const int64_t nx = wide ? cols : rows;
  const int64_t per = (nx + CS - 1) / CS;
  const int64_t x0 = imin(nx, int64_t(rank) * per), x1 = imin(nx, x0 + per);
  double* Gp = gpart + int64_t(rank) * n * n;
  auto unf = [&](int64_t i, int64_t c) {
    const int64_t o = c / inner, t = c - o * inner;
    return P[(o * rows + i) * inner + t];
  };
  if (x1 <= x0) {
    for (int64_t idx = threadIdx.x; idx < int64_t(n) * n; idx += blockDim.x) Gp[idx] = 0.0;
    __syncthreads();
  } else if (wide) {  // G = A A^T: x over the columns
    gram_tiled(n, x1 - x0, [&](int64_t c, int a) { return unf(a, x0 + c); }, true, Gp, dsm, sc.dsm_cap);
  } else {  // G = A^T A: x over the rows
    gram_tiled(n, x1 - x0, [&](int64_t i, int a) { return unf(x0 + i, a); }, false, Gp, dsm, sc.dsm_cap);
  }
  cl_sync();
  if (rank == 0) {
    for (int64_t idx = threadIdx.x; idx < int64_t(n) * n; idx += blockDim.x) {
      double v = 0.0;
      for (int r = 0; r < CS; ++r) v += gpart[int64_t(r) * n * n + idx];
      G[idx] = v;
    }
    __syncthreads();
    tstop(sc, kPhGram, tg);
    llsv_unfold(P, outer, rows, inner, k, U, G, V, misc, dsm, sc, kprev, si, /*gram_ready=*/true);
  }
}


extern std::atomic<int64_t> g_launches;

// Sets a kernel's dynamic shared-memory cap on the current device, once per
// (kernel slot, device): the attribute is per device, so a process driving
// several devices sets it on each. Returns the attribute call's error.
cudaError_t ensure_dyn_smem(const void* fn, int slot, size_t bytes);

}  // namespace ttb
