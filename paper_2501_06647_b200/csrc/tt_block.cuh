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
  int eig_calls, eig_sweeps;  // instrumentation (Jacobi sweeps per problem)
  int si_ok, si_fail, si_iters;  // subspace-iteration outcomes and iterations
  int dsm_cap;                   // doubles of dynamic shared memory in this launch
  long long cyc[12];          // instrumentation: cycles per phase (see kPh*, kSi*)
};

// Phase-timer slots (thread 0 accumulates clock64 deltas; instrumentation).
enum { kPhEig = 0, kPhGram = 1, kPhTtm = 2, kPhGemm = 3, kPhOrtho = 4, kPhU0 = 5, kPhBig = 6, kPhAll = 7 };
// subspace-iteration internals (subsets of kPhEig): A^T U + Gram, A Y + residual, CholeskyQR2, Rayleigh-Ritz
enum { kSiAtU = 8, kSiAY = 9, kSiQR = 10, kSiRR = 11 };
#ifdef TT_INSTRUMENT
__device__ __forceinline__ long long tstart() { return threadIdx.x == 0 ? clock64() : 0; }
__device__ __forceinline__ void tstop(BlockScratch& sc, int slot, long long t0) {
  if (threadIdx.x == 0) sc.cyc[slot] += clock64() - t0;
}
#else
__device__ __forceinline__ long long tstart() { return 0; }
__device__ __forceinline__ void tstop(BlockScratch&, int, long long) {}
#endif

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
// TMA bulk-copy (cp.async.bulk) + mbarrier helpers for streaming global memory
// through a shared-memory ring (sm_90+; the B200 bulk-copy engine).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TT_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TT_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// sum_k a[k*as] * b[k*bs] with four independent accumulators: the loads of
// four iterations are issued back to back, so a runtime-length dot product
// over L2-resident operands waits for one load latency per four terms.
__device__ __forceinline__ double dot4(const double* __restrict__ a, int64_t as, const double* __restrict__ b,
                                       int64_t bs, int64_t n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t k = 0;
  for (; k + 3 < n; k += 4) {
    const double a0 = a[k * as], a1 = a[(k + 1) * as], a2 = a[(k + 2) * as], a3 = a[(k + 3) * as];
    const double b0 = b[k * bs], b1 = b[(k + 1) * bs], b2 = b[(k + 2) * bs], b3 = b[(k + 3) * bs];
    s0 = fma(a0, b0, s0);
    s1 = fma(a1, b1, s1);
    s2 = fma(a2, b2, s2);
    s3 = fma(a3, b3, s3);
  }
  for (; k < n; ++k) s0 = fma(a[k * as], b[k * bs], s0);
  return (s0 + s1) + (s2 + s3);
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

// C(i,j) (+)= sum_k A(i,k) B(k,j); element (i,j) of X at X[i*rs + j*cs].
// Few outputs with a long K (e.g. V_sub^T V_sub over thousands of rows) split
// K across the block and reduce the partials through shared memory.
__device__ __forceinline__ void gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t ars, int64_t acs,
                                     const double* B, int64_t brs, int64_t bcs, double* C, int64_t crs, int64_t ccs,
                                     bool acc, BlockScratch& sc) {
  const int64_t tot = M * N;
  const int64_t split = (tot <= 128 && K >= 64) ? imin(int64_t(blockDim.x) / tot, K / 16) : 1;
  if (split >= 2) {
    const int64_t kc = (K + split - 1) / split;
    const int64_t work = tot * split;
    if (threadIdx.x < work) {
      const int64_t e = threadIdx.x % tot, part = threadIdx.x / tot;
      const int64_t i = e % M, j = e / M;
      const int64_t k0 = part * kc, k1 = imin(K, k0 + kc);
      const double* a = A + i * ars;
      const double* b = B + j * bcs;
      sc.red[threadIdx.x] = dot4(a + k0 * acs, acs, b + k0 * brs, brs, k1 - k0);
    }
    __syncthreads();
    if (threadIdx.x < tot) {
      const int64_t i = threadIdx.x % M, j = threadIdx.x / M;
      double s = 0.0;
      for (int64_t part = 0; part < split; ++part) s += sc.red[part * tot + threadIdx.x];
      double* c = C + i * crs + j * ccs;
      *c = acc ? *c + s : s;
    }
    __syncthreads();
    return;
  }
  for (int64_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int64_t i = idx % M, j = idx / M;
    const double s = dot4(A + i * ars, acs, B + j * bcs, brs, K);
    double* c = C + i * crs + j * ccs;
    *c = acc ? *c + s : s;
  }
  __syncthreads();
}

// G = V^T V for a tall column-major V (rows x k, ld), k small: warps own pair
// groups (i <= j), lanes stride over rows, warp shuffles reduce.  G: k x k.
__device__ __forceinline__ void gram_tall(const double* __restrict__ V, int64_t ld, int64_t rows, int k,
                                          double* __restrict__ G) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = int(blockDim.x >> 5);
  const int npairs = k * (k + 1) / 2;
  constexpr int PB = 8;
  for (int base = warp * PB; base < npairs; base += nw * PB) {
    int pi[PB], pj[PB];
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      int e = base + u, i = 0;
      if (e >= npairs) e = npairs - 1;
      while (e >= k - i) {  // pair index -> (i, j) in the upper triangle, row-major
        e -= k - i;
        ++i;
      }
      pi[u] = i;
      pj[u] = i + e;
    }
    double acc[PB];
#pragma unroll
    for (int u = 0; u < PB; ++u) acc[u] = 0.0;
#pragma unroll 4
    for (int64_t r = lane; r < rows; r += 32) {
#pragma unroll
      for (int u = 0; u < PB; ++u) acc[u] = fma(V[r + pi[u] * ld], V[r + pj[u] * ld], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      const double v = warp_sum(acc[u]);
      if (lane == 0 && base + u < npairs) {
        G[pi[u] + pj[u] * k] = v;
        G[pj[u] + pi[u] * k] = v;
      }
    }
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
      s += dot4(pi, 1, pj, 1, inner);
    }
    G[i + j * rows] = s;
    G[j + i * rows] = s;
  }
  __syncthreads();
}

// Register-tiled Gram for larger n: G (n x n, col-major) = sum_x T(x, :)^T T(x, :)
// with T(x, a) = elem(x, a), x < nx. Chunks of x are staged in shared memory
// (cx x n, row-major; `x_fast` picks the staging order so that consecutive
// threads read consecutive global addresses), and each thread accumulates a
// 4x4 block of the upper triangle in registers: per staged row, 8 shared loads
// feed 16 FMAs, against 2 uncoalesced global loads per FMA for a
// thread-per-entry Gram. Blocks beyond one per thread take further passes.
// FP64 tensor-core (DMMA) accumulate: c += a b over one m8n8k4 fragment.
__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Gram on the FP64 tensor cores: G (n x n, col-major) = sum_x T(x, :)^T T(x, :),
// T(x, a) = elem(x, a). Chunks of x are staged in shared memory as for
// gram_tiled; each warp owns up to kTpw 8x8 tiles of the upper triangle and
// accumulates them with mma.sync.m8n8k4.f64 over groups of 4 staged rows: lane
// (g, q) = (lane / 4, lane % 4) feeds A(g, q) = T(x0 + q, i0 + g) and
// B(q, g) = T(x0 + q, j0 + g) and receives G(i0 + g, j0 + 2q + {0, 1}). One
// DMMA replaces 8 per-thread FMAs and the register tiles' shared-memory reloads.
template <class Elem>
__device__ __forceinline__ void gram_tiled_mma(int n, int64_t nx, Elem elem, bool x_fast, double* __restrict__ G,
                                               double* stage, int stage_cap) {
  constexpr int kTpw = 12;
  const int nb = (n + 7) / 8;
  const int ntiles = nb * (nb + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = int(blockDim.x >> 5);
  const int g = lane >> 2, q = lane & 3;
  const int ch = int(imax(4, imin((nx + 3) / 4 * 4, (stage_cap / n) / 4 * 4)));
  for (int base = 0; base < ntiles; base += nw * kTpw) {  // tile groups: each warp takes kTpw tiles
    int ti[kTpw], tj[kTpw];
    double acc[kTpw][2];
#pragma unroll
    for (int u = 0; u < kTpw; ++u) {
      int e = base + warp * kTpw + u, bi = 0;
      if (e >= ntiles) e = -1;
      if (e >= 0) {
        while (e >= nb - bi) {
          e -= nb - bi;
          ++bi;
        }
      }
      ti[u] = e >= 0 ? 8 * bi : -1;
      tj[u] = e >= 0 ? 8 * (bi + e) : -1;
      acc[u][0] = acc[u][1] = 0.0;
    }
    for (int64_t x0 = 0; x0 < nx; x0 += ch) {
      const int cx = int(imin(ch, nx - x0));
      const int cx4 = (cx + 3) & ~3;
      __syncthreads();
      if (x_fast) {
        for (int idx = threadIdx.x; idx < cx4 * n; idx += blockDim.x) {
          const int x = idx % cx4, a = idx / cx4;
          stage[x * n + a] = x < cx ? elem(x0 + x, a) : 0.0;
        }
      } else {
        for (int idx = threadIdx.x; idx < cx4 * n; idx += blockDim.x) {
          const int a = idx % n, x = idx / n;
          stage[x * n + a] = x < cx ? elem(x0 + x, a) : 0.0;
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kTpw; ++u) {
        if (ti[u] < 0) continue;  // warp-uniform
        const int ia = ti[u] + g, ja = tj[u] + g;
        const bool iok = ia < n, jok = ja < n;
        for (int x = 0; x < cx4; x += 4) {
          const double* row = stage + (x + q) * n;
          dmma_884(acc[u][0], acc[u][1], iok ? row[ia] : 0.0, jok ? row[ja] : 0.0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kTpw; ++u) {
      if (ti[u] < 0) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ti[u] + g, j = tj[u] + 2 * q + h;
        if (i < n && j < n) {
          G[i + int64_t(j) * n] = acc[u][h];
          G[j + int64_t(i) * n] = acc[u][h];
        }
      }
    }
  }
  __syncthreads();
}

template <class Elem>
__device__ __forceinline__ void gram_tiled(int n, int64_t nx, Elem elem, bool x_fast, double* __restrict__ G,
                                           double* stage, int stage_cap) {
#ifndef TT_NO_DMMA
  if (n >= 16) {
    gram_tiled_mma(n, nx, elem, x_fast, G, stage, stage_cap);
    return;
  }
#endif
  const int nb = (n + 3) / 4;
  const int ntiles = nb * (nb + 1) / 2;
  const int ch = int(imax(1, imin(nx, stage_cap / n)));
  for (int tile0 = 0; tile0 < ntiles; tile0 += blockDim.x) {
    const int tile = tile0 + threadIdx.x;
    int bi = 0, bj = 0;
    if (tile < ntiles) {  // tile -> (bi <= bj), row-major over the upper triangle
      int e = tile;
      while (e >= nb - bi) {
        e -= nb - bi;
        ++bi;
      }
      bj = bi + e;
    }
    double acc[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
    for (int64_t x0 = 0; x0 < nx; x0 += ch) {
      const int cx = int(imin(ch, nx - x0));
      __syncthreads();
      if (x_fast) {
        for (int idx = threadIdx.x; idx < cx * n; idx += blockDim.x) {
          const int x = idx % cx, a = idx / cx;
          stage[x * n + a] = elem(x0 + x, a);
        }
      } else {
        for (int idx = threadIdx.x; idx < cx * n; idx += blockDim.x) {
          const int a = idx % n, x = idx / n;
          stage[x * n + a] = elem(x0 + x, a);
        }
      }
      __syncthreads();
      if (tile < ntiles) {
        const int i0 = 4 * bi, j0 = 4 * bj;
        for (int x = 0; x < cx; ++x) {
          const double* row = stage + x * n;
          double u[4], v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            u[q] = i0 + q < n ? row[i0 + q] : 0.0;
            v[q] = j0 + q < n ? row[j0 + q] : 0.0;
          }
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] = fma(u[p], v[q], acc[p][q]);
        }
      }
    }
    if (tile < ntiles) {
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = 4 * bi + p, j = 4 * bj + q;
          if (i < n && j < n && i <= j) {
            G[i + int64_t(j) * n] = acc[p][q];
            G[j + int64_t(i) * n] = acc[p][q];
          }
        }
    }
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
    s = dot4(p1, inner, p2, inner, rows);
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
static __device__ int sym_eig(double* A, int n, double* V, int* order, BlockScratch& sc) {
  const int n2 = n + (n & 1);
  const int np = n2 / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nwk = kWarps;
  for (int j = warp; j < n; j += nwk)
    for (int i = lane; i < n; i += 32) V[i + j * n] = (i == j) ? 1.0 : 0.0;
  if (threadIdx.x < 2) sc.rotated[threadIdx.x] = 0;
  if (n <= 1) {
    if (threadIdx.x == 0 && n == 1) order[0] = 0;
    __syncthreads();
    return 0;
  }
  // Skip a rotation when |a_pq| <= max(eps_r sqrt(|a_pp a_qq|), eps_a ||A||_F):
  // the relative test keeps the large eigenpairs accurate to working
  // precision, the absolute floor stops the solver from chasing rounding noise
  // between numerically-zero eigenvalues (eigenvector error <= eps_a/gap).
  double fro = 0.0;
  for (int j = warp; j < n; j += nwk)
    for (int i = lane; i < n; i += 32) fro = fma(A[i + j * n], A[i + j * n], fro);
  const double abs_thr = 1e-15 * sqrt(block_sum(fro, sc));
  const double eps2 = 1e-28;  // relative test (1e-14)^2
  int sweeps_done = 0;
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
          const double a2 = apq * apq;
          if (a2 > eps2 * fabs(app * aqq) && fabs(apq) > abs_thr) {
            // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = (aqq - app) / (2 apq),
            // rewritten without the division by apq (GvL sym.schur2).
            const double th = aqq - app, tw = 2.0 * apq;
            const double den = fabs(th) + sqrt(fma(th, th, tw * tw));
            t = (th >= 0.0 ? tw : -tw) / den;
            c = rsqrt(fma(t, t, 1.0));
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
      for (int P2 = warp; P2 < np; P2 += nwk) {
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
      for (int P1 = warp; P1 < np; P1 += nwk) {
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
    ++sweeps_done;
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
  return sweeps_done;
}

// Shared-memory Jacobi for n <= 52 (pairs <= 26 fit one warp's lanes): every
// warp recomputes the round's rotations in its lanes (lane k <-> pair k) and
// exchanges them by shuffles, A is double-buffered (A0 -> A1) so a round is a
// single barrier, and the round-robin pairing uses conditional subtraction.
// S = dynamic shared base: A0 | A1 | V, each n*n doubles (col-major).
constexpr int kFastEigN = 52;  // np <= 26 lanes; <= 4 pairs per warp needs >= 7 warps

__device__ __forceinline__ void rr_pair(int r, int k, int n2, int& p, int& q) {
  const int m = n2 - 1;
  if (k == 0) {
    p = r;
    q = m;
  } else {
    p = r + k;
    if (p >= m) p -= m;
    q = r - k;
    if (q < 0) q += m;
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

static __device__ int sym_eig_smem(double* S, int n, int* order, BlockScratch& sc) {
  const int n2 = n + (n & 1);
  const int np = n2 / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* A = S;
  double* B = S + n * n;
  double* V = S + 2 * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) V[idx] = (idx % (n + 1) == 0) ? 1.0 : 0.0;
  double fro = 0.0;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) fro = fma(A[idx], A[idx], fro);
  const double abs_thr = 1e-15 * sqrt(block_sum(fro, sc));  // block_sum ends with a barrier
  const double eps2 = 1e-28;
  int sweeps_done = 0;
  if (n <= 1) {
    if (threadIdx.x == 0) order[0] = 0;
    __syncthreads();
    return 0;
  }
  const int nwarps = int(blockDim.x >> 5);
  for (int sweep = 0; sweep < 20; ++sweep) {
    int any = 0;
    for (int r = 0; r < n2 - 1; ++r) {
      // rotation of pair `lane` (identical in every warp)
      int p = 0, q = 0;
      double c = 1.0, sn = 0.0, t = 0.0;
      if (lane < np) {
        rr_pair(r, lane, n2, p, q);
        if (q < n) {
          const double apq = A[p + q * n];
          const double app = A[p + p * n], aqq = A[q + q * n];
          const double th = aqq - app, tw = 2.0 * apq;
          const double h2 = fma(th, th, tw * tw);
          const double den = fabs(th) + sqrt(h2);  // sqrt issued before the threshold test resolves
          if (apq * apq > eps2 * fabs(app * aqq) && fabs(apq) > abs_thr) {
            t = (th >= 0.0 ? tw : -tw) / den;
            c = rsqrt(fma(t, t, 1.0));
            sn = t * c;
          }
        }
      }
      any |= __any_sync(0xffffffffu, sn != 0.0);
      // gather the pair parameters this warp needs up front (overlapped shuffles)
      constexpr int PU = 4;  // pairs per warp: needs >= 7 warps for np <= 26 (256-thread CTAs)
      int p2v[PU], q2v[PU];
      double c2v[PU], s2v[PU];
#pragma unroll
      for (int u = 0; u < PU; ++u) {
        const int P2 = warp + u * nwarps;
        const int src = P2 < 32 ? P2 : 0;
        p2v[u] = __shfl_sync(0xffffffffu, p, src);
        q2v[u] = __shfl_sync(0xffffffffu, q, src);
        c2v[u] = __shfl_sync(0xffffffffu, c, src);
        s2v[u] = __shfl_sync(0xffffffffu, sn, src);
      }
      // B = J^T A J, one owner per 2x2 block (warp <-> P2, lane <-> P1)
      if (lane < np) {
        const bool hq = q < n;
#pragma unroll
        for (int u = 0; u < PU; ++u) {
          const int P2 = warp + u * nwarps;
          if (P2 >= np) break;
          const int p2 = p2v[u], q2 = q2v[u];
          const double c2 = c2v[u], s2 = s2v[u];
          const bool hq2 = q2 < n;
          if (lane == P2) {
            const double app = A[p + p * n];
            if (hq) {
              const double apq = A[p + q * n], aqq = A[q + q * n];
              B[p + p * n] = app - t * apq;
              B[q + q * n] = aqq + t * apq;
              B[p + q * n] = (sn != 0.0) ? 0.0 : apq;
              B[q + p * n] = (sn != 0.0) ? 0.0 : apq;
            } else {
              B[p + p * n] = app;
            }
          } else {
            const double m00 = A[p + p2 * n];
            const double m01 = hq2 ? A[p + q2 * n] : 0.0;
            const double m10 = hq ? A[q + p2 * n] : 0.0;
            const double m11 = (hq && hq2) ? A[q + q2 * n] : 0.0;
            const double x00 = c * m00 - sn * m10, x01 = c * m01 - sn * m11;
            const double x10 = sn * m00 + c * m10, x11 = sn * m01 + c * m11;
            B[p + p2 * n] = c2 * x00 - s2 * x01;
            if (hq2) B[p + q2 * n] = s2 * x00 + c2 * x01;
            if (hq) B[q + p2 * n] = c2 * x10 - s2 * x11;
            if (hq && hq2) B[q + q2 * n] = s2 * x10 + c2 * x11;
          }
        }
      }
      // V = V J (warp <-> pair, lanes <-> rows); same pairs as the P2 set above
#pragma unroll
      for (int u = 0; u < PU; ++u) {
        const int P1 = warp + u * nwarps;
        if (P1 >= np) break;
        const double s1 = s2v[u];
        if (s1 == 0.0) continue;
        const double c1 = c2v[u];
        double* vp = V + p2v[u] * n;
        double* vq = V + q2v[u] * n;
        for (int i = lane; i < n; i += 32) {
          const double a = vp[i], b = vq[i];
          vp[i] = c1 * a - s1 * b;
          vq[i] = s1 * a + c1 * b;
        }
      }
      __syncthreads();
      double* tmp = A;
      A = B;
      B = tmp;
    }
    ++sweeps_done;
    if (!__syncthreads_or(any)) break;
  }
  // the diagonalised matrix must end in S[0 .. n*n)
  if (A != S) {
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) S[idx] = A[idx];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double li = S[i + i * n];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = S[j + j * n];
      if (lj > li || (lj == li && j < i)) ++rank;
    }
    order[rank] = i;
  }
  __syncthreads();
  return sweeps_done;
}

// Sign convention of linalg.cpp:15-31: each column's first max-|.| entry is
// made nonnegative. flips[j] = 1 when column j was negated.
static __device__ void sign_fix(double* U, int64_t rows, int k, int64_t ld, int* flips, BlockScratch& sc) {
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
static __device__ void orthonormalize(double* U, int64_t rows, int j0, int k, int64_t ld, BlockScratch& sc) {
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
