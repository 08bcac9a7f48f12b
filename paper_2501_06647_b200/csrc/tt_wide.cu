// leaf_wide_kernel — tucker_als (tucker.cpp:86-119) on one leaf block per
// thread-block CLUSTER (8 or 16 CTAs, one per SM), for launches with few large
// problems: the streamed leaf of a single-slice append, the raw tail of a range
// query, the brute-force ALS of a few ranges. The one-CTA-per-problem
// leaf_als_kernel (tt_leaf.cu) stays the path for wide batches.
//
// Work split per sweep (same arithmetic and mode order as leaf_als_kernel):
//   * the two streamed passes over X (Y = X x_1 U_1^T, W = X x_0 U_0^T) are
//     split by output tile across the cluster; each CTA streams its tiles
//     through a 6-stage TMA ring (the block stays L2-resident across passes);
//   * the small mode products of the projected tensors are split by output
//     column range;
//   * the leader CTA (rank 0) runs the eigensolvers (llsv), the core and the
//     fit/stop test; with 176 KB of dynamic shared memory a 100 x 100 Jacobi
//     fallback runs in shared memory.
// Phases are separated by cluster barriers (barrier.cluster release/acquire:
// MEMBAR + CCTL.IVALL in the SASS, so every CTA reads the others' global
// writes of the previous phase). Per-CTA partial sums go through the problem's
// exchange slots (LeafWs::xch) and are reduced in rank order by every CTA, so
// all CTAs hold bit-identical scalars and take the same control path.
#include <mutex>

#include "tt_dev.cuh"

namespace ttb {

constexpr int kWideStages = 6;
constexpr size_t kWideDynSmem = size_t(kWideStages * kTileD + kUStage) * sizeof(double);  // 176 KB

struct WPipe {
  uint64_t full[kWideStages];
  uint32_t uses[kWideStages];
};

// ttm_stream_r (tt_dev.cuh) restricted to this CTA's output tiles
// (ot = rank, rank + CS, ...), every j-tile of each, through a kWideStages
// ring: out[o][a][t] = sum_j U[j][a] in[o][j][t].
template <int R>
__device__ __noinline__ void ttm_stream_w(const double* in, int64_t outer, int64_t d, int64_t inner, const double* U,
                                          double* out, double* dyn, WPipe& pp, double* norm_acc, const void* tmap,
                                          int tmap_rank, int rank, int CS) {
  const StreamTile tile = stream_tile(outer, d, inner);
  const int64_t tw = tile.tw, G = tile.G, cj = tile.cj;
  const int64_t ngrp = (outer + G - 1) / G, ntt = (inner + tw - 1) / tw, njt = (d + cj - 1) / cj;
  const int64_t nout = ngrp * ntt;
  const int64_t mine = rank < nout ? (nout - 1 - rank) / CS + 1 : 0;
  const int64_t ntiles = mine * njt;
  double* ring = dyn;
  double* Ut = dyn + kWideStages * kTileD;
  const bool u_smem = d * R <= kUStage;
  if (u_smem) {
    for (int64_t idx = threadIdx.x; idx < d * R; idx += blockDim.x) {
      const int64_t j = idx / R, a = idx - j * R;
      Ut[idx] = U[j + a * d];
    }
  }
  fence_proxy_async();
  __syncthreads();
  auto coords = [&](int64_t u, int64_t& o0, int64_t& j0, int64_t& t0) {
    const int64_t jt = u % njt, ot = rank + (u / njt) * CS;
    const int64_t tt = ot % ntt, grp = ot / ntt;
    o0 = grp * G;
    j0 = jt * cj;
    t0 = tt * tw;
  };
  auto issue = [&](int64_t u) {  // warp 0: fill the stage of local tile u
    const int st = int(u % kWideStages);
    int64_t o0, j0, t0;
    coords(u, o0, j0, t0);
    const int64_t g_n = imin(G, outer - o0), jn = imin(cj, d - j0), tn = imin(tw, inner - t0);
    double* dst = ring + int64_t(st) * kTileD;
    const int lane = threadIdx.x & 31;
    if (tmap != nullptr) {
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&pp.full[st], uint32_t(G * cj * tw * sizeof(double)));
        if (tmap_rank == 3)
          tma_load_3d(dst, tmap, int(t0), int(j0), int(o0), &pp.full[st]);
        else
          tma_load_2d(dst, tmap, int(t0), int(j0), &pp.full[st]);
      }
      return;
    }
    const bool whole_rows = (tn == inner);
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
      bulk_g2s(dst + (g * cj + jj) * tw, in + ((o0 + g) * d + j0 + jj) * inner + t0, seg_bytes, &pp.full[st]);
    }
  };
  if (threadIdx.x < 32)
    for (int64_t u = 0; u < imin(int64_t(kWideStages), ntiles); ++u) issue(u);
  double acc[R];
  double nrm = 0.0;
  for (int64_t u = 0; u < ntiles; ++u) {
    const int st = int(u % kWideStages);
    int64_t o0, j0, t0;
    coords(u, o0, j0, t0);
    const int64_t jt = u % njt;
    const int64_t g_n = imin(G, outer - o0), jn = imin(cj, d - j0), tn = imin(tw, inner - t0);
    const int64_t g = threadIdx.x / tw, tl = threadIdx.x - g * tw;
    const bool active = threadIdx.x < G * tw && g < g_n && tl < tn;
    if (jt == 0) {
#pragma unroll
      for (int a = 0; a < R; ++a) acc[a] = 0.0;
    }
    mbar_wait(&pp.full[st], pp.uses[st] & 1u);
    if (active) {
      const double* x = ring + int64_t(st) * kTileD + g * cj * tw + tl;
      if (u_smem) {
#pragma unroll 2
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
          for (int a = 0; a < R; ++a) acc[a] = fma(U[(j0 + jj) + a * d], xv, acc[a]);
        }
      }
      if (jt == njt - 1) {
        double* dst = out + (o0 + g) * R * inner + t0 + tl;
#pragma unroll
        for (int a = 0; a < R; ++a) dst[a * inner] = acc[a];
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) pp.uses[st] += 1;
    if (threadIdx.x < 32 && u + kWideStages < ntiles) issue(u + kWideStages);
  }
  if (norm_acc) *norm_acc += nrm;
  __syncthreads();
}

__device__ __forceinline__ void ttm_stream_wide(const double* in, int64_t outer, int64_t d, int64_t inner,
                                                const double* U, int r, double* out, double* dyn, WPipe& pp,
                                                double* norm_acc, const void* tmap, int tmap_rank, int rank, int CS) {
  switch (r) {
#define TT_CASE(N)                                                                                  \
  case N:                                                                                           \
    ttm_stream_w<N>(in, outer, d, inner, U, out, dyn, pp, norm_acc, tmap, tmap_rank, rank, CS); \
    break;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10) TT_CASE(11) TT_CASE(12) TT_CASE(13) TT_CASE(14) TT_CASE(15) TT_CASE(16)
#undef TT_CASE
    default:
      break;
  }
}

// Mode product out[o][a][t] = sum_j M(a, j) in[o][j][t] (M(a, j) =
// M[a*ms_a + j*ms_j]) over this CTA's share [c0, c1) of the output columns
// c = o*inner + t. Plain (coherent) loads: `in` was written by other CTAs.
template <int RT>
__device__ __forceinline__ void ttm_cols_chunk(const double* in, int64_t d, int64_t inner, const double* M,
                                               int64_t ms_a, int64_t ms_j, int a0, int na, double* out,
                                               int64_t r_total, int64_t c0, int64_t c1) {
  for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const int64_t o = c / inner, t = c - o * inner;
    const double* src = in + o * d * inner + t;
    double s[RT];
#pragma unroll
    for (int a = 0; a < RT; ++a) s[a] = 0.0;
    for (int64_t j = 0; j < d; ++j) {
      const double x = src[j * inner];
      const double* mj = M + j * ms_j + int64_t(a0) * ms_a;
#pragma unroll
      for (int a = 0; a < RT; ++a)
        if (a < na) s[a] = fma(mj[a * ms_a], x, s[a]);
    }
    double* dst = out + o * r_total * inner + t;
#pragma unroll
    for (int a = 0; a < RT; ++a)
      if (a < na) dst[int64_t(a0 + a) * inner] = s[a];
  }
}

__device__ __forceinline__ void mode_product_cl(const double* in, int64_t outer, int64_t d, int64_t inner,
                                                const double* M, int64_t ms_a, int64_t ms_j, int64_t r, double* out,
                                                int rank, int CS) {
  const int64_t ncol = outer * inner;
  const int64_t per = (ncol + CS - 1) / CS;
  const int64_t c0 = imin(ncol, int64_t(rank) * per), c1 = imin(ncol, c0 + per);
  for (int a0 = 0; a0 < r; a0 += 16) {
    const int na = int(imin(16, r - a0));
    if (na <= 4)
      ttm_cols_chunk<4>(in, d, inner, M, ms_a, ms_j, a0, na, out, r, c0, c1);
    else if (na <= 8)
      ttm_cols_chunk<8>(in, d, inner, M, ms_a, ms_j, a0, na, out, r, c0, c1);
    else
      ttm_cols_chunk<16>(in, d, inner, M, ms_a, ms_j, a0, na, out, r, c0, c1);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1) leaf_wide_kernel(Params prm, const LeafDesc* __restrict__ descs) {
  __shared__ BlockScratch sc;
  __shared__ WPipe pipe;
  extern __shared__ __align__(128) double dsm[];
  const long long t_kernel = tstart();
  const int rank = int(cl_rank()), CS = int(cl_size());
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    sc.eig_calls = sc.eig_sweeps = sc.si_ok = sc.si_fail = sc.si_iters = 0;
    sc.dsm_cap = int(dyn_smem_doubles());
    for (int i = 0; i < 12; ++i) sc.cyc[i] = 0;
    for (int i = 0; i < kWideStages; ++i) {
      mbar_init(&pipe.full[i], 1);
      pipe.uses[i] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  const LeafDesc D = descs[cl_id()];
  const int p = prm.p;
  int64_t d[kMaxP], rc[kMaxP], k[kMaxP];
  d[0] = D.len;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, rc);
  const LeafWs lay = leaf_ws_layout(p, D.len, prm.d, prm.req, CS);
  double* W = D.ws + lay.W;
  double* gpart = D.ws + lay.gpart;
  double* B[2] = {D.ws + lay.B1, D.ws + lay.B2};
  double* G = D.ws + lay.G;
  double* V = D.ws + lay.V;
  double* misc = D.ws + lay.misc;
  double* xch = D.ws + lay.xch;  // [0, CS): per-CTA partial sums; [32]: stop flag
  const double* X = D.x;
  const int64_t ns = prod_range(d, 1, p);
  for (int n = 0; n < p; ++n) {
    if (leader) bcopy(D.out_f[n], D.init[n], d[n] * rc[n]);
    k[n] = rc[n];
  }
  cl_sync();
  int sweeps = 0, converged = 0;
  double norm_sq = 0.0, norm = 0.0;
  double prev_fit = nan("");
  for (int sweep = 0; sweep < prm.max_iters; ++sweep) {
    // ---- mode 0: Y = X x_1 U_1^T ... x_{p-1} U_{p-1}^T (split), U_0 = llsv(M_0(Y)) (leader)
    const int64_t k0n = leaf_mode_rank(p, d, k, 0);
    int64_t cur[kMaxP];
    for (int m = 0; m < p; ++m) cur[m] = d[m];
    const double* src = X;
    int tog = 0;
    for (int m = 1; m < p; ++m) {
      double* dst = B[tog];
      const int64_t inner = prod_range(cur, m + 1, p);
      if (m == 1) {
        const long long tb = tstart();
        double nacc = 0.0;
        if (stream_ok(X, inner, int(k[1]))) {
          ttm_stream_wide(X, d[0], d[1], inner, D.out_f[1], int(k[1]), dst, dsm, pipe, sweep == 0 ? &nacc : nullptr,
                          D.tmaps, 3, rank, CS);
        } else {
          if (sweep == 0) {
            const int64_t tot = D.len * ns, per = (tot + CS - 1) / CS;
            const int64_t e0 = imin(tot, rank * per), e1 = imin(tot, e0 + per);
            for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) nacc = fma(X[i], X[i], nacc);
          }
          mode_product_cl(src, prod_range(cur, 0, m), cur[m], inner, D.out_f[m], d[m], 1, k[m], dst, rank, CS);
        }
        if (sweep == 0) {
          const double part = block_sum(nacc, sc);
          if (threadIdx.x == 0) xch[rank] = part;
        }
        tstop(sc, kPhBig, tb);
      } else {
        mode_product_cl(src, prod_range(cur, 0, m), cur[m], inner, D.out_f[m], d[m], 1, k[m], dst, rank, CS);
      }
      cl_sync();
      cur[m] = k[m];
      src = dst;
      tog ^= 1;
    }
    if (sweep == 0) {
      norm_sq = 0.0;
      for (int r = 0; r < CS; ++r) norm_sq += xch[r];  // rank order: identical in every CTA
      if (norm_sq == 0.0) {  // tucker.cpp:96-100: init factors, zero core
        if (leader) bzero(D.out_core, prod_range(rc, 0, p));
        converged = 1;
        break;
      }
      norm = sqrt(norm_sq);
    }
    wide_llsv(src, 1, d[0], prod_range(cur, 1, p), k0n, D.out_f[0], G, V, misc, dsm, sc, k[0], D.ws + lay.SI, gpart,
              rank, CS);
    k[0] = k0n;
    cl_sync();
    // ---- W = X x_0 U_0^T : (k0, D_1, ..., D_{p-1}), split
    {
      const long long tb = tstart();
      if (stream_ok(X, ns, int(k[0])))
        ttm_stream_wide(X, 1, d[0], ns, D.out_f[0], int(k[0]), W, dsm, pipe, nullptr,
                        D.tmaps ? static_cast<const char*>(D.tmaps) + 128 : nullptr, 2, rank, CS);
      else
        mode_product_cl(X, 1, d[0], ns, D.out_f[0], d[0], 1, k[0], W, rank, CS);
      tstop(sc, kPhBig, tb);
    }
    cl_sync();
    // ---- modes n >= 1 from W: products split, llsv on the leader
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
        const long long tt = tstart();
        mode_product_cl(s2, prod_range(pc, 0, m), pc[m], prod_range(pc, m + 1, p), D.out_f[m], d[m], 1, k[m], dst,
                        rank, CS);
        tstop(sc, kPhTtm, tt);
        cl_sync();
        pc[m] = k[m];
        s2 = dst;
        t2 ^= 1;
      }
      wide_llsv(s2, prod_range(pc, 0, n), d[n], prod_range(pc, n + 1, p), kn, D.out_f[n], G, V, misc, dsm, sc, k[n],
                D.ws + lay.SI, gpart, rank, CS);
      k[n] = kn;
      Pn = s2;
      cl_sync();
    }
    // ---- core = P_{p-1} x_{p-1} U_{p-1}^T (== core_of(x, U), tucker.cpp:67-76), fit and stop (leader)
    if (leader) {
      mode_product(Pn, prod_range(k, 0, p - 1), d[p - 1], 1, D.out_f[p - 1], d[p - 1], 1, k[p - 1], D.out_core,
                   false, sc);
      const double core_sq = bsumsq(D.out_core, prod_range(k, 0, p), sc);
      const double res = fmax(0.0, norm_sq - core_sq);
      const double fit = 1.0 - sqrt(res) / norm;
      if (threadIdx.x == 0) {
        D.objective[sweep] = res;
        xch[32] = (sweep > 0 && fabs(fit - prev_fit) < prm.tol) ? 1.0 : 0.0;
        xch[33] = fit;
      }
    }
    cl_sync();
    sweeps = sweep + 1;
    if (xch[32] != 0.0) {
      converged = 1;
      break;
    }
    prev_fit = xch[33];
  }
  if (leader && threadIdx.x == 0) {
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
  // no CTA may exit while another can still read the exchange slots
  cl_sync();
}

// Cluster size for the wide leaf kernel on the current device: 16 CTAs (one
// per SM, non-portable size) when the GPU can co-schedule such a cluster, else
// the portable 8. 0 when neither fits.
int leaf_wide_cluster() {
  static std::mutex mu;
  static int cs[64];
  static uint64_t done = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(mu);
  if (done >> (dev & 63) & 1) return cs[dev & 63];
  int best = 0;
  if (ensure_dyn_smem(reinterpret_cast<const void*>(leaf_wide_kernel), 2, kWideDynSmem) == cudaSuccess) {
    cudaFuncSetAttribute(leaf_wide_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {16, 8}) {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = kWideDynSmem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, leaf_wide_kernel, &cfg) == cudaSuccess && ncl > 0) {
        best = c;
        break;
      }
      cudaGetLastError();
    }
  }
  cudaGetLastError();
  cs[dev & 63] = best;
  done |= uint64_t(1) << (dev & 63);
  return best;
}

cudaError_t launch_leaf_wide(const Params& prm, const LeafDesc* d_descs, int n, int cs, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(unsigned(n * cs));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kWideDynSmem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, leaf_wide_kernel, prm, d_descs);
  g_launches.fetch_add(1);
  return e;
}

}  // namespace ttb
