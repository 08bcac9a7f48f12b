// Grid-wide leaf path — tucker_als (tucker.cpp:86-119) on a batch of
// equal-length leaf blocks (a tree build, a streamed leaf, a query's raw
// tail), run as phase kernels over all leaves instead of one CTA per leaf:
//
//   per sweep   grid_ttm_kernel   Y_l = X_l x_1 U_1^T   every leaf, tiles across the whole GPU
//               grid_last_kernel  Y x_2 U_2^T (order 3)  whole GPU
//               grid_solve0       remaining small products, U_0 = llsv(M_0(Y))   one CTA per leaf
//               grid_ttm_kernel   W_l = X_l x_0 U_0^T   every leaf, tiles across the whole GPU
//   per mode    grid_ttm / grid_last   first (W-sized) product of the mode's chain, whole GPU
//     n >= 1    grid_gram_kernel  partial Grams of the dense mode-1 unfolding (16 row chunks per leaf)
//               grid_solve_mode   rest of the chain, U_n = llsv; last mode: core, fit / stop   one CTA per leaf
//
// Same arithmetic, mode order and stop rule as leaf_als_kernel (tt_leaf.cu;
// the streamed products accumulate in the same order, so the two paths agree
// bit for bit on a build); the passes over X — >95% of a C3 leaf's bytes and
// flops — and the W-sized products leave the per-leaf CTA. grid_ttm_kernel is
// a persistent kernel (one CTA per SM): a producer warp streams X tiles and
// the matching rows of the transposed, zero-padded factor through a 5-stage
// cp.async.bulk ring (full/empty mbarriers), and 256 consumer threads each own
// TT consecutive columns of one slab and RC accumulator columns in registers
// (RC*TT DFMAs per 1-2 LDS.128 of X and RC/2 broadcast LDS.128 of U^T). X is
// read from HBM once per pass (ncu: 4.34 GB for 4.33 GB of X at C3) and never
// staged through a per-leaf workspace. Small batches take one slab and two
// columns per thread so that a single leaf still spreads over the GPU.
//
// The per-leaf ALS state (column counts, ||X||^2, previous fit, stop flag)
// lives in the leaf's workspace (GridWs::state); converged leaves are skipped
// by every later phase. The host runs sweeps until the device-side count of
// unconverged leaves reaches zero (one 4-byte readback per sweep).
#include <mutex>

#include "tt_dev.cuh"

namespace ttb {

constexpr int kGridStages = 5;
constexpr int kGridUtStage = int(kGridCjMax * kGridUtLd);              // staged U^T doubles per stage
constexpr int kGridStageD = int(kGridTileDoubles) + kGridUtStage;      // 36 KB
constexpr size_t kGridDynSmem = size_t(kGridStages) * kGridStageD * sizeof(double);  // 180 KB: one CTA per SM
constexpr int kGridConsumers = 256;
constexpr int kGridThreads = kGridConsumers + 32;

struct GridPipe {
  uint64_t full[kGridStages];
  uint64_t empty[kGridStages];
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Shapes of one streamed pass over a leaf: pass 1 is Y = X x_1 U_1^T (X as
// (len, D_1, rest)), pass 2 is W = X x_0 U_0^T (X as (1, len, ns)), pass 3 is
// W x_1 U_1^T (W as (k0, D_1, rest)): the first product of every mode n >= 2.
struct GridPassShape {
  int64_t outer, d, inner;
};
__host__ __device__ __forceinline__ GridPassShape grid_pass_shape(const Params& prm, int64_t len, int pass, int64_t k0) {
  GridPassShape s;
  if (pass == 1 || pass == 3) {
    s.outer = pass == 1 ? len : k0;
    s.d = prm.d[1];
    s.inner = prod_range(prm.d, 2, prm.p);
  } else {
    s.outer = 1;
    s.d = len;
    s.inner = prod_range(prm.d, 1, prm.p);
  }
  return s;
}

// One work item = (leaf, accumulator chunk, slab group, column tile).
template <int RC, int TT>
__global__ void __launch_bounds__(kGridThreads, 1)
grid_ttm_kernel(Params prm, const LeafDesc* __restrict__ descs, int nleaves, int pass, int R, int want_norm,
                int k0, int gcap) {
  __shared__ GridPipe pipe;
  __shared__ double red[8];
  extern __shared__ __align__(128) double dsm[];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGridStages; ++i) {
      mbar_init(&pipe.full[i], 1);
      mbar_init(&pipe.empty[i], kGridConsumers / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t len = descs[0].len;  // equal-length batch
  const GridPassShape sh = grid_pass_shape(prm, len, pass, k0);
  const GridTile tile = grid_tile(sh.outer, sh.d, sh.inner, gcap, TT);
  const GridChunks ch = grid_chunks(R);
  const LeafWs lay = leaf_ws_layout(prm.p, len, prm.d, prm.req);
  const GridWs gw = grid_ws_layout(prm.p, len, prm.d, prm.req);
  const int64_t tw = tile.tw, G = tile.G, cj = tile.cj, njt = tile.njt;
  const int64_t per_leaf = int64_t(ch.nchunk) * tile.ngrp * tile.ntt;
  const int64_t nitems = per_leaf * nleaves;
  const bool whole = tw == sh.inner;  // a slab's cj rows are one contiguous segment
  uint32_t it = 0;                    // ring step, continuous across items
  if (threadIdx.x >= kGridConsumers) {
    // ---------------- producer warp ----------------
    const int lane = threadIdx.x & 31;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
      const int64_t leaf = item / per_leaf, r0 = item - leaf * per_leaf;
      const LeafDesc& D = descs[leaf];
      if (D.ws[gw.state + kGsDone] != 0.0) continue;
      const int64_t r1 = r0 % (tile.ngrp * tile.ntt);
      const int64_t grp = r1 / tile.ntt, tt = r1 - grp * tile.ntt;
      const int64_t o0 = grp * G, g_n = imin(G, sh.outer - o0);
      const int64_t t0 = tt * tw, tn = imin(tw, sh.inner - t0);
      const double* in = pass == 3 ? D.ws + lay.W : D.x;
      const double* Ut = D.ws + (pass == 2 ? gw.ut0 : gw.ut1);
      for (int64_t u = 0; u < njt; ++u, ++it) {
        const int st = int(it % kGridStages);
        const uint32_t use = it / kGridStages;
        if (use > 0) mbar_wait(&pipe.empty[st], (use - 1) & 1u);
        const int64_t j0 = u * cj, jn = imin(cj, sh.d - j0);
        const int64_t nseg = whole ? g_n : g_n * jn;
        const uint32_t seg_bytes = uint32_t((whole ? jn * sh.inner : tn) * sizeof(double));
        const uint32_t ut_bytes = uint32_t(jn * ch.rp * sizeof(double));
        double* dst = dsm + int64_t(st) * kGridStageD;
        if (lane == 0) {
          mbar_arrive_expect_tx(&pipe.full[st], uint32_t(nseg) * seg_bytes + ut_bytes);
          bulk_g2s(dst + kGridTileDoubles, Ut + j0 * ch.rp, ut_bytes, &pipe.full[st]);
        }
        __syncwarp();
        for (int64_t sg = lane; sg < nseg; sg += 32) {
          int64_t g, jj;
          if (whole) {
            g = sg;
            jj = 0;
          } else {
            g = sg / jn;
            jj = sg - g * jn;
          }
          bulk_g2s(dst + (g * cj + jj) * tw, in + ((o0 + g) * sh.d + j0 + jj) * sh.inner + t0, seg_bytes,
                   &pipe.full[st]);
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const int tid = threadIdx.x;
  const int64_t g = tid / tile.tpo, tq = tid - g * tile.tpo;
  const int xoff = int((g * cj) * tw + tq * TT), itw = int(tw), irp = ch.rp;
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int64_t leaf = item / per_leaf, r0 = item - leaf * per_leaf;
    const LeafDesc& D = descs[leaf];
    if (D.ws[gw.state + kGsDone] != 0.0) continue;
    const int64_t chunk = r0 / (tile.ngrp * tile.ntt), r1 = r0 - chunk * (tile.ngrp * tile.ntt);
    const int64_t grp = r1 / tile.ntt, tt = r1 - grp * tile.ntt;
    const int64_t o0 = grp * G, g_n = imin(G, sh.outer - o0);
    const int64_t t0 = tt * tw, tn = imin(tw, sh.inner - t0);
    const int a0 = int(chunk) * RC;
    const bool active = g < g_n && tq * TT < tn;
    double acc[RC][TT];
#pragma unroll
    for (int a = 0; a < RC; ++a)
#pragma unroll
      for (int q = 0; q < TT; ++q) acc[a][q] = 0.0;
    double nrm = 0.0;
    for (int64_t u = 0; u < njt; ++u, ++it) {
      const int st = int(it % kGridStages);
      mbar_wait(&pipe.full[st], (it / kGridStages) & 1u);
      if (active) {
        const int jn = int(imin(cj, sh.d - u * cj));
        const double* xs = dsm + st * kGridStageD + xoff;
        const double* ur = dsm + st * kGridStageD + int(kGridTileDoubles) + a0;
#pragma unroll 1
        for (int jj = 0; jj < jn; ++jj, xs += itw, ur += irp) {
          double xv[TT];
#pragma unroll
          for (int q = 0; q < TT; q += 2) {
            const double2 t2 = *reinterpret_cast<const double2*>(xs + q);
            xv[q] = t2.x;
            xv[q + 1] = t2.y;
          }
          if (want_norm) {
#pragma unroll
            for (int q = 0; q < TT; ++q) nrm = fma(xv[q], xv[q], nrm);
          }
#pragma unroll
          for (int a = 0; a + 1 < RC; a += 2) {
            const double2 u2 = *reinterpret_cast<const double2*>(ur + a);
#pragma unroll
            for (int q = 0; q < TT; ++q) acc[a][q] = fma(u2.x, xv[q], acc[a][q]);
#pragma unroll
            for (int q = 0; q < TT; ++q) acc[a + 1][q] = fma(u2.y, xv[q], acc[a + 1][q]);
          }
          if (RC & 1) {
            const double u1 = ur[RC - 1];
#pragma unroll
            for (int q = 0; q < TT; ++q) acc[RC - 1][q] = fma(u1, xv[q], acc[RC - 1][q]);
          }
        }
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&pipe.empty[st]);
    }
    if (active) {
      double* out = D.ws + (pass == 2 ? lay.W : lay.B1) + (o0 + g) * R * sh.inner + t0 + tq * TT;
#pragma unroll
      for (int a = 0; a < RC; ++a) {
        if (a0 + a < R) {
#pragma unroll
          for (int q = 0; q < TT; q += 2)
            *reinterpret_cast<double2*>(out + int64_t(a0 + a) * sh.inner + q) = make_double2(acc[a][q], acc[a][q + 1]);
        }
      }
    }
    if (want_norm) {  // block-uniform: ||X||^2 partial of this tile, fixed summation order
      const double w = warp_sum(nrm);
      consumer_sync();
      if ((tid & 31) == 0) red[tid >> 5] = w;
      consumer_sync();
      if (tid == 0 && chunk == 0) {
        double s = 0.0;
        for (int i = 0; i < kGridConsumers / 32; ++i) s += red[i];
        D.ws[gw.npart + r1] = s;
      }
    }
  }
}

// Last-mode contraction of W for order-3 series: sum_t W[c][t] U[t][a] over the
// k0*D_1 rows c = (o, j) of every leaf (the first product of mode 1,
// W x_2 U_2^T), written as the mode-1 unfolding itself: a dense row-major
// D_1 x (k0*R) matrix out[j][o*R + a], so the solver's Gram, warm start and
// back-multiplication read contiguous rows. A CTA stages 128 contiguous rows (padded against bank
// conflicts) and U^T in shared memory; a thread owns one row and half of the
// R columns.
constexpr int kLastRows = 128;
constexpr int64_t kLastMaxD = 94;  // (d + 2) * 128 rows * 8 B <= 96 KB
template <int RH>
__global__ void __launch_bounds__(256, 2)
grid_last_kernel(Params prm, const LeafDesc* __restrict__ descs, int64_t rows, int R, int which) {
  extern __shared__ __align__(128) double dsm[];
  const int64_t tiles = (rows + kLastRows - 1) / kLastRows;
  const int64_t leaf = blockIdx.x / tiles, tile = blockIdx.x - leaf * tiles;
  const LeafDesc& D = descs[leaf];
  const int p = prm.p;
  const LeafWs lay = leaf_ws_layout(p, D.len, prm.d, prm.req);
  const GridWs gw = grid_ws_layout(p, D.len, prm.d, prm.req);
  if (D.ws[gw.state + kGsDone] != 0.0) return;
  const int d = int(prm.d[p - 1]), ldx = d + 2;
  constexpr int rp = 2 * RH;
  double* xs = dsm;
  double* us = dsm + kLastRows * ldx;
  const int64_t c0 = tile * kLastRows;
  const int nr = int(imin(kLastRows, rows - c0));
  const double* U = D.out_f[p - 1];
  for (int idx = threadIdx.x; idx < d * rp; idx += blockDim.x) {
    const int a = idx / d, t = idx - a * d;
    us[t * rp + a] = a < R ? U[t + int64_t(a) * d] : 0.0;
  }
  // which = 1: W (k0*D_1 rows) -> dense mode-1 unfolding in B1; which = 0: pass-1 output Y in B1 (len*k1 rows)
  // -> Y x_2 U_2^T in B2, natural order (the dense len x (k1*R) mode-0 unfolding)
  const double2* src = reinterpret_cast<const double2*>(D.ws + (which ? lay.W : lay.B1) + c0 * d);
  for (int i2 = threadIdx.x; i2 < nr * d / 2; i2 += blockDim.x) {
    const int e = 2 * i2, r = e / d, t = e - r * d;
    *reinterpret_cast<double2*>(xs + r * ldx + t) = src[i2];
  }
  __syncthreads();
  const int r = threadIdx.x >> 1, a0 = (threadIdx.x & 1) * RH;
  if (r >= nr) return;
  double acc[RH];
#pragma unroll
  for (int a = 0; a < RH; ++a) acc[a] = 0.0;
  const double* xr = xs + r * ldx;
  const double* ur = us + a0;
#pragma unroll 4
  for (int t = 0; t < d; ++t) {
    const double x = xr[t];
#pragma unroll
    for (int a = 0; a < RH; ++a) acc[a] = fma(ur[t * rp + a], x, acc[a]);
  }
  const int64_t c = c0 + r, d1 = prm.d[1], o = c / d1, j = c - o * d1;
  double* out = which ? D.ws + lay.B1 + j * (rows / d1) * R + o * R + a0 : D.ws + lay.B2 + c * R + a0;
#pragma unroll
  for (int a = 0; a < RH; ++a)
    if (a0 + a < R) out[a] = acc[a];
}

cudaError_t grid_solve_prepare();
void launch_grid_prep(const Params& prm, const LeafDesc* d_descs, int n, int* d_active, cudaStream_t st);
void launch_grid_solve0(const Params& prm, const LeafDesc* d_descs, int n, int sweep, int gcap, int tt1, int y_done,
                        cudaStream_t st);
void launch_grid_solve_mode(const Params& prm, const LeafDesc* d_descs, int n, int sweep, int mode, int first_done,
                            int gram_ready, int* d_active, cudaStream_t st);
bool grid_gram_applies(int64_t rows, int64_t cols, int64_t k);
void launch_grid_gram(const Params& prm, const LeafDesc* d_descs, int n, int cols, cudaStream_t st);

// ---------------------------------------------------------------------------
using GridTtmFn = void (*)(Params, const LeafDesc*, int, int, int, int, int, int);
template <int TT>
static GridTtmFn grid_ttm_fn(int rc) {
  switch (rc) {
#define TT_CASE(N) \
  case N:          \
    return grid_ttm_kernel<N, TT>;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8) TT_CASE(9) TT_CASE(10)
#undef TT_CASE
    default:
      return nullptr;
  }
}

using GridLastFn = void (*)(Params, const LeafDesc*, int64_t, int, int);
static GridLastFn grid_last_fn(int rh) {
  switch (rh) {
#define TT_CASE(N) \
  case N:          \
    return grid_last_kernel<N>;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10) TT_CASE(11) TT_CASE(12) TT_CASE(13) TT_CASE(14) TT_CASE(15) TT_CASE(16)
#undef TT_CASE
    default:
      return nullptr;
  }
}
constexpr size_t kLastDynSmem = size_t(kLastRows * (kLastMaxD + 2) + kLastMaxD * 32) * sizeof(double);  // 120 KB cap

// Device time of the streamed passes over X (passes 1 and 2), for the bench's
// live roofline: events around each launch, read after the sweep's sync.
static std::mutex g_pass_mu;
static double g_pass_stats[3] = {0.0, 0.0, 0.0};  // launches, ms, X bytes
void grid_pass_stats(double* out3) {
  std::lock_guard<std::mutex> lk(g_pass_mu);
  for (int i = 0; i < 3; ++i) out3[i] = g_pass_stats[i];
}
struct PassEvents {
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int dev = -1;
  bool ensure() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return false;
    if (d == dev) return true;
    for (auto& e : ev) {
      if (e) cudaEventDestroy(e);
      if (cudaEventCreate(&e) != cudaSuccess) return false;
    }
    dev = d;
    return true;
  }
};

// Per-device launch state: shared-memory caps set once, resident CTA count.
static cudaError_t grid_prepare(int* ctas_out) {
  static std::mutex mu;
  static uint64_t done = 0;
  static int ctas[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (!(done >> (dev & 63) & 1)) {
    for (int rc = 1; rc <= int(kGridRcMax); ++rc) {
      e = cudaFuncSetAttribute(grid_ttm_fn<2>(rc), cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGridDynSmem));
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(grid_ttm_fn<4>(rc), cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGridDynSmem));
      if (e != cudaSuccess) return e;
    }
    for (int rh = 1; rh <= 16; ++rh) {
      e = cudaFuncSetAttribute(grid_last_fn(rh), cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLastDynSmem));
      if (e != cudaSuccess) return e;
    }
    if ((e = grid_solve_prepare()) != cudaSuccess) return e;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    ctas[dev & 63] = nsm;
    done |= uint64_t(1) << (dev & 63);
  }
  *ctas_out = ctas[dev & 63];
  return cudaSuccess;
}

// Whether a batch of n equal-length leaves can take the grid-wide path.
bool leaf_grid_ok(const Params& prm, int64_t len) {
  if (prm.p < 3) return false;
  const int64_t rest = prod_range(prm.d, 2, prm.p);
  if (rest % 2 != 0) return false;
  int64_t d[kMaxP], rc[kMaxP];
  d[0] = len;
  for (int m = 1; m < prm.p; ++m) d[m] = prm.d[m];
  clamp_ranks(prm.p, d, prm.req, rc);
  for (int m = 0; m < prm.p; ++m)
    if (rc[m] > kGridUtLd) return false;
  return true;
}

// Runs the whole ALS of the batch on `st` (asynchronous except for the
// per-sweep 4-byte readback of the unconverged count). `active`: max_iters
// device ints. Returns the first CUDA error.
cudaError_t launch_leaf_grid(const Params& prm, const LeafDesc* d_descs, int n, int64_t len, int* d_active,
                             cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int ctas = 0;
  cudaError_t e = grid_prepare(&ctas);
  if (e != cudaSuccess) return e;
  const int p = prm.p;
  int64_t d[kMaxP], k[kMaxP];
  d[0] = len;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, k);
  launch_grid_prep(prm, d_descs, n, d_active, st);
  int tt_pass1 = 4;  // columns per thread of pass 1 (the solve sums that pass's norm partials)
  static thread_local PassEvents pe;
  const bool timed = pe.ensure();
  auto ttm = [&](int pass, int64_t R, int want_norm) -> cudaError_t {
    const GridPassShape sh = grid_pass_shape(prm, len, pass, k[0]);
    // slabs per tile: enough items for two per SM when the batch is small
    const int64_t gcap = imax(1, sh.outer * n / (2 * ctas));
    GridTile t = grid_tile(sh.outer, sh.d, sh.inner, gcap);
    // too few work items to fill the SMs: two columns per thread instead of four
    if (t.tt == 4 && t.ngrp * t.ntt * n < ctas) t = grid_tile(sh.outer, sh.d, sh.inner, gcap, 2);
    const GridChunks ch = grid_chunks(R);
    const int64_t items = int64_t(ch.nchunk) * t.ngrp * t.ntt * n;
    if (pass == 1) tt_pass1 = int(t.tt);
    GridTtmFn fn = t.tt == 4 ? grid_ttm_fn<4>(ch.rc) : grid_ttm_fn<2>(ch.rc);
    if (!fn) return cudaErrorInvalidValue;
    if (timed && pass <= 2) cudaEventRecord(pe.ev[2 * (pass - 1)], st);
    fn<<<unsigned(imin(items, ctas)), kGridThreads, kGridDynSmem, st>>>(prm, d_descs, n, pass, int(R), want_norm,
                                                                         int(k[0]), int(gcap));
    if (timed && pass <= 2) cudaEventRecord(pe.ev[2 * (pass - 1) + 1], st);
    g_launches.fetch_add(1);
    return cudaGetLastError();
  };
  // W x_2 U_2^T for order-3 series (the first product of mode 1)
  auto last = [&](int which) -> cudaError_t {
    const int64_t rows = which ? k[0] * d[1] : len * k[1], R = k[2];
    const int rh = int((R + 1) / 2);
    GridLastFn fn = grid_last_fn(rh);
    if (!fn) return cudaErrorInvalidValue;
    const int64_t tiles = (rows + kLastRows - 1) / kLastRows;
    const size_t smem = size_t(kLastRows * (d[2] + 2) + d[2] * 2 * rh) * sizeof(double);
    fn<<<unsigned(tiles * n), 256, smem, st>>>(prm, d_descs, rows, int(R), which);
    g_launches.fetch_add(1);
    return cudaGetLastError();
  };
  int prev_left = n;
  for (int sweep = 0; sweep < prm.max_iters; ++sweep) {
    if ((e = ttm(1, k[1], sweep == 0)) != cudaSuccess) return e;
    const bool last_ok = p == 3 && d[2] <= kLastMaxD && d[2] % 2 == 0 && k[2] <= 32;
    if (last_ok && (e = last(0)) != cudaSuccess) return e;  // Y x_2 U_2^T, grid-wide
    launch_grid_solve0(prm, d_descs, n, sweep, int(imax(1, len * n / (2 * ctas))), tt_pass1, last_ok ? 1 : 0, st);
    k[0] = leaf_mode_rank(p, d, k, 0);
    if ((e = ttm(2, k[0], 0)) != cudaSuccess) return e;
    for (int m = 1; m < p; ++m) {
      // the W-sized first product of the mode's chain, grid-wide where a kernel covers its shape
      int first_done = 0, gram_ready = 0;
      if (m >= 2) {
        if ((e = ttm(3, k[1], 0)) != cudaSuccess) return e;
        first_done = 1;
      } else if (last_ok) {
        if ((e = last(1)) != cudaSuccess) return e;
        first_done = 1;
        // its Gram, split over row chunks across the GPU
        if (grid_gram_applies(d[1], k[0] * k[2], leaf_mode_rank(p, d, k, 1))) {
          launch_grid_gram(prm, d_descs, n, int(k[0] * k[2]), st);
          gram_ready = 1;
        }
      }
      launch_grid_solve_mode(prm, d_descs, n, sweep, m, first_done, gram_ready, d_active, st);
      k[m] = leaf_mode_rank(p, d, k, m);
    }
    int left = 0;
    if ((e = cudaMemcpyAsync(&left, d_active + sweep, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    if (timed) {  // converged leaves are skipped: count the leaves this sweep streamed
      const int streamed = sweep == 0 ? n : prev_left;
      float ms1 = 0.f, ms2 = 0.f;
      if (cudaEventElapsedTime(&ms1, pe.ev[0], pe.ev[1]) == cudaSuccess &&
          cudaEventElapsedTime(&ms2, pe.ev[2], pe.ev[3]) == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_pass_mu);
        g_pass_stats[0] += 2.0;
        g_pass_stats[1] += double(ms1) + double(ms2);
        g_pass_stats[2] += 2.0 * 8.0 * double(streamed) * double(len) * double(prod_range(d, 1, p));
      }
    }
    prev_left = left;
    if (left == 0) break;
  }
  return cudaGetLastError();
}

}  // namespace ttb
