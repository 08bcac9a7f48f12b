// Per-leaf solver kernels of the grid-wide leaf path (see tt_grid.cu): one CTA
// per leaf between the streamed passes — the remaining small mode products,
// the llsv solves, the core, the fit and the stop test of tucker_als
// (tucker.cpp:54-119), with the ALS state carried in the leaf's workspace.
#include <mutex>

#include "tt_dev.cuh"

namespace ttb {

// U (rows x R, col-major, ld rows) -> Ut (row-major, row stride rp, zero-padded)
__device__ __forceinline__ void write_ut(const double* U, int64_t rows, int64_t R, double* Ut) {
  const GridChunks ch = grid_chunks(R);
  for (int64_t idx = threadIdx.x; idx < rows * ch.rp; idx += blockDim.x) {
    const int64_t j = idx / ch.rp, a = idx - j * ch.rp;
    Ut[idx] = a < R ? U[j + a * rows] : 0.0;
  }
  __syncthreads();
}

__device__ __forceinline__ void grid_status(const LeafDesc& D, const double* st, int p, const BlockScratch& sc) {
  if (threadIdx.x == 0) {
    D.status[0] = int(st[kGsSweeps]);
    D.status[1] = int(st[kGsConv]);
    D.status[2] = int(st[kGsZero]);
    D.status[3] = 0;
    for (int m = 0; m < kMaxP; ++m) D.status[4 + m] = m < p ? int(st[kGsK + m]) : 0;
    D.status[4 + kMaxP] += sc.eig_calls;
    D.status[5 + kMaxP] += sc.eig_sweeps;
    for (int i = 0; i < 8; ++i) D.status[6 + kMaxP + i] += int(sc.cyc[i] >> 10);
    D.status[14 + kMaxP] += sc.si_ok;
    D.status[15 + kMaxP] += sc.si_fail;
    D.status[16 + kMaxP] += sc.si_iters;
    for (int i = 0; i < 4; ++i) D.status[17 + kMaxP + i] += int(sc.cyc[8 + i] >> 10);
  }
}

__device__ __forceinline__ void grid_scratch_init(BlockScratch& sc) {
  if (threadIdx.x == 0) {
    sc.eig_calls = sc.eig_sweeps = sc.si_ok = sc.si_fail = sc.si_iters = 0;
    sc.dsm_cap = int(dyn_smem_doubles());
    for (int i = 0; i < 12; ++i) sc.cyc[i] = 0;
  }
  __syncthreads();
}

// Init factors, state, status and the first pass's U_1^T (one CTA per leaf).
__global__ void __launch_bounds__(kThreads) grid_prep_kernel(Params prm, const LeafDesc* __restrict__ descs,
                                                             int* __restrict__ active) {
  const LeafDesc D = descs[blockIdx.x];
  const int p = prm.p;
  int64_t d[kMaxP], rc[kMaxP];
  d[0] = D.len;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, rc);
  const GridWs gw = grid_ws_layout(p, D.len, prm.d, prm.req);
  double* st = D.ws + gw.state;
  for (int n = 0; n < p; ++n) bcopy(D.out_f[n], D.init[n], d[n] * rc[n]);
  if (threadIdx.x < kGsSize) st[threadIdx.x] = threadIdx.x >= kGsK && threadIdx.x < kGsK + p ? double(rc[threadIdx.x - kGsK]) : 0.0;
  if (threadIdx.x < kStatusInts) D.status[threadIdx.x] = 0;
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < prm.max_iters; i += blockDim.x) active[i] = 0;
  write_ut(D.init[1], d[1], rc[1], D.ws + gw.ut1);
}

// After pass 1: the remaining contractions of Y, then U_0 = llsv(M_0(Y)).
__global__ void __launch_bounds__(kThreads, 2) grid_solve0_kernel(Params prm, const LeafDesc* __restrict__ descs,
                                                                  int sweep, int gcap, int tt1, int y_done) {
  __shared__ BlockScratch sc;
  extern __shared__ __align__(128) double dsm[];
  const LeafDesc D = descs[blockIdx.x];
  const int p = prm.p;
  const LeafWs lay = leaf_ws_layout(p, D.len, prm.d, prm.req);
  const GridWs gw = grid_ws_layout(p, D.len, prm.d, prm.req);
  double* st = D.ws + gw.state;
  if (st[kGsDone] != 0.0) return;
  grid_scratch_init(sc);
  int64_t d[kMaxP], rc[kMaxP], k[kMaxP];
  d[0] = D.len;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, rc);
  for (int m = 0; m < p; ++m) k[m] = int64_t(st[kGsK + m]);
  double* B[2] = {D.ws + lay.B1, D.ws + lay.B2};
  if (sweep == 0) {
    const GridTile t1 = grid_tile(D.len, prm.d[1], prod_range(prm.d, 2, p), gcap, tt1);
    double s = 0.0;
    if (threadIdx.x == 0)
      for (int64_t i = 0; i < t1.ngrp * t1.ntt; ++i) s += D.ws[gw.npart + i];
    if (threadIdx.x == 0) sc.bcast[1] = s;
    __syncthreads();
    const double norm_sq = sc.bcast[1];
    if (norm_sq == 0.0) {  // tucker.cpp:96-100: init factors, zero core
      bzero(D.out_core, prod_range(rc, 0, p));
      if (threadIdx.x == 0) {
        st[kGsNorm] = 0.0;
        st[kGsDone] = 1.0;
        st[kGsConv] = 1.0;
        st[kGsZero] = 1.0;
      }
      __syncthreads();
      grid_status(D, st, p, sc);
      return;
    }
    if (threadIdx.x == 0) st[kGsNorm] = norm_sq;
  }
  const int64_t k0n = leaf_mode_rank(p, d, k, 0);
  int64_t cur[kMaxP];
  for (int m = 0; m < p; ++m) cur[m] = d[m];
  cur[1] = k[1];
  const double* src = B[0];
  int tog = 1;
  for (int m = 2; m < p; ++m) {
    double* dst = B[tog];
    if (!(m == 2 && y_done))  // order 3: Y x_2 U_2^T came from grid_last_kernel (tt_grid.cu)
      mode_product(src, prod_range(cur, 0, m), cur[m], prod_range(cur, m + 1, p), D.out_f[m], d[m], 1, k[m], dst, false,
                   sc);
    cur[m] = k[m];
    src = dst;
    tog ^= 1;
  }
  llsv_unfold(src, 1, d[0], prod_range(cur, 1, p), k0n, D.out_f[0], D.ws + lay.G, D.ws + lay.V, D.ws + lay.misc, dsm, sc,
              k[0], D.ws + lay.SI);
  write_ut(D.out_f[0], d[0], k0n, D.ws + gw.ut0);
  if (threadIdx.x == 0) st[kGsK] = double(k0n);
  __syncthreads();
  grid_status(D, st, p, sc);
}

// Partial Grams A^T A of the dense mode-1 unfolding (D_1 x cols, row-major in B1,
// written by grid_last_kernel) over kGridGramCtas row chunks per leaf:
// blockIdx.x = chunk, blockIdx.y = leaf. grid_solve_mode_kernel sums the
// partials in chunk order (bit-identical across runs) and goes straight to the
// eigensolver (the cluster kernel's wide_llsv, spread over the grid).
__global__ void __launch_bounds__(kThreads, 2) grid_gram_kernel(Params prm, const LeafDesc* __restrict__ descs,
                                                                int cols) {
  extern __shared__ __align__(128) double dsm[];
  const LeafDesc D = descs[blockIdx.y];
  const int p = prm.p;
  const LeafWs lay = leaf_ws_layout(p, D.len, prm.d, prm.req);
  const GridWs gw = grid_ws_layout(p, D.len, prm.d, prm.req);
  if (D.ws[gw.state + kGsDone] != 0.0) return;
  const int64_t rows = prm.d[1], per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t x0 = imin(rows, int64_t(blockIdx.x) * per), x1 = imin(rows, x0 + per);
  const double* A = D.ws + lay.B1;
  double* Gp = D.ws + gw.gpart + int64_t(blockIdx.x) * cols * cols;
  if (x1 <= x0) {
    for (int64_t idx = threadIdx.x; idx < int64_t(cols) * cols; idx += blockDim.x) Gp[idx] = 0.0;
    return;
  }
  gram_tiled(cols, x1 - x0, [&](int64_t i, int a) { return A[(x0 + i) * cols + a]; }, false, Gp, dsm,
             int(dyn_smem_doubles()));
}

// After pass 2, once per mode n >= 1: the contraction chain W x_{m != 0,n} U_m^T
// (its first, W-sized product already in B1 when `first_done`: computed
// grid-wide by tt_grid.cu), then U_n = llsv. The last mode's call also forms
// the core, the fit and the stop test (tucker.cpp:67-76, 104-116).
__global__ void __launch_bounds__(kThreads, 2) grid_solve_mode_kernel(Params prm, const LeafDesc* __restrict__ descs,
                                                                      int sweep, int n, int first_done,
                                                                      int gram_ready, int* __restrict__ active) {
  __shared__ BlockScratch sc;
  extern __shared__ __align__(128) double dsm[];
  const LeafDesc D = descs[blockIdx.x];
  const int p = prm.p;
  const LeafWs lay = leaf_ws_layout(p, D.len, prm.d, prm.req);
  const GridWs gw = grid_ws_layout(p, D.len, prm.d, prm.req);
  double* st = D.ws + gw.state;
  if (st[kGsDone] != 0.0) return;
  grid_scratch_init(sc);
  int64_t d[kMaxP], k[kMaxP];
  d[0] = D.len;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  for (int m = 0; m < p; ++m) k[m] = int64_t(st[kGsK + m]);
  const double* W = D.ws + lay.W;
  double* B[2] = {D.ws + lay.B1, D.ws + lay.B2};
  int64_t pc[kMaxP];
  const int64_t kn = leaf_mode_rank(p, d, k, n);
  pc[0] = k[0];
  for (int m = 1; m < p; ++m) pc[m] = d[m];
  const double* s2 = W;
  int t2 = 0;
  bool first = true;
  for (int m = 1; m < p; ++m) {
    if (m == n) continue;
    double* dst = B[t2];
    if (!(first && first_done))
      mode_product(s2, prod_range(pc, 0, m), pc[m], prod_range(pc, m + 1, p), D.out_f[m], d[m], 1, k[m], dst, false, sc);
    first = false;
    pc[m] = k[m];
    s2 = dst;
    t2 ^= 1;
  }
  if (first_done && n == 1 && p == 3) {  // grid_last_kernel wrote the unfolding as a dense D_1 x (k0*k2) matrix
    const int64_t cols = pc[0] * pc[2];
    if (gram_ready) {  // grid_gram_kernel's partials, summed in chunk order
      double* G = D.ws + lay.G;
      const double* gp = D.ws + gw.gpart;
      for (int64_t idx = threadIdx.x; idx < cols * cols; idx += blockDim.x) {
        double v = 0.0;
        for (int r = 0; r < int(kGridGramCtas); ++r) v += gp[int64_t(r) * cols * cols + idx];
        G[idx] = v;
      }
      __syncthreads();
    }
    llsv_unfold(s2, 1, d[1], cols, kn, D.out_f[1], D.ws + lay.G, D.ws + lay.V, D.ws + lay.misc, dsm, sc, k[1],
                D.ws + lay.SI, gram_ready != 0);
  } else
    llsv_unfold(s2, prod_range(pc, 0, n), d[n], prod_range(pc, n + 1, p), kn, D.out_f[n], D.ws + lay.G, D.ws + lay.V,
                D.ws + lay.misc, dsm, sc, k[n], D.ws + lay.SI);
  k[n] = kn;
  if (n == 1) write_ut(D.out_f[1], d[1], k[1], D.ws + gw.ut1);
  if (threadIdx.x == 0) st[kGsK + n] = double(kn);
  if (n == p - 1) {
    const double norm_sq = st[kGsNorm], prev_fit = st[kGsPrevFit];
    // core = P_{p-1} x_{p-1} U_{p-1}^T (== core_of(x, U), tucker.cpp:67-76)
    mode_product(s2, prod_range(k, 0, p - 1), d[p - 1], 1, D.out_f[p - 1], d[p - 1], 1, k[p - 1], D.out_core, false, sc);
    const double core_sq = bsumsq(D.out_core, prod_range(k, 0, p), sc);
    const double res = fmax(0.0, norm_sq - core_sq);
    const double fit = 1.0 - sqrt(res) / sqrt(norm_sq);
    const bool stop = sweep > 0 && fabs(fit - prev_fit) < prm.tol;
    if (threadIdx.x == 0) {
      D.objective[sweep] = res;
      st[kGsSweeps] = double(sweep + 1);
      if (stop) {
        st[kGsConv] = 1.0;
        st[kGsDone] = 1.0;
      } else {
        st[kGsPrevFit] = fit;
        atomicAdd(active + sweep, 1);
      }
    }
  }
  __syncthreads();
  grid_status(D, st, p, sc);
}

// ---------------------------------------------------------------------------
// Dynamic shared memory of the solver kernels: batches of up to four leaves per
// SM get most of the SM and run in waves of one CTA per SM (the eigensolvers
// keep a 100 x 100 Gram and its iterates in shared memory, as in the cluster
// kernel: a staged solve is ~3x faster than two unstaged ones sharing an SM);
// wider batches run two CTAs per SM with the one-CTA leaf kernel's budget.
constexpr size_t kGridSolveSmemBig = size_t(176) * 1024;
static size_t grid_solve_smem(int n) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return n <= 4 * nsm ? kGridSolveSmemBig : kLeafDynSmem;
}

cudaError_t grid_solve_prepare() {
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done >> (dev & 63) & 1) return cudaSuccess;
  e = cudaFuncSetAttribute(grid_solve0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGridSolveSmemBig));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(grid_solve_mode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGridSolveSmemBig));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(grid_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLeafDynSmem));
  if (e != cudaSuccess) return e;
  done |= uint64_t(1) << (dev & 63);
  return cudaSuccess;
}
void launch_grid_prep(const Params& prm, const LeafDesc* d_descs, int n, int* d_active, cudaStream_t st) {
  grid_prep_kernel<<<n, kThreads, 0, st>>>(prm, d_descs, d_active);
  g_launches.fetch_add(1);
}
void launch_grid_solve0(const Params& prm, const LeafDesc* d_descs, int n, int sweep, int gcap, int tt1, int y_done,
                        cudaStream_t st) {
  grid_solve0_kernel<<<n, kThreads, grid_solve_smem(n), st>>>(prm, d_descs, sweep, gcap, tt1, y_done);
  g_launches.fetch_add(1);
}
void launch_grid_solve_mode(const Params& prm, const LeafDesc* d_descs, int n, int sweep, int mode, int first_done,
                            int gram_ready, int* d_active, cudaStream_t st) {
  grid_solve_mode_kernel<<<n, kThreads, grid_solve_smem(n), st>>>(prm, d_descs, sweep, mode, first_done, gram_ready,
                                                                 d_active);
  g_launches.fetch_add(1);
}
// Whether the mode-1 Gram of a dense rows x cols unfolding (k columns wanted) is
// formed grid-wide: exactly when llsv_unfold would take its tiled-Gram route
// (tall, no tall subspace iteration: see llsv_uses_subspace).
bool grid_gram_applies(int64_t rows, int64_t cols, int64_t k) {
  const bool tall_si = cols >= 2 * k && cols * k <= kSiMaxYK && k <= kSiMaxK;
  return rows > cols && !tall_si && cols >= kGramTiledMinN && cols * 4 <= int64_t(kLeafDynSmem / sizeof(double));
}
void launch_grid_gram(const Params& prm, const LeafDesc* d_descs, int n, int cols, cudaStream_t st) {
  grid_gram_kernel<<<dim3(unsigned(kGridGramCtas), unsigned(n)), kThreads, kLeafDynSmem, st>>>(prm, d_descs, cols);
  g_launches.fetch_add(1);
}

}  // namespace ttb
