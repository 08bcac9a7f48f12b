// stitch_als_kernel — stitch() (stitch.cpp:110-184) for appends (2 parts) and
// range queries (s parts), one CTA per problem, entirely in compressed
// r-sized coordinates: the L-row temporal unfolding is never formed
// (SURVEY.md A.2); partial hits enter through the Gram S = Vsub^T Vsub of
// their kept temporal rows instead of a QR.
#include <mutex>

#include "tt_stitch_body.cuh"

namespace ttb {

__global__ void __launch_bounds__(kStitchThreads, kStitchCtas)
    stitch_als_kernel(Params prm, const StitchDesc* __restrict__ descs, const StitchPart* __restrict__ parts_all) {
  stitch_body<false>(prm, descs, parts_all, int(blockIdx.x), 0, 1);
}

// Gathers small device-staged outputs (cores, non-temporal factors) into the
// caller's pinned, UVA-mapped host buffers in one launch (one CTA per segment).
__global__ void __launch_bounds__(256) copy_segments_kernel(const CopySeg* __restrict__ segs, int n) {
  const CopySeg sg = segs[blockIdx.x];
  for (int64_t i = threadIdx.x; i < sg.n; i += blockDim.x) sg.dst[i] = sg.src[i];
}

std::atomic<int64_t> g_launches{0};

cudaError_t ensure_dyn_smem(const void* fn, int slot, size_t bytes) {
  static std::mutex mu;
  static uint64_t done[8] = {};  // bit d of done[slot]: set on device d
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (done[slot] & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e == cudaSuccess) done[slot] |= bit;
  return e;
}

// ---------------------------------------------------------------------------
// partial_hit_factors (stitch.cpp:36-47) for the standalone API: thin
// Householder QR of the kept temporal rows V0[b:e, :] (len x n, n <= 32), in
// the LAPACK dgeqr2 / dorg2r convention, the reference's sign rule on Q's
// columns (linalg.cpp:15-31, R's rows follow), and core <- core x_0 R. One CTA;
// W (len x n) is the in-place factorisation, Q is len x k (k = min(len, n)).
// Range queries never call this: they fold partial hits into the stitch
// through the metric S = V_sub^T V_sub.
__global__ void __launch_bounds__(256) partial_hit_kernel(const double* __restrict__ V0, int64_t ld, int64_t b,
                                                          int64_t len, int n, const double* __restrict__ core,
                                                          int64_t rest, double* W, double* Q, double* R,
                                                          double* out_core, double* tau) {
  __shared__ BlockScratch sc;
  __shared__ int flips[kMaxVec];
  const int k = int(imin(len, n));
  for (int64_t idx = threadIdx.x; idx < len * n; idx += blockDim.x) {
    const int64_t i = idx % len, c = idx / len;
    W[idx] = V0[b + i + c * ld];
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    double* wj = W + int64_t(j) * len;
    double xs = 0.0;
    for (int64_t i = j + 1 + threadIdx.x; i < len; i += blockDim.x) xs = fma(wj[i], wj[i], xs);
    const double xnorm2 = block_sum(xs, sc);
    const double alpha = wj[j];
    double t = 0.0, beta = alpha;
    if (xnorm2 > 0.0) {  // dlarfg
      beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
      t = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int64_t i = j + 1 + threadIdx.x; i < len; i += blockDim.x) wj[i] *= scal;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      wj[j] = beta;
      tau[j] = t;
    }
    __syncthreads();
    // H_j = I - t v v^T (v = [1; W[j+1:, j]]) on the trailing columns
    if (t != 0.0 && j + 1 < n) {
      double part[kMaxVec];
#pragma unroll
      for (int c = 0; c < kMaxVec; ++c) part[c] = 0.0;
      for (int64_t i = j + threadIdx.x; i < len; i += blockDim.x) {
        const double v = i == j ? 1.0 : wj[i];
#pragma unroll
        for (int c = 0; c < kMaxVec; ++c)
          if (j + 1 + c < n) part[c] = fma(v, W[i + int64_t(j + 1 + c) * len], part[c]);
      }
      block_sum_vec<kMaxVec>(part, n - j - 1, sc);
      for (int64_t idx = threadIdx.x; idx < (len - j) * (n - j - 1); idx += blockDim.x) {
        const int64_t i = j + idx % (len - j), c = j + 1 + idx / (len - j);
        const double v = i == j ? 1.0 : wj[i];
        W[i + c * len] -= t * v * sc.vec[c - j - 1];
      }
      __syncthreads();
    }
  }
  // R = triu(W[0:k, :]) (k x n, ld k)
  for (int idx = threadIdx.x; idx < k * n; idx += blockDim.x) {
    const int a = idx % k, c = idx / k;
    R[idx] = a <= c ? W[a + int64_t(c) * len] : 0.0;
  }
  // Q = H_0 ... H_{k-1} [I_k; 0] (dorg2r order: reflectors applied backwards)
  for (int64_t idx = threadIdx.x; idx < len * k; idx += blockDim.x) {
    const int64_t i = idx % len, c = idx / len;
    Q[idx] = i == c ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    const double* wj = W + int64_t(j) * len;
    double part[kMaxVec];
#pragma unroll
    for (int c = 0; c < kMaxVec; ++c) part[c] = 0.0;
    for (int64_t i = j + threadIdx.x; i < len; i += blockDim.x) {
      const double v = i == j ? 1.0 : wj[i];
#pragma unroll
      for (int c = 0; c < kMaxVec; ++c)
        if (j + c < k) part[c] = fma(v, Q[i + int64_t(j + c) * len], part[c]);
    }
    block_sum_vec<kMaxVec>(part, k - j, sc);
    for (int64_t idx = threadIdx.x; idx < (len - j) * (k - j); idx += blockDim.x) {
      const int64_t i = j + idx % (len - j), c = j + idx / (len - j);
      const double v = i == j ? 1.0 : wj[i];
      Q[i + c * len] -= t * v * sc.vec[c - j];
    }
    __syncthreads();
  }
  // sign rule on Q's columns; R's rows follow (linalg.cpp:15-31)
  sign_fix(Q, len, k, len, flips, sc);
  for (int idx = threadIdx.x; idx < k * n; idx += blockDim.x)
    if (flips[idx % k]) R[idx] = -R[idx];
  __syncthreads();
  // core <- core x_0 R : (k x rest) = R (k x n) * core (n x rest, row-major)
  for (int64_t idx = threadIdx.x; idx < int64_t(k) * rest; idx += blockDim.x) {
    const int64_t a = idx / rest, tt = idx - a * rest;
    double v = 0.0;
    for (int c = 0; c < n; ++c) v = fma(R[a + int64_t(c) * k], core[int64_t(c) * rest + tt], v);
    out_core[idx] = v;
  }
}

cudaError_t launch_partial_hit(const double* V0, int64_t ld, int64_t b, int64_t len, int n, const double* core,
                               int64_t rest, double* W, double* Q, double* R, double* out_core, double* tau,
                               cudaStream_t st) {
  partial_hit_kernel<<<1, 256, 0, st>>>(V0, ld, b, len, n, core, rest, W, Q, R, out_core, tau);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}



cudaError_t launch_copy_segments(const CopySeg* d_segs, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  copy_segments_kernel<<<n, 256, 0, st>>>(d_segs, n);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_stitch(const Params& prm, const StitchDesc* d_descs, const StitchPart* d_parts, int n,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  // Batches that leave most SMs idle (streamed appends, single queries) run one
  // CTA per SM with 200 KB of dynamic shared memory: the solvers then keep
  // their 100 x 100 Grams and iteration state on chip (sc.dsm_cap adapts).
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t dyn = n <= nsm ? kDynSmemSolo : kDynSmem;
  const cudaError_t ae = ensure_dyn_smem(reinterpret_cast<const void*>(stitch_als_kernel), 1, kDynSmemSolo);
  if (ae != cudaSuccess) return ae;
  stitch_als_kernel<<<n, kStitchThreads, dyn, st>>>(prm, d_descs, d_parts);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

int64_t launches() { return g_launches.load(); }

}  // namespace ttb
