// stitch_wide_kernel — the stitch of one problem per thread-block cluster
// (body in tt_stitch_body.cuh): the launch path of small stitch batches
// (streamed appends' stitch chains, single range queries).
#include <mutex>

#include "tt_stitch_body.cuh"

namespace ttb {

// One problem per thread-block cluster (small batches: streamed appends and
// single queries), one CTA per SM with 200 KB of dynamic shared memory.
__global__ void __launch_bounds__(kStitchThreads, 1)
    stitch_wide_kernel(Params prm, const StitchDesc* __restrict__ descs, const StitchPart* __restrict__ parts_all) {
  stitch_body<true>(prm, descs, parts_all, int(cl_id()), int(cl_rank()), int(cl_size()));
}


// Cluster size for stitch_wide_kernel on the current device (16 when such a
// cluster fits, else 8; 0 when neither does).
int stitch_wide_cluster() {
  static std::mutex mu;
  static int cs[64];
  static uint64_t done = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(mu);
  if (done >> (dev & 63) & 1) return cs[dev & 63];
  int best = 0;
  if (ensure_dyn_smem(reinterpret_cast<const void*>(stitch_wide_kernel), 3, kDynSmemSolo) == cudaSuccess) {
    cudaFuncSetAttribute(stitch_wide_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {16, 8}) {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kStitchThreads);
      cfg.dynamicSmemBytes = kDynSmemSolo;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, stitch_wide_kernel, &cfg) == cudaSuccess && ncl > 0) {
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

cudaError_t launch_stitch_wide(const Params& prm, const StitchDesc* d_descs, const StitchPart* d_parts, int n, int cs,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(unsigned(n * cs));
  cfg.blockDim = dim3(kStitchThreads);
  cfg.dynamicSmemBytes = kDynSmemSolo;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, stitch_wide_kernel, prm, d_descs, d_parts);
  g_launches.fetch_add(1);
  return e;
}

}  // namespace ttb
