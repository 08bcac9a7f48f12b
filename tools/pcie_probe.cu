// D2H bandwidth: DMA copy engine (cudaMemcpyAsync, pinned) vs SM stores into
// UVA-mapped pinned host memory. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pcie_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void store_kernel(const double* __restrict__ src, double* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) dst[i] = src[i];
}
int main() {
  const size_t bytes = size_t(1393) << 20, n = bytes / 8;
  double *d, *h, *hd;
  cudaMalloc(&d, bytes);
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaMemset(d, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("DMA D2H  %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(a);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("DMA H2D  %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(a);
    store_kernel<<<148 * 8, 256>>>(d, hd, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("SM stores to mapped host %.1f GB/s (%s)\n", bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    // 1 MB copies (one per query-sized U0)
    cudaEventRecord(a);
    for (size_t off = 0; off < bytes; off += (size_t(1) << 20)) cudaMemcpyAsync((char*)h + off, (char*)d + off, size_t(1) << 20, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("DMA D2H in 1 MB copies %.1f GB/s\n", bytes / ms / 1e6);
  }
  return 0;
}
