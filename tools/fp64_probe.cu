// B200 FP64 micro-probe: dependent-chain latencies (DFMA, DMUL, div, sqrt,
// rsqrt, LDS.64, SHFL) and the DFMA throughput peak of the chip, measured with
// clock64 / CUDA events. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, double x0, int iters) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x * 0.5 + 1.0;
  __syncthreads();
  double a = x0, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) a = a * b;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) a = 1.0 / (a + 1.0);
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) a = sqrt(a + 2.0);
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) a = rsqrt(a + 2.0);
  long long t5 = clock64();
  int idx = 1;
  for (int i = 0; i < iters; ++i) idx = int(sm[idx & 63]) & 63;
  long long t6 = clock64();
  double sv = a;
  for (int i = 0; i < iters; ++i) sv = __shfl_sync(0xffffffffu, sv, (threadIdx.x + 1) & 31);
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    out[0] = a + idx + sv;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    cyc[6] = t7 - t6;
  }
}

__global__ void __launch_bounds__(256) tput_kernel(double* out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;
}

// FP64 tensor-core (DMMA) throughput: mma.sync.aligned.m8n8k4 f64, 8
// independent accumulator fragments per warp (2 flops x 8x8x4 per mma).
__global__ void __launch_bounds__(256) dmma_kernel(double* out, int iters) {
  double acc[8][2];
  for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = threadIdx.x * 1e-3 + k;
  const double a = 0.999999 + threadIdx.x * 1e-9, b = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 64 * sizeof(long long));
  const int it = 4096;
  lat_kernel<<<1, 32>>>(d, c, 0.5, it);
  lat_kernel<<<1, 32>>>(d, c, 0.5, it);
  long long h[8];
  cudaMemcpy(h, c, 7 * sizeof(long long), cudaMemcpyDeviceToHost);
  const char* names[7] = {"DFMA", "DMUL", "div", "sqrt", "rsqrt", "LDS.64+cvt", "SHFL(f64)"};
  for (int i = 0; i < 7; ++i) printf("latency %-10s %.1f cycles\n", names[i], double(h[i]) / it);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = nsm * 8;
  tput_kernel<<<blocks, 256>>>(d, 100);
  cudaEventRecord(e0);
  tput_kernel<<<blocks, 256>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * iters * double(blocks) * 256;
  printf("DFMA throughput %.2f TFLOP/s (%d SMs, %.3f ms)\n", flops / ms / 1e9, nsm, ms);
  {
    const int dit = 4096;
    dmma_kernel<<<nsm * 8, 256>>>(d, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dmma_kernel<<<nsm * 8, 256>>>(d, dit);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = double(nsm) * 8 * (256 / 32) * dit * 8 * (2.0 * 8 * 8 * 4);
    printf("DMMA (mma.sync m8n8k4 f64) throughput %.2f TFLOP/s (%d SMs, %.3f ms)\n", flops / (ms * 1e-3) / 1e12, nsm, ms);
  }
  return 0;
}
