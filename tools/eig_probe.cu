// Isolated timing of the block Jacobi eigensolvers on random SPD Gram
// matrices (n x n), one CTA per matrix: cycles per call, sweeps, and the
// residual max |A v - lambda v| / ||A|| against the input.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2501_06647_b200/csrc tools/eig_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#include "tt_block.cuh"

using namespace ttb;

__global__ void __launch_bounds__(256, 2) probe(const double* G, int n, int which, long long* cyc, int* sweeps,
                                                double* evals, double* evecs) {
  __shared__ BlockScratch sc;
  extern __shared__ double dsm[];
  __shared__ int order[64];
  const double* g = G + size_t(blockIdx.x) * n * n;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) dsm[i] = g[i];
  __syncthreads();
  long long t0 = clock64();
  int sw;
  double* V;
  if (which == 0) {
    sw = sym_eig_smem(dsm, n, order, sc);
    V = dsm + 2 * n * n;
  } else {
    sw = sym_eig(dsm, n, dsm + n * n, order, sc);
    V = dsm + n * n;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    sweeps[blockIdx.x] = sw;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) evals[blockIdx.x * n + i] = dsm[order[i] * (n + 1)];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int r = i % n, c = i / n;
    evecs[size_t(blockIdx.x) * n * n + i] = V[r + order[c] * n];
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 40;
  const int nb = 148;
  std::vector<double> h(size_t(nb) * n * n);
  srand(1);
  for (int b = 0; b < nb; ++b) {
    // G = Y^T Y with Y (3n x n) having a decaying spectrum (signal + noise)
    std::vector<double> y(3 * n * n);
    for (int i = 0; i < 3 * n; ++i)
      for (int j = 0; j < n; ++j)
        y[i * n + j] = ((rand() / double(RAND_MAX)) - 0.5) * (j < 10 ? 10.0 / (j + 1) : 0.05);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0;
        for (int k = 0; k < 3 * n; ++k) s += y[k * n + i] * y[k * n + j];
        h[size_t(b) * n * n + i + j * n] = s;
      }
  }
  double *dG, *dE, *dV;
  long long* dc;
  int* ds;
  cudaMalloc(&dG, h.size() * 8);
  cudaMalloc(&dE, nb * n * 8);
  cudaMalloc(&dV, h.size() * 8);
  cudaMalloc(&dc, nb * 8);
  cudaMalloc(&ds, nb * 4);
  cudaMemcpy(dG, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = 3 * n * n * 8;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int which = 0; which < 2; ++which) {
    if (which == 0 && n > kFastEigN) continue;
    probe<<<nb, 256, smem>>>(dG, n, which, dc, ds, dE, dV);
    probe<<<nb, 256, smem>>>(dG, n, which, dc, ds, dE, dV);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<long long> c(nb);
    std::vector<int> s(nb);
    std::vector<double> ev(nb * n), vv(h.size());
    cudaMemcpy(c.data(), dc, nb * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(s.data(), ds, nb * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ev.data(), dE, nb * n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(vv.data(), dV, h.size() * 8, cudaMemcpyDeviceToHost);
    double cs = 0, ss = 0, worst = 0;
    for (int b = 0; b < nb; ++b) {
      cs += c[b];
      ss += s[b];
      const double* G = h.data() + size_t(b) * n * n;
      double nrm = 0;
      for (int i = 0; i < n * n; ++i) nrm += G[i] * G[i];
      nrm = sqrt(nrm);
      for (int k = 0; k < n; ++k)
        for (int i = 0; i < n; ++i) {
          double r = -ev[b * n + k] * vv[size_t(b) * n * n + i + k * n];
          for (int j = 0; j < n; ++j) r += G[i + j * n] * vv[size_t(b) * n * n + j + k * n];
          worst = fmax(worst, fabs(r) / nrm);
        }
    }
    printf("%s n=%d: %.0f cycles/call, %.2f sweeps, %.0f cycles/round, resid %.2e\n",
           which == 0 ? "smem1sync" : "generic  ", n, cs / nb, ss / nb, cs / ss / (n + (n & 1) - 1), worst);
  }
  return 0;
}
