// leaf_als_kernel — tucker_als on one leaf block (tucker.cpp:86-119), one CTA
// per leaf; X is streamed from HBM twice per sweep through a TMA ring
// (Y = X x_{m>=1} U_m^T for the mode-0 update, W = X x_0 U_0^T reused by every
// other mode and the core).
#include "tt_dev.cuh"

namespace ttb {

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2) leaf_als_kernel(Params prm, const LeafDesc* __restrict__ descs) {
  __shared__ BlockScratch sc;
  __shared__ Pipe pipe;
  extern __shared__ __align__(128) double dsm[];
  const long long t_kernel = tstart();
  if (threadIdx.x == 0) {
    sc.eig_calls = sc.eig_sweeps = sc.si_ok = sc.si_fail = sc.si_iters = 0;
    sc.dsm_cap = int(dyn_smem_doubles());
    for (int i = 0; i < 12; ++i) sc.cyc[i] = 0;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&pipe.full[i], 1);
      pipe.uses[i] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  const LeafDesc D = descs[blockIdx.x];
  const int p = prm.p;
  int64_t d[kMaxP], rc[kMaxP], k[kMaxP];
  d[0] = D.len;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, rc);
  const LeafWs lay = leaf_ws_layout(p, D.len, prm.d, prm.req);
  double* W = D.ws + lay.W;
  double* B[2] = {D.ws + lay.B1, D.ws + lay.B2};
  double* G = D.ws + lay.G;
  double* V = D.ws + lay.V;
  double* misc = D.ws + lay.misc;
  const double* X = D.x;
  const int64_t ns = prod_range(d, 1, p);
  for (int n = 0; n < p; ++n) {
    bcopy(D.out_f[n], D.init[n], d[n] * rc[n]);
    k[n] = rc[n];
  }
  int sweeps = 0, converged = 0;
  double norm_sq = 0.0, norm = 0.0;
  double prev_fit = nan("");
  for (int sweep = 0; sweep < prm.max_iters; ++sweep) {
    // ---- mode 0: Y = X x_1 U_1^T ... x_{p-1} U_{p-1}^T, U_0 = llsv(M_0(Y))
    const int64_t k0n = leaf_mode_rank(p, d, k, 0);
    int64_t cur[kMaxP];
    for (int m = 0; m < p; ++m) cur[m] = d[m];
    const double* src = X;
    int tog = 0;
    for (int m = 1; m < p; ++m) {
      double* dst = B[tog];
      const int64_t inner = prod_range(cur, m + 1, p);
      if (m == 1 && stream_ok(X, inner, int(k[1]))) {
        // first contraction streams X through the TMA ring; sweep 0 also
        // accumulates ||X||^2 (tucker.cpp:96)
        const long long tb = tstart();
        double nacc = 0.0;
        ttm_stream(X, d[0], d[1], inner, D.out_f[1], int(k[1]), dst, dsm, pipe, sweep == 0 ? &nacc : nullptr,
                   D.tmaps, 3);
        if (sweep == 0) norm_sq = block_sum(nacc, sc);
        tstop(sc, kPhBig, tb);
      } else {
        if (m == 1 && sweep == 0) norm_sq = bsumsq(X, D.len * ns, sc);
        mode_product(src, prod_range(cur, 0, m), cur[m], inner, D.out_f[m], d[m], 1, k[m], dst, false, sc,
                     m == 1 ? kPhBig : kPhTtm);
      }
      cur[m] = k[m];
      src = dst;
      tog ^= 1;
    }
    if (sweep == 0) {
      if (norm_sq == 0.0) {  // tucker.cpp:96-100: init factors, zero core
        bzero(D.out_core, prod_range(rc, 0, p));
        converged = 1;
        break;
      }
      norm = sqrt(norm_sq);
    }
    llsv_unfold(src, 1, d[0], prod_range(cur, 1, p), k0n, D.out_f[0], G, V, misc, dsm, sc, k[0], D.ws + lay.SI);
    k[0] = k0n;
    // ---- W = X x_0 U_0^T : (k0, D_1, ..., D_{p-1})
    if (stream_ok(X, ns, int(k[0]))) {
      const long long tb = tstart();
      ttm_stream(X, 1, d[0], ns, D.out_f[0], int(k[0]), W, dsm, pipe, nullptr,
                 D.tmaps ? static_cast<const char*>(D.tmaps) + 128 : nullptr, 2);
      tstop(sc, kPhBig, tb);
    } else {
      mode_product(X, 1, d[0], ns, D.out_f[0], d[0], 1, k[0], W, false, sc, kPhBig);
    }
    // ---- modes n >= 1 from W
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
        mode_product(s2, prod_range(pc, 0, m), pc[m], prod_range(pc, m + 1, p), D.out_f[m], d[m], 1, k[m], dst,
                     false, sc);
        pc[m] = k[m];
        s2 = dst;
        t2 ^= 1;
      }
      llsv_unfold(s2, prod_range(pc, 0, n), d[n], prod_range(pc, n + 1, p), kn, D.out_f[n], G, V, misc, dsm, sc,
                  k[n], D.ws + lay.SI);
      k[n] = kn;
      Pn = s2;
    }
    // ---- core = P_{p-1} x_{p-1} U_{p-1}^T  (== core_of(x, U), tucker.cpp:67-76)
    mode_product(Pn, prod_range(k, 0, p - 1), d[p - 1], 1, D.out_f[p - 1], d[p - 1], 1, k[p - 1], D.out_core,
                 false, sc);
    const double core_sq = bsumsq(D.out_core, prod_range(k, 0, p), sc);
    const double res = fmax(0.0, norm_sq - core_sq);
    if (threadIdx.x == 0) D.objective[sweep] = res;
    sweeps = sweep + 1;
    const double fit = 1.0 - sqrt(res) / norm;
    if (sweep > 0 && fabs(fit - prev_fit) < prm.tol) {
      converged = 1;
      break;
    }
    prev_fit = fit;
  }
  if (threadIdx.x == 0) {
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
}

cudaError_t launch_leaf(const Params& prm, const LeafDesc* d_descs, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const cudaError_t ae = ensure_dyn_smem(reinterpret_cast<const void*>(leaf_als_kernel), 0, kLeafDynSmem);
  if (ae != cudaSuccess) return ae;
  leaf_als_kernel<<<n, kThreads, kLeafDynSmem, st>>>(prm, d_descs);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace ttb
