// Device code of the stitch (stitch.cpp:110-184) shared by the one-CTA
// kernel (tt_stitch.cu) and the cluster kernel (tt_stitch_wide.cu): the body
// is a template on the cluster mode, each kernel lives in its own translation
// unit so the two instantiations compile in parallel.
#pragma once
#include "tt_dev.cuh"

namespace ttb {

// ---------------------------------------------------------------------------
// U_0 = blockdiag(V_sub,i) [E_i]  (L x K0, ld L), sign-fixed (linalg.cpp:15-31);
// E_i = rows [roff[i], roff[i+1]) of the stacked E (ld R).
// Pass 0 evaluates the rows without storing and finds each column's first
// max-|.| row; pass 1 recomputes and stores U_0 once with the signs applied.
// Two rows per thread are in flight, E_i is staged in shared memory.
template <int K0>
__device__ __noinline__ void materialize_u0_k(const StitchPart* __restrict__ parts, int s, const double* Est,
                                              int R, const int* roff, double* __restrict__ U0, int64_t L, int* flips,
                                              int64_t* idxbuf, double* Es, BlockScratch& sc) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nt = int(blockDim.x);
  for (int pass = 0; pass < 2; ++pass) {
    double best[K0], sg[K0];
    int64_t bidx[K0];
#pragma unroll
    for (int c = 0; c < K0; ++c) {
      best[c] = -1.0;
      bidx[c] = 0;
      sg[c] = (pass == 1 && flips[c]) ? -1.0 : 1.0;
    }
    int64_t off = 0;
    for (int i = 0; i < s; ++i) {
      const int64_t r0 = parts[i].rho[0], len = parts[i].len, ld = parts[i].ld0;
      const double* vs = parts[i].v0 + parts[i].row0;
      const double* E = Est + roff[i];  // stacked E, ld R
      __syncthreads();
      for (int64_t e = threadIdx.x; e < r0 * K0; e += nt) Es[e] = E[(e % r0) + (e / r0) * R];
      __syncthreads();
      for (int64_t rb = threadIdx.x; rb < len; rb += 2 * nt) {
        const int64_t ra = rb, rc = rb + nt;
        const bool has_c = rc < len;
        double oa[K0], ob[K0];
#pragma unroll
        for (int c = 0; c < K0; ++c) oa[c] = ob[c] = 0.0;
        for (int64_t a = 0; a < r0; ++a) {
          const double va = vs[ra + a * ld];
          const double vb = has_c ? vs[rc + a * ld] : 0.0;
#pragma unroll
          for (int c = 0; c < K0; ++c) {
            const double ev = Es[a + c * r0];
            oa[c] = fma(va, ev, oa[c]);
            ob[c] = fma(vb, ev, ob[c]);
          }
        }
        if (pass == 1) {
#pragma unroll
          for (int c = 0; c < K0; ++c) {
            U0[off + ra + c * L] = sg[c] * oa[c];
            if (has_c) U0[off + rc + c * L] = sg[c] * ob[c];
          }
        } else {
#pragma unroll
          for (int c = 0; c < K0; ++c) {
            const double ma = fabs(oa[c]);
            if (ma > best[c]) {
              best[c] = ma;
              bidx[c] = off + ra;
              sg[c] = oa[c];
            }
            const double mb = has_c ? fabs(ob[c]) : -1.0;
            if (mb > best[c]) {  // rc > ra: a tie keeps the earlier row
              best[c] = mb;
              bidx[c] = off + rc;
              sg[c] = ob[c];
            }
          }
        }
      }
      off += len;
    }
    if (pass == 0) {
#pragma unroll
      for (int c = 0; c < K0; ++c) {
        double b = best[c], v = sg[c];
        int64_t bi = bidx[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, b, o);
          const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
          const double ov = __shfl_xor_sync(0xffffffffu, v, o);
          if (ob > b || (ob == b && oi < bi)) {
            b = ob;
            bi = oi;
            v = ov;
          }
        }
        if (l == 0) {
          sc.red[w * kMaxVec + c] = b;
          idxbuf[w * kMaxVec + c] = v < 0.0 ? -(bi + 1) : (bi + 1);
        }
      }
      __syncthreads();
      if (threadIdx.x < K0) {
        const int c = threadIdx.x;
        double b = sc.red[c];
        int64_t bi = idxbuf[c];
        for (int ww = 1; ww < kWarps; ++ww) {
          const double ob = sc.red[ww * kMaxVec + c];
          const int64_t oi = idxbuf[ww * kMaxVec + c];
          const int64_t ai = bi < 0 ? -bi : bi, ao = oi < 0 ? -oi : oi;
          if (ob > b || (ob == b && ao < ai)) {
            b = ob;
            bi = oi;
          }
        }
        flips[c] = bi < 0;
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

static __device__ bool materialize_u0(int k0, const StitchPart* parts, int s, const double* Est, int R, const int* roff,
                               double* U0, int64_t L, int* flips, int64_t* idxbuf, double* Es, BlockScratch& sc) {
  switch (k0) {
#define TT_CASE(N) \
  case N:          \
    materialize_u0_k<N>(parts, s, Est, R, roff, U0, L, flips, idxbuf, Es, sc); \
    return true;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8)
    TT_CASE(9) TT_CASE(10) TT_CASE(11) TT_CASE(12) TT_CASE(13) TT_CASE(14) TT_CASE(15) TT_CASE(16)
#undef TT_CASE
    default:
      return false;
  }
}

// ---------------------------------------------------------------------------
// S = V^T V for a tall V (rows x K, ld) with many rows (a partial hit's kept
// temporal rows: up to tens of thousands): every thread keeps all K(K+1)/2
// upper-triangle sums for its rows (K loads feed K(K+1)/2 FMAs per row, rows
// strided over the block so each load instruction is coalesced), then a warp
// butterfly and a shared-memory pass reduce them. `red` holds kWarps*K(K+1)/2
// doubles.
template <int K>
__device__ __noinline__ void gram_long_k(const double* __restrict__ V, int64_t ld, int64_t rows,
                                         double* __restrict__ G, double* red) {
  constexpr int NP = K * (K + 1) / 2;
  double acc[NP];
#pragma unroll
  for (int e = 0; e < NP; ++e) acc[e] = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    double v[K];
#pragma unroll
    for (int a = 0; a < K; ++a) v[a] = V[r + a * ld];
    int e = 0;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a; b < K; ++b) {
        acc[e] = fma(v[a], v[b], acc[e]);
        ++e;
      }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < NP; ++e) {
    const double s = warp_sum(acc[e]);
    if (l == 0) red[w * NP + e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NP; e += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < int(blockDim.x >> 5); ++q) s += red[q * NP + e];
    int a = 0, rem = e;  // e -> (a, b), upper triangle row-major
    while (rem >= K - a) {
      rem -= K - a;
      ++a;
    }
    const int b = a + rem;
    G[a + b * K] = s;
    G[b + a * K] = s;
  }
  __syncthreads();
}

static __device__ void gram_long(const double* V, int64_t ld, int64_t rows, int k, double* G, double* red) {
  switch (k) {
#define TT_CASE(N)                         \
  case N:                                  \
    gram_long_k<N>(V, ld, rows, G, red);   \
    return;
    TT_CASE(1) TT_CASE(2) TT_CASE(3) TT_CASE(4) TT_CASE(5) TT_CASE(6) TT_CASE(7) TT_CASE(8) TT_CASE(9) TT_CASE(10)
#undef TT_CASE
    default:
      gram_tall(V, ld, rows, k, G);
  }
}

// ---------------------------------------------------------------------------
struct PartView {
  const double* core;
  int64_t rho[kMaxP];
  const double* v0;
  int64_t ld0, row0, len;
  int partial;
  const double* v[kMaxP];
};

__device__ __forceinline__ PartView load_part(const StitchPart& s) {
  PartView v;
  v.core = s.core;
  for (int m = 0; m < kMaxP; ++m) {
    v.rho[m] = s.rho[m];
    v.v[m] = s.v[m];
  }
  v.v0 = s.v0;
  v.ld0 = s.ld0;
  v.row0 = s.row0;
  v.len = s.len;
  v.partial = s.partial;
  return v;
}

// ---------------------------------------------------------------------------
// Part-batched small products. A stitch touches s parts, and most of its work
// is the same tiny product per part (mode products of r-sized cores, U^T V
// projections). Issuing them part by part costs one barrier and one L2 round
// trip per part; a batch flattens the outputs of all parts into one index
// space so one block-wide pass (one barrier) covers every part.
//
// One batch entry: C[o] (M x N) (+)= A[o] (M x K) B[o] (K x N) for o < outer,
// element (i, j) of X[o] at X[o*xos + i*xrs + j*xcs].
struct BGemm {
  const double* A;
  const double* B;
  double* C;
  int M, N, K, outer;
  int ars, acs, aos, brs, bcs, bos, crs, ccs, cos;
  int acc;
};

// A mode product (in: row-major (outer, d, inner); M(a, j) = M[a*ms_a + j*ms_j],
// a < r) as a batch entry.
__device__ __forceinline__ BGemm bg_mode_product(const double* in, int64_t outer, int64_t d, int64_t inner,
                                                 const double* M, int64_t ms_a, int64_t ms_j, int64_t r,
                                                 double* out) {
  BGemm g;
  g.A = M;
  g.B = in;
  g.C = out;
  g.M = int(r);
  g.N = int(inner);
  g.K = int(d);
  g.outer = int(outer);
  g.ars = int(ms_a);
  g.acs = int(ms_j);
  g.aos = 0;
  g.brs = int(inner);
  g.bcs = 1;
  g.bos = int(d * inner);
  g.crs = int(inner);
  g.ccs = 1;
  g.cos = int(r * inner);
  g.acc = 0;
  return g;
}

// Runs entries gen(0..n-1) in one pass; ends with a barrier.
template <class Gen>
__device__ __forceinline__ void gemm_batched(int n, Gen gen, BlockScratch& sc) {
  const long long t0 = tstart();
  if (n > 0) {
    int i = 0;
    BGemm g = gen(0);
    int64_t base = 0, sz = int64_t(g.outer) * g.M * g.N;
    for (int64_t e = threadIdx.x;; e += blockDim.x) {
      while (e >= base + sz) {
        base += sz;
        if (++i >= n) break;
        g = gen(i);
        sz = int64_t(g.outer) * g.M * g.N;
      }
      if (i >= n) break;
      const int64_t l = e - base;
      const int jj = int(l % g.N);
      const int64_t q = l / g.N;
      const int ii = int(q % g.M);
      const int o = int(q / g.M);
      const double* __restrict__ a = g.A + int64_t(o) * g.aos + int64_t(ii) * g.ars;
      const double* __restrict__ b = g.B + int64_t(o) * g.bos + int64_t(jj) * g.bcs;
      const double sum = dot4(a, g.acs, b, g.brs, g.K);
      double* c = g.C + int64_t(o) * g.cos + int64_t(ii) * g.crs + int64_t(jj) * g.ccs;
      *c = g.acc ? *c + sum : sum;
    }
  }
  __syncthreads();
  tstop(sc, kPhTtm, t0);
}

// Stacked temporal rows of all parts (mode-0 coordinates): part i owns rows
// [roff[i], roff[i+1]) of the stacked E / A / C matrices (R = sum rho_i0 rows);
// rt_pp[r] = the part of row r if it is a partial hit (rows carrying the
// metric S_i), else -1. The host rejects stitches with more rows.
constexpr int kRowTab = kStitchMaxRows;
#ifndef TT_ONE_PASS_MIN_PARTS
#define TT_ONE_PASS_MIN_PARTS 2  // one-pass Z_n from two parts up (measured: append stitches 3% faster)
#endif

// The stitch, one problem per CTA (CL = false) or per thread-block cluster
// (CL = true: rank 0 leads and runs every solver; all CTAs form each Z_n by row
// range and its Gram by column/row range — the phases whose shape is
// data-independent — separated by cluster barriers; per-sweep scalars travel
// through the problem's exchange slots).
template <bool CL>
__device__ __forceinline__ void stitch_body(const Params& prm, const StitchDesc* __restrict__ descs,
                                            const StitchPart* __restrict__ parts_all, int prob, int rank, int CS) {
  __shared__ BlockScratch sc;
  __shared__ int flips[kMaxVec];
  __shared__ int64_t idxbuf[kWarps * kMaxVec];
  __shared__ int roff[kRowTab + 1], rt_pp[kRowTab];
  extern __shared__ double dsm[];
  const long long t_kernel = tstart();
  if (threadIdx.x == 0) {
    sc.eig_calls = sc.eig_sweeps = sc.si_ok = sc.si_fail = sc.si_iters = 0;
    sc.dsm_cap = int(dyn_smem_doubles());
    for (int i = 0; i < 12; ++i) sc.cyc[i] = 0;
  }
  const StitchDesc D = descs[prob];
  const StitchPart* parts = parts_all + D.part0;
  const bool leader = rank == 0;
  const int p = prm.p, s = D.nparts;
  int64_t d[kMaxP], rc[kMaxP], k[kMaxP], rho_max[kMaxP], rcx[kMaxP];
  d[0] = D.L;
  for (int m = 1; m < p; ++m) d[m] = prm.d[m];
  clamp_ranks(p, d, prm.req, rc);
  for (int m = 0; m < p; ++m) rho_max[m] = 0;
  for (int i = 0; i < s; ++i)
    for (int m = 0; m < p; ++m) rho_max[m] = imax(rho_max[m], parts[i].rho[m]);
  for (int m = 0; m < p; ++m) rcx[m] = imax(rc[m], rho_max[m]);
  const StitchWs lay = stitch_ws_layout(p, D.L, prm.d, prm.req, rho_max, s, CL ? CS : 0);
  double* ws = D.ws;
  double* xch = ws + lay.xch;      // cluster: [0] ||X||^2, [1] stop flag
  double* gpart = ws + lay.gpart;  // cluster: per-CTA partial Grams
  double* T[2] = {ws + lay.T1, ws + lay.T2};
  double* G = ws + lay.G;
  double* Vg = ws + lay.V;
  double* Z = ws + lay.Z;
  double* misc = ws + lay.misc;
  double* wk = ws + lay.WK;  // Q x k0 scaled eigenvectors
  double* HH = ws + lay.HH;  // rho0 x rho0 scratch
  auto Pm = [&](int i, int m) {  // P_im = U_m^T V_im, k_m x rho_im (ld k_m)
    int64_t off = 0;
    for (int q = 1; q < m; ++q) off += rc[q] * rcx[q];
    return ws + lay.P + int64_t(i) * lay.per_part_P + off;
  };

  auto Sp = [&](int i) { return ws + lay.S + int64_t(i) * lay.per_part_S; };
  double* TB[2] = {ws + lay.TB1, ws + lay.TB2};  // part-batched chain scratch, stride lay.chain
  // stacked temporal rows: part i owns rows [roff[i], roff[i+1])
  int R = 0;
  bool any_partial = false;
  for (int i = 0; i < s; ++i) {
    R += int(parts[i].rho[0]);
    any_partial = any_partial || parts[i].partial;
  }
  if (threadIdx.x == 0) {
    int o = 0;
    for (int i = 0; i < s; ++i) {
      roff[i] = o;
      o += int(parts[i].rho[0]);
    }
    roff[s] = o;
  }
  __syncthreads();
  for (int i = 0; i < s; ++i) {
    const int pp = parts[i].partial ? i : -1;
    for (int r = roff[i] + threadIdx.x; r < roff[i + 1]; r += blockDim.x) rt_pp[r] = pp;
  }
  __syncthreads();
  int longest = -1;  // the part with the most temporal rows (warm starts)
  for (int i = 0, best = 0; i < s; ++i)
    if (parts[i].len > best) {
      best = int(parts[i].len);
      longest = i;
    }
  double* Est = ws + lay.E;  // stacked E (R x k0, ld R): U0 = blockdiag(V_sub,i) E
  double* Ast = ws + lay.A;  // stacked A = S E (rows of partial parts)
  double* Cst = ws + lay.C;  // stacked C (R x Q, row-major)
  auto Ep = [&](int i) { return Est + roff[i]; };  // ld R
  auto Ap = [&](int i) { return Ast + roff[i]; };  // ld R

  // ---- partial-hit metric S_i = Vsub^T Vsub and the norm of the implied tensor
  double norm_sq = 0.0;
  if (leader) {
  {  // entire parts: sum of the squared cores, one pass over all parts
    double acc = 0.0;
    for (int i = 0; i < s; ++i) {
      if (parts[i].partial) continue;
      const double* c = parts[i].core;
      const int64_t ne = prod_range(parts[i].rho, 0, p);
      for (int64_t e = threadIdx.x; e < ne; e += blockDim.x) acc = fma(c[e], c[e], acc);
    }
    norm_sq = block_sum(acc, sc);
  }
  for (int i = 0; i < s; ++i) {
    if (!parts[i].partial) continue;
    const PartView pv = load_part(parts[i]);
    const int64_t r0 = pv.rho[0];
    const int64_t hk = prod_range(pv.rho, 1, p);
    {
      const double* vs = pv.v0 + pv.row0;
      {
        const long long tg = tstart();
        gram_long(vs, pv.ld0, pv.len, int(r0), Sp(i), dsm);
        tstop(sc, kPhGram, tg);
      }
      // ||H x_0 R||^2 = sum_ab S_ab (M0(H) M0(H)^T)_ab
      tgemm(r0, r0, hk, pv.core, hk, 1, pv.core, 1, hk, HH, 1, r0, false, sc);
      double acc = 0.0;
      for (int64_t e = threadIdx.x; e < r0 * r0; e += blockDim.x) acc = fma(Sp(i)[e], HH[e], acc);
      norm_sq += block_sum(acc, sc);
    }
  }
  }  // leader
  if constexpr (CL) {
    if (leader && threadIdx.x == 0) xch[0] = norm_sq;
    cl_sync();
    norm_sq = xch[0];
  }
  // ---- init (stitch.cpp:135-144): U_m = random_orthonormal(D_m, r_m), m >= 1
  for (int m = 1; m < p; ++m) {
    if (leader) bcopy(D.out_f[m], prm.stitch_init[m], d[m] * rc[m]);
    k[m] = rc[m];
  }
  k[0] = rc[0];
  int sweeps = 0, converged = 0, any_zero_sigma = 0;
  if (norm_sq == 0.0) {  // stitch.cpp:146-150; U_0 is drawn by the host
    if (leader) bzero(D.out_core, prod_range(rc, 0, p));
    converged = 1;
  } else {
    // P_im = U_m^T V_im for every part and mode m >= 1, one batched pass
    auto pm_entry = [&](int i, int m) {
      BGemm g;
      g.A = D.out_f[m];
      g.B = parts[i].v[m];
      g.C = Pm(i, m);
      g.M = int(k[m]);
      g.N = int(parts[i].rho[m]);
      g.K = int(d[m]);
      g.outer = 1;
      g.ars = int(d[m]);
      g.acs = 1;
      g.brs = 1;
      g.bcs = int(d[m]);
      g.crs = 1;
      g.ccs = int(k[m]);
      g.aos = g.bos = g.cos = 0;
      g.acc = 0;
      return g;
    };
    if (leader) gemm_batched(s * (p - 1), [&](int e) { return pm_entry(e / (p - 1), 1 + e % (p - 1)); }, sc);
    const double norm = sqrt(norm_sq);
    double prev_fit = nan("");
    bool wk_valid = false;  // wk holds the previous sweep's G0 eigenvectors (mode-0 fallback warm start)
    for (int sweep = 0; sweep < prm.max_iters; ++sweep) {
      // ================= mode 0 (stitch_temporal_unfolding, stitch.cpp:49-73)
      const int64_t k0n = stitch_mode_rank(p, d, rc, k, 0);
      const int64_t Q = prod_range(k, 1, p);
      if (leader) {
      auto Cp = [&](int i) { return Cst + int64_t(roff[i]) * Q; };  // rows of part i (row-major, stride Q)
      // C_i = M0(H_i x_{p-1} P_{i,p-1} ... x_1 P_i1), descending as the reference;
      // one batched pass per mode over all parts
      for (int m = p - 1; m >= 1; --m) {
        const int step = p - 1 - m;
        gemm_batched(s, [&](int i) {
          int64_t cur[kMaxP];
          for (int q = 0; q < p; ++q) cur[q] = q > m ? k[q] : parts[i].rho[q];
          const double* src = step == 0 ? parts[i].core : TB[(step - 1) & 1] + int64_t(i) * lay.chain;
          double* dst = (m == 1) ? Cst + int64_t(roff[i]) * Q : TB[step & 1] + int64_t(i) * lay.chain;
          return bg_mode_product(src, prod_range(cur, 0, m), cur[m], prod_range(cur, m + 1, p), Pm(i, m), 1, k[m],
                                 k[m], dst);
        }, sc);
      }
      // ---- subspace iteration on the implicit Z0 in compressed coordinates:
      // U0 = blockdiag(V_sub,i) E with E^T S E = I; Z0 Z0^T U0 maps to
      // E <- C (C^T S E). Warm start: the previous sweep's E, or in sweep 0 the
      // k0 columns of C with the largest S-norm. Rayleigh-Ritz makes E the exact
      // left singular vectors; any failure falls through to the eigen paths.
      // All parts are processed together as stacked R-row matrices (E, A = S E
      // in shared memory, C row-major in the workspace), so an iteration costs
      // a fixed number of block passes whatever s is.
      bool mode0_done = false;
      const int kk = int(k0n);
      // shared memory: [0, 768) Rayleigh-Ritz eigensolver scratch, Y (Q x k),
      // G/L/Linv/B (k x k), E and A (R x k each)
      const int64_t si_smem = 768 + Q * kk + 5 * kk * kk + 2 * int64_t(R) * kk;
      if (kk <= kSiMaxK && Q >= 2 * kk && R >= kk && si_smem <= sc.dsm_cap) {
        const long long t_si = tstart();
        const int nt = int(blockDim.x);
        const int Qi = int(Q);
        double* Y = dsm + 768;            // Q x kk
        double* small = Y + Q * kk;       // G, L, Linv (kk x kk each)
        double* B = small + 4 * kk * kk;  // kk x kk
        double* Es = B + kk * kk;         // R x kk (ld R)
        double* As = Es + R * kk;         // R x kk (ld R)
        double* Rg = Z;                   // residual rows of partial parts (ld R)
        // dst = S src (entire rows: S = I); both stacked, ld R
        auto apply_S_all = [&](const double* src, double* dst) {
          for (int idx = threadIdx.x; idx < R * kk; idx += nt) {
            const int r = idx % R, j = idx / R;
            const int i = rt_pp[r];
            double v;
            if (i < 0) {
              v = src[idx];
            } else {
              const int o = roff[i], r0 = roff[i + 1] - o;
              const double* S = Sp(i) + (r - o);
              const double* e = src + o + j * R;
              v = 0.0;
              for (int b = 0; b < r0; ++b) v = fma(S[b * r0], e[b], v);
            }
            dst[idx] = v;
          }
          __syncthreads();
        };
        // S-orthonormalise Es in place (two CholeskyQR passes in the metric S)
        auto s_orth = [&]() -> bool {
          const int tot = kk * kk;
          const int nsplit = nt / tot > 0 ? nt / tot : 1;
          double* Gk = small;
          double* Li = small + 2 * kk * kk;
          for (int pass = 0; pass < 2; ++pass) {
            apply_S_all(Es, As);
            if (threadIdx.x < tot * nsplit) {  // G = E^T A, rows split across the block
              const int e = threadIdx.x % tot, part = threadIdx.x / tot;
              const double* x = Es + (e % kk) * R;
              const double* y = As + (e / kk) * R;
              double v = 0.0;
              for (int r = part; r < R; r += nsplit) v = fma(x[r], y[r], v);
              sc.red[threadIdx.x] = v;
            }
            if (threadIdx.x == 0) sc.ibcast[2] = 0;
            __syncthreads();
            if (threadIdx.x < tot) {
              double v = 0.0;
              for (int part = 0; part < nsplit; ++part) v += sc.red[part * tot + threadIdx.x];
              Gk[threadIdx.x] = v;
            }
            __syncthreads();
            chol_inv_warp(Gk, kk, small + tot, Li, sc);
            __syncthreads();
            if (sc.ibcast[2]) return false;
            for (int r = threadIdx.x; r < R; r += nt) {
              double w[kSiMaxK];
#pragma unroll
              for (int l = 0; l < kSiMaxK; ++l) w[l] = l < kk ? Es[r + l * R] : 0.0;
#pragma unroll
              for (int j = 0; j < kSiMaxK; ++j) {
                if (j < kk) {
                  double v = 0.0;
#pragma unroll
                  for (int l = 0; l <= j; ++l) v = fma(w[l], Li[j + l * kk], v);
                  Es[r + j * R] = v;
                }
              }
            }
            __syncthreads();
          }
          return true;
        };
        bool ok = true;
        long long tp = tstart();
        if (sweep == 0 || k[0] < k0n) {
          // start: the k0 columns of C with the largest S-norm
          double* cn = misc + kMisc / 2;  // Q norms
          for (int q = threadIdx.x; q < Qi; q += nt) {
            double v = 0.0;
            for (int i = 0; i < s; ++i) {
              const int o = roff[i], r0 = roff[i + 1] - o;
              const double* Ci = Cst + int64_t(o) * Qi + q;
              if (parts[i].partial) {
                const double* S = Sp(i);
                for (int a = 0; a < r0; ++a)
                  for (int b = 0; b < r0; ++b) v = fma(Ci[a * Qi] * S[a + b * r0], Ci[b * Qi], v);
              } else {
                for (int a = 0; a < r0; ++a) v = fma(Ci[a * Qi], Ci[a * Qi], v);
              }
            }
            cn[q] = v;
          }
          __syncthreads();
          int* pick = reinterpret_cast<int*>(misc);
          for (int q = threadIdx.x; q < Qi; q += nt) {
            int rank = 0;
            for (int l = 0; l < Qi; ++l) rank += (cn[l] > cn[q] || (cn[l] == cn[q] && l < q));
            if (rank < kk) pick[rank] = q;
          }
          __syncthreads();
          for (int idx = threadIdx.x; idx < R * kk; idx += nt) {
            const int r = idx % R, c = idx / R;
            Es[idx] = Cst[int64_t(r) * Qi + pick[c]];
          }
          __syncthreads();
          ok = s_orth();
        } else {
          // warm start: the previous sweep's E (first k0n columns, ld R)
          for (int idx = threadIdx.x; idx < R * kk; idx += nt) Es[idx] = Est[idx];
          __syncthreads();
        }
        tstop_m0(sc, kSiAtU, tp);
        bool conv = false;
        for (int it = 0; ok && it < kSiMaxIter; ++it) {
          // A = S E ; Y = C^T A (Q x k) ; B = Y^T Y ; W = C Y
          tp = tstart();
          apply_S_all(Es, As);
          for (int idx = threadIdx.x; idx < Qi * kk; idx += nt) {
            const int q = idx % Qi, j = idx / Qi;
            const double* a = As + j * R;
            const double* c = Cst + q;
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
            int r = 0;
            for (; r + 3 < R; r += 4) {
              v0 = fma(c[int64_t(r) * Qi], a[r], v0);
              v1 = fma(c[int64_t(r + 1) * Qi], a[r + 1], v1);
              v2 = fma(c[int64_t(r + 2) * Qi], a[r + 2], v2);
              v3 = fma(c[int64_t(r + 3) * Qi], a[r + 3], v3);
            }
            for (; r < R; ++r) v0 = fma(c[int64_t(r) * Qi], a[r], v0);
            Y[idx] = (v0 + v1) + (v2 + v3);
          }
          __syncthreads();
          for (int e = threadIdx.x; e < kk * kk; e += nt) {
            const double* y1 = Y + (e % kk) * Qi;
            const double* y2 = Y + (e / kk) * Qi;
            double v = 0.0;
            for (int q = 0; q < Qi; ++q) v = fma(y1[q], y2[q], v);
            B[e] = v;
          }
          __syncthreads();
          tstop_m0(sc, kSiAY, tp);
          tp = tstart();
          // per row: W = C Y (into As), residual W - E B: rsq += |.|^2 on entire
          // rows, partial rows keep it for the metric term
          double rsq = 0.0;
          for (int r = threadIdx.x; r < R; r += nt) {
            double w[kSiMaxK], e[kSiMaxK];
#pragma unroll
            for (int l = 0; l < kSiMaxK; ++l) {
              w[l] = 0.0;
              e[l] = l < kk ? Es[r + l * R] : 0.0;
            }
            const double* Cr = Cst + int64_t(r) * Qi;
            int q = 0;
            for (; q + 3 < Qi; q += 4) {  // four C loads in flight
              const double c0 = Cr[q], c1 = Cr[q + 1], c2 = Cr[q + 2], c3 = Cr[q + 3];
#pragma unroll
              for (int l = 0; l < kSiMaxK; ++l)
                if (l < kk) {
                  const double* y = Y + q + l * Qi;
                  w[l] = fma(c3, y[3], fma(c2, y[2], fma(c1, y[1], fma(c0, y[0], w[l]))));
                }
            }
            for (; q < Qi; ++q) {
              const double cv = Cr[q];
#pragma unroll
              for (int l = 0; l < kSiMaxK; ++l)
                if (l < kk) w[l] = fma(cv, Y[q + l * Qi], w[l]);
            }
            const bool part_row = rt_pp[r] >= 0;
#pragma unroll
            for (int j = 0; j < kSiMaxK; ++j) {
              if (j < kk) {
                double v = w[j];
#pragma unroll
                for (int l = 0; l < kSiMaxK; ++l)
                  if (l < kk) v = fma(-e[l], B[l + j * kk], v);
                As[r + j * R] = w[j];
                if (part_row)
                  Rg[r + j * R] = v;
                else
                  rsq = fma(v, v, rsq);
              }
            }
          }
          __syncthreads();
          if (any_partial) {
            for (int idx = threadIdx.x; idx < R * kk; idx += nt) {
              const int r = idx % R, j = idx / R;
              const int i = rt_pp[r];
              if (i < 0) continue;
              const int o = roff[i], r0 = roff[i + 1] - o;
              const double* S = Sp(i) + (r - o);
              const double* e = Rg + o + j * R;
              double v = 0.0;
              for (int b = 0; b < r0; ++b) v = fma(S[b * r0], e[b], v);
              rsq = fma(v, Rg[idx], rsq);
            }
          }
          double bsq = 0.0;
          for (int e = threadIdx.x; e < kk * kk; e += nt) bsq = fma(B[e], B[e], bsq);
          rsq = block_sum(rsq, sc);
          bsq = block_sum(bsq, sc);
          if (!(bsq > 0.0)) {
            ok = false;
            break;
          }
          if (rsq <= 1e-26 * bsq) {
            conv = true;
            if (threadIdx.x == 0) sc.si_iters += it + 1;
            break;
          }
          tstop_m0(sc, kSiQR, tp);
          tp = tstart();
          for (int idx = threadIdx.x; idx < R * kk; idx += nt) Es[idx] = As[idx];
          __syncthreads();
          ok = s_orth();
          tstop_m0(sc, kSiRR, tp);
        }
        if (ok && conv) {
          // Rayleigh-Ritz: E <- E R (descending); store E and A = S E
          int* order = reinterpret_cast<int*>(misc);
          double* diag = nullptr;
          const double* Rv = eig_run(B, kk, small, order, dsm, &diag, sc);
          for (int r = threadIdx.x; r < R; r += nt) {
            double w[kSiMaxK];
#pragma unroll
            for (int l = 0; l < kSiMaxK; ++l) w[l] = l < kk ? Es[r + l * R] : 0.0;
            for (int j = 0; j < kk; ++j) {
              const double* rj = Rv + order[j] * kk;
              double v = 0.0;
#pragma unroll
              for (int l = 0; l < kSiMaxK; ++l)
                if (l < kk) v = fma(w[l], rj[l], v);
              Est[r + j * R] = v;
              Es[r + j * R] = v;
            }
          }
          __syncthreads();
          if (any_partial) {
            apply_S_all(Es, As);
            for (int idx = threadIdx.x; idx < R * kk; idx += nt) Ast[idx] = As[idx];
            __syncthreads();
          }
          any_zero_sigma = 0;
          mode0_done = true;
          if (threadIdx.x == 0) sc.si_ok += 1;
        } else if (threadIdx.x == 0) {
          sc.si_fail += 1;
        }
        tstop(sc, kPhEig, t_si);
      }
      // Row-compressed variant: with entire parts only, Z0 = blockdiag(V_i0) C
      // (C = [C_1; ...; C_s], R = sum rho_i0 rows) and V_i0 orthonormal, so the
      // left singular vectors of Z0 are blockdiag(V_i0) times the eigenvectors
      // of C C^T — an R^2 problem instead of Q^2 when that is smaller, with no
      // Sigma^-1 amplification.
      if (mode0_done) {
        // E, A already set by the subspace iteration
      } else if (!any_partial && R < Q && k0n <= R) {  // else: rank-deficient Z0 needs the completion path
        tgemm(R, R, Q, Cst, Q, 1, Cst, 1, Q, G, 1, R, false, sc);
        int* order = reinterpret_cast<int*>(misc);
        double* diag = nullptr;
        const double* Vp = eig_run(G, R, Vg, order, dsm, &diag, sc);
        for (int64_t idx = threadIdx.x; idx < int64_t(R) * k0n; idx += blockDim.x) {
          const int64_t r = idx % R, c = idx / R;
          Est[idx] = Vp[r + int64_t(order[c]) * R];
        }
        __syncthreads();
        any_zero_sigma = 0;
      } else {
        // G0 = Z0^T Z0 = sum_i C_i^T S_i C_i   (Q x Q)
        for (int i = 0; i < s; ++i) {
          const int64_t r0 = parts[i].rho[0];
          const double* rhs = Cp(i);
          if (parts[i].partial) {
            tgemm(r0, Q, r0, Sp(i), 1, r0, Cp(i), Q, 1, T[0], Q, 1, false, sc);
            rhs = T[0];
          }
          tgemm(Q, Q, r0, Cp(i), 1, Q, rhs, Q, 1, G, 1, Q, i > 0, sc);
        }
        {
          int* order = reinterpret_cast<int*>(misc);
          double* sig = misc + kMisc / 2;
          double* lamv = misc + kMisc / 2 + 512;
          double* diag = nullptr;
          if (threadIdx.x == 0) sc.ibcast[1] = 0;
          // ranks beyond the E-coordinate iteration (C5: k0 = 20 on a 400 x 400
          // G0): warm-started top-k Gram iteration instead of a full Jacobi of G0
          // — start from the previous sweep's eigenvectors (wk, same directions),
          // or in sweep 0 from the canonical vectors of G0's k0 largest diagonal
          // entries; the Jacobi path remains the fallback
          const double* Vsi = nullptr;
          if (k0n > kSiMaxK && k0n <= kGramSiMaxK && Q >= 2 * k0n && Q > kGramSiMinN &&
              7 * k0n * k0n + 256 <= sc.dsm_cap) {
            double* Us = Vg;
            double* Ws = Vg + Q * k0n;
            if (wk_valid) {
              for (int64_t idx = threadIdx.x; idx < Q * k0n; idx += blockDim.x) Us[idx] = wk[idx];
            } else {
              int* pick = reinterpret_cast<int*>(misc);
              for (int q = threadIdx.x; q < int(Q); q += blockDim.x) {
                int rank = 0;
                const double gq = G[q + q * Q];
                for (int l = 0; l < int(Q); ++l) {
                  const double gl = G[l + l * Q];
                  rank += (gl > gq || (gl == gq && l < q));
                }
                if (rank < k0n) pick[rank] = q;
              }
              __syncthreads();
              for (int64_t idx = threadIdx.x; idx < Q * k0n; idx += blockDim.x) {
                const int64_t j = idx % Q, c = idx / Q;
                Us[idx] = (j == pick[c]) ? 1.0 : 0.0;
              }
            }
            __syncthreads();
            Vsi = sym_topk_si(G, int(Q), int(k0n), Us, Ws, lamv, order, dsm, sc);
            if (threadIdx.x == 0) {
              if (Vsi)
                sc.si_ok += 1;
              else
                sc.si_fail += 1;
            }
          }
          const double* Vp = Vsi;
          if (!Vsi) Vp = eig_run(G, int(Q), Vg, order, dsm, &diag, sc);
          auto vcol = [&](int64_t c) { return Vsi ? Vsi + c * Q : Vp + int64_t(order[c]) * Q; };
          auto lamc = [&](int64_t c) { return Vsi ? lamv[c] : diag[order[c] * (Q + 1)]; };
          if (threadIdx.x < k0n) {
            const double l0 = fmax(lamc(0), 0.0);
            const double lc = fmax(lamc(threadIdx.x), 0.0);
            const bool ok = gram_sigma_ok(lc, l0);
            sig[threadIdx.x] = ok ? 1.0 / sqrt(lc) : 0.0;
            if (!ok) atomicOr(&sc.ibcast[1], 1);
          }
          __syncthreads();
          for (int64_t idx = threadIdx.x; idx < Q * k0n; idx += blockDim.x) {
            const int64_t j = idx % Q, c = idx / Q;
            wk[idx] = vcol(c)[j] * sig[c];
          }
          __syncthreads();
          any_zero_sigma = sc.ibcast[1];
          wk_valid = !any_zero_sigma;
        }
        // E = C W Sigma^-1 (R x k0, stacked);  A_i = S_i E_i = (U0[rows_i]^T V_i0)^T
        tgemm(R, k0n, Q, Cst, Q, 1, wk, 1, Q, Est, 1, R, false, sc);
        for (int i = 0; i < s; ++i)
          if (parts[i].partial) {
            const int64_t r0 = parts[i].rho[0];
            tgemm(r0, k0n, r0, Sp(i), 1, r0, Ep(i), 1, R, Ap(i), 1, R, false, sc);
          }
      }
      }  // leader: mode 0
      k[0] = k0n;
      // ================= modes n >= 1 (stitch_nontemporal_unfolding, stitch.cpp:75-108)
      for (int n = 1; n < p; ++n) {
        const int64_t kn = stitch_mode_rank(p, d, rc, k, n);
        int64_t zc[kMaxP];
        for (int m = 0; m < p; ++m) zc[m] = (m == n) ? d[n] : k[m];
        const int64_t zo = prod_range(zc, 0, n), zi = prod_range(zc, n + 1, p);
        // F_i = H_i x_0 (U0[rows_i]^T V_i0) x_{m != 0,n} P_im, shape (zo, rho_in, zi)
        const int64_t Qn = zo * zi;
        int64_t rho_n_sum = 0;
        for (int i = 0; i < s; ++i) rho_n_sum += parts[i].rho[n];
        const bool one_pass = rho_n_sum * Qn <= int64_t(sc.dsm_cap) && s >= TT_ONE_PASS_MIN_PARTS && s <= 64;
        // F_i chain, one batched pass per contracted mode over all parts:
        // x_0 (U0[rows_i]^T V_i0) with M(a, j) = A0[j + a*rho0], then x_m P_im
        // for m != 0, n ascending; F_i ends in TB[(nsteps-1)&1] + i*chain
        int nsteps = 0;
        for (int m = 0; m < p; ++m) {
          if (m == n) continue;
          const int step = nsteps++;
          if (leader) gemm_batched(s, [&](int i) {
            int64_t cur[kMaxP];
            for (int q = 0; q < p; ++q) cur[q] = (q < m && q != n) ? k[q] : parts[i].rho[q];
            double* dst = TB[step & 1] + int64_t(i) * lay.chain;
            if (m == 0) {
              const double* A0 = parts[i].partial ? Ap(i) : Ep(i);
              return bg_mode_product(parts[i].core, 1, cur[0], prod_range(cur, 1, p), A0, R, 1, k[0], dst);
            }
            const double* src = TB[(step - 1) & 1] + int64_t(i) * lay.chain;
            return bg_mode_product(src, prod_range(cur, 0, m), cur[m], prod_range(cur, m + 1, p), Pm(i, m), 1, k[m],
                                   k[m], dst);
          }, sc);
        }
        double* Fb = TB[(nsteps - 1) & 1];
        if constexpr (CL) cl_sync();  // F_i complete
        if (!one_pass && leader) {
          // per-part accumulation: Z_n += F_i x_n V_in
          for (int i = 0; i < s; ++i)
            mode_product(Fb + int64_t(i) * lay.chain, zo, parts[i].rho[n], zi, parts[i].v[n], 1, d[n], d[n], Z,
                         i > 0, sc);
        }
        // Every mode but the last writes Z_n as the dense row-major unfolding
        // (d_n x Qn): llsv then reads contiguous rows (coalesced warm start,
        // shared-memory back-multiplication). The last mode's Z feeds the core
        // and keeps the tensor layout.
        const bool dense_z = one_pass && n < p - 1;
        if (one_pass) {
          // Z_n = sum_i F_i x_n V_in written once: the stacked F (sum rho_in x Qn)
          // is staged in shared memory; a thread owns one row a of Z and 8
          // columns, streaming V_in[a, :] from global (coalesced over a).
          const long long tz = tstart();
          __shared__ const double* vptr[64];
          __shared__ int64_t foff[65];
          if (threadIdx.x == 0) {
            int64_t o = 0;
            for (int i = 0; i < s; ++i) {
              vptr[i] = parts[i].v[n];
              foff[i] = o;
              o += parts[i].rho[n];
            }
            foff[s] = o;
          }
          __syncthreads();
          double* Fs = dsm;
          for (int i = 0; i < s; ++i) {
            const int64_t rn = foff[i + 1] - foff[i];
            const double* F = Fb + int64_t(i) * lay.chain;
            for (int64_t e = threadIdx.x; e < rn * Qn; e += blockDim.x) {
              const int64_t j = e / Qn, c = e - j * Qn;
              const int64_t o = c / zi, t = c - o * zi;
              Fs[(foff[i] + j) * Qn + c] = F[(o * rn + j) * zi + t];
            }
          }
          __syncthreads();
          const int64_t dn = d[n];
          const int64_t ncb = (Qn + 7) / 8;
          // this CTA's rows of Z_n (all of them outside a cluster)
          const int64_t rper = (dn + CS - 1) / CS;
          const int64_t a_lo = imin(dn, int64_t(rank) * rper), a_n = imin(dn, a_lo + rper) - a_lo;
          for (int64_t w = threadIdx.x; w < a_n * ncb; w += blockDim.x) {
            const int64_t a = a_lo + w % a_n, cb = w / a_n;
            const int64_t c0 = cb * 8;
            double acc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = 0.0;
            for (int i = 0; i < s; ++i) {
              const double* V = vptr[i] + a;
              const int64_t j0 = foff[i], rn = foff[i + 1] - j0;
              int64_t j = 0;
              for (; j + 3 < rn; j += 4) {  // four V loads in flight
                const double v0 = V[j * dn], v1 = V[(j + 1) * dn], v2 = V[(j + 2) * dn], v3 = V[(j + 3) * dn];
                const double* fr = Fs + (j0 + j) * Qn + c0;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                  if (c0 + c < Qn)
                    acc[c] = fma(v3, fr[c + 3 * Qn], fma(v2, fr[c + 2 * Qn], fma(v1, fr[c + Qn], fma(v0, fr[c], acc[c]))));
              }
              for (; j < rn; ++j) {
                const double v = V[j * dn];
                const double* fr = Fs + (j0 + j) * Qn + c0;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                  if (c0 + c < Qn) acc[c] = fma(v, fr[c], acc[c]);
              }
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int64_t cc = c0 + c;
              if (cc < Qn) {
                if (dense_z) {  // the mode-n unfolding itself: dense row-major d_n x Qn
                  Z[a * Qn + cc] = acc[c];
                } else {
                  const int64_t o = cc / zi, t = cc - o * zi;
                  Z[(o * dn + a) * zi + t] = acc[c];
                }
              }
            }
          }
          __syncthreads();
          tstop(sc, kPhTtm, tz);
        }
        // Warm start of the eigen-iterations: in sweep 0 the factor still holds the
        // random init; the longest part's own mode-n factor spans nearly the same
        // subspace and cuts the iterations. The init value of U_n is not used again
        // (P_in is recomputed below), and the converged top-k vectors do not depend
        // on the start.
        int64_t kprev = k[n];
        if (sweep == 0 && longest >= 0) {
          kprev = imin(parts[longest].rho[n], k[n]);
          if (leader) bcopy(D.out_f[n], parts[longest].v[n], d[n] * kprev);
        }
        if constexpr (CL) {
          cl_sync();  // Z_n complete
          wide_llsv(Z, dense_z ? 1 : zo, d[n], dense_z ? Qn : zi, kn, D.out_f[n], G, Vg, misc, dsm, sc, kprev,
                    ws + lay.SI, gpart, rank, CS);
        } else {
          llsv_unfold(Z, dense_z ? 1 : zo, d[n], dense_z ? Qn : zi, kn, D.out_f[n], G, Vg, misc, dsm, sc, kprev,
                      ws + lay.SI);
        }
        k[n] = kn;
        if (leader) gemm_batched(s, [&](int i) { return pm_entry(i, n); }, sc);
      }
      // ================= core: fold Z_{p-1} and project the last mode (stitch.cpp:163-172)
      double stop = 0.0;
      if (leader) {
        mode_product(Z, prod_range(k, 0, p - 1), d[p - 1], 1, D.out_f[p - 1], d[p - 1], 1, k[p - 1], D.out_core,
                     false, sc);
        const double core_sq = bsumsq(D.out_core, prod_range(k, 0, p), sc);
        const double res = fmax(0.0, norm_sq - core_sq);
        if (threadIdx.x == 0) D.objective[sweep] = res;
        const double fit = 1.0 - sqrt(res) / norm;
        stop = (sweep > 0 && fabs(fit - prev_fit) < prm.tol) ? 1.0 : 0.0;
        prev_fit = fit;
      }
      if constexpr (CL) {
        if (leader && threadIdx.x == 0) xch[1] = stop;
        cl_sync();
        stop = xch[1];
      }
      sweeps = sweep + 1;
      if (stop != 0.0) {
        converged = 1;
        break;
      }
    }
    if constexpr (CL) {
      if (!leader) return;  // the leader materialises U_0 and reports
    }
    // ================= materialise U_0 = blockdiag(Vsub_i) [E_i] (L x k0), sign-fixed
    const int64_t k0 = k[0];
    double* U0 = D.out_f[0];
    const long long tu = tstart();
    if (any_zero_sigma ||
        !materialize_u0(int(k0), parts, s, Est, R, roff, U0, D.L, flips, idxbuf, dsm, sc)) {
      // Row-parallel materialisation in column chunks of KU: each thread owns
      // rows, keeps the first max-|.| row per column (sign convention), then a
      // block argmax picks each column's sign. Rows of part i: Vsub_i[r,:] E_i.
      constexpr int KU = 8;
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      for (int c0 = 0; c0 < k0; c0 += KU) {
        const int nc = int(imin(KU, k0 - c0));
        double best[KU];
        int64_t bidx[KU];
  #pragma unroll
        for (int c = 0; c < KU; ++c) {
          best[c] = -1.0;
          bidx[c] = 0;
        }
        int64_t off = 0;
        for (int i = 0; i < s; ++i) {
          const PartView pv = load_part(parts[i]);
          const int64_t r0 = pv.rho[0];
          const double* vs = pv.v0 + pv.row0;
          const double* E = Ep(i) + c0 * R;
          for (int64_t r = threadIdx.x; r < pv.len; r += blockDim.x) {
            double out[KU];
  #pragma unroll
            for (int c = 0; c < KU; ++c) out[c] = 0.0;
            for (int64_t a = 0; a < r0; ++a) {
              const double v = vs[r + a * pv.ld0];
  #pragma unroll
              for (int c = 0; c < KU; ++c)
                if (c < nc) out[c] = fma(v, E[a + c * R], out[c]);
            }
  #pragma unroll
            for (int c = 0; c < KU; ++c)
              if (c < nc) {
                U0[off + r + (c0 + c) * D.L] = out[c];
                const double m = fabs(out[c]);
                if (m > best[c]) {
                  best[c] = m;
                  bidx[c] = off + r;
                }
              }
          }
          off += pv.len;
        }
  #pragma unroll
        for (int c = 0; c < KU; ++c) {
          double b = best[c];
          int64_t bi = bidx[c];
  #pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, b, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > b || (ob == b && oi < bi)) {
              b = ob;
              bi = oi;
            }
          }
          if (l == 0 && c < nc) {
            sc.red[w * kMaxVec + c0 + c] = b;
            idxbuf[w * kMaxVec + c0 + c] = bi;
          }
        }
      }
      __syncthreads();
      if (any_zero_sigma) {
        orthonormalize(U0, D.L, 0, int(k0), D.L, sc);
        sign_fix(U0, D.L, int(k0), D.L, flips, sc);
      } else {
        if (threadIdx.x < k0) {
          const int c = threadIdx.x;
          double b = sc.red[c];
          int64_t bi = idxbuf[c];
          for (int ww = 1; ww < kWarps; ++ww) {
            const double ob = sc.red[ww * kMaxVec + c];
            const int64_t oi = idxbuf[ww * kMaxVec + c];
            if (ob > b || (ob == b && oi < bi)) {
              b = ob;
              bi = oi;
            }
          }
          flips[c] = U0[bi + c * D.L] < 0.0;
        }
        __syncthreads();
        for (int64_t idx = threadIdx.x; idx < D.L * k0; idx += blockDim.x)
          if (flips[idx / D.L]) U0[idx] = -U0[idx];
        __syncthreads();
      }
    }
    const int64_t slice = prod_range(k, 1, p);
    for (int64_t e = threadIdx.x; e < k0 * slice; e += blockDim.x)
      if (flips[e / slice]) D.out_core[e] = -D.out_core[e];
    __syncthreads();
    tstop(sc, kPhU0, tu);
  }
  if (leader && threadIdx.x == 0) {
    D.status[0] = sweeps;
    D.status[1] = converged;
    D.status[2] = norm_sq == 0.0;
    D.status[3] = any_zero_sigma;
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

// ---------------------------------------------------------------------------
}  // namespace ttb
