// Shared host/device definitions: problem descriptors, rank planning and
// workspace layout. Everything here is data-independent integer arithmetic,
// evaluated identically on the host (planning, buffer sizing) and on the
// device (per-sweep shapes inside the ALS kernels).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define TT_HD __host__ __device__ __forceinline__
#else
#define TT_HD inline
#endif

namespace ttb {

constexpr int kMaxP = 8;
// Bound on the stacked temporal rows (sum of the parts' rho_0) of one stitch
// (shared-memory row tables of the stitch kernel).
constexpr int kStitchMaxRows = 1024;

TT_HD int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
TT_HD int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

TT_HD int64_t prod_except(const int64_t* a, int p, int skip) {
  int64_t r = 1;
  for (int m = 0; m < p; ++m)
    if (m != skip) r *= a[m];
  return r;
}
TT_HD int64_t prod_range(const int64_t* a, int b, int e) {
  int64_t r = 1;
  for (int m = b; m < e; ++m) r *= a[m];
  return r;
}

// clamp_ranks (tucker.cpp:41-52): r_n <- min(r_n, D_n).
TT_HD void clamp_ranks(int p, const int64_t* d, const int64_t* req, int64_t* rc) {
  for (int m = 0; m < p; ++m) rc[m] = imin(req[m], d[m]);
}

// Column count returned by leading_left_singular_vectors (linalg.cpp:47):
// k = min(rank, rows, cols) with cols = prod of the other factors' columns.
// tucker_als requests the current column count (tucker.cpp:63-64) ...
TT_HD int64_t leaf_mode_rank(int p, const int64_t* d, const int64_t* k, int n) {
  return imin(imin(k[n], d[n]), prod_except(k, p, n));
}
// ... stitch requests the clamped rank every sweep (stitch.cpp:155-161).
TT_HD int64_t stitch_mode_rank(int p, const int64_t* d, const int64_t* rc, const int64_t* k, int n) {
  return imin(imin(rc[n], d[n]), prod_except(k, p, n));
}

// ---------------------------------------------------------------------------
// Problem descriptors (device-visible PODs).
// Tile shape of the streamed mode products (shared by the host, which encodes
// the TMA tensor maps, and the device loop): G slabs x cj rows x tw columns.
struct StreamTile {
  int64_t tw, G, cj;
};
#ifndef TT_STREAM_TILE_DOUBLES
#define TT_STREAM_TILE_DOUBLES 3072
#endif
constexpr int64_t kStreamTileDoubles = TT_STREAM_TILE_DOUBLES;  // 24 KB per ring stage (measured best of 20/24/32 KB at 2 stages)
TT_HD StreamTile stream_tile(int64_t outer, int64_t d, int64_t inner) {
  StreamTile t;
  t.tw = imin(inner, 256);
  t.G = imax(1, imin(imin(outer, 256 / t.tw), 256));
  t.cj = imax(1, imin(imin(d, kStreamTileDoubles / (t.G * t.tw)), 256));
  return t;
}

struct LeafDesc {
  const double* x;                 // row-major (len, D_1, ..., D_{p-1})
  const void* tmaps;               // 2 CUtensorMaps (128 B each): [0] X as (inner, D_1, len), [1] X as (ns, len); or null
  int64_t len;                     // temporal extent of this block
  const double* init[kMaxP];       // init factors for this length (D_n x rc_n, col-major)
  double* out_f[kMaxP];            // output factor slots (ld = D_n; factor 0: ld = len)
  double* out_core;                // row-major core, capacity prod rc
  double* ws;                      // workspace (leaf_ws_size doubles)
  int32_t* status;                 // [sweeps, converged, zero, deficient, k_0..k_7, eig calls, eig sweeps]
  double* objective;               // max_iters doubles
};

struct StitchPart {
  const double* core;              // row-major (rho_0, ..., rho_{p-1})
  int64_t rho[kMaxP];
  const double* v0;                // temporal factor of the stored node (col-major)
  int64_t ld0;                     // its leading dimension (node length)
  int64_t row0;                    // first row used (partial hit) or 0
  int64_t len;                     // rows used
  int32_t partial;                 // 1: rows [row0, row0+len) of a longer factor
  int32_t pad;
  const double* v[kMaxP];          // non-temporal factors, m >= 1 (D_m x rho_m)
};

struct StitchDesc {
  int32_t part0, nparts;
  int64_t L;                       // total temporal length
  double* out_f[kMaxP];            // factor 0: L x rc0 (ld = L); m: D_m x rc_m
  double* out_core;
  double* ws;
  int32_t* status;
  double* objective;
};

struct Params {
  int32_t p;
  int32_t max_iters;
  double tol;
  int64_t d[kMaxP];                // d[0] ignored (per problem); d[m] = D_m
  int64_t req[kMaxP];              // requested ranks
  const double* stitch_init[kMaxP];  // stitch init factors U_m (m >= 1), D_m x rc_m
};

struct CopySeg {
  const double* src;
  double* dst;
  int64_t n;
};

constexpr int kStatusInts = 4 + kMaxP + 17;  // ..., eig calls, Jacobi sweeps, kcycles[8], subspace ok/fail

// ---------------------------------------------------------------------------
// Workspace layouts (in doubles). The misc tail holds reductions, sigma, order.
constexpr int64_t kMisc = 2048;

struct LeafWs {
  int64_t W, B1, B2, G, V, SI, misc, xch, gpart, total, gram_n;
};
// Cross-CTA exchange slots of the cluster leaf kernel (per-CTA partial sums, stop flag).
constexpr int64_t kXch = 64;

// Subspace-iteration scratch: U/W (rows x k), Y (cols x k), small k x k
// matrices and the unfolding column-offset table.
TT_HD int64_t si_size(int64_t max_rows, int64_t max_cols, int64_t kmax) {
  return 2 * max_rows * kmax + max_cols * kmax + 8 * kmax * kmax + max_cols + 64;
}

// cs > 0: the cluster kernel's per-CTA partial Gram slots (cs x gram_n^2).
TT_HD LeafWs leaf_ws_layout(int p, int64_t len, const int64_t* d, const int64_t* req, int64_t cs = 0) {
  int64_t dd[kMaxP], rc[kMaxP];
  dd[0] = len;
  for (int m = 1; m < p; ++m) dd[m] = d[m];
  clamp_ranks(p, dd, req, rc);
  const int64_t ns = prod_range(dd, 1, p);
  const int64_t sW = rc[0] * ns;
  const int64_t sT = len * rc[1] * prod_range(dd, 2, p);
  const int64_t sB = imax(sT, sW);
  int64_t g = imin(len, prod_range(rc, 1, p));
  for (int n = 1; n < p; ++n) g = imax(g, imin(dd[n], prod_except(rc, p, n)));
  LeafWs w;
  w.gram_n = g;
  w.W = 0;
  w.B1 = w.W + sW;
  w.B2 = w.B1 + sB;
  w.G = w.B2 + sB;
  w.V = w.G + g * g;
  int64_t maxrows = len, kmax = 1;
  for (int m = 0; m < p; ++m) {
    maxrows = imax(maxrows, dd[m]);
    kmax = imax(kmax, rc[m]);
  }
  w.SI = w.V + g * g;
  w.misc = w.SI + si_size(maxrows, g, kmax);
  w.xch = w.misc + kMisc + 4 * g;
  w.gpart = w.xch + kXch;
  w.total = w.gpart + cs * g * g;
  w.total = (w.total + 31) & ~int64_t(31);
  return w;
}

// ---------------------------------------------------------------------------
// Grid-wide leaf path (tt_grid.cu): wide batches of equal-length leaf blocks,
// run as phase kernels over ALL leaves (streamed products split across the
// whole GPU, per-leaf solver kernels in between).
//
// Tile of a streamed product out[o][a][t] = sum_j Ut[j][a] in[o][j][t]: each of
// the 256 consumer threads owns tt consecutive columns t of one slab o and all
// R accumulators; a tile is G slabs x tw columns, streamed in chunks of cj rows.
struct GridTile {
  int64_t tt, tw, tpo, G, cj, ngrp, ntt, njt;
};
constexpr int64_t kGridTileDoubles = 4096;  // X doubles per ring stage (32 KB)
constexpr int64_t kGridCjMax = 16;          // rows of j per stage (bounds the staged U^T rows)
constexpr int64_t kGridRcMax = 10;          // accumulator columns per thread (x tt columns of t)
// gcap bounds the slabs per tile: small batches take fewer slabs per tile so the
// pass has enough work items for every SM.
// ttmax = 2 halves the columns per thread (small batches: twice the active threads).
TT_HD GridTile grid_tile(int64_t outer, int64_t d, int64_t inner, int64_t gcap = 256, int64_t ttmax = 4) {  // requires inner % 2 == 0
  GridTile t;
  t.tt = (inner % 4 == 0 && ttmax >= 4) ? 4 : 2;
  t.tw = imin(inner, 256 * t.tt);
  t.tpo = t.tw / t.tt;
  t.G = imax(1, imin(imin(outer, 256 / t.tpo), gcap));
  t.cj = imax(1, imin(imin(d, kGridTileDoubles / (t.G * t.tw)), kGridCjMax));
  t.ngrp = (outer + t.G - 1) / t.G;
  t.ntt = (inner + t.tw - 1) / t.tw;
  t.njt = (d + t.cj - 1) / t.cj;
  return t;
}
// R accumulator columns are split into nchunk equal chunks of rc columns (even
// when nchunk > 1, so every chunk starts 16-byte aligned); the staged U^T rows
// are zero-padded to rp = nchunk*rc (rounded up to even) columns.
struct GridChunks {
  int nchunk, rc, rp;
};
TT_HD GridChunks grid_chunks(int64_t R) {
  GridChunks c;
  c.nchunk = int((R + kGridRcMax - 1) / kGridRcMax);
  c.rc = int((R + c.nchunk - 1) / c.nchunk);
  if (c.nchunk > 1) c.rc = (c.rc + 1) & ~1;
  c.rp = (c.nchunk * c.rc + 1) & ~1;
  return c;
}
// Extra per-leaf workspace behind leaf_ws_layout(): the row-major, zero-padded
// U_1^T / U_0^T copies the streamed passes read (row stride grid_chunks(R).rp,
// capacity 32 columns), per-tile partial
// sums of ||X||^2, and the leaf's ALS state carried between the phase kernels.
constexpr int64_t kGridUtLd = 32;
enum { kGsNorm = 0, kGsPrevFit = 1, kGsDone = 2, kGsSweeps = 3, kGsConv = 4, kGsZero = 5, kGsK = 8, kGsSize = 16 };
constexpr int64_t kGridGramCtas = 16;  // row chunks (CTAs) of a grid-wide partial Gram per leaf
struct GridWs {
  int64_t ut1, ut0, npart, state, gpart, total;
};
TT_HD GridWs grid_ws_layout(int p, int64_t len, const int64_t* d, const int64_t* req) {
  const LeafWs l = leaf_ws_layout(p, len, d, req);
  const GridTile t = grid_tile(len, d[1], prod_range(d, 2, p), 1, 2);  // most tiles: one slab each, narrow
  GridWs g;
  g.ut1 = l.total;
  g.ut0 = g.ut1 + d[1] * kGridUtLd;
  g.npart = g.ut0 + len * kGridUtLd;
  g.state = g.npart + ((t.ngrp * t.ntt + 1) & ~int64_t(1));
  g.gpart = (g.state + kGsSize + 31) & ~int64_t(31);  // kGridGramCtas partial Grams (gram_n^2 each)
  g.total = (g.gpart + kGridGramCtas * l.gram_n * l.gram_n + 31) & ~int64_t(31);
  return g;
}

struct StitchWs {
  int64_t P, C, S, E, A, G, V, T1, T2, TB1, TB2, Z, WK, HH, SI, misc, xch, gpart, total, gram_n;
  int64_t chain;  // per-part stride of the part-batched mode-product chains (TB1/TB2)
  int64_t per_part_P, per_part_C, per_part_S, per_part_E;
};

// rcx[m] = max(rc[m], max_i rho_im): bound on every intermediate extent. The C, E
// and A regions hold the parts' stacked temporal rows (R = sum rho_i0 <=
// nparts*rcx0 rows; C row-major R x Q, E and A column-major R x k0, ld R).
// cs > 0: the cluster stitch kernel's exchange slots and per-CTA partial Grams.
TT_HD StitchWs stitch_ws_layout(int p, int64_t L, const int64_t* d, const int64_t* req, const int64_t* rho_max,
                                int nparts, int64_t cs = 0) {
  int64_t dd[kMaxP], rc[kMaxP], rcx[kMaxP];
  dd[0] = L;
  for (int m = 1; m < p; ++m) dd[m] = d[m];
  clamp_ranks(p, dd, req, rc);
  for (int m = 0; m < p; ++m) rcx[m] = imax(rc[m], rho_max[m]);
  const int64_t Q = prod_range(rc, 1, p);
  int64_t g = Q;
  for (int n = 1; n < p; ++n) g = imax(g, imin(dd[n], prod_except(rc, p, n)));
  int64_t pp = 0;
  for (int m = 1; m < p; ++m) pp += rc[m] * rcx[m];
  const int64_t chain = prod_range(rcx, 0, p);
  int64_t z = 0;
  for (int n = 1; n < p; ++n) z = imax(z, prod_except(rc, p, n) * dd[n]);
  z = imax(z, int64_t(nparts) * rcx[0] * rc[0]);  // Z doubles as the mode-0 residual scratch
  StitchWs w;
  w.gram_n = g;
  w.per_part_P = pp;
  w.per_part_C = rcx[0] * Q;
  w.per_part_S = rcx[0] * rcx[0];
  w.per_part_E = rcx[0] * rc[0];
  w.P = 0;
  w.C = w.P + nparts * w.per_part_P;
  w.S = w.C + nparts * w.per_part_C;
  w.E = w.S + nparts * w.per_part_S;
  w.A = w.E + nparts * w.per_part_E;
  w.G = w.A + nparts * w.per_part_E;
  w.V = w.G + g * g;
  w.T1 = w.V + g * g;
  w.T2 = w.T1 + chain;
  w.chain = chain;
  w.TB1 = w.T2 + chain;
  w.TB2 = w.TB1 + int64_t(nparts) * chain;
  w.Z = w.TB2 + int64_t(nparts) * chain;
  w.WK = w.Z + z;
  w.HH = w.WK + g * rc[0];
  int64_t maxrows = 1, kmax = 1;
  for (int m = 1; m < p; ++m) maxrows = imax(maxrows, dd[m]);
  for (int m = 0; m < p; ++m) kmax = imax(kmax, rc[m]);
  w.SI = w.HH + rcx[0] * rcx[0];
  w.misc = w.SI + si_size(maxrows, g, kmax);
  w.xch = w.misc + kMisc + 4 * g;
  w.gpart = w.xch + kXch;
  w.total = w.gpart + cs * g * g;
  w.total = (w.total + 31) & ~int64_t(31);
  return w;
}

}  // namespace ttb
