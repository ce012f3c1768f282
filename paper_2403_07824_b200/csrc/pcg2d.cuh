// pcg2d.cuh — kernels (e) and (d), 2-D: IC(0) centroid factors and batched PCG
// on the structured r x r P1 mesh (BASELINE C4: r = 256, 65,025 unknowns).
//
// Replaces, per sample, assemble (proj/src/fem.cpp:213-256) + pcg
// (proj/src/solver.cpp:186-245) with the IC(0) preconditioner of SURVEY
// Appendix A (not in the reference), and, per centroid, the factorisation
// step of run_campaign_with (driver.cpp:212-219).
//
// Storage: every per-node array lives in HBM in anti-diagonal ("wavefront")
// order: level l = ix + iy (0 .. 2m-2, m = r-1), nodes of a level contiguous
// by increasing iy. Thread t of a CTA owns grid row iy = t (T = 256 >= m), so
// at level l it touches node (l - t, t); its W/S neighbours lie in level l-1
// and its E/N neighbours in level l+1, so every access of a warp is one
// coalesced segment.
//
// Exactness: the coefficients are assembled in the oracle's insertion order
// (kbar = ((k_a + k_b) + k_c) / 3, local entries scale * (b_i b_j + c_i c_j),
// the diagonal summed over the node's six triangles in cell order), the CSR
// row products use the reference's column order without contraction, and the
// IC(0) sweeps are level-scheduled: each node performs exactly the sequential
// sweep's operations on exactly the same inputs. Hence A, b, the IC(0) factor,
// A v and M^{-1} r are bit-identical to the CPU oracle; only the dot-product
// summation order differs (block tree vs serial). In exact mode the products
// are stored at their natural index and summed serially by one thread, and the
// whole solve (J, residual history, x) is bit-identical to the reference's
// arithmetic; the tree mode is faster and reproduces the oracle built with
// pairwise dot products.
//
// One CTA per sample (persistent grid, samples in bucket order). Per PCG
// iteration three passes over the levels:
//   P1 (barrier-free): p_new = z + beta p_old (ping-pong halves); A p; pAp
//   P2 (barrier-free): x_new = x_old + alpha p (ping-pong); r -= alpha A p;
//       r_true = b - A x_new with neighbours' x_new recomputed by the same FMA
//   P3 (one barrier per level): forward and backward IC(0) sweeps; r.z
// Ap is recomputed in P2 (bit-identical) instead of stored.
#pragma once
#include "common.cuh"

namespace vqpc {

constexpr int P2_T = 256;            // threads per CTA, one per grid row (r <= 257: two CTAs per SM)
constexpr int P2_TBIG = 512;         // the same kernels with 512 threads, one CTA per SM (257 < r <= 513)
constexpr int P2_FAC = 4;            // factor vectors per centroid: D, aW, aS, RN(1/D)
constexpr int P2_MAXL = 2 * P2_TBIG;  // max levels (2m - 1 <= 1023)

// Order in which the reference's SparseBuilder sums a row's six diagonal
// contributions (fem.cpp:177-211: std::sort by column, then duplicates summed in
// sorted order), per row pattern W | E << 1 | S << 2 | N << 3 of present
// neighbours; entry k = index (in triangle order) of the k-th term. The same for
// every structured mesh; filled once on the host with the same std::sort
// (diag_orders in vqpc.cu).
__constant__ unsigned char vqpc_dperm[16][6];

struct Grid2D {
  int r;       // mesh resolution
  int m;       // interior nodes per row (r - 1)
  int n;       // m * m
  int L;       // levels 2m - 1
  double h;    // 1 / r
};

__host__ __device__ inline int lvl_lo(int l, int m) { return l - (m - 1) > 0 ? l - (m - 1) : 0; }
__host__ __device__ inline int lvl_hi(int l, int m) { return l < m - 1 ? l : m - 1; }

// ---- coefficient assembly for one interior node, oracle insertion order ------
// kappa: nodal, (r+1)^2, natural mesh order id = Y (r+1) + X.
struct RowCoef {
  double d, w, s, e, nn, b;
};

__device__ inline void tri_geom(int X0, int Y0, int X1, int Y1, int X2, int Y2, double h, double& area, double bb[3],
                                double cc[3]) {
  const double x0 = X0 * h, y0 = Y0 * h, x1 = X1 * h, y1 = Y1 * h, x2 = X2 * h, y2 = Y2 * h;
  area = __dmul_rn(0.5, __dsub_rn(__dmul_rn(__dsub_rn(x1, x0), __dsub_rn(y2, y0)),
                                  __dmul_rn(__dsub_rn(x2, x0), __dsub_rn(y1, y0))));
  bb[0] = __dsub_rn(y1, y2);
  bb[1] = __dsub_rn(y2, y0);
  bb[2] = __dsub_rn(y0, y1);
  cc[0] = __dsub_rn(x2, x1);
  cc[1] = __dsub_rn(x0, x2);
  cc[2] = __dsub_rn(x1, x0);
}

// entry (i, j) of triangle with vertices V[0..2] (mesh coords), i,j local vertex ids
__device__ inline double tri_entry(const double* kappa, int side, int X[3], int Y[3], int i, int j, double h,
                                   double* area_out) {
  double area, bb[3], cc[3];
  tri_geom(X[0], Y[0], X[1], Y[1], X[2], Y[2], h, area, bb, cc);
  const double ka = kappa[Y[0] * side + X[0]], kb = kappa[Y[1] * side + X[1]], kc = kappa[Y[2] * side + X[2]];
  const double kbar = __ddiv_rn(__dadd_rn(__dadd_rn(ka, kb), kc), 3.0);
  const double scale = __ddiv_rn(kbar, __dmul_rn(4.0, area));
  if (area_out) *area_out = area;
  return __dmul_rn(scale, __dadd_rn(__dmul_rn(bb[i], bb[j]), __dmul_rn(cc[i], cc[j])));
}

// T1 of cell (cx, cy): {a, b, d}; T2: {a, d, c}; a=(cx,cy) b=(cx+1,cy) c=(cx,cy+1) d=(cx+1,cy+1)
__device__ inline void cell_tri(int cx, int cy, int which, int X[3], int Y[3]) {
  if (which == 1) {
    X[0] = cx; Y[0] = cy; X[1] = cx + 1; Y[1] = cy; X[2] = cx + 1; Y[2] = cy + 1;
  } else {
    X[0] = cx; Y[0] = cy; X[1] = cx + 1; Y[1] = cy + 1; X[2] = cx; Y[2] = cy + 1;
  }
}

// Row of interior node (ix, iy) (mesh node X = ix+1, Y = iy+1): diagonal summed in
// the oracle's triangle order, couplings as the two-triangle sums, b = area_sum / 3.
__device__ inline RowCoef assemble_row(const double* kappa, const Grid2D g, int ix, int iy) {
  const int side = g.r + 1, X = ix + 1, Y = iy + 1;
  int tx[3], ty[3];
  double area, asum, e1, e2, dt[6];  // dt: the six diagonal contributions in triangle order
  // 1) T1(X-1,Y-1): node is d (local 2)
  cell_tri(X - 1, Y - 1, 1, tx, ty);
  dt[0] = tri_entry(kappa, side, tx, ty, 2, 2, g.h, &area);
  asum = area;
  const double s1 = tri_entry(kappa, side, tx, ty, 2, 1, g.h, nullptr);  // S via T1(X-1,Y-1): (d, b)
  // 2) T2(X-1,Y-1): node is d (local 1)
  cell_tri(X - 1, Y - 1, 2, tx, ty);
  dt[1] = tri_entry(kappa, side, tx, ty, 1, 1, g.h, &area);
  asum = __dadd_rn(asum, area);
  const double w1 = tri_entry(kappa, side, tx, ty, 1, 2, g.h, nullptr);  // W via T2(X-1,Y-1): (d, c)
  // 3) T2(X,Y-1): node is c (local 2)
  cell_tri(X, Y - 1, 2, tx, ty);
  dt[2] = tri_entry(kappa, side, tx, ty, 2, 2, g.h, &area);
  asum = __dadd_rn(asum, area);
  const double s2 = tri_entry(kappa, side, tx, ty, 2, 0, g.h, nullptr);  // S via T2(X,Y-1): (c, a)
  e1 = tri_entry(kappa, side, tx, ty, 2, 1, g.h, nullptr);                // E via T2(X,Y-1): (c, d)
  // 4) T1(X-1,Y): node is b (local 1)
  cell_tri(X - 1, Y, 1, tx, ty);
  dt[3] = tri_entry(kappa, side, tx, ty, 1, 1, g.h, &area);
  asum = __dadd_rn(asum, area);
  const double w2 = tri_entry(kappa, side, tx, ty, 1, 0, g.h, nullptr);  // W via T1(X-1,Y): (b, a)
  const double n1 = tri_entry(kappa, side, tx, ty, 1, 2, g.h, nullptr);  // N via T1(X-1,Y): (b, d)
  // 5) T1(X,Y): node is a (local 0)
  cell_tri(X, Y, 1, tx, ty);
  dt[4] = tri_entry(kappa, side, tx, ty, 0, 0, g.h, &area);
  asum = __dadd_rn(asum, area);
  e2 = tri_entry(kappa, side, tx, ty, 0, 1, g.h, nullptr);  // E via T1(X,Y): (a, b)
  // 6) T2(X,Y): node is a (local 0)
  cell_tri(X, Y, 2, tx, ty);
  dt[5] = tri_entry(kappa, side, tx, ty, 0, 0, g.h, &area);
  asum = __dadd_rn(asum, area);
  const double n2 = tri_entry(kappa, side, tx, ty, 0, 2, g.h, nullptr);  // N via T2(X,Y): (a, c)
  // the diagonal in the reference's sorted-duplicate order for this row pattern
  const int pat = (ix > 0 ? 1 : 0) | (ix < g.m - 1 ? 2 : 0) | (iy > 0 ? 4 : 0) | (iy < g.m - 1 ? 8 : 0);
  double diag = dt[vqpc_dperm[pat][0]];
#pragma unroll
  for (int k = 1; k < 6; ++k) diag = __dadd_rn(diag, dt[vqpc_dperm[pat][k]]);
  RowCoef rc;
  rc.d = diag;
  rc.w = ix > 0 ? __dadd_rn(w1, w2) : 0.0;
  rc.s = iy > 0 ? __dadd_rn(s1, s2) : 0.0;
  rc.e = ix < g.m - 1 ? __dadd_rn(e1, e2) : 0.0;
  rc.nn = iy < g.m - 1 ? __dadd_rn(n1, n2) : 0.0;
  rc.b = __ddiv_rn(asum, 3.0);
  return rc;
}

// CSR row product in the reference's column order (S, W, diag, E, N), no contraction
__device__ __forceinline__ double row_apply(double as, double aw, double d, double ae, double an, double vs, double vw,
                                            double v, double ve, double vn) {
  double s = __dmul_rn(as, vs);
  s = __dadd_rn(s, __dmul_rn(aw, vw));
  s = __dadd_rn(s, __dmul_rn(d, v));
  s = __dadd_rn(s, __dmul_rn(ae, ve));
  return __dadd_rn(s, __dmul_rn(an, vn));
}

struct LevelTab {
  int off[P2_MAXL + 2];  // level offsets (off[L] = n)
  int lo[P2_MAXL + 2];   // smallest iy of each level
  int dw[P2_MAXL + 2];   // a - a_W for nodes of level l (a_S = a_W - 1)
  int de[P2_MAXL + 2];   // a_E - a for nodes of level l (a_N = a_E + 1)
};

__device__ inline void build_levels(LevelTab& tab, const Grid2D g) {
  if (threadIdx.x == 0) {
    int off = 0;
    for (int l = 0; l < g.L; ++l) {
      tab.off[l] = off;
      tab.lo[l] = lvl_lo(l, g.m);
      off += lvl_hi(l, g.m) - tab.lo[l] + 1;
    }
    tab.off[g.L] = off;
    tab.lo[g.L] = 0;
    for (int l = 0; l < g.L; ++l) {
      const int size_l = tab.off[l + 1] - tab.off[l];
      tab.dw[l] = l > 0 ? (tab.off[l] - tab.off[l - 1]) + tab.lo[l - 1] - tab.lo[l] : 0;
      tab.de[l] = l + 1 < g.L ? size_l + tab.lo[l] - tab.lo[l + 1] : 0;
    }
  }
  __syncthreads();
}

// address of node (l - t, t) in wavefront order, or -1 if not on level l.
// Closed form (no table lookups on the sweeps' critical path): levels l < m hold
// l + 1 nodes, levels l >= m hold 2m - 1 - l, so off(l) = l(l+1)/2 below m and
// m^2 - r(r+1)/2 with r = 2m - 1 - l above.
__device__ __forceinline__ int wf_addr(const Grid2D g, int l, int t) {
  const int m = g.m;
  if (static_cast<unsigned>(l) >= static_cast<unsigned>(g.L)) return -1;
  int off, lo, hi;
  if (l < m) {
    off = (l * (l + 1)) >> 1;
    lo = 0;
    hi = l;
  } else {
    const int r = 2 * m - 1 - l;
    off = m * m - ((r * (r + 1)) >> 1);
    lo = l - m + 1;
    hi = m - 1;
  }
  return (t >= lo && t <= hi) ? off + t - lo : -1;
}
__device__ __forceinline__ int wf_addr(const LevelTab&, const Grid2D g, int l, int t) { return wf_addr(g, l, t); }

__device__ __forceinline__ int wf_size(int l, int m) { return l < m ? l + 1 : 2 * m - 1 - l; }
// a - a_W for the nodes of level l (a_S = a_W - 1), and a_E - a (a_N = a_E + 1)
__device__ __forceinline__ int wf_dw(int l, int m) { return wf_size(l - 1, m) + lvl_lo(l - 1, m) - lvl_lo(l, m); }
__device__ __forceinline__ int wf_de(int l, int m) { return wf_size(l, m) + lvl_lo(l, m) - lvl_lo(l + 1, m); }

// level of a wavefront address, tracked instead of looked up: {level, its first address, its size}
struct LvlCursor {
  int l, off, sz;
};
__device__ __forceinline__ void lvl_advance(LvlCursor& c, int a, int m) {
  while (a >= c.off + c.sz) {
    c.off += c.sz;
    ++c.l;
    c.sz = wf_size(c.l, m);
  }
}

#ifdef VQPC_PHASE_TIMING
__device__ unsigned long long g_pcg2d_phase[4];  // cycles: setup, sweeps, P1, P2 (CTA thread 0)
#define P2_TIC(v) const long long v = clock64()
#define P2_TOC(i, v) \
  if (threadIdx.x == 0) atomicAdd(&g_pcg2d_phase[i], static_cast<unsigned long long>(clock64() - v))
#else
#define P2_TIC(v)
#define P2_TOC(i, v)
#endif

// Division by a pivot with its correctly rounded reciprocal R = RN(1/D):
// q0 = x R, e = fma(-D, q0, x) (exact), q = fma(e, R, q0) equals RN(x / D)
// (Markstein's theorem; normal range, which the IC(0) pivots and sweep values
// are in). Three dependent FP64 ops instead of the division sequence on the
// sweeps' per-level critical path; exact-mode tests check the bits.
__device__ __forceinline__ double div_by_pivot(double x, double d, double r) {
  const double q0 = __dmul_rn(x, r);
  const double e = __fma_rn(-d, q0, x);
  return __fma_rn(e, r, q0);
}

// ---- (e) IC(0) factor of every centroid matrix (one CTA per centroid) ---------
// fac layout per centroid (P2_FAC n doubles, wavefront order): D, aW, aS of A_c, RN(1/D).
template <int TT>
__global__ void __launch_bounds__(TT) factor2d_kernel(const double* kappa_c, int64_t ldk, int P, const Grid2D g,
                                                         double* fac, int* err) {
  __shared__ LevelTab tab;
  __shared__ double dprev[2][TT + 1];
  build_levels(tab, g);
  const int p = blockIdx.x, t = threadIdx.x;
  if (p >= P) return;
  const double* kap = kappa_c + static_cast<size_t>(p) * ldk;
  double* D = fac + static_cast<size_t>(p) * P2_FAC * g.n;
  double* W = D + g.n;
  double* S = W + g.n;
  double* R = S + g.n;
  for (int k = t; k <= TT; k += blockDim.x) dprev[0][k] = dprev[1][k] = 1.0;
  __syncthreads();
  bool ok = true;
  for (int l = 0; l < g.L; ++l) {
    const int cur = l & 1, prv = cur ^ 1;
    const int a = wf_addr(tab, g, l, t);
    if (a >= 0) {
      const int ix = l - t, iy = t;
      const RowCoef rc = assemble_row(kap, g, ix, iy);
      // oracle: t = a_ii; t -= aW*aW / D_W; t -= aS*aS / D_S
      double v = rc.d;
      if (ix > 0) v = __dsub_rn(v, __ddiv_rn(__dmul_rn(rc.w, rc.w), dprev[prv][t]));
      if (iy > 0) v = __dsub_rn(v, __ddiv_rn(__dmul_rn(rc.s, rc.s), dprev[prv][t - 1]));
      if (!(v > 0.0)) ok = false;
      dprev[cur][t] = v;
      D[a] = v;
      W[a] = rc.w;
      S[a] = rc.s;
      R[a] = __drcp_rn(v);
    }
    __syncthreads();
  }
  if (!ok) atomicExch(err, 1);
}

// ---- (d) batched PCG, one CTA per sample --------------------------------------
struct Pcg2dParams {
  Grid2D g;
  const double* kappa;      // samples x ldk nodal kappa (natural mesh order)
  int64_t ldk;
  const uint8_t* kflag;
  const int32_t* perm;
  const int32_t* labels;
  const double* fac;        // P x 3n (D, aW, aS), wavefront order
  double* work;             // per CTA: P2_WORK n doubles
  int64_t B, out_base, solve_limit;
  double eps;
  int max_iter;
  const int32_t* max_iter_arr;
  int* counter;
  int32_t* iters;
  double* rel;
  uint8_t* status;
  double* x_out;            // nullable, natural interior order
  int exact;                // 1: dot products summed serially in natural order (reference bits)
  const int* gmap;          // per wavefront address: level | (iy << 16)
  const double* bvec;       // per wavefront address: b_i = area_sum_i / 3 when the mesh's b is not
                            // uniform (h = 1/r inexact: every triangle area rounds differently); null:
                            // b is the same for every node (r a power of two, e.g. C4) and read once
};

constexpr int P2_WORK = 11;  // per-CTA scratch vectors: d, w, s, x[2], r, p[2], y, z, prod
#ifndef P2_DEPTH_OVERRIDE
constexpr int P2_DEPTH = 6;
#else
constexpr int P2_DEPTH = P2_DEPTH_OVERRIDE;
#endif  // cp.async prefetch ring depth (levels) for the IC(0) sweeps
constexpr int P2_NOPS = 6;   // operands per node in the ring
// Flat passes (P1, P2) stream the wavefront array in chunks of TT addresses:
// each thread prefetches its own address of chunk k + P2_SD with cp.async into
// a raw slot only it reads, and publishes the vector values its neighbours need
// into 4-slot exchange rings (a node's neighbours lie in chunks k-1..k+1 since a
// level holds <= TT nodes). One barrier per chunk.
#ifndef P2_SD_OVERRIDE
constexpr int P2_SD = 3;       // chunks in flight
#else
constexpr int P2_SD = P2_SD_OVERRIDE;
#endif
constexpr int P2_RSLOT = P2_SD + 1;  // raw slots: the slot refilled in step k is the one read in step k-1
constexpr int P2_RAW = 6;      // raw double vectors per address
constexpr int P2_XCH = 4;      // exchange rings: p (or p_new), x_new, aW, aS; 4 chunk slots each (k-2..k+1 live)
// dynamic shared memory of pcg2d_kernel<MC, TT>: the larger of the sweeps' ring and the flat passes' slots
constexpr size_t p2_dsmem(int tt) {
  const size_t ring = sizeof(double) * P2_DEPTH * P2_NOPS * tt;
  const size_t flat = sizeof(double) * (P2_RSLOT * P2_RAW + 4 * P2_XCH) * tt;
  return ring > flat ? ring : flat;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8s(unsigned sa, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
// same with an L2 eviction-priority policy (createpolicy): the centroid factors
// are shared by every CTA of a bucket and should stay in L2 (evict_last) while
// the per-sample vectors stream through it (evict_first)
__device__ __forceinline__ unsigned long long l2_policy_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async8h(unsigned sa, const void* gmem, unsigned long long pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async8p(void* smem, const void* gmem, unsigned long long pol) {
  cp_async8h(static_cast<unsigned>(__cvta_generic_to_shared(smem)), gmem, pol);
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int NW>
__device__ __forceinline__ double block_sum2d(double v, double* red, int warp, int lane) {
  v = warp_allsum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) s[i] = red[i];
#pragma unroll
  for (int w = 1; w < NW; w <<= 1)
#pragma unroll
    for (int i = 0; i + w < NW; i += 2 * w) s[i] += s[i + w];
  return s[0];
}

// Exact mode: the products were stored at their natural index; one thread sums
// them serially (s = 0; s += t_i for i = 0..n-1), i.e. solver.cpp:176-180's bits.
__device__ __forceinline__ double serial_sum2d(const double* prod, int n, double* slot) {
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll 8
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, prod[i]);
    *slot = s;
  }
  __syncthreads();
  const double v = *slot;
  __syncthreads();
  return v;
}

// MC > 0 compiles the kernel for a fixed interior size m = MC (BASELINE C4: 255):
// every vector offset j*n becomes an immediate and the level arithmetic folds.
template <int MC, int TT>
__global__ void __launch_bounds__(TT, TT == TT ? 2 : 1) pcg2d_kernel(const Pcg2dParams prm) {
  constexpr int NW = TT / 32;
  extern __shared__ __align__(16) double dsm[];
  __shared__ double sbuf[2][TT + 2];  // previous level of the running sweep (index iy + 1)
  __shared__ int2 lvl_dd[2 * TT];         // per level: a - a_W, a_E - a
  __shared__ double red[4][NW];
  __shared__ int64_t s_item;
  __shared__ double s_bval;
  static_assert((TT & (TT - 1)) == 0, "the exchange rings index addresses modulo 4 TT");
  Grid2D g = prm.g;
  if constexpr (MC > 0) {
    g.m = MC;
    g.n = MC * MC;
    g.L = 2 * MC - 1;
  }
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int l = t; l < g.L; l += TT) lvl_dd[l] = make_int2(l > 0 ? wf_dw(l, g.m) : 0, l + 1 < g.L ? wf_de(l, g.m) : 0);
  LvlCursor lc0{0, 0, 1};  // level of wavefront address t (the first chunk of the flat passes)
  if (t < g.n) lvl_advance(lc0, t, g.m);
  __syncthreads();
  const int n = g.n;
  double* base = prm.work + static_cast<size_t>(blockIdx.x) * P2_WORK * n;
  double* Ad = base;          // diagonal
  double* Aw = base + n;      // W coupling (the E coupling of node i is Aw[E])
  double* As = base + 2 * n;  // S coupling (the N coupling of node i is As[N])
  double* Xb[2] = {base + 3 * n, base + 4 * n};
  double* Rv = base + 5 * n;
  double* Pb[2] = {base + 6 * n, base + 7 * n};
  double* Y = base + 8 * n;
  double* Z = base + 9 * n;
  double* Prod = base + 10 * n;  // exact mode: products at natural index iy*m + ix
  const bool exact = prm.exact != 0;
  // reduce a thread partial (fast) or the stored products (exact)
  auto reduce = [&](double part, double* red_slot) {
    return exact ? serial_sum2d(Prod, n, red_slot) : block_sum2d<NW>(part, red_slot, warp, lane);
  };
  auto nat = [&](int l) { return t * g.m + (l - t); };

  for (;;) {
    if (t == 0) s_item = atomicAdd(prm.counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    __syncthreads();
    if (item >= prm.B) break;
    const int s = prm.perm[item];
    const int64_t gs = prm.out_base + s;
    const int label = prm.labels[s];
    if (label < 0 || prm.kflag[s] || gs >= prm.solve_limit) {
      if (t == 0) {
        prm.iters[gs] = 0;
        prm.rel[gs] = 0.0;
        prm.status[gs] = gs >= prm.solve_limit ? VQPC_S_NOT_SOLVED
                         : label < 0           ? VQPC_S_INVALID_LATENT
                                               : (prm.kflag[s] & 1) ? VQPC_S_COEFF_OVERFLOW : VQPC_S_INVALID_COEFF;
      }
      continue;
    }
    const double* kap = prm.kappa + static_cast<size_t>(s) * prm.ldk;
    const double* FD = prm.fac + static_cast<size_t>(label) * P2_FAC * n;
    const double* FW = FD + n;
    const double* FS = FW + n;
    const double* FR = FS + n;
    int xc = 0, pc = 0;  // current ping-pong halves

    // ---- setup: assemble the sample's rows, x = 0, r = b ----------------------
    double bb_loc = 0.0;
    for (int l = 0; l < g.L; ++l) {
      const int a = wf_addr(g, l, t);
      if (a >= 0) {
        const RowCoef rc = assemble_row(kap, g, l - t, t);
        Ad[a] = rc.d;
        Aw[a] = rc.w;
        As[a] = rc.s;
        Xb[0][a] = 0.0;
        Rv[a] = rc.b;
        if (t == 0 && l == 0) s_bval = rc.b;  // b_i = area_sum / 3: uniform unless prm.bvec is set
        bb_loc = fma(rc.b, rc.b, bb_loc);
        if (exact) Prod[nat(l)] = __dmul_rn(rc.b, rc.b);
      }
    }
    __syncthreads();
    // the flat passes below touch nodes of every thread, so b comes from one shared copy
    const double bval = s_bval;
    const int max_iter = prm.max_iter_arr ? prm.max_iter_arr[gs] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);

    // z = M^{-1} r by the level-scheduled IC(0) sweeps (oracle arithmetic); returns the r.z partial.
    // Each thread prefetches ITS OWN node's operands P2_DEPTH-1 levels ahead with
    // cp.async into a shared-memory ring (no registers held; a thread only reads
    // what it copied, so the ring needs no barrier), hiding the HBM latency that
    // otherwise stalls every one of the 2 x (2m-1) dependent levels.
    double (*ring)[P2_NOPS][TT] = reinterpret_cast<double (*)[P2_NOPS][TT]>(dsm);
    // Per-thread address cursors (no per-level table lookups): lin(l) is the
    // wavefront address of row t on level l (linear in t, valid or not), up(l) =
    // lin(l+1) - lin(l); row t has a node on level l iff 0 <= l - t < m.
    const int m = g.m;
    const bool trow = t < m;
    auto lin = [&](int l) {
      if (l < m) return ((l * (l + 1)) >> 1) + t;
      const int r = 2 * m - 1 - l;
      return m * m - ((r * (r + 1)) >> 1) + t - (l - m + 1);
    };
    auto up = [&](int l) { return l < m - 1 ? l + 1 : 2 * m - 2 - l; };
    auto on = [&](int l) { return trow && static_cast<unsigned>(l - t) < static_cast<unsigned>(m); };
    // ring slots as 32-bit shared addresses; slot counters instead of l % depth
    const unsigned ring_sa = static_cast<unsigned>(__cvta_generic_to_shared(dsm)) + t * 8u;
    const unsigned long long pol_fac = l2_policy_last();
    constexpr unsigned OPB = TT * 8u, SLOTB = P2_NOPS * TT * 8u;
    auto next_slot = [](int sl) { return sl + 1 == P2_DEPTH ? 0 : sl + 1; };
    auto fwd_issue = [&](int l, int a, int sl) {
      if (on(l)) {
        const unsigned r0 = ring_sa + sl * SLOTB;
        cp_async8s(r0, Rv + a);
        cp_async8h(r0 + OPB, FW + a, pol_fac);
        cp_async8h(r0 + 2 * OPB, FS + a, pol_fac);
        cp_async8h(r0 + 3 * OPB, FD + a, pol_fac);
        cp_async8h(r0 + 4 * OPB, FR + a, pol_fac);
      }
      cp_commit();
    };
    auto bwd_issue = [&](int l, int a, int sl) {
      if (l >= 0 && on(l)) {
        const unsigned r0 = ring_sa + sl * SLOTB;
        const int ae = a + up(l);  // (ix+1, iy) on level l+1; (ix, iy+1) is the next address
        if (l - t < m - 1) cp_async8h(r0, FW + ae, pol_fac);
        if (t < m - 1) cp_async8h(r0 + OPB, FS + ae + 1, pol_fac);
        cp_async8h(r0 + 2 * OPB, FD + a, pol_fac);
        cp_async8s(r0 + 3 * OPB, Y + a);
        cp_async8s(r0 + 4 * OPB, Rv + a);
        cp_async8h(r0 + 5 * OPB, FR + a, pol_fac);
      }
      cp_commit();
    };
    auto sweeps = [&]() -> double {
      // forward (D + L) y = r, ascending levels; level l lives in ring slot l % depth
      __syncthreads();
      int ai = lin(0), ac = ai;  // issue / compute cursors
      int si = 0, sc = 0;        // issue / compute slots
      for (int l = 0; l < P2_DEPTH - 1; ++l) {
        fwd_issue(l, ai, si);
        ai += up(l);
        si = next_slot(si);
      }
      for (int l = 0; l < g.L; ++l) {
        fwd_issue(l + P2_DEPTH - 1, ai, si);  // slot of level l-1, already consumed
        ai += up(l + P2_DEPTH - 1);
        si = next_slot(si);
        cp_wait<P2_DEPTH - 1>();
        const int cur = l & 1, prv = cur ^ 1;
        if (on(l)) {
          const double* op = &ring[sc][0][t];
          double v = op[0];
          if (l - t > 0) v = __dsub_rn(v, __dmul_rn(op[TT], sbuf[prv][t + 1]));
          if (t > 0) v = __dsub_rn(v, __dmul_rn(op[2 * TT], sbuf[prv][t]));
          v = div_by_pivot(v, op[3 * TT], op[4 * TT]);
          VQPC_DCHECK(ac >= 0 && ac < n);
          Y[ac] = v;
          sbuf[cur][t + 1] = v;
        }
        ac += up(l);
        sc = next_slot(sc);
        __syncthreads();
      }
      cp_wait<0>();
      __syncthreads();  // Y complete before the backward prefetch reads it
      // backward (D + L^T) z = D y, descending levels: z_i = y_i - (aE z_E + aN z_N) / D_i;
      // level l lives in ring slot (L - 1 - l) % depth
      double rz_part = 0.0;
      ai = lin(g.L - 1);
      ac = ai;
      si = sc = 0;
      for (int l = g.L - 1; l > g.L - P2_DEPTH; --l) {
        bwd_issue(l, ai, si);
        ai -= up(l - 1);
        si = next_slot(si);
      }
      for (int l = g.L - 1; l >= 0; --l) {
        bwd_issue(l - (P2_DEPTH - 1), ai, si);
        ai -= up(l - P2_DEPTH);
        si = next_slot(si);
        cp_wait<P2_DEPTH - 1>();
        const int cur = l & 1, prv = cur ^ 1;
        if (on(l)) {
          const double* op = &ring[sc][0][t];
          double acc = 0.0;
          if (l - t < m - 1) acc = __dadd_rn(acc, __dmul_rn(op[0], sbuf[prv][t + 1]));
          if (t < m - 1) acc = __dadd_rn(acc, __dmul_rn(op[TT], sbuf[prv][t + 2]));
          const double z = __dsub_rn(op[3 * TT], div_by_pivot(acc, op[2 * TT], op[5 * TT]));
          VQPC_DCHECK(ac >= 0 && ac < n);
          Z[ac] = z;
          sbuf[cur][t + 1] = z;
          rz_part = fma(op[4 * TT], z, rz_part);
          if (exact) Prod[t * m + (l - t)] = __dmul_rn(op[4 * TT], z);
        }
        ac -= up(l - 1);
        sc = next_slot(sc);
        __syncthreads();
      }
      cp_wait<0>();
      return rz_part;
    };

    // norm_b first: in exact mode Prod holds b_i^2 until the sweeps overwrite it
    const double norm_b = sqrt(reduce(bb_loc, red[3]));
    double rz = reduce(sweeps(), red[2]);
    int J = 0;
    double rel_rec = 0.0;
    uint8_t st = VQPC_S_MAX_ITER;
    if (norm_b == 0.0) st = VQPC_S_CONVERGED;
    else if (!(rz > 0.0)) st = VQPC_S_BREAKDOWN;
    else {
      double beta = 0.0;
      for (int j = 1; j <= max_iter; ++j) {
        // ---- P1: p_new = z + beta p_old into the other half; pAp (chunk-streamed) ----
        P2_TIC(t_p1);
        const double* Po = Pb[pc];
        double* Pn = Pb[pc ^ 1];
        const bool first = j == 1;
        const int NC = (n + TT - 1) / TT;
        double* raw = dsm;                                   // [P2_RSLOT][P2_RAW][TT]
        double* xch = dsm + P2_RSLOT * P2_RAW * TT;        // [P2_XCH][4][TT]
        auto RAW = [&](int k, int v) -> double* { return raw + ((static_cast<unsigned>(k) % P2_RSLOT) * P2_RAW + v) * TT + t; };
        // chunk slot (q >> 8) & 3, column q & 255: together q & 1023
        auto XCH = [&](int x, int q) -> double& { return xch[x * 4 * TT + (q & (4 * TT - 1))]; };
        const unsigned long long pol_str = l2_policy_first();
        auto flat_issue = [&](int k, const double* v0, const double* v1, const double* v2) {
          const int a = k * TT + t;
          if (k < NC && a < n) {
            if (v0) cp_async8p(RAW(k, 0), v0 + a, pol_str);
            if (v1) cp_async8p(RAW(k, 1), v1 + a, pol_str);
            if (v2) cp_async8p(RAW(k, 2), v2 + a, pol_str);
            cp_async8p(RAW(k, 3), As + a, pol_str);
            cp_async8p(RAW(k, 4), Aw + a, pol_str);
            cp_async8p(RAW(k, 5), Ad + a, pol_str);
          }
          cp_commit();
        };
        // neighbour addresses of wavefront address a (level l, row iy); -1 off the mesh. The
        // level of a thread's address is tracked by a cursor {level, its offset, its size} that
        // advances with the address (one or two levels per chunk away from the corners), so the
        // flat passes read no per-address map.
        struct Nb { int s, w, e, nn, ix, iy; };
        auto nbrs = [&](int a, const LvlCursor& c) {
          const int l = c.l, iy = lvl_lo(l, g.m) + (a - c.off), ix = l - iy;
          Nb b;
          const int2 dd = lvl_dd[l];
          const int dw = dd.x, de = dd.y;
          b.w = ix > 0 ? a - dw : -1;
          b.s = iy > 0 ? a - dw - 1 : -1;
          b.e = ix < g.m - 1 ? a + de : -1;
          b.nn = iy < g.m - 1 ? a + de + 1 : -1;
          b.ix = ix;
          b.iy = iy;
          return b;
        };
        auto xv = [&](int x, int q) { return q < 0 ? 0.0 : XCH(x, q); };
        double pap = 0.0;
        {
          for (int k = 0; k < P2_SD; ++k) flat_issue(k, Z, first ? nullptr : Po, nullptr);
          double cs = 0.0, cw = 0.0, cd = 0.0;
          LvlCursor lc = lc0;  // level of address (k - 1) TT + t
          for (int k = 0; k <= NC; ++k) {
            const double ps = cs, pw = cw, pd = cd;
            if (k < NC) {
              cp_wait<P2_SD - 1>();
              const int a = k * TT + t;
              if (a < n) {
                const double z = *RAW(k, 0);
                const double pcv = first ? z : __dadd_rn(z, __dmul_rn(beta, *RAW(k, 1)));
                cs = *RAW(k, 3);
                cw = *RAW(k, 4);
                cd = *RAW(k, 5);
                XCH(0, a) = pcv;
                XCH(2, a) = cw;
                XCH(3, a) = cs;
                Pn[a] = pcv;
              }
            }
            flat_issue(k + P2_SD, Z, first ? nullptr : Po, nullptr);
            __syncthreads();
            const int a = (k - 1) * TT + t;
            if (k >= 1 && a < n) {
              lvl_advance(lc, a, g.m);
              const Nb b = nbrs(a, lc);
              const double pcv = XCH(0, a);
              const double ap = row_apply(ps, pw, pd, xv(2, b.e), xv(3, b.nn), xv(0, b.s), xv(0, b.w), pcv,
                                          xv(0, b.e), xv(0, b.nn));
              pap = fma(pcv, ap, pap);
              if (exact) Prod[b.iy * g.m + b.ix] = __dmul_rn(pcv, ap);
            }
          }
        }
        pc ^= 1;
        const double pAp = reduce(pap, red[0]);
        P2_TOC(2, t_p1);
        if (!(pAp > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        const double alpha = rz / pAp;
        // ---- P2: x_new = x + alpha p, r -= alpha A p, |b - A x_new|^2 (chunk-streamed) --
        P2_TIC(t_p2);
        // every x_new is recomputed with the operation its owner uses (bit-identical);
        // updates follow solver.cpp:216-218/241 without contraction
        const double* Pv = Pb[pc];
        const double* Xo = Xb[xc];
        double* Xn = Xb[xc ^ 1];
        double rr = 0.0;
        {
          for (int k = 0; k < P2_SD; ++k) flat_issue(k, Pv, Xo, Rv);
          double cs = 0.0, cw = 0.0, cd = 0.0, cr = 0.0;
          LvlCursor lc = lc0;  // level of address (k - 1) TT + t
          double cb = bval;  // b of this thread's address in the chunk being loaded
          for (int k = 0; k <= NC; ++k) {
            const double ps = cs, pw = cw, pd = cd, pr = cr, pb = cb;
            if (k < NC) {
              cp_wait<P2_SD - 1>();
              const int a = k * TT + t;
              if (a < n) {
                if (prm.bvec) cb = __ldg(prm.bvec + a);  // consumed one chunk later (latency hidden)
                const double pvv = *RAW(k, 0);
                const double xn = __dadd_rn(*RAW(k, 1), __dmul_rn(alpha, pvv));
                cr = *RAW(k, 2);
                cs = *RAW(k, 3);
                cw = *RAW(k, 4);
                cd = *RAW(k, 5);
                XCH(0, a) = pvv;
                XCH(1, a) = xn;
                XCH(2, a) = cw;
                XCH(3, a) = cs;
                Xn[a] = xn;
              }
            }
            flat_issue(k + P2_SD, Pv, Xo, Rv);
            __syncthreads();
            const int a = (k - 1) * TT + t;
            if (k >= 1 && a < n) {
              lvl_advance(lc, a, g.m);
              const Nb b = nbrs(a, lc);
              const double aE = xv(2, b.e), aN = xv(3, b.nn);
              const double ap = row_apply(ps, pw, pd, aE, aN, xv(0, b.s), xv(0, b.w), XCH(0, a), xv(0, b.e),
                                          xv(0, b.nn));
              const double ax = row_apply(ps, pw, pd, aE, aN, xv(1, b.s), xv(1, b.w), XCH(1, a), xv(1, b.e),
                                          xv(1, b.nn));
              const double rt = __dsub_rn(pb, ax);
              rr = fma(rt, rt, rr);
              if (exact) Prod[b.iy * g.m + b.ix] = __dmul_rn(rt, rt);
              Rv[a] = __dsub_rn(pr, __dmul_rn(alpha, ap));
            }
          }
        }
        xc ^= 1;
        const double rel = sqrt(reduce(rr, red[1])) / norm_b;
        P2_TOC(3, t_p2);
        J = j;
        rel_rec = rel;
        if (rel < prm.eps) {
          st = VQPC_S_CONVERGED;
          break;
        }
        // ---- P3: z = M^{-1} r; r.z (level-ordered sweeps) ---------------------------
        P2_TIC(t_sw);
        const double rz_next = reduce(sweeps(), red[2]);
        P2_TOC(1, t_sw);
        if (!(rz_next > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        beta = rz_next / rz;
        rz = rz_next;
      }
    }
    if (t == 0) {
      prm.iters[gs] = J;
      prm.rel[gs] = rel_rec;
      prm.status[gs] = st;
    }
    if (prm.x_out) {
      double* xo = prm.x_out + static_cast<size_t>(gs) * n;
      for (int l = 0; l < g.L; ++l) {
        const int a = wf_addr(g, l, t);
        if (a >= 0) xo[t * g.m + (l - t)] = Xb[xc][a];
      }
    }
    __syncthreads();
  }
}

// per wavefront address: level | (iy << 16) (shared by every sample of the grid)
__global__ void __launch_bounds__(P2_T) build_gmap_kernel(const Grid2D g, int* gmap) {
  __shared__ LevelTab tab;
  build_levels(tab, g);
  for (int l = blockIdx.x; l < g.L; l += gridDim.x) {
    const int lo = tab.lo[l], hi = lvl_hi(l, g.m);
    for (int iy = lo + threadIdx.x; iy <= hi; iy += blockDim.x) gmap[tab.off[l] + iy - lo] = l | (iy << 16);
  }
}

// per wavefront address: b_i = area_sum_i / 3 with the assembly's own operations
// (assemble_row; kappa does not enter b). Used when the mesh's b is not uniform.
__global__ void __launch_bounds__(P2_T) build_bvec_kernel(const Grid2D g, const double* kappa_any, const int* gmap,
                                                          double* bvec) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < g.n; a += gridDim.x * blockDim.x) {
    const int lv = gmap[a], l = lv & 0xffff, iy = lv >> 16;
    bvec[a] = assemble_row(kappa_any, g, l - iy, iy).b;
  }
}

// natural-order IC(0) apply for one vector (parity tests), single CTA
template <int TT>
__global__ void __launch_bounds__(TT) precond2d_apply_kernel(const double* fac, int p, const Grid2D g,
                                                                const double* r_nat, double* z_nat, double* ws) {
  __shared__ LevelTab tab;
  __shared__ double sbuf[2][TT + 2];
  build_levels(tab, g);
  const int t = threadIdx.x, n = g.n;
  const double* FD = fac + static_cast<size_t>(p) * P2_FAC * n;
  const double* FW = FD + n;
  const double* FS = FW + n;
  double* Y = ws;
  sbuf[0][t + 1] = sbuf[1][t + 1] = 0.0;
  if (t == 0) sbuf[0][0] = sbuf[1][0] = sbuf[0][TT + 1] = sbuf[1][TT + 1] = 0.0;
  __syncthreads();
  for (int l = 0; l < g.L; ++l) {
    const int cur = l & 1, prv = cur ^ 1;
    const int a = wf_addr(tab, g, l, t);
    if (a >= 0) {
      const int ix = l - t;
      double v = r_nat[t * g.m + ix];
      if (ix > 0) v = __dsub_rn(v, __dmul_rn(FW[a], sbuf[prv][t + 1]));
      if (t > 0) v = __dsub_rn(v, __dmul_rn(FS[a], sbuf[prv][t]));
      v = __ddiv_rn(v, FD[a]);
      Y[a] = v;
      sbuf[cur][t + 1] = v;
    }
    __syncthreads();
  }
  sbuf[0][t + 1] = sbuf[1][t + 1] = 0.0;
  __syncthreads();
  for (int l = g.L - 1; l >= 0; --l) {
    const int cur = l & 1, prv = cur ^ 1;
    const int a = wf_addr(tab, g, l, t);
    if (a >= 0) {
      const int ix = l - t;
      double acc = 0.0;
      if (ix < g.m - 1) acc = __dadd_rn(acc, __dmul_rn(FW[wf_addr(tab, g, l + 1, t)], sbuf[prv][t + 1]));
      if (t < g.m - 1) acc = __dadd_rn(acc, __dmul_rn(FS[wf_addr(tab, g, l + 1, t + 1)], sbuf[prv][t + 2]));
      const double z = __dsub_rn(Y[a], __ddiv_rn(acc, FD[a]));
      z_nat[t * g.m + ix] = z;
      sbuf[cur][t + 1] = z;
    }
    __syncthreads();
  }
}

}  // namespace vqpc
