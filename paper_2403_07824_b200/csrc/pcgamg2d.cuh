// pcgamg2d.cuh — kernel (d) with the reference's DEFAULT preconditioner kind:
// smoothed-aggregation AMG applied as one symmetric V-cycle per PCG iteration
// (AmgPreconditioner::apply / cycle, proj/src/amg.cpp:199-225; PrecondKind::Amg
// is the default at proj/include/vqp/driver.hpp:36), on the structured 2-D mesh.
//
// One CTA per sample (persistent grid over the bucket-ordered queue, so CTAs
// that run at the same time mostly share a label and its hierarchy stays hot in
// L2). The sample's operator is assembled from its nodal kappa with the
// oracle's operations (assemble_row, pcg2d.cuh) and applied matrix-free in the
// reference's CSR column order; the centroid's hierarchy (built on the host by
// amg_setup.cuh, packed as sliced ELL: 32-row slices, entries column-major
// within a slice, -1 padding) drives the V-cycle. Every vector lives in HBM in
// natural interior order, so the serial (reference-order) dot products of the
// exact mode need no reordering.
//
// Exactness: each row of every V-cycle operation is one serial chain in the
// order the reference's Eigen expressions evaluate it (amg_setup.cuh header);
// rows are independent, so the V-cycle is bit-identical to the oracle's. PCG
// arithmetic is solver.cpp:186-245's without contraction; only the dot
// products' summation order differs in the fast mode (block tree), and the
// exact mode sums stored products serially (bit-identical solve).
#pragma once
#include "common.cuh"
#include "pcg2d.cuh"
#include "pcgchol2d.cuh"

namespace vqpc {

constexpr int AMG_T = 256;          // threads per CTA
constexpr int AMG_MAXLEV = 16;      // hierarchy depth handled on the device
constexpr int AMG_MAXDENSE = 1024;  // coarsest dense solve size (shared-memory vector)
#ifndef AMG_ROWU
#define AMG_ROWU 1                   // rows per thread interleaved in the V-cycle passes (A/B builds)
#endif
constexpr int kAmgRowU = AMG_ROWU;
#ifndef AMG_PF
#define AMG_PF 1                     // rows ahead (in units of AMG_T) the streamed level-0 operands are prefetched into L2 (0: off;
                                     // 1: 1.10x, 2: 1.08x, 3: 1.08x on 2,664 C4amg samples, profiles/r02q_*)
#endif
constexpr int kAmgPf = AMG_PF;
#ifdef AMG_PF_L1
__device__ __forceinline__ void amg_prefetch(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
#else
__device__ __forceinline__ void amg_prefetch(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
#endif
#ifndef AMG_ELLU
#define AMG_ELLU 4                   // entries of an ELL row whose loads issue together (A and P^T rows; A/B builds)
#endif
constexpr int kAmgEllU = AMG_ELLU;
#ifndef AMG_PCGU
#define AMG_PCGU 1                   // rows per thread interleaved in the two PCG passes (A/B builds)
#endif
constexpr int kAmgPcgU = AMG_PCGU;
#ifndef AMG_MINB
#define AMG_MINB 3                   // resident CTAs per SM the register budget targets (3: +12 % over 2, r02f A/B)
#endif

// Sliced ELL: rows in slices of 32; slice s holds width_s entries per row, entry k of
// row i at e0_i + 32 k for k < len_i, with row[i] = {e0_i, len_i} (e0_i = the slice's
// offset + (i & 31)). An entry is one 16-byte record {value, column (low 32 bits of the
// second word)}: one load per entry instead of a column and a value load, and one
// 8-byte load per row for its offset and length. The row loops run to len_i with no exit
// that depends on a loaded column, so the unrolled iterations' loads issue together,
// and every loop fetches the next row's {e0, len} while it works on the current row.
struct AmgEll {
  const int2* row;          // per row: first record, stored entries
  const double2* rec;       // records {val, col}
  int rows, cols;           // shape (bounds checks of the check build)
};
__device__ __forceinline__ int ell_col(const double2& rc) { return __double2loint(rc.y); }

struct AmgLevelD {
  int n, nc;                // rows; rows of the next level (0 on the coarsest)
  AmgEll A, P, Pt;
  const double* inv_diag;
  int voff;                 // levels >= 1: offset of (r, x, o) in the per-CTA coarse scratch
  // level 0 of a structured mesh: the centroid matrix as its stencil (S, W, diagonal per
  // row; row i's E / N couplings are the W of i + 1 / the S of i + m, bitwise equal), so
  // the two level-0 A passes stream instead of gathering through the ELL columns. The
  // reference's stored SW / NE zeros are skipped: r_i - (+-0) and a sum started at +0
  // plus (+-0) are unchanged (the V-cycle's r is never -0), so the bits are the ELL path's.
  const double *st_s, *st_w, *st_c;
  int st_m;
};

struct AmgHierD {
  int nlev, dense_n;
  const double* L;          // dense_n x dense_n row-major lower factor of the coarsest operator
  AmgLevelD lv[AMG_MAXLEV];
};

__device__ __forceinline__ int2 ell_row(const AmgEll& M, int i) {
  VQPC_DCHECK(i >= 0 && i < M.rows);
  return __ldg(M.row + i);
}

// ---- one V-cycle z = M^{-1} r for S right-hand sides on hierarchy H ---------------
// (amg.cpp:210-225), block-wide. Vectors hold the S slots interleaved per row
// (v[i * S + s]): every ELL entry of the centroid's hierarchy is loaded once and
// applied to S samples, and each gather of a neighbour row brings all S slots in
// one sector. Level 0: r0 (input), x0 / res0 scratch, z (output); levels >= 1 in cv.
// rz[s] accumulates this thread's r.z partial of slot s (fast mode); in exact mode
// the products are stored at prod[s * n0 + i].
template <int S>
__device__ void amg_vcycle(const AmgHierD& H, double omega, const double* r0, double* x0, double* res0, double* z,
                           double* cv, double* sdense, bool exact, double* prod, double (&rz)[S]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  auto vr = [&](int l) -> double* { return l == 0 ? const_cast<double*>(r0) : cv + static_cast<size_t>(H.lv[l].voff) * S; };
  auto vx = [&](int l) -> double* { return l == 0 ? x0 : cv + (static_cast<size_t>(H.lv[l].voff) + H.lv[l].n) * S; };
  auto vo = [&](int l) -> double* { return l == 0 ? res0 : cv + (static_cast<size_t>(H.lv[l].voff) + 2 * H.lv[l].n) * S; };
  const int last = H.nlev - 1;
  const int n0 = H.lv[0].n;
#pragma unroll
  for (int s = 0; s < S; ++s) rz[s] = 0.0;
  // ---- down: pre-smooth from zero, residual, restriction -------------------------
  for (int l = 0; l < last; ++l) {
    const AmgLevelD L = H.lv[l];
    const double* __restrict__ r = vr(l);
    double* __restrict__ x = vx(l);
    double* __restrict__ res = vo(l);  // the residual; later this level's output
    int2 rw_n = make_int2(0, 0);
    if (!L.st_c && t < L.n) rw_n = ell_row(L.A, t);
#pragma unroll kAmgRowU
    for (int i = t; i < L.n; i += AMG_T) {
      const int2 rw = rw_n;
      if (!L.st_c && i + AMG_T < L.n) rw_n = ell_row(L.A, i + AMG_T);
      const double di = __ldg(L.inv_diag + i);
      double acc[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        acc[s] = r[i * S + s];
        x[i * S + s] = __dmul_rn(omega, __dmul_rn(di, acc[s]));
      }
      // res = r; res -= A x (Eigen's rewrite of `r - A x`), x_c recomputed with its owner's operations
      if (L.st_c) {  // level 0, structured: CSR column order S, W, C, E, N
        if (kAmgPf > 0 && i + kAmgPf * AMG_T < L.n) {
          const int ip = i + kAmgPf * AMG_T;
          amg_prefetch(r + static_cast<size_t>(ip) * S);
          amg_prefetch(L.inv_diag + ip);
          amg_prefetch(L.st_s + ip);
          amg_prefetch(L.st_w + ip);
          amg_prefetch(L.st_c + ip);
        }
        const int m = L.st_m, ix = i % m, iy = i / m;
        auto sub = [&](double a, int c) {
          const double dc = __ldg(L.inv_diag + c);
#pragma unroll
          for (int s = 0; s < S; ++s)
            acc[s] = __dsub_rn(acc[s], __dmul_rn(a, __dmul_rn(omega, __dmul_rn(dc, r[c * S + s]))));
        };
        if (iy > 0) sub(__ldg(L.st_s + i), i - m);
        if (ix > 0) sub(__ldg(L.st_w + i), i - 1);
        sub(__ldg(L.st_c + i), i);
        if (ix < m - 1) sub(__ldg(L.st_w + i + 1), i + 1);
        if (iy < m - 1) sub(__ldg(L.st_s + i + m), i + m);
      } else {
      const int w = rw.y;
      int e = rw.x;
      #pragma unroll kAmgEllU
      for (int k = 0; k < w; ++k, e += 32) {
        const double2 rc = __ldg(L.A.rec + e);
        const int c = ell_col(rc);
        VQPC_DCHECK(c >= 0 && c < L.A.cols);
        const double a = rc.x, dc = __ldg(L.inv_diag + c);
#pragma unroll
        for (int s = 0; s < S; ++s)
          acc[s] = __dsub_rn(acc[s], __dmul_rn(a, __dmul_rn(omega, __dmul_rn(dc, r[c * S + s]))));
      }
      }
#pragma unroll
      for (int s = 0; s < S; ++s) res[i * S + s] = acc[s];
    }
    __syncthreads();
    double* __restrict__ rn = vr(l + 1);
    const double* __restrict__ rs = res;
    rw_n = t < L.nc ? ell_row(L.Pt, t) : make_int2(0, 0);
#pragma unroll kAmgRowU
    for (int c = t; c < L.nc; c += AMG_T) {  // P^T residual: 0 + sum, ascending fine rows
      const int2 rw = rw_n;
      if (c + AMG_T < L.nc) rw_n = ell_row(L.Pt, c + AMG_T);
      double acc[S];
#pragma unroll
      for (int s = 0; s < S; ++s) acc[s] = 0.0;
      const int w = rw.y;
      int e = rw.x;
      #pragma unroll kAmgEllU
      for (int k = 0; k < w; ++k, e += 32) {
        const double2 rc = __ldg(L.Pt.rec + e);
        const int q = ell_col(rc);
        VQPC_DCHECK(q >= 0 && q < L.Pt.cols);
        const double v = rc.x;
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] = __dadd_rn(acc[s], __dmul_rn(v, rs[q * S + s]));
      }
#pragma unroll
      for (int s = 0; s < S; ++s) rn[c * S + s] = acc[s];
    }
    __syncthreads();
  }
  // ---- coarsest ----------------------------------------------------------------
  {
    const AmgLevelD L = H.lv[last];
    const double* r = vr(last);
    double* o = last == 0 ? z : vo(last);
    if (H.dense_n > 0) {
      const int nc = H.dense_n;
      VQPC_DCHECK(nc == L.n && nc <= AMG_MAXDENSE);
      if (warp == 0) {  // column-oriented substitutions, S right-hand sides, rows dealt to lanes
        for (int q = lane; q < nc * S; q += 32) sdense[q] = r[q];
        __syncwarp();
        for (int k = 0; k < nc; ++k) {  // L y = r
          const double lkk = __ldg(H.L + static_cast<size_t>(k) * nc + k);
          if (lane < S) sdense[k * S + lane] = __ddiv_rn(sdense[k * S + lane], lkk);
          __syncwarp();
          double yk[S];
#pragma unroll
          for (int s = 0; s < S; ++s) yk[s] = sdense[k * S + s];
          for (int i = k + 1 + lane; i < nc; i += 32) {
            const double lik = __ldg(H.L + static_cast<size_t>(i) * nc + k);
#pragma unroll
            for (int s = 0; s < S; ++s) sdense[i * S + s] = __dsub_rn(sdense[i * S + s], __dmul_rn(lik, yk[s]));
          }
          __syncwarp();
        }
        for (int k = nc - 1; k >= 0; --k) {  // L^T x = y
          const double lkk = __ldg(H.L + static_cast<size_t>(k) * nc + k);
          if (lane < S) sdense[k * S + lane] = __ddiv_rn(sdense[k * S + lane], lkk);
          __syncwarp();
          double xk[S];
#pragma unroll
          for (int s = 0; s < S; ++s) xk[s] = sdense[k * S + s];
          for (int i = lane; i < k; i += 32) {
            const double lki = __ldg(H.L + static_cast<size_t>(k) * nc + i);
#pragma unroll
            for (int s = 0; s < S; ++s) sdense[i * S + s] = __dsub_rn(sdense[i * S + s], __dmul_rn(lki, xk[s]));
          }
          __syncwarp();
        }
        for (int q = lane; q < nc * S; q += 32) o[q] = sdense[q];
      }
    } else {  // smoother-only bottom (amg.cpp:214-217)
      double* x = vx(last);
      for (int i = t; i < L.n; i += AMG_T) {
        const double di = __ldg(L.inv_diag + i);
#pragma unroll
        for (int s = 0; s < S; ++s) x[i * S + s] = __dmul_rn(omega, __dmul_rn(di, r[i * S + s]));
      }
      __syncthreads();
      for (int i = t; i < L.n; i += AMG_T) {
        double acc[S];
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] = 0.0;
        const int2 rw = ell_row(L.A, i);
        const int w = rw.y;
        int e = rw.x;
        #pragma unroll kAmgEllU
        for (int k = 0; k < w; ++k, e += 32) {
          const double2 rc = __ldg(L.A.rec + e);
          const int c = ell_col(rc);
          const double a = rc.x;
#pragma unroll
          for (int s = 0; s < S; ++s) acc[s] = __dadd_rn(acc[s], __dmul_rn(a, x[c * S + s]));
        }
        const double di = __ldg(L.inv_diag + i);
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double oi = __dadd_rn(x[i * S + s], __dmul_rn(omega, __dmul_rn(di, __dsub_rn(r[i * S + s], acc[s]))));
          o[i * S + s] = oi;
          if (last == 0) {
            rz[s] = fma(r[i * S + s], oi, rz[s]);
            if (exact) prod[static_cast<size_t>(s) * n0 + i] = __dmul_rn(r[i * S + s], oi);
          }
        }
      }
    }
    __syncthreads();
    if (last == 0 && H.dense_n > 0) {  // single dense level: r.z here
      for (int i = t; i < n0; i += AMG_T)
#pragma unroll
        for (int s = 0; s < S; ++s) {
          rz[s] = fma(r0[i * S + s], z[i * S + s], rz[s]);
          if (exact) prod[static_cast<size_t>(s) * n0 + i] = __dmul_rn(r0[i * S + s], z[i * S + s]);
        }
      __syncthreads();
    }
  }
  // ---- up: prolongation, post-smooth ---------------------------------------------
  for (int l = last - 1; l >= 0; --l) {
    const AmgLevelD L = H.lv[l];
    const double* __restrict__ r = vr(l);
    double* __restrict__ x = vx(l);
    const double* __restrict__ oc = vo(l + 1);
    int2 rw_n = t < L.n ? ell_row(L.P, t) : make_int2(0, 0);
#pragma unroll kAmgRowU
    for (int i = t; i < L.n; i += AMG_T) {  // x += P coarse (x_i + P_ik c_k, ascending k)
      const int2 rw = rw_n;
      if (i + AMG_T < L.n) rw_n = ell_row(L.P, i + AMG_T);
      if (kAmgPf > 0 && i + kAmgPf * AMG_T < L.n) amg_prefetch(x + static_cast<size_t>(i + kAmgPf * AMG_T) * S);
      double acc[S];
#pragma unroll
      for (int s = 0; s < S; ++s) acc[s] = x[i * S + s];
      const int w = rw.y;
      int e = rw.x;
      #pragma unroll 4
      for (int k = 0; k < w; ++k, e += 32) {
        const double2 rc = __ldg(L.P.rec + e);
        const int c = ell_col(rc);
        VQPC_DCHECK(c >= 0 && c < L.P.cols);
        const double v = rc.x;
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] = __dadd_rn(acc[s], __dmul_rn(v, oc[c * S + s]));
      }
#pragma unroll
      for (int s = 0; s < S; ++s) x[i * S + s] = acc[s];
    }
    __syncthreads();
    double* __restrict__ o = l == 0 ? z : vo(l);
    const double* __restrict__ xs = x;
    rw_n = (!L.st_c && t < L.n) ? ell_row(L.A, t) : make_int2(0, 0);
#pragma unroll kAmgRowU
    for (int i = t; i < L.n; i += AMG_T) {  // x += omega D^-1 (r - A x), A x into a fresh vector
      const int2 rw = rw_n;
      if (!L.st_c && i + AMG_T < L.n) rw_n = ell_row(L.A, i + AMG_T);
      double acc[S];
#pragma unroll
      for (int s = 0; s < S; ++s) acc[s] = 0.0;
      if (L.st_c) {  // level 0, structured: 0 + S, W, C, E, N products
        if (kAmgPf > 0 && i + kAmgPf * AMG_T < L.n) {
          const int ip = i + kAmgPf * AMG_T;
          amg_prefetch(xs + static_cast<size_t>(ip) * S);
          amg_prefetch(r + static_cast<size_t>(ip) * S);
          amg_prefetch(L.inv_diag + ip);
          amg_prefetch(L.st_s + ip);
          amg_prefetch(L.st_w + ip);
          amg_prefetch(L.st_c + ip);
        }
        const int m = L.st_m, ix = i % m, iy = i / m;
        auto add = [&](double a, int c) {
#pragma unroll
          for (int s = 0; s < S; ++s) acc[s] = __dadd_rn(acc[s], __dmul_rn(a, xs[c * S + s]));
        };
        if (iy > 0) add(__ldg(L.st_s + i), i - m);
        if (ix > 0) add(__ldg(L.st_w + i), i - 1);
        add(__ldg(L.st_c + i), i);
        if (ix < m - 1) add(__ldg(L.st_w + i + 1), i + 1);
        if (iy < m - 1) add(__ldg(L.st_s + i + m), i + m);
      } else {
      const int w = rw.y;
      int e = rw.x;
      #pragma unroll kAmgEllU
      for (int k = 0; k < w; ++k, e += 32) {
        const double2 rc = __ldg(L.A.rec + e);
        const int c = ell_col(rc);
        VQPC_DCHECK(c >= 0 && c < L.A.cols);
        const double a = rc.x;
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] = __dadd_rn(acc[s], __dmul_rn(a, xs[c * S + s]));
      }
      }
      const double di = __ldg(L.inv_diag + i);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double ri = r[i * S + s];
        const double oi = __dadd_rn(xs[i * S + s], __dmul_rn(omega, __dmul_rn(di, __dsub_rn(ri, acc[s]))));
        o[i * S + s] = oi;
        if (l == 0) {
          rz[s] = fma(ri, oi, rz[s]);
          if (exact) prod[static_cast<size_t>(s) * n0 + i] = __dmul_rn(ri, oi);
        }
      }
    }
    __syncthreads();
  }
}

struct PcgAmgParams {
  Grid2D g;
  const double* kappa;      // samples x ldk nodal kappa (natural mesh order)
  int64_t ldk;
  const uint8_t* kflag;
  const int32_t* perm;      // label-major order (groups index into it)
  const int32_t* labels;
  const int2* groups;       // (first entry in perm, count <= S), one label each
  const int* ngroups;
  const AmgHierD* hier;     // P hierarchies
  double omega;
  double* work;             // per CTA: cta_stride doubles
  int64_t cta_stride;
  int64_t cv_off;           // offset of the coarse-level scratch inside a CTA's block
  int64_t B, out_base, solve_limit;
  double eps;
  int max_iter;
  const int32_t* max_iter_arr;
  int* counter;
  int32_t* iters;
  double* rel;
  uint8_t* status;
  double* x_out;            // nullable, natural interior order
  int exact;
};

constexpr int AMG_WORK = 13;  // per slot: Ad, Aw, As, b, x[2], r, p[2], z, x0, res0, prod

// block sums of S partials (one reduction round for all slots)
template <int S>
__device__ __forceinline__ void amg_block_sums(double (&v)[S], double (*red)[AMG_T / 32], int warp, int lane) {
#pragma unroll
  for (int s = 0; s < S; ++s) v[s] = warp_allsum(v[s]);
  if (lane == 0)
#pragma unroll
    for (int s = 0; s < S; ++s) red[s][warp] = v[s];
  __syncthreads();
#pragma unroll
  for (int s = 0; s < S; ++s) {
    double a[AMG_T / 32];
#pragma unroll
    for (int i = 0; i < AMG_T / 32; ++i) a[i] = red[s][i];
#pragma unroll
    for (int w = 1; w < AMG_T / 32; w <<= 1)
#pragma unroll
      for (int i = 0; i + w < AMG_T / 32; i += 2 * w) a[i] += a[i + w];
    v[s] = a[0];
  }
  __syncthreads();
}

// exact mode: slot s's products summed serially (s = 0; s += t_i, i = 0..n-1) by thread s
template <int S>
__device__ __forceinline__ void amg_serial_sums(double (&v)[S], const double* prod, int n, double* sval) {
  __syncthreads();
  if (threadIdx.x < S) {
    const double* q = prod + static_cast<size_t>(threadIdx.x) * n;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, q[i]);
    sval[threadIdx.x] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < S; ++s) v[s] = sval[s];
  __syncthreads();
}

// One CTA per group of up to S samples of one label (the centroid's hierarchy is
// streamed once for all of them); slots that terminate keep iterating with
// alpha = beta = 0 (their vectors stay put) until the whole group is done.
template <int S>
__global__ void __launch_bounds__(AMG_T, AMG_MINB) pcgamg2d_kernel(const PcgAmgParams prm) {
  constexpr int NW = AMG_T / 32;
  extern __shared__ double sdense[];  // dense_n * S
  __shared__ double red[S][NW];
  __shared__ double sval[S];
  __shared__ int s_grp;
  const Grid2D g = prm.g;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n = g.n, m = g.m;
  double* base = prm.work + static_cast<size_t>(blockIdx.x) * prm.cta_stride;
  const size_t nS = static_cast<size_t>(n) * S;
  double* Ad = base;
  double* Aw = base + nS;       // W coupling of node i; the E coupling of i is Aw[i + 1]
  double* As = base + 2 * nS;   // S coupling of node i; the N coupling of i is As[i + m]
  double* Bv = base + 3 * nS;
  double* Xb[2] = {base + 4 * nS, base + 5 * nS};
  double* Rv = base + 6 * nS;
  double* Pb[2] = {base + 7 * nS, base + 8 * nS};
  double* Z = base + 9 * nS;
  double* X0 = base + 10 * nS;
  double* Res0 = base + 11 * nS;
  double* Prod = base + 12 * nS;  // exact mode: slot s's products at Prod[s * n + i]
  double* cv = base + prm.cv_off;
  const bool exact = prm.exact != 0;
  auto reduce = [&](double (&v)[S]) {
    if (exact) amg_serial_sums<S>(v, Prod, n, sval);
    else amg_block_sums<S>(v, red, warp, lane);
  };

  for (;;) {
    if (t == 0) s_grp = atomicAdd(prm.counter, 1);
    __syncthreads();
    const int grp = s_grp;
    __syncthreads();
    if (grp >= *prm.ngroups) break;
    const int2 gr = prm.groups[grp];
    int sid[S], mit[S], J[S];
    int64_t gsv[S];
    bool act[S];
    double rel_rec[S];
    uint8_t st[S];
    int label = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      act[s] = false;
      J[s] = 0;
      rel_rec[s] = 0.0;
      st[s] = VQPC_S_MAX_ITER;
      sid[s] = -1;
      gsv[s] = 0;
      mit[s] = 0;
      if (s < gr.y) {
        const int sm = prm.perm[gr.x + s];
        sid[s] = sm;
        gsv[s] = prm.out_base + sm;
        const int lb = prm.labels[sm];
        if (lb < 0 || prm.kflag[sm] || gsv[s] >= prm.solve_limit) {
          st[s] = gsv[s] >= prm.solve_limit ? VQPC_S_NOT_SOLVED
                  : lb < 0                  ? VQPC_S_INVALID_LATENT
                                            : (prm.kflag[sm] & 1) ? VQPC_S_COEFF_OVERFLOW : VQPC_S_INVALID_COEFF;
        } else {
          act[s] = true;
          label = lb;  // a group shares one label (bucketed)
        }
        mit[s] = prm.max_iter_arr ? prm.max_iter_arr[gsv[s]] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);
      }
    }
    const AmgHierD& H = prm.hier[label];
    int xc = 0, pc = 0;

    // ---- setup: every slot's rows (fem.cpp:213-256), x = 0, r = b; idle slots r = 0 ----
    double part[S];
#pragma unroll
    for (int s = 0; s < S; ++s) part[s] = 0.0;
    for (int i = t; i < n; i += AMG_T) {
      const int ix = i % m, iy = i / m;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        RowCoef rc;
        if (act[s]) {
          rc = assemble_row(prm.kappa + static_cast<size_t>(sid[s]) * prm.ldk, g, ix, iy);
        } else {
          rc.d = 1.0;
          rc.w = rc.s = rc.e = rc.nn = rc.b = 0.0;
        }
        const size_t q = static_cast<size_t>(i) * S + s;
        Ad[q] = rc.d;
        Aw[q] = rc.w;
        As[q] = rc.s;
        Bv[q] = rc.b;
        Xb[0][q] = 0.0;
        Rv[q] = rc.b;
        part[s] = fma(rc.b, rc.b, part[s]);
        if (exact) Prod[static_cast<size_t>(s) * n + i] = __dmul_rn(rc.b, rc.b);
      }
    }
    __syncthreads();
    reduce(part);
    double norm_b[S], rz[S], beta[S], alpha[S];
#pragma unroll
    for (int s = 0; s < S; ++s) norm_b[s] = sqrt(part[s]);
    amg_vcycle<S>(H, prm.omega, Rv, X0, Res0, Z, cv, sdense, exact, Prod, rz);
    reduce(rz);
    bool any = false;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      beta[s] = alpha[s] = 0.0;
      if (!act[s]) continue;
      if (norm_b[s] == 0.0) {
        st[s] = VQPC_S_CONVERGED;
        act[s] = false;
      } else if (!(rz[s] > 0.0)) {
        st[s] = VQPC_S_BREAKDOWN;
        act[s] = false;
      } else if (mit[s] < 1) {
        act[s] = false;
      }
      any |= act[s];
    }
    for (int j = 1; any; ++j) {
      // ---- p_new = z + beta p (solver.cpp:241) and A p, p.Ap; neighbours' p_new recomputed
      const double* Po = Pb[pc];
      double* Pn = Pb[pc ^ 1];
      const bool first = j == 1;
#pragma unroll
      for (int s = 0; s < S; ++s) part[s] = 0.0;
#pragma unroll kAmgPcgU
      for (int i = t; i < n; i += AMG_T) {
        if (kAmgPf > 0 && i + kAmgPf * AMG_T < n) {
          const size_t up = static_cast<size_t>(i + kAmgPf * AMG_T) * S;
          amg_prefetch(Z + up);
          if (!first) amg_prefetch(Po + up);
          amg_prefetch(As + up);
          amg_prefetch(Aw + up);
          amg_prefetch(Ad + up);
        }
        const int ix = i % m, iy = i / m;
        const bool hs = iy > 0, hw = ix > 0, he = ix < m - 1, hn = iy < m - 1;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          auto pnew = [&](int q) {
            const size_t u = static_cast<size_t>(q) * S + s;
            return first ? Z[u] : __dadd_rn(Z[u], __dmul_rn(beta[s], Po[u]));
          };
          const size_t u = static_cast<size_t>(i) * S + s;
          const double pi = pnew(i);
          Pn[u] = pi;
          const double ae = he ? Aw[u + S] : 0.0, an = hn ? As[u + static_cast<size_t>(m) * S] : 0.0;
          const double ap = row_apply(As[u], Aw[u], Ad[u], ae, an, hs ? pnew(i - m) : 0.0, hw ? pnew(i - 1) : 0.0, pi,
                                      he ? pnew(i + 1) : 0.0, hn ? pnew(i + m) : 0.0);
          part[s] = fma(pi, ap, part[s]);
          if (exact) Prod[static_cast<size_t>(s) * n + i] = __dmul_rn(pi, ap);
        }
      }
      pc ^= 1;
      reduce(part);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        alpha[s] = 0.0;
        if (!act[s]) continue;
        if (!(part[s] > 0.0)) {
          st[s] = VQPC_S_BREAKDOWN;
          act[s] = false;
          continue;
        }
        alpha[s] = rz[s] / part[s];
      }
      // ---- x += alpha p; r -= alpha A p; r_true = b - A x (solver.cpp:215-222) ----------
      const double* Pv = Pb[pc];
      const double* Xo = Xb[xc];
      double* Xn = Xb[xc ^ 1];
#pragma unroll
      for (int s = 0; s < S; ++s) part[s] = 0.0;
#pragma unroll kAmgPcgU
      for (int i = t; i < n; i += AMG_T) {
        if (kAmgPf > 0 && i + kAmgPf * AMG_T < n) {
          const size_t up = static_cast<size_t>(i + kAmgPf * AMG_T) * S;
          amg_prefetch(Pv + up);
          amg_prefetch(Xo + up);
          amg_prefetch(Rv + up);
          amg_prefetch(Bv + up);
          amg_prefetch(As + up);
          amg_prefetch(Aw + up);
          amg_prefetch(Ad + up);
        }
        const int ix = i % m, iy = i / m;
        const bool hs = iy > 0, hw = ix > 0, he = ix < m - 1, hn = iy < m - 1;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const size_t u = static_cast<size_t>(i) * S + s, dm = static_cast<size_t>(m) * S;
          auto xnew = [&](size_t q) { return __dadd_rn(Xo[q], __dmul_rn(alpha[s], Pv[q])); };
          const double as = As[u], aw = Aw[u], ad = Ad[u];
          const double ae = he ? Aw[u + S] : 0.0, an = hn ? As[u + dm] : 0.0;
          const double ap = row_apply(as, aw, ad, ae, an, hs ? Pv[u - dm] : 0.0, hw ? Pv[u - S] : 0.0, Pv[u],
                                      he ? Pv[u + S] : 0.0, hn ? Pv[u + dm] : 0.0);
          const double xi = xnew(u);
          Xn[u] = xi;
          Rv[u] = __dsub_rn(Rv[u], __dmul_rn(alpha[s], ap));
          const double ax = row_apply(as, aw, ad, ae, an, hs ? xnew(u - dm) : 0.0, hw ? xnew(u - S) : 0.0, xi,
                                      he ? xnew(u + S) : 0.0, hn ? xnew(u + dm) : 0.0);
          const double rt = __dsub_rn(Bv[u], ax);
          part[s] = fma(rt, rt, part[s]);
          if (exact) Prod[static_cast<size_t>(s) * n + i] = __dmul_rn(rt, rt);
        }
      }
      xc ^= 1;
      reduce(part);
      bool need = false;
      bool done_now[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        done_now[s] = false;
        if (!act[s]) continue;
        const double rel = sqrt(part[s]) / norm_b[s];
        J[s] = j;
        rel_rec[s] = rel;
        if (rel < prm.eps) {
          st[s] = VQPC_S_CONVERGED;
          act[s] = false;
          done_now[s] = true;
        } else if (j >= mit[s]) {  // loop exhausted: MAX_ITER (x is this iterate)
          act[s] = false;
          done_now[s] = true;
        } else {
          need = true;
        }
      }
      if (prm.x_out) {  // a slot's x at its exit iteration (later iterations leave it with alpha = 0 anyway)
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (done_now[s]) {
            double* xo = prm.x_out + static_cast<size_t>(gsv[s]) * n;
            for (int i = t; i < n; i += AMG_T) xo[i] = Xn[static_cast<size_t>(i) * S + s];
          }
      }
      if (!need) break;
      // ---- z = M^{-1} r (one V-cycle for every slot); r.z -----------------------------
      amg_vcycle<S>(H, prm.omega, Rv, X0, Res0, Z, cv, sdense, exact, Prod, part);
      reduce(part);
      any = false;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        beta[s] = 0.0;
        if (!act[s]) continue;
        if (!(part[s] > 0.0)) {
          st[s] = VQPC_S_BREAKDOWN;
          act[s] = false;
          continue;
        }
        beta[s] = part[s] / rz[s];
        rz[s] = part[s];
        any = true;
      }
    }
    // slots whose solve ended in a breakdown (or never started) report x as it stands
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (s >= gr.y) continue;
      if (t == 0) {
        prm.iters[gsv[s]] = J[s];
        prm.rel[gsv[s]] = rel_rec[s];
        prm.status[gsv[s]] = st[s];
      }
      if (prm.x_out && (st[s] == VQPC_S_BREAKDOWN)) {
        double* xo = prm.x_out + static_cast<size_t>(gsv[s]) * n;
        for (int i = t; i < n; i += AMG_T) xo[i] = Xb[xc][static_cast<size_t>(i) * S + s];
      }
    }
    __syncthreads();
  }
}

// M^{-1} r for one vector (Preconditioner::apply; parity tests), one CTA
__global__ void __launch_bounds__(AMG_T) amg_apply_kernel(const AmgHierD* hier, int p, double omega, const double* r,
                                                          double* z, double* x0, double* res0, double* cv) {
  extern __shared__ double sdense[];
  double rz[1];
  amg_vcycle<1>(hier[p], omega, r, x0, res0, z, cv, sdense, false, nullptr, rz);
}

// CSR values of the 2-D centroid matrices in the reference's stored pattern
// (fem.cpp:177-211: SW, S, W, C, E, N, NE per interior row, the SW/NE entries
// the exact zeros the reference stores): row i of centroid p at
// vals[(p * n + i) * 7 + k]; absent neighbours (boundary) are marked NaN.
__global__ void amg_centroid_rows_kernel(const double* kappa_c, int64_t ldk, int P, const Grid2D g, double* vals) {
  const int64_t total = static_cast<int64_t>(P) * g.n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(q / g.n), i = static_cast<int>(q % g.n);
    const int ix = i % g.m, iy = i / g.m;
    const RowCoef rc = assemble_row(kappa_c + static_cast<size_t>(p) * ldk, g, ix, iy);
    double* v = vals + static_cast<size_t>(q) * 7;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    v[0] = (ix > 0 && iy > 0) ? 0.0 : nan;
    v[1] = iy > 0 ? rc.s : nan;
    v[2] = ix > 0 ? rc.w : nan;
    v[3] = rc.d;
    v[4] = ix < g.m - 1 ? rc.e : nan;
    v[5] = iy < g.m - 1 ? rc.nn : nan;
    v[6] = (ix < g.m - 1 && iy < g.m - 1) ? 0.0 : nan;
  }
}

}  // namespace vqpc
