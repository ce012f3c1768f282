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

namespace vqpc {

constexpr int AMG_T = 256;          // threads per CTA
constexpr int AMG_MAXLEV = 16;      // hierarchy depth handled on the device
constexpr int AMG_MAXDENSE = 1024;  // coarsest dense solve size (shared-memory vector)

// Sliced ELL: rows in slices of 32; slice s holds width_s = (soff[s+1]-soff[s])/32
// entries per row, entry k of row i at soff[s] + 32 k + (i & 31); col -1 pads.
struct AmgEll {
  const int* soff;
  const int* col;
  const double* val;
};

struct AmgLevelD {
  int n, nc;                // rows; rows of the next level (0 on the coarsest)
  AmgEll A, P, Pt;
  const double* inv_diag;
  int voff;                 // levels >= 1: offset of (r, x, o) in the per-CTA coarse scratch
};

struct AmgHierD {
  int nlev, dense_n;
  const double* L;          // dense_n x dense_n row-major lower factor of the coarsest operator
  AmgLevelD lv[AMG_MAXLEV];
};

__device__ __forceinline__ int ell_row(const AmgEll& M, int i, int& width) {
  const int s = i >> 5;
  const int b = __ldg(M.soff + s);
  width = (__ldg(M.soff + s + 1) - b) >> 5;
  return b + (i & 31);
}

// y = 0 + sum_k v_k x[c_k] (ascending columns): Eigen's sparse * dense into a fresh vector
__device__ __forceinline__ double ell_dot(const AmgEll& M, int i, const double* x) {
  int w;
  int e = ell_row(M, i, w);
  double s = 0.0;
  for (int k = 0; k < w; ++k, e += 32) {
    const int c = __ldg(M.col + e);
    if (c < 0) break;
    s = __dadd_rn(s, __dmul_rn(__ldg(M.val + e), x[c]));
  }
  return s;
}

// ---- one V-cycle z = M^{-1} r on hierarchy H (amg.cpp:210-225), block-wide ---------
// Level 0: r0 (input, n0), x0 and res0 scratch, z (output). Levels >= 1 in cv
// (per CTA). Returns this thread's r.z partial (fast mode); in exact mode the
// products r_i z_i are stored at prod[i].
__device__ double amg_vcycle(const AmgHierD& H, double omega, const double* r0, double* x0, double* res0, double* z,
                             double* cv, double* sdense, bool exact, double* prod) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  auto vr = [&](int l) -> double* { return l == 0 ? const_cast<double*>(r0) : cv + H.lv[l].voff; };
  auto vx = [&](int l) -> double* { return l == 0 ? x0 : cv + H.lv[l].voff + H.lv[l].n; };
  auto vo = [&](int l) -> double* { return l == 0 ? res0 : cv + H.lv[l].voff + 2 * H.lv[l].n; };
  const int last = H.nlev - 1;
  // ---- down: pre-smooth from zero, residual, restriction -------------------------
  for (int l = 0; l < last; ++l) {
    const AmgLevelD& L = H.lv[l];
    const double* r = vr(l);
    double* x = vx(l);
    double* res = vo(l);  // the residual; later this level's output
    for (int i = t; i < L.n; i += AMG_T) {
      const double xi = __dmul_rn(omega, __dmul_rn(__ldg(L.inv_diag + i), r[i]));
      x[i] = xi;
      // res = r; res -= A x (Eigen's rewrite of `r - A x`), x_j recomputed with its owner's operations
      int w;
      int e = ell_row(L.A, i, w);
      double s = r[i];
      for (int k = 0; k < w; ++k, e += 32) {
        const int c = __ldg(L.A.col + e);
        if (c < 0) break;
        const double xc = __dmul_rn(omega, __dmul_rn(__ldg(L.inv_diag + c), r[c]));
        s = __dsub_rn(s, __dmul_rn(__ldg(L.A.val + e), xc));
      }
      res[i] = s;
    }
    __syncthreads();
    double* rn = vr(l + 1);
    for (int c = t; c < L.nc; c += AMG_T) rn[c] = ell_dot(L.Pt, c, res);
    __syncthreads();
  }
  // ---- coarsest ----------------------------------------------------------------
  {
    const AmgLevelD& L = H.lv[last];
    const double* r = vr(last);
    double* o = last == 0 ? z : vo(last);
    if (H.dense_n > 0) {
      const int nc = H.dense_n;
      if (warp == 0) {
        for (int i = lane; i < nc; i += 32) sdense[i] = r[i];
        __syncwarp();
        for (int k = 0; k < nc; ++k) {  // L y = r, column-oriented
          if (lane == (k & 31)) sdense[k] = __ddiv_rn(sdense[k], __ldg(H.L + static_cast<size_t>(k) * nc + k));
          __syncwarp();
          const double yk = sdense[k];
          for (int i = lane; i < nc; i += 32)
            if (i > k) sdense[i] = __dsub_rn(sdense[i], __dmul_rn(__ldg(H.L + static_cast<size_t>(i) * nc + k), yk));
          __syncwarp();
        }
        for (int k = nc - 1; k >= 0; --k) {  // L^T x = y, column-oriented
          if (lane == (k & 31)) sdense[k] = __ddiv_rn(sdense[k], __ldg(H.L + static_cast<size_t>(k) * nc + k));
          __syncwarp();
          const double xk = sdense[k];
          for (int i = lane; i < k; i += 32)
            sdense[i] = __dsub_rn(sdense[i], __dmul_rn(__ldg(H.L + static_cast<size_t>(k) * nc + i), xk));
          __syncwarp();
        }
        for (int i = lane; i < nc; i += 32) o[i] = sdense[i];
      }
    } else {  // smoother-only bottom (amg.cpp:214-217)
      double* x = vx(last);
      for (int i = t; i < L.n; i += AMG_T) x[i] = __dmul_rn(omega, __dmul_rn(__ldg(L.inv_diag + i), r[i]));
      __syncthreads();
      for (int i = t; i < L.n; i += AMG_T) {
        const double ti = ell_dot(L.A, i, x);
        o[i] = __dadd_rn(x[i], __dmul_rn(omega, __dmul_rn(__ldg(L.inv_diag + i), __dsub_rn(r[i], ti))));
      }
    }
    __syncthreads();
  }
  // ---- up: prolongation, post-smooth ---------------------------------------------
  double rz = 0.0;
  for (int l = last - 1; l >= 0; --l) {
    const AmgLevelD& L = H.lv[l];
    const double* r = vr(l);
    double* x = vx(l);
    const double* oc = l + 1 == last && H.dense_n == 0 && last == 0 ? z : vo(l + 1);
    for (int i = t; i < L.n; i += AMG_T) {  // x += P coarse (x_i + P_ik c_k, ascending k)
      int w;
      int e = ell_row(L.P, i, w);
      double s = x[i];
      for (int k = 0; k < w; ++k, e += 32) {
        const int c = __ldg(L.P.col + e);
        if (c < 0) break;
        s = __dadd_rn(s, __dmul_rn(__ldg(L.P.val + e), oc[c]));
      }
      x[i] = s;
    }
    __syncthreads();
    double* o = l == 0 ? z : vo(l);
    for (int i = t; i < L.n; i += AMG_T) {  // x += omega D^-1 (r - A x), A x into a fresh vector
      const double ti = ell_dot(L.A, i, x);
      const double oi = __dadd_rn(x[i], __dmul_rn(omega, __dmul_rn(__ldg(L.inv_diag + i), __dsub_rn(r[i], ti))));
      o[i] = oi;
      if (l == 0) {
        rz = fma(r[i], oi, rz);
        if (exact) prod[i] = __dmul_rn(r[i], oi);
      }
    }
    __syncthreads();
  }
  if (last == 0) {  // single-level hierarchy: the smoother (or the dense solve) wrote z
    for (int i = t; i < H.lv[0].n; i += AMG_T) {
      rz = fma(r0[i], z[i], rz);
      if (exact) prod[i] = __dmul_rn(r0[i], z[i]);
    }
    __syncthreads();
  }
  return rz;
}

struct PcgAmgParams {
  Grid2D g;
  const double* kappa;      // samples x ldk nodal kappa (natural mesh order)
  int64_t ldk;
  const uint8_t* kflag;
  const int32_t* perm;
  const int32_t* labels;
  const AmgHierD* hier;     // P hierarchies
  double omega;
  double* work;             // per CTA: AMG_WORK n + cv_len doubles
  int64_t cta_stride;       // doubles per CTA
  int cv_off;               // offset of the coarse-level scratch inside a CTA's block
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

constexpr int AMG_WORK = 13;  // Ad, Aw, As, b, x[2], r, p[2], z, x0, res0, prod

template <int NW>
__device__ __forceinline__ double amg_reduce(bool exact, double part, const double* prod, int n, double* slot,
                                             int warp, int lane) {
  return exact ? serial_sum2d(prod, n, slot) : block_sum2d<NW>(part, slot, warp, lane);
}

__global__ void __launch_bounds__(AMG_T, 2) pcgamg2d_kernel(const PcgAmgParams prm) {
  constexpr int NW = AMG_T / 32;
  __shared__ double red[4][NW];
  __shared__ double sdense[AMG_MAXDENSE];
  __shared__ int64_t s_item;
  const Grid2D g = prm.g;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n = g.n, m = g.m;
  double* base = prm.work + static_cast<size_t>(blockIdx.x) * prm.cta_stride;
  double* Ad = base;
  double* Aw = base + n;       // W coupling of node i; the E coupling of i is Aw[i + 1]
  double* As = base + 2 * n;   // S coupling of node i; the N coupling of i is As[i + m]
  double* Bv = base + 3 * n;
  double* Xb[2] = {base + 4 * n, base + 5 * n};
  double* Rv = base + 6 * n;
  double* Pb[2] = {base + 7 * n, base + 8 * n};
  double* Z = base + 9 * n;
  double* X0 = base + 10 * n;
  double* Res0 = base + 11 * n;
  double* Prod = base + 12 * n;
  double* cv = base + prm.cv_off;
  const bool exact = prm.exact != 0;
  auto reduce = [&](double part, double* slot) { return amg_reduce<NW>(exact, part, Prod, n, slot, warp, lane); };

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
    const AmgHierD& H = prm.hier[label];
    int xc = 0, pc = 0;

    // ---- setup: the sample's rows (fem.cpp:213-256), x = 0, r = b --------------------
    double bb = 0.0;
    for (int i = t; i < n; i += AMG_T) {
      const RowCoef rc = assemble_row(kap, g, i % m, i / m);
      Ad[i] = rc.d;
      Aw[i] = rc.w;
      As[i] = rc.s;
      Bv[i] = rc.b;
      Xb[0][i] = 0.0;
      Rv[i] = rc.b;
      bb = fma(rc.b, rc.b, bb);
      if (exact) Prod[i] = __dmul_rn(rc.b, rc.b);
    }
    __syncthreads();
    const int max_iter = prm.max_iter_arr ? prm.max_iter_arr[gs] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);
    const double norm_b = sqrt(reduce(bb, red[3]));
    double rz = reduce(amg_vcycle(H, prm.omega, Rv, X0, Res0, Z, cv, sdense, exact, Prod), red[2]);
    int J = 0;
    double rel_rec = 0.0;
    uint8_t st = VQPC_S_MAX_ITER;
    if (norm_b == 0.0) st = VQPC_S_CONVERGED;
    else if (!(rz > 0.0)) st = VQPC_S_BREAKDOWN;
    else {
      double beta = 0.0;
      for (int j = 1; j <= max_iter; ++j) {
        // ---- p_new = z + beta p (solver.cpp:241) and A p, p.Ap; neighbours' p_new recomputed
        const double* Po = Pb[pc];
        double* Pn = Pb[pc ^ 1];
        const bool first = j == 1;
        auto pnew = [&](int q) { return first ? Z[q] : __dadd_rn(Z[q], __dmul_rn(beta, Po[q])); };
        double pap = 0.0;
        for (int i = t; i < n; i += AMG_T) {
          const int ix = i % m, iy = i / m;
          const double pi = pnew(i);
          Pn[i] = pi;
          const double ps = iy > 0 ? pnew(i - m) : 0.0, pw = ix > 0 ? pnew(i - 1) : 0.0;
          const double pe = ix < m - 1 ? pnew(i + 1) : 0.0, pn = iy < m - 1 ? pnew(i + m) : 0.0;
          const double ae = ix < m - 1 ? Aw[i + 1] : 0.0, an = iy < m - 1 ? As[i + m] : 0.0;
          const double ap = row_apply(As[i], Aw[i], Ad[i], ae, an, ps, pw, pi, pe, pn);
          pap = fma(pi, ap, pap);
          if (exact) Prod[i] = __dmul_rn(pi, ap);
        }
        pc ^= 1;
        const double pAp = reduce(pap, red[0]);
        if (!(pAp > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        const double alpha = rz / pAp;
        // ---- x += alpha p; r -= alpha A p; r_true = b - A x (solver.cpp:215-222) ----------
        const double* Pv = Pb[pc];
        const double* Xo = Xb[xc];
        double* Xn = Xb[xc ^ 1];
        auto xnew = [&](int q) { return __dadd_rn(Xo[q], __dmul_rn(alpha, Pv[q])); };
        double rr = 0.0;
        for (int i = t; i < n; i += AMG_T) {
          const int ix = i % m, iy = i / m;
          const bool hs = iy > 0, hw = ix > 0, he = ix < m - 1, hn = iy < m - 1;
          const double as = As[i], aw = Aw[i], ad = Ad[i];
          const double ae = he ? Aw[i + 1] : 0.0, an = hn ? As[i + m] : 0.0;
          const double ap = row_apply(as, aw, ad, ae, an, hs ? Pv[i - m] : 0.0, hw ? Pv[i - 1] : 0.0, Pv[i],
                                      he ? Pv[i + 1] : 0.0, hn ? Pv[i + m] : 0.0);
          const double xi = xnew(i);
          Xn[i] = xi;
          Rv[i] = __dsub_rn(Rv[i], __dmul_rn(alpha, ap));
          const double ax = row_apply(as, aw, ad, ae, an, hs ? xnew(i - m) : 0.0, hw ? xnew(i - 1) : 0.0, xi,
                                      he ? xnew(i + 1) : 0.0, hn ? xnew(i + m) : 0.0);
          const double rt = __dsub_rn(Bv[i], ax);
          rr = fma(rt, rt, rr);
          if (exact) Prod[i] = __dmul_rn(rt, rt);
        }
        xc ^= 1;
        const double rel = sqrt(reduce(rr, red[1])) / norm_b;
        J = j;
        rel_rec = rel;
        if (rel < prm.eps) {
          st = VQPC_S_CONVERGED;
          break;
        }
        // ---- z = M^{-1} r (one V-cycle); r.z ------------------------------------------
        const double rz_next = reduce(amg_vcycle(H, prm.omega, Rv, X0, Res0, Z, cv, sdense, exact, Prod), red[2]);
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
      for (int i = t; i < n; i += AMG_T) xo[i] = Xb[xc][i];
    }
    __syncthreads();
  }
}

// M^{-1} r for one vector (Preconditioner::apply; parity tests), one CTA
__global__ void __launch_bounds__(AMG_T) amg_apply_kernel(const AmgHierD* hier, int p, double omega, const double* r,
                                                          double* z, double* x0, double* res0, double* cv) {
  __shared__ double sdense[AMG_MAXDENSE];
  amg_vcycle(hier[p], omega, r, x0, res0, z, cv, sdense, false, nullptr);
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
