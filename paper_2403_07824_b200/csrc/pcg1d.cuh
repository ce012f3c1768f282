// pcg1d.cuh — kernel (d), 1-D: batched PCG, one CTA per sample, persistent grid.
//
// Replaces, for every sample of a bucket, the reference's per-sample loop body
// (proj/src/driver.cpp:228-239): transport(lift) -> assemble -> pcg with the
// centroid's Cholesky preconditioner (proj/src/solver.cpp:186-245, :80-111).
//
// Layout. One CTA of T threads owns one sample at a time; thread t owns the R
// consecutive rows [tR, tR+R) of the n unknowns (n <= R*T; padding rows are
// dead and provably inert, see below). Registers per thread: x, r, p (R each),
// the preconditioner couplings n_j and the transient w/z (or A p). Shared
// memory is thread-major ([i*T + t] holds row tR+i, so warp accesses are
// bank-conflict free): the sample's element conductances c_j = kappa_j/h and
// the centroid factor {n_j, 1/u_j^2}, reloaded only when the bucket changes.
//
// Operator: A_jj = c_j + c_{j+1}, A_{j,j+1} = -c_{j+1}
// with c_j = kappa_j / h — the same IEEE values the oracle's CSR holds; b_j = h.
// Matrix-free: no CSR is ever formed.
//
// Preconditioner: the exact factor of the centroid matrix, M = U U^T with U the
// upper-bidiagonal Cholesky factor of the reference's RCM (= reversed) order
// (solver.cpp:32-70 on a path graph), stored as U = (I+N) D:
//   sweep 1 (descending)  y_j = r_j - n_j y_{j+1};   y_j <- y_j / u_j^2
//   sweep 2 (ascending)   z_j = y_j - n_{j-1} z_{j-1}
// Each sweep is a first-order linear recurrence, solved as a chunked scan:
// serial over a thread's rows (two interleaved half-chains for ILP), an
// affine scan over lanes with shuffles whose multipliers are per-centroid
// constants precomputed into shared memory (one SHFL pair + one FMA per
// level), one barrier for the warp aggregates, a short fold over warps, and a
// fix-up pass.
//
// Per iteration, in the reference's operation order (solver.cpp:211-242):
//   Ap = A p; pAp = p.Ap               -> barrier 1 (reduction)
//   alpha; x += alpha p; r -= alpha Ap
//   r_true = b - A x; rr = |r_true|^2   (rides barrier 2)
//   sweep 1                             -> barrier 2 (warp aggregates + rr)
//   rel = sqrt(rr)/|b|; record; rel < eps -> converged
//   sweep 2                             -> barrier 3 (warp aggregates)
//   rz' = r.z                            -> barrier 4 (reduction + z halos)
//   beta = rz'/rz; p = z + beta p
// Halo values of x and p are never exchanged: each thread updates its copy of
// the neighbours' boundary entries with the same FMA the neighbour executes,
// so they stay bit-identical; only z boundary values travel (barrier 4).
// Block reductions: butterfly inside the warp, then every warp reduces the
// NW warp partials with the same butterfly — all threads hold identical bits,
// and the order is fixed, so results do not depend on scheduling.
// Breakdown checks use !(v > 0) exactly like the reference (NaN-safe).
//
// Dead rows j >= n: n_j = 1/u_j^2 = 0 (so z_j = p_j = x_j = 0) and
// n_{n-1} = 0 (no coupling into them); A p leaks -c_n p_{n-1} into r_n only,
// which sweep 1 never propagates (n_{n-1} = 0) and scales by 0; the true
// residual is masked in the one thread that owns dead rows.
#pragma once
#include "common.cuh"

namespace vqpc {

struct Pcg1dParams {
  int n;                      // unknowns
  int N;                      // elements (= n + 1)
  double h;                   // 1 / N
  const double* kappa;        // samples x N (row stride ldk), natural sample order
  int64_t ldk;
  const uint8_t* kflag;       // per sample: nonzero -> coefficient overflow
  const int32_t* perm;        // bucket order -> local sample index
  const int32_t* labels;      // per local sample
  const double2* factors;     // P x NP {n_j, 1/u_j^2}
  int NP;                     // padded rows per factor (= R*T)
  int64_t B;                  // samples in this batch
  int64_t out_base;           // global index of local sample 0 (outputs)
  double eps;
  int max_iter;               // < 0 -> 10 n
  const int32_t* max_iter_arr;  // nullable, indexed by global sample
  int* counter;               // work queue head
  int32_t* iters;
  double* rel;
  uint8_t* status;
  double* x_out;              // nullable, (global sample) x n
};

template <int R, int T>
struct Pcg1dShared {
  static constexpr int NW = T / 32;
  double2 fac[R * T];     // {n_j, 1/u_j^2}, thread-major
  double cs[R * T + 1];   // c_j = kappa_j / h, thread-major; [R*T] = c_{R*T}
  double lev[12 * T];     // per-thread scan multipliers: L1[5], Q1, L2[5], Q2
  double wa1[NW], wa2[NW];  // per-warp products of the sweep multipliers
  double sw1[NW], sw2[NW];  // per-iteration warp aggregates
  double red[4][NW];        // reduction partials: pAp, rr, rz, |b|^2
  double zf[T], zl[T];      // first / last z of every thread
  int item;
};

// sum over the NW warp partials in a fixed butterfly order (identical in all threads)
template <int NW>
__device__ __forceinline__ double cross_warp_sum(const double* part, int lane) {
  double t = lane < NW ? part[lane] : 0.0;
  return warp_allsum(t);
}

template <int R, int T>
__global__ void __launch_bounds__(T, 1) pcg1d_kernel(const Pcg1dParams prm) {
  using Sh = Pcg1dShared<R, T>;
  constexpr int NW = Sh::NW;
  constexpr int H = R / 2;
  static_assert(R % 2 == 0 && R >= 4, "two half-chains per thread");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sh& S = *reinterpret_cast<Sh*>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j0 = tid * R;
  const int n = prm.n;
  const bool tail_thread = j0 + R > n;  // owns dead rows

  int cur_label = -1;
  double nc[R];         // n_j of own rows
  double n_left = 0.0;  // n_{j0-1}
  double A1lo = 0, A1hi = 0, A2lo = 0, A2hi = 0;

  for (;;) {
    if (tid == 0) S.item = atomicAdd(prm.counter, 1);
    __syncthreads();
    const int64_t item = S.item;
    __syncthreads();
    if (item >= prm.B) break;
    const int s = prm.perm[item];
    const int64_t gs = prm.out_base + s;
    const int label = prm.labels[s];
    if (label < 0 || prm.kflag[s]) {
      if (tid == 0) {
        prm.iters[gs] = 0;
        prm.rel[gs] = 0.0;
        prm.status[gs] = label < 0 ? VQPC_S_INVALID_LATENT : VQPC_S_COEFF_OVERFLOW;
      }
      continue;
    }
    if (label != cur_label) {
      // ---- new bucket: factor to smem, per-thread / per-lane scan constants ----
      const double2* src = prm.factors + static_cast<size_t>(label) * prm.NP;
      for (int e = tid; e < R * T; e += T) S.fac[(e % R) * T + e / R] = src[e];  // coalesced read
      __syncthreads();
#pragma unroll
      for (int i = 0; i < R; ++i) nc[i] = S.fac[i * T + tid].x;
      n_left = tid > 0 ? S.fac[(R - 1) * T + tid - 1].x : 0.0;
      A1lo = 1.0;
      A1hi = 1.0;
#pragma unroll
      for (int i = 0; i < H; ++i) A1lo *= -nc[i];
#pragma unroll
      for (int i = H; i < R; ++i) A1hi *= -nc[i];
      A2lo = -n_left;
#pragma unroll
      for (int i = 0; i < H - 1; ++i) A2lo *= -nc[i];
      A2hi = 1.0;
#pragma unroll
      for (int i = H - 1; i < R - 1; ++i) A2hi *= -nc[i];
      // lane-range products for the shuffle scans
      double P1 = A1lo * A1hi, P2 = A2lo * A2hi;  // current inclusive range products
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int off = 1 << k;
        S.lev[k * T + tid] = lane + off < 32 ? P1 : 0.0;    // suffix-scan multiplier
        S.lev[(6 + k) * T + tid] = lane >= off ? P2 : 0.0;  // prefix-scan multiplier
        const double o1 = shfl_down(P1, off), o2 = shfl_up(P2, off);
        if (lane + off < 32) P1 *= o1;
        if (lane >= off) P2 *= o2;
      }
      // now P1 = prod over lanes [lane, 31], P2 = prod over lanes [0, lane]
      const double q1 = shfl_down(P1, 1), q2 = shfl_up(P2, 1);
      S.lev[5 * T + tid] = lane < 31 ? q1 : 1.0;
      S.lev[11 * T + tid] = lane > 0 ? q2 : 1.0;
      if (lane == 0) S.wa1[warp] = P1;
      if (lane == 31) S.wa2[warp] = P2;
      cur_label = label;
      __syncthreads();
    }

    // ---- sample setup: c_j = kappa_j / h, b = h, x = 0, r = b --------------
    const double* kap = prm.kappa + static_cast<size_t>(s) * prm.ldk;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int j = j0 + i;
      S.cs[i * T + tid] = j <= n ? kap[j] / prm.h : 0.0;  // IEEE division: the oracle's kappa/h
    }
    if (tid == T - 1) S.cs[R * T] = R * T <= n ? kap[R * T] / prm.h : 0.0;
    double x[R], r[R], p[R], wz[R];
    double bb = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      x[i] = 0.0;
      r[i] = j0 + i < n ? prm.h : 0.0;
      bb = fma(r[i], r[i], bb);
    }
    const int max_iter = prm.max_iter_arr ? prm.max_iter_arr[gs] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);

    double rz = 0.0, norm_b = 0.0, rel_rec = 0.0;
    int J = 0;
    uint8_t st = VQPC_S_MAX_ITER;
    double rr_loc = 0.0;
    double p_left = 0.0, p_right = 0.0, x_left = 0.0, x_right = 0.0;
    int j = 0;  // 0: setup pass (z = M^{-1} b); >= 1: iteration j
    for (;;) {
      // ================= sweep 1 (descending) + rr: barrier 2 ===============
      {
        double vh = 0.0, vl = 0.0;
#pragma unroll
        for (int i = 0; i < H; ++i) {  // two independent chains, incoming 0
          vh = fma(-nc[R - 1 - i], vh, r[R - 1 - i]);
          vl = fma(-nc[H - 1 - i], vl, r[H - 1 - i]);
        }
        const double Wh = vh;
        double W = fma(A1lo, vh, vl);
#pragma unroll
        for (int k = 0; k < 5; ++k) W = fma(S.lev[k * T + tid], shfl_down(W, 1 << k), W);
        const double rrw = warp_allsum(rr_loc);
        if (lane == 0) {
          S.sw1[warp] = W;
          S.red[1][warp] = rrw;
        }
        __syncthreads();  // barrier 2
        double v = 0.0;
#pragma unroll
        for (int w2 = NW - 1; w2 > 0; --w2)
          if (w2 > warp) v = fma(S.wa1[w2], v, S.sw1[w2]);
        const double Wn = shfl_down(W, 1);
        const double vin = fma(S.lev[5 * T + tid], v, lane == 31 ? 0.0 : Wn);
        // fix-up: hi half from vin, lo half from y at row j0+H
        double uh = vin, ul = fma(A1hi, vin, Wh);
#pragma unroll
        for (int i = 0; i < H; ++i) {
          uh = fma(-nc[R - 1 - i], uh, r[R - 1 - i]);
          ul = fma(-nc[H - 1 - i], ul, r[H - 1 - i]);
          wz[R - 1 - i] = uh;
          wz[H - 1 - i] = ul;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) wz[i] *= S.fac[i * T + tid].y;
      }
      if (j > 0) {
        const double rr = cross_warp_sum<NW>(S.red[1], lane);
        const double rel = sqrt(rr) / norm_b;
        J = j;
        rel_rec = rel;
        if (rel < prm.eps) {
          st = VQPC_S_CONVERGED;
          break;
        }
      }
      // ================= sweep 2 (ascending): barrier 3 =====================
      {
        double vl = wz[0], vh = wz[H];  // incoming 0 for both halves
#pragma unroll
        for (int i = 1; i < H; ++i) {
          vl = fma(-nc[i - 1], vl, wz[i]);
          vh = fma(-nc[H + i - 1], vh, wz[H + i]);
        }
        const double Zl = vl;
        double W = fma(A2hi, vl, vh);
#pragma unroll
        for (int k = 0; k < 5; ++k) W = fma(S.lev[(6 + k) * T + tid], shfl_up(W, 1 << k), W);
        if (lane == 31) S.sw2[warp] = W;
        __syncthreads();  // barrier 3
        double v = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < NW - 1; ++w2)
          if (w2 < warp) v = fma(S.wa2[w2], v, S.sw2[w2]);
        const double Wp = shfl_up(W, 1);
        const double vin = fma(S.lev[11 * T + tid], v, lane == 0 ? 0.0 : Wp);
        double ul = fma(-n_left, vin, wz[0]);
        double uh = fma(-nc[H - 1], fma(A2lo, vin, Zl), wz[H]);
        wz[0] = ul;
        wz[H] = uh;
#pragma unroll
        for (int i = 1; i < H; ++i) {
          ul = fma(-nc[i - 1], ul, wz[i]);
          uh = fma(-nc[H + i - 1], uh, wz[H + i]);
          wz[i] = ul;
          wz[H + i] = uh;
        }
      }
      // ================= rz (+|b|^2 at setup), z halos: barrier 4 ===========
      {
        double rz_loc = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) rz_loc = fma(r[i], wz[i], rz_loc);
        const double a = warp_allsum(rz_loc);
        const double b2 = j == 0 ? warp_allsum(bb) : 0.0;
        if (lane == 0) {
          S.red[2][warp] = a;
          S.red[3][warp] = b2;
        }
        S.zf[tid] = wz[0];
        S.zl[tid] = wz[R - 1];
        __syncthreads();  // barrier 4
      }
      const double rz_next = cross_warp_sum<NW>(S.red[2], lane);
      const double zl_left = tid > 0 ? S.zl[tid - 1] : 0.0;
      const double zf_right = tid < T - 1 ? S.zf[tid + 1] : 0.0;
      if (j == 0) {
        norm_b = sqrt(cross_warp_sum<NW>(S.red[3], lane));
        if (norm_b == 0.0) {
          st = VQPC_S_CONVERGED;
          break;
        }
        if (!(rz_next > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        rz = rz_next;
#pragma unroll
        for (int i = 0; i < R; ++i) p[i] = wz[i];
        p_left = zl_left;
        p_right = zf_right;
      } else {
        if (!(rz_next > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        const double beta = rz_next / rz;
        rz = rz_next;
#pragma unroll
        for (int i = 0; i < R; ++i) p[i] = fma(beta, p[i], wz[i]);
        p_left = fma(beta, p_left, zl_left);
        p_right = fma(beta, p_right, zf_right);
      }
      // ================= next iteration: Ap, pAp -> barrier 1 ===============
      ++j;
      if (j > max_iter) {
        st = VQPC_S_MAX_ITER;
        break;
      }
      {
        double pap_loc = 0.0;
        double c_lo = S.cs[tid];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const double c_hi = i + 1 < R ? S.cs[(i + 1) * T + tid] : S.cs[tid + 1];
          const double pl = i == 0 ? p_left : p[i - 1];
          const double pr = i == R - 1 ? p_right : p[i + 1];
          const double t = fma(c_hi, pr, c_lo * pl);
          wz[i] = fma(c_lo + c_hi, p[i], -t);  // (A p)_j, reusing wz
          pap_loc = fma(p[i], wz[i], pap_loc);
          c_lo = c_hi;
        }
        const double a = warp_allsum(pap_loc);
        if (lane == 0) S.red[0][warp] = a;
        __syncthreads();  // barrier 1
      }
      const double pAp = cross_warp_sum<NW>(S.red[0], lane);
      if (!(pAp > 0.0)) {
        st = VQPC_S_BREAKDOWN;
        break;
      }
      const double alpha = rz / pAp;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        x[i] = fma(alpha, p[i], x[i]);
        r[i] = fma(-alpha, wz[i], r[i]);
      }
      x_left = fma(alpha, p_left, x_left);
      x_right = fma(alpha, p_right, x_right);
      // true residual b - A x
      rr_loc = 0.0;
      {
        double c_lo = S.cs[tid];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const double c_hi = i + 1 < R ? S.cs[(i + 1) * T + tid] : S.cs[tid + 1];
          const double xl = i == 0 ? x_left : x[i - 1];
          const double xr = i == R - 1 ? x_right : x[i + 1];
          const double t = fma(c_hi, xr, c_lo * xl);
          double rt = prm.h - fma(c_lo + c_hi, x[i], -t);
          if (tail_thread && j0 + i >= n) rt = 0.0;
          rr_loc = fma(rt, rt, rr_loc);
          c_lo = c_hi;
        }
      }
    }

    if (tid == 0) {
      prm.iters[gs] = J;
      prm.rel[gs] = rel_rec;
      prm.status[gs] = st;
    }
    if (prm.x_out) {
      double* xo = prm.x_out + static_cast<size_t>(gs) * n;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (j0 + i < n) xo[j0 + i] = x[i];
    }
  }
}

template <int R, int T>
constexpr size_t pcg1d_smem_bytes() {
  return sizeof(Pcg1dShared<R, T>);
}

}  // namespace vqpc
