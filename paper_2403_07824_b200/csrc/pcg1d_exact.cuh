// pcg1d_exact.cuh — kernel (d), 1-D, reference-order mode (vqpc_set_exact_reductions).
//
// The fast kernel (pcg1d.cuh) differs from the reference only in summation and
// scan order (tree dot products, a chunked-scan tridiagonal solve) and in
// contracting the vector updates into FMAs. This kernel removes those three
// differences, so that given the same kappa it reproduces the oracle's (and the
// reference's) PCG bit for bit — iteration counts, residual records, status and
// x — which pins every other piece of GPU arithmetic on the 1-D path:
//
//  * dot / norm2 (solver.cpp:176-182): products rounded, summed serially in
//    natural row order (s += a_i * b_i, no contraction);
//  * matvec (fem.cpp:142-148): s = 0; s += a_jk v_k over the CSR row in column
//    order, values -c_j, c_j + c_{j+1}, -c_{j+1} (the 1-D assembly's IEEE values);
//  * the updates x += alpha p, r -= alpha Ap, p = z + beta p (solver.cpp:224-241)
//    as separate multiply and add;
//  * the preconditioner apply (solver.cpp:98-110): Eigen's SimplicialLLT solve
//    of the RCM-permuted (= reversed) system with the factor {l_j, u_j} that
//    factor1d_kernel computes with the reference's own IEEE operations:
//      forward  (k = n-1-j ascending):  y_j = (r_j - y_{j+1} l_j) / u_j
//      backward (j ascending):          z_j = y_j / u_j,  y_{j+1} -= l_j z_j.
//
// Serial parts (dots, both sweeps) run on one thread per sample; everything
// elementwise is spread over the CTA. It is a parity instrument (tests,
// diagnostics), not the throughput path: ~0.5 ms per iteration at n = 4095.
#pragma once
#include "common.cuh"

namespace vqpc {

struct Pcg1dExactParams {
  int n;
  double h;
  const double* kappa;  // samples x (n + 1), row stride ldk
  int64_t ldk;
  const uint8_t* kflag;
  const int32_t* perm;
  const int32_t* labels;
  const double2* lu;  // P x NP {l_j, u_j} (reference factor values)
  int NP;
  int64_t B;
  int64_t out_base;
  int64_t solve_limit;
  double eps;
  int max_iter;
  const int32_t* max_iter_arr;
  int* counter;
  int32_t* iters;
  double* rel;
  uint8_t* status;
  double* x_out;
  double* work;  // per CTA: c (n + 1), x, r, p, z, v (n each)
};

constexpr int PX_T = 128;

// serial natural-order sum of prod[0..n) by one thread
__device__ __forceinline__ double serial_sum(const double* prod, int n) {
  double s = 0.0;
  int j = 0;
  for (; j + 4 <= n; j += 4) {
    const double a = prod[j], b = prod[j + 1], c = prod[j + 2], d = prod[j + 3];
    s = __dadd_rn(s, a);
    s = __dadd_rn(s, b);
    s = __dadd_rn(s, c);
    s = __dadd_rn(s, d);
  }
  for (; j < n; ++j) s = __dadd_rn(s, prod[j]);
  return s;
}

// CSR row j of the 1-D operator times v, in the reference's order
__device__ __forceinline__ double exact_row(const double* c, const double* v, int j, int n) {
  double s = 0.0;
  if (j > 0) s = __dadd_rn(s, __dmul_rn(-c[j], v[j - 1]));
  s = __dadd_rn(s, __dmul_rn(__dadd_rn(c[j], c[j + 1]), v[j]));
  if (j + 1 < n) s = __dadd_rn(s, __dmul_rn(-c[j + 1], v[j + 1]));
  return s;
}

// z = M^{-1} r by one thread (Eigen's triangular solves on the reversed order)
__device__ void exact_apply(const double2* lu, const double* r, double* z, int n) {
  double y = 0.0;
  for (int j = n - 1; j >= 0; --j) {  // L y = P r
    const double2 f = lu[j];
    double t = r[j];
    if (j + 1 < n) t = __dsub_rn(t, __dmul_rn(y, f.x));
    y = __ddiv_rn(t, f.y);
    z[j] = y;
  }
  for (int j = 0; j < n; ++j) {  // L^T w = y, column-oriented
    const double2 f = lu[j];
    const double w = __ddiv_rn(z[j], f.y);
    z[j] = w;
    if (j + 1 < n) z[j + 1] = __dsub_rn(z[j + 1], __dmul_rn(f.x, w));
  }
}

static __global__ void __launch_bounds__(PX_T) pcg1d_exact_kernel(const Pcg1dExactParams prm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* prod = reinterpret_cast<double*>(smem_raw);  // n products
  __shared__ double s_val;
  __shared__ int64_t s_item;
  const int tid = threadIdx.x, n = prm.n;
  double* c = prm.work + static_cast<size_t>(blockIdx.x) * (6 * static_cast<size_t>(n) + 1);
  double* x = c + n + 1;
  double* r = x + n;
  double* p = r + n;
  double* z = p + n;
  double* v = z + n;
  const double h = prm.h;
  // s = serial dot over prod[] after every thread wrote its products; broadcast
  auto reduce = [&]() -> double {
    __syncthreads();
    if (tid == 0) s_val = serial_sum(prod, n);
    __syncthreads();
    return s_val;
  };
  auto precond = [&](const double2* f) {
    __syncthreads();
    if (tid == 0) exact_apply(f, r, z, n);
    __syncthreads();
  };
  for (;;) {
    if (tid == 0) s_item = atomicAdd(prm.counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    __syncthreads();
    if (item >= prm.B) break;
    const int s = prm.perm[item];
    const int64_t gs = prm.out_base + s;
    const int label = prm.labels[s];
    if (label < 0 || prm.kflag[s] || gs >= prm.solve_limit) {
      if (tid == 0) {
        prm.iters[gs] = 0;
        prm.rel[gs] = 0.0;
        prm.status[gs] = gs >= prm.solve_limit ? VQPC_S_NOT_SOLVED
                         : label < 0           ? VQPC_S_INVALID_LATENT
                                               : (prm.kflag[s] & 1) ? VQPC_S_COEFF_OVERFLOW : VQPC_S_INVALID_COEFF;
      }
      continue;
    }
    const double2* f = prm.lu + static_cast<size_t>(label) * prm.NP;
    const double* kap = prm.kappa + static_cast<size_t>(s) * prm.ldk;
    for (int j = tid; j <= n; j += PX_T) c[j] = __ddiv_rn(kap[j], h);  // element stiffness kappa_e / h
    for (int j = tid; j < n; j += PX_T) {
      x[j] = 0.0;
      r[j] = h;
      prod[j] = __dmul_rn(h, h);
    }
    const int max_iter = prm.max_iter_arr ? prm.max_iter_arr[gs] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);
    const double norm_b = __dsqrt_rn(reduce());
    int J = 0;
    double rel_rec = 0.0;
    uint8_t st = VQPC_S_MAX_ITER;
    if (norm_b == 0.0) {
      st = VQPC_S_CONVERGED;
    } else {
      precond(f);
      for (int j = tid; j < n; j += PX_T) {
        p[j] = z[j];
        prod[j] = __dmul_rn(r[j], z[j]);
      }
      double rz = reduce();
      if (!(rz > 0.0)) st = VQPC_S_BREAKDOWN;
      for (int it = 1; st == VQPC_S_MAX_ITER && it <= max_iter; ++it) {
        for (int j = tid; j < n; j += PX_T) {
          const double a = exact_row(c, p, j, n);
          v[j] = a;
          prod[j] = __dmul_rn(p[j], a);
        }
        const double pAp = reduce();
        if (!(pAp > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        const double alpha = __ddiv_rn(rz, pAp);
        for (int j = tid; j < n; j += PX_T) {
          x[j] = __dadd_rn(x[j], __dmul_rn(alpha, p[j]));
          r[j] = __dsub_rn(r[j], __dmul_rn(alpha, v[j]));
        }
        __syncthreads();
        for (int j = tid; j < n; j += PX_T) {
          const double t = __dsub_rn(h, exact_row(c, x, j, n));
          prod[j] = __dmul_rn(t, t);
        }
        const double rel = __ddiv_rn(__dsqrt_rn(reduce()), norm_b);
        J = it;
        rel_rec = rel;
        if (rel < prm.eps) {
          st = VQPC_S_CONVERGED;
          break;
        }
        precond(f);
        for (int j = tid; j < n; j += PX_T) prod[j] = __dmul_rn(r[j], z[j]);
        const double rz_next = reduce();
        if (!(rz_next > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        const double beta = __ddiv_rn(rz_next, rz);
        rz = rz_next;
        for (int j = tid; j < n; j += PX_T) p[j] = __dadd_rn(z[j], __dmul_rn(beta, p[j]));
        __syncthreads();
      }
    }
    if (tid == 0) {
      prm.iters[gs] = J;
      prm.rel[gs] = rel_rec;
      prm.status[gs] = st;
    }
    if (prm.x_out) {
      double* xo = prm.x_out + static_cast<size_t>(gs) * n;
      for (int j = tid; j < n; j += PX_T) xo[j] = x[j];
    }
    __syncthreads();
  }
}

}  // namespace vqpc
