// factor.cuh — kernel (e), 1-D: exact Cholesky factor of every centroid matrix.
//
// Replaces, per centroid p, assemble(centroid_coefficient) -> build_cholesky
// (proj/src/driver.cpp:212-219, solver.cpp:80-111). On the 1-D path graph the
// reference's RCM order is the reversal (solver.cpp:32-70: minimum-degree
// start at row 0, BFS 0..n-1, reversed), so its SimplicialLLT factors from the
// last row up:
//   u_{n-1} = sqrt(A_{n-1,n-1})
//   l_j     = A_{j,j+1} / u_{j+1},   u_j = sqrt(A_jj - l_j * l_j)
// with A_jj = kappa_j/h + kappa_{j+1}/h, A_{j,j+1} = -(kappa_{j+1}/h). Computed
// with __ddiv_rn/__dmul_rn/__dsub_rn/__dsqrt_rn: the same IEEE operations, so
// u and l are bit-identical to the oracle's factor of the same kappa. The
// stored form is the unit-bidiagonal split U = (I+N) D used by pcg1d:
//   n_j = l_j / u_{j+1}  (n_{n-1} = 0),   dinv2_j = 1 / u_j^2;  dead rows {0,0}.
// One thread per centroid (one-time setup; latency-bound by design). With lu_out
// the pass-1 values {l_j, u_j} are kept as well (pcg1d_exact_kernel applies them
// exactly as the reference's SimplicialLLT solve does).
#pragma once
#include "common.cuh"

namespace vqpc {

static __global__ void factor1d_kernel(const double* kappa, int64_t ldk, int P, int n, double h, double2* fac, int NP,
                                int* err, double2* lu_out = nullptr) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double* kp = kappa + static_cast<size_t>(p) * ldk;
  double2* f = fac + static_cast<size_t>(p) * NP;
  // pass 1 (descending): store {l_j, u_j}
  double s_next = __ddiv_rn(kp[n], h);  // s_{j+1} for j = n-1
  double u_next = 0.0;
  bool ok = true;
  for (int j = n - 1; j >= 0; --j) {
    const double s_j = __ddiv_rn(kp[j], h);
    const double diag = __dadd_rn(s_j, s_next);
    double l = 0.0, d;
    if (j == n - 1) {
      d = diag;
    } else {
      l = __ddiv_rn(-s_next, u_next);
      d = __dsub_rn(diag, __dmul_rn(l, l));
    }
    if (!(d > 0.0)) ok = false;
    const double u = __dsqrt_rn(d);
    f[j] = make_double2(l, u);
    if (lu_out) lu_out[static_cast<size_t>(p) * NP + j] = make_double2(l, u);  // reference-order mode
    u_next = u;
    s_next = s_j;
  }
  // pass 2 (ascending): {n_j, dinv2_j}
  for (int j = 0; j < n; ++j) {
    const double2 lu = f[j];
    const double nj = j + 1 < n ? __ddiv_rn(lu.x, f[j + 1].y) : 0.0;
    const double uinv = __drcp_rn(lu.y);
    f[j] = make_double2(nj, __dmul_rn(uinv, uinv));
  }
  for (int j = n; j < NP; ++j) f[j] = make_double2(0.0, 0.0);
  if (!ok) atomicExch(err, 1);
}

// Reference apply of the same factor for a single vector (parity tests):
// z = M_p^{-1} r with the unit-bidiagonal form (one thread, serial).
static __global__ void precond1d_apply_kernel(const double2* fac, int NP, int p, int n, const double* r, double* z) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const double2* f = fac + static_cast<size_t>(p) * NP;
  double y = 0.0;
  for (int j = n - 1; j >= 0; --j) {
    y = fma(-f[j].x, y, r[j]);
    z[j] = y;
  }
  for (int j = 0; j < n; ++j) z[j] *= f[j].y;
  double v = 0.0;
  for (int j = 0; j < n; ++j) {
    const double nl = j > 0 ? f[j - 1].x : 0.0;
    v = fma(-nl, v, z[j]);
    z[j] = v;
  }
}

}  // namespace vqpc
