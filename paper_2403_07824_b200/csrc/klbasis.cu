// klbasis.cu — build_kl_basis (proj/src/field.cpp:22-82) on the device.
//
// The reference forms the dense lumped-Galerkin operator W = M^1/2 C M^1/2
// (n_nodes^2 entries) and calls Eigen's SelfAdjointEigenSolver — infeasible at
// C4's 66,049 nodes. Here the same discrete eigenproblem is solved by
// Lanczos with full reorthogonalisation on the device:
//   * the operator is applied matrix-free: 1-D (element midpoints, w_e = h) by a
//     DGEMV with the N x N kernel matrix; 2-D through the tensor structure of the
//     squared-exponential kernel on the structured node grid,
//     C = sigma^2 C1 (x) C1, so W v = s .* vec(sigma^2 C1 V C1^T) with V = s .* v
//     reshaped side x side (two (r+1)^3 DGEMMs per product; s = sqrt(mass));
//   * every Lanczos vector is orthogonalised against all previous ones twice
//     (classical Gram-Schmidt, DGEMV with the basis block), so the Ritz values of
//     the small tridiagonal T agree with the dense eigensolver's to rounding;
//   * T's eigenpairs come from the implicit QL method on the host (k <= a few
//     hundred), the Ritz vectors from one DGEMM.
// Then the reference's post-processing (field.cpp:48-80): eigenvalues
// descending, the degeneracy cutoff lambda >= 1e-12 lambda_1 (optional, SURVEY
// F5), Phi = v / sqrt(mass), sign: the first entry of largest magnitude positive
// (ties within 1e-9 relative go to the first index, as klbasis.py).
// GEMMs/GEMVs are cuBLAS calls (plain library GEMMs on a one-time setup path).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "vqpc.h"

namespace {

struct KlFail {
  int code;
};

#define KCK(call)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw KlFail{e_ == cudaErrorMemoryAllocation ? VQPC_OUT_OF_MEMORY : VQPC_CUDA_ERROR}; \
  } while (0)
#define KCB(call)                                                \
  do {                                                           \
    if ((call) != CUBLAS_STATUS_SUCCESS) throw KlFail{VQPC_CUDA_ERROR}; \
  } while (0)

template <class T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) { KCK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

// y = scale * s .* y (elementwise), s = sqrt(mass)
__global__ void scale_kernel(double* y, const double* s, double scale, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = scale * (s[i] * y[i]);
}
__global__ void mul_kernel(double* y, const double* x, const double* s, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = s[i] * x[i];
}

// symmetric tridiagonal eigenproblem by the implicit QL method (diagonal d,
// off-diagonal e[i] = T(i, i+1)); Z (k x k, column-major) receives the eigenvectors
bool tridiagonal_ql(std::vector<double>& d, std::vector<double> e, std::vector<double>& Z, int k) {
  Z.assign(static_cast<size_t>(k) * k, 0.0);
  for (int i = 0; i < k; ++i) Z[static_cast<size_t>(i) * k + i] = 1.0;
  e.resize(k, 0.0);
  double tnorm = 0.0;  // deflation floor: off-diagonals below eps * ||T|| are zero (the noise-level
  for (int i = 0; i < k; ++i) tnorm = std::max(tnorm, std::abs(d[i]) + std::abs(e[i]));  // tail of T)
  const double floor_e = 1e-17 * tnorm;
  for (int l = 0; l < k; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < k - 1; ++m) {
        const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
        if (std::abs(e[m]) <= 1e-17 * dd || std::abs(e[m]) <= floor_e) break;
      }
      if (m != l) {
        if (++iter > 1000) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0 ? std::abs(r) : -std::abs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i], b = c * e[i];
          e[i + 1] = (r = std::hypot(f, g));
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          d[i + 1] = g + (p = s * r);
          g = c * r - b;
          double* zi = Z.data() + static_cast<size_t>(i) * k;
          double* zi1 = zi + k;
          for (int q = 0; q < k; ++q) {
            f = zi1[q];
            zi1[q] = s * zi[q] + c * f;
            zi[q] = c * zi[q] - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return true;
}

}  // namespace

extern "C" int vqpc_kl_basis(int device, int dim, int size, double sigma2, double ell, int n_kl, int cutoff,
                             double* eigenvalues_out, double* eigenvectors_out, double* mass_out, int* kept_out) {
  if (!eigenvalues_out || !eigenvectors_out || !kept_out) return VQPC_INVALID_ARGUMENT;
  if (!(sigma2 > 0.0) || !(ell > 0.0)) return VQPC_INVALID_CONFIG;  // "invalid-kernel"
  if (dim != 1 && dim != 2) return VQPC_INVALID_CONFIG;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) return VQPC_NO_DEVICE;
  const int side = dim == 1 ? size : size + 1;
  const int64_t nn = dim == 1 ? size : static_cast<int64_t>(side) * side;
  if (size < 2 || n_kl < 1 || n_kl > nn) return VQPC_INVALID_CONFIG;  // "rank-exceeds-dofs"
  cublasHandle_t hb = nullptr;
  try {
    KCK(cudaSetDevice(device));
    KCB(cublasCreate(&hb));
    // ---- nodes, lumped mass, kernel factor ----------------------------------------
    const double h = 1.0 / size;
    std::vector<double> mass(nn), t(side);
    if (dim == 1) {
      for (int e = 0; e < size; ++e) t[e] = (e + 0.5) * h;  // element midpoints
      std::fill(mass.begin(), mass.end(), h);
    } else {
      for (int a = 0; a < side; ++a) t[a] = a * h;
      // lumped P1 mass of the structured mesh (fem.cpp:132-140): a third of the area of
      // the triangles at each node; each cell {a,b,d},{a,d,c} (a=(cx,cy), d=(cx+1,cy+1))
      const double area = 0.5 * h * h;
      std::vector<double> acc(nn, 0.0);
      for (int cy = 0; cy < size; ++cy)
        for (int cx = 0; cx < size; ++cx) {
          acc[static_cast<size_t>(cy) * side + cx] += 2 * area;
          acc[static_cast<size_t>(cy) * side + cx + 1] += area;
          acc[static_cast<size_t>(cy + 1) * side + cx + 1] += 2 * area;
          acc[static_cast<size_t>(cy + 1) * side + cx] += area;
        }
      for (int64_t i = 0; i < nn; ++i) mass[i] = acc[i] / 3.0;
    }
    std::vector<double> sm(nn);
    for (int64_t i = 0; i < nn; ++i) sm[i] = std::sqrt(mass[i]);
    // C1[a][b] = exp(-(t_a - t_b)^2 / ell^2) (field.cpp:16-20 with the separable factor)
    std::vector<double> C1(static_cast<size_t>(side) * side);
    for (int a = 0; a < side; ++a)
      for (int b = 0; b < side; ++b) {
        const double d = t[a] - t[b];
        C1[static_cast<size_t>(a) * side + b] = std::exp(-(d * d) / (ell * ell));
      }
    Dev<double> dC(C1.size()), dS(nn);
    KCK(cudaMemcpy(dC.p, C1.data(), sizeof(double) * C1.size(), cudaMemcpyHostToDevice));
    KCK(cudaMemcpy(dS.p, sm.data(), sizeof(double) * nn, cudaMemcpyHostToDevice));
    // 1-D: W = sigma2 * diag(s) C1 diag(s) formed once (N x N)
    std::unique_ptr<Dev<double>> dW;
    Dev<double> dV(nn), dT(nn);
    if (dim == 1) {
      std::vector<double> W(C1.size());
      for (int a = 0; a < side; ++a)
        for (int b = 0; b < side; ++b)
          W[static_cast<size_t>(a) * side + b] = sm[a] * (sigma2 * C1[static_cast<size_t>(a) * side + b]) * sm[b];
      dW = std::make_unique<Dev<double>>(W.size());
      KCK(cudaMemcpy(dW->p, W.data(), sizeof(double) * W.size(), cudaMemcpyHostToDevice));
    }
    const unsigned eg = 256, tb = 256;
    auto apply = [&](const double* x, double* y) {  // y = W x
      const double one = 1.0, zero = 0.0;
      if (dim == 1) {
        KCB(cublasDgemv(hb, CUBLAS_OP_N, side, side, &one, dW->p, side, x, 1, &zero, y, 1));  // W symmetric
        return;
      }
      mul_kernel<<<eg, tb>>>(dV.p, x, dS.p, nn);
      // V is side x side with V[iy][ix] at iy*side+ix (row-major) = column-major V^T.
      // Y = C1 V C1^T  <=>  Y^T = C1 V^T C1^T (C1 symmetric): T = V^T C1, Y^T = C1 T (column-major)
      KCB(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, side, side, side, &one, dV.p, side, dC.p, side, &zero, dT.p, side));
      KCB(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, side, side, side, &one, dC.p, side, dT.p, side, &zero, y, side));
      scale_kernel<<<eg, tb>>>(y, dS.p, sigma2, nn);
    };
    // ---- Lanczos with full reorthogonalisation -------------------------------------
    const int k = static_cast<int>(std::min<int64_t>(nn, 3LL * n_kl + 64));
    Dev<double> dQ(static_cast<size_t>(nn) * (k + 1)), dw(nn), dh(k + 1);
    std::vector<double> q0(nn);
    double nrm = 0.0;
    for (int64_t i = 0; i < nn; ++i) {
      q0[i] = (static_cast<double>(vqpc_counter_hash(0x6b6c62617369ull, static_cast<uint64_t>(i), 0) >> 11) + 0.5) *
                  0x1.0p-53 - 0.5;
      nrm += q0[i] * q0[i];
    }
    nrm = std::sqrt(nrm);
    for (auto& v : q0) v /= nrm;
    KCK(cudaMemcpy(dQ.p, q0.data(), sizeof(double) * nn, cudaMemcpyHostToDevice));
    std::vector<double> alpha, beta;
    int steps = 0;
    for (int j = 0; j < k; ++j) {
      double* qj = dQ.p + static_cast<size_t>(j) * nn;
      apply(qj, dw.p);
      // two passes of classical Gram-Schmidt against q_0 .. q_j (alpha_j from the first)
      const double one = 1.0, zero = 0.0, mone = -1.0;
      double aj = 0.0;
      for (int pass = 0; pass < 2; ++pass) {
        KCB(cublasDgemv(hb, CUBLAS_OP_T, static_cast<int>(nn), j + 1, &one, dQ.p, static_cast<int>(nn), dw.p, 1, &zero,
                        dh.p, 1));
        if (pass == 0) KCK(cudaMemcpy(&aj, dh.p + j, sizeof(double), cudaMemcpyDeviceToHost));
        KCB(cublasDgemv(hb, CUBLAS_OP_N, static_cast<int>(nn), j + 1, &mone, dQ.p, static_cast<int>(nn), dh.p, 1, &one,
                        dw.p, 1));
      }
      double bj = 0.0;
      KCB(cublasDnrm2(hb, static_cast<int>(nn), dw.p, 1, &bj));
      alpha.push_back(aj);
      steps = j + 1;
      if (!(bj > 1e-300) || j + 1 == k) break;
      beta.push_back(bj);
      const double inv = 1.0 / bj;
      KCK(cudaMemcpy(dQ.p + static_cast<size_t>(j + 1) * nn, dw.p, sizeof(double) * nn, cudaMemcpyDeviceToDevice));
      KCB(cublasDscal(hb, static_cast<int>(nn), &inv, dQ.p + static_cast<size_t>(j + 1) * nn, 1));
    }
    // ---- Ritz pairs ------------------------------------------------------------------
    std::vector<double> d(alpha), Z;
    std::vector<double> e(beta);
    if (!tridiagonal_ql(d, e, Z, steps)) throw KlFail{VQPC_INVALID_CONFIG};
    std::vector<int> order(steps);
    for (int i = 0; i < steps; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return d[a] > d[b]; });
    const int want = std::min(n_kl, steps);
    std::vector<double> S(static_cast<size_t>(steps) * want);
    for (int c = 0; c < want; ++c)
      std::copy_n(Z.data() + static_cast<size_t>(order[c]) * steps, steps, S.data() + static_cast<size_t>(c) * steps);
    Dev<double> dSm(S.size()), dX(static_cast<size_t>(nn) * want);
    KCK(cudaMemcpy(dSm.p, S.data(), sizeof(double) * S.size(), cudaMemcpyHostToDevice));
    {
      const double one = 1.0, zero = 0.0;
      KCB(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(nn), want, steps, &one, dQ.p,
                      static_cast<int>(nn), dSm.p, steps, &zero, dX.p, static_cast<int>(nn)));
    }
    std::vector<double> X(static_cast<size_t>(nn) * want);
    KCK(cudaMemcpy(X.data(), dX.p, sizeof(double) * X.size(), cudaMemcpyDeviceToHost));
    // ---- the reference's post-processing (field.cpp:48-80) ----------------------------
    const double lead = d[order[0]];
    if (!(lead > 0.0)) throw KlFail{VQPC_INVALID_CONFIG};  // "kl-eigensolve-failed"
    int kept = 0;
    while (kept < want && (cutoff ? d[order[kept]] >= 1e-12 * lead : d[order[kept]] > 0.0)) ++kept;
    for (int c = 0; c < kept; ++c) {
      eigenvalues_out[c] = d[order[c]];
      double* phi = eigenvectors_out + static_cast<size_t>(c) * nn;
      const double* v = X.data() + static_cast<size_t>(c) * nn;
      double amax = 0.0;
      for (int64_t i = 0; i < nn; ++i) {
        phi[i] = v[i] / sm[i];
        amax = std::max(amax, std::abs(phi[i]));
      }
      int64_t imax = 0;
      while (std::abs(phi[imax]) < amax * (1.0 - 1e-9)) ++imax;
      if (phi[imax] < 0.0)
        for (int64_t i = 0; i < nn; ++i) phi[i] = -phi[i];
    }
    if (mass_out) std::copy(mass.begin(), mass.end(), mass_out);
    *kept_out = kept;
    cublasDestroy(hb);
    return VQPC_OK;
  } catch (const KlFail& f) {
    if (hb) cublasDestroy(hb);
    return f.code;
  }
}
