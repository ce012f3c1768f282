// amg_setup.cuh — host part of the SA-AMG preconditioner kind (VQPC_PC_AMG):
// the per-centroid smoothed-aggregation hierarchy (setup (e), once per
// centroid) and its packing into the device layout pcgamg2d.cuh reads.
//
// Restates AmgPreconditioner's constructor (proj/src/amg.cpp:132-197) with the
// reference's defaults (AmgOptions, proj/include/vqp/solver.hpp:35-43):
//   strength |a_ij| >= theta sqrt(a_ii a_jj)            amg.cpp:46-58
//   greedy aggregation, three passes                      amg.cpp:60-105
//   rho(D^-1 A) by 10 power steps from the counter-RNG    amg.cpp:108-124
//   P = (I - (4/3 / rho) D^-1 A) T, T piecewise constant  amg.cpp:157-177
//   A_c = P^T A P (Galerkin), until n <= coarse_size      amg.cpp:179-181
//   dense LL^T of the coarsest operator                   amg.cpp:186-193
// Where the reference hands arithmetic to Eigen, the evaluation order is
// written out: sparse products accumulate every entry
// from its first product in ascending inner index (Eigen's conservative
// sparse product; computed here row-wise, Gustavson order, which visits the
// inner index in the same ascending order); vector norms are serial sums; the
// coarsest factor is a left-looking column Cholesky with sequential
// subtraction in ascending k. The oracle (oracle/src/vqp_oracle.cpp) states
// the same definitions independently; tests compare the hierarchies bit for bit.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "vqpc.h"

namespace vqpc {
namespace amg {

struct Options {
  double theta = 0.08;         // strength_threshold
  double omega = 2.0 / 3.0;    // jacobi_weight
  double damping = 4.0 / 3.0;  // prolongator_damping
  int power_iterations = 10;
  int coarse_size = 64;
  int max_levels = 32;
};

struct Csr {
  int rows = 0, cols = 0;
  std::vector<int> ptr, idx;
  std::vector<double> val;
  int nnz() const { return ptr.empty() ? 0 : ptr[rows]; }
};

struct Level {
  Csr A, P, Pt;                // operator; prolongator (rows x nc) and its transpose (empty on the coarsest)
  std::vector<double> inv_diag;
};

struct Hierarchy {
  std::vector<Level> lv;
  int dense_n = 0;             // > 0: coarsest operator factored densely (row-major L, lower)
  std::vector<double> L;
};

struct NotSpd {};

inline double counter_uniform(uint64_t seed, uint64_t index) {  // uniform_open01(seed, index, 0), rng.hpp:27-31
  return (static_cast<double>(vqpc_counter_hash(seed, index, 0) >> 11) + 0.5) * 0x1.0p-53;
}

inline Csr transpose(const Csr& A) {
  Csr T;
  T.rows = A.cols;
  T.cols = A.rows;
  T.ptr.assign(T.rows + 1, 0);
  for (int e = 0; e < A.nnz(); ++e) ++T.ptr[A.idx[e] + 1];
  for (int r = 0; r < T.rows; ++r) T.ptr[r + 1] += T.ptr[r];
  T.idx.resize(A.nnz());
  T.val.resize(A.nnz());
  std::vector<int> fill(T.ptr.begin(), T.ptr.end() - 1);
  for (int r = 0; r < A.rows; ++r)  // rows ascending: every transposed row lists ascending indices
    for (int e = A.ptr[r]; e < A.ptr[r + 1]; ++e) {
      const int q = fill[A.idx[e]]++;
      T.idx[q] = r;
      T.val[q] = A.val[e];
    }
  return T;
}

// C = X Y, row-wise (Gustavson). Entry (i, j) = X(i,k0) Y(k0,j), then += X(i,k) Y(k,j)
// for the following k in ascending order; every touched entry is stored.
inline Csr multiply(const Csr& X, const Csr& Y) {
  Csr C;
  C.rows = X.rows;
  C.cols = Y.cols;
  C.ptr.assign(C.rows + 1, 0);
  std::vector<double> acc(Y.cols, 0.0);
  std::vector<int> seen(Y.cols, -1), cols;
  for (int i = 0; i < X.rows; ++i) {
    cols.clear();
    for (int e = X.ptr[i]; e < X.ptr[i + 1]; ++e) {
      const int k = X.idx[e];
      const double x = X.val[e];
      for (int f = Y.ptr[k]; f < Y.ptr[k + 1]; ++f) {
        const int j = Y.idx[f];
        const double prod = x * Y.val[f];
        if (seen[j] != i) {
          seen[j] = i;
          acc[j] = prod;
          cols.push_back(j);
        } else {
          acc[j] += prod;
        }
      }
    }
    std::sort(cols.begin(), cols.end());
    for (int j : cols) {
      C.idx.push_back(j);
      C.val.push_back(acc[j]);
    }
    C.ptr[i + 1] = static_cast<int>(C.idx.size());
  }
  return C;
}

inline double diagonal_of(const Csr& A, int i) {
  for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
    if (A.idx[e] == i) return A.val[e];
  return 0.0;
}

// amg.cpp:40-106. strong[i] from row i (|A(i,j)| with the row's own diagonal
// first in the product, as the reference's column sweep evaluates it); pass 2
// weighs candidate j by |A(j, i)| (the reference iterates column i).
inline std::vector<int> aggregate(const Csr& A, const Csr& At, const std::vector<double>& diag, double theta,
                                  int& count) {
  const int n = A.rows;
  std::vector<int> sptr(n + 1, 0), sidx;
  sidx.reserve(A.nnz());
  for (int i = 0; i < n; ++i) {
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
      const int j = A.idx[e];
      if (j != i && std::abs(A.val[e]) >= theta * std::sqrt(diag[i] * diag[j])) sidx.push_back(j);
    }
    sptr[i + 1] = static_cast<int>(sidx.size());
  }
  auto is_strong = [&](int i, int j) { return std::binary_search(sidx.begin() + sptr[i], sidx.begin() + sptr[i + 1], j); };
  std::vector<int> agg(n, -1);
  count = 0;
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    bool untouched = true;
    for (int e = sptr[i]; e < sptr[i + 1] && untouched; ++e) untouched = agg[sidx[e]] < 0;
    if (!untouched) continue;
    agg[i] = count;
    for (int e = sptr[i]; e < sptr[i + 1]; ++e) agg[sidx[e]] = count;
    ++count;
  }
  const std::vector<int> first_pass(agg);
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    int pick = -1;
    double wmax = -1.0;
    for (int e = At.ptr[i]; e < At.ptr[i + 1]; ++e) {
      const int j = At.idx[e];
      if (j == i || first_pass[j] < 0 || !is_strong(i, j)) continue;
      const double w = std::abs(At.val[e]);
      if (w > wmax) {
        wmax = w;
        pick = first_pass[j];
      }
    }
    if (pick >= 0) agg[i] = pick;
  }
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    agg[i] = count;
    for (int e = sptr[i]; e < sptr[i + 1]; ++e)
      if (agg[sidx[e]] < 0) agg[sidx[e]] = count;
    ++count;
  }
  return agg;
}

inline void matvec(const Csr& A, const double* x, double* y) {  // Eigen sparse * dense: 0 + sum, ascending
  for (int i = 0; i < A.rows; ++i) {
    double s = 0.0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) s += A.val[e] * x[A.idx[e]];
    y[i] = s;
  }
}

// amg.cpp:108-124
inline double spectral_radius(const Csr& A, const std::vector<double>& inv_diag, int steps) {
  const int n = A.rows;
  std::vector<double> v(n), w(n);
  for (int i = 0; i < n; ++i) v[i] = counter_uniform(0x5ca1ab1eu, static_cast<uint64_t>(i)) - 0.5;
  double ss = 0.0;
  for (double t : v) ss += t * t;
  const double len = std::sqrt(ss);
  if (len > 0.0)
    for (double& t : v) t /= len;
  double rho = 1.0;
  for (int s = 0; s < steps; ++s) {
    matvec(A, v.data(), w.data());
    double q = 0.0;
    for (int i = 0; i < n; ++i) {
      w[i] = inv_diag[i] * w[i];
      q += w[i] * w[i];
    }
    rho = std::sqrt(q);
    if (!(rho > 0.0)) return 1.0;
    for (int i = 0; i < n; ++i) v[i] = w[i] / rho;
  }
  return rho;
}

// amg.cpp:132-197 for one centroid matrix A0 (throws NotSpd)
inline Hierarchy build(const Csr& A0, const Options& o = {}) {
  Hierarchy H;
  Csr A = A0;
  for (int depth = 0;; ++depth) {
    Level lv;
    const int n = A.rows;
    std::vector<double> diag(n);
    lv.inv_diag.resize(n);
    for (int i = 0; i < n; ++i) {
      diag[i] = diagonal_of(A, i);
      lv.inv_diag[i] = 1.0 / diag[i];
      if (!std::isfinite(lv.inv_diag[i])) throw NotSpd{};
    }
    const bool coarsen = depth + 1 < o.max_levels && n > o.coarse_size;
    int nc = 0;
    std::vector<int> agg;
    Csr At;
    if (coarsen) {
      At = transpose(A);
      agg = aggregate(A, At, diag, o.theta, nc);
    }
    if (!coarsen || nc >= n) {
      lv.A = std::move(A);
      H.lv.push_back(std::move(lv));
      break;
    }
    std::vector<int> agg_size(nc, 0);
    for (int c : agg) ++agg_size[c];
    const double rho = spectral_radius(A, lv.inv_diag, o.power_iterations);
    const double c = o.damping / rho;
    // smoother S = I - c D^-1 A (the pattern of A, the identity where A lacks a diagonal)
    Csr S;
    S.rows = S.cols = n;
    S.ptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      bool diag_done = false;
      for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        const int j = A.idx[e];
        if (!diag_done && j > i) {
          S.idx.push_back(i);
          S.val.push_back(1.0);
          diag_done = true;
        }
        const double x = c * (lv.inv_diag[i] * A.val[e]);
        S.idx.push_back(j);
        S.val.push_back(j == i ? 1.0 - x : 0.0 - x);
        diag_done = diag_done || j == i;
      }
      if (!diag_done) {
        S.idx.push_back(i);
        S.val.push_back(1.0);
      }
      S.ptr[i + 1] = static_cast<int>(S.idx.size());
    }
    // tentative prolongator T: row i = (agg_i, 1/sqrt(|agg_i|))
    Csr T;
    T.rows = n;
    T.cols = nc;
    T.ptr.resize(n + 1);
    T.idx.resize(n);
    T.val.resize(n);
    for (int i = 0; i < n; ++i) {
      T.ptr[i] = i;
      T.idx[i] = agg[i];
      T.val[i] = 1.0 / std::sqrt(static_cast<double>(agg_size[agg[i]]));
    }
    T.ptr[n] = n;
    lv.P = multiply(S, T);
    lv.Pt = transpose(lv.P);
    Csr Ac = multiply(multiply(lv.Pt, A), lv.P);
    lv.A = std::move(A);
    H.lv.push_back(std::move(lv));
    A = std::move(Ac);
  }
  const Csr& Ac = H.lv.back().A;
  const int nc = Ac.rows;
  if (nc <= o.coarse_size || H.lv.size() > 1) {
    H.dense_n = nc;
    std::vector<double> D(static_cast<size_t>(nc) * nc, 0.0);  // lower triangle of the coarsest operator
    for (int i = 0; i < nc; ++i)
      for (int e = Ac.ptr[i]; e < Ac.ptr[i + 1]; ++e)
        if (Ac.idx[e] <= i) D[static_cast<size_t>(i) * nc + Ac.idx[e]] = Ac.val[e];
    H.L.assign(D.size(), 0.0);
    double* L = H.L.data();
    for (int j = 0; j < nc; ++j) {
      double d = D[static_cast<size_t>(j) * nc + j];
      for (int k = 0; k < j; ++k) d -= L[static_cast<size_t>(j) * nc + k] * L[static_cast<size_t>(j) * nc + k];
      if (!(d > 0.0)) throw NotSpd{};
      const double ljj = std::sqrt(d);
      L[static_cast<size_t>(j) * nc + j] = ljj;
      for (int i = j + 1; i < nc; ++i) {
        double s = D[static_cast<size_t>(i) * nc + j];
        for (int k = 0; k < j; ++k) s -= L[static_cast<size_t>(i) * nc + k] * L[static_cast<size_t>(j) * nc + k];
        L[static_cast<size_t>(i) * nc + j] = s / ljj;
      }
    }
  }
  return H;
}

}  // namespace amg
}  // namespace vqpc
