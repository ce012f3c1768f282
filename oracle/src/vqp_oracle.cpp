// =============================================================================
// vqp_oracle.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// CPU restatement of the reference library `vqp` (arXiv 2403.07824,
// /root/reference/proj) along the Monte-Carlo sample -> realise -> assign ->
// solve hot path. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.
//
// Parity anchors:
//  * rng/counter hash is bit-identical to proj/include/vqp/rng.hpp:8-31 and is
//    pinned against oracle/_ref (the reference header compiled here).
//  * The normal quantile replaces Boost.Math (absent; proj/src/rng.cpp:3):
//    A&S 26.2.23 start + 3 Halley steps on erfc. Exact xi bits are therefore
//    "parity unpinned" vs Boost; both sides consume the same saved xi arrays.
//  * assign / kmeans / grid are checked bit-for-bit against the reference's own
//    proj/src/quantizer.cpp compiled into oracle/_ref.
//  * 2-D assembly is checked against the reference's own proj/src/fem.cpp.
//  * pcg follows proj/src/solver.cpp:186-245 operation for operation; the
//    Eigen SimplicialLLT factor (solver.cpp:80-111) is restated as an
//    envelope LL^T after the same RCM permutation (solver.cpp:32-70); for the
//    1-D tridiagonal systems this is the identical arithmetic.
//  * The 1-D model, the sign grid and IC(0) are not in the reference; they are
//    defined in SURVEY.md Appendix A and restated here (parity vs the GPU only).
//
// Build: g++ -O3 -DNDEBUG -std=gnu++20 -ffp-contract=off (no -march), matching
// the reference's Release build (proj/CMakeLists.txt:6-8) so that no FMA
// contraction changes the rounding of serial sums.
// =============================================================================
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <numbers>
#include <queue>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace vqpo {

// ---- error codes (same table as include/vqpc.h; duplicated so the oracle is
// self-contained) --------------------------------------------------------------
enum Code : int {
  OK = 0,
  INVALID_LATENT = 1,        // quantizer.cpp:135-138
  INVALID_COEFFICIENT = 2,   // fem.cpp:216-219
  COEFFICIENT_OVERFLOW = 3,  // field.cpp:141-142
  NOT_SPD = 4,               // solver.cpp:96
  PCG_BREAKDOWN = 5,         // solver.cpp:207,214,238
  INVALID_TOLERANCE = 6,     // solver.cpp:190
  MODE_COUNT_OUT_OF_RANGE = 7,
  INVALID_CODEBOOK = 8,
  INSUFFICIENT_SAMPLES = 9,
  INVALID_CONFIG = 10,
  INVALID_ARGUMENT = 11,
};

struct Err : std::runtime_error {
  int code;
  explicit Err(int c) : std::runtime_error("vqp-oracle"), code(c) {}
};

// per-sample status (Appendix B classes)
enum Status : uint8_t {
  ST_CONVERGED = 0,
  ST_MAX_ITER = 1,
  ST_BREAKDOWN = 2,
  ST_COEFF_OVERFLOW = 3,
  ST_INVALID_LATENT = 4,
  ST_INVALID_COEFF = 5,
};

// ---- rng: proj/include/vqp/rng.hpp:8-31 ------------------------------------
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static inline uint64_t counter_hash(uint64_t seed, uint64_t index, uint64_t comp) {
  uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ull);
  h = mix64(h ^ mix64(index + 0x6a09e667f3bcc909ull));
  return mix64(h ^ mix64(comp + 0xbb67ae8584caa73bull));
}
static inline double uniform_open01(uint64_t seed, uint64_t index, uint64_t comp) {
  const uint64_t bits = counter_hash(seed, index, comp) >> 11;
  return (static_cast<double>(bits) + 0.5) * 0x1.0p-53;
}

// normal CDF, quantizer.cpp:15-17
static inline double normal_cdf(double x) {
  return 0.5 * std::erfc(-x / std::numbers::sqrt2);
}

// Boost-free inverse normal CDF (replaces boost::math::quantile, rng.cpp:9-11,
// quantizer.cpp:19-23). Start: Abramowitz & Stegun 26.2.23 (|err| < 4.5e-4),
// then three Halley steps on F(z) - q with F from erfc.
static double normal_quantile(double p) {
  if (!(p > 0.0 && p < 1.0)) throw Err(INVALID_LATENT);
  const double q = p < 0.5 ? p : 1.0 - p;  // exact for p >= 0.5
  const double t = std::sqrt(-2.0 * std::log(q));
  double z = -(t - (2.515517 + t * (0.802853 + t * 0.010328)) /
                       (1.0 + t * (1.432788 + t * (0.189269 + t * 0.001308))));
  const double sqrt2pi = std::sqrt(2.0 * std::numbers::pi);
  for (int it = 0; it < 3; ++it) {
    // central region: erf form keeps relative accuracy of F(z) - q near z = 0
    const double e = q > 0.25 ? 0.5 * std::erf(z / std::numbers::sqrt2) - (q - 0.5)
                              : normal_cdf(z) - q;
    const double u = e * sqrt2pi * std::exp(0.5 * z * z);
    z = z - u / (1.0 + 0.5 * z * u);
  }
  return p < 0.5 ? z : -z;
}

static inline double gaussian_draw(uint64_t seed, uint64_t index, uint64_t comp) {
  return normal_quantile(uniform_open01(seed, index, comp));
}

// ---- threads: driver.cpp:143-162 (slots claimed via an atomic counter; each
// slot writes only its own outputs) -------------------------------------------
static void parallel_for_slots(long count, int threads, const std::function<void(long)>& fn) {
  threads = std::max<long>(1, std::min<long>(threads, count));
  if (threads <= 1) {
    for (long s = 0; s < count; ++s) fn(s);
    return;
  }
  std::atomic<long> next{0};
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) {
    pool.emplace_back([&]() {
      for (;;) {
        const long s = next.fetch_add(1);
        if (s >= count) return;
        fn(s);
      }
    });
  }
  for (auto& t : pool) t.join();
}

// ---- field: lift (field.cpp:113-125) and transport (field.cpp:138-145) -----
// evecs is mode-major (n_kl x n_nodes, field.hpp:25).
static void lift(const double* evals, const double* evecs, int n_nodes, const double* xi,
                 int m, double* h) {
  std::fill(h, h + n_nodes, 0.0);
  for (int k = 0; k < m; ++k) {
    const double w = std::sqrt(evals[k]) * xi[k];
    if (w == 0.0) continue;
    const double* phi = evecs + static_cast<size_t>(k) * n_nodes;
    for (int i = 0; i < n_nodes; ++i) h[i] += w * phi[i];
  }
}
static void transport(double* v, int n) {
  for (int i = 0; i < n; ++i) {
    v[i] = std::exp(v[i]);
    if (!std::isfinite(v[i])) throw Err(COEFFICIENT_OVERFLOW);
  }
}

// ---- sparse matrices: fem.hpp:45-72, matvec fem.cpp:142-148 -----------------
struct Csr {
  int n = 0;
  std::vector<int> row_ptr, col;
  std::vector<double> val;
  void matvec(const double* x, double* y) const {
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s += val[k] * x[col[k]];
      y[i] = s;
    }
  }
  double at(int i, int j) const {
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
      if (col[k] == j) return val[k];
    return 0.0;
  }
};
struct System {
  Csr A;
  std::vector<double> b;
};

// Scattered (i, j, v) contributions merged per row in column order; duplicate
// columns are summed in insertion order (the reference's SparseBuilder,
// fem.cpp:177-211, sums them in std::sort order; the two agree to rounding,
// checked against oracle/_ref in tests).
struct RowAccumulator {
  int n;
  std::vector<std::vector<std::pair<int, double>>> rows;
  explicit RowAccumulator(int n_) : n(n_), rows(n_) {}
  void add(int i, int j, double v) {
    auto& r = rows[i];
    for (auto& e : r)
      if (e.first == j) {
        e.second += v;
        return;
      }
    r.emplace_back(j, v);
  }
  Csr finish() {
    Csr A;
    A.n = n;
    A.row_ptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      std::stable_sort(rows[i].begin(), rows[i].end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      A.row_ptr[i + 1] = A.row_ptr[i] + static_cast<int>(rows[i].size());
    }
    for (int i = 0; i < n; ++i)
      for (auto& e : rows[i]) {
        A.col.push_back(e.first);
        A.val.push_back(e.second);
      }
    return A;
  }
};

static void check_coefficient(const double* kappa, int nn) {
  for (int i = 0; i < nn; ++i)
    if (!(kappa[i] > 0.0) || !std::isfinite(kappa[i])) throw Err(INVALID_COEFFICIENT);
}

// The reference's SparseBuilder (fem.cpp:177-211) operation for operation: every
// contribution is appended in insertion order, each row is ordered with std::sort
// on the column (not stable: for rows of more than 16 entries libstdc++'s
// introsort permutes equal columns), and duplicates are summed in that order,
// the first one initialising the entry. Used for the 2-D assembly so the CSR
// values are bit-identical to the reference's (same standard library).
struct RefSparseBuilder {
  int n;
  std::vector<std::vector<std::pair<int, double>>> rows;
  explicit RefSparseBuilder(int n_) : n(n_), rows(n_) {}
  void add(int i, int j, double v) { rows[i].emplace_back(j, v); }
  Csr finish() {
    Csr A;
    A.n = n;
    A.row_ptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      auto row = rows[i];
      std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      int last = -1;
      for (const auto& [j, v] : row) {
        if (j != last) {
          A.col.push_back(j);
          A.val.push_back(v);
          last = j;
        } else {
          A.val.back() += v;
        }
      }
      A.row_ptr[i + 1] = static_cast<int>(A.col.size());
    }
    return A;
  }
};

// 1-D model: N elements of length h = 1/N, coefficient per
// element (midpoint value), unknowns at interior nodes 1..N-1 numbered 0..N-2.
static System assemble_1d(int N, const double* kappa) {
  if (N < 2) throw Err(INVALID_CONFIG);
  check_coefficient(kappa, N);
  const int n = N - 1;
  const double h = 1.0 / N;
  RowAccumulator acc(n);
  for (int e = 0; e < N; ++e) {
    const double s = kappa[e] / h;  // element stiffness kappa_e / h * [1 -1; -1 1]
    const int gl = e - 1, gr = e;   // unknowns of nodes e and e+1 (-1 / n: Dirichlet)
    const bool il = gl >= 0, ir = gr < n;
    if (il) acc.add(gl, gl, s);
    if (il && ir) acc.add(gl, gr, -s);
    if (ir && il) acc.add(gr, gl, -s);
    if (ir) acc.add(gr, gr, s);
  }
  System sys;
  sys.A = acc.finish();
  sys.b.assign(n, h);  // int phi_j = h/2 + h/2 over its two elements
  return sys;
}

// 2-D structured mesh (make_mesh, fem.cpp:53-81): (r+1)^2 nodes, node id =
// iy*(r+1)+ix, each cell split along the a-d diagonal into {a,b,d},{a,d,c};
// interior dofs numbered in node order (fem.cpp:28-42). Assembly restates
// fem.cpp:213-256 (kbar = vertex mean, local stiffness kbar/(4 area)(bb+cc)).
static System assemble_2d(int r, const double* kappa) {
  if (r < 2) throw Err(INVALID_CONFIG);
  const int side = r + 1, nn = side * side;
  check_coefficient(kappa, nn);
  const double h = 1.0 / r;
  std::vector<int> interior(nn, -1);
  int n = 0;
  for (int iy = 0; iy < side; ++iy)
    for (int ix = 0; ix < side; ++ix)
      if (ix > 0 && iy > 0 && ix < r && iy < r) interior[iy * side + ix] = n++;
  auto X = [&](int id) { return (id % side) * h; };
  auto Y = [&](int id) { return (id / side) * h; };
  RefSparseBuilder acc(n);
  std::vector<double> area_sum(nn, 0.0);
  for (int cy = 0; cy < r; ++cy)
    for (int cx = 0; cx < r; ++cx) {
      const int a = cy * side + cx, b = a + 1, c = (cy + 1) * side + cx, d = c + 1;
      const int tris[2][3] = {{a, b, d}, {a, d, c}};
      for (const auto& t : tris) {
        const double x0 = X(t[0]), y0 = Y(t[0]), x1 = X(t[1]), y1 = Y(t[1]);
        const double x2 = X(t[2]), y2 = Y(t[2]);
        const double area = 0.5 * ((x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0));
        const double bb[3] = {y1 - y2, y2 - y0, y0 - y1};
        const double cc[3] = {x2 - x1, x0 - x2, x1 - x0};
        const double kbar = (kappa[t[0]] + kappa[t[1]] + kappa[t[2]]) / 3.0;
        const double scale = kbar / (4.0 * area);
        for (int i = 0; i < 3; ++i) {
          const int gi = interior[t[i]];
          if (gi < 0) continue;
          for (int j = 0; j < 3; ++j) {
            const int gj = interior[t[j]];
            if (gj < 0) continue;
            acc.add(gi, gj, scale * (bb[i] * bb[j] + cc[i] * cc[j]));
          }
        }
        for (int v : t) area_sum[v] += area;
      }
    }
  System sys;
  sys.A = acc.finish();
  sys.b.assign(n, 0.0);
  for (int id = 0; id < nn; ++id)
    if (interior[id] >= 0) sys.b[interior[id]] = area_sum[id] / 3.0;
  return sys;
}

// ---- preconditioners: interface solver.hpp:13-20 ----------------------------
struct Preconditioner {
  virtual ~Preconditioner() = default;
  virtual void apply(const double* r, double* z) const = 0;
  virtual const char* kind() const = 0;
  int built_from = -1;
};

struct IdentityPreconditioner final : Preconditioner {
  int n;
  explicit IdentityPreconditioner(int n_) : n(n_) {}
  void apply(const double* r, double* z) const override { std::copy(r, r + n, z); }
  const char* kind() const override { return "identity"; }
};

// RCM (solver.cpp:32-70): BFS from a minimum-degree start in each component,
// neighbours visited by increasing (degree, index), final order reversed.
static std::vector<int> rcm_permutation(const Csr& A) {
  const int n = A.n;
  std::vector<int> degree(n), by_degree(n), order;
  for (int i = 0; i < n; ++i) degree[i] = A.row_ptr[i + 1] - A.row_ptr[i];
  for (int i = 0; i < n; ++i) by_degree[i] = i;
  auto less = [&](int a, int b) { return degree[a] != degree[b] ? degree[a] < degree[b] : a < b; };
  std::sort(by_degree.begin(), by_degree.end(), less);
  std::vector<char> seen(n, 0);
  std::vector<int> nb;
  order.reserve(n);
  for (int s : by_degree) {
    if (seen[s]) continue;
    seen[s] = 1;
    std::queue<int> q;
    q.push(s);
    while (!q.empty()) {
      const int u = q.front();
      q.pop();
      order.push_back(u);
      nb.clear();
      for (int k = A.row_ptr[u]; k < A.row_ptr[u + 1]; ++k) {
        const int v = A.col[k];
        if (v != u && !seen[v]) {
          seen[v] = 1;
          nb.push_back(v);
        }
      }
      std::sort(nb.begin(), nb.end(), less);
      for (int v : nb) q.push(v);
    }
  }
  std::reverse(order.begin(), order.end());
  return order;  // order[k] = original row of permuted row k
}

// Exact Cholesky with RCM ordering (solver.cpp:80-111). The permuted matrix
// B = P A P^T is factored row by row over its envelope; for each row k the
// off-diagonal L_kl = (B_kl - sum_j L_kj L_lj) / L_ll and the pivot
// L_kk = sqrt(B_kk - sum_j L_kj^2) (Eigen SimplicialLLT's up-looking rows; on
// tridiagonal matrices the arithmetic is identical). Solves follow Eigen's
// sparse triangular solves (SimplicialCholeskyBase::_solve_impl): forward with
// the column-major lower factor (each y_k receives its column contributions in
// increasing column order, then the division by the pivot), backward with the
// row-major upper view L^T (row by row from the bottom, each row's stored
// entries in increasing column order).
struct CholeskyPreconditioner final : Preconditioner {
  int n = 0, W = 0;
  std::vector<int> perm, first;    // envelope start per permuted row
  std::vector<size_t> start;       // offset of row k in L (entries first[k]..k)
  std::vector<double> L;
  explicit CholeskyPreconditioner(const Csr& A) : n(A.n) {
    perm = rcm_permutation(A);
    std::vector<int> inv(n);
    for (int k = 0; k < n; ++k) inv[perm[k]] = k;
    first.assign(n, 0);
    for (int k = 0; k < n; ++k) {
      int f = k;
      const int i = perm[k];
      for (int e = A.row_ptr[i]; e < A.row_ptr[i + 1]; ++e) f = std::min(f, inv[A.col[e]]);
      first[k] = f;
    }
    start.assign(n + 1, 0);
    for (int k = 0; k < n; ++k) start[k + 1] = start[k] + static_cast<size_t>(k - first[k] + 1);
    for (int k = 0; k < n; ++k) W = std::max(W, k - first[k]);
    L.assign(start[n], 0.0);
    for (int k = 0; k < n; ++k) {
      double* Lk = L.data() + start[k] - first[k];  // Lk[l] = L(k, l)
      const int i = perm[k];
      for (int e = A.row_ptr[i]; e < A.row_ptr[i + 1]; ++e) {
        const int l = inv[A.col[e]];
        if (l <= k) Lk[l] = A.val[e];
      }
      double d = Lk[k];
      for (int l = first[k]; l < k; ++l) {
        const double* Ll = L.data() + start[l] - first[l];
        double s = Lk[l];
        for (int j = std::max(first[k], first[l]); j < l; ++j) s -= Lk[j] * Ll[j];
        const double lkl = s / Ll[l];
        Lk[l] = lkl;
        d -= lkl * lkl;
      }
      if (!(d > 0.0)) throw Err(NOT_SPD);
      Lk[k] = std::sqrt(d);
    }
  }
  void apply(const double* r, double* z) const override {
    std::vector<double> y(n);
    for (int k = 0; k < n; ++k) y[k] = r[perm[k]];
    for (int k = 0; k < n; ++k) {  // L y = r_perm
      const double* Lk = L.data() + start[k] - first[k];
      double t = y[k];
      for (int j = first[k]; j < k; ++j) t -= y[j] * Lk[j];
      y[k] = t / Lk[k];
    }
    // L^T z = y as Eigen evaluates it: SimplicialLLT::solve applies matrixU() =
    // L.adjoint(), an upper-triangular ROW-major view of the column-major factor, so
    // the sparse triangular solve goes row by row from the bottom: z_i = (y_i -
    // L(j1,i) z_j1 - L(j2,i) z_j2 - ...) / L(i,i) over the stored column i of L in
    // ascending j (sequential subtraction). Row j holds column i iff first[j] <= i,
    // and j - first[j] <= W bounds the scan.
    for (int i = n - 1; i >= 0; --i) {
      double t = y[i];
      const int jmax = std::min(n - 1, i + W);
      for (int j = i + 1; j <= jmax; ++j) {
        if (first[j] > i) continue;
        t -= L[start[j] - first[j] + i] * y[j];
      }
      y[i] = t / L[start[i] - first[i] + i];
    }
    for (int k = 0; k < n; ++k) z[perm[k]] = y[k];
  }
  const char* kind() const override { return "cholesky"; }
};

// IC(0) of the 2-D P1 stiffness (new). Natural interior
// ordering, 5-point pattern. Root-free form M = (D + L_A) D^{-1} (D + L_A^T)
// with D_i = a_ii - a_iW^2/D_W - a_iS^2/D_S. The NE/SW stored zeros get no fill.
struct IC0Preconditioner final : Preconditioner {
  int m = 0, n = 0;  // m = r-1 interior nodes per row
  std::vector<double> D, aW, aS, aE, aN;
  IC0Preconditioner(const Csr& A, int r) : m(r - 1), n(A.n) {
    if (n != m * m) throw Err(INVALID_CONFIG);
    D.assign(n, 0.0);
    aW.assign(n, 0.0);
    aS.assign(n, 0.0);
    aE.assign(n, 0.0);
    aN.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
      const int ix = i % m, iy = i / m;
      if (ix > 0) aW[i] = A.at(i, i - 1);
      if (iy > 0) aS[i] = A.at(i, i - m);
      if (ix < m - 1) aE[i] = A.at(i, i + 1);
      if (iy < m - 1) aN[i] = A.at(i, i + m);
      double t = A.at(i, i);
      if (ix > 0) t -= aW[i] * aW[i] / D[i - 1];
      if (iy > 0) t -= aS[i] * aS[i] / D[i - m];
      if (!(t > 0.0)) throw Err(NOT_SPD);
      D[i] = t;
    }
  }
  void apply(const double* r, double* z) const override {
    for (int i = 0; i < n; ++i) {  // (D + L_A) y = r
      const int ix = i % m, iy = i / m;
      double t = r[i];
      if (ix > 0) t -= aW[i] * z[i - 1];
      if (iy > 0) t -= aS[i] * z[i - m];
      z[i] = t / D[i];
    }
    for (int i = n - 1; i >= 0; --i) {  // (D + L_A^T) z = D y
      const int ix = i % m, iy = i / m;
      double t = 0.0;
      if (ix < m - 1) t += aE[i] * z[i + 1];
      if (iy < m - 1) t += aN[i] * z[i + m];
      z[i] = z[i] - t / D[i];
    }
  }
  const char* kind() const override { return "ic0"; }
};

// ---- SA-AMG (amg.cpp:40-230; the reference's default kind, driver.hpp:36) ----
// Restated operation for operation where the reference's arithmetic is its own
// (strength test, aggregation passes, power iteration seed, damping constant),
// and with Eigen's evaluation orders written out where it delegates to Eigen:
//  * sparse * dense into a fresh vector: per row, sum from the first product in
//    ascending column order (col-major scatter, amg.cpp:114, 206, 223);
//  * `r - A x` assigned to a vector (amg.cpp:219): Eigen rewrites it to
//    res = r; res -= A x, i.e. per row r_i - a_ij1 x_j1 - a_ij2 x_j2 - ...;
//  * `x += P c` (amg.cpp:221): x_i += P_ik c_k in ascending k;
//  * P^T v (amg.cpp:220): per coarse row, sum over the fine rows in ascending order;
//  * sparse * sparse (amg.cpp:177, 179): Eigen's conservative product, every
//    result entry the first product then += in ascending inner index, every
//    touched entry stored (explicit zeros included);
//  * norms (v.normalize(), w.norm()): serial sums (Eigen vectorises them:
//    parity with Eigen's bits is unpinned there, as everywhere Eigen computes);
//  * the coarsest direct solve (Eigen LLT / SimplicialLLT, amg.cpp:186-193):
//    a dense column Cholesky, left-looking with sequential subtraction in
//    ascending k, and column-oriented forward (k ascending) / backward (k
//    descending) substitution — the order the GPU's warp solve reproduces.
struct AmgOptions {
  double theta = 0.08;           // strength_threshold (solver.hpp:36)
  double omega = 2.0 / 3.0;      // jacobi_weight
  double damping = 4.0 / 3.0;    // prolongator_damping
  int power_iterations = 10;
  int coarse_size = 64;
  int max_levels = 32;
};

// Transpose of an (n x ncols) CSR: row j lists column j's entries in ascending row order.
static Csr csr_transpose(const Csr& A, int ncols) {
  Csr T;
  T.n = ncols;
  T.row_ptr.assign(ncols + 1, 0);
  for (int k = 0; k < A.row_ptr[A.n]; ++k) T.row_ptr[A.col[k] + 1]++;
  for (int j = 0; j < ncols; ++j) T.row_ptr[j + 1] += T.row_ptr[j];
  T.col.resize(A.col.size());
  T.val.resize(A.val.size());
  std::vector<int> pos(T.row_ptr.begin(), T.row_ptr.end() - 1);
  for (int i = 0; i < A.n; ++i)
    for (int k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
      const int p = pos[A.col[k]]++;
      T.col[p] = i;
      T.val[p] = A.val[k];
    }
  return T;
}

// Eigen's conservative sparse product C = A B (A: n x m by rows, B: m x q by
// rows), column-major semantics: C(i, j) = sum over k ascending of A(i, k) B(k, j),
// the first product assigned. Computed here from B's columns (Bt) and A's
// columns (At): for column j, for k ascending in B(:, j), for i in A(:, k).
static Csr spgemm_eigen(const Csr& At, int n, const Csr& Bt) {
  const int q = Bt.n;
  std::vector<std::vector<std::pair<int, double>>> cols(q);
  std::vector<double> vals(n, 0.0);
  std::vector<char> mask(n, 0);
  std::vector<int> touched;
  for (int j = 0; j < q; ++j) {
    touched.clear();
    for (int e = Bt.row_ptr[j]; e < Bt.row_ptr[j + 1]; ++e) {
      const int k = Bt.col[e];
      const double y = Bt.val[e];
      for (int f = At.row_ptr[k]; f < At.row_ptr[k + 1]; ++f) {
        const int i = At.col[f];
        const double x = At.val[f];
        if (!mask[i]) {
          mask[i] = 1;
          vals[i] = x * y;
          touched.push_back(i);
        } else {
          vals[i] += x * y;
        }
      }
    }
    std::sort(touched.begin(), touched.end());
    for (int i : touched) {
      cols[j].push_back({i, vals[i]});
      mask[i] = 0;
    }
  }
  // assemble by rows (n x q)
  Csr C;
  C.n = n;
  C.row_ptr.assign(n + 1, 0);
  for (int j = 0; j < q; ++j)
    for (auto& e : cols[j]) C.row_ptr[e.first + 1]++;
  for (int i = 0; i < n; ++i) C.row_ptr[i + 1] += C.row_ptr[i];
  C.col.resize(C.row_ptr[n]);
  C.val.resize(C.row_ptr[n]);
  std::vector<int> pos(C.row_ptr.begin(), C.row_ptr.end() - 1);
  for (int j = 0; j < q; ++j)
    for (auto& e : cols[j]) {
      const int p = pos[e.first]++;
      C.col[p] = j;
      C.val[p] = e.second;
    }
  return C;
}

// greedy aggregation over the strength graph (amg.cpp:40-106)
static std::vector<int> amg_aggregate(const Csr& A, const Csr& At, const std::vector<double>& diag, double theta,
                                      int& count) {
  const int n = A.n;
  std::vector<std::vector<int>> strong(n);
  for (int i = 0; i < n; ++i)
    for (int k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
      const int j = A.col[k];
      if (j == i) continue;
      if (std::abs(A.val[k]) >= theta * std::sqrt(diag[i] * diag[j])) strong[i].push_back(j);
    }  // row i's columns ascend, so strong[i] is already sorted (amg.cpp:56)
  std::vector<int> agg(n, -1);
  count = 0;
  for (int i = 0; i < n; ++i) {  // pass 1
    if (agg[i] >= 0) continue;
    bool free = true;
    for (int j : strong[i])
      if (agg[j] >= 0) {
        free = false;
        break;
      }
    if (!free) continue;
    agg[i] = count;
    for (int j : strong[i]) agg[j] = count;
    ++count;
  }
  const std::vector<int> pass1 = agg;
  for (int i = 0; i < n; ++i) {  // pass 2: column i of A (InnerIterator over column i)
    if (agg[i] >= 0) continue;
    int best = -1;
    double best_w = -1.0;
    for (int k = At.row_ptr[i]; k < At.row_ptr[i + 1]; ++k) {
      const int j = At.col[k];
      if (j == i || pass1[j] < 0) continue;
      if (!std::binary_search(strong[i].begin(), strong[i].end(), j)) continue;
      const double w = std::abs(At.val[k]);
      if (w > best_w) {
        best_w = w;
        best = pass1[j];
      }
    }
    if (best >= 0) agg[i] = best;
  }
  for (int i = 0; i < n; ++i) {  // pass 3
    if (agg[i] >= 0) continue;
    agg[i] = count;
    for (int j : strong[i])
      if (agg[j] < 0) agg[j] = count;
    ++count;
  }
  return agg;
}

static double amg_spectral_radius(const Csr& A, const std::vector<double>& inv_diag, int iterations) {
  const int n = A.n;
  std::vector<double> v(n), w(n);
  for (int i = 0; i < n; ++i) v[i] = uniform_open01(0x5ca1ab1eu, static_cast<uint64_t>(i), 0) - 0.5;
  double nrm = 0.0;
  for (int i = 0; i < n; ++i) nrm += v[i] * v[i];
  nrm = std::sqrt(nrm);
  if (nrm > 0.0)
    for (int i = 0; i < n; ++i) v[i] /= nrm;
  double rho = 1.0;
  for (int it = 0; it < iterations; ++it) {
    A.matvec(v.data(), w.data());
    for (int i = 0; i < n; ++i) w[i] = inv_diag[i] * w[i];
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += w[i] * w[i];
    rho = std::sqrt(s);
    if (!(rho > 0.0)) return 1.0;
    for (int i = 0; i < n; ++i) v[i] = w[i] / rho;
  }
  return rho;
}

struct AmgLevel {
  Csr A;                     // this level's operator (by rows)
  std::vector<double> inv_diag;
  Csr P, Pt;                 // prolongator (n x nc) by rows, and by columns; empty on the coarsest
  int nc = 0;
};

struct AmgPreconditioner final : Preconditioner {
  AmgOptions opt;
  std::vector<AmgLevel> levels;
  int dense_n = 0;           // > 0: dense Cholesky of the coarsest operator
  std::vector<double> Lc;    // dense_n x dense_n, row-major, lower triangle

  explicit AmgPreconditioner(const Csr& A_in, const AmgOptions& o = {}) : opt(o) {
    Csr A = A_in;
    for (int depth = 0;; ++depth) {
      AmgLevel lv;
      lv.A = A;
      const int n = A.n;
      std::vector<double> diag(n, 0.0);
      for (int i = 0; i < n; ++i) diag[i] = A.at(i, i);
      lv.inv_diag.resize(n);
      for (int i = 0; i < n; ++i) {
        lv.inv_diag[i] = 1.0 / diag[i];
        if (!std::isfinite(lv.inv_diag[i])) throw Err(NOT_SPD);
      }
      const bool can_coarsen = depth + 1 < opt.max_levels && n > opt.coarse_size;
      if (!can_coarsen) {
        levels.push_back(std::move(lv));
        break;
      }
      const Csr At = csr_transpose(A, n);
      int nc = 0;
      const std::vector<int> agg = amg_aggregate(A, At, diag, opt.theta, nc);
      if (nc >= n) {
        levels.push_back(std::move(lv));
        break;
      }
      std::vector<int> size(nc, 0);
      for (int i = 0; i < n; ++i) size[agg[i]] += 1;
      // tentative prolongator T (n x nc), by columns: column c = aggregate c's rows ascending
      Csr Tt;
      Tt.n = nc;
      Tt.row_ptr.assign(nc + 1, 0);
      for (int i = 0; i < n; ++i) Tt.row_ptr[agg[i] + 1]++;
      for (int c = 0; c < nc; ++c) Tt.row_ptr[c + 1] += Tt.row_ptr[c];
      Tt.col.resize(n);
      Tt.val.resize(n);
      {
        std::vector<int> pos(Tt.row_ptr.begin(), Tt.row_ptr.end() - 1);
        for (int i = 0; i < n; ++i) {
          const int p = pos[agg[i]]++;
          Tt.col[p] = i;
          Tt.val[p] = 1.0 / std::sqrt(static_cast<double>(size[agg[i]]));
        }
      }
      const double rho = amg_spectral_radius(A, lv.inv_diag, opt.power_iterations);
      // S = I - (damping / rho) (D^{-1} A), the pattern of A plus the diagonal
      const double c = opt.damping / rho;
      Csr S;
      S.n = n;
      S.row_ptr.assign(n + 1, 0);
      for (int i = 0; i < n; ++i) {
        bool has_diag = false;
        for (int k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
          const int j = A.col[k];
          if (!has_diag && j > i) {  // identity entry where A stores no diagonal (not on SPD input)
            S.col.push_back(i);
            S.val.push_back(1.0);
            has_diag = true;
          }
          const double x = c * (lv.inv_diag[i] * A.val[k]);
          S.col.push_back(j);
          S.val.push_back(j == i ? 1.0 - x : 0.0 - x);
          if (j == i) has_diag = true;
        }
        if (!has_diag) {
          S.col.push_back(i);
          S.val.push_back(1.0);
        }
        S.row_ptr[i + 1] = static_cast<int>(S.col.size());
      }
      const Csr St = csr_transpose(S, n);
      lv.P = spgemm_eigen(St, n, Tt);          // P = S T (n x nc)
      lv.Pt = csr_transpose(lv.P, nc);
      lv.nc = nc;
      // A_c = (P^T A) P: first PtA (nc x n), then (PtA) P
      const Csr PtA = spgemm_eigen(lv.P, nc, At);    // columns of P^T are P's rows; B = A by columns
      const Csr PtAt = csr_transpose(PtA, n);
      Csr Ac = spgemm_eigen(PtAt, nc, lv.Pt);
      levels.push_back(std::move(lv));
      A = std::move(Ac);
    }
    const AmgLevel& last = levels.back();
    const int nc = last.A.n;
    if (nc <= opt.coarse_size || levels.size() > 1) {
      dense_n = nc;
      Lc.assign(static_cast<size_t>(nc) * nc, 0.0);
      for (int j = 0; j < nc; ++j) {
        double d = last.A.at(j, j);
        for (int k = 0; k < j; ++k) d -= Lc[j * nc + k] * Lc[j * nc + k];
        if (!(d > 0.0)) throw Err(NOT_SPD);
        const double ljj = std::sqrt(d);
        Lc[j * nc + j] = ljj;
        for (int i = j + 1; i < nc; ++i) {
          double s = last.A.at(i, j);
          for (int k = 0; k < j; ++k) s -= Lc[i * nc + k] * Lc[j * nc + k];
          Lc[i * nc + j] = s / ljj;
        }
      }
    }
  }

  void dense_solve(const double* r, double* x) const {
    const int nc = dense_n;
    std::vector<double> s(r, r + nc);
    for (int k = 0; k < nc; ++k) {  // L y = r, column-oriented
      const double yk = s[k] / Lc[k * nc + k];
      s[k] = yk;
      for (int i = k + 1; i < nc; ++i) s[i] -= Lc[i * nc + k] * yk;
    }
    for (int k = nc - 1; k >= 0; --k) {  // L^T x = y, column-oriented
      const double xk = s[k] / Lc[k * nc + k];
      s[k] = xk;
      for (int i = 0; i < k; ++i) s[i] -= Lc[k * nc + i] * xk;
    }
    std::copy(s.begin(), s.end(), x);
  }

  // one V-cycle from zero on level l (amg.cpp:210-225)
  void cycle(size_t l, const double* r, double* x) const {
    const AmgLevel& lv = levels[l];
    const int n = lv.A.n;
    const double w = opt.omega;
    if (l + 1 == levels.size()) {
      if (dense_n > 0) {
        dense_solve(r, x);
        return;
      }
      std::vector<double> t(n);
      for (int i = 0; i < n; ++i) x[i] = w * (lv.inv_diag[i] * r[i]);
      lv.A.matvec(x, t.data());
      for (int i = 0; i < n; ++i) x[i] += w * (lv.inv_diag[i] * (r[i] - t[i]));
      return;
    }
    std::vector<double> res(n), t(n), rc(lv.nc), xc(lv.nc);
    for (int i = 0; i < n; ++i) x[i] = w * (lv.inv_diag[i] * r[i]);  // pre-smooth from 0
    for (int i = 0; i < n; ++i) {  // residual = r - A x (Eigen: res = r; res -= A x)
      double s = r[i];
      for (int k = lv.A.row_ptr[i]; k < lv.A.row_ptr[i + 1]; ++k) s -= lv.A.val[k] * x[lv.A.col[k]];
      res[i] = s;
    }
    lv.Pt.matvec(res.data(), rc.data());  // P^T residual
    cycle(l + 1, rc.data(), xc.data());
    for (int i = 0; i < n; ++i) {  // x += P coarse
      double s = x[i];
      for (int k = lv.P.row_ptr[i]; k < lv.P.row_ptr[i + 1]; ++k) s += lv.P.val[k] * xc[lv.P.col[k]];
      x[i] = s;
    }
    lv.A.matvec(x, t.data());  // post-smooth
    for (int i = 0; i < n; ++i) x[i] += w * (lv.inv_diag[i] * (r[i] - t[i]));
  }

  void apply(const double* r, double* z) const override { cycle(0, r, z); }
  const char* kind() const override { return "amg"; }
};

// ---- pcg: solver.cpp:186-245 -------------------------------------------------
struct Record {
  int iterations = 0;
  double rel = 0.0;
  uint8_t status = ST_MAX_ITER;
};

#ifndef VQPO_PAIRWISE_DOT
static double dot(const double* a, const double* b, int n) {  // solver.cpp:176-180: serial
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
#else
// investigation build only (not the oracle): pairwise summation, to measure how
// much of a GPU/CPU iteration-count difference the summation order explains
static double dot_rec(const double* a, const double* b, int n) {
  if (n <= 8) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
  }
  const int h = n / 2;
  return dot_rec(a, b, h) + dot_rec(a + h, b + h, n - h);
}
static double dot(const double* a, const double* b, int n) { return dot_rec(a, b, n); }
#endif

// Returns the record the reference would hold at exit. A breakdown (where the
// reference throws "pcg-breakdown") is reported as status ST_BREAKDOWN with the
// last recorded iteration count and residual.
static Record pcg(const System& sys, const Preconditioner& M, double eps, int max_iter,
                  double* x_out, std::vector<double>* trace) {
  const Csr& A = sys.A;
  const int n = A.n;
  if (!(eps > 0.0) || eps >= 1.0) throw Err(INVALID_TOLERANCE);
  if (max_iter < 0) max_iter = 10 * n;
  Record rec;
  std::vector<double> x(n, 0.0);
  const double norm_b = std::sqrt(dot(sys.b.data(), sys.b.data(), n));
  if (norm_b == 0.0) {
    rec.status = ST_CONVERGED;
    if (x_out) std::copy(x.begin(), x.end(), x_out);
    return rec;
  }
  std::vector<double> r = sys.b, z(n), p(n), Ap(n), rt(n);
  M.apply(r.data(), z.data());
  std::copy(z.begin(), z.end(), p.begin());
  double rz = dot(r.data(), z.data(), n);
  if (!(rz > 0.0)) {
    rec.status = ST_BREAKDOWN;
    if (x_out) std::copy(x.begin(), x.end(), x_out);
    return rec;
  }
  rec.status = ST_MAX_ITER;
  for (int j = 1; j <= max_iter; ++j) {
    A.matvec(p.data(), Ap.data());
    const double pAp = dot(p.data(), Ap.data(), n);
    if (!(pAp > 0.0)) {
      rec.status = ST_BREAKDOWN;
      break;
    }
    const double alpha = rz / pAp;
    for (int i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * Ap[i];
    }
    A.matvec(x.data(), rt.data());
    for (int i = 0; i < n; ++i) rt[i] = sys.b[i] - rt[i];
    const double rel = std::sqrt(dot(rt.data(), rt.data(), n)) / norm_b;
    if (trace) trace->push_back(rel);
    rec.iterations = j;
    rec.rel = rel;
    if (rel < eps) {
      rec.status = ST_CONVERGED;
      break;
    }
    M.apply(r.data(), z.data());
    const double rz_next = dot(r.data(), z.data(), n);
    if (!(rz_next > 0.0)) {
      rec.status = ST_BREAKDOWN;
      break;
    }
    const double beta = rz_next / rz;
    rz = rz_next;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  if (x_out) std::copy(x.begin(), x.end(), x_out);
  return rec;
}

// ---- quantizer: T2Map (quantizer.cpp:50-63), nearest_row (113-130), assign
// (134-145), kmeans (181-357), grid (425-463), sign grid (new), centroid
// coefficient (465-476) ------------------------------------------------------
enum Method : int { KMEANS = 0, CLVQ = 1, GRID = 2, SIGN_GRID = 3 };
enum MapKind : int { SCALE = 0, CDF = 1 };

struct Codebook {
  int m = 0, P = 0, method = KMEANS, map = SCALE;
  const double* lambdas = nullptr;   // m
  const double* centroids = nullptr; // P x m, quantization space
  const double* latent = nullptr;    // P x m, grids only
};

static void to_quant(const Codebook& cb, const double* chi, double* eta) {
  for (int k = 0; k < cb.m; ++k) {
    const double root = std::sqrt(cb.lambdas[k]);
    eta[k] = cb.map == SCALE ? root * chi[k] : root * normal_cdf(chi[k]);
  }
}
static void to_latent(const Codebook& cb, const double* eta, double* chi) {
  for (int k = 0; k < cb.m; ++k) {
    const double root = std::sqrt(cb.lambdas[k]);
    chi[k] = cb.map == SCALE ? eta[k] / root : normal_quantile(eta[k] / root);
  }
}

static int nearest_row(const double* x, const double* sites, int P, int m, double* best_out) {
  int best = 0;
  double best_d = std::numeric_limits<double>::infinity();
  for (int p = 0; p < P; ++p) {
    const double* c = sites + static_cast<size_t>(p) * m;
    double d = 0.0;
    for (int k = 0; k < m; ++k) {
      const double t = x[k] - c[k];
      d += t * t;
    }
    if (d < best_d) {  // strict: ties keep the smallest index
      best_d = d;
      best = p;
    }
  }
  if (best_out) *best_out = best_d;
  return best;
}

static int assign(const Codebook& cb, const double* xi) {
  for (int k = 0; k < cb.m; ++k)
    if (!std::isfinite(xi[k])) throw Err(INVALID_LATENT);
  if (cb.method == GRID || cb.method == SIGN_GRID)
    return nearest_row(xi, cb.latent, cb.P, cb.m, nullptr);
  std::vector<double> eta(cb.m);
  to_quant(cb, xi, eta.data());
  return nearest_row(eta.data(), cb.centroids, cb.P, cb.m, nullptr);
}

static double sqdist(const double* a, const double* b, int m) {
  double d = 0.0;
  for (int k = 0; k < m; ++k) {
    const double t = a[k] - b[k];
    d += t * t;
  }
  return d;
}

// minmax (farthest point) seeding, quantizer.cpp:181-213
static std::vector<double> minmax_seed(const std::vector<double>& pts, int n, int m, int P,
                                       uint64_t init_seed) {
  std::vector<double> c(static_cast<size_t>(P) * m);
  const int first = static_cast<int>(counter_hash(init_seed, 0, 0) % static_cast<uint64_t>(n));
  std::copy_n(pts.data() + static_cast<size_t>(first) * m, m, c.data());
  std::vector<double> min_d(n);
  for (int i = 0; i < n; ++i) min_d[i] = sqdist(pts.data() + static_cast<size_t>(i) * m, c.data(), m);
  for (int p = 1; p < P; ++p) {
    int far = 0;
    for (int i = 1; i < n; ++i)
      if (min_d[i] > min_d[far]) far = i;
    if (!(min_d[far] > 0.0)) throw Err(INSUFFICIENT_SAMPLES);
    double* cp = c.data() + static_cast<size_t>(p) * m;
    std::copy_n(pts.data() + static_cast<size_t>(far) * m, m, cp);
    for (int i = 0; i < n; ++i)
      min_d[i] = std::min(min_d[i], sqdist(pts.data() + static_cast<size_t>(i) * m, cp, m));
  }
  return c;
}

static double assign_all(const std::vector<double>& pts, int n, int m, const std::vector<double>& c,
                         int P, std::vector<int>& labels) {
  double total = 0.0;
  for (int i = 0; i < n; ++i) {
    double bd;
    labels[i] = nearest_row(pts.data() + static_cast<size_t>(i) * m, c.data(), P, m, &bd);
    total += bd;
  }
  return total / n;
}

// empty-cell repair, quantizer.cpp:260-294
static bool repair_empty_cells(const std::vector<double>& pts, int n, int m, std::vector<double>& c,
                               int P, std::vector<int>& labels) {
  bool repaired = false;
  for (;;) {
    std::vector<long> counts(P, 0);
    for (int i = 0; i < n; ++i) counts[labels[i]] += 1;
    int empty = -1;
    for (int p = 0; p < P; ++p)
      if (counts[p] == 0) {
        empty = p;
        break;
      }
    if (empty < 0) return repaired;
    repaired = true;
    int worst = 0;
    double worst_d = -1.0;
    for (int i = 0; i < n; ++i) {
      const double d = sqdist(pts.data() + static_cast<size_t>(i) * m,
                              c.data() + static_cast<size_t>(labels[i]) * m, m);
      if (d > worst_d) {
        worst_d = d;
        worst = i;
      }
    }
    std::copy_n(pts.data() + static_cast<size_t>(worst) * m, m,
                c.data() + static_cast<size_t>(empty) * m);
    assign_all(pts, n, m, c, P, labels);
  }
}

// kmeans = minmax seed + Lloyd (quantizer.cpp:296-357)
static std::vector<double> kmeans(const double* samples, int n, int m, const double* lambdas,
                                  int map, int P, uint64_t init_seed, int max_iter, double rel_tol,
                                  std::vector<double>* history) {
  if (P < 1) throw Err(INVALID_CODEBOOK);
  if (n < P) throw Err(INSUFFICIENT_SAMPLES);
  Codebook t2;
  t2.m = m;
  t2.map = map;
  t2.lambdas = lambdas;
  std::vector<double> pts(static_cast<size_t>(n) * m);
  for (int i = 0; i < n; ++i)
    to_quant(t2, samples + static_cast<size_t>(i) * m, pts.data() + static_cast<size_t>(i) * m);
  std::vector<double> c = minmax_seed(pts, n, m, P, init_seed);
  std::vector<int> labels(n);
  double prev = std::numeric_limits<double>::infinity();
  for (int iter = 0; iter < max_iter; ++iter) {
    double w = assign_all(pts, n, m, c, P, labels);
    if (repair_empty_cells(pts, n, m, c, P, labels)) w = assign_all(pts, n, m, c, P, labels);
    if (history) history->push_back(w);
    std::vector<double> sums(static_cast<size_t>(P) * m, 0.0);
    std::vector<long> counts(P, 0);
    for (int i = 0; i < n; ++i) {
      const double* x = pts.data() + static_cast<size_t>(i) * m;
      double* s = sums.data() + static_cast<size_t>(labels[i]) * m;
      for (int k = 0; k < m; ++k) s[k] += x[k];
      counts[labels[i]] += 1;
    }
    for (int p = 0; p < P; ++p) {
      if (counts[p] == 0) continue;
      for (int k = 0; k < m; ++k)
        c[static_cast<size_t>(p) * m + k] = sums[static_cast<size_t>(p) * m + k] / counts[p];
    }
    if (prev < std::numeric_limits<double>::infinity() && prev - w <= rel_tol * std::abs(prev)) break;
    prev = w;
  }
  // Codebook::validate (quantizer.cpp:95-109): pairwise distinct
  for (int p = 0; p < P; ++p)
    for (int q = p + 1; q < P; ++q)
      if (sqdist(c.data() + static_cast<size_t>(p) * m, c.data() + static_cast<size_t>(q) * m, m) == 0.0)
        throw Err(INVALID_CODEBOOK);
  return c;
}

// ---- campaign: driver.cpp:193-281 with the 1-D/2-D model switch ---------------
enum Precond : int { PC_IDENTITY = 0, PC_CHOLESKY = 1, PC_AMG = 3, PC_IC0 = 4 };

struct Model {
  int dim = 1;   // 1: N elements; 2: r x r structured mesh
  int size = 0;  // N (dim 1) or r (dim 2)
  int n_nodes() const { return dim == 1 ? size : (size + 1) * (size + 1); }
  int n_unknowns() const { return dim == 1 ? size - 1 : (size - 1) * (size - 1); }
  System assemble(const double* kappa) const {
    return dim == 1 ? assemble_1d(size, kappa) : assemble_2d(size, kappa);
  }
};

static std::unique_ptr<Preconditioner> build_preconditioner(int kind, const Model& model, const Csr& A) {
  switch (kind) {
    case PC_IDENTITY: return std::make_unique<IdentityPreconditioner>(A.n);
    case PC_CHOLESKY: return std::make_unique<CholeskyPreconditioner>(A);
    case PC_AMG: return std::make_unique<AmgPreconditioner>(A);
    case PC_IC0:
      if (model.dim != 2) throw Err(INVALID_CONFIG);
      return std::make_unique<IC0Preconditioner>(A, model.size);
    default: throw Err(INVALID_CONFIG);
  }
}

struct Basis {
  const double* evals = nullptr;
  const double* evecs = nullptr;
  int n_kl = 0, n_nodes = 0;
};

// centroid coefficient (quantizer.cpp:465-476): chi = latent site (grids) or
// T2(centroid); kappa_p = transport(lift(basis, chi)) over the first m modes.
static std::vector<double> centroid_coefficient(const Codebook& cb, int p, const Basis& basis) {
  std::vector<double> chi(cb.m), h(basis.n_nodes);
  if (cb.method == GRID || cb.method == SIGN_GRID)
    std::copy_n(cb.latent + static_cast<size_t>(p) * cb.m, cb.m, chi.data());
  else
    to_latent(cb, cb.centroids + static_cast<size_t>(p) * cb.m, chi.data());
  if (cb.m > basis.n_kl) throw Err(MODE_COUNT_OUT_OF_RANGE);
  lift(basis.evals, basis.evecs, basis.n_nodes, chi.data(), cb.m, h.data());
  transport(h.data(), basis.n_nodes);
  return h;
}

struct PreconditionerSet {
  Model model;
  std::vector<std::unique_ptr<Preconditioner>> M;
};

static void solve_one(const Model& model, const Basis& basis, const double* xi, int m_xi,
                      const Preconditioner& M, double eps, int max_iter, Record& rec, double* x_out,
                      std::vector<double>& h) {
  try {
    // no finiteness check here: like the reference (driver.cpp:230-233), a
    // non-finite xi_k reaches lift and transport reports coefficient-overflow
    // (only assign's first m components raise invalid-latent)
    lift(basis.evals, basis.evecs, basis.n_nodes, xi, m_xi, h.data());
    transport(h.data(), basis.n_nodes);
    const System sys = model.assemble(h.data());
    rec = pcg(sys, M, eps, max_iter, x_out, nullptr);
  } catch (const Err& e) {
    rec = Record{};
    rec.status = e.code == COEFFICIENT_OVERFLOW ? ST_COEFF_OVERFLOW
                 : e.code == INVALID_LATENT     ? ST_INVALID_LATENT
                                                : ST_INVALID_COEFF;
    if (e.code == INVALID_TOLERANCE) throw;
  }
}

}  // namespace vqpo

// =============================================================================
// C entry points (ctypes). All return an error code (0 = ok).
// =============================================================================
using namespace vqpo;

#define VQPO_GUARD(...)                  \
  try {                                  \
    __VA_ARGS__;                         \
  } catch (const Err& e) {               \
    return e.code;                       \
  } catch (...) {                        \
    return INVALID_ARGUMENT;             \
  }                                      \
  return OK;

extern "C" {

uint64_t vqpo_counter_hash(uint64_t seed, uint64_t index, uint64_t comp) {
  return counter_hash(seed, index, comp);
}
double vqpo_uniform_open01(uint64_t seed, uint64_t index, uint64_t comp) {
  return uniform_open01(seed, index, comp);
}
double vqpo_normal_quantile(double p) {
  try {
    return normal_quantile(p);
  } catch (...) {
    return std::numeric_limits<double>::quiet_NaN();
  }
}
double vqpo_normal_cdf(double x) { return normal_cdf(x); }

// draw_standard_normal (quantizer.cpp:77-87): out[i*m + k] = gaussian_draw(seed,
// index0 + i, k). Rows are independent, so threads do not change the bits.
int vqpo_draw_standard_normal(int64_t n, int m, uint64_t seed, int64_t index0, double* out, int threads) {
  VQPO_GUARD({
    const long chunk = 4096;
    const long nchunks = (n + chunk - 1) / chunk;
    parallel_for_slots(nchunks, threads, [&](long c) {
      const long lo = c * chunk, hi = std::min<long>(n, lo + chunk);
      for (long i = lo; i < hi; ++i)
        for (int k = 0; k < m; ++k)
          out[i * m + k] = gaussian_draw(seed, static_cast<uint64_t>(index0 + i), static_cast<uint64_t>(k));
    });
  })
}

// lift + transport for B samples (field.cpp:113-145). kappa_out: B x n_nodes.
// status_out[i]: 0 ok or ST_COEFF_OVERFLOW.
int vqpo_realise(const double* evals, const double* evecs, int n_kl, int n_nodes, const double* xi,
                 int64_t B, int ld, int m, double* kappa_out, uint8_t* status_out, int threads) {
  VQPO_GUARD({
    if (m > n_kl) throw Err(MODE_COUNT_OUT_OF_RANGE);
    parallel_for_slots(B, threads, [&](long i) {
      double* h = kappa_out + static_cast<size_t>(i) * n_nodes;
      lift(evals, evecs, n_nodes, xi + static_cast<size_t>(i) * ld, m, h);
      uint8_t st = ST_CONVERGED;
      for (int j = 0; j < n_nodes; ++j) {
        h[j] = std::exp(h[j]);
        if (!std::isfinite(h[j])) st = ST_COEFF_OVERFLOW;
      }
      if (status_out) status_out[i] = st;
    });
  })
}

// assemble: returns CSR into caller buffers sized by vqpo_assemble_nnz.
int vqpo_assemble(int dim, int size, const double* kappa, int* n_out, int* nnz_out, int* row_ptr,
                  int* col, double* val, double* b) {
  VQPO_GUARD({
    Model model{dim, size};
    const System s = model.assemble(kappa);
    *n_out = s.A.n;
    *nnz_out = static_cast<int>(s.A.val.size());
    if (row_ptr) std::copy(s.A.row_ptr.begin(), s.A.row_ptr.end(), row_ptr);
    if (col) std::copy(s.A.col.begin(), s.A.col.end(), col);
    if (val) std::copy(s.A.val.begin(), s.A.val.end(), val);
    if (b) std::copy(s.b.begin(), s.b.end(), b);
  })
}

int vqpo_rcm_permutation(int n, const int* row_ptr, const int* col, int* perm_out) {
  VQPO_GUARD({
    Csr A;
    A.n = n;
    A.row_ptr.assign(row_ptr, row_ptr + n + 1);
    A.col.assign(col, col + row_ptr[n]);
    A.val.assign(row_ptr[n], 1.0);
    const auto p = rcm_permutation(A);
    std::copy(p.begin(), p.end(), perm_out);
  })
}

// nearest-centroid assignment for B samples (quantizer.cpp:134-145; the driver's
// serial loop driver.cpp:206-210). xi rows have stride ld; the first m are used.
int vqpo_assign(int method, int map, int P, int m, const double* lambdas, const double* centroids,
                const double* latent, const double* xi, int64_t B, int ld, int32_t* labels) {
  VQPO_GUARD({
    Codebook cb{m, P, method, map, lambdas, centroids, latent};
    for (long i = 0; i < B; ++i) labels[i] = assign(cb, xi + static_cast<size_t>(i) * ld);
  })
}

int vqpo_kmeans(const double* samples, int n, int m, const double* lambdas, int map, int P,
                uint64_t init_seed, int max_iter, double rel_tol, double* centroids_out,
                double* history_out, int* n_history) {
  VQPO_GUARD({
    std::vector<double> hist;
    const auto c = kmeans(samples, n, m, lambdas, map, P, init_seed, max_iter, rel_tol, &hist);
    std::copy(c.begin(), c.end(), centroids_out);
    if (history_out) std::copy(hist.begin(), hist.end(), history_out);
    if (n_history) *n_history = static_cast<int>(hist.size());
  })
}

// reference grid (quantizer.cpp:425-463): origin + 2^m vertices at +-s.
int vqpo_grid_sites(int m, double s, double* sites) {
  VQPO_GUARD({
    const int P = m == 0 ? 1 : 1 + (1 << m);
    std::fill(sites, sites + static_cast<size_t>(P) * m, 0.0);
    for (int v = 1; v < P; ++v) {
      const unsigned bits = static_cast<unsigned>(v - 1);
      for (int k = 0; k < m; ++k) sites[static_cast<size_t>(v) * m + k] = (bits >> k) & 1u ? s : -s;
    }
  })
}

// sign grid (new): P = 2^m sites, component k = +s if bit k
// of p is set else -s, s = sqrt(2/pi) (the half-normal mean).
int vqpo_sign_grid_sites(int m, double* sites) {
  VQPO_GUARD({
    const double s = std::sqrt(2.0 / std::numbers::pi);
    const int P = 1 << m;
    for (int p = 0; p < P; ++p)
      for (int k = 0; k < m; ++k) sites[static_cast<size_t>(p) * m + k] = (p >> k) & 1 ? s : -s;
  })
}

int vqpo_to_quant(int map, int m, const double* lambdas, const double* chi, int64_t B, double* eta) {
  VQPO_GUARD({
    Codebook cb;
    cb.m = m;
    cb.map = map;
    cb.lambdas = lambdas;
    for (long i = 0; i < B; ++i) to_quant(cb, chi + static_cast<size_t>(i) * m, eta + static_cast<size_t>(i) * m);
  })
}

int vqpo_centroid_coefficients(int method, int map, int P, int m, const double* lambdas,
                               const double* centroids, const double* latent, const double* evals,
                               const double* evecs, int n_kl, int n_nodes, double* kappa_out) {
  VQPO_GUARD({
    Codebook cb{m, P, method, map, lambdas, centroids, latent};
    Basis basis{evals, evecs, n_kl, n_nodes};
    for (int p = 0; p < P; ++p) {
      const auto k = centroid_coefficient(cb, p, basis);
      std::copy(k.begin(), k.end(), kappa_out + static_cast<size_t>(p) * n_nodes);
    }
  })
}

// --- preconditioner sets (driver.cpp:212-219) ---------------------------------
void vqpo_pset_destroy(void* h) { delete static_cast<PreconditionerSet*>(h); }

int vqpo_pset_build(int dim, int size, int kind, int method, int map, int P, int m, const double* lambdas,
                    const double* centroids, const double* latent, const double* evals,
                    const double* evecs, int n_kl, int n_nodes, void** out) {
  VQPO_GUARD({
    auto set = std::make_unique<PreconditionerSet>();
    set->model = Model{dim, size};
    if (set->model.n_nodes() != n_nodes) throw Err(INVALID_CONFIG);
    Codebook cb{m, P, method, map, lambdas, centroids, latent};
    Basis basis{evals, evecs, n_kl, n_nodes};
    for (int p = 0; p < P; ++p) {
      const auto coeff = centroid_coefficient(cb, p, basis);
      const System cs = set->model.assemble(coeff.data());
      set->M.push_back(build_preconditioner(kind, set->model, cs.A));
      set->M.back()->built_from = p;
    }
    *out = set.release();
  })
}

// preconditioner from an explicit coefficient (tests: J = 1 with the exact factor)
int vqpo_pset_from_coefficients(int dim, int size, int kind, int P, const double* kappa, void** out) {
  VQPO_GUARD({
    auto set = std::make_unique<PreconditionerSet>();
    set->model = Model{dim, size};
    const int nn = set->model.n_nodes();
    for (int p = 0; p < P; ++p) {
      const System cs = set->model.assemble(kappa + static_cast<size_t>(p) * nn);
      set->M.push_back(build_preconditioner(kind, set->model, cs.A));
      set->M.back()->built_from = p;
    }
    *out = set.release();
  })
}

// SA-AMG hierarchy of centroid p (AmgOptions::level_sizes_out, solver.hpp:42, plus
// the operators, for bit-level checks of the GPU library's own setup).
// info[l*4 + 0..3] = n_l, nnz(A_l), nnz(P_l), nc_l; returns the level count in *nlev
// and the coarsest dense size in *dense_n.
int vqpo_pset_amg_info(void* h, int p, int max_levels, int64_t* info, int* nlev, int* dense_n) {
  VQPO_GUARD({
    auto* set = static_cast<PreconditionerSet*>(h);
    const auto* amg = dynamic_cast<const AmgPreconditioner*>(set->M.at(p).get());
    if (!amg) throw Err(INVALID_CONFIG);
    *nlev = static_cast<int>(amg->levels.size());
    *dense_n = amg->dense_n;
    for (int l = 0; l < *nlev && l < max_levels; ++l) {
      const AmgLevel& lv = amg->levels[l];
      info[l * 4 + 0] = lv.A.n;
      info[l * 4 + 1] = lv.A.row_ptr[lv.A.n];
      info[l * 4 + 2] = lv.P.n ? lv.P.row_ptr[lv.P.n] : 0;
      info[l * 4 + 3] = lv.nc;
    }
  })
}

// copy level l's A (row_ptr n+1, col, val), inv_diag (n) and P (row_ptr n+1,
// col, val; empty on the coarsest); L (dense_n^2, row-major) when l is the last level
int vqpo_pset_amg_level(void* h, int p, int l, int* a_rp, int* a_col, double* a_val, double* inv_diag, int* p_rp,
                        int* p_col, double* p_val, double* L) {
  VQPO_GUARD({
    auto* set = static_cast<PreconditionerSet*>(h);
    const auto* amg = dynamic_cast<const AmgPreconditioner*>(set->M.at(p).get());
    if (!amg) throw Err(INVALID_CONFIG);
    const AmgLevel& lv = amg->levels.at(l);
    std::copy(lv.A.row_ptr.begin(), lv.A.row_ptr.end(), a_rp);
    std::copy(lv.A.col.begin(), lv.A.col.end(), a_col);
    std::copy(lv.A.val.begin(), lv.A.val.end(), a_val);
    std::copy(lv.inv_diag.begin(), lv.inv_diag.end(), inv_diag);
    if (lv.P.n) {
      std::copy(lv.P.row_ptr.begin(), lv.P.row_ptr.end(), p_rp);
      std::copy(lv.P.col.begin(), lv.P.col.end(), p_col);
      std::copy(lv.P.val.begin(), lv.P.val.end(), p_val);
    }
    if (L && l + 1 == static_cast<int>(amg->levels.size())) std::copy(amg->Lc.begin(), amg->Lc.end(), L);
  })
}

int vqpo_pset_apply(void* h, int p, const double* r, double* z) {
  VQPO_GUARD({
    auto* set = static_cast<PreconditionerSet*>(h);
    set->M.at(p)->apply(r, z);
  })
}

// Per-sample solves with labels supplied: coefficient = transport(lift(xi_i))
// over m_xi modes, system assembled, pcg with M_{label_i}. max_iter_arr
// (nullable) overrides max_iter per sample (Appendix B.5 fixed-K runs).
int vqpo_solve_batch(void* h, const double* evals, const double* evecs, int n_kl, int n_nodes,
                     const double* xi, int64_t B, int ld, int m_xi, const int32_t* labels, double eps,
                     int max_iter, const int32_t* max_iter_arr, int threads, int32_t* iters,
                     double* rel, uint8_t* status, double* x_out) {
  VQPO_GUARD({
    auto* set = static_cast<PreconditionerSet*>(h);
    if (!(eps > 0.0) || eps >= 1.0) throw Err(INVALID_TOLERANCE);
    if (m_xi > n_kl) throw Err(MODE_COUNT_OUT_OF_RANGE);
    Basis basis{evals, evecs, n_kl, n_nodes};
    const int n = set->model.n_unknowns();
    parallel_for_slots(B, threads, [&](long i) {
      std::vector<double> hbuf(n_nodes);
      Record rec;
      const int mi = max_iter_arr ? max_iter_arr[i] : max_iter;
      solve_one(set->model, basis, xi + static_cast<size_t>(i) * ld, m_xi, *set->M.at(labels[i]), eps,
                mi, rec, x_out ? x_out + static_cast<size_t>(i) * n : nullptr, hbuf);
      iters[i] = rec.iterations;
      rel[i] = rec.rel;
      status[i] = rec.status;
    });
  })
}

// Single system with an explicit coefficient and preconditioner index; trace
// (nullable, capacity max_iter) receives the true relative residual history.
int vqpo_pcg_coefficient(void* h, int p, const double* kappa, double eps, int max_iter, double* x_out,
                         int32_t* iters, double* rel, uint8_t* status, double* trace, int* n_trace) {
  VQPO_GUARD({
    auto* set = static_cast<PreconditionerSet*>(h);
    const System sys = set->model.assemble(kappa);
    std::vector<double> tr;
    const Record rec = pcg(sys, *set->M.at(p), eps, max_iter, x_out, trace ? &tr : nullptr);
    *iters = rec.iterations;
    *rel = rec.rel;
    *status = rec.status;
    if (trace) {
      std::copy(tr.begin(), tr.end(), trace);
      *n_trace = static_cast<int>(tr.size());
    }
  })
}

// Full campaign (driver.cpp:193-281): assign all (serial), build the P
// preconditioners up front (serial), group by label in index order, solve the
// groups on `threads` workers (one slot per centroid group), then reduce.
// stats (length 4P): [n_p | sum_j | conv_count | conv_sum]; summary[0..3] =
// {total_iterations, unconverged, conv_total, conv_sum_total};
// timings[0..3] = seconds {assign, build, solve, reduce}.
// ideal_sweep (driver.cpp:290-340): for every realisation i (threads over
// realisations, driver.cpp:313) and every m of m_list, the preconditioner of the
// kind built from the m-truncated coefficient transport(lift(basis, xi_i[0:m]))
// applied to the full-coefficient system; records[i * n_m + im]. The rows
// (m, relative energy, mean J over converged) are formed by the caller.
int vqpo_ideal_sweep(int dim, int size, int kind, const double* evals, const double* evecs, int n_kl, int n_nodes,
                     const double* xi, int64_t B, int ld, const int* m_list, int n_m, double eps, int max_iter,
                     int threads, int32_t* iters, double* rel, uint8_t* status) {
  VQPO_GUARD({
    if (!(eps > 0.0) || eps >= 1.0) throw Err(INVALID_TOLERANCE);
    Model model{dim, size};
    if (model.n_nodes() != n_nodes || ld < n_kl) throw Err(INVALID_CONFIG);
    for (int im = 0; im < n_m; ++im)
      if (m_list[im] < 0 || m_list[im] > n_kl) throw Err(MODE_COUNT_OUT_OF_RANGE);
    parallel_for_slots(static_cast<long>(B), threads, [&](long i) {
      const double* xr = xi + static_cast<size_t>(i) * ld;
      std::vector<double> h(n_nodes), ht(n_nodes);
      for (int im = 0; im < n_m; ++im) {
        Record rec;
        try {
          lift(evals, evecs, n_nodes, xr, n_kl, h.data());
          transport(h.data(), n_nodes);
          const System sys = model.assemble(h.data());
          lift(evals, evecs, n_nodes, xr, m_list[im], ht.data());
          transport(ht.data(), n_nodes);
          const System trunc = model.assemble(ht.data());
          const auto M = build_preconditioner(kind, model, trunc.A);
          rec = pcg(sys, *M, eps, max_iter, nullptr, nullptr);
        } catch (const Err& e) {
          rec = Record{};
          rec.status = e.code == COEFFICIENT_OVERFLOW ? ST_COEFF_OVERFLOW : ST_INVALID_COEFF;
        }
        const size_t q = static_cast<size_t>(i) * n_m + im;
        iters[q] = rec.iterations;
        rel[q] = rec.rel;
        status[q] = rec.status;
      }
    });
  })
}

int vqpo_run_campaign(int dim, int size, int kind, int method, int map, int P, int m,
                      const double* lambdas, const double* centroids, const double* latent,
                      const double* evals, const double* evecs, int n_kl, int n_nodes, const double* xi,
                      int64_t B, int ld, double eps, int max_iter, int threads, int32_t* labels,
                      int32_t* iters, double* rel, uint8_t* status, int64_t* stats, int64_t* summary,
                      double* timings) {
  VQPO_GUARD({
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double>(b - a).count();
    };
    if (!(eps > 0.0) || eps >= 1.0) throw Err(INVALID_TOLERANCE);
    Codebook cb{m, P, method, map, lambdas, centroids, latent};
    Basis basis{evals, evecs, n_kl, n_nodes};
    Model model{dim, size};
    if (model.n_nodes() != n_nodes || ld < n_kl) throw Err(INVALID_CONFIG);
    const auto t0 = clk::now();
    for (long i = 0; i < B; ++i) labels[i] = assign(cb, xi + static_cast<size_t>(i) * ld);
    const auto t1 = clk::now();
    std::vector<std::unique_ptr<Preconditioner>> M(P);
    for (int p = 0; p < P; ++p) {
      const auto coeff = centroid_coefficient(cb, p, basis);
      const System cs = model.assemble(coeff.data());
      M[p] = build_preconditioner(kind, model, cs.A);
      M[p]->built_from = p;
    }
    const auto t2 = clk::now();
    std::vector<std::vector<long>> groups(P);
    for (long i = 0; i < B; ++i) groups[labels[i]].push_back(i);
    std::vector<int> active;
    for (int p = 0; p < P; ++p)
      if (!groups[p].empty()) active.push_back(p);
    parallel_for_slots(static_cast<long>(active.size()), threads, [&](long slot) {
      const int p = active[slot];
      std::vector<double> hbuf(n_nodes);
      for (long i : groups[p]) {
        Record rec;
        solve_one(model, basis, xi + static_cast<size_t>(i) * ld, n_kl, *M[p], eps, max_iter, rec,
                  nullptr, hbuf);
        iters[i] = rec.iterations;
        rel[i] = rec.rel;
        status[i] = rec.status;
      }
    });
    const auto t3 = clk::now();
    std::fill(stats, stats + 4 * static_cast<size_t>(P), 0);
    int64_t total = 0, unconv = 0, ctot = 0, csum = 0;
    for (long i = 0; i < B; ++i) {
      const int p = labels[i];
      stats[p] += 1;
      stats[P + p] += iters[i];
      total += iters[i];
      if (status[i] == ST_CONVERGED) {
        stats[2 * P + p] += 1;
        stats[3 * P + p] += iters[i];
        ctot += 1;
        csum += iters[i];
      } else {
        unconv += 1;
      }
    }
    summary[0] = total;
    summary[1] = unconv;
    summary[2] = ctot;
    summary[3] = csum;
    const auto t4 = clk::now();
    if (timings) {
      timings[0] = secs(t0, t1);
      timings[1] = secs(t1, t2);
      timings[2] = secs(t2, t3);
      timings[3] = secs(t3, t4);
    }
  })
}

}  // extern "C"
