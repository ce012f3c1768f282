// oracle/ref/ref_glue.cpp — TEST INFRASTRUCTURE ONLY.
// C entry points over the reference's OWN translation units compiled here
// unchanged from /root/reference/proj/src (fem.cpp, quantizer.cpp, rng.cpp,
// artifacts.cpp). Used only by tests/ to pin the oracle restatement.
// The two field.cpp functions quantizer.cpp links against (lift, transport;
// field.cpp needs Eigen, which is absent) are restated below with the
// semantics of proj/src/field.cpp:113-125 and :138-145.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "vqp/artifacts.hpp"
#include "vqp/error.hpp"
#include "vqp/fem.hpp"
#include "vqp/field.hpp"
#include "vqp/quantizer.hpp"
#include "vqp/rng.hpp"

namespace vqp {
std::vector<double> lift(const KLBasis& basis, std::span<const double> xi) {
  const int m = static_cast<int>(xi.size());
  if (m > basis.n_kl()) throw Error("mode-count-out-of-range");
  std::vector<double> h(basis.n_nodes(), 0.0);
  for (int k = 0; k < m; ++k) {
    const double w = std::sqrt(basis.eigenvalues[k]) * xi[k];
    if (w == 0.0) continue;
    const auto phi = basis.mode(k);
    for (int i = 0; i < basis.n_nodes(); ++i) h[i] += w * phi[i];
  }
  return h;
}
std::vector<double> transport(std::span<const double> v) {
  std::vector<double> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    out[i] = std::exp(v[i]);
    if (!std::isfinite(out[i])) throw Error("coefficient-overflow");
  }
  return out;
}
}  // namespace vqp

using namespace vqp;

static thread_local std::string g_last_error;

static vqp::Codebook make_codebook(int method, int map, int P, int m, const double* lambdas,
                                   const double* centroids) {
  Codebook cb;
  cb.m = m;
  cb.P = P;
  cb.t2.kind = map == 0 ? MapKind::Scale : MapKind::ScaledCdf;
  cb.t2.lambdas.assign(lambdas, lambdas + m);
  cb.method = method == 0 ? QuantMethod::KMeans : method == 1 ? QuantMethod::Clvq : QuantMethod::Grid;
  cb.centroids.assign(centroids, centroids + static_cast<size_t>(P) * m);
  if (cb.method == QuantMethod::Grid) {
    cb.grid_s = grid_parameter();
    cb.latent_centroids = grid_latent_sites(m, cb.grid_s);
  }
  return cb;
}

#define GUARD(...)                      \
  try {                                 \
    __VA_ARGS__;                        \
  } catch (const vqp::Error& e) {       \
    g_last_error = e.code();            \
    return 1;                           \
  } catch (const std::exception& e) {   \
    g_last_error = e.what();            \
    return 2;                           \
  }                                     \
  return 0;

extern "C" {

const char* vqpref_last_error() { return g_last_error.c_str(); }

uint64_t vqpref_counter_hash(uint64_t s, uint64_t i, uint64_t k) { return counter_hash(s, i, k); }
double vqpref_uniform_open01(uint64_t s, uint64_t i, uint64_t k) { return uniform_open01(s, i, k); }

// reference make_mesh + assemble (fem.cpp:53-81, 213-256); nnz query when val == nullptr
int vqpref_assemble_2d(int r, const double* kappa, int* n, int* nnz, int* row_ptr, int* col,
                       double* val, double* b) {
  GUARD({
    const TriMesh mesh = make_mesh(r);
    const LinearSystem sys = assemble(mesh, {kappa, static_cast<size_t>(mesh.n_nodes())});
    *n = sys.A.n;
    *nnz = sys.A.nnz();
    if (val) {
      std::memcpy(row_ptr, sys.A.row_ptr.data(), sizeof(int) * (sys.A.n + 1));
      std::memcpy(col, sys.A.col_idx.data(), sizeof(int) * sys.A.nnz());
      std::memcpy(val, sys.A.vals.data(), sizeof(double) * sys.A.nnz());
      std::memcpy(b, sys.b.data(), sizeof(double) * sys.A.n);
    }
  })
}

uint64_t vqpref_mesh_fingerprint(int r) { return mesh_fingerprint(make_mesh(r)); }

int vqpref_lumped_mass(int r, double* mass) {
  GUARD({
    const auto m = lumped_mass(make_mesh(r));
    std::memcpy(mass, m.data(), sizeof(double) * m.size());
  })
}

// reference assign (quantizer.cpp:134-145) for B rows of stride ld
int vqpref_assign(int method, int map, int P, int m, const double* lambdas, const double* centroids,
                  const double* xi, int64_t B, int ld, int32_t* labels) {
  GUARD({
    const Codebook cb = make_codebook(method, map, P, m, lambdas, centroids);
    for (int64_t i = 0; i < B; ++i)
      labels[i] = assign(cb, {xi + static_cast<size_t>(i) * ld, static_cast<size_t>(m)});
  })
}

// reference kmeans (quantizer.cpp:347-357)
int vqpref_kmeans(const double* samples, int n, int m, const double* lambdas, int map, int P,
                  uint64_t init_seed, int max_iter, double rel_tol, double* centroids_out,
                  double* history_out, int* n_history) {
  GUARD({
    SampleSet s;
    s.n = n;
    s.m = m;
    s.data.assign(samples, samples + static_cast<size_t>(n) * m);
    T2Map t2{map == 0 ? MapKind::Scale : MapKind::ScaledCdf, {lambdas, lambdas + m}};
    std::vector<double> hist;
    const Codebook cb = kmeans(s, t2, P, init_seed, max_iter, rel_tol, &hist);
    std::memcpy(centroids_out, cb.centroids.data(), sizeof(double) * cb.centroids.size());
    if (history_out) std::memcpy(history_out, hist.data(), sizeof(double) * hist.size());
    if (n_history) *n_history = static_cast<int>(hist.size());
  })
}

int vqpref_grid_latent_sites(int m, double s, double* out) {
  GUARD({
    const auto v = grid_latent_sites(m, s);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  })
}

// reference centroid_coefficient (quantizer.cpp:465-476) over a caller basis
int vqpref_centroid_coefficient(int method, int map, int P, int m, const double* lambdas,
                                const double* centroids, int p, const double* evals,
                                const double* evecs, int n_kl, int n_nodes, double* out) {
  GUARD({
    const Codebook cb = make_codebook(method, map, P, m, lambdas, centroids);
    KLBasis basis;
    basis.eigenvalues.assign(evals, evals + n_kl);
    basis.eigenvectors.assign(evecs, evecs + static_cast<size_t>(n_kl) * n_nodes);
    basis.mass.assign(n_nodes, 1.0);
    const auto k = centroid_coefficient(cb, p, basis);
    std::memcpy(out, k.data(), sizeof(double) * k.size());
  })
}

// artifact round trips with the reference's own reader/writer (artifacts.cpp)
int vqpref_load_codebook(const char* path, int* m, int* P, int* map, int* method, double* lambdas,
                         double* centroids) {
  GUARD({
    const Codebook cb = load_codebook(path);
    *m = cb.m;
    *P = cb.P;
    *map = cb.t2.kind == MapKind::Scale ? 0 : 1;
    *method = cb.method == QuantMethod::KMeans ? 0 : cb.method == QuantMethod::Clvq ? 1 : 2;
    if (lambdas) std::memcpy(lambdas, cb.t2.lambdas.data(), sizeof(double) * cb.m);
    if (centroids) std::memcpy(centroids, cb.centroids.data(), sizeof(double) * cb.centroids.size());
  })
}

int vqpref_save_codebook(const char* path, int method, int map, int P, int m, const double* lambdas,
                         const double* centroids, uint64_t seed) {
  GUARD({
    Codebook cb = make_codebook(method, map, P, m, lambdas, centroids);
    cb.seed = seed;
    save_codebook(path, cb);
  })
}

int vqpref_load_kl_basis(const char* path, int* n_kl, int* n_nodes, double* evals, double* evecs,
                         double* mass, double* total_variance) {
  GUARD({
    const KLBasis b = load_kl_basis(path);
    *n_kl = b.n_kl();
    *n_nodes = b.n_nodes();
    *total_variance = b.total_variance;
    if (evals) std::memcpy(evals, b.eigenvalues.data(), sizeof(double) * b.eigenvalues.size());
    if (evecs) std::memcpy(evecs, b.eigenvectors.data(), sizeof(double) * b.eigenvectors.size());
    if (mass) std::memcpy(mass, b.mass.data(), sizeof(double) * b.mass.size());
  })
}

int vqpref_save_kl_basis(const char* path, int n_kl, int n_nodes, const double* evals,
                         const double* evecs, const double* mass, double total_variance, double sigma2,
                         double ell, int mesh_resolution, uint64_t mesh_hash) {
  GUARD({
    KLBasis b;
    b.eigenvalues.assign(evals, evals + n_kl);
    b.eigenvectors.assign(evecs, evecs + static_cast<size_t>(n_kl) * n_nodes);
    b.mass.assign(mass, mass + n_nodes);
    b.total_variance = total_variance;
    b.sigma2 = sigma2;
    b.ell = ell;
    b.mesh_resolution = mesh_resolution;
    b.mesh_hash = mesh_hash;
    save_kl_basis(path, b);
  })
}

}  // extern "C"
