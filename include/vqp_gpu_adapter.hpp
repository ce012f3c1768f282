// vqp_gpu_adapter.hpp — the reference-side binding of include/vqpc.h.
//
// Header-only C++20 adapter a maintainer drops next to the reference library
// (/root/reference/proj, namespace vqp): it implements the reference's own
// interfaces on top of the C ABI, so a driver can switch its hot path with a
// one-line change. Types come from the reference headers:
//   vqp::CampaignConfig / CampaignArtifacts / SimulationReport  (driver.hpp:17-95)
//   vqp::SampleSet / Codebook / KLBasis                          (quantizer.hpp, field.hpp)
//   vqp::Preconditioner                                          (solver.hpp:13-20)
//   vqp::Error                                                   (error.hpp:10-19)
// Compile: -I<reference>/include -I<this repo>/include, link libvqpc.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "vqp/driver.hpp"
#include "vqp/error.hpp"
#include "vqp/solver.hpp"
#include "vqpc.h"

namespace vqp::gpu {

// What the reference's CampaignConfig cannot express (it is 2-D only and has
// no IC(0)): the model dimension/size, an optional override of the
// preconditioner kind, the chunking and the solve subset (BASELINE C5).
struct GpuOptions {
  int dim = 2;          // 1: N-element 1-D model (size = N); 2: r x r mesh (size = r)
  int size = 0;         // 0: take artifacts.mesh.resolution
  int precond = -1;     // -1: CampaignConfig::precond (gpu_precond); else a vqpc_precond (e.g. VQPC_PC_IC0)
  int64_t chunk = 0;
  int64_t solve_limit = -1;
  bool exact_reductions = false;
  int device = 0;
};

// vqp::Error whose code() is the reference's stable code string (error.hpp:8-19)
// and whose what() adds the library's detail message (vqpc_last_error).
class Error : public vqp::Error {
 public:
  Error(const char* code, std::string detail) : vqp::Error(code), what_(std::move(detail)) {}
  const char* what() const noexcept override { return what_.c_str(); }

 private:
  std::string what_;
};

inline void check(int code, const vqpc_ctx* ctx = nullptr) {
  if (code == VQPC_OK) return;
  std::string msg = vqpc_error_string(code);
  if (ctx && *vqpc_last_error(ctx)) msg = msg + ": " + vqpc_last_error(ctx);
  throw Error(vqpc_error_string(code), msg);
}

// CampaignConfig::precond (driver.hpp:13,36) -> the GPU kind that implements it, as
// build_preconditioner chooses the reference's (driver.cpp:117-126). Kinds without a
// GPU implementation raise invalid-config instead of silently substituting another.
inline int gpu_precond(PrecondKind kind) {
  switch (kind) {
    case PrecondKind::Cholesky: return VQPC_PC_CHOLESKY;
    case PrecondKind::Amg: return VQPC_PC_AMG;
    default:
      throw Error("invalid-config", std::string("invalid-config: preconditioner kind '") +
                                        (kind == PrecondKind::Identity ? "identity" : "block_jacobi") +
                                        "' has no GPU implementation (cholesky, amg; ic0 via GpuOptions::precond)");
  }
}

// Device-resident basis + codebook + the P centroid factors. Owns a vqpc_ctx.
class Context {
 public:
  Context(const CampaignArtifacts& art, const GpuOptions& opt, int precond) {
    const Codebook& cb = art.codebook;
    const KLBasis& basis = art.basis;
    // import_mesh (fem.cpp:83-114) leaves resolution = 0: the device kernels are written for
    // the structured mesh of make_mesh (fem.cpp:53-81) and refuse an unstructured one
    if (opt.dim == 2 && opt.size <= 0 && art.mesh.resolution <= 0)
      throw Error("invalid-config",
                  "invalid-config: the mesh was imported (TriMesh::resolution == 0); the GPU path needs the "
                  "structured r x r mesh of make_mesh (any r with the amg kind, r <= 513 ic0, r <= 257 cholesky)");
    vqpc_problem pb{};
    pb.dim = opt.dim;
    pb.size = opt.size > 0 ? opt.size : art.mesh.resolution;
    pb.n_kl = basis.n_kl();
    pb.n_nodes = basis.n_nodes();
    pb.eigenvalues = basis.eigenvalues.data();
    pb.eigenvectors = basis.eigenvectors.data();
    pb.method = cb.method == QuantMethod::KMeans ? VQPC_KMEANS : cb.method == QuantMethod::Clvq ? VQPC_CLVQ : VQPC_GRID;
    pb.map = cb.t2.kind == MapKind::Scale ? VQPC_SCALE : VQPC_CDF;
    pb.P = cb.P;
    pb.m = cb.m;
    pb.lambdas = cb.t2.lambdas.data();
    pb.centroids = cb.centroids.data();
    pb.latent = cb.latent_centroids.empty() ? nullptr : cb.latent_centroids.data();
    pb.precond = precond;
    pb.device = opt.device;
    vqpc_ctx* c = nullptr;
    check(vqpc_ctx_create(&pb, &c));
    ctx_.reset(c);
    if (opt.exact_reductions) check(vqpc_set_exact_reductions(ctx(), 1), ctx());
    check(vqpc_factor_centroids(ctx()), ctx());  // driver.cpp:212-219 on the device
  }
  vqpc_ctx* ctx() const { return ctx_.get(); }
  int unknowns() const { return vqpc_unknowns(ctx_.get()); }

 private:
  struct Del {
    void operator()(vqpc_ctx* c) const { vqpc_ctx_destroy(c); }
  };
  std::unique_ptr<vqpc_ctx, Del> ctx_;
};

// The reference's Preconditioner interface (solver.hpp:13-20) backed by a GPU
// centroid factor: apply() solves M_p z = r on the device.
class GpuCentroidPreconditioner final : public Preconditioner {
 public:
  GpuCentroidPreconditioner(std::shared_ptr<Context> c, int p) : c_(std::move(c)) { built_from = p; }
  void apply(std::span<const double> r, std::span<double> z) const override {
    check(vqpc_precond_apply(c_->ctx(), built_from, r.data(), z.data()), c_->ctx());
  }
  const char* kind() const override { return "gpu-centroid-factor"; }

 private:
  std::shared_ptr<Context> c_;
};

// int assign(const Codebook&, span<const double>) (quantizer.hpp:92), batched.
inline std::vector<int> assign_all(const Context& c, const SampleSet& xi) {
  std::vector<int32_t> lab(static_cast<size_t>(xi.n));
  check(vqpc_assign(c.ctx(), xi.data.data(), xi.n, xi.m, lab.data()), c.ctx());
  for (int32_t l : lab)
    if (l < 0) throw vqp::Error("invalid-latent");  // the reference throws on non-finite xi
  return {lab.begin(), lab.end()};
}

// SimulationReport run_campaign_with(config, artifacts, realizations)
// (driver.hpp:93-95) on the GPU. Per-sample failures that make the reference
// throw (pcg-breakdown inside a worker) are reported as unconverged
// records instead of aborting the process.
namespace detail {
inline SimulationReport campaign(const CampaignConfig& config, const CampaignArtifacts& artifacts,
                                 const SampleSet& realizations, const GpuOptions& opt, std::vector<double>* x) {
  Context c(artifacts, opt, opt.precond >= 0 ? opt.precond : gpu_precond(config.precond));
  const int64_t B = realizations.n;
  const int P = artifacts.codebook.P;
  std::vector<int32_t> labels(B), iters(B);
  std::vector<double> rel(B);
  std::vector<uint8_t> status(B);
  std::vector<int64_t> stats(4 * static_cast<size_t>(P)), summary(4);
  if (x) {
    x->assign(static_cast<size_t>(B) * vqpc_unknowns(c.ctx()), 0.0);
    check(vqpc_run_campaign_x(c.ctx(), realizations.data.data(), B, realizations.m, config.eps, -1, opt.chunk,
                              opt.solve_limit, labels.data(), iters.data(), rel.data(), status.data(), stats.data(),
                              summary.data(), x->data()),
          c.ctx());
  } else {
    check(vqpc_run_campaign_ex(c.ctx(), realizations.data.data(), B, realizations.m, config.eps, -1, opt.chunk,
                               opt.solve_limit, labels.data(), iters.data(), rel.data(), status.data(), stats.data(),
                               summary.data()),
          c.ctx());
  }
  SimulationReport rep;
  rep.n_realizations = B;
  rep.assignments.assign(labels.begin(), labels.end());
  rep.records.resize(B);
  for (int64_t i = 0; i < B; ++i)
    rep.records[i] = {iters[i], rel[i], status[i] == VQPC_S_CONVERGED, labels[i]};
  rep.per_centroid.assign(P, {});
  for (int p = 0; p < P; ++p) {
    auto& s = rep.per_centroid[p];
    s.n_p = stats[p];
    s.sum_j = stats[P + p];
    s.mean_j = stats[2 * P + p] > 0 ? static_cast<double>(stats[3 * P + p]) / stats[2 * P + p] : 0.0;
    double nsq = 0.0;  // Codebook::centroid_norm (quantizer.cpp:89-93), inlined to stay header-only
    for (double v : artifacts.codebook.centroid(p)) nsq += v * v;
    s.centroid_norm = std::sqrt(nsq);
  }
  rep.total_iterations = summary[0];
  rep.unconverged = summary[1];
  rep.mean_j = summary[2] > 0 ? static_cast<double>(summary[3]) / summary[2] : 0.0;
  rep.max_sum_j = rep.min_sum_j = 0;
  if (P > 0) {
    rep.max_sum_j = rep.min_sum_j = rep.per_centroid[0].sum_j;
    for (const auto& s : rep.per_centroid) {
      rep.max_sum_j = std::max(rep.max_sum_j, s.sum_j);
      rep.min_sum_j = std::min(rep.min_sum_j, s.sum_j);
    }
  }
  return rep;
}
}  // namespace detail

inline SimulationReport run_campaign_with(const CampaignConfig& config, const CampaignArtifacts& artifacts,
                                          const SampleSet& realizations, const GpuOptions& opt) {
  return detail::campaign(config, artifacts, realizations, opt, nullptr);
}

// run_campaign_with plus the solutions the reference computes and discards
// (driver.cpp:236-237; SURVEY §8b run_campaign_with_solutions): x is resized to
// B x n, row i = the PCG iterate of realisation i at its exit (zeros for
// realisations that were not solved).
inline SimulationReport run_campaign_with_solutions(const CampaignConfig& config, const CampaignArtifacts& artifacts,
                                                    const SampleSet& realizations, const GpuOptions& opt,
                                                    std::vector<double>& x) {
  return detail::campaign(config, artifacts, realizations, opt, &x);
}

}  // namespace vqp::gpu
