// drive_adapter.cpp — TEST PROGRAM: the reference-side drop-in, executed.
//
// A stand-in for the reference's own run_campaign (proj/src/driver.cpp:283-288)
// after the one-line switch INTEGRATION.md describes: the artifacts are loaded by
// the REFERENCE's own loaders (vqp::load_kl_basis / vqp::load_codebook,
// proj/src/artifacts.cpp:69-127, compiled unchanged into oracle/_ref/libvqpref.so),
// the mesh by the reference's make_mesh (fem.cpp:53-81), and the campaign runs
// through include/vqp_gpu_adapter.hpp's vqp::gpu::run_campaign_with, which returns
// the reference's SimulationReport (driver.hpp:65-75). The report is written as
// JSON so tests/test_integration.py can compare it with the ctypes run.
//
// usage: drive_adapter <basis.klb> <codebook.qnt> <xi.bin> <out.json> <precond> <dim> <size> [gpu_precond]
//   precond: the CampaignConfig::precond string (cholesky | amg | identity | block_jacobi)
//   gpu_precond: optional GpuOptions::precond override (vqpc_precond number, e.g. 4 = IC(0))
//   xi.bin: int64 n, int64 m, then n x m doubles (row-major SampleSet)
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "vqp/artifacts.hpp"
#include "vqp/fem.hpp"
#include "vqp_gpu_adapter.hpp"

static vqp::PrecondKind kind_of(const std::string& s) {
  if (s == "cholesky") return vqp::PrecondKind::Cholesky;
  if (s == "amg") return vqp::PrecondKind::Amg;
  if (s == "identity") return vqp::PrecondKind::Identity;
  return vqp::PrecondKind::BlockJacobi;
}

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s basis.klb codebook.qnt xi.bin out.json precond dim size [gpu_precond]\n", argv[0]);
    return 2;
  }
  std::FILE* out = std::fopen(argv[4], "w");
  if (!out) return 2;
  try {
    vqp::CampaignArtifacts art;
    art.basis = vqp::load_kl_basis(argv[1]);
    art.codebook = vqp::load_codebook(argv[2]);
    const int dim = std::atoi(argv[6]), size = std::atoi(argv[7]);
    if (dim == 2) art.mesh = vqp::make_mesh(size);
    vqp::SampleSet xi;
    {
      std::ifstream f(argv[3], std::ios::binary);
      int64_t hdr[2];
      f.read(reinterpret_cast<char*>(hdr), sizeof hdr);
      xi.n = static_cast<int>(hdr[0]);
      xi.m = static_cast<int>(hdr[1]);
      xi.data.resize(static_cast<size_t>(hdr[0] * hdr[1]));
      f.read(reinterpret_cast<char*>(xi.data.data()), static_cast<std::streamsize>(sizeof(double) * xi.data.size()));
      if (!f) throw vqp::Error("artifact-not-found");
    }
    vqp::CampaignConfig config;
    config.mesh_resolution = size;
    config.eps = 1e-8;
    config.precond = kind_of(argv[5]);
    config.n_realizations = xi.n;
    vqp::gpu::GpuOptions opt;
    opt.dim = dim;
    opt.size = size;
    if (argc > 8) opt.precond = std::atoi(argv[8]);
    const vqp::SimulationReport rep = vqp::gpu::run_campaign_with(config, art, xi, opt);
    std::fprintf(out, "{\"ok\": true, \"n_realizations\": %ld, \"mean_j\": %.17g, \"total_iterations\": %ld, "
                 "\"max_sum_j\": %ld, \"min_sum_j\": %ld, \"unconverged\": %ld, \"per_centroid\": [",
                 rep.n_realizations, rep.mean_j, rep.total_iterations, rep.max_sum_j, rep.min_sum_j, rep.unconverged);
    for (size_t p = 0; p < rep.per_centroid.size(); ++p) {
      const auto& c = rep.per_centroid[p];
      std::fprintf(out, "%s{\"n_p\": %ld, \"sum_j\": %ld, \"mean_j\": %.17g, \"centroid_norm\": %.17g}", p ? ", " : "",
                   c.n_p, c.sum_j, c.mean_j, c.centroid_norm);
    }
    std::fprintf(out, "], \"assignments\": [");
    for (size_t i = 0; i < rep.assignments.size(); ++i) std::fprintf(out, "%s%d", i ? ", " : "", rep.assignments[i]);
    std::fprintf(out, "], \"iterations\": [");
    for (size_t i = 0; i < rep.records.size(); ++i) std::fprintf(out, "%s%d", i ? ", " : "", rep.records[i].iterations);
    std::fprintf(out, "], \"converged\": [");
    for (size_t i = 0; i < rep.records.size(); ++i) std::fprintf(out, "%s%d", i ? ", " : "", rep.records[i].converged ? 1 : 0);
    std::fprintf(out, "], \"final_rel\": [");
    for (size_t i = 0; i < rep.records.size(); ++i)
      std::fprintf(out, "%s%.17g", i ? ", " : "", rep.records[i].final_relative_residual);
    std::fprintf(out, "]}\n");
  } catch (const vqp::Error& e) {
    std::fprintf(out, "{\"ok\": false, \"code\": \"%s\", \"what\": \"%s\"}\n", e.code().c_str(), e.what());
    std::fclose(out);
    return 1;
  }
  std::fclose(out);
  return 0;
}
