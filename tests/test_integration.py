"""The reference-side binding compiles against the REAL reference headers and
links against libvqpc.so (no GPU needed: compile + link only; on a B200 box the
same program also runs a small 2-D campaign)."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
PROGRAM = r'''
#include "vqp_gpu_adapter.hpp"
#include <cstdio>
int main(int argc, char** argv) {
  if (argc < 2) return 0;  // link check only
  // a tiny 2-D campaign through the reference's own types
  vqp::CampaignArtifacts art;
  art.mesh.resolution = 8;
  const int nn = 81, K = 3;
  art.basis.eigenvalues = {0.1, 0.05, 0.02};
  art.basis.eigenvectors.assign(K * nn, 0.0);
  for (int k = 0; k < K; ++k)
    for (int i = 0; i < nn; ++i) art.basis.eigenvectors[k * nn + i] = 0.1 * ((i * (k + 1)) % 7 - 3);
  art.basis.mass.assign(nn, 1.0 / 64);
  art.codebook.m = 2; art.codebook.P = 2;
  art.codebook.t2.lambdas = {0.1, 0.05};
  art.codebook.centroids = {0.1, 0.0, -0.1, 0.0};
  vqp::CampaignConfig cfg; cfg.eps = 1e-8;
  vqp::SampleSet xi; xi.n = 16; xi.m = K; xi.data.assign(16 * K, 0.3);
  for (int i = 0; i < 16 * K; ++i) xi.data[i] = 0.1 * ((i * 5) % 11 - 5);
  vqp::gpu::GpuOptions opt;
  const vqp::SimulationReport rep = vqp::gpu::run_campaign_with(cfg, art, xi, opt);
  std::printf("n=%ld mean_j=%.3f unconverged=%ld\n", rep.n_realizations, rep.mean_j, rep.unconverged);
  return rep.unconverged == 0 ? 0 : 1;
}
'''


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not mounted")
def test_adapter_compiles_against_reference_headers_and_links():
    from paper_2403_07824_b200 import build
    lib = build.build()
    with tempfile.TemporaryDirectory() as t:
        src = os.path.join(t, "drv.cpp")
        open(src, "w").write(PROGRAM)
        exe = os.path.join(t, "drv")
        libdir = os.path.dirname(lib)
        cmd = ["g++", "-std=c++20", "-O1", f"-I{REF_INC}", f"-I{os.path.join(ROOT, 'include')}", src,
               f"-L{libdir}", "-l:" + os.path.basename(lib), f"-Wl,-rpath,{libdir}", "-o", exe]
        r = subprocess.run(cmd, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]
        assert subprocess.run([exe], capture_output=True).returncode == 0
