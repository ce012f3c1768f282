"""C4chol phase breakdown of the grouped 2-D Cholesky PCG (cycles summed over CTAs by
thread 0): run with VQPC_LIB pointing at a -DVQPC_PHASE_TIMING build."""
import sys
import time

from paper_2403_07824_b200 import campaign, lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = campaign.CONFIGS["C4chol"]
basis = campaign.load_or_build_basis(cfg)
cb = campaign.load_or_build_codebook(cfg, basis)
xi = lib.draw_standard_normal(n, basis["eigenvalues"].size, 0)
ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
ctx.run_campaign(xi[:8], cfg["eps"], max_iter=2)
lib.pcg2d_phase_cycles(reset=True)
t = time.time()
res = ctx.run_campaign(xi, cfg["eps"], max_iter=maxit)
dt = time.time() - t
ph = lib.pcg2d_phase_cycles(reset=True)
it = res["iterations"].sum()
print(f"C4chol n={n} maxit={maxit} wall {dt:.3f}s iters {it}")
for name, c in zip(("issue", "solves", "mbar wait", "fwd compute"), ph):
    print(f"  {name:14s} {c / 1e6:10.1f} Mcycles summed over CTAs, {c / it:12.0f} per sample-iteration")
