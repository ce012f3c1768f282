"""C4 phase breakdown of the 2-D PCG: run with VQPC_LIB pointing at a -DVQPC_PHASE_TIMING build."""
import sys, time
import numpy as np
from paper_2403_07824_b200 import campaign, lib
from tests.helpers import setup_case
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg, basis, cb, _ = setup_case("C4", 8)
xi = lib.draw_standard_normal(n, basis["eigenvalues"].size, 0)
ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
lib.pcg2d_phase_cycles(reset=True)
t = time.time(); res = ctx.run_campaign(xi, cfg["eps"]); dt = time.time() - t
ph = lib.pcg2d_phase_cycles(reset=True)
it = res["iterations"].sum()
print(f"C4 n={n} wall {dt:.3f}s samples/s {n/dt:.0f} iters {it}")
for name, c in zip(("setup", "sweeps", "P1", "P2"), ph):
    print(f"  {name:7s} {c / it:10.0f} cycles/iteration/CTA")
