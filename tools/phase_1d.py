"""Per-barrier phase cycles of the 1-D PCG (run with VQPC_LIB pointing at a -DVQPC_PHASE_TIMING build)."""
import sys, time
import numpy as np
from paper_2403_07824_b200 import campaign, lib
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(n, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts)
ctx.run_campaign(xi, cfg["eps"])
lib.pcg1d_phase_cycles(reset=True)
t = time.time(); res = ctx.run_campaign(xi, cfg["eps"]); dt = time.time() - t
ph = lib.pcg1d_phase_cycles(reset=True)
it = res["iterations"].sum()
print(f"{name} n={n} wall {dt:.3f}s iters {it}  total {sum(ph) / it:.0f} cycles/iteration")
for nm, c in zip(("Ap+pAp", "update+resid+sweep1", "sweep2", "rz"), ph):
    print(f"  {nm:22s} {c / it:8.0f} cycles/iteration")
