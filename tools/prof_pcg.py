"""One C2 campaign over n samples (for ncu captures of the pcg kernel)."""
import sys, time
import numpy as np
from paper_2403_07824_b200 import campaign, lib
from tests.helpers import setup_case
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg, basis, cb, _ = setup_case(name, 8192)
xi = lib.draw_standard_normal(n, basis["eigenvalues"].size, 0)
ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
t = time.time(); res = ctx.run_campaign(xi, cfg["eps"]); dt = time.time() - t
st, it = res["status"], res["iterations"]
print(f"{name} n={n} wall {dt:.3f}s status {np.bincount(st, minlength=3)} iters {it.sum()} "
      f"max {it.max()} ns/sample-iter/SM {dt/it.sum()*148*1e9:.0f}")
