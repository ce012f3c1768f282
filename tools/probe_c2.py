"""Quick timing probe of the C2 campaign (host arrays, wall clock)."""
import sys, time
import numpy as np
from paper_2403_07824_b200 import campaign, lib
from tests.helpers import setup_case
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 17
cfg, basis, cb, _ = setup_case(name, 8192)
K = basis["eigenvalues"].size
t = time.time(); xi = lib.draw_standard_normal(n, K, 0); print("draw", time.time() - t, flush=True)
ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
for rep in range(2):
    t = time.time(); res = ctx.run_campaign(xi, cfg["eps"]); dt = time.time() - t
    st = res["status"]; it = res["iterations"]
    print(f"{name} n={n} wall {dt:.3f}s  samples/s {n/dt:.0f}  status {np.bincount(st, minlength=3)}  "
          f"meanJ(conv) {it[st==0].mean():.3f}  total_iters {it.sum()}  launches {ctx.launches}", flush=True)
