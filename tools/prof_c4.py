"""C4 campaign over n samples (ncu captures of the 2-D kernel)."""
import sys, time
import numpy as np
from paper_2403_07824_b200 import campaign, lib
from tests.helpers import setup_case
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg, basis, cb, _ = setup_case("C4", 8)
xi = lib.draw_standard_normal(n, basis["eigenvalues"].size, 0)
ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
t = time.time(); res = ctx.run_campaign(xi, cfg["eps"]); dt = time.time() - t
print(f"C4 n={n} wall {dt:.3f}s iters {res['iterations'].sum()} status {np.bincount(res['status'])}")
