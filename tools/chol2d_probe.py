"""C4chol probe: factor time of the 32 centroid envelopes at r = 256 and the
grouped-PCG throughput for the S given by VQPC_CHOL_S (GPU; diagnostics only)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
MAXIT = int(sys.argv[2]) if len(sys.argv) > 2 else -1
cfg = campaign.CONFIGS["C4chol"]
basis = campaign.load_or_build_basis(cfg)
cb = campaign.load_or_build_codebook(cfg, basis)
t0 = time.perf_counter()
ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
t1 = time.perf_counter()
K = basis["eigenvalues"].size
rng = np.random.default_rng(1)
xi = rng.standard_normal((B, K))
ctx.run_campaign(xi[:64], cfg["eps"])  # warm-up
ctx.profile(True)
t2 = time.perf_counter()
res = ctx.run_campaign(xi, cfg["eps"], max_iter=MAXIT)
t3 = time.perf_counter()
prof = ctx.profile_read()
print(f"S={os.environ.get('VQPC_CHOL_S', '8')} context+factor {t1 - t0:.2f} s; campaign {B} samples {t3 - t2:.2f} s "
      f"-> {B / (t3 - t2):.1f} samples/s, mean J {res['iterations'].mean():.2f}, status {np.bincount(res['status'])}; "
      f"prof {prof}")
