"""Time the realisation kernel in both modes (DMMA vs the reference-order CUDA-core
AXPY of vqpc_set_exact_reductions) on one config's shape."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(n, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts, factor=False)
N = ctx.n_nodes
for exact in (False, True):
    ctx.set_exact_reductions(exact)
    ctx.realise(xi)
    ctx.profile(True)
    ctx.profile_read(reset=True)
    ctx.realise(xi)
    ms = ctx.profile_read(reset=True)["realise"]["ms"]
    ctx.profile(False)
    print(f"{name} {n} samples: {'reference-order' if exact else 'DMMA'} realise {ms:.3f} ms, "
          f"{2.0 * N * K * n / ms / 1e9:.2f} TFLOP/s")
