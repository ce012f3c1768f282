"""Work-queue study: per-sample J of a full campaign and the relative true residual
after T iterations (a capped campaign), for a two-phase (probe, then resume
longest-first) schedule simulation. Writes gpurun_out/<name>_probe.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
B = cfg.get("solve_subset") or cfg["n_realizations"]
xi = lib.draw_standard_normal(B, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts)
full = ctx.run_campaign(xi, cfg["eps"])
out = dict(it=full["iterations"], st=full["status"], labels=full["labels"])
for T in (50, 100, 200, 400):
    r = ctx.run_campaign(xi, cfg["eps"], max_iter=T)
    out[f"rel{T}"] = r["rel"]
    out[f"st{T}"] = r["status"]
np.savez_compressed(f"gpurun_out/{name}_probe.npz", **out)
print("saved", B)
