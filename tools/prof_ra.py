"""One C5-shaped chunk through realise and assign (ncu captures of kernels (a), (b))."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

cfg = campaign.CONFIGS["C5"]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(16384, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts, factor=False)
lab = ctx.assign(xi)
kap, st = ctx.realise(xi)
print("ok", lab[:4], kap.shape)
