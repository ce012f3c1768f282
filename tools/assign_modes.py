"""Time the assignment kernel on one config's shape (run twice, with and without
VQPC_ASSIGN_DIRECT=1, to compare the contraction-plus-recheck path with the direct one)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(n, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts, factor=False)
lab0 = ctx.assign(xi)
ctx.profile(True)
ctx.profile_read(reset=True)
lab = ctx.assign(xi)
ms = ctx.profile_read(reset=True)["assign"]["ms"]
P, m = arts["codebook"]["P"], cfg["m"]
mode = "direct" if os.environ.get("VQPC_ASSIGN_DIRECT") else "contraction+recheck"
print(f"{name} {n} samples, m={m} P={P}: {mode} assign {ms:.3f} ms, {3.0 * P * m * n / ms / 1e9:.2f} T exact-op-equivalents/s")
import numpy as np  # noqa: E402
np.save(f"/tmp/labels_{mode[:6]}.npy", lab)
