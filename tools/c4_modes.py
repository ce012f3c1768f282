"""C4 (or another 2-D config) samples/s in the fast mode (block-tree dot
products) and in reference-order mode (serial natural-order dots,
vqpc_set_exact_reductions), on the same samples, with the J statistics of both.

usage: python tools/c4_modes.py [config] [n_samples]
"""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(n, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts)
out = {}
for exact in (False, True):
    ctx.set_exact_reductions(exact)
    ctx.run_campaign(xi[:64], cfg["eps"])
    t = time.perf_counter()
    res = ctx.run_campaign(xi, cfg["eps"])
    dt = time.perf_counter() - t
    out[exact] = res
    conv = res["status"] == 0
    print(f"{name} {'exact' if exact else 'fast '} mode: {n / dt:.1f} samples/s, mean J {res['iterations'][conv].mean():.3f}, "
          f"statuses {np.bincount(res['status'])}", flush=True)
a, b = out[False], out[True]
both = (a["status"] == 0) & (b["status"] == 0)
dj = a["iterations"][both].astype(int) - b["iterations"][both]
print("fast - exact dJ: mean %.3f, |dJ| hist %s" % (dj.mean(), np.bincount(np.minimum(np.abs(dj), 10))))
