"""A/B the pcg kernel layouts on one config: samples/s of the device campaign and
whether per-sample results are bit-identical across layouts.

usage: python tools/pcg_variants.py C2 32768 VAR=VAL[,VAR=VAL] ...   ("-" = defaults)
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2])
variants = sys.argv[3:] or ["-"]
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(n, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts)
base = None
for v in variants:
    env = {} if v == "-" else dict(kv.split("=") for kv in v.split(","))
    for k, val in env.items():
        os.environ[k] = val
    ctx.run_campaign(xi, cfg["eps"])  # warm
    ctx.profile(True)
    ctx.profile_read(reset=True)
    t = time.perf_counter()
    res = ctx.run_campaign(xi, cfg["eps"])
    dt = time.perf_counter() - t
    prof = ctx.profile_read(reset=True)
    ctx.profile(False)
    for k in env:
        del os.environ[k]
    same = None
    if base is None:
        base = res
    else:
        same = all(np.array_equal(res[k], base[k]) for k in ("iterations", "status", "rel", "labels"))
    it = res["iterations"].astype(np.int64).sum()
    print(f"{name} n={n} [{v}] {n / dt:,.0f} samples/s wall, pcg {prof['pcg']['ms']:.2f} ms, "
          f"{it / (prof['pcg']['ms'] / 1e3) / 1e6:.2f} M iter/s, identical={same}", flush=True)
ctx.close()
