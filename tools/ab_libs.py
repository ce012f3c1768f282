"""A/B two builds of libvqpc.so on one config: device-campaign samples/s and
whether every per-sample result is bit-identical.

usage: python tools/ab_libs.py C2 32768 path/to/libA.so path/to/libB.so [reps]
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CHILD = r"""
import os, sys, time
import numpy as np
sys.path.insert(0, %(root)r)
from paper_2403_07824_b200 import campaign, lib
cfg = campaign.CONFIGS[%(name)r]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(%(n)d, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts)
kw = dict(chunk=cfg.get("chunk", 0), solve_limit=cfg.get("solve_subset") or -1)
ctx.run_campaign(xi, cfg["eps"], **kw)
best = None
for _ in range(%(reps)d):
    ctx.profile(True); ctx.profile_read(reset=True)
    res = ctx.run_campaign(xi, cfg["eps"], **kw)
    prof = ctx.profile_read(reset=True); ctx.profile(False)
    ms = prof["pcg"]["ms"]
    step = sum(v["ms"] for v in prof.values())
    best = ms if best is None else min(best, ms)
np.savez(%(out)r, pcg_ms=best, step_ms=step, **{k: res[k] for k in ("iterations", "status", "rel", "labels")})
"""


def run(libpath, name, n, reps, out):
    env = dict(os.environ, VQPC_LIB=os.path.abspath(libpath))
    code = CHILD % dict(root=ROOT, name=name, n=n, reps=reps, out=out)
    subprocess.check_call([sys.executable, "-c", code], env=env)
    return np.load(out)


def main():
    name, n, a, b = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    d = tempfile.mkdtemp()
    ra = run(a, name, n, reps, os.path.join(d, "a.npz"))
    rb = run(b, name, n, reps, os.path.join(d, "b.npz"))
    it = ra["iterations"].astype(np.int64).sum()
    same = all(np.array_equal(ra[k], rb[k]) for k in ("iterations", "status", "rel", "labels"))
    for tag, r, p in (("A", ra, a), ("B", rb, b)):
        ms = float(r["pcg_ms"])
        print(f"{name} n={n} {tag} {os.path.basename(p)}: pcg {ms:.2f} ms, {it / ms / 1e3:.2f} M iter/s, "
              f"all kernels {float(r['step_ms']):.2f} ms")
    print(f"speedup B/A {float(ra['pcg_ms']) / float(rb['pcg_ms']):.4f}  bit-identical={same}")
    if not same:
        for k in ("iterations", "status", "rel"):
            print(k, "differs in", int((ra[k] != rb[k]).sum()), "samples")


if __name__ == "__main__":
    main()
