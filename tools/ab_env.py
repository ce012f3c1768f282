"""A/B one build of libvqpc.so under two environment settings (e.g. VQPC_MAX_GROUPS=148
vs 296) on one config: device-campaign time and whether every per-sample record is
bit-identical.

usage: python tools/ab_env.py C4 2048 VQPC_MAX_GROUPS=148 VQPC_MAX_GROUPS=296 [reps] [exact]
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from ab_libs import CHILD  # noqa: E402


def run(env_kv, name, n, reps, out, exact):
    env = dict(os.environ)
    for kv in env_kv.split(","):
        if kv:
            k, v = kv.split("=", 1)
            env[k] = v
    code = CHILD % dict(root=ROOT, name=name, n=n, reps=reps, out=out)
    if exact:
        code = code.replace("ctx = campaign.make_context(cfg, arts)",
                            "ctx = campaign.make_context(cfg, arts); ctx.set_exact_reductions(True)")
    subprocess.check_call([sys.executable, "-c", code], env=env)
    return np.load(out)


def main():
    name, n, a, b = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    exact = len(sys.argv) > 6 and sys.argv[6] == "exact"
    d = tempfile.mkdtemp()
    ra = run(a, name, n, reps, os.path.join(d, "a.npz"), exact)
    rb = run(b, name, n, reps, os.path.join(d, "b.npz"), exact)
    same = all(np.array_equal(ra[k], rb[k]) for k in ("iterations", "status", "rel", "labels"))
    for tag, r, e in (("A", ra, a), ("B", rb, b)):
        print(f"{name} n={n} {'exact ' if exact else ''}{tag} [{e}]: pcg {float(r['pcg_ms']):.1f} ms, "
              f"{n / float(r['step_ms']) * 1e3:.1f} samples/s")
    print(f"speedup B/A {float(ra['pcg_ms']) / float(rb['pcg_ms']):.4f}  bit-identical={same}")
    if not same:
        for k in ("iterations", "status", "rel"):
            print(k, "differs in", int((ra[k] != rb[k]).sum()), "samples")


if __name__ == "__main__":
    main()
