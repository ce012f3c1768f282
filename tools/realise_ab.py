"""A/B two builds of libvqpc.so on the realisation kernel (a): DMMA TFLOP/s on one
config's shape and whether kappa is bit-identical.

usage: python tools/realise_ab.py C5 16384 libA.so libB.so
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, %(root)r)
from paper_2403_07824_b200 import campaign, lib
cfg = campaign.CONFIGS[%(name)r]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
xi = lib.draw_standard_normal(%(n)d, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts, factor=False)
kap, st = ctx.realise(xi)
best = 1e30
for _ in range(5):
    ctx.profile(True); ctx.profile_read(reset=True)
    ctx.realise(xi)
    best = min(best, ctx.profile_read(reset=True)["realise"]["ms"]); ctx.profile(False)
np.savez(%(out)r, kap=kap, st=st, ms=best, flops=2.0 * ctx.n_nodes * K * %(n)d)
"""
name, n, a, b = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
d = tempfile.mkdtemp()
res = []
for tag, libp in (("A", a), ("B", b)):
    out = os.path.join(d, tag + ".npz")
    subprocess.check_call([sys.executable, "-c", CHILD % dict(root=ROOT, name=name, n=n, out=out)],
                          env=dict(os.environ, VQPC_LIB=os.path.abspath(libp)))
    r = np.load(out)
    res.append(r)
    print(f"{name} {n} samples {tag} {os.path.basename(libp)}: realise {float(r['ms']):.3f} ms, "
          f"{float(r['flops']) / float(r['ms']) / 1e9:.2f} TFLOP/s")
print("speedup B/A %.4f  kappa bit-identical=%s" % (float(res[0]["ms"]) / float(res[1]["ms"]),
                                                    np.array_equal(res[0]["kap"], res[1]["kap"])))
