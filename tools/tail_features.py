"""Per-sample work and candidate cost predictors of a full campaign (work-queue
ordering study): J, status, label, the current key (KL-weighted distance to the
centroid field) and features of the realised log-field h = Phi^T (sqrt(lambda) xi):
its range, its maximum deviation from the centroid's field and the deviation's
mass-weighted mean square. Writes gpurun_out/<name>_tail.npz.

usage: python tools/tail_features.py C2
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign, lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
basis, cb = arts["basis"], arts["codebook"]
lam = basis["eigenvalues"]
K, m = lam.size, cfg["m"]
B = cfg.get("solve_subset") or cfg["n_realizations"]
xi = lib.draw_standard_normal(B, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts)
res = ctx.run_campaign(xi, cfg["eps"])
dev = torch.device("cuda", 0)
phi = torch.from_numpy(basis["eigenvectors"]).to(dev)  # K x N
sl = torch.from_numpy(np.sqrt(lam)).to(dev)
chi = np.asarray(cb["centroids"]) / np.sqrt(np.asarray(cb["lambdas"]))[None, :]
hc = (torch.from_numpy(chi).to(dev) * sl[:m]) @ phi[:m]  # P x N centroid log-fields
lab = torch.from_numpy(res["labels"].astype(np.int64)).to(dev)
out = {k: [] for k in ("hrange", "hmax", "hmin", "dmax", "dms", "key")}
for c0 in range(0, B, 8192):
    x = torch.from_numpy(xi[c0:c0 + 8192]).to(dev)
    h = (x * sl) @ phi
    d = h - hc[lab[c0:c0 + 8192]]
    out["hmax"].append(h.max(1).values)
    out["hmin"].append(h.min(1).values)
    out["hrange"].append(h.max(1).values - h.min(1).values)
    out["dmax"].append(d.abs().max(1).values)
    out["dms"].append((d * d).mean(1))
    xc = x.clone()
    xc[:, :m] -= torch.from_numpy(chi).to(dev)[lab[c0:c0 + 8192]]
    out["key"].append(((xc * sl) ** 2).sum(1))
np.savez_compressed(f"gpurun_out/{name}_tail.npz", it=res["iterations"], st=res["status"], labels=res["labels"],
                    **{k: torch.cat(v).cpu().numpy() for k, v in out.items()})
print("saved", B, np.bincount(res["status"]), "hmax[:3]", torch.cat(out["hmax"])[:3].cpu().numpy(), "xi0", xi[0, :3])
