"""Dump per-sample labels / J / status of a full campaign (work-queue ordering analysis)."""
import sys
import numpy as np
from paper_2403_07824_b200 import campaign, lib
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = campaign.CONFIGS[name]
arts = campaign.prepare_campaign(cfg)
K = arts["basis"]["eigenvalues"].size
B = cfg["n_realizations"]
xi = lib.draw_standard_normal(B, K, cfg["master_seed"])
ctx = campaign.make_context(cfg, arts)
res = ctx.run_campaign(xi, cfg["eps"], chunk=cfg.get("chunk", 0))
np.savez_compressed(f"gpurun_out/{name}_res.npz", labels=res["labels"], it=res["iterations"], st=res["status"],
                    rel=res["rel"], xi8=xi[:, :cfg["m"]])
print("saved", B)
