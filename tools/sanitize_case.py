"""One small campaign per kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck):

  C1     pcg1d (single CTA per sample), realise, assign, bucket
  C5     pcg1d 2-CTA cluster variant (DSMEM st.async + mbarrier exchanges), assign_mma
  C4s    pcg2d (cp.async rings, level sweeps), IC(0) factor
  C4chol pcgchol2d (TMA bulk copies, mbarriers, DMMA), cholfactor2d (shared-flag spins)
  C4amg  pcgamg2d (V-cycle, warp-level dense coarse solve)
  exact  the reference-order kernels (1-D exact, 2-D chol exact)

usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py C4chol
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2403_07824_b200 import campaign, lib  # noqa: E402

CASES = {
    "C1": (campaign.scaled(campaign.CONFIGS["C1"], n_realizations=64), {}),
    "C5": (campaign.scaled(campaign.CONFIGS["C5"], n_realizations=8, chunk=0, solve_subset=None), {}),
    "C4s": (campaign.scaled(campaign.CONFIGS["C4"], mesh_resolution=32, name="C4s", n_realizations=8), {}),
    "C4chol": (campaign.scaled(campaign.CONFIGS["C4chol"], mesh_resolution=32, name="C4chols", n_realizations=16),
               {"VQPC_CHOL_S": "8"}),
    "C4amg": (campaign.scaled(campaign.CONFIGS["C4amg"], mesh_resolution=32, name="C4amgs", n_realizations=8), {}),
}


def run(name):
    if name == "exact":
        for sub in ("C1", "C4chol"):
            cfg, env = CASES[sub]
            os.environ.update(env)
            arts = campaign.prepare_campaign(cfg)
            xi = lib.draw_standard_normal(4, arts["basis"]["eigenvalues"].size, cfg["master_seed"])
            ctx = campaign.make_context(cfg, arts)
            ctx.set_exact_reductions(True)
            res = ctx.run_campaign(xi, cfg["eps"], max_iter=200)
            print(sub, "exact:", res["iterations"].tolist(), res["status"].tolist())
            ctx.close()
        return
    cfg, env = CASES[name]
    os.environ.update(env)
    arts = campaign.prepare_campaign(cfg)
    xi = lib.draw_standard_normal(cfg["n_realizations"], arts["basis"]["eigenvalues"].size, cfg["master_seed"])
    res = campaign.run_campaign_with(cfg, arts, xi)
    print(name, "J:", res["iterations"].tolist(), "status:", np.bincount(res["status"]).tolist())


if __name__ == "__main__":
    run(sys.argv[1])
