"""Shared setup for parity tests: artifacts are built once (KL basis by the
product's setup code, codebooks by the CPU oracle's kmeans — the same bits the
GPU-assisted kmeans produces, which test_gpu_parity checks separately) and
both sides consume identical xi arrays."""
import numpy as np

import oracle
from paper_2403_07824_b200 import campaign

CONFIGS = dict(campaign.CONFIGS)
# reduced 2-D case with C4's field and solver settings (r = 32: 961 unknowns) for
# parity runs the CPU oracle finishes in seconds
CONFIGS["C4s"] = campaign.scaled(campaign.CONFIGS["C4"], mesh_resolution=32, name="C4s")


def setup_case(name, n_real=None, ns=None, **over):
    cfg = campaign.scaled(CONFIGS[name], n_realizations=n_real, ns=ns, **over)
    basis = campaign.load_or_build_basis(cfg)
    if name == "C5":
        # P = 4096 on 2^18 pilot points: hours for the CPU oracle's Lloyd, seconds
        # with the GPU sweeps (bit-identical; tested on smaller cases)
        cb = campaign.load_or_build_codebook(cfg, basis)
    else:
        cb = campaign.load_or_build_codebook(cfg, basis, kmeans_fn=oracle.kmeans, draw_fn=oracle.draw_standard_normal)
    K = basis["eigenvalues"].size
    xi = oracle.draw_standard_normal(cfg["n_realizations"], K, cfg["master_seed"])
    return cfg, basis, cb, xi


def oracle_codebook(cb):
    return oracle.Codebook(cb["method"], cb["map"], cb["lambdas"], cb["centroids"], cb.get("latent"))


def compare_runs(j_cpu, s_cpu, j_gpu, s_gpu):
    """Appendix B protocol summary: status agreement, |dJ| on converged-both,
    mean J over converged-both samples."""
    both = (s_cpu == 0) & (s_gpu == 0)
    dj = np.abs(j_cpu[both].astype(np.int64) - j_gpu[both])
    return dict(status_agree=float(np.mean(s_cpu == s_gpu)), n_both=int(both.sum()),
                max_dj=int(dj.max()) if dj.size else 0, frac_dj=float(np.mean(dj > 0)) if dj.size else 0.0,
                mean_cpu=float(j_cpu[both].mean()) if both.any() else 0.0,
                mean_gpu=float(j_gpu[both].mean()) if both.any() else 0.0,
                disagree=np.nonzero(s_cpu != s_gpu)[0])
