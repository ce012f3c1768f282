"""Parity at BASELINE sizes (north_star "every config
reproduces the CPU oracle"), against the multi-threaded CPU oracle.

* B.2: labels bit-identical over EVERY sample of C2 (2^17), C3 (2^16) and C5
  (2^20 x 4096 x 64), the oracle's nearest_row (quantizer.cpp:113-130) threaded
  over rows.
* B.3/B.4 on >= 4096 full-size samples of C2, C3 and C5: status agreement, the
  |dJ| histogram and mean J, against the same statistics of the oracle's own
  FMA-contracted build (the rounding-level yardstick) where that is affordable.
* 2-D at r = 256 (65,025 unknowns): C4 (IC(0)) on 256 samples and C4chol (the
  reference's cholesky kind) on 64 samples, with the 2-D FMA yardstick; and
  C4's reference-order mode bit-identical to the oracle at full size.
Every test prints its statistics (the GPU logs under profiles/ are these prints).
"""
import os

import numpy as np
import pytest

import oracle
from paper_2403_07824_b200 import campaign, lib
from tests.helpers import compare_runs, oracle_codebook, setup_case

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


def _hist(dj):
    h = np.bincount(np.minimum(dj, 10))
    return {("%d" % k if k < 10 else ">=10"): int(v) for k, v in enumerate(h) if v}


def _stats(ref, res):
    cmp = compare_runs(ref["iterations"], ref["status"], res["iterations"], res["status"])
    both = (ref["status"] == 0) & (res["status"] == 0)
    dj = np.abs(ref["iterations"][both].astype(np.int64) - res["iterations"][both])
    cmp["hist"] = _hist(dj)
    cmp["mean_diff"] = abs(cmp["mean_cpu"] - cmp["mean_gpu"])
    return cmp


def _show(tag, cmp):
    print(tag, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in cmp.items() if k != "disagree"},
          "status disagreements:", cmp["disagree"][:20].tolist(), flush=True)


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_full_b_labels_bit_identical(name):
    """Appendix B.2 at the configuration's full B."""
    cfg = campaign.CONFIGS[name]
    arts = campaign.prepare_campaign(cfg)
    basis, cb = arts["basis"], arts["codebook"]
    K = basis["eigenvalues"].size
    B = cfg["n_realizations"]
    xi = lib.draw_standard_normal(B, K, cfg["master_seed"])
    ctx = campaign.make_context(cfg, arts, factor=False)
    lab = ctx.assign(xi)
    ctx.close()
    ref = oracle.assign(oracle_codebook(cb), xi, threads=THREADS)
    bad = np.nonzero(lab != ref)[0]
    print(name, f"labels: {B} samples, {bad.size} differ", flush=True)
    assert bad.size == 0, bad[:10]


def _full_j(name, n, yardstick):
    cfg, basis, cb, xi = setup_case(name, n)
    ocb = oracle_codebook(cb)
    res = campaign.run_campaign_with(cfg, dict(basis=basis, codebook=cb), xi)
    args = (cfg["dim"], cfg["mesh_resolution"], cfg["precond"], ocb, basis["eigenvalues"], basis["eigenvectors"], xi,
            cfg["eps"])
    ref = oracle.run_campaign(*args, threads=THREADS)
    assert np.array_equal(res["labels"], ref["labels"])
    cmp = _stats(ref, res)
    _show(f"{name} n={n} gpu-vs-oracle", cmp)
    yard = None
    if yardstick:
        with oracle.fma_variant():
            ref_fma = oracle.run_campaign(*args, threads=THREADS)
        yard = _stats(ref, ref_fma)
        _show(f"{name} n={n} fma-yardstick", yard)
    return cfg, cmp, yard


@pytest.mark.parametrize("name,n,yardstick", [("C2", 4096, True), ("C3", 4096, True), ("C5", 4096, False)])
def test_full_size_j_parity(name, n, yardstick):
    """Appendix B.3/B.4 on 4096 full-size samples. The GPU's spread must not
    exceed the reference's own rounding-level spread (its FMA build) beyond small
    absolute floors; C5 (the oracle needs ~7 min for 4096 samples) uses the floors
    measured on the yardstick of the other 1-D configurations."""
    cfg, cmp, yard = _full_j(name, n, yardstick)
    if yard is None:  # C5: floors from the C2/C3 yardsticks (profiles/r02_fullsize_gpu.log)
        yard = dict(status_agree=0.98, frac_dj=0.07, mean_diff=0.01)
    else:
        # samples converged on both sides: as many as the yardstick keeps (rtol 1e-8 sits at the
        # attainable accuracy: ~10 % of C2's and ~40 % of C5's samples stagnate to a breakdown)
        assert cmp["n_both"] >= yard["n_both"] - 0.01 * n
    assert cmp["status_agree"] >= min(yard["status_agree"], 0.995) - 0.01, (cmp, yard)
    assert cmp["frac_dj"] <= max(1.5 * yard["frac_dj"], 0.01), (cmp, yard)
    assert cmp["mean_diff"] <= max(3 * yard["mean_diff"], 0.01), (cmp, yard)


def test_c4_full_size_256_samples():
    """C4 at r = 256 (65,025 unknowns, IC(0)): 256 samples vs the 16-thread oracle,
    beside the 2-D FMA yardstick. Fast mode differs from the oracle only in the
    dot-product summation order (block tree vs serial)."""
    cfg, cmp, yard = _full_j("C4", 256, True)
    assert cmp["status_agree"] == 1.0 and cmp["n_both"] == 256
    # mean J (~900) within 0.5 % and per-sample |dJ| small; the yardstick is printed beside
    assert cmp["mean_diff"] <= max(0.005 * cmp["mean_cpu"], 3 * yard["mean_diff"]), (cmp, yard)
    assert cmp["max_dj"] <= max(20, 2 * yard["max_dj"]), (cmp, yard)


def test_c4_full_size_exact_mode_bit_identical():
    """C4 at r = 256 in reference-order mode (serial natural-order dot products):
    J, status, final residual and x bit-identical to the oracle given the same
    coefficient bits, at the full BASELINE mesh."""
    cfg, basis, cb, xi = setup_case("C4", 24)
    ocb = oracle_codebook(cb)
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    ctx.set_exact_reductions(True)
    kc = ctx.centroid_coefficients()
    labels = oracle.assign(ocb, xi)
    assert np.array_equal(ctx.assign(xi), labels)
    kap, _ = ctx.realise(xi)
    it, rel, st, x = ctx.solve_batch(xi, labels, cfg["eps"], want_x=True)
    ctx.close()
    pset = oracle.PreconditionerSet.from_coefficients(2, cfg["mesh_resolution"], "ic0", kc)
    from concurrent.futures import ThreadPoolExecutor

    def one(i):
        return pset.pcg(int(labels[i]), kap[i], cfg["eps"])

    with ThreadPoolExecutor(THREADS) as ex:
        outs = list(ex.map(one, range(len(xi))))
    for i, out in enumerate(outs):
        assert out["iterations"] == it[i] and out["status"] == st[i], (i, out["iterations"], it[i])
        assert out["rel"] == rel[i], i
        assert np.array_equal(out["x"], x[i]), i
    print("C4 exact mode r=256: %d samples bit-identical, mean J %.2f" % (len(xi), it.mean()), flush=True)


def test_c4chol_full_size_64_samples():
    """C4chol (the reference's cholesky kind, RCM + LL^T of every centroid matrix)
    at r = 256 on 64 samples vs the 16-thread oracle, beside the FMA yardstick."""
    cfg, cmp, yard = _full_j("C4chol", 64, True)
    assert cmp["status_agree"] == 1.0 and cmp["n_both"] == 64
    assert cmp["max_dj"] <= max(2, yard["max_dj"]), (cmp, yard)
    assert cmp["mean_diff"] <= max(3 * yard["mean_diff"], 0.05), (cmp, yard)


def test_ic0_paper_size_mesh():
    """The paper's problem size (n = 99,681 unknowns) on the structured
    mesh r = 317 (99,856 unknowns) with the IC(0) kind: meshes beyond r = 257 run the
    level sweeps with 512-thread CTAs (one thread per grid row). Reference-order mode
    is bit-identical to the oracle; the fast mode's J stays within the C4 band."""
    from concurrent.futures import ThreadPoolExecutor

    from tests.helpers import CONFIGS
    name = "C4ic317"
    CONFIGS.setdefault(name, campaign.scaled(campaign.CONFIGS["C4"], mesh_resolution=317, name=name))
    cfg, basis, cb, xi = setup_case(name, 16)
    ocb = oracle_codebook(cb)
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    assert ctx.n == 316 * 316
    fast = ctx.run_campaign(xi, cfg["eps"])
    ctx.set_exact_reductions(True)
    kc = ctx.centroid_coefficients()
    labels = oracle.assign(ocb, xi)
    assert np.array_equal(fast["labels"], labels)
    kap, _ = ctx.realise(xi)
    it, rel, st, x = ctx.solve_batch(xi, labels, cfg["eps"], want_x=True)
    ctx.close()
    pset = oracle.PreconditionerSet.from_coefficients(2, cfg["mesh_resolution"], "ic0", kc)
    with ThreadPoolExecutor(THREADS) as ex:
        outs = list(ex.map(lambda i: pset.pcg(int(labels[i]), kap[i], cfg["eps"]), range(len(xi))))
    for i, out in enumerate(outs):
        assert out["iterations"] == it[i] and out["status"] == st[i] and out["rel"] == rel[i], (i, out["iterations"], it[i])
        assert np.array_equal(out["x"], x[i]), i
    dj = np.abs(fast["iterations"].astype(int) - it)
    print("r=317 (n=99,856) IC(0): J exact", it.tolist(), "fast", fast["iterations"].tolist(), flush=True)
    assert (fast["status"] == 0).all() and dj.max() <= 20 and abs(fast["iterations"].mean() - it.mean()) <= 0.005 * it.mean()
