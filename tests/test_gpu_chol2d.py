"""2-D campaigns with the reference's own `cholesky` preconditioner
(solver.cpp:72-111: RCM + LL^T of each centroid matrix; pcgchol2d.cuh) against
the CPU oracle's restatement (oracle/src/vqp_oracle.cpp CholeskyPreconditioner).

* the factor is bit-identical: the GPU's serial apply (vqpc_precond_apply) equals
  the oracle's apply bit for bit, which needs the same RCM permutation, envelope
  and every factor entry;
* the batched solve (blocked triangular solves, tree dot products) reproduces the
  oracle's iteration counts within +-1 and its solutions to 1e-10 (relative l2),
  for 1, 2 and 4 right-hand sides per CTA and meshes whose row count is not a
  multiple of the 32-row block.
"""
import numpy as np
import pytest

import oracle
from paper_2403_07824_b200 import campaign, lib

from tests.helpers import CONFIGS, oracle_codebook, setup_case

pytestmark = pytest.mark.gpu


def _cfg_name(r):
    name = f"C4chol{r}"
    if name not in CONFIGS:
        CONFIGS[name] = campaign.scaled(campaign.CONFIGS["C4"], mesh_resolution=r, precond="cholesky", name=name)
    return name


@pytest.mark.parametrize("r", [17, 30, 32])
def test_chol2d_factor_and_apply_bit_identical(r):
    cfg, basis, cb, _ = setup_case(_cfg_name(r), 4)
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    kc = ctx.centroid_coefficients()
    pset = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", kc)
    rng = np.random.default_rng(r)
    for p in (0, cb["P"] // 2, cb["P"] - 1):
        v = rng.standard_normal(ctx.n)
        assert np.array_equal(ctx.precond_apply(p, v), pset.apply(p, v)), (r, p)
    ctx.close()


@pytest.mark.parametrize("S", [1, 2, 4, 8])
@pytest.mark.parametrize("r,n_real", [(32, 48), (30, 24)])
def test_chol2d_solve_parity(monkeypatch, S, r, n_real):
    monkeypatch.setenv("VQPC_CHOL_S", str(S))
    cfg, basis, cb, xi = setup_case(_cfg_name(r), n_real)
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    kc = ctx.centroid_coefficients()
    labels = oracle.assign(oracle_codebook(cb), xi)
    kap, _ = ctx.realise(xi)
    pset = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", kc)
    it, rel, st, x = ctx.solve_batch(xi, labels, cfg["eps"], want_x=True)
    jc = np.empty(len(xi), dtype=np.int64)
    dx = np.empty(len(xi))
    for i in range(len(xi)):
        out = pset.pcg(int(labels[i]), kap[i], cfg["eps"])
        assert out["status"] == st[i], i
        assert rel[i] < cfg["eps"]
        jc[i] = out["iterations"]
        dx[i] = np.linalg.norm(out["x"] - x[i]) / np.linalg.norm(out["x"])
    dj = np.abs(jc - it)
    print(f"r={r} S={S}: J gpu {it.mean():.3f} cpu {jc.mean():.3f}, |dJ| max {dj.max()} frac>0 {np.mean(dj > 0):.3f};"
          f" rel-l2(x) max {dx.max():.2e}, on equal J {dx[dj == 0].max():.2e}")
    assert dj.max() <= 2 and np.mean(dj > 1) <= 0.05
    assert abs(it.mean() - jc.mean()) < 0.5
    assert dx[dj == 0].max() < 1e-10
    ctx.close()


def test_chol2d_campaign_vs_oracle():
    """run_campaign_with end to end (assign, bucket, realise, grouped PCG, stats)."""
    name = _cfg_name(32)
    cfg, basis, cb, xi = setup_case(name, 96)
    res = campaign.run_campaign_with(cfg, dict(basis=basis, codebook=cb), xi)
    ref = oracle.run_campaign(2, 32, "cholesky", oracle_codebook(cb), basis["eigenvalues"], basis["eigenvectors"], xi,
                              cfg["eps"])
    assert np.array_equal(res["labels"], ref["labels"])
    assert np.array_equal(res["status"], ref["status"])
    with oracle.fma_variant():  # yardstick: the reference's own arithmetic with FMA contraction
        yard = oracle.run_campaign(2, 32, "cholesky", oracle_codebook(cb), basis["eigenvalues"],
                                   basis["eigenvectors"], xi, cfg["eps"])
    dj = np.abs(res["iterations"].astype(int) - ref["iterations"])
    dy = np.abs(yard["iterations"].astype(int) - ref["iterations"])
    print(f"chol2d r=32 campaign: J gpu {res['iterations'].mean():.3f} cpu {ref['iterations'].mean():.3f} "
          f"cpu+fma {yard['iterations'].mean():.3f}; |dJ| gpu max {dj.max()} frac>0 {np.mean(dj > 0):.3f}, "
          f"cpu+fma max {dy.max()} frac>0 {np.mean(dy > 0):.3f}")
    assert dj.max() <= max(2, dy.max()) and np.mean(dj > 1) <= 0.05
    assert abs(res["iterations"].mean() - ref["iterations"].mean()) < 0.5


def test_chol2d_records_edges(monkeypatch):
    """Invalid latents, a solve limit and an iteration cap inside one S = 4 group."""
    monkeypatch.setenv("VQPC_CHOL_S", "4")
    cfg, basis, cb, xi = setup_case(_cfg_name(32), 16)
    xi = xi.copy()
    xi[3, 0] = np.nan
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    full = ctx.run_campaign(xi, cfg["eps"])
    assert full["status"][3] == 4 and full["iterations"][3] == 0  # invalid latent
    ok = np.arange(16) != 3
    assert np.all(full["status"][ok] == 0)
    lim = ctx.run_campaign(xi, cfg["eps"], solve_limit=8)
    assert np.all(lim["status"][8:] == 6)
    assert np.array_equal(lim["iterations"][:8], full["iterations"][:8])
    labels = ctx.assign(xi)
    it, rel, st, _ = ctx.solve_batch(xi, labels, cfg["eps"], max_iter=3)
    assert np.all(it[ok] == 3) and np.all(st[ok] == 1)
    ctx.close()


def test_chol2d_rejects_exact_mode():
    cfg, basis, cb, xi = setup_case(_cfg_name(32), 4)
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    ctx.set_exact_reductions(True)
    labels = oracle.assign(oracle_codebook(cb), xi)
    with pytest.raises(lib.VqpcError, match="invalid-config"):
        ctx.solve_batch(xi, labels, cfg["eps"])
    ctx.close()
