"""2-D campaigns with the reference's own `cholesky` preconditioner
(solver.cpp:72-111: RCM + LL^T of each centroid matrix; pcgchol2d.cuh) against
the CPU oracle's restatement (oracle/src/vqp_oracle.cpp CholeskyPreconditioner).

* the factor is bit-identical: the GPU's serial apply (vqpc_precond_apply) equals
  the oracle's apply bit for bit, which needs the same RCM permutation, envelope
  and every factor entry;
* the reference-order mode (serial dots, Eigen-order triangular solves:
  forward column-major lower, backward row-major upper view) is bit-identical to
  the oracle: J, status, final residual and x;
* the batched throughput solve (blocked DMMA triangular solves, tree dot
  products) is compared with the oracle beside the oracle's own FMA build (the
  rounding-level yardstick): statuses identical, max |dJ| and the mean-J gap no
  larger than the yardstick's plus one iteration / 0.5 iterations, x to 1e-10
  (relative l2) where J agrees; for 1, 2, 4 and 8 right-hand sides per CTA, on
  meshes whose row count is not a multiple of the 32-row block, and at r = 64,
  128, 200 and 257 (envelope width W = 256, the DMMA window's limit; the ring
  wraps and the backward sweep reloads y blocks).
"""
from concurrent.futures import ThreadPoolExecutor
import os

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


def _oracle_solves(pset, labels, kap, eps, n_threads=None):
    def one(i):
        return pset.pcg(int(labels[i]), kap[i], eps)
    with ThreadPoolExecutor(n_threads or os.cpu_count()) as ex:
        return list(ex.map(one, range(len(labels))))


@pytest.mark.parametrize("S,r,n_real", [(S, r, n) for S in (1, 2, 4, 8) for r, n in ((32, 48), (30, 24))]
                         + [(2, 64, 32), (8, 64, 32), (4, 128, 16), (8, 128, 16), (8, 200, 8), (2, 257, 6),
                            (8, 257, 8)])
def test_chol2d_solve_parity(monkeypatch, S, r, n_real):
    monkeypatch.setenv("VQPC_CHOL_S", str(S))
    cfg, basis, cb, xi = setup_case(_cfg_name(r), n_real)
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    kc = ctx.centroid_coefficients()
    labels = oracle.assign(oracle_codebook(cb), xi)
    kap, _ = ctx.realise(xi)
    it, rel, st, x = ctx.solve_batch(xi, labels, cfg["eps"], want_x=True)
    ctx.close()
    pset = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", kc)
    outs = _oracle_solves(pset, labels, kap, cfg["eps"])
    with oracle.fma_variant():
        pf = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", kc)
        outs_f = _oracle_solves(pf, labels, kap, cfg["eps"])
    jc = np.array([o["iterations"] for o in outs])
    jf = np.array([o["iterations"] for o in outs_f])
    assert [o["status"] for o in outs] == list(st)
    assert (rel < cfg["eps"]).all()
    dx = np.array([np.linalg.norm(o["x"] - x[i]) / np.linalg.norm(o["x"]) for i, o in enumerate(outs)])
    dj, dy = np.abs(jc - it), np.abs(jc - jf)
    print(f"r={r} S={S}: J gpu {it.mean():.3f} cpu {jc.mean():.3f} cpu+fma {jf.mean():.3f}; |dJ| max {dj.max()} "
          f"(fma {dy.max()}) frac>0 {np.mean(dj > 0):.3f} (fma {np.mean(dy > 0):.3f}); rel-l2(x) max {dx.max():.2e}, "
          f"on equal J {dx[dj == 0].max() if (dj == 0).any() else 0:.2e}")
    assert dj.max() <= dy.max() + 1
    assert abs(it.mean() - jc.mean()) <= abs(jf.mean() - jc.mean()) + 0.5
    if (dj == 0).any():
        assert dx[dj == 0].max() < 1e-10


@pytest.mark.parametrize("r,n_real", [(17, 16), (32, 24), (64, 8)])
def test_chol2d_exact_mode_bit_identical(r, n_real):
    """Reference-order mode of the 2-D cholesky kind (pcgchol2d_exact_kernel): with
    the same coefficient bits, J, status, final residual and x equal the oracle's
    (Eigen's solve order in both triangular sweeps, serial natural-order dots)."""
    cfg, basis, cb, xi = setup_case(_cfg_name(r), n_real)
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    ctx.set_exact_reductions(True)
    kc = ctx.centroid_coefficients()
    labels = oracle.assign(oracle_codebook(cb), xi)
    kap, _ = ctx.realise(xi)
    it, rel, st, x = ctx.solve_batch(xi, labels, cfg["eps"], want_x=True)
    ctx.close()
    pset = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", kc)
    for i, out in enumerate(_oracle_solves(pset, labels, kap, cfg["eps"])):
        assert out["iterations"] == it[i] and out["status"] == st[i], (i, out["iterations"], it[i])
        assert out["rel"] == rel[i], i
        assert np.array_equal(out["x"], x[i]), i
    print(f"chol2d exact mode r={r}: {n_real} samples bit-identical, mean J {it.mean():.2f}")


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


def test_chol_groups_cover_every_sample(monkeypatch):
    """The parallel group builder (chol_groups_kernel) emits every solved sample in
    exactly one group: a campaign with skewed buckets gives the same records for
    S = 1 and S = 8."""
    cfg, basis, cb, xi = setup_case(_cfg_name(17), 64)
    out = []
    for S in ("1", "8"):  # the group size is read when the context is created
        monkeypatch.setenv("VQPC_CHOL_S", S)
        ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
        out.append(ctx.run_campaign(xi, cfg["eps"]))
        ctx.close()
    a, b = out
    assert np.array_equal(a["labels"], b["labels"]) and np.array_equal(a["status"], b["status"])
    assert (a["status"] == 0).all() and np.array_equal(a["n_p"], b["n_p"])
