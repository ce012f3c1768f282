"""GPU edge cases through the C ABI: empty and ragged batches, non-finite and
extreme inputs, invalid arguments, size limits — each checked against the
reference's semantics (and the oracle where it restates them)."""
import numpy as np
import pytest

import oracle
from paper_2403_07824_b200 import campaign, lib
from tests.helpers import oracle_codebook, setup_case

pytestmark = pytest.mark.gpu


def _case(name, n):
    cfg, basis, cb, xi = setup_case(name, n)
    return cfg, basis, cb, xi, campaign.make_context(cfg, dict(basis=basis, codebook=cb))


def test_empty_batch():
    cfg, basis, cb, xi, ctx = _case("C1", 16)
    res = ctx.run_campaign(xi[:0], cfg["eps"])
    assert res["labels"].size == 0 and res["iterations"].size == 0
    assert int(res["n_p"].sum()) == 0 and res["total_iterations"] == 0
    assert ctx.assign(xi[:0]).size == 0
    it, _, st, _ = ctx.solve_batch(xi[:0], np.zeros(0, np.int32), cfg["eps"])
    assert it.size == 0 and st.size == 0
    kap, st = ctx.realise(xi[:0])
    assert kap.shape == (0, ctx.n_nodes)
    # and the context still works afterwards
    assert np.array_equal(ctx.assign(xi), oracle.assign(oracle_codebook(cb), xi))


@pytest.mark.parametrize("name", ["C2", "C4s"])
def test_non_finite_and_extreme_inputs_follow_reference_semantics(name):
    """Per-sample statuses where the reference throws:
    * non-finite xi_k, k < m: assign's invalid-latent (quantizer.cpp:135-138), label -1;
    * non-finite xi_k, k >= m: lift -> transport's coefficient-overflow (field.cpp:141-142);
    * exp overflow: coefficient-overflow; exp underflow to kappa == 0: assembly's
      invalid-coefficient (the first KL mode is positive, so xi_0 = -3000 drives
      every h below -745).
    Well-formed neighbours in the same batch are unaffected."""
    cfg, basis, cb, xi, ctx = _case(name, 8)
    m = cfg["m"]
    x = xi.copy()
    x[1, 0] = np.nan
    x[2, m + 1] = np.nan
    x[3, 0] = 3.0e3
    x[4, 0] = -3.0e3
    x[5, 1] = np.inf
    res = ctx.run_campaign(x, cfg["eps"])
    st, lab = res["status"], res["labels"]
    assert lab[1] == -1 and lab[5] == -1 and (lab[[0, 2, 3, 4, 6, 7]] >= 0).all()
    assert list(st[1:6]) == [4, 3, 3, 5, 4], st
    assert (res["iterations"][1:6] == 0).all()
    ok = [0, 6, 7]
    ref = ctx.run_campaign(xi[ok], cfg["eps"])
    for k in ("labels", "iterations", "rel", "status"):
        assert np.array_equal(res[k][ok], ref[k]), k
    # realise alone reports the same coefficient statuses
    _, rst = ctx.realise(x[2:5])
    assert list(rst) == [3, 3, 5]
    # the oracle's per-sample solve (reference lift/transport/assemble semantics)
    ocb = oracle_codebook(cb)
    pset = oracle.PreconditionerSet.build(cfg["dim"], cfg["mesh_resolution"], cfg["precond"], ocb,
                                          basis["eigenvalues"], basis["eigenvectors"])
    _, _, st_o, _ = pset.solve_batch(basis["eigenvalues"], basis["eigenvectors"], x[2:5], lab[2:5], cfg["eps"])
    assert list(st_o) == [3, 3, 5]
    # the reference's campaign aborts on the first invalid latent; the oracle restates that
    with pytest.raises(oracle.OracleError, match="invalid-latent"):
        oracle.run_campaign(cfg["dim"], cfg["mesh_resolution"], cfg["precond"], ocb, basis["eigenvalues"],
                            basis["eigenvectors"], x[:2], cfg["eps"])


def test_invalid_tolerance_and_zero_iterations():
    cfg, basis, cb, xi, ctx = _case("C1", 8)
    lab = ctx.assign(xi)
    for eps in (0.0, -1.0, 1.0, 2.0, float("nan")):  # solver.cpp:188-190
        with pytest.raises(lib.VqpcError, match="invalid-tolerance"):
            ctx.run_campaign(xi, eps)
        with pytest.raises(lib.VqpcError, match="invalid-tolerance"):
            ctx.solve_batch(xi, lab, eps)
    # max_iter = 0: the loop never runs -> J = 0, not converged (the oracle agrees)
    it, rel, st, _ = ctx.solve_batch(xi, lab, cfg["eps"], max_iter=0)
    assert (it == 0).all() and (st == 1).all()
    ocb = oracle_codebook(cb)
    pset = oracle.PreconditionerSet.build(1, cfg["mesh_resolution"], "cholesky", ocb, basis["eigenvalues"],
                                          basis["eigenvectors"])
    jo, _, so, _ = pset.solve_batch(basis["eigenvalues"], basis["eigenvectors"], xi, lab, cfg["eps"], max_iter=0)
    assert np.array_equal(jo, it) and np.array_equal(so, st)
    # max_iter = 1 everywhere, and a ragged per-sample cap, both match the oracle bit for bit in J/status
    cap = np.arange(len(xi), dtype=np.int32) % 5
    it2, _, st2, _ = ctx.solve_batch(xi, lab, cfg["eps"], max_iter_arr=cap)
    jo2, _, so2, _ = pset.solve_batch(basis["eigenvalues"], basis["eigenvectors"], xi, lab, cfg["eps"],
                                      max_iter_arr=cap)
    assert np.array_equal(it2, jo2) and np.array_equal(st2, so2)


def test_duplicate_rows_and_ragged_chunks():
    """Identical realisations give identical records wherever they sit in the
    batch; chunk sizes that do not divide B (1, 7, 333) change nothing."""
    cfg, basis, cb, xi, ctx = _case("C3", 700)
    x = np.concatenate([xi[:50], xi[:50], xi[50:]])
    a = ctx.run_campaign(x, cfg["eps"])
    for k in ("labels", "iterations", "rel", "status"):
        assert np.array_equal(a[k][:50], a[k][50:100]), k
    for chunk in (7, 333):
        b = ctx.run_campaign(x, cfg["eps"], chunk=chunk)
        for k in ("labels", "iterations", "rel", "status", "n_p", "sum_j"):
            assert np.array_equal(a[k], b[k]), (chunk, k)
    c = ctx.run_campaign(x[:3], cfg["eps"], chunk=1)
    for k in ("labels", "iterations", "rel", "status"):
        assert np.array_equal(a[k][:3], c[k]), k


def test_size_limits():
    """n = 8192 rows is the largest 1-D system (2-CTA clusters; C5 has 8191); beyond it the
    context refuses with invalid-config instead of failing at launch. The 2-D
    IC(0) kind puts one thread on each grid row: r <= 513 (512-thread CTAs above
    r = 257), beyond it invalid-config likewise."""
    rng = np.random.default_rng(0)
    cb = dict(method="kmeans", map="scale", lambdas=np.ones(2), centroids=rng.standard_normal((4, 2)))
    for dim, size in ((1, 8193), (2, 257), (2, 513)):
        nn = size if dim == 1 else (size + 1) ** 2
        basis = dict(eigenvalues=np.array([1.0, 0.5]), eigenvectors=rng.standard_normal((2, nn)) * 1e-3)
        ctx = lib.Context(dim, size, basis, cb, "cholesky" if dim == 1 else "ic0")
        ctx.factor_centroids()
        ctx.close()
    for dim, size in ((1, 8194), (2, 514)):
        nn = size if dim == 1 else (size + 1) ** 2
        basis = dict(eigenvalues=np.array([1.0, 0.5]), eigenvectors=np.zeros((2, nn)))
        with pytest.raises(lib.VqpcError, match="invalid-config"):
            lib.Context(dim, size, basis, cb, "cholesky" if dim == 1 else "ic0")


def test_async_campaigns_on_two_contexts_match_sync():
    """vqpc_run_campaign_async: batches enqueued alternately on two contexts (the
    bench's pipelined steps) give the synchronous call's records and statistics."""
    cfg, basis, cb, xi, ctx = _case("C3", 300)
    ref = ctx.run_campaign(xi, cfg["eps"])
    ctx2 = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    outs = [c.campaign_outputs(len(xi)) for c in (ctx, ctx2)]
    for k in range(4):
        c = (ctx, ctx2)[k % 2]
        c.run_campaign_async(xi, cfg["eps"], outs[k % 2])
    ctx.synchronize()
    ctx2.synchronize()
    for o in outs:
        assert np.array_equal(o["labels"], ref["labels"]) and np.array_equal(o["iterations"], ref["iterations"])
        assert np.array_equal(o["rel"], ref["rel"]) and np.array_equal(o["status"], ref["status"])
        assert np.array_equal(o["stats"][:ctx.P], ref["n_p"]) and int(o["summary"][0]) == ref["total_iterations"]
