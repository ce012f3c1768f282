"""ideal_sweep (driver.cpp:290-340): per-realisation
preconditioners built from the m-truncated coefficient, applied to the
full-coefficient systems — the paper's Fig. 2 "ideal" curve.

CPU: the oracle's restatement has the reference's properties (mean J falls as m
grows; m = n_kl is the exact factor of the sample's own matrix, so the cholesky
kind needs exactly one iteration; relative energy rises to 1).
GPU: the device sweep (per-realisation factors through the campaign's own PCG
kernels) equals the oracle record for record in reference-order mode, and
matches its statistics in the throughput mode; the context's centroid factors
survive the sweep.
"""
import numpy as np
import pytest

import oracle
from paper_2403_07824_b200 import campaign
from tests.helpers import CONFIGS, setup_case

CONFIGS.setdefault("C4amgs", campaign.scaled(campaign.CONFIGS["C4amg"], mesh_resolution=32, name="C4amgs"))
CONFIGS.setdefault("C4chols", campaign.scaled(campaign.CONFIGS["C4chol"], mesh_resolution=32, name="C4chols"))


def _oracle_sweep(cfg, basis, xi, m_list, kind=None):
    return oracle.ideal_sweep(cfg["dim"], cfg["mesh_resolution"], kind or cfg["precond"], basis["eigenvalues"],
                              basis["eigenvectors"], xi, m_list, cfg["eps"])


def test_oracle_ideal_sweep_properties():
    cfg, basis, cb, xi = setup_case("C1", 48)
    K = basis["eigenvalues"].size
    m_list = [0, 2, 8, K]
    rec = _oracle_sweep(cfg, basis, xi, m_list)
    rows = campaign.sweep_rows(basis, m_list, rec)
    assert rows[0]["relative_energy"] == 0.0 and rows[-1]["relative_energy"] == pytest.approx(1.0, abs=1e-6)
    assert all(a["mean_j"] >= b["mean_j"] for a, b in zip(rows, rows[1:]))
    assert (rec["iterations"][:, -1] == 1).all()  # the exact factor of the sample's own matrix


@pytest.mark.gpu
@pytest.mark.parametrize("name,n", [("C1", 64), ("C4s", 24), ("C4chols", 12), ("C4amgs", 24)])
def test_gpu_ideal_sweep_exact_mode_bit_identical(name, n):
    """Reference-order mode: every (realisation, m) record equals the oracle's pcg
    with the oracle's preconditioner built from the same truncated coefficient bits
    (ctx.realise over the first m modes) on the same full-coefficient system; the
    context's centroid factors are intact after the sweep."""
    cfg, basis, cb, xi = setup_case(name, n)
    K = basis["eigenvalues"].size
    m_list = [0, 3, cfg["m"], K]
    ctx = campaign.make_context(cfg, dict(basis=basis, codebook=cb))
    before = ctx.run_campaign(xi, cfg["eps"])
    ctx.set_exact_reductions(True)
    g = ctx.ideal_sweep(xi, m_list, cfg["eps"], max_iter=2000)
    kap, _ = ctx.realise(xi)
    kap_m = [ctx.realise(xi, m)[0] for m in m_list]
    ctx.set_exact_reductions(False)
    after = ctx.run_campaign(xi, cfg["eps"])  # the centroid factors are intact
    ctx.close()
    for k in ("labels", "iterations", "rel", "status"):
        assert np.array_equal(before[k], after[k]), k
    nn = cfg["mesh_resolution"] if cfg["dim"] == 1 else (cfg["mesh_resolution"] + 1) ** 2
    for j, m in enumerate(m_list):
        pset = oracle.PreconditionerSet.from_coefficients(cfg["dim"], cfg["mesh_resolution"], cfg["precond"],
                                                          kap_m[j][:, :nn])
        for i in range(n):
            out = pset.pcg(i, kap[i, :nn], cfg["eps"], max_iter=2000)
            assert out["iterations"] == g["iterations"][i, j] and out["status"] == g["status"][i, j], (i, m)
            assert out["rel"] == g["rel"][i, j], (i, m)
    rows = campaign.sweep_rows(basis, m_list, g)
    print(name, "ideal sweep (exact mode, bit-identical):", [(r["m"], round(r["relative_energy"], 4),
                                                               round(r["mean_j"], 3)) for r in rows])
    if cfg["precond"] == "cholesky":
        assert (g["iterations"][:, -1] == 1).all()


@pytest.mark.gpu
def test_gpu_ideal_sweep_c2_throughput_mode():
    """The throughput kernels on C2's full-size systems: rows within the oracle's
    rounding spread (its FMA build) and the m = n_kl column exactly one iteration."""
    cfg, basis, cb, xi = setup_case("C2", 256)
    K = basis["eigenvalues"].size
    m_list = [0, 4, 8, 16, K]
    res = campaign.ideal_sweep(cfg, dict(basis=basis, codebook=cb), xi, m_list)
    o = _oracle_sweep(cfg, basis, xi, m_list)
    with oracle.fma_variant():
        f = _oracle_sweep(cfg, basis, xi, m_list)
    rg, ro, rf = (campaign.sweep_rows(basis, m_list, r) for r in (res, o, f))
    print("C2 ideal sweep rows (m, energy, mean J gpu / oracle / oracle+fma):",
          [(a["m"], round(a["relative_energy"], 4), round(a["mean_j"], 3), round(b["mean_j"], 3), round(c["mean_j"], 3))
           for a, b, c in zip(rg, ro, rf)])
    assert (res["iterations"][:, -1] == 1).all()
    for a, b, c in zip(rg, ro, rf):
        assert abs(a["mean_j"] - b["mean_j"]) <= max(3 * abs(c["mean_j"] - b["mean_j"]), 0.05 * b["mean_j"])
    assert np.mean(res["status"] == o["status"]) >= 0.98
