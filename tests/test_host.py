"""Host-side pieces of the product that run without a GPU: KL basis setup,
artifacts, the C-ABI library's exported symbols, no-fallback behaviour and
the host coefficient sampler."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from paper_2403_07824_b200 import artifacts as art
from paper_2403_07824_b200 import campaign, klbasis, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_kl_basis_1d_properties():  # SPEC acceptance 2 (M-orthonormality, energy)
    b = klbasis.build_kl_basis_1d(1024, 1.0, 0.1, 50)
    lam, phi, mass = b["eigenvalues"], b["eigenvectors"], b["mass"]
    assert lam.size == 39  # degeneracy cutoff 1e-12 lambda_1 (field.cpp:51-54)
    assert np.all(np.diff(lam) <= 0)
    G = (phi * mass) @ phi.T
    assert np.abs(G - np.eye(lam.size)).max() < 1e-10
    for k in range(lam.size):  # sign convention (field.cpp:72-79), exact ties to the first index
        i = klbasis._sign_index(phi[k])
        assert phi[k, i] > 0
        a = np.abs(phi[k])
        assert a[i] >= a.max() * (1 - 1e-9) and np.all(a[:i] < a.max() * (1 - 1e-9))
    xi = np.random.default_rng(0).standard_normal((10, lam.size))
    h = (xi * np.sqrt(lam)) @ phi
    e1 = (h * h * mass).sum(1)
    e2 = ((xi * np.sqrt(lam)) ** 2).sum(1)
    assert np.allclose(e1, e2, rtol=1e-10)
    c5 = klbasis.build_kl_basis_1d(2048, 2.0, 0.1, 100, cutoff=False)
    assert c5["eigenvalues"].size == 100 and np.all(c5["eigenvalues"] > 0)


def test_kl_basis_2d_small_matches_dense():
    r = 8
    b = klbasis.build_kl_basis_2d(r, 1.0, 0.3, 12)
    side = r + 1
    t = np.arange(side) / r
    X, Y = np.meshgrid(t, t)
    x, y = X.ravel(), Y.ravel()
    C2 = np.exp(-((x[:, None] - x[None]) ** 2 + (y[:, None] - y[None]) ** 2) / 0.09)
    sm = np.sqrt(klbasis.lumped_mass_2d(r))
    w = np.linalg.eigvalsh(sm[:, None] * C2 * sm[None])[::-1]
    assert np.allclose(b["eigenvalues"], w[:12], rtol=1e-9)
    G = (b["eigenvectors"] * b["mass"]) @ b["eigenvectors"].T
    assert np.abs(G - np.eye(12)).max() < 1e-9


def test_kl_basis_2d_host_independent():
    """The basis does not depend on the eigensolver's start vector (a stand-in for
    the host): the corner masses split the lambda_ij / lambda_ji pairs of the
    separable kernel, so every mode is simple and even or odd under the grid
    transposition T, and the sign rule's exact ties (odd modes) go to the first
    index."""
    r = 20
    a = klbasis.build_kl_basis_2d(r, 1.0, 0.2, 24, v0_seed=1)
    b = klbasis.build_kl_basis_2d(r, 1.0, 0.2, 24, v0_seed=2)
    assert np.allclose(a["eigenvalues"], b["eigenvalues"], rtol=1e-11, atol=0)
    assert np.abs(a["eigenvectors"] - b["eigenvectors"]).max() < 1e-7
    lam = a["eigenvalues"]
    assert np.all(np.diff(lam) < 0)
    side = r + 1
    perm = np.arange(side * side).reshape(side, side).T.reshape(-1)
    for phi in a["eigenvectors"]:
        assert min(np.abs(phi[perm] - phi).max(), np.abs(phi[perm] + phi).max()) < 1e-6 * np.abs(phi).max()


def test_sign_rule_ties_take_first_index():
    v = np.array([0.1, -0.5, 0.2, 0.5 * (1 + 1e-13), -0.3])
    assert klbasis._sign_index(v) == 1
    assert klbasis._sign_index(np.array([0.1, 0.4, -0.5])) == 2


def test_artifact_round_trip(tmp_path):
    b = klbasis.build_kl_basis_1d(64, 1.0, 0.2, 8)
    b["mesh_hash"] = 123
    art.save_kl_basis(tmp_path / "b.klb", b)
    b2 = art.load_kl_basis(tmp_path / "b.klb")
    assert np.array_equal(b2["eigenvectors"], b["eigenvectors"]) and b2["mesh_hash"] == 123
    sites = art.sign_grid_sites(3)
    cb = dict(m=3, P=8, map="scale", method="sign_grid", seed=0, lambdas=b["eigenvalues"][:3],
              centroids=sites * np.sqrt(b["eigenvalues"][:3]))
    art.save_codebook(tmp_path / "c.qnt", cb)
    c2 = art.load_codebook(tmp_path / "c.qnt")
    assert np.array_equal(c2["latent"], sites) and np.array_equal(c2["centroids"], cb["centroids"])
    with pytest.raises(RuntimeError, match="artifact-corrupt"):
        (tmp_path / "x.qnt").write_bytes(b'{"format":"klb"}\n')
        art.load_codebook(tmp_path / "x.qnt")


def _header_functions():
    text = open(os.path.join(ROOT, "include", "vqpc.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vqpc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = lib.load()
    names = _header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and nothing in the header is a torch / C++ type
    hdr = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "vqpc.h")).read(), flags=re.S)
    assert "torch" not in hdr and "std::" not in hdr and "at::" not in hdr


def test_no_cpu_fallback_without_device():
    """Without a B200 the compute entry points fail loudly (no-device)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    b = klbasis.build_kl_basis_1d(64, 1.0, 0.2, 8)
    cb = dict(m=2, P=2, map="scale", method="kmeans", lambdas=b["eigenvalues"][:2],
              centroids=np.array([[0.1, 0.0], [-0.1, 0.0]]))
    with pytest.raises(lib.VqpcError, match="no-device"):
        lib.Context(1, 64, b, cb)
    with pytest.raises(lib.VqpcError, match="no-device"):
        lib.kmeans(np.zeros((10, 2)), np.ones(2), 2)


def test_host_sampler_matches_oracle():
    a = lib.draw_standard_normal(500, 7, 3, index0=11, threads=3)
    b = oracle.draw_standard_normal(500, 7, 3, index0=11)
    assert np.array_equal(a, b)
    assert lib.counter_hash(0, 0, 0) == 0x2B64F8B9232EFE85


def test_configs_describe_baseline():
    C1, C2, C5 = campaign.CONFIGS["C1"], campaign.CONFIGS["C2"], campaign.CONFIGS["C5"]
    assert campaign.unknowns(C1) == 1023 and campaign.unknowns(C2) == 4095 and campaign.unknowns(C5) == 8191
    assert campaign.unknowns(campaign.CONFIGS["C4"]) == 65025
    assert C2["n_realizations"] == 1 << 17 and C2["quantizer"]["P"] == 64 and C2["m"] == 8
    assert campaign.CONFIGS["C3"]["quantizer"]["method"] == "sign_grid"
