"""Pin the CPU oracle against the reference's own code: golden fixtures made by
tests/golden/make_golden.py from oracle/_ref (the reference's fem/quantizer/
rng/artifacts TUs compiled unchanged), plus live cross-checks when _ref is
built in this container."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_2403_07824_b200 import artifacts as art

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def test_counter_rng_goldens():
    d = np.load(os.path.join(G, "rng.npz"))
    for (s, i, k), h, u in zip(d["grid"], d["hash"], d["uniform"]):
        assert oracle.counter_hash(int(s), int(i), int(k)) == int(h)
        assert oracle.uniform_open01(int(s), int(i), int(k)) == u
    # SURVEY §8c known answers
    assert oracle.counter_hash(0, 0, 0) == 0x2B64F8B9232EFE85
    assert oracle.uniform_open01(0, 0, 0) == 0.16950945396382261
    assert oracle.uniform_open01(1, 5, 2) == 0.34279012049220753


def test_normal_quantile_accuracy():
    """Boost is absent, so xi bits are 'parity unpinned'; the replacement must
    still be a correct inverse CDF to a few ulps."""
    scipy_special = pytest.importorskip("scipy.special")
    u = np.array([oracle.uniform_open01(3, i, 0) for i in range(20000)] + [2.0 ** -54, 1e-300, 0.25, 1 - 2.0 ** -53])
    q = np.array([oracle.normal_quantile(x) for x in u])
    ref = scipy_special.ndtri(u)
    rel = np.abs(q - ref) / np.maximum(np.abs(ref), 1e-300)
    assert rel.max() < 5e-15
    assert np.isnan(oracle.normal_quantile(0.0)) and np.isnan(oracle.normal_quantile(1.0))


@pytest.mark.parametrize("r", [2, 4, 8])
@pytest.mark.parametrize("tag", ["one", "rough"])
def test_assemble_2d_matches_reference(r, tag):
    d = np.load(os.path.join(G, "assemble2d.npz"))
    k = f"r{r}_{tag}"
    rp, col, val, b = oracle.assemble(2, r, d[k + "_kappa"])
    assert np.array_equal(rp, d[k + "_rp"]) and np.array_equal(col, d[k + "_col"])
    assert np.array_equal(b, d[k + "_b"])
    # duplicates summed in the reference SparseBuilder's std::sort order: bit-identical
    assert np.array_equal(val, d[k + "_val"])


def test_lumped_mass_2d_matches_reference():
    from paper_2403_07824_b200 import klbasis
    d = np.load(os.path.join(G, "assemble2d.npz"))
    for r in (2, 4, 8):
        assert np.array_equal(klbasis.lumped_mass_2d(r), d[f"r{r}_mass"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_kmeans_and_assign_bit_identical_to_reference(tag):
    d = np.load(os.path.join(G, "quantizer.npz"))
    P, seed = int(d[f"{tag}_P"][0]), int(d[f"{tag}_seed"][0])
    cen, hist = oracle.kmeans(d[f"{tag}_samples"], d[f"{tag}_lam"], P, init_seed=seed)
    assert np.array_equal(cen, d[f"{tag}_centroids"])
    assert np.array_equal(hist, d[f"{tag}_history"])
    cb = oracle.Codebook("kmeans", "scale", d[f"{tag}_lam"], cen)
    assert np.array_equal(oracle.assign(cb, d[f"{tag}_xi"]), d[f"{tag}_labels"])


def test_assign_ties_and_spec_example():
    d = np.load(os.path.join(G, "quantizer.npz"))
    cb = oracle.Codebook("kmeans", "scale", d["tie_lam"], d["tie_centroids"])
    assert np.array_equal(oracle.assign(cb, d["tie_xi"]), d["tie_labels"])
    assert list(d["tie_labels"][:2]) == [0, 0]  # equidistant -> smallest index
    cen, _ = oracle.kmeans(d["spec_pts"], np.ones(1), 2)
    assert np.array_equal(np.sort(cen.ravel()), [1.0, 10.0])
    assert np.array_equal(cen, d["spec_centroids"])


def test_grid_sites_match_reference():
    d = np.load(os.path.join(G, "quantizer.npz"))
    assert np.array_equal(oracle.grid_sites(3, 0.8614), d["grid3_sites"])
    assert np.array_equal(art.grid_latent_sites(3, 0.8614), d["grid3_sites"])


def test_artifact_formats_byte_exact():
    """Our .qnt/.klb writer reproduces the reference writer's bytes and reads them back."""
    cb = art.load_codebook(os.path.join(G, "ref_codebook.qnt"))
    assert cb["P"] == 4 and cb["m"] == 3 and cb["seed"] == 42
    assert np.array_equal(cb["centroids"], np.arange(12, dtype=np.float64).reshape(4, 3) / 7.0)
    import tempfile
    with tempfile.TemporaryDirectory() as t:
        pth = os.path.join(t, "c.qnt")
        art.save_codebook(pth, cb)
        assert open(pth, "rb").read() == open(os.path.join(G, "ref_codebook.qnt"), "rb").read()
        b = art.load_kl_basis(os.path.join(G, "ref_basis.klb"))
        assert b["mesh_hash"] == 0xABCDEF and b["eigenvectors"].shape == (2, 5)
        pth = os.path.join(t, "b.klb")
        art.save_kl_basis(pth, b)
        assert open(pth, "rb").read() == open(os.path.join(G, "ref_basis.klb"), "rb").read()


@needs_ref
def test_live_reference_assign_kmeans_random():
    R = oracle.ref()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rs = np.random.default_rng(5)
    for m, P in [(4, 16), (8, 64), (10, 33)]:
        samples = oracle.draw_standard_normal(3000, m, 77 + m)
        lam = np.sort(rs.uniform(1e-3, 0.2, m))[::-1].copy()
        cen = np.empty((P, m))
        hist = np.empty(200)
        nh = C.c_int()
        oracle._ref_check(R.vqpref_kmeans(p(samples), 3000, m, p(lam), 0, P, 3, 200, 1e-6, p(cen), p(hist),
                                          C.byref(nh)))
        mine, h2 = oracle.kmeans(samples, lam, P, init_seed=3)
        assert np.array_equal(mine, cen) and np.array_equal(h2, hist[: nh.value])
        xi = rs.standard_normal((2000, m))
        lab = np.empty(2000, np.int32)
        oracle._ref_check(R.vqpref_assign(0, 0, P, m, p(lam), p(cen), p(xi), 2000, m, p(lab)))
        assert np.array_equal(oracle.assign(oracle.Codebook("kmeans", "scale", lam, cen), xi), lab)


@needs_ref
def test_live_reference_centroid_coefficient():
    R = oracle.ref()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rs = np.random.default_rng(8)
    K, nn, m, P = 6, 50, 4, 5
    ev = np.sort(rs.uniform(0.01, 0.3, K))[::-1].copy()
    vec = rs.standard_normal((K, nn))
    lam = ev[:m].copy()
    cen = rs.standard_normal((P, m)) * np.sqrt(lam)
    mine = oracle.centroid_coefficients(oracle.Codebook("kmeans", "scale", lam, cen), ev, vec)
    for q in range(P):
        out = np.empty(nn)
        oracle._ref_check(R.vqpref_centroid_coefficient(0, 0, P, m, p(lam), p(cen), q, p(ev), p(vec), K, nn, p(out)))
        assert np.array_equal(out, mine[q])


@needs_ref
@pytest.mark.parametrize("r", [17, 100, 256])
def test_live_reference_assemble_2d_rough(r):
    """The oracle's 2-D assembly against the reference's own fem.cpp (compiled
    here) on rough coefficients and meshes whose h = 1/r is inexact: CSR and b
    bit-identical — duplicates summed in SparseBuilder's std::sort order."""
    R = oracle.ref()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    kappa = np.exp(np.random.default_rng(r).standard_normal((r + 1) ** 2))
    n, nnz = C.c_int(), C.c_int()
    oracle._ref_check(R.vqpref_assemble_2d(r, p(kappa), C.byref(n), C.byref(nnz), None, None, None, None))
    rp = np.empty(n.value + 1, np.int32)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value)
    b = np.empty(n.value)
    oracle._ref_check(R.vqpref_assemble_2d(r, p(kappa), C.byref(n), C.byref(nnz), p(rp), p(col), p(val), p(b)))
    mrp, mcol, mval, mb = oracle.assemble(2, r, kappa)
    assert np.array_equal(mrp, rp) and np.array_equal(mcol, col)
    assert np.array_equal(mval, val) and np.array_equal(mb, b)
