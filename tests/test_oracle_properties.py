"""The reference's own unit tests (proj/tests/test_fem.cpp) and SPEC.md
acceptance properties, restated against the CPU oracle."""
import numpy as np
import pytest

import oracle


def dense(rp, col, val):
    n = len(rp) - 1
    A = np.zeros((n, n))
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            A[i, col[k]] += val[k]
    return A


def test_hand_assembled_r2():  # test_fem.cpp:38-48
    rp, col, val, b = oracle.assemble(2, 2, np.ones(9))
    assert list(val) == [4.0] and list(b) == [0.25]
    ps = oracle.PreconditionerSet.from_coefficients(2, 2, "identity", np.ones(9))
    out = ps.pcg(0, np.ones(9), 1e-12)
    assert out["status"] == 0 and abs(out["x"][0] - 0.0625) <= 1e-12 * 0.0625


def test_unit_coefficient_five_point_stencil():  # test_fem.cpp:50-62
    rp, col, val, b = oracle.assemble(2, 4, np.ones(25))
    A = dense(rp, col, val)
    assert np.all(np.diag(A) == 4.0)
    assert A[4, 1] == A[4, 3] == A[4, 5] == A[4, 7] == -1.0
    assert A[4, 0] == 0.0
    # the diagonal neighbour is a stored (zero) entry of the 7-point pattern
    assert 0 in col[rp[4]:rp[5]]


def test_linear_scaling_and_cholesky_solution():  # test_fem.cpp:64-79
    r = 6
    nn = (r + 1) ** 2
    _, _, v1, b1 = oracle.assemble(2, r, np.ones(nn))
    _, _, v2, b2 = oracle.assemble(2, r, 2 * np.ones(nn))
    assert np.array_equal(v2, 2 * v1) and np.array_equal(b1, b2)
    p1 = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", np.ones(nn))
    p2 = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", 2 * np.ones(nn))
    u1 = p1.pcg(0, np.ones(nn), 1e-13)["x"]
    u2 = p2.pcg(0, 2 * np.ones(nn), 1e-13)["x"]
    assert np.allclose(u2, 0.5 * u1, rtol=1e-10, atol=0)


def test_interior_row_sums_vanish():  # test_fem.cpp:81-112
    r = 32
    rp, col, val, _ = oracle.assemble(2, r, np.ones((r + 1) ** 2))
    m = r - 1
    for i in range((r - 1) ** 2):
        ix, iy = i % m, i // m
        if 1 <= ix <= m - 2 and 1 <= iy <= m - 2:
            assert abs(val[rp[i]:rp[i + 1]].sum()) < 1e-12


def test_symmetry_spd_and_positive_load():  # test_fem.cpp:114-129
    r = 12
    nn = (r + 1) ** 2
    kappa = np.exp(2.0 * (np.array([oracle.uniform_open01(7, i, 0) for i in range(nn)]) - 0.5))
    rp, col, val, b = oracle.assemble(2, r, kappa)
    A = dense(rp, col, val)
    assert np.abs(A - A.T).max() < 1e-12
    oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", kappa)  # no not-spd
    assert np.all(b > 0)
    oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", np.maximum(kappa, 0.8))


def _sine_series(x, y, terms=100):  # proj/tests/oracles.hpp:28-41
    u = 0.0
    for a in range(terms):
        j = 2 * a + 1
        sx = np.sin(j * np.pi * x)
        for bb in range(terms):
            k = 2 * bb + 1
            u += 16.0 / (np.pi ** 4 * j * k * (j * j + k * k)) * sx * np.sin(k * np.pi * y)
    return u


def test_sine_series_oracle_r32():  # test_fem.cpp:131-145
    r = 32
    nn = (r + 1) ** 2
    ps = oracle.PreconditionerSet.from_coefficients(2, r, "cholesky", np.ones(nn))
    out = ps.pcg(0, np.ones(nn), 1e-12)
    assert out["status"] == 0
    m = r - 1
    h = 1.0 / r
    worst = 0.0
    for i in range(m * m):
        x, y = (i % m + 1) * h, (i // m + 1) * h
        worst = max(worst, abs(out["x"][i] - _sine_series(x, y, 40)))
    assert worst < 5e-3


def test_invalid_coefficient():  # test_fem.cpp:147-154
    kappa = np.ones(16)
    for bad in (0.0, -2.0, np.inf, np.nan):
        kappa[5] = bad
        with pytest.raises(oracle.OracleError, match="invalid-coefficient"):
            oracle.assemble(2, 3, kappa)
    with pytest.raises(oracle.OracleError, match="invalid-coefficient"):
        oracle.assemble(1, 8, np.array([1, 1, 1, 0.0, 1, 1, 1, 1]))


@pytest.mark.parametrize("dim,size", [(2, 32), (1, 1024)])
def test_exact_factor_gives_one_iteration(dim, size):  # SPEC.md:460 (acceptance 1)
    nn = size if dim == 1 else (size + 1) ** 2
    rs = np.random.default_rng(1)
    for _ in range(5):
        kappa = np.exp(rs.normal(0, 0.7, nn))
        ps = oracle.PreconditionerSet.from_coefficients(dim, size, "cholesky", kappa)
        out = ps.pcg(0, kappa, 1e-8)
        assert out["iterations"] == 1 and out["status"] == 0


def test_one_d_model_structure():
    N = 16
    kappa = np.linspace(0.5, 2.0, N)
    rp, col, val, b = oracle.assemble(1, N, kappa)
    n = N - 1
    assert len(val) == 3 * n - 2 and np.all(b == 1.0 / N)
    A = dense(rp, col, val)
    for j in range(n):
        assert A[j, j] == kappa[j] * N + kappa[j + 1] * N
        if j + 1 < n:
            assert A[j, j + 1] == -kappa[j + 1] * N == A[j + 1, j]
    assert np.all(np.linalg.eigvalsh(A) > 0)


def test_rcm_on_path_graph_is_reversal():  # solver.cpp:32-70 on the 1-D pattern
    rp, col, _, _ = oracle.assemble(1, 64, np.ones(64))
    assert np.array_equal(oracle.rcm_permutation(rp, col), np.arange(62, -1, -1))


def test_cholesky_apply_solves_centroid_matrix():
    rs = np.random.default_rng(2)
    for dim, size in [(1, 300), (2, 10)]:
        nn = size if dim == 1 else (size + 1) ** 2
        kappa = np.exp(rs.normal(0, 1, nn))
        rp, col, val, _ = oracle.assemble(dim, size, kappa)
        A = dense(rp, col, val)
        ps = oracle.PreconditionerSet.from_coefficients(dim, size, "cholesky", kappa)
        r = rs.standard_normal(A.shape[0])
        z = ps.apply(0, r)
        assert np.linalg.norm(A @ z - r) / np.linalg.norm(r) < 1e-10


def test_ic0_is_the_no_fill_factor():
    """IC(0) of the 5-point pattern: M = (D + L) D^-1 (D + L^T) reproduces A on
    the pattern, and its apply is that operator's inverse."""
    r = 9
    nn = (r + 1) ** 2
    kappa = np.exp(np.random.default_rng(4).normal(0, 1, nn))
    rp, col, val, _ = oracle.assemble(2, r, kappa)
    A = dense(rp, col, val)
    n = A.shape[0]
    ps = oracle.PreconditionerSet.from_coefficients(2, r, "ic0", kappa)
    M = np.column_stack([np.linalg.solve(np.eye(n), ps.apply(0, e)) for e in np.eye(n)])
    Minv = M
    Mfull = np.linalg.inv(Minv)
    m = r - 1
    for i in range(n):
        for j in (i, i - 1, i + 1, i - m, i + m):
            if 0 <= j < n and (j == i or abs(A[i, j]) > 0):
                assert abs(Mfull[i, j] - A[i, j]) < 1e-9 * abs(A[i, i])
    assert np.allclose(Mfull, Mfull.T, atol=1e-9 * np.abs(Mfull).max())


def test_pcg_status_semantics():
    kappa = np.exp(np.random.default_rng(3).normal(0, 1, 256))
    ps = oracle.PreconditionerSet.from_coefficients(1, 256, "identity", kappa)
    out = ps.pcg(0, kappa, 1e-8, max_iter=3)
    assert out["status"] == 1 and out["iterations"] == 3  # max_iter -> not converged
    with pytest.raises(oracle.OracleError, match="invalid-tolerance"):
        ps.pcg(0, kappa, 1.0)


def test_assign_brute_force_and_scale_invariance():  # oracles.hpp:44-60; SPEC invariants
    rs = np.random.default_rng(9)
    m, P = 6, 40
    lam = np.sort(rs.uniform(0.1, 1.0, m))[::-1].copy()
    cen = rs.standard_normal((P, m))
    xi = rs.standard_normal((500, m))
    cb = oracle.Codebook("kmeans", "scale", lam, cen)
    lab = oracle.assign(cb, xi)
    eta = xi * np.sqrt(lam)
    d = ((eta[:, None, :] - cen[None]) ** 2).sum(-1)
    assert np.array_equal(lab, d.argmin(1))
    # multiplying all lambdas (and centroids' eta accordingly) by 4 keeps the argmin
    cb4 = oracle.Codebook("kmeans", "scale", 4 * lam, 2 * cen)
    assert np.array_equal(oracle.assign(cb4, xi), lab)
    with pytest.raises(oracle.OracleError, match="invalid-latent"):
        oracle.assign(cb, np.array([[np.nan] * m]))


def test_lloyd_monotone_and_fixed_point():  # SPEC acceptance 3
    x = oracle.draw_standard_normal(3000, 3, 5)
    lam = np.array([1.0, 0.5, 0.25])
    cen, hist = oracle.kmeans(x, lam, 12)
    assert np.all(np.diff(hist) <= 1e-12 * hist[:-1])
    cb = oracle.Codebook("kmeans", "scale", lam, cen)
    lab = oracle.assign(cb, x)
    eta = x * np.sqrt(lam)
    for p in range(12):
        assert np.allclose(cen[p], eta[lab == p].mean(0), atol=1e-3 * np.abs(eta).max())


def test_sign_grid_cells_are_sign_patterns():
    m = 6
    sites = oracle.sign_grid_sites(m)
    xi = oracle.draw_standard_normal(2000, m, 3)
    cb = oracle.Codebook("sign_grid", "scale", np.ones(m), sites, sites)
    lab = oracle.assign(cb, xi)
    expect = ((xi > 0).astype(int) << np.arange(m)).sum(1)
    assert np.array_equal(lab, expect)
