"""KL basis construction (one-time host setup; output is a ``.klb`` artifact).

Restates ``build_kl_basis`` (/root/reference/proj/src/field.cpp:22-82): the
lumped-mass Galerkin covariance operator W = M^{1/2} C M^{1/2} is
diagonalised, the ``n_kl`` dominant eigenpairs are kept subject to the
degeneracy cutoff lambda >= 1e-12 * lambda_1 (field.cpp:51-54), and each
eigenvector is mapped to Phi = M^{-1/2} v with the sign convention "first entry
of largest magnitude is positive" (field.cpp:72-79).

Two discretisations:

* 1-D: element midpoints x_e = (e + 1/2) h, weights w_e = h, so W = h C.
  Solved with LAPACK ``dsyevr`` on the top ``n_kl`` eigenvalues (scipy).
* 2-D: the reference's structured mesh nodes and lumped mass
  (fem.cpp:132-140). The dense W (66,049^2 for r = 256) is infeasible, so the
  same discrete eigenproblem is solved by Lanczos (ARPACK) with the Kronecker
  matvec C = C_y (x) C_x on the tensor node grid.

The eigensolver is a library call (the reference uses Eigen's
SelfAdjointEigenSolver); bits are not reproducible across eigensolvers, which is
why the basis is an artifact shared by the oracle and the GPU path.

``kl_cutoff=False`` keeps the top ``n_kl`` modes with lambda > 0 (SURVEY F5:
configuration C5 needs d = 64 modes while only ~39 survive the reference cutoff).
"""
from __future__ import annotations

import numpy as np


TIE_RTOL = 1e-9  # magnitudes within this relative distance of the maximum count as tied


def _sign_index(row):
    """First index of the largest magnitude (field.cpp:72-79), with entries within
    TIE_RTOL of the maximum treated as tied. On the symmetric domains here the
    odd modes have exact ties |v_i| = |v_j| in exact arithmetic, which rounding
    breaks differently on different hosts; the tolerance makes the first index
    win deterministically (the reference's rule whenever it is unambiguous)."""
    a = np.abs(row)
    return int(np.nonzero(a >= a.max() * (1.0 - TIE_RTOL))[0][0])


def _finish(evals_desc, vecs_desc, sqrt_mass, n_kl, cutoff):
    lead = evals_desc[0]
    if not lead > 0:
        raise RuntimeError("kl-eigensolve-failed")
    thr = 1e-12 * lead if cutoff else 0.0
    kept = 0
    while kept < min(n_kl, len(evals_desc)) and (evals_desc[kept] >= thr if cutoff else evals_desc[kept] > 0):
        kept += 1
    lam = np.ascontiguousarray(evals_desc[:kept])
    phi = np.ascontiguousarray((vecs_desc[:, :kept] / sqrt_mass[:, None]).T)  # mode-major
    for k in range(kept):
        imax = _sign_index(phi[k])  # first index of the largest magnitude (ties: see _sign_index)
        if phi[k, imax] < 0:
            phi[k] = -phi[k]
    return lam, phi


def build_kl_basis_1d(n_elements: int, sigma2: float, ell: float, n_kl: int, cutoff: bool = True):
    """Return dict(eigenvalues, eigenvectors (K x N), mass (N), total_variance)."""
    import scipy.linalg as sl

    if not (sigma2 > 0 and ell > 0):
        raise ValueError("invalid-kernel")
    N = int(n_elements)
    if n_kl < 1 or n_kl > N:
        raise ValueError("rank-exceeds-dofs")
    h = 1.0 / N
    x = (np.arange(N) + 0.5) * h
    mass = np.full(N, h)
    sm = np.sqrt(mass)
    d = x[:, None] - x[None, :]
    C = sigma2 * np.exp(-(d * d) / (ell * ell))
    W = sm[:, None] * C * sm[None, :]
    w, v = sl.eigh(W, subset_by_index=[N - n_kl, N - 1], driver="evr")
    lam, phi = _finish(w[::-1], v[:, ::-1], sm, n_kl, cutoff)
    return dict(eigenvalues=lam, eigenvectors=phi, mass=mass, total_variance=sigma2 * float(mass.sum()),
                sigma2=sigma2, ell=ell, mesh_resolution=N, dim=1)


def lumped_mass_2d(r: int):
    """Lumped P1 mass of the structured r x r mesh (fem.cpp:132-140): a third of
    the area of the triangles touching each node (corner masses h^2/3, h^2/6)."""
    side = r + 1
    h = 1.0 / r
    area = 0.5 * h * h
    acc = np.zeros((side, side))
    # cell (cx, cy): triangles {a,b,d} and {a,d,c}; a=(cx,cy) b=(cx+1,cy) c=(cx,cy+1) d=(cx+1,cy+1)
    acc[:-1, :-1] += 2 * area  # a in both   (index [iy, ix])
    acc[:-1, 1:] += area       # b
    acc[1:, 1:] += 2 * area    # d in both
    acc[1:, :-1] += area       # c
    return (acc / 3.0).reshape(-1)


def build_kl_basis_2d(r: int, sigma2: float, ell: float, n_kl: int, cutoff: bool = True, tol: float = 0.0,
                      v0_seed: int = 12345):
    """Lanczos with the Kronecker matvec on the (r+1)^2 node grid."""
    from scipy.sparse.linalg import LinearOperator, eigsh

    side = r + 1
    h = 1.0 / r
    t = np.arange(side) * h
    d = t[:, None] - t[None, :]
    C1 = np.exp(-(d * d) / (ell * ell))  # C = sigma2 * C1 (x) C1 (separable squared exponential)
    mass = lumped_mass_2d(r)
    sm = np.sqrt(mass)
    nn = side * side

    def mv(v):
        V = (sm * v.reshape(-1)).reshape(side, side)  # [iy, ix]
        Y = sigma2 * (C1 @ V @ C1.T)
        return sm * Y.reshape(-1)

    if n_kl >= nn - 1:
        # tiny meshes (n_kl modes are all of them): the dense W (Lanczos needs k < N)
        import scipy.linalg as sl
        W = (sm[:, None] * (sigma2 * np.kron(C1, C1))) * sm[None, :]
        k = min(n_kl, nn)
        w, v = sl.eigh(W, subset_by_index=[nn - k, nn - 1])
    else:
        op = LinearOperator((nn, nn), matvec=mv, dtype=np.float64)
        rng = np.random.default_rng(v0_seed)
        w, v = eigsh(op, k=n_kl, which="LA", tol=tol, v0=rng.standard_normal(nn),
                     ncv=min(nn, max(2 * n_kl + 1, n_kl + 64)))
    order = np.argsort(w)[::-1]
    lam, phi = _finish(w[order], v[:, order], sm, n_kl, cutoff)
    return dict(eigenvalues=lam, eigenvectors=phi, mass=mass, total_variance=sigma2 * float(mass.sum()),
                sigma2=sigma2, ell=ell, mesh_resolution=r, dim=2)
