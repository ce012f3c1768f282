"""Artifact files shared by the GPU path and the CPU oracle.

Formats follow /root/reference/proj/src/artifacts.cpp: one line of JSON
metadata, then little-endian float64 blocks; every float in the header is
printed with ``%.17g`` (artifacts.cpp:18-22).

* ``.klb`` (artifacts.cpp:50-86): header {format, version, n_nodes, n_kl,
  total_variance, sigma2, ell, mesh_resolution, mesh_hash}, then eigenvalues,
  eigenvectors (mode-major), lumped mass.
* ``.qnt`` (artifacts.cpp:88-127): header {format, version, m, P, map, method,
  seed, lambdas[, s]}, then the P x m centroid block. Grid codebooks rebuild
  their latent sites from ``s``. The sign grid (new) uses
  method "sign_grid" and rebuilds its sites from m.
* ``.xis`` (new): header {format, version, n, m, seed, index0}, then
  the n x m row-major xi block — the seeded inputs both sides consume.

Only the ``.klb``/``.qnt`` kinds the reference knows are readable by the
reference's own loader (checked against oracle/_ref in tests).
"""
from __future__ import annotations

import json
import math

import numpy as np


def fmt(v: float) -> str:
    """printf("%.17g") (artifacts.cpp:18-22)."""
    return "%.17g" % v


def _write(path, header: str, blocks):
    with open(path, "wb") as f:
        f.write(header.encode() + b"\n")
        for b in blocks:
            f.write(np.ascontiguousarray(b, dtype="<f8").tobytes())


def _read(path, fmt_name):
    with open(path, "rb") as f:
        line = f.readline()
        try:
            hdr = json.loads(line)
        except json.JSONDecodeError as e:
            raise RuntimeError("artifact-corrupt") from e
        if hdr.get("format") != fmt_name:
            raise RuntimeError("artifact-corrupt")
        return hdr, f.read()


def _block(raw, off, count):
    need = 8 * count
    if off + need > len(raw):
        raise RuntimeError("artifact-corrupt")
    return np.frombuffer(raw, dtype="<f8", count=count, offset=off).copy(), off + need


def save_kl_basis(path, basis: dict):
    lam = np.asarray(basis["eigenvalues"], np.float64)
    phi = np.asarray(basis["eigenvectors"], np.float64)
    mass = np.asarray(basis["mass"], np.float64)
    hdr = ('{"format":"klb","version":1,"n_nodes":%d,"n_kl":%d,"total_variance":%s,"sigma2":%s,'
           '"ell":%s,"mesh_resolution":%d,"mesh_hash":"%016x"}') % (
        mass.size, lam.size, fmt(basis["total_variance"]), fmt(basis["sigma2"]), fmt(basis["ell"]),
        int(basis["mesh_resolution"]), int(basis.get("mesh_hash", 0)))
    _write(path, hdr, [lam, phi.reshape(-1), mass])


def load_kl_basis(path) -> dict:
    hdr, raw = _read(path, "klb")
    nn, K = int(hdr["n_nodes"]), int(hdr["n_kl"])
    lam, off = _block(raw, 0, K)
    phi, off = _block(raw, off, K * nn)
    mass, off = _block(raw, off, nn)
    return dict(eigenvalues=lam, eigenvectors=phi.reshape(K, nn), mass=mass,
                total_variance=float(hdr["total_variance"]), sigma2=float(hdr["sigma2"]),
                ell=float(hdr["ell"]), mesh_resolution=int(hdr["mesh_resolution"]),
                mesh_hash=int(hdr["mesh_hash"], 16))


def sign_grid_sites(m: int) -> np.ndarray:
    """Sign-grid latent sites: component k of site p is
    +sqrt(2/pi) if bit k of p is set, else -sqrt(2/pi)."""
    s = math.sqrt(2.0 / math.pi)
    p = np.arange(1 << m)[:, None]
    k = np.arange(m)[None, :]
    return np.where((p >> k) & 1, s, -s).astype(np.float64)


def grid_latent_sites(m: int, s: float) -> np.ndarray:
    """Reference grid sites (quantizer.cpp:427-440): origin, then vertex v maps
    component k to +-s from bit k of (v - 1)."""
    if m == 0:
        return np.zeros((1, 0))
    P = 1 + (1 << m)
    out = np.zeros((P, m))
    bits = np.arange(P - 1)[:, None]
    out[1:] = np.where((bits >> np.arange(m)[None, :]) & 1, s, -s)
    return out


def save_codebook(path, cb: dict):
    lam = np.asarray(cb["lambdas"], np.float64)
    cen = np.asarray(cb["centroids"], np.float64)
    hdr = '{"format":"qnt","version":1,"m":%d,"P":%d,"map":"%s","method":"%s","seed":%d,"lambdas":[%s]' % (
        cb["m"], cb["P"], cb["map"], cb["method"], int(cb.get("seed", 0)), ",".join(fmt(v) for v in lam))
    if cb["method"] == "grid":
        hdr += ',"s":%s' % fmt(cb["s"])
    hdr += "}"
    _write(path, hdr, [cen.reshape(-1)])


def load_codebook(path) -> dict:
    hdr, raw = _read(path, "qnt")
    m, P = int(hdr["m"]), int(hdr["P"])
    cen, _ = _block(raw, 0, P * m)
    cb = dict(m=m, P=P, map=hdr["map"], method=hdr["method"], seed=int(hdr.get("seed", 0)),
              lambdas=np.asarray(hdr["lambdas"], np.float64), centroids=cen.reshape(P, m), latent=None)
    if cb["method"] == "grid":
        cb["s"] = float(hdr["s"])
        cb["latent"] = grid_latent_sites(m, cb["s"])
    elif cb["method"] == "sign_grid":
        cb["latent"] = sign_grid_sites(m)
    return cb


def save_xis(path, xi: np.ndarray, seed: int, index0: int = 0):
    xi = np.ascontiguousarray(xi, np.float64)
    hdr = '{"format":"xis","version":1,"n":%d,"m":%d,"seed":%d,"index0":%d}' % (xi.shape[0], xi.shape[1], seed, index0)
    _write(path, hdr, [xi.reshape(-1)])


def load_xis(path) -> np.ndarray:
    hdr, raw = _read(path, "xis")
    n, m = int(hdr["n"]), int(hdr["m"])
    xi, _ = _block(raw, 0, n * m)
    return xi.reshape(n, m)
