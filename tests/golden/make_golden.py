"""Generate tests/golden/*.npz from the REFERENCE'S OWN code (oracle/_ref: the
reference's fem.cpp / quantizer.cpp / rng.cpp / artifacts.cpp compiled
unchanged). Run in the container that mounts /root/reference:

    python -m tests.golden.make_golden

The fixtures pin the CPU oracle (tests/test_oracle_golden.py) on machines
where the reference is not available."""
import ctypes as C
import os

import numpy as np

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
p = lambda a: a.ctypes.data_as(C.c_void_p)


def rng():
    R = oracle.ref()
    seeds = [0, 1, 7, 12345, 2**63 + 11]
    idx = [0, 1, 5, 1000, 2**40 + 3]
    comp = [0, 1, 2, 63, 255]
    grid = np.array([(s, i, k) for s in seeds for i in idx for k in comp], dtype=np.uint64)
    h = np.array([R.vqpref_counter_hash(int(s), int(i), int(k)) for s, i, k in grid], dtype=np.uint64)
    u = np.array([R.vqpref_uniform_open01(int(s), int(i), int(k)) for s, i, k in grid])
    np.savez_compressed(os.path.join(HERE, "rng.npz"), grid=grid, hash=h, uniform=u)


def assemble2d():
    R = oracle.ref()
    out = {}
    rs = np.random.default_rng(3)
    for r in (2, 4, 8):
        nn = (r + 1) ** 2
        for tag, kappa in (("one", np.ones(nn)), ("rough", np.exp(rs.uniform(-1.5, 1.5, nn)))):
            n, nnz = C.c_int(), C.c_int()
            oracle._ref_check(R.vqpref_assemble_2d(r, p(kappa), C.byref(n), C.byref(nnz), None, None, None, None))
            rp = np.empty(n.value + 1, np.int32)
            col = np.empty(nnz.value, np.int32)
            val = np.empty(nnz.value)
            b = np.empty(n.value)
            oracle._ref_check(R.vqpref_assemble_2d(r, p(kappa), C.byref(n), C.byref(nnz), p(rp), p(col), p(val), p(b)))
            k = f"r{r}_{tag}"
            out.update({k + "_kappa": kappa, k + "_rp": rp, k + "_col": col, k + "_val": val, k + "_b": b})
        mass = np.empty(nn)
        oracle._ref_check(R.vqpref_lumped_mass(r, p(mass)))
        out[f"r{r}_mass"] = mass
        out[f"r{r}_hash"] = np.array([R.vqpref_mesh_fingerprint(r)], np.uint64)
    np.savez_compressed(os.path.join(HERE, "assemble2d.npz"), **out)


def quantizer():
    R = oracle.ref()
    rs = np.random.default_rng(11)
    out = {}
    # kmeans codebooks (Scale map) + assignments of fresh draws, reference code
    for tag, (n, m, P, seed) in {"a": (2000, 3, 7, 1), "b": (3000, 5, 16, 4), "c": (2000, 8, 12, 9)}.items():
        samples = oracle.draw_standard_normal(n, m, seed)
        lam = np.sort(rs.uniform(0.01, 1.0, m))[::-1].copy()
        cen = np.empty((P, m))
        hist = np.empty(200)
        nh = C.c_int()
        oracle._ref_check(R.vqpref_kmeans(p(samples), n, m, p(lam), 0, P, C.c_uint64(seed), 200, C.c_double(1e-6),
                                          p(cen), p(hist), C.byref(nh)))
        xi = oracle.draw_standard_normal(1000, m + 3, seed + 100)  # stride ld = m + 3
        lab = np.empty(len(xi), np.int32)
        oracle._ref_check(R.vqpref_assign(0, 0, P, m, p(lam), p(cen), p(xi), len(xi), m + 3, p(lab)))
        out.update({f"{tag}_samples": samples, f"{tag}_lam": lam, f"{tag}_P": np.array([P]),
                    f"{tag}_seed": np.array([seed]), f"{tag}_centroids": cen, f"{tag}_history": hist[:nh.value],
                    f"{tag}_xi": xi, f"{tag}_labels": lab})
    # ties: points exactly equidistant between centroids -> smallest index
    cen = np.array([[0.0, 0.0], [2.0, 0.0], [1.0, 1.0], [1.0, -1.0]])
    lam = np.array([1.0, 1.0])
    xi = np.array([[1.0, 0.0], [0.5, 0.5], [1.0, 0.25], [-3.0, 0.0], [1.5, 0.5]])
    lab = np.empty(len(xi), np.int32)
    oracle._ref_check(R.vqpref_assign(0, 0, 4, 2, p(lam), p(cen), p(xi), len(xi), 2, p(lab)))
    out.update(tie_centroids=cen, tie_lam=lam, tie_xi=xi, tie_labels=lab)
    # {0,1,2,9,10,11}, P = 2 -> {1, 10}
    pts = np.array([[0.0], [1.0], [2.0], [9.0], [10.0], [11.0]])
    cen = np.empty((2, 1))
    hist = np.empty(200)
    nh = C.c_int()
    oracle._ref_check(R.vqpref_kmeans(p(pts), 6, 1, p(np.ones(1)), 0, 2, C.c_uint64(1), 200, C.c_double(1e-6),
                                      p(cen), p(hist), C.byref(nh)))
    out.update(spec_pts=pts, spec_centroids=cen)
    # reference grid sites (quantizer.cpp:427-440)
    sites = np.empty((9, 3))
    oracle._ref_check(R.vqpref_grid_latent_sites(3, C.c_double(0.8614), p(sites)))
    out.update(grid3_sites=sites)
    np.savez_compressed(os.path.join(HERE, "quantizer.npz"), **out)


def artifacts_bytes():
    """Reference-written .qnt / .klb files (byte-exact format pins)."""
    R = oracle.ref()
    lam = np.array([0.5, 0.25, 0.125])
    cen = np.arange(12, dtype=np.float64).reshape(4, 3) / 7.0
    path_q = os.path.join(HERE, "ref_codebook.qnt")
    oracle._ref_check(R.vqpref_save_codebook(path_q.encode(), 0, 0, 4, 3, p(lam), p(cen), C.c_uint64(42)))
    ev = np.array([0.3, 0.2])
    vec = np.arange(10, dtype=np.float64).reshape(2, 5) / 3.0
    mass = np.full(5, 0.2)
    path_k = os.path.join(HERE, "ref_basis.klb")
    oracle._ref_check(R.vqpref_save_kl_basis(path_k.encode(), 2, 5, p(ev), p(vec), p(mass), C.c_double(1.0),
                                             C.c_double(1.0), C.c_double(0.1), 5, C.c_uint64(0xabcdef)))


if __name__ == "__main__":
    oracle.build()
    rng()
    assemble2d()
    quantizer()
    artifacts_bytes()
    print("golden fixtures written to", HERE)
