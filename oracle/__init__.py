"""CPU oracle — TEST INFRASTRUCTURE ONLY.

ctypes front-end for ``oracle/liboracle.so`` (the C++ restatement of the
reference ``vqp`` hot path, ``oracle/src/vqp_oracle.cpp``) and for
``oracle/_ref/libvqpref.so`` (the reference's own fem/quantizer/rng/artifacts
translation units compiled unchanged, see ``oracle/ref/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
FMA_PATH = os.path.join(HERE, "liboracle_fma.so")
REF_PATH = os.path.join(HERE, "_ref", "libvqpref.so")

ERRORS = {
    0: "ok", 1: "invalid-latent", 2: "invalid-coefficient", 3: "coefficient-overflow",
    4: "not-spd", 5: "pcg-breakdown", 6: "invalid-tolerance", 7: "mode-count-out-of-range",
    8: "invalid-codebook", 9: "insufficient-samples", 10: "invalid-config", 11: "invalid-argument",
}
METHODS = {"kmeans": 0, "clvq": 1, "grid": 2, "sign_grid": 3}
MAPS = {"scale": 0, "cdf": 1}
PRECONDS = {"identity": 0, "cholesky": 1, "amg": 3, "ic0": 4}


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(ERRORS.get(code, f"error-{code}"))
        self.code = code


def build(force: bool = False) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    # make tracks the sources' timestamps (a stale build would check the GPU
    # against an outdated restatement)
    subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so", "liboracle_fma.so"] + (["-B"] if force else []))
    if os.path.isdir("/root/reference/proj") and (force or not os.path.exists(REF_PATH)):
        subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "ref")])


_lib = None
_ref = None
_use_fma = False


class fma_variant:
    """Context manager: route oracle calls to the FMA-contracted build (a
    rounding-level variant of the same restatement)."""

    def __enter__(self):
        global _use_fma
        self.prev = _use_fma
        _use_fma = True

    def __exit__(self, *a):
        global _use_fma
        _use_fma = self.prev

D = C.c_double
I = C.c_int
I64 = C.c_int64
U64 = C.c_uint64
VP = C.c_void_p
PD = C.POINTER(C.c_double)


def _p(a):
    return None if a is None else a.ctypes.data_as(VP)


_libs = {}


def lib():
    path = FMA_PATH if _use_fma else LIB_PATH
    if path not in _libs:
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.vqpo_counter_hash.restype = U64
        L.vqpo_counter_hash.argtypes = [U64, U64, U64]
        L.vqpo_uniform_open01.restype = D
        L.vqpo_uniform_open01.argtypes = [U64, U64, U64]
        L.vqpo_normal_quantile.restype = D
        L.vqpo_normal_quantile.argtypes = [D]
        L.vqpo_normal_cdf.restype = D
        L.vqpo_normal_cdf.argtypes = [D]
        L.vqpo_pset_destroy.restype = None
        L.vqpo_pset_destroy.argtypes = [VP]
        _libs[path] = L
    return _libs[path]


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The reference's own TUs (oracle/_ref). Raises if not built."""
    global _ref
    if _ref is None:
        R = C.CDLL(REF_PATH)
        R.vqpref_counter_hash.restype = U64
        R.vqpref_counter_hash.argtypes = [U64, U64, U64]
        R.vqpref_uniform_open01.restype = D
        R.vqpref_uniform_open01.argtypes = [U64, U64, U64]
        R.vqpref_mesh_fingerprint.restype = U64
        R.vqpref_mesh_fingerprint.argtypes = [I]
        R.vqpref_last_error.restype = C.c_char_p
        CP = C.c_char_p
        sigs = {
            "vqpref_assemble_2d": [I, VP, VP, VP, VP, VP, VP, VP],
            "vqpref_lumped_mass": [I, VP],
            "vqpref_assign": [I, I, I, I, VP, VP, VP, I64, I, VP],
            "vqpref_kmeans": [VP, I, I, VP, I, I, U64, I, D, VP, VP, VP],
            "vqpref_grid_latent_sites": [I, D, VP],
            "vqpref_centroid_coefficient": [I, I, I, I, VP, VP, I, VP, VP, I, I, VP],
            "vqpref_load_codebook": [CP, VP, VP, VP, VP, VP, VP],
            "vqpref_save_codebook": [CP, I, I, I, I, VP, VP, U64],
            "vqpref_load_kl_basis": [CP, VP, VP, VP, VP, VP, VP],
            "vqpref_save_kl_basis": [CP, I, I, VP, VP, VP, D, D, D, I, U64],
        }
        for name, args in sigs.items():
            getattr(R, name).restype = I
            getattr(R, name).argtypes = args
        _ref = R
    return _ref


def _check(code):
    if code != 0:
        raise OracleError(code)


def _ref_check(code):
    if code != 0:
        raise RuntimeError(ref().vqpref_last_error().decode())


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------------------------- rng
def counter_hash(seed, index, comp):
    return lib().vqpo_counter_hash(seed, index, comp)


def uniform_open01(seed, index, comp):
    return lib().vqpo_uniform_open01(seed, index, comp)


def normal_quantile(p):
    return lib().vqpo_normal_quantile(p)


def draw_standard_normal(n, m, seed, index0=0, threads=None):
    out = np.empty((n, m), dtype=np.float64)
    threads = threads or os.cpu_count() or 1
    _check(lib().vqpo_draw_standard_normal(I64(n), I(m), U64(seed), I64(index0), _p(out), I(threads)))
    return out


# ---------------------------------------------------------------------------- field
def realise(evals, evecs, xi, m=None, threads=None):
    """kappa = transport(lift(basis, xi_i)) for every row (field.cpp:113-145)."""
    evals, evecs, xi = f64(evals), f64(evecs), f64(np.atleast_2d(xi))
    n_kl, n_nodes = evecs.shape
    B, ld = xi.shape
    m = ld if m is None else m
    out = np.empty((B, n_nodes))
    st = np.empty(B, dtype=np.uint8)
    _check(lib().vqpo_realise(_p(evals), _p(evecs), I(n_kl), I(n_nodes), _p(xi), I64(B), I(ld), I(m),
                              _p(out), _p(st), I(threads or os.cpu_count() or 1)))
    return out, st


def assemble(dim, size, kappa):
    """CSR (row_ptr, col, val) and b of the model system (dim 1: N elements, dim 2: r x r)."""
    kappa = f64(kappa)
    n, nnz = C.c_int(), C.c_int()
    _check(lib().vqpo_assemble(I(dim), I(size), _p(kappa), C.byref(n), C.byref(nnz), None, None, None, None))
    rp = np.empty(n.value + 1, np.int32)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value)
    b = np.empty(n.value)
    _check(lib().vqpo_assemble(I(dim), I(size), _p(kappa), C.byref(n), C.byref(nnz), _p(rp), _p(col), _p(val), _p(b)))
    return rp, col, val, b


def rcm_permutation(row_ptr, col):
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    n = len(row_ptr) - 1
    out = np.empty(n, np.int32)
    _check(lib().vqpo_rcm_permutation(I(n), _p(row_ptr), _p(col), _p(out)))
    return out


# ------------------------------------------------------------------------ quantizer
class Codebook:
    """Flat codebook: method, map, lambdas (m), centroids (P x m, quantization
    space) and latent sites (grids). Mirrors quantizer.hpp:69-87."""

    def __init__(self, method, map, lambdas, centroids, latent=None):
        self.method = method
        self.map = map
        self.lambdas = f64(lambdas)
        self.centroids = f64(centroids)
        self.P, self.m = self.centroids.shape
        self.latent = None if latent is None else f64(latent)

    @property
    def args(self):
        return (I(METHODS[self.method]), I(MAPS[self.map]), I(self.P), I(self.m), _p(self.lambdas),
                _p(self.centroids), _p(self.latent))


def assign(cb: Codebook, xi, threads=1):
    """quantizer.cpp:134-145 per row. threads > 1 splits the rows over Python
    threads (ctypes releases the GIL; rows are independent, so the labels do not
    depend on the split)."""
    xi = f64(np.atleast_2d(xi))
    B, ld = xi.shape
    labels = np.empty(B, np.int32)
    if threads <= 1 or B < 2 * threads:
        _check(lib().vqpo_assign(*cb.args, _p(xi), I64(B), I(ld), _p(labels)))
        return labels
    from concurrent.futures import ThreadPoolExecutor
    bounds = np.linspace(0, B, threads + 1).astype(np.int64)

    def part(t):
        a, b = int(bounds[t]), int(bounds[t + 1])
        sub = xi[a:b]
        out = np.empty(b - a, np.int32)
        _check(lib().vqpo_assign(*cb.args, _p(sub), I64(b - a), I(ld), _p(out)))
        labels[a:b] = out

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(part, range(threads)))
    return labels


def to_quant(map, lambdas, chi):
    chi = f64(np.atleast_2d(chi))
    lambdas = f64(lambdas)
    out = np.empty_like(chi)
    _check(lib().vqpo_to_quant(I(MAPS[map]), I(chi.shape[1]), _p(lambdas), _p(chi), I64(chi.shape[0]), _p(out)))
    return out


def kmeans(samples, lambdas, P, map="scale", init_seed=1, max_iter=200, rel_tol=1e-6):
    samples, lambdas = f64(samples), f64(lambdas)
    n, m = samples.shape
    out = np.empty((P, m))
    hist = np.empty(max_iter)
    nh = C.c_int()
    _check(lib().vqpo_kmeans(_p(samples), I(n), I(m), _p(lambdas), I(MAPS[map]), I(P), U64(init_seed),
                             I(max_iter), D(rel_tol), _p(out), _p(hist), C.byref(nh)))
    return out, hist[: nh.value].copy()


def grid_sites(m, s):
    P = 1 if m == 0 else 1 + (1 << m)
    out = np.empty((P, m))
    _check(lib().vqpo_grid_sites(I(m), D(s), _p(out)))
    return out


def sign_grid_sites(m):
    out = np.empty((1 << m, m))
    _check(lib().vqpo_sign_grid_sites(I(m), _p(out)))
    return out


def centroid_coefficients(cb: Codebook, evals, evecs):
    evals, evecs = f64(evals), f64(evecs)
    n_kl, n_nodes = evecs.shape
    out = np.empty((cb.P, n_nodes))
    _check(lib().vqpo_centroid_coefficients(*cb.args, _p(evals), _p(evecs), I(n_kl), I(n_nodes), _p(out)))
    return out


# --------------------------------------------------------------------------- solver
class PreconditionerSet:
    """The P centroid preconditioners, built up front (driver.cpp:212-219)."""

    def __init__(self, handle, dim, size):
        self.lib = lib()
        self.h = handle
        self.dim, self.size = dim, size
        self.n = size - 1 if dim == 1 else (size - 1) ** 2

    @classmethod
    def build(cls, dim, size, kind, cb: Codebook, evals, evecs):
        evals, evecs = f64(evals), f64(evecs)
        h = VP()
        _check(lib().vqpo_pset_build(I(dim), I(size), I(PRECONDS[kind]), *cb.args, _p(evals), _p(evecs),
                                     I(evecs.shape[0]), I(evecs.shape[1]), C.byref(h)))
        return cls(h, dim, size)

    @classmethod
    def from_coefficients(cls, dim, size, kind, kappa):
        kappa = f64(np.atleast_2d(kappa))
        h = VP()
        _check(lib().vqpo_pset_from_coefficients(I(dim), I(size), I(PRECONDS[kind]), I(kappa.shape[0]), _p(kappa),
                                                 C.byref(h)))
        return cls(h, dim, size)

    def amg_levels(self, p):
        """SA-AMG hierarchy of centroid p: list of dicts (A CSR, inv_diag, P CSR) and
        the coarsest dense Cholesky factor (amg.cpp:132-197 restated)."""
        info = np.zeros(4 * 64, np.int64)
        nlev, dn = I(), I()
        _check(lib().vqpo_pset_amg_info(self.h, I(p), I(64), _p(info), C.byref(nlev), C.byref(dn)))
        out = []
        for l in range(nlev.value):
            n, nnz, pnnz, nc = (int(v) for v in info[4 * l:4 * l + 4])
            a_rp, a_col, a_val = np.empty(n + 1, np.int32), np.empty(nnz, np.int32), np.empty(nnz)
            inv = np.empty(n)
            p_rp = np.empty(n + 1, np.int32) if pnnz else np.empty(1, np.int32)
            p_col, p_val = np.empty(max(pnnz, 1), np.int32), np.empty(max(pnnz, 1))
            last = l + 1 == nlev.value
            L = np.empty(dn.value * dn.value) if last and dn.value else None
            _check(lib().vqpo_pset_amg_level(self.h, I(p), I(l), _p(a_rp), _p(a_col), _p(a_val), _p(inv), _p(p_rp),
                                             _p(p_col), _p(p_val), _p(L) if L is not None else None))
            lv = dict(n=n, A=(a_rp, a_col, a_val), inv_diag=inv, nc=nc)
            if pnnz:
                lv["P"] = (p_rp, p_col[:pnnz], p_val[:pnnz])
            if L is not None:
                lv["L"] = L.reshape(dn.value, dn.value)
            out.append(lv)
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.vqpo_pset_destroy(self.h)
            self.h = None

    def apply(self, p, r):
        r = f64(r)
        z = np.empty_like(r)
        _check(lib().vqpo_pset_apply(self.h, I(p), _p(r), _p(z)))
        return z

    def solve_batch(self, evals, evecs, xi, labels, eps, max_iter=-1, max_iter_arr=None, threads=None,
                    m_xi=None, want_x=False):
        evals, evecs, xi = f64(evals), f64(evecs), f64(np.atleast_2d(xi))
        B, ld = xi.shape
        labels = np.ascontiguousarray(labels, np.int32)
        it = np.empty(B, np.int32)
        rel = np.empty(B)
        st = np.empty(B, np.uint8)
        x = np.empty((B, self.n)) if want_x else None
        mia = None if max_iter_arr is None else np.ascontiguousarray(max_iter_arr, np.int32)
        _check(lib().vqpo_solve_batch(self.h, _p(evals), _p(evecs), I(evecs.shape[0]), I(evecs.shape[1]), _p(xi),
                                      I64(B), I(ld), I(ld if m_xi is None else m_xi), _p(labels), D(eps),
                                      I(max_iter), _p(mia), I(threads or os.cpu_count() or 1), _p(it), _p(rel),
                                      _p(st), _p(x)))
        return it, rel, st, x

    def pcg(self, p, kappa, eps, max_iter=-1, trace=False):
        kappa = f64(kappa)
        x = np.empty(self.n)
        it, rel, st, nt = C.c_int32(), C.c_double(), C.c_uint8(), C.c_int()
        cap = max_iter if max_iter > 0 else 10 * self.n
        tr = np.empty(cap) if trace else None
        _check(lib().vqpo_pcg_coefficient(self.h, I(p), _p(kappa), D(eps), I(max_iter), _p(x), C.byref(it),
                                          C.byref(rel), C.byref(st), _p(tr), C.byref(nt)))
        out = dict(x=x, iterations=it.value, rel=rel.value, status=st.value)
        if trace:
            out["trace"] = tr[: nt.value].copy()
        return out


def ideal_sweep(dim, size, kind, evals, evecs, xi, m_list, eps, max_iter=-1, threads=None):
    """driver.cpp:290-340 restated: per-(realisation, m) records (B x n_m arrays)."""
    evals, evecs, xi = f64(evals), f64(evecs), f64(np.atleast_2d(xi))
    B, ld = xi.shape
    ml = np.ascontiguousarray(m_list, dtype=np.int32)
    it = np.empty((B, ml.size), np.int32)
    rel = np.empty((B, ml.size))
    st = np.empty((B, ml.size), np.uint8)
    _check(lib().vqpo_ideal_sweep(I(dim), I(size), I(PRECONDS[kind]), _p(evals), _p(evecs), I(evecs.shape[0]),
                                  I(evecs.shape[1]), _p(xi), I64(B), I(ld), _p(ml), I(ml.size), D(eps), I(max_iter),
                                  I(threads or os.cpu_count() or 1), _p(it), _p(rel), _p(st)))
    return dict(iterations=it, rel=rel, status=st)


def run_campaign(dim, size, kind, cb: Codebook, evals, evecs, xi, eps, max_iter=-1, threads=None):
    """driver.cpp:193-281 restated: returns per-sample arrays, per-centroid stats
    and stage timings (seconds)."""
    evals, evecs, xi = f64(evals), f64(evecs), f64(xi)
    B, ld = xi.shape
    P = cb.P
    labels = np.empty(B, np.int32)
    it = np.empty(B, np.int32)
    rel = np.empty(B)
    st = np.empty(B, np.uint8)
    stats = np.empty(4 * P, np.int64)
    summary = np.empty(4, np.int64)
    timings = np.empty(4)
    _check(lib().vqpo_run_campaign(I(dim), I(size), I(PRECONDS[kind]), *cb.args, _p(evals), _p(evecs),
                                   I(evecs.shape[0]), I(evecs.shape[1]), _p(xi), I64(B), I(ld), D(eps), I(max_iter),
                                   I(threads or os.cpu_count() or 1), _p(labels), _p(it), _p(rel), _p(st),
                                   _p(stats), _p(summary), _p(timings)))
    return dict(labels=labels, iterations=it, rel=rel, status=st, n_p=stats[:P], sum_j=stats[P:2 * P],
                conv_count=stats[2 * P:3 * P], conv_sum=stats[3 * P:], total_iterations=int(summary[0]),
                unconverged=int(summary[1]), conv_total=int(summary[2]), conv_sum_total=int(summary[3]),
                timings=dict(assign=timings[0], build=timings[1], solve=timings[2], reduce=timings[3]))
