"""ctypes binding of the C ABI (include/vqpc.h) — the drop-in boundary.

There is no CPU fallback: loading fails loudly when ``libvqpc.so`` is missing,
and every compute call fails with ``no-device`` on a machine without a B200.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VQPC_LIB", os.path.join(HERE, "libvqpc.so"))

METHODS = {"kmeans": 0, "clvq": 1, "grid": 2, "sign_grid": 3}
MAPS = {"scale": 0, "cdf": 1}
PRECONDS = {"identity": 0, "cholesky": 1, "amg": 3, "ic0": 4}
STATUS = {0: "converged", 1: "max_iter", 2: "breakdown", 3: "coefficient-overflow", 4: "invalid-latent",
          5: "invalid-coefficient", 6: "not-solved"}


class VqpcError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        self.code = code
        super().__init__(f"{error_string(code)}{': ' + msg if msg else ''}")


class _Problem(C.Structure):
    _fields_ = [("dim", C.c_int), ("size", C.c_int), ("n_kl", C.c_int), ("n_nodes", C.c_int),
                ("eigenvalues", C.c_void_p), ("eigenvectors", C.c_void_p), ("method", C.c_int), ("map", C.c_int),
                ("P", C.c_int), ("m", C.c_int), ("lambdas", C.c_void_p), ("centroids", C.c_void_p),
                ("latent", C.c_void_p), ("precond", C.c_int), ("device", C.c_int)]


_lib = None


def load():
    """Load libvqpc.so (built in-tree by paper_2403_07824_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2403_07824_b200.build.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        VP, I, I64, D, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64
        sig = {
            "vqpc_ctx_create": (I, [C.POINTER(_Problem), C.POINTER(VP)]),
            "vqpc_ctx_destroy": (None, [VP]),
            "vqpc_last_error": (C.c_char_p, [VP]),
            "vqpc_error_string": (C.c_char_p, [I]),
            "vqpc_set_stream": (I, [VP, VP]),
            "vqpc_synchronize": (I, [VP]),
            "vqpc_set_exact_reductions": (I, [VP, I]),
            "vqpc_unknowns": (I, [VP]),
            "vqpc_factor_entries": (C.c_int64, [VP]),
            "vqpc_launch_count": (I64, [VP]),
            "vqpc_factor_centroids": (I, [VP]),
            "vqpc_centroid_coefficients": (I, [VP, VP]),
            "vqpc_precond_apply": (I, [VP, I, VP, VP]),
            "vqpc_assign": (I, [VP, VP, I64, I, VP]),
            "vqpc_assign_d": (I, [VP, VP, I64, I, VP]),
            "vqpc_bucket_d": (I, [VP, VP, I64, VP, VP]),
            "vqpc_realise": (I, [VP, VP, I64, I, I, VP, VP]),
            "vqpc_solve_batch": (I, [VP, VP, I64, I, VP, D, I, VP, VP, VP, VP, VP]),
            "vqpc_run_campaign": (I, [VP, VP, I64, I, D, I, I64, VP, VP, VP, VP, VP, VP]),
            "vqpc_run_campaign_d": (I, [VP, VP, I64, I, D, I, I64, VP, VP, VP, VP, VP, VP]),
            "vqpc_run_campaign_ex": (I, [VP, VP, I64, I, D, I, I64, I64, VP, VP, VP, VP, VP, VP]),
            "vqpc_run_campaign_ex_d": (I, [VP, VP, I64, I, D, I, I64, I64, VP, VP, VP, VP, VP, VP]),
            "vqpc_run_campaign_x": (I, [VP, VP, I64, I, D, I, I64, I64, VP, VP, VP, VP, VP, VP, VP]),
            "vqpc_run_campaign_async": (I, [VP, VP, I64, I, D, I, I64, I64, VP, VP, VP, VP, VP, VP]),
            "vqpc_kmeans": (I, [I, VP, I, I, VP, I, I, U64, I, D, VP, VP, C.POINTER(C.c_int)]),
            "vqpc_draw_standard_normal": (I, [I64, I, U64, I64, VP, I]),
            "vqpc_profile": (I, [VP, I]),
            "vqpc_profile_read": (I, [VP, VP, VP, I]),
            "vqpc_fp64_peak": (I, [I, C.POINTER(C.c_double)]),
            "vqpc_debug_pcg2d_phase_cycles": (I, [C.POINTER(C.c_ulonglong), I]),
            "vqpc_debug_pcg1d_phase_cycles": (I, [C.POINTER(C.c_ulonglong), I]),
            "vqpc_counter_hash": (U64, [U64, U64, U64]),
            "vqpc_amg_info": (I, [VP, I, I, VP, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "vqpc_ideal_sweep": (I, [VP, VP, I64, I, VP, I, D, I, VP, VP, VP]),
            "vqpc_kl_basis": (I, [I, I, I, D, D, I, I, VP, VP, VP, C.POINTER(C.c_int)]),
            "vqpc_amg_level": (I, [VP, I, I, VP, VP, VP, VP, VP, VP, VP, VP]),
            "vqpc_normal_quantile": (D, [D]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def error_string(code: int) -> str:
    try:
        return load().vqpc_error_string(code).decode()
    except ImportError:
        return f"error-{code}"


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(code, ctx=None):
    if code != 0:
        msg = load().vqpc_last_error(ctx).decode() if ctx else ""
        raise VqpcError(code, msg)


# --------------------------------------------------------------- host utilities
def draw_standard_normal(n, m, seed, index0=0, threads=None):
    """draw_standard_normal (quantizer.cpp:77-87): out[i, k] = gaussian_draw(seed, index0+i, k)."""
    out = np.empty((n, m), np.float64)
    _check(load().vqpc_draw_standard_normal(n, m, seed, index0, _p(out), threads or os.cpu_count() or 1))
    return out


KERNEL_KINDS = ("assign", "bucket", "realise", "pcg", "other")


def fp64_peak(device=0):
    """Measured fp64 FMA-pipe throughput (TFLOP/s) of this device."""
    v = C.c_double()
    _check(load().vqpc_fp64_peak(device, C.byref(v)))
    return v.value


def pcg2d_phase_cycles(reset=True):
    """Cycles of the 2-D PCG phases (setup, sweeps, P1, P2); zeros unless built with -DVQPC_PHASE_TIMING."""
    out = (C.c_ulonglong * 4)()
    _check(load().vqpc_debug_pcg2d_phase_cycles(out, int(reset)))
    return list(out)


def pcg1d_phase_cycles(reset=True):
    """Cycles between the 1-D PCG's barriers (Ap; update+residual+sweep 1; sweep 2; r.z); zeros unless
    built with -DVQPC_PHASE_TIMING."""
    out = (C.c_ulonglong * 4)()
    _check(load().vqpc_debug_pcg1d_phase_cycles(out, int(reset)))
    return list(out)


def counter_hash(seed, index, comp):
    return load().vqpc_counter_hash(seed, index, comp)


def normal_quantile(p):
    return load().vqpc_normal_quantile(p)


def kmeans(samples, lambdas, P, map="scale", init_seed=1, max_iter=200, rel_tol=1e-6, device=0):
    """Reference kmeans (quantizer.cpp:347-357) with GPU distance sweeps; returns
    (centroids P x m in quantization space, distortion history)."""
    samples, lambdas = f64(samples), f64(lambdas)
    n, m = samples.shape
    out = np.empty((P, m))
    hist = np.empty(max(max_iter, 1))
    nh = C.c_int()
    _check(load().vqpc_kmeans(device, _p(samples), n, m, _p(lambdas), MAPS[map], P, init_seed, max_iter, rel_tol,
                              _p(out), _p(hist), C.byref(nh)))
    return out, hist[: nh.value].copy()


# ---------------------------------------------------------------------- context
def kl_basis(dim, size, sigma2, ell, n_kl, cutoff=True, device=0):
    """build_kl_basis (field.cpp:22-82) on the device (Lanczos, matrix-free
    operator): dict(eigenvalues, eigenvectors (K x N), mass, total_variance)."""
    nn = size if dim == 1 else (size + 1) ** 2
    lam = np.empty(n_kl)
    phi = np.empty((n_kl, nn))
    mass = np.empty(nn)
    kept = C.c_int()
    _check(load().vqpc_kl_basis(device, dim, size, sigma2, ell, n_kl, 1 if cutoff else 0, _p(lam), _p(phi),
                                _p(mass), C.byref(kept)))
    k = kept.value
    return dict(eigenvalues=lam[:k].copy(), eigenvectors=np.ascontiguousarray(phi[:k]), mass=mass,
                total_variance=sigma2 * float(mass.sum()), sigma2=sigma2, ell=ell, mesh_resolution=size, dim=dim)


class Context:
    """One device context: basis, codebook and (after factor_centroids) the P
    centroid factors resident in HBM. Mirrors CampaignArtifacts + the P
    preconditioners of run_campaign_with (driver.cpp:212-219)."""

    def __init__(self, dim, size, basis, codebook, precond="cholesky", device=0):
        self._keep = []
        lam = f64(basis["eigenvalues"])
        phi = f64(basis["eigenvectors"])
        cb_l = f64(codebook["lambdas"])
        cen = f64(codebook["centroids"])
        lat = None if codebook.get("latent") is None else f64(codebook["latent"])
        self._keep += [lam, phi, cb_l, cen, lat]
        K, nn = phi.shape
        self.dim, self.size, self.n_kl, self.n_nodes = dim, size, K, nn
        self.P, self.m = cen.shape
        pb = _Problem(dim, size, K, nn, lam.ctypes.data, phi.ctypes.data, METHODS[codebook["method"]],
                      MAPS[codebook["map"]], self.P, self.m, cb_l.ctypes.data, cen.ctypes.data,
                      None if lat is None else lat.ctypes.data, PRECONDS[precond], device)
        h = C.c_void_p()
        _check(load().vqpc_ctx_create(C.byref(pb), C.byref(h)))
        self.h = h
        self.n = load().vqpc_unknowns(h)
        self.factor_entries = int(load().vqpc_factor_entries(h))
        self.factored = False

    def close(self):
        if getattr(self, "h", None):
            load().vqpc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, code):
        _check(code, self.h)

    @property
    def launches(self):
        return load().vqpc_launch_count(self.h)

    def set_stream(self, stream_ptr):
        self._c(load().vqpc_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def profile(self, enable=True):
        self._c(load().vqpc_profile(self.h, 1 if enable else 0))

    def profile_read(self, reset=True):
        ms = np.zeros(len(KERNEL_KINDS))
        n = np.zeros(len(KERNEL_KINDS), np.int64)
        self._c(load().vqpc_profile_read(self.h, _p(ms), _p(n), 1 if reset else 0))
        return {k: dict(ms=float(ms[i]), launches=int(n[i])) for i, k in enumerate(KERNEL_KINDS)}

    def synchronize(self):
        self._c(load().vqpc_synchronize(self.h))

    def set_exact_reductions(self, enable=True):
        """Reference-order mode: serial dots (2-D), plus Eigen-order LL^T solves and
        unfused updates (1-D, pcg1d_exact_kernel); bit-identical solves."""
        self._c(load().vqpc_set_exact_reductions(self.h, 1 if enable else 0))

    def factor_centroids(self):
        self._c(load().vqpc_factor_centroids(self.h))
        self.factored = True
        self.factor_entries = int(load().vqpc_factor_entries(self.h))

    def ideal_sweep(self, xi, m_list, eps, max_iter=-1):
        """ideal_sweep records (driver.cpp:290-340): B x len(m_list) arrays."""
        xi = f64(np.atleast_2d(xi))
        B, ld = xi.shape
        ml = np.ascontiguousarray(m_list, dtype=np.int32)
        it = np.empty((B, ml.size), np.int32)
        rel = np.empty((B, ml.size))
        st = np.empty((B, ml.size), np.uint8)
        self._c(load().vqpc_ideal_sweep(self.h, _p(xi), B, ld, _p(ml), ml.size, eps, max_iter, _p(it), _p(rel),
                                        _p(st)))
        return dict(iterations=it, rel=rel, status=st)

    def amg_levels(self, p):
        """SA-AMG hierarchy of centroid p as built by the library (same layout as
        oracle.PreconditionerSet.amg_levels)."""
        info = np.zeros(4 * 64, np.int64)
        nlev, dn = C.c_int(), C.c_int()
        self._c(load().vqpc_amg_info(self.h, p, 64, _p(info), C.byref(nlev), C.byref(dn)))
        out = []
        for l in range(nlev.value):
            n, nnz, pnnz, nc = (int(v) for v in info[4 * l:4 * l + 4])
            a_rp, a_col, a_val = np.empty(n + 1, np.int32), np.empty(nnz, np.int32), np.empty(nnz)
            inv = np.empty(n)
            p_rp = np.empty(n + 1, np.int32) if pnnz else np.empty(1, np.int32)
            p_col, p_val = np.empty(max(pnnz, 1), np.int32), np.empty(max(pnnz, 1))
            last = l + 1 == nlev.value
            L = np.empty(dn.value * dn.value) if last and dn.value else None
            self._c(load().vqpc_amg_level(self.h, p, l, _p(a_rp), _p(a_col), _p(a_val), _p(inv), _p(p_rp),
                                          _p(p_col), _p(p_val), _p(L) if L is not None else None))
            lv = dict(n=n, A=(a_rp, a_col, a_val), inv_diag=inv, nc=nc)
            if pnnz:
                lv["P"] = (p_rp, p_col[:pnnz], p_val[:pnnz])
            if L is not None:
                lv["L"] = L.reshape(dn.value, dn.value)
            out.append(lv)
        return out

    def centroid_coefficients(self):
        out = np.empty((self.P, self.n_nodes))
        self._c(load().vqpc_centroid_coefficients(self.h, _p(out)))
        return out

    def precond_apply(self, p, r):
        r = f64(r)
        z = np.empty_like(r)
        self._c(load().vqpc_precond_apply(self.h, p, _p(r), _p(z)))
        return z

    def assign(self, xi):
        xi = f64(np.atleast_2d(xi))
        B, ld = xi.shape
        labels = np.empty(B, np.int32)
        self._c(load().vqpc_assign(self.h, _p(xi), B, ld, _p(labels)))
        return labels

    def realise(self, xi, m=None):
        xi = f64(np.atleast_2d(xi))
        B, ld = xi.shape
        out = np.empty((B, self.n_nodes))
        st = np.empty(B, np.uint8)
        self._c(load().vqpc_realise(self.h, _p(xi), B, ld, ld if m is None else m, _p(out), _p(st)))
        return out, st

    def solve_batch(self, xi, labels, eps, max_iter=-1, max_iter_arr=None, want_x=False):
        xi = f64(np.atleast_2d(xi))
        B, ld = xi.shape
        labels = np.ascontiguousarray(labels, np.int32)
        mia = None if max_iter_arr is None else np.ascontiguousarray(max_iter_arr, np.int32)
        it = np.empty(B, np.int32)
        rel = np.empty(B)
        st = np.empty(B, np.uint8)
        x = np.empty((B, self.n)) if want_x else None
        self._c(load().vqpc_solve_batch(self.h, _p(xi), B, ld, _p(labels), eps, max_iter, _p(mia), _p(it), _p(rel),
                                        _p(st), _p(x)))
        return it, rel, st, x

    def run_campaign(self, xi, eps, max_iter=-1, chunk=0, solve_limit=-1, want_x=False):
        """run_campaign_with (driver.cpp:193-281) on host arrays (copies included);
        solve_limit >= 0 solves only the first solve_limit samples (C5);
        want_x also returns the solutions the reference discards (driver.cpp:236-237)
        as res["x"] (B x n; rows of unsolved samples are NaN)."""
        xi = f64(xi)
        B, ld = xi.shape
        P = self.P
        labels = np.empty(B, np.int32)
        it = np.empty(B, np.int32)
        rel = np.empty(B)
        st = np.empty(B, np.uint8)
        stats = np.empty(4 * P, np.int64)
        summary = np.empty(4, np.int64)
        x = None
        if want_x:
            x = np.full((B, self.n), np.nan)
            self._c(load().vqpc_run_campaign_x(self.h, _p(xi), B, ld, eps, max_iter, chunk, solve_limit, _p(labels),
                                               _p(it), _p(rel), _p(st), _p(stats), _p(summary), _p(x)))
        else:
            self._c(load().vqpc_run_campaign_ex(self.h, _p(xi), B, ld, eps, max_iter, chunk, solve_limit,
                                                _p(labels), _p(it), _p(rel), _p(st), _p(stats), _p(summary)))
        return dict(x=x, labels=labels, iterations=it, rel=rel, status=st, n_p=stats[:P], sum_j=stats[P:2 * P],
                    conv_count=stats[2 * P:3 * P], conv_sum=stats[3 * P:], total_iterations=int(summary[0]),
                    unconverged=int(summary[1]), conv_total=int(summary[2]), conv_sum_total=int(summary[3]))

    def run_campaign_async(self, xi, eps, out, max_iter=-1, chunk=0, solve_limit=-1):
        """vqpc_run_campaign_async: enqueue a campaign over host xi (pinned for overlap)
        into the preallocated host arrays of ``out`` (labels, iterations, rel, status,
        stats, summary — see campaign_outputs) and return at once; results are valid
        after synchronize()."""
        B, ld = xi.shape
        self._c(load().vqpc_run_campaign_async(self.h, _p(xi), B, ld, eps, max_iter, chunk, solve_limit,
                                               _p(out["labels"]), _p(out["iterations"]), _p(out["rel"]),
                                               _p(out["status"]), _p(out["stats"]), _p(out["summary"])))

    def campaign_outputs(self, B, alloc=np.empty):
        """Host result arrays for run_campaign_async (alloc: e.g. a pinned-memory allocator)."""
        return dict(labels=alloc(B, np.int32), iterations=alloc(B, np.int32), rel=alloc(B, np.float64),
                    status=alloc(B, np.uint8), stats=alloc(4 * self.P, np.int64), summary=alloc(4, np.int64))

    def run_campaign_device(self, d_xi_ptr, B, ld, eps, d_labels, d_iters, d_rel, d_status, d_stats, d_summary,
                            max_iter=-1, chunk=0, solve_limit=-1):
        """Device-resident variant: every argument is a raw device pointer (int)."""
        V = C.c_void_p
        self._c(load().vqpc_run_campaign_ex_d(self.h, V(d_xi_ptr), B, ld, eps, max_iter, chunk, solve_limit,
                                              V(d_labels), V(d_iters), V(d_rel), V(d_status), V(d_stats),
                                              V(d_summary)))
