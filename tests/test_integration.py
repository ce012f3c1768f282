"""The reference-side drop-in (include/vqp_gpu_adapter.hpp), compiled against the
REAL reference headers and EXECUTED.

tests/adapter/drive_adapter.cpp stands in for the reference's run_campaign
(driver.cpp:283-288) after the one-line switch INTEGRATION.md shows: it loads the
.klb/.qnt artifacts with the reference's own loaders (artifacts.cpp, compiled
unchanged into oracle/_ref), runs vqp::gpu::run_campaign_with and writes the
reference's SimulationReport as JSON. The binary is built in this container
(tests/adapter/Makefile; the GPU box has no /root/reference) and travels with the
repo. CPU tests: it links, and the error mapping (CampaignConfig::precond kinds
without a GPU implementation -> invalid-config with a detailed what(); no device
-> no-device). GPU tests: its report equals the ctypes run's field for field.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from tests.conftest import HAS_GPU

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
ADIR = os.path.join(ROOT, "tests", "adapter")
EXE = os.path.join(ADIR, "_bin", "drive_adapter")


def build_adapter():
    """Compile the test program (only where the reference headers are mounted)."""
    if os.path.isdir(REF_INC):
        from paper_2403_07824_b200 import build
        build.build()
        import oracle
        oracle.build()
        subprocess.check_call(["make", "-s", "-C", ADIR])
    return EXE


def _write_xi(path, xi):
    with open(path, "wb") as f:
        np.array(xi.shape, dtype=np.int64).tofile(f)
        np.ascontiguousarray(xi, dtype=np.float64).tofile(f)


def _run(tmp_path, name, n, precond, gpu_precond=None):
    from paper_2403_07824_b200 import campaign
    from tests.helpers import setup_case
    cfg, basis, cb, xi = setup_case(name, n)
    kb = os.path.join(campaign.CACHE, f"basis_{campaign._key(cfg, 'basis')}.klb")
    qn = os.path.join(campaign.CACHE, f"codebook_{campaign._key(cfg, 'codebook')}.qnt")
    assert os.path.exists(kb) and os.path.exists(qn)
    xp, op = str(tmp_path / f"{name}.xi"), str(tmp_path / f"{name}_{precond}.json")
    _write_xi(xp, xi)
    args = [EXE, kb, qn, xp, op, precond, str(cfg["dim"]), str(cfg["mesh_resolution"])]
    if gpu_precond is not None:
        args.append(str(gpu_precond))
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    return cfg, basis, cb, xi, r.returncode, json.load(open(op))


@pytest.fixture(scope="module")
def exe():
    build_adapter()
    if not os.path.exists(EXE):
        pytest.fail("tests/adapter/_bin/drive_adapter missing: build it where /root/reference is mounted")
    return EXE


def test_adapter_builds_against_reference_headers(exe):
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libvqpc.so" in out and "libvqpref.so" in out


@pytest.mark.parametrize("kind", ["identity", "block_jacobi"])
def test_adapter_rejects_kinds_without_gpu_implementation(exe, tmp_path, kind):
    """CampaignConfig::precond is honoured (driver.cpp:117-126): kinds with no GPU
    implementation raise vqp::Error("invalid-config") whose what() keeps the detail,
    instead of silently substituting another preconditioner."""
    *_, rc, rep = _run(tmp_path, "C1", 8, kind)
    assert rc == 1 and rep["ok"] is False and rep["code"] == "invalid-config"
    assert kind in rep["what"] and "no GPU implementation" in rep["what"]


@pytest.mark.skipif(HAS_GPU, reason="CPU-only check")
def test_adapter_without_device_reports_no_device(exe, tmp_path):
    *_, rc, rep = _run(tmp_path, "C1", 8, "cholesky")
    assert rc == 1 and rep["code"] == "no-device" and rep["what"].startswith("no-device")


def _compare(rep, res):
    r = res["report"]
    assert rep["ok"] is True and rep["n_realizations"] == r["n_realizations"]
    assert rep["assignments"] == [int(v) for v in res["labels"]]
    assert rep["iterations"] == [int(v) for v in res["iterations"]]
    assert rep["converged"] == [int(v == 0) for v in res["status"]]
    assert np.array_equal(np.array(rep["final_rel"]), res["rel"])
    for a, b in zip(rep["per_centroid"], r["per_centroid"]):
        assert (a["n_p"], a["sum_j"]) == (b["n_p"], b["sum_j"])
        assert a["mean_j"] == b["mean_j"] and a["centroid_norm"] == pytest.approx(b["centroid_norm"], rel=1e-15)
    for k in ("mean_j", "total_iterations", "max_sum_j", "min_sum_j", "unconverged"):
        assert rep[k] == r[k], k


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,precond,override", [
    ("C1", 256, "cholesky", None),   # 1-D, the reference's cholesky kind
    ("C4s", 48, "cholesky", None),   # 2-D, the reference's cholesky kind (RCM + LL^T)
    ("C4s", 48, "amg", None),        # 2-D, the reference's default kind (SA-AMG)
    ("C4s", 48, "amg", 4),           # GpuOptions override: IC(0)
])
def test_adapter_report_equals_ctypes_run(exe, tmp_path, name, n, precond, override):
    """The reference-side program's SimulationReport equals the ctypes campaign over
    the same artifacts and xi (same labels, records and per-centroid statistics)."""
    from paper_2403_07824_b200 import campaign
    cfg, basis, cb, xi, rc, rep = _run(tmp_path, name, n, precond, override)
    assert rc == 0, rep
    kind = {None: precond, 4: "ic0"}[override]
    res = campaign.run_campaign_with(dict(cfg, precond=kind), dict(basis=basis, codebook=cb), xi)
    _compare(rep, res)
