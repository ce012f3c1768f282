"""bench.py host logic (no GPU): workload description per config, roofline
arithmetic for every dominant-kernel kind, CPU sample sizing, and the JSON
contract of the reference arm's line."""
import importlib.util
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_workload_describes_config(name):
    from paper_2403_07824_b200 import campaign
    b = _bench()
    cfg = campaign.CONFIGS[name]
    w = b.workload(cfg, cfg["n_realizations"], cfg["n_kl"])
    n = (cfg["mesh_resolution"] - 1) ** cfg["dim"]
    assert w["unknowns"] == n and w["P"] == cfg["quantizer"]["P"] and w["d"] == cfg["m"]
    assert w["workload"].startswith(name + ":")
    assert ("IC(0)" in w["workload"]) == (cfg["dim"] == 2)
    assert (w["solve_subset"] is not None) == (name == "C5")
    json.dumps(w)


def test_cpu_sample_size_bounded():
    from paper_2403_07824_b200 import campaign
    b = _bench()
    sizes = {k: b.cpu_sample_size(campaign.CONFIGS[k]) for k in ("C1", "C2", "C3", "C4", "C5")}
    # (all threads, one thread): C4 >= 32 samples, C2 >= 8192, one-thread legs bounded
    assert 32 <= sizes["C4"][0] <= 64 and sizes["C4"][1] <= 8
    assert sizes["C2"][0] >= 8192 and sizes["C2"][1] <= 512
    assert all(a >= 16 and 1 <= o <= a for a, o in sizes.values())


def test_default_workload_is_c4():
    b = _bench()
    import sys as _s
    old = _s.argv
    _s.argv = ["bench.py"]
    try:
        assert b.parse().config == "C4"
    finally:
        _s.argv = old


def test_c5_value_counts_solved_samples():
    from paper_2403_07824_b200 import campaign
    b = _bench()
    assert b.solved_count(campaign.CONFIGS["C5"], 1 << 20) == 1 << 16
    assert b.solved_count(campaign.CONFIGS["C2"], 1 << 17) == 1 << 17


def _prof(kind, ms, launches=3):
    p = {k: {"ms": 0.0, "launches": 0} for k in ("assign", "bucket", "realise", "pcg", "other")}
    p[kind] = {"ms": ms, "launches": launches}
    return p


def test_roofline_pcg2d_is_hbm_bound(monkeypatch):
    from paper_2403_07824_b200 import campaign
    b = _bench()
    monkeypatch.setattr(b, "measured_peaks", lambda: {"hbm_gbs": 6536.4})
    cfg = campaign.CONFIGS["C4"]
    r = cfg["mesh_resolution"]
    n, npts = (r - 1) ** 2, (r + 1) ** 2
    iters = 1000
    roof = b.roofline(cfg, _prof("pcg", 3 * 1000.0), iters, 8, 3, 0)  # 1 s per launch
    assert roof["kernel"] == "pcg2d" and roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    assert roof["achieved"] == pytest.approx(8.0 * (2 * npts + 14 * n) * iters / 1e9)
    assert roof["frac"] == pytest.approx(roof["achieved"] / 6536.4)


def test_roofline_pcg1d_and_realise_fp64(monkeypatch):
    from paper_2403_07824_b200 import campaign, lib
    b = _bench()
    monkeypatch.setattr(lib, "fp64_peak", lambda device=0: 33.5)
    cfg = campaign.CONFIGS["C2"]
    n = cfg["mesh_resolution"] - 1
    roof = b.roofline(cfg, _prof("pcg", 3 * 500.0), 10 ** 6, 1 << 17, 3, 0)
    assert roof["kernel"] == "pcg1d" and roof["bound"] == "fp64"
    assert roof["achieved"] == pytest.approx(31.0 * n * 1e6 / 0.5 / 1e12)
    assert roof["frac"] == pytest.approx(roof["achieved"] / 33.5)
    cfg5 = campaign.CONFIGS["C5"]
    roof = b.roofline(cfg5, _prof("realise", 3 * 100.0), 0, 1 << 14, 3, 0)
    assert roof["kernel"] == "realise"
    assert roof["achieved"] == pytest.approx(2.0 * cfg5["mesh_resolution"] * cfg5["n_kl"] * (1 << 14) / 0.1 / 1e12)
    # the effective mode count (after the cutoff) is what the contraction uses
    roof = b.roofline(dict(cfg5, _K=39), _prof("realise", 3 * 100.0), 0, 1 << 14, 3, 0)
    assert roof["achieved"] == pytest.approx(2.0 * cfg5["mesh_resolution"] * 39 * (1 << 14) / 0.1 / 1e12)


def test_per_kernel_rooflines():
    """Every kernel kind of the step gets its SURVEY §8(d) work rate and roof:
    pcg (1-D fp64 / 2-D HBM), realise (DGEMM roof), assign (fp64), bucket (HBM)."""
    from paper_2403_07824_b200 import campaign
    b = _bench()
    cfg = campaign.CONFIGS["C2"]
    n, N, K, B = cfg["mesh_resolution"] - 1, cfg["mesh_resolution"], 73, 1 << 17
    prof = {"pcg": {"ms": 3 * 600.0, "launches": 3}, "realise": {"ms": 3 * 5.0, "launches": 3},
            "assign": {"ms": 3 * 0.05, "launches": 3}, "bucket": {"ms": 3 * 0.1, "launches": 6},
            "other": {"ms": 0.3, "launches": 3}}
    peaks = {"fp64": 33.5, "dgemm": 36.0, "hbm": 6536.4}
    r = b.kernel_rooflines(cfg, prof, 10 ** 7, B, K, 3, peaks)
    assert set(r) == {"pcg", "realise", "assign", "bucket"}
    assert r["pcg"]["achieved"] == pytest.approx(31.0 * n * 1e7 / 0.6 / 1e12) and r["pcg"]["roof"] == "fp64"
    assert r["realise"]["achieved"] == pytest.approx(2.0 * N * K * B / 0.005 / 1e12)
    assert r["realise"]["frac"] == pytest.approx(r["realise"]["achieved"] / 36.0)
    assert r["assign"]["achieved"] == pytest.approx(3.0 * 64 * 8 * B / 0.00005 / 1e12)
    assert r["bucket"]["unit"] == "GB/s" and r["bucket"]["frac"] == pytest.approx(r["bucket"]["achieved"] / 6536.4)
    c4 = campaign.CONFIGS["C4"]
    r4 = b.kernel_rooflines(c4, prof, 10 ** 6, 8192, 100, 3, peaks)
    assert r4["pcg"]["roof"] == "hbm" and r4["pcg"]["unit"] == "GB/s"


def test_reference_arm_contract(monkeypatch, capsys):
    """--impl reference on rank != 0 exits without output; rank 0 prints the
    contract keys (timed on a tiny C1 sample through the oracle)."""
    b = _bench()
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--config", "C1", "--steps", "1",
                                      "--warmup", "0", "--cpu-samples", "16"])
    args = b.parse()
    b.run_reference(args, rank=1, world=2)
    assert capsys.readouterr().out == ""
    b.run_reference(args, rank=0, world=1)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["value"] > 0
