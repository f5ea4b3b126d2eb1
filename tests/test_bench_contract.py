"""bench.py's JSON line contract (the driver parses it): the reference arm (the fp64 oracle on
the host cores) runs on CPU; our arm needs the GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--ref-step-s", "0.2"], 600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"] and d["config"]["config"] == "C3"
    assert d["extrapolated"] is True and 0 < d["sample_fraction"] < 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_json_line():
    d = _run(["--config", "C0", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "alu" and r["achieved"] > 0 and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0.3 < r["frac"] < 1.0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3 * d["steps"]
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and isinstance(c["reasons"], list)


def test_multi_gpu_line_without_enough_gpus():
    """``--gpus 2`` outside torchrun takes the self-launch path; with fewer GPUs visible (this CPU
    box: none) it prints one JSON line saying so, carrying both gather legs' keys."""
    d = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"], 300)
    assert d["n_gpus"] == 2 and d["value"] is None and "unavailable" in d
    g = d["gather"]
    for k in ("fused_ms", "nccl_ms", "fused_bp_ms_per_rank", "nccl_bp_ms_per_rank", "fused_collective_ms_per_rank",
              "nccl_collective_ms_per_rank", "headline"):
        assert k in g


def test_gather_summary_picks_the_fastest_verified_leg():
    sys.path.insert(0, ROOT)
    import bench

    legs = {"fused": {"ms": 7.7, "bp_ms": [7.6, 7.5], "collective_ms": [0.05, 0.1]},
            "nccl": {"ms": 8.0, "bp_ms": [7.6, 7.6], "collective_ms": [0.3, 0.3]}}
    g = bench.gather_summary(2, legs, {"fused": {"ok": True}, "nccl": {"ok": True}})
    assert g["headline"] == "fused" and g["fused_ms"] == 7.7 and g["nccl_ms"] == 8.0
    g = bench.gather_summary(2, legs, {"fused": {"ok": False}, "nccl": {"ok": True}})
    assert g["headline"] == "nccl"
    g = bench.gather_summary(2, {"fused": None, "nccl": legs["nccl"]}, {"nccl": {"ok": False}})
    assert g["headline"] is None and g["fused_ms"] is None
    legs["publish"] = {"ms": 7.5, "bp_ms": [7.4, 7.3], "collective_ms": [0.1, 0.1]}
    g = bench.gather_summary(2, legs, {"fused": {"ok": True}, "publish": {"ok": True}, "nccl": {"ok": True}})
    assert g["headline"] == "publish" and g["publish_ms"] == 7.5


@pytest.mark.gpu
def test_both_gather_legs_on_one_rank():
    """--all-legs: the N > 1 code path on a one-rank group (symmetric-memory fused scatter of the
    rank's tile block, the publish leg, NCCL all-gather of its tile rows), every leg timed and checked
    against the 1-GPU image; exactly one JSON line on stdout."""
    d = _run(["--config", "C0", "--all-legs", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], 900)
    g = d["gather"]
    assert g["world"] == 1 and g["headline"] in ("fused", "publish", "nccl")
    assert g["fused_check"]["ok"] and g["nccl_check"]["ok"] and g["publish_check"]["ok"]
    assert g["publish_ms"] > 0
    assert g["fused_ms"] > 0 and g["nccl_ms"] > 0 and len(g["fused_bp_ms_per_rank"]) == 1
