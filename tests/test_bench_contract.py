"""The bench.py JSON-line contract, checked on the committed round profiles (CPU only).

Every key the driver and the judge read must be present with the right shape: the base
contract (metric ... config), `e2e`, `gpu_launches`, `roofline`, `cpu_baseline`, `clocks`; and
for the reference arm `impl`, `cpu_baseline` and a zero-byte `e2e`.
"""
import json
from pathlib import Path

import pytest

PROFILES = Path(__file__).resolve().parents[1] / "profiles" / "r2"
ARM_FILES = ["bench_c1.jsonl", "bench_c2.jsonl", "bench_c3.jsonl", "bench_c4.jsonl",
             "bench_c5.jsonl"]


def last_line(name):
    lines = [l for l in (PROFILES / name).read_text().splitlines() if l.startswith("{")]
    assert lines, name
    return json.loads(lines[-1])


@pytest.mark.parametrize("name", ARM_FILES)
def test_isg_arm_line(name):
    d = last_line(name)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, (name, k)
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["warmup"] >= 3
    assert d["scaling"] in ("weak", "strong") and d["higher_is_better"] is True
    assert "workload" in d["config"] and "l2" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] >= 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, (name, k)
    assert 0 < r["frac"] < 1 and r["achieved"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9)
    c = d["cpu_baseline"]
    assert c is not None, name
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, (name, k)
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1
    clk = d["clocks"]
    assert clk["sm_mhz"] and clk["sm_max_mhz"] and isinstance(clk["reasons"], list)
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(clk["reasons"])


@pytest.mark.parametrize("name", ["bench_reference.jsonl", "bench_reference_c2.jsonl"])
def test_reference_arm_line(name):
    d = last_line(name)
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] in ("iters/s", "frames/s")
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_headline_is_c3_train():
    """The default bench line is BASELINE.json's train metric on the C3 workload."""
    base = json.loads((PROFILES.parents[1] / "BASELINE.json").read_text())
    d = last_line("bench_c3.jsonl")
    assert d["metric"] in base["metric"]
    assert d["config"]["n_gaussians"] == 1_000_000
    assert (d["config"]["width"], d["config"]["height"]) == (1920, 1080)


def test_headline_carries_render_fps():
    """The default line also reports BASELINE's second metric (C2 render FPS) with its own e2e
    and the reference's own render() beside it."""
    d = last_line("bench_c3.jsonl")
    r = d["render"]
    assert r["unit"] == "frames/s" and r["value"] > 0 and r["e2e"]["value"] > 0
    assert r["e2e"]["d2h_bytes_per_step"] == 1920 * 1080 * 3 * 4
    assert r["cpu_baseline"]["kind"] == "reference" and r["cpu_baseline"]["value"] > 0


def test_reference_arm_shares_the_config():
    a, b = last_line("bench_c3.jsonl"), last_line("bench_reference.jsonl")
    assert a["config"] == b["config"] and a["metric"] == b["metric"] and a["unit"] == b["unit"]
