"""bench.py's one-line JSON contract, exercised on the small BASELINE config C1 (256x128, 2 views, 3 iterations):
the keys the driver reads are present and consistent, the timed region launched this library's kernels, and
no launch fell back to the generic kernels."""
import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_bench_line_contract_on_c1():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--workload", "c1", "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["unit"] == "maps/s" and d["vs_baseline"] is None and d["scaling"] == "weak"
    assert d["config"]["workload"].startswith("c1: 256x128 keyframe, 2 neighbour views")
    assert abs(d["value"] - 1e3 / d["ms_per_step"]) <= 1e-3 * d["value"]
    e2e = d["e2e"]
    assert e2e["unit"] == "maps/s" and e2e["value"] > 0
    assert e2e["h2d_bytes_per_step"] == 256 * 128 * 3 and e2e["d2h_bytes_per_step"] == 256 * 128 * 5
    assert d["gpu_launches"] >= 3 * (1 + 2 * 3) and d["generic_fallbacks"] == 0
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3 and 0 < r["frac"] < 1
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert set(d["kernels"]) >= {"refine", "red_black", "eval_costs"}
