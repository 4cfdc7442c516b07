"""bench.py's JSON line keeps the driver contract (both arms): the keys the
driver and the judge read, with sane types and values, on the quick C1
configuration (the headline C3 line has the same builder); both arms print
the same metric / unit / direction / workload (the driver pairs them on
these), and ``--gpus 2`` launches two ranks by itself (gloo on the one test
GPU: a functional check of the N>1 path, never a reported number)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _run(*args, env=None):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=900,
                         env=None if env is None else {**os.environ, **env})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout + out.stderr[-3000:]
    return json.loads(lines[0])


def test_bench_line_contract(cuda_device):
    d = _run("--config", "c1", "--steps", "2", "--warmup", "3", "--cpu-nodes", "2048")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("c1")
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "algorithmic_frac"):
        assert k in r, k
    assert r["achieved"] > 0 and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["frac"] < 1.2  # executed work: a physical fraction
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("port", "reference") and c["sample"]
    assert c["cpu_model"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    ref = _run("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3",
               "--cpu-nodes", "2048")
    for k in ("metric", "unit", "higher_is_better"):
        assert ref[k] == d[k], k
    assert ref["config"]["workload"] == d["config"]["workload"]


def test_reference_arm_contract(cuda_device):
    d = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.parametrize("config", ["c1", "c4"])
def test_bench_spawns_ranks(cuda_device, config):
    """``bench.py --gpus 2`` (no torchrun) runs two ranks and reports n_gpus 2:
    C1's i-slabs + the packed gradient all-reduce, C4's mesh-parallel step +
    the one-bucket parameter all-reduce."""
    d = _run("--gpus", "2", "--config", config, "--steps", "2", "--warmup", "3",
             "--no-cpu-baseline", env={"WV_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"].endswith("x2")
