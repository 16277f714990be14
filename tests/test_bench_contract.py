"""bench.py contract checks that run on CPU: the reference arm prints one JSON line with the required
keys, and the algorithmic byte model matches SURVEY 8(d) D.3 on the configs of BASELINE.md."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from lf_synth import CONFIGS  # noqa: E402


def test_alg_bytes_match_baseline_md():
    # BASELINE.md section 3 (bf16 out): tiny 33,540; q7 4,212,752; q3 1,075,316,736; r 8,596,234,240
    assert bench.alg_bytes_per_step(CONFIGS["tiny"], 1, 2) == 33540
    assert bench.alg_bytes_per_step(CONFIGS["q7"], 1, 2) == 4212752
    assert bench.alg_bytes_per_step(CONFIGS["q3"], 64, 2) == 1075316736
    assert bench.alg_bytes_per_step(CONFIGS["r"], 256, 2) == 8596234240
    assert bench.alg_bytes_per_step(CONFIGS["f1"], 128, 2) == 1680871424


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "tiny",
                        "--steps", "3", "--warmup", "3", "--ref-seconds", "0.2"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == "tiny"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_warmup_floor():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "2"], capture_output=True,
                       text=True, timeout=120, cwd=ROOT)
    assert r.returncode != 0 and "warmup" in r.stderr


def test_l2_methods():
    """Caches larger than L2 run back to back; L2-resident ones cycle >= 8 x L2 of layer caches; only
    caches too small for <= 256 layers fall back to per-step timing after an L2 flush."""
    big = bench.cache_bytes_per_gpu(CONFIGS["r"], 256)
    assert big > bench.FLUSH_BELOW and bench.layers_for(big) == 1
    q7 = bench.cache_bytes_per_gpu(CONFIGS["q7"], 1)
    L = bench.layers_for(q7)
    assert 1 < L <= bench.MAX_LAYERS and L * q7 >= bench.CYCLE_FACTOR * bench.L2_BYTES
    assert bench.layers_for(bench.cache_bytes_per_gpu(CONFIGS["tiny"], 1)) == 0
    assert "flushed" in bench.l2_note(bench.cache_bytes_per_gpu(CONFIGS["tiny"], 1))
    assert "layer caches" in bench.l2_note(q7) and "larger than L2" in bench.l2_note(big)
