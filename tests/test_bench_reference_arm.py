"""The `bench.py --impl reference` line (the oracle timed on the host cores) keeps the bench contract:
the GPU arm's metric / unit / config.workload, a cpu_baseline describing the run, a zero-copy e2e."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                        "--config", "C1", "--ref-pixels", "4"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    # (the GPU arm's config dict, key for key: the driver compares the two)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    sys.path.insert(0, ROOT)
    import bench
    from synth import CONFIGS
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == "iters/s"
    assert d["higher_is_better"] is True and d["warmup"] >= 3 and d["steps"] == 1
    assert d["config"] == bench.mapping_config(CONFIGS["C1"], True, "CUDA graph of the whole step (2 streams)", 1)
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    # ms_per_step is the measured sample, the extrapolation is declared
    cb = d["cpu_baseline"]
    assert cb["extrapolated"] is True and 0 < cb["sample_fraction"] <= 1.0
    assert abs(d["ms_per_step"] * 1e-3 - cb["sample_fraction"] / d["value"]) < 1e-6 * d["ms_per_step"] + 1e-9
    assert d["e2e"] == {"value": d["value"], "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
