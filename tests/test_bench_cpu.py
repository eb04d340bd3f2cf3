"""bench.py contract checks that run without a GPU: the reference arm (the CPU
oracle, this tier's reference implementation) prints one JSON line with the
driver's keys, and the metric arithmetic follows Eq.(13)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "worked_examples.json")))


def test_reference_arm_json_line():
    env = dict(os.environ, FBS_REF_BUDGET_S="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "synthetic", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "steps", "warmup", "higher_is_better", "impl", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "Mdisp/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_mdisp_matches_eq13_worked_example():
    sys.path.insert(0, ROOT)
    import bench
    import stereo_synth as synth
    g = GOLD["mde_s"]
    cfg = synth.Config("x", g["W"], g["H"], 0, g["D"] - 1, 4, 0)
    assert abs(bench.mdisp(cfg, 1, g["t_s"]) - g["expected"]) < 1e-9
    assert abs(bench.mdisp(cfg, 1, g["t_s"]) - g["paper"]) < 0.5  # paper's 344.16 at ~0.0294 s


def test_warmup_floor():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "2"],
                         capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "warmup" in out.stderr
