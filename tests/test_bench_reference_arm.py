"""bench.py --impl reference (the reference algorithm, oracle mode A, on the
host cores) keeps the driver's JSON contract: one JSON line on stdout with the
arm's metric / unit / direction, the workload it timed, a cpu_baseline that
describes the run, and an e2e object with no host<->device bytes.  Runs on
CPU (cfg1: a few seconds)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, EPFEM_REF_BUDGET_S="60")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "3", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "ip/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("tangent-stiffness assembly")
    assert d["config"]["workload"] == "cfg1" and d["config"]["same_config"] is True
    assert d["config"]["n_int"] == 131072 and d["steps"] == 3 and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and "cfg1" in cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "ip/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert abs(d["value"] - d["config"]["n_int"] / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
