"""bench.py's reference arm runs on CPU (the oracle port): its JSON line keeps
the driver's contract -- one line on stdout, the iterations it actually timed
in `steps`, the same `config` dict as our arm, host facts."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "C1",
           "--steps", "3", "--warmup", "1", "--no-ttt-c1"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "it/s" and d["value"] > 0
    assert d["steps"] == 3 and d["steps_requested"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert {"cpu_model", "nproc", "numpy", "scipy"} <= set(d["host"])
    sys.path.insert(0, REPO)
    import bench
    from paper_2603_15504_b200 import instances

    class A:
        config = "C1"

    assert d["config"] == json.loads(json.dumps(bench.workload_config(A, instances.lp_random(2000, 4000, 0.01, 0))))
