"""bench.py's reference arm on the CPU (the contract's JSON line): runs here without a GPU, on a small sample budget.
Under a multi-rank launch only rank 0 prints; the other ranks exit 0 without work."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                           "--warmup", "0", "--cpu-budget", "1"], capture_output=True, text=True, env=env, timeout=600)


def test_reference_arm_prints_the_contract_line():
    res = run()
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["unit"] == "DOF/s" and line["higher_is_better"] is True and line["vs_baseline"] is None
    assert "configs[2]" in line["config"]["workload"] and set(line["config"]) == {"workload", "ndof", "nt", "m", "l2"}
    assert line["e2e"] == {"value": line["value"], "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and "sample" in cb
    # a step of this arm is one bounded sample: its wall time, not the extrapolated time-to-solution
    assert line["ms_per_step"] < 120e3 < cb["extrapolated_tts_s"] * 1e3
    assert line["value"] > 0


def test_reference_arm_other_ranks_exit_quietly():
    res = run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert res.returncode == 0 and res.stdout.strip() == ""
