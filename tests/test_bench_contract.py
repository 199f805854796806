"""bench.py keeps the driver's JSON contract: one line on stdout with the
required keys -- the reference arm on CPU here, our arm on the B200."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, cwd=REPO,
                         capture_output=True, text=True, timeout=timeout, check=True)
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"], 600)
    assert BASE <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    # crossdict itself when baseline/_ref is installed, else the C port
    has_ref = os.path.isdir(os.path.join(REPO, "baseline", "_ref", "crossdict"))
    assert d["cpu_baseline"]["kind"] == ("reference" if has_ref else "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the same config object as our arm's line; the bounded sample is named beside it
    assert d["config"]["signals"] == 1_000_000 and "configs[4]" in d["config"]["workload"]
    assert d["signals_per_step"] > 0


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--no-extras"], 1200)
    assert BASE <= set(d) and d.get("impl", "ours") != "reference"
    assert d["value"] > 0 and d["scaling"] == "strong" and "workload" in d["config"]
    assert d["config"]["signals"] == 1_000_000 and "configs[4]" in d["config"]["workload"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    # algorithmic flops / time against P_emu: the Gram form of step 2 does fewer
    # flops than SURVEY 8(d) charges it, so the fraction may pass 1
    assert d["roofline"]["frac"] > 0 and d["roofline"]["step"]["frac"] > 0
    assert d["full_omp"]["value"] > 0
    assert d["e2e_api"]["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] > 0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
