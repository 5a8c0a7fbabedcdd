"""bench.py's JSON contract where it does not need a GPU: the reference arm
(`--impl reference`) runs the unmodified reference on the host and prints one
line with the driver's keys."""
import json
import os
import subprocess
import sys

import pytest

from checkers import reference_available
from conftest import ROOT

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("path", ["factor", "symbolic"])
def test_reference_arm_prints_one_contract_line(path):
    d = run_bench("--impl", "reference", "--path", path, "--config", "c1", "--steps", "1", "--warmup", "3")
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("C1")


def test_reference_arm_for_the_solve_says_why_it_is_unavailable():
    d = run_bench("--impl", "reference", "--path", "solve", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and "unavailable" in d
