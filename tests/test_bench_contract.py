"""bench.py's reference arm runs on CPU: its JSON line carries the driver
contract's keys (impl, metric/unit/value, steps/warmup, the cpu_baseline and
e2e objects) and the reference's own digest for the workload."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "bfs16",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    if "unavailable" in line:
        pytest.skip(line["unavailable"])
    assert line["impl"] == "reference" and line["metric"] == "GTEPS"
    assert line["steps"] == 2 and line["warmup"] == 1 and line["n_gpus"] == 1
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["parity"]["digest"] == line["parity"]["expected"] == "591673cb243fad4e"  # survey §8(c) s16 BFS
    # the stock reference driver, never the product library
    assert line["reference"]["driver"].startswith("wedgegraph.run_until_convergence")
    assert not any("libwedge_b200" in so for so in line["loaded_so"]), line["loaded_so"]
    assert line["config"]["workload"].startswith("BFS on symmetrized RMAT s16")
