"""bench.py's reference arm (the fp64 oracle timed on the host) keeps the
driver contract: one JSON line with impl, metric/unit of our arm, cpu_baseline
and an e2e block with zero copy bytes.  CPU only (a small workload)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "c1_n8_2d8", "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         check=True).stdout.strip().splitlines()
    line = json.loads(out[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "steps/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["metric"].startswith("SOS grad steps/sec")
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "steps/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("c1_n8_2d8")
