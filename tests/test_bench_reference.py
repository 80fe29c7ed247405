"""bench.py's reference arm (`--impl reference`) runs on CPU: it prints one JSON line with the
contract's keys (the CPU oracle port on the host cores, plus the reference's own ToyModel engine).
Small model and sample so the test takes seconds; the driver runs it at the 8B shape."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--model", "llama-tiny:bench",
                        "--steps", "1", "--warmup", "1", "--cpu-sample-prompt", "2", "--cpu-sample-gen", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config"):
        assert k in line, k
    assert line["value"] > 0 and line["unit"] == "tok/s"
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
