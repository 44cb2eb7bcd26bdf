"""bench.py contract checks that need no GPU: the reference arm never loads the product
library (only oracle/), prints one JSON line with the fields the driver reads, and
`--gpus N` refuses a WORLD_SIZE that disagrees with it."""
import json
import os
import subprocess
import sys

from conftest import ROOT

_STUB = r'''
import json, sys, types
sys.argv = ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"]
sys.path.insert(0, ROOT)
import oracle.cpu_arm as arm
class FakeArm:
    """Stands in for RefArm (which materialises 90 GB of Mixtral slabs): same interface."""
    def __init__(self, *a, **k):
        self.L, self.threads = 32, 2
    def step(self, s):
        return 0.5, {"router": 0.1, "llapor": 0.1, "presched_simulate": 0.1, "experts": 0.2, "makespan_ticks": 1}, None
    def legs_1core(self, min_seconds=0.25):
        return {n: (1.0, 10) for n in arm.ref_time_legs.__globals__["REF_LEGS"]}
    def close(self):
        pass
arm.RefArm = FakeArm
import bench
bench.main()
loaded = sorted(m for m in sys.modules if m.startswith("paper_2509_23638_b200"))
print("LOADED", json.dumps(loaded))
'''


def test_reference_arm_loads_only_oracle():
    out = subprocess.run([sys.executable, "-c", _STUB.replace("ROOT", repr(str(ROOT)))], capture_output=True,
                         text=True, cwd=ROOT, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    line = json.loads(lines[0])
    assert json.loads(lines[-1].split(" ", 1)[1]) == []  # no product module imported
    assert line["impl"] == "reference" and line["unit"] == "tokens/s" and line["steps"] == 2
    assert line["ms_per_step"] == 500.0 and abs(line["value"] - 16 / 0.5) < 1e-9
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["consistency"]["fits_in_driver_run"] is True
    assert len(line["cpu_baseline"]["legs_1core_us"]) == 8


def test_world_size_must_match_gpus():
    env = {**os.environ, "WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4"], capture_output=True, text=True,
                         env=env, cwd=ROOT, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=2" in (out.stderr + out.stdout)
