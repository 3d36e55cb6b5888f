"""bench.py's reference arm (the CPU leg the driver runs beside the GPU arm):
runs at a reduced size here and must print ONE JSON line with the contract's
keys — same metric / unit / config as the GPU arm, impl = reference, the
cpu_baseline description and an e2e object with zero copy bytes."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--n", "32",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "certificate voxel-candidates/s"
    assert d["unit"] == "voxel-candidates/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["config"]["grid"] == 32 and d["config"]["candidates"] == 16
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_both_arms_share_the_config_dict():
    sys.path.insert(0, str(ROOT))
    import bench
    a = bench.workload_config(512, 16)
    assert set(a) == {"workload", "grid", "candidates", "l2"} and a["grid"] == 512
