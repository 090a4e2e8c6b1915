"""Host logic of bench.py (CPU, -m "not gpu"): the algorithmic flop model's
per-kernel split, and the reference arm's output contract (exactly one JSON
line on stdout, whatever libraries print)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_flops_parts_sum_to_total():
    mesh, orders, _ = bench.cfg5_sample(4)
    total = bench.flops_residual(mesh, orders)
    parts = bench.flops_residual(mesh, orders, parts=True)
    assert set(parts) == {"k_ns_res", "k_ns_grad", "qhat_faces", "flux_faces"}
    assert all(v > 0 for v in parts.values())
    assert abs(sum(parts.values()) - total) <= 1e-9 * total


def test_reference_arm_prints_one_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GDOF/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("cfg5")
