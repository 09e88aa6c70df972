"""bench.py host logic on CPU: the R7 gate used outside the cpu_baseline leg, JSON-serialisable results,
busBW convention (R15), and the reference arm's output line."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402


def _bf16(f32):
    return (np.asarray(f32, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def test_fp64_gate_accepts_exact_and_rejects_wrong():
    xs = [synth.normal(2, r, 4096, "bf16") for r in range(4)]
    F = np.stack([bench.bf16_to_f64(x) for x in xs]).sum(0)
    y = _bf16(F.astype(np.float32))
    ok = bench.fp64_gate(y, xs)
    assert ok is True and json.dumps({"ok": ok})
    bad = y.copy()
    bad[17] ^= 0x4000  # flip an exponent bit
    assert bench.fp64_gate(bad, xs) is False


def test_busbw_convention():
    alg, bus = bench.busbw(2 << 30, 1.0, 8)
    assert abs(alg - (2 << 30) / 1e9) < 1e-9 and abs(bus - alg * 14 / 8) < 1e-9


def test_reference_arm_line():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                          "--warmup", "3", "--mib", "1"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0
