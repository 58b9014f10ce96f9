"""The bench.py contract on CPU: the reference arm's JSON line (the oracle on a tiny sample) carries
every key the driver reads, and the roofline model's per-frame-iteration work matches DESIGN.md 9."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0", "--ref-frames", "4"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert "workload" in d["config"]


def test_roofline_model_c2():
    import bench
    import synth

    cfg = synth.CONFIGS["C2"]
    mufu, fma, byts = bench.per_frame_iter(cfg, 0)
    assert mufu == 2 * 2048 * 64 + 1024 * 64  # packed log messages at q = 64: 2 E q + N q
    assert bench.per_frame_iter(synth.CONFIGS["C4"], 0)[0] == 4096  # linear messages at q = 256: 1 rcp per edge
    assert fma == 2048 * 6 * 64 + 1024 * 7 * 64  # separable VN + the decision points
    assert byts == 2 * 2048 * 64 * 4 + 4 * 1024 * 6 + 1024  # one message set read + written, channel, symbols
    r = bench.roofline(cfg, 0, frame_iters=1000, seconds=1000 * 427e-9, traffic=None)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["achieved"] - byts * 1000 / (1000 * 427e-9) / 1e9) < 1e-6
    assert 0.3 < r["frac"] < 0.5
