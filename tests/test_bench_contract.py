"""bench.py's reference arm on CPU (no GPU needed): the oracle timed as it stands, one JSON line
with the contract's keys; under torchrun with 2 ranks only rank 0 prints and the others exit 0."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def test_reference_arm_single():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg3", "--steps", "1",
                        "--warmup", "1", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["impl"] == "reference" and line["unit"] == "motifs/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["steps"] == 1 and line["warmup"] == 1
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_torchrun_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
                        "--config", "cfg3", "--gpus", "2", "--steps", "1", "--warmup", "1", "--cpu-seconds", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_line_gpu_small():
    """bench.py's own arm on the GPU (small config): one JSON line with the contract's keys."""
    r = subprocess.run([sys.executable, "bench.py", "--config", "cfg3", "--k", "3", "--steps", "2", "--warmup", "3",
                        "--e2e-steps", "1", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    roof = line["roofline"]
    assert roof["bound"] == "alu" and roof["peak"] > 0 and roof["unit"] == "Gwarp-inst/s"
    assert roof["frac"] is None or 0 < roof["frac"] <= 1.0
    assert roof["frac"] is None or 0 < roof["hbm"]["frac"] <= 1.0
    assert line["dtype"] in ("u32", "u64")
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert "workload" in line["config"]
