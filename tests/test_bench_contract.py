"""bench.py's JSON-line contract (the driver parses it): the reference arm on CPU, our arm
on a B200.  Runs bench.py as a subprocess, as the driver does."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    """--impl reference: the fp64 oracle on a bounded sample, one JSON line with impl,
    cpu_baseline and a zero-transfer e2e (task contract)."""
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3", "--config", "c1_tiny")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["vs_baseline"] is None
    assert d["config"]["workload"] == "c1_tiny"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_contract():
    """Default-path line on a small config: roofline, e2e, clocks, launch count, cpu_baseline."""
    d = run_bench("--steps", "20", "--warmup", "3", "--config", "c1_tiny", "--no-prefill")
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["steps"] == 20 and d["warmup"] == 3 and d["scaling"] in ("weak", "strong")
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert d["config"]["layer_caches"] >= 2 and d["step_us"]["p10"] <= d["step_us"]["p50"] <= d["step_us"]["p90"]
    assert d["read_probe"]["gbs"] > 0 and abs(r["frac_of_read_peak"] - r["achieved"] / r["read_peak"]) < 1e-9
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_c5_defaults_to_sharing_aware_decode():
    """C5 (beam groups of 4) runs the N1 tcgen05 kernel by default, coop with --grouped 0 and
    the CUDA-core shared kernel with --shared 4; the roofline is quoted on unique K/V bytes
    either way."""
    common = ("--steps", "5", "--warmup", "3", "--config", "c5_beam", "--no-cpu-baseline", "--no-e2e", "--no-prefill")
    a = run_bench(*common)
    b = run_bench(*common, "--grouped", "0")
    c = run_bench(*common, "--shared", "4")
    assert a["config"]["decode_kernel"].startswith("grouped4") and b["config"]["decode_kernel"] == "coop"
    assert c["config"]["decode_kernel"].startswith("shared4")
    for d in (a, b, c):
        assert d["roofline"]["basis"].startswith("unique") and d["roofline"]["kv_unique_over_logical"] < 0.5


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.gpu
@pytest.mark.parametrize("gather", ["nccl", "fused"])
def test_two_rank_bench_line(gather):
    """bench.py under torchrun with 2 ranks sharing the one GPU (gloo for the plumbing and
    the all-gather; the fused path over CUDA IPC): rank 0 prints one line with the N>1
    fields (per-rank GB/s, gather us for the NCCL-style path, rotated layer caches)."""
    env = dict(os.environ, PA_BENCH_SAME_DEVICE="1", PA_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "5", "--warmup", "3", "--config", "c2_alpaca", "--tp-gather", gather,
                        "--no-cpu-baseline", "--no-prefill", "--no-e2e"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "tp2" and d["config"]["layer_caches"] >= 2
    assert d["config"]["tp_gather"] == gather
    pr = d["per_rank"]
    assert len(pr["attention_gbs"]) == 2 and all(v > 0 for v in pr["attention_gbs"])
    if gather == "nccl":
        assert len(pr["gather_us"]) == 2
    assert d["step_us"]["p10"] <= d["step_us"]["p50"] <= d["step_us"]["p90"]
