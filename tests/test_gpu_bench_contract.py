"""bench.py keeps the driver contract: one JSON line with the required keys,
single process and under torchrun (2 ranks sharing the one GPU over gloo --
the SFFT_BENCH_BACKEND test hook; the production multi-GPU run uses NCCL)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"}


def last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_single_process_line(cuda):
    out = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--cpu-seconds", "0.5",
                          "--e2e-steps", "2"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = last_json(out.stdout)
    assert KEYS <= set(d) and {"e2e", "cpu_baseline"} <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["gpu_launches"] == 5
    assert d["roofline"]["bound"] == "hbm" and 0.3 < d["roofline"]["frac"] < 1.2
    # default workload: BASELINE configs[2] fp64 (the reference's arithmetic)
    assert d["config"]["workload"] == "cfg3_n1024_f64" and d["dtype"] == "f64"
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * (1 << 18) * 1024 * 8 and d["e2e"]["matches_device_result"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["one_process"]["cores"] == 1 and d["cpu_baseline"]["one_process"]["value"] > 0
    # the checker after the timed region: fp64 bitwise the oracle
    assert d["parity"]["pass"] and d["parity"]["bitwise"] and d["parity"]["rows_checked"] == 64


def test_torchrun_two_ranks(cuda):
    env = dict(os.environ, SFFT_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29537", "bench.py", "--gpus", "2",
                          "--config", "cfg2_n64_f32", "--scaling", "weak",
                          "--steps", "4", "--warmup", "3", "--no-e2e"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = last_json(out.stdout)
    assert KEYS <= set(d) and d["n_gpus"] == 2 and d["config"]["global_batch"] == 2 * (1 << 20)
    assert d["scaling"] == "weak"
    assert "cpu_baseline" not in d          # rank 0 at N=1 only


def test_gpus_flag_spawns_ranks_strong(cuda):
    # `bench.py --gpus 2` without a launcher spawns the ranks itself; strong
    # scaling splits the config's B rows into two contiguous blocks
    env = dict(os.environ, SFFT_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "4", "--warmup", "3", "--no-e2e"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = last_json(out.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 1 << 18 and d["config"]["batch_per_gpu"] == 1 << 17
    assert d["parity"]["pass"]


def test_reference_arm_line(cuda):
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = last_json(out.stdout)
    assert d["impl"] == "reference" and d["unit"] == "transforms/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
