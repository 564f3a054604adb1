"""bench.py keeps the driver's contract: one JSON line with the required keys, at N=1 and (on one
GPU, MOM_BENCH_SHARED_GPU test mode) through the N=2 torchrun path with the fused gather."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"]


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_contract(cuda_device):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    res = _last_json(r.stdout)
    for k in REQUIRED:
        assert k in res, k
    assert res["n_gpus"] == 1 and res["steps"] == 3 and res["warmup"] == 3
    assert res["value"] > 0 and res["ms_per_step"] > 0
    assert res["roofline"]["bound"] == "tensor" and 0 < res["roofline"]["frac"] < 1.5
    assert res["gpu_launches"] == 3 * (2 * res["config"]["M"] + 4)
    assert res["e2e"]["h2d_bytes_per_step"] > 0 and res["e2e"]["value"] > 0
    assert 0 < res["e2e"]["pcie_h2d_gbs_incl_kv_reload"] < 200  # host-link rate: physical (PCIe Gen5 x16)
    # a 3-step region is far below 3 s: the roofline compares with the burst figure
    assert "burst" in res["roofline"]["peak_source"] and res["roofline"]["frac"] == res["roofline"]["frac_of_burst_peak"]
    assert res["serial"]["value"] > 0
    assert res["activation_reduction_x"] > res["config"]["M"] * 0.99
    kt = res["kernel_trace"]  # in-kernel timeline: clocks and MMA-issue efficiency are physical
    assert "error" not in kt, kt
    assert 500 < kt["phaseA_mhz"] <= res["clocks"]["sm_max_mhz"] + 50
    assert 0.8 < kt["mlp_step_mma_issue_efficiency"] <= 1.02
    assert kt["launches"] == 2 * 2 * res["config"]["M"]
    st = res["stack_cfg5"]  # config 5 (32 layers, 455 000 tokens) measured in the same run
    assert "error" not in st, st
    assert "skipped" in st or (st["value"] > 0 and st["gather_verified"] is True and st["n_gpus"] == 1
                               and st["scaling"] == "strong"), st


def test_bench_reference_arm():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--config", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = _last_json(r.stdout)
    assert res["impl"] == "reference" and res["value"] > 0 and res["cpu_baseline"]["kind"] == "oracle"


def test_bench_two_ranks_shared_gpu(cuda_device):
    env = dict(os.environ, MOM_BENCH_SHARED_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--config", "0", "--no-stack"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    res = _last_json(r.stdout)
    assert res["n_gpus"] == 2 and res["config"]["global_tokens"] == 2 * res["config"]["seq_len_per_gpu"]
