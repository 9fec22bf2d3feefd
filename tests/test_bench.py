"""bench.py keeps the driver's JSON-line contract (task spec): the reference
arm on CPU here, the B200 arm on a GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--ref-seconds", "0.5",
              "--cpals-cpu-iters", "0"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    # the installed reference itself (baseline/_ref) when present, else the port
    from pathlib import Path as _P

    want = "reference" if (_P(ROOT) / "baseline" / "_ref" / "cpkern").exists() else "port"
    assert d["cpu_baseline"]["kind"] == want
    assert {"logical_cpus", "threading_layer"} <= set(d["cpu_baseline"]["cpu"])
    assert d["value"] > 0 and d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run(["--steps", "1", "--warmup", "3", "--e2e-steps", "1", "--dfma-steps", "0", "--gemm-steps", "0",
              "--f32-steps", "0", "--cpals-iters", "2", "--c5-iters", "0", "--cpu-seconds", "0.5"], 900)
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["dtype"] == "f64"
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and r["frac"] > 0
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 8 * 1024 ** 3 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] < d["value"]
    assert d["gpu_launches"] > 0 and {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
def test_b200_arm_multi_rank_path():
    """The N > 1 path of bench.py (torchrun, mode-2 slabs, allreduce of the
    other modes, max-over-ranks timing, e2e per rank) with 2 ranks on the one
    GPU over gloo: one JSON line from rank 0, n_gpus = 2, the global
    workload's flops."""
    import os

    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", str(ROOT / "bench.py"), "--gpus", "2", "--steps",
           "1", "--warmup", "3", "--e2e-steps", "1", "--c5-iters", "2", "--c5-dims", "96,40,36", "--c5-rank", "16",
           "--cpu-seconds", "0.5"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "mode-2 block partition x2"
    # the sharded CP-ALS leg ran through the strict (device-only) communicator
    c5 = d["cp_als_c5"]
    assert "error" not in c5, c5
    assert c5["gpus"] == 2 and c5["sec_per_iter"] > 0 and len(c5["fits"]) == 2
    assert c5["comm_calls_per_iter"] >= 5 and c5["rollbacks"] == 0
