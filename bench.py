"""Benchmark: rank-2000 dense MTTKRP over all modes (BASELINE config 4) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = the MTTKRP of every mode (0, 1, 2) of the 1024^3 float64 tensor
against rank-2000 factors (the north star's headline case).  `value` is
algorithmic GFLOP/s, 2 N R (d-1) flops per mode (BASELINE.json's roofline
numerator), with inputs resident in HBM; the 8 GiB tensor is 65x the L2, so
no flush is needed between steps.  `e2e` is the same metric through the
public API from pinned HOST buffers, H2D of tensor + factors and D2H of the
three results inside the timed region.  Multi-GPU (torchrun): the tensor is
block-partitioned along mode 0; mode 0 needs no communication, modes 1 and 2
allreduce their I_k x R partials over NCCL (strong scaling, fixed tensor).

`--impl reference` times the CPU restatement of the reference TILE kernel
(oracle/, C + OpenMP, all host threads) on a bounded slab of the same
workload; only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "dense MTTKRP GFLOP/s & roofline fraction vs rank R; CP-ALS sec/iter at 1/2/4/8 GPU"
DIMS = (1024, 1024, 1024)
RANK = 2000
SM = 2  # shard mode of the c4 leg at N > 1 (see run_b200)
SEED = 0
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
NCU_SUMMARY = ROOT / "profiles" / "ncu_summary.json"


def _hbm_peak_gbs():
    """The pod's measured copy bandwidth (MEASURED_PEAKS.json), else the
    B200_PROFILING.md fallback the perfmodel carries."""
    try:
        return float(json.loads(PEAKS_FILE.read_text())["hbm_gbs"])
    except Exception:  # noqa: BLE001
        from paper_2510_14891_b200.perfmodel import B200_HBM_BYTES_PER_S

        return B200_HBM_BYTES_PER_S / 1e9


HBM_PEAK_GBS = _hbm_peak_gbs()
FP64_NOMINAL_TFS = 37.22496  # 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz


def algo_flops(dims, rank):
    n = int(np.prod(dims))
    return 2 * n * rank * (len(dims) - 1)


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 4 + i and s[4 + i] == "Active"})
        power = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_median": statistics.median(power) if power else None}


# ------------------------------------------------------------ reference (CPU)
REF_DIR = ROOT / "baseline" / "_ref"  # the unmodified reference, pip-installed


def reference_cpkern():
    """The reference package itself (`cpkern`, Python + numba), installed
    under baseline/_ref; None when it is absent or numba cannot import (the
    oracle's C port then stands in, kind "port")."""
    if not (REF_DIR / "cpkern").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/cpk_numba_cache")
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 1))
    if str(REF_DIR) not in sys.path:
        sys.path.append(str(REF_DIR))
    try:
        import cpkern

        return cpkern
    except Exception:  # noqa: BLE001
        return None


def host_cpu_info(ref=None):
    """lscpu model / sockets / cores and the threading layer the CPU path used."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keys = {"Model name": "model", "Socket(s)": "sockets", "Core(s) per socket": "cores_per_socket",
                "Thread(s) per core": "threads_per_core"}
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in keys:
                info[keys[k.strip()]] = v.strip()
    except Exception:  # noqa: BLE001
        pass
    if ref is not None:
        import numba

        try:
            info["threading_layer"] = f"numba {numba.__version__} {numba.threading_layer()}"
        except Exception:  # noqa: BLE001  (no parallel region has run yet)
            info["threading_layer"] = f"numba {numba.__version__}"
    else:
        info["threading_layer"] = "OpenMP (gcc, oracle/liboracle.so)"
    return info


def cpu_sample(target_seconds: float, threads: int = 0):
    """Time the reference's TILE MTTKRP on the host on a slab of config 4.

    The slab keeps I_0 = I_1 = 1024 and R = 2000 and cuts mode 2 to `depth`
    slices; all three modes are run, like one GPU step.  With the reference
    installed (baseline/_ref) this is `cpkern.run(y, m, MttkrpPlan(TILE, k,
    unroll=16, tile_volume=N_T))` itself -- numba, all host threads -- with
    N_T from the reference's own Eq. 6 heuristic on its intel-8480p spec
    (w = 362, N_T = 131044, clamped per mode by plan_for_mode); otherwise
    the oracle's C + OpenMP restatement of the same kernel (kind "port",
    bit-identical to it and ~2x faster, profiles/r01_port_vs_reference.json).
    """
    from oracle import gen

    fs = gen.bench_factors(DIMS, RANK, SEED)
    ck = reference_cpkern()
    if ck is not None:
        import numba

        from cpkern.mttkrp import MttkrpPlan, Variant, heuristic_tile_volume, plan_for_mode

        if threads > 0:
            numba.set_num_threads(threads)
        w = numba.get_num_threads()
        n_t = heuristic_tile_volume(DIMS, ck.bundled_machine("intel-8480p"))

        def run_modes(dims, y, sub):
            t = ck.DenseTensor(dims, y)
            m = ck.KruskalTensor(np.ones(RANK), sub, validate=False)
            base = MttkrpPlan(Variant.TILE, 0, unroll=16, tile_volume=n_t, workers=0)
            for k in range(3):
                ck.run(t, m, plan_for_mode(base, dims, k))

        # numba compiles on the first call: a tiny warm-up outside the timing
        run_modes((4, 4, 2), np.ones(32), [fs[0][:4], fs[1][:4], fs[2][:2]])
        kind = "reference"
        what = f"cpkern.run TILE (the reference, numba), N_T={n_t} F=16"
    else:
        from oracle import oracle

        w = oracle.max_threads() if threads <= 0 else threads

        def run_modes(dims, y, sub):
            for k in range(3):
                oracle.mttkrp_tile(y, dims, k, sub, None, f_cols=16, n_t=131044, workers=w)

        kind = "port"
        what = "oracle TILE port (C+OpenMP), N_T=131044 F=16"

    def run(depth):
        dims = (DIMS[0], DIMS[1], depth)
        y = gen.splitmix_uniform(int(np.prod(dims)), SEED)
        sub = [fs[0], fs[1], fs[2][:depth]]
        t0 = time.perf_counter()
        run_modes(dims, y, sub)
        return time.perf_counter() - t0, algo_flops(dims, RANK) * 3

    # calibrate on one slice, then size the sample to ~target_seconds
    t1, f1 = run(1)
    depth = max(1, min(DIMS[2], int(target_seconds / max(t1, 1e-3))))
    if depth == 1:
        t, f = t1, f1
    else:
        t, f = run(depth)
    return {"seconds": t, "flops": f, "depth": depth, "threads": w, "kind": kind, "what": what,
            "cpu": host_cpu_info(ck)}


def cpu_cpals_sample(iters: int = 1):
    """The reference's own cp_als (baseline/_ref) on config 3 (128^4,
    R = 256) for `iters` sweeps on the host, with the GEMM plan -- its
    fastest CPU MTTKRP (the default SLICE / TILE plans take ~85 s per mode
    here); seconds per sweep.  None without the reference."""
    ck = reference_cpkern()
    if ck is None:
        return None
    from cpkern.mttkrp import MttkrpPlan, Variant

    dims = (128, 128, 128, 128)
    y = ck.DenseTensor(dims, np.random.Generator(np.random.Philox(SEED)).random(int(np.prod(dims))))
    cfg = ck.AlsConfig(rank=256, tol=0.0, max_iters=iters, seed=0, plan=MttkrpPlan(Variant.GEMM, 0))
    t0 = time.perf_counter()
    _, tr = ck.cp_als(y, cfg)
    dt = time.perf_counter() - t0
    return {"config": "c3: 4-way 128^4 f64, rank 256", "impl": "cpkern.cp_als (the reference), plan GEMM",
            "iters": iters, "sec_per_iter": dt / iters,
            "mttkrp_sec_per_iter": sum(sum(s) for s in tr.mttkrp_seconds) / iters,
            "other_sec_per_iter": sum(tr.other_seconds) / iters, "fits": tr.fits,
            "cores": os.cpu_count(), "cpu": host_cpu_info(ck)}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    budget = args.ref_seconds or max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(budget / 4)
    vals, secs = [], []
    s = None
    for _ in range(args.steps):
        s = cpu_sample(budget)
        vals.append(s["flops"] / s["seconds"] / 1e9)
        secs.append(s["seconds"])
    value = statistics.median(vals)
    sample = f"slab 1024x1024x{s['depth']} of config 4 (R=2000), all 3 modes, {s['what']}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (splitmix64 counter-based U[0,1) tensor, Philox(1) factors)",
        "config": {"workload": "c4: 3-way 1024^3 f64 tensor, rank 2000, MTTKRP all modes (CPU slab sample)",
                   "dims": list(DIMS), "rank": RANK, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": s["threads"], "kind": s["kind"],
                         "sample": sample, "cpu": s["cpu"]},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if args.cpals_cpu_iters > 0:
        try:
            line["cp_als"] = cpu_cpals_sample(args.cpals_cpu_iters)
        except Exception as exc:  # noqa: BLE001  (report, do not lose the line)
            line["cp_als"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU path
def shard_rows(n, world, rank):
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def run_b200(args):
    import torch

    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as dist

        # one process per GPU over NCCL; BENCH_DIST_BACKEND=gloo lets the
        # tests run this multi-rank path with several ranks on one GPU
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if backend == "nccl":
            # CUDA tensors go over NCCL; the group also carries a gloo
            # backend so a stray CPU tensor could never hang the run (the
            # sharded sweep's communicator is strict and raises on one)
            dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_2510_14891_b200 as ck
    from paper_2510_14891_b200 import _lib
    from paper_2510_14891_b200 import harness
    from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device, mttkrp_modes, resolve_plan

    # ---- inputs resident in HBM: this rank's slab of config 4 along SM
    # (every mode of the cube is "the longest"; the slowest one gives
    # contiguous slabs and keeps the other modes' o-groups long: a mode-0
    # slab of 128 rows at 8 GPUs would flush modes 1 and 2 every 8 chunks)
    lo, hi = shard_rows(DIMS[SM], world, rank)
    local_dims = tuple(hi - lo if m == SM else e for m, e in enumerate(DIMS))
    n_local = int(np.prod(local_dims))
    lib = _lib.load()
    # element (i0, i1, i2) of the global tensor is splitmix(i0 + 1024 i1 + 1024^2 i2)
    full = torch.empty(int(np.prod(DIMS)), dtype=torch.float64, device=dev)
    _lib.check(lib.cpk_fill_uniform_f64(full.data_ptr(), full.numel(), SEED, 0,
                                        torch.cuda.current_stream().cuda_stream), "fill")
    if world == 1:
        y = full
    else:  # the slowest mode's slab is one contiguous range
        plane = DIMS[0] * DIMS[1]
        y = full[lo * plane:hi * plane].clone()
        del full
    # the reference CLI's factor recipe (cli.py:137-141): Philox(seed + 1)
    fs_host = [np.asarray(a) for a in harness.bench_factors(DIMS, RANK, SEED).factors]
    fs_host[SM] = np.ascontiguousarray(fs_host[SM][lo:hi])
    fs = [torch.from_numpy(a).to(dev) for a in fs_host]
    torch.cuda.synchronize()

    def step(events=None):
        outs = []
        for k in range(3):
            if events is not None:
                events[k][0].record()
            g, _, _ = mttkrp_device(y, local_dims, fs, k, None, MttkrpPlan(Variant.B200, k))
            if events is not None:
                events[k][1].record()
            if world > 1 and k != SM:
                dist.all_reduce(g)
            outs.append(g)
        return outs

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    mode_events = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
                   for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        barrier()
        t0.record()
        for s in range(args.steps):
            step(mode_events[s])
        t1.record()
        barrier()
    elapsed = t0.elapsed_time(t1) * 1e-3
    if world > 1:
        tt = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    per_mode = [statistics.median(mode_events[s][k][0].elapsed_time(mode_events[s][k][1]) for s in range(args.steps))
                for k in range(3)]
    plans = [resolve_plan(MttkrpPlan(Variant.B200, k), local_dims, RANK) for k in range(3)]

    # ---- the same step with the DFMA (CUDA-core FMA) consumers, for the
    # north star's literal math choice; not part of `value`
    dfma = None
    if args.dfma_steps > 0 and world == 1:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        ms = [[] for _ in range(3)]
        for it in range(args.dfma_steps + 1):
            for k in range(3):
                ev[k][0].record()
                mttkrp_device(y, local_dims, fs, k, None, MttkrpPlan(Variant.B200, k, engine="tma"))
                ev[k][1].record()
            torch.cuda.synchronize()
            if it > 0:  # first pass warms the kernels up
                for k in range(3):
                    ms[k].append(ev[k][0].elapsed_time(ev[k][1]))
        dfma_mode = [statistics.median(m) for m in ms]
        dplan = resolve_plan(MttkrpPlan(Variant.B200, 0, engine="tma"), local_dims, RANK)
        dfma = {"engine": "tma (DFMA outer products, warp-specialized TMA)", "rank_tile": dplan["rank_tile"],
                "per_mode_ms": dfma_mode,
                "gflops": algo_flops(local_dims, RANK) * 3 / (sum(dfma_mode) * 1e-3) / 1e9}

    # ---- the same three MTTKRPs through a dimension tree (mttkrp_modes
    # tree=True: M_0, then W = Y x_0 A_0 (I_1 I_2 x R) once and M_1, M_2 read
    # out of it): two tensor passes per step; not part of `value`
    tree_leg = None
    if args.tree_steps > 0 and world == 1:
        ref_outs = step()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.tree_steps + 1)]
        outs = mttkrp_modes(y, fs, tree=True)  # warm-up
        torch.cuda.synchronize()
        evs[0].record()
        for i in range(args.tree_steps):
            outs = mttkrp_modes(y, fs, tree=True)
            evs[i + 1].record()
        evs[-1].synchronize()
        t_ms = evs[0].elapsed_time(evs[-1]) / args.tree_steps
        per_call = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.tree_steps)]
        dev_rel = max(float(torch.linalg.norm(a - b) / torch.linalg.norm(b)) for a, b in zip(outs, ref_outs))
        tree_leg = {"what": "mttkrp_modes(tree=True): M_0 + one W_R = Y x_0 A_0 MTTKRP (16.8 GB) + 2 contractions",
                    "ms_per_step": t_ms, "gflops": algo_flops(DIMS, RANK) * 3 / (t_ms * 1e-3) / 1e9,
                    "max_rel_frobenius_vs_per_mode": dev_rel, "steps": args.tree_steps, "per_call_ms": per_call}
        del outs, ref_outs
        torch.cuda.empty_cache()

    total_flops = algo_flops(DIMS, RANK) * 3 * args.steps
    value = total_flops / elapsed / 1e9

    # ---- GFLOP/s and roofline fraction vs rank R (BASELINE.json's metric
    # name) on the config-2 shape, every mode, auto plans; not part of `value`
    rank_sweep = None
    if args.rank_sweep and world == 1:
        from paper_2510_14891_b200.perfmodel import roofline_seconds

        d2 = (512, 512, 512)
        y2 = torch.empty(int(np.prod(d2)), dtype=torch.float64, device=dev)
        _lib.check(lib.cpk_fill_uniform_f64(y2.data_ptr(), y2.numel(), SEED, 0,
                                            torch.cuda.current_stream().cuda_stream), "fill")
        n2 = int(np.prod(d2))
        rank_sweep = {"shape": list(d2), "roofline": "max(8N/HBM, 2NR(d-1)/FP64 nominal)",
                      "timing": "per call, calls issued back to back between two CUDA events (host work "
                                "overlaps the previous call, as inside a CP-ALS sweep)",
                      "hbm_peak_gbs": HBM_PEAK_GBS, "points": []}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for r in (8, 16, 24, 32, 48, 64, 128, 256, 512, 1000, 2000):
            rng = np.random.Generator(np.random.Philox(1))
            f2 = [torch.from_numpy(rng.random((n, r))).to(dev) for n in d2]
            ms, tiles = [], []
            for k in range(3):
                plan = MttkrpPlan(Variant.B200, k)
                mttkrp_device(y2, d2, f2, k, None, plan)  # warm-up (plan, workspace, tensor maps)
                reps = 20 if r <= 64 else 5
                e0.record()
                for _ in range(reps):
                    mttkrp_device(y2, d2, f2, k, None, plan)
                e1.record()
                e1.synchronize()
                ms.append(e0.elapsed_time(e1) / reps)
                tiles.append(resolve_plan(plan, d2, r)["rank_tile"])
            roof = roofline_seconds(d2, r) * 1e3  # nominal FP64 peak (37.2 TF/s at 1965 MHz)
            t_mode = sum(ms) / 3 * 1e-3
            rank_sweep["points"].append({"rank": r, "ms_per_mode": ms, "rank_tiles": tiles,
                                         "gflops": algo_flops(d2, r) * 3 / (sum(ms) * 1e-3) / 1e9,
                                         "roofline_frac": 3 * roof / sum(ms),
                                         "hbm_frac": 8 * n2 / t_mode / (HBM_PEAK_GBS * 1e9),
                                         "fp64_issued_frac": 2 * n2 * r / t_mode / (FP64_NOMINAL_TFS * 1e12)})
        del y2, f2
        torch.cuda.empty_cache()

    # ---- the library baseline on the same GPU: partial KRPs + cuBLAS DGEMM
    # (the reference's mttkrp_gemm, mttkrp.py:230-276); not part of `value`
    gemm = None
    if args.gemm_steps > 0 and world == 1:
        from paper_2510_14891_b200.baselines import gemm_scratch_bytes, mttkrp_gemm_cublas

        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        ms = [[] for _ in range(3)]
        try:
            for it in range(args.gemm_steps + 1):
                for k in range(3):
                    ev[k][0].record()
                    g = mttkrp_gemm_cublas(y, local_dims, fs, k)
                    ev[k][1].record()
                    del g
                torch.cuda.synchronize()
                if it > 0:
                    for k in range(3):
                        ms[k].append(ev[k][0].elapsed_time(ev[k][1]))
            gm = [statistics.median(m) for m in ms]
            gemm = {"impl": "partial KRPs (torch) + cuBLAS DGEMM, mttkrp.py:230-276", "per_mode_ms": gm,
                    "gflops": algo_flops(local_dims, RANK) * 3 / (sum(gm) * 1e-3) / 1e9,
                    "scratch_bytes_per_mode": [gemm_scratch_bytes(local_dims, RANK, k) for k in range(3)]}
        except torch.OutOfMemoryError as exc:
            gemm = {"error": f"OOM: {exc}"[:200]}
        torch.cuda.empty_cache()

    # ---- optional float32 path (north star: <= 1e-4): the tcgen05 3xTF32
    # kernel on the same values rounded to fp32, checked against the FP64
    # result of those values; not part of `value`
    f32 = None
    if args.f32_steps > 0 and world == 1:
        try:
            y32 = y.float()
            f32s = [f.float() for f in fs]
            y64r = y32.double()
            f64r = [f.double() for f in f32s]
            errs, ms = [], [[] for _ in range(3)]
            for k in range(3):
                g64, _, _ = mttkrp_device(y64r, local_dims, f64r, k)
                for it in range(args.f32_steps + 1):
                    g32, _, t = mttkrp_device(y32, local_dims, f32s, k)
                    if it > 0:
                        ms[k].append(t.seconds * 1e3)
                errs.append(float(torch.linalg.norm(g32.double() - g64) / torch.linalg.norm(g64)))
                del g64, g32
            del y64r, f64r, y32
            fm = [statistics.median(m) for m in ms]
            f32 = {"impl": "tcgen05.mma kind::tf32, 3xTF32 split, TMEM accumulators (cpk_mttkrp_f32)",
                   "per_mode_ms": fm, "gflops": algo_flops(local_dims, RANK) * 3 / (sum(fm) * 1e-3) / 1e9,
                   "rel_frobenius_vs_fp64": errs, "tolerance": 1e-4}
        except Exception as exc:  # report, do not lose the headline line
            f32 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()

    # ---- e2e through the public API from pinned host buffers (N=1 only: the
    # per-rank host slab at N>1 is the same code path)
    e2e = None
    if args.e2e_steps > 0:
        y_host = torch.empty(n_local, dtype=torch.float64, pin_memory=True)
        y_host.copy_(y)
        fs_pinned = [torch.from_numpy(a).pin_memory() for a in fs_host]
        h2d = 8 * n_local + sum(8 * a.size for a in fs_host)
        d2h = 8 * RANK * sum(local_dims)

        g_pinned = [torch.empty((local_dims[k], RANK), dtype=torch.float64, pin_memory=True)
                    for k in range(3)]

        def e2e_step():
            # a host-resident DenseTensor through ck.mttkrp_modes: the copy
            # runs in slabs and the work of all three modes is issued per
            # landed slab, so the copy hides under the compute.  Results come
            # back into pinned buffers (no host sync until the end).
            yt = ck.DenseTensor(local_dims, y_host)
            fd = [a.to(dev, non_blocking=True) for a in fs_pinned]
            for k, g in enumerate(ck.mttkrp_modes(yt, fd, (0, 1, 2))):
                if world > 1 and k != SM:
                    dist.all_reduce(g)
                g_pinned[k].copy_(g, non_blocking=True)
            torch.cuda.synchronize()
            return g_pinned

        e2e_step()
        barrier()
        te = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        e2e_t = time.perf_counter() - te
        if world > 1:
            tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_t = float(tt.item())
        e2e = {"value": algo_flops(DIMS, RANK) * 3 * args.e2e_steps / e2e_t / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
               "ms_per_step": 1e3 * e2e_t / args.e2e_steps}
        del y_host

    # ---- roofline of the dominant kernel (mttkrp_f64_sm100, per launch)
    fp64_peak = None
    if rank == 0:
        pk = (_lib.C.c_double(0), _lib.C.c_double(0))
        _lib.check(lib.cpk_fp64_peak_probe(_lib.C.byref(pk[0]), _lib.C.byref(pk[1])), "probe")
        fp64_peak = pk[0].value
    nominal = 148 * 64 * 2 * 1.965e9
    flops_per_launch = algo_flops(local_dims, RANK)  # one mode
    mean_launch_s = statistics.mean(per_mode) * 1e-3
    achieved = flops_per_launch / mean_launch_s
    # issued work: the kernel runs the DMMA fragments of live 8-column
    # blocks only (a warp whose 64 columns straddle R skips its dead tail),
    # so the columns it issues are R rounded up to 8, not to the rank tile
    live_cols = -(-RANK // 8) * 8
    traffic = None
    traffic_src = None
    if NCU_SUMMARY.exists():
        try:
            summ = json.loads(NCU_SUMMARY.read_text())
            traffic = summ.get("dram_bytes_per_launch")
            traffic_src = (f"{NCU_SUMMARY.relative_to(ROOT)} (ncu --set full capture '{summ.get('tag')}', "
                           "dram__bytes_read.sum + dram__bytes_write.sum per launch; not measured in this run)")
        except Exception:
            traffic = None

    del y, fs
    torch.cuda.empty_cache()
    cp = None
    if args.cpals_iters > 0 and world == 1:
        cp = bench_cpals(ck, dev, args.cpals_iters)
        torch.cuda.empty_cache()
    c5 = None
    c5_dims = tuple(int(x) for x in args.c5_dims.split(","))
    if args.c5_iters > 0:
        try:
            c5 = bench_c5(dev, args.c5_iters, c5_dims, args.c5_rank)
        except Exception as exc:  # report, do not lose the headline line
            c5 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()
        if world == 1 and args.c5_projection and c5 and "error" not in c5:
            try:
                proj = bench_c5_projection(dev, args.c5_iters, c5_dims, args.c5_rank)
                for pt in proj["points"]:
                    pt["projected_speedup"] = c5["sec_per_iter"] / pt["rank0_sec_per_iter"]
                    pt["per_mode_projected_speedup"] = (c5["per_mode"]["sec_per_iter"]
                                                        / pt["per_mode_rank0_sec_per_iter"])
                c5["projection"] = proj
            except Exception as exc:  # noqa: BLE001
                c5["projection"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        s = cpu_sample(args.cpu_seconds)
        cpu = {"value": s["flops"] / s["seconds"] / 1e9, "unit": "GFLOP/s", "cores": s["threads"], "kind": s["kind"],
               "sample": f"{s['what']} on slab 1024x1024x{s['depth']} of config 4, R=2000, all 3 modes, "
                         f"{s['seconds']:.1f} s", "cpu": s["cpu"]}
        if cp is not None and args.cpals_cpu_iters > 0:
            try:
                cp["cpu_reference"] = cpu_cpals_sample(args.cpals_cpu_iters)
            except Exception as exc:  # noqa: BLE001
                cp["cpu_reference"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if rank == 0:
        hbm = 6508.2e9
        try:
            hbm = json.loads(PEAKS_FILE.read_text())["hbm_gbs"] * 1e9
        except Exception:
            pass
        peak = fp64_peak or nominal
        roof_t = max(8 * int(np.prod(DIMS)) / hbm, algo_flops(DIMS, RANK) / peak)
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (splitmix64 counter-based U[0,1) tensor generated on device, Philox(1) factors)",
            "config": {"workload": "c4: 3-way 1024x1024x1024 f64 tensor, rank 2000, MTTKRP of all 3 modes per step",
                       "dims": list(DIMS), "rank": RANK, "parallelism": f"mode-{SM} block partition x{world}",
                       "l2": "inputs 8 GiB >> 126 MB L2; no flush needed"},
            "per_mode_ms": per_mode,
            "paper_gflops": int(np.prod(DIMS)) * RANK * 3 * 3 * args.steps / elapsed / 1024 ** 3,
            # bound "tensor": the DMMA kernel is bound by the tensor pipe's
            # FP64 (DMMA) subpipe (ncu sm__inst_executed_pipe_tensor_subpipe_dmma
            # ~96 %); its peak is the FP64 one, measured live -- not the bf16
            # peak of MEASURED_PEAKS.json
            "roofline": {"bound": "tensor", "pipe": "fp64 (DMMA = DFMA datapath)",
                         "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": "cpk_fp64_peak_probe (max of register DFMA and DMMA loops, this run)"
                         if fp64_peak else "nominal 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz",
                         "nominal_peak": nominal / 1e12,
                         "kernel": "mttkrp_f64_ws_sm100 (TMA + DMMA consumers) + splitk_reduce_f64, per mode",
                         "plans": [{key: p[key] for key in ("engine", "rank_tile", "block_rows", "block_k", "splits")}
                                   for p in plans],
                         "flops_per_launch": flops_per_launch,
                         "issued_fp64_frac": (int(np.prod(local_dims)) * 2 * live_cols / mean_launch_s) / peak,
                         "north_star_roofline_ms_per_mode": roof_t * 1e3,
                         "north_star_frac": roof_t * 3 * args.steps / elapsed},
            "dfma_engine": dfma,
            "all_modes_dimension_tree": tree_leg,
            "rank_sweep": rank_sweep,
            "gemm_baseline": gemm,
            "fp32_path": f32,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": 6 * args.steps,
            "clocks": clocks.summary(),
        }
        if cp:
            line["cp_als"] = cp
        if c5:
            line["cp_als_c5"] = c5
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_cpals(ck, dev, iters):
    """CP-ALS seconds per sweep at config 3 (128^4, R=256): the API default
    (dimension tree, split 2: two tensor passes per sweep), its graph
    replay, and the per-mode sweep (four passes, the reference's structure)."""
    import torch

    from paper_2510_14891_b200.perfmodel import roofline_seconds

    dims = (128, 128, 128, 128)
    t = ck.DenseTensor.uniform(dims, seed=SEED, device=dev)
    roof = 4 * roofline_seconds(dims, 256)  # the sweep's 4 MTTKRPs at the north-star roofline
    res = {"config": "c3: 4-way 128^4 f64, rank 256", "iters": iters, "roofline_sec_per_iter": roof}
    for tree, graph in ((None, None), (None, True), (False, None), (False, True)):
        cfg = ck.AlsConfig(rank=256, tol=0.0, max_iters=iters, seed=0, dimtree=tree)
        ck.cp_als(t, replace(cfg, max_iters=2), graph=graph)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, tr = ck.cp_als(t, cfg, graph=graph)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        dst = res if tree is None else res.setdefault("per_mode", {"what": "dimtree=False: 4 MTTKRPs per sweep"})
        if graph is None:  # eager below GRAPH_MIN_ITERS sweeps
            dst.update({"sec_per_iter": dt / iters, "roofline_frac": roof / (dt / iters),
                        "mttkrp_sec_per_iter": statistics.median(sum(s) for s in tr.mttkrp_seconds),
                        "other_sec_per_iter": statistics.median(tr.other_seconds), "fit_last": tr.fits[-1],
                        "tree_split": tr.tree_split})
        else:  # forced capture: sweeps 2.. are one CUDA-graph replay each
            dst.update({"graph_sec_per_iter": dt / iters,
                        "graph_sec_per_replayed_sweep": statistics.median(
                            sum(m) + o for m, o in zip(tr.mttkrp_seconds[1:], tr.other_seconds[1:]))})
    return res


def bench_c5(dev, iters, dims=(4096, 2048, 2048), r=512):
    """Sharded CP-ALS at config 5 (4096 x 2048 x 2048, R = 512): seconds per
    sweep (CUDA events on each rank, max over ranks).  Each rank generates
    its mode-0 slab on its GPU; the sweep is the single-GPU engine with the
    NCCL exchange steps (sharded.py)."""
    import torch

    from paper_2510_14891_b200 import sharded
    from paper_2510_14891_b200.cpals import AlsConfig

    comm = sharded.Comm(device=dev)
    part = sharded.partition_for(dims, comm.world)
    y = sharded.uniform_slab(part, comm.rank, seed=SEED, device=dev)
    sharded.cp_als_sharded(y, part, AlsConfig(rank=r, tol=0.0, max_iters=1, seed=0), comm, gather=False)  # warm-up
    torch.cuda.empty_cache()
    comm.reset()
    _, tr = sharded.cp_als_sharded(y, part, AlsConfig(rank=r, tol=0.0, max_iters=iters, seed=0), comm,
                                   gather=False)
    sec = statistics.median(tr.sweep_seconds)
    mt = statistics.median(sum(s) for s in tr.mttkrp_seconds)
    comm_s = tr.comm_seconds / max(1, len(tr.fits))
    # the per-mode sweep (dimtree=False: 3 tensor passes, the reference's structure)
    torch.cuda.empty_cache()
    _, tr_pm = sharded.cp_als_sharded(y, part, AlsConfig(rank=r, tol=0.0, max_iters=iters, seed=0, dimtree=False),
                                      comm, gather=False)
    sec_pm = statistics.median(tr_pm.sweep_seconds)
    if comm.world > 1:
        t = torch.tensor([sec, mt, comm_s, sec_pm], dtype=torch.float64, device=dev)
        comm.dist.all_reduce(t, op=comm.dist.ReduceOp.MAX)
        sec, mt, comm_s, sec_pm = (float(v) for v in t.tolist())
    del y
    flops = 3 * algo_flops(dims, r)
    from paper_2510_14891_b200.perfmodel import roofline_seconds

    # the sweep's 3 MTTKRPs of the whole tensor at the roofline of this many GPUs
    roof = 3 * roofline_seconds(dims, r) / comm.world
    return {"config": f"c5: 3-way {'x'.join(map(str, dims))} f64, rank {r}, mode-{part.mode} block partition",
            "gpus": comm.world, "iters": iters, "sec_per_iter": sec, "roofline_sec_per_iter": roof,
            "roofline_frac": roof / sec, "mttkrp_sec_per_iter": mt,
            "mttkrp_gflops": flops / mt / 1e9, "mttkrp_gflops_per_gpu": flops / mt / 1e9 / comm.world,
            "comm_sec_per_iter": comm_s, "comm_bytes_per_iter": tr.comm_bytes // max(1, len(tr.fits)),
            "comm_calls_per_iter": tr.comm_calls / max(1, len(tr.fits)), "rollbacks": tr.rollbacks,
            "tree_split": tr.tree_split,
            "timing": "CUDA events per sweep (sweep start -> stats readback), max over ranks", "fits": tr.fits,
            "per_mode": {"what": "dimtree=False: 3 MTTKRPs per sweep", "sec_per_iter": sec_pm,
                         "mttkrp_gflops": flops / statistics.median(sum(s) for s in tr_pm.mttkrp_seconds) / 1e9,
                         "fits": tr_pm.fits}}


def bench_c5_projection(dev, iters, dims=(4096, 2048, 2048), r=512, worlds=(2, 4, 8)):
    """One-GPU projection of the sharded c5 sweep: rank 0's own work at P
    ranks (its 1/P slab, the same engine and plans), with the collectives
    elided by a loopback communicator -- so the sweep time is what one rank
    computes, and the projected speed-up is sec(P=1) / sec(P).  Fits are
    meaningless (partial sums are never combined); the transfers it leaves
    out are ~18 MiB per sweep (tens of microseconds over NVLink 5).  This box
    has one GPU; the real N-GPU number is `cp_als_c5` under torchrun."""
    import torch

    from paper_2510_14891_b200 import sharded
    from paper_2510_14891_b200.cpals import AlsConfig

    class Loopback(sharded.Comm):
        def __init__(self, world):
            super().__init__(device=dev)
            self.world, self.rank = world, 0

        def allreduce_(self, t, op=None):
            self._check(t)
            self.calls += 1
            self.bytes += t.numel() * t.element_size()
            return t

    out = []
    for world in worlds:
        comm = Loopback(world)
        part = sharded.partition_for(dims, world)
        y = sharded.uniform_slab(part, 0, seed=SEED, device=dev)
        sharded.cp_als_sharded(y, part, AlsConfig(rank=r, tol=0.0, max_iters=1, seed=0), comm, gather=False)
        comm.bytes = 0
        _, tr = sharded.cp_als_sharded(y, part, AlsConfig(rank=r, tol=0.0, max_iters=iters, seed=0), comm,
                                       gather=False)
        elided = comm.bytes // max(1, len(tr.fits))
        torch.cuda.empty_cache()
        _, tr_pm = sharded.cp_als_sharded(y, part, AlsConfig(rank=r, tol=0.0, max_iters=iters, seed=0,
                                                             dimtree=False), comm, gather=False)
        out.append({"gpus": world, "rank0_sec_per_iter": statistics.median(tr.sweep_seconds),
                    "rank0_mttkrp_sec_per_iter": statistics.median(sum(m) for m in tr.mttkrp_seconds),
                    "elided_bytes_per_iter": elided, "rollbacks": tr.rollbacks,
                    "tree_split": tr.tree_split,
                    "per_mode_rank0_sec_per_iter": statistics.median(tr_pm.sweep_seconds)})
        del y
        torch.cuda.empty_cache()
    return {"what": "rank 0's sweep at P ranks on this one GPU, collectives elided (loopback)",
            "config": f"c5: {'x'.join(map(str, dims))} f64, rank {r}", "iters": iters, "points": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--dfma-steps", type=int, default=2)
    ap.add_argument("--gemm-steps", type=int, default=2)
    ap.add_argument("--rank-sweep", type=int, default=1, help="1: add the GFLOP/s-vs-rank leg (c2 shape)")
    ap.add_argument("--f32-steps", type=int, default=2)
    ap.add_argument("--tree-steps", type=int, default=3, help="c4 step through mttkrp_modes(tree=True)")
    ap.add_argument("--cpals-iters", type=int, default=10)
    ap.add_argument("--c5-iters", type=int, default=3)
    ap.add_argument("--c5-dims", default="4096,2048,2048", help="CP-ALS leg shape (tests shrink it)")
    ap.add_argument("--c5-rank", type=int, default=512)
    ap.add_argument("--c5-projection", type=int, default=1, help="1: add the one-GPU P=2/4/8 rank-0 projection")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpals-cpu-iters", type=int, default=1, help="reference cp_als sweeps on the host (c3)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=0.0, help="reference arm: CPU seconds per step (0 = auto)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
