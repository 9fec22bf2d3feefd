"""The reference's tile-width sweep (cpkern `sweep`, cli.py:343-464) on B200.

Same protocol and CSV dialect: for each variant x rank x tile width x mode,
`warmup` untimed runs then `reps` timed runs; one row per rep with the
columns of cli.py:361-364 (modes 1-based, floats at 17 significant digits,
cli.py:338-340), and an aggregate file whose gflops is the mean over modes
of each mode's best rep, with `best` marking the argmax per (variant, rank)
(cli.py:433-450).  Model columns use the paper's traffic models on the
chosen machine spec (perfmodel.py:121-184; default the bundled nvidia-b200
spec).  Three B200 columns are appended to the per-rep rows: the rank tile,
split count and engine the planner used.

Inputs follow the reference CLI recipe (cli.py:121-141): tensor
Philox(seed).random(N), factors Philox(seed + 1), unit weights.  Paper
Table III used the tile width as its knob; on the GPU the width sets N_T =
w^(d-1), i.e. the split-K granularity (mttkrp.py:345-375 semantics).

    python -m paper_2510_14891_b200 sweep --shape 401,201,12,501 --ranks 32 \\
        --variants tile --tile-widths 2,4,6,8,12 --out sweep.csv
"""

from __future__ import annotations

import csv
import json
import math
import os
import statistics

import numpy as np

import importlib

from . import perfmodel as pm
from .dtensor import DenseTensor, num_elements
from .errors import ParameterError
from .kruskal import KruskalTensor

mt = importlib.import_module(".mttkrp", __package__)  # the module (the package re-exports a function of this name)

COLUMNS = ["variant", "mode", "rank", "tile_width", "N_T", "rep", "time_s", "gflops",
           "mops0", "mopsInf", "T0", "T0LM", "TInf", "atomic_updates"]
B200_COLUMNS = ["rank_tile", "splits", "engine"]
AGG_COLUMNS = ["variant", "rank", "tile_width", "N_T", "gflops", "best"]
SWEEP_VARIANTS = (mt.Variant.ELEM, mt.Variant.SLICE, mt.Variant.TILE, mt.Variant.B200)


def _cell(v):
    return f"{v:.17g}" if isinstance(v, float) else v


def bench_factors(dims, rank: int, seed: int):
    """cli.py:137-141: Philox(seed + 1) uniform factors in mode order, unit weights."""
    rng = np.random.Generator(np.random.Philox(seed + 1))
    return KruskalTensor(np.ones(rank), [rng.random((n, rank)) for n in dims], validate=False)


def sweep(y: DenseTensor, ranks, variants=(mt.Variant.TILE,), tile_widths=None, modes=None, reps: int = 3,
          warmup: int = 1, machine: pm.MachineSpec | None = None, seed: int = 0, out: str = "sweep.csv",
          agg_out: str | None = None) -> dict:
    machine = machine or pm.bundled_machine("nvidia-b200")
    d = y.ndim
    variants = [mt.Variant(v) for v in variants]
    for v in variants:
        if v not in SWEEP_VARIANTS:
            raise ParameterError(f"sweep benchmarks {[b.value for b in SWEEP_VARIANTS]}, not {v.value}")
    modes = list(range(d)) if modes is None else [int(m) for m in modes]
    widths = list(tile_widths) if tile_widths else [mt.heuristic_tile_width(y.dims, machine)]
    if any(w < 1 for w in widths):
        raise ParameterError("tile widths must be >= 1")
    rows, agg_rows = [], []
    for variant in variants:
        for rank in ranks:
            m = bench_factors(y.dims, rank, seed)
            f = pm.flops(y.dims, rank)
            m_inf = pm.mem_infty(y.dims, rank, machine.s_f_bytes)
            t_inf = pm.predict_seconds(f, m_inf, machine)
            for width in (widths if variant == mt.Variant.TILE else [None]):
                per_mode = []
                agg_nt = width ** (d - 1) if variant == mt.Variant.TILE else (1 if variant == mt.Variant.ELEM else "")
                for mode in modes:
                    n_s = y.size // y.dims[mode]
                    nt = {mt.Variant.TILE: max(1, min((width or 1) ** (d - 1), n_s)),
                          mt.Variant.SLICE: n_s, mt.Variant.ELEM: 1}.get(variant)
                    plan = mt.MttkrpPlan(variant, mode, tile_volume=nt if variant == mt.Variant.TILE else None)
                    if nt is not None:
                        m0 = pm.mem_zero(y.dims, rank, mode, nt, machine.s_f_bytes)
                        m0lm = pm.mem_zero_lm(y.dims, rank, mode, nt, machine.l, machine.s_f_bytes)
                        t0, t0lm = pm.predict_seconds(f, m0, machine), pm.predict_seconds(f, m0lm, machine)
                    else:
                        m0 = t0 = t0lm = None
                    for _ in range(warmup):
                        mt.run(y, m, plan)
                    best = math.inf
                    for rep in range(reps):
                        o = mt.run(y, m, plan)
                        t = o.stats.seconds
                        best = min(best, t)
                        rows.append({
                            "variant": variant.value, "mode": mode + 1, "rank": rank,
                            "tile_width": "" if width is None else width, "N_T": "" if nt is None else nt,
                            "rep": rep, "time_s": t, "gflops": pm.gflops(f, t),
                            "mops0": "" if m0 is None else pm.gbytes_per_s(m0, t),
                            "mopsInf": pm.gbytes_per_s(m_inf, t), "T0": "" if t0 is None else t0,
                            "T0LM": "" if t0lm is None else t0lm, "TInf": t_inf,
                            "atomic_updates": o.stats.atomic_updates, "rank_tile": o.stats.rank_tile,
                            "splits": o.stats.splits, "engine": mt.resolve_plan(plan, y.dims, rank)["engine"],
                        })
                    per_mode.append(pm.gflops(f, best))
                agg_rows.append({"variant": variant.value, "rank": rank, "tile_width": "" if width is None else width,
                                 "N_T": agg_nt, "gflops": statistics.fmean(per_mode), "best": 0})
    groups = {}
    for r in agg_rows:
        groups.setdefault((r["variant"], r["rank"]), []).append(r)
    for g in groups.values():
        max(g, key=lambda r: r["gflops"])["best"] = 1
    with open(out, "w", newline="", encoding="utf-8") as fh:
        w = csv.DictWriter(fh, fieldnames=COLUMNS + B200_COLUMNS)
        w.writeheader()
        w.writerows([{k: _cell(v) for k, v in r.items()} for r in rows])
    agg_out = agg_out or (os.path.splitext(out)[0] + ".agg.csv")
    with open(agg_out, "w", newline="", encoding="utf-8") as fh:
        w = csv.DictWriter(fh, fieldnames=AGG_COLUMNS)
        w.writeheader()
        w.writerows([{k: _cell(v) for k, v in r.items()} for r in agg_rows])
    return {"rows": len(rows), "out": out, "agg_out": agg_out}


def _ints(s: str, what: str) -> list:
    try:
        return [int(x) for x in s.split(",") if x.strip()]
    except ValueError as exc:
        raise ParameterError(f"bad {what} list {s!r}") from exc


# Named shapes of the reference CLI (cli.py:42-47): the paper's tearing and
# island tensors and their small twins.
PRESETS = {
    "tearing": (401, 201, 12, 501),
    "island": (129, 129, 129, 12, 39),
    "tearing-small": (51, 26, 12, 51),
    "island-small": (17, 17, 17, 12, 9),
}


def model_report(dims, ranks, modes=None, machine: pm.MachineSpec | None = None) -> dict:
    """The reference's `cpkern model` document (cli.py:470-545): work, traffic
    models and predicted times per rank, per variant (ELEM N_T = 1, SLICE
    N_T = N_S, TILE the Eq. 6 heuristic) and mode, the dense-GEMM footprint
    and capacity-only device counts -- no kernels run.  Same keys and values
    (tests/golden/model_cli.json); a "b200" entry adds the north-star
    roofline per mode (max(8 N / HBM, 2 N R (d-1) / FP64)) on the measured
    B200 denominators."""
    machine = machine or pm.bundled_machine("nvidia-b200")
    dims = tuple(int(x) for x in dims)
    d, n = len(dims), num_elements(dims)
    modes = list(range(d)) if modes is None else [int(k) for k in modes]
    width = mt.heuristic_tile_width(dims, machine) if d >= 2 else 1
    rows = []
    for rank in ranks:
        f = pm.flops(dims, rank)
        m_inf = pm.mem_infty(dims, rank, machine.s_f_bytes)
        inten = pm.intensity(f, m_inf)
        worst, worst_k = pm.mem_gemm_worst(dims, rank, machine.s_f_bytes)
        variants = {}
        for name, n_t in (("elem", lambda k: 1), ("slice", lambda k: n // dims[k]),
                          ("tile", lambda k: max(1, min(width ** (d - 1), n // dims[k])))):
            per = []
            for k in modes:
                m0 = pm.mem_zero(dims, rank, k, n_t(k), machine.s_f_bytes)
                m0lm = pm.mem_zero_lm(dims, rank, k, n_t(k), machine.l, machine.s_f_bytes)
                per.append({"mode": k + 1, "N_T": n_t(k), "m_zero": m0, "m_zero_lm": m0lm,
                            "T0": pm.predict_seconds(f, m0, machine), "T0LM": pm.predict_seconds(f, m0lm, machine)})
            variants[name] = {"T0_mean": statistics.fmean(r["T0"] for r in per),
                              "T0LM_mean": statistics.fmean(r["T0LM"] for r in per), "per_mode": per}
        rows.append({
            "rank": rank, "f": f, "matrix_free_bytes": m_inf, "matrix_free_gib": m_inf / pm.GIB,
            "intensity": inten, "compute_bound": pm.is_compute_bound(inten, machine),
            "TInf": pm.predict_seconds(f, m_inf, machine),
            "gemm_per_mode_bytes": [pm.mem_gemm(dims, rank, k, machine.s_f_bytes) for k in range(d)],
            "gemm_worst_bytes": worst, "gemm_worst_gib": worst / pm.GIB, "gemm_worst_mode": worst_k + 1,
            "matrix_free_pct_of_gemm": 100.0 * m_inf / worst,
            "devices_matrix_free": pm.device_count(m_inf, machine), "devices_gemm": pm.device_count(worst, machine),
            "variants": variants,
            "b200": {"roofline_seconds_per_mode": pm.roofline_seconds(dims, rank),
                     "algorithmic_flops_per_mode": pm.algorithmic_flops(dims, rank)},
        })
    return {"machine": machine.to_dict(), "dims": list(dims), "n_elements": n,
            "tensor_bytes": machine.s_f_bytes * n, "heuristic_tile_width": width,
            "heuristic_tile_volume": width ** (d - 1) if d >= 2 else 1, "modes": [k + 1 for k in modes],
            "ranks": rows}


def _print_model(doc: dict) -> None:
    m = doc["machine"]
    print(f"shape {tuple(doc['dims'])}  N={doc['n_elements']}  tensor "
          f"{doc['tensor_bytes'] / pm.GIB:.3f} GiB  machine {m['name']}")
    print(f"heuristic tile width {doc['heuristic_tile_width']} (N_T={doc['heuristic_tile_volume']})")
    for r in doc["ranks"]:
        print(f"\nrank {r['rank']}:")
        print(f"  f = {r['f']} flops   intensity {r['intensity']:.3f} flop/B"
              f"   {'compute' if r['compute_bound'] else 'memory'}-bound")
        print(f"  matrix-free footprint {r['matrix_free_bytes']} B = {r['matrix_free_gib']:.2f} GiB"
              f"  ({r['matrix_free_pct_of_gemm']:.2f}% of dense baseline)")
        print(f"  dense baseline worst mode {r['gemm_worst_mode']}: {r['gemm_worst_bytes']} B"
              f" = {r['gemm_worst_gib']:.2f} GiB")
        print(f"  devices needed (capacity lower bound): {r['devices_matrix_free']} matrix-free,"
              f" {r['devices_gemm']} dense")
        print(f"  T_inf {r['TInf']:.6f} s")
        for name, v in r["variants"].items():
            print(f"  {name:6s} T0 {v['T0_mean']:.6f} s   T0,LM {v['T0LM_mean']:.6f} s  (mean over modes)")
        print(f"  B200 north-star roofline {r['b200']['roofline_seconds_per_mode']:.6f} s per mode")


def main(argv=None) -> int:
    import argparse

    ap = argparse.ArgumentParser(prog="python -m paper_2510_14891_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sp = sub.add_parser("sweep", help="tile-width / variant sweep (cpkern sweep, cli.py:343-464)")
    sp.add_argument("--shape", help="comma-separated extents (synthetic Philox tensor)")
    sp.add_argument("--tensor", help="DTEN file instead of --shape")
    sp.add_argument("--ranks", default="32")
    sp.add_argument("--variants", default="tile")
    sp.add_argument("--tile-widths", default="")
    sp.add_argument("--modes", default="all", help="'all' or 1-based, comma-separated")
    sp.add_argument("--reps", type=int, default=3)
    sp.add_argument("--warmup", type=int, default=1)
    sp.add_argument("--machine", default="nvidia-b200", help="bundled spec name or JSON path")
    sp.add_argument("--seed", type=int, default=0)
    sp.add_argument("--out", default="sweep.csv")
    sp.add_argument("--agg-out", default=None)
    mp = sub.add_parser("model", help="analytic work/traffic/time numbers, no kernels (cpkern model, cli.py:470-545)")
    mp.add_argument("--tensor", help="read the shape from a DTEN header")
    mp.add_argument("--shape", help="comma-separated extents")
    mp.add_argument("--preset", choices=sorted(PRESETS), help="named shape (cli.py:42-47)")
    mp.add_argument("--ranks", default="32")
    mp.add_argument("--modes", default="all", help="'all' or 1-based, comma-separated")
    mp.add_argument("--machine", default="nvidia-b200", help="bundled spec name or JSON path")
    mp.add_argument("--json", action="store_true", help="machine-readable output")
    a = ap.parse_args(argv)
    if a.cmd == "model":
        if a.tensor:
            from .dtensor import read_dten_header

            dims = read_dten_header(a.tensor)
        elif a.preset:
            dims = PRESETS[a.preset]
        elif a.shape:
            dims = tuple(_ints(a.shape, "shape"))
        else:
            raise ParameterError("give --shape, --preset or --tensor")
        machine = (pm.bundled_machine(a.machine) if a.machine in pm.bundled_machine_names()
                   else pm.load_machine(a.machine))
        if a.modes.strip().lower() == "all":
            modes = None
        else:
            modes = [m - 1 for m in _ints(a.modes, "modes")]
            if any(not 0 <= k < len(dims) for k in modes):
                raise ParameterError(f"modes must lie in [1, {len(dims)}]")
        doc = model_report(dims, _ints(a.ranks, "ranks"), modes, machine)
        if a.json:
            print(json.dumps(doc, indent=2))
        else:
            _print_model(doc)
        return 0
    if a.tensor:
        from .dtensor import read_dten

        y = read_dten(a.tensor, device="cuda")
    else:
        if not a.shape:
            raise ParameterError("give --shape or --tensor")
        dims = tuple(_ints(a.shape, "shape"))
        y = DenseTensor(dims, np.random.Generator(np.random.Philox(a.seed)).random(num_elements(dims)))
    machine = pm.bundled_machine(a.machine) if a.machine in pm.bundled_machine_names() else pm.load_machine(a.machine)
    modes = None if a.modes.strip().lower() in ("", "all") else [m - 1 for m in _ints(a.modes, "modes")]
    res = sweep(y, _ints(a.ranks, "ranks"), a.variants.split(","), _ints(a.tile_widths, "tile widths") or None,
                modes, a.reps, a.warmup, machine, a.seed, a.out, a.agg_out)
    print(json.dumps(res))
    return 0
