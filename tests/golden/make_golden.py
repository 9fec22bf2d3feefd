"""Generate the golden fixtures by running the REFERENCE implementation itself.

Run in a container where /root/reference is present (it is not on the GPU
box).  The reference is imported read-only from /root/reference/pkg/src with
its numba cache redirected; nothing from it is copied into this repo -- only
its outputs on seeded inputs are stored.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Fixtures (numpy .npz, float64):
  small.npz  -- CASES of test_mttkrp.py (kernel parity, all modes) and the
                50-instance acceptance family (test_acceptance.py:52-62):
                inputs + G from cpkern.mttkrp_reference (canonical order)
  c1.npz     -- BASELINE config 1 (64^3, R=16): G for all modes (reference)
  c2.npz     -- config 2 (512^3, R=64): G for all modes (cpkern.mttkrp_gemm,
                which the reference's tests pin to mttkrp_reference at 1e-12),
                plus 8 rows per mode from mttkrp_reference on single-slice
                sub-tensors
  c3.npz     -- config 3 (128^4, R=256): G for all modes (mttkrp_gemm)
  dten/      -- DTEN v1 files written by cpkern.dtensor.write_dten (a 4-way
                Philox tensor and a 1-way one) and the reference's verdict
                (shape, or the FormatError message) on malformed variants
  model.json -- cpkern.perfmodel traffic models / predicted times (sweep columns)
  model_cli.json -- `cpkern model --json` documents (cli.py:470-545) for
                presets / shapes / machines / ranks / modes
  step.npz   -- one CP-ALS mode update from identical factors (SURVEY.md 8(c)
                plan (i)): the CP-ALS init factors (Philox(seed)), then for
                each mode G_k (unit-weight MTTKRP), Gamma_k, the reference's
                _solve_normal and column normalization (cpals.py:122-140);
                config 3 (modes 0 and 3) and a rank-512 3-way case (all
                modes) that takes the R > 256 solve path
  als.npz    -- cp_als fit trajectories: the planted suites of test_cpals.py
                (REFERENCE and GEMM plans), and config 3 for 10 sweeps (GEMM)
Inputs for c1-c3 follow the reference CLI recipe (cli.py:133-141):
tensor Philox(0).random(N), factors Philox(1).random((I_k, R)) per mode.
"""

import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("NUMBA_NUM_THREADS", "8")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import cpkern as ck  # noqa: E402
from cpkern.mttkrp import MttkrpPlan, Variant  # noqa: E402

OUT = Path(__file__).resolve().parent
CASES = [((5, 4, 6), 3), ((3, 8, 2, 5), 4), ((6, 6), 2), ((2, 3, 2, 2, 3), 5)]


def rng_for(seed):
    return np.random.Generator(np.random.Philox(seed))


def random_tensor(dims, seed):
    r = rng_for(seed)
    return ck.DenseTensor(dims, r.random(int(np.prod(dims))))


def random_model(dims, rank, seed):
    r = rng_for(seed + 1009)
    lam = r.random(rank) + 0.5
    return ck.KruskalTensor(lam, [r.random((i, rank)) for i in dims])


def seeded_instance(i):
    rng = np.random.Generator(np.random.Philox(1000 + i))
    d = 3 + i % 3
    dims = tuple(int(x) for x in rng.integers(2, 9, size=d))
    rank = (1, 3, 8, 32)[i % 4]
    y = ck.DenseTensor(dims, rng.random(int(np.prod(dims))))
    factors = [rng.random((n, rank)) for n in dims]
    weights = rng.random(rank) + 0.5
    return y, ck.KruskalTensor(weights, factors)


def pack_instance(store, key, y, m):
    store[f"{key}/dims"] = np.asarray(y.dims, dtype=np.int64)
    store[f"{key}/data"] = y.data
    store[f"{key}/lam"] = m.weights
    for j, a in enumerate(m.factors):
        store[f"{key}/A{j}"] = a
    for k in range(y.ndim):
        store[f"{key}/G{k}"] = ck.mttkrp_reference(y, m, k).matrix


def make_small():
    store = {}
    for c, (dims, rank) in enumerate(CASES):
        pack_instance(store, f"case{c}", random_tensor(dims, 15), random_model(dims, rank, 16))
    for i in range(50):
        y, m = seeded_instance(i)
        pack_instance(store, f"inst{i}", y, m)
    np.savez_compressed(OUT / "small.npz", **store)


def config_inputs(dims, rank, seed=0):
    y = ck.DenseTensor(dims, rng_for(seed).random(int(np.prod(dims))))
    r = rng_for(seed + 1)
    m = ck.KruskalTensor(np.ones(rank), [r.random((i, rank)) for i in dims], validate=False)
    return y, m


def sampled_rows_reference(y, m, k, rows):
    """G[rows] through the reference's own serial kernel on single-slice sub-tensors."""
    arr = y.to_ndarray()
    out = []
    for n in rows:
        sub = np.take(arr, [n], axis=k)
        ys = ck.DenseTensor.from_ndarray(sub)
        fs = [a if j != k else a[n:n + 1] for j, a in enumerate(m.factors)]
        ms = ck.KruskalTensor(m.weights, fs, validate=False)
        out.append(ck.mttkrp_reference(ys, ms, k).matrix[0])
    return np.asarray(out)


def make_config(name, dims, rank, use_gemm, sample_rows=0):
    t0 = time.time()
    y, m = config_inputs(dims, rank)
    store = {"dims": np.asarray(dims, dtype=np.int64), "rank": np.int64(rank)}
    for k in range(len(dims)):
        g = (ck.mttkrp_gemm(y, m, k) if use_gemm else ck.mttkrp_reference(y, m, k)).matrix
        store[f"G{k}"] = g
        if sample_rows:
            rows = np.linspace(0, dims[k] - 1, sample_rows).astype(np.int64)
            store[f"rows{k}"] = rows
            store[f"Grows{k}"] = sampled_rows_reference(y, m, k, rows)
    np.savez_compressed(OUT / f"{name}.npz", **store)
    print(f"{name}: {time.time() - t0:.1f} s", flush=True)


def make_step():
    """One mode update per mode, from the same (init) factors, through the
    reference's own gram / Gamma loop / _solve_normal / normalization."""
    from cpkern.cpals import _solve_normal
    from cpkern.kruskal import gram

    t0 = time.time()
    store = {}
    for name, dims, rank, modes in (("c3", (128, 128, 128, 128), 256, (0, 3)), ("r512", (64, 56, 48), 512, (0, 1, 2))):
        y = ck.DenseTensor(dims, rng_for(0).random(int(np.prod(dims))))
        rng = np.random.Generator(np.random.Philox(0))  # cp_als init, seed 0 (cpals.py:108-109)
        factors = [rng.random((i, rank)) for i in dims]
        grams = [gram(a) for a in factors]
        unit = np.ones(rank)
        store[f"{name}/dims"] = np.asarray(dims, dtype=np.int64)
        for k in modes:
            g = ck.mttkrp_gemm(y, ck.KruskalTensor(unit, factors, validate=False), k).matrix
            gamma = np.ones((rank, rank))
            for m in range(len(dims)):
                if m != k:
                    gamma *= grams[m]
            a_hat = _solve_normal(gamma, g.copy())
            nrm = np.linalg.norm(a_hat, axis=0)
            nz = nrm > 0
            a_hat[:, nz] /= nrm[nz]
            store[f"{name}/G{k}"] = g
            store[f"{name}/A{k}"] = np.ascontiguousarray(a_hat)
            store[f"{name}/lam{k}"] = np.where(nz, nrm, 0.0)
            store[f"{name}/cond{k}"] = np.float64(np.linalg.cond(gamma))
    np.savez_compressed(OUT / "step.npz", **store)
    print(f"step: {time.time() - t0:.1f} s", flush=True)


def planted(dims, rank, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    truth = ck.KruskalTensor(np.ones(rank), [rng.standard_normal((i, rank)) for i in dims])
    return truth.full()


def make_als():
    store = {}
    for dims, rank, tseed, sweeps in [((6, 7, 8), 3, 101, 14), ((4, 5, 6, 7), 2, 33, 12), ((5, 5, 5), 2, 42, 20)]:
        y = planted(dims, rank, tseed)
        key = f"planted_{'x'.join(map(str, dims))}_r{rank}"
        store[f"{key}/data"] = y.data
        store[f"{key}/dims"] = np.asarray(dims, dtype=np.int64)
        for pname, plan in [("reference", MttkrpPlan(Variant.REFERENCE, 0)), ("gemm", MttkrpPlan(Variant.GEMM, 0))]:
            model, tr = ck.cp_als(y, ck.AlsConfig(rank=rank, tol=0.0, max_iters=sweeps, seed=0, plan=plan))
            store[f"{key}/fits_{pname}"] = np.asarray(tr.fits)
            store[f"{key}/lam_{pname}"] = model.weights
    # random (non-planted) tensor: fit identity regime (test_cpals.py:46-55)
    y = ck.DenseTensor((7, 6, 5), rng_for(5).random(210))
    model, tr = ck.cp_als(y, ck.AlsConfig(rank=3, tol=0.0, max_iters=20, seed=2))
    store["rand765/data"] = y.data
    store["rand765/fits"] = np.asarray(tr.fits)
    store["rand765/lam"] = model.weights
    for j, a in enumerate(model.factors):
        store[f"rand765/A{j}"] = a
    # config 3: 10 sweeps, GEMM plan (the fast CPU path)
    t0 = time.time()
    y, _ = config_inputs((128, 128, 128, 128), 256)
    model, tr = ck.cp_als(y, ck.AlsConfig(rank=256, tol=0.0, max_iters=10, seed=0,
                                          plan=MttkrpPlan(Variant.GEMM, 0)))
    store["c3/fits"] = np.asarray(tr.fits)
    store["c3/lam"] = model.weights
    store["c3/mttkrp_seconds"] = np.asarray(tr.mttkrp_seconds)
    print(f"c3 cp_als: {time.time() - t0:.1f} s", flush=True)
    np.savez_compressed(OUT / "als.npz", **store)


def make_model():
    """Traffic-model values from cpkern.perfmodel on a few shapes/specs."""
    import json

    from cpkern import perfmodel as pmr

    cases = []
    for dims, rank, mode, nt in [((401, 201, 12, 501), 32, 0, 256), ((129, 129, 129, 12, 39), 32, 2, 4096),
                                 ((1024, 1024, 1024), 2000, 1, 131044), ((64, 64, 64), 16, 2, 1)]:
        for mach in ("nvidia-h100", "intel-8480p"):
            ms = pmr.bundled_machine(mach)
            f = pmr.flops(dims, rank)
            m0 = pmr.mem_zero(dims, rank, mode, nt)
            m0lm = pmr.mem_zero_lm(dims, rank, mode, nt, ms.l)
            minf = pmr.mem_infty(dims, rank)
            cases.append({"dims": list(dims), "rank": rank, "mode": mode, "nt": nt, "machine": mach, "f": f,
                          "mem_zero": m0, "mem_zero_lm": m0lm, "mem_infty": minf,
                          "T0": pmr.predict_seconds(f, m0, ms), "T0LM": pmr.predict_seconds(f, m0lm, ms),
                          "TInf": pmr.predict_seconds(f, minf, ms), "gbps": pmr.gbytes_per_s(m0, 0.37)})
    (OUT / "model.json").write_text(json.dumps(cases, indent=1) + "\n")


MODEL_CLI_CASES = [
    ["--preset", "tearing", "--ranks", "16,32", "--machine", "nvidia-h100"],
    ["--preset", "island", "--ranks", "32", "--modes", "1,3,5", "--machine", "intel-8480p"],
    ["--shape", "1024,1024,1024", "--ranks", "2000", "--machine", "nvidia-h100"],
    ["--shape", "4096,2048,2048", "--ranks", "512", "--machine", "intel-8480p"],
    ["--shape", "64,64,64", "--ranks", "1,16", "--machine", "nvidia-h100"],
    ["--shape", "7", "--ranks", "3", "--machine", "intel-8480p"],
]


def make_model_cli():
    """`cpkern model --json` (the reference CLI itself) on MODEL_CLI_CASES."""
    import contextlib
    import io
    import json

    from cpkern import cli

    docs = []
    for args in MODEL_CLI_CASES:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert cli.main(["model", *args, "--json"]) == 0
        docs.append({"args": args, "doc": json.loads(buf.getvalue())})
    (OUT / "model_cli.json").write_text(json.dumps(docs, indent=1) + "\n")


def make_dten():
    import json

    from cpkern.dtensor import read_dten, read_dten_header, write_dten
    from cpkern.errors import FormatError

    d = OUT / "dten"
    d.mkdir(exist_ok=True)
    good = {"t4.dten": (6, 5, 4, 3), "t1.dten": (7,)}
    for name, dims in good.items():
        write_dten(d / name, ck.DenseTensor(dims, random_tensor(dims, 5).data))
    raw = (d / "t4.dten").read_bytes()
    bad = {
        "bad_magic.dten": b"DTEX" + raw[4:],
        "bad_version.dten": raw[:4] + (2).to_bytes(4, "little") + raw[8:],
        "zero_modes.dten": raw[:8] + (0).to_bytes(4, "little") + raw[12:],
        "bad_etype.dten": raw[:12 + 32] + (2).to_bytes(4, "little") + raw[12 + 36:],
        "zero_extent.dten": raw[:12] + (0).to_bytes(8, "little") + raw[20:],
        "truncated_header.dten": raw[:10],
        "truncated_dims.dten": raw[:30],
        "short_payload.dten": raw[:-8],
        "long_payload.dten": raw + bytes(8),
    }
    verdict = {}
    for name, blob in bad.items():
        (d / name).write_bytes(blob)
    for name in list(good) + list(bad):
        try:
            shape = read_dten_header(d / name)
            read_dten(d / name)
            verdict[name] = {"dims": list(shape)}
        except FormatError as exc:
            verdict[name] = {"error": str(exc)}
    (d / "verdict.json").write_text(json.dumps(verdict, indent=1) + "\n")


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "c1", "c2", "c3", "als", "dten", "model", "model_cli", "step"]
    if "model" in which:
        make_model()
    if "model_cli" in which:
        make_model_cli()
    if "dten" in which:
        make_dten()
    if "small" in which:
        make_small()
    if "c1" in which:
        make_config("c1", (64, 64, 64), 16, use_gemm=False)
    if "c2" in which:
        make_config("c2", (512, 512, 512), 64, use_gemm=True, sample_rows=4)
    if "c3" in which:
        make_config("c3", (128, 128, 128, 128), 256, use_gemm=True)
    if "als" in which:
        make_als()
    if "step" in which:
        make_step()
    print("done")
