"""ORACLE -- test infrastructure only.  Synthetic inputs.

* `philox_tensor` / `bench_factors` restate the reference CLI recipe
  (pkg/src/cpkern/cli.py:133-141): tensor = Generator(Philox(seed)).random(N)
  flat in first-mode-fastest order; factors = Generator(Philox(seed + 1)),
  rng.random((I_k, R)) in mode order, unit weights.
* `splitmix_uniform` is the CPU twin of the device generator
  cpk_fill_uniform_f64 (paper_2510_14891_b200/csrc/capi.cu), used for the
  BASELINE tensors too large to stage through the host (c4, c5):
      key  = mix64(seed * G + 0x632BE59BD9B4E019)
      x[i] = (mix64(key + (offset + i + 1) * G) >> 11) * 2^-53,  G = 0x9E3779B97F4A7C15
  with mix64 the splitmix64 finalizer.
"""

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def num_elements(dims):
    n = 1
    for x in dims:
        n *= int(x)
    return n


def philox_tensor(dims, seed=0):
    rng = np.random.Generator(np.random.Philox(seed))
    return rng.random(num_elements(dims))


def bench_factors(dims, rank, seed=0):
    rng = np.random.Generator(np.random.Philox(seed + 1))
    return [rng.random((int(i), rank)) for i in dims]


def _mix64(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix_key(seed):
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * _G + np.uint64(0x632BE59BD9B4E019)
        return _mix64(np.array(z, dtype=np.uint64))


def splitmix_uniform(n, seed=0, offset=0):
    with np.errstate(over="ignore"):
        key = splitmix_key(seed)
        c = np.arange(offset, offset + n, dtype=np.uint64) + np.uint64(1)
        z = _mix64(key + c * _G)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def splitmix_at(flat_idx, seed=0):
    """Values of the splitmix tensor at the given flat indices."""
    with np.errstate(over="ignore"):
        key = splitmix_key(seed)
        z = _mix64(key + (np.asarray(flat_idx).astype(np.uint64) + np.uint64(1)) * _G)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def slice_flat_indices(dims, mode, index):
    """Flat indices of slice `index` of mode `mode`, in the reference's
    in-slice order (first remaining mode fastest; dtensor.py:97-122)."""
    dims = [int(x) for x in dims]
    strides = np.cumprod([1] + dims[:-1]).astype(np.int64)
    axes = [np.arange(e, dtype=np.int64) * strides[m] for m, e in enumerate(dims) if m != mode]
    if not axes:
        return np.array([index * strides[mode]], dtype=np.int64)
    grids = np.meshgrid(*axes, indexing="ij")
    return (int(index) * int(strides[mode]) + sum(grids)).ravel(order="F")


def splitmix_slice(dims, mode, index, seed=0):
    """In-slice data of one mode-`mode` slice of the splitmix tensor."""
    return splitmix_at(slice_flat_indices(dims, mode, index), seed)
