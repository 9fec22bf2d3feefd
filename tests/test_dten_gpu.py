"""DTEN ingest straight into device memory (cpk_dten_load_slab_f64): whole
tensors and slabs along every mode land bit-exactly, including across the
64 MiB staging-buffer boundary, and feed the MTTKRP / sharded driver."""

import numpy as np
import pytest
import torch

import paper_2510_14891_b200 as ck
from conftest import rng_for
from oracle import oracle
from paper_2510_14891_b200 import sharded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(6, 5, 4, 3), (7,), (33, 1, 20), (300, 200, 250)])
def test_slabs_of_every_mode_land_bit_exact(tmp_path, dims):
    y = rng_for(len(dims) + dims[0]).random(int(np.prod(dims)))
    path = tmp_path / "t.dten"
    ck.write_dten(path, ck.DenseTensor(dims, y))
    arr = y.reshape(dims, order="F")
    whole = ck.read_dten(path, device="cuda")
    assert whole.dims == dims and torch.equal(whole.data.cpu(), torch.from_numpy(y))
    rng = rng_for(3)
    for mode in range(len(dims)):
        for _ in range(3):
            lo = int(rng.integers(0, dims[mode]))
            hi = int(rng.integers(lo + 1, dims[mode] + 1))
            t = ck.read_dten(path, device="cuda", mode=mode, lo=lo, hi=hi)
            ref = np.take(arr, range(lo, hi), axis=mode).ravel(order="F")
            assert np.array_equal(t.data.cpu().numpy(), ref), (dims, mode, lo, hi)


def test_dten_errors(tmp_path):
    path = tmp_path / "t.dten"
    ck.write_dten(path, ck.DenseTensor((4, 3), np.arange(12.0)))
    with pytest.raises(ck.IndexRangeError):
        ck.read_dten(path, device="cuda", mode=2)
    with pytest.raises(ck.IndexRangeError):
        ck.read_dten(path, device="cuda", mode=0, lo=2, hi=9)
    with pytest.raises(ck.ParameterError):
        ck.read_dten(path, mode=0, lo=1, hi=2)  # host reads are whole-tensor


def test_sharded_slabs_from_dten_feed_the_mttkrp(tmp_path):
    """Each rank's DTEN slab (partition mode 0) gives the same local MTTKRP
    as the slab cut from the resident tensor; their mode-1 partials sum to
    the full G."""
    dims, rank, world = (40, 12, 9), 17, 3
    y = rng_for(77).random(int(np.prod(dims)))
    path = tmp_path / "y.dten"
    ck.write_dten(path, ck.DenseTensor(dims, y))
    part = sharded.partition_for(dims, world, mode=0)
    fs = [rng_for(80 + j).random((n, rank)) for j, n in enumerate(dims)]
    total = np.zeros((dims[1], rank))
    for r in range(world):
        slab = sharded.dten_slab(path, part, r, device="cuda")
        lo, hi = part.bounds(r)
        ref_slab = sharded.local_slab(ck.DenseTensor(dims, y), part, r)
        assert np.array_equal(slab.data.cpu().numpy(), np.asarray(ref_slab.data if not torch.is_tensor(ref_slab.data)
                                                                   else ref_slab.data.cpu()))
        local_f = [fs[0][lo:hi], fs[1], fs[2]]
        g = ck.run(slab, ck.KruskalTensor(np.ones(rank), local_f), ck.MttkrpPlan(ck.Variant.B200, 1)).matrix
        total += g.cpu().numpy() if torch.is_tensor(g) else g
    assert oracle.rel_err(total, oracle.mttkrp_ref(y, dims, 1, fs)) <= 1e-10
