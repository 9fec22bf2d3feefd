"""Optional float32 path (north star: <= 1e-4 relative Frobenius): the
tcgen05 kind::tf32 kernel with a 3xTF32 split, against the FP64 oracle on
the same (fp32-representable) inputs."""

import numpy as np
import pytest
import torch

import paper_2510_14891_b200 as ck
from conftest import rng_for
from oracle import oracle
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, f32_eligible, mttkrp_device

pytestmark = pytest.mark.gpu
TOL32 = 1e-4


def _inputs(dims, rank, seed, signed=False):
    y = rng_for(seed).random(int(np.prod(dims))).astype(np.float32)
    fs = [rng_for(seed + 1 + j).random((n, rank)).astype(np.float32) for j, n in enumerate(dims)]
    if signed:
        y = (2 * y - 1).astype(np.float32)
        fs = [(2 * a - 1).astype(np.float32) for a in fs]
    return y, fs


@pytest.mark.parametrize("dims", [(40, 36, 34), (64, 20, 12, 8), (128, 9), (8, 4, 6, 5, 3), (300, 44, 17)])
@pytest.mark.parametrize("rank", [1, 37, 128, 300])
def test_f32_every_mode_matches_oracle(dims, rank):
    y, fs = _inputs(dims, rank, sum(dims) + rank)
    dev = torch.device("cuda", 0)
    yd = torch.from_numpy(y).to(dev)
    fd = [torch.from_numpy(a).to(dev) for a in fs]
    assert f32_eligible(dims)
    for k in range(len(dims)):
        ref = oracle.mttkrp_ref(y.astype(np.float64), dims, k, [a.astype(np.float64) for a in fs])
        for splits in (0, 1, 3):
            g, _, _ = mttkrp_device(yd, dims, fd, k, None, MttkrpPlan(Variant.B200, k, splits=splits))
            assert g.dtype == torch.float32
            err = oracle.rel_err(g.double().cpu().numpy(), ref)
            assert err <= TOL32, (dims, rank, k, splits, err)


def test_f32_weights_signed_data_and_public_api():
    dims, rank = (48, 30, 20), 70
    y, fs = _inputs(dims, rank, 5, signed=True)
    lam = (rng_for(6).random(rank) + 0.5).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    fd = [torch.from_numpy(a).cuda() for a in fs]
    for k in range(3):
        ref = oracle.mttkrp_ref(y.astype(np.float64), dims, k, [a.astype(np.float64) for a in fs],
                                lam.astype(np.float64))
        got = ck.mttkrp(yd, fd, k, weights=torch.from_numpy(lam).cuda())
        assert got.dtype == torch.float32 and got.is_cuda
        assert oracle.rel_err(got.double().cpu().numpy(), ref) <= TOL32, k


def test_f32_ineligible_shapes_run_on_the_fp64_kernel():
    """I_0 % 4 != 0 (TMA strides): float64 copies through the FP64 kernel."""
    dims, rank = (41, 7, 9), 5
    y, fs = _inputs(dims, rank, 9)
    yd = torch.from_numpy(y).cuda()
    fd = [torch.from_numpy(a).cuda() for a in fs]
    assert not f32_eligible(dims)
    for k in range(3):
        got = ck.mttkrp(yd, fd, k)
        ref = oracle.mttkrp_ref(y.astype(np.float64), dims, k, [a.astype(np.float64) for a in fs])
        assert got.dtype == torch.float32 and oracle.rel_err(got.double().cpu().numpy(), ref) <= TOL32
