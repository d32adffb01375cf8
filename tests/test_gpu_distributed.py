"""Order/ring-sharded wavelet transform on one GPU with virtual ranks.

The virtual exchanger runs P ranks stage by stage in one process (no rank ever
waits on another), so the partition, the exchange packing and the sharded
kernels are checked against the unsharded transform without more GPUs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1211_1680_b200 as sw
    from paper_1211_1680_b200 import distributed as D
    from paper_1211_1680_b200.device import WaveletTransform

    return torch, sw, D, WaveletTransform


@pytest.mark.parametrize("P", [1, 2, 3])
@pytest.mark.parametrize("real", [False, True])
@pytest.mark.parametrize("scheme", ["MW", "GL"])
def test_sharded_matches_unsharded(env, P, real, scheme):
    torch, sw, D, WT = env
    L = 96
    sch = getattr(sw.SamplingScheme, scheme)
    cfg = sw.TransformConfig(L, 2.0, 1, scheme=sch, multires=True)
    rng = np.random.default_rng(P + 10 * real)
    f = sw.gaussian_coeffs(L, rng, real_signal=real)
    x = torch.from_numpy(sw.sh_synthesis(f, sw.make_grid(sch, L)).values.copy()).cuda()
    if real:
        x = x.real.contiguous()
    x = x[None]
    ref = WT(cfg, batch=1, real=real)
    ref_maps = ref.analysis(x)
    ex = D.VirtualExchange(P)
    sh = D.ShardedWaveletTransform(cfg, ex, batch=1, real=real)
    rows = {r: x[:, slice(*sh.ring_block(L, r)), :].contiguous() for r in range(P)}
    out = sh.analysis(rows)
    for j, k in enumerate(sh.bands):
        full = torch.cat([out[r][j] for r in range(P)], dim=1)
        err = (full - ref_maps[j]).abs().max().item() / max(ref_maps[j].abs().max().item(), 1e-300)
        assert err <= 1e-12, (j, err)
    back = sh.synthesis(out)
    y = torch.cat([back[r] for r in range(P)], dim=1)
    assert (y - x).abs().max().item() <= 1e-10 * x.abs().max().item()


def test_partition_covers_everything(env):
    _, _, D, _ = env
    for L, P in [(64, 3), (2048, 8), (7, 4)]:
        owner = D.order_owner(L, P)
        assert set(owner.tolist()) <= set(range(P))
        cost = np.zeros(P)
        for m in range(L):
            cost[owner[m]] += L - m
        assert cost.max() / max(cost.mean(), 1) < 1.0 + 2.0 * P / L + 0.05
        blocks = D.ring_blocks(L, P)
        assert blocks[0][0] == 0 and blocks[-1][1] == L
        assert all(b[1] == c[0] for b, c in zip(blocks, blocks[1:]))
