"""Device jump-ahead of std::mt19937_64 (mg_mt64_jump / mg_mt64_split):
bit-exact against the sequential stream of the oracle, and the segmented
mt64 mode of the fused mini-render run identical to the sequential one."""
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2309_15676_b200 import api as a
    return a


@pytest.mark.parametrize("J", [1, 313, 123457, 10 ** 9 + 7])
def test_device_jump_matches_discard(api, oracle, J, record_property):
    from paper_2309_15676_b200 import _lib
    L = _lib.load()
    seeds = [(42, 7), (1, 0), (909, 3)]
    rng = api.Rng([L.mg_stream_seed(s, r) for s, r in seeds])
    t0 = time.time()
    rng.jump(J)
    torch.cuda.synchronize()
    record_property("jump_seconds_incl_poly", time.time() - t0)
    got = rng.raw(700).cpu().numpy()
    for i, (s, r) in enumerate(seeds):
        if J <= 200000:
            want = oracle.rng_draws(s, r, 1, J + 700)[J:]
            assert np.array_equal(got[i], want), i


def test_device_jump_composes(api):
    """jump(a) then jump(b) == jump(a + b) (covers distances too far to
    check against a sequential discard)."""
    from paper_2309_15676_b200 import _lib
    L = _lib.load()
    seed = L.mg_stream_seed(7, 1)
    a, b = api.Rng([seed]), api.Rng([seed])
    a.jump(10 ** 9 + 7)
    a.jump(123456789)
    b.jump(10 ** 9 + 7 + 123456789)
    assert np.array_equal(a.raw(1000).cpu().numpy(), b.raw(1000).cpu().numpy())


def test_jump_requires_block_boundary(api):
    rng = api.Rng.stream(3, 0)
    rng.raw(100)
    with pytest.raises(api.InvalidArgument):
        rng.jump(1000)
    rng.raw(212)  # back on a boundary (312 drawn)
    rng.jump(1000)


def test_split_segments_tile_the_stream(api, oracle):
    from paper_2309_15676_b200 import _lib
    L = _lib.load()
    G, seg, D = 5, 312 * 3, 4000
    rng = api.Rng.split(L.mg_stream_seed(11, 2), G, seg)
    first = rng.uniform(seg).cpu().numpy().reshape(-1)
    rng.jump(D - seg)
    second = rng.uniform(seg).cpu().numpy().reshape(-1)
    seq = oracle.rng_draws(11, 2, 2, D + G * seg)
    assert np.array_equal(first.view(np.uint64), seq[:G * seg].view(np.uint64))
    assert np.array_equal(second.view(np.uint64), seq[D:D + G * seg].view(np.uint64))


@pytest.mark.parametrize("P,spp", [(4096, 2), (1000, 3)])
def test_segmented_mt64_render_equals_sequential(api, P, spp):
    kw = dict(gen_seed=3, lr=0.02, seed=8, replicate=0, rng="mt64", dtype=torch.float64)
    seq = api.MiniRenderRun(P, spp, mt64_segments=1, **kw)
    seg = api.MiniRenderRun(P, spp, mt64_segments=7, **kw)
    assert seg.seg_len is not None and seq.seg_len is None
    for _ in range(6):
        seq.step()
        seg.step()
        assert torch.equal(seq.params, seg.params)
