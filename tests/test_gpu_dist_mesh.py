"""Image-tile sharding of a shared-parameter renderer through the real
multi-GPU plumbing (dist.tile_rows + SharedParamStep over NCCL, and
SharedParamStepP2P over torch symmetric memory), run as a 1-rank NCCL group
on the single GPU of this environment: the sharded loop reproduces the
single-process MeshTextureRun (bit-identical through SharedParamStep; the
peer-memory kernel within reduction-order tolerance).  Multi-rank host logic
is covered by tests/test_dist_gloo.py; exact tile sums by
tests/test_gpu_mesh.py."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def _problem(api):
    geo = api.mesh_scene_geometry((6, 8), (8, 10))
    return api.MeshTextureProblem(24, 18, 8, max_vertices=4, target_spp=4, dtype=torch.float32,
                                  geometry=geo, view=api.mesh_scene_view(max_vertices=4))


def test_tile_sharded_shared_param_step_matches_single_process(pg):
    from paper_2309_15676_b200 import api
    from paper_2309_15676_b200.dist import SharedParamStep, tile_rows
    K = 8
    prob = _problem(api)
    ref = api.MeshTextureRun(prob, "meta", lr=0.02, fused=False)
    ref_traj = []
    for _ in range(K):
        ref.step()
        ref_traj.append(ref.params.clone())
    rank, world = pg.get_rank(), pg.get_world_size()
    n = prob.dim()
    upd = api.FusedMetaUpdate(n // world, dtype=prob.dtype, lr=0.02, project_lo=0.0,
                              project_hi=1.0)
    step = SharedParamStep(upd, n)
    params = prob.initial_params()
    prev = params.clone()
    key = ref.key
    for t in range(K):
        pair = prob.sample_pair(params, prev, t, key, rows=tile_rows(prob.H, rank, world))
        new = torch.empty_like(params)
        step(pair.prop, pair.diff, params, new)
        prev, params = params, new
        assert torch.equal(params, ref_traj[t]), t


def test_peer_memory_shared_step_tracks_single_process(pg):
    from paper_2309_15676_b200 import api
    from paper_2309_15676_b200.dist import SharedParamStepP2P, tile_rows
    K = 8
    prob = _problem(api)
    ref = api.MeshTextureRun(prob, "meta", lr=0.02, fused=False)
    ref_traj = []
    for _ in range(K):
        ref.step()
        ref_traj.append(ref.params.clone())
    rank, world = pg.get_rank(), pg.get_world_size()
    n = prob.dim()
    step = SharedParamStepP2P(n, dtype=prob.dtype, lr=0.02, project_lo=0.0, project_hi=1.0,
                              init=0.5)
    prev = prob.initial_params()
    for t in range(K):
        pair = prob.sample_pair(step.params, prev, t, ref.key,
                                rows=tile_rows(prob.H, rank, world))
        step.prop.copy_(pair.prop)
        step.diff.copy_(pair.diff)
        prev = step.params.clone()
        step()
        got = step.params.cpu().numpy()
        want = ref_traj[t].cpu().numpy()
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6, err_msg=str(t))


@pytest.mark.parametrize("world", [2, 3])
def test_fused_scatter_reduce_scatter_emulated_ranks(world):
    """mg_meshscene_sample_pair_sharded with `world` ranks emulated on this
    GPU (distinct accumulator shards; each rank's launch renders its own rows
    and adds into every owner's shard; no launch waits on another): the
    finalized shards concatenate to the single-process pair bit for bit."""
    from paper_2309_15676_b200 import api
    from paper_2309_15676_b200.dist import tile_rows
    geo = api.mesh_scene_geometry((6, 8), (8, 10))
    prob = api.MeshTextureProblem(20, 15, 6, max_vertices=4, target_spp=2, dtype=torch.float64,
                                  channels=5, prop_paths=3, geometry=geo,
                                  view=api.mesh_scene_view(max_vertices=4))
    n = prob.dim()
    assert n % world == 0
    S = n // world
    rs = np.random.RandomState(world)
    now = torch.tensor(rs.uniform(0.2, 0.8, n), device="cuda")
    prev = (now - 0.01).clamp(0, 1)
    full = prob.sample_pair(now, prev, 5, key=21)
    full = (full.prop.clone(), full.diff.clone())
    accs = [torch.zeros(2 * S, dtype=torch.int64, device="cuda") for _ in range(world)]
    ptrs = [a.data_ptr() for a in accs]
    for r in range(world):
        prob.sample_pair_sharded(now, prev, 5, 21, tile_rows(prob.H, r, world), ptrs, S)
    props, diffs = [], []
    for r in range(world):
        p = torch.empty(S, dtype=torch.float64, device="cuda")
        d = torch.empty_like(p)
        api.fixed_finalize(accs[r], p, d)
        props.append(p)
        diffs.append(d)
        assert int(torch.count_nonzero(accs[r])) == 0
    assert torch.equal(torch.cat(props), full[0])
    assert torch.equal(torch.cat(diffs), full[1])


def test_tiled_render_step_p2p_matches_single_process(pg):
    """The symmetric-memory TiledRenderStepP2P (1-rank group here) follows the
    single-process MeshTextureRun trajectory bit for bit."""
    from paper_2309_15676_b200 import api
    from paper_2309_15676_b200.dist import TiledRenderStepP2P
    prob = _problem(api)
    ref = api.MeshTextureRun(prob, "meta", lr=0.02, fused=False)
    step = TiledRenderStepP2P(prob, lr=0.02)
    for t in range(6):
        ref.step()
        step.step()
        assert torch.equal(step.params, ref.params), t
