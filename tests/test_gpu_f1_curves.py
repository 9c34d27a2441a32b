"""F1 loss-versus-iteration curves agree (north_star: "loss-versus-iteration
curves that agree"): each path-traced problem runs K optimisation
iterations on the device (sample-pair launch + fused meta update, fp64) and
the same loop runs on the CPU oracle (mgo_*_sample_pair + mgo_meta_update,
identical per-step arguments).  Per-iteration loss estimates agree to
1e-12; the parameter trajectory is bit-identical until the global step
norm enters (iteration 2: the device reduces ||delta pi||^2 as a tree, the
oracle sequentially) and within 1e-10 relative afterwards."""
import numpy as np
import pytest
import torch

from oracle_bind import Oracle
from paper_2309_15676_b200 import _abi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2309_15676_b200 import api
    return api


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


def oracle_loop(oracle, run, pair_fn, K):
    """Replays run (a QuadTextureRun-like object, freshly constructed) on the
    oracle: the FusedMetaUpdate argument sequence with device-side step norm
    (ssn_from_host = 0), ping-pong parameter buffers as in QuadTextureRun."""
    upd = run.upd
    n = upd.n
    st = {k: np.zeros(n) for k in ("m2_prop", "m2_diff", "mean", "var", "alpha_prev")}
    sc = _abi.fresh_scalars()
    params = run.params.cpu().numpy().copy()
    prev = params.copy()
    bfp = 1.0
    losses, traj = [], []
    for t in range(K):
        prop, diff, loss = pair_fn(params, prev, t)
        bfp *= upd.beta_f
        a = _abi.MetaUpdateArgs(
            meta=upd.meta, prop_coef=(1.0 - upd.beta_f) / (1.0 - bfp), beta_delta=upd.beta_delta,
            first_step=int(t == 0), diff_norm=upd.diff_norm,
            project=(2 if upd.project_hi is not None else int(upd.project_lo is not None)),
            ssn_from_host=0, proj_lo=0.0 if upd.project_lo is None else upd.project_lo,
            ssn_host=0.0, proj_hi=0.0 if upd.project_hi is None else upd.project_hi)
        new, _, rc = oracle.meta_update(a, st, prop, diff, params, sc)
        assert rc == 0
        prev, params = params, new
        losses.append(loss)
        traj.append(params.copy())
    return losses, traj


def device_loop(run, K):
    losses, traj = [], []
    for _ in range(K):
        run.step()
        losses.append(run.loss_estimate())
        traj.append(run.params.cpu().numpy().copy())
    return losses, traj


def check_curves(dev, ora):
    (dl, dt), (ol, ot) = dev, ora
    np.testing.assert_allclose(dl, ol, rtol=1e-12, atol=1e-14)
    for k, (a, b) in enumerate(zip(dt, ot)):
        if k < 2:
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), f"iteration {k}"
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-13, err_msg=f"iteration {k}")


def test_quad_loss_curve_matches_oracle(api, oracle):
    W, H, R, K = 20, 16, 4, 25
    prob = api.QuadTextureProblem(W, H, R, target_spp=16, dtype=torch.float64)
    run = api.QuadTextureRun(prob, "meta", lr=0.02)
    Le = np.array(list(prob.Le))
    tgt = prob.target_img.cpu().numpy()
    ora = oracle_loop(oracle, run, lambda p, q, t: oracle.quad_sample_pair(
        W, H, R, Le, tgt, p, q, run.key, t), K)
    check_curves(device_loop(run, K), ora)


def test_helix_loss_curve_matches_oracle(api, oracle):
    W, H, K = 24, 20, 20
    prob = api.HelixProblem(W, H, target_spp=8, dtype=torch.float64)
    run = api.HelixRun(prob, "meta", lr=0.02)
    sph = prob.spheres_host
    Le, env, ground = (np.array(list(x)) for x in (prob.Le, prob.env, prob.ground))
    tgt = prob.target_img.cpu().numpy()
    ora = oracle_loop(oracle, run, lambda p, q, t: oracle.helix_sample_pair(
        W, H, sph, Le, env, ground, tgt, p, q, run.key, t), K)
    check_curves(device_loop(run, K), ora)


@pytest.mark.parametrize("channels,nprop", [(4, 2), (5, 4)])
def test_mesh_loss_curve_matches_oracle(api, oracle, channels, nprop):
    W, H, R, K = 14, 10, 4, 12
    geo = api.mesh_scene_geometry((6, 8), (8, 10))
    view = api.mesh_scene_view(max_vertices=4)
    prob = api.MeshTextureProblem(W, H, R, max_vertices=4, target_spp=4, dtype=torch.float64,
                                  channels=channels, prop_paths=nprop, geometry=geo, view=view)
    run = api.MeshTextureRun(prob, "meta", lr=0.02)
    rec, obj, nobj = geo
    tgt = prob.target_img.cpu().numpy()
    ora = oracle_loop(oracle, run, lambda p, q, t: oracle.meshx_sample_pair(
        W, H, rec, obj, nobj, channels, R, view, tgt, p, q, run.key, t, nprop), K)
    check_curves(device_loop(run, K), ora)
