"""F1 slice: path-traced gradient samples of the textured
quad (BASELINE.json configs[0]) against the repo's own CPU oracle
(oracle/metagrad_oracle.c mgo_quad_*; the reference has no renderer).

  * fp64: render and gradient sample pairs BIT-EXACT (only IEEE + - * / sqrt,
    Philox-addressed samples, fixed-point adjoint accumulation);
  * fp32: <= 1e-5 of the gradient scale;
  * the finite-difference sample is unbiased for the change of the
    proportional sample's expectation (z-test over 4000 iterations);
  * the meta-estimator and Adam both fit the target texture.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

LE = (8.0, 7.0, 6.0)


@pytest.fixture(scope="module")
def api():
    from paper_2309_15676_b200 import api as a
    return a


def host(t):
    return t.detach().double().cpu().numpy()


def bits_equal(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_quad_render_and_target_bit_exact(api, oracle):
    prob = api.QuadTextureProblem(64, 64, 32, LE, target_spp=64)
    from paper_2309_15676_b200 import _lib
    key = _lib.load().mg_mix64(1)
    ref = oracle.quad_render(64, 64, 32, host(prob.target_tex), LE, 64, key, 7)
    assert bits_equal(host(prob.target_img), ref)
    assert (ref >= 0).all() and ref.max() > 0.05


@pytest.mark.parametrize("W,H,R", [(64, 64, 32), (96, 80, 16), (256, 256, 64)])
def test_quad_sample_pair_bit_exact_fp64(api, oracle, W, H, R):
    prob = api.QuadTextureProblem(W, H, R, LE, target_spp=16)
    rs = np.random.RandomState(R)
    now = rs.uniform(0, 1, 3 * R * R)
    prev = now - 0.01 * rs.uniform(0, 1, now.size)
    tnow = torch.tensor(now, device="cuda")
    tprev = torch.tensor(prev, device="cuda")
    for it in (0, 5):
        pair = prob.sample_pair(tnow, tprev, it, key=12345)
        p, d, loss = oracle.quad_sample_pair(W, H, R, LE, host(prob.target_img), now, prev,
                                             12345, it)
        assert bits_equal(host(pair.prop), p), it
        assert bits_equal(host(pair.diff), d), it
        assert float(prob.loss_buf[0]) == pytest.approx(loss, rel=1e-12)
    same = prob.sample_pair(tnow, tnow, 3, key=1)
    assert (host(same.diff) == 0).all()


def test_quad_sample_pair_fp32(api, oracle):
    W, H, R = 64, 64, 32
    prob = api.QuadTextureProblem(W, H, R, LE, target_spp=16, dtype=torch.float32)
    rs = np.random.RandomState(0)
    now = rs.uniform(0, 1, 3 * R * R).astype(np.float32)
    prev = (now - 0.01 * rs.uniform(0, 1, now.size)).astype(np.float32)
    pair = prob.sample_pair(torch.tensor(now, device="cuda"), torch.tensor(prev, device="cuda"),
                            2, key=99)
    p, d, _ = oracle.quad_sample_pair(W, H, R, LE, host(prob.target_img), now, prev, 99, 2)
    scale = np.abs(p).max()
    assert np.abs(host(pair.prop) - p).max() < 1e-5 * scale
    assert np.abs(host(pair.diff) - d).max() < 1e-5 * max(np.abs(d).max(), 1e-30) + 1e-9


def test_quad_fd_sample_is_unbiased(api):
    """E[diff(theta_t, theta_{t-1})] = E[prop(theta_t)] - E[prop(theta_{t-1})]:
    the common-random-number difference estimates the gradient change."""
    W, H, R, K = 32, 32, 8, 4000
    prob = api.QuadTextureProblem(W, H, R, LE, target_spp=256)
    rs = np.random.RandomState(3)
    a = torch.tensor(rs.uniform(0.2, 0.8, 3 * R * R), device="cuda")
    b = a - torch.tensor(0.05 * rs.uniform(0.5, 1.0, 3 * R * R), device="cuda")
    d_sum = torch.zeros_like(a)
    d_sq = torch.zeros_like(a)
    pa = torch.zeros_like(a)
    pa_sq = torch.zeros_like(a)
    pb = torch.zeros_like(a)
    pb_sq = torch.zeros_like(a)
    for it in range(K):
        x = prob.sample_pair(a, b, it, key=5)
        d_sum += x.diff
        d_sq += x.diff ** 2
        ya = prob.sample_pair(a, a, it, key=6).prop  # independent draws
        yb = prob.sample_pair(b, b, it, key=7).prop
        pa += ya
        pa_sq += ya ** 2
        pb += yb
        pb_sq += yb ** 2
    mean = lambda s: host(s) / K  # noqa: E731
    var = lambda s, q: (host(q) / K - (host(s) / K) ** 2) / K  # noqa: E731 (variance of the mean)
    md = mean(d_sum)
    me = mean(pa) - mean(pb)
    se = np.sqrt(var(d_sum, d_sq) + var(pa, pa_sq) + var(pb, pb_sq)) + 1e-300
    z = np.abs(md - me) / se
    assert np.mean(z > 3.0) < 0.02, np.mean(z > 3.0)
    assert z.max() < 6.0, z.max()
    # and the FD sample has far lower variance than the difference of props
    assert np.median(var(d_sum, d_sq) / (var(pa, pa_sq) + var(pb, pb_sq))) < 0.2


@pytest.mark.parametrize("opt,lr", [("meta", 0.01), ("adam", 0.01)])
def test_quad_config1_optimisation_fits_target(api, opt, lr, record_property):
    """configs[0]: 64x64, 32x32 RGB texture from seed 0 towards seed 1, 200
    iterations, lr 0.01 — the texture error must drop."""
    prob = api.QuadTextureProblem(64, 64, 32, LE, target_spp=1024)
    run = api.QuadTextureRun(prob, optimizer=opt, lr=lr, seed=0)
    e0 = run.texture_error()
    losses = []
    for _ in range(200):
        run.step()
        losses.append(run.loss_estimate())
    e1 = run.texture_error()
    record_property("texture_error", [e0, e1])
    record_property("loss_first_last", [losses[0], float(np.mean(losses[-20:]))])
    assert e1 < 0.6 * e0
    assert np.mean(losses[-20:]) < 0.2 * losses[0]


@pytest.mark.parametrize("tiles", [2, 3])
def test_tile_sharded_gradients_sum_exactly(api, tiles):
    """Image tiles shard across GPUs: the partial gradient
    pairs of disjoint row tiles — computed as separate launches here, one
    per emulated rank — sum EXACTLY (fixed-point accumulation) to the
    unsharded pair, so the all-reduce/reduce-scatter of the partials gives
    a result independent of the rank count."""
    W, H, R = 64, 64, 32
    prob = api.QuadTextureProblem(W, H, R, LE, target_spp=16)
    rs = np.random.RandomState(1)
    now = torch.tensor(rs.uniform(0, 1, 3 * R * R), device="cuda")
    prev = now - 0.01
    full = prob.sample_pair(now, prev, 4, key=3)
    full = (full.prop.clone(), full.diff.clone())
    from paper_2309_15676_b200.dist import tile_rows
    sp = torch.zeros_like(now)
    sd = torch.zeros_like(now)
    for r in range(tiles):
        part = prob.sample_pair(now, prev, 4, key=3, rows=tile_rows(H, r, tiles))
        sp += part.prop
        sd += part.diff
    assert torch.equal(sp, full[0]) and torch.equal(sd, full[1])


@pytest.mark.parametrize("kind,dtype", [("quad", torch.float32), ("quad", torch.float64),
                                        ("helix", torch.float32), ("mesh", torch.float32),
                                        ("meshx", torch.float32)])
def test_graph_replayed_run_is_bit_identical(api, kind, dtype):
    """run(k, graph=True) replays one captured two-step block (device
    iteration counter, device Moment2 coefficient): the parameters, the
    optimiser state and the loss equal the eager loop's bit for bit, over
    an odd count (the last step eager) and a second run() call."""
    side = torch.cuda.Stream()
    ctx = api.Context(0, stream=side)

    def make():
        if kind == "quad":
            prob = api.QuadTextureProblem(32, 32, 8, target_spp=16, dtype=dtype, ctx=ctx)
            return prob, api.QuadTextureRun(prob, optimizer="meta", lr=0.01)
        if kind == "helix":
            prob = api.HelixProblem(32, 24, target_spp=4, dtype=dtype, ctx=ctx)
            return prob, api.HelixRun(prob, optimizer="meta", lr=0.01)
        # mesh wavefront (28 launches per iteration, prev-copy reuse on);
        # meshx: 5 channels, 4 proportional paths (the configs[4] form)
        ch, nprop = (4, 2) if kind == "mesh" else (5, 4)
        prob = api.MeshTextureProblem(32, 24, 8, (8, 12), (10, 12), max_vertices=4, target_spp=4,
                                      dtype=dtype, ctx=ctx, channels=ch, prop_paths=nprop)
        return prob, api.MeshTextureRun(prob, "meta", lr=0.01)

    with torch.cuda.stream(side):
        pe, re_ = make()
        re_.run(13)
        re_.run(6)
        pg, rg = make()
        rg.run(13, graph=True)
        rg.run(6, graph=True)
        torch.cuda.synchronize()
    assert re_.t == rg.t == 19
    assert torch.equal(re_.params, rg.params) and torch.equal(re_.prev, rg.prev)
    for a in ("m2_prop", "m2_diff", "mean", "var", "alpha_prev"):
        assert torch.equal(getattr(re_.upd, a), getattr(rg.upd, a)), a
    assert pe.loss_buf.item() == pg.loss_buf.item()
    se, sg = re_.upd.scalars(), rg.upd.scalars()
    assert (se.ssn, se.diff_count, se.prop_decay_pow) == (sg.ssn, sg.diff_count, sg.prop_decay_pow)
    assert se.prop_decay_pow == re_.upd.beta_f_pow  # device chain == host chain


@pytest.mark.parametrize("kind", ["quad", "mesh"])
def test_graph_run_after_odd_eager_tail_realigns(api, kind):
    """A graph captured with pi_t in buffer A must not be replayed while
    pi_t sits in buffer B (after a trailing eager step, or a user step()):
    run(13, graph) -> run(5, graph) -> step() -> run(4, graph) equals 23
    eager steps bit for bit.  The calls are made OUTSIDE any stream context
    (the replays must still be ordered on ctx.stream)."""
    side = torch.cuda.Stream()
    ctx = api.Context(0, stream=side)

    def make():
        if kind == "quad":
            prob = api.QuadTextureProblem(32, 32, 8, target_spp=16, dtype=torch.float32, ctx=ctx)
            return prob, api.QuadTextureRun(prob, optimizer="meta", lr=0.01)
        prob = api.MeshTextureProblem(32, 24, 8, (8, 12), (10, 12), max_vertices=4, target_spp=4,
                                      dtype=torch.float32, ctx=ctx, channels=4, prop_paths=2)
        return prob, api.MeshTextureRun(prob, "meta", lr=0.01)

    with torch.cuda.stream(side):
        pe, re_ = make()
        re_.run(23)
        pg, rg = make()
    torch.cuda.synchronize()
    rg.run(13, graph=True)
    rg.run(5, graph=True)
    with torch.cuda.stream(side):
        rg.step()
    rg.run(4, graph=True)
    torch.cuda.synchronize()
    assert re_.t == rg.t == 23
    assert torch.equal(re_.params, rg.params) and torch.equal(re_.prev, rg.prev)
    for a in ("m2_prop", "m2_diff", "mean", "var", "alpha_prev"):
        assert torch.equal(getattr(re_.upd, a), getattr(rg.upd, a)), a
    assert pe.loss_buf.item() == pg.loss_buf.item()


def test_device_coef_beta_f_zero(api):
    """beta_f = 0 is a valid Moment2 decay (coefficient 1, moment2.hpp:36-38):
    with the device-formed coefficient (graph runs) the state equals the
    host-coefficient run bit for bit and stays finite."""
    n = 5000
    g = torch.Generator(device="cuda").manual_seed(3)
    props = [torch.randn(n, device="cuda", generator=g) for _ in range(4)]
    diffs = [0.1 * torch.randn(n, device="cuda", generator=g) for _ in range(4)]
    outs = []
    for dev_coef in (False, True):
        u = api.FusedMetaUpdate(n, lr=0.01, beta_f=0.0, device_coef=dev_coef)
        bufs = [torch.zeros(n, device="cuda"), torch.empty(n, device="cuda")]
        for t in range(6):
            u.step(props[t % 4], diffs[t % 4] if t else torch.zeros(n, device="cuda"),
                   bufs[t % 2], bufs[(t + 1) % 2])
        torch.cuda.synchronize()
        outs.append((bufs[0].clone(), u.m2_prop.clone(), u.var.clone()))
    for a, b in zip(*outs):
        assert torch.isfinite(a).all() and torch.equal(a, b)
