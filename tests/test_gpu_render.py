"""Fused mini-render iteration (mg_minirender_meta_iteration): the sample
pair computed in registers and fed straight into the fused meta update.

  * mt64 mode, fp64: the whole trajectory against the reference run (oracle
    run_single, same seeds) — params and loss rel <= 1e-9 (CUDA vs glibc pow,
    and the device's tree-ordered step norm over 4096 pixels).
  * Philox mode: the pair math bit-for-bit against the oracle fed the same
    Philox uniforms (fp64, <= 1e-9 term-scale for pow), fp32 <= 1e-4, and
    the estimator's unbiasedness (problems.hpp:175-178) as a z-test over 2^20
    independent pixels.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2309_15676_b200 import _abi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2309_15676_b200 import api as a
    return a


def host(t):
    return t.detach().double().cpu().numpy()


def test_fused_minirender_mt64_trajectory_matches_reference(api, oracle):
    P, spp, iters = 4096, 2, 21
    cfg = _abi.config_from(problem="mini-render", pixel_count=P, spp=spp, iterations=iters,
                           seed=0, problem_seed=1, lr=0.01)
    rec = oracle.run_single(cfg, 0)
    run = api.MiniRenderRun(P, spp, gen_seed=1, lr=0.01, seed=0, replicate=0, rng="mt64",
                            dtype=torch.float64)
    for k in range(1, iters):
        run.step()
        np.testing.assert_allclose(host(run.params), rec["params"][k], rtol=1e-9, atol=1e-13,
                                   err_msg=f"iteration {k}")
        assert run.scalars().loss == pytest.approx(rec["loss"][k], rel=1e-9)


def test_fused_minirender_f32_mt64_tolerance(api, oracle):
    P, spp, iters = 4096, 2, 21
    cfg = _abi.config_from(problem="mini-render", pixel_count=P, spp=spp, iterations=iters,
                           seed=3, problem_seed=1, lr=0.01)
    rec = oracle.run_single(cfg, 0)
    run = api.MiniRenderRun(P, spp, gen_seed=1, lr=0.01, seed=3, replicate=0, rng="mt64",
                            dtype=torch.float32)
    for _ in range(1, iters):
        run.step()
    ref = rec["params"][iters - 1]
    assert np.max(np.abs(host(run.params) - ref) / np.maximum(np.abs(ref), 0.1)) < 1e-4


@pytest.mark.parametrize("dt,tol", [(torch.float64, 1e-9), (torch.float32, 1e-4)])
def test_fused_minirender_philox_pair_math(api, oracle, dt, tol):
    P, spp = 1000, 3
    run = api.MiniRenderRun(P, spp, gen_seed=11, lr=0.05, seed=9, replicate=2, rng="philox",
                            dtype=dt)
    b = host(run.problem.exponents)
    T = host(run.problem.target)
    prev = host(run.params)
    for it in range(3):
        now = host(run.params)
        prop = torch.empty(P, dtype=dt, device="cuda")
        diff = torch.empty(P, dtype=dt, device="cuda")
        run.step(prop_out=prop, diff_out=diff)
        u = oracle.philox_uniforms(run.key, P, spp, it)
        cross, mb = oracle.minirender_kernel_terms(b, u, spp)
        ref_prop = (2.0 * now) * cross - (2.0 * T) * mb
        ref_diff = np.zeros(P) if it == 0 else (2.0 * (now - prev)) * cross
        scale = 2 * np.abs(now) * 25.0 + 10.0
        assert np.max(np.abs(host(prop) - ref_prop) / scale) < tol, it
        assert np.max(np.abs(host(diff) - ref_diff) / scale) < tol, it
        prev = now


def test_philox_estimator_is_unbiased(api):
    """problems.hpp:175-178: E[prop] = 2 (a - T) — z-test over 2^20 pixels with
    identical (b, T, a), each drawing independent Philox uniforms."""
    from paper_2309_15676_b200 import _lib
    L = _lib.load()
    ctx = api.Context.default()
    P, spp = 1 << 20, 4
    dt = torch.float64
    b = torch.full((P,), 2.5, dtype=dt, device="cuda")
    T = torch.full((P,), 0.5, dtype=dt, device="cuda")
    now = torch.full((P,), 0.7, dtype=dt, device="cuda")
    prev = now.clone()
    st = [torch.empty(P, dtype=dt, device="cuda") for _ in range(5)]
    sc = torch.zeros(8, dtype=torch.float64, device="cuda")
    L.mg_scalars_write(ctx.h, C.c_void_p(sc.data_ptr()), C.byref(_abi.fresh_scalars()))
    prop = torch.empty(P, dtype=dt, device="cuda")
    upd = _abi.MetaUpdateArgs(meta=_abi.MetaParams(0.01, 1e-8, 1e-30, 1), prop_coef=1.0,
                              beta_delta=0.5, first_step=1, project=1)
    a = _abi.RenderArgs(update=upd, spp=spp, rng_kind=_abi.MG_RNG_PHILOX, key=777, iteration=0)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    assert L.mg_minirender_meta_iteration(ctx.h, _abi.MG_F64, P, C.byref(a), p(b), p(T), None,
                                          p(now), p(prev), *[p(x) for x in st], p(sc), p(prop),
                                          None) == 0
    x = host(prop)
    z = abs(x.mean() - 2 * (0.7 - 0.5)) / (x.std(ddof=1) / np.sqrt(P))
    assert z < 4.0, z


@pytest.mark.parametrize("rng", ["philox", "mt64"])
def test_pixel_sharded_run_matches_unsharded(api, rng):
    """Two pixel shards of ONE run, executed one after the other on this GPU
    with the 4 reducible scalars summed between iterations (what ShardedStep's
    NCCL all-reduce does across GPUs), reproduce the unsharded run: the
    per-pixel draws are addressed by global pixel index (Philox) or sliced
    from the replicate's full stream (mt64), so only the step-norm summation
    order differs."""
    P, spp, cut = 5003, 3, 2048
    kw = dict(gen_seed=5, lr=0.02, seed=4, replicate=1, rng=rng, dtype=torch.float64)
    full = api.MiniRenderRun(P, spp, **kw)
    shards = [api.MiniRenderRun(P, spp, pixel_range=(0, cut), **kw),
              api.MiniRenderRun(P, spp, pixel_range=(cut, P), **kw)]
    for _ in range(12):
        full.step()
        for s in shards:
            s.step()
        tot = shards[0].scalars_buf[:4] + shards[1].scalars_buf[:4]
        for s in shards:
            s.scalars_buf[:4] = tot
    got = np.concatenate([host(s.params) for s in shards])
    np.testing.assert_allclose(got, host(full.params), rtol=1e-12, atol=1e-15)
    assert full.scalars().loss == pytest.approx(float(tot[2]), rel=1e-12)


@pytest.mark.parametrize("dt,rtol", [("f64", 1e-9), ("f32", 1e-4)])
def test_scaled_run_single_matches_reference_series(api, oracle, dt, rtol):
    """run_single of a large mini-render replicate dispatches to the fused
    whole-GPU iteration (exact mt64 stream) and reproduces the reference's
    extractor series and counters."""
    P = api.SCALED_MIN_PIXELS + 1000
    kw = dict(problem="mini-render", pixel_count=P, spp=2, iterations=15, seed=2,
              problem_seed=9, lr=0.02, coord=777)
    cfg = api.ExperimentConfig(dtype=dt, **kw)
    assert api._scaled_eligible(cfg)
    rec = api.run_single(cfg, 1)
    ser, recs, finals = oracle.run_series(_abi.config_from(**kw), 2)
    assert (rec.iterations_run, rec.draws_used, rec.evals_used) == recs[1][0:1] + recs[1][2:4]
    for name in ("loss", "param_err", "prop", "diff", "grad_est", "est_var", "alpha", "delta",
                 "true_grad", "step_sq_norm", "param"):
        ref = ser[name][1]
        scale = np.max(np.abs(ref)) + 1e-300
        np.testing.assert_allclose(rec.series[name], ref, rtol=rtol, atol=rtol * scale,
                                   err_msg=name)


@pytest.mark.parametrize("rng", ["philox", "mt64"])
@pytest.mark.parametrize("spp", [2, 3, 4])
def test_fast_f32_kernel_tracks_fp64_run(api, spp, rng):
    """The TMA-fed fp32 fast kernel (render_fast.cu: FMA, approximate
    divide/sqrt/rcp, fp32 per-thread partial sums) at a size that runs it
    (>= one 1024-pixel tile per SM, ring wrapping, plus a ragged tail) stays
    within the fp32 bar of the fp64 run on the same draws — Philox, or the
    exact mt19937_64 stream streamed in as a tenth TMA array; both pair
    maths are pinned to the oracle above — over 12 iterations, and within
    1e-5 of the IEEE fp32 kernel."""
    from paper_2309_15676_b200 import _lib
    L = _lib.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    P = 1024 * sms * 9 + 333
    kw = dict(gen_seed=3, lr=0.02, seed=5, replicate=0, rng=rng)
    runs = {"f64": api.MiniRenderRun(P, spp, dtype=torch.float64, **kw),
            "fast": api.MiniRenderRun(P, spp, dtype=torch.float32, **kw)}
    L.mg_set_option(b"render_fast", 0)
    try:
        runs["ieee"] = api.MiniRenderRun(P, spp, dtype=torch.float32, **kw)
    finally:
        L.mg_set_option(b"render_fast", 1)
    for _ in range(12):
        for name, r in runs.items():
            L.mg_set_option(b"render_fast", 0 if name == "ieee" else 1)
            try:
                r.step()
            finally:
                L.mg_set_option(b"render_fast", 1)
    torch.cuda.synchronize()
    ref = host(runs["f64"].params)
    for name, tol in (("fast", 1e-4), ("ieee", 1e-4)):
        got = host(runs[name].params)
        assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 0.1)) < tol, name
        for st in ("mean", "var", "alpha_prev", "m2_prop"):
            a, b = host(getattr(runs[name], st)), host(getattr(runs["f64"], st))
            floor = np.sqrt(np.mean(b ** 2))
            assert np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)) < tol, (name, st)
    fast, ieee = host(runs["fast"].params), host(runs["ieee"].params)
    assert np.max(np.abs(fast - ieee) / np.maximum(np.abs(ieee), 0.1)) < 1e-5
    s64, s32 = runs["f64"].scalars(), runs["fast"].scalars()
    assert s32.nonfinite == 0
    assert s32.loss == pytest.approx(s64.loss, rel=1e-4)
    assert s32.ssn == pytest.approx(s64.ssn, rel=1e-3)
