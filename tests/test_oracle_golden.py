"""Pin the C restatement (oracle/metagrad_oracle.c) against golden vectors
produced by the UNMODIFIED reference (tests/golden/, oracle/gen_golden.py).

Everything here is bit-exact: the oracle and the reference perform the same
IEEE operations in the same order (both built without FMA contraction; the
reference's reductions are sequential under the shim).
CPU only.
"""
import ast

import numpy as np
import pytest

from paper_2309_15676_b200 import _abi


def bits_equal(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


# ------------------------------------------------------------------ A1 RNG
@pytest.mark.parametrize("s", [0, 7, 42])
@pytest.mark.parametrize("r", [0, 1, 999])
def test_rng_streams_bit_exact(oracle, golden, s, r):
    g = golden("rng")
    raw = oracle.rng_draws(s, r, 1, 100000)
    assert np.array_equal(raw[:2000], g[f"rng_raw_s{s}_r{r}"])
    assert np.bitwise_xor.reduce(raw) == g[f"rng_xor_s{s}_r{r}"]
    assert np.sum(raw, dtype=np.uint64) == g[f"rng_sum_s{s}_r{r}"]
    assert bits_equal(oracle.rng_draws(s, r, 2, 2000), g[f"rng_uni_s{s}_r{r}"])
    assert bits_equal(oracle.rng_draws(s, r, 3, 2000), g[f"rng_upos_s{s}_r{r}"])


def test_mt19937_64_standard_value(oracle, golden):
    # C++ standard [rand.predef]: the 10000th output of a default-constructed
    # mt19937_64 (seed 5489) is 9981545732273789042.
    raw = oracle.rng_draws(5489, 0, 0, 10000)
    assert int(raw[-1]) == 9981545732273789042
    assert np.array_equal(raw, golden("rng")["rng_engine_raw_seed5489"])


def test_mix64_matches_reference_stream_seed(oracle):
    # rng.hpp:9-14 on a few fixed inputs (values from the splitmix64 finaliser)
    assert oracle.mix64(0) == 0xE220A8397B1DCDAF
    assert oracle.mix64(1) == 0x910A2DEC89025CC1


# ------------------------------------------------------- A2-A7 problems
@pytest.mark.parametrize("P,seed", [(16, 2024), (4096, 1), (8, 1234), (6, 11)])
def test_minirender_generate(oracle, golden, P, seed):
    g = golden("problems")
    b, T = oracle.minirender_generate(P, seed)
    assert bits_equal(b, g[f"gen_P{P}_s{seed}_b"])
    assert bits_equal(T, g[f"gen_P{P}_s{seed}_T"])


@pytest.mark.parametrize("P,spp,seed", [(16, 4, 2024), (4096, 2, 1), (6, 3, 11)])
def test_minirender_kernel_terms_and_pairs(oracle, golden, P, spp, seed):
    g = golden("problems")
    b, T = oracle.minirender_generate(P, seed)
    cross, mb = oracle.minirender_kernel_terms(b, g[f"kt_P{P}_spp{spp}_u"], spp)
    assert bits_equal(cross, g[f"kt_P{P}_spp{spp}_cross"])
    assert bits_equal(mb, g[f"kt_P{P}_spp{spp}_mb"])
    now, prev = g[f"sp_P{P}_spp{spp}_now"], g[f"sp_P{P}_spp{spp}_prev"]
    for skip in (0, 2):
        prop, diff, ssn = oracle.minirender_sample_pair(spp, b, T, now, prev, 909, 3, skip)
        assert bits_equal(prop, g[f"sp_P{P}_spp{spp}_k{skip}_prop"])
        assert bits_equal(diff, g[f"sp_P{P}_spp{spp}_k{skip}_diff"])
        assert bits_equal(ssn, g[f"sp_P{P}_spp{spp}_k{skip}_ssn"])
    prop, diff, ssn = oracle.minirender_sample_pair(spp, b, T, now, now, 909, 3, 0)
    assert bits_equal(prop, g[f"sp_P{P}_spp{spp}_same_prop"])
    assert bits_equal(diff, g[f"sp_P{P}_spp{spp}_same_diff"]) and ssn == 0.0


def test_exprate_pairs(oracle, golden):
    g = golden("problems")
    for now, prev, skip, p, d, s in g["exprate"]:
        op, od, os_, rc = oracle.exprate_sample_pair(2.0, 32, now, prev, 808, 7, int(skip))
        assert rc == 0
        assert bits_equal([op, od, os_], [p, d, s])
    assert oracle.exprate_sample_pair(2.0, 32, -0.5, 1.0, 1, 0)[3] == _abi.MG_EDOMAIN
    assert int(g["exprate_domain_rc"]) == 3  # reference raised std::domain_error


def test_multnoise_pairs(oracle, golden):
    g = golden("problems")
    now = np.array([1.5, -0.7, 2.2, 0.3])
    prev = np.array([1.45, -0.75, 2.14, 0.33])
    for skip in (0, 3):
        prop, diff, ssn = oracle.multnoise_sample_pair(1.0, 2, np.zeros(4), now, prev, 404, 0, skip)
        assert bits_equal(prop, g[f"mn_k{skip}_prop"])
        assert bits_equal(diff, g[f"mn_k{skip}_diff"])
        assert bits_equal(ssn, g[f"mn_k{skip}_ssn"])


# ------------------------------------------------------ A8-A12 estimators
@pytest.mark.parametrize("decay", [0.5, 0.9, 0.99])
def test_moment2(oracle, golden, decay):
    g = golden("estimators")
    out = oracle.moment2_run(decay, g[f"m2_d{decay}_xs"])
    assert bits_equal(out, g[f"m2_d{decay}_out"])
    assert bits_equal(out[0], g[f"m2_d{decay}_xs"][0] ** 2)  # first step is the raw square


@pytest.mark.parametrize("k", [0, 1, 2])
def test_meta_step(oracle, golden, k):
    g = golden("estimators")
    prop, diff, vp, vd = g[f"meta{k}_in"]
    st = None
    if f"meta{k}_state_in" in g:
        m, v, a = g[f"meta{k}_state_in"]
        st = {"mean": m, "var": v, "alpha_prev": a}
    out, delta, rc = oracle.meta_step(0.01, 1e-8, 1e-30, int(g[f"meta{k}_clip"]), st, prop, diff,
                                      vp, vd)
    assert rc == 0
    assert bits_equal(np.stack([out["mean"], out["var"], out["alpha_prev"]]),
                      g[f"meta{k}_state_out"])
    assert bits_equal(delta, g[f"meta{k}_delta"])


def test_meta_step_rejects_negative_variance(oracle):
    _, _, rc = oracle.meta_step(0.01, 1e-8, 1e-30, 1, None, [1.0], [0.0], [-1.0], [0.0])
    assert rc == _abi.MG_ELOGIC


def test_meta_hand_evaluated_injected_state(oracle):
    # tests/test_meta.cpp:83-96 (alpha=0.5, mean=1.5, var=0.5)
    st = {"mean": np.zeros(1), "var": np.ones(1), "alpha_prev": np.full(1, 0.5)}
    out, _, _ = oracle.meta_step(0.01, 1e-8, 1e-30, 1, st, [2.0], [1.0], [1.0], [0.0])
    assert out["alpha_prev"][0] == pytest.approx(0.5, rel=1e-14)
    assert out["mean"][0] == pytest.approx(1.5, rel=1e-14)
    assert out["var"][0] == pytest.approx(0.5, rel=1e-14)


def test_adam(oracle, golden):
    g = golden("estimators")
    m, v, d, _ = oracle.adam_run(g["adam_grads"], lr=0.02)
    assert bits_equal(m, g["adam_m"]) and bits_equal(v, g["adam_v"])
    assert bits_equal(d, g["adam_delta"])


# ----------------------------------------------------------- A13 harness
RUNS = ["accept9_r0", "accept9_r3", "accept9_noclip_r0", "noiseless_r0", "scripted_exp_r0",
        "exprate_r0", "exprate_adam_r0", "multnoise_indep_r0", "multnoise_perparam_r0",
        "diverge_r0", "minirender_adam_r0", "s1_standin_r0"]


@pytest.mark.parametrize("key", RUNS)
def test_run_single_full_record(oracle, golden, key):
    g = golden("runs")
    kw = ast.literal_eval(str(g[f"{key}__cfg"]))
    rep = int(key.rsplit("_r", 1)[1])
    cfg = _abi.config_from(**kw)
    rec = oracle.run_single(cfg, rep)
    assert rec["rc"] == 0
    for k in ("iterations_run", "status", "draws_used", "evals_used"):
        assert rec[k] == int(g[f"{key}__{k}"]), k
    for k in ("params", "loss", "prop", "diff", "ssn", "mean_est", "var_est", "delta",
              "true_grad"):
        assert bits_equal(rec[k], g[f"{key}__{k}"]), k
    if kw.get("optimizer", "meta") == "meta":
        assert bits_equal(rec["alpha"], g[f"{key}__alpha"])


def test_noiseless_recurrence_hand_values(oracle):
    # tests/test_harness.cpp:102-134
    cfg = _abi.config_from(problem="mult-noise", dim=1, sigma=0.0, samples_per_iter=1,
                           trajectory="scripted-linear", iterations=3)
    rec = oracle.run_single(cfg, 0)
    assert rec["prop"][0, 0] == 2.0 and rec["diff"][0, 0] == 0.0 and rec["alpha"][0, 0] == 0.0
    var_prop = 4.0 + (0.1 / 0.19) * (1.0 - 4.0)
    var_folded = 5.0
    alpha = var_prop / (var_prop + var_folded + 1e-30)
    assert rec["ssn"][1] == 1.0
    assert rec["alpha"][1, 0] == pytest.approx(alpha, rel=1e-14)
    assert rec["mean_est"][1, 0] == pytest.approx(1.0, rel=1e-14)


def test_philox4x32_10_known_answers(oracle):
    """Random123 published known-answer vectors for philox4x32-10."""
    assert oracle.philox([0, 0, 0, 0], 0) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert oracle.philox([0xffffffff] * 4, 0xffffffffffffffff) == [
        0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert oracle.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                         (0x299f31d0 << 32) | 0xa4093822) == [
        0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]
    u = oracle.philox_uniforms(12345, 4, 3, 7)
    assert u.shape == (12,) and (u >= 0).all() and (u < 1).all()


# ------------------------------------------------ F1 slice (own renderer)
def test_quad_oracle_properties(oracle):
    """The F1 oracle (mgo_quad_*; the reference has no renderer): identical
    textures give an exactly zero FD sample; the gradient sample is affine
    in the texture (Lambertian direct lighting is linear in the albedo);
    renders are deterministic in (key, stream)."""
    W, H, R, Le = 32, 32, 8, (8.0, 7.0, 6.0)
    rs = np.random.RandomState(0)
    tex = rs.uniform(0, 1, 3 * R * R)
    img = oracle.quad_render(W, H, R, tex, Le, 8, 11, 7)
    assert np.array_equal(img, oracle.quad_render(W, H, R, tex, Le, 8, 11, 7))
    assert img.max() > 0 and (img >= 0).all()
    p0, d0, _ = oracle.quad_sample_pair(W, H, R, Le, img, tex, tex, 3, 0)
    assert (d0 == 0).all()
    # affine: prop(a + s*e) - prop(a) is linear in s
    e = rs.uniform(-1, 1, tex.size)
    p1, _, _ = oracle.quad_sample_pair(W, H, R, Le, img, tex + 0.1 * e, tex + 0.1 * e, 3, 0)
    p2, _, _ = oracle.quad_sample_pair(W, H, R, Le, img, tex + 0.2 * e, tex + 0.2 * e, 3, 0)
    np.testing.assert_allclose(p2 - p0, 2 * (p1 - p0), atol=1e-9)
    # FD sample == linear response to the texture step on shared draws
    _, d1, _ = oracle.quad_sample_pair(W, H, R, Le, img, tex + 0.1 * e, tex, 3, 0)
    _, d2, _ = oracle.quad_sample_pair(W, H, R, Le, img, tex + 0.2 * e, tex, 3, 0)
    np.testing.assert_allclose(d2, 2 * d1, atol=1e-9)
