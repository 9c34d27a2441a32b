"""F1 slice 2 (BASELINE.json configs[2]): depth-4 path-traced
gradients of a principled BSDF's 5 global parameters on the helix scene,
against the repo's own CPU oracle (mgo_helix_*; no reference renderer).
fp64 render and sample pairs are BIT-EXACT (IEEE + - * / sqrt only,
Philox-addressed sampling, fixed-point reduction)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
LE, ENV, GR = (10.0, 10.0, 10.0), (0.2, 0.2, 0.2), (0.5, 0.5, 0.5)


@pytest.fixture(scope="module")
def api():
    from paper_2309_15676_b200 import api as a
    return a


def host(t):
    return t.detach().double().cpu().numpy()


def bits_equal(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_helix_render_bit_exact(api, oracle):
    prob = api.HelixProblem(48, 40, target_spp=4)
    from paper_2309_15676_b200 import _lib
    key = _lib.load().mg_mix64(1)
    ref = oracle.helix_render(48, 40, prob.spheres_host, LE, ENV, GR, host(prob.target_theta), 4,
                              key)
    assert bits_equal(host(prob.target_img), ref)
    assert ref.max() > 0.1


def test_helix_sample_pair_bit_exact(api, oracle):
    W, H = 40, 40
    prob = api.HelixProblem(W, H, target_spp=4)
    now = np.array([0.6, 0.35, 0.2, 0.3, 0.45])
    prev = now - np.array([0.01, -0.02, 0.005, 0.01, -0.015])
    for it in (0, 3):
        pair = prob.sample_pair(torch.tensor(now, device="cuda"), torch.tensor(prev, device="cuda"),
                                it, key=77)
        p, d, loss = oracle.helix_sample_pair(W, H, prob.spheres_host, LE, ENV, GR,
                                              host(prob.target_img), now, prev, 77, it)
        assert bits_equal(host(pair.prop), p), (host(pair.prop), p)
        assert bits_equal(host(pair.diff), d), (host(pair.diff), d)
        assert float(prob.loss_buf[0]) == pytest.approx(loss, rel=1e-11)
    same = prob.sample_pair(torch.tensor(now, device="cuda"), torch.tensor(now, device="cuda"), 1,
                            key=77)
    assert (host(same.diff) == 0).all()


def test_helix_fd_sample_is_unbiased(api):
    W, H, K = 32, 32, 1500
    prob = api.HelixProblem(W, H, target_spp=16)
    a = torch.tensor([0.6, 0.35, 0.2, 0.3, 0.45], device="cuda", dtype=torch.float64)
    b = a - torch.tensor([0.03, -0.02, 0.02, 0.03, -0.04], device="cuda", dtype=torch.float64)
    sums = {k: torch.zeros(5, dtype=torch.float64, device="cuda") for k in ("d", "d2", "pa", "pa2",
                                                                               "pb", "pb2")}
    for it in range(K):
        d = prob.sample_pair(a, b, it, key=5).diff
        ya = prob.sample_pair(a, a, it, key=6).prop
        yb = prob.sample_pair(b, b, it, key=7).prop
        sums["d"] += d
        sums["d2"] += d * d
        sums["pa"] += ya
        sums["pa2"] += ya * ya
        sums["pb"] += yb
        sums["pb2"] += yb * yb
    s = {k: host(v) / K for k, v in sums.items()}
    vd = (s["d2"] - s["d"] ** 2) / K
    vp = (s["pa2"] - s["pa"] ** 2) / K + (s["pb2"] - s["pb"] ** 2) / K
    z = np.abs(s["d"] - (s["pa"] - s["pb"])) / np.sqrt(vd + vp)
    assert z.max() < 4.0, z
    assert np.all(vd < 0.5 * vp)  # common random numbers: FD far less noisy


def test_helix_optimisation_fits_target(api, record_property):
    prob = api.HelixProblem(64, 64, target_spp=64)
    run = api.HelixRun(prob, optimizer="meta", lr=0.01)
    e0 = float(torch.linalg.vector_norm(run.params - prob.target_theta))
    for _ in range(300):
        run.step()
    e1 = float(torch.linalg.vector_norm(run.params - prob.target_theta))
    record_property("theta_error", [e0, e1])
    print("helix theta error", e0, "->", e1, host(run.params), host(prob.target_theta))
    assert e1 < 0.7 * e0, (e0, e1, host(run.params), host(prob.target_theta))


def test_helix_tile_sharded_gradients_sum_exactly(api):
    prob = api.HelixProblem(40, 40, target_spp=4)
    a = torch.tensor([0.6, 0.35, 0.2, 0.3, 0.45], device="cuda", dtype=torch.float64)
    b = a - 0.01
    full = prob.sample_pair(a, b, 2, key=9)
    full = (full.prop.clone(), full.diff.clone())
    sp, sd = torch.zeros_like(a), torch.zeros_like(a)
    for r0, r1 in ((0, 13), (13, 29), (29, 40)):
        part = prob.sample_pair(a, b, 2, key=9, rows=(r0, r1))
        sp += part.prop
        sd += part.diff
    assert torch.equal(sp, full[0]) and torch.equal(sd, full[1])


def test_helix_f32_path_divergence_pixel_fraction(api, record_property):
    """fp32 mode traces the helix geometry in fp32: a path can take a
    different branch than the fp64 path on the same random numbers (grazing
    hits, shadow-ray edges).  Reported as the fraction of pixels whose
    1-spp radiance differs by more than 1e-3 (relative) — same-path pixels
    differ by ~1e-6."""
    W = H = 128
    p64 = api.HelixProblem(W, H, target_spp=1, dtype=torch.float64)
    theta = torch.tensor([0.6, 0.35, 0.2, 0.3, 0.45], device="cuda", dtype=torch.float64)
    i64 = p64.render(theta, 1, 1234).cpu().numpy().reshape(3, -1)
    i32 = p64.render(theta.float(), 1, 1234).double().cpu().numpy().reshape(3, -1)
    rel = np.abs(i32 - i64) / np.maximum(np.abs(i64), 1e-2)
    diverged = float(np.mean(rel.max(axis=0) > 1e-3))
    record_property("helix_f32_diverged_pixel_fraction", diverged)
    print("helix f32 path-divergence pixel fraction", diverged)
    # measured 3.7e-4 (128 x 128, 1 spp) with the cancellation-free fp32
    # sphere test (3.5e-2 with the fp64 expression order evaluated in fp32)
    assert diverged < 2e-3
    # the remaining pixels agree to fp32 precision
    same = rel.max(axis=0) <= 1e-3
    assert np.median(rel.max(axis=0)[same]) < 1e-5
