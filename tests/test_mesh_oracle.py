"""F1 slice 3 oracle (mgo_mesh_*, CPU): the reverse-mode texture gradient of
one pixel's proportional sample equals central finite differences of the
path radiances (paths are parameter-independent, so I(theta) is smooth
along them), and the estimator pieces behave as specified.  Parity is
unpinned against any external renderer (the reference has none); the GPU
kernels are pinned bit-exactly to this oracle in tests/test_gpu_mesh.py."""
import numpy as np
import pytest

from oracle_bind import Oracle
from paper_2309_15676_b200 import api


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.fixture(scope="module")
def scene():
    rec, obj, nobj = api.mesh_scene_geometry((6, 8), (8, 10))
    view = api.mesh_scene_view(max_vertices=4)
    return rec, obj, nobj, view


def test_brute_force_hit_is_the_nearest_triangle(oracle, scene):
    rec = scene[0]
    o = np.array([0.0, 1.6, 4.5])
    d = np.array([0.0, -0.25, -0.97])
    d /= np.linalg.norm(d)
    k, t = oracle.mesh_closest_hit(rec, o, d)
    assert k >= 0 and np.isfinite(t)
    # every other triangle hit along the ray is farther
    for j in range(rec.shape[0]):
        kk, tt = oracle.mesh_closest_hit(rec[j:j + 1], o, d)
        if kk == 0:
            assert tt >= t


def test_reverse_mode_gradient_matches_finite_differences(oracle, scene):
    rec, obj, nobj, view = scene
    R, W, H = 4, 3, 2
    n = nobj * 4 * R * R
    rs = np.random.RandomState(0)
    theta = rs.uniform(0.2, 0.8, n)
    target = np.full(3 * W * H, 0.05)
    key, it = 77, 3
    prop, diff, loss = oracle.mesh_sample_pair(W, H, rec, obj, nobj, R, view, target, theta, theta,
                                               key, it)
    assert np.all(diff == 0.0)          # theta_t == theta_{t-1}: the FD sample vanishes exactly
    # prop = sum_pixels sum_c r_A dI_B + r_B dI_A with I from mgo_mesh_path_radiance
    eps = 1e-6
    touched = np.flatnonzero(prop)
    assert touched.size > 4
    check = touched[rs.choice(touched.size, min(24, touched.size), replace=False)]
    fd = np.zeros(check.size)
    for px in range(W):
        for py in range(H):
            pix = py * W + px
            LA, _ = oracle.mesh_path_radiance(W, H, rec, obj, R, view, theta, px, py, key, it, 0)
            LB, _ = oracle.mesh_path_radiance(W, H, rec, obj, R, view, theta, px, py, key, it, 1)
            Is = target[np.arange(3) * W * H + pix]
            rA, rB = LA - Is, LB - Is
            for i, k in enumerate(check):
                tp, tm = theta.copy(), theta.copy()
                tp[k] += eps
                tm[k] -= eps
                dA = (oracle.mesh_path_radiance(W, H, rec, obj, R, view, tp, px, py, key, it, 0)[0] -
                      oracle.mesh_path_radiance(W, H, rec, obj, R, view, tm, px, py, key, it, 0)[0]) \
                    / (2 * eps)
                dB = (oracle.mesh_path_radiance(W, H, rec, obj, R, view, tp, px, py, key, it, 1)[0] -
                      oracle.mesh_path_radiance(W, H, rec, obj, R, view, tm, px, py, key, it, 1)[0]) \
                    / (2 * eps)
                fd[i] += float(np.sum(rA * dB + rB * dA))
    np.testing.assert_allclose(prop[check], fd, rtol=2e-5, atol=1e-8)


def test_sample_pair_rows_partition_exactly(oracle, scene):
    rec, obj, nobj, view = scene
    R, W, H = 4, 5, 4
    n = nobj * 4 * R * R
    rs = np.random.RandomState(1)
    now = rs.uniform(0.2, 0.8, n)
    prev = now - 0.01
    target = np.full(3 * W * H, 0.1)
    full = oracle.mesh_sample_pair(W, H, rec, obj, nobj, R, view, target, now, prev, 5, 1)
    a = oracle.mesh_sample_pair(W, H, rec, obj, nobj, R, view, target, now, prev, 5, 1, rows=(0, 3))
    b = oracle.mesh_sample_pair(W, H, rec, obj, nobj, R, view, target, now, prev, 5, 1, rows=(3, 4))
    assert np.array_equal(a[0] + b[0], full[0]) and np.array_equal(a[1] + b[1], full[1])


@pytest.mark.parametrize("nprop", [2, 4])
def test_metalness_reverse_mode_matches_finite_differences(oracle, scene, nprop):
    """configs[4] form: 5 texture channels (base rgb, roughness, metalness)
    with the full principled-BSDF derivatives, and n proportional paths:
    prop = 2/(n(n-1)) sum_j (sum_{i!=j} r_i) dI_j."""
    rec, obj, nobj, view = scene
    R, W, H, nch = 4, 3, 2, 5
    n = nobj * nch * R * R
    rs = np.random.RandomState(nprop)
    theta = rs.uniform(0.2, 0.8, n)
    target = np.full(3 * W * H, 0.05)
    key, it = 91, 2
    prop, diff, loss = oracle.meshx_sample_pair(W, H, rec, obj, nobj, nch, R, view, target, theta,
                                                theta, key, it, nprop)
    assert np.all(diff == 0.0)
    touched = np.flatnonzero(prop)
    # metalness entries are among the touched parameters
    assert np.any((touched // (R * R)) % nch == 4)
    check = touched[rs.choice(touched.size, min(20, touched.size), replace=False)]
    eps = 1e-6
    scale = 2.0 / (nprop * (nprop - 1.0))
    fd = np.zeros(check.size)

    def rad(th, px, py, j):
        return oracle.meshx_path_radiance(W, H, rec, obj, nch, R, view, th, px, py, key, it, j)[0]
    for px in range(W):
        for py in range(H):
            pix = py * W + px
            Is = target[np.arange(3) * W * H + pix]
            r = [rad(theta, px, py, j) - Is for j in range(nprop)]
            for i, k in enumerate(check):
                tp, tm = theta.copy(), theta.copy()
                tp[k] += eps
                tm[k] -= eps
                for j in range(nprop):
                    dI = (rad(tp, px, py, j) - rad(tm, px, py, j)) / (2 * eps)
                    others = sum(r[m] for m in range(nprop) if m != j)
                    fd[i] += scale * float(np.sum(others * dI))
    np.testing.assert_allclose(prop[check], fd, rtol=2e-5, atol=1e-8)


def test_general_form_reduces_to_the_configs3_estimator(oracle, scene):
    rec, obj, nobj, view = scene
    R, W, H = 4, 4, 3
    n = nobj * 4 * R * R
    rs = np.random.RandomState(4)
    now = rs.uniform(0.2, 0.8, n)
    prev = now - 0.01
    target = np.full(3 * W * H, 0.1)
    a = oracle.mesh_sample_pair(W, H, rec, obj, nobj, R, view, target, now, prev, 3, 1)
    b = oracle.meshx_sample_pair(W, H, rec, obj, nobj, 4, R, view, target, now, prev, 3, 1, 2)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
