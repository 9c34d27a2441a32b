"""Test-side ctypes bindings to the CPU checkers (TEST INFRASTRUCTURE ONLY).

  Oracle  — oracle/_build/libmgoracle.so: the plain-C restatement of the
            reference hot path (oracle/metagrad_oracle.c).
  RefLib  — oracle/_ref/libmetagrad_ref.so: the UNMODIFIED reference sources
            compiled against the Eigen shim (oracle/ref/Makefile), when built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may use these.  The product path (paper_2309_15676_b200) never does.
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2309_15676_b200 import _abi  # noqa: E402

ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libmgoracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libmetagrad_ref.so")

_dp = C.POINTER(C.c_double)


def _ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays must be contiguous"
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def build_oracle():
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


class Oracle:
    """ctypes view of oracle/metagrad_oracle.h."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        self.lib = L = C.CDLL(path)
        L.mgo_mix64.restype = C.c_uint64
        L.mgo_mix64.argtypes = [C.c_uint64]
        L.mgo_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int64, C.c_void_p]
        L.mgo_moment2_step.argtypes = [C.c_int64, C.c_double, _dp, C.POINTER(C.c_int64),
                                       C.c_void_p, C.c_void_p]
        L.mgo_meta_step.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int,
                                    C.c_int] + [C.c_void_p] * 8
        L.mgo_adam_step.argtypes = [C.c_int64, C.POINTER(_abi.AdamScalars)] + [C.c_void_p] * 4
        L.mgo_meta_update.argtypes = ([C.c_int64, C.POINTER(_abi.MetaUpdateArgs)] +
                                      [C.c_void_p] * 13 +
                                      [C.POINTER(_abi.UpdateScalars), C.c_void_p])
        L.mgo_adam_update.argtypes = ([C.c_int64, C.POINTER(_abi.AdamScalars), C.c_int,
                                       C.c_double] + [C.c_void_p] * 6 +
                                      [C.POINTER(_abi.UpdateScalars)])
        L.mgo_minirender_generate.argtypes = [C.c_int32, C.c_uint64, C.c_double, C.c_void_p,
                                              C.c_void_p]
        L.mgo_minirender_kernel_terms.argtypes = [C.c_int32, C.c_int32] + [C.c_void_p] * 4
        L.mgo_exprate_gradient_from_batch.restype = C.c_double
        L.mgo_exprate_gradient_from_batch.argtypes = [C.c_double, C.c_int32, C.c_double,
                                                      C.c_double, C.c_double]
        L.mgo_problem_dim.argtypes = [C.POINTER(_abi.ExperimentConfigC)]
        L.mgo_run_single.argtypes = [C.POINTER(_abi.ExperimentConfigC), C.c_int32,
                                     C.POINTER(_abi.RunRecordC), C.c_void_p]
        L.mgo_run_single_series.argtypes = [C.POINTER(_abi.ExperimentConfigC), C.c_int32,
                                            C.POINTER(_abi.RunRecordC),
                                            C.POINTER(_abi.RunSeriesC), C.c_int32, C.c_void_p]
        L.mgo_philox4x32_10.argtypes = [C.POINTER(C.c_uint32 * 4), C.c_uint64,
                                        C.POINTER(C.c_uint32 * 4)]
        L.mgo_philox_uniform.restype = C.c_double
        L.mgo_philox_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint32]
        # sample-pair helpers take an mgo_mt64*; we re-create streams per call
        self._mt_size = 312 * 8 + 8

    # ------------------------------------------------------------ rng
    def philox(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        o = (C.c_uint32 * 4)()
        self.lib.mgo_philox4x32_10(C.byref(c), key, C.byref(o))
        return list(o)

    def philox_uniforms(self, key, P, spp, it, stream=0):
        f = self.lib.mgo_philox_uniform
        return np.array([f(key, j, it, s, stream) for j in range(P) for s in range(spp)])

    def mix64(self, x):
        return self.lib.mgo_mix64(x)

    def rng_draws(self, seed, rep, mode, n):
        out = np.empty(n, dtype=np.uint64 if mode in (0, 1) else np.float64)
        self.lib.mgo_rng_draws(seed, rep, mode, n, _ptr(out))
        return out

    def new_stream(self, seed, rep):
        buf = C.create_string_buffer(self._mt_size)
        self.lib.mgo_rng_stream(buf, C.c_uint64(seed), C.c_uint64(rep))
        return buf

    # ------------------------------------------------------ estimators
    def moment2_run(self, decay, xs):
        xs = _f64(xs)
        steps, n = xs.shape
        m2 = np.zeros(n)
        out = np.empty_like(xs)
        pw, cnt = C.c_double(1.0), C.c_int64(0)
        for s in range(steps):
            row = np.ascontiguousarray(xs[s])
            self.lib.mgo_moment2_step(n, decay, C.byref(pw), C.byref(cnt), _ptr(m2), _ptr(row))
            out[s] = m2
        return out

    def meta_step(self, lr, eps_step, eps_alpha, clip, state, prop, diff, var_prop, var_diff):
        """state = None (fresh) or dict(mean, var, alpha_prev); returns (state, delta, rc)."""
        prop, diff, var_prop, var_diff = map(_f64, (prop, diff, var_prop, var_diff))
        n = prop.size
        first = state is None
        st = {k: np.zeros(n) for k in ("mean", "var", "alpha_prev")} if first else \
            {k: _f64(v).copy() for k, v in state.items()}
        delta = np.empty(n)
        rc = self.lib.mgo_meta_step(n, lr, eps_step, eps_alpha, int(clip), int(first),
                                    _ptr(st["mean"]), _ptr(st["var"]), _ptr(st["alpha_prev"]),
                                    _ptr(prop), _ptr(diff), _ptr(var_prop), _ptr(var_diff),
                                    _ptr(delta))
        return st, delta, rc

    def adam_run(self, grads, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8):
        grads = _f64(grads)
        steps, n = grads.shape
        s = _abi.AdamScalars(lr, beta1, beta2, eps, 1.0, 1.0, 0)
        m, v, d = np.zeros(n), np.zeros(n), np.zeros(n)
        for k in range(steps):
            row = np.ascontiguousarray(grads[k])
            self.lib.mgo_adam_step(n, C.byref(s), _ptr(m), _ptr(v), _ptr(row), _ptr(d))
        return m, v, d, s

    def meta_update(self, args, state, prop, diff, params_in, scalars, target=None,
                    vprop=None, vdiff=None, params_prev=None):
        """One fused iteration; state dict of fp64 arrays (m2_prop, m2_diff,
        mean, var, alpha_prev) updated in place; returns (params_out, delta, rc)."""
        prop, diff, params_in = _f64(prop), _f64(diff), _f64(params_in)
        n = prop.size
        out = np.empty(n)
        delta = np.empty(n)
        rc = self.lib.mgo_meta_update(
            n, C.byref(args), _ptr(prop), _ptr(diff),
            _ptr(None if vprop is None else _f64(vprop)),
            _ptr(None if vdiff is None else _f64(vdiff)),
            _ptr(state["m2_prop"]), _ptr(state["m2_diff"]), _ptr(state["mean"]),
            _ptr(state["var"]), _ptr(state["alpha_prev"]), _ptr(params_in), _ptr(out),
            _ptr(None if params_prev is None else _f64(params_prev)),
            _ptr(None if target is None else _f64(target)), C.byref(scalars), _ptr(delta))
        return out, delta, rc

    def adam_update(self, s, grad, m, v, params_in, scalars, target=None, project=False,
                    proj_lo=0.0):
        grad, params_in = _f64(grad), _f64(params_in)
        out = np.empty_like(params_in)
        self.lib.mgo_adam_update(grad.size, C.byref(s), int(project), proj_lo, _ptr(grad),
                                 _ptr(m), _ptr(v), _ptr(params_in), _ptr(out),
                                 _ptr(None if target is None else _f64(target)),
                                 C.byref(scalars))
        return out

    # --------------------------------------------------------- problems
    def minirender_generate(self, P, gen_seed, exponent_max=4.0):
        b, T = np.empty(P), np.empty(P)
        self.lib.mgo_minirender_generate(P, gen_seed, exponent_max, _ptr(b), _ptr(T))
        return b, T

    def minirender_kernel_terms(self, exponents, uniforms, spp):
        P = exponents.size
        cross, mb = np.empty(P), np.empty(P)
        self.lib.mgo_minirender_kernel_terms(P, spp, _ptr(_f64(exponents)), _ptr(_f64(uniforms)),
                                             _ptr(cross), _ptr(mb))
        return cross, mb

    def minirender_sample_pair(self, spp, exponents, target, now, prev, seed, rep, skip=0):
        P = exponents.size
        g = self.new_stream(seed, rep)
        f = self.lib.mgo_minirender_sample_pair
        f.restype = C.c_double
        f.argtypes = [C.c_int32, C.c_int32] + [C.c_void_p] * 7
        args = [_ptr(_f64(exponents)), _ptr(_f64(target)), g, _ptr(_f64(now)), _ptr(_f64(prev))]
        prop, diff = np.empty(P), np.empty(P)
        ssn = None
        for _ in range(skip + 1):
            ssn = f(P, spp, *args, _ptr(prop), _ptr(diff))
        return prop, diff, ssn

    def exprate_sample_pair(self, target_mean, n, rate_now, rate_prev, seed, rep, skip=0):
        g = self.new_stream(seed, rep)
        f = self.lib.mgo_exprate_sample_pair
        f.argtypes = [C.c_double, C.c_int32, C.c_void_p, C.c_double, C.c_double, _dp, _dp, _dp]
        p, d, s = C.c_double(), C.c_double(), C.c_double()
        rc = 0
        for _ in range(skip + 1):
            rc = f(target_mean, n, g, rate_now, rate_prev, C.byref(p), C.byref(d), C.byref(s))
        return p.value, d.value, s.value, rc

    def multnoise_sample_pair(self, sigma, n, target, now, prev, seed, rep, skip=0):
        d = target.size
        g = self.new_stream(seed, rep)
        f = self.lib.mgo_multnoise_sample_pair
        f.restype = C.c_double
        f.argtypes = [C.c_int32, C.c_double, C.c_int32] + [C.c_void_p] * 6
        prop, diff = np.empty(d), np.empty(d)
        ssn = None
        for _ in range(skip + 1):
            ssn = f(d, sigma, n, _ptr(_f64(target)), g, _ptr(_f64(now)), _ptr(_f64(prev)),
                    _ptr(prop), _ptr(diff))
        return prop, diff, ssn

    # ------------------------------------------------------ F1 quad slice
    def quad_render(self, W, H, R, tex, Le, spp, key, stream):
        f = self.lib.mgo_quad_render
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_uint64,
                      C.c_uint32, C.c_void_p]
        img = np.empty(3 * W * H)
        le = _f64(Le)
        f(W, H, R, _ptr(_f64(tex)), _ptr(le), spp, key, stream, _ptr(img))
        return img

    def quad_sample_pair(self, W, H, R, Le, target_img, now, prev, key, it, stream=0):
        f = self.lib.mgo_quad_sample_pair
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, _dp]
        n = 3 * R * R
        prop, diff, loss = np.empty(n), np.empty(n), C.c_double()
        f(W, H, R, _ptr(_f64(Le)), _ptr(_f64(target_img)), _ptr(_f64(now)), _ptr(_f64(prev)),
          key, it, stream, _ptr(prop), _ptr(diff), C.byref(loss))
        return prop, diff, loss.value

    def helix_render(self, W, H, sph, Le, env, ground, theta, spp, key):
        f = self.lib.mgo_helix_render
        f.argtypes = [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 5 + [C.c_int, C.c_uint64,
                                                                      C.c_void_p]
        img = np.empty(3 * W * H)
        sph = _f64(sph)
        f(W, H, sph.shape[0], _ptr(sph), _ptr(_f64(Le)), _ptr(_f64(env)), _ptr(_f64(ground)),
          _ptr(_f64(theta)), spp, key, _ptr(img))
        return img

    def helix_sample_pair(self, W, H, sph, Le, env, ground, target_img, now, prev, key, it):
        f = self.lib.mgo_helix_sample_pair
        f.argtypes = [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 7 + [C.c_uint64, C.c_uint32,
                                                                      C.c_void_p, C.c_void_p, _dp]
        prop, diff, loss = np.empty(5), np.empty(5), C.c_double()
        sph = _f64(sph)
        f(W, H, sph.shape[0], _ptr(sph), _ptr(_f64(Le)), _ptr(_f64(env)), _ptr(_f64(ground)),
          _ptr(_f64(target_img)), _ptr(_f64(now)), _ptr(_f64(prev)), key, it, _ptr(prop),
          _ptr(diff), C.byref(loss))
        return prop, diff, loss.value

    # ------------------------------------------------- F1 slice 3: meshes
    def mesh_closest_hit(self, rec, o, d):
        f = self.lib.mgo_mesh_closest_hit
        f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, _dp, _dp, _dp]
        f.restype = C.c_int
        t, u, v = C.c_double(), C.c_double(), C.c_double()
        rec = _f64(rec)
        k = f(rec.shape[0], _ptr(rec), _ptr(_f64(o)), _ptr(_f64(d)), C.byref(t), C.byref(u),
              C.byref(v))
        return k, t.value

    def mesh_render(self, W, H, rec, obj, R, view, theta, spp, key):
        f = self.lib.mgo_mesh_render
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                      C.c_void_p, C.c_int, C.c_uint64, C.c_void_p]
        img = np.empty(3 * W * H)
        rec = _f64(rec)
        obj = np.ascontiguousarray(obj, dtype=np.int32)
        f(W, H, rec.shape[0], _ptr(rec), obj.ctypes.data_as(C.c_void_p), R, _ptr(_f64(view)),
          _ptr(_f64(theta)), spp, key, _ptr(img))
        return img

    def mesh_sample_pair(self, W, H, rec, obj, nobj, R, view, target_img, now, prev, key, it,
                         rows=None):
        f = self.lib.mgo_mesh_sample_pair
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                      C.c_int, C.c_int, C.c_void_p, C.c_void_p, _dp]
        r0, r1 = rows if rows is not None else (0, H)
        n = nobj * 4 * R * R
        prop, diff, loss = np.empty(n), np.empty(n), C.c_double()
        rec = _f64(rec)
        obj = np.ascontiguousarray(obj, dtype=np.int32)
        f(W, H, rec.shape[0], _ptr(rec), obj.ctypes.data_as(C.c_void_p), nobj, R, _ptr(_f64(view)),
          _ptr(_f64(target_img)), _ptr(_f64(now)), _ptr(_f64(prev)), key, it, r0, r1, _ptr(prop),
          _ptr(diff), C.byref(loss))
        return prop, diff, loss.value

    def meshx_render(self, W, H, rec, obj, nch, R, view, theta, spp, key):
        f = self.lib.mgo_meshx_render
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                      C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_void_p]
        img = np.empty(3 * W * H)
        rec = _f64(rec)
        obj = np.ascontiguousarray(obj, dtype=np.int32)
        f(W, H, rec.shape[0], _ptr(rec), obj.ctypes.data_as(C.c_void_p), nch, R, _ptr(_f64(view)),
          _ptr(_f64(theta)), spp, key, _ptr(img))
        return img

    def meshx_sample_pair(self, W, H, rec, obj, nobj, nch, R, view, target_img, now, prev, key,
                          it, nprop, rows=None):
        f = self.lib.mgo_meshx_sample_pair
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                      C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                      C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, _dp]
        r0, r1 = rows if rows is not None else (0, H)
        n = nobj * nch * R * R
        prop, diff, loss = np.empty(n), np.empty(n), C.c_double()
        rec = _f64(rec)
        obj = np.ascontiguousarray(obj, dtype=np.int32)
        f(W, H, rec.shape[0], _ptr(rec), obj.ctypes.data_as(C.c_void_p), nobj, nch, R,
          _ptr(_f64(view)), _ptr(_f64(target_img)), _ptr(_f64(now)), _ptr(_f64(prev)), key, it,
          r0, r1, nprop, _ptr(prop), _ptr(diff), C.byref(loss))
        return prop, diff, loss.value

    def meshx_path_radiance(self, W, H, rec, obj, nch, R, view, theta, px, py, key, it, path):
        f = self.lib.mgo_meshx_path_radiance
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                      C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32,
                      C.c_uint32, C.c_void_p]
        f.restype = C.c_int
        L = np.empty(3)
        rec = _f64(rec)
        obj = np.ascontiguousarray(obj, dtype=np.int32)
        nv = f(W, H, rec.shape[0], _ptr(rec), obj.ctypes.data_as(C.c_void_p), nch, R,
               _ptr(_f64(view)), _ptr(_f64(theta)), px, py, key, it, path, _ptr(L))
        return L, nv

    def mesh_path_radiance(self, W, H, rec, obj, R, view, theta, px, py, key, it, path):
        f = self.lib.mgo_mesh_path_radiance
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                      C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]
        f.restype = C.c_int
        L = np.empty(3)
        rec = _f64(rec)
        obj = np.ascontiguousarray(obj, dtype=np.int32)
        nv = f(W, H, rec.shape[0], _ptr(rec), obj.ctypes.data_as(C.c_void_p), R, _ptr(_f64(view)),
               _ptr(_f64(theta)), px, py, key, it, path, _ptr(L))
        return L, nv

    # ----------------------------------------------------------- harness
    def run_single(self, cfg, replicate):
        dim = self.lib.mgo_problem_dim(C.byref(cfg))
        it = cfg.iterations
        names = ("params", "loss", "prop", "diff", "ssn", "mean_est", "var_est", "alpha",
                 "delta", "true_grad")
        vec = {"params", "prop", "diff", "mean_est", "var_est", "alpha", "delta", "true_grad"}
        bufs = {k: np.full((it, dim) if k in vec else (it,), np.nan) for k in names}

        class Full(C.Structure):
            _fields_ = [(k, C.c_void_p) for k in names]
        full = Full(*[_ptr(bufs[k]) for k in names])
        rec = _abi.RunRecordC()
        rc = self.lib.mgo_run_single(C.byref(cfg), replicate, C.byref(rec), C.byref(full))
        n = rec.iterations_run
        out = {k: v[:n] for k, v in bufs.items()}
        out.update(status=rec.status, iterations_run=n, draws_used=rec.draws_used,
                   evals_used=rec.evals_used, rc=rc)
        return out

    def run_series(self, cfg, replicates):
        """Coordinate series for replicates [0, replicates): dict name -> [R][it]."""
        it = cfg.iterations
        dim = self.lib.mgo_problem_dim(C.byref(cfg))
        out = {n: np.full((replicates, it), np.nan) for n in _abi.SERIES_NAMES}
        recs = []
        finals = np.full((replicates, dim), np.nan)
        for r in range(replicates):
            s = _abi.RunSeriesC(*[_ptr(out[n][r]) for n in _abi.SERIES_NAMES])
            rec = _abi.RunRecordC()
            fp = np.empty(dim)
            rc = self.lib.mgo_run_single_series(C.byref(cfg), r, C.byref(rec), C.byref(s), 1,
                                                _ptr(fp))
            if rc:
                raise RuntimeError(f"oracle run_single failed rc={rc}")
            finals[r] = fp
            recs.append((rec.iterations_run, rec.status, rec.draws_used, rec.evals_used))
        return out, recs, finals


class RefLib:
    """ctypes view of oracle/ref/ref_capi.cpp over the unmodified reference."""

    def __init__(self, path=REF_SO):
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int64, C.c_void_p]
        L.ref_minirender_gen.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_minirender_kernel_terms.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double,
                                                  C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_minirender_sample_pair.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double,
                                                 C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                                 C.c_int, C.c_void_p, C.c_void_p, _dp]
        L.ref_exprate_sample_pair.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double,
                                              C.c_uint64, C.c_uint64, C.c_int, _dp, _dp, _dp]
        L.ref_multnoise_sample_pair.argtypes = [C.c_int, C.c_double, C.c_int, C.c_void_p,
                                                C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                                C.c_int, C.c_void_p, C.c_void_p, _dp]
        L.ref_moment2_run.argtypes = [C.c_double, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_meta_step.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int,
                                    C.c_int] + [C.c_void_p] * 5 + [C.c_double] + [C.c_void_p] * 3
        L.ref_adam_run.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_run_single.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64)] + [C.c_void_p] * 10
        L.ref_run_experiment.argtypes = [C.c_char_p, C.c_char_p, _dp, C.POINTER(C.c_int)]
        L.ref_meta_update_bench.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_void_p, C.c_void_p, C.c_double, _dp, _dp]
        L.ref_validation_suite.argtypes = [C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int)]

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"reference raised (rc={rc}): {self.lib.ref_last_error().decode()}")

    def rng_draws(self, seed, rep, mode, n):
        out = np.empty(n, dtype=np.uint64 if mode in (0, 1) else np.float64)
        self.lib.ref_rng_draws(seed, rep, mode, n, _ptr(out))
        return out

    def minirender_gen(self, P, spp, gen_seed, albedo_init=0.1, exponent_max=4.0):
        b, T, init = np.empty(P), np.empty(P), np.empty(P)
        self._check(self.lib.ref_minirender_gen(P, spp, gen_seed, albedo_init, exponent_max,
                                                _ptr(b), _ptr(T), _ptr(init)))
        return b, T, init

    def minirender_kernel_terms(self, P, spp, gen_seed, uniforms, exponent_max=4.0):
        cross, mb = np.empty(P), np.empty(P)
        self._check(self.lib.ref_minirender_kernel_terms(P, spp, gen_seed, exponent_max,
                                                         _ptr(_f64(uniforms)), _ptr(cross),
                                                         _ptr(mb)))
        return cross, mb

    def minirender_sample_pair(self, P, spp, gen_seed, now, prev, seed, rep, skip=0,
                               exponent_max=4.0):
        prop, diff, ssn = np.empty(P), np.empty(P), C.c_double()
        self._check(self.lib.ref_minirender_sample_pair(P, spp, gen_seed, exponent_max,
                                                        _ptr(_f64(now)), _ptr(_f64(prev)), seed,
                                                        rep, skip, _ptr(prop), _ptr(diff),
                                                        C.byref(ssn)))
        return prop, diff, ssn.value

    def exprate_sample_pair(self, target_mean, n, rate_now, rate_prev, seed, rep, skip=0):
        p, d, s = C.c_double(), C.c_double(), C.c_double()
        rc = self.lib.ref_exprate_sample_pair(target_mean, n, rate_now, rate_prev, seed, rep,
                                              skip, C.byref(p), C.byref(d), C.byref(s))
        return p.value, d.value, s.value, rc

    def multnoise_sample_pair(self, sigma, n, target, now, prev, seed, rep, skip=0):
        dim = target.size
        prop, diff, ssn = np.empty(dim), np.empty(dim), C.c_double()
        self._check(self.lib.ref_multnoise_sample_pair(dim, sigma, n, _ptr(_f64(target)),
                                                       _ptr(_f64(now)), _ptr(_f64(prev)), seed,
                                                       rep, skip, _ptr(prop), _ptr(diff),
                                                       C.byref(ssn)))
        return prop, diff, ssn.value

    def moment2_run(self, decay, xs):
        xs = _f64(xs)
        out = np.empty_like(xs)
        self._check(self.lib.ref_moment2_run(decay, xs.shape[1], xs.shape[0], _ptr(xs),
                                             _ptr(out)))
        return out

    def meta_step(self, lr, eps_step, eps_alpha, clip, state, prop, diff, ssn, var_prop,
                  var_diff):
        prop = _f64(prop)
        n = prop.size
        has = state is not None
        st = {k: (_f64(state[k]).copy() if has else np.zeros(n))
              for k in ("mean", "var", "alpha_prev")}
        delta = np.empty(n)
        rc = self.lib.ref_meta_step(n, lr, eps_step, eps_alpha, int(clip), int(has),
                                    _ptr(st["mean"]), _ptr(st["var"]), _ptr(st["alpha_prev"]),
                                    _ptr(prop), _ptr(_f64(diff)), ssn, _ptr(_f64(var_prop)),
                                    _ptr(_f64(var_diff)), _ptr(delta))
        return st, delta, rc

    def adam_run(self, grads, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8):
        grads = _f64(grads)
        steps, n = grads.shape
        m, v, d = np.empty(n), np.empty(n), np.empty(n)
        self._check(self.lib.ref_adam_run(n, steps, lr, beta1, beta2, eps, _ptr(grads), _ptr(m),
                                          _ptr(v), _ptr(d)))
        return m, v, d

    def run_single(self, cfg_kw, replicate):
        text = _abi.config_text(**cfg_kw).encode()
        cfg = _abi.config_from(**cfg_kw)
        dim = {0: 1, 1: cfg.dim, 2: cfg.pixel_count}[cfg.problem]
        it = cfg.iterations
        names = ("params", "loss", "prop", "diff", "ssn", "mean_est", "var_est", "alpha",
                 "delta", "true_grad")
        vec = {"params", "prop", "diff", "mean_est", "var_est", "alpha", "delta", "true_grad"}
        bufs = {k: np.full((it, dim) if k in vec else (it,), np.nan) for k in names}
        iters, status = C.c_int(), C.c_int()
        draws, evals = C.c_int64(), C.c_int64()
        self._check(self.lib.ref_run_single(text, replicate, C.byref(iters), C.byref(status),
                                            C.byref(draws), C.byref(evals),
                                            *[_ptr(bufs[k]) for k in names]))
        n = iters.value
        out = {k: v[:n] for k, v in bufs.items()}
        out.update(status=status.value, iterations_run=n, draws_used=draws.value,
                   evals_used=evals.value)
        return out

    def run_experiment_seconds(self, cfg_kw, csv_path=None):
        sec, div = C.c_double(), C.c_int()
        self._check(self.lib.ref_run_experiment(_abi.config_text(**cfg_kw).encode(),
                                                (csv_path or "").encode(), C.byref(sec),
                                                C.byref(div)))
        return sec.value, div.value

    def meta_update_bench(self, props, diffs, ssn, steps, threads, warmup=0):
        """Seconds per timed step (mean, median) of the reference's meta
        update over `threads` contiguous chunks; props/diffs [pool][n]."""
        props, diffs = _f64(props), _f64(diffs)
        pool, n = props.shape
        out, med = C.c_double(), C.c_double()
        self._check(self.lib.ref_meta_update_bench(n, warmup, steps, threads, pool, _ptr(props),
                                                   _ptr(diffs), ssn, C.byref(out), C.byref(med)))
        return out.value, med.value


def ref_available():
    return os.path.exists(REF_SO)
