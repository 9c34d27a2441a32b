"""Host-side mirror of the reference `metagrad` API for the hot path, backed by
the sm_100a kernels behind include/mgcuda.h.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/metagrad/*.hpp):

  Rng.stream(seed, r)                      rng.hpp:23-25   (device mt19937_64)
  Moment2(decay).step(x)                   moment2.hpp:21-50
  GradientSamplePair(prop, diff, ssn)      meta.hpp:20-24
  MetaEstimator(lr, ...).step(pair, vp, vd) meta.hpp:71-114 (mean/var/alpha_prev injectable)
  Adam(lr, b1, b2, eps).step(grad)         adam.hpp:14-50
  MiniRenderProblem / ExpRateProblem / MultNoiseQuadratic .sample_pair(now, prev, rng)
                                           problems.hpp:74-195
  FusedMetaUpdate                          the one-pass hot path (harness.cpp:144-188)
  ExperimentConfig, run_single, run_experiment   harness.hpp:18-112

Vectors are torch CUDA tensors (float64 = parity mode, float32 = fast mode);
torch is only the device-memory/stream plumbing.  Exceptions: InvalidArgument
(std::invalid_argument), LogicError (std::logic_error), DomainError
(std::domain_error).  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np
import torch

from . import _abi
from ._lib import DomainError, InvalidArgument, LogicError, MgError, check, load  # noqa: F401

__all__ = ["Context", "Rng", "Moment2", "GradientSamplePair", "MetaEstimator", "Adam",
           "MiniRenderProblem", "ExpRateProblem", "MultNoiseQuadratic", "FusedMetaUpdate",
           "FusedAdamUpdate", "MiniRenderRun", "QuadTextureProblem", "QuadTextureRun",
           "HelixProblem", "HelixRun", "helix_spheres", "MeshScene", "MeshTextureProblem",
           "MeshTextureRun", "mesh_scene_geometry", "mesh_scene_view", "smooth_noise_textures",
           "MeshLargeProblem", "mesh_large_scene_geometry", "large_scene_view",
           "ExperimentConfig", "RunRecord", "AggregateReport", "run_single",
           "run_experiment", "InvalidArgument", "LogicError", "DomainError", "mix64"]


def _p(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise InvalidArgument(_abi.MG_EINVAL, "tensor must be on the CUDA device")
    if not t.is_contiguous():
        raise InvalidArgument(_abi.MG_EINVAL, "tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return _abi.MG_F64
    if t.dtype == torch.float32:
        return _abi.MG_F32
    raise InvalidArgument(_abi.MG_EINVAL, f"unsupported dtype {t.dtype} (float32/float64)")


class Context:
    """One device + the current torch stream (mg_ctx_create)."""

    _default: Dict[int, "Context"] = {}

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        L = load()
        self.device = device
        torch.cuda.set_device(device)
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        h = C.c_void_p()
        # torch's default stream is the legacy NULL stream: adopt it as
        # cudaStreamLegacy ((void*)1) so our kernels stay ordered with torch's
        # copies (NULL would make mg_ctx_create create a private stream).
        check(L.mg_ctx_create(device, C.c_void_p(s.cuda_stream or 1), C.byref(h)))
        self.h = h

    @classmethod
    def default(cls, device: Optional[int] = None) -> "Context":
        dev = torch.cuda.current_device() if device is None else device
        if dev not in cls._default:
            cls._default[dev] = Context(dev)
        return cls._default[dev]

    def synchronize(self):
        check(load().mg_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(load().mg_ctx_launch_count(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load().mg_ctx_destroy(self.h)
        except Exception:
            pass


def mix64(x: int) -> int:
    return int(load().mg_mix64(x))


# ------------------------------------------------------------------- RNG
class Rng:
    """A batch of device std::mt19937_64 engines (rng.hpp:18-37).

    Rng(seed) is one engine seeded with `seed` (rng.hpp:20);
    Rng.stream(seed, r) is the replicate stream (rng.hpp:23-25);
    Rng.streams(seed, reps) batches several replicates."""

    def __init__(self, engine_seeds, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        seeds = np.ascontiguousarray(np.atleast_1d(np.asarray(engine_seeds, dtype=np.uint64)))
        self.n = seeds.size
        h = C.c_void_p()
        check(load().mg_mt64_create(self.ctx.h, self.n, seeds.ctypes.data_as(C.c_void_p),
                                    C.byref(h)))
        self.h = h

    @classmethod
    def stream(cls, base_seed: int, replicate: int, ctx=None) -> "Rng":
        return cls([load().mg_stream_seed(base_seed, replicate)], ctx)

    @classmethod
    def split(cls, engine_seed: int, segments: int, segment_len: int, ctx=None) -> "Rng":
        """`segments` engines at draws c*segment_len of ONE stream seeded with
        engine_seed (GF(2) jump-ahead; mg_mt64_split)."""
        self = cls.__new__(cls)
        self.ctx = ctx or Context.default()
        self.n = segments
        h = C.c_void_p()
        check(load().mg_mt64_split(self.ctx.h, engine_seed, segments, segment_len, C.byref(h)))
        self.h = h
        return self

    def jump(self, distance: int):
        """Advance every engine by `distance` draws (mg_mt64_jump)."""
        check(load().mg_mt64_jump(self.ctx.h, self.h, distance))

    @classmethod
    def streams(cls, base_seed: int, replicates, ctx=None) -> "Rng":
        L = load()
        return cls([L.mg_stream_seed(base_seed, int(r)) for r in replicates], ctx)

    def _draw(self, n: int, kind: int) -> torch.Tensor:
        out = torch.empty((self.n, n), dtype=torch.uint64 if kind == 0 else torch.float64,
                          device=f"cuda:{self.ctx.device}")
        check(load().mg_mt64_draw(self.ctx.h, self.h, n, kind, _p(out)))
        return out

    def raw(self, n: int = 1) -> torch.Tensor:
        return self._draw(n, 0)

    def uniform(self, n: int = 1) -> torch.Tensor:
        return self._draw(n, 1)

    def uniform_pos(self, n: int = 1) -> torch.Tensor:
        return self._draw(n, 2)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load().mg_mt64_destroy(self.h)
        except Exception:
            pass


# ------------------------------------------------------------ estimators
class Moment2:
    """Zero-centred EMA of squares (moment2.hpp:21-50)."""

    def __init__(self, decay: float = 0.9, dim: Optional[int] = None, ctx=None):
        if not (0.0 <= decay < 1.0):
            raise InvalidArgument(_abi.MG_EINVAL, "Moment2: decay must lie in [0, 1)")
        self.ctx = ctx or Context.default()
        self.s = _abi.Moment2Scalars(decay, 1.0, 0)
        self._m2 = None if dim is None else torch.zeros(dim, dtype=torch.float64, device="cuda")

    def step(self, x: torch.Tensor):
        if self.s.count == 0 and (self._m2 is None or self._m2.numel() == 0):
            self._m2 = torch.empty_like(x)
        if x.numel() != self._m2.numel():
            raise InvalidArgument(_abi.MG_EINVAL, "Moment2: sample dimension mismatch")
        if x.dtype != self._m2.dtype:
            self._m2 = self._m2.to(x.dtype)
        check(load().mg_moment2_step(self.ctx.h, _dtype_code(x), x.numel(), C.byref(self.s),
                                     _p(self._m2), _p(x.contiguous())))

    def m2(self) -> torch.Tensor:
        return self._m2 if self._m2 is not None else torch.zeros(0, device="cuda")

    def count(self) -> int:
        return int(self.s.count)

    def decay(self) -> float:
        return float(self.s.decay)


@dataclasses.dataclass
class GradientSamplePair:
    """meta.hpp:20-24"""
    prop: torch.Tensor
    diff: torch.Tensor
    step_sq_norm: float = 0.0


class MetaEstimator:
    """Recurrent gradient meta-estimator (meta.hpp:71-114).  mean, var and
    alpha_prev are public device tensors and may be injected (as the
    reference's tests do, tests/test_meta.cpp:213-218)."""

    def __init__(self, lr: float = 0.001, eps_step: float = 1e-8, eps_alpha: float = 1e-30,
                 ctx=None):
        if not lr > 0.0:
            raise InvalidArgument(_abi.MG_EINVAL, "MetaEstimator: lr must be positive")
        self.ctx = ctx or Context.default()
        self.lr, self.eps_step, self.eps_alpha = lr, eps_step, eps_alpha
        self.clip_enabled = True
        self.mean: Optional[torch.Tensor] = None
        self.var: Optional[torch.Tensor] = None
        self.alpha_prev: Optional[torch.Tensor] = None

    def step(self, sample: GradientSamplePair, var_prop: torch.Tensor,
             var_diff: torch.Tensor) -> torch.Tensor:
        n = sample.prop.numel()
        first = self.mean is None or self.mean.numel() == 0
        if first:
            self.mean = torch.empty_like(sample.prop)
            self.var = torch.empty_like(sample.prop)
            self.alpha_prev = torch.empty_like(sample.prop)
        if (sample.diff.numel() != n or var_prop.numel() != n or var_diff.numel() != n or
                self.mean.numel() != n):
            raise InvalidArgument(_abi.MG_EINVAL, "MetaEstimator: dimension mismatch")
        delta = torch.empty_like(sample.prop)
        p = _abi.MetaParams(self.lr, self.eps_step, self.eps_alpha, int(self.clip_enabled))
        check(load().mg_meta_step(self.ctx.h, _dtype_code(sample.prop), n, C.byref(p),
                                  int(first), _p(self.mean), _p(self.var), _p(self.alpha_prev),
                                  _p(sample.prop), _p(sample.diff), _p(var_prop),
                                  _p(var_diff), _p(delta)))
        return delta


class Adam:
    """Bias-corrected Adam (adam.hpp:14-50)."""

    def __init__(self, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 ctx=None):
        if not lr > 0.0:
            raise InvalidArgument(_abi.MG_EINVAL, "Adam: lr must be positive")
        if not (0.0 <= beta1 < 1.0 and 0.0 <= beta2 < 1.0):
            raise InvalidArgument(_abi.MG_EINVAL, "Adam: betas must lie in [0, 1)")
        self.ctx = ctx or Context.default()
        self.s = _abi.AdamScalars(lr, beta1, beta2, eps, 1.0, 1.0, 0)
        self._m = self._v = None

    def step(self, grad: torch.Tensor) -> torch.Tensor:
        if self.s.t == 0 and self._m is None:
            self._m, self._v = torch.empty_like(grad), torch.empty_like(grad)
        if grad.numel() != self._m.numel():
            raise InvalidArgument(_abi.MG_EINVAL, "Adam: gradient dimension mismatch")
        delta = torch.empty_like(grad)
        check(load().mg_adam_step(self.ctx.h, _dtype_code(grad), grad.numel(), C.byref(self.s),
                                  _p(self._m), _p(self._v), _p(grad), _p(delta)))
        return delta

    def t(self) -> int:
        return int(self.s.t)

    def m(self):
        return self._m

    def v(self):
        return self._v

    def m_hat(self):
        return self._m / (1.0 - self.s.beta1_pow) if self.s.t > 0 else self._m

    def v_hat(self):
        return self._v / (1.0 - self.s.beta2_pow) if self.s.t > 0 else self._v


# --------------------------------------------------------------- problems
class _Problem:
    def loss(self, params):
        raise NotImplementedError

    def project(self, params):
        return params


class MiniRenderProblem(_Problem):
    """problems.hpp:157-195 / problems.cpp:162-228, target and exponents
    generated on the device from Rng(mix64(gen_seed))."""

    def __init__(self, pixel_count: int, spp: int, gen_seed: int = 1234, albedo_init: float = 0.1,
                 exponent_max: float = 4.0, ctx=None):
        if pixel_count < 1:
            raise InvalidArgument(_abi.MG_EINVAL, "mini-render: pixel_count must be >= 1")
        if spp < 2:
            raise InvalidArgument(_abi.MG_EINVAL, "mini-render: spp must be at least 2")
        if not exponent_max >= 0.0:
            raise InvalidArgument(_abi.MG_EINVAL, "mini-render: exponent_max must be >= 0")
        self.ctx = ctx or Context.default()
        self.pixel_count, self.spp_, self.albedo_init = pixel_count, spp, albedo_init
        self.exponents = torch.empty(pixel_count, dtype=torch.float64, device="cuda")
        self.target = torch.empty(pixel_count, dtype=torch.float64, device="cuda")
        check(load().mg_minirender_generate(self.ctx.h, pixel_count, gen_seed, exponent_max,
                                            _p(self.exponents), _p(self.target)))

    def name(self):
        return "mini-render"

    def dim(self):
        return self.pixel_count

    def spp(self):
        return self.spp_

    def draws_per_sample(self):
        return self.pixel_count * self.spp_

    def initial_params(self, dtype=torch.float64):
        return torch.full((self.pixel_count,), self.albedo_init, dtype=dtype, device="cuda")

    def truth_params(self):
        return self.target

    def target_image(self):
        return self.target

    def shape_exponents(self):
        return self.exponents

    def sample_pair(self, params_now, params_prev, rng: Rng):
        """One pair per engine in rng: now/prev are [P] or [R, P]."""
        R = rng.n
        now = params_now.reshape(R, -1).contiguous()
        prev = params_prev.reshape(R, -1).contiguous()
        if now.shape[1] != self.pixel_count or prev.shape != now.shape:
            raise InvalidArgument(_abi.MG_EINVAL, "mini-render: parameter dimension mismatch")
        prop, diff = torch.empty_like(now), torch.empty_like(now)
        ssn = torch.empty(R, dtype=torch.float64, device="cuda")
        check(load().mg_minirender_sample_pair(self.ctx.h, _dtype_code(now), R, self.pixel_count,
                                               self.spp_, _p(self.exponents), _p(self.target),
                                               rng.h, _p(now), _p(prev), _p(prop), _p(diff),
                                               _p(ssn)))
        if R == 1:
            return GradientSamplePair(prop[0], diff[0], float(ssn[0]))
        return GradientSamplePair(prop, diff, ssn)

    def true_gradient(self, params):
        return 2.0 * (params - self.target.to(params.dtype))

    def loss(self, params):
        return float(((params.double() - self.target) ** 2).sum())

    def project(self, params):
        return torch.clamp_min(params, 0.0)


class ExpRateProblem(_Problem):
    """problems.hpp:81-111 / problems.cpp:30-94 (dim 1)."""

    def __init__(self, target_mean: float = 2.0, samples_per_iter: int = 32,
                 rate_init: float = 2.0, ctx=None):
        if not target_mean > 0.0:
            raise InvalidArgument(_abi.MG_EINVAL, "exp-rate: target mean must be positive")
        if samples_per_iter < 2:
            raise InvalidArgument(_abi.MG_EINVAL, "exp-rate: samples_per_iter must be at least 2")
        if not rate_init > 0.0:
            raise InvalidArgument(_abi.MG_EINVAL, "exp-rate: initial rate must be positive")
        self.ctx = ctx or Context.default()
        self.target_mean_, self.n, self.rate_init = target_mean, samples_per_iter, rate_init

    def dim(self):
        return 1

    def draws_per_sample(self):
        return self.n

    def sample_pair(self, now, prev, rng: Rng):
        R = rng.n
        now = now.reshape(R).double().contiguous()
        prev = prev.reshape(R).double().contiguous()
        prop, diff, ssn = (torch.empty(R, dtype=torch.float64, device="cuda") for _ in range(3))
        check(load().mg_exprate_sample_pair(self.ctx.h, R, self.target_mean_, self.n, rng.h,
                                            _p(now), _p(prev), _p(prop), _p(diff), _p(ssn)))
        return GradientSamplePair(prop, diff, ssn)

    def true_gradient(self, params):
        r = params
        return 2.0 * (1.0 / r - self.target_mean_) * (-1.0 / (r * r))


class MultNoiseQuadratic(_Problem):
    """problems.hpp:118-148 / problems.cpp:99-157."""

    def __init__(self, target: torch.Tensor, noise_amp: float, samples_per_iter: int = 1,
                 ctx=None):
        if target.numel() == 0:
            raise InvalidArgument(_abi.MG_EINVAL, "mult-noise: empty target")
        if noise_amp < 0.0:
            raise InvalidArgument(_abi.MG_EINVAL, "mult-noise: noise amplitude must be >= 0")
        if samples_per_iter < 1:
            raise InvalidArgument(_abi.MG_EINVAL, "mult-noise: samples_per_iter must be >= 1")
        self.ctx = ctx or Context.default()
        self.target = target.double().cuda().contiguous()
        self.sigma, self.n = noise_amp, samples_per_iter

    def dim(self):
        return self.target.numel()

    def draws_per_sample(self):
        return self.n * self.target.numel()

    def sample_pair(self, now, prev, rng: Rng):
        R, d = rng.n, self.target.numel()
        now = now.reshape(R, d).double().contiguous()
        prev = prev.reshape(R, d).double().contiguous()
        prop, diff = torch.empty_like(now), torch.empty_like(now)
        ssn = torch.empty(R, dtype=torch.float64, device="cuda")
        check(load().mg_multnoise_sample_pair(self.ctx.h, R, d, self.sigma, self.n,
                                              _p(self.target), rng.h, _p(now), _p(prev),
                                              _p(prop), _p(diff), _p(ssn)))
        if R == 1:
            return GradientSamplePair(prop[0], diff[0], float(ssn[0]))
        return GradientSamplePair(prop, diff, ssn)


# ------------------------------------------------------- fused hot path
class FusedMetaUpdate:
    """Device-resident state of one meta-estimator run over n parameters and
    the one-pass update of harness.cpp:144-188 (mg_meta_update).

    step(prop, diff, params_in, params_out) runs one iteration; the step norm
    of the NEXT iteration and the loss of the new parameters are reduced on
    the device into self.scalars (mg_update_scalars), so consecutive steps
    need no host synchronisation."""

    def __init__(self, n: int, dtype=torch.float32, lr: float = 0.01, beta_f: float = 0.9,
                 beta_delta: float = 0.5, eps_step: float = 1e-8, eps_alpha: float = 1e-30,
                 clip: bool = True, project_lo: Optional[float] = None,
                 diff_norm: str = "global", ctx=None, device="cuda",
                 project_hi: Optional[float] = None):
        self.ctx = ctx or Context.default()
        self.n, self.dtype = n, dtype
        self.beta_f, self.beta_delta = beta_f, beta_delta
        self.meta = _abi.MetaParams(lr, eps_step, eps_alpha, int(clip))
        self.project_lo, self.project_hi = project_lo, project_hi
        self.diff_norm = _abi.DIFF_NORMS[diff_norm]
        mk = lambda: torch.empty(n, dtype=dtype, device=device)  # noqa: E731
        self.m2_prop, self.m2_diff, self.mean, self.var, self.alpha_prev = (mk() for _ in range(5))
        self.scalars_buf = torch.zeros(C.sizeof(_abi.UpdateScalars) // 8, dtype=torch.float64,
                                       device=device)
        self.reset()

    def reset(self):
        self.t = 0
        self.beta_f_pow = 1.0
        host = _abi.fresh_scalars()
        check(load().mg_scalars_write(self.ctx.h, _p(self.scalars_buf), C.byref(host)))

    def scalars(self) -> _abi.UpdateScalars:
        out = _abi.UpdateScalars()
        check(load().mg_scalars_read(self.ctx.h, _p(self.scalars_buf), C.byref(out)))
        return out

    def args(self, ssn_host: Optional[float] = None) -> _abi.MetaUpdateArgs:
        """Advance the host-side Moment2(beta_f) scalars (moment2.hpp:34-38)."""
        self.t += 1
        self.beta_f_pow *= self.beta_f
        c_prop = (1.0 - self.beta_f) / (1.0 - self.beta_f_pow)
        return _abi.MetaUpdateArgs(
            meta=self.meta, prop_coef=c_prop, beta_delta=self.beta_delta,
            first_step=int(self.t == 1), diff_norm=self.diff_norm,
            project=(2 if self.project_hi is not None else int(self.project_lo is not None)),
            ssn_from_host=int(ssn_host is not None),
            proj_lo=0.0 if self.project_lo is None else self.project_lo,
            ssn_host=0.0 if ssn_host is None else ssn_host,
            proj_hi=0.0 if self.project_hi is None else self.project_hi)

    def step(self, prop, diff, params_in, params_out, target=None, vprop=None, vdiff=None,
             params_prev=None, delta_out=None, ssn_host=None):
        a = self.args(ssn_host)
        x = _abi.MetaExtras(_p(vprop), _p(vdiff), _p(params_prev), _p(target), _p(delta_out))
        check(load().mg_meta_update(self.ctx.h, _dtype_code(prop), self.n, C.byref(a), _p(prop),
                                    _p(diff), _p(self.m2_prop), _p(self.m2_diff), _p(self.mean),
                                    _p(self.var), _p(self.alpha_prev), _p(params_in),
                                    _p(params_out), _p(self.scalars_buf), C.byref(x)))


class FusedAdamUpdate:
    """Adam baseline with the same fused update/reductions (mg_adam_update)."""

    def __init__(self, n: int, dtype=torch.float32, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8,
                 project_lo: Optional[float] = None, ctx=None, device="cuda"):
        self.ctx = ctx or Context.default()
        self.n = n
        self.s = _abi.AdamScalars(lr, beta1, beta2, eps, 1.0, 1.0, 0)
        self.m = torch.empty(n, dtype=dtype, device=device)
        self.v = torch.empty(n, dtype=dtype, device=device)
        self.project_lo = project_lo
        self.scalars_buf = torch.zeros(C.sizeof(_abi.UpdateScalars) // 8, dtype=torch.float64,
                                       device=device)
        host = _abi.fresh_scalars()
        check(load().mg_scalars_write(self.ctx.h, _p(self.scalars_buf), C.byref(host)))

    def step(self, grad, params_in, params_out, target=None):
        check(load().mg_adam_update(self.ctx.h, _dtype_code(grad), self.n, C.byref(self.s),
                                    int(self.project_lo is not None),
                                    0.0 if self.project_lo is None else self.project_lo,
                                    _p(grad), _p(self.m), _p(self.v), _p(params_in),
                                    _p(params_out), _p(target), _p(self.scalars_buf)))


class MiniRenderRun:
    """One mini-render optimisation run at scale, each iteration ONE fused
    kernel (mg_minirender_meta_iteration): sample_pair + Moment2 x2 +
    MetaEstimator + projected update, the pair never leaving registers.

    rng="mt64": the replicate's exact std::mt19937_64 stream (Rng::stream(seed,
    replicate), pixel-major draws, problems.cpp:201-202) — bit-compatible with
    the reference, but the stream is sequential (one CTA draws P*spp values
    per iteration).  rng="philox": counter-based, every pixel draws its own
    uniforms in-kernel (statistically equivalent; the scale mode)."""

    def __init__(self, pixel_count: int, spp: int, gen_seed: int = 1234, albedo_init: float = 0.1,
                 exponent_max: float = 4.0, lr: float = 0.01, beta_f: float = 0.9,
                 beta_delta: float = 0.5, eps_step: float = 1e-8, eps_alpha: float = 1e-30,
                 clip: bool = True, seed: int = 0, replicate: int = 0, rng: str = "philox",
                 dtype=torch.float32, pixel_range=None, mt64_segments=None, ctx=None):
        self.ctx = ctx or Context.default()
        self.problem = MiniRenderProblem(pixel_count, spp, gen_seed, albedo_init, exponent_max,
                                         ctx=self.ctx)
        lo, hi = pixel_range if pixel_range is not None else (0, pixel_count)
        if not 0 <= lo < hi <= pixel_count:
            raise InvalidArgument(_abi.MG_EINVAL, "MiniRenderRun: bad pixel_range")
        self.lo, self.hi, self.P_total = lo, hi, pixel_count
        self.P, self.spp, self.dtype = hi - lo, spp, dtype
        self.b = self.problem.exponents[lo:hi].to(dtype).contiguous()
        self.T = self.problem.target[lo:hi].to(dtype).contiguous()
        self.params = torch.full((self.P,), albedo_init, dtype=dtype, device="cuda")
        pixel_count = self.P
        self.prev = self.params.clone()
        mk = lambda: torch.empty(pixel_count, dtype=dtype, device="cuda")  # noqa: E731
        self.m2_prop, self.m2_diff, self.mean, self.var, self.alpha_prev = (mk() for _ in range(5))
        self.scalars_buf = torch.zeros(C.sizeof(_abi.UpdateScalars) // 8, dtype=torch.float64,
                                       device="cuda")
        check(load().mg_scalars_write(self.ctx.h, _p(self.scalars_buf),
                                      C.byref(_abi.fresh_scalars())))
        self.meta = _abi.MetaParams(lr, eps_step, eps_alpha, int(clip))
        self.beta_f, self.beta_delta = beta_f, beta_delta
        self.rng_kind = {"mt64": _abi.MG_RNG_MT64, "philox": _abi.MG_RNG_PHILOX}[rng]
        self.key = int(load().mg_stream_seed(seed, replicate))
        if self.rng_kind == _abi.MG_RNG_MT64:
            # the replicate's stream covers ALL pixels; a shard reads its slice.
            # D = P*spp draws per iteration come from G engines positioned
            # L = 312*k draws apart on the SAME stream (jump-ahead), each
            # drawing L per iteration, then jumping D - L: bit-identical to
            # the sequential stream, generated in parallel.
            D = self.P_total * spp
            self.D = D
            # one engine draws ~3e5 values in the time a jump takes (~1 ms,
            # latency-bound), so split only large per-iteration blocks; the
            # engines then tile K iterations' worth of the stream (K*D draws,
            # <= ~2 GB of uniforms) so each engine jumps once per K iterations.
            auto = mt64_segments is None and D >= (1 << 20)
            if D >= 312 and (auto or (mt64_segments or 1) > 1):
                gmax = mt64_segments or 592
                K = max(1, min(16, (1 << 28) // D))
                block = K * D
                L = 312 * (-(-(-(-block // gmax)) // 312))
                G = -(-block // L)
                self.rng = Rng.split(int(load().mg_stream_seed(seed, replicate)), G, L,
                                     ctx=self.ctx)
                self.seg_len, self.block_iters = L, K
            else:
                self.rng = Rng.stream(seed, replicate, ctx=self.ctx)
                self.seg_len, self.block_iters = None, 1
            rows = self.rng.n * self.seg_len if self.seg_len else D
            self.u = torch.empty(rows, dtype=torch.float64, device="cuda")
        else:
            self.rng, self.u = None, None
            self.seg_len, self.block_iters = None, 1
        self.t = 0
        self.beta_f_pow = 1.0

    def draws_per_sample(self) -> int:
        return self.P * self.spp

    def step(self, prop_out=None, diff_out=None, record: Optional[int] = None):
        """One iteration.  prop_out/diff_out receive this iteration's sample
        pair: full [P] tensors, or (record=k) one-element tensors receiving
        local pixel k only."""
        self.t += 1
        self.beta_f_pow *= self.beta_f
        upd = _abi.MetaUpdateArgs(meta=self.meta,
                                  prop_coef=(1.0 - self.beta_f) / (1.0 - self.beta_f_pow),
                                  beta_delta=self.beta_delta, first_step=int(self.t == 1),
                                  diff_norm=_abi.MG_DIFF_NORM_GLOBAL, project=1)
        a = _abi.RenderArgs(update=upd, spp=self.spp, rng_kind=self.rng_kind, key=self.key,
                            iteration=self.t - 1, stream=0, pixel_offset=self.lo,
                            record_plus1=0 if record is None else record + 1)
        L = load()
        u = None
        if self.rng is not None:
            k = (self.t - 1) % self.block_iters
            if self.seg_len:
                if k == 0:  # draws for the next K iterations, then jump past them
                    check(L.mg_mt64_draw(self.ctx.h, self.rng.h, self.seg_len, 1, _p(self.u)))
                    self.rng.jump(self.block_iters * self.D - self.seg_len)
            else:
                check(L.mg_mt64_draw(self.ctx.h, self.rng.h, self.D, 1, _p(self.u)))
            u = C.c_void_p(self.u.data_ptr() + 8 * (k * self.D + self.lo * self.spp))
        check(L.mg_minirender_meta_iteration(
            self.ctx.h, _dtype_code(self.params), self.P, C.byref(a), _p(self.b), _p(self.T),
            u, _p(self.params), _p(self.prev), _p(self.m2_prop), _p(self.m2_diff),
            _p(self.mean), _p(self.var), _p(self.alpha_prev), _p(self.scalars_buf),
            _p(prop_out), _p(diff_out)))
        # prev now holds pi_{t+1}: swap roles
        self.params, self.prev = self.prev, self.params

    def scalars(self) -> _abi.UpdateScalars:
        out = _abi.UpdateScalars()
        check(load().mg_scalars_read(self.ctx.h, _p(self.scalars_buf), C.byref(out)))
        return out


# ------------------------------------------------- F1 slice: textured quad
class QuadTextureProblem:
    """BASELINE.json configs[0] ("PR1 ref"): W x H image of one textured quad
    lit by one rectangular area light, direct lighting only, Lambertian BSDF;
    the parameters are an R x R RGB albedo texture ([3][R*R], channel-major).
    The reference has no renderer; scene and estimators are this
    repo's own, restated in oracle/metagrad_oracle.c.

    Textures: Rng(mix64(seed)).uniform() x 3R^2 (init seed 0, target seed 1,
    as the mini-render construction draws, problems.cpp:168-172); the target
    image is a target_spp-sample render of the target texture."""

    STREAM_TARGET = 7

    def __init__(self, width: int = 64, height: int = 64, tex_res: int = 32,
                 light=(8.0, 7.0, 6.0), init_seed: int = 0, target_seed: int = 1,
                 target_spp: int = 1024, dtype=torch.float64, ctx=None):
        self.ctx = ctx or Context.default()
        self.W, self.H, self.R, self.dtype = width, height, tex_res, dtype
        self.Le = (C.c_double * 3)(*light)
        n = 3 * tex_res * tex_res
        L = load()
        self.init = Rng([L.mg_mix64(init_seed)], ctx=self.ctx).uniform(n)[0].to(dtype)
        self.target_tex = Rng([L.mg_mix64(target_seed)], ctx=self.ctx).uniform(n)[0].to(dtype)
        self.target_img = torch.empty(3 * width * height, dtype=dtype, device="cuda")
        check(L.mg_quad_render(self.ctx.h, _dtype_code(self.target_tex), width, height, tex_res,
                               self.Le, target_spp, L.mg_mix64(target_seed), self.STREAM_TARGET,
                               _p(self.target_tex), _p(self.target_img)))
        self.accum = torch.zeros(6 * tex_res * tex_res, dtype=torch.int64, device="cuda")
        self.loss_buf = torch.zeros(1, dtype=torch.float64, device="cuda")

    def dim(self) -> int:
        return 3 * self.R * self.R

    def draws_per_sample(self) -> int:
        """Path samples per iteration: 2 proportional + 1 finite-difference spp."""
        return 3 * self.W * self.H

    def initial_params(self):
        return self.init.clone()

    def truth_params(self):
        return self.target_tex

    def render(self, tex, spp: int, key: int, stream: int = 3):
        img = torch.empty(3 * self.W * self.H, dtype=tex.dtype, device="cuda")
        check(load().mg_quad_render(self.ctx.h, _dtype_code(tex), self.W, self.H, self.R,
                                    self.Le, spp, key, stream, _p(tex.contiguous()), _p(img)))
        return img

    def sample_pair(self, now, prev, iteration: int, key: int, stream: int = 0, rows=None):
        """One gradient sample pair (prop, diff) for the L2 image loss; the
        returned pair's step_sq_norm is left to the fused update (device).
        rows=(r0, r1) restricts it to an image tile (partials of disjoint
        tiles sum exactly to the full pair)."""
        r0, r1 = rows if rows is not None else (0, self.H)
        prop, diff = torch.empty_like(now), torch.empty_like(now)
        check(load().mg_quad_sample_pair(self.ctx.h, _dtype_code(now), self.W, self.H, self.R,
                                         self.Le, _p(self.target_img), _p(now.contiguous()),
                                         _p(prev.contiguous()), key, iteration, stream, r0, r1,
                                         _p(self.accum), _p(prop), _p(diff), _p(self.loss_buf)))
        return GradientSamplePair(prop, diff)


class QuadTextureRun:
    """configs[0] optimisation loop on the device: per iteration one
    gradient-sample-pair launch (render + adjoint scatter) and one fused
    update (meta-estimator, or the Adam baseline), projection max(p, 0)."""

    def __init__(self, problem: QuadTextureProblem, optimizer: str = "meta", lr: float = 0.01,
                 seed: int = 0, replicate: int = 0, **kw):
        self.p = problem
        self.params = problem.initial_params()
        self.prev = self.params.clone()
        self.key = int(load().mg_stream_seed(seed, replicate))
        n = problem.dim()
        if optimizer == "meta":
            self.upd = FusedMetaUpdate(n, dtype=problem.dtype, lr=lr, project_lo=0.0,
                                       ctx=problem.ctx, **kw)
        elif optimizer == "adam":
            self.upd = FusedAdamUpdate(n, dtype=problem.dtype, lr=lr, project_lo=0.0,
                                       ctx=problem.ctx, **kw)
        else:
            raise InvalidArgument(_abi.MG_EINVAL, "optimizer must be meta or adam")
        self.optimizer = optimizer
        self.t = 0

    def step(self):
        pair = self.p.sample_pair(self.params, self.prev if self.optimizer == "meta" else
                                  self.params, self.t, self.key)
        new = self.prev  # ping-pong: pi_{t-1} buffer receives pi_{t+1}
        if self.optimizer == "meta":
            self.upd.step(pair.prop, pair.diff, self.params, new)
        else:
            self.upd.step(pair.prop, self.params, new)
        self.prev, self.params = self.params, new
        self.t += 1
        return pair

    def loss_estimate(self) -> float:
        return float(self.p.loss_buf[0])

    def texture_error(self) -> float:
        return float(torch.linalg.vector_norm((self.params - self.p.target_tex).double()))


def helix_spheres(n: int = 64, radius: float = 0.1, turns: float = 4.0, helix_radius: float = 1.0,
                  y0: float = 0.3, y1: float = 2.3) -> np.ndarray:
    """configs[2] geometry: n spheres evenly along a helix (host libm
    cos/sin, computed once and shared by the device and the oracle)."""
    out = np.empty((n, 4))
    for k in range(n):
        phi = 2.0 * math.pi * turns * k / n
        out[k] = (helix_radius * math.cos(phi), y0 + (y1 - y0) * k / max(n - 1, 1),
                  helix_radius * math.sin(phi), radius)
    return out


class HelixProblem:
    """BASELINE.json configs[2]: a W x H render of a procedural helix of 64
    spheres (radius 0.1, 4 turns) on a diffuse ground plane under one area
    light plus a constant environment, depth-4 path tracing with NEE; the
    spheres' principled BSDF has 5 global parameters theta = (base r, g, b,
    metalness, roughness), initialised U(0,1) from seed 0 against seeded
    target values (seed 1).  Own renderer (oracle
    mgo_helix_*)."""

    def __init__(self, width: int = 256, height: int = 256, light=(10.0, 10.0, 10.0),
                 env=(0.2, 0.2, 0.2), ground=(0.5, 0.5, 0.5), init_seed: int = 0,
                 target_seed: int = 1, target_spp: int = 64, dtype=torch.float64, ctx=None):
        self.ctx = ctx or Context.default()
        self.W, self.H, self.dtype = width, height, dtype
        self.spheres_host = helix_spheres()
        self.spheres = torch.tensor(self.spheres_host, dtype=torch.float64, device="cuda")
        self.Le = (C.c_double * 3)(*light)
        self.env = (C.c_double * 3)(*env)
        self.ground = (C.c_double * 3)(*ground)
        L = load()
        self.init = Rng([L.mg_mix64(init_seed)], ctx=self.ctx).uniform(5)[0].to(dtype)
        tt = Rng([L.mg_mix64(target_seed)], ctx=self.ctx).uniform(5)[0]
        tt[4] = 0.3 + 0.7 * tt[4]  # target roughness in [0.3, 1] (well-conditioned highlights)
        self.target_theta = tt.to(dtype)
        self.target_img = self.render(self.target_theta, target_spp, int(L.mg_mix64(target_seed)))
        self.accum = torch.zeros(10, dtype=torch.int64, device="cuda")
        self.loss_buf = torch.zeros(1, dtype=torch.float64, device="cuda")

    def dim(self) -> int:
        return 5

    def draws_per_sample(self) -> int:
        """Paths per iteration: 2 proportional + 1 finite-difference spp."""
        return 3 * self.W * self.H

    def initial_params(self):
        return self.init.clone()

    def render(self, theta, spp: int, key: int):
        img = torch.empty(3 * self.W * self.H, dtype=theta.dtype, device="cuda")
        check(load().mg_helix_render(self.ctx.h, _dtype_code(theta), self.W, self.H,
                                     self.spheres.shape[0], _p(self.spheres), self.Le, self.env,
                                     self.ground, _p(theta.contiguous()), spp, key, _p(img)))
        return img

    def sample_pair(self, now, prev, iteration: int, key: int, rows=None):
        r0, r1 = rows if rows is not None else (0, self.H)
        prop, diff = torch.empty_like(now), torch.empty_like(now)
        check(load().mg_helix_sample_pair(
            self.ctx.h, _dtype_code(now), self.W, self.H, self.spheres.shape[0], _p(self.spheres),
            self.Le, self.env, self.ground, _p(self.target_img), _p(now.contiguous()),
            _p(prev.contiguous()), key, iteration, r0, r1, _p(self.accum), _p(prop), _p(diff),
            _p(self.loss_buf)))
        return GradientSamplePair(prop, diff)


class HelixRun(QuadTextureRun):
    """configs[2] optimisation loop (same structure as QuadTextureRun); the 5
    parameters (colours, metalness, roughness) are projected to [0, 1]."""

    def __init__(self, problem, optimizer: str = "meta", lr: float = 0.01, seed: int = 0,
                 replicate: int = 0, **kw):
        if optimizer == "meta":
            kw.setdefault("project_hi", 1.0)
        super().__init__(problem, optimizer, lr, seed, replicate, **kw)


# ------------------------------------- F1 slice 3: textured mesh scene
MESH_VIEW_LAYOUT = ("cam[3] fwd[3] right[3] up[3] tan_half_fov light_y light_x0 light_x1 "
                    "light_z0 light_z1 Le[3] env[3] max_vertices")


def _sphere_triangles(center, radius_fn, n_theta: int, n_phi: int):
    """UV-sphere tessellation: (v0, v1, v2, uv0, uv1, uv2) lists; single
    triangles at the poles (no degenerate ones).  uv = (phi/2pi, theta/pi)."""
    th = np.pi * np.arange(n_theta + 1) / n_theta
    ph = 2.0 * np.pi * np.arange(n_phi + 1) / n_phi
    T_, P_ = np.meshgrid(th, ph, indexing="ij")
    rad = radius_fn(T_, P_)
    pos = np.stack([center[0] + rad * np.sin(T_) * np.cos(P_), center[1] + rad * np.cos(T_),
                    center[2] + rad * np.sin(T_) * np.sin(P_)], axis=-1)
    uv = np.stack([P_ / (2.0 * np.pi), T_ / np.pi], axis=-1)
    tris = []
    for i in range(n_theta):
        for j in range(n_phi):
            a, b, c, d = (i, j), (i, j + 1), (i + 1, j), (i + 1, j + 1)
            if i != 0:
                tris.append((a, b, d))
            if i != n_theta - 1:
                tris.append((a, d, c))
    v = np.array([[pos[k] for k in t] for t in tris])
    w = np.array([[uv[k] for k in t] for t in tris])
    return v, w


def mesh_scene_geometry(sphere_res=(24, 48), displaced_res=(100, 100), seed: int = 3,
                        displacement: float = 0.12):
    """BASELINE.json configs[3] geometry (seed-generated):
    object 0 a ground quad (y = 0, x, z in [-2.5, 2.5]), object 1 a sphere
    (centre (-0.9, 0.5, 0), radius 0.5), object 2 a seeded displaced sphere
    (centre (0.8, 0.55, 0.1), radius 0.5 (1 + displacement * noise),
    ~2 * n_theta * n_phi triangles: 19.8k at the default 100 x 100).
    Returns (records [T][18] fp64, object ids [T] int32, nobj)."""
    quad_v = np.array([[[-2.5, 0.0, -2.5], [2.5, 0.0, -2.5], [2.5, 0.0, 2.5]],
                       [[-2.5, 0.0, -2.5], [2.5, 0.0, 2.5], [-2.5, 0.0, 2.5]]])
    quad_w = (quad_v[:, :, [0, 2]] + 2.5) / 5.0
    sph_v, sph_w = _sphere_triangles((-0.9, 0.5, 0.0), lambda t, p: 0.5 + 0.0 * t, *sphere_res)
    rs = np.random.RandomState(seed)
    waves = [(rs.uniform(-1, 1), rs.randint(1, 6), rs.randint(1, 7), rs.uniform(0, 2 * np.pi))
             for _ in range(6)]

    def disp(t, p):
        noise = sum(a * np.sin(m * t) * np.cos(g * p + q) for a, m, g, q in waves) / len(waves)
        return 0.5 * (1.0 + displacement * noise * 2.0)
    dsp_v, dsp_w = _sphere_triangles((0.8, 0.55, 0.1), disp, *displaced_res)
    V = np.concatenate([quad_v, sph_v, dsp_v])
    Wuv = np.concatenate([quad_w, sph_w, dsp_w])
    obj = np.concatenate([np.zeros(len(quad_v)), np.ones(len(sph_v)),
                          np.full(len(dsp_v), 2)]).astype(np.int32)
    e1 = V[:, 1] - V[:, 0]
    e2 = V[:, 2] - V[:, 0]
    n = np.cross(e1, e2)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    rec = np.concatenate([V[:, 0], e1, e2, n, Wuv[:, 0], Wuv[:, 1] - Wuv[:, 0],
                          Wuv[:, 2] - Wuv[:, 0]], axis=1)
    return np.ascontiguousarray(rec), obj, 3


def mesh_large_scene_geometry(n_spheres: int = 15, res=(130, 130), seed: int = 5,
                              displacement: float = 0.15):
    """BASELINE.json configs[4] geometry: object 0 a ground quad, objects
    1..n_spheres seeded displaced spheres (radius 0.35) on a 5-wide grid —
    16 objects and ~502k triangles at the default 130 x 130 tessellation."""
    quad_v = np.array([[[-3.0, 0.0, -2.5], [3.0, 0.0, -2.5], [3.0, 0.0, 2.5]],
                       [[-3.0, 0.0, -2.5], [3.0, 0.0, 2.5], [-3.0, 0.0, 2.5]]])
    quad_w = np.stack([(quad_v[:, :, 0] + 3.0) / 6.0, (quad_v[:, :, 2] + 2.5) / 5.0], axis=-1)
    rs = np.random.RandomState(seed)
    Vs, Ws, objs = [quad_v], [quad_w], [np.zeros(2)]
    for k in range(n_spheres):
        cx = -2.0 + 1.0 * (k % 5) + rs.uniform(-0.1, 0.1)
        cz = -1.2 + 1.0 * (k // 5) + rs.uniform(-0.1, 0.1)
        waves = [(rs.uniform(-1, 1), rs.randint(1, 6), rs.randint(1, 7), rs.uniform(0, 2 * np.pi))
                 for _ in range(5)]

        def rad(t, p, waves=waves):
            noise = sum(a * np.sin(m * t) * np.cos(g * p + q) for a, m, g, q in waves) / len(waves)
            return 0.35 * (1.0 + displacement * noise * 2.0)
        v, w = _sphere_triangles((cx, 0.4, cz), rad, *res)
        Vs.append(v)
        Ws.append(w)
        objs.append(np.full(len(v), k + 1))
    V, Wuv = np.concatenate(Vs), np.concatenate(Ws)
    obj = np.concatenate(objs).astype(np.int32)
    e1 = V[:, 1] - V[:, 0]
    e2 = V[:, 2] - V[:, 0]
    n = np.cross(e1, e2)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    rec = np.concatenate([V[:, 0], e1, e2, n, Wuv[:, 0], Wuv[:, 1] - Wuv[:, 0],
                          Wuv[:, 2] - Wuv[:, 0]], axis=1)
    return np.ascontiguousarray(rec), obj, n_spheres + 1


def mesh_scene_view(max_vertices: int = 6, light=(6.0, 6.0, 6.0), env=(0.25, 0.3, 0.35),
                    cam=(0.0, 1.6, 4.5), look_at=(0.0, 0.45, 0.0), tan_half_fov: float = 0.45,
                    light_y: float = 3.0, light_rect=(-1.0, 1.0, -1.0, 1.0)):
    """view[25] (layout MESH_VIEW_LAYOUT): pinhole camera, rectangular light
    at y = light_y over x in [x0, x1], z in [z0, z1] facing down, constant
    environment."""
    cam = np.asarray(cam, dtype=np.float64)
    fwd = np.asarray(look_at, dtype=np.float64) - cam
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, [0.0, 1.0, 0.0])
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    return np.concatenate([cam, fwd, right, up, [tan_half_fov, light_y, *light_rect],
                           light, env, [float(max_vertices)]]).astype(np.float64)


def smooth_noise_textures(nobj: int, R: int, seed: int, grid: int = 6,
                          base_range=(0.15, 0.85), rough_range=(0.25, 0.9), channels: int = 4,
                          metal_range=(0.0, 0.6)) -> np.ndarray:
    """Seeded smooth-noise textures [nobj][channels][R*R] (bilinear upsampling
    of a grid x grid lattice of uniforms): base colour, roughness and (5
    channels) metalness."""
    rs = np.random.RandomState(seed)
    x = (np.arange(R) + 0.5) / R * (grid - 1)
    i0 = np.minimum(x.astype(int), grid - 2)
    f = x - i0
    out = np.empty((nobj, channels, R * R))
    for o in range(nobj):
        for c in range(channels):
            g = rs.uniform(0, 1, (grid, grid))
            rows = g[i0] * (1 - f)[:, None] + g[i0 + 1] * f[:, None]
            img = rows[:, i0] * (1 - f)[None, :] + rows[:, i0 + 1] * f[None, :]
            lo, hi = base_range if c < 3 else (rough_range if c == 3 else metal_range)
            out[o, c] = (lo + (hi - lo) * img).reshape(-1)
    return out


class MeshScene:
    """A triangle scene on the device (BVH built on the host, mg_meshscene_*)."""

    def __init__(self, records: np.ndarray, obj: np.ndarray, nobj: int, tex_res: int, view,
                 ctx=None, channels: int = 4):
        self.ctx = ctx or Context.default()
        self.records = np.ascontiguousarray(records, dtype=np.float64)
        self.obj = np.ascontiguousarray(obj, dtype=np.int32)
        self.nobj, self.R, self.channels = nobj, tex_res, channels
        self.view = np.ascontiguousarray(view, dtype=np.float64)
        h = C.c_void_p()
        check(load().mg_meshscene_create(self.ctx.h, self.records.shape[0],
                                         self.records.ctypes.data_as(C.c_void_p),
                                         self.obj.ctypes.data_as(C.c_void_p), nobj, tex_res,
                                         channels, C.byref(h)))
        self.h = h

    def info(self):
        nodes, depth, params = C.c_int32(), C.c_int32(), C.c_int64()
        check(load().mg_meshscene_info(self.h, C.byref(nodes), C.byref(depth), C.byref(params)))
        return {"nodes": nodes.value, "depth": depth.value, "params": params.value,
                "triangles": self.records.shape[0]}

    def params(self) -> int:
        return self.nobj * self.channels * self.R * self.R

    def intersect(self, rays: torch.Tensor):
        """rays: CUDA fp64 [n][6] -> (t [n], triangle [n])"""
        n = rays.shape[0]
        t = torch.empty(n, dtype=torch.float64, device=rays.device)
        k = torch.empty(n, dtype=torch.int32, device=rays.device)
        check(load().mg_meshscene_intersect(self.ctx.h, self.h, n, _p(rays.contiguous()), _p(t),
                                            _p(k)))
        return t, k

    def render(self, theta, W: int, H: int, spp: int, key: int):
        img = torch.empty(3 * W * H, dtype=theta.dtype, device="cuda")
        check(load().mg_meshscene_render(self.ctx.h, self.h, _dtype_code(theta), W, H,
                                         self.view.ctypes.data_as(C.c_void_p), spp, key,
                                         _p(theta.contiguous()), _p(img)))
        return img

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load().mg_meshscene_destroy(self.h)
        except Exception:
            pass


class MeshTextureProblem:
    """BASELINE.json configs[3]: W x H render of the 3-object mesh scene,
    each object with an R x R RGB albedo + roughness texture (3 * 4 * R^2
    parameters, ~3.1M at R = 512), targets seeded smooth noise (seed 1),
    initialised to base 0.5 / roughness 0.5, depth-6 NEE path tracing,
    1 FD + 2 proportional spp (paths A, B, C).  Own renderer (DESIGN.md §12,
    oracle mgo_mesh_*)."""

    def __init__(self, width: int = 512, height: int = 512, tex_res: int = 512,
                 sphere_res=(24, 48), displaced_res=(100, 100), max_vertices: int = 6,
                 target_seed: int = 1, target_spp: int = 16, dtype=torch.float32, ctx=None,
                 channels: int = 4, prop_paths: int = 2, geometry=None, view=None):
        self.ctx = ctx or Context.default()
        self.W, self.H, self.R, self.dtype = width, height, tex_res, dtype
        self.channels, self.prop_paths = channels, prop_paths
        rec, obj, nobj = geometry if geometry is not None else \
            mesh_scene_geometry(sphere_res, displaced_res)
        view = view if view is not None else mesh_scene_view(max_vertices)
        self.scene = MeshScene(rec, obj, nobj, tex_res, view, self.ctx, channels)
        n = self.scene.params()
        self.target_tex = torch.tensor(
            smooth_noise_textures(nobj, tex_res, target_seed, channels=channels).reshape(-1),
            device="cuda").to(dtype)
        init = np.full((nobj, channels, tex_res * tex_res), 0.5)
        if channels == 5:
            init[:, 4] = 0.1
        self.init = torch.tensor(init.reshape(-1), device="cuda").to(dtype)
        self.target_img = self.scene.render(self.target_tex, width, height, target_spp,
                                            int(load().mg_mix64(target_seed)))
        self.accum = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
        self.loss_buf = torch.zeros(1, dtype=torch.float64, device="cuda")

    def dim(self) -> int:
        return self.scene.params()

    def draws_per_sample(self) -> int:
        """Paths per iteration: prop_paths proportional + 1 finite-difference spp."""
        return (self.prop_paths + 1) * self.W * self.H

    def initial_params(self):
        return self.init.clone()

    def sample_pair(self, now, prev, iteration: int, key: int, rows=None):
        r0, r1 = rows if rows is not None else (0, self.H)
        prop, diff = torch.empty_like(now), torch.empty_like(now)
        check(load().mg_meshscene_sample_pair(
            self.ctx.h, self.scene.h, _dtype_code(now), self.W, self.H,
            self.scene.view.ctypes.data_as(C.c_void_p), _p(self.target_img), _p(now.contiguous()),
            _p(prev.contiguous()), key, iteration, r0, r1, self.prop_paths, _p(self.accum),
            _p(prop), _p(diff), _p(self.loss_buf)))
        return GradientSamplePair(prop, diff)


def large_scene_view(max_vertices: int = 8):
    """configs[4] camera/light over the 5 x 3 grid of objects."""
    return mesh_scene_view(max_vertices, light=(8.0, 8.0, 8.0), cam=(0.0, 2.8, 4.4),
                           look_at=(0.0, 0.2, -0.3), tan_half_fov=0.55, light_y=3.5,
                           light_rect=(-1.5, 1.5, -1.5, 1.0))


class MeshLargeProblem(MeshTextureProblem):
    """BASELINE.json configs[4]: 1024 x 1024 image, 16 objects (ground quad +
    15 seeded displaced spheres, ~502k triangles), each with a 1024 x 1024
    texture of base r, g, b, roughness and metalness (16 * 5 * 1024^2 =
    83.9M parameters), depth 8 with NEE, 1 FD + 4 proportional spp."""

    def __init__(self, width: int = 1024, height: int = 1024, tex_res: int = 1024,
                 res=(130, 130), max_vertices: int = 8, target_seed: int = 1,
                 target_spp: int = 4, dtype=torch.float32, ctx=None, prop_paths: int = 4):
        super().__init__(width, height, tex_res, max_vertices=max_vertices,
                         target_seed=target_seed, target_spp=target_spp, dtype=dtype, ctx=ctx,
                         channels=5, prop_paths=prop_paths,
                         geometry=mesh_large_scene_geometry(res=res),
                         view=large_scene_view(max_vertices))


class MeshTextureRun(QuadTextureRun):
    """configs[3] optimisation loop: sample pair + fused update per
    iteration; texture values projected to [0, 1] (meta)."""

    def __init__(self, problem, optimizer: str = "meta", lr: float = 0.01, seed: int = 0,
                 replicate: int = 0, **kw):
        if optimizer == "meta":
            kw.setdefault("project_hi", 1.0)
        super().__init__(problem, optimizer, lr, seed, replicate, **kw)


# ------------------------------------------------------------- harness
@dataclasses.dataclass
class ExperimentConfig:
    """harness.hpp:18-67 (+ B200 knobs dtype/rng)."""
    problem: str = "exp-rate"
    optimizer: str = "meta"
    iterations: int = 100
    replicates: int = 1
    seed: int = 0
    lr: float = 0.01
    beta_f: float = 0.9
    beta_delta: float = 0.5
    beta1: float = 0.9
    beta2: float = 0.999
    eps_step: float = 1e-8
    eps_alpha: float = 1e-30
    adam_eps: float = 1e-8
    dim: int = 4
    sigma: float = 1.0
    samples_per_iter: int = 32
    target_mean: float = 2.0
    rate_init: float = 2.0
    pixel_count: int = 8
    spp: int = 4
    problem_seed: int = 1234
    albedo_init: float = 0.1
    exponent_max: float = 4.0
    trajectory: str = "optimise"
    traj_rate: float = 0.05
    no_alpha_clip: bool = False
    independent_variance_samples: bool = False
    non_zero_centred: bool = False
    diff_norm: str = "global"
    coord: int = 0
    converge_threshold: float = -1.0
    threads: int = 0
    dtype: str = "f64"
    rng: str = "mt64"

    def to_c(self) -> _abi.ExperimentConfigC:
        kw = dataclasses.asdict(self)
        kw.pop("threads")
        return _abi.config_from(**kw)

    def validate(self):
        try:
            c = self.to_c()
        except ValueError as e:
            raise InvalidArgument(_abi.MG_EINVAL, str(e)) from None
        check(load().mg_config_validate(C.byref(c)))

    def problem_dim(self) -> int:
        return {"exp-rate": 1, "mult-noise": self.dim, "mini-render": self.pixel_count}[self.problem]


STATUS = {0: "completed", 1: "converged", 2: "diverged"}


@dataclasses.dataclass
class RunRecord:
    """Per-replicate record (harness.hpp:73-90), scalar series for `coord`."""
    status: str
    iterations_run: int
    draws_used: int
    evals_used: int
    series: Dict[str, np.ndarray]
    final_params: np.ndarray
    # full per-iteration vectors (harness.hpp:79-88), [iterations_run][dim]
    # each, when requested (run_single(..., full=True)); alpha is None for Adam
    vectors: Optional[Dict[str, Optional[np.ndarray]]] = None


SCALED_MIN_PIXELS = 1 << 16


def _scaled_eligible(cfg: ExperimentConfig) -> bool:
    """Large mini-render replicates run on the whole GPU (fused iteration
    kernel + jump-ahead mt64 engines) instead of one CTA of the runner."""
    return (cfg.problem == "mini-render" and cfg.optimizer == "meta" and
            cfg.pixel_count >= SCALED_MIN_PIXELS and cfg.trajectory == "optimise" and
            cfg.diff_norm == "global" and not cfg.independent_variance_samples and
            cfg.rng == "mt64")


def _run_minirender_scaled(cfg: ExperimentConfig, replicate: int, ctx=None) -> "RunRecord":
    """harness.cpp:90-200 for one large mini-render replicate: each iteration
    is one fused kernel; the extractor series of coordinate `coord` and the
    scalars are gathered on the device (no per-iteration host sync) and read
    back once.  Divergence (non-finite params, harness.cpp:116) truncates."""
    ctx = ctx or Context.default()
    dt = torch.float64 if cfg.dtype == "f64" else torch.float32
    run = MiniRenderRun(cfg.pixel_count, cfg.spp, gen_seed=cfg.problem_seed,
                        albedo_init=cfg.albedo_init, exponent_max=cfg.exponent_max, lr=cfg.lr,
                        beta_f=cfg.beta_f, beta_delta=cfg.beta_delta, eps_step=cfg.eps_step,
                        eps_alpha=cfg.eps_alpha, clip=not cfg.no_alpha_clip, seed=cfg.seed,
                        replicate=replicate, rng="mt64", dtype=dt, ctx=ctx)
    it, c = cfg.iterations, cfg.coord
    T = run.problem.target  # fp64 truth
    ser = torch.full((11, it), float("nan"), dtype=torch.float64, device="cuda")
    pr = torch.empty(1, dtype=dt, device="cuda")
    df = torch.empty(1, dtype=dt, device="cuda")
    loss0 = ((run.params.double() - T) ** 2).sum()
    n, status, finals = it, "completed", None
    D = cfg.pixel_count * cfg.spp
    draws = evals = 0
    changed_prev = 0.0  # params == prev before the first step (no diff)
    for i in range(it):
        p_i = run.params[c].double().clone()
        loss_i = loss0 if i == 0 else run.scalars_buf[2].clone()  # step i overwrites it
        run.step(prop_out=pr, diff_out=df, record=c)
        m, v = run.mean[c].double(), run.var[c].double()
        delta = (-cfg.lr * m) / (torch.sqrt(v) + cfg.eps_step)  # meta.hpp:112
        ser[:, i] = torch.stack([torch.sqrt(loss_i), loss_i, pr[0].double(), df[0].double(), m, v,
                                 run.alpha_prev[c].double(), delta, 2.0 * (p_i - T[c]),
                                 run.scalars_buf[6], p_i])
        draws += D
        evals += D * (2 if changed_prev > 0 else 1)  # harness.cpp:129-131
        sc = run.scalars()
        changed_prev = sc.changed
        if sc.nonfinite > 0:  # params of iteration i+1 non-finite: harness.cpp:116-119
            n, status = i + 1, ("diverged" if i + 1 < it else "completed")
            finals = run.prev  # params of iteration i (the last recorded)
            if i + 1 < it:
                break
    if finals is None:
        finals = run.prev
    ser_h = ser.cpu().numpy()
    ser_h[:, n:] = np.nan
    finals = finals.double().cpu().numpy()
    rec = RunRecord(status, n, draws, evals,
                    {nm: ser_h[k] for k, nm in enumerate(_abi.SERIES_NAMES)}, finals)
    if status != "diverged" and cfg.converge_threshold > 0.0 and n > 0:
        if ser_h[0][n - 1] < cfg.converge_threshold:  # harness.cpp:191-198
            rec.status = "converged"
    return rec


def _run_device(cfg: ExperimentConfig, rep_begin: int, rep_count: int, ctx=None,
                full: bool = False):
    if _scaled_eligible(cfg) and not full:
        return [_run_minirender_scaled(cfg, r, ctx) for r in range(rep_begin, rep_begin + rep_count)]
    ctx = ctx or Context.default()
    c = cfg.to_c()
    it = cfg.iterations
    dim = cfg.problem_dim()
    bufs = {n: np.full((rep_count, it), np.nan) for n in _abi.SERIES_NAMES}
    ser = _abi.RunSeriesC(*[b.ctypes.data_as(C.c_void_p) for b in bufs.values()])
    recs = (_abi.RunRecordC * rep_count)()
    finals = np.empty((rep_count, dim))
    if full:
        vecs = np.empty((rep_count, it, 8, dim))
        check(load().mg_run_replicates_full(ctx.h, C.byref(c), rep_begin, rep_count,
                                            C.cast(recs, C.c_void_p), C.byref(ser),
                                            finals.ctypes.data_as(C.c_void_p),
                                            vecs.ctypes.data_as(C.c_void_p)))
    else:
        check(load().mg_run_replicates(ctx.h, C.byref(c), rep_begin, rep_count,
                                       C.cast(recs, C.c_void_p), C.byref(ser),
                                       finals.ctypes.data_as(C.c_void_p)))
    out = []
    for r in range(rep_count):
        rec = recs[r]
        vectors = None
        if full:
            from .report import REPLICATE_VECTORS
            n_run = rec.iterations_run
            vectors = {n: vecs[r, :n_run, k].copy() for k, n in enumerate(REPLICATE_VECTORS)}
            if cfg.optimizer != "meta":
                vectors["alpha"] = None
        out.append(RunRecord(STATUS[rec.status], rec.iterations_run, rec.draws_used,
                             rec.evals_used, {n: bufs[n][r] for n in bufs}, finals[r], vectors))
    return out


def run_single(cfg: ExperimentConfig, replicate_index: int, ctx=None,
               full: bool = False) -> RunRecord:
    """harness.cpp:90-200 on the device.  full=True also returns every
    per-iteration vector of the reference's RunRecord (record.vectors),
    e.g. for report.write_replicate_csv."""
    cfg.validate()
    if cfg.coord >= cfg.problem_dim():
        raise InvalidArgument(_abi.MG_EINVAL, "coord exceeds problem dimension")
    return _run_device(cfg, replicate_index, 1, ctx, full=full)[0]


@dataclasses.dataclass
class SeriesStats:
    mean: np.ndarray
    variance: np.ndarray
    median: np.ndarray
    q25: np.ndarray
    q75: np.ndarray


@dataclasses.dataclass
class AggregateReport:
    config: ExperimentConfig
    series_names: List[str]
    stats: Dict[str, SeriesStats]
    active_replicates: np.ndarray
    diverged_count: int
    records: List[RunRecord]


def _seq_sum(x: np.ndarray, axis: int = 0) -> np.ndarray:
    """Sequential (index-order) sum along axis: the last element of a prefix
    sum, which numpy evaluates left to right — identical to stats.hpp's
    `for (double x : xs) s += x` (np.sum would sum pairwise)."""
    if x.shape[axis] == 0:
        return np.zeros(np.delete(x.shape, axis))
    return np.take(np.cumsum(x, axis=axis), -1, axis=axis)


def _column_stats(vals: np.ndarray):
    """mean_of / variance_of / quantile (stats.hpp:45-68) of one sample."""
    n = vals.size
    if n == 0:
        return math.nan, 0.0, math.nan, math.nan, math.nan
    mean = float(_seq_sum(vals)) / n
    var = float(_seq_sum((vals - mean) * (vals - mean))) / (n - 1) if n >= 2 else 0.0
    s = np.sort(vals)

    def q(p):
        pos = p * (n - 1)
        lo = int(pos)
        if lo + 1 >= n:
            return float(s[-1])
        frac = pos - lo
        return float(s[lo] * (1.0 - frac) + s[lo + 1] * frac)
    return mean, var, q(0.5), q(0.25), q(0.75)


SERIES_ORDER = ["param_err", "loss", "prop", "diff", "grad_est", "est_var", "alpha", "delta",
                "true_grad", "step_sq_norm"]


def aggregate(cfg: ExperimentConfig, records: List[RunRecord]) -> AggregateReport:
    """Per-iteration reduction in replicate order (harness.cpp:274-302)."""
    it = cfg.iterations
    names = [n for n in SERIES_ORDER if cfg.optimizer == "meta" or n != "alpha"]
    runs = np.array([r.iterations_run for r in records])
    active = np.array([int(np.sum(runs > i)) for i in range(it)])
    stats = {}
    for n in names:
        cols = np.stack([r.series[n] for r in records])  # [R][it], replicate order
        st = SeriesStats(*(np.empty(it) for _ in range(5)))
        for i in range(it):
            vals = cols[runs > i, i]
            st.mean[i], st.variance[i], st.median[i], st.q25[i], st.q75[i] = _column_stats(vals)
        stats[n] = st
    div = sum(1 for r in records if r.status == "diverged")
    return AggregateReport(cfg, names, stats, active, div, records)


def aggregate_series_device(series, iterations_run, ctx=None):
    """F2: across-replicate statistics on the device (harness.cpp:274-302).
    series: CUDA fp64 [S][R][T]; iterations_run: CUDA int32 [R].  Returns
    (stats [S][5][T] = mean, variance, median, q25, q75; active [T]),
    bit-identical to `aggregate` (sequential sums in replicate order)."""
    import torch
    if series.dim() != 3 or series.dtype != torch.float64 or not series.is_cuda:
        raise InvalidArgument(_abi.MG_EINVAL, "series must be a CUDA fp64 [S][R][T] tensor")
    ctx = ctx or Context.default()
    S, R, T = series.shape
    runs = iterations_run.to(device=series.device, dtype=torch.int32).contiguous()
    if runs.numel() != R:
        raise InvalidArgument(_abi.MG_EINVAL, "iterations_run must hold one entry per replicate")
    stats = torch.empty((S, 5, T), dtype=torch.float64, device=series.device)
    active = torch.empty(T, dtype=torch.int32, device=series.device)
    check(load().mg_aggregate_series(ctx.h, S, R, T, _p(series.contiguous()), _p(runs), _p(stats),
                                     _p(active)))
    return stats, active


def _run_experiment_device_stats(cfg: ExperimentConfig, rep_begin: int, rep_count: int,
                                 ctx=None) -> AggregateReport:
    ctx = ctx or Context.default()
    c = cfg.to_c()
    it = cfg.iterations
    recs = (_abi.RunRecordC * rep_count)()
    stats = np.empty((len(_abi.SERIES_NAMES), 5, it))
    active = np.empty(it, dtype=np.int32)
    check(load().mg_run_experiment_stats(ctx.h, C.byref(c), rep_begin, rep_count,
                                         C.cast(recs, C.c_void_p),
                                         stats.ctypes.data_as(C.c_void_p),
                                         active.ctypes.data_as(C.c_void_p)))
    records = [RunRecord(STATUS[r.status], r.iterations_run, r.draws_used, r.evals_used, {}, None)
               for r in recs]
    names = [n for n in SERIES_ORDER if cfg.optimizer == "meta" or n != "alpha"]
    st = {n: SeriesStats(*(stats[_abi.SERIES_NAMES.index(n), q].copy() for q in range(5)))
          for n in names}
    div = sum(1 for r in records if r.status == "diverged")
    return AggregateReport(cfg, names, st, active.astype(np.int64), div, records)


def run_experiment(cfg: ExperimentConfig, ctx=None, rep_begin: int = 0,
                   rep_count: Optional[int] = None,
                   device_aggregate: bool = False) -> AggregateReport:
    """harness.cpp:249-302: all replicates as one device launch (the thread
    pool becomes the grid); reduction in replicate order on the host, or on
    the device with device_aggregate=True (F2: only the statistics leave the
    GPU; records then carry no per-iteration series)."""
    cfg.validate()
    if cfg.coord >= cfg.problem_dim():
        raise InvalidArgument(_abi.MG_EINVAL, "coord exceeds problem dimension")
    n = cfg.replicates if rep_count is None else rep_count
    if device_aggregate and not _scaled_eligible(cfg):
        return _run_experiment_device_stats(cfg, rep_begin, n, ctx)
    recs = _run_device(cfg, rep_begin, n, ctx)
    return aggregate(cfg, recs)
