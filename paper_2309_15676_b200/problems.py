"""The reference's gradient-sample problems (problems.hpp:74-195) on the
device, and the fused mini-render iteration at scale."""
from __future__ import annotations

import ctypes as C
import dataclasses  # noqa: F401
import math  # noqa: F401
from typing import Dict, List, Optional  # noqa: F401

import numpy as np
import torch

from . import _abi
from ._lib import DomainError, InvalidArgument, LogicError, MgError, check, load  # noqa: F401
from ._core import Context, Rng, _dtype_code, _p  # noqa: F401
from .estimators import FusedMetaUpdate, GradientSamplePair  # noqa: F401


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
                # the engines run on their own stream: block b+1's draws and
                # jump overlap block b's render iterations (double buffer)
                self.side = torch.cuda.Stream(device=self.ctx.device)
                self.rng_ctx = Context(self.ctx.device, stream=self.side)
                self.rng = Rng.split(int(load().mg_stream_seed(seed, replicate)), G, L,
                                     ctx=self.rng_ctx)
                self.seg_len, self.block_iters = L, K
            else:
                self.rng = Rng.stream(seed, replicate, ctx=self.ctx)
                self.seg_len, self.block_iters = None, 1
            rows = self.rng.n * self.seg_len if self.seg_len else D
            self.u = torch.empty(rows, dtype=torch.float64, device="cuda")
            if self.seg_len:
                self.ubuf = [self.u, torch.empty(rows, dtype=torch.float64, device="cuda")]
                self.ready = [torch.cuda.Event(), torch.cuda.Event()]
                self.done = [torch.cuda.Event(), torch.cuda.Event()]
                self._fill(0)
        else:
            self.rng, self.u = None, None
            self.seg_len, self.block_iters = None, 1
        self.t = 0
        self.beta_f_pow = 1.0

    def draws_per_sample(self) -> int:
        return self.P * self.spp

    def _fill(self, blk: int):
        """Block blk's draws (K iterations of the stream, all engines) into
        ubuf[blk % 2] on the side stream, then jump the engines past them."""
        j = blk % 2
        if blk >= 2:
            self.side.wait_event(self.done[j])       # block blk-2 no longer reads it
        check(load().mg_mt64_draw(self.rng_ctx.h, self.rng.h, self.seg_len, 1,
                                  _p(self.ubuf[j])))
        self.rng.jump(self.block_iters * self.D - self.seg_len)
        self.ready[j].record(self.side)

    def step(self, prop_out=None, diff_out=None, record: Optional[int] = None):
        """One iteration.  prop_out/diff_out receive this iteration's sample
        pair: full [P] tensors, or (record=k) one-element tensors receiving
        local pixel k only."""
        self.t += 1
        self.beta_f_pow *= self.beta_f
        upd = _abi.MetaUpdateArgs(meta=self.meta,
                                  prop_coef=(1.0 - self.beta_f) / (1.0 - self.beta_f_pow),
                                  beta_delta=self.beta_delta, first_step=int(self.t == 1),
                                  diff_norm=_abi.MG_DIFF_NORM_GLOBAL, project=1,
                                  beta_f=self.beta_f, prop_pow_advance=1)
        a = _abi.RenderArgs(update=upd, spp=self.spp, rng_kind=self.rng_kind, key=self.key,
                            iteration=self.t - 1, stream=0, pixel_offset=self.lo,
                            record_plus1=0 if record is None else record + 1)
        L = load()
        u = None
        main = self.ctx.stream
        if self.rng is not None:
            k = (self.t - 1) % self.block_iters
            if self.seg_len:
                blk = (self.t - 1) // self.block_iters
                if k == 0:  # block blk ready; start generating block blk + 1
                    main.wait_event(self.ready[blk % 2])
                    self._fill(blk + 1)
                self.u = self.ubuf[blk % 2]
            else:
                check(L.mg_mt64_draw(self.ctx.h, self.rng.h, self.D, 1, _p(self.u)))
            u = C.c_void_p(self.u.data_ptr() + 8 * (k * self.D + self.lo * self.spp))
        check(L.mg_minirender_meta_iteration(
            self.ctx.h, _dtype_code(self.params), self.P, C.byref(a), _p(self.b), _p(self.T),
            u, _p(self.params), _p(self.prev), _p(self.m2_prop), _p(self.m2_diff),
            _p(self.mean), _p(self.var), _p(self.alpha_prev), _p(self.scalars_buf),
            _p(prop_out), _p(diff_out)))
        if self.seg_len and k == self.block_iters - 1:
            self.done[blk % 2].record(main)            # buffer free for block blk + 2
        # prev now holds pi_{t+1}: swap roles
        self.params, self.prev = self.prev, self.params

    def scalars(self) -> _abi.UpdateScalars:
        out = _abi.UpdateScalars()
        check(load().mg_scalars_read(self.ctx.h, _p(self.scalars_buf), C.byref(out)))
        return out
