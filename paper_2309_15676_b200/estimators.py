"""Moment2 / GradientSamplePair / MetaEstimator / Adam (moment2.hpp,
meta.hpp, adam.hpp) on the device, and the fused one-pass updates
(mg_meta_update, mg_adam_update) of the hot path (harness.cpp:144-188)."""
from __future__ import annotations

import ctypes as C
import dataclasses  # noqa: F401
import math  # noqa: F401
from typing import Dict, List, Optional  # noqa: F401

import numpy as np
import torch

from . import _abi
from ._lib import DomainError, InvalidArgument, LogicError, MgError, check, load  # noqa: F401
from ._core import Context, _dtype_code, _p  # noqa: F401


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
                 project_hi: Optional[float] = None, device_coef: bool = False):
        self.ctx = ctx or Context.default()
        self.n, self.dtype = n, dtype
        self.beta_f, self.beta_delta = beta_f, beta_delta
        self.meta = _abi.MetaParams(lr, eps_step, eps_alpha, int(clip))
        self.project_lo, self.project_hi = project_lo, project_hi
        self.diff_norm = _abi.DIFF_NORMS[diff_norm]
        # device_coef: the Moment2(beta_f) coefficient of steps after the
        # first is formed on the device (mg_meta_update_args.prop_coef_device),
        # so a captured step is replayable
        self.device_coef = device_coef
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
            proj_hi=0.0 if self.project_hi is None else self.project_hi,
            beta_f=self.beta_f, prop_coef_device=int(self.device_coef and self.t > 1),
            prop_pow_advance=1)

    def step(self, prop, diff, params_in, params_out, target=None, vprop=None, vdiff=None,
             params_prev=None, delta_out=None, ssn_host=None):
        a = self.args(ssn_host)
        x = _abi.MetaExtras(_p(vprop), _p(vdiff), _p(params_prev), _p(target), _p(delta_out))
        check(load().mg_meta_update(self.ctx.h, _dtype_code(prop), self.n, C.byref(a), _p(prop),
                                    _p(diff), _p(self.m2_prop), _p(self.m2_diff), _p(self.mean),
                                    _p(self.var), _p(self.alpha_prev), _p(params_in),
                                    _p(params_out), _p(self.scalars_buf), C.byref(x)))


    def step_fixed(self, accum, cells: int, nch: int, r2: int, params_in, params_out,
                   params_prev=None, target=None, touch=None):
        """step() with the sample pair still in a mesh scene's texel-interleaved
        fixed-point accumulator (MeshTextureProblem.sample_pair(...,
        finalize=False)): converted, consumed and zeroed in the same pass
        (mg_meta_update_fixed); every element as finalize + step().
        touch: the accumulator's touch map (MeshTextureProblem.enable_touch_map)
        — only the cells a path reached are read and zeroed."""
        a = self.args(None)
        x = _abi.MetaExtras(None, None, _p(params_prev), _p(target), None)
        check(load().mg_meta_update_fixed_touch(self.ctx.h, _dtype_code(params_in), cells, nch,
                                                r2, C.byref(a), _p(accum), _p(touch),
                                                _p(self.m2_prop), _p(self.m2_diff),
                                                _p(self.mean), _p(self.var),
                                                _p(self.alpha_prev), _p(params_in),
                                                _p(params_out), _p(self.scalars_buf),
                                                C.byref(x)))


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

    def scalars(self) -> _abi.UpdateScalars:
        out = _abi.UpdateScalars()
        check(load().mg_scalars_read(self.ctx.h, _p(self.scalars_buf), C.byref(out)))
        return out

    def step(self, grad, params_in, params_out, target=None):
        check(load().mg_adam_update(self.ctx.h, _dtype_code(grad), self.n, C.byref(self.s),
                                    int(self.project_lo is not None),
                                    0.0 if self.project_lo is None else self.project_lo,
                                    _p(grad), _p(self.m), _p(self.v), _p(params_in),
                                    _p(params_out), _p(target), _p(self.scalars_buf)))
