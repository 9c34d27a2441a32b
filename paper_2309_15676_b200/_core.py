"""Device plumbing shared by the host API: tensor/pointer helpers, the
context (device + stream) and the device mt19937_64 engines (rng.hpp)."""
from __future__ import annotations

import ctypes as C
import dataclasses  # noqa: F401
import math  # noqa: F401
from typing import Dict, List, Optional  # noqa: F401

import numpy as np
import torch

from . import _abi
from ._lib import DomainError, InvalidArgument, LogicError, MgError, check, load  # noqa: F401


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
