"""run_single / run_experiment (harness.hpp:18-112, harness.cpp:90-302) on
the device: the persistent replicate runner, the scaled mini-render path,
across-replicate aggregation (host or device)."""
from __future__ import annotations

import ctypes as C
import dataclasses  # noqa: F401
import math  # noqa: F401
from typing import Dict, List, Optional  # noqa: F401

import numpy as np
import torch

from . import _abi
from ._lib import DomainError, InvalidArgument, LogicError, MgError, check, load  # noqa: F401
from ._core import Context, _p  # noqa: F401
from .problems import MiniRenderRun  # noqa: F401


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
    """Sequential (index-order) sum along axis starting from 0.0: the last
    element of a prefix sum over a leading zero, which numpy evaluates left
    to right — identical to stats.hpp's `double s = 0.0; for (double x : xs)
    s += x` (np.sum would sum pairwise; a bare cumsum would keep a lone -0.0)."""
    x = np.moveaxis(np.asarray(x, dtype=np.float64), axis, 0)
    z = np.concatenate([np.zeros((1,) + x.shape[1:]), x], axis=0)
    return np.cumsum(z, axis=0)[-1]


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


def _stats_columns(cols: np.ndarray, mask: np.ndarray):
    """_column_stats of every iteration column at once: cols [R][T] in
    replicate order, mask [R][T] = replicate active at that iteration.
    The same arithmetic per column (stats.hpp:45-68): sums sequential in
    replicate order starting from 0.0 (cumsum over a leading zero row; the
    masked-out entries add +0.0, which leaves every partial sum unchanged),
    quantiles by linear interpolation over the sorted active values (NaN
    last, as std::sort places them for these inputs)."""
    R, T = cols.shape
    n = mask.sum(axis=0)
    z = np.zeros((R + 1, T))
    z[1:] = np.where(mask, cols, 0.0)
    with np.errstate(invalid="ignore", divide="ignore"):
        mean = np.cumsum(z, axis=0)[-1] / n
        mean = np.where(n > 0, mean, math.nan)
        dev = cols - mean
        z[1:] = np.where(mask, dev * dev, 0.0)
        var = np.where(n >= 2, np.cumsum(z, axis=0)[-1] / (n - 1), 0.0)
    srt = np.sort(np.where(mask, cols, math.nan), axis=0)
    cidx = np.arange(T)

    def q(p):
        pos = p * (n - 1)
        lo = np.maximum(pos, 0).astype(np.int64)
        last = srt[np.maximum(n - 1, 0), cidx]
        lo_c = np.minimum(lo, max(R - 1, 0))
        hi_c = np.minimum(lo + 1, max(R - 1, 0))
        frac = pos - lo
        interp = srt[lo_c, cidx] * (1.0 - frac) + srt[hi_c, cidx] * frac
        out = np.where(lo + 1 >= n, last, interp)
        return np.where(n > 0, out, math.nan)
    return mean, var, q(0.5), q(0.25), q(0.75)


def aggregate(cfg: ExperimentConfig, records: List[RunRecord]) -> AggregateReport:
    """Per-iteration reduction in replicate order (harness.cpp:274-302)."""
    it = cfg.iterations
    names = [n for n in SERIES_ORDER if cfg.optimizer == "meta" or n != "alpha"]
    runs = np.array([r.iterations_run for r in records])
    mask = runs[:, None] > np.arange(it)[None, :]
    active = mask.sum(axis=0)
    # every (series, iteration) column of every series in one pass: [R][S*T]
    S = len(names)
    cols = np.stack([np.concatenate([np.asarray(r.series[n], dtype=np.float64) for n in names])
                     for r in records]) if records else np.zeros((0, S * it))
    st = _stats_columns(cols, np.tile(mask, (1, S)))
    stats = {n: SeriesStats(*(q[k * it:(k + 1) * it] for q in st)) for k, n in enumerate(names)}
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
