"""World-size-2 tests of the multi-GPU host logic on CPU (gloo).

The device compute is replaced by the oracle (this is the host-side
sharding/collective logic under test, not the kernels): a parameter-sharded
run with the per-step scalar all-reduce must reproduce the single-process
run, and a replicate-sharded run_experiment must produce the identical
report.  The same ShardedStep / run_experiment_sharded drive NCCL on B200s.
"""
import ctypes as C
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2309_15676_b200 import _abi, dist as mgdist  # noqa: E402


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for n in (1, 1000, 1024 * 7 + 3, 10 ** 6):
        for world in (1, 2, 3, 8):
            cuts = [mgdist.shard_range(n, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            for (a, b), (c, d) in zip(cuts, cuts[1:]):
                assert b == c and a <= b
            assert all(lo % 1024 == 0 for lo, _ in cuts)
    for R in (1, 5, 100, 1000):
        rr = [mgdist.replicate_range(R, r, 4) for r in range(4)]
        assert rr[0][0] == 0 and rr[-1][1] == R
        assert sum(e - b for b, e in rr) == R


class OracleUpdater:
    """CPU stand-in for api.FusedMetaUpdate (same scalars_buf layout)."""

    def __init__(self, oracle, n):
        self.o = oracle
        self.st = {k: np.zeros(n) for k in ("m2_prop", "m2_diff", "mean", "var", "alpha_prev")}
        self.sc = _abi.fresh_scalars()
        self.scalars_buf = torch.zeros(8, dtype=torch.float64)
        self._sync_out()
        self.t, self.bp = 0, 1.0

    def _sync_out(self):
        raw = np.frombuffer(bytes(self.sc), dtype=np.float64).copy()
        self.scalars_buf.copy_(torch.from_numpy(raw))

    def _sync_in(self):
        raw = self.scalars_buf.numpy().tobytes()
        C.memmove(C.addressof(self.sc), raw, len(raw))

    def step(self, prop, diff, params):
        self._sync_in()
        self.t += 1
        self.bp *= 0.9
        a = _abi.MetaUpdateArgs(meta=_abi.MetaParams(0.01, 1e-8, 1e-30, 1),
                                prop_coef=(1 - 0.9) / (1 - self.bp), beta_delta=0.5,
                                first_step=int(self.t == 1), project=1)
        out, _, rc = self.o.meta_update(a, self.st, prop, diff, params, self.sc)
        assert rc == 0
        self._sync_out()
        self.out = out


def _inputs(n, steps):
    rs = np.random.RandomState(5)
    props = [rs.standard_normal(n) for _ in range(steps)]
    diffs = [np.zeros(n)] + [0.1 * rs.standard_normal(n) for _ in range(steps - 1)]
    return props, diffs


def _sharded_worker(rank, world, port, n, steps, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_bind import Oracle
    lo, hi = mgdist.shard_range(n, rank, world, align=64)
    props, diffs = _inputs(n, steps)
    up = OracleUpdater(Oracle(), hi - lo)
    step = mgdist.ShardedStep(up)
    p = np.full(hi - lo, 0.2)
    for t in range(steps):
        step(props[t][lo:hi], diffs[t][lo:hi], p)
        p = up.out
    parts = [None] * world
    dist.all_gather_object(parts, (lo, p, up.scalars_buf.numpy().copy()))
    if rank == 0:
        full = np.concatenate([x[1] for x in sorted(parts, key=lambda x: x[0])])
        np.save(result_path, np.concatenate([full, parts[0][2]]))
    dist.destroy_process_group()


def test_parameter_sharded_run_matches_single_process(oracle, tmp_path):
    n, steps, world = 5000, 12, 2
    out = str(tmp_path / "sharded.npy")
    mp.spawn(_sharded_worker, args=(world, free_port(), n, steps, out), nprocs=world, join=True)
    got = np.load(out)
    params, scal = got[:n], got[n:]
    # single process, same inputs
    props, diffs = _inputs(n, steps)
    up = OracleUpdater(oracle, n)
    p = np.full(n, 0.2)
    for t in range(steps):
        up.step(props[t], diffs[t], p)
        p = up.out
    # the global step norm is summed in a different order (2 shards) -> ulps
    np.testing.assert_allclose(params, p, rtol=1e-12, atol=1e-15)
    ref = up.scalars_buf.numpy()
    np.testing.assert_allclose(scal[0], ref[0], rtol=1e-12)  # ssn
    assert scal[1] == ref[1] and scal[3] == ref[3]           # changed, nonfinite
    assert scal[5] == ref[5]                                 # diff-EMA count (bit pattern)


def _oracle_run_fn(cfg, begin, count):
    from oracle_bind import Oracle
    from paper_2309_15676_b200.api import RunRecord, STATUS
    o = Oracle()
    c = cfg.to_c()
    it = cfg.iterations
    dim = cfg.problem_dim()
    recs = []
    for r in range(begin, begin + count):
        bufs = {nm: np.full(it, np.nan) for nm in _abi.SERIES_NAMES}
        ser = _abi.RunSeriesC(*[b.ctypes.data_as(C.c_void_p) for b in bufs.values()])
        rec = _abi.RunRecordC()
        fp = np.empty(dim)
        rc = o.lib.mgo_run_single_series(C.byref(c), r, C.byref(rec), C.byref(ser), 1,
                                         fp.ctypes.data_as(C.c_void_p))
        assert rc == 0
        recs.append(RunRecord(STATUS[rec.status], rec.iterations_run, rec.draws_used,
                              rec.evals_used, bufs, fp))
    return recs


def _replicate_worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2309_15676_b200.api import ExperimentConfig
    cfg = ExperimentConfig(problem="mini-render", pixel_count=6, spp=3, iterations=30,
                           replicates=7, seed=42)
    rep = mgdist.run_experiment_sharded(cfg, _oracle_run_fn)
    if rank == 0:
        np.save(result_path, np.stack([rep.stats[nm].median for nm in rep.series_names] +
                                      [rep.stats[nm].mean for nm in rep.series_names]))
    dist.destroy_process_group()


def test_replicate_sharded_experiment_is_world_size_invariant(tmp_path):
    out = str(tmp_path / "rep.npy")
    mp.spawn(_replicate_worker, args=(2, free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    from paper_2309_15676_b200.api import ExperimentConfig, aggregate
    cfg = ExperimentConfig(problem="mini-render", pixel_count=6, spp=3, iterations=30,
                           replicates=7, seed=42)
    rep = aggregate(cfg, _oracle_run_fn(cfg, 0, 7))
    want = np.stack([rep.stats[nm].median for nm in rep.series_names] +
                    [rep.stats[nm].mean for nm in rep.series_names])
    assert np.array_equal(got, want, equal_nan=True)


class OracleShardUpdater(OracleUpdater):
    """OracleUpdater with the FusedMetaUpdate.step(prop, diff, p_in, p_out) shape."""

    def step(self, prop, diff, p_in, p_out):
        super().step(prop.numpy(), diff.numpy(), p_in.numpy())
        p_out.copy_(torch.from_numpy(self.out))


def _shared_worker(rank, world, port, n, steps, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_bind import Oracle
    rs = np.random.RandomState(100 + rank)  # each rank renders different tiles
    step = mgdist.SharedParamStep(OracleShardUpdater(Oracle(), n // world), n)
    params = torch.full((n,), 0.2, dtype=torch.float64)
    out = torch.empty_like(params)
    for t in range(steps):
        prop = torch.from_numpy(rs.standard_normal(n))
        diff = torch.zeros(n, dtype=torch.float64) if t == 0 else \
            torch.from_numpy(0.1 * rs.standard_normal(n))
        step(prop, diff, params, out)
        params, out = out, params
    if rank == 0:
        np.save(result_path, params.numpy())
    dist.destroy_process_group()


def test_shared_parameter_reduce_scatter_update(oracle, tmp_path):
    """Tile-sharded shared parameters: reduce-scatter of the partial sample
    pairs + sharded fused update + all-gather == the single-process update on
    the summed pairs."""
    n, steps, world = 4096, 8, 2
    out = str(tmp_path / "shared.npy")
    mp.spawn(_shared_worker, args=(world, free_port(), n, steps, out), nprocs=world, join=True)
    got = np.load(out)
    rss = [np.random.RandomState(100 + r) for r in range(world)]
    up = OracleUpdater(oracle, n)
    p = np.full(n, 0.2)
    for t in range(steps):
        props = [r.standard_normal(n) for r in rss]
        diffs = [np.zeros(n) if t == 0 else 0.1 * r.standard_normal(n) for r in rss]
        up.step(props[0] + props[1], diffs[0] + diffs[1], p)
        p = up.out
    np.testing.assert_allclose(got, p, rtol=1e-12, atol=1e-15)
