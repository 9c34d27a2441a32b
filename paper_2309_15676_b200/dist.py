"""Multi-GPU plumbing for the hot path (one process per GPU, torch.distributed).

Two ways the path shards:

* Parameter sharding of ONE run (bench configs[1], large mini-render): each
  rank owns a contiguous shard of the parameter vector and runs the fused
  update on it; the only exchange per iteration is a SUM all-reduce of the 4
  reducible scalars (step norm, #changed, loss, #nonfinite) because the next
  iteration's diff decoupling needs the GLOBAL ||delta pi||^2
  (problems.cpp:214).  NCCL on the device, no host sync.
* Replicate sharding (run_experiment, harness.cpp:249-272): ranks run
  disjoint replicate ranges with no communication, then rank 0 gathers the
  records and reduces them in replicate order (harness.cpp:274-302), so the
  report is identical for any world size.

The compute is injected (an updater / a run function), so the same host
logic is exercised on CPU with gloo in tests/test_dist_gloo.py and on B200s
with NCCL in bench.py.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple


def shard_range(n: int, rank: int, world: int, align: int = 1024) -> Tuple[int, int]:
    """Contiguous [lo, hi) shard of n parameters; boundaries are multiples of
    `align` elements (keeps every shard 16-byte aligned and TMA-tileable)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    blocks = -(-n // align)
    lo_b = blocks * rank // world
    hi_b = blocks * (rank + 1) // world
    return min(lo_b * align, n), min(hi_b * align, n)


def replicate_range(replicates: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [begin, end) replicate range of this rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return replicates * rank // world, replicates * (rank + 1) // world


def tile_rows(height: int, rank: int, world: int) -> Tuple[int, int]:
    """Image rows [r0, r1) this rank renders for a shared-parameter problem
    (the `rows=` argument of QuadTextureProblem/HelixProblem.sample_pair).
    The renderers accumulate adjoints in 2^-40 fixed point, so the partial
    pairs of disjoint tiles sum EXACTLY to the unsharded pair: the summed
    gradient (and hence the whole run) is independent of the world size."""
    return replicate_range(height, rank, world)


class ShardedStep:
    """One iteration of a parameter-sharded run: local fused update, then one
    SUM all-reduce of the 4 reducible scalars (in place, on the scalars'
    device; NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, updater, group=None):
        self.updater = updater
        self.group = group

    def __call__(self, *args, **kwargs):
        import torch.distributed as dist
        self.updater.step(*args, **kwargs)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(self.updater.scalars_buf[:4], op=dist.ReduceOp.SUM, group=self.group)


def run_experiment_sharded(cfg, run_fn: Callable[[object, int, int], Sequence], group=None,
                           aggregate_fn: Callable | None = None):
    """Replicate-sharded run_experiment.  run_fn(cfg, begin, count) -> list of
    per-replicate records (the device runner on a GPU rank).  Returns the
    aggregate report on rank 0 (None elsewhere)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b, e = replicate_range(cfg.replicates, rank, world)
    local = list(run_fn(cfg, b, e - b)) if e > b else []
    if world > 1:
        gathered: List = [None] * world if rank == 0 else None
        dist.gather_object((b, local), gathered, dst=0, group=group)
        if rank != 0:
            return None
        records = [r for _, recs in sorted(gathered, key=lambda x: x[0]) for r in recs]
    else:
        records = local
    if aggregate_fn is None:
        from .api import aggregate as aggregate_fn
    return aggregate_fn(cfg, records)


def _reduce_scatter_sum(full, shard_out, group=None):
    """SUM-reduce `full` over ranks and keep this rank's contiguous slice
    (NCCL reduce_scatter_tensor; gloo has no reduce-scatter, so all-reduce
    + slice there — same result)."""
    import torch.distributed as dist
    if full.is_cuda:
        dist.reduce_scatter_tensor(shard_out, full, op=dist.ReduceOp.SUM, group=group)
    else:
        buf = full.clone()
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        rank = dist.get_rank(group)
        n = shard_out.numel()
        shard_out.copy_(buf[rank * n:(rank + 1) * n])


class SharedParamStep:
    """One iteration of a shared-parameter problem sharded by image tiles
    (SURVEY.md §8(e), configs 4/5): every rank renders its tiles and produces
    FULL-length partial gradient samples (prop, diff) for the one shared
    parameter vector; the partials are SUM-reduce-scattered so each rank
    owns the summed pair for its parameter shard, the fused meta update runs
    on that shard only (state is sharded too: 1/G of the optimiser memory
    per GPU), the new parameters are all-gathered, and the 4 reducible
    scalars all-reduced.  Parameter count must be divisible by world*align.

    updater: FusedMetaUpdate-like object over n/world parameters."""

    def __init__(self, updater, n: int, group=None):
        import torch.distributed as dist
        self.updater = updater
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if n % self.world:
            raise ValueError("shared parameter count must divide evenly across ranks")
        self.n, self.shard = n, n // self.world

    def __call__(self, prop_partial, diff_partial, params_full, params_full_out):
        import torch
        import torch.distributed as dist
        lo = self.rank * self.shard
        prop = torch.empty(self.shard, dtype=prop_partial.dtype, device=prop_partial.device)
        diff = torch.empty_like(prop)
        pair = torch.cat([prop_partial.view(self.world, self.shard),
                          diff_partial.view(self.world, self.shard)], dim=1).reshape(-1)
        pair_shard = torch.empty(2 * self.shard, dtype=pair.dtype, device=pair.device)
        _reduce_scatter_sum(pair, pair_shard, self.group)          # one collective for both
        prop.copy_(pair_shard[:self.shard])
        diff.copy_(pair_shard[self.shard:])
        p_in = params_full[lo:lo + self.shard].contiguous()
        p_out = torch.empty_like(p_in)
        self.updater.step(prop, diff, p_in, p_out)
        if self.world > 1:
            dist.all_reduce(self.updater.scalars_buf[:4], op=dist.ReduceOp.SUM, group=self.group)
            dist.all_gather_into_tensor(params_full_out, p_out, group=self.group)
        else:
            params_full_out.copy_(p_out)


class SharedParamStepP2P:
    """SharedParamStep as ONE kernel over NVLink peer memory per rank
    (mg_shared_meta_update): the partial sample pairs and both parameter
    ping-pong buffers live in torch symmetric memory, so each rank reduces its
    shard straight out of the peers' buffers (rank order, deterministic) and
    stores the updated shard into every peer's parameter buffer — no NCCL
    reduce-scatter/all-gather, no staging copies.  Two symmetric-memory
    barriers fence the step; the 4 scalars are all-reduced with NCCL.

    Tested with emulated ranks on one GPU (tests/test_gpu_parity.py::
    test_shared_param_peer_kernel_emulated_ranks); this round's environment
    has a single GPU, so the symmetric-memory plumbing itself is not
    exercised on >1 GPU yet."""

    def __init__(self, n: int, dtype=None, group=None, lr=0.01, beta_f=0.9, beta_delta=0.5,
                 eps_step=1e-8, eps_alpha=1e-30, clip=True, project_lo=None, init=0.0,
                 project_hi=None):
        import ctypes as C

        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        from . import _abi
        from .api import Context

        dtype = dtype or torch.float32
        self.C, self._abi, self.torch, self.dist = C, _abi, torch, dist
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        if n % self.world:
            raise ValueError("shared parameter count must divide evenly across ranks")
        self.n, self.S, self.dtype = n, n // self.world, dtype
        dev = torch.device("cuda", torch.cuda.current_device())
        self.ctx = Context.default()

        def symm(fill=None):
            t = symm_mem.empty(n, dtype=dtype, device=dev)
            if fill is not None:
                t.fill_(fill)
            h = symm_mem.rendezvous(t, self.group)
            assert t.data_ptr() == h.buffer_ptrs[self.rank], "tensor not at allocation base"
            return t, h

        self.prop, self.h_prop = symm()
        self.diff, self.h_diff = symm()
        self.params, self.h_params = symm(init)
        self.params_next, self.h_next = symm(init)
        mk = lambda: torch.empty(self.S, dtype=dtype, device=dev)  # noqa: E731
        self.state = [mk() for _ in range(5)]
        self.scalars_buf = torch.zeros(8, dtype=torch.float64, device=dev)
        from ._lib import check, load
        self._check, self._L = check, load()
        self._check(self._L.mg_scalars_write(self.ctx.h, C.c_void_p(self.scalars_buf.data_ptr()),
                                             C.byref(_abi.fresh_scalars())))
        self.meta = _abi.MetaParams(lr, eps_step, eps_alpha, int(clip))
        self.beta_f, self.beta_delta, self.project_lo = beta_f, beta_delta, project_lo
        self.project_hi = project_hi
        self.t, self.bp = 0, 1.0

    def __call__(self, target_shard=None):
        """One iteration; the caller has written this rank's partial pair into
        self.prop / self.diff (e.g. rendered straight into them)."""
        C, _abi = self.C, self._abi
        self.t += 1
        self.bp *= self.beta_f
        a = _abi.MetaUpdateArgs(meta=self.meta, prop_coef=(1.0 - self.beta_f) / (1.0 - self.bp),
                                beta_delta=self.beta_delta, first_step=int(self.t == 1),
                                project=(2 if self.project_hi is not None
                                         else int(self.project_lo is not None)),
                                proj_lo=self.project_lo or 0.0,
                                proj_hi=self.project_hi or 0.0, beta_f=self.beta_f,
                                prop_pow_advance=1)
        arr = lambda ptrs: (C.c_void_p * self.world)(*ptrs)  # noqa: E731
        self.h_prop.barrier()                      # every rank's partials are written
        self._check(self._L.mg_shared_meta_update(
            self.ctx.h, _abi.MG_F32 if self.dtype == self.torch.float32 else _abi.MG_F64,
            self.S, self.rank * self.S, self.world, C.byref(a), arr(self.h_prop.buffer_ptrs),
            arr(self.h_diff.buffer_ptrs), arr(self.h_next.buffer_ptrs),
            C.c_void_p(self.params.data_ptr()),
            *[C.c_void_p(x.data_ptr()) for x in self.state],
            None if target_shard is None else C.c_void_p(target_shard.data_ptr()),
            C.c_void_p(self.scalars_buf.data_ptr())))
        self.h_next.barrier()                      # every shard stored everywhere
        if self.world > 1:
            self.dist.all_reduce(self.scalars_buf[:4], op=self.dist.ReduceOp.SUM, group=self.group)
        self.params, self.params_next = self.params_next, self.params
        self.h_params, self.h_next = self.h_next, self.h_params


class TiledRenderStepP2P:
    """One iteration of a tile-sharded shared-parameter renderer
    (configs[3]/[4] over NVLink) with the reduce-scatter FUSED into the
    adjoint scatter: every rank renders its image rows (tile_rows) and adds
    each parameter's fixed-point contribution straight into the owning
    rank's accumulator shard through symmetric-memory peer pointers
    (mg_meshscene_sample_pair_sharded) — no full-length partial buffers, no
    reduce-scatter launch.  After a barrier each rank converts its own shard
    (mg_fixed_finalize), runs the fused meta update on it, and the new
    parameters are all-gathered (NCCL); the 4 update scalars are
    all-reduced.  Integer atomics commute, so the result is bit-identical to
    the single-process run for any number of ranks.

    problem: a MeshTextureProblem (identical on every rank)."""

    def __init__(self, problem, lr: float = 0.01, group=None, seed: int = 0, replicate: int = 0):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        from .api import FusedMetaUpdate, load
        self.torch, self.dist = torch, dist
        self.p = problem
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        n = problem.dim()
        if n % self.world:
            raise ValueError("parameter count must divide evenly across ranks")
        self.n, self.S = n, n // self.world
        dev = torch.device("cuda", torch.cuda.current_device())
        self.acc = symm_mem.empty(2 * self.S, dtype=torch.int64, device=dev)
        self.acc.zero_()
        self.h = symm_mem.rendezvous(self.acc, self.group)
        self.upd = FusedMetaUpdate(self.S, dtype=problem.dtype, lr=lr, project_lo=0.0,
                                   project_hi=1.0, ctx=problem.ctx)
        self.params = problem.initial_params()
        self.prev = self.params.clone()
        self.prop = torch.empty(self.S, dtype=problem.dtype, device=dev)
        self.diff = torch.empty_like(self.prop)
        self.key = int(load().mg_stream_seed(seed, replicate))
        self.t = 0

    def step(self):
        torch, dist = self.torch, self.dist
        from .api import fixed_finalize
        lo = self.rank * self.S
        self.h.barrier()                 # owners' accumulators are zero again
        self.p.sample_pair_sharded(self.params, self.prev, self.t, self.key,
                                   tile_rows(self.p.H, self.rank, self.world),
                                   self.h.buffer_ptrs, self.S)
        self.h.barrier()                 # every rank's atomics have landed
        fixed_finalize(self.acc, self.prop, self.diff, self.p.ctx)
        shard_new = torch.empty(self.S, dtype=self.p.dtype, device=self.prop.device)
        self.upd.step(self.prop, self.diff, self.params[lo:lo + self.S].contiguous(), shard_new)
        new = torch.empty_like(self.params)
        if self.world > 1:
            dist.all_reduce(self.upd.scalars_buf[:4], op=dist.ReduceOp.SUM, group=self.group)
            dist.all_gather_into_tensor(new, shard_new, group=self.group)
        else:
            new.copy_(shard_new)
        self.prev, self.params = self.params, new
        self.t += 1
