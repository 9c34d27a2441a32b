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
