#!/usr/bin/env python
"""Benchmark of the B200 hot path: BASELINE.json configs[1], the fused
meta-estimator update (Moment2 x2 + decoupled diff variance + MetaEstimator
step + parameter update + step-norm/loss reductions, harness.cpp:144-188).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n PARAMS] [--impl ours|reference]

One step = one mg_meta_update over N fp32 parameters per GPU with the state
carried across steps (weak scaling: every rank owns N parameters of one
logical parameter vector; the global step norm / loss are all-reduced with
NCCL each step, on the device, because the diff decoupling of the next step
needs the GLOBAL ||delta pi||^2, problems.cpp:214 / SPEC.md:131).

Inputs: prop ~ N(mu_i, sigma_i^2), diff ~ N(0, (0.1 sigma_i)^2), mu_i ~ U(-1,1),
sigma_i ~ U(0.1, 2) (seeded synthetic, BASELINE.json configs[1]); a pool of 4
batches resident in HBM (2 x 4 x N bytes each, far larger than L2, so no L2
flush is needed) cycled over the steps.  The timed region contains only the
update kernels (and the scalar all-reduce for N>1).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gradient samples/sec (prop+FD pairs) & optimisation iterations/sec vs roofline"
UNIT = "pairs/s"
BYTES_PER_PARAM = {"f32": 56, "f64": 112}  # 8 streams read + 6 written


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # configs[1]: 100 steps, state carried
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=1 << 28, help="parameters per GPU")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pool", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-n", type=int, default=None,
                    help="cpu_baseline sample size (default: --n, the full workload)")
    ap.add_argument("--dry-run", action="store_true",
                    help="form the process group (gloo without a GPU) and print its shape only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--extras", action="store_true",
                    help="force the secondary measurements (default: on for a single GPU)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary measurements (Adam, fused renders, F1 scenes)")
    ap.add_argument("--no-tma", action="store_true", help="register-streaming kernel instead of TMA")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples)}


TRAFFIC_FILE = os.path.join("profiles", "r02_meta_update_traffic.json")


def ncu_traffic(n, dtype):
    """DRAM bytes per launch of the fused update: NOT measured by this run —
    the committed ncu capture (TRAFFIC_FILE: dram__bytes_read.sum +
    dram__bytes_write.sum of one launch at 2^28 fp32, tools/profile_r02.sh)
    scaled to n; None for a dtype not captured."""
    try:
        with open(os.path.join(ROOT, TRAFFIC_FILE)) as f:
            d = json.load(f)
        return d["bytes_per_param"] * n if dtype == "f32" else None
    except Exception:
        return None


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload_config(n, world):
    """The `config` object of BOTH arms (same workload, same keys)."""
    return {"workload": "meta-update-microbench (BASELINE configs[1])",
            "params_per_gpu": n, "global_params": n * world,
            "l2": "inputs > L2 (no flush)", "parallelism": f"param-shard x{world}",
            "beta_f": 0.9, "beta_delta": 0.5, "lr": 0.01, "steps_state_carried": True}


# --------------------------------------------------------------- reference
def cpu_reference(n, steps, threads, warmup=1, pool=2, seed=0):
    """Times the UNMODIFIED reference (oracle/_ref) meta update: Moment2 x2 +
    diff decoupling + MetaEstimator::step + params += delta, fp64, on the
    configs[1] input distributions (seeded numpy PCG64).  Returns (pairs/s,
    mean seconds per timed step, kind)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import RefLib, ref_available
    if not ref_available():
        raise RuntimeError("oracle/_ref not built (make -C oracle/ref)")
    rs = np.random.default_rng(seed)
    mu = rs.uniform(-1, 1, n)
    sig = rs.uniform(0.1, 2.0, n)
    props = np.empty((pool, n))
    diffs = np.empty((pool, n))
    for k in range(pool):
        rs.standard_normal(out=props[k])
        props[k] *= sig
        props[k] += mu
        rs.standard_normal(out=diffs[k])
        diffs[k] *= sig
        diffs[k] *= 0.1
    del mu, sig
    sec, _ = RefLib().meta_update_bench(props, diffs, 1e-4, steps, threads, warmup=warmup)
    return n / sec, sec, "reference"


def run_reference_arm(args):
    """The reference's own CPU implementation of the path (oracle/_ref: the
    unmodified reference sources), on the SAME workload as our arm: N =
    --n parameters per GPU (2^28 by default), configs[1] inputs, state
    carried, all host threads.  At --gpus N the job's N x --n parameters
    are processed shard after shard by the same cores, so the throughput
    (pairs/s) is the one measured on one shard.  Rank 0 alone runs."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = args.n
    gpus = max(args.gpus, world)
    t0 = time.time()
    val, sec, kind = cpu_reference(n, args.steps, threads, warmup=args.warmup)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(n, gpus),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{n} params/step (the full per-GPU workload), mean of "
                                   f"{args.steps} timed steps after {args.warmup} warm-up, "
                                   f"{threads} std::threads over contiguous chunks, fp64"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    from paper_2309_15676_b200 import api

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:  # torchrun: NCCL even for N = 1
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    ctx = api.Context(local)
    stream = ctx.stream
    if args.no_tma:
        from paper_2309_15676_b200 import _lib
        _lib.load().mg_set_option(b"disable_tma", 1)
    n = args.n
    dt = torch.float32 if args.dtype == "f32" else torch.float64

    # ---- synthetic inputs (untimed), BASELINE.json configs[1]
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    mu = torch.rand(n, device=dev, dtype=dt, generator=g) * 2 - 1
    sig = torch.rand(n, device=dev, dtype=dt, generator=g) * 1.9 + 0.1
    props = [mu + sig * torch.randn(n, device=dev, dtype=dt, generator=g) for _ in range(args.pool)]
    diffs = [0.1 * sig * torch.randn(n, device=dev, dtype=dt, generator=g) for _ in range(args.pool)]
    zero_diff = torch.zeros(n, device=dev, dtype=dt)
    del mu
    pa = torch.zeros(n, device=dev, dtype=dt)
    pb = torch.empty_like(pa)
    upd = api.FusedMetaUpdate(n, dtype=dt, lr=0.01, beta_f=0.9, beta_delta=0.5, ctx=ctx)
    torch.cuda.synchronize()

    sc = upd.scalars_buf  # 4 reducible doubles first

    kev = []  # (start, end) events around each kernel launch of the timed region

    def step(t, timed=False):
        src, dst = (pa, pb) if t % 2 == 0 else (pb, pa)
        d = zero_diff if t == 0 else diffs[t % args.pool]
        if timed:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(stream)
        upd.step(props[t % args.pool], d, src, dst)
        if timed:
            ev[1].record(stream)
            kev.append(ev)
        if pg is not None:  # global ||dpi||^2, #changed, loss, #nonfinite
            pg.all_reduce(sc[:4])

    t = 0
    for _ in range(args.warmup):
        step(t)
        t += 1
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step(t, timed=True)
            t += 1
        e1.record(stream)
        torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launches - launches0
    if pg is not None:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = n * world * args.steps / (ms / 1e3)
    scal = upd.scalars()

    # ---- roofline: the kernel's average launch duration over the timed
    # region (events around every launch, on the launching stream)
    k_ms = sum(a.elapsed_time(b) for a, b in kev) / len(kev)
    peak, peak_kind = measured_peak()
    algo_bytes = BYTES_PER_PARAM[args.dtype] * n
    achieved = algo_bytes / (k_ms / 1e3) / 1e9

    # ---- e2e through the public API with HOST buffers (pinned), H2D of the
    # step's sample pair and D2H of its scalars inside the timed region
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    hp = [x.cpu().pin_memory() for x in props[:2]]
    hd = [x.cpu().pin_memory() for x in diffs[:2]]
    # double-buffered device inputs: step k+1's H2D copy (copy stream)
    # overlaps step k's update (compute stream); the copy is PCIe-bound
    dbuf = [(torch.empty_like(pa), torch.empty_like(pa)) for _ in range(2)]
    host_sc = torch.empty(8, dtype=torch.float64).pin_memory()
    cstream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def prefetch(k):
        with torch.cuda.stream(cstream):
            if k >= 2:
                cstream.wait_event(consumed[k % 2])     # buffer free again
            dbuf[k % 2][0].copy_(hp[k % 2], non_blocking=True)
            dbuf[k % 2][1].copy_(hd[k % 2], non_blocking=True)
            copied[k % 2].record(cstream)

    f0.record(stream)
    cstream.wait_event(f0)
    prefetch(0)
    for k in range(e2e_steps):
        if k + 1 < e2e_steps:
            prefetch(k + 1)
        stream.wait_event(copied[k % 2])
        src, dst = (pa, pb) if t % 2 == 0 else (pb, pa)
        upd.step(dbuf[k % 2][0], dbuf[k % 2][1], src, dst)
        consumed[k % 2].record(stream)
        if pg is not None:
            pg.all_reduce(sc[:4])
        host_sc.copy_(sc, non_blocking=True)
        t += 1
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    if pg is not None:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_val = n * world * e2e_steps / (e2e_ms / 1e3)
    esz = 4 if args.dtype == "f32" else 8

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "iterations_per_s": 1e3 / ms_step,
            "impl": "ours", "config": workload_config(n, world),
            "kernel": "register-streaming" if args.no_tma else "tma-bulk-pipeline",
            "pool_batches": args.pool,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(n, args.dtype),
                         "traffic_source": f"committed ncu capture {TRAFFIC_FILE} "
                                           "(bytes/param x n), not this run",
                         "frac_vs_8tbs_spec": achieved / 8000.0,
                         "peak_kind": peak_kind,
                         "kernel_ms": k_ms, "algorithmic_bytes": algo_bytes},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 2 * esz * n,
                    "d2h_bytes_per_step": 64, "steps": e2e_steps},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "final_scalars": {"ssn": scal.ssn, "changed": scal.changed,
                              "nonfinite": scal.nonfinite},
        }
    if pg is not None:
        pg.barrier()
    del props, diffs
    torch.cuda.empty_cache()
    if world > 1 and not args.no_extras:
        # first multi-rank run of the peer-memory path happens on the
        # driver's box: a watchdog keeps the headline line if the extra
        # hangs (every rank exits 0 after rank 0 has printed it)
        def give_up():
            if rank == 0:
                out = dict(line)
                out["extras"] = {"mesh_large_tiled_error": "timed out after 300 s"}
                print(json.dumps(out), flush=True)
            os._exit(0)
        dog = threading.Timer(300.0, give_up)
        dog.daemon = True
        dog.start()
        try:
            sh = sharded_extras(args, ctx, pg, rank, world)
        except Exception as e:  # recorded; the other ranks hit the watchdog
            sh = {"mesh_large_tiled_error": f"{type(e).__name__}: {e}"}
        dog.cancel()
        if rank == 0:
            line["extras"] = sh
    if rank == 0 and not args.no_extras and (world == 1 or args.extras):
        line.setdefault("extras", {}).update(extras(args, ctx))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cn = args.cpu_n or n
        try:
            cv, csec, kind = cpu_reference(cn, 1, 1, warmup=1)
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": 1, "kind": kind,
                                    "sample": f"{cn} params fp64 (the full workload), 1 warm-up "
                                              f"+ 1 timed step, 1 thread (the reference's "
                                              f"per-run math is single-threaded)"}
        except Exception as e:  # reported, never replaces our number
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def sharded_extras(args, ctx, pg, rank, world):
    """N > 1: north_star's real split, BASELINE configs[4] (1024^2, 16
    objects / ~503k triangles, 83.9M texture parameters, depth 8, 1 FD + 4
    proportional spp) with the image rows sharded across the ranks
    (dist.TiledRenderStepP2P: each rank adds its adjoints straight into the
    owning rank's fixed-point shard over NVLink, fused update on the shard,
    parameters all-gathered, 4 scalars all-reduced).  Strong scaling (same
    image).  Also the all-gather of the 83.9M-float parameter vector alone,
    as bus bandwidth.  Every rank takes part; times are max over ranks
    (CUDA events)."""
    import torch
    from paper_2309_15676_b200 import api
    from paper_2309_15676_b200.dist import TiledRenderStepP2P
    out = {}
    dev = torch.device("cuda", ctx.device)

    def agree(ok):
        f = torch.tensor([0.0 if ok else 1.0], device=dev, dtype=torch.float64)
        pg.all_reduce(f)
        return f.item() == 0.0

    def max_ms(ms):
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    err = None
    try:
        prob = api.MeshLargeProblem(target_spp=2, ctx=ctx)
        step = TiledRenderStepP2P(prob, lr=0.005)
    except Exception as e:
        err = f"{type(e).__name__}: {e}"
    if not agree(err is None):
        out["mesh_large_tiled_error"] = err or "another rank failed to build the scene"
        return out
    try:
        for _ in range(2):
            step.step()
        torch.cuda.synchronize()
        ok = True
    except Exception as e:
        err, ok = f"{type(e).__name__}: {e}", False
    if not agree(ok):
        out["mesh_large_tiled_error"] = err or "another rank failed in the warm-up iterations"
        return out
    pg.barrier()
    K = 5
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream)
    for _ in range(K):
        step.step()
    b.record(ctx.stream)
    torch.cuda.synchronize()
    ms = max_ms(a.elapsed_time(b) / K)
    n = prob.dim()
    gather_bytes = 4 * n  # the whole parameter vector lands on every rank
    # the all-gather alone (NCCL over NVLink), bus bandwidth convention
    shard = torch.empty(n // world, device=dev)
    full = torch.empty(n, device=dev)
    for _ in range(2):
        pg.all_gather_into_tensor(full, shard)
    torch.cuda.synchronize()
    pg.barrier()
    a.record()
    for _ in range(5):
        pg.all_gather_into_tensor(full, shard)
    b.record()
    torch.cuda.synchronize()
    ag_ms = max_ms(a.elapsed_time(b) / 5)
    out["mesh_large_1024px_tiled_p2p"] = {
        "n_gpus": world, "ms_per_iteration": ms, "iterations_per_s": 1e3 / ms,
        "paths_per_s": prob.draws_per_sample() / (ms / 1e3), "texture_params": n,
        "scaling": "strong (same image, rows split)",
        "allgather_bytes_per_iteration": gather_bytes,
        "allgather_ms": ag_ms,
        "allgather_busbw_gbs": gather_bytes * (world - 1) / world / (ag_ms / 1e3) / 1e9,
        "scalar_allreduce_bytes": 32}
    del step, prob, shard, full
    torch.cuda.empty_cache()
    return out


def extras(args, ctx):
    """Secondary measurements, each guarded (a failure is recorded, never
    fatal): Adam kernel roofline, fused mini-render iterations, the F1
    path-traced scenes of BASELINE configs[0], [2], [3], [4], BVH ray
    throughput, the replicate runner."""
    import torch
    from paper_2309_15676_b200 import api
    out = {}
    n = args.n
    dev = torch.device("cuda", ctx.device)
    peak, _ = measured_peak()

    def timed(step, iters, warm=2):
        """ms per call of step() on ctx's stream (CUDA events)."""
        for _ in range(warm):
            step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream)
        for _ in range(iters):
            step()
        b.record(ctx.stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters

    def adam():
        g = torch.randn(n, device=dev)
        buf = [torch.zeros(n, device=dev), torch.empty(n, device=dev)]
        ad = api.FusedAdamUpdate(n, ctx=ctx)
        k = [0]

        def step():
            ad.step(g, buf[k[0] % 2], buf[(k[0] + 1) % 2])
            k[0] += 1
        ms = timed(step, 10, warm=3)
        out["adam_update_f32"] = {"ms": ms, "gbs": 28 * n / (ms / 1e3) / 1e9,
                                  "frac": 28 * n / (ms / 1e3) / 1e9 / peak}

    def update_sizes():
        # configs[1]'s smaller sizes, 100 steps with state carried: 2^24 eager;
        # 2^20 (59 MB, L2-resident, launch-bound) as ONE CUDA graph holding
        # the 100 captured steps (each step's host scalars baked in at
        # capture), replayed; no roofline judgement at 2^20
        side = torch.cuda.Stream(device=dev)
        gctx = api.Context(ctx.device, stream=side)
        for m in (1 << 20, 1 << 24):
            gen = torch.Generator(device=dev).manual_seed(7)
            mu = torch.rand(m, device=dev, generator=gen) * 2 - 1
            sg = torch.rand(m, device=dev, generator=gen) * 1.9 + 0.1
            pr = [mu + sg * torch.randn(m, device=dev, generator=gen) for _ in range(2)]
            df = [0.1 * sg * torch.randn(m, device=dev, generator=gen) for _ in range(2)]
            bufs = [torch.zeros(m, device=dev), torch.empty(m, device=dev)]
            up = api.FusedMetaUpdate(m, lr=0.01, ctx=gctx)

            def hundred():
                up.reset()
                for t in range(100):
                    up.step(pr[t % 2], df[t % 2], bufs[t % 2], bufs[(t + 1) % 2])
            torch.cuda.synchronize()
            with torch.cuda.stream(side):
                hundred()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if m == 1 << 20:
                    g = torch.cuda.CUDAGraph()
                    up.reset()
                    with torch.cuda.graph(g, stream=side):
                        for t in range(100):
                            up.step(pr[t % 2], df[t % 2], bufs[t % 2], bufs[(t + 1) % 2])
                    g.replay()
                    torch.cuda.synchronize()
                    a.record(side)
                    for _ in range(5):
                        g.replay()
                    b.record(side)
                    torch.cuda.synchronize()
                    ms = a.elapsed_time(b) / 500
                    mode = "cuda graph of 100 steps"
                else:
                    a.record(side)
                    hundred()
                    b.record(side)
                    torch.cuda.synchronize()
                    ms = a.elapsed_time(b) / 100
                    mode = "eager"
            gbs = BYTES_PER_PARAM["f32"] * m / (ms / 1e3) / 1e9
            r = {"params": m, "ms_per_step": ms, "pairs_per_s": m / (ms / 1e3), "gbs": gbs,
                 "mode": mode}
            if m == 1 << 24:
                r["frac"] = gbs / peak
            else:
                r["note"] = "L2-resident (59 MB < 126 MB L2): launch-bound, not roofline-judged"
            out[f"meta_update_2^{m.bit_length() - 1}_f32"] = r
            del pr, df, bufs, up

    def update_f64():
        # the parity-mode (fp64, bit-exact with the reference) fused update at
        # the headline size, 2^28 parameters, state carried, 20 steps (the
        # like-for-like arithmetic of the reference arm)
        m = n
        gen = torch.Generator(device=dev).manual_seed(8)
        mu = torch.rand(m, device=dev, dtype=torch.float64, generator=gen) * 2 - 1
        sg = torch.rand(m, device=dev, dtype=torch.float64, generator=gen) * 1.9 + 0.1
        pr = [mu + sg * torch.randn(m, device=dev, dtype=torch.float64, generator=gen)
              for _ in range(2)]
        del mu
        df = [0.1 * sg * torch.randn(m, device=dev, dtype=torch.float64, generator=gen)
              for _ in range(2)]
        del sg
        bufs = [torch.zeros(m, device=dev, dtype=torch.float64),
                torch.empty(m, device=dev, dtype=torch.float64)]
        up = api.FusedMetaUpdate(m, dtype=torch.float64, lr=0.01, ctx=ctx)
        ev = []
        for t in range(24):
            if t >= 4:
                e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                e[0].record(ctx.stream)
            up.step(pr[t % 2], df[t % 2] if t else torch.zeros_like(bufs[0]), bufs[t % 2],
                    bufs[(t + 1) % 2])
            if t >= 4:
                e[1].record(ctx.stream)
                ev.append(e)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)
        gbs = BYTES_PER_PARAM["f64"] * m / (ms / 1e3) / 1e9
        out["meta_update_2^28_f64"] = {"params": m, "ms_per_step": ms,
                                       "pairs_per_s": m / (ms / 1e3), "gbs": gbs,
                                       "frac": gbs / peak, "steps_timed": len(ev),
                                       "bytes_per_param": BYTES_PER_PARAM["f64"]}
        del pr, df, bufs, up

    def minirender(rng):
        # fused mini-render iteration at scale (16.7M pixels): one kernel per
        # iteration, sample pair in registers; philox draws, or the
        # reference's exact mt19937_64 stream (engines tiling ONE stream via
        # GF(2) jump-ahead, bit-identical draws)
        P, spp = 1 << 24, 2
        run = api.MiniRenderRun(P, spp, gen_seed=1, lr=0.01, rng=rng, dtype=torch.float32,
                                ctx=ctx)
        ms = timed(run.step, 50 if rng == "philox" else 10, warm=3 if rng == "philox" else 2)
        r = {"pixels": P, "spp": spp, "ms_per_iteration": ms,
             "pairs_per_s": P * spp / (ms / 1e3)}
        if rng == "philox":
            r.update({"gbs": 60 * P / (ms / 1e3) / 1e9, "frac": 60 * P / (ms / 1e3) / 1e9 / peak,
                      "loss": run.scalars().loss})
        else:
            r["engines"] = run.rng.n
        out["minirender_fused_philox_f32" if rng == "philox" else
            "minirender_fused_mt64_exact_f32"] = r

    def quad():
        # F1 slice, configs[0]: 64x64 textured quad, 32x32 RGB texture, 1 FD +
        # 2 proportional spp; and a 1024^2 / 512^2-texture variant.  A context
        # on its own stream, so the loop can also run as a CUDA graph.
        qs = torch.cuda.Stream(device=dev)
        qctx = api.Context(ctx.device, stream=qs)

        def qtimed(fn, iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(qs)
            fn(iters)
            b.record(qs)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / iters

        for W, R, iters in ((64, 32, 200), (1024, 512, 50)):
            with torch.cuda.stream(qs):
                prob = api.QuadTextureProblem(W, W, R, target_spp=64, dtype=torch.float32,
                                              ctx=qctx)
                run = api.QuadTextureRun(prob, optimizer="meta", lr=0.01)
                run.run(3)
                ms = qtimed(run.run, iters)
                # the same loop as one captured two-step CUDA graph, replayed
                # (device iteration counter and Moment2 coefficient;
                # bit-identical to the eager loop, tests/test_gpu_quad.py)
                run.run(2, graph=True)
                ms_g = qtimed(lambda k: run.run(k, graph=True), iters)
            out[f"quad_texture_{W}px_{R}tex_f32"] = {
                "iterations": iters, "ms_per_iteration": ms, "iterations_per_s": 1e3 / ms,
                "path_samples_per_s": prob.draws_per_sample() / (ms / 1e3),
                "graph_ms_per_iteration": ms_g, "graph_iterations_per_s": 1e3 / ms_g,
                "texture_params": prob.dim()}

    def helix():
        # F1 slice 2, configs[2]: 256x256 helix of 64 spheres, depth 4 + NEE,
        # 5 principled-BSDF parameters
        for dtn, dt in (("f32", torch.float32), ("f64", torch.float64)):
            prob = api.HelixProblem(256, 256, target_spp=16, dtype=dt, ctx=ctx)
            run = api.HelixRun(prob, optimizer="meta", lr=0.01)
            ms = timed(run.step, 10)
            out[f"helix_256px_{dtn}"] = {"ms_per_iteration": ms, "iterations_per_s": 1e3 / ms,
                                         "paths_per_s": prob.draws_per_sample() / (ms / 1e3)}

    def mesh():
        # F1 slice 3, configs[3]: 512^2, 3 objects / 22k triangles (BVH),
        # 3 x 4 x 512^2 = 3.1M texture parameters, depth 6, 1 FD + 2 prop spp
        prob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4,
                                      dtype=torch.float32, ctx=ctx)
        run = api.MeshTextureRun(prob, optimizer="meta", lr=0.005)
        ms = timed(run.step, 5)
        # the same loop replayed as a captured two-iteration CUDA graph (56
        # launches), on a context of its own stream; bit-identical
        gs = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(gs):
            gprob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4,
                                           dtype=torch.float32, ctx=api.Context(ctx.device, stream=gs))
            grun = api.MeshTextureRun(gprob, optimizer="meta", lr=0.005)
            grun.run(3)
            grun.run(2, graph=True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(gs)
            grun.run(10, graph=True)
            b.record(gs)
            torch.cuda.synchronize()
            ms_g = a.elapsed_time(b) / 10
        out["mesh_texture_512px_f32"] = {"ms_per_iteration": ms, "iterations_per_s": 1e3 / ms,
                                         "graph_ms_per_iteration": ms_g,
                                         "paths_per_s": prob.draws_per_sample() / (ms / 1e3),
                                         "texture_params": prob.dim(), **prob.scene.info()}
        # BVH closest-hit throughput on the same scene (rays aimed at the objects)
        nr = 1 << 22
        g = torch.Generator(device="cuda").manual_seed(0)
        rnd = lambda: torch.rand(nr, device="cuda", generator=g, dtype=torch.float64)  # noqa: E731
        org = torch.stack([rnd() * 4 - 2, rnd() * 2 + 0.1,
                           torch.full((nr,), 4.0, device="cuda", dtype=torch.float64)], 1)
        tgt = torch.stack([rnd() * 3 - 1.5, rnd() * 1.1,
                           torch.zeros(nr, device="cuda", dtype=torch.float64)], 1)
        dirs = tgt - org
        dirs /= torch.linalg.vector_norm(dirs, dim=1, keepdim=True)
        rays = torch.cat([org, dirs], 1).contiguous()
        ms = timed(lambda: prob.scene.intersect(rays), 1, warm=1)
        out["mesh_bvh_closest_hit"] = {"rays": nr, "ms": ms, "rays_per_s": nr / (ms / 1e3)}

    def mesh_large():
        # F1 slice 4, configs[4]: 1024^2, 16 objects / ~503k triangles,
        # 16 x 5 x 1024^2 = 83.9M texture parameters (base rgb, roughness,
        # metalness), depth 8, 1 FD + 4 proportional spp
        prob = api.MeshLargeProblem(target_spp=2, ctx=ctx)
        run = api.MeshTextureRun(prob, optimizer="meta", lr=0.005)
        ms = timed(run.step, 3)
        out["mesh_large_1024px_f32"] = {"ms_per_iteration": ms, "iterations_per_s": 1e3 / ms,
                                        "paths_per_s": prob.draws_per_sample() / (ms / 1e3),
                                        "texture_params": prob.dim(), **prob.scene.info()}

    def runner():
        # reference harness stand-in for configs[0] (S1: mini-render P=4096,
        # spp=2, 200 iterations, meta) through api.run_experiment, wall clock
        # around the call (median of 5 after one warm-up): one replicate (a
        # thread-block cluster: producer CTA for the exact mt19937_64 stream,
        # consumer CTAs holding the state in registers) and 148 replicates
        # (one CTA each, one launch)
        import statistics
        for reps, key in ((1, "minirender_s1_single_replicate"), (148, "minirender_runner")):
            cfg = api.ExperimentConfig(problem="mini-render", pixel_count=4096, spp=2,
                                       iterations=200, seed=0, problem_seed=1, lr=0.01,
                                       replicates=reps)
            api.run_experiment(cfg, ctx=ctx)
            walls = []
            for _ in range(5):
                t0 = time.time()
                api.run_experiment(cfg, ctx=ctx)
                walls.append(time.time() - t0)
            wall = statistics.median(walls)
            out[key] = {"replicates": reps, "iterations": 200, "wall_s": wall,
                        "wall_min_s": min(walls),
                        "walls_ms": [round(x * 1e3, 3) for x in walls],
                        "pairs_per_s": reps * 200 * 4096 * 2 / wall,
                        "runner": "cluster" if reps == 1 else "one CTA per replicate"}

    for name, fn in (("update_f64", update_f64), ("update_sizes", update_sizes), ("adam", adam), ("minirender_philox", lambda: minirender("philox")),
                     ("minirender_mt64", lambda: minirender("mt64")), ("quad", quad),
                     ("helix", helix), ("mesh", mesh), ("mesh_large", mesh_large),
                     ("runner", runner)):
        try:
            fn()
        except Exception as e:  # recorded, never fatal to the headline line
            out[f"{name}_error"] = f"{type(e).__name__}: {e}"
        torch.cuda.empty_cache()
    return out


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: re-exec this command as N
    ranks under torch.distributed.run (one process per GPU, rendezvous on
    127.0.0.1); rank 0 prints the JSON line.  Returns the launcher's exit
    code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def dry_run(args):
    """Form the process group exactly as a real run would (NCCL on GPUs,
    gloo without) and print its shape: the launcher's CPU test."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend)
        ranks = [None] * world
        dist.all_gather_object(ranks, (rank, local, os.getpid()))
        dist.destroy_process_group()
    else:
        ranks = [(rank, local, os.getpid())]
    if rank == 0:
        print(json.dumps({"dry_run": True, "impl": args.impl, "n_gpus": world,
                          "ranks": [r[0] for r in ranks], "local_ranks": [r[1] for r in ranks],
                          "distinct_pids": len({r[2] for r in ranks})}), flush=True)
    return 0


def main():
    args = parse()
    launched = "WORLD_SIZE" in os.environ
    if not launched and args.gpus > 1 and args.impl == "ours":
        return spawn_ranks(args.gpus)
    _, world, _ = dist_env()
    if launched and args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks",
              file=sys.stderr)
        return 2
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
