"""Times the fused mini-render iteration (fp32, 16.7M pixels; argv: spp
[default 2], rng philox|mt64 [default philox]) for the IEEE kernel and every schedule of the TMA-fed fast kernel
(mg_set_option render_fast / render_fast_variant), interleaved, CUDA events
on the run's stream.  Prints one JSON line per schedule."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15676_b200 import _lib, api  # noqa: E402

L = _lib.load()
P, spp = 1 << 24, int(sys.argv[1]) if len(sys.argv) > 1 else 2
rng = sys.argv[2] if len(sys.argv) > 2 else "philox"
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
run = api.MiniRenderRun(P, spp, gen_seed=1, lr=0.01, rng=rng, dtype=torch.float32)
nv = int(os.environ.get("RF_VARIANTS", "16"))
only = [int(x) for x in os.environ.get("RF_ONLY", "").split(",") if x]
cfgs = [("ieee", 0, -1), ("fast_default", 1, -1)] + [(f"fast{v}", 1, v) for v in (only or range(nv))]
res = {c[0]: [] for c in cfgs}
s = run.ctx.stream
for _ in range(3):
    run.step()
for rep in range(int(os.environ.get("RF_REPS", "4"))):
    for name, fast, v in cfgs:
        L.mg_set_option(b"render_fast", fast)
        L.mg_set_option(b"render_fast_variant", v)
        run.step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(20):
            run.step()
        b.record(s)
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / 20)
L.mg_set_option(b"render_fast", 1)
L.mg_set_option(b"render_fast_variant", -1)
for name, ts in res.items():
    ms = min(ts)
    gbs = 60 * P / (ms / 1e3) / 1e9
    # bytes: the nine-array pass (60 B/pixel); mt64 adds the draws' write+read
    print(json.dumps({"kernel": name, "spp": spp, "rng": rng, "ms": ms, "all_ms": ts, "gbs": gbs,
                      "frac": gbs / peak, "pairs_per_s": P * spp / (ms / 1e3)}), flush=True)
