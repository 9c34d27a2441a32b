"""configs[4] / configs[3]: fused update with and without the touch map
(interleaved rounds, ms per iteration) and the touched-cell fraction."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

c3 = "--c3" in sys.argv
mk = (lambda: api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4,
                                     dtype=torch.float32)) if c3 else \
     (lambda: api.MeshLargeProblem(target_spp=2))
runs = {}
for tm in (True, False):
    prob = mk()
    runs[tm] = (prob, api.MeshTextureRun(prob, "meta", lr=0.005, touch_map=tm))
    for _ in range(3):
        runs[tm][1].step()
torch.cuda.synchronize()
prob, run = runs[True]
prob.sample_pair(run.params, run.prev, 99, run.key, finalize=False)
torch.cuda.synchronize()
bits = prob.touch.view(torch.uint8)
frac = float(sum(int(((bits >> k) & 1).sum()) for k in range(8))) / (prob.touch.numel() * 32)
run.upd.step_fixed(prob.accum, *prob.fixed_layout(), run.params, run.prev.clone(), touch=prob.touch)
res = {True: [], False: []}
for _ in range(5):
    for tm in (True, False):
        r = runs[tm][1]
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            r.step()
        b.record()
        torch.cuda.synchronize()
        res[tm].append(round(a.elapsed_time(b) / 3, 4))
same = torch.equal(runs[True][1].params, runs[False][1].params)
print(json.dumps({"scene": "configs3" if c3 else "configs4", "touched_cell_fraction": round(frac, 4),
                  "ms_touch": res[True], "ms_plain": res[False]}), flush=True)
