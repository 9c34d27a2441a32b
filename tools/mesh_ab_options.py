"""In-process A/B of mesh renderer options (mg_set_option) on BASELINE
configs[4] (1024^2, 16 objects / ~503k triangles, depth 8, 1 FD + 4 prop
spp, fp32) and configs[3] (512^2, 22k triangles, depth 6): first the
sample pair of both settings on the same parameters must be bit-identical,
then interleaved timing of full optimisation iterations (sample pair +
fused update), CUDA events, min over rounds.

  python tools/mesh_ab_options.py OPTION [VALUE_A VALUE_B] [--c3]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2309_15676_b200 import _lib, api  # noqa: E402

L = _lib.load()
opt = sys.argv[1].encode()
vals = [int(sys.argv[2]), int(sys.argv[3])] if len(sys.argv) > 3 else [0, 1]
scenes = []
if "--c3" in sys.argv:
    scenes.append(("configs3", lambda: api.MeshTextureProblem(512, 512, 512, max_vertices=6,
                                                             target_spp=4, dtype=torch.float32)))
else:
    scenes.append(("configs4", lambda: api.MeshLargeProblem(target_spp=2)))
for name, make in scenes:
    prob = make()
    run = api.MeshTextureRun(prob, "meta", lr=0.005)
    for _ in range(3):
        run.step()
    torch.cuda.synchronize()
    pairs = []
    for v in vals:
        L.mg_set_option(opt, v)
        pr = prob.sample_pair(run.params, run.prev, 5, run.key)
        torch.cuda.synchronize()
        pairs.append((pr.prop.clone(), pr.diff.clone(), float(prob.loss_buf[0])))
    same = all(torch.equal(a, b) for a, b in zip(pairs[0][:2], pairs[1][:2]))
    res = {v: [] for v in vals}
    for _ in range(4):
        for v in vals:
            L.mg_set_option(opt, v)
            run.step()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                run.step()
            b.record()
            torch.cuda.synchronize()
            res[v].append(a.elapsed_time(b) / 3)
    print(json.dumps({"scene": name, "option": opt.decode(), "bit_identical_pair": same,
                      "loss": [p[2] for p in pairs],
                      "ms": {str(v): round(min(t), 4) for v, t in res.items()},
                      "all": {str(v): [round(x, 3) for x in t] for v, t in res.items()}}),
          flush=True)
