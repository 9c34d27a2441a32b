"""BVH builder A/B (python tools/bvh_axes_probe.py [OPTION A B]; default
bvh_sah_axes 1 3): binned SAH on the longest centroid axis (1) against all
three axes (3): configs[3] and configs[4] iteration time, node count, depth,
build time; the sample pairs must be bit-identical (closest hit does not
depend on the tree)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402
from paper_2309_15676_b200._lib import check, load  # noqa: E402

OPT = sys.argv[1].encode() if len(sys.argv) > 3 else b"bvh_sah_axes"
VA, VB = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1, 3)
for name, make in (("configs3", lambda: api.MeshTextureProblem(512, 512, 512, max_vertices=6,
                                                               target_spp=4, dtype=torch.float32)),
                   ("configs4", lambda: api.MeshLargeProblem(target_spp=2))):
    runs, pairs, info = {}, {}, {}
    for axes in (VA, VB):
        check(load().mg_set_option(OPT, axes))
        t0 = time.time()
        prob = make()
        info[axes] = dict(prob.scene.info(), setup_s=round(time.time() - t0, 2))
        runs[axes] = api.MeshTextureRun(prob, "meta", lr=0.005)
        pr = prob.sample_pair(runs[axes].params, runs[axes].prev, 3, runs[axes].key)
        pairs[axes] = (pr.prop.clone(), pr.diff.clone())
        for _ in range(2):
            runs[axes].step()
    same = all(torch.equal(a, b) for a, b in zip(pairs[VA], pairs[VB]))
    res = {VA: [], VB: []}
    for _ in range(4):
        for axes in (VA, VB):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                runs[axes].step()
            b.record()
            torch.cuda.synchronize()
            res[axes].append(round(a.elapsed_time(b) / 3, 4))
    print(json.dumps({"scene": name, "bit_identical_pair": same, "info": info,
                      "ms": {str(k): min(v) for k, v in res.items()}, "all": res}), flush=True)
    del runs, pairs
check(load().mg_set_option(OPT, VB))
