import sys, torch
sys.path.insert(0, ".")
from paper_2309_15676_b200 import api
from paper_2309_15676_b200._lib import check, load
for leaf in (1, 2, 3, 4, 6):
    check(load().mg_set_option(b"bvh_leaf_size", leaf))
    prob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4, dtype=torch.float32)
    run = api.MeshTextureRun(prob, "meta", lr=0.005)
    for _ in range(2): run.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): run.step()
    b.record(); torch.cuda.synchronize()
    print("leaf", leaf, prob.scene.info(), "ms/it", round(a.elapsed_time(b)/5, 3), flush=True)
