import sys, time, torch
sys.path.insert(0, ".")
from paper_2309_15676_b200 import api
ctx = api.Context.default()
t0 = time.time()
mprob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4, dtype=torch.float32, ctx=ctx)
print("setup", time.time() - t0, mprob.scene.info(), flush=True)
mrun = api.MeshTextureRun(mprob, optimizer="meta", lr=0.005)
for _ in range(2): mrun.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); 
for _ in range(5): mrun.step()
b.record(); torch.cuda.synchronize()
print("ms/it", a.elapsed_time(b) / 5, "loss", mrun.loss_estimate(), flush=True)
