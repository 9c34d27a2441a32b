"""Tile-sharded mesh optimisation across GPUs (BASELINE configs[3] / [4]:
"image-tile-sharded at 2/4/8 GPUs with gradient allreduce"), one process
per GPU:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mesh_scaling.py [configs3|configs4]

Each rank renders its image rows and adds its adjoints straight into the
owning rank's fixed-point shard over NVLink (dist.TiledRenderStepP2P), then
runs the fused update on its shard; the parameters are all-gathered.
Prints one JSON line (rank 0): iterations/s and paths/s over the timed
iterations, max over ranks (CUDA events)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15676_b200 import api  # noqa: E402
from paper_2309_15676_b200.dist import TiledRenderStepP2P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "configs3"
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
if which == "configs4":
    prob = api.MeshLargeProblem(target_spp=2)
else:
    prob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4)
step = TiledRenderStepP2P(prob, lr=0.005)
for _ in range(2):
    step.step()
torch.cuda.synchronize()
dist.barrier()
K = 10
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(K):
    step.step()
b.record()
torch.cuda.synchronize()
ms = torch.tensor([a.elapsed_time(b) / K], device="cuda", dtype=torch.float64)
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
if rank == 0:
    m = float(ms.item())
    print(json.dumps({"workload": which, "n_gpus": world, "ms_per_iteration": m,
                      "iterations_per_s": 1e3 / m,
                      "paths_per_s": prob.draws_per_sample() / (m / 1e3),
                      "texture_params": prob.dim(), "scaling": "strong (same image, rows split)"}),
          flush=True)
dist.barrier()
dist.destroy_process_group()
