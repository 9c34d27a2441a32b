#!/bin/bash
# A/B of the fp32 traversal variants (tools/mesh_ab_options.py, in-process,
# bit-identity checked) on configs[4] and configs[3], plus the mesh tests.
for opt in mesh_smem_stack mesh_bvh8; do
  python tools/mesh_ab_options.py $opt 0 1 > gpurun_out/ab_${opt}_4.json 2>&1
  python tools/mesh_ab_options.py $opt 0 1 --c3 > gpurun_out/ab_${opt}_3.json 2>&1
done
python -m pytest -q -p no:cacheprovider tests/test_gpu_mesh.py -x > gpurun_out/t_mesh8.log 2>&1
tail -2 gpurun_out/t_mesh8.log
for f in gpurun_out/ab_mesh_*.json; do echo $f; cut -c1-260 $f; done
