mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_dist_mesh.py -x -q > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
for i in 1 2; do
MG_LIB=$PWD/ab/libmgcuda.so timeout 300 python tools/mesh_large_probe.py > gpurun_out/ab_large_base$i.log 2>&1
timeout 300 python tools/mesh_large_probe.py > gpurun_out/ab_large_new$i.log 2>&1
done
MG_LIB=$PWD/ab/libmgcuda.so timeout 300 python tools/mesh_bench_probe.py > gpurun_out/ab_c3_base.log 2>&1
timeout 300 python tools/mesh_bench_probe.py > gpurun_out/ab_c3_new.log 2>&1
tail -3 gpurun_out/ab_tests.log; grep ms gpurun_out/ab_*.log
