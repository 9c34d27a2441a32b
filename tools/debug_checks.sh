#!/bin/bash
# In place of compute-sanitizer (closed on the GPU pool): the -m gpu subset
# that exercises every synchronisation-heavy kernel, run against the
# device-check build libmgcuda_debug.so (MG_DCHECK asserts: TMA ring and tile
# bounds, queue / traversal-stack capacities, accumulator cells, reduction
# grid sizes, cluster ranks) — a violated invariant is a device assert and a
# failed test.  Run ON THE GPU BOX; log gpurun_out/debug_checks.log.
mkdir -p gpurun_out
export MG_LIB=$PWD/paper_2309_15676_b200/libmgcuda_debug.so
test -f "$MG_LIB" || { echo "no $MG_LIB (make -C paper_2309_15676_b200/csrc debug)"; exit 1; }
python -c "from paper_2309_15676_b200 import _lib; print('library:', _lib.LIB_PATH)" \
  > gpurun_out/debug_checks.log 2>&1
# negative control: a deliberately failing check must surface as MG_ECUDA
python -c "
from paper_2309_15676_b200 import _lib, api
rc = _lib.load().mg_debug_selftest(api.Context.default().h)
print('selftest rc', rc, '(MG_ECUDA expected: checks are live)')
" >> gpurun_out/debug_checks.log 2>&1
timeout 3000 python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_parity.py tests/test_gpu_update_scale.py tests/test_gpu_render.py \
  tests/test_gpu_mt64_jump.py tests/test_gpu_aggregate.py tests/test_gpu_mesh.py \
  tests/test_gpu_quad.py tests/test_gpu_helix.py tests/test_gpu_acceptance.py \
  >> gpurun_out/debug_checks.log 2>&1
echo "rc=$?" >> gpurun_out/debug_checks.log
grep -c "Assertion \`" gpurun_out/debug_checks.log | sed 's/^/device asserts: /' >> gpurun_out/debug_checks.log
tail -4 gpurun_out/debug_checks.log
