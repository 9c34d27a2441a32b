#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over a reduced -m gpu
# subset that exercises every synchronisation-heavy kernel: the TMA
# bulk-copy rings (meta update, Adam, fast mini-render), the last-CTA grid
# reductions, the block-cooperative mt19937_64 twist and the GF(2) jump,
# the cluster runner (DSMEM exchange, producer/consumer flags), the mesh
# wavefront (persistent traversal, adjoint scatter atomics) and the
# peer-memory shared-parameter kernel (emulated ranks).  Run ON THE GPU BOX.
# Logs: gpurun_out/sanitizer_<tool>.log; one summary line per tool in
# gpurun_out/sanitizer_summary.txt.
mkdir -p gpurun_out
SEL_PARITY="test_tma_pipeline_matches_register_kernel or test_adam_tma_matches_register_kernel or test_fused_meta_update_f64_bit_exact_per_step or test_mt64_streams_bit_exact or test_moment2_bit_exact or test_shared_param_peer_kernel_emulated_ranks or (test_cluster_runner_matches_cta_runner and f64-0) or test_fused_adam_update_matches_oracle or test_run_single_matches_reference_record"
TESTS=(
  "tests/test_gpu_parity.py -k"
  "tests/test_gpu_render.py -k fast_f32_kernel_tracks_fp64_run and 2"
  "tests/test_gpu_mt64_jump.py"
  "tests/test_gpu_aggregate.py"
  "tests/test_gpu_mesh.py -k sample_pair_bit_exact or tiles_sum_exactly or prev_copy_reuse or divergence_pixel_fraction"
)
: > gpurun_out/sanitizer_summary.txt
for tool in memcheck racecheck synccheck; do
  log=gpurun_out/sanitizer_$tool.log
  : > $log
  for t in "${TESTS[@]}"; do
    if [[ "$t" == "tests/test_gpu_parity.py -k" ]]; then
      args=(tests/test_gpu_parity.py -k "$SEL_PARITY")
    elif [[ "$t" == *" -k "* ]]; then
      args=(${t%% -k *} -k "${t#* -k }")
    else
      args=($t)
    fi
    echo "=== $tool: ${args[*]}" >> $log
    timeout 3000 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest -q -p no:cacheprovider -x "${args[@]}" >> $log 2>&1
    echo "rc=$?" >> $log
  done
  echo "$tool: $(grep -c 'ERROR SUMMARY: 0 errors' $log) clean processes, $(grep 'ERROR SUMMARY' $log | grep -vc ': 0 errors') with errors; pytest: $(grep -E '[0-9]+ passed' $log | tr '\n' ' ')" >> gpurun_out/sanitizer_summary.txt
done
cat gpurun_out/sanitizer_summary.txt
