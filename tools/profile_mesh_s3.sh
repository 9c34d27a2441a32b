#!/bin/bash
# Run ON THE GPU BOX: configs[4] launch list (whole iterations) + --set full
# captures with source of the shade (depths 1, 2), scatter and isect (depth 2)
# launches; .ncu-rep copied into gpurun_out/ for per-line analysis here.
set -u
mkdir -p gpurun_out
CMD="python tools/mesh_large_probe.py"
timeout 600 $CMD > gpurun_out/ps_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/ps_plain.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 1200 ncu --metrics $M --clock-control none --csv -k regex:'wf_|mesh_|meta_update|fixed|tex_ilv' \
  --log-file gpurun_out/ps_launches.csv $CMD > gpurun_out/ps_ncu_launch.log 2>&1
for k in wf_shade:16 wf_shade:17 wf_scatter:2 wf_isect:17; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
    -o gpurun_out/ps_${name}_$skip -f $CMD > gpurun_out/ps_ncu_${name}_$skip.log 2>&1
done
echo done
