#!/bin/bash
# Run ON THE GPU BOX (under gpurun): configs[4] (and configs[3]) mesh
# iteration — plain timing, then a per-launch metric list over whole
# iterations (duration, DRAM bytes, issue activity, SIMT efficiency), then
# one `--set full` capture per wavefront stage (the depth-1 launch of the
# third iteration).  Summaries in gpurun_out/; .ncu-rep files in /tmp.
set -u
mkdir -p gpurun_out
CMD="python tools/mesh_large_probe.py"
timeout 600 $CMD > gpurun_out/pm_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/pm_plain.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum
timeout 1200 ncu --metrics $M --clock-control none --csv -k regex:'wf_|mesh_|meta_update|fixed|tex_ilv' \
  --log-file gpurun_out/pm_launches.csv $CMD > gpurun_out/pm_ncu_launch.log 2>&1
for k in wf_isect:17 wf_shade:17 wf_shadow:17 wf_scatter:2 mesh_finalize:2; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
    -o /tmp/pm_$name -f $CMD > gpurun_out/pm_ncu_$name.log 2>&1
  bash tools/ncu_extract.sh /tmp/pm_$name.ncu-rep gpurun_out/pm_full_$name.csv
  ncu -i /tmp/pm_$name.ncu-rep --page details > gpurun_out/pm_details_$name.txt 2>&1
done
echo done
