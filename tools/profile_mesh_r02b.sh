#!/bin/bash
# Run ON THE GPU BOX: configs[4] after the wavefront tail kernel and the
# fused fixed-point update — plain timing, the per-launch metric list over
# whole iterations (for tools/mesh_stage_table.py) and one `--set full`
# capture each of the tail kernel and the fused update.
set -u
mkdir -p gpurun_out
CMD="python tools/mesh_large_probe.py"
timeout 600 $CMD > gpurun_out/pb_plain.log 2>&1 || { cat gpurun_out/pb_plain.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 1200 ncu --metrics $M --clock-control none --csv -k regex:'wf_|mesh_|meta_update|tex_ilv' \
  --log-file gpurun_out/pb_launches.csv $CMD > /dev/null 2>&1
for k in wf_tail:2 meta_update_fixed:3 wf_scatter:2; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
    -o /tmp/pb_$name -f $CMD > /dev/null 2>&1
  bash tools/ncu_extract.sh /tmp/pb_$name.ncu-rep gpurun_out/pb_full_$name.csv
  ncu -i /tmp/pb_$name.ncu-rep --page details > gpurun_out/pb_details_$name.txt 2>&1
done
python tools/mesh_stage_table.py gpurun_out/pb_launches.csv > gpurun_out/pb_stage_table.md
cat gpurun_out/pb_plain.log gpurun_out/pb_stage_table.md
