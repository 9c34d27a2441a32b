#!/bin/bash
# per-stage ncu launch list (durations, DRAM bytes) of one configs[4] iteration
# for the in-tree library and every ab/<variant>; tables via tools/mesh_stage_table.py
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
for v in new $(ls ab 2>/dev/null); do
  if [ $v = new ]; then unset MG_LIB; else export MG_LIB=$PWD/ab/$v/libmgcuda.so; fi
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:'wf_|mesh_|meta_update|tex_' \
    --log-file gpurun_out/abn_$v.csv python tools/mesh_large_probe.py > gpurun_out/abn_$v.log 2>&1
done
