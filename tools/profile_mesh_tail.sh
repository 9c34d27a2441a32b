set -u
mkdir -p gpurun_out
CMD="python tools/mesh_large_probe.py"
timeout 600 $CMD > gpurun_out/pt_plain.log 2>&1
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 1200 ncu --metrics $M --clock-control none --csv -k regex:'wf_|mesh_|meta_update|tex_ilv' --log-file gpurun_out/pt_launches.csv $CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wf_tail -s 2 -c 1 -o gpurun_out/pt_tail -f $CMD > gpurun_out/pt_ncu.log 2>&1
echo done
