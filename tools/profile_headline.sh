#!/bin/bash
# Run ON THE GPU BOX (under gpurun): the headline bench command plain, then
# its ncu launch list, then one `--set full` capture of the fused update;
# text summaries land in gpurun_out/ (the .ncu-rep stays in /tmp).
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
timeout 600 $CMD > gpurun_out/hl_plain.jsonl 2> gpurun_out/hl_plain.err || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/hl_launches.csv $CMD > gpurun_out/hl_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:meta_update_tma \
  -s 4 -c 1 -o /tmp/hl_update -f $CMD > gpurun_out/hl_ncu_update.log 2>&1
ncu -i /tmp/hl_update.ncu-rep --page details > gpurun_out/hl_update_details.txt 2>&1
ncu -i /tmp/hl_update.ncu-rep --page raw --csv --metrics \
  dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread \
  > gpurun_out/hl_update_raw.csv 2>&1
echo done
