#!/bin/bash
# Round-2 evidence, run ON THE GPU BOX: the driver's bench commands (our arm
# and the reference arm), the ncu launch list of the headline command, one
# `--set full` capture each of the headline fused update (meta_update_tma)
# and of the fast fused mini-render kernel, DRAM bytes per launch.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.jsonl 2> gpurun_out/r02_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.jsonl 2> gpurun_out/r02_bench_ref.err
CMD="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --e2e-steps 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:meta_update_tma \
  -s 5 -c 1 -o /tmp/r02_update -f $CMD > gpurun_out/r02_ncu_update.log 2>&1
ncu -i /tmp/r02_update.ncu-rep --page details > gpurun_out/r02_update_details.txt 2>&1
ncu -i /tmp/r02_update.ncu-rep --page raw --csv --metrics \
  dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread \
  > gpurun_out/r02_update_raw.csv 2>&1
RCMD="python tools/run_render.py --iters 5"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:minirender_fast \
  -s 3 -c 1 -o /tmp/r02_render -f $RCMD > gpurun_out/r02_ncu_render.log 2>&1
ncu -i /tmp/r02_render.ncu-rep --page details > gpurun_out/r02_render_details.txt 2>&1
ncu -i /tmp/r02_render.ncu-rep --page raw --csv --metrics \
  dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread \
  > gpurun_out/r02_render_raw.csv 2>&1
echo done
