#!/bin/bash
# Run ON THE GPU BOX (under gpurun): plain bench run, then the ncu launch
# list of the same command, then one `--set full` capture of the fused
# update and of the fused mini-render kernel.  Outputs in gpurun_out/.
set -u
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:meta_update \
  -s 5 -c 1 -o gpurun_out/prof_update $CMD > gpurun_out/ncu_update.log 2>&1
RCMD="python tools/run_render.py --iters 4"
timeout 300 $RCMD > gpurun_out/render_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:minirender_meta \
  -s 2 -c 1 -o gpurun_out/prof_render $RCMD > gpurun_out/ncu_render.log 2>&1
echo done
