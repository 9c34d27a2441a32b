# per-kernel A/B of the configs[4] scatter/finalize stages (ncu durations + DRAM bytes)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum
for v in base new; do
  if [ $v = base ]; then export MG_LIB=$PWD/ab/libmgcuda.so; else unset MG_LIB; fi
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:'scatter|finalize' -s 4 -c 4 \
    --log-file gpurun_out/abn_$v.csv python tools/mesh_large_probe.py > gpurun_out/abn_$v.log 2>&1
done
