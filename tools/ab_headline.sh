#!/bin/bash
# Interleaved A/B of the headline update kernel: in-tree library vs
# ab/<variant>/libmgcuda.so, bench.py --no-extras (2^28 fp32, 20 steps).
for i in 1 2 3; do
  for v in new $(ls ab 2>/dev/null); do
    if [ $v = new ]; then unset MG_LIB; else export MG_LIB=$PWD/ab/$v/libmgcuda.so; fi
    python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --e2e-steps 3 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4))"
  done
done
