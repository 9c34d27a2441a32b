#!/bin/bash
# A/B timing of the configs[2] helix iteration: in-tree library vs ab/<variant>/.
for i in 1 2; do
  for v in new $(ls ab 2>/dev/null); do
    if [ $v = new ]; then unset MG_LIB; else export MG_LIB=$PWD/ab/$v/libmgcuda.so; fi
    timeout 300 python tools/helix_probe.py 2>&1 | grep ms/it | sed "s/^/$v /"
  done
done
