#!/bin/bash
# Run ON THE GPU BOX: mesh parity tests, then the A/B of the per-vertex
# field layout (planes at every depth vs records from depth d).
set -u
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "mesh or smoke or f1" ) > gpurun_out/vfrec_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/vfrec_pytest.log
: > gpurun_out/vfrec_ab.jsonl
for d in 1 0; do
  timeout 600 python tools/mesh_ab_options.py mesh_vf_records -1 $d >> gpurun_out/vfrec_ab.jsonl 2>> gpurun_out/vfrec_ab.err
done
timeout 600 python tools/mesh_ab_options.py mesh_vf_records -1 0 --c3 >> gpurun_out/vfrec_ab.jsonl 2>> gpurun_out/vfrec_ab.err
timeout 600 python tools/mesh_ab_options.py mesh_vf_records -1 1 --c3 >> gpurun_out/vfrec_ab.jsonl 2>> gpurun_out/vfrec_ab.err
echo done
