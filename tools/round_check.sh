#!/bin/bash
# Run ON THE GPU BOX: the driver's round-end checks (pytest -m gpu, smoke)
# followed by the round-2 evidence script (bench arms + ncu captures).
set -u
mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/rc_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/rc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rc_smoke.log 2>&1
bash tools/profile_r02.sh
