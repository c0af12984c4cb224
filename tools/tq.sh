#!/bin/bash
# tests + quick benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log; grep -E "^E  |Error" gpurun_out/gpu_tests.log | head -5
WORKLOADS="${WORKLOADS:-c1 c2 c3}" ./tools/quick_bench.sh
