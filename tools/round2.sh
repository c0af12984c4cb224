#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/quick.txt
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
WORKLOADS="c1 c2 c3 c4 c5" ./tools/quick_bench.sh
python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_c2b python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
echo ncu rc=$?
