#!/bin/bash
# One GPU session: build check, gpu tests, benches. Logs -> gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/gpu_tests.log >> gpurun_out/summary.txt
for w in ${WORKLOADS:-c2 c3 c4 c5 c1}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc=$?" >> gpurun_out/summary.txt
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; echo "ref rc=$?" >> gpurun_out/summary.txt
nproc >> gpurun_out/summary.txt; lscpu | grep "Model name" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
