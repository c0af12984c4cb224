mkdir -p gpurun_out/q1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q1/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/q1/gpu_tests.log 2>&1; echo "tests rc=$?" > gpurun_out/q1/summary.txt
tail -3 gpurun_out/q1/gpu_tests.log >> gpurun_out/q1/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/q1/summary.txt
for w in c2 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/q1/bench_$w.json 2> gpurun_out/q1/bench_$w.err; echo "bench $w rc=$?" >> gpurun_out/q1/summary.txt; done
cat gpurun_out/q1/summary.txt
