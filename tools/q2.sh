mkdir -p gpurun_out/q2; rm -f gpurun_out/q2/*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q2/build.log 2>&1
for w in c2 c3 c1; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/q2/bench_$w.json 2> gpurun_out/q2/bench_$w.err; echo "bench $w rc=$?" >> gpurun_out/q2/summary.txt; done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/q2/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q2/summary.txt
tail -3 gpurun_out/q2/gpu_tests.log >> gpurun_out/q2/summary.txt
cat gpurun_out/q2/summary.txt
