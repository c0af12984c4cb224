mkdir -p gpurun_out/q3; rm -f gpurun_out/q3/*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q3/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/q3/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q3/summary.txt
tail -3 gpurun_out/q3/gpu_tests.log >> gpurun_out/q3/summary.txt
for w in c1 c2 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/q3/bench_$w.json 2> gpurun_out/q3/bench_$w.err; echo "bench $w rc=$?" >> gpurun_out/q3/summary.txt; done
FPS_PLANEQ=0 timeout 600 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/q3/bench_c1_popc.json 2> gpurun_out/q3/bench_c1_popc.err
FPS_PLANEQ=0 timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/q3/bench_c2_popc.json 2> gpurun_out/q3/bench_c2_popc.err
cat gpurun_out/q3/summary.txt
