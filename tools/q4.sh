mkdir -p gpurun_out/q4; rm -f gpurun_out/q4/*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q4/build.log 2>&1
for w in c1 c2 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/q4/bench_$w.json 2> gpurun_out/q4/bench_$w.err; done
for w in c1 c2; do FPS_DEBUG=1 timeout 600 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/q4/dbg_$w.err; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "plane or tail or ties or adversarial" > gpurun_out/q4/tests.log 2>&1; tail -2 gpurun_out/q4/tests.log
