#!/bin/bash
D=gpurun_out/final; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu > $D/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $D/summary.txt
tail -2 $D/gpu_tests.log >> $D/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/summary.txt
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo "bench default rc=$?" >> $D/summary.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $D/bench_reference.json 2> $D/bench_reference.err; echo "ref rc=$?" >> $D/summary.txt
cat $D/summary.txt; tail -c 400 $D/bench_default.json
