#!/bin/bash
# Tensor-core path: parity tests + C4/C5 benches (+ bit-sliced C5 for comparison)
D=gpurun_out/mq; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -q -m gpu -k "mma or range" -x > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/summary.txt
tail -2 $D/tests.log >> $D/summary.txt
for w in c4 c5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $D/bench_$w.json 2> $D/bench_$w.err; echo "bench $w rc=$?" >> $D/summary.txt
done
FPS_MMA=0 timeout 600 python bench.py --workload c5 --no-cpu-baseline > $D/bench_c5_bs.json 2> $D/bench_c5_bs.err
for w in c4 c5; do
C="python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mma_scan_kernel" -s 1 -c 1 -o $D/prof_${w}_mma $C > $D/ncu_$w.log 2>&1; echo "ncu $w rc=$?" >> $D/summary.txt
done
cat $D/summary.txt
