#!/bin/bash
# Round evidence (tensor-core multi-query refresh): tests, smoke, benches, reference arm, launch lists, ncu captures.
D=gpurun_out/ev6; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
nvidia-smi > $D/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $D/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $D/summary.txt
tail -2 $D/gpu_tests.log >> $D/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/summary.txt
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo "bench default rc=$?" >> $D/summary.txt
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w > $D/bench_$w.json 2> $D/bench_$w.err; echo "bench $w rc=$?" >> $D/summary.txt
done
FPS_MMA=0 timeout 900 python bench.py --workload c4 --no-cpu-baseline > $D/bench_c4_bitslice.json 2> $D/bench_c4_bitslice.err
FPS_MMA=1 timeout 900 python bench.py --workload c5 --no-cpu-baseline > $D/bench_c5_mma.json 2> $D/bench_c5_mma.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $D/bench_reference.json 2> $D/bench_reference.err; echo "ref rc=$?" >> $D/summary.txt
for w in c2 c4; do
  CMD="python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_$w.csv $CMD > /dev/null 2>&1; echo "launches $w rc=$?" >> $D/summary.txt
done
C="python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline"
$C > /dev/null 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"mma_scan_kernel" -s 1 -c 1 -o $D/prof_c4_mma $C > $D/ncu_c4.log 2>&1; echo "ncu c4 rc=$?" >> $D/summary.txt
cat $D/summary.txt
