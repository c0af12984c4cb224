#!/bin/bash
# Round evidence: tests, benches for every workload, reference arm, launch list + ncu captures.
mkdir -p gpurun_out/ev; rm -f gpurun_out/ev/*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev/build.log 2>&1 || exit 1
nvidia-smi > gpurun_out/ev/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/ev/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/ev/summary.txt
tail -2 gpurun_out/ev/gpu_tests.log >> gpurun_out/ev/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev/summary.txt
for w in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w > gpurun_out/ev/bench_$w.json 2> gpurun_out/ev/bench_$w.err; echo "bench $w rc=$?" >> gpurun_out/ev/summary.txt
done
timeout 900 python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.err; echo "bench default rc=$?" >> gpurun_out/ev/summary.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err; echo "ref rc=$?" >> gpurun_out/ev/summary.txt
CMD="python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c2.csv $CMD > /dev/null 2>&1
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"scan_kernel|select_kernel" -s 6 -c 2 -o gpurun_out/ev/prof_c2 $CMD > gpurun_out/ev/ncu_c2.log 2>&1; echo "ncu c2 rc=$?" >> gpurun_out/ev/summary.txt
CMD3="python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"scan_kernel" -s 2 -c 1 -o gpurun_out/ev/prof_c3 $CMD3 > gpurun_out/ev/ncu_c3.log 2>&1; echo "ncu c3 rc=$?" >> gpurun_out/ev/summary.txt
CMD4="python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"scan_kernel" -s 1 -c 1 -o gpurun_out/ev/prof_c4 $CMD4 > gpurun_out/ev/ncu_c4.log 2>&1; echo "ncu c4 rc=$?" >> gpurun_out/ev/summary.txt
cat gpurun_out/ev/summary.txt
