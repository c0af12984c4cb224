#!/usr/bin/env bash
# End-of-round GPU pass: full GPU suite, smoke, default bench + reference arm,
# every workload's bench line, ncu launch list + --set full of the C4 scan.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref_c3.err
for w in c1 c2 c4 c5; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
CMD="python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_c4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mma4x_scan -s 3 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"
# plane scan captures (C3: the headline kernel; C2: the short, latency-bound scan)
for w in c3 c2; do
  CMD="python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline"
  $CMD > gpurun_out/plain_$w.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv $CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pq_scan -s 3 -c 1 -o gpurun_out/prof_$w $CMD > gpurun_out/ncu_$w.log 2>&1
  echo "ncu $w rc=$?"
done
