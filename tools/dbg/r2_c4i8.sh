# full GPU suite + C4 bench (default int8) + ncu launch list and --set full of the int8 full pass
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
CMD="python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_c4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mma_scan -s 3 -c 1 -o gpurun_out/prof_c4i8 $CMD > gpurun_out/ncu_c4i8.log 2>&1
echo "ncu rc=$?"
