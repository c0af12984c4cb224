cd "$(dirname "$0")/../.."
timeout 600 python tools/dbg/overflow_probe.py > gpurun_out/fp4_probe.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "mma or tensor or config4 or config5 or group or batch_min" > gpurun_out/fp4_tests.log 2>&1; echo rc=$? >> gpurun_out/fp4_tests.log
for kind in fp4 i8; do
  FPS_MMA_KIND=$kind timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fp4_bench_$kind.log 2>&1
done
