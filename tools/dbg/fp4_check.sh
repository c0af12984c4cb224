cd "$(dirname "$0")/../.."
timeout 600 python tools/dbg/overflow_probe.py > gpurun_out/fp4_probe.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "mma or tensor or config4 or config5 or group or batch_min" > gpurun_out/fp4_tests.log 2>&1; echo rc=$? >> gpurun_out/fp4_tests.log
for v in "FPS_MMA_KIND=fp4" "FPS_MMA_KIND=fp4 FPS_SCAN_FLAGS=4096" "FPS_MMA_KIND=i8"; do
  echo "== $v" >> gpurun_out/fp4_bench.log
  env $v timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['scan_kernel_ms'], r['frac'], r['kernel'])" >> gpurun_out/fp4_bench.log 2>&1
done
