cd "$(dirname "$0")/../.."
for v in ${VARIANTS:-"FPS_MM_SUSPEND_NS=20000" "FPS_MM_SUSPEND_NS=0" "FPS_MM_SUSPEND_NS=200" "FPS_MM_SUSPEND_NS=0 FPS_SCAN_FLAGS=36864"}; do
  echo "== $v" >> gpurun_out/fp4_env.log
  env $v timeout 600 python bench.py --workload ${WL:-c4} --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['scan_kernel_ms'])" >> gpurun_out/fp4_env.log 2>&1
done
