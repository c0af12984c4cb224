cd "$(dirname "$0")/../.."
for f in ${FLAGS:-0 4096 32768 36864}; do
  echo "== flags $f" >> gpurun_out/fp4_flags.log
  FPS_SCAN_FLAGS=$f timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['scan_kernel_ms'])" >> gpurun_out/fp4_flags.log 2>&1
done
