cd "$(dirname "$0")/../.."
run() { wl=$1; shift; echo "== $wl $*" >> gpurun_out/mma_bench.log; env "$@" timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['scan_kernel_ms'], r.get('frac'), r['kernel'], d['e2e']['ms_per_step'])" >> gpurun_out/mma_bench.log 2>&1; }
timeout 900 python -m pytest tests -q -m gpu -x -k "mma or tensor or config4 or config5 or group or batch_min" > gpurun_out/mma_tests.log 2>&1; echo rc=$? >> gpurun_out/mma_tests.log
run c4 X=1
run c4 FPS_MMA_KIND=fp4
run c5 X=1
run c5 FPS_MMA=1
run c5 FPS_MMA=1 FPS_MMA_KIND=fp4
