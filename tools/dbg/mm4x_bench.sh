# tensor-core scan variants: parity subset + C4/C5 timings
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out; rm -f gpurun_out/mm4x_bench.log
run() { wl=$1; shift; envs=(); args=(); for x in "$@"; do case "$x" in *=*) envs+=("$x");; *) args+=("$x");; esac; done; echo "== $wl $*" >> gpurun_out/mm4x_bench.log; env "${envs[@]}" timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline "${args[@]}" 2>gpurun_out/mm4x_err.log | python tools/dbg/summ.py >> gpurun_out/mm4x_bench.log 2>&1 || tail -5 gpurun_out/mm4x_err.log >> gpurun_out/mm4x_bench.log; }
timeout 900 python -m pytest tests -q -m gpu -x -k "${TESTK:-mma or tensor or config4 or config5 or batch_min or smoke}" > gpurun_out/mm4x_tests.log 2>&1; echo rc=$? >> gpurun_out/mm4x_tests.log
# variants: one per line of $VARIANTS_FILE ("<workload> VAR=value ...")
if [ -n "$VARIANTS_FILE" ]; then
  while read -r line; do [ -n "$line" ] && run $line; done < "$VARIANTS_FILE"
else
  for v in "c4 X=1" "c4 FPS_MMA_KIND=i8" "c5 FPS_MMA=1" "c5 X=1"; do run $v; done
fi
