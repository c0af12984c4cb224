#!/bin/bash
# plane-scan seed phase: parity tests, then C1/C2/C3 with the seed off / on / delayed / waiting
mkdir -p gpurun_out; rm -f gpurun_out/seed.txt
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -x -q -m gpu -k "${KEXPR:-plane or pq or single or topk or fullsize}" > gpurun_out/seed_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/seed.txt
tail -3 gpurun_out/seed_tests.log >> gpurun_out/seed.txt
run() {
  for w in ${WORKLOADS:-c2 c1 c3}; do
    env "$@" timeout 300 python bench.py --workload $w --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > gpurun_out/q_$w.json 2>gpurun_out/q_$w.err
    python -c "
import json; d=json.loads(open('gpurun_out/q_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$* | $w ms/step=%.4f scan_ms=%.4f frac=%.3f e2e_ms=%.4f best=%s'%(d['ms_per_step'], r['scan_kernel_ms'], r['frac'], d['e2e']['ms_per_step'], d.get('check')))" >> gpurun_out/seed.txt 2>&1 || tail -3 gpurun_out/q_$w.err >> gpurun_out/seed.txt
  done
}
while read -r line; do [ -n "$line" ] && run $line; done < ${VARIANTS:-tools/dbg/variants_seed.txt}
cat gpurun_out/seed.txt
