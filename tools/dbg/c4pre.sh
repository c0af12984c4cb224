#!/bin/bash
# C4 call overhead: seed (POPC) and prefix (tensor-core) pass lengths
mkdir -p gpurun_out; rm -f gpurun_out/c4pre.txt
python -c "import __graft_entry__ as g; g.build()" || exit 1
while read -r line; do
  [ -z "$line" ] && continue
  env $line timeout 300 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_c4.json 2>gpurun_out/q_c4.err
  python -c "
import json; d=json.loads(open('gpurun_out/q_c4.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$line | c4 ms/step=%.4f scan_ms=%.4f e2e_ms=%.4f best=%s'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step'], d.get('check')))" >> gpurun_out/c4pre.txt 2>&1 || tail -3 gpurun_out/q_c4.err >> gpurun_out/c4pre.txt
done < ${VARIANTS:-tools/dbg/variants_c4pre.txt}
cat gpurun_out/c4pre.txt
