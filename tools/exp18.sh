#!/bin/bash
# bit-slice: 2 blocks per lane; warps per CTA x min CTAs
IFS=";" read -ra CL <<< "${CFGS:-8 1;16 1}"
for cfg in "${CL[@]}"; do
  set -- $cfg
  nvcc -DFPS_BS_WARPS=$1 -DFPS_BS_MINB=$2 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1 | sed "s/^/warps=$1 minb=$2 tests: /"
  for w in c4 c5; do
    timeout 600 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('warps=$1 minb=$2 $w ms/step=%.3f value=%.3e %s frac=%.3f'%(d['ms_per_step'], d['value'], r['bound'], r['frac']))"
  done
done
