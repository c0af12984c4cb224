#!/bin/bash
# bit-slice kernel: queries per warp x min CTAs per SM (register cap)
mkdir -p gpurun_out
IFS=";" read -ra CL <<< "${CFGS:-4 1;2 3;2 2;4 3}"
for cfg in "${CL[@]}"; do
  set -- $cfg
  nvcc -DFPS_BS_QPW=$1 -DFPS_BS_MINB=$2 -DFPS_BS_DUAL=${3:-1} -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  for w in ${WLS:-c4 c5}; do
    timeout 600 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('qpw=$1 minb=$2 dual=${3:-1} $w ms/step=%.3f value=%.3e %s frac=%.3f check=%s'%(d['ms_per_step'], d['value'], r['bound'], r['frac'], d.get('check')))"
  done
done
