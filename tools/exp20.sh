#!/bin/bash
# long scans: global tail share x chunk (compact tiles)
IFS=";" read -ra CL <<< "${CFGS:-50 8;50 4;50 16;30 8;70 8;0 8}"
for cfg in "${CL[@]}"; do
  set -- $cfg
  nvcc -DFPS_DYN_STATIC_PCT=$1 -DFPS_DYN_CHUNK_ITERS=$2 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  for rep in 1 2; do
    timeout 300 python bench.py --workload c3 --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('static=$1 chunk=$2 c3 ms/step=%.4f scan_ms=%.4f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step']))"
  done
done
