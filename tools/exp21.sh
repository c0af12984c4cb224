#!/bin/bash
# short scans: CTA-dynamic vs the global tail (min iterations per warp for the tail)
IFS=";" read -ra CL <<< "${CFGS:-128 50 12;0 50 12;0 70 12;0 50 24}"
for cfg in "${CL[@]}"; do
  set -- $cfg
  nvcc -DFPS_DYN_MIN_ITERS=$1 -DFPS_DYN_STATIC_PCT=$2 -DFPS_DYN_CHUNK_ITERS=$3 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  for rep in 1 2; do for w in c2 c1; do
    timeout 300 python bench.py --workload $w --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('min=$1 static=$2 chunk=$3 $w ms/step=%.4f scan_ms=%.4f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step']))"
  done; done
done
