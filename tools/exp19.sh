#!/bin/bash
# short scans: CTA-dynamic + global tail (percent static, chunk)
IFS=";" read -ra CL <<< "${CFGS:-0 2;80 2;90 2;80 4;70 1}"
for cfg in "${CL[@]}"; do
  set -- $cfg
  nvcc -DFPS_QW1_CTA_TAIL_PCT=$1 -DFPS_QW1_CTA_TAIL_CHUNK=$2 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  [ "$1" = "80" ] && [ "$2" = "2" ] && timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
  for rep in 1 2; do for w in c2 c1; do
    timeout 300 python bench.py --workload $w --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('tail=$1/$2 $w ms/step=%.4f scan_ms=%.4f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step']))"
  done; done
done
