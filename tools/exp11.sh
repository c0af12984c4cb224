#!/bin/bash
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('minb=$MINB $*', 'ms/step=%.4f scan_ms=%.4f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step']))"; }
for MINB in 2 3 4; do
  nvcc -DFPS_QW1_MINB=$MINB -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp
  MINB=$MINB run --workload c2 --radius 0
  MINB=$MINB run --workload c2
  MINB=$MINB run --workload c3
done
