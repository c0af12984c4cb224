#!/bin/bash
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$CFG $*', 'ms/step=%.4f scan_ms=%.4f e2e=%.4f best=%s'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step'], d.get('check')))"; }
for cfg in "1 2 1" "0 4 1" "0 5 1" "0 6 1" "0 4 2" "0 3 2"; do
  set -- $cfg
  nvcc -DFPS_QW1_PIPE=$1 -DFPS_QW1_MINB=$2 -DFPS_QW1_U=$3 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  CFG="pipe=$1,minb=$2,U=$3" run --workload c2
  CFG="pipe=$1,minb=$2,U=$3" run --workload c3
  CFG="pipe=$1,minb=$2,U=$3" run --workload c1
done
