#!/bin/bash
# single-query scan: load width (E) x trip depth (U) x pipelining x CTAs/SM
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$CFG $*', 'ms/step=%.4f scan_ms=%.4f e2e=%.4f best=%s'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step'], d.get('check')))"; }
for cfg in "4 1 1 2" "2 1 1 2" "2 2 1 2" "2 4 0 2" "2 2 0 3" "2 2 1 3" "2 1 1 3"; do
  set -- $cfg
  nvcc -DFPS_QW1_E=$1 -DFPS_QW1_U=$2 -DFPS_QW1_PIPE=$3 -DFPS_QW1_MINB=$4 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  CFG="E=$1,U=$2,pipe=$3,minb=$4" run --workload c2
  CFG="E=$1,U=$2,pipe=$3,minb=$4" run --workload c3
  CFG="E=$1,U=$2,pipe=$3,minb=$4" run --workload c1
done
