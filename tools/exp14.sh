#!/bin/bash
# single-query scan: bulk-copy ring depth (FPS_QW1_STAGES), TMA on/off
mkdir -p gpurun_out
run() { timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$CFG $*', 'ms/step=%.4f scan_ms=%.4f e2e=%.4f best=%s'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step'], d.get('check')))"; }
IFS=";" read -ra CL <<< "${CFGS:-1 4;1 2;1 3;1 6;0 4}"
for cfg in "${CL[@]}"; do
  set -- $cfg
  nvcc -DFPS_QW1_TMA=$1 -DFPS_QW1_STAGES=$2 -DFPS_QW1_DYN_PCT=${3:-85} -DFPS_QW1_DYN_CHUNK=${4:-2} -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || continue
  if [ "$cfg" = "${CL[0]}" ]; then timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2; fi
  for w in ${WLS:-c2 c3 c1}; do CFG="tma=$1,S=$2,dyn=${3:-85}/${4:-2}" run --workload $w; done
done
