#!/bin/bash
# timelines of the seed phase variants (trace build)
mkdir -p gpurun_out
nvcc -DFPS_SCAN_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -ldl -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp 2>/dev/null || exit 1
while read -r line; do
  echo "=== $line"
  env $line python tools/scan_trace.py ${WLS:-c2} 2>&1 | grep -v "run 0" | sed -n '/run 1/,/run 2/p'
done < ${VARIANTS:-tools/dbg/variants_seed.txt} > gpurun_out/seed_trace.txt 2>&1
cat gpurun_out/seed_trace.txt
