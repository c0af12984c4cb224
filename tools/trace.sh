#!/bin/bash
mkdir -p gpurun_out
nvcc -DFPS_SCAN_TRACE ${NVFLAGS} -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || exit 1
python tools/scan_trace.py ${WLS:-c2 c3}
