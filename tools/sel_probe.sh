#!/bin/bash
# select_kernel phase probe: build with FPS_SEL_PROBE, print phase cycles
nvcc -DFPS_SEL_PROBE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp || exit 1
python tools/sel_phases.py ${WLS:-c1 c2 c3} 2>&1 | grep phases
