#!/usr/bin/env bash
# GPU-box measurement pass: quick bench of every workload, tensor-core variants,
# tcgen05 peak microbenchmark, ncu launch list + --set full capture (WL=c3).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/umma_peak tools/microbench/umma_peak.cu && timeout 120 gpurun_out/umma_peak > gpurun_out/umma_peak.txt 2>&1
WORKLOADS="c1 c2 c4 c5" bash tools/quick_bench.sh > /dev/null 2>&1
VARIANTS_FILE=tools/dbg/variants_c4.txt bash tools/dbg/mm4x_bench.sh
WL=${WL:-c3} TAG=${TAG:-r02} bash tools/prof.sh
