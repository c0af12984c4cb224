cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/tmem_ld tools/microbench/tmem_ld.cu && timeout 120 gpurun_out/tmem_ld > gpurun_out/tmem_ld.txt 2>&1
CMD="python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mma_scan -s 2 -c 4 -o gpurun_out/prof_r02_c4 $CMD > gpurun_out/ncu_full_c4.log 2>&1
echo ncu rc=$?
