# TMEM alignment microbench + ncu source capture of the fp4 operand-copy scan (EPI=${EPI:-8})
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/tmem_ld tools/microbench/tmem_ld.cu && timeout 120 gpurun_out/tmem_ld align > gpurun_out/tmem_align.txt 2>&1
CMD="python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline"
export FPS_MM4X_EPI=${EPI:-8} FPS_MM_SUSPEND_NS=0
$CMD > gpurun_out/plain_c4x.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mma4x -s 1 -c 1 -o gpurun_out/prof_c4x_e$FPS_MM4X_EPI $CMD > gpurun_out/ncu_c4x.log 2>&1
echo ncu rc=$?
