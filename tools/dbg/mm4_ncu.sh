cd "$(dirname "$0")/../.."
timeout 300 python tools/dbg/mm4_run.py > gpurun_out/mm4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mma4_scan_kernel -s 2 -c 1 -o gpurun_out/mm4_prof -f python tools/dbg/mm4_run.py > gpurun_out/mm4_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/mm4_ncu.log
