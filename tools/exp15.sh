#!/bin/bash
# select warm-up pass on/off: trace + bench
for wv in 1 0; do
  NVFLAGS="-DFPS_SEL_WARM=$wv" WLS="c1 c2" ./tools/trace.sh 2>&1 | grep -E "run 2|select" | tail -4 | sed "s/^/warm=$wv /"
  nvcc -DFPS_SEL_WARM=$wv -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -cudart static -Xcompiler -pthread -o paper_1906_06170_b200/libfpsgpu.so paper_1906_06170_b200/csrc/fps_capi.cu paper_1906_06170_b200/csrc/fps_ingest.cpp
  for w in c1 c2; do timeout 300 python bench.py --workload $w --steps 50 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('warm=$wv $w ms/step=%.4f e2e_ms=%.4f'%(d['ms_per_step'], d['e2e']['ms_per_step']))"; done
  CMD="python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w$wv.csv $CMD > /dev/null 2>&1
  grep select_kernel gpurun_out/launches_w$wv.csv | tail -3 | awk -F'","' '{print "warm='$wv' ncu select ns", $NF}'
done
