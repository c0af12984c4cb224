#!/bin/bash
D=gpurun_out/mn; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
C="python tools/mma_time.py"
MODES=1 WL=c4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mma_scan_kernel" -s 1 -c 1 -o $D/prof_c4 $C > $D/ncu_c4.log 2>&1; echo "ncu rc=$?" >> $D/summary.txt
cat $D/summary.txt
