#!/bin/bash
D=gpurun_out/mb; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -q -m gpu -x -k "mma or range or bitslice" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/time.log; tail -2 $D/tests.log >> $D/time.log
for n in 256 128 64; do
  echo "N cap $n" >> $D/time.log
  FPS_MMA_N=$n MODES=1 WL=c4 timeout 300 python tools/mma_time.py >> $D/time.log 2>&1
done
MODES=1 WL=c5 timeout 300 python tools/mma_time.py >> $D/time.log 2>&1
FPS_SCAN_FLAGS=4096 MODES=1 WL=c5 timeout 300 python tools/mma_time.py >> $D/time.log 2>&1
cat $D/time.log
