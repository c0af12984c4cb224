#!/bin/bash
D=gpurun_out/ms; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -q -m gpu -x -k "mma or range or bitslice" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/time.log; tail -2 $D/tests.log >> $D/time.log
for pf in 22 21 23 0; do
  echo "prefix $pf" >> $D/time.log
  FPS_MMA_PREFIX=$pf MODES=1 WL=c4 timeout 300 python tools/mma_time.py >> $D/time.log 2>&1
  FPS_DEBUG=1 FPS_MMA_PREFIX=$pf MODES=1 WL=c4 timeout 300 python tools/mma_time.py 2>&1 | grep "mma scan" | tail -2 >> $D/time.log
done
cat $D/time.log
