#!/bin/bash
D=gpurun_out/mx; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests -q -m gpu -x -k "mma or range or bitslice" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/summary.txt
for f in ${FLAGS:-0 4096}; do
  echo "flags $f" >> $D/time.log
  MODES=1 FPS_SCAN_FLAGS=$f WL=c4 timeout 300 python tools/mma_time.py >> $D/time.log 2>&1
  MODES=1 FPS_SCAN_FLAGS=$f WL=c5 timeout 300 python tools/mma_time.py >> $D/time.log 2>&1
done
cat $D/time.log $D/summary.txt; tail -3 $D/tests.log
