#!/bin/bash
D=gpurun_out/ms; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
FPS_DEBUG=1 MODES=1 WL=c4 timeout 300 python tools/mma_time.py 2>&1 | grep "mma scan" | tail -2 >> $D/time.log
cat $D/time.log
