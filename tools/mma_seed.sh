#!/bin/bash
D=gpurun_out/ms; mkdir -p $D; rm -f $D/*
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || exit 1
for cfg in "18 22" "18 21" "18 20" "16 20" "18 0" "20 0" "16 22"; do
  set -- $cfg
  echo "seed $1 prefix $2" >> $D/time.log
  FPS_MMA_SEED=$1 FPS_MMA_PREFIX=$2 MODES=1 WL=c4 timeout 300 python tools/mma_time.py >> $D/time.log 2>&1
done
timeout 600 python bench.py --workload c4 > $D/bench_c4.json 2> $D/bench_c4.err
cat $D/time.log; tail -c 600 $D/bench_c4.json
