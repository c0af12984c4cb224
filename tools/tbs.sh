#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "query_counts or range or large_k or golden" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "config4 or config5" 2>&1 | tail -3
WORKLOADS="c4 c5" ./tools/quick_bench.sh
