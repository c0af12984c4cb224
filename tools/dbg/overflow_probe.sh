cd "$(dirname "$0")/../.."
for v in "FPS_GRAPHS=0 CUDA_LAUNCH_BLOCKING=1" "CUDA_LAUNCH_BLOCKING=1" "FPS_GRAPHS=0 FPS_DEBUG=1" "FPS_MMA=0" "Q=64 FPS_MMA=1 FPS_GRAPHS=0 CUDA_LAUNCH_BLOCKING=1"; do
  echo "== $v"; env $v timeout 120 python tools/dbg/overflow_probe.py 2>&1 | tail -8
done
