// Dependent-chain latency of warp shuffles and of one bitonic compare-exchange
// stage (u64 keys), single warp. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void k(u64* out, u64 seed, int reps) {
  unsigned t = threadIdx.x;
  unsigned x = (unsigned)seed + t;
  u64 key = seed * (t + 1);
  __syncwarp();
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1 << (i & 3)) + 1;
  }
  long long c1 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (unsigned st = 16; st >= 1; st >>= 1) {
      u64 o = __shfl_xor_sync(0xffffffffu, key, st);
      bool lt = o < key;
      key = (lt == ((t & st) == 0)) ? o : key;
    }
  }
  long long c2 = clock64();
  if (t == 0) { out[0] = c1 - c0; out[1] = c2 - c1; }
  out[2 + t] = x + key;
}
int main() {
  u64* d; cudaMalloc(&d, 64 * 8);
  for (int it = 0; it < 3; ++it) {
    k<<<1, 32>>>(d, 12345, 64);
    u64 h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("shfl u32 dep-chain: %.1f cyc/op; bitonic u64 shuffle stage: %.1f cyc/stage\n", h[0] / (64.0 * 16), h[1] / (64.0 * 5));
  }
  return 0;
}
