// tcgen05.ld (TMEM -> registers) throughput on B200 (sm_100a).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tools/microbench/tmem_ld.cu && ./tmem_ld
//
// The tensor-core fingerprint scan's epilogue reads one accumulator per
// (entry, query) pair. This measures how fast TMEM can be read back, per SM,
// for the load shapes the epilogue can use: 32x32b.x16 / .x32 / .x64, with
// and without .pack::16b (two 16-bit columns per register), W warps per CTA
// (a warp may only touch its lane quadrant: warp % 4), one CTA per SM, and
// L loads in flight per tcgen05.wait::ld. Reports TMEM cells (32-bit) read
// per clock per SM and register bytes delivered per clock per SM.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X, bool PACK>
__device__ __forceinline__ void ld(uint32_t addr, uint32_t (&r)[X]);

#define R16(r) "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
               "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
#define S16 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}"
template <>
__device__ __forceinline__ void ld<16, false>(uint32_t a, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 " S16 ", [%16];" : R16(r) : "r"(a));
}
template <>
__device__ __forceinline__ void ld<16, true>(uint32_t a, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 " S16 ", [%16];" : R16(r) : "r"(a));
}
#define R32(r) R16(r), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), \
               "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),       \
               "=r"(r[30]), "=r"(r[31])
#define S32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
template <>
__device__ __forceinline__ void ld<32, false>(uint32_t a, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " S32 ", [%32];" : R32(r) : "r"(a));
}
template <>
__device__ __forceinline__ void ld<32, true>(uint32_t a, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 " S32 ", [%32];" : R32(r) : "r"(a));
}

// each warp: ITER rounds of L loads (X registers each) then one wait
template <int X, bool PACK, int L>
__global__ void __launch_bounds__(512, 1) k_ld(int iters, unsigned long long* clk, uint32_t* sink, uint32_t shift) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base + ((uint32_t)(32 * (warp % 4)) << 16);
  constexpr uint32_t COLS = PACK ? 2 * X : X;  // TMEM columns one load reads
  const uint32_t nw = blockDim.x / 32;
  // warps sharing a quadrant read different column ranges
  // shift = 0: a moving base; shift = 1 + b: fixed column base b (+ the warp's part)
  const uint32_t c0 = (warp / 4) * (shift ? 64u : 512 / (nw / 4 > 0 ? nw / 4 : 1)) + (shift ? shift - 1 : 0);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[L][X];
#pragma unroll
    for (int l = 0; l < L; ++l) ld<X, PACK>(tm + (shift ? c0 + l * COLS : (c0 + l * COLS + it * 8) & (512 - COLS)), r[l]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int l = 0; l < L; ++l)
#pragma unroll
      for (int i = 0; i < X; ++i) acc ^= r[l][i];
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

template <int X, bool PACK, int L>
void run(int warps, uint32_t shift = 0) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* clk;
  uint32_t* sink;
  CK(cudaMalloc(&clk, sms * 8));
  CK(cudaMalloc(&sink, 4096));
  const int iters = 4096;
  k_ld<X, PACK, L><<<sms, warps * 32>>>(64, clk, sink, shift);
  CK(cudaDeviceSynchronize());
  k_ld<X, PACK, L><<<sms, warps * 32>>>(iters, clk, sink, shift);
  CK(cudaDeviceSynchronize());
  unsigned long long h[1024];
  CK(cudaMemcpy(h, clk, sms * 8, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += (double)h[i];
  avg /= sms;
  const double cells = (double)warps * iters * L * 32 * (PACK ? 2 * X : X);  // 32-bit TMEM cells per CTA
  const double regb = (double)warps * iters * L * 32 * X * 4;                 // register bytes per CTA
  printf("base=%3d 32x32b.x%-2d %-9s warps=%2d loads/wait=%d: %7.1f clk/round  cells %6.1f B/clk/SM  regs %6.1f B/clk/SM\n",
         (int)shift - 1, X, PACK ? "pack::16b" : "", warps, L, avg / iters, cells * 4 / avg, regb / avg);
  CK(cudaFree(clk));
  CK(cudaFree(sink));
}

int main(int argc, char** argv) {
  if (argc > 1) {  // column alignment: fixed column bases 0 / 8 / 16 / 24 / 56 / 104 (+ warp part)
    for (uint32_t sh : {0u, 8u, 16u, 24u, 56u, 104u}) {
      run<32, false, 1>(8, sh + 1);
      run<32, false, 1>(16, sh + 1);
      run<16, false, 1>(16, sh + 1);
    }
    return 0;
  }
  for (int w : {4, 8, 16}) {
    run<16, false, 1>(w);
    run<16, true, 1>(w);
    run<32, false, 1>(w);
    run<32, true, 1>(w);
    run<16, false, 2>(w);
    run<16, true, 2>(w);
    run<32, true, 2>(w);
  }
  return 0;
}
