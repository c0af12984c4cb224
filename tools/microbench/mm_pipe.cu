// Per-tile pipeline cost of the fp4 tensor-core scan's structure, feature by
// feature (B200, sm_100a):
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mm_pipe tools/microbench/mm_pipe.cu && ./mm_pipe
//
// One CTA per SM; an MMA lane issues 3 x kind::mxf4 (M = 128, N = 208,
// K = 64) per tile into one of two TMEM accumulators and commits to the
// accumulator's barrier; EPI epilogue warps wait for it, read their columns
// (tcgen05.ld), and release it. Options switch on, one at a time, what the
// product kernel (fps_mma4x.cuh) adds: a loader lane streaming 12 KB A tiles
// from global memory into a ring (MMA waits for the stage, commits its
// release), per-warp instead of per-thread releases, the epilogue's AND of
// the loaded registers. Prints clocks per tile (max over CTAs).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

constexpr int M = 128, N = 208, KB = 96, TILE = M * KB, STAGES = 12;
enum : unsigned { LOADER = 1, WARP_ARRIVE = 2, TESTS = 4, NO_LDTM = 8, RANDOM_B = 16, SHARED5 = 32, NO_MMA = 64 };

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | (uint64_t)((lbo >> 4) & 0x3fff) << 16 |
         (uint64_t)((sbo >> 4) & 0x3fff) << 32 | (uint64_t)1 << 46;
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(bar),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t sfa,
                                    uint32_t sfb) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

template <int W>
__device__ __forceinline__ void ld_cols(uint32_t ta, uint32_t* r) {
  if constexpr (W >= 32) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta));
    ld_cols<W - 32>(ta + 32, r + 32);
  } else if constexpr (W >= 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta));
    ld_cols<W - 8>(ta + 8, r + 8);
  }
}

// EPI epilogue warps (warps 0 .. EPI-1), MMA lane (warp EPI), loader lane (warp EPI+1)
template <int EPI>
__global__ void __launch_bounds__((EPI + 2) * 32, 1)
    k_pipe(int tiles, unsigned opt, const uint8_t* __restrict__ gA, unsigned long long* clk, uint32_t* sink) {
  constexpr int W = N / (EPI / 4);  // columns per epilogue warp (208 / 2 = 104 or 208 / 4 = 52 -> 48/56)
  constexpr int WL = W / 8 * 8;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sb = sm;
  uint8_t* sa = sm + N * KB;  // [STAGES][TILE]
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (N * KB + STAGES * TILE) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = (opt & RANDOM_B) ? (uint32_t)i * 2654435761u : 0u;
  if (warp == EPI) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&tfull[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&tempty[b])),
                   "r"((opt & WARP_ARRIVE) ? EPI : EPI * 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  if (warp < 4) {
    for (uint32_t c = 480; c < 512; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tm + ((uint32_t)(32 * warp) << 16) + c),
                   "r"(0x7f7f7f7fu));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned long long t0 = clock64();
  if (warp == EPI + 1) {
    if (lane == 0 && (opt & LOADER)) {
      const uint8_t* src = gA + (size_t)((opt & SHARED5) ? blockIdx.x / 5 : blockIdx.x) * tiles * TILE;
      for (int t = 0; t < tiles; ++t) {
        const int s = t % STAGES;
        if (t >= STAGES) wait(su32(&empty[s]), (uint32_t)((t / STAGES) - 1) & 1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(TILE)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(sa + s * TILE)),
                     "l"(src + (size_t)t * TILE), "r"(TILE), "r"(su32(&full[s]))
                     : "memory");
      }
    }
  } else if (warp == EPI) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
      const uint64_t db0 = desc(su32(sb), N / 8 * 128, 128), da0 = desc(su32(sa), M / 8 * 128, 128);
      constexpr uint64_t DA = 2 * (M / 8 * 128) / 16, DB = 2 * (N / 8 * 128) / 16, DS = TILE / 16;
      for (int t = 0; t < tiles; ++t) {
        const int b = t & 1, s = t % STAGES;
        if (t >= 2) wait(su32(&tempty[b]), (uint32_t)((t >> 1) - 1) & 1u);
        if (opt & LOADER) wait(su32(&full[s]), (uint32_t)(t / STAGES) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t das = da0 + ((opt & LOADER) ? (uint64_t)s * DS : 0);
        if (!(opt & NO_MMA)) {
#pragma unroll
          for (int ks = 0; ks < 3; ++ks) mma(tm + b * N, das + ks * DA, db0 + ks * DB, idesc, ks > 0, tm + 480, tm + 496);
        }
        if (opt & LOADER) commit(su32(&empty[s]));
        commit(su32(&tfull[b]));
      }
    }
  } else {
    const int quad = warp % 4, part = warp / 4;
    const uint32_t ta = tm + ((uint32_t)(32 * quad) << 16) + (uint32_t)(part * WL);
    uint32_t acc = 0;
    for (int t = 0; t < tiles; ++t) {
      const int b = t & 1;
      wait(su32(&tfull[b]), (uint32_t)(t >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[WL];
      if (!(opt & NO_LDTM)) ld_cols<WL>(ta + b * N, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (opt & WARP_ARRIVE) {
        __syncwarp();
        if (lane == 0) arrive(su32(&tempty[b]));
      } else {
        arrive(su32(&tempty[b]));
      }
      if ((opt & TESTS) && !(opt & NO_LDTM)) {
        uint32_t x = r[0];
#pragma unroll
        for (int i = 1; i < WL; ++i) x &= r[i];
        acc |= __any_sync(0xffffffffu, (int)x >= 0) ? 1u : 0u;
      }
    }
    if (acc == 0x12345u) sink[0] = acc;
  }
  __syncwarp();
  const unsigned long long t1 = clock64();
  if (warp == EPI && lane == 0) clk[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == EPI) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int EPI>
void run(int ctas, unsigned opt, const uint8_t* gA, int tiles, const char* what) {
  const int smem = N * KB + STAGES * TILE;
  CK(cudaFuncSetAttribute(k_pipe<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* dclk;
  uint32_t* sink;
  CK(cudaMalloc(&dclk, ctas * 8));
  CK(cudaMalloc(&sink, 64));
  k_pipe<EPI><<<ctas, (EPI + 2) * 32, smem>>>(64, opt, gA, dclk, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pipe<EPI><<<ctas, (EPI + 2) * 32, smem>>>(tiles, opt, gA, dclk, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> c(ctas);
  CK(cudaMemcpy(c.data(), dclk, ctas * 8, cudaMemcpyDeviceToHost));
  unsigned long long mx = 0;
  for (auto v : c) mx = v > mx ? v : mx;
  printf("EPI=%2d ctas=%3d opt=%2u %-48s %7.1f clk/tile  (%.3f ms for %d tiles)\n", EPI, ctas, opt, what,
         (double)mx / tiles, ms, tiles);
  cudaFree(dclk);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int tiles = 4000;
  uint8_t* gA;
  CK(cudaMalloc(&gA, (size_t)sms * tiles * TILE));
  {
    std::vector<uint32_t> h((size_t)sms * tiles * TILE / 4);
    uint32_t x = 12345;
    for (auto& v : h) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; v = x; }
    CK(cudaMemcpy(gA, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  }
  struct V { unsigned opt; const char* what; } vs[] = {
      {WARP_ARRIVE | TESTS | LOADER | RANDOM_B | SHARED5, "full (loader shared by 5, tests)"},
      {WARP_ARRIVE | NO_LDTM | NO_MMA, "barriers only (no loader)"},
      {WARP_ARRIVE | NO_LDTM | NO_MMA | LOADER, "barriers only + loader ring"},
      {WARP_ARRIVE | NO_MMA | LOADER, "no MMA, LDTM, loader"},
      {WARP_ARRIVE | NO_LDTM | LOADER | RANDOM_B, "MMA + loader, no LDTM"},
  };
  for (const V& v : vs) run<8>(sms, v.opt, gA, tiles, v.what);
  return 0;
}
