// Issue cost of the tensor-core scan's MMA lane, piece by piece (B200, sm_100a):
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_lane tools/microbench/mma_lane.cu && ./mma_lane
//
// One CTA per SM; lane 0 of warp 0 runs the per-tile loop of the MMA issuer
// (fps_mma4x.cuh) with each ingredient switched on separately: mbarrier
// try_wait on an already-completed phase, tcgen05.commit to an mbarrier, 3 x
// kind::mxf4 (M = 128, K = 64) at N = 64 / 208 into alternating TMEM
// accumulators. Operands are uninitialised shared memory (timing only).
// Prints clocks per loop iteration (max over CTAs).
#include <cstdint>
#include <cstdio>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

enum : unsigned { WAITS = 1, COMMITS = 2, MMAS = 4, TEST_WAIT = 8, ONE_COMMIT = 16, ONE_WAIT = 32, WIDE = 64, WARP = 128 };

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
__device__ __forceinline__ void test_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n T: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra T;\n}\n" ::"r"(bar),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// whole-warp variants: every lane runs the loop, one elected lane issues
__device__ __forceinline__ void commit_el(uint32_t bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void mma_el(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t sfa,
                                       uint32_t sfb) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t sfa,
                                    uint32_t sfb) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

__global__ void __launch_bounds__(128, 1) k_lane(int iters, unsigned opt, unsigned long long* clk) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t done_bar[2], sink_bar[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done_bar[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sink_bar[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // complete phase 0 of the done barriers: try_wait(parity 0) then succeeds at once
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&done_bar[i])) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0 || ((opt & WARP) && warp == 0)) {
    const bool W = opt & WARP;
    const int N = (opt & WIDE) ? 208 : 64;
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = desc(su32(sm), 128 / 8 * 128, 128), db = desc(su32(sm + 12288), N / 8 * 128, 128);
    const uint32_t sfa = tmem + 480, sfb = tmem + 496;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int b = it & 1;
      if (opt & WAITS) {
        if (opt & TEST_WAIT) {
          test_wait(su32(&done_bar[0]), 0);
          if (!(opt & ONE_WAIT)) test_wait(su32(&done_bar[1]), 0);
        } else {
          wait(su32(&done_bar[0]), 0);
          if (!(opt & ONE_WAIT)) wait(su32(&done_bar[1]), 0);
        }
      }
      if (opt & MMAS) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int ks = 0; ks < 3; ++ks) if (W) mma_el(tmem + (uint32_t)b * N, da + ks * 16, db + ks * (2 * (N / 8 * 128) / 16), idesc, ks > 0, sfa, sfb); else mma(tmem + (uint32_t)b * N, da + ks * 16, db + ks * (2 * (N / 8 * 128) / 16), idesc, ks > 0, sfa, sfb);
      }
      if (opt & COMMITS) {
        if (W) commit_el(su32(&sink_bar[0])); else commit(su32(&sink_bar[0]));
        if (!(opt & ONE_COMMIT)) { if (W) commit_el(su32(&sink_bar[1])); else commit(su32(&sink_bar[1])); }
      }
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = (t1 - t0) / (unsigned long long)iters;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  // drain the MMAs before freeing TMEM
  if (threadIdx.x == 0 && (opt & MMAS)) {
    commit(su32(&done_bar[0]));
    wait(su32(&done_bar[0]), 1);
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Warp-uniform MMA role (the CUTLASS pattern): the role is chosen on a warp
// index the compiler can prove uniform (__shfl_sync), the whole warp runs the
// loop, one elected lane issues each tcgen05 instruction.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}\n" : "=r"(pred));
  return pred != 0;
}
__global__ void __launch_bounds__(128, 1) k_uni(int iters, unsigned opt, unsigned long long* clk) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t done_bar[2], sink_bar[2];
  __shared__ uint32_t tmem_base;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done_bar[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sink_bar[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&done_bar[i])) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_base, 0);
  if (warp == 0) {
    const int N = (opt & WIDE) ? 208 : 64;
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = desc(su32(sm), 128 / 8 * 128, 128), db = desc(su32(sm + 12288), N / 8 * 128, 128);
    const uint32_t sfa = tmem + 480, sfb = tmem + 496;
    const uint32_t bar0 = su32(&done_bar[0]), bar1 = su32(&done_bar[1]), sk0 = su32(&sink_bar[0]), sk1 = su32(&sink_bar[1]);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int b = it & 1;
      if (opt & WAITS) {
        wait(bar0, 0);
        if (!(opt & ONE_WAIT)) wait(bar1, 0);
      }
      if (opt & MMAS) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (elect_one())
          for (int ks = 0; ks < 3; ++ks) mma(tmem + (uint32_t)b * N, da + ks * 16, db + ks * (2 * (N / 8 * 128) / 16), idesc, ks > 0, sfa, sfb);
        __syncwarp();
      }
      if (opt & COMMITS) {
        if (elect_one()) {
          commit(sk0);
          if (!(opt & ONE_COMMIT)) commit(sk1);
        }
        __syncwarp();
      }
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = (t1 - t0) / (unsigned long long)iters;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && (opt & MMAS)) {
    commit(su32(&done_bar[0]));
    wait(su32(&done_bar[0]), 1);
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  const int ctas = 148, iters = 20000;
  unsigned long long* d;
  CK(cudaMalloc(&d, ctas * 8));
  const int smem = 12288 + 208 * 96;
  CK(cudaFuncSetAttribute(k_lane, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_uni, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const unsigned UNI = 1u << 16;
  struct V { unsigned opt; const char* what; } vs[] = {
      {UNI, "uniform: empty loop"},
      {UNI | WAITS, "uniform: 2 try_wait"},
      {UNI | COMMITS, "uniform: 2 commits"},
      {UNI | MMAS, "uniform: 3 mxf4 N=64"},
      {UNI | MMAS | COMMITS, "uniform: 3 mxf4 N=64 + 2 commits"},
      {UNI | MMAS | COMMITS | WAITS, "uniform: 3 mxf4 N=64 + 2 commits + 2 try_wait"},
      {UNI | MMAS | WIDE, "uniform: 3 mxf4 N=208"},
      {UNI | MMAS | COMMITS | WAITS | WIDE, "uniform: 3 mxf4 N=208 + 2 commits + 2 try_wait"},
      {0, "empty loop"},
      {WAITS, "2 try_wait (phase already complete)"},
      {WAITS | ONE_WAIT, "1 try_wait"},
      {WAITS | TEST_WAIT, "2 test_wait"},
      {COMMITS, "2 commits (no MMA)"},
      {COMMITS | ONE_COMMIT, "1 commit"},
      {WAITS | COMMITS, "2 try_wait + 2 commits"},
      {MMAS, "3 mxf4 N=64 (no commit)"},
      {MMAS | COMMITS, "3 mxf4 N=64 + 2 commits"},
      {MMAS | COMMITS | ONE_COMMIT, "3 mxf4 N=64 + 1 commit"},
      {MMAS | COMMITS | WAITS, "3 mxf4 N=64 + 2 commits + 2 try_wait"},
      {MMAS | COMMITS | WAITS | ONE_WAIT | ONE_COMMIT, "3 mxf4 N=64 + 1 commit + 1 try_wait"},
      {MMAS | WIDE, "3 mxf4 N=208 (no commit)"},
      {MMAS | COMMITS | WAITS | WIDE, "3 mxf4 N=208 + 2 commits + 2 try_wait"},
      {WARP, "warp: empty loop"},
      {WARP | WAITS, "warp: 2 try_wait"},
      {WARP | COMMITS, "warp: 2 commits"},
      {WARP | MMAS, "warp: 3 mxf4 N=64"},
      {WARP | MMAS | COMMITS | WAITS, "warp: 3 mxf4 N=64 + 2 commits + 2 try_wait"},
      {WARP | MMAS | WIDE, "warp: 3 mxf4 N=208"},
      {WARP | MMAS | COMMITS | WAITS | WIDE, "warp: 3 mxf4 N=208 + 2 commits + 2 try_wait"},
  };
  for (const V& v : vs) {
    if (v.opt & UNI) k_uni<<<ctas, 128, smem>>>(iters, v.opt & ~UNI, d);
    else k_lane<<<ctas, 128, smem>>>(iters, v.opt, d);
    CK(cudaDeviceSynchronize());
    unsigned long long h[ctas], mx = 0;
    CK(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));
    for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-44s %6llu clk per iteration\n", v.what, mx);
  }
  return 0;
}
