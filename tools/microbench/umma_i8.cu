// Bring-up of the tcgen05 int8 MMA path (D[tmem] = A[smem] . B[smem]^T) with
// the K-major no-swizzle canonical layout: one CTA, M = 128, N = 256, K = 192.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mb_umma umma_i8.cu && ./mb_umma
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int M = 128, N = 256, K = 192;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: byte (row, k) at (k / 16) * (rows / 8 * 128) + (row / 8) * 128 + (row % 8) * 16 + k % 16
__device__ __forceinline__ uint32_t canon(int row, int k, int rows) {
  return (k / 16) * (rows / 8 * 128) + (row / 8) * 128 + (row % 8) * 16 + (k % 16);
}

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void k_umma(const uint8_t* A, const uint8_t* B, int* C) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;
  uint8_t* sb = sm + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) sa[canon(i / K, i % K, M)] = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) sb[canon(i / K, i % K, N)] = B[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int s = 0; s < K / 32; ++s) {
      const uint64_t da = desc(su32(sa + s * 2 * (M / 8 * 128)), M / 8 * 128, 128);
      const uint64_t db = desc(su32(sb + s * 2 * (N / 8 * 128)), N / 8 * 128, 128);
      const uint32_t acc = s > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(tm),
          "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(su32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tm + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) C[(32 * warp + lane) * N + c0 + j] = (int)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  std::vector<uint8_t> A(M * K), B(N * K);
  srand(7);
  for (auto& x : A) x = rand() % 4 == 0;
  for (auto& x : B) x = rand() % 3 == 0;
  uint8_t *dA, *dB;
  int* dC;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dC, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0xff, M * N * 4));
  const int smem = (M + N) * K;
  CK(cudaFuncSetAttribute(k_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_umma<<<1, 128, smem>>>(dA, dB, dC);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int> C(M * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int ref = 0;
      for (int k = 0; k < K; ++k) ref += A[i * K + k] * B[j * K + k];
      if (ref != C[i * N + j]) {
        if (bad < 8) printf("mismatch (%d,%d): got %d ref %d\n", i, j, C[i * N + j], ref);
        ++bad;
      }
    }
  printf("umma i8: %d mismatches of %d\n", bad, M * N);
  return bad != 0;
}
