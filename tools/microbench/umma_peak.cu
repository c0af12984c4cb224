// tcgen05 tensor-core peak + fp4 bring-up microbenchmark (B200, sm_100a).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_peak tools/microbench/umma_peak.cu && ./umma_peak
//
// 1. correctness of the block-scaled fp4 formulation of the fingerprint test
//    (kind::mxf4, e2m1 operands, all scale factors 1.0 = ue8m0 127): A = entry
//    bits as 1.0 plus the per-row digits of -|a|, B = 2.0 x query bits plus the
//    per-column digits of T - |q| + 0.5, so D = T - d + 0.5 exactly (f32);
//    checked against the CPU for random and extreme rows / columns;
// 2. peak issue rate: one CTA per SM issuing back-to-back MMAs from shared
//    memory into two alternating TMEM accumulators (operand contents do not
//    matter for the rate), kind::i8 (K = 32 per instruction) and kind::mxf4
//    (K = 64), M = 128, several N. Reports dense ops/s (2 per multiply-add)
//    against the nominal 4.5 (int8) / 9 (fp4) POP/s of a B200.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

constexpr int M = 128;
constexpr int KB = 96;  // bytes per row of a fp4 operand (192 elements)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ __forceinline__ uint32_t canon(uint32_t row, uint32_t kbyte, uint32_t rows) {
  return (kbyte / 16) * (rows / 8 * 128) + (row / 8) * 128 + (row % 8) * 16 + (kbyte % 16);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                   su32(bar)),
               "r"(parity)
               : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
// instruction descriptors
__host__ __device__ constexpr uint32_t idesc_i8(int n) {  // s32 += u8 x s8
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_mxf4(int n) {  // f32 += e2m1 x e2m1, ue8m0 scales, K = 64
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                         uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// fill TMEM columns [c0, c0 + ncols) of all 128 lanes with `v` (4 warps)
__device__ void tmem_fill(uint32_t tmem, uint32_t c0, uint32_t ncols, uint32_t v) {
  const int warp = threadIdx.x >> 5;
  if (warp >= 4) return;
  for (uint32_t c = c0; c < c0 + ncols; c += 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                     tmem + ((uint32_t)(32 * warp) << 16) + c),
                 "r"(v));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ------------------------------------------------------------------ 1. correctness
template <int N>
__global__ void k_check(const uint8_t* A, const uint8_t* B, float* C) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;
  uint8_t* sb = sm + M * KB;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * KB; i += blockDim.x) sa[canon(i / KB, i % KB, M)] = A[i];
  for (int i = tid; i < N * KB; i += blockDim.x) sb[canon(i / KB, i % KB, N)] = B[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
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
  // accumulator garbage first (so a scale factor read outside the filled
  // region would show), then scale factors 1.0 in columns 448..511
  tmem_fill(tm, 0, 448, 0x40404040u);
  tmem_fill(tm, 448, 64, 0x7f7f7f7fu);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t id = idesc_mxf4(N);
    for (int s = 0; s < 3; ++s) {  // K = 64 elements = 32 bytes = 2 core matrices per MMA
      const uint64_t da = desc(su32(sa + s * 2 * (M / 8 * 128)), M / 8 * 128, 128);
      const uint64_t db = desc(su32(sb + s * 2 * (N / 8 * 128)), N / 8 * 128, 128);
      mma_mxf4(tm, da, db, id, s > 0, tm + 480, tm + 496);
    }
    commit(&bar);
  }
  bar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tm + ((uint32_t)(32 * warp) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) C[(32 * warp + lane) * N + c0 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// e2m1 codes: value -> nibble (sign bit 3; exp 2 bits; mantissa 1 bit)
static int e2m1_code(double v) {
  static const double vals[8] = {0, 0.5, 1, 1.5, 2, 3, 4, 6};
  const int sg = v < 0 ? 8 : 0;
  const double a = v < 0 ? -v : v;
  for (int i = 0; i < 8; ++i)
    if (vals[i] == a) return i == 0 ? 0 : (sg | i);
  printf("not e2m1: %f\n", v);
  exit(1);
}
// greedy e2m1 digits of x (a multiple of 0.5) into `slots` codes
static void digits(double x, int slots, int* out) {
  static const double vals[7] = {6, 4, 3, 2, 1.5, 1, 0.5};
  const double sg = x < 0 ? -1 : 1;
  double a = x * sg;
  for (int i = 0; i < slots; ++i) {
    out[i] = 0;
    for (double v : vals)
      if (v <= a + 1e-9) { out[i] = e2m1_code(v * sg); a -= v; break; }
  }
  if (a > 1e-9) { printf("digits: %f left of %f\n", a, x); exit(1); }
}
static void put(std::vector<uint8_t>& m, int row, int k, int code) {  // element k: 2 per byte, low nibble first
  uint8_t& b = m[row * KB + k / 2];
  b = (k & 1) ? (uint8_t)((b & 0x0f) | (code << 4)) : (uint8_t)((b & 0xf0) | code);
}

// Test-term slots (elements 168..191 are zero bits in a compact library):
//   168..172  A = e2m1 digits of P = |a| / 6      B = -6
//   173..174  A = digits of R = |a| % 6           B = -1
//   175..182  A = 6                               B = digits of X = trunc(v / 6), v = T - |q| + 0.5
//   183..184  A = 1                               B = digits of Y = v - 6 X
// so D = 2c - |a| + v = T - d + 0.5 (never 0: pass iff the f32 sign bit is clear).
template <int N>
static int check() {
  std::vector<uint8_t> A(M * KB, 0), B(N * KB, 0);
  std::vector<int> abits(M * 192, 0), qbits(N * 192, 0), pa(M), T(N), pq(N);
  srand(1234 + N);
  for (int i = 0; i < M; ++i) {
    const int dens = i == 0 ? 0 : rand() % 100;
    for (int k = 0; k < 168; ++k) abits[i * 192 + k] = i == 1 ? 1 : (rand() % 100) < dens;
    pa[i] = 0;
    for (int k = 0; k < 192; ++k) pa[i] += abits[i * 192 + k];
    for (int k = 0; k < 168; ++k) put(A, i, k, abits[i * 192 + k] ? e2m1_code(1.0) : 0);
    int d[7];
    digits(pa[i] / 6, 5, d);
    digits(pa[i] % 6, 2, d + 5);
    for (int s = 0; s < 7; ++s) put(A, i, 168 + s, d[s]);
    for (int s = 175; s < 183; ++s) put(A, i, s, e2m1_code(6.0));
    for (int s = 183; s < 185; ++s) put(A, i, s, e2m1_code(1.0));
  }
  for (int j = 0; j < N; ++j) {
    const int dens = j == 0 ? 0 : rand() % 100;
    for (int k = 0; k < 166; ++k) qbits[j * 192 + k] = j == 1 ? 1 : (rand() % 100) < dens;
    pq[j] = 0;
    for (int k = 0; k < 192; ++k) pq[j] += qbits[j * 192 + k];
    T[j] = j == 2 ? 255 : j == 3 ? 0 : j == 4 ? 255 : rand() % 256;
    for (int k = 0; k < 168; ++k) put(B, j, k, qbits[j * 192 + k] ? e2m1_code(2.0) : 0);
    for (int s = 168; s < 173; ++s) put(B, j, s, e2m1_code(-6.0));
    for (int s = 173; s < 175; ++s) put(B, j, s, e2m1_code(-1.0));
    const double v = T[j] - pq[j] + 0.5;
    const int X = (int)(v / 6.0);  // trunc toward 0
    const double Y = v - 6.0 * X;
    int dx[8], dy[2];
    digits(X, 8, dx);
    digits(Y, 2, dy);
    for (int s = 0; s < 8; ++s) put(B, j, 175 + s, dx[s]);
    for (int s = 0; s < 2; ++s) put(B, j, 183 + s, dy[s]);
  }
  uint8_t *dA, *dB;
  float* dC;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dC, (size_t)M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const int smem = (M + N) * KB;
  CK(cudaFuncSetAttribute(k_check<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_check<N><<<1, 128, smem>>>(dA, dB, dC);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> C((size_t)M * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int c = 0;
      for (int k = 0; k < 192; ++k) c += abits[i * 192 + k] & qbits[j * 192 + k];
      const int d = pa[i] + pq[j] - 2 * c;
      const float ref = (float)(T[j] - d) + 0.5f;
      if (C[(size_t)i * N + j] != ref) {
        if (bad < 8) printf("  mismatch (%d,%d): got %f ref %f\n", i, j, C[(size_t)i * N + j], ref);
        ++bad;
      }
    }
  printf("mxf4 N=%d encoding check: %d mismatches of %d\n", N, bad, M * N);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  return bad;
}

// ------------------------------------------------------------------ 2. peak issue rate
// KIND 0: i8 (6 x K32 per 192-K tile), 1: mxf4 (3 x K64). Two accumulators, a
// commit per tile; the issuing thread waits for tile t-2 before reusing its
// accumulator (as a real kernel would for the epilogue).
template <int KIND, int N>
__global__ void __launch_bounds__(128, 1) k_peak(int tiles, unsigned long long* clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int ABYTES = KIND == 0 ? M * 192 : M * KB;
  uint8_t* sa = sm;
  uint8_t* sb = sm + ABYTES;
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (ABYTES + N * (KIND == 0 ? 192 : KB)) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x22222222u * (i & 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  if (KIND == 1) tmem_fill(tm, 480, 32, 0x7f7f7f7fu);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const unsigned long long t0 = clock64();
    const uint64_t da0 = desc(su32(sa), M / 8 * 128, 128);
    const uint64_t db0 = desc(su32(sb), N / 8 * 128, 128);
    constexpr uint64_t DA = 2 * (M / 8 * 128) / 16, DB = 2 * (N / 8 * 128) / 16;
    for (int t = 0; t < tiles; ++t) {
      const int b = t & 1;
      if (t >= 2) bar_wait(&bar[b], (uint32_t)((t >> 1) - 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tm + (uint32_t)b * N;
      if (KIND == 0) {
#pragma unroll
        for (int ks = 0; ks < 6; ++ks) mma_i8(dt, da0 + ks * DA, db0 + ks * DB, idesc_i8(N), ks > 0);
      } else {
#pragma unroll
        for (int ks = 0; ks < 3; ++ks)
          mma_mxf4(dt, da0 + ks * DA, db0 + ks * DB, idesc_mxf4(N), ks > 0, tm + 480, tm + 496);
      }
      commit(&bar[b]);
    }
    bar_wait(&bar[(tiles - 1) & 1], (uint32_t)(((tiles - 1) >> 1)) & 1u);
    clk[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int KIND, int N>
static void peak(int sms) {
  const int tiles = 20000;
  constexpr int ABYTES = KIND == 0 ? M * 192 : M * KB;
  const int smem = ABYTES + N * (KIND == 0 ? 192 : KB);
  CK(cudaFuncSetAttribute(k_peak<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* dclk;
  CK(cudaMalloc(&dclk, sms * 8));
  k_peak<KIND, N><<<sms, 128, smem>>>(100, dclk);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_peak<KIND, N><<<sms, 128, smem>>>(tiles, dclk);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> clk(sms);
  CK(cudaMemcpy(clk.data(), dclk, sms * 8, cudaMemcpyDeviceToHost));
  unsigned long long mx = 0;
  for (auto c : clk) mx = c > mx ? c : mx;
  const double ops = 2.0 * M * N * 192 * (double)tiles * sms;
  const double clk_per_tile = (double)mx / tiles;
  printf("%s N=%3d: %8.1f TOP/s dense (%.3f of nominal %.1f POP/s), %.1f clk per 128x%dx192 tile per SM\n",
         KIND == 0 ? "i8  " : "mxf4", N, ops / (ms / 1e3) / 1e12, ops / (ms / 1e3) / (KIND == 0 ? 4.5e15 : 9e15),
         KIND == 0 ? 4.5 : 9.0, clk_per_tile, N);
  cudaFree(dclk);
}


// ------------------------------------------------------------------ 3. pipeline round trip
// As k_peak, plus 16 epilogue warps that, per tile, wait for the accumulator
// (tcgen05.commit -> mbarrier), load their quarter of it from TMEM, and
// release it (mbarrier arrive) before the issuer may reuse it: the
// MMA -> epilogue -> MMA round trip with NACC accumulator buffers.
template <int N, int NACC>
__global__ void __launch_bounds__(32 * 18, 1) k_pipe(int tiles, unsigned long long* clk, int spin) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;
  uint8_t* sb = sm + M * KB;
  __shared__ uint64_t tfull[NACC], tempty[NACC];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (M * KB + N * KB) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int b = 0; b < NACC; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&tfull[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 512;" ::"r"(su32(&tempty[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  tmem_fill(tm, 480, 32, 0x7f7f7f7fu);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp >= 2) {  // 16 epilogue warps: quadrant warp % 4, quarter (warp - 2) / 4
    const int ew = warp - 2, quad = warp % 4, qt = ew / 4;
    constexpr int W = (N / 4) / 8 * 8;
    for (int t = 0; t < tiles; ++t) {
      const int b = t % NACC;
      bar_wait(&tfull[b], (uint32_t)(t / NACC) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ta = tm + ((uint32_t)(32 * quad) << 16) + (uint32_t)(b * N + qt * W);
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
            "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
            "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
      if (r[0] == 0x12345678u && r[31] == 7u) clk[0] = 1;  // keep the loads
    }
  } else if (tid == 0) {
    const unsigned long long t0 = clock64();
    const uint64_t da0 = desc(su32(sa), M / 8 * 128, 128);
    const uint64_t db0 = desc(su32(sb), N / 8 * 128, 128);
    constexpr uint64_t DA = 2 * (M / 8 * 128) / 16, DB = 2 * (N / 8 * 128) / 16;
    for (int t = 0; t < tiles; ++t) {
      const int b = t % NACC;
      if (t >= NACC) {
        if (spin) bar_wait(&tempty[b], (uint32_t)((t / NACC) - 1) & 1u);
        else
          asm volatile(
              "{\n .reg .pred p;\n WS: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 20000;\n @!p bra WS;\n}\n" ::"r"(
                  su32(&tempty[b])),
              "r"((uint32_t)((t / NACC) - 1) & 1u)
              : "memory");
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tm + (uint32_t)b * N;
#pragma unroll
      for (int ks = 0; ks < 3; ++ks)
        mma_mxf4(dt, da0 + ks * DA, db0 + ks * DB, idesc_mxf4(N), ks > 0, tm + 480, tm + 496);
      commit(&tfull[b]);
    }
    clk[blockIdx.x + 1] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int NACC>
static void pipe(int sms, int spin) {
  const int tiles = 20000;
  const int smem = M * KB + N * KB;
  CK(cudaFuncSetAttribute(k_pipe<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* dclk;
  CK(cudaMalloc(&dclk, (sms + 1) * 8));
  k_pipe<N, NACC><<<sms, 32 * 18, smem>>>(100, dclk, spin);
  CK(cudaDeviceSynchronize());
  k_pipe<N, NACC><<<sms, 32 * 18, smem>>>(tiles, dclk, spin);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> clk(sms + 1);
  CK(cudaMemcpy(clk.data(), dclk, (sms + 1) * 8, cudaMemcpyDeviceToHost));
  unsigned long long mx = 0;
  for (int i = 1; i <= sms; ++i) mx = clk[i] > mx ? clk[i] : mx;
  printf("pipe mxf4 N=%3d, %d accumulators, %s: %.1f clk per tile (MMA + epilogue round trip)\n", N, NACC,
         spin ? "spin waits" : "suspend-hint waits", (double)mx / tiles);
  cudaFree(dclk);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int bad = check<64>() + check<208>() + check<240>();
  peak<0, 256>(sms);
  peak<0, 208>(sms);
  peak<0, 128>(sms);
  peak<0, 64>(sms);
  peak<1, 240>(sms);
  peak<1, 208>(sms);
  peak<1, 128>(sms);
  peak<1, 64>(sms);
  pipe<208, 2>(sms, 1);
  pipe<208, 2>(sms, 0);
  pipe<160, 3>(sms, 1);
  pipe<112, 4>(sms, 1);
  pipe<128, 2>(sms, 1);
  return bad != 0;
}
