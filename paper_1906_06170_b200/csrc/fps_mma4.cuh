// fps_mma4.cuh — the multi-query scan on the block-scaled fp4 tensor-core
// path (tcgen05.mma kind::mxf4, e2m1 operands, f32 accumulators in TMEM):
// twice the MMA rate of kind::i8 on B200 (measured: 8.84 vs 4.56 dense POP/s,
// tools/microbench/umma_peak.cu, profiles/r02_umma_peak.txt).
//
// Same algebra as fps_mma.cuh (for 0/1 vectors the AND-popcount is a dot
// product; the reference distance popcount(a XOR q) over the three words,
// scan.py:137-143, is d = |a| + |q| - 2c), with the operands as e2m1 values
// and every block scale factor 1.0 (ue8m0 127):
//   A (library row)  : element k = 1.0 if bit k is set (k < 168), then test digits
//   B (query column) : element k = 2.0 if query bit k is set, then test digits
// Element order (any permutation of K applied to both operands leaves the
// dot product unchanged): in each 32-element block c, u32 word t (elements
// 8t..8t+7), nibble j holds bit 32c + 4j + t, so a producer builds a word as
// ((x >> t) << 1) & 0x22222222 from the block's 32 bits x -- two ALU ops, no
// table. Bits 168..191 are zero in a compact library (the 21 B/entry layout
// keeps 168 bits), so in block 5 only nibbles 0-1 of each word carry bits
// (160..167) and nibbles 2-7 of words 0-2 carry the test terms (e2m1 values
// are 0, .5, 1, 1.5, 2, 3, 4, 6 and negatives):
//   word 0 nibbles 2-6   A = digits of P = |a| / 6      B = -6
//   word 0 nibble 7,
//   word 1 nibble 2      A = digits of R = |a| % 6      B = -1
//   word 1 nibbles 3-7,
//   word 2 nibbles 2-4   A = 6                          B = digits of X = trunc(v / 6), v = T - |q| + 0.5
//   word 2 nibbles 5-6   A = 1                          B = digits of Y = v - 6X
// so the accumulator is D = 2c - |a| + v = T - d + 0.5: never zero, and the
// pair passes (d <= T) iff the f32 sign bit is clear. All terms are small
// integers or halves: the f32 sums are exact (checked bit-exactly on random
// and extreme rows / columns by the microbenchmark, and end to end by the
// parity tests against the reference goldens and the C oracle).
//
// Pipeline as in fps_mma.cuh (one CTA per SM): a loader warp streams library
// tiles (bulk copies), 4 producer warps expand a 128-entry tile to the
// canonical K-major fp4 layout (two ALU ops per 8 elements, 96 B per row
// instead of 192), one lane issues 3 x K=64 MMAs per tile into one of two
// TMEM accumulators, 16 epilogue warps (4 lane quadrants x 4 column
// quarters, every tile) test the sign bits. TMEM: two N-column
// accumulators (N <= 240) and the scale factors in columns 480..511.
#pragma once
#include "fps_mma.cuh"

namespace fps {

__device__ unsigned long long g_mm4_trace[64 * 8];  // debug (scan flag 1 << 20): CTA 0, tiles 2000..2063
#define MM4_TRACE(slot)                                                                      \
  do {                                                                                       \
    if ((a.flags & (1u << 20)) && blockIdx.x == 0 && it >= 2000 && it < 2064)                \
      g_mm4_trace[(it - 2000) * 8 + (slot)] = clock64();                                     \
  } while (0)

constexpr int MM4_KB = 96;                       // bytes per operand row (192 e2m1 elements)
constexpr u32 MM4_A_BYTES = MM_M * MM4_KB;       // 12 KB per stage
constexpr int MM4_STAGES = 6;
constexpr u32 MM4_SF_COL = 480;                  // scale factors (all 1.0): SFA at 480, SFB at 496
__host__ __device__ constexpr u32 mm4_b_bytes(int n) { return (u32)n * MM4_KB; }
__host__ __device__ constexpr size_t mm4_smem(int n) {
  return mm4_b_bytes(n) + (size_t)MM4_STAGES * MM4_A_BYTES + (size_t)MM_RAW * MM_RAW_BYTES_MAX;
}

// e2m1 code of a value in {0, .5, 1, 1.5, 2, 3, 4, 6} (and negatives)
__host__ __device__ __forceinline__ u32 e2m1(int twice) {  // argument: 2 x value
  const u32 s = twice < 0 ? 8u : 0u;
  const int a = twice < 0 ? -twice : twice;
  const u32 c = a == 0 ? 0u : a == 1 ? 1u : a == 2 ? 2u : a == 3 ? 3u : a == 4 ? 4u : a == 6 ? 5u : a == 8 ? 6u : 7u;
  return c ? (s | c) : 0u;
}
// greedy e2m1 digits of x/2 (x = 2 x the value, a multiple of 1) into `slots`
// nibbles of `out` starting at nibble `pos` (values 6, 4, 3, 2, 1.5, 1, .5)
__host__ __device__ inline u64 e2m1_digits(int x, int slots) {
  const int sg = x < 0 ? -1 : 1;
  int a = x * sg;
  u64 out = 0;
  for (int i = 0; i < slots; ++i) {
    const int v = a >= 12 ? 12 : a >= 8 ? 8 : a >= 6 ? 6 : a >= 4 ? 4 : a;  // 2 x {6, 4, 3, 2, <=1.5}
    a -= v;
    out |= (u64)e2m1(sg * v) << (4 * i);
  }
  return out;
}

// Block-5 test slots, as (word, nibble) -> a flat nibble index 8 * word + nibble.
constexpr int MM4_P0 = 2;    // P digits: word 0 nibbles 2..6
constexpr int MM4_R0 = 7;    // R digits: word 0 nibble 7, word 1 nibble 2 (flat 7 and 10)
constexpr int MM4_X0 = 11;   // X digits: word 1 nibbles 3..7 (flat 11..15), word 2 nibbles 2..4 (flat 18..20)
constexpr int MM4_Y0 = 21;   // Y digits: word 2 nibbles 5..6 (flat 21..22)

// The four u32 words of a 32-element block from its 32 bits x (element order above).
__host__ __device__ __forceinline__ void mm4_words(u32 x, u32 code, u32 (&o)[4]) {
  // code = e2m1 code of the operand's "1" value (1.0 = 2 for A, 2.0 = 4 for B), placed by a multiply
  const u32 m = 0x11111111u;
  o[0] = (x & m) * code;
  o[1] = ((x >> 1) & m) * code;
  o[2] = ((x >> 2) & m) * code;
  o[3] = ((x >> 3) & m) * code;
}

// B of the fp4 fused test: columns ordered by u = T - |q| (as mm_prep_kernel),
// padding columns (past Q) get v = -0.5 (D < 0 for every entry).
__global__ void mm4_prep_kernel(const u64* __restrict__ q, u32 Q, const u32* __restrict__ tq,
                                unsigned char* __restrict__ bop, int* __restrict__ tcol, u32* __restrict__ qpop,
                                u32 nchunks, const u64* __restrict__ order, u32* __restrict__ qcol, u32 NN) {
  const u32 col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= nchunks * NN) return;
  const u32 chunk = col / NN, j = col % NN;
  u64 w[3] = {0, 0, 0};
  const bool ok = col < Q;
  const u32 qi = ok ? (u32)(order[col] & 0xffffffffu) : 0u;
  if (ok) { w[0] = q[3 * (u64)qi]; w[1] = q[3 * (u64)qi + 1]; w[2] = q[3 * (u64)qi + 2]; }
  qcol[col] = qi;
  const u32 pop = (u32)(__popcll(w[0]) + __popcll(w[1]) + __popcll(w[2]));
  qpop[col] = pop;
  tcol[col] = ok ? (int)tq[qi] : 0;
  // v = T - |q| + 0.5 in halves: 2v = 2(T - |q|) + 1
  const int v2 = ok ? 2 * ((int)tq[qi] - (int)pop) + 1 : -1;
  const int X = v2 / 12;                  // trunc(v / 6)
  const int Y2 = v2 - 12 * X;             // 2 x (v - 6X)
  const u64 dx = e2m1_digits(2 * X, 8), dy = e2m1_digits(Y2, 2);
  u32 t5[4] = {0, 0, 0, 0};               // block 5 test nibbles (flat index 8 * word + nibble)
  auto setn = [&](int flat, u32 code) { t5[flat >> 3] |= code << (4 * (flat & 7)); };
  for (int i = 0; i < 5; ++i) setn(MM4_P0 + i, e2m1(-12));            // -6
  setn(MM4_R0, e2m1(-2));                                              // -1
  setn(MM4_R0 + 3, e2m1(-2));
  for (int i = 0; i < 8; ++i) setn(i < 5 ? MM4_X0 + i : 18 + (i - 5), (u32)(dx >> (4 * i)) & 15u);
  for (int i = 0; i < 2; ++i) setn(MM4_Y0 + i, (u32)(dy >> (4 * i)) & 15u);
  unsigned char* b = bop + (u64)chunk * mm4_b_bytes((int)NN);
  for (int c = 0; c < 6; ++c) {
    const u32 x = (u32)(w[c >> 1] >> (32 * (c & 1)));
    u32 o[4];
    mm4_words(x, 4u, o);  // 2.0 per set query bit
    if (c == 5)
      for (int t = 0; t < 4; ++t) o[t] = (o[t] & 0xffu) | t5[t];
    for (int t = 0; t < 4; ++t)
      for (int by = 0; by < 4; ++by) b[mm_canon(j, 16 * c + 4 * t + by, NN)] = (unsigned char)(o[t] >> (8 * by));
  }
}

__device__ __forceinline__ void mm4_mma(u32 d, u64 a, u64 b, u32 idesc, u32 acc, u32 sfa, u32 sfb) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

template <int NREG>
__device__ __forceinline__ void mm4_ld(u32 taddr, u32 (&r)[NREG]);
template <>
__device__ __forceinline__ void mm4_ld<32>(u32 taddr, u32 (&r)[32]) { mm_ld32(taddr, r); }
template <>
__device__ __forceinline__ void mm4_ld<16>(u32 taddr, u32 (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void mm4_ld<8>(u32 taddr, u32 (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// Issue the TMEM loads of CNT consecutive columns (CNT a multiple of 8, <= 64)
// into r[0, CNT): x32 / x16 / x8 pieces, one wait for all of them afterwards.
template <int CNT>
__device__ __forceinline__ void mm4_issue(u32 taddr, u32* r) {
  if constexpr (CNT >= 32) {
    mm4_ld<32>(taddr, *reinterpret_cast<u32(*)[32]>(r));
    mm4_issue<CNT - 32>(taddr + 32, r + 32);
  } else if constexpr (CNT >= 16) {
    mm4_ld<16>(taddr, *reinterpret_cast<u32(*)[16]>(r));
    mm4_issue<CNT - 16>(taddr + 16, r + 16);
  } else if constexpr (CNT >= 8) {
    mm4_ld<8>(taddr, *reinterpret_cast<u32(*)[8]>(r));
    mm4_issue<CNT - 8>(taddr + 8, r + 8);
  }
}

// Test CNT loaded columns (f32 D = T - d + 0.5: a pair passes iff the sign
// bit is clear): the AND of the sign bits first, the per-column extraction
// only for lanes that hold a passing pair. cb0 = the first column's index.
template <int CNT, int N>
__device__ __forceinline__ void mm4_test(const MmArgs& a, const u32* r, int cb0, u64 e, u32* s_pcnt,
                                         const u32* s_qcol) {
  u32 t = r[0];
#pragma unroll
  for (int i = 1; i < CNT; ++i) t &= r[i];
  const bool any = (t & 0x80000000u) == 0 && e < a.n;
  if (!__any_sync(0xffffffffu, any) || !any) return;
  const u64 idx = a.index_base + e;
#pragma unroll
  for (int g0 = 0; g0 < CNT; g0 += 64) {  // passing columns as 64-bit masks
    u64 hm = 0;
#pragma unroll
    for (int i = g0; i < (g0 + 64 < CNT ? g0 + 64 : CNT); ++i) hm |= (u64)((~r[i]) >> 31) << (i - g0);
    while (hm) {
      const int c = cb0 + g0 + __ffsll((long long)hm) - 1;
      hm &= hm - 1;
      if (a.mode == 0) {
        // the CTA's private list of this column: a shared-memory counter and a
        // store nothing waits on; published at the end
        const u32 pos = atomicAdd(s_pcnt + c, 1u);
        if (pos < a.pcap) a.priv[((u64)blockIdx.x * N + c) * a.pcap + pos] = idx;
      } else {
        const u64 pos = atomicAdd(a.out_cnt, 1ull);
        if (pos < a.out_cap) a.out[pos] = ((u64)s_qcol[c] << 48) | idx;
      }
    }
  }
}

// Epilogue columns of a warp: the N accumulator columns in 4 quarters of
// multiples of 8 (e.g. N = 208: 56, 56, 48, 48).
template <int N>
struct Mm4Quarters {
  static constexpr int U = N / 8;                       // 8-column units
  static constexpr int W_HI = 8 * ((U + 3) / 4), W_LO = 8 * (U / 4);
  static constexpr int N_HI = U % 4 ? U % 4 : 4;        // quarters of width W_HI
  __device__ static constexpr int off(int q) { return q < N_HI ? q * W_HI : N_HI * W_HI + (q - N_HI) * W_LO; }
};

// One tile of one epilogue warp: load the quarter (one wait), release the
// accumulator, test.
template <int CNT, int N>
__device__ __forceinline__ void mm4_tile(const MmArgs& a, u32 taddr, int cb0, u64 e, u64* tempty_bar, u32* s_pcnt,
                                         const u32* s_qcol) {
  u32 r[CNT];
  mm4_issue<CNT>(taddr, r);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  mm_bar_arrive_warp(tempty_bar);
  if (a.flags & 4096) return;
  mm4_test<CNT, N>(a, r, cb0, e, s_pcnt, s_qcol);
}

__device__ __forceinline__ void mm4x_wait(u32 bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n M4XW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra M4XW;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Record the passing columns of one row (rare): W <= 128 columns as two
// 64-bit masks, then one private-list append (top-k) or range-output append
// per passing pair. Out of line: inlined, the epilogue loop outgrows the
// instruction cache (C4 scan 9.8 -> 12.7 ms).
template <int W, int N>
__device__ __noinline__ void mm4x_hits(const MmArgs& a, u64 hm0, u64 hm1, int cb0, u64 idx, u32* s_pcnt,
                                       const u32* s_qcol) {
#pragma unroll 1
  for (int g = 0; g < 2; ++g) {
    u64 hm = g ? hm1 : hm0;
    while (hm) {
      const int c = cb0 + 64 * g + __ffsll((long long)hm) - 1;
      hm &= hm - 1;
      if (a.mode == 0) {
        const u32 pos = atomicAdd(s_pcnt + c, 1u);
        if (pos < a.pcap) a.priv[((u64)blockIdx.x * N + c) * a.pcap + pos] = idx;
      } else {
        const u64 pos = atomicAdd(a.out_cnt, 1ull);
        if (pos < a.out_cap) a.out[pos] = ((u64)s_qcol[c] << 48) | idx;
      }
    }
  }
}

// The epilogue loop of one warp: W accumulator columns starting at TMEM
// address ta0 (accumulator 0; accumulator 1 is N columns on), barriers
// tfull[0..1] / tempty[0..1] at bf / be (8 bytes apart).
template <int W, int N, int NACC>
__device__ __forceinline__ void mm4x_epilogue(const MmArgs& a, u32 ntile, u64 e0, u32 bf, u32 be, u32 ta0, int cb0,
                                              bool tests, u32* s_pcnt, const u32* s_qcol, u32 it0, u32 istep) {
  static_assert(W % 8 == 0 && W <= 128, "columns per warp");
  const u32 lane = threadIdx.x & 31;
#pragma unroll 1
  for (u32 it = it0; it < ntile; it += istep) {
    const u32 b = it % NACC;
    mm4x_wait(bf + 8 * b, (it / NACC) & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    u32 r[W];
    mm4_issue<W>(ta0 + b * N, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(be + 8 * b) : "memory");
    if (!tests) continue;
    u32 t = r[0];
#pragma unroll
    for (int i = 1; i < W; ++i) t &= r[i];
    const bool any = (int)t >= 0;  // some column's sign bit is clear: D > 0, the pair passes
    if (!__any_sync(0xffffffffu, any) || !any) continue;
    const u64 e = e0 + (u64)it * MM_M;
    if (e >= a.n) continue;  // padding rows of the last tile (zero operands: D > 0)
    u64 hm0 = 0, hm1 = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const u64 bit = (u64)((~r[i]) >> 31);
      if (i < 64) hm0 |= bit << i;
      else hm1 |= bit << (i - 64);
    }
    mm4x_hits<W, N>(a, hm0, hm1, cb0, a.index_base + e, s_pcnt, s_qcol);
  }
}

// The same loop for a warp owning W = 2 H columns (H <= 64) of a wide
// accumulator in a group that drains every other tile: two rounds of H
// loaded columns (half the registers), each tested as it lands; the
// accumulator is released after the second round's loads.
template <int W, int N, int NACC>
__device__ __forceinline__ void mm4x_epilogue2(const MmArgs& a, u32 ntile, u64 e0, u32 bf, u32 be, u32 ta0, int cb0,
                                               bool tests, u32* s_pcnt, const u32* s_qcol, u32 it0, u32 istep) {
  constexpr int H0 = 8 * ((W / 8 + 1) / 2), H1 = W - H0;  // e.g. 104 = 56 + 48
  static_assert(W % 8 == 0 && H0 <= 64 && H1 > 0, "two rounds of at most 64 columns");
  const u32 lane = threadIdx.x & 31;
#pragma unroll 1
  for (u32 it = it0; it < ntile; it += istep) {
    const u32 b = it % NACC;
    mm4x_wait(bf + 8 * b, (it / NACC) & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    u32 r[H0];
    mm4_issue<H0>(ta0 + b * N, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    u64 m0 = 0, m1 = 0;
    bool any = false;
    if (tests) {
      u32 t = r[0];
#pragma unroll
      for (int i = 1; i < H0; ++i) t &= r[i];
      if ((int)t >= 0) {
        any = true;
#pragma unroll
        for (int i = 0; i < H0; ++i) m0 |= (u64)((~r[i]) >> 31) << i;
      }
    }
    mm4_issue<H1>(ta0 + b * N + H0, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(be + 8 * b) : "memory");
    if (!tests) continue;
    u32 t = r[0];
#pragma unroll
    for (int i = 1; i < H1; ++i) t &= r[i];
    if ((int)t >= 0) {
      any = true;
#pragma unroll
      for (int i = 0; i < H1; ++i) m1 |= (u64)((~r[i]) >> 31) << i;
    }
    if (!__any_sync(0xffffffffu, any) || !any) continue;
    const u64 e = e0 + (u64)it * MM_M;
    if (e >= a.n) continue;  // padding rows of the last tile
    // columns [0, H0) in m0, [H0, W) in m1 -> 64-bit halves of the W columns
    u64 hm0 = m0, hm1 = m1;  // (H0 == 64: already the halves)
    if constexpr (H0 < 64) hm0 |= m1 << H0, hm1 = m1 >> (64 - H0);
    mm4x_hits<W, N>(a, hm0, hm1, cb0, a.index_base + e, s_pcnt, s_qcol);
  }
}

template <int N>
__global__ void __launch_bounds__(MM_THREADS, 1) mma4_scan_kernel(const MmArgs a) {
  static_assert(N % 16 == 0 && N >= 64 && N <= 240, "accumulator width (two accumulators + scale factors in 512 columns)");
  constexpr u32 B_BYTES = mm4_b_bytes(N);
  constexpr u32 TMEM_COLS = 512;
  extern __shared__ __align__(1024) unsigned char msm[];
  unsigned char* sB = msm;
  unsigned char* sA = msm + B_BYTES;  // [MM4_STAGES][12 KB]
  char* raw = reinterpret_cast<char*>(msm + B_BYTES + MM4_STAGES * MM4_A_BYTES);  // [MM_RAW][library tile]
  // N = 64: 4 accumulators and 4 epilogue groups of 4 warps (group g drains
  // accumulator g of every four tiles); wider: 2 accumulators, all 16
  // epilogue warps on every tile
  constexpr int NACC = N <= 64 ? 4 : 2;
  constexpr bool GROUPED = N <= 64;
  __shared__ __align__(8) u64 full_bar[MM4_STAGES], empty_bar[MM4_STAGES], tfull[NACC], tempty[NACC];
  __shared__ __align__(8) u64 raw_full[MM_RAW], raw_empty[MM_RAW];
  __shared__ u32 tmem_base;
  __shared__ uint2 luta[176];  // |a| -> block-5 test nibbles of words 0 and 1 (digits of -|a|, A = 6)
  __shared__ u32 s_qcol[N], s_pcnt[N];
  const int tid = threadIdx.x, warp = mm_warp_uniform(tid >> 5), lane = tid & 31;
  const u32 chunk = blockIdx.x % a.nchunks;
  const u64 part = blockIdx.x / a.nchunks;
  const u32 SUB = a.lib.compact ? TILE_CMP / MM_M : TILE_FULL / MM_M;
  const u32 RAW_BYTES = (u32)tile_bytes(a.lib.compact);
  const u64 n_raw = (a.n + tile_entries(a.lib.compact) - 1) / tile_entries(a.lib.compact);
  const u64 raw0 = a.tile0 / (tile_entries(a.lib.compact) / MM_M);
  const u64 r0 = raw0 + part * (n_raw - raw0) / a.parts, r1 = raw0 + (part + 1) * (n_raw - raw0) / a.parts;
  const u64 nraw = r1 > r0 ? r1 - r0 : 0;
  const u64 t0 = r0 * SUB;

  // ---- setup: B chunk, tables, barriers, TMEM (+ scale factors)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.bop + (u64)chunk * B_BYTES);
    uint4* dst = reinterpret_cast<uint4*>(sB);
    for (u32 i = tid; i < B_BYTES / 16; i += blockDim.x) dst[i] = src[i];
  }
  for (int i = tid; i < N; i += blockDim.x) {
    s_qcol[i] = a.qcol[chunk * N + i];
    s_pcnt[i] = 0;
  }
  for (int i = tid; i < 176; i += blockDim.x) {
    const u64 p = e2m1_digits(2 * (i / 6), 5), r = e2m1_digits(2 * (i % 6), 2);
    u32 t5[2] = {0, 0};
    auto setn = [&](int flat, u32 code) { t5[flat >> 3] |= code << (4 * (flat & 7)); };
    for (int d = 0; d < 5; ++d) setn(MM4_P0 + d, (u32)(p >> (4 * d)) & 15u);
    setn(MM4_R0, (u32)r & 15u);
    setn(MM4_R0 + 3, (u32)(r >> 4) & 15u);
    for (int d = 0; d < 5; ++d) setn(MM4_X0 + d, e2m1(12));  // A = 6 (word 1 nibbles 3..7)
    luta[i] = make_uint2(t5[0], t5[1]);
  }
  if (tid == 0) {
    for (int s = 0; s < MM4_STAGES; ++s) {
      mm_bar_init(&full_bar[s], 4);  // one arrival per producer warp
      mm_bar_init(&empty_bar[s], 1);
    }
    for (int r = 0; r < MM_RAW; ++r) {
      mm_bar_init(&raw_full[r], 1);
      mm_bar_init(&raw_empty[r], 4);
    }
    for (int b = 0; b < NACC; ++b) {
      mm_bar_init(&tfull[b], 1);
      mm_bar_init(&tempty[b], GROUPED ? MM_EPI / NACC : MM_EPI);  // one arrival per warp that drains it
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4 + MM_EPI) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = (u32)mm_warp_uniform((int)tmem_base);
  if (warp < 4) {  // scale factors: every byte of columns 480..511 = ue8m0 127 (1.0)
    for (u32 c = MM4_SF_COL; c < TMEM_COLS; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + ((u32)(32 * warp) << 16) + c),
                   "r"(0x7f7f7f7fu));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u64 ntile = nraw * SUB;

  if (warp < 4) {
    // ===== producers: thread = entry row; 6 x 16 B of e2m1 nibbles per row
    const u32 row = (u32)tid;
    for (u64 it = 0; it < ntile; ++it) {
      const int s = (int)(it % MM4_STAGES);
      const u64 r = it / SUB;
      const u32 sub = (u32)(it % SUB);
      const int rs = (int)(r % MM_RAW);
      if (sub == 0) mm_bar_wait(&raw_full[rs], (u32)(r / MM_RAW) & 1u);
      if (tid == 0) MM4_TRACE(3);
      u64 w[3];
      {
        const char* tb = raw + (u64)rs * RAW_BYTES;
        const u32 e = sub * MM_M + row;
        if (a.lib.compact) {
          w[0] = reinterpret_cast<const u64*>(tb)[e];
          w[1] = reinterpret_cast<const u64*>(tb + 8 * TILE_CMP)[e];
          w[2] = (u64)reinterpret_cast<const u32*>(tb + 16 * TILE_CMP)[e] |
                 ((u64)reinterpret_cast<const unsigned char*>(tb + 20 * TILE_CMP)[e] << 32);
        } else {
          w[0] = reinterpret_cast<const u64*>(tb)[e];
          w[1] = reinterpret_cast<const u64*>(tb + 8 * TILE_FULL)[e];
          w[2] = reinterpret_cast<const u64*>(tb + 16 * TILE_FULL)[e];
        }
      }
      if (sub == SUB - 1) mm_bar_arrive_warp(&raw_empty[rs]);
      const u32 pa = (u32)(__popcll(w[0]) + __popcll(w[1]) + __popcll(w[2]));
      if (it >= MM4_STAGES) mm_bar_wait(&empty_bar[s], (u32)((it / MM4_STAGES) - 1) & 1u);
      if (tid == 0) MM4_TRACE(4);
      unsigned char* A = sA + s * MM4_A_BYTES;
      const uint2 ta = luta[pa < 176 ? pa : 175];
      if (a.flags & 65536) {  // experiment: no expansion (stage left as is)
        if (!(a.flags & 32768)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mm_bar_arrive_warp(&full_bar[s]);
        continue;
      }
#pragma unroll
      for (int c = 0; c < 6; ++c) {  // 16 B = one 32-element block
        u32 o[4];
        mm4_words((u32)(w[c >> 1] >> (32 * (c & 1))), 2u, o);  // 1.0 per set bit
        if (c == 5) {  // block 5: bits 160..167 in nibbles 0-1, test terms in 2-7
          o[0] = (o[0] & 0xffu) | ta.x;
          o[1] = (o[1] & 0xffu) | ta.y;
          o[2] = (o[2] & 0xffu) | e2m1(12) * 0x111u << 8 | e2m1(2) * 0x11u << 20;  // A = 6 (nibbles 2-4), 1 (5-6)
          o[3] = o[3] & 0xffu;
        }
        *reinterpret_cast<uint4*>(A + mm_canon(row, 16 * c, MM_M)) = make_uint4(o[0], o[1], o[2], o[3]);
      }
      if (!(a.flags & 32768)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mm_bar_arrive_warp(&full_bar[s]);
      if (tid == 0) MM4_TRACE(5);
    }
  } else if (warp == 5 + MM_EPI) {
    // ===== loader (the whole warp waits, one elected lane issues): library
    // tiles -> raw ring, cp.async.bulk
    const u64 pol = l2_evict_first_policy();
    for (u64 r = 0; r < nraw; ++r) {
      const int rs = (int)(r % MM_RAW);
      if (r >= MM_RAW) mm_bar_wait(&raw_empty[rs], (u32)((r / MM_RAW) - 1) & 1u);
      if (mm_elect_one()) {
        if (a.flags & 8192) {  // experiment: no library loads
          mm_bar_arrive(&raw_full[rs]);
        } else {
          mbar_expect_tx(&raw_full[rs], RAW_BYTES);
          bulk_g2s_stream(raw + (u64)rs * RAW_BYTES, a.lib.base + (r0 + r) * RAW_BYTES, RAW_BYTES, &raw_full[rs], pol);
        }
      }
      __syncwarp();
    }
  } else if (warp < 4 + MM_EPI) {
   if constexpr (GROUPED) {
    // ===== epilogue, N = 64: 4 groups of 4 warps (one per lane quadrant, all
    // 64 columns), group g drains accumulator g of every four tiles
    const u32 ew = (u32)(warp - 4);
    const u32 quad = (u32)warp % 4, grp = ew / 4;
    mm4x_epilogue<(N <= 128 ? N : 128), N, NACC>(a, (u32)ntile, t0 * MM_M + quad * 32 + lane, smem_u32(&tfull[0]),
                                               smem_u32(&tempty[0]), tmem + (quad * 32u << 16), 0,
                                               !(a.flags & 4096), s_pcnt, s_qcol, grp, (u32)NACC);
   } else {
    // ===== epilogue: 16 warps, every tile; warp e reads TMEM lane quadrant
    // e % 4 (its warp id mod 4) and column quarter e / 4 -- one load wait
    // per tile per warp, then the accumulator is released and tested
    const u32 ew = (u32)(warp - 4);
    const u32 quad = ew % 4, qt = ew / 4;
    const u32 row = quad * 32 + lane;
    using QS = Mm4Quarters<N>;
    const int c0 = QS::off((int)qt);
    for (u64 it = 0; it < ntile; ++it) {
      const int b = (int)(it & 1);
      const u64 e = (t0 + it) * MM_M + row;
      if (a.suspend_ns) mm_bar_wait_ns(&tfull[b], (u32)(it >> 1) & 1u, a.suspend_ns);
      else mm_bar_wait_spin(&tfull[b], (u32)(it >> 1) & 1u);
      if (ew == 0 && lane == 0) MM4_TRACE(6);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const u32 taddr = tmem + (quad * 32u << 16) + (u32)b * N + (u32)c0;
      if ((int)qt < QS::N_HI) mm4_tile<QS::W_HI, N>(a, taddr, c0, e, &tempty[b], s_pcnt, s_qcol);
      else mm4_tile<QS::W_LO, N>(a, taddr, c0, e, &tempty[b], s_pcnt, s_qcol);
      if (ew == 0 && lane == 0) MM4_TRACE(7);
    }
   }
  } else {
    // ===== MMA issuer (the whole warp waits, one elected lane issues):
    // f32 += e2m1 (library) x e2m1 (queries, test terms), K-major
    const u32 idesc = (1u << 7) | (1u << 10) | ((u32)(N >> 3) << 17) | (1u << 23) | ((u32)(MM_M >> 4) << 24);
    const u64 db0 = mm_desc(smem_u32(sB), N / 8 * 128, 128);
    const u64 da0 = mm_desc(smem_u32(sA), MM_M / 8 * 128, 128);
    // K = 64 elements = 32 bytes = two core matrices per MMA
    constexpr u64 DA_K = 2 * (MM_M / 8 * 128) / 16, DB_K = 2 * (N / 8 * 128) / 16, DA_S = MM4_A_BYTES / 16;
    const u32 sfa = tmem + MM4_SF_COL, sfb = tmem + MM4_SF_COL + 16;
    for (u64 it = 0; it < ntile; ++it) {
      const int s = (int)(it % MM4_STAGES), b = (int)(it % NACC);
      if (a.suspend_ns) {
        if (it >= NACC) mm_bar_wait_ns(&tempty[b], (u32)((it / NACC) - 1) & 1u, a.suspend_ns);
        mm_bar_wait_ns(&full_bar[s], (u32)(it / MM4_STAGES) & 1u, a.suspend_ns);
      } else {
        if (it >= NACC) mm_bar_wait_spin(&tempty[b], (u32)((it / NACC) - 1) & 1u);
        MM4_TRACE(0);
        mm_bar_wait_spin(&full_bar[s], (u32)(it / MM4_STAGES) & 1u);
      }
      MM4_TRACE(1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (mm_elect_one()) {
        const u64 das = da0 + (u64)s * DA_S;
        const u32 dt = tmem + (u32)b * N;
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) mm4_mma(dt, das + ks * DA_K, db0 + ks * DB_K, idesc, ks > 0, sfa, sfb);
        mm_commit(&empty_bar[s]);
        mm_commit(&tfull[b]);
      }
      __syncwarp();
      MM4_TRACE(2);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (a.mode == 0) {
    // publish the private lists: one global atomic per (column, CTA); a list
    // past its capacity poisons its query's count (> cap: the device fallback)
    for (int c = warp; c < N; c += MM_THREADS / 32) {
      const u32 cnt = s_pcnt[c];
      if (cnt == 0) continue;
      const u32 qi = s_qcol[c];
      if (qi >= a.Q || chunk * N + c >= a.Q) continue;
      u32 base = 0;
      if (lane == 0) base = atomicAdd(a.cand_cnt + qi, cnt > a.pcap ? a.cap + 1 : cnt);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (cnt > a.pcap) continue;
      const u64* src = a.priv + ((u64)blockIdx.x * N + c) * a.pcap;
      for (u32 i = lane; i < cnt; i += 32)
        if (base + i < a.cap) a.cand[(u64)qi * a.cap + base + i] = src[i];
    }
  }
  if (warp == 4 + MM_EPI) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

}  // namespace fps
