// fps_mma.cuh — multi-query scan on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM). Default for batches of
// >= 192 queries (top-k and range); FPS_MMA=0 disables it, FPS_MMA=1 forces it.
//
// For 0/1 vectors the AND-popcount is a dot product: c = |a AND q| = a . q,
// and the reference distance (scan.py:137-143, popcount of the XOR of the
// three full words) is d = |a| + |q| - 2c, with |a|, |q| counted over all
// 192 bits (pad bits included, as the reference XORs them). So a batch of
// queries against a library tile is an int8 GEMM with K = 192 (keys 1..166 +
// pad bits): A = 128 library entries x 192 bytes (0/1), B = N (64/128/256)
// queries x 192 bytes, D = 128 x N int32 in TMEM. The test d <= T_q is
// folded into the GEMM (compact libraries, whose bits 168.. are zero): B
// holds 2 x the query bits and, in K slots 168..171, T_q - |q| (three s8
// parts) and -1; A holds the entry bits and 1, 1, 1, |a|. So D = T_q - d:
// a pair passes iff D >= 0, and its distance is T_q - D.
//
// Exactness (top-k): T_q is the k-th distance of an exact top-k of a library
// prefix (every prefix entry is in the library, so the true k-th distance is
// <= T_q); every pair with d <= T_q is collected into the query's candidate
// list and select_kernel keeps the k smallest (distance, index). Lists that
// overflow their capacity are reported and the batch is recomputed by the
// bit-sliced kernel. Range: T_q is the radius.
//
// CTA = 22 warps, one CTA per SM: a loader warp streams library tiles into a
// raw ring (cp.async.bulk); producer warps 0-3 expand them to the canonical
// K-major int8 layout (a thread per entry row) in a 4-stage ring; one lane of
// the MMA warp issues 6 x K=32 MMAs per tile into one of two TMEM
// accumulators and commits them to mbarriers; 16 epilogue warps (two groups
// on alternate tiles) read the accumulators with tcgen05.ld .pack::16b and
// test 16 columns at a time (max first, exact check only when it can pass).
#pragma once
#include "fps_kernels.cuh"

namespace fps {

constexpr int MM_M = 128;          // entries per tile (TMEM lanes)
constexpr int MM_N = 256;          // queries per CTA chunk (TMEM columns per accumulator), largest shape
                                   // (mma_scan_kernel<N>: N = 64 / 128 / 256 by batch size)
constexpr int MM_K = 192;          // bytes per row (3 x 64 bits)
constexpr int MM_KX = 168;         // first K slot of the fused-test terms (bits 168.. are zero in compact libraries)
constexpr int MM_STAGES = 4;
constexpr u32 MM_A_BYTES = MM_M * MM_K;  // 24 KB
constexpr u32 MM_B_BYTES = MM_N * MM_K;  // 48 KB (N = 256)
__host__ __device__ constexpr u32 mm_b_bytes(int n) { return (u32)n * MM_K; }
constexpr int MM_EPI = 16;                // epilogue warps: 2 groups (alternate tiles) x 4 lane quadrants x 2 column halves
#ifndef FPS_MM_SUSPEND_NS
#define FPS_MM_SUSPEND_NS 20000
#endif
constexpr unsigned MM_SUSPEND_NS = FPS_MM_SUSPEND_NS;  // try_wait suspend hint: waiting warps sleep instead of spinning
constexpr int MM_RAW = 8;                 // raw library tiles in flight per CTA (bulk-copy ring)
constexpr u32 MM_RAW_BYTES_MAX = 24 * 256; // >= tile_bytes(compact) and tile_bytes(full)
constexpr int MM_THREADS = (4 + MM_EPI + 2) * 32;  // producers, epilogue, MMA issuer, loader

// byte (row, k) of a K-major, no-swizzle canonical operand with `rows` rows
__host__ __device__ __forceinline__ u32 mm_canon(u32 row, u32 k, u32 rows) {
  return (k / 16) * (rows / 8 * 128) + (row / 8) * 128 + (row % 8) * 16 + (k % 16);
}

__device__ __forceinline__ u64 mm_desc(u32 saddr, u32 lbo, u32 sbo) {
  u64 d = (u64)((saddr >> 4) & 0x3fff);
  d |= (u64)((lbo >> 4) & 0x3fff) << 16;
  d |= (u64)((sbo >> 4) & 0x3fff) << 32;
  d |= (u64)1 << 46;  // descriptor version (sm_100); base offset 0, SWIZZLE_NONE
  return d;
}

// Query chunk operands, built once per call: B in the canonical layout
// (queries past Q are zero rows) and per column u = T - |q| (INT_MIN/2: never passes).
// Columns are ordered by u (sorted keys (u + 2^20) << 32 | query), so the 16
// columns a thread tests together have nearly the same u and their shared
// bound (max u) rarely lets a chunk through that no column passes.
__global__ void mm_ukeys_kernel(const u64* __restrict__ q, u32 Q, const u32* __restrict__ tq, u64* __restrict__ keys) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Q) return;
  const u32 pop = (u32)(__popcll(q[3 * (u64)i]) + __popcll(q[3 * (u64)i + 1]) + __popcll(q[3 * (u64)i + 2]));
  keys[i] = ((u64)((int)tq[i] - (int)pop + (1 << 20)) << 32) | i;
}

// B of the fused test (compact libraries: bits 168..191 of every entry and
// query are zero, so K slots 168..171 are free): B[k] = 2 x bit k of the query
// (s8), B[168..170] = T - |q| split into three s8 parts, B[171] = -1; the
// library side sets A[168..170] = 1 and A[171] = |a|. The accumulator is then
// D = 2c + (T - |q|) - |a| = T - d: the pair passes iff D >= 0, and d = T - D.
// Padding columns (past Q) get T - |q| = -384: D < 0 for every entry.
__global__ void mm_prep_kernel(const u64* __restrict__ q, u32 Q, const u32* __restrict__ tq, unsigned char* __restrict__ bop,
                               int* __restrict__ tcol, u32* __restrict__ qpop, u32 nchunks,
                               const u64* __restrict__ order, u32* __restrict__ qcol, u32 NN) {
  const u32 col = blockIdx.x * blockDim.x + threadIdx.x;  // global column = chunk * NN + j
  if (col >= nchunks * NN) return;
  const u32 chunk = col / NN, j = col % NN;
  u64 w[3] = {0, 0, 0};
  const bool ok = col < Q;
  const u32 qi = ok ? (u32)(order[col] & 0xffffffffu) : 0u;
  if (ok) { w[0] = q[3 * (u64)qi]; w[1] = q[3 * (u64)qi + 1]; w[2] = q[3 * (u64)qi + 2]; }
  qcol[col] = qi;
  unsigned char* b = bop + (u64)chunk * mm_b_bytes((int)NN);
  for (u32 k = 0; k < MM_K; ++k) b[mm_canon(j, k, NN)] = (unsigned char)(((w[k >> 6] >> (k & 63)) & 1) * 2);
  const u32 pop = (u32)(__popcll(w[0]) + __popcll(w[1]) + __popcll(w[2]));
  qpop[col] = pop;
  int u = ok ? (int)tq[qi] - (int)pop : -384;
  for (u32 k = MM_KX; k < MM_KX + 3; ++k) {
    const int part = u < -128 ? -128 : (u > 127 ? 127 : u);
    u -= part;
    b[mm_canon(j, k, NN)] = (unsigned char)(signed char)part;
  }
  b[mm_canon(j, MM_KX + 3, NN)] = (unsigned char)(signed char)-1;
  tcol[col] = ok ? (int)tq[qi] : 0;
}

// range: the bound of query q is its radius
__global__ void mm_radius_kernel(const unsigned char* __restrict__ radius, u32 Q, u32* __restrict__ tq) {
  const u32 q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < Q) tq[q] = radius[q];
}

// Per query: the seed bound T_q = k-th distance of the seed top-k (255 when
// the seed holds fewer than k entries: everything is a candidate).
__global__ void mm_seed_kernel(const u64* __restrict__ keys, const u32* __restrict__ cnt, u32 Q, u32 k, u32* tq) {
  const u32 q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < Q) tq[q] = cnt[q] >= k ? key_d(keys[(u64)q * k + k - 1]) : 255u;
}

// Distances of the collected pairs (the scan stores indices only): top-k
// lists [Q][cap] (counts clamped to cap) or range keys (query << 48 | index).
__global__ void mm_fix_kernel(PlanesOut lib, u64 index_base, const u64* __restrict__ q, u64* __restrict__ keys,
                              const u32* __restrict__ cnt, u32 cap, const u64* __restrict__ n_range, u64 range_cap) {
  if (n_range) {
    const u64 n = min(*n_range, range_cap);
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
      const u64 k = keys[i];
      const u64 qi = k >> 48, idx = k & ((1ull << 40) - 1);
      u64 w0, w1, w2;
      lib.get(idx - index_base, w0, w1, w2);
      const u32 d = (u32)(__popcll(w0 ^ q[3 * qi]) + __popcll(w1 ^ q[3 * qi + 1]) + __popcll(w2 ^ q[3 * qi + 2]));
      keys[i] = (qi << 48) | make_key(d, idx);
    }
    return;
  }
  const u32 qi = blockIdx.y;
  if (cnt[qi] > cap) return;  // overflowed list (unwritten slots): the gated fallback pass recomputes the batch
  const u32 n = cnt[qi];
  const u64 q0 = q[3 * (u64)qi], q1 = q[3 * (u64)qi + 1], q2 = q[3 * (u64)qi + 2];
  u64* kq = keys + (u64)qi * cap;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 idx = kq[i];
    u64 w0, w1, w2;
    lib.get(idx - index_base, w0, w1, w2);
    kq[i] = make_key((u32)(__popcll(w0 ^ q0) + __popcll(w1 ^ q1) + __popcll(w2 ^ q2)), idx);
  }
}

// The exact top-k so far (keys, cnt: the previous pass's select) opens the
// candidate lists of the next range pass: indices only, as the scan stores
// them (mm_fix_kernel recomputes the distances of the whole list).
__global__ void mm_carry_kernel(const u64* __restrict__ keys, const u32* __restrict__ cnt, u32 k,
                                u64* __restrict__ cand, u32* __restrict__ cand_cnt, u32 cap) {
  const u32 qi = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  const u32 n = min(cnt[qi], k);
  if (i < n && i < cap) cand[(u64)qi * cap + i] = keys[(u64)qi * k + i] & IDX_MASK;
  if (i == 0) cand_cnt[qi] = n;
}

struct MmArgs {
  PlanesOut lib;
  u64 n, index_base;
  u64 n_tiles;              // ceil(n / 128)
  u64 tile0;                // first 128-entry tile of this pass (a multiple of the library tile): entries [128 tile0, n)
  u32 Q, nchunks, parts;    // CTA c: chunk c % nchunks, tile range part c / nchunks
  const unsigned char* bop; // [nchunks][48 KB] canonical B
  const int* tcol;          // [nchunks * 256] T of each column's query (d = T - D)
  const u32* qpop;          // [nchunks * 256] |q| per column
  const u32* qcol;          // [nchunks * 256] query of each column
  u64* cand;                // [Q][cap] keys d << 40 | index
  u32* cand_cnt;            // [Q]
  u32 cap;
  u32 mode;                 // 0 top-k candidates (keys), 1 range hits (query << 48 | key) into out
  u64* out;
  u64* out_cnt;
  u64 out_cap;
  u32 flags;                // experiments: 4096 = epilogue without tests, 8192 = producer without library loads
  u64* priv;                // top-k: [CTA][N columns][pcap] private candidate lists (no global atomics on the scan path)
  u32 pcap;
  u32 suspend_ns;           // fp4 kernel: try_wait suspend hint on the MMA / epilogue barriers (0: spin)
};

__device__ __forceinline__ void mm_bar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mm_bar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// One arrival per warp (after every lane's prior accesses): the fp4 kernels'
// epilogue warps release an accumulator with one arrival each.
__device__ __forceinline__ void mm_bar_arrive_warp(u64* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mm_bar_arrive(bar);
}
__device__ __forceinline__ void mm_bar_wait_ns(u64* bar, u32 parity, u32 ns) {
  asm volatile(
      "{\n .reg .pred p;\n MMWN: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra MMWN;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity), "r"(ns)
      : "memory");
}
__device__ __forceinline__ void mm_bar_wait_spin(u64* bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n MMWS: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra MMWS;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mm_bar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n MMW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra MMW;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity), "r"(MM_SUSPEND_NS)
      : "memory");
}
// One elected lane of a converged warp. The single-thread roles (MMA issuer,
// TMA loader) run their loops with the whole warp and issue under this: in a
// lane-0-only branch every tcgen05 / TMA instruction's operands live in vector
// registers and ptxas wraps each in a per-lane loop (R2UR, ELECT, BRA.U.ANY),
// which costs ~775 clk per tile of 3 MMAs + 2 commits + 2 waits against 312 clk
// warp-uniform (tools/microbench/mma_lane.cu, profiles/r02_mma_lane.txt).
__device__ __forceinline__ bool mm_elect_one() {
  u32 pred = 0;
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}\n" : "=r"(pred));
  return pred != 0;
}
// A warp index / shared value the compiler can treat as warp-uniform.
__device__ __forceinline__ int mm_warp_uniform(int v) { return __shfl_sync(0xffffffffu, v, 0); }
__device__ __forceinline__ void mm_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 consecutive TMEM columns of the warp's lane quadrant (one row per lane)
__device__ __forceinline__ void mm_ld32(u32 taddr, u32 (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 consecutive TMEM columns, the low 16 bits of each, two per register
// (column 2i in bits 0-15 of r[i], column 2i+1 in bits 16-31)
__device__ __forceinline__ void mm_ld32p(u32 taddr, u32 (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void mm_ld16p(u32 taddr, u32 (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ u32 mm_max16(const u32* v) {
  const u32 a0 = max(max(v[0], v[1]), v[2]), a1 = max(max(v[3], v[4]), v[5]), a2 = max(max(v[6], v[7]), v[8]);
  const u32 a3 = max(max(v[9], v[10]), v[11]), a4 = max(max(v[12], v[13]), v[14]);
  return max(max(max(a0, a1), max(a2, a3)), max(a4, v[15]));
}

template <int N>
__global__ void __launch_bounds__(MM_THREADS, 1) mma_scan_kernel(const MmArgs a) {
  static_assert(N == 64 || N == 128 || N == 256, "accumulator width");
  constexpr u32 B_BYTES = mm_b_bytes(N);
  constexpr u32 TMEM_COLS = 2 * N;         // two accumulators (power of two >= 32)
  extern __shared__ __align__(1024) unsigned char msm[];
  unsigned char* sB = msm;
  unsigned char* sA = msm + B_BYTES;  // [MM_STAGES][24 KB]
  char* raw = reinterpret_cast<char*>(msm + B_BYTES + MM_STAGES * MM_A_BYTES);  // [MM_RAW][library tile]
  __shared__ __align__(8) u64 full_bar[MM_STAGES], empty_bar[MM_STAGES], tfull[2], tempty[2];
  __shared__ __align__(8) u64 raw_full[MM_RAW], raw_empty[MM_RAW];
  __shared__ u32 tmem_base;
  __shared__ u32 lut[16];
  __shared__ int s_t[N];
  __shared__ u32 s_qcol[N], s_qpop[N], s_pcnt[N];
  const int tid = threadIdx.x, warp = mm_warp_uniform(tid >> 5), lane = tid & 31;
  const u32 chunk = blockIdx.x % a.nchunks;
  const u64 part = blockIdx.x / a.nchunks;
  // CTA work: a contiguous run of library tiles (SUB MMA tiles of 128 entries each)
  const u32 SUB = a.lib.compact ? TILE_CMP / MM_M : TILE_FULL / MM_M;
  const u32 RAW_BYTES = (u32)tile_bytes(a.lib.compact);
  const u64 n_raw = (a.n + tile_entries(a.lib.compact) - 1) / tile_entries(a.lib.compact);
  const u64 raw0 = a.tile0 / (tile_entries(a.lib.compact) / MM_M);
  const u64 r0 = raw0 + part * (n_raw - raw0) / a.parts, r1 = raw0 + (part + 1) * (n_raw - raw0) / a.parts;
  const u64 nraw = r1 > r0 ? r1 - r0 : 0;
  const u64 t0 = r0 * SUB;

  // ---- setup: B chunk, thresholds, table, barriers, TMEM
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.bop + (u64)chunk * B_BYTES);
    uint4* dst = reinterpret_cast<uint4*>(sB);
    for (u32 i = tid; i < B_BYTES / 16; i += blockDim.x) dst[i] = src[i];
  }
  for (int i = tid; i < N; i += blockDim.x) {
    s_t[i] = a.tcol[chunk * N + i];
    s_qcol[i] = a.qcol[chunk * N + i];
    s_qpop[i] = a.qpop[chunk * N + i];
    s_pcnt[i] = 0;
  }
  if (tid < 16) lut[tid] = (tid & 1) | ((tid >> 1) & 1) << 8 | ((tid >> 2) & 1) << 16 | ((tid >> 3) & 1) << 24;
  if (tid == 0) {
    for (int s = 0; s < MM_STAGES; ++s) {
      mm_bar_init(&full_bar[s], 128);
      mm_bar_init(&empty_bar[s], 1);
    }
    for (int r = 0; r < MM_RAW; ++r) {
      mm_bar_init(&raw_full[r], 1);
      mm_bar_init(&raw_empty[r], 128);
    }
    for (int b = 0; b < 2; ++b) {
      mm_bar_init(&tfull[b], 1);
      mm_bar_init(&tempty[b], MM_EPI / 2 * 32);  // one epilogue group per accumulator
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
  const u64 ntile = nraw * SUB;

  if (warp < 4) {
    // ===== producers: thread = entry row of the tile; the entry's words come
    // from the raw-tile ring the loader warp fills with bulk copies
    const u32 row = (u32)tid;
    for (u64 it = 0; it < ntile; ++it) {
      const int s = (int)(it % MM_STAGES);
      const u64 r = it / SUB;
      const u32 sub = (u32)(it % SUB);
      const int rs = (int)(r % MM_RAW);
      if (sub == 0) mm_bar_wait(&raw_full[rs], (u32)(r / MM_RAW) & 1u);
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
      if (sub == SUB - 1) mm_bar_arrive(&raw_empty[rs]);
      if (it >= MM_STAGES) mm_bar_wait(&empty_bar[s], (u32)((it / MM_STAGES) - 1) & 1u);
      unsigned char* A = sA + s * MM_A_BYTES;
#pragma unroll
      for (int c = 0; c < MM_K / 16; ++c) {
        const u32 bits = (u32)(w[c >> 2] >> (16 * (c & 3))) & 0xffffu;
        // 4 bits -> 4 bytes: the shifted copies of a nibble at bits 0/7/14/21
        // do not overlap, so one multiply spreads them (then keep bit 0 of each byte)
        uint4 v;
        v.x = ((bits & 15u) * 0x204081u) & 0x01010101u;
        v.y = (((bits >> 4) & 15u) * 0x204081u) & 0x01010101u;
        v.z = (((bits >> 8) & 15u) * 0x204081u) & 0x01010101u;
        v.w = ((bits >> 12) * 0x204081u) & 0x01010101u;
        if (c == MM_KX / 16) {  // bytes 168..171: the fused-test terms 1, 1, 1, |a|
          const u32 pa = (u32)(__popcll(w[0]) + __popcll(w[1]) + __popcll(w[2]));
          v.z = 0x00010101u | (pa << 24);
        }
        *reinterpret_cast<uint4*>(A + mm_canon(row, 16 * c, MM_M)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mm_bar_arrive(&full_bar[s]);
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
    // ===== epilogue: two groups of 8 warps take alternate tiles (group g
    // always reads accumulator g), so a group has two MMA tiles of time for
    // its loads and tests and the accumulator it holds is released as soon as
    // its loads land. Warp (quad, half) of a group reads TMEM lane quadrant
    // quad (rows 32 quad .. + 31), columns [half * N / 2, (half + 1) * N / 2),
    // in rounds of <= 64 columns. The accumulators D = T - d fit 16 bits, so
    // tcgen05.ld .pack::16b brings two columns per register. Common path: the
    // AND of a round's registers (a column passes iff its sign bit is clear);
    // the per-column extraction runs only for lanes that hold a passing pair.
    const u32 grp = (u32)(warp - 4) / 8;
    const u32 wq = (u32)(warp - 4) % 8;
    const u32 quad = wq % 4, half = wq / 4;
    const u32 row = quad * 32 + lane;
    constexpr int NC = N / 2;                  // columns per warp
    constexpr int RC = NC < 64 ? NC : 64;      // columns per round
    constexpr int NRND = NC / RC;
    constexpr int RR = RC / 2;                 // packed registers per round
    for (u64 it = grp; it < ntile; it += 2) {
      const int b = (int)grp;
      const u64 e = (t0 + it) * MM_M + row;
      mm_bar_wait(&tfull[b], (u32)(it >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const u32 taddr = tmem + (quad * 32u << 16) + (u32)b * N + half * NC;
#pragma unroll 1
      for (int rnd = 0; rnd < NRND; ++rnd) {
        u32 r[RR];
        if constexpr (RR == 16) {
          mm_ld32p(taddr + RC * rnd, r);
        } else {
#pragma unroll
          for (int g = 0; g < RR / 16; ++g) mm_ld32p(taddr + RC * rnd + 32 * g, *reinterpret_cast<u32(*)[16]>(r + 16 * g));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (rnd == NRND - 1) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mm_bar_arrive(&tempty[b]);
        }
        if (a.flags & 4096) continue;
        // D = T - d per column (s16 halves): some column passes iff a sign
        // bit of the AND of all halves is clear
        u32 t = r[0];
#pragma unroll
        for (int i = 1; i < RR; ++i) t &= r[i];
        bool any = (t & 0x80008000u) != 0x80008000u && e < a.n;
        if (a.flags & 16384) any = false;  // experiment: no hits (timing only)
        if (!__any_sync(0xffffffffu, any)) continue;
        if (!any) continue;
        const int cb0 = (int)half * NC + RC * rnd;
        // passing columns as a bit mask (straight-line), then a compact loop:
        // the hit path stays small (instruction cache) and needs no register
        // indexing. Keys carry the index only; mm_fix_kernel computes the
        // distances of the (few) collected pairs from the library words.
        u64 hm = 0;
#pragma unroll
        for (int i = 0; i < RR; ++i) {
          const u32 nn = ~r[i];
          hm |= ((u64)((nn >> 15) & 1u) << (2 * i)) | ((u64)(nn >> 31) << (2 * i + 1));
        }
        const u64 idx = a.index_base + e;
        while (hm) {
          const int c = cb0 + __ffsll((long long)hm) - 1;
          hm &= hm - 1;
          if (a.mode == 0) {
            // the CTA's private list of this column: a shared-memory counter,
            // a store that nothing waits on; published at the end
            const u32 pos = atomicAdd(s_pcnt + c, 1u);
            if (pos < a.pcap) a.priv[((u64)blockIdx.x * N + c) * a.pcap + pos] = idx;
          } else {
            const u64 pos = atomicAdd(a.out_cnt, 1ull);
            if (pos < a.out_cap) a.out[pos] = ((u64)s_qcol[c] << 48) | idx;
          }
        }
      }
    }
  } else {
    // ===== MMA issuer (the whole warp waits, one elected lane issues)
    // s32 += u8 (library) x s8 (queries, fused-test terms), both K-major
    const u32 idesc = (2u << 4) | (1u << 10) | ((u32)(N >> 3) << 17) | ((u32)(MM_M >> 4) << 24);
    // descriptors: built once; a K step / stage only moves the start
    // address field (bits 0-13, in 16-byte units; shared addresses < 256 KB
    // never carry out of it), so the issue loop is a few uniform adds per MMA
    const u64 db0 = mm_desc(smem_u32(sB), N / 8 * 128, 128);
    const u64 da0 = mm_desc(smem_u32(sA), MM_M / 8 * 128, 128);
    constexpr u64 DA_K = 2 * (MM_M / 8 * 128) / 16, DB_K = 2 * (N / 8 * 128) / 16, DA_S = MM_A_BYTES / 16;
    for (u64 it = 0; it < ntile; ++it) {
      const int s = (int)(it % MM_STAGES), b = (int)(it & 1);
      if (it >= 2) mm_bar_wait(&tempty[b], (u32)((it >> 1) - 1) & 1u);
      mm_bar_wait(&full_bar[s], (u32)(it / MM_STAGES) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (mm_elect_one()) {
        const u64 das = da0 + (u64)s * DA_S;
        const u32 dt = tmem + (u32)b * N;
#pragma unroll
        for (int ks = 0; ks < MM_K / 32; ++ks) {
          if (ks == 0)
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;" ::"r"(dt), "l"(das), "l"(db0),
                         "r"(idesc));
          else
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(dt), "l"(das + ks * DA_K),
                         "l"(db0 + ks * DB_K), "r"(idesc));
        }
        mm_commit(&empty_bar[s]);
        mm_commit(&tfull[b]);
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (a.mode == 0) {
    // publish the private lists: one global atomic per (column, CTA); a list
    // past its capacity poisons its query's count (> cap: the host falls back)
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
