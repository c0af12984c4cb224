// fps_mma4x.cuh — the block-scaled fp4 tensor-core scan fed from an
// operand copy of the library (the default multi-query path for large
// batches; configs 4-5 shapes).
//
// fps_mma4.cuh expands every library tile to e2m1 operands on the fly: four
// producer warps spend ~260 issue slots per 128-entry tile, once per query
// chunk, and the SM runs out of issue slots before the MMA does (ncu:
// profiles/r02_ncu_c4_i8_16warp_variant_details.csv). Here the expansion happens once per
// library: `mm4x_build_kernel` writes every 128-entry tile as the MMA's A
// operand, already in the canonical K-major layout (12 KB per tile, 96 B per
// entry: the 166 key bits as e2m1 1.0, then the |a|-dependent test digits of
// fps_mma4.cuh), so the scan CTA is a loader lane (one cp.async.bulk per
// tile straight into the A stage ring), one MMA lane (3 x K=64
// kind::mxf4 per tile into one of two TMEM accumulators) and 16 epilogue
// warps (sign tests). The query chunks of a library range run on
// neighbouring CTAs and read each A tile at about the same time, so HBM
// sees the operand copy about once per pass and the rest hits L2.
//
// Algebra, element order and the exactness argument are fps_mma4.cuh's:
// D = 2c - |a| + (T - |q| + 0.5) = T - d + 0.5 with d the reference distance
// (scan.py:137-143); a pair passes iff the f32 sign bit of D is clear.
#pragma once
#include <cuda.h>  // CUtensorMap (the map itself is encoded on the host, fps_capi.cu)

#include "fps_mma4.cuh"

namespace fps {

constexpr u32 MM4X_TILE = MM_M * MM4_KB;  // 12,288 B of A operand per 128 entries
constexpr int MM4X_STAGES = 12;
// Epilogue warps: 4 lane quadrants x EPI / 4 column parts. Fewer, wider
// warps spend fewer issue slots per tile on waits and loop overhead (the f32
// accumulators need one AND per two columns whatever the split).
__host__ __device__ constexpr int mm4x_threads(int epi) { return (epi + 2) * 32; }  // + MMA issuer, loader

// Columns of epilogue part p (of P) of an N-column accumulator: multiples of
// 8, widths differing by at most 8.
template <int N, int P>
struct Mm4Split {
  static constexpr int U = N / 8;  // 8-column units
  static constexpr int W_HI = 8 * ((U + P - 1) / P), W_LO = 8 * (U / P);
  static constexpr int N_HI = U % P ? U % P : P;  // parts of width W_HI
  __device__ static constexpr int off(int q) { return q < N_HI ? q * W_HI : N_HI * W_HI + (q - N_HI) * W_LO; }
};
__host__ __device__ constexpr size_t mm4x_smem(int n) { return mm4_b_bytes(n) + (size_t)MM4X_STAGES * MM4X_TILE; }

// Block-5 test nibbles of an entry with popcount pa (words 0 and 1; word 2
// carries the constants A = 6 at nibbles 2-4 and A = 1 at 5-6): the e2m1
// digits of P = pa / 6 (B = -6) and R = pa % 6 (B = -1), as fps_mma4.cuh.
__host__ __device__ inline uint2 mm4_test_nibbles(u32 pa) {
  const u64 p = e2m1_digits(2 * (int)(pa / 6), 5), r = e2m1_digits(2 * (int)(pa % 6), 2);
  u32 t5[2] = {0, 0};
  auto setn = [&](int flat, u32 code) { t5[flat >> 3] |= code << (4 * (flat & 7)); };
  for (int d = 0; d < 5; ++d) setn(MM4_P0 + d, (u32)(p >> (4 * d)) & 15u);
  setn(MM4_R0, (u32)r & 15u);
  setn(MM4_R0 + 3, (u32)(r >> 4) & 15u);
  for (int d = 0; d < 5; ++d) setn(MM4_X0 + d, e2m1(12));  // A = 6 against the X digits of B
  return make_uint2(t5[0], t5[1]);
}

// The operand copy: tile t (entries 128t ..) = [6 chunks][128 rows][16 B],
// i.e. byte mm_canon(row, 16 c + j, 128) = c * 2048 + 16 row + j. One thread
// per (tile, chunk, row): a warp writes 512 contiguous bytes. Rows past n are
// zero. Compact libraries only (bits 168.. must be zero: they carry the test
// terms).
__global__ void mm4x_build_kernel(PlanesOut lib, u64 n, u64 n_tiles, unsigned char* __restrict__ op) {
  const u64 total = n_tiles * 6 * MM_M;
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (u64)gridDim.x * blockDim.x) {
    const u64 tile = t / (6 * MM_M);
    const u32 c = (u32)(t / MM_M % 6), row = (u32)(t % MM_M);
    const u64 e = tile * MM_M + row;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (e < n) {
      u64 w[3];
      lib.get(e, w[0], w[1], w[2]);
      u32 o[4];
      mm4_words((u32)(w[c >> 1] >> (32 * (c & 1))), 2u, o);  // 1.0 per set bit
      if (c == 5) {
        const u32 pa = (u32)(__popcll(w[0]) + __popcll(w[1]) + __popcll(w[2]));
        const uint2 ta = mm4_test_nibbles(pa < 176 ? pa : 175);
        o[0] = (o[0] & 0xffu) | ta.x;
        o[1] = (o[1] & 0xffu) | ta.y;
        o[2] = (o[2] & 0xffu) | e2m1(12) * 0x111u << 8 | e2m1(2) * 0x11u << 20;  // A = 6 (nibbles 2-4), 1 (5-6)
        o[3] = o[3] & 0xffu;
      }
      v = make_uint4(o[0], o[1], o[2], o[3]);
    }
    *reinterpret_cast<uint4*>(op + tile * MM4X_TILE + (u64)c * (16 * MM_M) + 16 * row) = v;
  }
}

// The operand copy as a 2-D tensor for the TMA engine: rows of 256 B, a
// 128-entry tile = 48 rows (one box).
constexpr u32 MM4X_ROW = 256, MM4X_BOX_ROWS = MM4X_TILE / MM4X_ROW;

// NACC accumulators in flight; EPI epilogue warps, in NACC groups of
// EPI / NACC (>= 4, whole lane quadrants) when EPI > 8 -- group g drains
// accumulator g of every NACC tiles, so it has NACC MMA tiles of time -- or
// 8 warps on every tile (EPI = 8).
template <int N, int EPI, int NACC = 2>
__global__ void __launch_bounds__(mm4x_threads(EPI), 1)
    mma4x_scan_kernel(const MmArgs a, const unsigned char* __restrict__ op, const __grid_constant__ CUtensorMap tmap) {
  static_assert(N % 16 == 0 && N >= 64 && N <= 240, "accumulator width (two accumulators + scale factors in 512 columns)");
  static_assert(EPI % 4 == 0 && EPI >= 8 && EPI <= 28, "epilogue warps: whole lane quadrants");
  static_assert(NACC >= 2 && NACC * N + 32 <= 512, "accumulators + scale factors fit 512 TMEM columns");
  static_assert(EPI == 8 || (EPI % NACC == 0 && (EPI / NACC) % 4 == 0), "whole groups of lane quadrants");
  constexpr int MM4X_EPI = EPI;
  // 16 epilogue warps: two groups of 8 on alternate tiles (group g always
  // drains accumulator g, so it has two MMA tiles of time); 8: every tile
  constexpr int GROUPS = EPI == 8 ? 1 : NACC, GW = EPI / GROUPS;
  static_assert(N / (GW / 4) <= 128, "a warp's columns fit its registers (in two rounds when grouped)");
  constexpr int MM4X_THREADS = mm4x_threads(EPI);
  constexpr u32 B_BYTES = mm4_b_bytes(N);
  constexpr u32 TMEM_COLS = 512;
  extern __shared__ __align__(1024) unsigned char msm[];
  unsigned char* sB = msm;
  unsigned char* sA = msm + B_BYTES;  // [MM4X_STAGES][12 KB]
  __shared__ __align__(8) u64 full_bar[MM4X_STAGES], empty_bar[MM4X_STAGES], tfull[NACC], tempty[NACC];
  __shared__ u32 tmem_base;
  __shared__ u32 s_qcol[N], s_pcnt[N];
  const int tid = threadIdx.x, warp = mm_warp_uniform(tid >> 5), lane = tid & 31;
  const u32 chunk = blockIdx.x % a.nchunks;
  const u64 part = blockIdx.x / a.nchunks;
  const u64 nt = a.n_tiles - a.tile0;  // tiles of this pass
  const u64 t0 = a.tile0 + part * nt / a.parts, t1 = a.tile0 + (part + 1) * nt / a.parts;
  const u64 ntile = t1 > t0 ? t1 - t0 : 0;

  // ---- setup: B chunk, barriers, TMEM (+ scale factors)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.bop + (u64)chunk * B_BYTES);
    uint4* dst = reinterpret_cast<uint4*>(sB);
    for (u32 i = tid; i < B_BYTES / 16; i += blockDim.x) dst[i] = src[i];
  }
  for (int i = tid; i < N; i += blockDim.x) {
    s_qcol[i] = a.qcol[chunk * N + i];
    s_pcnt[i] = 0;
  }
  if (tid == 0) {
    for (int s = 0; s < MM4X_STAGES; ++s) {
      mm_bar_init(&full_bar[s], 1);
      mm_bar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mm_bar_init(&tfull[b], 1);
      mm_bar_init(&tempty[b], (u32)(MM4X_EPI / GROUPS));  // one arrival per warp of the accumulator's group
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MM4X_EPI) {
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

  if (warp == MM4X_EPI + 1) {
    // ===== loader (the whole warp waits, one elected lane issues): A tiles
    // of the operand copy -> stage ring
    const bool first = (a.flags & (1u << 22)) != 0;  // experiment: L2 evict-first on the operand tiles
    const u64 pol = l2_evict_first_policy();
    for (u64 it = 0; it < ntile; ++it) {
      const int s = (int)(it % MM4X_STAGES);
      if (it >= (u64)MM4X_STAGES) mm_bar_wait_spin(&empty_bar[s], (u32)((it / MM4X_STAGES) - 1) & 1u);
      MM4_TRACE(3);
      if (mm_elect_one()) {
        if (a.flags & 8192) {  // experiment: no operand loads (timing only)
          mm_bar_arrive(&full_bar[s]);
        } else {
          mbar_expect_tx(&full_bar[s], MM4X_TILE);
          const unsigned char* src = op + (t0 + it) * MM4X_TILE;
          if (!(a.flags & (1u << 24))) {  // default: one TMA tensor box (flag 1 << 24: a 1-D bulk copy)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];" ::"r"(smem_u32(sA + (u64)s * MM4X_TILE)),
                "l"(reinterpret_cast<u64>(&tmap)), "r"(0), "r"((u32)((t0 + it) * MM4X_BOX_ROWS)),
                "r"(smem_u32(&full_bar[s]))
                : "memory");
          } else if (first) {
            bulk_g2s_stream(sA + (u64)s * MM4X_TILE, src, MM4X_TILE, &full_bar[s], pol);
          } else {
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sA + (u64)s * MM4X_TILE)),
                "l"(src), "r"(MM4X_TILE), "r"(smem_u32(&full_bar[s]))
                : "memory");
          }
        }
      }
      __syncwarp();
    }
  } else if (warp < MM4X_EPI) {
    // ===== epilogue: EPI warps, every tile; warp e reads TMEM lane quadrant
    // e % 4 and column part e / 4 -- one load wait per tile per warp, one
    // arrival per warp releases the accumulator, then the sign bits are
    // tested (addresses, parities and the row index are carried in
    // registers: the loop is the loads, the AND chain and a vote).
    const u32 ew = (u32)warp;
    const u32 grp = ew / GW, wg = ew % GW;
    const u32 quad = wg % 4, qt = wg / 4;
    using QS = Mm4Split<N, GW / 4>;
    const int c0 = QS::off((int)qt);
    const u32 ta0 = tmem + (quad * 32u << 16) + (u32)c0;
    const u64 e0 = t0 * MM_M + quad * 32 + lane;
    const bool tests = !(a.flags & 4096);
    if constexpr (GROUPS > 1 && QS::W_HI > 64) {  // wide columns in groups: two rounds per tile
      if ((int)qt < QS::N_HI)
        mm4x_epilogue2<QS::W_HI, N, NACC>(a, (u32)ntile, e0, smem_u32(&tfull[0]), smem_u32(&tempty[0]), ta0, c0,
                                          tests, s_pcnt, s_qcol, grp, (u32)GROUPS);
      else
        mm4x_epilogue2<QS::W_LO, N, NACC>(a, (u32)ntile, e0, smem_u32(&tfull[0]), smem_u32(&tempty[0]), ta0, c0,
                                          tests, s_pcnt, s_qcol, grp, (u32)GROUPS);
    } else {
      if ((int)qt < QS::N_HI)
        mm4x_epilogue<QS::W_HI, N, NACC>(a, (u32)ntile, e0, smem_u32(&tfull[0]), smem_u32(&tempty[0]), ta0, c0,
                                         tests, s_pcnt, s_qcol, grp, (u32)GROUPS);
      else
        mm4x_epilogue<QS::W_LO, N, NACC>(a, (u32)ntile, e0, smem_u32(&tfull[0]), smem_u32(&tempty[0]), ta0, c0,
                                         tests, s_pcnt, s_qcol, grp, (u32)GROUPS);
    }
  } else {
    // ===== MMA issuer (the whole warp waits, one elected lane issues):
    // f32 += e2m1 (library) x e2m1 (queries, test terms), K-major
    const u32 idesc = (1u << 7) | (1u << 10) | ((u32)(N >> 3) << 17) | (1u << 23) | ((u32)(MM_M >> 4) << 24);
    const u64 db0 = mm_desc(smem_u32(sB), N / 8 * 128, 128);
    const u64 da0 = mm_desc(smem_u32(sA), MM_M / 8 * 128, 128);
    // K = 64 elements = 32 bytes = two core matrices per MMA
    constexpr u64 DA_K = 2 * (MM_M / 8 * 128) / 16, DB_K = 2 * (N / 8 * 128) / 16, DA_S = MM4X_TILE / 16;
    const u32 sfa = tmem + MM4_SF_COL, sfb = tmem + MM4_SF_COL + 16;
    for (u64 it = 0; it < ntile; ++it) {
      const int s = (int)(it % MM4X_STAGES), b = (int)(it % NACC);
      MM4_TRACE(0);
      if (it >= NACC) mm_bar_wait_spin(&tempty[b], (u32)((it / NACC) - 1) & 1u);
      mm_bar_wait_spin(&full_bar[s], (u32)(it / MM4X_STAGES) & 1u);
      MM4_TRACE(1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (mm_elect_one()) {
        const u64 das = da0 + (u64)s * DA_S;
        const u32 dt = tmem + (u32)b * N;
        if (!(a.flags & (1u << 23))) {  // (experiment: no MMAs, timing only)
#pragma unroll
          for (int ks = 0; ks < 3; ++ks) mm4_mma(dt, das + ks * DA_K, db0 + ks * DB_K, idesc, ks > 0, sfa, sfb);
        }
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
    for (int c = warp; c < N; c += MM4X_THREADS / 32) {
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
  if (warp == MM4X_EPI) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

}  // namespace fps
