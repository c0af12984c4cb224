// fps_bitslice.cuh — bit-sliced multi-query scan (configs 4 and 5).
//
// The per-comparison POPC formulation is XU-pipe bound (16 POPC/clk/SM on
// B200, 4-6 POPC per comparison). Here the library is transposed once into
// bit-plane tiles: for a block of 32 entries, plane p is one u32 whose bit e
// is key p+1 of entry e. A lane then evaluates one query against 32 entries
// at once with LOP3 only:
//   c   = |a AND q| = sum over the query's set keys of plane p   (carry-save
//         counter, ~2.6 LOP3 per set key, a few LDS),
//   d   = |a| + |q| - 2c                                         (|a| planes
//         are stored with the tile),
//   d < T  <=>  |a| - 2c - (T - |q|) < 0                         (bit-sliced
//         10-bit two's-complement ripple, sign plane = pass mask).
// Dense queries (|q| > 83) count over their zero keys instead:
//   d = |q| - |a| + 2 |a AND NOT q|.
// Roughly 150 LOP3/LDS per 32 x 32 = 1024 comparisons per warp instruction
// stream, versus ~4.5 k instructions (4 k POPC-pipe slots) for the POPC scan.
//
// Tiles of 2048 entries (64 blocks, 44.5 KB) are streamed into shared memory
// with the Blackwell bulk-copy engine (cp.async.bulk + mbarrier, double
// buffered); the 16 warps of a CTA (one CTA per SM) share each tile and split
// the CTA's 64 queries. A lane owns two consecutive blocks: one 64-bit shared
// load fetches a plane word of both, so the plane-address arithmetic and the
// loads are amortised over 64 entries and the two carry-save chains
// interleave (C4: 46.0 -> 33.7 ms against one block per lane).
// Results go through the same per-(warp, query) ordered candidate buffers,
// exact tie rule and select_kernel as the POPC scan (fps_kernels.cuh).
#pragma once
#include "fps_kernels.cuh"

namespace fps {

constexpr int BS_PLANES = 174;               // 166 key planes + 8 popcount planes
constexpr int BS_ZERO = 174;                 // index of an all-zero plane (padding)
#ifndef FPS_BS_BPL
#define FPS_BS_BPL 2
#endif
constexpr int BS_BPL = FPS_BS_BPL;           // 32-entry blocks per lane (one LDS.64 reads a plane of both)
static_assert(BS_BPL == 2, "the scan reads both blocks of a lane with one 64-bit shared load");
constexpr int BS_BLOCKS = 32 * BS_BPL;       // blocks per tile
constexpr int BS_TILE_ENTRIES = 32 * BS_BLOCKS;
constexpr int BS_TILE_WORDS = BS_PLANES * BS_BLOCKS;
constexpr u32 BS_TILE_BYTES = BS_TILE_WORDS * 4;  // 44,544 B at 2 blocks per lane
constexpr u32 BS_PLANE_BYTES = BS_BLOCKS * 4;
constexpr int BS_LIST = 88;                  // max plane indices per query (83 rounded to 8)
#ifndef FPS_BS_QPW
#define FPS_BS_QPW 4
#endif
#ifndef FPS_BS_MINB
#define FPS_BS_MINB 1
#endif
constexpr int BS_QPW = FPS_BS_QPW;           // queries per warp (the maximum; small batches use 1 or 2)
#ifndef FPS_BS_WARPS
#define FPS_BS_WARPS 16
#endif
constexpr int BS_WARPS = FPS_BS_WARPS;
constexpr int BS_QPC = BS_QPW * BS_WARPS;    // queries per CTA

// ---------------------------------------------------------------------------
// one-time transpose: tiled u64 library -> bit-plane tiles
// ---------------------------------------------------------------------------
// One warp per 32-entry block: lane e holds entry e, plane p = ballot(bit p).
__global__ void bs_build_kernel(PlanesOut lib, u64 n, u32* __restrict__ bs, u32* wide) {
  const int lane = threadIdx.x & 31;
  const u64 nblocks = (n + 31) / 32;
  for (u64 blk = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; blk < nblocks;
       blk += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 i = blk * 32 + lane;
    u64 w[3] = {0, 0, 0};
    if (i < n) lib.get(i, w[0], w[1], w[2]);
    // bits past key 166 (FPS1 pad bytes) are not represented in the planes:
    // such libraries keep using the POPC scan, which counts them like the reference
    if (w[2] >> 38) atomicAdd(wide, 1u);
    u32* tile = bs + (blk / BS_BLOCKS) * BS_TILE_WORDS;
    const u32 b = (u32)(blk % BS_BLOCKS);
#pragma unroll 2
    for (int p = 0; p < 166; ++p) {
      const u32 m = __ballot_sync(FULL, (w[p >> 6] >> (p & 63)) & 1);
      if (lane == 0) tile[p * BS_BLOCKS + b] = m;
    }
    const u32 pc = (u32)(__popcll(w[0]) + __popcll(w[1]) + __popcll(w[2] & ((1ull << 38) - 1)));
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const u32 m = __ballot_sync(FULL, (pc >> k) & 1);
      if (lane == 0) tile[(166 + k) * BS_BLOCKS + b] = m;
    }
  }
}

// Per query: popcount, dense flag and the padded list of planes to count.
struct BsQuery {
  u32 pop;     // |q|
  u32 dense;   // 1: list = zero keys (count |a AND NOT q|)
  u32 len;     // list length, multiple of 8
  u32 pad;
  u32 list[BS_LIST];  // byte offsets (plane * BS_PLANE_BYTES) of the planes to count, padded with the zero plane
};

__global__ void bs_prep_queries(const u64* __restrict__ q, u32 Q, BsQuery* __restrict__ out) {
  const u32 qi = blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= Q) return;
  const u64 w0 = q[3 * (u64)qi], w1 = q[3 * (u64)qi + 1], w2 = q[3 * (u64)qi + 2];
  const u32 pop = (u32)(__popcll(w0) + __popcll(w1) + __popcll(w2));
  BsQuery r;
  r.pop = pop;
  r.dense = pop > 83 ? 1u : 0u;
  u32 len = 0;
  for (int p = 0; p < 166; ++p) {
    const u32 bit = (u32)(((p < 64 ? w0 : p < 128 ? w1 : w2) >> (p & 63)) & 1);
    if (bit != r.dense) r.list[len++] = (u32)p * BS_PLANE_BYTES;
  }
  while (len % 8) r.list[len++] = (u32)BS_ZERO * BS_PLANE_BYTES;
  for (u32 i = len; i < BS_LIST; ++i) r.list[i] = (u32)BS_ZERO * BS_PLANE_BYTES;
  r.len = len;
  r.pad = 0;
  out[qi] = r;
}

// tg[q] (every replica) = the k-th distance of the seed pass: an exact upper
// bound of the full library's k-th distance (the seed entries are in it).
__global__ void bs_seed_tg(const u64* __restrict__ keys, const u32* __restrict__ cnt, u32 Q, u32 k, u32* tg,
                           u32 tg_rep, u32 gstride) {
  const u32 q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  const u32 t = cnt[q] >= k ? key_d(keys[(u64)q * k + k - 1]) : T_OPEN;
  for (u32 r = 0; r < tg_rep; ++r) tg[((u64)q * tg_rep + r) * gstride] = t;
}

struct BsArgs {
  const u32* bs;        // bit-plane tiles
  u64 n;                // valid entries
  u64 index_base;
  const BsQuery* qs;    // [Q]
  const unsigned char* radius;  // RANGE
  u32 Q, k, cap;
  u32 n_qg;             // query groups of BS_QPC
  u64 n_parts;          // library parts (CTAs per query group)
  u64 tiles;            // ceil(n / 1024)
  u32* tg;
  u32 tg_rep, gstride;
  u64* buf;             // [warps][BS_QPW][cap]
  u64* cand;
  u32* cand_cnt;
  u64 cand_cap;
  u64* out;             // RANGE keys
  u64* out_cnt;
  u64 out_cap;
};

// ripple add of a bit-sliced value and a uniform constant: returns the sign
// plane (bit 9) of x + w over 10 bits
__device__ __forceinline__ u32 bs_sign_after_add(const u32 (&x)[10], u32 w) {
  u32 cy = 0, s9 = 0;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const u32 wm = ((w >> i) & 1u) ? FULL : 0u;
    if (i == 9) s9 = x[i] ^ wm ^ cy;
    cy = (x[i] & wm) | (cy & (x[i] ^ wm));
  }
  return s9;
}

// Sign plane of (P - N) + w over 10 bits: (P, N) = (2c, |a|) if DENSE else
// (|a|, 2c); bit e set <=> entry e passes d < T (see the header).
// Same with the constant's bit masks (0 or ~0 per bit) precomputed in shared memory.
__device__ __forceinline__ u32 bs_sign_after_add_m(const u32 (&x)[10], const u32* wm) {
  u32 cy = 0, s9 = 0;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const u32 w = wm[i];
    if (i == 9) s9 = x[i] ^ w ^ cy;
    cy = (x[i] & w) | (cy & (x[i] ^ w));
  }
  return s9;
}

template <bool DENSE>
__device__ __forceinline__ u32 bs_pass_mask(const u32 (&A)[8], const u32 (&C)[8], const u32* wm) {
  u32 X[10];
  u32 cy = FULL;  // +1 of the two's complement of N
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const u32 p = i < 8 ? (DENSE ? C[i] : A[i]) : 0u;
    const u32 nn = ~(i < 8 ? (DENSE ? A[i] : C[i]) : 0u);
    X[i] = p ^ nn ^ cy;
    cy = (p & nn) | (cy & (p ^ nn));
  }
  return bs_sign_after_add_m(X, wm);
}

template <int MODE, int QPW>
__global__ void __launch_bounds__(BS_WARPS * 32, FPS_BS_MINB) bs_scan_kernel(const BsArgs a) {
  constexpr int QPC = QPW * BS_WARPS;  // queries per CTA
  extern __shared__ __align__(128) unsigned char bsm[];
  u32* tiles = reinterpret_cast<u32*>(bsm);  // 2 x (BS_TILE_WORDS + a zero plane)
  u64* bars = reinterpret_cast<u64*>(bsm + 2 * (BS_TILE_BYTES + BS_PLANE_BYTES));  // 2 mbarriers
  BsQuery* sq = reinterpret_cast<BsQuery*>(bars + 2);                 // [QPC]
  u32* hist_all = reinterpret_cast<u32*>(sq + QPC);               // [BS_WARPS][QPW][HB] (TOPK)
  WarpState<QPW>* ws_all = reinterpret_cast<WarpState<QPW>*>(hist_all + BS_WARPS * QPW * HB);
  // per (warp, slot): bit masks of (|q| - T) mod 2^10, refreshed whenever T changes
  u32* wmask_all = reinterpret_cast<u32*>(ws_all + BS_WARPS);

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 qg = blockIdx.x % a.n_qg;
  const u64 part = blockIdx.x / a.n_qg;
  const u64 t0 = part * a.tiles / a.n_parts, t1 = (part + 1) * a.tiles / a.n_parts;
  const u64 g = (u64)blockIdx.x * BS_WARPS + wid;  // global warp id (buffers)

  // queries of this CTA
  for (int i = threadIdx.x; i < QPC; i += blockDim.x) {
    const u32 qi = qg * QPC + i;
    if (qi < a.Q) sq[i] = a.qs[qi];
    else { sq[i].pop = 0; sq[i].dense = 0; sq[i].len = 0; }
  }
  for (int b = 0; b < 2; ++b)
    for (int i = threadIdx.x; i < BS_BLOCKS; i += blockDim.x) tiles[b * (BS_TILE_WORDS + BS_BLOCKS) + BS_TILE_WORDS + i] = 0;
  u32* hist = hist_all + wid * QPW * HB;
  WarpState<QPW>* ws = ws_all + wid;
  if (MODE == MODE_TOPK) {
    for (int i = lane; i < QPW * HB; i += 32) hist[i] = 0;
    if (lane < QPW) { ws->town[lane] = T_OPEN; ws->pubd[lane] = 0; ws->cnt[lane] = 0; }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // per-slot thresholds (accept d < T)
  u32 T[QPW];
#pragma unroll
  for (int j = 0; j < QPW; ++j) {
    const u32 qi = qg * QPC + wid * QPW + j;
    if (qi >= a.Q) T[j] = 0;
    else if (MODE == MODE_RANGE) T[j] = (u32)a.radius[qi] + 1;
    else {
      const u32 t = *(volatile const u32*)(a.tg + ((u64)qi * a.tg_rep) * a.gstride);
      T[j] = (t < T_OPEN ? t : T_OPEN - 1) + 1;
    }
  }
  u64* wbuf = (MODE == MODE_TOPK) ? a.buf + g * QPW * (u64)a.cap : nullptr;
  u32* wmask = wmask_all + wid * QPW * 10;
  auto set_wmask = [&](int j, u32 Tj) {
    const u32 w = (u32)((int)sq[wid * QPW + j].pop - (int)Tj) & 0x3ffu;
    if (lane < 10) wmask[j * 10 + lane] = ((w >> lane) & 1u) ? FULL : 0u;
    __syncwarp();
  };
#pragma unroll
  for (int j = 0; j < QPW; ++j) set_wmask(j, T[j]);

  auto issue = [&](u64 t, int b) {
    mbar_expect_tx(&bars[b], BS_TILE_BYTES);
    bulk_g2s(tiles + b * (BS_TILE_WORDS + BS_BLOCKS), a.bs + t * BS_TILE_WORDS, BS_TILE_BYTES, &bars[b]);
  };
  if (threadIdx.x == 0) {
    if (t0 < t1) issue(t0, 0);
    if (t0 + 1 < t1) issue(t0 + 1, 1);
  }

  u32 phase[2] = {0, 0};
  for (u64 t = t0; t < t1; ++t) {
    const int b = (int)((t - t0) & 1);
    mbar_wait(&bars[b], phase[b]);
    phase[b] ^= 1;
    const u32* tile = tiles + b * (BS_TILE_WORDS + BS_BLOCKS);
    // popcount planes of this lane's blocks (shared by every query)
    u32 A[BS_BPL][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint2 v = *reinterpret_cast<const uint2*>(tile + (166 + i) * BS_BLOCKS + lane * BS_BPL);
      A[0][i] = v.x;
      A[1][i] = v.y;
    }
    const u64 blk_first = t * BS_TILE_ENTRIES + (u64)lane * 32 * BS_BPL;  // local index of this lane's bit 0
    // entries past n (last tile) never pass: mask them out
    u32 valid[BS_BPL];
#pragma unroll
    for (int h = 0; h < BS_BPL; ++h) {
      const u64 f = blk_first + 32 * h;
      valid[h] = f >= a.n ? 0u : (a.n - f >= 32 ? FULL : ((1u << (a.n - f)) - 1u));
    }

#pragma unroll 1
    for (int j = 0; j < QPW; ++j) {
      u32 Tj = 0;
#pragma unroll
      for (int jj = 0; jj < QPW; ++jj)
        if (jj == j) Tj = T[jj];
      if (Tj == 0) continue;  // padding slot or nothing can pass
      const BsQuery& qq = sq[wid * QPW + j];
      // carry-save count of the listed planes for both blocks: ones..s64 =
      // binary digits (two independent chains per lane)
      u32 ones[BS_BPL], twos[BS_BPL], fours[BS_BPL], eights[BS_BPL], s16[BS_BPL], s32[BS_BPL], s64[BS_BPL];
#pragma unroll
      for (int h = 0; h < BS_BPL; ++h) ones[h] = twos[h] = fours[h] = eights[h] = s16[h] = s32[h] = s64[h] = 0;
      const char* lane_base = reinterpret_cast<const char*>(tile) + 4 * BS_BPL * lane;
#define CSA(h, l, x, y)              \
  do {                               \
    const u32 u_ = l ^ x;            \
    h = (l & x) | (u_ & y);          \
    l = u_ ^ y;                      \
  } while (0)
      // 8 listed planes of both blocks -> the eights-weight carry of each
      // block (ones/twos/fours absorb the rest)
      auto load8 = [&](u32 c, u32 (&d)[BS_BPL][8]) {
        const uint4 o0 = *reinterpret_cast<const uint4*>(qq.list + c);
        const uint4 o1 = *reinterpret_cast<const uint4*>(qq.list + c + 4);
        const u32 off[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint2 v = *reinterpret_cast<const uint2*>(lane_base + off[i]);
          d[0][i] = v.x;
          d[1][i] = v.y;
        }
      };
      auto tree8 = [&](const u32 (&d)[BS_BPL][8], u32 (&e8)[BS_BPL]) {
#pragma unroll
        for (int h = 0; h < BS_BPL; ++h) {
          u32 twosA, twosB, foursA, foursB;
          CSA(twosA, ones[h], d[h][0], d[h][1]);
          CSA(twosB, ones[h], d[h][2], d[h][3]);
          CSA(foursA, twos[h], twosA, twosB);
          CSA(twosA, ones[h], d[h][4], d[h][5]);
          CSA(twosB, ones[h], d[h][6], d[h][7]);
          CSA(foursB, twos[h], twosA, twosB);
          CSA(e8[h], fours[h], foursA, foursB);
        }
      };
      u32 c0 = 0;
      // 16 planes per step: two 8-plane trees and one more carry-save adder
      // at weight 8 (35 LOP3 per 16 planes instead of 42)
      for (; c0 + 16 <= qq.len; c0 += 16) {
        u32 d[BS_BPL][8], e8a[BS_BPL], e8b[BS_BPL];
        load8(c0, d);
        tree8(d, e8a);
        load8(c0 + 8, d);
        tree8(d, e8b);
#pragma unroll
        for (int h = 0; h < BS_BPL; ++h) {
          u32 e16;
          CSA(e16, eights[h], e8a[h], e8b[h]);
          const u32 c2 = s16[h] & e16;
          s16[h] ^= e16;
          const u32 c3 = s32[h] & c2;
          s32[h] ^= c2;
          s64[h] ^= c3;
        }
      }
      if (c0 < qq.len) {  // a last group of 8 (lists are padded to multiples of 8)
        u32 d[BS_BPL][8], e8[BS_BPL];
        load8(c0, d);
        tree8(d, e8);
#pragma unroll
        for (int h = 0; h < BS_BPL; ++h) {
          const u32 c1 = eights[h] & e8[h];
          eights[h] ^= e8[h];
          const u32 c2 = s16[h] & c1;
          s16[h] ^= c1;
          const u32 c3 = s32[h] & c2;
          s32[h] ^= c2;
          s64[h] ^= c3;
        }
      }
#undef CSA
      // pass mask: sign of X + (|q| - T), X = |a| - 2c (sparse) or 2c - |a|
      // (dense); a warp-uniform branch picks the operand order (no selects)
      const u32* wm = wmask + j * 10;
      u32 m[BS_BPL];
#pragma unroll
      for (int h = 0; h < BS_BPL; ++h) {
        const u32 C[8] = {0, ones[h], twos[h], fours[h], eights[h], s16[h], s32[h], s64[h]};  // 2c
        m[h] = (qq.dense ? bs_pass_mask<true>(A[h], C, wm) : bs_pass_mask<false>(A[h], C, wm)) & valid[h];
      }
      if (!__any_sync(FULL, m[0] | m[1])) continue;

      // ---- slow path: exact distances of the passing entries, in index order
      // (bit e of mm = entry blk_first + e; the lane's blocks are consecutive)
      const u64 mm = (u64)m[0] | ((u64)m[1] << 32);
      const u32 qi = qg * QPC + wid * QPW + j;
      const u32 cntl = (u32)__popcll(mm);
      const u32 incl = warp_incl_scan(cntl, lane);
      const u32 total = __shfl_sync(FULL, incl, 31);
      auto dist_of_bit = [&](int e) -> u32 {
        const int h = e >> 5, bit = e & 31;
        u32 av = 0, cv = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) av |= (((h ? A[1][i] : A[0][i]) >> bit) & 1u) << i;
        const u32 cb[7] = {h ? ones[1] : ones[0], h ? twos[1] : twos[0], h ? fours[1] : fours[0],
                           h ? eights[1] : eights[0], h ? s16[1] : s16[0], h ? s32[1] : s32[0],
                           h ? s64[1] : s64[0]};
#pragma unroll
        for (int i = 0; i < 7; ++i) cv |= ((cb[i] >> bit) & 1u) << i;
        return qq.dense ? qq.pop - av + 2 * cv : av + qq.pop - 2 * cv;
      };
      if (MODE == MODE_RANGE) {
        u64 base = 0;
        if (lane == 31) base = atomicAdd(a.out_cnt, (u64)total);
        base = __shfl_sync(FULL, base, 31);
        u64 pos = base + incl - cntl;
        for (u64 rest = mm; rest; rest &= rest - 1) {
          const int e = __ffsll((long long)rest) - 1;
          if (pos < a.out_cap)
            a.out[pos] = ((u64)qi << 48) | make_key(dist_of_bit(e), a.index_base + blk_first + e);
          ++pos;
        }
        continue;
      }
      // MODE_TOPK: the per-(warp, query) buffer of fps_kernels.cuh
      u32* hj = hist + j * HB;
      u64* bj = wbuf + (u64)j * a.cap;
      if (ws->cnt[j] + total > a.cap) {
        // ordered compaction to the k best (entries are in index order)
        const u32 n0 = ws->cnt[j];
        u32 less;
        const u32 tt = warp_kth_bin(hj, a.k, lane, &less);
        const u32 mk = a.k - less;
        u32 outp = 0, ties = 0;
        for (u32 i0 = 0; i0 < n0; i0 += 32) {
          const u32 i = i0 + lane;
          const bool vld = i < n0;
          const u64 key = vld ? bj[i] : ~0ull;
          const u32 d = key_d(key);
          const bool lt = vld && d < tt, tie = vld && d == tt;
          const u32 tb = __ballot_sync(FULL, tie);
          const bool keep = lt || (tie && ties + __popc(tb & lanemask_lt()) < mk);
          const u32 kb = __ballot_sync(FULL, keep);
          const u32 pp = outp + __popc(kb & lanemask_lt());
          __syncwarp();
          if (keep) bj[pp] = key;
          outp += __popc(kb);
          ties += __popc(tb);
        }
        for (u32 bb = lane; bb < HB; bb += 32) {
          if (bb > tt) hj[bb] = 0;
          else if (bb == tt) hj[bb] = mk;
        }
        if (lane == 0) ws->cnt[j] = outp;
        __syncwarp();
      }
      const u32 cnt0 = ws->cnt[j];
      u32 pos = cnt0 + incl - cntl;
#ifdef FPS_BS_DEBUG
      if (cnt0 + total > a.cap) { printf("BS overflow cnt0 %u total %u cap %u\n", cnt0, total, a.cap); __trap(); }
#endif
      for (u64 rest = mm; rest; rest &= rest - 1) {
        const int e = __ffsll((long long)rest) - 1;
        const u32 d = dist_of_bit(e);
#ifdef FPS_BS_DEBUG
        if (d >= HB || d >= Tj) { printf("BS bad d %u T %u pop %u dense %u lane %d e %d\n", d, Tj, qq.pop, qq.dense, lane, e); __trap(); }
#endif
        bj[pos++] = make_key(d, a.index_base + blk_first + e);
        atomicAdd(hj + d, 1u);
      }
      __syncwarp();
      if (lane == 0) ws->cnt[j] = cnt0 + total;
      __syncwarp();
      if (cnt0 + total >= a.k) {
        u32 less;
        const u32 tt = warp_kth_bin(hj, a.k, lane, &less);
        const u32 nt = tt < Tj ? tt : Tj;
#pragma unroll
        for (int jj = 0; jj < QPW; ++jj)
          if (jj == j) T[jj] = nt;
        set_wmask(j, nt);
        if (lane == 0) ws->town[j] = tt;
        __syncwarp();
      }
    }
    __syncthreads();  // every warp is done with buffer b
    if (threadIdx.x == 0 && t + 2 < t1) issue(t + 2, b);
  }

  if (MODE == MODE_TOPK) {
#pragma unroll 1
    for (int j = 0; j < QPW; ++j) {
      const u32 qi = qg * QPC + wid * QPW + j;
      if (qi >= a.Q) continue;
      u32* hj = hist + j * HB;
      u64* bj = wbuf + (u64)j * a.cap;
      u32 n0 = ws->cnt[j];
      if (n0 > a.k) {
        u32 less;
        const u32 tt = warp_kth_bin(hj, a.k, lane, &less);
        const u32 mk = a.k - less;
        u32 outp = 0, ties = 0;
        for (u32 i0 = 0; i0 < n0; i0 += 32) {
          const u32 i = i0 + lane;
          const bool vld = i < n0;
          const u64 key = vld ? bj[i] : ~0ull;
          const u32 d = key_d(key);
          const bool lt = vld && d < tt, tie = vld && d == tt;
          const u32 tb = __ballot_sync(FULL, tie);
          const bool keep = lt || (tie && ties + __popc(tb & lanemask_lt()) < mk);
          const u32 kb = __ballot_sync(FULL, keep);
          const u32 pp = outp + __popc(kb & lanemask_lt());
          __syncwarp();
          if (keep) bj[pp] = key;
          outp += __popc(kb);
          ties += __popc(tb);
        }
        n0 = outp;
        __syncwarp();
      }
      const u32 bound = *(volatile const u32*)(a.tg + ((u64)qi * a.tg_rep) * a.gstride);
      for (u32 i0 = 0; i0 < n0; i0 += 32) {
        const u32 i = i0 + lane;
        const u64 key = i < n0 ? bj[i] : ~0ull;
        const bool keep = i < n0 && key_d(key) <= bound;
        const u32 kb = __ballot_sync(FULL, keep);
        const u32 nk = __popc(kb);
        if (nk == 0) continue;
        u32 base = 0;
        if (lane == 0) base = atomicAdd(a.cand_cnt + qi, nk);
        base = __shfl_sync(FULL, base, 0);
#ifdef FPS_BS_DEBUG
        if (base + nk > a.cand_cap) { printf("BS cand overflow %u %u %llu\n", base, nk, a.cand_cap); __trap(); }
#endif
        if (keep) a.cand[(u64)qi * a.cand_cap + base + __popc(kb & lanemask_lt())] = key;
      }
    }
  }
}

}  // namespace fps
