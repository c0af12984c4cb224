// fps_planeq.cuh — single-query scan that reads only the bit planes the query
// needs (configs 1-3, the HBM-bound path).
//
// The distance contract is the reference's (scan.py:137-143): d = sum over the
// three words of popcount(entry XOR query). With the library stored as bit
// planes (plane p of a 32-entry block = one u32 whose bit e is key p+1 of
// entry e; planes 166..173 = the entry's popcount |a|, bit by bit):
//   d = |a| + |q| - 2 |a AND q|          (c counted over the query's set keys)
//   d = |q| - |a| + 2 |a AND NOT q|      (dense queries, |q| > 83: zero keys)
// so one query needs only its m = min(|q|, 166 - |q|) listed planes plus the
// 8 popcount planes: (8 + m) / 8 bytes per entry instead of 21-24 B for the
// whole fingerprint. MACCS-like queries (|q| ~ 38 keys) read 5.75 B/entry —
// the HBM stream, which bounds the single-query scan, shrinks ~3.7x.
//
// Layout (plane-major): plane p occupies pstride u32 words from pm + p *
// pstride; word w is 32-entry block w. A warp step covers 1,024 x BPL entries
// (a lane owns BPL consecutive blocks; BPL = 2 reads both with one 64-bit
// shared load, as in fps_bitslice.cuh), i.e. 128 x BPL bytes of every listed
// plane. The host picks the shape per query (topk_pq in fps_capi.cu): BPL = 1
// with as many warps (<= 16) as hold two stages of the query's plane list on
// libraries with at least two steps per warp, 6 warps x BPL = 2 on shorter
// ones; a list wider than the ring was sized for (a device-resident query of
// unknown width) keeps as many warps active as the ring memory allows.
//
// Per warp, a ring of S stages in shared memory: position 0..7 = popcount
// planes, 8.. = the query's list (zero-padded to a multiple of 8). COPY 1
// (default) fills a stage with cp.async, 16 B per lane and 512 B per warp
// instruction, completing on the stage's mbarrier (arrive.noinc per lane);
// COPY 0 issues one cp.async.bulk per plane chunk (TMA engine), which tops out
// at ~15 B/clk/SM with 256 B copies. The count c runs through the carry-save
// adder tree of the multi-query kernel; the pass mask is the sign plane of
// X + (|q| - T) with X = |a| - 2c (or 2c - |a|).
//
// Selection is the single-query POPC scan's (fps_kernels.cuh): per-warp
// ordered candidate buffer with its distance histogram and the exact tie
// rule, sampled warps publishing witnesses into ghist, the global bound tg,
// survivors d <= tg to the flat list, then select_kernel. A warp's first step
// has no bound yet: it computes the step's distances bit-sliced, finds the
// k-th smallest by radix select (no per-entry work), publishes witnesses at a
// few ranks, and holds its entries back one step so they are inserted under
// the tighter global bound the first wave of witnesses produces: before its
// second step's test a warp takes the bound of the whole first wave (one
// warp per CTA polls the global histogram, the others read shared memory).
#pragma once
#include "fps_bitslice.cuh"

namespace fps {

// A warp step covers 1,024 x BPL entries: BPL consecutive 32-entry blocks per
// lane, i.e. 32 x BPL u32 words = 128 x BPL bytes of every listed plane.
template <int BPL> struct PqStep {
  static constexpr u32 WORDS = 32 * BPL;       // u32 words of one plane per step
  static constexpr u32 CHUNK = WORDS * 4;      // bytes of one plane per step
  static constexpr u64 ENTRIES = 32ull * WORDS;
};
constexpr u32 PQ_STRIDE_WORDS = 64;             // plane stride granule (whole steps at BPL <= 2)
constexpr int PQ_NPMAX = 8 + BS_LIST;           // stage positions: popcount planes + padded list
constexpr int PQ_SMAX = 4;                      // ring stages per warp (at most)
constexpr u64 PQ_NONE = ~0ull;

// Plane-major copy of the library: one warp per 32-entry block, plane p =
// ballot of key p+1; lane (p mod 32) stores it. Libraries with bits past key
// 166 (FPS1 pad bytes) are flagged in *wide and keep the POPC scan. With
// `order` (popcount-sorted keys |a| << 32 | index) position j holds entry
// order[j] and perm[j] records its index.
__global__ void pm_build_kernel(PlanesOut lib, u64 n, u32* __restrict__ pm, u64 pstride, u32* wide,
                                const u64* __restrict__ order, u32* __restrict__ perm) {
  const int lane = threadIdx.x & 31;
  const u64 nblocks = (n + 31) / 32;
  for (u64 blk = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; blk < nblocks;
       blk += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 j = blk * 32 + lane;
    u64 w[3] = {0, 0, 0};
    if (j < n) {
      const u64 i = order ? (order[j] & 0xffffffffull) : j;
      if (order) perm[j] = (u32)i;
      lib.get(i, w[0], w[1], w[2]);
    }
    if (w[2] >> 38) atomicAdd(wide, 1u);
    u32 mine[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int p = 0; p < 166; ++p) {
      const u32 m = __ballot_sync(FULL, (u32)(w[p >> 6] >> (p & 63)) & 1u);
      if ((p & 31) == lane) mine[p >> 5] = m;
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const int p = c * 32 + lane;
      if (p < 166) pm[(u64)p * pstride + blk] = mine[c];
    }
    const u32 pc = (u32)(__popcll(w[0]) + __popcll(w[1]) + __popcll(w[2] & ((1ull << 38) - 1)));
    u32 pcm = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const u32 m = __ballot_sync(FULL, (pc >> b) & 1u);
      if (lane == b) pcm = m;
    }
    if (lane < 8) pm[(u64)(166 + lane) * pstride + blk] = pcm;
  }
}

// Sort keys of the popcount-sorted copy: |a| << 32 | index (index < 2^32 on a device).
__global__ void pm_sort_keys_kernel(PlanesOut lib, u64 n, u64* __restrict__ keys) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 w0, w1, w2;
    lib.get(i, w0, w1, w2);
    const u64 pc = (u64)(__popcll(w0) + __popcll(w1) + __popcll(w2 & ((1ull << 38) - 1)));
    keys[i] = (pc << 32) | i;
  }
}

// Popcount range of every 1,024 sorted entries: min | max << 8.
__global__ void pm_meta_kernel(const u64* __restrict__ sorted, u64 n, unsigned short* __restrict__ meta) {
  const u64 nb = (n + 1023) / 1024;
  for (u64 b = (u64)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (u64)gridDim.x * blockDim.x) {
    const u64 f = b * 1024, l = (f + 1023 < n ? f + 1023 : n - 1);
    meta[b] = (unsigned short)((sorted[f] >> 32) | ((sorted[l] >> 32) << 8));
  }
}

struct PqArgs {
  const u32* pm;        // plane-major planes (174 x pstride words)
  u64 pstride;          // words per plane (>= 64 * n_steps; padding words are zero)
  u64 n;                // valid entries
  u64 index_base;
  const u64* queries;   // the query (3 words) on the device; nullptr: inline in qin
  u64 qin[3];
  u32 k, cap;           // top-k, per-warp buffer capacity (>= k + PQ_STEP)
  u64 n_steps;          // ceil(n / PQ_STEP)
  u32 ring_bytes;       // shared-memory ring per warp (before warps are folded, see below)
  u32 pub_every;        // warps with g % pub_every == 0 publish witnesses
  u32 flags;            // FPS_SCAN_FLAGS: 1 = no publishing, 2 = no tg refresh
  u32 refresh;          // steps between reads of the global bound (1 = every step)
  u32 wave_pct;         // first wave: a warp's second step waits for the witnesses of this share of the
                        // active warps with a full first step (0: no wave)
  u64 wave_steps;       // full steps of the library (warps with one post k witnesses each)
  u32 wave_wait_ns;     // ... for at most this long
  u32* tg;
  u32* ghist;
  u32 gstride, tg_rep;
  u64* buf;             // [warps][cap]
  u64* cand;            // [cand_cap] survivors of the query
  u32* cand_cnt;
  u64 cand_cap;
  // popcount-sorted copy (SORTED kernels): sorted position -> local index, and
  // per 1,024 sorted entries the popcount range (min | max << 8)
  const u32* perm;
  const unsigned short* meta;
  u32 meta_cap;         // steps of a CTA's run the shared-memory copy of meta holds
};

// Dynamic shared memory: [warps][ring_bytes] ring | [warps][PQ_SMAX] mbarriers
// | [warps][PQ_SMAX] slot steps | [warps][HB] histograms | [warps] WarpState
// | [warps][32] u64 tie scratch | [meta_cap] u16 popcount ranges (SORTED).
__host__ __device__ inline size_t pq_smem(int nwb, u32 ring_bytes, u32 meta_cap = 0) {
  return (size_t)nwb * ring_bytes + (size_t)nwb * PQ_SMAX * 16 + (size_t)nwb * HB * 4 +
         ((size_t)nwb * sizeof(WarpState<1>) + 15) / 16 * 16 + (size_t)nwb * 32 * 8 + (size_t)meta_cap * 2;
}

// COPY 0: per-plane 256 B cp.async.bulk (TMA engine); 1: 16 B cp.async
// (LDGSTS) per lane, two planes per warp instruction, completion through
// cp.async.mbarrier.arrive.noinc on the same stage barriers.
#ifdef FPS_SCAN_TRACE
__device__ u64 g_pq_pro[16384 * 4];    // per warp, prologue: list built, ring initialised, requests issued, dependency wait over
__device__ u64 g_pq_s1[16384 * 4];     // per warp, second step: bound taken, held-back entries inserted, CSA done
__device__ u64 g_pq_steps[16384 * 8];  // per warp: tile-ready time of its first 8 steps
__device__ u64 g_pq_phase[16384 * 8];  // per warp, first step: CSA done, refill issued, bound, mask, inserted, published
#endif
// SORTED: the plane copy is ordered by popcount |a| (then index). A step whose
// entries share one |a| (all but ~one per popcount value) skips the popcount
// planes (|a| is a constant), steps whose |a| range cannot reach the bound
// (d >= ||a| - |q||) are not read at all, and since a warp no longer meets
// entries in index order, ties at its own k-th distance are kept and resolved
// by index (full (d, index) key order) when the buffer is compacted.
__device__ __forceinline__ u64 pq_now_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <int COPY, int BPL, bool SORTED>
__global__ void __launch_bounds__(512, 1) pq_scan_kernel(const PqArgs a) {
  static_assert(!SORTED || COPY == 1, "the sorted copy is read with cp.async");
  constexpr u32 PQ_WORDS = PqStep<BPL>::WORDS, PQ_CHUNK = PqStep<BPL>::CHUNK;
  constexpr u64 PQ_STEP = PqStep<BPL>::ENTRIES;
  constexpr u32 LPP = 8 * BPL;      // cp.async: lanes per position (16 B each)
  constexpr u32 PPI = 32 / LPP;     // positions per warp instruction (512 B)
  extern __shared__ __align__(128) unsigned char pqs[];
  // the select kernel may launch now; it waits for this grid before reading
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
#ifdef FPS_SCAN_TRACE
  u64 tr_start = gtimer(), tr_first = 0, tr_step1 = 0;
  bool ph_done = false;
  u32 tr_iter = ~0u;  // steps taken so far - 1
#endif
  __shared__ u32 s_list[PQ_NPMAX];  // source plane of each stage position (BS_ZERO: zero padding)
  __shared__ u32 s_np, s_nc, s_pop, s_dense, s_next;
  __shared__ u32 s_wave_poll, s_wave_T;  // first wave: poller election, the bound it found (| 1 << 31)
  __shared__ const u32* s_base[PQ_NPMAX];  // plane base of each copied position (COPY 1)

  // ---- the query's plane list (read-only inputs: safe before the dependency wait)
  if (wib == 0) {
    const u64 q0 = a.queries ? a.queries[0] : a.qin[0];
    const u64 q1 = a.queries ? a.queries[1] : a.qin[1];
    const u64 q2 = a.queries ? a.queries[2] : a.qin[2];
    // |q| over all 192 bits (pad bits of a query count once each; the
    // library's are zero on this path), as the POPC distance does
    const u32 pop = (u32)(__popcll(q0) + __popcll(q1) + __popcll(q2));
    const u32 dense = pop > 83 ? 1u : 0u;
    u32 base = 0;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const int p = c * 32 + lane;
      const u64 wv = c < 2 ? q0 : (c < 4 ? q1 : q2);
      const u32 bit = (u32)(wv >> (p & 63)) & 1u;
      const bool sel = p < 166 && bit != dense;
      const u32 bal = __ballot_sync(FULL, sel);
      if (sel) s_list[8 + base + __popc(bal & lanemask_lt())] = (u32)p;
      base += __popc(bal);
    }
    const u32 mpad = (base + 7) & ~7u;
    if (lane < 8) s_list[lane] = 166 + lane;
    for (u32 i = 8 + base + lane; i < 8 + mpad; i += 32) s_list[i] = BS_ZERO;
    if (lane == 0) {
      s_np = 8 + mpad;
      s_nc = 8 + base;
      s_pop = pop;
      s_dense = dense;
      s_next = 0;
      s_wave_poll = 0;
      s_wave_T = 0;
    }
  }
  __syncthreads();
  if (COPY == 1)
    for (u32 i = threadIdx.x; i < s_nc; i += blockDim.x) s_base[i] = a.pm + (u64)s_list[i] * a.pstride;
  // CTA-dynamic schedule: the CTA owns a contiguous run of steps; its warps
  // claim them one at a time (each warp sees ascending steps: the ordered
  // buffers rely on it) so warps that draw more bandwidth take more.
  const u64 cta_lo = (u64)blockIdx.x * a.n_steps / gridDim.x;
  const u64 cta_hi = ((u64)blockIdx.x + 1) * a.n_steps / gridDim.x;
  unsigned short* s_meta = reinterpret_cast<unsigned short*>(
      pqs + pq_smem(nwb, a.ring_bytes) );  // (meta region follows the tie scratch)
  if (SORTED) {
    // popcount range of each step of the run: BPL consecutive 1,024-entry blocks
    for (u64 i = threadIdx.x; i < cta_hi - cta_lo; i += blockDim.x) {
      u32 lo = 255, hi = 0;
#pragma unroll
      for (int h = 0; h < BPL; ++h) {
        const u64 b = (cta_lo + i) * BPL + h;
        if (b * 1024 < a.n) {
          const u32 m = a.meta[b];
          lo = min(lo, m & 0xffu);
          hi = max(hi, m >> 8);
        }
      }
      s_meta[i] = (unsigned short)(lo | (hi << 8));
    }
  }
  __syncthreads();  // the last block-level barrier
#ifdef FPS_SCAN_TRACE
  const u64 tr_p0 = gtimer();
#endif
  const u32 np = s_np, nc = s_nc, pop = s_pop;
  const bool dense = s_dense != 0;
  const u32 stage_bytes = np * PQ_CHUNK;
  // Lists wider than the ring was sized for (a device-resident query of
  // unknown width): as many warps as the CTA's ring memory gives two stages
  // stay active (16 -> 13 at 56 positions, 8 at 96), the others leave.
  const u32 total_ring = a.ring_bytes * (u32)nwb;
  u32 nact = total_ring / (2 * stage_bytes);
  nact = nact > (u32)nwb ? (u32)nwb : (nact < 1 ? 1u : nact);
  if ((u32)wib >= nact) return;
  const u32 rbytes = (total_ring / nact) / 256 * 256;
  const u32 S = min((u32)PQ_SMAX, max(1u, rbytes / stage_bytes));

  char* ring = reinterpret_cast<char*>(pqs) + (size_t)wib * rbytes;
  u64* bars = reinterpret_cast<u64*>(pqs + (size_t)nwb * a.ring_bytes) + wib * PQ_SMAX;
  u64* slot_step = reinterpret_cast<u64*>(pqs + (size_t)nwb * a.ring_bytes) + nwb * PQ_SMAX + wib * PQ_SMAX;
  u32* hist = reinterpret_cast<u32*>(reinterpret_cast<u64*>(pqs + (size_t)nwb * a.ring_bytes) + 2 * nwb * PQ_SMAX) +
              wib * HB;
  WarpState<1>* ws = reinterpret_cast<WarpState<1>*>(
                         reinterpret_cast<u32*>(reinterpret_cast<u64*>(pqs + (size_t)nwb * a.ring_bytes) +
                                                2 * nwb * PQ_SMAX) + nwb * HB) + wib;
  const u64 g = (u64)blockIdx.x * nact + wib;  // global warp id (buffers, publishing)

  // the stage barriers first: the requests go out as early as possible, the
  // rest of the per-warp state is set up while they fly
  const u32* src[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const u32 pos = lane + 32 * r;
    src[r] = pos < nc ? a.pm + (u64)s_list[pos] * a.pstride : nullptr;
  }
  if (lane == 0) {
    for (u32 st = 0; st < S; ++st) mbar_init(&bars[st], COPY == 1 ? 32u : 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

#ifdef FPS_SCAN_TRACE
  const u64 tr_p1 = gtimer();
#endif
  const u64 pol = l2_evict_first_policy();
  const u32 half = (u32)lane / LPP;  // position within a cp.async group
  u32 T = T_OPEN;  // accept d < T
  auto issue = [&](u32 st) {
    u64 t = 0;
    u32 mt = 0;
    if (lane == 0) {
      for (;;) {
        t = cta_lo + atomicAdd(&s_next, 1u);
        if (t >= cta_hi) {
          t = PQ_NONE;
          break;
        }
        if (!SORTED) break;
        // d >= ||a| - |q||: a step whose popcount range stays T away is not read
        mt = s_meta[t - cta_lo];
        const u32 lo = mt & 0xffu, hi = mt >> 8;
        const u32 lb = pop < lo ? lo - pop : (pop > hi ? pop - hi : 0u);
        if (lb < T) break;
      }
      slot_step[st] = t;
      if (COPY == 0) {
        if (t == PQ_NONE) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[st])) : "memory");
        else mbar_expect_tx(&bars[st], nc * PQ_CHUNK);
      }
    }
    t = __shfl_sync(FULL, t, 0);
    if (COPY == 1) {
      if (t != PQ_NONE) {
        // one |a| for the whole step: its popcount planes are not needed
        mt = __shfl_sync(FULL, mt, 0);
        const u32 g0 = (SORTED && (mt & 0xffu) == (mt >> 8)) ? 8 / PPI : 0u;
        // one instruction moves 512 B: lanes [LPP*j, LPP*j + LPP) copy 16 B
        // each of position PPI*i + j; source = plane base + a per-stage offset
        u32 dst = smem_u32(ring + st * stage_bytes) + half * PQ_CHUNK + (lane % LPP) * 16 + g0 * PPI * PQ_CHUNK;
        const u64 off = t * PQ_CHUNK + (lane % LPP) * 16;
        const u64* bp = reinterpret_cast<const u64*>(s_base) + half;
        const u32 ngrp = nc / PPI;
#pragma unroll 4
        for (u32 i = g0; i < ngrp; ++i) {
          const char* sp = reinterpret_cast<const char*>(bp[PPI * i]) + off;
          asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(sp), "l"(pol)
                       : "memory");
          dst += PPI * PQ_CHUNK;
        }
        if (half < nc % PPI) {
          const char* sp = reinterpret_cast<const char*>(bp[PPI * ngrp]) + off;
          asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(sp), "l"(pol)
                       : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[st])) : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[st])) : "memory");
      }
      return;
    }
    if (t == PQ_NONE) return;
    char* dst = ring + st * stage_bytes;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const u32 pos = lane + 32 * r;
      if (pos < nc) bulk_g2s_stream(dst + pos * PQ_CHUNK, src[r] + t * PQ_WORDS, PQ_CHUNK, &bars[st], pol);
    }
  };
  for (u32 st = 0; st < S; ++st) issue(st);
  // zero padding positions of every slot (never written by the copies)
  for (u32 st = 0; st < S; ++st) {
    u32* sp = reinterpret_cast<u32*>(ring + st * stage_bytes);
    for (u32 i = nc * PQ_WORDS + lane; i < np * PQ_WORDS; i += 32) sp[i] = 0;
  }
  for (int i = lane; i < HB; i += 32) hist[i] = 0;
  if (lane == 0) {
    ws->town[0] = T_OPEN;
    ws->pubd[0] = 0;
    ws->cnt[0] = 0;
  }
  __syncwarp();
#ifdef FPS_SCAN_TRACE
  const u64 tr_p2 = gtimer();
#endif
  // ---- everything below touches the per-call state the previous select resets
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef FPS_SCAN_TRACE
  if (lane == 0 && g < 16384) {
    g_pq_pro[g * 4 + 0] = tr_p0;
    g_pq_pro[g * 4 + 1] = tr_p1;
    g_pq_pro[g * 4 + 2] = tr_p2;
    g_pq_pro[g * 4 + 3] = gtimer();
  }
#endif

  u64* wbuf = a.buf + g * (u64)a.cap;
  u64* tie_scratch = reinterpret_cast<u64*>(pqs + pq_smem(nwb, a.ring_bytes) - (size_t)nwb * 32 * 8) + wib * 32;
  const volatile u32* tgw = tgrep(a, 0, (u32)(g % a.tg_rep));  // this warp's replica of the bound
  u32 tgp = (a.flags & 2) ? T_OPEN : *tgw;
  const bool publisher = !(a.flags & 1) && (g % a.pub_every) == 0;
  u32 since_refresh = 0;
  u32 hv[7];          // published-witness histogram snapshot (deferred tighten)
  bool tpend = false;
  // smallest T with >= k published witnesses d <= T -> every replica of tg;
  // returns the new filter limit (accept d < limit)
  auto finish_tighten = [&](bool post = true) -> u32 {
    tpend = false;
    u32 sum = 0;
#pragma unroll
    for (int i = 0; i < 7; ++i) sum += hv[i];
    const u32 incl = warp_incl_scan(sum, lane);
    const u32 bal = __ballot_sync(FULL, incl >= a.k);
    if (!bal) return T_OPEN;
    const int src = __ffs(bal) - 1;
    u32 tt = 0;
    if (lane == src) {
      u32 cc = incl - sum;
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        if (cc + hv[i] >= a.k) { tt = lane * 7 + i; break; }
        cc += hv[i];
      }
    }
    tt = __shfl_sync(FULL, tt, src);
    if (post)
      for (u32 r = lane; r < a.tg_rep; r += 32) atomicMin(tgrep(a, 0, r), tt);
    return (tt < T_OPEN ? tt : T_OPEN - 1) + 1;
  };
  bool first = true;  // the warp's first tile: the bound is read afresh
  // (the active warps of this launch: wide plane lists fold warps)
  const u32 wave_target = (u32)min((min((u64)gridDim.x * nact, a.wave_steps) * a.wave_pct / 100) * a.k, (u64)0x7fffffffu);
  bool wave = false;  // first-step witnesses posted: the second step waits for the first wave's

  // Compaction to the k best by (d, index): every entry with d < tt (the
  // k-th distance), then m = k - count(d < tt) of the ties. In index order
  // (unsorted copy) those are the first m ties in the buffer; on the sorted
  // copy the m smallest indices among the ties.
  auto compact = [&]() {
    const u32 n0 = ws->cnt[0];
    u32 less;
    const u32 tt = warp_kth_bin(hist, a.k, lane, &less);
    const u32 mk = a.k - less;
    u64 cut = IDX_MASK;  // SORTED: keep ties with index <= cut
    if (SORTED && hist[tt] > mk) {
      const u32 ntie = hist[tt];
      if (ntie <= 32) {
        u32 tp = 0;
        for (u32 i0 = 0; i0 < n0; i0 += 32) {
          const u32 i = i0 + lane;
          const u64 key = i < n0 ? wbuf[i] : ~0ull;
          const bool tie = i < n0 && key_d(key) == tt;
          const u32 tb = __ballot_sync(FULL, tie);
          if (tie) tie_scratch[tp + __popc(tb & lanemask_lt())] = key & IDX_MASK;
          tp += __popc(tb);
        }
        __syncwarp();
        const u64 mine = (u32)lane < ntie ? tie_scratch[lane] : ~0ull;
        u32 rank = 0;
        for (u32 j = 0; j < ntie; ++j) rank += tie_scratch[j] < mine ? 1u : 0u;
        const u32 sel = __ballot_sync(FULL, (u32)lane < ntie && rank == mk - 1);
        cut = __shfl_sync(FULL, mine, __ffs(sel) - 1);
        __syncwarp();
      } else {
        // many ties: the mk-th smallest tie index, MSB first over the buffer
        u64 pref = 0;
        u32 r = mk;
        for (int b = IDX_BITS - 1; b >= 0; --b) {
          u32 c = 0;
          for (u32 i0 = 0; i0 < n0; i0 += 32) {
            const u32 i = i0 + lane;
            const u64 key = i < n0 ? wbuf[i] : ~0ull;
            const u64 idx = key & IDX_MASK;
            const bool ok = i < n0 && key_d(key) == tt && (idx >> (b + 1)) == (pref >> (b + 1)) && !((idx >> b) & 1ull);
            c += __popc(__ballot_sync(FULL, ok));
          }
          if (c < r) {
            r -= c;
            pref |= 1ull << b;
          }
        }
        cut = pref;
      }
    }
    u32 outp = 0, ties = 0;
    for (u32 i0 = 0; i0 < n0; i0 += 32) {
      const u32 i = i0 + lane;
      const bool vld = i < n0;
      const u64 key = vld ? wbuf[i] : ~0ull;
      const u32 d = key_d(key);
      const bool lt = vld && d < tt, tie = vld && d == tt;
      const u32 tb = __ballot_sync(FULL, tie);
      const bool keep = lt || (tie && (SORTED ? (key & IDX_MASK) <= cut : ties + __popc(tb & lanemask_lt()) < mk));
      const u32 kb = __ballot_sync(FULL, keep);
      const u32 pp = outp + __popc(kb & lanemask_lt());
      __syncwarp();
      if (keep) wbuf[pp] = key;
      outp += __popc(kb);
      ties += __popc(tb);
    }
    for (u32 bb = lane; bb < HB; bb += 32) {
      if (bb > tt) hist[bb] = 0;
      else if (bb == tt) hist[bb] = mk;
    }
    if (lane == 0) ws->cnt[0] = outp;
    __syncwarp();
  };

  // Insert the entries of masks em (bit e of block h = entry bfirst + 32 h + e)
  // into the ordered buffer with distances dfn(h, bit); then the own bound and,
  // for new entries of publishers, their witnesses.
  auto insert = [&](const u32 (&em)[BPL], u64 bfirst, auto&& dfn, bool pub_new) {
    const u64 mm = (u64)em[0] | (BPL == 2 ? ((u64)em[BPL - 1] << 32) : 0ull);
    if (!__any_sync(FULL, mm != 0)) return;
    const u32 cntl = (u32)__popcll(mm);
    const u32 incl = warp_incl_scan(cntl, lane);
    const u32 total = __shfl_sync(FULL, incl, 31);
    if (ws->cnt[0] + total > a.cap) compact();
    const u32 cnt0 = ws->cnt[0];
    u32 pos = cnt0 + incl - cntl;
    if (SORTED) {
      // eight index lookups in flight at a time (a dependent load per entry
      // would cost a memory round trip each)
      for (u64 rest = mm; rest;) {
        int es[8];
        u32 li[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          es[j] = -1;
          if (rest) {
            es[j] = __ffsll((long long)rest) - 1;
            rest &= rest - 1;
            li[j] = __ldg(a.perm + bfirst + es[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (es[j] >= 0) {
            const u32 d = dfn(BPL == 2 ? (es[j] >> 5) : 0, es[j] & 31);
            wbuf[pos++] = make_key(d, a.index_base + li[j]);
            atomicAdd(hist + d, 1u);
          }
        }
      }
    } else {
      for (u64 rest = mm; rest; rest &= rest - 1) {
        const int e = __ffsll((long long)rest) - 1;
        const u32 d = dfn(BPL == 2 ? (e >> 5) : 0, e & 31);
        wbuf[pos++] = make_key(d, a.index_base + bfirst + e);
        atomicAdd(hist + d, 1u);
      }
    }
    __syncwarp();
    if (lane == 0) ws->cnt[0] = cnt0 + total;
    __syncwarp();
    if (cnt0 + total < a.k) return;
    u32 less;
    const u32 town = warp_kth_bin(hist, a.k, lane, &less);
    if (lane == 0) ws->town[0] = town;
    if (publisher && pub_new) {
      if (!ws->pubd[0]) {
        // first publication: every buffered candidate with d <= town
        for (u32 b = lane; b <= town && b < HB; b += 32) {
          const u32 cb = hist[b];
          if (cb) atomicAdd(gbin(a, 0, b), cb);
        }
      } else {
        // later: the entries just inserted with d <= town
        for (u64 rest = mm; rest; rest &= rest - 1) {
          const int e = __ffsll((long long)rest) - 1;
          const u32 d = dfn(BPL == 2 ? (e >> 5) : 0, e & 31);
          if (d <= town) atomicAdd(gbin(a, 0, d), 1u);
        }
      }
      __syncwarp();
      if (lane == 0) ws->pubd[0] = 1;
      __syncwarp();
      // tighten the global bound one step later: the histogram loads are
      // in flight while the next stage is awaited (an L2 round trip under a
      // saturated memory system costs microseconds)
#pragma unroll
      for (int i = 0; i < 7; ++i) hv[i] = *(volatile const u32*)gbin(a, 0, lane * 7 + i);
      tpend = true;
    }
    // (sorted order: entries at the own k-th distance may still precede by index)
    const u32 tn = SORTED ? town + 1 : town;
    T = tn < T ? tn : T;
    __syncwarp();
  };
  // first-step entries held back (bit-sliced distances, valid masks)
  u32 Dsv[BPL][8], vsv[BPL];
  u64 bsv = 0;
  u32 Tsv = 256, tlim = T_OPEN;  // their own limit; the last applied global limit
  bool pending = false;
  // insert them: d < min(own limit, global limit), no new witnesses (a
  // publisher already posted the step's)
  auto flush_pending = [&](bool fresh) {
    pending = false;
    u32 lim = Tsv < tlim ? Tsv : tlim;
    if (fresh && !(a.flags & 2)) {
      const u32 tf = *tgw;
      const u32 tl = (tf < T_OPEN ? tf : T_OPEN - 1) + 1;
      lim = tl < lim ? tl : lim;
    }
    u32 em[BPL];
#pragma unroll
    for (int h = 0; h < BPL; ++h) {  // D < lim, MSB first over 9 bits (D < 256)
      u32 lt = 0, eq = FULL;
#pragma unroll
      for (int b = 8; b >= 0; --b) {
        const u32 db = b < 8 ? Dsv[h][b] : 0u;
        const u32 lb = ((lim >> b) & 1u) ? FULL : 0u;
        lt |= eq & ~db & lb;
        eq &= ~(db ^ lb);
      }
      em[h] = lt & vsv[h];
    }
    insert(em, bsv, [&](int h, int bit) -> u32 {
      u32 d = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) d |= (((h ? Dsv[BPL - 1][b] : Dsv[0][b]) >> bit) & 1u) << b;
      return d;
    }, false);
  };

  // The first wave's exchange and the held-back entries of the previous step
  // (index order: before this step's entries). Called after the step's
  // carry-save count so part of the exchange hides under it (C2 scan 25.8 ->
  // 24.9 us); the sorted-copy kernels, short of registers, call it first.
  auto wave_and_flush = [&]() {
      if (wave) {
        // Second step (after its carry-save count): every warp posted its first
        // step's witnesses at about the same time. Wait (bounded) until wave_target of them are visible,
        // then take the bound from the histogram: this step, the held-back
        // first-step entries and everything after run under a bound drawn from
        // hundreds of thousands of entries instead of the warp's own 2,048 --
        // inserts become rare and the scan streams.
        wave = false;
        // one warp per CTA polls the global histogram (every warp polling its
        // 224 lines costs ~4 us of L2 hot-line traffic); the others take the
        // bound from shared memory
        u32 r = 0;
        if (lane == 0) r = atomicAdd(&s_wave_poll, 1u);
        r = __shfl_sync(FULL, r, 0);
        const u64 t0 = pq_now_ns();
        u32 lim = T_OPEN;
        if (r == 0) {
          for (;;) {
#pragma unroll
            for (int i = 0; i < 7; ++i) hv[i] = *(volatile const u32*)gbin(a, 0, lane * 7 + i);
            u32 sum = 0;
#pragma unroll
            for (int i = 0; i < 7; ++i) sum += hv[i];
            sum = __reduce_add_sync(FULL, sum);
            if (sum >= wave_target || pq_now_ns() - t0 > a.wave_wait_ns) break;
          }
          lim = finish_tighten(true);
          if (lane == 0) *(volatile u32*)&s_wave_T = lim | 0x80000000u;
        } else {
          u32 v;
          while (!(v = *(volatile const u32*)&s_wave_T) && pq_now_ns() - t0 < (u64)a.wave_wait_ns + 2000) __nanosleep(40);
          if (v) lim = v & 0xffffu;
        }
        T = lim < T ? lim : T;
        tlim = lim < tlim ? lim : tlim;
      }
#ifdef FPS_SCAN_TRACE
      if (lane == 0 && g < 16384 && tr_iter == 1) g_pq_s1[g * 4 + 0] = gtimer();
#endif
      // the previous step's held-back entries first (index order) -- after this
      // step's count, so part of the first wave's exchange above hides under it
      // (C2 scan 25.8 -> 24.9 us)
      if (pending) flush_pending(false);
#ifdef FPS_SCAN_TRACE
      if (lane == 0 && g < 16384 && tr_iter == 1) g_pq_s1[g * 4 + 1] = gtimer();
#endif
  };
#pragma unroll 1
  for (u32 st = 0, ph = 0;; st = (st + 1 == S) ? 0 : st + 1, ph ^= (st == 0) ? 1u : 0u) {
#ifdef FPS_SCAN_TRACE
    if (tr_first && !tr_step1) tr_step1 = gtimer();  // (slot 2: end of the first step's compute)
#endif
    mbar_wait(&bars[st], ph);
    const u64 t = *(volatile const u64*)&slot_step[st];
    if (t == PQ_NONE) break;
#ifdef FPS_SCAN_TRACE
    if (!tr_first) tr_first = gtimer();
    ++tr_iter;
    if (lane == 0 && g < 16384 && tr_iter < 8) g_pq_steps[g * 8 + tr_iter] = gtimer();  // start of every step (a store: no stall)
#endif
    // first tile: the bound other warps may have set meanwhile (the load
    // flies under the carry-save count)
    u32 tfresh = T_OPEN;
    if (first && !(a.flags & 2)) tfresh = *tgw;
    if (a.flags & 512) {  // experiment: stream only (no compute; results are not valid)
      __syncwarp();
      issue(st);
      continue;
    }
    if (tpend) {
      const u32 lim = finish_tighten();
      T = lim < T ? lim : T;
      tlim = lim < tlim ? lim : tlim;
    }
    // the bound prefetched one step ago
    {
      const u32 tl = (tgp < T_OPEN ? tgp : T_OPEN - 1) + 1;
      T = tl < T ? tl : T;
      tlim = tl < tlim ? tl : tlim;
    }
    if constexpr (SORTED) wave_and_flush();
    const char* stage = ring + st * stage_bytes;
    const char* lb = stage + 4 * BPL * lane;  // this lane's BPL words of every position
    // one shared load fetches a plane word of all BPL blocks of the lane
    auto ldp = [&](const char* p, u32* d) {
      if constexpr (BPL == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        d[0] = v.x;
        d[1] = v.y;
      } else {
        d[0] = *reinterpret_cast<const u32*>(p);
      }
    };
    u32 A[BPL][8];
    const u32 mt = SORTED ? (u32)s_meta[t - cta_lo] : 0u;
    if (SORTED && (mt & 0xffu) == (mt >> 8)) {  // one popcount for the step
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int h = 0; h < BPL; ++h) A[h][i] = ((mt >> i) & 1u) ? FULL : 0u;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        u32 v[BPL];
        ldp(lb + i * PQ_CHUNK, v);
#pragma unroll
        for (int h = 0; h < BPL; ++h) A[h][i] = v[h];
      }
    }
    const u64 blk_first = t * PQ_STEP + (u64)lane * 32 * BPL;  // local index of bit 0 of this lane's first block
    u32 valid[BPL];
#pragma unroll
    for (int h = 0; h < BPL; ++h) {
      const u64 f = blk_first + 32 * h;
      valid[h] = f >= a.n ? 0u : (a.n - f >= 32 ? FULL : ((1u << (a.n - f)) - 1u));
    }
    // carry-save count of the listed planes (positions 8 .. np-1)
    u32 ones[BPL], twos[BPL], fours[BPL], eights[BPL], s16[BPL], s32[BPL], s64[BPL];
#pragma unroll
    for (int h = 0; h < BPL; ++h) ones[h] = twos[h] = fours[h] = eights[h] = s16[h] = s32[h] = s64[h] = 0;
#define CSA(h, l, x, y)   \
  do {                    \
    const u32 u_ = l ^ x; \
    h = (l & x) | (u_ & y); \
    l = u_ ^ y;           \
  } while (0)
    const char* lp = lb + 8 * PQ_CHUNK;
    auto load8 = [&](u32 c, u32 (&d)[BPL][8]) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        u32 v[BPL];
        ldp(lp + (c + i) * PQ_CHUNK, v);
#pragma unroll
        for (int h = 0; h < BPL; ++h) d[h][i] = v[h];
      }
    };
    auto tree8 = [&](const u32 (&d)[BPL][8], u32 (&e8)[BPL]) {
#pragma unroll
      for (int h = 0; h < BPL; ++h) {
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
    const u32 mlen = np - 8;
    u32 c0 = 0;
#pragma unroll 1
    for (; c0 + 16 <= mlen; c0 += 16) {
      u32 d[BPL][8], e8a[BPL], e8b[BPL];
      load8(c0, d);
      tree8(d, e8a);
      load8(c0 + 8, d);
      tree8(d, e8b);
#pragma unroll
      for (int h = 0; h < BPL; ++h) {
        u32 e16;
        CSA(e16, eights[h], e8a[h], e8b[h]);
        const u32 c2 = s16[h] & e16;
        s16[h] ^= e16;
        const u32 c3 = s32[h] & c2;
        s32[h] ^= c2;
        s64[h] ^= c3;
      }
    }
    if (c0 < mlen) {
      u32 d[BPL][8], e8[BPL];
      load8(c0, d);
      tree8(d, e8);
#pragma unroll
      for (int h = 0; h < BPL; ++h) {
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

#ifdef FPS_SCAN_TRACE
    if (lane == 0 && g < 16384 && tr_iter == 0) g_pq_phase[g * 8 + 0] = gtimer();
    if (lane == 0 && g < 16384 && tr_iter == 1) g_pq_s1[g * 4 + 2] = gtimer();
#endif
    // every lane is done reading this slot: refill it with the step S ahead
    __syncwarp();
    if (COPY == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

#ifdef FPS_SCAN_TRACE
    if (lane == 0 && g < 16384 && tr_iter == 0) g_pq_phase[g * 8 + 1] = gtimer();
#endif
    issue(st);
    if (!(a.flags & 2) && ++since_refresh >= a.refresh) {  // applied at the next step
      since_refresh = 0;
      tgp = *tgw;
    }

    // X = P - N over 10 bits: (P, N) = (|a|, 2c) sparse, (2c, |a|) dense
    u32 X[BPL][10];
#pragma unroll
    for (int h = 0; h < BPL; ++h) {
      const u32 C[8] = {0, ones[h], twos[h], fours[h], eights[h], s16[h], s32[h], s64[h]};  // 2c
      u32 cy = FULL;
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        const u32 p = i < 8 ? (dense ? C[i] : A[h][i]) : 0u;
        const u32 nn = ~(i < 8 ? (dense ? A[h][i] : C[i]) : 0u);
        X[h][i] = p ^ nn ^ cy;
        cy = (p & nn) | (cy & (p ^ nn));
      }
    }
    // entries with d < Tq: sign plane of X + (|q| - Tq)
    auto pass = [&](int h, u32 Tq) -> u32 {
      return bs_sign_after_add(X[h], (pop - Tq) & 0x3ffu) & valid[h];
    };
#ifdef FPS_SCAN_TRACE
    if (lane == 0 && g < 16384 && tr_iter == 0) g_pq_phase[g * 8 + 2] = gtimer();
#endif

    if constexpr (!SORTED) wave_and_flush();
    if (first) {
      first = false;
      const u32 tl = (tfresh < T_OPEN ? tfresh : T_OPEN - 1) + 1;
      T = tl < T ? tl : T;
      tlim = tl < tlim ? tl : tlim;
    }
    if (T >= T_OPEN && !pending) {
      // ---- the warp's first step, no bound known yet. Distances of the
      // whole step bit-sliced (D = X + |q|), the k-th smallest by radix
      // select (no per-entry work); publishers post witnesses at the 1st,
      // 2nd, 4th, 8th and k-th smallest distance. The step's entries are
      // inserted at the next step, when more witnesses have been published
      // and the global bound is tighter (typically: far fewer inserts).
#pragma unroll
      for (int h = 0; h < BPL; ++h) {
        u32 cy = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const u32 w = ((pop >> b) & 1u) ? FULL : 0u;
          Dsv[h][b] = X[h][b] ^ w ^ cy;
          cy = (X[h][b] & w) | (cy & (X[h][b] ^ w));
        }
        vsv[h] = valid[h];
      }
#ifdef FPS_SCAN_TRACE
      if (lane == 0 && g < 16384) g_pq_phase[g * 8 + 6] = gtimer();
#endif
      u32 nv = 0;
#pragma unroll
      for (int h = 0; h < BPL; ++h) nv += __popc(valid[h]);
      nv = __reduce_add_sync(FULL, nv);
      // r-th smallest distance of the step (1-based, r <= nv), MSB first
      // NR radix selects at once (r-th smallest distance of the step, 1-based,
      // r <= nv), MSB first: the NR warp reductions of a bit are independent
      // and overlap their latency
      auto rsel = [&](const auto& rs, auto& out) {
        constexpr int NR = sizeof(rs) / sizeof(rs[0]);
        u32 msk[NR][BPL], rr[NR];
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          rr[j] = rs[j];
          out[j] = 0;
#pragma unroll
          for (int h = 0; h < BPL; ++h) msk[j][h] = valid[h];
        }
#pragma unroll
        for (int b = 7; b >= 0; --b) {
          u32 c[NR];
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            c[j] = 0;
#pragma unroll
            for (int h = 0; h < BPL; ++h) c[j] += __popc(msk[j][h] & ~Dsv[h][b]);
          }
#pragma unroll
          for (int j = 0; j < NR; ++j) c[j] = __reduce_add_sync(FULL, c[j]);
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const bool zero = c[j] >= rr[j];
            if (!zero) {
              rr[j] -= c[j];
              out[j] |= 1u << b;
            }
#pragma unroll
            for (int h = 0; h < BPL; ++h) msk[j][h] &= zero ? ~Dsv[h][b] : Dsv[h][b];
          }
        }
      };
      Tsv = 256;  // fewer than k entries: every one is a candidate
      if (nv >= a.k) {
        u32 town1 = 0;
        const bool wv = wave_target != 0 && !(a.flags & 1);
        if (publisher || wv) {
          // witnesses: 1 at the smallest distance, 1 at the 2nd, 2 at the 4th,
          // k - 4 at the k-th (ranks capped at k). With many more warps than
          // k the bound is set by the warps' smallest distances: higher ranks
          // (8th ... 64th) bought nothing.
          const u32 rs[4] = {1u, min(2u, a.k), min(4u, a.k), a.k};
          u32 ts[4];
          rsel(rs, ts);
          if (lane < 4) {
            const u32 prev = lane == 0 ? 0u : lane == 1 ? rs[0] : lane == 2 ? rs[1] : rs[2];
            const u32 tl = lane == 0 ? ts[0] : lane == 1 ? ts[1] : lane == 2 ? ts[2] : ts[3];
            const u32 rl = lane == 0 ? rs[0] : lane == 1 ? rs[1] : lane == 2 ? rs[2] : rs[3];
            if (rl > prev) atomicAdd(gbin(a, 0, tl), rl - prev);
          }
          town1 = ts[3];
          if (publisher && lane == 0) ws->pubd[0] = 1;
          if (wv) {
            // first wave: every warp posts; the second step takes the bound
            // from all of them (below)
            wave = true;
          } else {
#pragma unroll
            for (int i = 0; i < 7; ++i) hv[i] = *(volatile const u32*)gbin(a, 0, lane * 7 + i);
            tpend = true;
          }
        } else {
          const u32 rs[1] = {a.k};
          u32 ts[1];
          rsel(rs, ts);
          town1 = ts[0];
        }
        // >= k entries of this step have d <= town1 and a smaller index than
        // any later entry: later entries need d < town1
        const u32 tn = SORTED ? town1 + 1 : town1;
        T = tn < T ? tn : T;
        Tsv = town1 + 1;
      }
#ifdef FPS_SCAN_TRACE
      if (lane == 0 && g < 16384) g_pq_phase[g * 8 + 7] = gtimer();
#endif
      bsv = blk_first;
      pending = true;
      __syncwarp();
      continue;
    }

#ifdef FPS_SCAN_TRACE
    if (lane == 0 && g < 16384 && tr_iter == 1) g_pq_phase[g * 8 + 3] = gtimer();
#endif
    u32 em[BPL];
#pragma unroll
    for (int h = 0; h < BPL; ++h) em[h] = pass(h, T);
    insert(em, blk_first, [&](int h, int bit) -> u32 {
      constexpr int H1 = BPL - 1;
      u32 av = 0, cv = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) av |= (((h ? A[H1][i] : A[0][i]) >> bit) & 1u) << i;
      const u32 cb[7] = {h ? ones[H1] : ones[0], h ? twos[H1] : twos[0], h ? fours[H1] : fours[0],
                         h ? eights[H1] : eights[0], h ? s16[H1] : s16[0], h ? s32[H1] : s32[0],
                         h ? s64[H1] : s64[0]};
#pragma unroll
      for (int i = 0; i < 7; ++i) cv |= ((cb[i] >> bit) & 1u) << i;
      return dense ? pop - av + 2 * cv : av + pop - 2 * cv;
    }, true);
#ifdef FPS_SCAN_TRACE
    if (lane == 0 && g < 16384 && tr_iter == 1) g_pq_phase[g * 8 + 5] = gtimer();
    ph_done = true;
#endif
    __syncwarp();
  }
  if (pending) flush_pending(true);

#ifdef FPS_SCAN_TRACE
  if (lane == 0 && g < 16384) {
    g_scan_trace[g * 4 + 0] = tr_start;
    g_scan_trace[g * 4 + 1] = gtimer();
    g_scan_trace[g * 4 + 3] = tr_first;
    g_scan_trace[g * 4 + 2] = tr_step1;
  }
#endif
  // ---- survivors (d <= the bound, re-read: short scans end before their
  // first prefetch sees the witnesses published in the same step) to the flat list
  if (tpend) finish_tighten();
  u32 tb = tgp;
  if (!(a.flags & 2)) {
    const u32 tf = *tgw;
    tb = tf < tb ? tf : tb;
  }
  u32 c = 0;
  for (u32 b = lane; b < (u32)HB; b += 32) c += b <= tb ? hist[b] : 0u;
  c = __reduce_add_sync(FULL, c);
  if (c == 0) return;
  if (c > a.k) compact();
  const u32 n0 = ws->cnt[0];
  for (u32 i0 = 0; i0 < n0; i0 += 32) {
    const u32 i = i0 + lane;
    const u64 key = i < n0 ? wbuf[i] : ~0ull;
    const bool keep = i < n0 && key_d(key) <= tb;
    const u32 kb = __ballot_sync(FULL, keep);
    const u32 nk = __popc(kb);
    if (nk == 0) continue;
    u32 base = 0;
    if (lane == 0) base = atomicAdd(a.cand_cnt, nk);
    base = __shfl_sync(FULL, base, 0);
    if (keep) a.cand[base + __popc(kb & lanemask_lt())] = key;
  }
}

}  // namespace fps
