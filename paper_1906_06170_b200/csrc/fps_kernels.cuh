// fps_kernels.cuh — sm_100a device code for the MACCS-166 Hamming scan.
//
// Replaces the reference's per-block numpy kernel + heap
// (/root/reference/pkg/src/fpscan/scan.py:137-143, :91-126, :173-209) and the
// shard merge (scan.py:225-236) with:
//   * scan_kernel<QW,E,MODE>  — one pass over the HBM-resident SoA library
//     (three u64 planes); each warp owns a contiguous library part and QW
//     queries held in registers; distance = sum of popcount(word XOR query)
//     over the three full 64-bit words (exactly what scan.py:142 XORs);
//     MODE_TOPK keeps a per-(warp,query) candidate buffer in index order with
//     an incremental distance histogram and an exact filter threshold;
//     MODE_RANGE appends every hit with warp-ballot compaction;
//     MODE_HIST counts distances (large-k path).
//   * select_kernel — per query, exact top-k over the flat candidate list
//     (histogram on distance, then tie resolution by index).
//   * merge_kernel — rank-0 merge of G sorted per-shard top-k lists
//     (merge_topk semantics) by merge-path ranking.
//   * gen_kernel / transpose kernels — synthetic library and FPS1/row-major
//     ingestion into planes.
//
// Ordering everywhere is the reference total order (distance, then id) with
// id = global library index (cid = index + 1 in the reference's synthetic
// libraries, synth.py:37). Keys pack (d << 40) | index (index < 2^40).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef FPS_QW1_MINB
#define FPS_QW1_MINB 2  // CTAs per SM the single-query kernels are register-limited for
#endif
#ifndef FPS_QW1_TMA
#define FPS_QW1_TMA 1  // single-query scans stream tiles through a per-warp shared-memory ring (bulk copies)
#endif
#ifndef FPS_QW1_STAGES
#define FPS_QW1_STAGES 2  // tiles in flight per warp in the bulk-copy ring
#endif

namespace fps {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr u32 FULL = 0xffffffffu;
constexpr int IDX_BITS = 40;
constexpr u64 IDX_MASK = (1ull << IDX_BITS) - 1;
constexpr int HB = 224;       // histogram bins (distances 0..192 used; 7 per lane)
constexpr u32 DMASKED = 255;  // distance given to masked (out-of-range) entries
constexpr u32 T_OPEN = 255;   // "accept everything" threshold

enum { MODE_TOPK = 0, MODE_RANGE = 1, MODE_HIST = 2 };

// HBM layout: tiles, each a small structure of arrays
//   full    (24 B/entry): w0[128] u64 | w1[128] u64 | w2[128] u64                 = 3072 B
//   compact (21 B/entry): w0[256] u64 | w1[256] u64 | w2lo[256] u32 | w2hi[256] u8 = 5376 B
// One warp iteration of the single-query scan (32 lanes x 4 entries) reads
// one full tile (or half a compact one): its loads fall in one 3-5 KB span.
// (compact tiles hold 256 entries so a tile, 5376 B, is a whole number of
// 256 B DRAM interleave chunks, like the 3072 B full tile)
constexpr int TILE_FULL = 128;
constexpr int TILE_CMP = 256;
constexpr u64 TILE_BYTES_FULL = 24 * TILE_FULL;
constexpr u64 TILE_BYTES_CMP = 21 * TILE_CMP;
__host__ __device__ __forceinline__ u64 tile_bytes(bool compact) { return compact ? TILE_BYTES_CMP : TILE_BYTES_FULL; }
__host__ __device__ __forceinline__ u64 tile_entries(bool compact) { return compact ? TILE_CMP : TILE_FULL; }

__host__ __device__ __forceinline__ u64 make_key(u32 d, u64 idx) { return ((u64)d << IDX_BITS) | idx; }
__host__ __device__ __forceinline__ u32 key_d(u64 key) { return (u32)(key >> IDX_BITS) & 0xffu; }

struct __align__(32) u64x4 { u64 x, y, z, w; };

// Streaming loads: read-only, do not allocate in L1 (each byte is read once).
__device__ __forceinline__ void ld_entries(const u64* p, u64 (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld_entries(const u64* p, u64 (&v)[2]) {
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p));
}
__device__ __forceinline__ void ld_entries(const u64* p, u64 (&v)[1]) {
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v[0]) : "l"(p));
}

// Compact layout: word 2 is split into a u32 plane (bits 0..31, keys
// 129..160) and a u8 plane (bits 32..39: keys 161..166 + the 2 low pad bits).
__device__ __forceinline__ void ld_w2c(const u32* lo, const unsigned char* hi, u64 (&v)[4]) {
  u32 a, b, c, d, h;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(lo));
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(h) : "l"(hi));
  v[0] = (u64)a | ((u64)(h & 0xffu) << 32);
  v[1] = (u64)b | ((u64)((h >> 8) & 0xffu) << 32);
  v[2] = (u64)c | ((u64)((h >> 16) & 0xffu) << 32);
  v[3] = (u64)d | ((u64)(h >> 24) << 32);
}
__device__ __forceinline__ void ld_w2c(const u32* lo, const unsigned char* hi, u64 (&v)[2]) {
  u32 a, b;
  unsigned short h;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(lo));
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(h) : "l"(hi));
  v[0] = (u64)a | ((u64)(h & 0xffu) << 32);
  v[1] = (u64)b | ((u64)(h >> 8) << 32);
}
__device__ __forceinline__ void ld_w2c(const u32* lo, const unsigned char* hi, u64 (&v)[1]) {
  u32 a;
  unsigned short h;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(a) : "l"(lo));
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(h) : "l"(hi));
  v[0] = (u64)a | ((u64)(h & 0xffu) << 32);
}

__device__ __forceinline__ u32 dist3(u64 a, u64 b, u64 c, u64 q0, u64 q1, u64 q2) {
  return (u32)(__popcll(a ^ q0) + __popcll(b ^ q1) + __popcll(c ^ q2));
}

// Same distance with 4 POPC instead of 6: two full adders (carry-save) fold
// the six 32-bit XOR words into sums s1, s2 and carries c1, c2 with
// popc(x0)+popc(x1)+popc(x2) = popc(s1) + 2 popc(c1). POPC issues at 16/clk/SM
// on B200 vs 64/clk for LOP3, so the compute-bound multi-query scan trades
// two POPC for four LOP3 per comparison.
__device__ __forceinline__ u32 dist3_csa(u64 a, u64 b, u64 c, u64 q0, u64 q1, u64 q2) {
  const u64 ya = a ^ q0, yb = b ^ q1, yc = c ^ q2;
  const u32 x0 = (u32)ya, x1 = (u32)(ya >> 32), x2 = (u32)yb;
  const u32 x3 = (u32)(yb >> 32), x4 = (u32)yc, x5 = (u32)(yc >> 32);
  const u32 s1 = x0 ^ x1 ^ x2, c1 = (x0 & x1) | (x2 & (x0 ^ x1));
  const u32 s2 = x3 ^ x4 ^ x5, c2 = (x3 & x4) | (x5 & (x3 ^ x4));
  return (u32)(__popc(s1) + __popc(s2)) + 2u * (u32)(__popc(c1) + __popc(c2));
}

// Release/acquire fence at GPU scope (cheaper than __threadfence()'s fence.sc).
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ u32 warp_incl_scan(u32 v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Smallest t with sum_{d<=t} hist[d] >= k (hist has HB bins, warp-cooperative).
// Returns T_OPEN when the total is below k. Also returns count(d < t) in *less.
__device__ __forceinline__ u32 warp_kth_bin(const u32* hist, u32 k, int lane, u32* less) {
  u32 h[7];
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < 7; ++i) { h[i] = hist[lane * 7 + i]; s += h[i]; }
  u32 incl = warp_incl_scan(s, lane);
  u32 ballot = __ballot_sync(FULL, incl >= k);
  if (ballot == 0) { *less = 0; return T_OPEN; }
  int src = __ffs(ballot) - 1;
  u32 t = 0, lt = 0;
  if (lane == src) {
    u32 c = incl - s;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      if (c + h[i] >= k) { t = lane * 7 + i; lt = c; break; }
      c += h[i];
    }
  }
  t = __shfl_sync(FULL, t, src);
  *less = __shfl_sync(FULL, lt, src);
  return t;
}

struct ScanArgs {
  const char* lib;               // tiled library (see TILE_BYTES_*)
  u64 n;           // valid entries on this device
  u64 index_base;  // global index of entry 0
  const u64* queries;  // Q x 3 (device); nullptr: the single query is inline in qin
  u64 qin[3];          // inline query words (host API, Q == 1: no H2D copy)
  const unsigned char* radius;  // MODE_RANGE: per-query radius
  u32 Q;
  u32 Qmin;        // MINQ: number of queries the distance is minimised over
  u32 k;
  u32 cap;         // MODE_TOPK: per-(warp, query) buffer capacity
  u32 n_qg;        // query groups (ceil(Q / QW))
  u32 flags;       // experiment knobs (FPS_SCAN_FLAGS): 1 = no global publish, 2 = no tg refresh,
                   // 32 = select without programmatic dependent launch
  u32 gstride;     // words between consecutive ghist bins / tg replicas (spreads hot lines over L2 slices)
  u32 tg_rep;      // replicas of tg[q] (all receive every atomicMin; warp g reads replica g % tg_rep)
  u32 pub_every;   // only library parts with part % pub_every == 0 publish to ghist
  u64 n_parts;     // library parts
  u64 iters;       // ceil(n / (32*E))
  u32* dyn_ctr;    // bulk-copy single-query scan: tail chunk counter (nullptr: static parts only)
  u64 dyn_start;   // first tile of the dynamically claimed tail
  u64 dyn_chunk;   // tiles per claim
  // MODE_TOPK state (all per query unless noted)
  u32* tg;         // global filter bound: entries with d > tg[q] are not in the top-k
  u32* ghist;      // [Q][HB] distances of published candidates (distinct entries)
  u64* buf;        // [warps][QW][cap] candidate buffers
  u64* cand;       // [Q][cand_cap] flat survivor list
  u32* cand_cnt;   // [Q]
  u64 cand_cap;
  // MODE_RANGE output
  u64* out;        // keys (q << 48) | (d << 40) | idx
  u64* out_cnt;    // single counter
  u64 out_cap;
  // MODE_HIST output: ghist reused
  const u32* gate;  // non-null: the grid does nothing unless *gate != 0 (device-side
                    // fallback of the tensor-core path, decided without the host)
};

// Global bound maintenance. ghist[q] counts distances of *published*
// candidates; every published candidate is a distinct library entry, so if
// the cumulative count up to T reaches k, no entry with d > T can be in the
// top-k and tg[q] = min(tg[q], T) is exact. Reads of ghist see monotone
// counters, so any snapshot is a valid lower count.
template <class A>
__device__ __forceinline__ u32* gbin(const A& a, u32 qi, u32 b) {
  return a.ghist + ((u64)qi * HB + b) * a.gstride;
}
template <class A>
__device__ __forceinline__ u32* tgrep(const A& a, u32 qi, u32 r) {
  return a.tg + ((u64)qi * a.tg_rep + r) * a.gstride;
}

template <class A>
__device__ __forceinline__ u32 tighten_tg(const A& a, u32 qi, int lane) {
  u32 hv[7], s = 0;
#pragma unroll
  for (int i = 0; i < 7; ++i) { hv[i] = *(volatile const u32*)gbin(a, qi, lane * 7 + i); s += hv[i]; }
  u32 incl = warp_incl_scan(s, lane);
  u32 bal = __ballot_sync(FULL, incl >= a.k);
  if (!bal) return T_OPEN;
  const int src = __ffs(bal) - 1;
  u32 tt = 0;
  if (lane == src) {
    u32 cc = incl - s;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      if (cc + hv[i] >= a.k) { tt = lane * 7 + i; break; }
      cc += hv[i];
    }
  }
  tt = __shfl_sync(FULL, tt, src);
  for (u32 r = lane; r < a.tg_rep; r += 32) atomicMin(tgrep(a, qi, r), tt);
  return tt;
}

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Streaming variant: an L2 evict-first policy, so a library scanned once per
// call does not displace the small hot scan state (bounds, histograms).
__device__ __forceinline__ u64 l2_evict_first_policy() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, u32 bytes, u64* bar, u64 pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Per-warp slow-path state, kept in shared memory (only touched on inserts).
template <int QW>
struct WarpState {
  u32 town[QW];   // own k-th distance (T_OPEN until k candidates)
  u32 pubd[QW];   // 1 once the warp has published its candidates
  u32 cnt[QW];    // buffer fill
};

// Dynamic shared-memory layout of scan_kernel (host and device agree on it):
// [per-warp histograms][per-warp WarpState] then, for the bulk-copy
// single-query variant, [per-warp ring of STAGES tiles][per-warp mbarriers]
// [per-warp slot tile indices].
template <int QW, int E, int MODE, bool CMP>
struct ScanSmem {
  static constexpr bool TMA = (QW == 1 && E == 4 && FPS_QW1_TMA != 0);
  static constexpr int STAGES = FPS_QW1_STAGES;
  static constexpr u64 SLOT = CMP ? TILE_BYTES_CMP : TILE_BYTES_FULL;  // one library tile per ring slot
  static constexpr int SUB = CMP ? TILE_CMP / 128 : TILE_FULL / 128;   // 128-entry iterations per tile
  __host__ __device__ static constexpr size_t base(int nwb) {
    return MODE == MODE_RANGE ? 0 : (size_t)nwb * (QW * HB * sizeof(u32) + sizeof(WarpState<QW>));
  }
  __host__ __device__ static constexpr size_t ring_off(int nwb) { return TMA ? (base(nwb) + 127) / 128 * 128 : base(nwb); }
  __host__ __device__ static constexpr size_t bars_off(int nwb) {
    return ring_off(nwb) + (TMA ? (size_t)nwb * STAGES * SLOT : 0);
  }
  __host__ __device__ static constexpr size_t tiles_off(int nwb) { return bars_off(nwb) + (TMA ? (size_t)nwb * STAGES * 8 : 0); }
  __host__ __device__ static constexpr size_t total(int nwb) { return tiles_off(nwb) + (TMA ? (size_t)nwb * STAGES * 8 : 0); }
};

#ifdef FPS_SCAN_TRACE
__device__ u64 g_scan_trace[16384 * 4];  // per warp: start, end (globaltimer ns), SM id, first data
__device__ u64 g_mark[8];                // marker kernel / select start / select end (globaltimer ns)
__device__ __forceinline__ u64 gtimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void mark_kernel(int slot) { g_mark[slot] = gtimer(); }
#endif
template <int QW, int E, int MODE, bool MINQ = false, bool CMP = false>
__global__ void __launch_bounds__(256, (QW == 1 ? FPS_QW1_MINB : (QW >= 4 ? 2 : 3))) scan_kernel(const ScanArgs a) {
  extern __shared__ u32 smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nwb = blockDim.x >> 5;
  const u64 g = (u64)blockIdx.x * nwb + wib;
  // let a programmatic dependent (select_kernel) launch early; it still waits
  // for this grid to complete before reading its results
  asm volatile("griddepcontrol.launch_dependents;");
  using SL = ScanSmem<QW, E, MODE, CMP>;
  // Launched as a programmatic dependent of the previous call's select_kernel
  // (host API / graphs): the CTAs get resident while it runs and wait until it
  // has completed (it resets the bounds, histograms and counters) before
  // touching that state. The bulk-copy scan first puts its first library
  // tiles in flight -- the library is read-only -- so the HBM ramp overlaps
  // the previous select.
  if constexpr (!SL::TMA) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.gate && *(volatile const u32*)a.gate == 0) return;  // block-uniform
  }
  __shared__ u32 s_cta_next;  // bulk-copy scan: next tile of the CTA's run (CTA-dynamic mode)
  if constexpr (SL::TMA) {
    if (threadIdx.x == 0) s_cta_next = 0;
    __syncthreads();  // the only block-level barrier: before any warp leaves
  }
  if (g >= (u64)a.n_qg * a.n_parts) return;  // warp-uniform; no block-level sync below
#ifdef FPS_SCAN_TRACE
  u64 tr_start, tr_first = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_start));
#endif
  const u32 qg = (u32)(g % a.n_qg);
  const u64 part = g / a.n_qg;
  const u64 it0 = part * a.iters / a.n_parts;
  const u64 it1 = (part + 1) * a.iters / a.n_parts;
  const u64 n_full = a.n / (32 * E);  // iterations whose entries are all valid

  u64 q0[QW], q1[QW], q2[QW];
  u32 T[QW];  // hot filter: accept d < T[j]
#pragma unroll
  for (int j = 0; j < QW; ++j) {
    u32 qi = qg * QW + j;
    bool ok = qi < a.Q;
    q0[j] = ok ? (a.queries ? a.queries[3 * (u64)qi + 0] : a.qin[0]) : 0;
    q1[j] = ok ? (a.queries ? a.queries[3 * (u64)qi + 1] : a.qin[1]) : 0;
    q2[j] = ok ? (a.queries ? a.queries[3 * (u64)qi + 2] : a.qin[2]) : 0;
    if (MODE == MODE_TOPK) T[j] = ok ? T_OPEN : 0;
    else if (MODE == MODE_RANGE) T[j] = ok ? (u32)a.radius[qi] + 1 : 0;
    else T[j] = ok ? 256 : 0;
  }
  u32* hist = smem + (u64)wib * QW * HB;  // [QW][HB] (TOPK / HIST)
  WarpState<QW>* ws = reinterpret_cast<WarpState<QW>*>(smem + (u64)nwb * QW * HB) + wib;
  if (MODE != MODE_RANGE) {
    for (int i = lane; i < QW * HB; i += 32) hist[i] = 0;
    if (lane < QW) { ws->town[lane] = T_OPEN; ws->pubd[lane] = 0; ws->cnt[lane] = 0; }
    __syncwarp();
  }
  u64* wbuf = (MODE == MODE_TOPK) ? a.buf + g * QW * (u64)a.cap : nullptr;

  // Register arrays indexed by a runtime slot j would be demoted to local
  // memory; the slow path selects / updates slot j with unrolled compares.
  auto setT = [&](int j, u32 v) {
#pragma unroll
    for (int jj = 0; jj < QW; ++jj)
      if (jj == j) T[jj] = v;
  };
  auto refresh_tg = [&](int j) {
    u32 qi = qg * QW + j;
    if (qi < a.Q && !(a.flags & 2)) {
      u32 t = *(volatile const u32*)tgrep(a, qi, (u32)(g % a.tg_rep));
      t = (t < T_OPEN ? t : T_OPEN - 1) + 1;
      u32 own = ws->town[j];
      setT(j, t < own ? t : own);
    }
  };

  // Warp-collective ordered compaction of query slot j's buffer down to its
  // k best: every entry with d < T_own, then the first m ties in index order
  // (the buffer is always in ascending index order).
  auto compact = [&](int j) {
    u32* hj = hist + j * HB;
    u64* bj = wbuf + (u64)j * a.cap;
    const u32 n = ws->cnt[j];
    u32 less;
    const u32 t = warp_kth_bin(hj, a.k, lane, &less);
    const u32 m = a.k - less;
    u32 out = 0, ties = 0;
    for (u32 i0 = 0; i0 < n; i0 += 32) {
      const u32 i = i0 + lane;
      const bool valid = i < n;
      const u64 key = valid ? bj[i] : ~0ull;
      const u32 d = key_d(key);
      const bool lt = valid && d < t;
      const bool tie = valid && d == t;
      const u32 tb = __ballot_sync(FULL, tie);
      const u32 tr = ties + __popc(tb & lanemask_lt());
      const bool keep = lt || (tie && tr < m);
      const u32 kb = __ballot_sync(FULL, keep);
      const u32 p = out + __popc(kb & lanemask_lt());
      __syncwarp();
      if (keep) bj[p] = key;
      out += __popc(kb);
      ties += __popc(tb);
    }
    for (u32 b = lane; b < HB; b += 32) {
      if (b > t) hj[b] = 0;
      else if (b == t) hj[b] = m;
    }
    if (lane == 0) ws->cnt[j] = out;
    __syncwarp();
  };

  // MINQ (reference batch_search, scan.py:137-143 + :306-318): the score of
  // an entry is its minimum distance over all Qmin queries.
  auto dist_of = [&](u64 x, u64 y, u64 z, int j) -> u32 {
    if (MINQ) {
      u32 best = 0xffffffffu;
      for (u32 t = 0; t < a.Qmin; ++t) {
        const u32 d = dist3(x, y, z, __ldg(a.queries + 3 * (u64)t), __ldg(a.queries + 3 * (u64)t + 1),
                            __ldg(a.queries + 3 * (u64)t + 2));
        best = d < best ? d : best;
      }
      return best;
    }
    return QW >= 2 ? dist3_csa(x, y, z, q0[j], q1[j], q2[j]) : dist3(x, y, z, q0[j], q1[j], q2[j]);
  };

  auto process = [&](const u64 (&A)[E], const u64 (&B)[E], const u64 (&C)[E], u64 it, bool masked) {
    const u64 first = it * (32 * E) + (u64)lane * E;  // local index of this lane's entry 0
    u32 hit = 0;
#pragma unroll
    for (int j = 0; j < QW; ++j) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        u32 d = dist_of(A[e], B[e], C[e], j);
        if (masked && first + e >= a.n) d = DMASKED;
        if (MODE == MODE_HIST) {
          if (d != DMASKED && T[j]) atomicAdd(hist + j * HB + d, 1u);
        } else {
          hit |= (d < T[j]) ? 1u : 0u;
        }
      }
    }
    if (MODE == MODE_HIST) return;
    if (!__any_sync(FULL, hit)) return;
    // slow path: rare once thresholds settle
#pragma unroll 1
    for (int j = 0; j < QW; ++j) {
      u64 x0 = 0, x1 = 0, x2 = 0;
      u32 Tj = 0;
#pragma unroll
      for (int jj = 0; jj < QW; ++jj)
        if (jj == j) { x0 = q0[jj]; x1 = q1[jj]; x2 = q2[jj]; Tj = T[jj]; }
      u32 dd[E];
      u32 m = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        dd[e] = MINQ ? dist_of(A[e], B[e], C[e], 0)
                     : (QW >= 2 ? dist3_csa(A[e], B[e], C[e], x0, x1, x2) : dist3(A[e], B[e], C[e], x0, x1, x2));
        if (masked && first + e >= a.n) dd[e] = DMASKED;
        if (dd[e] < Tj) m |= 1u << e;
      }
      if (!__any_sync(FULL, m)) continue;
      const u32 qi = qg * QW + j;
      const u32 c = __popc(m);
      const u32 incl = warp_incl_scan(c, lane);
      const u32 total = __shfl_sync(FULL, incl, 31);
      if (MODE == MODE_RANGE) {
        u64 base = 0;
        if (lane == 31) base = atomicAdd(a.out_cnt, (u64)total);
        base = __shfl_sync(FULL, base, 31);
        u64 pos = base + incl - c;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (m >> e & 1u) {
            if (pos < a.out_cap) a.out[pos] = ((u64)qi << 48) | make_key(dd[e], a.index_base + first + e);
            ++pos;
          }
        }
        continue;
      }
      // MODE_TOPK: ordered insertion (lane-major, then e == ascending index)
      if (ws->cnt[j] + 32 * E > a.cap) compact(j);
      u32* hj = hist + j * HB;
      u64* bj = wbuf + (u64)j * a.cap;
      const u32 cnt0 = ws->cnt[j];
      u32 pos = cnt0 + incl - c;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (m >> e & 1u) {
          bj[pos++] = make_key(dd[e], a.index_base + first + e);
          atomicAdd(hj + dd[e], 1u);
        }
      }
      __syncwarp();
      if (lane == 0) ws->cnt[j] = cnt0 + total;
      __syncwarp();
      if (cnt0 + total >= a.k) {
        u32 less;
        const u32 t = warp_kth_bin(hj, a.k, lane, &less);
        if (lane == 0) ws->town[j] = t;
        if ((a.flags & 1) || (part % a.pub_every) != 0) {
          // not a publisher: the global bound arrives with the periodic refresh
          __syncwarp();
          setT(j, t < Tj ? t : Tj);
          continue;
        }
        if (!ws->pubd[j]) {
          // first publication: every buffered candidate with d <= t
          for (u32 b = lane; b <= t && b < HB; b += 32) {
            const u32 cb = hj[b];
            if (cb) atomicAdd(gbin(a, qi, b), cb);
          }
        } else {
          // later batches: the newly inserted entries with d <= t, one RED per
          // distinct distance
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const bool hb = (m >> e & 1u) && dd[e] <= t;
            const u32 key = hb ? dd[e] : 0xffffffffu;
            const u32 peers = __match_any_sync(FULL, key);
            if (hb && (u32)(__ffs(peers) - 1) == (u32)lane) atomicAdd(gbin(a, qi, dd[e]), (u32)__popc(peers));
          }
        }
        __syncwarp();
        if (lane == 0) ws->pubd[j] = 1;
        __syncwarp();
        const u32 tt = tighten_tg(a, qi, lane);
        const u32 lim = (tt < T_OPEN ? tt : T_OPEN - 1) + 1;
        const u32 nt = t < lim ? t : lim;
        setT(j, nt < Tj ? nt : Tj);
        __syncwarp();
      }
    }
  };

  constexpr int U = 1;  // iterations per trip
  // loop trips between global-bound refreshes (tg is replicated over L2 slices
  // for small Q, so the single-query kernel can afford one load per trip)
  constexpr int REFRESH = (QW == 1) ? 2 : 8;
  u64 it = it0;
  int since_refresh = 0;
  // The global bound is loaded one refresh period before it is applied, so the
  // load latency hides behind the scan instead of stalling it. Applying it is
  // monotone (T only decreases), and T <= T_own holds since every insertion.
  // (single-query kernel only: the multi-query kernels are compute bound and
  // refresh directly, keeping registers for the query words.)
  u32 tgp = T_OPEN;
  auto prefetch_tg = [&]() {
    if (QW == 1 && qg < a.Q) tgp = *(volatile const u32*)tgrep(a, qg, (u32)(g % a.tg_rep));
  };
  auto apply_tg = [&]() {
    if (QW == 1) {
      const u32 t = (tgp < T_OPEN ? tgp : T_OPEN - 1) + 1;
      T[0] = t < T[0] ? t : T[0];
    } else {
#pragma unroll
      for (int j = 0; j < QW; ++j) refresh_tg(j);
    }
  };
  if (MODE == MODE_TOPK && !(a.flags & 2) && !SL::TMA) prefetch_tg();
  // Only the globally last iteration can hold entries >= n; the main range is
  // scanned without per-entry masking.
  const u64 it_main = it1 < n_full ? it1 : n_full;
  struct Trip {
    u64 A[U][E], B[U][E], C[U][E];
  };
  auto load_trip = [&](Trip& t, u64 i0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const u64 first = (i0 + u) * (32 * E) + (u64)lane * E;
      constexpr u64 TL = CMP ? TILE_CMP : TILE_FULL;
      const char* tb = a.lib + (first / TL) * (CMP ? TILE_BYTES_CMP : TILE_BYTES_FULL);
      const u64 r = first % TL;
      ld_entries(reinterpret_cast<const u64*>(tb) + r, t.A[u]);
      ld_entries(reinterpret_cast<const u64*>(tb + 8 * TL) + r, t.B[u]);
      if (CMP) ld_w2c(reinterpret_cast<const u32*>(tb + 16 * TL) + r, reinterpret_cast<const unsigned char*>(tb + 20 * TL) + r, t.C[u]);
      else ld_entries(reinterpret_cast<const u64*>(tb + 16 * TL) + r, t.C[u]);
    }
  };
  auto run_trip = [&](const Trip& t, u64 i0) {
#pragma unroll
    for (int u = 0; u < U; ++u) process(t.A[u], t.B[u], t.C[u], i0 + u, false);
    if (MODE == MODE_TOPK && !(a.flags & 2) && ++since_refresh == REFRESH) {
      since_refresh = 0;
      apply_tg();
      prefetch_tg();
    }
  };
  if constexpr (SL::TMA) {
    // HBM-bound single-query scan. The warp's tiles stream through a
    // STAGES-deep shared-memory ring filled by the bulk-copy engine (one 3 KB
    // cp.async.bulk per tile, completion on a per-slot mbarrier), so the bytes
    // in flight cost no registers. Lane 0 is the producer: it refills a slot
    // once every lane has consumed it and records the slot's tile index.
    //
    // Tile sequence: the warp's static part of the first dyn_start tiles, then
    // (when dyn_ctr is set) chunks of the remaining tiles claimed from a global
    // counter -- warps that drew more bandwidth take more of the tail. Claims
    // are in increasing order, so each warp still sees ascending indices (the
    // ordered candidate buffers rely on it). The next claim is issued one
    // chunk ahead so its latency hides behind the copies.
    constexpr int S = SL::STAGES;
    constexpr u64 SLOT = SL::SLOT;
    constexpr int SUB = SL::SUB;
    constexpr u64 NONE = ~0ull;
    char* ring = reinterpret_cast<char*>(smem) + SL::ring_off(nwb) + (size_t)wib * S * SLOT;
    u64* bars = reinterpret_cast<u64*>(reinterpret_cast<char*>(smem) + SL::bars_off(nwb)) + wib * S;
    u64* slot_tile = reinterpret_cast<u64*>(reinterpret_cast<char*>(smem) + SL::tiles_off(nwb)) + wib * S;
    const u64 pol = l2_evict_first_policy();
    const u64 n_tiles = (a.iters + SUB - 1) / SUB;  // work unit: one library tile
    const bool dyn = a.dyn_ctr != nullptr;
    const u64 n_static = dyn ? a.dyn_start : n_tiles;
    u64 s_next = part * n_static / a.n_parts, s_end = (part + 1) * n_static / a.n_parts;
    // CTA-dynamic (short scans, one query group): the CTA's warps take the
    // tiles of the CTA's contiguous run one at a time from a shared counter,
    // so warps that draw more bandwidth take more tiles.
    const bool cta_dyn = !dyn && a.n_qg == 1 && !(a.flags & 256);
    u64 cta_lo = 0, cta_hi = 0;
    if (cta_dyn) {
      const u64 w0 = (u64)blockIdx.x * nwb;
      const u64 nv = (a.n_parts - w0) < (u64)nwb ? (a.n_parts - w0) : (u64)nwb;
      cta_lo = w0 * n_tiles / a.n_parts;
      cta_hi = (w0 + nv) * n_tiles / a.n_parts;
      s_next = s_end = 0;
    }
    u64 d_next = 0, d_end = 0;
    u32 pend = 0;
    bool has_pend = false;
    auto claim = [&]() {
      pend = atomicAdd(a.dyn_ctr, 1u);
      has_pend = true;
    };
    auto next_tile = [&]() -> u64 {
      if (cta_dyn) {
        const u64 t = cta_lo + atomicAdd(&s_cta_next, 1u);
        return t < cta_hi ? t : NONE;
      }
      if (s_next < s_end) {
        const u64 t = s_next++;
        if (s_next == s_end && dyn) claim();
        return t;
      }
      if (d_next >= d_end) {
        if (!has_pend) return NONE;
        const u64 c0 = a.dyn_start + (u64)pend * a.dyn_chunk;
        if (c0 >= n_tiles) {
          has_pend = false;
          return NONE;
        }
        d_next = c0;
        d_end = c0 + a.dyn_chunk < n_tiles ? c0 + a.dyn_chunk : n_tiles;
        claim();
      }
      return d_next++;
    };
    auto issue = [&](int st) {  // lane 0 only
      const u64 t = next_tile();
      slot_tile[st] = t;
      if (t != NONE) {
        mbar_expect_tx(&bars[st], (u32)SLOT);
        bulk_g2s_stream(ring + st * SLOT, a.lib + t * SLOT, (u32)SLOT, &bars[st], pol);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[st])) : "memory");
      }
    };
    // first tiles before the dependency wait, when no global claim is needed
    // for them (the tail counter belongs to the previous call until it ends)
    const bool pre = cta_dyn || s_end - s_next > (u64)S;
    if (lane == 0) {
#pragma unroll
      for (int st = 0; st < S; ++st) mbar_init(&bars[st], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (pre) {
#pragma unroll
        for (int st = 0; st < S; ++st) issue(st);
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (MODE == MODE_TOPK && !(a.flags & 2)) prefetch_tg();
    if (lane == 0 && !pre) {
      if (dyn && s_next == s_end) claim();
#pragma unroll
      for (int st = 0; st < S; ++st) issue(st);
    }
    __syncwarp();
#pragma unroll 1
    for (u64 j = 0;; ++j) {
      const int st = (int)(j % S);
      mbar_wait(&bars[st], (u32)(j / S) & 1u);
      const u64 t = *(volatile const u64*)&slot_tile[st];
      if (t == NONE) break;
#ifdef FPS_SCAN_TRACE
      if (j == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_first));
#endif
      const char* tb = ring + st * SLOT;
#pragma unroll
      for (int h = 0; h < SUB; ++h) {
        const u64 i = t * SUB + h;  // 128-entry iteration
        if (SUB > 1 && i >= a.iters) break;
        u64 A[4], B[4], C[4];
        constexpr int TL = CMP ? TILE_CMP : TILE_FULL;
        const u64* w0 = reinterpret_cast<const u64*>(tb) + h * 128 + lane * 4;
        const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(w0);
        const ulonglong2 a1 = *reinterpret_cast<const ulonglong2*>(w0 + 2);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(w0 + TL);
        const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(w0 + TL + 2);
        A[0] = a0.x; A[1] = a0.y; A[2] = a1.x; A[3] = a1.y;
        B[0] = b0.x; B[1] = b0.y; B[2] = b1.x; B[3] = b1.y;
        if constexpr (CMP) {
          // word 2 as a u32 plane (keys 129..160) + a u8 plane (keys 161..166 + 2 pad bits)
          const uint4 lo = *reinterpret_cast<const uint4*>(tb + 16 * TL + 4 * (h * 128 + lane * 4));
          const u32 hi = *reinterpret_cast<const u32*>(tb + 20 * TL + (h * 128 + lane * 4));
          C[0] = (u64)lo.x | ((u64)(hi & 0xffu) << 32);
          C[1] = (u64)lo.y | ((u64)((hi >> 8) & 0xffu) << 32);
          C[2] = (u64)lo.z | ((u64)((hi >> 16) & 0xffu) << 32);
          C[3] = (u64)lo.w | ((u64)(hi >> 24) << 32);
        } else {
          const ulonglong2 c0 = *reinterpret_cast<const ulonglong2*>(w0 + 2 * TL);
          const ulonglong2 c1 = *reinterpret_cast<const ulonglong2*>(w0 + 2 * TL + 2);
          C[0] = c0.x; C[1] = c0.y; C[2] = c1.x; C[3] = c1.y;
        }
        process(*reinterpret_cast<const u64(*)[E]>(A), *reinterpret_cast<const u64(*)[E]>(B),
                *reinterpret_cast<const u64(*)[E]>(C), i, i >= n_full);
      }
      __syncwarp();  // every lane's reads of slot st are complete (values consumed)
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(st);
      }
      if (MODE == MODE_TOPK && !(a.flags & 2) && ++since_refresh == REFRESH) {
        since_refresh = 0;
        apply_tg();
        prefetch_tg();
      }
    }
    it = it1;
  } else {
    for (; it + U <= it_main; it += U) {
      Trip t;
      load_trip(t, it);
      run_trip(t, it);
    }
  }
  for (; it < it1; ++it) {
    u64 A[E], B[E], C[E];
    const u64 first = it * (32 * E) + (u64)lane * E;
    constexpr u64 TL = CMP ? TILE_CMP : TILE_FULL;
    const char* tb = a.lib + (first / TL) * (CMP ? TILE_BYTES_CMP : TILE_BYTES_FULL);
    const u64 r = first % TL;
    ld_entries(reinterpret_cast<const u64*>(tb) + r, A);
    ld_entries(reinterpret_cast<const u64*>(tb + 8 * TL) + r, B);
    if (CMP) ld_w2c(reinterpret_cast<const u32*>(tb + 16 * TL) + r, reinterpret_cast<const unsigned char*>(tb + 20 * TL) + r, C);
    else ld_entries(reinterpret_cast<const u64*>(tb + 16 * TL) + r, C);
    process(A, B, C, it, it >= n_full);
  }

#ifdef FPS_SCAN_TRACE
  if (lane == 0 && g < 16384) {
    u64 tr_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_end));
    g_scan_trace[g * 4 + 0] = tr_start;
    g_scan_trace[g * 4 + 1] = tr_end;
    g_scan_trace[g * 4 + 3] = tr_first;
  }
#endif
  if (MODE == MODE_HIST) {
    __syncwarp();
#pragma unroll 1
    for (int j = 0; j < QW; ++j) {
      const u32 qi = qg * QW + j;
      if (qi >= a.Q) continue;
      for (int b = lane; b < HB; b += 32) {
        const u32 c = hist[j * HB + b];
        if (c) atomicAdd(gbin(a, qi, b), c);
      }
    }
    return;
  }
  if (MODE == MODE_TOPK) {
#pragma unroll 1
    for (int j = 0; j < QW; ++j) {
      const u32 qi = qg * QW + j;
      if (qi >= a.Q) continue;
      // single query: the bound prefetched during the scan (possibly looser
      // than the final one -- select re-filters) saves a load at exit
      const u32 t = (QW == 1) ? tgp : *(volatile const u32*)tgrep(a, qi, (u32)(g % a.tg_rep));
      // survivors (d <= t) counted from the histogram that mirrors the buffer:
      // most warps have none and skip reading their buffer back
      const u32* hj = hist + j * HB;
      u32 c = 0;
      for (u32 b = lane; b < (u32)HB; b += 32) c += b <= t ? hj[b] : 0u;
      c = __reduce_add_sync(FULL, c);
      if (c == 0) continue;
      if (c > a.k) compact(j);  // at most k per warp reach the candidate list
      const u32 n = ws->cnt[j];
      const u64* bj = wbuf + (u64)j * a.cap;
      // survivors: d <= tg (an exact bound on the k-th distance); four
      // independent loads per lane in flight
      for (u32 i0 = 0; i0 < n; i0 += 128) {
        u64 kk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const u32 i = i0 + u * 32 + lane;
          kk[u] = i < n ? bj[i] : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const u32 i = i0 + u * 32 + lane;
          const bool keep = i < n && key_d(kk[u]) <= t;
          const u32 kb = __ballot_sync(FULL, keep);
          const u32 nk = __popc(kb);
          if (nk == 0) continue;
          u32 base = 0;
          if (lane == 0) base = atomicAdd(a.cand_cnt + qi, nk);
          base = __shfl_sync(FULL, base, 0);
          if (keep) a.cand[(u64)qi * a.cand_cap + base + __popc(kb & lanemask_lt())] = kk[u];
        }
      }
    }
  }
#ifdef FPS_SCAN_TRACE
  if (lane == 0 && g < 16384) g_scan_trace[g * 4 + 2] = gtimer();
#endif
}

// ---------------------------------------------------------------------------
// select_kernel: exact top-k per query over the flat survivor list.
// One CTA per query. Resets the per-query scan state (tg, ghist, cand_cnt) so
// the next call starts clean without a memset launch.
// ---------------------------------------------------------------------------
constexpr int SEL_THREADS = 1024;

// Number of keys in s[0, n) smaller than x; four independent counters keep
// the dependent add chain short (shared-memory broadcast reads).
__device__ __forceinline__ u32 rank_in(const u64* s, u32 n, u64 x) {
  u32 r0 = 0, r1 = 0, r2 = 0, r3 = 0, j = 0;
  for (; j + 4 <= n; j += 4) {
    r0 += s[j] < x;
    r1 += s[j + 1] < x;
    r2 += s[j + 2] < x;
    r3 += s[j + 3] < x;
  }
  for (; j < n; ++j) r0 += s[j] < x;
  return r0 + r1 + r2 + r3;
}
// phase timestamps of the last select CTA (debug: FPS_DEBUG prints them)
__device__ unsigned long long g_sel_clock[12];
#define SEL_MARK(i) do { if (threadIdx.x == 0) g_sel_clock[i] = clock64(); } while (0)
constexpr int SEL_ECAP = 4096;      // ties at the threshold held in shared memory
constexpr u32 SEL_RANK_MAX = 2048;  // rank-select / rank-sort (one pass) up to this many keys

__device__ void block_bitonic_sort(u64* s, int n_pow2) {
  for (int size = 2; size <= n_pow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n_pow2 / 2; i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        u64 x = s[lo], y = s[hi];
        if ((x > y) == up) { s[lo] = y; s[hi] = x; }
      }
      __syncthreads();
    }
  }
}

// Barrier over the first nthreads threads of the CTA (named barrier 1).
__device__ __forceinline__ void bar_sync_n(u32 nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Bitonic sort of P keys, one per thread t < P (fully unrolled: every stride
// is a compile-time constant). Strides below 32 exchange through warp
// shuffles, wider ones through a double-buffered shared array with a
// P-thread named barrier (one barrier per stage).
template <u32 P>
__device__ __forceinline__ u64 bitonic_p(u64 key, u32 t, u64* sh) {
  int buf = 0;
#pragma unroll
  for (u32 size = 2; size <= P; size <<= 1) {
    const bool up = (t & size) == 0;
#pragma unroll
    for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
      u64 other;
      if (stride >= 32) {
        u64* b = sh + buf * SEL_THREADS;
        b[t] = key;
        bar_sync_n(P);
        other = b[t ^ stride];
        buf ^= 1;
      } else {
        other = __shfl_xor_sync(FULL, key, stride);
      }
      const bool lt = other < key;
      key = (lt == (((t & stride) == 0) == up)) ? other : key;
    }
  }
  return key;
}

// Small-select path: the survivors (n <= SEL_THREADS, one key per thread in
// `my`) that are within the final bound are sorted by the first p = pow2 >= m
// threads only (p >= 32); when some fall outside the bound they are first
// compacted through shared memory. The k smallest keys (padded with ~0) go to
// out; returns m.
__device__ __forceinline__ u32 select_small(u64 my, u32 n, bool keep, u64* sh, u32* s_wcnt, u32 k, u64* out) {
  const u32 t = threadIdx.x, lane = t & 31, w = t >> 5;
  const u32 m = (u32)__syncthreads_count(keep);
  u64 key = keep ? my : ~0ull;
  if (m != n) {  // uniform: survivors are not exactly threads [0, n) -- compact
    const u32 bal = __ballot_sync(FULL, keep);
    if (lane == 0) s_wcnt[w] = __popc(bal);
    __syncthreads();
    u32 off = 0;
#pragma unroll
    for (int i = 0; i < SEL_THREADS / 32; ++i) off += (i < (int)w) ? s_wcnt[i] : 0;
    u64* comp = sh + 2 * SEL_THREADS;
    if (keep) comp[off + __popc(bal & lanemask_lt())] = my;
    __syncthreads();
    key = t < m ? comp[t] : ~0ull;
  }
#ifdef FPS_SEL_PROBE
  if (t == 0) { g_sel_clock[10] = key; SEL_MARK(8); }
#endif
  u32 p = 32;
  while (p < m) p <<= 1;
  if (t < p) {
    switch (p) {
      case 32: key = bitonic_p<32>(key, t, sh); break;
      case 64: key = bitonic_p<64>(key, t, sh); break;
      case 128: key = bitonic_p<128>(key, t, sh); break;
      case 256: key = bitonic_p<256>(key, t, sh); break;
      case 512: key = bitonic_p<512>(key, t, sh); break;
      default: key = bitonic_p<1024>(key, t, sh); break;
    }
#ifdef FPS_SEL_PROBE
    if (t == 0) { g_sel_clock[10] = key; SEL_MARK(9); }
#endif
    if (t < k) out[t] = key;
  }
  for (u32 i = p + t; i < k; i += SEL_THREADS) out[i] = ~0ull;
  return m;
}

// Host-visible completion (single-query host path, one CTA): the results
// written by every thread, then the sequence number, at system scope.
__device__ __forceinline__ void post_done(u32* done_flag, u32 done_seq) {
  if (!done_flag) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *(volatile u32*)done_flag = done_seq;
  }
}

__global__ void __launch_bounds__(SEL_THREADS) select_kernel(u64* cand, u32* cand_cnt, u64 cand_cap, u32* tg,
                                                             u32* ghist, u32 gstride, u32 tg_rep, u32 k,
                                                             u64* out_keys, u32* out_cnt, int reset,
                                                             u32* dyn_ctr, u32* done_flag, u32 done_seq,
                                                             const u32* gate, u32* ovf) {
  extern __shared__ u64 ssel[];  // [k_pow2] result + [SEL_ECAP] ties
  __shared__ u32 hist[256];
  __shared__ u32 s_nres, s_ntie, s_T, s_m;
  __shared__ u64 s_cut;
  // the next call's scan may be launched as a programmatic dependent: let its
  // CTAs become resident now (they wait for this grid to finish)
  asm volatile("griddepcontrol.launch_dependents;");
  const u32 q = blockIdx.x;
  const u64* c = cand + (u64)q * cand_cap;
  // launched as a programmatic dependent of the scan: wait for its results
  __shared__ u32 s_wcnt[SEL_THREADS / 32];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (gate && *(volatile const u32*)gate == 0) return;  // gated off: the scan did nothing either
  SEL_MARK(0);
#ifdef FPS_SCAN_TRACE
  if (threadIdx.x == 0 && q == 0) g_mark[2] = gtimer();
#endif
  // speculative first-slot read, independent of the count load
  const u64 my = threadIdx.x < cand_cap ? c[threadIdx.x] : ~0ull;
  const u32 n = cand_cnt[q];
  if (n > cand_cap) {
    // a candidate list overflowed its capacity (tensor-core path; its slots
    // are not all written): flag it for the device-side fallback pass, which
    // recomputes the batch, and leave an empty, clean result
    if (ovf && threadIdx.x == 0) atomicOr(ovf, 1u);
    for (u32 i = threadIdx.x; i < k; i += blockDim.x) out_keys[(u64)q * k + i] = ~0ull;
    if (threadIdx.x == 0) out_cnt[q] = 0;
    if (reset) {
      for (int i = threadIdx.x; i < HB; i += blockDim.x) ghist[((u64)q * HB + i) * gstride] = 0;
      for (u32 r = threadIdx.x; r < tg_rep; r += blockDim.x) tg[((u64)q * tg_rep + r) * gstride] = T_OPEN;
      if (threadIdx.x == 0) cand_cnt[q] = 0;
      if (dyn_ctr && q == 0 && threadIdx.x == 0) *dyn_ctr = 0;
    }
    post_done(done_flag, done_seq);
    return;
  }
  const u32 bound = tg[(u64)q * tg_rep * gstride];  // every replica holds the same bound
#ifdef FPS_SEL_PROBE
  if (threadIdx.x == 0) g_sel_clock[1] = my + n + bound;  // wait for the loads
  SEL_MARK(2);
#endif
  u32 m_small = 0;
  if (n <= (u32)SEL_THREADS) {
    // common case: every survivor fits one key per thread -- sort the ones
    // within the bound (unique keys: the first k sorted are the answer)
    m_small = select_small(my, n, threadIdx.x < n && key_d(my) <= bound, ssel, s_wcnt, k, out_keys + (u64)q * k);
    SEL_MARK(3);
#ifdef FPS_SEL_PROBE
    if (threadIdx.x == 0) {
      g_sel_clock[5] = g_sel_clock[0] + m_small;
      g_sel_clock[6] = g_sel_clock[0] + bound;
      g_sel_clock[7] = g_sel_clock[0] + n;
    }
#endif
    __syncthreads();
  }
  if (n <= (u32)SEL_THREADS) {
    if (threadIdx.x == 0) out_cnt[q] = m_small < k ? m_small : k;
#ifdef FPS_SCAN_TRACE
    if (threadIdx.x == 0 && q == 0) g_mark[3] = gtimer();
#endif
    SEL_MARK(11);
    if (reset) {
      for (int i = threadIdx.x; i < HB; i += blockDim.x) ghist[((u64)q * HB + i) * gstride] = 0;
      for (u32 r = threadIdx.x; r < tg_rep; r += blockDim.x) tg[((u64)q * tg_rep + r) * gstride] = T_OPEN;
      if (threadIdx.x == 0) cand_cnt[q] = 0;
      if (dyn_ctr && q == 0 && threadIdx.x == 0) *dyn_ctr = 0;
    }
    post_done(done_flag, done_seq);
    return;
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) { s_nres = 0; s_ntie = 0; }
  __syncthreads(); SEL_MARK(1);
  const int lane = threadIdx.x & 31;
  // uniform trip counts so every warp-collective below sees the full warp
  for (u32 base = 0; base < n; base += blockDim.x) {
    const u32 i = base + threadIdx.x;
    const u32 d = i < n ? key_d(c[i]) : 0xffffu;
    const bool valid = i < n && d <= bound;
    // hot bins (many candidates share a distance): one shared atomic per
    // distinct distance per warp instead of one per candidate
    const u32 peers = __match_any_sync(FULL, valid ? d : 0xffffu);
    if (valid && (__ffs(peers) - 1) == lane) atomicAdd(&hist[d], (u32)__popc(peers));
  }
  __syncthreads(); SEL_MARK(2);
  if (threadIdx.x < 32) {
    // find T: smallest t with cum >= k (scan 256 bins, 8 per lane)
    int lane = threadIdx.x;
    u32 h[8], s = 0;
    for (int i = 0; i < 8; ++i) { h[i] = hist[lane * 8 + i]; s += h[i]; }
    u32 incl = warp_incl_scan(s, lane);
    u32 bal = __ballot_sync(FULL, incl >= k);
    if (bal == 0) {
      if (lane == 0) { s_T = 256; s_m = 0; }
    } else {
      int src = __ffs(bal) - 1;
      if (lane == src) {
        u32 cc = incl - s;
        for (int i = 0; i < 8; ++i) {
          if (cc + h[i] >= k) { s_T = lane * 8 + i; s_m = k - cc; break; }
          cc += h[i];
        }
      }
    }
  }
  __syncthreads(); SEL_MARK(3);
  const u32 T = s_T, m = s_m;
  u64* res = ssel;
  int kp = 1;
  while (kp < (int)k) kp <<= 1;
  u64* ties = ssel + kp;
  const u32 ntie_total = T < 256 ? hist[T] : 0;
  const bool ties_fit = ntie_total <= SEL_ECAP;
  for (u32 base = 0; base < n; base += blockDim.x) {
    const u32 i = base + threadIdx.x;
    const u64 key = i < n ? c[i] : ~0ull;
    const u32 d = key_d(key);
    const bool ok = i < n && d <= bound;
    const bool take = ok && d < T;
    const bool tie = ok && d == T && ties_fit;
    // warp-aggregated appends (one shared atomic per warp per list)
    const u32 tb = __ballot_sync(FULL, take), eb = __ballot_sync(FULL, tie);
    u32 rb = 0, ebase = 0;
    if (lane == 0) {
      if (tb) rb = atomicAdd(&s_nres, (u32)__popc(tb));
      if (eb) ebase = atomicAdd(&s_ntie, (u32)__popc(eb));
    }
    rb = __shfl_sync(FULL, rb, 0);
    ebase = __shfl_sync(FULL, ebase, 0);
    if (take) res[rb + __popc(tb & lanemask_lt())] = key;
    if (tie) ties[ebase + __popc(eb & lanemask_lt())] = key;
  }
  __syncthreads(); SEL_MARK(4);
  if (T < 256 && m > 0) {
    if (ntie_total <= m) {
      // every tie is in the answer
      for (u32 i = threadIdx.x; i < ntie_total; i += blockDim.x) res[s_nres + i] = ties[i];
      __syncthreads();
      if (threadIdx.x == 0) s_nres += ntie_total;
    } else if (ties_fit && ntie_total <= SEL_RANK_MAX) {
      // rank selection: keys are unique, so the m smallest have ranks 0..m-1
      const u32 base = s_nres;
      for (u32 i = threadIdx.x; i < ntie_total; i += blockDim.x) {
        const u32 r = rank_in(ties, ntie_total, ties[i]);
        if (r < m) res[base + r] = ties[i];
      }
      __syncthreads();
      if (threadIdx.x == 0) s_nres = base + m;
    } else if (ties_fit) {
      int tp = 1;
      while (tp < (int)ntie_total) tp <<= 1;
      for (int i = ntie_total + threadIdx.x; i < tp; i += blockDim.x) ties[i] = ~0ull;
      __syncthreads();
      block_bitonic_sort(ties, tp);
      const u32 base = s_nres;
      for (u32 i = threadIdx.x; i < m; i += blockDim.x) res[base + i] = ties[i];
      __syncthreads();
      if (threadIdx.x == 0) s_nres = base + m;
    } else {
      // radix select on the index bits of the ties: find the m-th smallest
      u64 prefix = 0;
      u32 need = m;
      for (int shift = IDX_BITS - 8; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const u64 hi_mask = (shift + 8 >= IDX_BITS) ? 0 : (IDX_MASK & ~((1ull << (shift + 8)) - 1));
        for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
          u64 key = c[i];
          if (key_d(key) != T) continue;
          u64 idx = key & IDX_MASK;
          if ((idx & hi_mask) != prefix) continue;
          atomicAdd(&hist[(idx >> shift) & 0xff], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          u32 cc = 0;
          for (int bb = 0; bb < 256; ++bb) {
            if (cc + hist[bb] >= need) { s_cut = prefix | ((u64)bb << shift); s_m = need - cc; break; }
            cc += hist[bb];
          }
        }
        __syncthreads();
        prefix = s_cut;
        need = s_m;
      }
      // prefix is now the m-th smallest tie index: keep ties with idx <= prefix
      for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
        u64 key = c[i];
        if (key_d(key) == T && (key & IDX_MASK) <= prefix) res[atomicAdd(&s_nres, 1u)] = key;
      }
    }
  }
  __syncthreads(); SEL_MARK(5);
  const u32 nres = s_nres;
  u64* out = out_keys + (u64)q * k;
  if (nres <= SEL_RANK_MAX) {
    // final order by rank (unique keys): one pass, no shared-memory sort
    for (u32 i = threadIdx.x; i < nres; i += blockDim.x) out[rank_in(res, nres, res[i])] = res[i];
    for (u32 i = nres + threadIdx.x; i < k; i += blockDim.x) out[i] = ~0ull;
  } else {
    for (int i = nres + threadIdx.x; i < kp; i += blockDim.x) res[i] = ~0ull;
    __syncthreads();
    block_bitonic_sort(res, kp);
    for (u32 i = threadIdx.x; i < k; i += blockDim.x) out[i] = i < nres ? res[i] : ~0ull;
  }
  if (threadIdx.x == 0) out_cnt[q] = nres;
  SEL_MARK(11);
  if (reset) {
    for (int i = threadIdx.x; i < HB; i += blockDim.x) ghist[((u64)q * HB + i) * gstride] = 0;
    for (u32 r = threadIdx.x; r < tg_rep; r += blockDim.x) tg[((u64)q * tg_rep + r) * gstride] = T_OPEN;
    if (threadIdx.x == 0) cand_cnt[q] = 0;
    if (dyn_ctr && q == 0 && threadIdx.x == 0) *dyn_ctr = 0;
  }
  post_done(done_flag, done_seq);
}

// ---------------------------------------------------------------------------
// merge_kernel: G per-shard sorted top-k lists -> global top-k per query
// (merge_topk, scan.py:225-236). Keys are unique (disjoint index ranges), so
// rank(x) = own position + sum over other lists of lower_bound(x).
// in_keys: [G][Q][k], in_cnt: [G][Q]; out_keys: [Q][k], out_cnt: [Q].
// ---------------------------------------------------------------------------
__global__ void merge_kernel(const u64* in_keys, const u32* in_cnt, u32 G, u32 Q, u32 k, u64* out_keys,
                             u32* out_cnt) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 total = (u64)G * Q * k;
  if (t < Q) {
    u32 s = 0;
    for (u32 gg = 0; gg < G; ++gg) s += in_cnt[(u64)gg * Q + t];
    out_cnt[t] = s < k ? s : k;
    for (u32 i = s; i < k; ++i) out_keys[t * k + i] = ~0ull;
  }
  if (t >= total) return;
  const u32 i = (u32)(t % k);
  const u32 q = (u32)((t / k) % Q);
  const u32 gg = (u32)(t / ((u64)k * Q));
  if (i >= in_cnt[(u64)gg * Q + q]) return;
  const u64 x = in_keys[((u64)gg * Q + q) * k + i];
  u64 rank = i;
  for (u32 h = 0; h < G; ++h) {
    if (h == gg) continue;
    const u64* L = in_keys + ((u64)h * Q + q) * k;
    u32 lo = 0, hi = in_cnt[(u64)h * Q + q];
    while (lo < hi) {
      u32 mid = (lo + hi) >> 1;
      if (L[mid] < x) lo = mid + 1; else hi = mid;
    }
    rank += lo;
  }
  if (rank < k) out_keys[(u64)q * k + rank] = x;
}

// ---------------------------------------------------------------------------
// Multi-device merges (fps_group_*): the same rank arithmetic as merge_kernel,
// but each shard's list is reached through its own pointer -- a peer-device
// pointer read over NVLink (fused gather + merge, no copy) or a slot of a
// root-side gather buffer filled by NCCL / peer copies.
// ---------------------------------------------------------------------------
constexpr int GROUP_MAX = 32;
struct ShardLists {
  const u64* keys[GROUP_MAX];  // top-k: [Q][k] sorted keys; range: a sorted run
  const u32* cnt[GROUP_MAX];   // top-k: [Q] counts (unused for runs)
  u64 len[GROUP_MAX];          // range: run lengths
  u64 off[GROUP_MAX];          // range: exclusive prefix of len
};

// Per-query top-k of G shard lists (merge_topk, scan.py:225-236): keys are
// unique across shards (disjoint index ranges), so a key's merged rank is its
// own position plus its lower bound in every other list.
__global__ void merge_lists_kernel(const ShardLists s, u32 G, u32 Q, u32 k, u64* __restrict__ out_keys,
                                   u32* __restrict__ out_cnt) {
  const u64 total = (u64)G * Q * k;
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < total + Q; t += (u64)gridDim.x * blockDim.x) {
    if (t >= total) {  // one thread per query: count and padding
      const u32 q = (u32)(t - total);
      u32 c = 0;
      for (u32 g = 0; g < G; ++g) c += s.cnt[g][q];
      out_cnt[q] = c < k ? c : k;
      for (u32 i = c; i < k; ++i) out_keys[(u64)q * k + i] = ~0ull;
      continue;
    }
    const u32 g = (u32)(t / ((u64)Q * k));
    const u32 q = (u32)((t / k) % Q);
    const u32 i = (u32)(t % k);
    if (i >= s.cnt[g][q]) continue;
    const u64 x = s.keys[g][(u64)q * k + i];
    u64 rank = i;
    for (u32 h = 0; h < G && rank < k; ++h) {
      if (h == g) continue;
      const u64* L = s.keys[h] + (u64)q * k;
      u32 lo = 0, hi = s.cnt[h][q];
      while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (L[mid] < x) lo = mid + 1; else hi = mid;
      }
      rank += lo;
    }
    if (rank < k) out_keys[(u64)q * k + rank] = x;
  }
}

// Range hits: G sorted runs of unique (q << 48 | d << 40 | index) keys ->
// one sorted array (a merge by rank, no re-sort of the union).
__global__ void merge_runs_kernel(const ShardLists s, u32 G, u64* __restrict__ out) {
  const u64 total = s.off[G - 1] + s.len[G - 1];
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (u64)gridDim.x * blockDim.x) {
    u32 g = 0;
    while (g + 1 < G && t >= s.off[g + 1]) ++g;
    const u64 i = t - s.off[g];
    const u64 x = s.keys[g][i];
    u64 rank = i;
    for (u32 h = 0; h < G; ++h) {
      if (h == g) continue;
      const u64* L = s.keys[h];
      u64 lo = 0, hi = s.len[h];
      while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (L[mid] < x) lo = mid + 1; else hi = mid;
      }
      rank += lo;
    }
    out[rank] = x;
  }
}

// ---------------------------------------------------------------------------
// Library ingestion
// ---------------------------------------------------------------------------
// Device view of the tiled library for ingestion / export kernels.
struct PlanesOut {
  char* base;
  int compact;
  __device__ __forceinline__ u64 te() const { return tile_entries(compact); }
  __device__ __forceinline__ char* tile(u64 i) const { return base + (i / te()) * tile_bytes(compact); }
  __device__ __forceinline__ void put(u64 i, u64 a, u64 b, u64 c) const {
    char* t = tile(i);
    const u64 T = te(), r = i % T;
    reinterpret_cast<u64*>(t)[r] = a;
    reinterpret_cast<u64*>(t + 8 * T)[r] = b;
    if (compact) {
      reinterpret_cast<u32*>(t + 16 * T)[r] = (u32)c;
      reinterpret_cast<unsigned char*>(t + 20 * T)[r] = (unsigned char)(c >> 32);
    } else {
      reinterpret_cast<u64*>(t + 16 * T)[r] = c;
    }
  }
  __device__ __forceinline__ void get(u64 i, u64& a, u64& b, u64& c) const {
    const char* t = tile(i);
    const u64 T = te(), r = i % T;
    a = reinterpret_cast<const u64*>(t)[r];
    b = reinterpret_cast<const u64*>(t + 8 * T)[r];
    c = compact ? ((u64)reinterpret_cast<const u32*>(t + 16 * T)[r] |
                   ((u64)reinterpret_cast<const unsigned char*>(t + 20 * T)[r] << 32))
                : reinterpret_cast<const u64*>(t + 16 * T)[r];
  }
};

// rows with `stride` u64 per row, fingerprint words at columns [col0, col0+3)
// (FPS1 record view: stride 4, col0 1 — scan.py:169; row-major words: 3, 0).
// bad_padding counts rows that set bits 38.. of word 2 (keys beyond 166).
__global__ void rows_to_planes(const u64* __restrict__ rows, u64 n_rows, int stride, int col0, PlanesOut o,
                               u64 dst_off, u32* bad_padding) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += (u64)gridDim.x * blockDim.x) {
    const u64* r = rows + i * stride + col0;
    const u64 a = r[0], b = r[1], c = r[2];
    o.put(dst_off + i, a, b, c);
    if (bad_padding && (c >> 38)) atomicAdd(bad_padding, 1u);
  }
}

// Count full-layout entries whose word 2 uses bits 40.. (they need 24 B/entry).
__global__ void count_wide(const u64* __restrict__ w2, u64 n, u32* wide) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    if (w2[i] >> 40) atomicAdd(wide, 1u);
}

// Library entries that use bits 40.. of word 2 (they need the 24 B tiles).
__global__ void count_wide_lib(PlanesOut src, u64 n, u32* wide) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 a, b, c;
    src.get(i, a, b, c);
    if (c >> 40) atomicAdd(wide, 1u);
  }
}

// Re-tile a library (24 B tiles -> 21 B tiles after loading, when it fits).
__global__ void retile_kernel(PlanesOut src, PlanesOut dst, u64 n) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 a, b, c;
    src.get(i, a, b, c);
    dst.put(i, a, b, c);
  }
}

// Three device planes (full layout) -> library planes.
__global__ void planes_to_planes(const u64* __restrict__ a, const u64* __restrict__ b, const u64* __restrict__ c,
                                 u64 n, PlanesOut o) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    o.put(i, a[i], b[i], c[i]);
}

// Library entries [start, start + m) back to rows (checking / export).
__global__ void planes_to_rows(PlanesOut o, u64 start, u64 m, u64* __restrict__ rows) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
    u64 x, y, z;
    o.get(start + i, x, y, z);
    rows[3 * i + 0] = x;
    rows[3 * i + 1] = y;
    rows[3 * i + 2] = z;
  }
}

__global__ void scatter_rows(const u64* __restrict__ idx, const u64* __restrict__ rows, u64 m, PlanesOut o,
                             u32* wide) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
    const u64 c = rows[3 * i + 2];
    if (o.compact && (c >> 40)) {
      atomicAdd(wide, 1u);
      continue;
    }
    o.put(idx[i], rows[3 * i + 0], rows[3 * i + 1], c);
  }
}

__device__ __forceinline__ u64 splitmix64_fin(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct GenArgs {
  PlanesOut o;
  u64 n;
  u64 start;     // global index of entry 0
  u64 seed_key;
  u32 thr[166];  // key j set iff u32 < thr[j-1]  (thr as 32-bit, thr_hi marks p == 1)
  unsigned char thr_hi[166];
};

// Synthetic library: key j set independently with probability
// p_j (p_j ~ Beta(0.6, 2), p_1 = 0 drawn on the host). Counter-based, so any
// chunk of the stream is reproducible; numpy twin: oracle generate_words.
__global__ void gen_kernel(const GenArgs a) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (u64)gridDim.x * blockDim.x) {
    const u64 gi = a.start + i;
    u64 w[3] = {0, 0, 0};
#pragma unroll 4
    for (int c = 0; c < 83; ++c) {
      const u64 z = a.seed_key + (gi * 83 + c + 1) * 0x9E3779B97F4A7C15ull;
      const u64 h = splitmix64_fin(z);
      const int j0 = 2 * c, j1 = 2 * c + 1;  // 0-based key slots
      const u32 lo = (u32)h, hi = (u32)(h >> 32);
      const bool b0 = a.thr_hi[j0] || lo < a.thr[j0];
      const bool b1 = a.thr_hi[j1] || hi < a.thr[j1];
      w[j0 >> 6] |= (u64)b0 << (j0 & 63);
      w[j1 >> 6] |= (u64)b1 << (j1 & 63);
    }
    a.o.put(i, w[0], w[1], w[2]);
  }
}

// Min-over-queries merge of Q per-query top-k lists (batch_search on the
// batched kernel): every listed entry becomes (index << 8 | distance) so one
// sort groups an entry's appearances with its smallest distance first.
__global__ void minq_flip(const u64* __restrict__ keys, const u32* __restrict__ cnt, u32 Q, u32 k,
                          u64* __restrict__ out) {
  const u64 n = (u64)Q * k;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u32 q = (u32)(i / k), r = (u32)(i % k);
    const u64 key = keys[i];
    out[i] = r < cnt[q] ? (((key & IDX_MASK) << 8) | key_d(key)) : ~0ull;
  }
}
// After that sort: keep each entry's first (minimum-distance) appearance as a
// (distance << 40 | index) key, everything else ~0; *firsts counts the kept.
__global__ void minq_first(const u64* __restrict__ sorted, u64 n, u64* __restrict__ out, u32* firsts) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 x = sorted[i];
    const bool first = x != ~0ull && (i == 0 || (sorted[i - 1] >> 8) != (x >> 8));
    out[i] = first ? make_key((u32)(x & 0xffu), x >> 8) : ~0ull;
    if (first) atomicAdd(firsts, 1u);
  }
}

// The first min(*firsts, k) keys of the re-sorted min-merge output -> out[k], *cnt.
__global__ void minq_emit(const u64* __restrict__ sorted, const u32* __restrict__ firsts, u32 k, u64* __restrict__ out,
                          u32* __restrict__ cnt) {
  const u32 m = min(*firsts, k);
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) out[i] = i < m ? sorted[i] : ~0ull;
  if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = m;
}

// Truncate sorted range output to the first k per query (large-k path).
__global__ void truncate_kernel(const u64* sorted, const u64* seg_off, u32 Q, u32 k, u64* out_keys, u32* out_cnt) {
  const u32 q = blockIdx.x;
  if (q >= Q) return;
  const u64 s = seg_off[q], e = seg_off[q + 1];
  const u64 n = e - s;
  const u32 r = n < k ? (u32)n : k;
  for (u32 i = threadIdx.x; i < k; i += blockDim.x)
    out_keys[(u64)q * k + i] = i < r ? (sorted[s + i] & ((1ull << 48) - 1)) : ~0ull;
  if (threadIdx.x == 0) out_cnt[q] = r;
}

}  // namespace fps
