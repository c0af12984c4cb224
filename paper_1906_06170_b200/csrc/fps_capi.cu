// fps_capi.cu — host side of libfpsgpu.so: the C ABI declared in include/fps.h.
//
// Owns the HBM-resident SoA library (three u64 planes) and the per-call
// scratch, launches the sm_100a kernels of fps_kernels.cuh, and maps CUDA
// failures to status codes. Reference interface replaced: fpscan.scan
// (search / batch_search / _search_multi / merge_topk, scan.py:225-318) plus
// the per-search shard streaming of scan.py:158-170 (the library is uploaded
// once instead of being re-read per search).
#include <cub/device/device_radix_sort.cuh>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fps.h"
#include "fps_bitslice.cuh"
#include "fps_kernels.cuh"
#include "fps_planeq.cuh"
#include "fps_mma.cuh"
#include "fps_mma4.cuh"
#include "fps_mma4x.cuh"

using fps::u32;
using fps::u64;

namespace {

thread_local std::string g_err;
// bumped by every device (re)allocation: CUDA graphs captured before it may
// hold stale pointers and are re-captured
std::atomic<u64> g_alloc_gen{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) {                                                                    \
      return fail(e_ == cudaErrorMemoryAllocation ? FPS_ENOMEM : FPS_ECUDA,                     \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                          \
    }                                                                                           \
  } while (0)

// launch check that names the kernel in the error message
#define LAUNCH_CHECK(name)                                                                      \
  do {                                                                                          \
    cudaError_t e_ = cudaGetLastError();                                                        \
    if (e_ != cudaSuccess) return fail(FPS_ECUDA, std::string(name) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int WPB = 8;  // warps per CTA in the scan kernels
constexpr u32 KMAX_FUSED = 1024;

// Device / pinned-host buffers own their allocation (move-only RAII): every
// member of a handle and every local scratch buffer is released when it goes
// out of scope. Release happens with the owning device current (destroy()
// and every entry point hold a DeviceGuard).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  int ensure(size_t want) {
    if (want <= bytes) return FPS_OK;
    release();
    size_t b = std::max<size_t>(want, 256);
    cudaError_t e = cudaMalloc(&p, b);
    g_alloc_gen++;
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return fail(FPS_ENOMEM, std::string("cudaMalloc(") + std::to_string(b) + "): " + cudaGetErrorString(e));
    }
    bytes = b;
    return FPS_OK;
  }
  void release() {
    if (p) {
      cudaFree(p);
      g_alloc_gen++;
    }
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  HostBuf(HostBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  ~HostBuf() { release(); }
  int ensure(size_t want) {
    if (want <= bytes) return FPS_OK;
    release();
    size_t b = std::max<size_t>(want, 4096);
    cudaError_t e = cudaMallocHost(&p, b);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return fail(FPS_ENOMEM, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
    }
    bytes = b;
    return FPS_OK;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

struct Config {
  int qw, e;
  u32 n_qg;
  u64 n_parts, iters, warps;
  u32 cap;
  u64 cand_cap;
  size_t smem;
  int grid;
};

}  // namespace

struct fps_lib {
  int device = 0;
  int sms = 148;
  u64 n = 0, n_alloc = 0, index_base = 0;
  // tiles of 128 entries (fps_kernels.cuh TILE_BYTES_*); compact (21 B / entry)
  // unless some entry uses bits 40.. of word 2, then full (24 B / entry)
  bool compact = false;
  char* mem = nullptr;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::atomic<u64> launches{0};
  // top-k state that must start clean (tg = 255, ghist = 0, cand_cnt = 0);
  // select_kernel restores it after every call
  DevBuf tg, ghist, cand_cnt;
  DevBuf dyn;  // tail-claim counter of the bulk-copy single-query scan (reset by select_kernel)
  u32 state_q = 0;
  DevBuf buf, cand, queries, keys, cnt, radius, rkeys, rcount, sort_tmp, sort_out, seg;
  // bit-plane copy of the library for the multi-query scans (built on first use)
  DevBuf bs, bsq;
  DevBuf mq;  // min-over-queries merge scratch (fps_topk_min on the batched kernel)
  int bs_state = 0;  // 0 unbuilt, 1 built, -1 ineligible (pad bits set)
  double derived_ms = 0;  // host time spent building derived copies (plane-major, bit-plane)
  // plane-major copy for the single-query plane scan (built on first use)
  DevBuf pm, pm_perm, pm_meta;
  int pm_state = 0;  // as bs_state
  bool pm_sorted = false;  // pm holds the popcount-sorted copy (pm_perm, pm_meta valid)
  // plane-scan knobs (FPS_PQ_*), read from the environment once per handle:
  // getenv is a linear scan of the environment, and this is the per-call path
  struct PqKnobs {
    bool init = false, sorted = false;
    int bpl = 0, warps = 8, stages = 2, smem_kb = 210, copy = 1, refresh = 0, wave_pct = 50, wave_ns = 8000, shape = 1;
  } pqk;
  u32 done_seq = 0;  // completion sequence of the single-query host path
  u32 pq_hint_np = 0;  // stage positions of the next device-resident single query (fps_query_hint; 0: unknown)
  // tensor-core multi-query path (fps_mma.cuh, FPS_MMA=1): |a| per entry and per-call operands
  DevBuf mm_bop, mm_ucol, mm_qpop, mm_tq, mm_qcol, mm_keys, mm_sorted, mm_tmp, mm_priv;
  DevBuf mm_ovf;  // candidate-list overflow flag of the tensor-core top-k (gates its fallback pass)
  // fp4 operand copy of the library for the tensor-core scan (fps_mma4x.cuh, built on first use)
  DevBuf mq4x;
  int mq4x_state = 0;  // as bs_state (-1: not compact, or no memory for it)
  alignas(64) CUtensorMap mq4x_map;  // the copy as rows of 256 B for TMA tensor loads
  u64 pm_stride = 0;  // u32 words per plane
  HostBuf h_stage;
  HostBuf h_range[2];     // pinned staging of range results (fps_range_fetch)
  u64 range_pending = 0;  // sorted range keys left on the device by fps_range_begin
  // mapped pinned result buffer of the single-query host path (written by the
  // select kernel over PCIe: no D2H copy) and its device alias
  void* hmap = nullptr;
  void* dmap = nullptr;
  size_t hmap_bytes = 0;
  // optional per-launch timing of the scan kernel (bench roofline evidence)
  int last_kernel = 0;  // fps_last_kernel
  int last_mma_kind = 0;  // fps_last_mma_kind: operand kind of the last tensor-core scan (1 + MmaKind)
  // host-API top-k calls replayed as one CUDA graph per (Q, k):
  // H2D queries -> scan -> select -> D2H, captured once
  struct TopkGraph {
    u32 Q = 0, k = 0;
    u64 gen = 0;
    bool mma = false;  // captured on the tensor-core path (re-captured when the choice changes)
    int kernel = 0;    // last_kernel of the captured path
    cudaGraphExec_t exec = nullptr;
    HostBuf hq, hout;
    DevBuf dq, dkeys, dcnt;
  };
  std::vector<TopkGraph*> graphs;
  bool timing = false;
  bool timing_suspend = false;  // helper passes (e.g. the bit-slice seed) are not timed
  bool timing_continue = false; // the next timed launch belongs to the previous one's scan (one count)
  size_t ev_groups = 0;         // timed scans (a scan may be several launches)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  cudaEvent_t ev_join = nullptr;  // orders the handle's stream after a caller's stream
  // shard of a multi-device group (fps_group_*): this shard's per-call result
  // block on its own device, and the event the root device waits on
  DevBuf gout;
  cudaEvent_t ev_done = nullptr;
  size_t ev_used = 0;
  fps::PlanesOut out() const { return fps::PlanesOut{mem, compact ? 1 : 0}; }
  u64 bytes_per_entry() const { return compact ? 21 : 24; }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device (per-context)
// attribute: remember, per (kernel, device), the largest opt-in set so far,
// so handles on several devices in one process all launch with it.
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, size_t> g_attr;

cudaError_t smem_optin(const void* func, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  size_t& have = g_attr[{func, dev}];
  if (have >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) have = smem;
  return e;
}

template <int QW, int E, int MODE, bool CMP = false>
size_t scan_smem() {
  return fps::ScanSmem<QW, E, MODE, CMP>::total(WPB);
}

template <int QW, int E, int MODE, bool MINQ = false, bool CMP = false>
int max_ctas_per_sm() {
  static int cached = 0;
  size_t smem = scan_smem<QW, E, MODE, CMP>();
  auto* k = fps::scan_kernel<QW, E, MODE, MINQ, CMP>;
  smem_optin((const void*)k, smem);  // per device: also before a cached return
  if (cached) return cached;
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, WPB * 32, smem);
  cached = std::max(1, blocks);
  return cached;
}

void pick_shape(u32 Q, int* qw, int* e) {
  if (Q == 1) { *qw = 1; *e = 4; }
  else if (Q == 2) { *qw = 2; *e = 2; }
  else if (Q <= 4) { *qw = 4; *e = 2; }
  else { *qw = 8; *e = 2; }
}

template <int QW, int E, int MODE, bool MINQ = false, bool CMP = false>
Config make_config(const fps_lib* L, u32 Q, u32 k, u64 n_prefix = 0) {
  Config c{};
  c.qw = QW;
  c.e = E;
  c.n_qg = (Q + QW - 1) / QW;
  const u64 n = n_prefix ? n_prefix : L->n;
  c.iters = (n + 32 * E - 1) / (32 * E);
  const u64 slots = (u64)L->sms * max_ctas_per_sm<QW, E, MODE, MINQ, CMP>() * WPB;
  u64 parts = std::max<u64>(1, slots / c.n_qg);
  const u64 min_iters = (QW == 1) ? 8 : 2;  // keep per-warp parts long enough to amortise warm-up
  parts = std::min<u64>(parts, std::max<u64>(1, c.iters / min_iters));
  c.n_parts = parts;
  c.warps = (u64)c.n_qg * parts;
  c.grid = (int)((c.warps + WPB - 1) / WPB);
  c.cap = 0;
  if (MODE == fps::MODE_TOPK) {
    u32 cap = std::max<u32>(2 * k + 32 * E, k + 256);
    cap = (cap + 31) / 32 * 32;
    c.cap = cap;
    c.cand_cap = parts * (u64)k;
  }
  c.smem = scan_smem<QW, E, MODE, CMP>();
  return c;
}

// Spread the per-query global histogram bins over distinct L2 lines/slices
// when many warps share a query (small Q); dense layout otherwise.
u32 ghist_stride(u32 Q) { return Q <= 64 ? 64u : 1u; }
u32 tg_replicas(u32 Q) { return Q <= 64 ? 16u : 1u; }

// tg[q] = T_OPEN (255) for every query slot the buffer holds.
cudaError_t fill_tg(fps_lib* L) {
  std::vector<u32> open(L->tg.bytes / 4, fps::T_OPEN);
  cudaError_t e = cudaMemcpyAsync(L->tg.p, open.data(), open.size() * 4, cudaMemcpyHostToDevice, L->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
  return e;
}

int ensure_state(fps_lib* L, u32 Q) {
  const size_t gh = (size_t)Q * fps::HB * 4 * ghist_stride(Q);
  const size_t tgb = (size_t)Q * tg_replicas(Q) * ghist_stride(Q) * 4;
  if (Q <= L->state_q && gh <= L->ghist.bytes && tgb <= L->tg.bytes) return FPS_OK;
  const u32 Qa = std::max(Q, L->state_q);
  int rc;
  if ((rc = L->tg.ensure(std::max((size_t)Qa * 4, (size_t)Q * tg_replicas(Q) * ghist_stride(Q) * 4)))) return rc;
  if ((rc = L->ghist.ensure(std::max(gh, (size_t)Qa * fps::HB * 4)))) return rc;
  if ((rc = L->cand_cnt.ensure((size_t)Qa * 4))) return rc;
  if ((rc = L->dyn.ensure(256))) return rc;
  CUDA_TRY(cudaMemsetAsync(L->dyn.p, 0, L->dyn.bytes, L->stream));
  CUDA_TRY(fill_tg(L));
  CUDA_TRY(cudaMemsetAsync(L->ghist.p, 0, L->ghist.bytes, L->stream));
  CUDA_TRY(cudaMemsetAsync(L->cand_cnt.p, 0, L->cand_cnt.bytes, L->stream));
  CUDA_TRY(cudaStreamSynchronize(L->stream));
  L->state_q = Qa;
  return FPS_OK;
}

// Restore the clean top-k state after a failed call.
void reset_state(fps_lib* L) {
  if (!L->state_q) return;
  fill_tg(L);
  cudaMemsetAsync(L->ghist.p, 0, L->ghist.bytes, L->stream);
  cudaMemsetAsync(L->cand_cnt.p, 0, L->cand_cnt.bytes, L->stream);
  if (L->dyn.p) cudaMemsetAsync(L->dyn.p, 0, L->dyn.bytes, L->stream);
}

u32 scan_flags() {
  static u32 f = [] {
    const char* e = std::getenv("FPS_SCAN_FLAGS");
    return e ? (u32)std::strtoul(e, nullptr, 0) : 0u;
  }();
  return f;
}

fps::ScanArgs base_args(const fps_lib* L, const u64* d_q, u32 Q) {
  fps::ScanArgs a{};
  a.flags = scan_flags();
  a.lib = L->mem;
  a.n = L->n;
  a.index_base = L->index_base;
  a.queries = d_q;
  a.Q = Q;
  return a;
}

// Dynamic tail of the bulk-copy single-query scan. Warps draw unequal HBM
// bandwidth (their static parts finish ~10 % apart on a 95 M library), so on
// long scans the second half of the tiles is claimed in 8-tile chunks from a
// global counter. Short scans (< 128 tiles per warp) stay static: the claim
// traffic there costs more than the imbalance (profiles/r01_experiments.md).
// Scan flag 64 disables it. Needs one query group: every warp scans for the
// same query.
#ifndef FPS_DYN_STATIC_PCT
#define FPS_DYN_STATIC_PCT 50  // share of the tiles split statically before the global tail
#endif
#ifndef FPS_DYN_MIN_ITERS
#define FPS_DYN_MIN_ITERS 128  // per-warp iterations below which a scan uses the CTA-dynamic schedule
#endif
#ifndef FPS_DYN_CHUNK_ITERS
#define FPS_DYN_CHUNK_ITERS 12  // 128-entry iterations per tail claim (6 compact tiles; 4 -> contention, 24 -> coarse tail)
#endif
template <int QW, int E, int MODE, bool CMP>
void set_dyn(fps_lib* L, fps::ScanArgs& a) {
  if (!fps::ScanSmem<QW, E, MODE, CMP>::TMA || MODE != fps::MODE_TOPK || a.n_qg != 1 || (a.flags & 64)) return;
  if (!L->dyn.p || a.iters < FPS_DYN_MIN_ITERS * a.n_parts) return;
  constexpr u64 SUB = fps::ScanSmem<QW, E, MODE, CMP>::SUB;  // iterations per tile (the kernel's work unit)
  a.dyn_ctr = L->dyn.as<u32>();
  a.dyn_start = (a.iters + SUB - 1) / SUB * FPS_DYN_STATIC_PCT / 100;
  a.dyn_chunk = std::max<u64>(1, FPS_DYN_CHUNK_ITERS / SUB);
}

// select_kernel launched as a programmatic dependent of the scan kernel: its
// launch and block scheduling overlap the scan's tail, and griddepcontrol.wait
// inside it orders it after the scan's completion (and memory flush).
cudaError_t launch_select(u32 Q, size_t smem, cudaStream_t s, u64* cand, u32* cand_cnt, u64 cand_cap, u32* tg,
                          u32* ghist, u32 gstride, u32 tg_rep, u32 k, u64* out_keys, u32* out_cnt, bool pdl,
                          u32* dyn_ctr = nullptr, u32* done_flag = nullptr, u32 done_seq = 0,
                          const u32* gate = nullptr, u32* ovf = nullptr) {
  smem_optin((const void*)fps::select_kernel, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(Q);
  cfg.blockDim = dim3(fps::SEL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fps::select_kernel, cand, cand_cnt, cand_cap, tg, ghist, gstride, tg_rep, k, out_keys,
                            out_cnt, 1, dyn_ctr, done_flag, done_seq, gate, ovf);
}

// Record an event pair around the next scan-kernel launch when timing is on.
std::pair<cudaEvent_t, cudaEvent_t>* timing_slot(fps_lib* L) {
  if (!L->timing || L->timing_suspend) return nullptr;
  if (L->ev_used == L->ev_pool.size()) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return nullptr;
    L->ev_pool.emplace_back(a, b);
  }
  if (!L->timing_continue || L->ev_groups == 0) L->ev_groups++;
  return &L->ev_pool[L->ev_used++];
}

template <int QW, int E, bool CMP>
int topk_fused(fps_lib* L, const u64* d_q, u32 Q, u32 k, u64* d_keys, u32* d_cnt, cudaStream_t s, bool prepare_only,
               u64 n_prefix = 0, const u64* h_qin = nullptr, const u32* gate = nullptr) {
  Config c = make_config<QW, E, fps::MODE_TOPK, false, CMP>(L, Q, k, n_prefix);
  int rc;
  if ((rc = ensure_state(L, Q))) return rc;
  if ((rc = L->buf.ensure(c.warps * QW * (size_t)c.cap * 8))) return rc;
  if ((rc = L->cand.ensure((size_t)Q * c.cand_cap * 8))) return rc;
  if (prepare_only) return FPS_OK;
  fps::ScanArgs a = base_args(L, d_q, Q);
  if (h_qin) {  // single query passed by value (host API): no H2D copy
    a.queries = nullptr;
    a.qin[0] = h_qin[0];
    a.qin[1] = h_qin[1];
    a.qin[2] = h_qin[2];
  }
  if (n_prefix) a.n = n_prefix;
  a.k = k;
  a.cap = c.cap;
  a.n_qg = c.n_qg;
  a.n_parts = c.n_parts;
  a.iters = c.iters;
  a.tg = L->tg.as<u32>();
  a.ghist = L->ghist.as<u32>();
  a.gstride = ghist_stride(Q);
  a.tg_rep = tg_replicas(Q);
  a.pub_every = (u32)std::max<u64>(1, c.n_parts / 512);
  a.buf = L->buf.as<u64>();
  a.cand = L->cand.as<u64>();
  a.cand_cnt = L->cand_cnt.as<u32>();
  a.cand_cap = c.cand_cap;
  a.gate = gate;
  set_dyn<QW, E, fps::MODE_TOPK, CMP>(L, a);
  if (c.warps > 0 && L->n > 0) {
    auto* ev = timing_slot(L);
    if (ev) cudaEventRecord(ev->first, s);
    if (ev) {
      fps::scan_kernel<QW, E, fps::MODE_TOPK, false, CMP><<<c.grid, WPB * 32, c.smem, s>>>(a);
    } else {
      // programmatic dependent of whatever kernel precedes it on the stream
      // (typically the previous call's select_kernel): launch latency hides
      // behind that kernel; griddepcontrol.wait in the scan orders the rest
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(c.grid);
      cfg.blockDim = dim3(WPB * 32);
      cfg.dynamicSmemBytes = c.smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      // (long scans with the global tail measured faster without it: C3
      // 306 vs 291-297 us; short ones faster with it: C2 48.3 vs 50.3 us)
      attr[0].val.programmaticStreamSerializationAllowed = ((a.flags & 128) || a.dyn_ctr) ? 0 : 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CUDA_TRY(cudaLaunchKernelEx(&cfg, fps::scan_kernel<QW, E, fps::MODE_TOPK, false, CMP>, a));
    }
    if (ev) cudaEventRecord(ev->second, s);
    L->launches++;
  }
  if (std::getenv("FPS_DEBUG")) {
    std::vector<u32> cc(std::min<u32>(Q, 8));
    cudaStreamSynchronize(s);
    cudaMemcpy(cc.data(), a.cand_cnt, cc.size() * 4, cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "[fps] Q=%u k=%u warps=%llu parts=%llu candidates:", Q, k, (unsigned long long)c.warps,
                 (unsigned long long)c.n_parts);
    for (u32 v : cc) std::fprintf(stderr, " %u", v);
    std::fprintf(stderr, "\n");
  }
  int kp = 1;
  while (kp < (int)k) kp <<= 1;
  size_t sel_smem = (size_t)(kp + fps::SEL_ECAP) * 8;
  LAUNCH_CHECK("scan_kernel<topk>");
  CUDA_TRY(launch_select(Q, sel_smem, s, a.cand, a.cand_cnt, c.cand_cap, a.tg, a.ghist, a.gstride, a.tg_rep, k,
                         d_keys, d_cnt, !(a.flags & 32), a.dyn_ctr, nullptr, 0, gate));
  L->launches++;
  LAUNCH_CHECK("select_kernel");
  if (std::getenv("FPS_DEBUG")) {
    unsigned long long t[12] = {0};
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(t, fps::g_sel_clock, sizeof(t));
    std::fprintf(stderr, "[fps] select phases (cycles from start):");
    for (int i = 1; i < 12; ++i) std::fprintf(stderr, " %lld", t[i] ? (long long)(t[i] - t[0]) : -1ll);
    std::fprintf(stderr, "\n");
  }
  CUDA_TRY(cudaGetLastError());
  return FPS_OK;
}

// ---------------------------------------------------------------------------
// bit-sliced multi-query path (fps_bitslice.cuh)
// ---------------------------------------------------------------------------
// Batches from 2 queries take the bit-sliced kernel: on the 95.4 M library it
// beats the POPC kernels at every Q >= 2 (Q = 2: 0.38 vs 0.46 ms, Q = 8: 0.51
// vs 1.22 ms, Q = 32: 1.20 vs 4.48 ms; tools/q_sweep.py). FPS_BS_MIN_Q
// overrides, FPS_BITSLICE=0 disables it.
u32 bs_min_q() {
  static u32 v = []() {
    const char* e = std::getenv("FPS_BS_MIN_Q");
    return e ? (u32)std::max(1, std::atoi(e)) : 2u;
  }();
  return v;
}

// Queries per warp of the bit-sliced kernel: small batches spread one or two
// queries over every warp of a CTA instead of four over a quarter of them.
u32 bs_qpw(u32 Q) { return Q <= (u32)fps::BS_WARPS ? 1u : Q <= 2u * fps::BS_WARPS ? 2u : (u32)fps::BS_QPW; }

template <int QPW>
size_t bs_smem_t() {
  return 2 * (fps::BS_TILE_BYTES + fps::BS_PLANE_BYTES) + 16 + (size_t)QPW * fps::BS_WARPS * sizeof(fps::BsQuery) +
         (size_t)fps::BS_WARPS * QPW * fps::HB * 4 + fps::BS_WARPS * sizeof(fps::WarpState<QPW>) +
         (size_t)fps::BS_WARPS * QPW * 10 * 4;
}
size_t bs_smem(u32 qpw) { return qpw == 1 ? bs_smem_t<1>() : qpw == 2 ? bs_smem_t<2>() : bs_smem_t<fps::BS_QPW>(); }

template <int MODE, int QPW>
int bs_ctas_per_sm() {
  static int cached = 0;
  const size_t sm = bs_smem_t<QPW>();
  smem_optin((const void*)fps::bs_scan_kernel<MODE, QPW>, sm);
  if (!cached) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached, fps::bs_scan_kernel<MODE, QPW>, fps::BS_WARPS * 32, sm);
    cached = std::max(1, cached);
  }
  return cached;
}

template <int MODE>
cudaError_t bs_launch(u32 qpw, u64 ctas, cudaStream_t s, const fps::BsArgs& b) {
  if (qpw == 1) {
    bs_ctas_per_sm<MODE, 1>();
    fps::bs_scan_kernel<MODE, 1><<<(unsigned)ctas, fps::BS_WARPS * 32, bs_smem_t<1>(), s>>>(b);
  } else if (qpw == 2) {
    bs_ctas_per_sm<MODE, 2>();
    fps::bs_scan_kernel<MODE, 2><<<(unsigned)ctas, fps::BS_WARPS * 32, bs_smem_t<2>(), s>>>(b);
  } else {
    bs_ctas_per_sm<MODE, fps::BS_QPW>();
    fps::bs_scan_kernel<MODE, fps::BS_QPW><<<(unsigned)ctas, fps::BS_WARPS * 32, bs_smem_t<fps::BS_QPW>(), s>>>(b);
  }
  return cudaGetLastError();
}

// Build (once) the bit-plane copy; libraries with pad bits past key 166 stay on the POPC path.
int bs_ensure(fps_lib* L) {
  if (L->bs_state) return FPS_OK;
  const auto t0 = std::chrono::steady_clock::now();
  struct Clock {
    fps_lib* L;
    std::chrono::steady_clock::time_point t0;
    ~Clock() { L->derived_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
  } clock{L, t0};
  const u64 tiles = (L->n + fps::BS_TILE_ENTRIES - 1) / fps::BS_TILE_ENTRIES;
  int rc;
  if ((rc = L->bs.ensure((size_t)std::max<u64>(tiles, 1) * fps::BS_TILE_BYTES))) {
    cudaGetLastError();
    L->bs_state = -1;  // not enough memory for the copy: keep the POPC scan
    return FPS_OK;
  }
  DevBuf wide;
  if ((rc = wide.ensure(4))) return rc;
  CUDA_TRY(cudaMemsetAsync(L->bs.p, 0, L->bs.bytes, L->stream));
  CUDA_TRY(cudaMemsetAsync(wide.p, 0, 4, L->stream));
  const u64 nblocks = (L->n + 31) / 32;
  const int grid = (int)std::min<u64>((nblocks * 32 + 255) / 256, (u64)L->sms * 32);
  fps::bs_build_kernel<<<std::max(grid, 1), 256, 0, L->stream>>>(L->out(), L->n, L->bs.as<u32>(), wide.as<u32>());
  L->launches++;
  u32 nwide = 0;
  CUDA_TRY(cudaMemcpyAsync(&nwide, wide.p, 4, cudaMemcpyDeviceToHost, L->stream));
  CUDA_TRY(cudaStreamSynchronize(L->stream));
  L->bs_state = nwide ? -1 : 1;
  if (nwide) L->bs.release();
  return FPS_OK;
}

bool bs_wanted(fps_lib* L, u32 Q) {
  const char* e = std::getenv("FPS_BITSLICE");
  if (e && std::string(e) == "0") return false;
  if (Q < bs_min_q() || L->n < fps::BS_TILE_ENTRIES) return false;
  if (bs_ensure(L) != FPS_OK) return false;
  return L->bs_state == 1;
}

fps::BsArgs bs_args(fps_lib* L, u32 Q, u32 qpw, u64* n_parts_out) {
  fps::BsArgs b{};
  b.bs = L->bs.as<u32>();
  b.n = L->n;
  b.index_base = L->index_base;
  b.qs = reinterpret_cast<const fps::BsQuery*>(L->bsq.p);
  b.Q = Q;
  const u32 qpc = qpw * fps::BS_WARPS;
  b.n_qg = (Q + qpc - 1) / qpc;
  b.tiles = (L->n + fps::BS_TILE_ENTRIES - 1) / fps::BS_TILE_ENTRIES;
  const int ctas_per_sm = qpw == 1 ? bs_ctas_per_sm<fps::MODE_TOPK, 1>()
                          : qpw == 2 ? bs_ctas_per_sm<fps::MODE_TOPK, 2>()
                                     : bs_ctas_per_sm<fps::MODE_TOPK, fps::BS_QPW>();
  const u64 slots = (u64)L->sms * ctas_per_sm;
  u64 parts = std::max<u64>(1, slots / b.n_qg);
  parts = std::min<u64>(parts, std::max<u64>(1, b.tiles / 4));  // >= 4 tiles per CTA
  b.n_parts = parts;
  *n_parts_out = parts;
  return b;
}

int bs_prep(fps_lib* L, const u64* d_q, u32 Q, cudaStream_t s) {
  int rc;
  if ((rc = L->bsq.ensure((size_t)Q * sizeof(fps::BsQuery)))) return rc;
  fps::bs_prep_queries<<<(Q + 127) / 128, 128, 0, s>>>(d_q, Q, reinterpret_cast<fps::BsQuery*>(L->bsq.p));
  L->launches++;
  LAUNCH_CHECK("bs_prep_queries");
  return FPS_OK;
}

template <bool CMP>
int topk_bs(fps_lib* L, const u64* d_q, u32 Q, u32 k, u64* d_keys, u32* d_cnt, cudaStream_t s, bool prepare_only) {
  int rc;
  // 1. seed: exact top-k of a library prefix with the POPC scan -> tg[q] bound
  const u64 seed_n = std::min<u64>(L->n, 1 << 18);
  L->timing_suspend = true;
  rc = topk_fused<8, 2, CMP>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only, seed_n);
  L->timing_suspend = false;
  if (rc) return rc;
  u64 parts = 0;
  const u32 qpw = bs_qpw(Q);
  fps::BsArgs b = bs_args(L, Q, qpw, &parts);
  const u64 ctas = (u64)b.n_qg * parts;
  // a warp step can pass a whole tile (every entry tied at the bound) after
  // the buffer was compacted to k: room for k + one tile
  const u32 cap = (std::max<u32>(2 * k, k + fps::BS_TILE_ENTRIES) + 31) / 32 * 32;
  const u64 cand_cap = parts * (u64)k;
  if ((rc = L->buf.ensure(ctas * fps::BS_WARPS * qpw * (size_t)cap * 8))) return rc;
  if ((rc = L->cand.ensure((size_t)Q * cand_cap * 8))) return rc;
  if ((rc = L->bsq.ensure((size_t)Q * sizeof(fps::BsQuery)))) return rc;
  if (prepare_only) return FPS_OK;
  fps::bs_seed_tg<<<(Q + 127) / 128, 128, 0, s>>>(d_keys, d_cnt, Q, k, L->tg.as<u32>(), tg_replicas(Q),
                                                   ghist_stride(Q));
  L->launches++;
  LAUNCH_CHECK("bs_seed_tg");
  if ((rc = bs_prep(L, d_q, Q, s))) return rc;
  b.qs = reinterpret_cast<const fps::BsQuery*>(L->bsq.p);  // (re)allocated by bs_prep
  // 2. bit-sliced scan of the whole library
  b.k = k;
  b.cap = cap;
  b.tg = L->tg.as<u32>();
  b.tg_rep = tg_replicas(Q);
  b.gstride = ghist_stride(Q);
  b.buf = L->buf.as<u64>();
  b.cand = L->cand.as<u64>();
  b.cand_cnt = L->cand_cnt.as<u32>();
  b.cand_cap = cand_cap;
  auto* ev = timing_slot(L);
  if (ev) cudaEventRecord(ev->first, s);
  CUDA_TRY(bs_launch<fps::MODE_TOPK>(qpw, ctas, s, b));
  if (ev) cudaEventRecord(ev->second, s);
  L->launches++;
  LAUNCH_CHECK("bs_scan_kernel<topk>");
  int kp = 1;
  while (kp < (int)k) kp <<= 1;
  CUDA_TRY(launch_select(Q, (size_t)(kp + fps::SEL_ECAP) * 8, s, b.cand, b.cand_cnt, cand_cap, b.tg, L->ghist.as<u32>(),
                         ghist_stride(Q), tg_replicas(Q), k, d_keys, d_cnt, false));
  L->launches++;
  LAUNCH_CHECK("select_kernel (bit-slice)");
  return FPS_OK;
}

int range_bs(fps_lib* L, const u64* d_q, u32 Q, const unsigned char* d_radius, u64* d_out, u64 cap, u64* d_count,
             cudaStream_t s) {
  int rc;
  if ((rc = bs_prep(L, d_q, Q, s))) return rc;
  u64 parts = 0;
  const u32 qpw = bs_qpw(Q);
  fps::BsArgs b = bs_args(L, Q, qpw, &parts);
  b.radius = d_radius;
  b.out = d_out;
  b.out_cnt = d_count;
  b.out_cap = cap;
  auto* ev = timing_slot(L);
  if (ev) cudaEventRecord(ev->first, s);
  CUDA_TRY(bs_launch<fps::MODE_RANGE>(qpw, (u64)b.n_qg * parts, s, b));
  if (ev) cudaEventRecord(ev->second, s);
  L->launches++;
  return FPS_OK;
}


// ---------------------------------------------------------------------------
// single-query plane scan (fps_planeq.cuh)
// ---------------------------------------------------------------------------
// Build (once) the plane-major copy; libraries with pad bits past key 166 keep
// the POPC scan (it counts them, like the reference).
int pm_ensure(fps_lib* L, bool sorted) {
  if (L->pm_state && (L->pm_state < 0 || L->pm_sorted == sorted)) return FPS_OK;
  struct Clock {
    fps_lib* L;
    std::chrono::steady_clock::time_point t0;
    ~Clock() { L->derived_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
  } clock{L, std::chrono::steady_clock::now()};
  L->pm.release();
  L->pm_perm.release();
  L->pm_meta.release();
  L->pm_sorted = sorted;
  const u64 steps = std::max<u64>(1, (L->n + 32 * fps::PQ_STRIDE_WORDS - 1) / (32 * fps::PQ_STRIDE_WORDS));
  // plane stride: whole steps, an odd number of 256 B chunks (planes read
  // side by side do not start on the same DRAM interleave phase)
  u64 stride_chunks = steps | 1;
  L->pm_stride = stride_chunks * fps::PQ_STRIDE_WORDS;
  int rc;
  if ((rc = L->pm.ensure((size_t)fps::BS_PLANES * L->pm_stride * 4))) {
    cudaGetLastError();
    L->pm_state = -1;
    return FPS_OK;
  }
  DevBuf wide, keys, sorted_keys, tmp;
  if ((rc = wide.ensure(4))) return rc;
  CUDA_TRY(cudaMemsetAsync(L->pm.p, 0, L->pm.bytes, L->stream));
  CUDA_TRY(cudaMemsetAsync(wide.p, 0, 4, L->stream));
  const u64 nblocks = (L->n + 31) / 32;
  const int grid = (int)std::min<u64>((nblocks * 32 + 255) / 256, (u64)L->sms * 32);
  if (sorted) {
    // order = entries sorted by (|a|, index): radix sort of |a| << 32 | index on bits 0..39
    if (L->n > (u64)INT32_MAX) return fail(FPS_EINVAL, "sorted plane copy: more than 2^31 entries on one device");
    if ((rc = keys.ensure(L->n * 8)) || (rc = sorted_keys.ensure(L->n * 8)) ||
        (rc = L->pm_perm.ensure(L->n * 4)) || (rc = L->pm_meta.ensure(((L->n + 1023) / 1024) * 2)))
      return rc;
    fps::pm_sort_keys_kernel<<<std::max(grid, 1), 256, 0, L->stream>>>(L->out(), L->n, keys.as<u64>());
    size_t tmp_bytes = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.as<u64>(), sorted_keys.as<u64>(), (int)L->n, 0,
                                            40, L->stream));
    if ((rc = tmp.ensure(tmp_bytes))) return rc;
    CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.as<u64>(), sorted_keys.as<u64>(), (int)L->n, 0,
                                            40, L->stream));
    const u64 nb = (L->n + 1023) / 1024;
    fps::pm_meta_kernel<<<(int)std::min<u64>((nb + 255) / 256, 4096), 256, 0, L->stream>>>(
        sorted_keys.as<u64>(), L->n, reinterpret_cast<unsigned short*>(L->pm_meta.p));
    L->launches += 4;
  }
  fps::pm_build_kernel<<<std::max(grid, 1), 256, 0, L->stream>>>(
      L->out(), L->n, L->pm.as<u32>(), L->pm_stride, wide.as<u32>(), sorted ? sorted_keys.as<u64>() : nullptr,
      sorted ? L->pm_perm.as<u32>() : nullptr);
  L->launches++;
  LAUNCH_CHECK("pm_build_kernel");
  u32 nwide = 0;
  CUDA_TRY(cudaMemcpyAsync(&nwide, wide.p, 4, cudaMemcpyDeviceToHost, L->stream));
  CUDA_TRY(cudaStreamSynchronize(L->stream));
  L->pm_state = nwide ? -1 : 1;
  if (nwide) {
    L->pm.release();
    L->pm_perm.release();
    L->pm_meta.release();
  }
  return FPS_OK;
}

bool pq_wanted(fps_lib* L) {
  const char* e = std::getenv("FPS_PLANEQ");  // "0": the POPC scan (tests cover both)
  if ((e && std::string(e) == "0") || L->n == 0) return false;
  if (!L->pqk.init) {
    auto ev = [](const char* name, int dflt) {
      const char* v = std::getenv(name);
      return v ? std::atoi(v) : dflt;
    };
    L->pqk.sorted = ev("FPS_PQ_SORTED", 0) == 1;  // the popcount-sorted plane copy (SORTED kernels)
    L->pqk.bpl = ev("FPS_PQ_BPL", 2) == 1 ? 1 : 2;
    L->pqk.warps = std::max(1, std::min(16, ev("FPS_PQ_WARPS", 8)));
    L->pqk.stages = std::max(1, std::min(fps::PQ_SMAX, ev("FPS_PQ_STAGES", 2)));
    L->pqk.smem_kb = ev("FPS_PQ_SMEM_KB", 210);
    L->pqk.copy = ev("FPS_PQ_COPY", 1) == 1 ? 1 : 0;
    L->pqk.refresh = ev("FPS_PQ_REFRESH", 0);
    // first wave: before its second step a warp waits (at most wave_ns) until
    // wave_pct % of the warps have posted their first step's witnesses
    L->pqk.wave_pct = std::max(0, std::min(100, ev("FPS_PQ_WAVE_PCT", 50)));
    L->pqk.wave_ns = std::max(0, ev("FPS_PQ_WAVE_NS", 8000));
    // shape policy: 1 (default) = 1,024-entry steps with as many warps (<= 16)
    // as hold two stages of the query's plane list; 0 = the knobs above for
    // every query (8 warps x 2,048-entry steps; lists wider than 48 positions
    // fold to 4 warps); 2 = policy 0 for lists of <= 48 positions, 1 for wider
    // ones. Explicit shape knobs imply 0.
    L->pqk.shape = ev("FPS_PQ_SHAPE", (std::getenv("FPS_PQ_BPL") || std::getenv("FPS_PQ_WARPS")) ? 0 : 1);
    L->pqk.init = true;
  }
  if (pm_ensure(L, L->pqk.sorted) != FPS_OK) {
    cudaGetLastError();
    return false;
  }
  return L->pm_state == 1;
}


// Stage positions of a query: 8 popcount planes + its listed planes padded to 8.
u32 pq_positions(const u64* q) {
  const u32 pop = (u32)(__builtin_popcountll(q[0]) + __builtin_popcountll(q[1]) + __builtin_popcountll(q[2]));
  const u32 pop166 = (u32)(__builtin_popcountll(q[0]) + __builtin_popcountll(q[1]) +
                           __builtin_popcountll(q[2] & ((1ull << 38) - 1)));
  const u32 m = pop > 83 ? 166 - pop166 : pop166;
  return 8 + (m + 7) / 8 * 8;
}

int topk_pq(fps_lib* L, const u64* d_q, const u64* h_qin, u32 k, u64* d_keys, u32* d_cnt, cudaStream_t s,
            bool prepare_only, u32* done_flag = nullptr, u32 done_seq = 0) {
  int rc;
  // Shape: sized to the query's plane list (below); long scans read the global
  // bound every 8th step (C3 109.5 -> 95.5 us), short ones every step (the
  // first steps set it: C2 29.1 vs 33.5 us).
  const bool long_scan = L->n >= (32u << 20);
  const bool srt = L->pm_sorted;
  // stage positions of the query's plane list: known when the query is on the
  // host (or hinted, fps_query_hint); 48 = up to 40 listed planes otherwise
  const u32 np = h_qin ? pq_positions(h_qin) : (L->pq_hint_np ? L->pq_hint_np : 48);
  int bpl = L->pqk.bpl;  // 32-entry blocks per lane
  int nwb = L->pqk.warps;
  const int stages = L->pqk.stages;
  u32 budget = (u32)L->pqk.smem_kb * 1024;
  // (short libraries, fewer than two 1,024-entry steps per warp at 16 warps,
  // keep the 8-warp shape unless the list is wide: C1 e2e 37 vs 40 us)
  const bool many_steps = L->n / fps::PqStep<1>::ENTRIES >= 32ull * (u64)L->sms;
  if (!srt && ((L->pqk.shape == 1 && (many_steps || np > 48)) || (L->pqk.shape == 2 && np > 48))) {
    // 1,024-entry steps and as many warps as hold two stages of this list
    // (16 below 48 positions, 14 at 48, 13 at 56, 8 at 96): two stages of 2,048-entry
    // steps fit 8 warps only up to 48 positions, beyond which the kernel folds
    // to 4 warps (C3: 98 -> 157 us from 48 to 49 planes; tools/dbg/pq_width.py:
    // now 98 -> 98.7 us, and 16 warps are 3-8 % faster on narrow lists too:
    // C3 |q| = 20 / 30 / 40: 76.1 / 88.1 / 98.2 -> 69.9 / 81.1 / 95.5 us).
    bpl = 1;
    budget = std::max<u32>(budget, 218u * 1024);
    // At most 14 warps at 48 positions (C3: 95.7 / 94.4 / 94.9 / 95.9 us at 13 /
    // 14 / 15 / 16 warps, 98.5 at 12), 16 on narrower lists (|q| = 20 / 30:
    // 70 / 81 us at 16 warps, 76 / 85 at 14); FPS_PQ_MAXW overrides.
    static const int maxw_env = std::getenv("FPS_PQ_MAXW") ? std::atoi(std::getenv("FPS_PQ_MAXW")) : 0;
    const int maxw = maxw_env > 0 ? maxw_env : (np >= 48 ? 14 : 16);
    for (nwb = std::max(5, std::min(16, maxw)); nwb > 4; --nwb)
      if (fps::pq_smem(nwb, (2 * np * fps::PqStep<1>::CHUNK + 255) / 256 * 256) <= budget) break;
  } else if (!srt && L->pqk.shape == 1) {
    // short libraries: 6 warps x 2,048-entry steps (a smaller CTA launches
    // faster; host-path call, tools/dbg/pq_small.py: 1 M entries 29.0 vs 30.8 us
    // with 8 warps, 2 M 28.1 vs 32.8, 4 M 28.8 vs 29.7)
    nwb = 6;
  }
  const u32 chunk = bpl == 1 ? fps::PqStep<1>::CHUNK : fps::PqStep<2>::CHUNK;
  const u64 step_entries = bpl == 1 ? fps::PqStep<1>::ENTRIES : fps::PqStep<2>::ENTRIES;
  // ring per warp: `stages` stages of the list; wider lists than the ring was
  // sized for fold warps in the kernel
  // (capped by the shared memory of one CTA; at least two stages of the
  // widest list over the whole CTA)
  const u32 ring_cap = (u32)((budget - (u32)fps::pq_smem(nwb, 0)) / nwb) / 256 * 256;
  u32 ring = std::min<u32>(((u32)stages * np * chunk + 255) / 256 * 256, ring_cap);
  ring = std::max<u32>(ring, (u32)((2 * fps::PQ_NPMAX * chunk + nwb - 1) / nwb + 255) / 256 * 256);
  const u64 steps = (L->n + step_entries - 1) / step_entries;
  const u64 grid = std::max<u64>(1, std::min<u64>((u64)L->sms, steps));
  const u32 meta_cap = srt ? (u32)((steps + grid - 1) / grid + 1) : 0u;
  const size_t smem = fps::pq_smem(nwb, ring, meta_cap);
  if (smem > 226 * 1024) return fail(FPS_EINVAL, "plane scan: shared memory ring too large (FPS_PQ_WARPS/STAGES)");
  const u64 warps = grid * nwb;
  const u32 cap = (std::max<u32>(2 * k, k + (u32)step_entries) + 31) / 32 * 32;
  const u64 cand_cap = warps * (u64)k;
  if ((rc = ensure_state(L, 1))) return rc;
  {
    // sized for every shape the policy may pick for later queries (a call must
    // not reallocate inside a captured or pipelined stream)
    const size_t c1 = (std::max<u32>(2 * k, k + (u32)fps::PqStep<1>::ENTRIES) + 31) / 32 * 32;
    const size_t c2 = (std::max<u32>(2 * k, k + (u32)fps::PqStep<2>::ENTRIES) + 31) / 32 * 32;
    const size_t per_cta = std::max<size_t>({(size_t)nwb * cap, 16 * c1, (size_t)L->pqk.warps * c2});
    if ((rc = L->buf.ensure((size_t)L->sms * per_cta * 8))) return rc;
    if ((rc = L->cand.ensure((size_t)L->sms * std::max<size_t>(16, nwb) * k * 8))) return rc;
  }
  const int copy = L->pqk.copy;  // 1: cp.async 16 B per lane (default, measured faster), 0: bulk copies
  const int kv = srt ? 4 + (bpl == 2 ? 1 : 0) : (copy == 1 ? 1 : 0) * 2 + (bpl == 2 ? 1 : 0);
  void (*const kerns[6])(fps::PqArgs) = {fps::pq_scan_kernel<0, 1, false>, fps::pq_scan_kernel<0, 2, false>,
                                         fps::pq_scan_kernel<1, 1, false>, fps::pq_scan_kernel<1, 2, false>,
                                         fps::pq_scan_kernel<1, 1, true>,  fps::pq_scan_kernel<1, 2, true>};
  auto* kern = kerns[kv];
  CUDA_TRY(smem_optin((const void*)kern, smem));  // (the kernel's static shared memory comes on top)
  if (prepare_only) return FPS_OK;
  fps::PqArgs a{};
  a.pm = L->pm.as<u32>();
  a.pstride = L->pm_stride;
  a.n = L->n;
  a.index_base = L->index_base;
  a.queries = h_qin ? nullptr : d_q;
  if (h_qin) { a.qin[0] = h_qin[0]; a.qin[1] = h_qin[1]; a.qin[2] = h_qin[2]; }
  a.k = k;
  a.cap = cap;
  a.n_steps = steps;
  a.ring_bytes = ring;
  // (every 8th 2,048-entry step = every 16th 1,024-entry step: C3 96.2 / 95.6 / 96.2 us at 8 / 16 / 32)
  a.refresh = (u32)(L->pqk.refresh > 0 ? L->pqk.refresh : (long_scan ? (bpl == 1 ? 16 : 8) : 1));
  a.perm = srt ? L->pm_perm.as<u32>() : nullptr;
  a.meta = srt ? reinterpret_cast<const unsigned short*>(L->pm_meta.p) : nullptr;
  a.meta_cap = meta_cap;
  a.pub_every = (u32)std::max<u64>(1, warps / 512);
  {
    // warps whose first step is a full one post k witnesses each; the kernel
    // sizes the wait from its active warps (wide plane lists fold warps).
    // (libraries with fewer than two steps per warp have no second step to speed up)
    const bool on = k <= step_entries && steps >= 2 * warps;
    a.wave_pct = on ? (u32)L->pqk.wave_pct : 0u;
    a.wave_steps = L->n / step_entries;
    a.wave_wait_ns = (u32)L->pqk.wave_ns;
  }
  a.flags = scan_flags();
  a.tg = L->tg.as<u32>();
  a.ghist = L->ghist.as<u32>();
  a.gstride = ghist_stride(1);
  a.tg_rep = tg_replicas(1);
  a.buf = L->buf.as<u64>();
  a.cand = L->cand.as<u64>();
  a.cand_cnt = L->cand_cnt.as<u32>();
  a.cand_cap = cand_cap;
  L->last_kernel = 5;
  auto* ev = timing_slot(L);
  if (ev) cudaEventRecord(ev->first, s);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(nwb * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (ev || (a.flags & 128)) ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  if (ev) cudaEventRecord(ev->second, s);
  L->launches++;
  LAUNCH_CHECK("pq_scan_kernel");
  int kp = 1;
  while (kp < (int)k) kp <<= 1;
  CUDA_TRY(launch_select(1, (size_t)(kp + fps::SEL_ECAP) * 8, s, a.cand, a.cand_cnt, cand_cap, a.tg, a.ghist,
                         a.gstride, a.tg_rep, k, d_keys, d_cnt, !(a.flags & 32), nullptr, done_flag, done_seq));
  L->launches++;
  LAUNCH_CHECK("select_kernel (plane scan)");
  static const bool dbg = std::getenv("FPS_DEBUG") != nullptr;
  if (dbg)
    std::fprintf(stderr, "[fps] plane scan: grid=%llu warps/CTA=%d ring=%u smem=%zu\n", (unsigned long long)grid, nwb,
                 ring, smem);
  return FPS_OK;
}


// ---------------------------------------------------------------------------
// tensor-core multi-query path (fps_mma.cuh)
// ---------------------------------------------------------------------------
// Batches of >= 64 queries take the tensor cores (95.4 M entries, top-k: 64
// queries 1.91 vs 2.12 ms bit-sliced, 128: 2.01 vs 4.08, 192: 2.41 vs 6.06;
// tools/dbg/mm4x_bench.sh with bench.py --queries). FPS_MMA=1 forces it for
// any batch >= 2, FPS_MMA=0 disables it. The call is stream ordered end to end
// (no host synchronisation, capturable): a candidate list that overflows its
// capacity raises a device flag, and a gated POPC pass recomputes the batch.
constexpr int MMA_MAX_PASS = 6;
struct MmaPlan {
  u64 seed_n = 0;               // seed prefix [0, seed_n): POPC top-k
  int npass = 0;                // tensor-core passes over [n_scan[i-1], n_scan[i]) (the first from seed_n)
  u64 n_scan[MMA_MAX_PASS] = {};  // (the last: the library)
  u32 cap[MMA_MAX_PASS] = {};   // per-query candidate capacity of each pass
};

// Passes and candidate capacities for (Q, k). The library is scanned ONCE, in
// growing ranges: a POPC top-k of the first 2^14 entries, then tensor-core
// passes over [2^14, 2^18), [2^18, 2^21), [2^21, 2^24) and the rest (ranges
// up to 1/2 of the library; FPS_MMA_PREFIX="18,21,24", FPS_MMA_SEED=14). Each
// pass starts from the exact top-k of everything before it (carried into its
// candidate lists), collects every pair within that bound, and its select is
// the exact top-k so far: the bound tightens 8-16x per pass while no entry is
// read twice. Candidates per query of a pass ~ k x n_scan / bound_n; the
// capacity is 8x that (+ the k carried), at least 16,384, and Q x cap x 8 B
// must fit the scratch budget (FPS_MMA_CAND_MB, default 1,024 MB). Returns
// false when it cannot: the batch then takes the bit-sliced kernel instead of
// overflowing. (C4: 8.81 ms per call with a 2^16 seed and a 2^22 prefix pass
// that the full pass scanned again; prefixes re-scanned by the full pass cost
// more than their tighter bound saves beyond 2^22.)
bool mma_plan(const fps_lib* L, u32 Q, u32 k, MmaPlan* p) {
  // (knobs read per call: batched calls are not latency bound, and tests set them at run time)
  const char* es = std::getenv("FPS_MMA_SEED");
  const int seed_log2 = es ? std::atoi(es) : 14;
  const char* ep = std::getenv("FPS_MMA_PREFIX");
  const std::string levels = ep ? ep : "18,21,24";
  const char* eb = std::getenv("FPS_MMA_CAND_MB");
  const u64 budget = (u64)(eb ? std::max(16, std::atoi(eb)) : 1024) << 20;
  // (whole 256-entry library tiles, at most half of the library; 0: no seed,
  // libraries below 512 entries are collected whole)
  p->seed_n = std::min<u64>(1ull << std::max(0, std::min(seed_log2, 40)), L->n / 2) / 256 * 256;
  p->npass = 0;
  u64 prev = p->seed_n;
  for (size_t pos = 0; pos < levels.size() && p->npass < MMA_MAX_PASS - 1;) {
    const size_t c = levels.find(',', pos);
    const int lg = std::atoi(levels.substr(pos, c == std::string::npos ? std::string::npos : c - pos).c_str());
    pos = c == std::string::npos ? levels.size() : c + 1;
    if (lg <= 0 || lg > 40) continue;
    const u64 m = 1ull << lg;
    if (m > prev && L->n >= 2 * m) p->n_scan[p->npass++] = prev = m;
  }
  p->n_scan[p->npass++] = L->n;
  for (int pass = 0; pass < p->npass; ++pass) {
    const u64 bound_n = pass == 0 ? p->seed_n : p->n_scan[pass - 1];
    const u64 expect = (u64)k * (p->n_scan[pass] / std::max<u64>(bound_n, 1) + 2);
    const u64 want = std::min<u64>(std::max<u64>(8 * expect, 16384), 1u << 22);
    const u64 fit = budget / ((u64)Q * 8);
    if (fit < 2 * expect || fit < 1024) return false;
    p->cap[pass] = (u32)std::min<u64>(want, fit);
  }
  return true;
}

bool mma_wanted(fps_lib* L, u32 Q, u32 k, MmaPlan* plan = nullptr) {
  const char* e = std::getenv("FPS_MMA");
  const int mode = e ? std::atoi(e) : -1;
  // compact libraries only: the fused test uses K slots 168.. (zero there)
  if (mode == 0 || Q < 2 || k > KMAX_FUSED || L->n < (u64)fps::MM_M || !L->compact) return false;
  if (mode != 1 && Q < 64) return false;  // (64-query top-k: 1.91 ms tensor vs 2.12 bit-sliced)
  MmaPlan p;
  if (!mma_plan(L, Q, k, &p)) return false;
  if (plan) *plan = p;
  return true;
}

// Operand kind of the tensor-core scan (FPS_MMA_KIND overrides). Default: the
// kind whose query chunks cost fewer ns per library tile -- "fp4x", the
// block-scaled fp4 kernel fed from the library's fp4 operand copy
// (fps_mma4x.cuh, chunks of <= 208 / 240 queries, ~303 ns per tile), or "i8",
// the int8 kernel (fps_mma.cuh, chunks of 256 queries, 16-bit packed
// accumulator reads, ~482 ns per tile). Measured on 95.4 M entries (scan
// kernel): 1,024 queries 7.63 ms fp4x vs 9.58 i8; 256 queries 2.43 ms i8 vs
// 2 fp4x chunks. "fp4" expands fp4 tiles in the kernel (fps_mma4.cuh). fp4x
// falls back to int8 when its copy (96 B/entry) does not fit.
enum MmaKind { MMA_I8 = 0, MMA_FP4 = 1, MMA_FP4X = 2 };
MmaKind mma_kind_env(u32 Q, u32 mode) {
  (void)mode;
  const char* e = std::getenv("FPS_MMA_KIND");
  if (!e) {
    // ties go to int8 (no operand copy)
    const u32 c4 = std::min((Q + 207) / 208, (Q + 239) / 240), c8 = (Q + 255) / 256;  // (mma_pick_n's chunks)
    return c4 * 310u < c8 * 482u ? MMA_FP4X : MMA_I8;
  }
  const std::string v(e);
  return v == "fp4" ? MMA_FP4 : v == "fp4x" ? MMA_FP4X : MMA_I8;
}

// Build (once) the fp4 operand copy; on failure (no memory) the scan uses int8.
int mq4x_ensure(fps_lib* L) {
  if (L->mq4x_state) return FPS_OK;
  if (!L->compact) {
    L->mq4x_state = -1;
    return FPS_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const u64 tiles = (L->n + fps::MM_M - 1) / fps::MM_M;
  if (L->mq4x.ensure((size_t)std::max<u64>(tiles, 1) * fps::MM4X_TILE)) {
    cudaGetLastError();
    L->mq4x_state = -1;
    return FPS_OK;
  }
  const int grid = (int)std::min<u64>((tiles * 6 * fps::MM_M + 255) / 256, (u64)L->sms * 32);
  fps::mm4x_build_kernel<<<std::max(grid, 1), 256, 0, L->stream>>>(L->out(), L->n, tiles, L->mq4x.as<unsigned char>());
  L->launches++;
  CUDA_TRY(cudaGetLastError());
  // tensor map over the copy: [tiles * 48 rows][256 B] u8, one 48-row box per tile
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      cudaGetLastError();
      return fail(FPS_ECUDA, "cuTensorMapEncodeTiled is not available from the driver");
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t gdim[2] = {fps::MM4X_ROW, (cuuint64_t)tiles * fps::MM4X_BOX_ROWS};
  const cuuint64_t gstride[1] = {fps::MM4X_ROW};
  const cuuint32_t box[2] = {fps::MM4X_ROW, fps::MM4X_BOX_ROWS};
  const cuuint32_t estride[2] = {1, 1};
  const CUresult cr = encode(&L->mq4x_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, L->mq4x.p, gdim, gstride, box, estride,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(FPS_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)cr) + ")");
  CUDA_TRY(cudaStreamSynchronize(L->stream));
  L->mq4x_state = 1;
  L->derived_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return FPS_OK;
}

// The kind a call runs: fp4x only once its operand copy exists.
MmaKind mma_kind(fps_lib* L, u32 Q, u32 mode) {
  MmaKind k = mma_kind_env(Q, mode);
  if (k == MMA_FP4X) {
    if (mq4x_ensure(L) != FPS_OK || L->mq4x_state != 1) k = MMA_I8;
  }
  return k;
}

// Accumulator width (queries per chunk). int8: 64 / 128 / 256. fp4: two
// accumulators + the scale factors fit 512 TMEM columns up to N = 240 (four
// at N = 64); e.g. 1,024 queries -> 5 chunks of 208.
u32 mma_pick_n(u32 Q, bool fp4) {
  if (!fp4) return Q <= 64 ? 64u : Q <= 128 ? 128u : 256u;
  if (Q <= 64) return 64u;
  if (Q <= 128) return 128u;
  // a tile costs about the same at any width (drain- and barrier-bound), so
  // the fewest chunks win; 208 over 240 on ties (measured: 9.21 ms for C4)
  return (Q + 239) / 240 < (Q + 207) / 208 ? 240u : 208u;
}

template <int N>
int mma_launch_n(fps_lib* L, u32 ctas, cudaStream_t s, const fps::MmArgs& a) {
  const size_t smem = fps::mm_b_bytes(N) + (size_t)fps::MM_STAGES * fps::MM_A_BYTES + (size_t)fps::MM_RAW * fps::MM_RAW_BYTES_MAX;
  CUDA_TRY(smem_optin((const void*)fps::mma_scan_kernel<N>, smem));
  auto* ev = timing_slot(L);
  if (ev) cudaEventRecord(ev->first, s);
  fps::mma_scan_kernel<N><<<ctas, fps::MM_THREADS, smem, s>>>(a);
  if (ev) cudaEventRecord(ev->second, s);
  L->launches++;
  LAUNCH_CHECK("mma_scan_kernel");
  return FPS_OK;
}

template <int N>
int mma4_launch_n(fps_lib* L, u32 ctas, cudaStream_t s, const fps::MmArgs& a) {
  const size_t smem = fps::mm4_smem(N);
  CUDA_TRY(smem_optin((const void*)fps::mma4_scan_kernel<N>, smem));
  auto* ev = timing_slot(L);
  if (ev) cudaEventRecord(ev->first, s);
  fps::mma4_scan_kernel<N><<<ctas, fps::MM_THREADS, smem, s>>>(a);
  if (ev) cudaEventRecord(ev->second, s);
  L->launches++;
  LAUNCH_CHECK("mma4_scan_kernel");
  return FPS_OK;
}

template <int N, int EPI, int NACC>
int mma4x_launch_ne(fps_lib* L, u32 ctas, cudaStream_t s, const fps::MmArgs& a) {
  const size_t smem = fps::mm4x_smem(N);
  CUDA_TRY(smem_optin((const void*)fps::mma4x_scan_kernel<N, EPI, NACC>, smem));
  auto* ev = timing_slot(L);
  if (ev) cudaEventRecord(ev->first, s);
  fps::mma4x_scan_kernel<N, EPI, NACC><<<ctas, fps::mm4x_threads(EPI), smem, s>>>(a, L->mq4x.as<unsigned char>(),
                                                                               L->mq4x_map);
  if (ev) cudaEventRecord(ev->second, s);
  L->launches++;
  LAUNCH_CHECK("mma4x_scan_kernel");
  return FPS_OK;
}
// Epilogue warps and accumulators of the fp4 operand-copy kernel.
template <int N>
int mma4x_launch_n(fps_lib* L, u32 ctas, cudaStream_t s, const fps::MmArgs& a) {
  // epilogue shape by width (FPS_MM4X_EPI=8 forces 8 warps on every tile):
  // N = 64: 4 accumulators, 4 groups of 4 warps (64 columns each; C5 scan
  // 1.87 -> 1.71 ms against 2 groups of 8); N = 128: 2 accumulators, 2 groups
  // of 8 warps (3 accumulators in 3 groups of 4 warps of 128 columns spill:
  // 13.7 -> 18.3 ms on C4 at N = 128)
  const char* e = std::getenv("FPS_MM4X_EPI");
  const int epi = e ? std::atoi(e) : 0;
  if constexpr (N <= 64) {
    if (epi != 8) return mma4x_launch_ne<N, 16, 4>(L, ctas, s, a);
  } else if constexpr (N <= 128) {
    if (epi != 8) return mma4x_launch_ne<N, 16, 2>(L, ctas, s, a);
  } else {
    // wider: 2 groups of 8 warps on alternate tiles, each warp draining its
    // <= 120 columns in two rounds (C4 scan 9.93 -> 9.21 ms against 8 warps
    // on every tile)
    if (epi != 8) return mma4x_launch_ne<N, 16, 2>(L, ctas, s, a);
  }
  return mma4x_launch_ne<N, 8, 2>(L, ctas, s, a);
}

// Shared part of the tensor-core calls: per-query operands from the bound
// mm_tq[q] (top-k: the seed's k-th distance; range: the radius), columns
// ordered by u = T - |q|, then the scan. mode 0 appends candidate keys to the
// per-query lists L->cand (capacity cap); mode 1 appends range hits to out.
int mma_run(fps_lib* L, const u64* d_q, u32 Q, u32 mode, u32 cap, u64* out, u64* out_cnt, u64 out_cap,
            cudaStream_t s, bool prepare_only, u64 n_scan = ~0ull, u64 n_start = 0) {
  int rc;
  const MmaKind kind = mma_kind(L, Q, mode);
  const bool fp4 = kind != MMA_I8;
  L->last_mma_kind = 1 + (int)kind;
  u32 NN = mma_pick_n(Q, fp4);
  if (const char* en = std::getenv("FPS_MMA_N"))  // experiments: accumulator width (fp4: 64/128/160/208/240)
    if (fp4) NN = (u32)std::atoi(en);
  const u32 nchunks = (Q + NN - 1) / NN;
  n_scan = std::min<u64>(n_scan, L->n);  // entries [n_start, n_scan) (a range pass of the top-k path)
  const u64 n_tiles = (n_scan + fps::MM_M - 1) / fps::MM_M;
  const u64 tile0 = std::min<u64>(n_start, n_scan) / 256 * 2;  // (whole 256-entry library tiles)
  const u32 parts = (u32)std::max<u64>(1, std::min<u64>(std::max<u32>(1, L->sms / nchunks), n_tiles - tile0));
  if ((rc = L->mm_bop.ensure((size_t)nchunks * (fp4 ? fps::mm4_b_bytes((int)NN) : fps::mm_b_bytes((int)NN)))) ||
      (rc = L->mm_ucol.ensure((size_t)nchunks * NN * 4)) || (rc = L->mm_qpop.ensure((size_t)nchunks * NN * 4)) ||
      (rc = L->mm_qcol.ensure((size_t)nchunks * NN * 4)) || (rc = L->mm_keys.ensure((size_t)Q * 8)) ||
      (rc = L->mm_sorted.ensure((size_t)Q * 8)))
    return rc;
  size_t tb = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, L->mm_keys.as<u64>(), L->mm_sorted.as<u64>(), (int)Q, 0, 64, s));
  if ((rc = L->mm_tmp.ensure(tb))) return rc;
  const u32 ctas = nchunks * parts;
  u64 pcap = 0;
  if (mode == 0) {
    // private per-(CTA, column) candidate lists: ~cap / parts expected per list
    pcap = std::max<u64>(256, 4 * (u64)cap / 8 / parts + 64);
    pcap = (pcap + 63) / 64 * 64;
    while (pcap > 256 && (u64)ctas * NN * pcap * 8 > (1ull << 30)) pcap /= 2;
    if ((rc = L->mm_priv.ensure((size_t)ctas * NN * pcap * 8))) return rc;  // before a graph capture
  }
  if (prepare_only) return FPS_OK;

  fps::mm_ukeys_kernel<<<(Q + 127) / 128, 128, 0, s>>>(d_q, Q, L->mm_tq.as<u32>(), L->mm_keys.as<u64>());
  CUDA_TRY(cub::DeviceRadixSort::SortKeys(L->mm_tmp.p, tb, L->mm_keys.as<u64>(), L->mm_sorted.as<u64>(), (int)Q, 0, 64, s));
  if (fp4)
    fps::mm4_prep_kernel<<<(nchunks * NN + 127) / 128, 128, 0, s>>>(
        d_q, Q, L->mm_tq.as<u32>(), L->mm_bop.as<unsigned char>(), L->mm_ucol.as<int>(), L->mm_qpop.as<u32>(), nchunks,
        L->mm_sorted.as<u64>(), L->mm_qcol.as<u32>(), NN);
  else
    fps::mm_prep_kernel<<<(nchunks * NN + 127) / 128, 128, 0, s>>>(
        d_q, Q, L->mm_tq.as<u32>(), L->mm_bop.as<unsigned char>(), L->mm_ucol.as<int>(), L->mm_qpop.as<u32>(), nchunks,
        L->mm_sorted.as<u64>(), L->mm_qcol.as<u32>(), NN);
  L->launches += 3;
  LAUNCH_CHECK("mm_prep");
  fps::MmArgs a{};
  a.lib = L->out();
  a.n = n_scan;
  a.index_base = L->index_base;
  a.n_tiles = n_tiles;
  a.tile0 = tile0;
  a.Q = Q;
  a.nchunks = nchunks;
  a.parts = parts;
  a.bop = L->mm_bop.as<unsigned char>();
  a.tcol = L->mm_ucol.as<int>();
  a.qpop = L->mm_qpop.as<u32>();
  a.qcol = L->mm_qcol.as<u32>();
  a.cand = L->cand.as<u64>();
  a.cand_cnt = L->cand_cnt.as<u32>();
  a.cap = cap;
  a.mode = mode;
  a.out = out;
  a.out_cnt = out_cnt;
  a.out_cap = out_cap;
  a.flags = scan_flags();
  {
    const char* e = std::getenv("FPS_MM_SUSPEND_NS");
    a.suspend_ns = e ? (u32)std::atoi(e) : 20000u;
  }
  if (mode == 0) {
    a.priv = L->mm_priv.as<u64>();
    a.pcap = (u32)pcap;
  }
  if (kind == MMA_FP4X) {
    if (NN == 64) return mma4x_launch_n<64>(L, ctas, s, a);
    if (NN == 128) return mma4x_launch_n<128>(L, ctas, s, a);
    if (NN == 160) return mma4x_launch_n<160>(L, ctas, s, a);
    if (NN == 208) return mma4x_launch_n<208>(L, ctas, s, a);
    return mma4x_launch_n<240>(L, ctas, s, a);
  }
  if (fp4) {
    if (NN == 64) return mma4_launch_n<64>(L, ctas, s, a);
    if (NN == 128) return mma4_launch_n<128>(L, ctas, s, a);
    if (NN == 160) return mma4_launch_n<160>(L, ctas, s, a);
    if (NN == 208) return mma4_launch_n<208>(L, ctas, s, a);
    return mma4_launch_n<240>(L, ctas, s, a);
  }
  if (NN == 64) return mma_launch_n<64>(L, ctas, s, a);
  if (NN == 128) return mma_launch_n<128>(L, ctas, s, a);
  return mma_launch_n<256>(L, ctas, s, a);
}

int topk_mma(fps_lib* L, const u64* d_q, u32 Q, u32 k, u64* d_keys, u32* d_cnt, cudaStream_t s, bool prepare_only,
             const MmaPlan& plan) {
  int rc;
  if ((rc = L->mm_ovf.ensure(256))) return rc;
  u32* ovf = L->mm_ovf.as<u32>();
  if ((rc = ensure_state(L, Q))) return rc;
  if (!prepare_only) CUDA_TRY(cudaMemsetAsync(ovf, 0, 4, s));
  // 1. seed bound: exact top-k of a short library prefix (POPC scan)
  if (plan.seed_n) {
    L->timing_suspend = true;
    rc = topk_fused<8, 2, true>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only, plan.seed_n);
    L->timing_suspend = false;
    if (rc) return rc;
  } else if (!prepare_only) {
    CUDA_TRY(cudaMemsetAsync(d_cnt, 0, (size_t)Q * 4, s));  // no seed: every pair is a candidate
  }
  // 2. tensor-core passes over growing ranges (mma_plan): each starts from the
  //    exact top-k of everything before it, carried into its candidate lists,
  //    and collects every pair within that bound -- so its select is the exact
  //    top-k so far and the next bound; no entry is read twice
  int kp = 1;
  while (kp < (int)k) kp <<= 1;
  for (int pass = 0; pass < plan.npass; ++pass) {
    const u64 n_start = pass == 0 ? plan.seed_n : plan.n_scan[pass - 1];
    const u64 n_scan = plan.n_scan[pass];
    const u32 cap = plan.cap[pass];
    if ((rc = L->mm_tq.ensure((size_t)Q * 4)) || (rc = L->cand.ensure((size_t)Q * cap * 8))) return rc;
    if (!prepare_only) {
      fps::mm_seed_kernel<<<(Q + 127) / 128, 128, 0, s>>>(d_keys, d_cnt, Q, k, L->mm_tq.as<u32>());
      fps::bs_seed_tg<<<(Q + 127) / 128, 128, 0, s>>>(d_keys, d_cnt, Q, k, L->tg.as<u32>(), tg_replicas(Q),
                                                       ghist_stride(Q));
      fps::mm_carry_kernel<<<dim3((k + 127) / 128, Q), 128, 0, s>>>(d_keys, d_cnt, k, L->cand.as<u64>(),
                                                                    L->cand_cnt.as<u32>(), cap);
      L->launches += 3;
    }
    L->timing_continue = pass > 0;  // the passes of a call are one timed scan
    rc = mma_run(L, d_q, Q, 0, cap, nullptr, nullptr, 0, s, prepare_only, n_scan, n_start);
    L->timing_continue = false;
    if (rc) return rc;
    if (prepare_only) continue;
    // distances of the collected pairs (the scan stores their indices)
    fps::mm_fix_kernel<<<dim3(4, Q), 256, 0, s>>>(L->out(), L->index_base, d_q, L->cand.as<u64>(),
                                                  L->cand_cnt.as<u32>(), cap, nullptr, 0);
    L->launches++;
    LAUNCH_CHECK("mm_fix_kernel");
    // a list past its capacity sets *ovf (its pass's bound, and so the next
    // pass, may then be wrong: the gated pass below recomputes everything)
    CUDA_TRY(launch_select(Q, (size_t)(kp + fps::SEL_ECAP) * 8, s, L->cand.as<u64>(), L->cand_cnt.as<u32>(), cap,
                           L->tg.as<u32>(), L->ghist.as<u32>(), ghist_stride(Q), tg_replicas(Q), k, d_keys, d_cnt,
                           false, nullptr, nullptr, 0, nullptr, ovf));
    L->launches++;
    LAUNCH_CHECK("select_kernel (mma)");
  }
  // 3. device-side fallback (adversarial ties): an exact POPC pass over the
  //    whole library that runs only when a candidate list overflowed
  L->timing_suspend = true;
  rc = topk_fused<8, 2, true>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only, 0, nullptr, ovf);
  L->timing_suspend = false;
  return rc;
}

// Range search on the tensor cores: the bound is the radius itself (exact,
// no seed); hits go straight to the range output. FPS_MMA=0 disables it,
// FPS_MMA=1 forces it for any batch >= 2; by default it serves batches of
// >= FPS_MMA_RANGE_MIN_Q (default 64) queries (C5, 64 queries: the fp4
// operand-copy kernel 1.87 ms against the bit-sliced kernel's 2.21 ms).
bool mma_range_wanted(fps_lib* L, u32 Q, cudaStream_t s) {
  const char* e = std::getenv("FPS_MMA");
  const int mode = e ? std::atoi(e) : -1;
  if (mode == 0 || Q < 2 || L->n < (u64)fps::MM_M || !L->compact) return false;
  const char* m = std::getenv("FPS_MMA_RANGE_MIN_Q");
  if (mode != 1 && Q < (u32)(m ? std::atoi(m) : 64)) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return false;
  }
  return true;
}

int range_mma(fps_lib* L, const u64* d_q, u32 Q, const unsigned char* d_radius, u64* d_out, u64 cap, u64* d_count,
              cudaStream_t s) {
  int rc;
  if ((rc = L->mm_tq.ensure((size_t)Q * 4))) return rc;
  fps::mm_radius_kernel<<<(Q + 127) / 128, 128, 0, s>>>(d_radius, Q, L->mm_tq.as<u32>());
  L->launches++;
  if ((rc = mma_run(L, d_q, Q, 1, 0, d_out, d_count, cap, s, false))) return rc;
  // distances of the hits (the scan stores query and index)
  fps::mm_fix_kernel<<<L->sms * 4, 256, 0, s>>>(L->out(), L->index_base, d_q, d_out, nullptr, 0, d_count, cap);
  L->launches++;
  LAUNCH_CHECK("mm_fix_kernel (range)");
  return FPS_OK;
}

int topk_dispatch(fps_lib* L, const u64* d_q, u32 Q, u32 k, u64* d_keys, u32* d_cnt, cudaStream_t s,
                  bool prepare_only) {
  MmaPlan plan;
  if (mma_wanted(L, Q, k, &plan)) {
    L->last_kernel = 6;
    return topk_mma(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only, plan);
  }
  if (Q == 1 && pq_wanted(L)) return topk_pq(L, d_q, nullptr, k, d_keys, d_cnt, s, prepare_only);
  if (bs_wanted(L, Q)) {
    L->last_kernel = 3;
    return L->compact ? topk_bs<true>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only)
                      : topk_bs<false>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
  }
  int qw, e;
  pick_shape(Q, &qw, &e);
  L->last_kernel = qw == 1 ? 1 : 2;
  if (L->compact) {
    if (qw == 1) return topk_fused<1, 4, true>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
    if (qw == 2) return topk_fused<2, 2, true>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
    if (qw == 4) return topk_fused<4, 2, true>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
    return topk_fused<8, 2, true>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
  }
  if (qw == 1) return topk_fused<1, 4, false>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
  if (qw == 2) return topk_fused<2, 2, false>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
  if (qw == 4) return topk_fused<4, 2, false>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
  return topk_fused<8, 2, false>(L, d_q, Q, k, d_keys, d_cnt, s, prepare_only);
}

template <int QW, int E, int MODE, bool CMP>
int launch_plain(fps_lib* L, fps::ScanArgs a, cudaStream_t s) {
  Config c = make_config<QW, E, MODE, false, CMP>(L, a.Q, 1);
  a.n_qg = c.n_qg;
  a.n_parts = c.n_parts;
  a.iters = c.iters;
  if (c.warps == 0 || L->n == 0) return FPS_OK;
  auto* ev = timing_slot(L);
  if (ev) cudaEventRecord(ev->first, s);
  fps::scan_kernel<QW, E, MODE, false, CMP><<<c.grid, WPB * 32, c.smem, s>>>(a);
  if (ev) cudaEventRecord(ev->second, s);
  L->launches++;
  CUDA_TRY(cudaGetLastError());
  return FPS_OK;
}

template <int MODE>
int plain_dispatch(fps_lib* L, const fps::ScanArgs& a, cudaStream_t s) {
  if (MODE == fps::MODE_RANGE && mma_range_wanted(L, a.Q, s)) {
    L->last_kernel = 6;
    return range_mma(L, a.queries, a.Q, a.radius, a.out, a.out_cap, a.out_cnt, s);
  }
  if (MODE == fps::MODE_RANGE && bs_wanted(L, a.Q)) {
    L->last_kernel = 3;
    return range_bs(L, a.queries, a.Q, a.radius, a.out, a.out_cap, a.out_cnt, s);
  }
  int qw, e;
  pick_shape(a.Q, &qw, &e);
  L->last_kernel = qw == 1 ? 1 : 2;
  if (L->compact) {
    if (qw == 1) return launch_plain<1, 4, MODE, true>(L, a, s);
    if (qw == 2) return launch_plain<2, 2, MODE, true>(L, a, s);
    if (qw == 4) return launch_plain<4, 2, MODE, true>(L, a, s);
    return launch_plain<8, 2, MODE, true>(L, a, s);
  }
  if (qw == 1) return launch_plain<1, 4, MODE, false>(L, a, s);
  if (qw == 2) return launch_plain<2, 2, MODE, false>(L, a, s);
  if (qw == 4) return launch_plain<4, 2, MODE, false>(L, a, s);
  return launch_plain<8, 2, MODE, false>(L, a, s);
}

int sort_keys(fps_lib* L, u64* d_keys, u64 n, cudaStream_t s) {
  if (n <= 1) return FPS_OK;
  if (n > (u64)INT32_MAX) return fail(FPS_ENOMEM, "range output exceeds 2^31 hits");
  DevBuf tmp_local, out_local;
  DevBuf& tmp = L ? L->sort_tmp : tmp_local;
  DevBuf& out = L ? L->sort_out : out_local;
  size_t tmp_bytes = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, d_keys, d_keys, (int)n, 0, 64, s));
  int rc;
  if ((rc = tmp.ensure(tmp_bytes))) return rc;
  if ((rc = out.ensure(n * 8))) return rc;
  CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, d_keys, out.as<u64>(), (int)n, 0, 64, s));
  CUDA_TRY(cudaMemcpyAsync(d_keys, out.p, n * 8, cudaMemcpyDeviceToDevice, s));
  if (L) L->launches += 2;
  if (!L) {
    cudaStreamSynchronize(s);
    tmp_local.release();
    out_local.release();
  }
  return FPS_OK;
}

// Range hits (unsorted) into L->rkeys; grows and retries on overflow.
int range_collect(fps_lib* L, const u64* d_q, u32 Q, const unsigned char* d_radius, u64* n_hits, u64 cap_hint) {
  u64 cap = std::max<u64>(cap_hint, 1 << 20);
  int rc;
  if ((rc = L->rcount.ensure(8))) return rc;
  for (int attempt = 0; attempt < 3; ++attempt) {
    if ((rc = L->rkeys.ensure(cap * 8))) return rc;
    cap = L->rkeys.bytes / 8;
    CUDA_TRY(cudaMemsetAsync(L->rcount.p, 0, 8, L->stream));
    fps::ScanArgs a = base_args(L, d_q, Q);
    a.radius = d_radius;
    a.out = L->rkeys.as<u64>();
    a.out_cnt = L->rcount.as<u64>();
    a.out_cap = cap;
    if ((rc = plain_dispatch<fps::MODE_RANGE>(L, a, L->stream))) return rc;
    u64 count = 0;
    CUDA_TRY(cudaMemcpyAsync(&count, L->rcount.p, 8, cudaMemcpyDeviceToHost, L->stream));
    CUDA_TRY(cudaStreamSynchronize(L->stream));
    if (count <= cap) {
      *n_hits = count;
      return FPS_OK;
    }
    cap = count + count / 8 + 1024;
  }
  return fail(FPS_ECUDA, "range output kept growing between attempts");
}

int check_lib(const fps_lib* L) {
  if (!L) return fail(FPS_EINVAL, "null library handle");
  return FPS_OK;
}

int stage_queries(fps_lib* L, const uint64_t* queries, u32 Q) {
  int rc;
  if ((rc = L->queries.ensure((size_t)Q * 24))) return rc;
  if ((rc = L->h_stage.ensure((size_t)Q * 24))) return rc;
  std::memcpy(L->h_stage.p, queries, (size_t)Q * 24);
  CUDA_TRY(cudaMemcpyAsync(L->queries.p, L->h_stage.p, (size_t)Q * 24, cudaMemcpyHostToDevice, L->stream));
  return FPS_OK;
}

// The compact 21 B/entry tiles (word 2 as u32 + u8) read 12.5 % fewer bytes;
// with the bulk-copy scan they are faster in every config (C3 scan 319 ->
// 289 us, profiles/r01_experiments.md), so they are the default whenever no
// entry uses bits 40.. of word 2. FPS_LAYOUT=full forces the 24 B tiles.
bool force_full_layout() {
  const char* e = std::getenv("FPS_LAYOUT");
  return e && std::string(e) == "full";
}

int alloc_planes(fps_lib* L, u64 n, bool compact) {
  L->n = n;
  L->compact = compact && !force_full_layout();
  // whole tiles plus two tiles of zero slack (vector loads never leave the allocation)
  const u64 te = fps::tile_entries(L->compact);
  const u64 tiles = (n + te - 1) / te + 2;
  L->n_alloc = tiles * te;
  const size_t bytes = (size_t)tiles * fps::tile_bytes(L->compact);
  cudaError_t e = cudaMalloc(&L->mem, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    L->mem = nullptr;
    return fail(FPS_ENOMEM, std::string("library cudaMalloc(") + std::to_string(bytes) +
                                "): " + cudaGetErrorString(e));
  }
  CUDA_TRY(cudaMemsetAsync(L->mem, 0, bytes, L->stream));
  return FPS_OK;
}

int new_lib(int device, u64 index_base, fps_lib** out) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(FPS_ENODEV, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail(FPS_EINVAL, "device ordinal out of range");
  if (index_base + 0 > fps::IDX_MASK) return fail(FPS_EINVAL, "index_base exceeds 2^40");
  CUDA_TRY(cudaSetDevice(device));
  fps_lib* L = new fps_lib();
  L->device = device;
  L->index_base = index_base;
  cudaDeviceGetAttribute(&L->sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete L;
    return fail(FPS_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
  }
  *out = L;
  return FPS_OK;
}

// Release everything the handle owns. The DevBuf / HostBuf members free
// themselves when the handle is deleted (with its device current); raw
// allocations, graphs, events and the stream are released here.
void destroy(fps_lib* L) {
  if (!L) return;
  DeviceGuard g(L->device);
  if (L->stream) cudaStreamSynchronize(L->stream);
  if (L->mem) cudaFree(L->mem);
  L->mem = nullptr;
  if (L->hmap) cudaFreeHost(L->hmap);
  L->hmap = nullptr;
  for (auto* gr : L->graphs) {
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    delete gr;
  }
  L->graphs.clear();
  for (auto& p : L->ev_pool) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  L->ev_pool.clear();
  if (L->ev_join) cudaEventDestroy(L->ev_join);
  if (L->ev_done) cudaEventDestroy(L->ev_done);
  if (L->stream) cudaStreamDestroy(L->stream);
  L->stream = nullptr;
  delete L;  // member buffers are freed here, device still current
}

void unpack_topk(const u64* keys, const u32* cnt, u32 Q, u32 k, uint64_t* out_idx, uint16_t* out_dist,
                 uint32_t* out_cnt) {
  for (u32 q = 0; q < Q; ++q) {
    out_cnt[q] = cnt[q];
    for (u32 i = 0; i < k; ++i) {
      u64 key = keys[(u64)q * k + i];
      bool ok = i < cnt[q];
      if (out_idx) out_idx[(u64)q * k + i] = ok ? (key & fps::IDX_MASK) : UINT64_MAX;
      if (out_dist) out_dist[(u64)q * k + i] = ok ? (uint16_t)fps::key_d(key) : 0xFFFF;
    }
  }
}

// Large-k path (k > KMAX_FUSED): exact distance histogram -> per-query
// threshold T_q -> range collection with radius T_q -> sort -> first k.
int topk_large(fps_lib* L, const u64* d_q, u32 Q, u32 k, u64* d_keys, u32* d_cnt) {
  int rc;
  L->last_kernel = 4;
  if ((rc = ensure_state(L, Q))) return rc;
  CUDA_TRY(cudaMemsetAsync(L->ghist.p, 0, (size_t)Q * fps::HB * 4, L->stream));
  fps::ScanArgs a = base_args(L, d_q, Q);
  a.ghist = L->ghist.as<u32>();
  a.gstride = 1;  // dense: read back by the host
  if ((rc = plain_dispatch<fps::MODE_HIST>(L, a, L->stream))) return rc;
  std::vector<u32> hist((size_t)Q * fps::HB);
  CUDA_TRY(cudaMemcpyAsync(hist.data(), L->ghist.p, hist.size() * 4, cudaMemcpyDeviceToHost, L->stream));
  CUDA_TRY(cudaMemsetAsync(L->ghist.p, 0, (size_t)Q * fps::HB * 4, L->stream));
  CUDA_TRY(cudaStreamSynchronize(L->stream));
  std::vector<unsigned char> rad(Q);
  std::vector<u64> seg(Q + 1, 0);
  for (u32 q = 0; q < Q; ++q) {
    u64 c = 0;
    int t = 255;
    for (int b = 0; b < fps::HB; ++b) {
      c += hist[(size_t)q * fps::HB + b];
      if (c >= k) { t = b; break; }
    }
    if (t == 255) {  // fewer than k entries: take all
      c = 0;
      for (int b = 0; b < fps::HB; ++b) c += hist[(size_t)q * fps::HB + b];
      t = 254;
    }
    rad[q] = (unsigned char)t;
    seg[q + 1] = seg[q] + c;
  }
  if ((rc = L->radius.ensure(Q))) return rc;
  CUDA_TRY(cudaMemcpyAsync(L->radius.p, rad.data(), Q, cudaMemcpyHostToDevice, L->stream));
  u64 hits = 0;
  if ((rc = range_collect(L, d_q, Q, L->radius.as<unsigned char>(), &hits, seg[Q] + 1))) return rc;
  if (hits != seg[Q]) return fail(FPS_ECUDA, "large-k collection count disagrees with the histogram");
  if ((rc = sort_keys(L, L->rkeys.as<u64>(), hits, L->stream))) return rc;
  if ((rc = L->seg.ensure((size_t)(Q + 1) * 8))) return rc;
  CUDA_TRY(cudaMemcpyAsync(L->seg.p, seg.data(), (size_t)(Q + 1) * 8, cudaMemcpyHostToDevice, L->stream));
  fps::truncate_kernel<<<Q, 256, 0, L->stream>>>(L->rkeys.as<u64>(), L->seg.as<u64>(), Q, k, d_keys, d_cnt);
  L->launches++;
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(L->stream));
  return FPS_OK;
}

// Sorted range keys on the device -> query / index / distance host columns,
// through a pinned double buffer: chunk c + 1 copies while chunk c is split
// (host threads measured slower: spawning them costs more than the split,
// which is bounded by first-touch faults on the fresh columns).
cudaError_t fetch_columns(cudaStream_t s, const u64* src, u64 n, HostBuf* hr, uint32_t* out_query,
                          uint64_t* out_index, uint16_t* out_dist) {
  constexpr u64 CH = 1 << 17;  // keys per chunk (1 MiB)
  if (n == 0) return cudaSuccess;
  if (hr[0].ensure(CH * 8) || hr[1].ensure(CH * 8)) return cudaErrorMemoryAllocation;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  auto issue = [&](u64 c) {
    const u64 lo = c * CH, m = std::min<u64>(CH, n - lo);
    cudaMemcpyAsync(hr[c & 1].p, src + lo, m * 8, cudaMemcpyDeviceToHost, s);
    cudaEventRecord(ev[c & 1], s);
  };
  const u64 chunks = (n + CH - 1) / CH;
  issue(0);
  cudaError_t e = cudaSuccess;
  for (u64 c = 0; c < chunks && e == cudaSuccess; ++c) {
    e = cudaEventSynchronize(ev[c & 1]);
    if (c + 1 < chunks) issue(c + 1);
    const u64 lo = c * CH, m = std::min<u64>(CH, n - lo);
    fps_range_unpack(reinterpret_cast<const uint64_t*>(hr[c & 1].p), m, out_query + lo, out_index + lo, out_dist + lo);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  for (auto& x : ev) cudaEventDestroy(x);
  return e;
}

// Order the handle's own stream after the work queued so far on s: the
// large-k path and the range collection run on L->stream and synchronise on
// it (their sizes are data dependent), so a caller's stream hands over here.
int join_stream(fps_lib* L, cudaStream_t s) {
  if (s == L->stream) return FPS_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return fail(FPS_EINVAL, "k > 1024 synchronises on the host and cannot be captured in a graph");
  }
  if (!L->ev_join) CUDA_TRY(cudaEventCreateWithFlags(&L->ev_join, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(L->ev_join, s));
  CUDA_TRY(cudaStreamWaitEvent(L->stream, L->ev_join, 0));
  return FPS_OK;
}

// Per-query top-k for any k >= 1 on stream s: the fused kernels for
// k <= 1024, else the large-k path (which synchronises).
int topk_any(fps_lib* L, const u64* d_q, u32 Q, u32 k, u64* d_keys, u32* d_cnt, cudaStream_t s) {
  if (k <= KMAX_FUSED) return topk_dispatch(L, d_q, Q, k, d_keys, d_cnt, s, false);
  int rc;
  if ((rc = join_stream(L, s))) return rc;
  return topk_large(L, d_q, Q, k, d_keys, d_cnt);
}

// Min-over-queries top-k (the reference batch_search, scan.py:306-318) on
// stream s, results left on the device: d_out[k] keys, *d_cnt.
//  * per-query path (batches on the bit-sliced / tensor-core kernels, and any
//    k > 1024): per-query top-k lists, then the min merge -- exact, because an
//    entry's best query ranks it no lower than the global order does, so the
//    global top-k is inside the union of the per-query lists, and its score
//    is its smallest listed distance;
//  * otherwise one POPC pass that scores every entry by its minimum distance.
int topk_min_dev(fps_lib* L, const u64* d_q, u32 Q, u32 k, u64* d_out, u32* d_cnt, cudaStream_t s) {
  int rc;
  if (Q == 0 || k == 0) return fail(FPS_EINVAL, "Q and k must be >= 1");
  const bool perq = (Q >= 2 && bs_wanted(L, Q)) || k > KMAX_FUSED;
  if (perq) {
    const u64 n = (u64)Q * k;
    if ((rc = L->mq.ensure(n * 8 * 3 + (size_t)Q * 4 + 16))) return rc;
    u64* pk = L->mq.as<u64>();  // per-query keys
    u64* tmp = pk + n;
    u64* out = tmp + n;
    u32* pc = reinterpret_cast<u32*>(out + n);
    u32* firsts = pc + Q;
    if ((rc = topk_any(L, d_q, Q, k, pk, pc, s))) return rc;
    const int blocks = (int)std::min<u64>((n + 255) / 256, 4096);
    fps::minq_flip<<<blocks, 256, 0, s>>>(pk, pc, Q, k, tmp);
    if ((rc = sort_keys(L, tmp, n, s))) return rc;
    CUDA_TRY(cudaMemsetAsync(firsts, 0, 4, s));
    fps::minq_first<<<blocks, 256, 0, s>>>(tmp, n, out, firsts);
    if ((rc = sort_keys(L, out, n, s))) return rc;
    fps::minq_emit<<<(k + 255) / 256, 256, 0, s>>>(out, firsts, k, d_out, d_cnt);
    L->launches += 3;
    LAUNCH_CHECK("minq merge");
    return FPS_OK;
  }
  Config c = L->compact ? make_config<1, 4, fps::MODE_TOPK, true, true>(L, 1, k)
                        : make_config<1, 4, fps::MODE_TOPK, true, false>(L, 1, k);
  if ((rc = ensure_state(L, 1))) return rc;
  if ((rc = L->buf.ensure(c.warps * (size_t)c.cap * 8))) return rc;
  if ((rc = L->cand.ensure(c.cand_cap * 8))) return rc;
  fps::ScanArgs a = base_args(L, d_q, 1);
  a.Qmin = Q;
  a.k = k;
  a.cap = c.cap;
  a.n_qg = 1;
  a.n_parts = c.n_parts;
  a.iters = c.iters;
  a.tg = L->tg.as<u32>();
  a.ghist = L->ghist.as<u32>();
  a.gstride = ghist_stride(1);
  a.tg_rep = tg_replicas(1);
  a.pub_every = (u32)std::max<u64>(1, c.n_parts / 512);
  a.buf = L->buf.as<u64>();
  a.cand = L->cand.as<u64>();
  a.cand_cnt = L->cand_cnt.as<u32>();
  a.cand_cap = c.cand_cap;
  if (L->compact) set_dyn<1, 4, fps::MODE_TOPK, true>(L, a);
  else set_dyn<1, 4, fps::MODE_TOPK, false>(L, a);
  L->last_kernel = 1;
  if (c.warps > 0 && L->n > 0) {
    if (L->compact) fps::scan_kernel<1, 4, fps::MODE_TOPK, true, true><<<c.grid, WPB * 32, c.smem, s>>>(a);
    else fps::scan_kernel<1, 4, fps::MODE_TOPK, true, false><<<c.grid, WPB * 32, c.smem, s>>>(a);
    L->launches++;
  }
  LAUNCH_CHECK("scan_kernel<min over queries>");
  int kp = 1;
  while (kp < (int)k) kp <<= 1;
  CUDA_TRY(launch_select(1, (size_t)(kp + fps::SEL_ECAP) * 8, s, a.cand, a.cand_cnt, c.cand_cap, a.tg, a.ghist,
                         a.gstride, a.tg_rep, k, d_out, d_cnt, true, a.dyn_ctr));
  L->launches++;
  LAUNCH_CHECK("select_kernel (min over queries)");
  return FPS_OK;
}

}  // namespace

// error message setter for the host-only ingestion code (fps_ingest.cpp)
void fps_set_last_error(const std::string& msg) { g_err = msg; }

extern "C" {

int fps_version(void) { return FPS_ABI_VERSION; }

const char* fps_last_error(void) { return g_err.c_str(); }

int fps_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return FPS_OK;
}

int fps_open(const uint64_t* words, uint64_t n, int layout, int device, uint64_t index_base, int check_padding,
             fps_lib** out) {
  if (!out) return fail(FPS_EINVAL, "out is null");
  *out = nullptr;
  if (n > 0 && !words) return fail(FPS_EINVAL, "words is null");
  if (index_base + n > fps::IDX_MASK) return fail(FPS_EINVAL, "library indices exceed 2^40");
  int stride, col0;
  if (layout == FPS_LAYOUT_ROWS3) { stride = 3; col0 = 0; }
  else if (layout == FPS_LAYOUT_FPS1) { stride = 4; col0 = 1; }
  else if (layout == FPS_LAYOUT_PLANES) { stride = 1; col0 = 0; }
  else return fail(FPS_EINVAL, "unknown layout");
  // Host pre-scan: the compact layout keeps bits 0..39 of word 2, so it is
  // exact iff no entry sets bits 40.. (always true for valid fingerprints;
  // FPS1 pad bytes are scanned as stored, like the reference).
  bool wide = false;
  for (u64 i = 0; i < n && !wide; ++i) {
    const u64 c = layout == FPS_LAYOUT_PLANES ? words[2 * n + i] : words[i * stride + col0 + 2];
    wide = (c >> 40) != 0;
  }
  fps_lib* L = nullptr;
  int rc = new_lib(device, index_base, &L);
  if (rc) return rc;
  DeviceGuard g(device);
  if ((rc = alloc_planes(L, n, !wide))) { destroy(L); return rc; }
  DevBuf bad;
  if ((rc = bad.ensure(4))) { destroy(L); return rc; }
  cudaMemsetAsync(bad.p, 0, 4, L->stream);
  if (layout == FPS_LAYOUT_PLANES && n) {
    DevBuf tmp;
    if ((rc = tmp.ensure((size_t)n * 24))) { destroy(L); return rc; }
    cudaMemcpyAsync(tmp.p, words, (size_t)n * 24, cudaMemcpyHostToDevice, L->stream);
    int blocks = (int)std::min<u64>((n + 255) / 256, 4096);
    fps::planes_to_planes<<<blocks, 256, 0, L->stream>>>(tmp.as<u64>(), tmp.as<u64>() + n, tmp.as<u64>() + 2 * n,
                                                          n, L->out());
    L->launches++;
    cudaStreamSynchronize(L->stream);
    tmp.release();
  } else if (n) {
    // stream rows through a pinned staging buffer in chunks, transposing on device
    const u64 chunk = 1 << 20;  // rows per chunk
    HostBuf hb;
    DevBuf db;
    if ((rc = hb.ensure((size_t)chunk * stride * 8)) || (rc = db.ensure((size_t)chunk * stride * 8))) {
      destroy(L);
      return rc;
    }
    for (u64 s = 0; s < n; s += chunk) {
      u64 m = std::min<u64>(chunk, n - s);
      cudaStreamSynchronize(L->stream);  // staging buffer reuse
      std::memcpy(hb.p, words + s * stride, (size_t)m * stride * 8);
      cudaMemcpyAsync(db.p, hb.p, (size_t)m * stride * 8, cudaMemcpyHostToDevice, L->stream);
      int blocks = (int)std::min<u64>((m + 255) / 256, 4096);
      fps::rows_to_planes<<<blocks, 256, 0, L->stream>>>(db.as<u64>(), m, stride, col0, L->out(), s,
                                                        check_padding ? bad.as<u32>() : nullptr);
      L->launches++;
    }
    cudaStreamSynchronize(L->stream);
    hb.release();
    db.release();
  }
  u32 nbad = 0;
  cudaMemcpyAsync(&nbad, bad.p, 4, cudaMemcpyDeviceToHost, L->stream);
  cudaError_t e = cudaStreamSynchronize(L->stream);
  bad.release();
  if (e != cudaSuccess) {
    destroy(L);
    return fail(FPS_ECUDA, std::string("library upload: ") + cudaGetErrorString(e));
  }
  if (layout == FPS_LAYOUT_PLANES && check_padding) {
    for (u64 i = 0; i < n; ++i)
      if (words[2 * n + i] >> 38) { nbad = 1; break; }
  }
  if (nbad) {
    destroy(L);
    return fail(FPS_EPADDING, "padding bits above key 166 must be zero");
  }
  *out = L;
  return FPS_OK;
}

int fps_open_device(const uint64_t* d_w0, const uint64_t* d_w1, const uint64_t* d_w2, uint64_t n, int device,
                    uint64_t index_base, fps_lib** out) {
  if (!out) return fail(FPS_EINVAL, "out is null");
  *out = nullptr;
  if (index_base + n > fps::IDX_MASK) return fail(FPS_EINVAL, "library indices exceed 2^40");
  fps_lib* L = nullptr;
  int rc = new_lib(device, index_base, &L);
  if (rc) return rc;
  DeviceGuard g(device);
  u32 nwide = 0;
  if (n) {
    DevBuf wide;
    if ((rc = wide.ensure(4))) { destroy(L); return rc; }
    cudaMemsetAsync(wide.p, 0, 4, L->stream);
    int blocks = (int)std::min<u64>((n + 255) / 256, 4096);
    fps::count_wide<<<blocks, 256, 0, L->stream>>>((const u64*)d_w2, n, wide.as<u32>());
    cudaMemcpyAsync(&nwide, wide.p, 4, cudaMemcpyDeviceToHost, L->stream);
    cudaStreamSynchronize(L->stream);
  }
  if ((rc = alloc_planes(L, n, nwide == 0))) { destroy(L); return rc; }
  if (n) {
    int blocks = (int)std::min<u64>((n + 255) / 256, 4096);
    fps::planes_to_planes<<<blocks, 256, 0, L->stream>>>((const u64*)d_w0, (const u64*)d_w1, (const u64*)d_w2, n,
                                                          L->out());
    L->launches++;
  }
  cudaError_t e = cudaStreamSynchronize(L->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    destroy(L);
    return fail(FPS_ECUDA, std::string("device upload: ") + cudaGetErrorString(e));
  }
  *out = L;
  return FPS_OK;
}

int fps_open_fps1(const char* const* paths, uint32_t n_paths, uint64_t start, uint64_t count, int device,
                  uint64_t* cids, fps_lib** out) {
  if (!out) return fail(FPS_EINVAL, "out is null");
  *out = nullptr;
  if (n_paths && !paths) return fail(FPS_EINVAL, "paths is null");
  // 1. validate every header first (no device work yet): magic, version, count vs size
  struct ShardFile {
    std::string path;
    u64 count;
  };
  std::vector<ShardFile> files;
  u64 total = 0;
  for (u32 f = 0; f < n_paths; ++f) {
    const std::string path = paths[f] ? paths[f] : "";
    FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) return fail(FPS_EIO, "shard " + path + ": " + std::strerror(errno));
    unsigned char h[16];
    const size_t got = std::fread(h, 1, 16, fp);
    std::fseek(fp, 0, SEEK_END);
    const long long size = std::ftell(fp);
    std::fclose(fp);
    if (got < 16) return fail(FPS_EIO, "shard " + path + ": header is " + std::to_string(got) + " bytes, expected 16");
    if (std::memcmp(h, "FPS1", 4) != 0) return fail(FPS_EIO, "shard " + path + ": bad magic, expected 'FPS1'");
    const unsigned version = h[4] | (h[5] << 8);
    if (version != 1)
      return fail(FPS_EIO, "shard " + path + ": format version " + std::to_string(version) + ", expected 1");
    u64 n = 0;
    for (int i = 0; i < 8; ++i) n |= (u64)h[8 + i] << (8 * i);
    if ((u64)size < 16 + n * 32) {
      return fail(FPS_EIO, "shard " + path + ": holds " + std::to_string(((u64)size - 16) / 32) +
                               " records, header declares " + std::to_string(n));
    }
    files.push_back({path, n});
    total += n;
  }
  if (start > total) return fail(FPS_EINVAL, "start beyond the last record");
  const u64 n = std::min<u64>(count, total - start);
  if (start + n > fps::IDX_MASK) return fail(FPS_EINVAL, "library indices exceed 2^40");
  fps_lib* L = nullptr;
  int rc = new_lib(device, start, &L);
  if (rc) return rc;
  DeviceGuard g(device);
  // 2. stream: read chunk i+1 from disk while chunk i is copied and transposed
  const u64 chunk = 1 << 20;  // records per chunk (32 MiB)
  HostBuf hb[2];
  DevBuf db[2];
  cudaEvent_t done[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b) {
    if ((rc = hb[b].ensure((size_t)chunk * 32)) || (rc = db[b].ensure((size_t)chunk * 32))) {
      destroy(L);
      return rc;
    }
    cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
  }
  // records of the slice use the compact layout only when no record sets bits 40.. of word 2;
  // decided up front from a full pass would cost a second read, so the 24 B layout is used
  if ((rc = alloc_planes(L, n, false))) { destroy(L); return rc; }
  u64 base = 0, dst = 0;  // global index of the current file's first record; entries written
  int slot = 0;
  for (const ShardFile& sf : files) {
    const u64 f0 = base, f1 = base + sf.count;
    base = f1;
    const u64 lo = std::max<u64>(f0, start), hi = std::min<u64>(f1, start + n);
    if (lo >= hi) continue;
    FILE* fp = std::fopen(sf.path.c_str(), "rb");
    if (!fp) { destroy(L); return fail(FPS_EIO, "shard " + sf.path + ": " + std::strerror(errno)); }
    std::fseek(fp, (long)(16 + (lo - f0) * 32), SEEK_SET);
    for (u64 r = lo; r < hi; r += chunk) {
      const u64 m = std::min<u64>(chunk, hi - r);
      cudaEventSynchronize(done[slot]);  // the copy that last used this pinned buffer has finished
      const size_t got = std::fread(hb[slot].p, 32, m, fp);
      if (got != m) {
        std::fclose(fp);
        destroy(L);
        return fail(FPS_EIO, "shard " + sf.path + ": truncated while reading");
      }
      if (cids) {
        const u64* rec = hb[slot].as<u64>();
        for (u64 i = 0; i < m; ++i) cids[dst + i] = rec[4 * i];
      }
      cudaMemcpyAsync(db[slot].p, hb[slot].p, m * 32, cudaMemcpyHostToDevice, L->stream);
      const int blocks = (int)std::min<u64>((m + 255) / 256, 4096);
      fps::rows_to_planes<<<blocks, 256, 0, L->stream>>>(db[slot].as<u64>(), m, 4, 1, L->out(), dst, nullptr);
      L->launches++;
      cudaEventRecord(done[slot], L->stream);
      dst += m;
      slot ^= 1;
    }
    std::fclose(fp);
  }
  cudaError_t e = cudaStreamSynchronize(L->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  for (int b = 0; b < 2; ++b) {
    cudaEventDestroy(done[b]);
    hb[b].release();
    db[b].release();
  }
  if (e != cudaSuccess) {
    destroy(L);
    return fail(FPS_ECUDA, std::string("shard upload: ") + cudaGetErrorString(e));
  }
  // The records streamed into 24 B tiles (their word-2 width is unknown up
  // front); re-tile to the 21 B layout when no record needs bits 40.. .
  if (n > 0 && !force_full_layout()) {
    DevBuf wide;
    if ((rc = wide.ensure(4))) { destroy(L); return rc; }
    CUDA_TRY(cudaMemsetAsync(wide.p, 0, 4, L->stream));
    const int blocks = (int)std::min<u64>((n + 255) / 256, (u64)L->sms * 16);
    fps::count_wide_lib<<<blocks, 256, 0, L->stream>>>(L->out(), n, wide.as<u32>());
    u32 nwide = 0;
    CUDA_TRY(cudaMemcpyAsync(&nwide, wide.p, 4, cudaMemcpyDeviceToHost, L->stream));
    CUDA_TRY(cudaStreamSynchronize(L->stream));
    if (nwide == 0) {
      const fps::PlanesOut full = L->out();
      char* old_mem = L->mem;
      const u64 old_alloc = L->n_alloc;
      L->mem = nullptr;
      if ((rc = alloc_planes(L, n, true)) == FPS_OK) {
        fps::retile_kernel<<<blocks, 256, 0, L->stream>>>(full, L->out(), n);
        L->launches += 2;
        e = cudaStreamSynchronize(L->stream);
        cudaFree(old_mem);
        if (e != cudaSuccess) {
          destroy(L);
          return fail(FPS_ECUDA, std::string("re-tiling: ") + cudaGetErrorString(e));
        }
      } else {  // no room for a second copy: keep the 24 B tiles
        cudaGetLastError();
        L->mem = old_mem;
        L->compact = false;
        L->n = n;
        L->n_alloc = old_alloc;
      }
    }
  }
  *out = L;
  return FPS_OK;
}

int fps_open_generated(uint64_t n, uint64_t start, uint64_t seed_key, const uint32_t* thr166,
                       const uint8_t* thr_all166, int device, uint64_t index_base, fps_lib** out) {
  if (!out || !thr166) return fail(FPS_EINVAL, "null argument");
  *out = nullptr;
  if (index_base + n > fps::IDX_MASK) return fail(FPS_EINVAL, "library indices exceed 2^40");
  fps_lib* L = nullptr;
  int rc = new_lib(device, index_base, &L);
  if (rc) return rc;
  DeviceGuard g(device);
  if ((rc = alloc_planes(L, n, true))) { destroy(L); return rc; }  // generated words never use bits 38..
  fps::GenArgs a{};
  a.o = L->out();
  a.n = n;
  a.start = start;
  a.seed_key = seed_key;
  for (int j = 0; j < 166; ++j) {
    a.thr[j] = thr166[j];
    a.thr_hi[j] = thr_all166 ? thr_all166[j] : 0;
  }
  if (n) {
    int blocks = (int)std::min<u64>((n + 255) / 256, (u64)L->sms * 16);
    fps::gen_kernel<<<blocks, 256, 0, L->stream>>>(a);
    L->launches++;
  }
  cudaError_t e = cudaStreamSynchronize(L->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    destroy(L);
    return fail(FPS_ECUDA, std::string("generate: ") + cudaGetErrorString(e));
  }
  *out = L;
  return FPS_OK;
}

int fps_close(fps_lib* lib) {
  if (!lib) return FPS_OK;
  // wait for a call in flight on another thread; the caller guarantees no new
  // call starts on a handle it closes (the Python layer reference-counts)
  { std::lock_guard<std::mutex> lk(lib->mu); }
  destroy(lib);
  return FPS_OK;
}

int fps_info(const fps_lib* lib, uint64_t* n, uint64_t* index_base, int* device) {
  if (int rc = check_lib(lib)) return rc;
  if (n) *n = lib->n;
  if (index_base) *index_base = lib->index_base;
  if (device) *device = lib->device;
  return FPS_OK;
}

int fps_layout(const fps_lib* lib, int* compact, uint64_t* bytes_per_entry) {
  if (int rc = check_lib(lib)) return rc;
  if (compact) *compact = lib->compact ? 1 : 0;
  if (bytes_per_entry) *bytes_per_entry = lib->bytes_per_entry();
  return FPS_OK;
}

int fps_read_entries(fps_lib* lib, uint64_t start, uint64_t count, uint64_t* rows) {
  if (int rc = check_lib(lib)) return rc;
  if (start > lib->n || count > lib->n - start) return fail(FPS_EINVAL, "entry range out of bounds");
  if (count == 0) return FPS_OK;
  if (!rows) return fail(FPS_EINVAL, "rows is null");
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  const u64 chunk = 1 << 22;
  DevBuf d_rows;
  int rc;
  if ((rc = d_rows.ensure((size_t)std::min<u64>(chunk, count) * 24))) return rc;
  for (u64 s0 = 0; s0 < count; s0 += chunk) {
    const u64 m = std::min<u64>(chunk, count - s0);
    int blocks = (int)std::min<u64>((m + 255) / 256, 4096);
    fps::planes_to_rows<<<blocks, 256, 0, lib->stream>>>(lib->out(), start + s0, m, d_rows.as<u64>());
    CUDA_TRY(cudaMemcpyAsync(rows + 3 * s0, d_rows.p, (size_t)m * 24, cudaMemcpyDeviceToHost, lib->stream));
    CUDA_TRY(cudaStreamSynchronize(lib->stream));
  }
  return FPS_OK;
}

int fps_write_entries(fps_lib* lib, const uint64_t* idx, const uint64_t* words, uint64_t m) {
  if (int rc = check_lib(lib)) return rc;
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  for (u64 i = 0; i < m; ++i)
    if (idx[i] >= lib->n) return fail(FPS_EINVAL, "entry index out of range");
  if (m == 0) return FPS_OK;
  int rc;
  DevBuf d_idx, d_rows, wide;
  if ((rc = d_idx.ensure((size_t)m * 8)) || (rc = d_rows.ensure((size_t)m * 24)) || (rc = wide.ensure(4))) return rc;
  CUDA_TRY(cudaMemsetAsync(wide.p, 0, 4, lib->stream));
  CUDA_TRY(cudaMemcpyAsync(d_idx.p, idx, (size_t)m * 8, cudaMemcpyHostToDevice, lib->stream));
  CUDA_TRY(cudaMemcpyAsync(d_rows.p, words, (size_t)m * 24, cudaMemcpyHostToDevice, lib->stream));
  int blocks = (int)std::min<u64>((m + 255) / 256, 4096);
  fps::scatter_rows<<<blocks, 256, 0, lib->stream>>>(d_idx.as<u64>(), d_rows.as<u64>(), m, lib->out(),
                                                     wide.as<u32>());
  lib->launches++;
  u32 nwide = 0;
  CUDA_TRY(cudaMemcpyAsync(&nwide, wide.p, 4, cudaMemcpyDeviceToHost, lib->stream));
  CUDA_TRY(cudaStreamSynchronize(lib->stream));
  // the bit-plane copies are derived from the entries: rebuild on next use
  lib->bs.release();
  lib->bs_state = 0;
  lib->mq4x.release();
  lib->mq4x_state = 0;
  lib->pm.release();
  lib->pm_perm.release();
  lib->pm_meta.release();
  lib->pm_state = 0;
  if (nwide) return fail(FPS_EINVAL, "entry sets bits 40.. of word 2; the library uses the compact layout");
  return FPS_OK;
}

int fps_topk_prepare(fps_lib* lib, uint32_t Q, uint32_t k) {
  if (int rc = check_lib(lib)) return rc;
  if (Q == 0 || k == 0) return fail(FPS_EINVAL, "Q and k must be >= 1");
  if (k > KMAX_FUSED) return FPS_OK;  // the large-k path sizes its scratch per call
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  int rc = topk_dispatch(lib, nullptr, Q, k, nullptr, nullptr, lib->stream, true);
  if (!rc) CUDA_TRY(cudaStreamSynchronize(lib->stream));
  return rc;
}

int fps_topk_async(fps_lib* lib, const uint64_t* d_queries, uint32_t Q, uint32_t k, uint64_t* d_keys,
                   uint32_t* d_cnt, void* stream) {
  if (int rc = check_lib(lib)) return rc;
  if (Q == 0 || k == 0) return fail(FPS_EINVAL, "Q and k must be >= 1");
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  cudaStream_t s = (cudaStream_t)stream;  // used as given (0 = legacy default stream)
  int rc = topk_any(lib, (const u64*)d_queries, Q, k, (u64*)d_keys, d_cnt, s);
  if (rc) reset_state(lib);
  return rc;
}

namespace {

// Host wait for a synchronous call: spin on cudaStreamQuery (a short scan
// finishes in tens of microseconds, and a blocking sync adds wake-up latency).
cudaError_t wait_stream(cudaStream_t s) {
  static const bool block = std::getenv("FPS_BLOCKING_SYNC") != nullptr;
  if (block) return cudaStreamSynchronize(s);
  for (;;) {
    cudaError_t e = cudaStreamQuery(s);
    if (e != cudaErrorNotReady) return e;
  }
}

bool graphs_enabled(const fps_lib* L) {
  static const bool off = [] {
    const char* e = std::getenv("FPS_GRAPHS");
    return (e && std::string(e) == "0") || std::getenv("FPS_DEBUG") != nullptr;
  }();
  return !off && !L->timing;
}

// Replay (capturing on first use) the whole host-API top-k call for (Q, k).
// Returns FPS_OK with results in gr->hout, or an error (the caller falls back).
int topk_graph(fps_lib* L, const uint64_t* queries, u32 Q, u32 k, fps_lib::TopkGraph** out) {
  fps_lib::TopkGraph* gr = nullptr;
  for (auto* x : L->graphs)
    if (x->Q == Q && x->k == k) gr = x;
  int rc;
  if (!gr) {
    if (L->graphs.size() >= 8) {  // bounded cache: drop the oldest
      auto* old = L->graphs.front();
      if (old->exec) cudaGraphExecDestroy(old->exec);
      delete old;
      L->graphs.erase(L->graphs.begin());
    }
    gr = new fps_lib::TopkGraph();
    gr->Q = Q;
    gr->k = k;
    L->graphs.push_back(gr);
    if ((rc = gr->hq.ensure((size_t)Q * 24)) || (rc = gr->hout.ensure((size_t)Q * k * 8 + (size_t)Q * 4)) ||
        (rc = gr->dq.ensure((size_t)Q * 24)) || (rc = gr->dkeys.ensure((size_t)Q * k * 8)) ||
        (rc = gr->dcnt.ensure((size_t)Q * 4)))
      return rc;
  }
  const bool mma_now = mma_wanted(L, Q, k);
  if (!gr->exec || gr->gen != g_alloc_gen.load() || gr->mma != mma_now) {
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    gr->exec = nullptr;
    // every scratch buffer must exist before capture (no allocation inside it)
    if ((rc = topk_dispatch(L, gr->dq.as<u64>(), Q, k, gr->dkeys.as<u64>(), gr->dcnt.as<u32>(), L->stream, true)))
      return rc;
    CUDA_TRY(cudaStreamSynchronize(L->stream));
    const u64 gen = g_alloc_gen.load();
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(L->stream, cudaStreamCaptureModeThreadLocal));
    cudaMemcpyAsync(gr->dq.p, gr->hq.p, (size_t)Q * 24, cudaMemcpyHostToDevice, L->stream);
    rc = topk_dispatch(L, gr->dq.as<u64>(), Q, k, gr->dkeys.as<u64>(), gr->dcnt.as<u32>(), L->stream, false);
    cudaMemcpyAsync(gr->hout.p, gr->dkeys.p, (size_t)Q * k * 8, cudaMemcpyDeviceToHost, L->stream);
    cudaMemcpyAsync(gr->hout.as<char>() + (size_t)Q * k * 8, gr->dcnt.p, (size_t)Q * 4, cudaMemcpyDeviceToHost,
                    L->stream);
    cudaError_t e = cudaStreamEndCapture(L->stream, &graph);
    if (rc || e != cudaSuccess || g_alloc_gen.load() != gen) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      return rc ? rc : fail(FPS_ECUDA, "graph capture failed");
    }
    e = cudaGraphInstantiate(&gr->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      cudaGetLastError();
      gr->exec = nullptr;
      return fail(FPS_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
    gr->gen = gen;
    gr->mma = mma_now;
    gr->kernel = L->last_kernel;
  }
  L->last_kernel = gr->kernel;
  std::memcpy(gr->hq.p, queries, (size_t)Q * 24);
  CUDA_TRY(cudaGraphLaunch(gr->exec, L->stream));
  cudaError_t e = wait_stream(L->stream);
  if (e != cudaSuccess) {
    reset_state(L);
    return fail(FPS_ECUDA, std::string("top-k graph: ") + cudaGetErrorString(e));
  }
  *out = gr;
  return FPS_OK;
}

}  // namespace

int fps_topk(fps_lib* lib, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx, uint16_t* out_dist,
             uint32_t* out_cnt) {
  if (int rc = check_lib(lib)) return rc;
  if (Q == 0) return FPS_OK;
  if (k == 0) return fail(FPS_EINVAL, "n must be >= 1");
  if (!queries || !out_cnt) return fail(FPS_EINVAL, "null argument");
  for (u32 q = 0; q < Q; ++q)
    if (queries[3 * (u64)q + 2] >> 38) return fail(FPS_EPADDING, "padding bits above key 166 must be zero");
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  int rc;
  if (Q == 1 && k <= KMAX_FUSED && !lib->timing) {
    // single query: the query travels as a kernel parameter and the select
    // kernel writes straight into mapped pinned memory -- two launches, no copies
    const size_t need = (size_t)k * 8 + 64 + 64;  // keys, count, completion flag
    if (lib->hmap_bytes < need) {
      if (lib->hmap) cudaFreeHost(lib->hmap);
      lib->hmap = nullptr;
      lib->hmap_bytes = 0;
      if (cudaHostAlloc(&lib->hmap, need, cudaHostAllocMapped) != cudaSuccess ||
          cudaHostGetDevicePointer(&lib->dmap, lib->hmap, 0) != cudaSuccess) {
        cudaGetLastError();
        lib->hmap = nullptr;
      } else {
        std::memset(lib->hmap, 0, need);  // completion flag starts below any sequence number
        lib->done_seq = 0;
        lib->hmap_bytes = need;
      }
    }
    if (lib->hmap) {
      u64* dk = reinterpret_cast<u64*>(lib->dmap);
      u32* dc = reinterpret_cast<u32*>(reinterpret_cast<char*>(lib->dmap) + (size_t)k * 8);
      lib->last_kernel = 1;
      // plane scan: select_kernel posts a sequence number into mapped memory
      // after the results; the host spins on it (no stream query per spin)
      u32* hflag = reinterpret_cast<u32*>(reinterpret_cast<char*>(lib->hmap) + (size_t)k * 8 + 64);
      u32* dflag = reinterpret_cast<u32*>(reinterpret_cast<char*>(lib->dmap) + (size_t)k * 8 + 64);
      const bool pq = pq_wanted(lib);
      const u32 seq = ++lib->done_seq;
      rc = pq ? topk_pq(lib, nullptr, reinterpret_cast<const u64*>(queries), k, dk, dc, lib->stream, false, dflag, seq)
         : lib->compact ? topk_fused<1, 4, true>(lib, nullptr, 1, k, dk, dc, lib->stream, false, 0, reinterpret_cast<const u64*>(queries))
                        : topk_fused<1, 4, false>(lib, nullptr, 1, k, dk, dc, lib->stream, false, 0, reinterpret_cast<const u64*>(queries));
      if (rc) { reset_state(lib); return rc; }
      cudaError_t e = cudaSuccess;
      if (pq) {
        for (u32 spin = 1; *(volatile u32*)hflag != seq; ++spin) {
          if ((spin & 255) == 0) {  // a failed launch never posts: check the stream now and then
            e = cudaStreamQuery(lib->stream);
            if (e == cudaErrorNotReady) { e = cudaSuccess; continue; }
            if (e != cudaSuccess || *(volatile u32*)hflag == seq) break;
            e = cudaErrorUnknown;  // stream idle without the flag
            break;
          }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
      } else {
        e = wait_stream(lib->stream);
      }
      if (e != cudaSuccess) {
        reset_state(lib);
        return fail(FPS_ECUDA, std::string("top-k: ") + cudaGetErrorString(e));
      }
      const u64* hk = reinterpret_cast<const u64*>(lib->hmap);
      const u32* hc = reinterpret_cast<const u32*>(reinterpret_cast<const char*>(lib->hmap) + (size_t)k * 8);
      unpack_topk(hk, hc, 1, k, out_idx, out_dist, out_cnt);
      return FPS_OK;
    }
  }
  if (k <= KMAX_FUSED && graphs_enabled(lib)) {
    fps_lib::TopkGraph* gr = nullptr;
    if (topk_graph(lib, queries, Q, k, &gr) == FPS_OK) {
      const u64* hk = gr->hout.as<u64>();
      const u32* hc = reinterpret_cast<const u32*>(gr->hout.as<char>() + (size_t)Q * k * 8);
      unpack_topk(hk, hc, Q, k, out_idx, out_dist, out_cnt);
      return FPS_OK;
    }
    cudaGetLastError();  // fall through to the stream path
  }
  if ((rc = stage_queries(lib, queries, Q))) return rc;
  if ((rc = lib->keys.ensure((size_t)Q * k * 8)) || (rc = lib->cnt.ensure((size_t)Q * 4))) return rc;
  if (k <= KMAX_FUSED) {
    rc = topk_dispatch(lib, lib->queries.as<u64>(), Q, k, lib->keys.as<u64>(), lib->cnt.as<u32>(), lib->stream, false);
    if (rc) { reset_state(lib); return rc; }
  } else {
    rc = topk_large(lib, lib->queries.as<u64>(), Q, k, lib->keys.as<u64>(), lib->cnt.as<u32>());
    if (rc) return rc;
  }
  size_t kb = (size_t)Q * k * 8;
  if ((rc = lib->h_stage.ensure(kb + (size_t)Q * 4))) return rc;
  u64* hk = lib->h_stage.as<u64>();
  u32* hc = reinterpret_cast<u32*>(lib->h_stage.as<char>() + kb);
  CUDA_TRY(cudaMemcpyAsync(hk, lib->keys.p, kb, cudaMemcpyDeviceToHost, lib->stream));
  CUDA_TRY(cudaMemcpyAsync(hc, lib->cnt.p, (size_t)Q * 4, cudaMemcpyDeviceToHost, lib->stream));
  cudaError_t e = cudaStreamSynchronize(lib->stream);
  if (e != cudaSuccess) {
    reset_state(lib);
    return fail(FPS_ECUDA, std::string("top-k: ") + cudaGetErrorString(e));
  }
  unpack_topk(hk, hc, Q, k, out_idx, out_dist, out_cnt);
  return FPS_OK;
}

// debug (not part of include/fps.h): per-tile timestamps of the fp4 scan
// (scan flag 1 << 20; tools/dbg/mm4_trace.py)
extern "C" int fps_dbg_mm4_trace(uint64_t* out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, fps::g_mm4_trace, sizeof(fps::g_mm4_trace));
}

#ifdef FPS_SCAN_TRACE
// debug builds only (not part of include/fps.h): timeline markers
extern "C" int fps_trace_mark(fps_lib* lib, int slot) {
  fps::mark_kernel<<<1, 1, 0, lib->stream>>>(slot);
  return (int)cudaGetLastError();
}
extern "C" int fps_trace_read(uint64_t* marks, uint64_t* warps) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(marks, fps::g_mark, 8 * sizeof(u64));
  return (int)cudaMemcpyFromSymbol(warps, fps::g_scan_trace, sizeof(fps::g_scan_trace));
}
extern "C" int fps_trace_phases(uint64_t* ph) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(ph, fps::g_pq_phase, sizeof(fps::g_pq_phase));
}
extern "C" int fps_trace_prologue(uint64_t* pro) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(pro, fps::g_pq_pro, sizeof(fps::g_pq_pro));
}
extern "C" int fps_trace_s1(uint64_t* st) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(st, fps::g_pq_s1, sizeof(fps::g_pq_s1));
}
extern "C" int fps_trace_steps(uint64_t* st) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(st, fps::g_pq_steps, sizeof(fps::g_pq_steps));
}
extern "C" int fps_trace_clear() {
  static u64 zeros[16384 * 8];
  cudaDeviceSynchronize();
  cudaMemcpyToSymbol(fps::g_mark, zeros, 8 * sizeof(u64));
  cudaMemcpyToSymbol(fps::g_pq_phase, zeros, sizeof(fps::g_pq_phase));
  cudaMemcpyToSymbol(fps::g_pq_steps, zeros, sizeof(fps::g_pq_steps));
  cudaMemcpyToSymbol(fps::g_pq_s1, zeros, sizeof(fps::g_pq_s1));
  return (int)cudaMemcpyToSymbol(fps::g_scan_trace, zeros, sizeof(fps::g_scan_trace));
}
#endif

int fps_topk_min(fps_lib* lib, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx,
                 uint16_t* out_dist, uint32_t* out_cnt) {
  if (int rc = check_lib(lib)) return rc;
  if (Q == 0) return fail(FPS_EINVAL, "batch_search requires at least one query");
  if (k == 0) return fail(FPS_EINVAL, "n must be >= 1");
  if (!queries || !out_cnt) return fail(FPS_EINVAL, "null argument");
  for (u32 q = 0; q < Q; ++q)
    if (queries[3 * (u64)q + 2] >> 38) return fail(FPS_EPADDING, "padding bits above key 166 must be zero");
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  int rc;
  if ((rc = stage_queries(lib, queries, Q))) return rc;
  if ((rc = lib->keys.ensure((size_t)k * 8)) || (rc = lib->cnt.ensure(4))) return rc;
  if ((rc = topk_min_dev(lib, lib->queries.as<u64>(), Q, k, lib->keys.as<u64>(), lib->cnt.as<u32>(), lib->stream))) {
    reset_state(lib);
    return rc;
  }
  if ((rc = lib->h_stage.ensure((size_t)k * 8 + 4))) return rc;
  u64* hk = lib->h_stage.as<u64>();
  u32* hc = reinterpret_cast<u32*>(lib->h_stage.as<char>() + (size_t)k * 8);
  CUDA_TRY(cudaMemcpyAsync(hk, lib->keys.p, (size_t)k * 8, cudaMemcpyDeviceToHost, lib->stream));
  CUDA_TRY(cudaMemcpyAsync(hc, lib->cnt.p, 4, cudaMemcpyDeviceToHost, lib->stream));
  cudaError_t e = cudaStreamSynchronize(lib->stream);
  if (e != cudaSuccess) {
    reset_state(lib);
    return fail(FPS_ECUDA, std::string("top-k min: ") + cudaGetErrorString(e));
  }
  unpack_topk(hk, hc, 1, k, out_idx, out_dist, out_cnt);
  return FPS_OK;
}

int fps_range_async(fps_lib* lib, const uint64_t* d_queries, uint32_t Q, const uint8_t* d_radius, uint64_t* d_out,
                    uint64_t cap, uint64_t* d_count, void* stream) {
  if (int rc = check_lib(lib)) return rc;
  if (Q == 0) return FPS_OK;
  if (Q > 65535) return fail(FPS_EINVAL, "at most 65535 queries per range call");
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  cudaStream_t s = (cudaStream_t)stream;  // used as given (0 = legacy default stream)
  CUDA_TRY(cudaMemsetAsync(d_count, 0, 8, s));
  fps::ScanArgs a = base_args(lib, (const u64*)d_queries, Q);
  a.radius = d_radius;
  a.out = (u64*)d_out;
  a.out_cnt = (u64*)d_count;
  a.out_cap = cap;
  return plain_dispatch<fps::MODE_RANGE>(lib, a, s);
}

int fps_range(fps_lib* lib, const uint64_t* queries, uint32_t Q, const uint8_t* radius, uint64_t** out_keys,
              uint64_t* n_out) {
  if (int rc = check_lib(lib)) return rc;
  if (!out_keys || !n_out) return fail(FPS_EINVAL, "null output");
  *out_keys = nullptr;
  *n_out = 0;
  if (Q == 0) return FPS_OK;
  if (Q > 65535) return fail(FPS_EINVAL, "at most 65535 queries per range call");
  if (!queries || !radius) return fail(FPS_EINVAL, "null argument");
  for (u32 q = 0; q < Q; ++q)
    if (queries[3 * (u64)q + 2] >> 38) return fail(FPS_EPADDING, "padding bits above key 166 must be zero");
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  int rc;
  if ((rc = stage_queries(lib, queries, Q))) return rc;
  if ((rc = lib->radius.ensure(Q))) return rc;
  CUDA_TRY(cudaMemcpyAsync(lib->radius.p, radius, Q, cudaMemcpyHostToDevice, lib->stream));
  u64 hits = 0;
  if ((rc = range_collect(lib, lib->queries.as<u64>(), Q, lib->radius.as<unsigned char>(), &hits, 0))) return rc;
  if ((rc = sort_keys(lib, lib->rkeys.as<u64>(), hits, lib->stream))) return rc;
  u64* host = (u64*)std::malloc(std::max<u64>(hits, 1) * 8);
  if (!host) return fail(FPS_ENOMEM, "host allocation for range output");
  if (hits) CUDA_TRY(cudaMemcpyAsync(host, lib->rkeys.p, hits * 8, cudaMemcpyDeviceToHost, lib->stream));
  cudaError_t e = cudaStreamSynchronize(lib->stream);
  if (e != cudaSuccess) {
    std::free(host);
    return fail(FPS_ECUDA, std::string("range: ") + cudaGetErrorString(e));
  }
  *out_keys = (uint64_t*)host;
  *n_out = hits;
  return FPS_OK;
}

void fps_free(void* p) { std::free(p); }

int fps_range_begin(fps_lib* lib, const uint64_t* queries, uint32_t Q, const uint8_t* radius, uint64_t* n_out) {
  if (int rc = check_lib(lib)) return rc;
  if (!n_out) return fail(FPS_EINVAL, "null output");
  *n_out = 0;
  if (Q > 65535) return fail(FPS_EINVAL, "at most 65535 queries per range call");
  if (Q && (!queries || !radius)) return fail(FPS_EINVAL, "null argument");
  for (u32 q = 0; q < Q; ++q)
    if (queries[3 * (u64)q + 2] >> 38) return fail(FPS_EPADDING, "padding bits above key 166 must be zero");
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  lib->range_pending = 0;
  if (Q == 0) return FPS_OK;
  int rc;
  if ((rc = stage_queries(lib, queries, Q))) return rc;
  if ((rc = lib->radius.ensure(Q))) return rc;
  CUDA_TRY(cudaMemcpyAsync(lib->radius.p, radius, Q, cudaMemcpyHostToDevice, lib->stream));
  u64 hits = 0;
  if ((rc = range_collect(lib, lib->queries.as<u64>(), Q, lib->radius.as<unsigned char>(), &hits, 0))) return rc;
  if ((rc = sort_keys(lib, lib->rkeys.as<u64>(), hits, lib->stream))) return rc;
  lib->range_pending = hits;
  *n_out = hits;
  return FPS_OK;
}

int fps_range_fetch(fps_lib* lib, uint32_t* out_query, uint64_t* out_index, uint16_t* out_dist, uint64_t n) {
  if (int rc = check_lib(lib)) return rc;
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  if (n != lib->range_pending) return fail(FPS_EINVAL, "fps_range_fetch: n does not match fps_range_begin");
  if (n && (!out_query || !out_index || !out_dist)) return fail(FPS_EINVAL, "null argument");
  const cudaError_t e = fetch_columns(lib->stream, lib->rkeys.as<u64>(), n, lib->h_range, out_query, out_index, out_dist);
  lib->range_pending = 0;
  if (e != cudaSuccess) return fail(FPS_ECUDA, std::string("range fetch: ") + cudaGetErrorString(e));
  return FPS_OK;
}

void fps_range_unpack(const uint64_t* keys, uint64_t n, uint32_t* out_query, uint64_t* out_index,
                      uint16_t* out_dist) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t x = keys[i];
    out_query[i] = (uint32_t)(x >> 48);
    out_index[i] = x & fps::IDX_MASK;
    out_dist[i] = (uint16_t)((x >> fps::IDX_BITS) & 0xffu);
  }
}

int fps_sort_keys(fps_lib* lib, uint64_t* d_keys, uint64_t n, void* stream) {
  if (lib) {
    std::lock_guard<std::mutex> lk(lib->mu);
    DeviceGuard g(lib->device);
    return sort_keys(lib, (u64*)d_keys, n, (cudaStream_t)stream);
  }
  return sort_keys(nullptr, (u64*)d_keys, n, (cudaStream_t)stream);
}

int fps_merge_async(const uint64_t* d_in_keys, const uint32_t* d_in_cnt, uint32_t G, uint32_t Q, uint32_t k,
                    uint64_t* d_out_keys, uint32_t* d_out_cnt, void* stream) {
  if (G == 0 || Q == 0 || k == 0) return fail(FPS_EINVAL, "G, Q and k must be >= 1");
  u64 total = std::max<u64>((u64)G * Q * k, Q);
  int blocks = (int)((total + 255) / 256);
  fps::merge_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const u64*)d_in_keys, d_in_cnt, G, Q, k, (u64*)d_out_keys, d_out_cnt);
  CUDA_TRY(cudaGetLastError());
  return FPS_OK;
}

int fps_merge_packed_async(const void* d_packed, uint64_t row_bytes, uint32_t G, uint32_t Q, uint32_t k,
                           uint64_t* d_out_keys, uint32_t* d_out_cnt, void* stream) {
  if (G == 0 || G > (uint32_t)fps::GROUP_MAX || Q == 0 || k == 0 || !d_packed)
    return fail(FPS_EINVAL, "1 <= G <= 32 blocks, Q, k >= 1 and a buffer are required");
  if (row_bytes < (u64)Q * k * 8 + (u64)Q * 4 || row_bytes % 8)
    return fail(FPS_EINVAL, "row_bytes must hold Q x k keys and Q counts (8-byte aligned)");
  fps::ShardLists lists{};
  for (u32 g = 0; g < G; ++g) {
    const char* row = (const char*)d_packed + (u64)g * row_bytes;
    lists.keys[g] = (const u64*)row;
    lists.cnt[g] = (const u32*)(row + (u64)Q * k * 8);
  }
  const u64 total = (u64)G * Q * k + Q;
  const int blocks = (int)std::min<u64>((total + 255) / 256, 4096);
  fps::merge_lists_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(lists, G, Q, k, (u64*)d_out_keys, d_out_cnt);
  CUDA_TRY(cudaGetLastError());
  return FPS_OK;
}

int fps_merge_runs_async(const uint64_t* const* d_runs, const uint64_t* run_len, uint32_t G, uint64_t* d_out,
                         void* stream) {
  if (G == 0 || G > (uint32_t)fps::GROUP_MAX || !d_runs || !run_len)
    return fail(FPS_EINVAL, "1 <= G <= 32 runs and their lengths are required");
  fps::ShardLists lists{};
  u64 off = 0;
  for (u32 g = 0; g < G; ++g) {
    lists.keys[g] = (const u64*)d_runs[g];
    lists.len[g] = run_len[g];
    lists.off[g] = off;
    off += run_len[g];
  }
  if (off == 0) return FPS_OK;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = (int)std::min<u64>((off + 255) / 256, (u64)sms * 8);
  fps::merge_runs_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(lists, G, (u64*)d_out);
  CUDA_TRY(cudaGetLastError());
  return FPS_OK;
}

int fps_memory(const fps_lib* lib, uint64_t* library_bytes, uint64_t* derived_bytes, uint64_t* scratch_bytes,
               double* derived_build_ms) {
  if (int rc = check_lib(lib)) return rc;
  fps_lib* L = const_cast<fps_lib*>(lib);
  std::lock_guard<std::mutex> lk(L->mu);
  const u64 te = fps::tile_entries(L->compact);
  const u64 lib_b = L->n_alloc / te * fps::tile_bytes(L->compact);
  const u64 der = L->pm.bytes + L->pm_perm.bytes + L->pm_meta.bytes + L->bs.bytes + L->mq4x.bytes;
  u64 scr = 0;
  for (const DevBuf* b : {&L->tg, &L->ghist, &L->cand_cnt, &L->dyn, &L->buf, &L->cand, &L->queries, &L->keys, &L->cnt,
                          &L->radius, &L->rkeys, &L->rcount, &L->sort_tmp, &L->sort_out, &L->seg, &L->bsq, &L->mq,
                          &L->mm_bop, &L->mm_ucol, &L->mm_qpop, &L->mm_tq, &L->mm_qcol, &L->mm_keys, &L->mm_sorted,
                          &L->mm_tmp, &L->mm_priv, &L->mm_ovf, &L->gout})
    scr += b->bytes;
  for (const auto* gr : L->graphs) scr += gr->dq.bytes + gr->dkeys.bytes + gr->dcnt.bytes;
  if (library_bytes) *library_bytes = lib_b;
  if (derived_bytes) *derived_bytes = der;
  if (scratch_bytes) *scratch_bytes = scr;
  if (derived_build_ms) *derived_build_ms = L->derived_ms;
  return FPS_OK;
}

int fps_release_derived(fps_lib* lib) {
  if (int rc = check_lib(lib)) return rc;
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  cudaStreamSynchronize(lib->stream);
  for (auto* gr : lib->graphs) {  // captured graphs may reference the copies
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    delete gr;
  }
  lib->graphs.clear();
  lib->pm.release();
  lib->pm_perm.release();
  lib->pm_meta.release();
  lib->bs.release();
  lib->mq4x.release();
  if (lib->pm_state > 0) lib->pm_state = 0;
  if (lib->bs_state > 0) lib->bs_state = 0;
  if (lib->mq4x_state > 0) lib->mq4x_state = 0;
  return FPS_OK;
}

uint64_t fps_launch_count(const fps_lib* lib) { return lib ? lib->launches.load() : 0; }

int fps_last_kernel(const fps_lib* lib) { return lib ? lib->last_kernel : 0; }
int fps_last_mma_kind(const fps_lib* lib) { return lib ? lib->last_mma_kind : 0; }

int fps_query_hint(fps_lib* lib, const uint64_t* query) {
  if (int rc = check_lib(lib)) return rc;
  std::lock_guard<std::mutex> lk(lib->mu);
  lib->pq_hint_np = query ? pq_positions(reinterpret_cast<const u64*>(query)) : 0u;
  return FPS_OK;
}

int fps_mma_overflowed(fps_lib* lib, int* flag) {
  if (int rc = check_lib(lib)) return rc;
  if (!flag) return FPS_EINVAL;
  std::lock_guard<std::mutex> lk(lib->mu);
  *flag = 0;
  if (!lib->mm_ovf.p) return FPS_OK;
  DeviceGuard g(lib->device);
  u32 v = 0;
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(&v, lib->mm_ovf.p, 4, cudaMemcpyDeviceToHost));
  *flag = v != 0;
  return FPS_OK;
}

int fps_timing(fps_lib* lib, int enable) {
  if (int rc = check_lib(lib)) return rc;
  std::lock_guard<std::mutex> lk(lib->mu);
  lib->timing = enable != 0;
  lib->ev_used = 0;
  lib->ev_groups = 0;
  return FPS_OK;
}

int fps_timing_read(fps_lib* lib, double* total_ms, uint64_t* count) {
  if (int rc = check_lib(lib)) return rc;
  std::lock_guard<std::mutex> lk(lib->mu);
  DeviceGuard g(lib->device);
  double t = 0;
  for (size_t i = 0; i < lib->ev_used; ++i) {
    CUDA_TRY(cudaEventSynchronize(lib->ev_pool[i].second));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, lib->ev_pool[i].first, lib->ev_pool[i].second));
    t += ms;
  }
  if (total_ms) *total_ms = t;
  if (count) *count = lib->ev_groups;
  lib->ev_used = 0;
  lib->ev_groups = 0;
  return FPS_OK;
}

}  // extern "C"

#include "fps_group.cuh"
