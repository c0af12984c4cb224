// fps_group.cuh — one library over several GPUs of one process (fps_group_*).
// Included at the end of fps_capi.cu (it drives the same per-device paths).
//
// Reference: the reference fans a search out over its shards inside one
// process (scan.py:256-287, a thread pool over contiguous, balanced shards,
// libstore.split_sizes, libstore.py:174-179) and merges the per-shard top-k
// with merge_topk (scan.py:225-236). Here each shard is a whole fps_lib on
// its own device (index_base = the shard's first global index), every shard
// scans concurrently on its own stream, and the root device (shard 0's)
// gathers and merges:
//   * FPS_GATHER_P2P  (default when every shard device is peer-accessible
//     from the root): the merge kernel reads each shard's result block
//     straight from peer HBM over NVLink -- gather and merge are one kernel,
//     no copy;
//   * FPS_GATHER_NCCL: grouped ncclSend / ncclRecv of the result blocks to
//     the root (libnccl loaded at run time; shard devices must be distinct),
//     then the same merge kernel on the gathered copy;
//   * FPS_GATHER_COPY: cudaMemcpyPeerAsync of the blocks, then the merge.
// The top-k of a union is the top-k of the per-shard top-ks under a total
// order, and shards are disjoint, so every mode is exact; range hits are
// per-shard sorted runs merged by rank (no re-sort of the union).
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is opened with dlopen when a group asks for it

namespace {

struct NcclApi {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

std::mutex g_nccl_mu;
NcclApi g_nccl;
int g_nccl_state = 0;  // 0 untried, 1 loaded, -1 unavailable
std::string g_nccl_err;

// libnccl.so.2: the copy already in the process (torch's) when there is one,
// else the system library; FPS_NCCL_LIB names another.
const NcclApi* nccl_api() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl_state) return g_nccl_state > 0 ? &g_nccl : nullptr;
  g_nccl_state = -1;
  const char* names[] = {std::getenv("FPS_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if (n && (h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) {
    const char* d = dlerror();
    g_nccl_err = std::string("cannot load libnccl: ") + (d ? d : "not found");
    return nullptr;
  }
  auto sym = [&](const char* name) { return dlsym(h, name); };
  g_nccl.CommInitAll = (decltype(g_nccl.CommInitAll))sym("ncclCommInitAll");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))sym("ncclCommDestroy");
  g_nccl.Send = (decltype(g_nccl.Send))sym("ncclSend");
  g_nccl.Recv = (decltype(g_nccl.Recv))sym("ncclRecv");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))sym("ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))sym("ncclGroupEnd");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))sym("ncclGetErrorString");
  g_nccl.GetVersion = (decltype(g_nccl.GetVersion))sym("ncclGetVersion");
  if (!g_nccl.CommInitAll || !g_nccl.CommDestroy || !g_nccl.Send || !g_nccl.Recv || !g_nccl.GroupStart ||
      !g_nccl.GroupEnd || !g_nccl.GetErrorString) {
    g_nccl_err = "libnccl lacks ncclSend / ncclRecv (NCCL >= 2.7 needed)";
    return nullptr;
  }
  g_nccl_state = 1;
  return &g_nccl;
}

#define NCCL_TRY(api, expr)                                                                      \
  do {                                                                                           \
    ncclResult_t r_ = (expr);                                                                    \
    if (r_ != ncclSuccess) return fail(FPS_ECUDA, std::string(#expr) + ": " + (api)->GetErrorString(r_)); \
  } while (0)

// libstore.split_sizes (libstore.py:174-179): parts differ by at most one,
// the first n % parts get the extra record.
std::vector<u64> split_sizes(u64 n, u32 parts) {
  std::vector<u64> s(parts, n / parts);
  for (u32 i = 0; i < n % parts; ++i) s[i]++;
  return s;
}

constexpr size_t blk_align(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

struct fps_group {
  std::vector<fps_lib*> shards;  // owned; shard i covers [base[i], base[i] + shards[i]->n)
  u64 n = 0;
  int root = 0;    // device of shard 0: queries arrive, results leave here
  int gather = 0;  // resolved FPS_GATHER_*
  std::mutex mu;
  std::atomic<u64> launches{0};
  std::vector<ncclComm_t> comms;  // NCCL mode: rank i = shard i
  DevBuf gbuf;                    // root: gathered shard blocks (NCCL / copy modes)
  DevBuf okeys, ocnt, rout;       // root: merged top-k, merged range hits
  HostBuf hq, hout, hr[2], hcount;
  u64 range_pending = 0;
  cudaEvent_t ev_in = nullptr;  // root: orders the shards after the caller's stream
  int last_kernel() const { return shards.empty() ? 0 : shards[0]->last_kernel; }
};

namespace {

int group_check(const fps_group* G) {
  if (!G) return fail(FPS_EINVAL, "null group handle");
  return FPS_OK;
}

int check_queries(const uint64_t* q, u32 Q) {
  for (u32 i = 0; i < Q; ++i)
    if (q[3 * (u64)i + 2] >> 38) return fail(FPS_EPADDING, "padding bits above key 166 must be zero");
  return FPS_OK;
}

// Root-side merge of one result block per shard. blk_bytes: the block size
// each shard wrote (keys [Q][k] u64, then counts [Q] u32). `out_*` on the root.
int group_merge(fps_group* G, u32 Q, u32 k, size_t blk_bytes, u64* out_keys, u32* out_cnt, cudaStream_t sr) {
  const u32 ng = (u32)G->shards.size();
  fps::ShardLists lists{};
  const size_t blk = blk_align(blk_bytes);
  if (G->gather == FPS_GATHER_P2P) {
    for (u32 i = 0; i < ng; ++i) {
      CUDA_TRY(cudaStreamWaitEvent(sr, G->shards[i]->ev_done, 0));
      lists.keys[i] = G->shards[i]->gout.as<u64>();
    }
  } else {
    int rc;
    if ((rc = G->gbuf.ensure(blk * ng))) return rc;
    if (G->gather == FPS_GATHER_COPY) {
      for (u32 i = 0; i < ng; ++i) {
        fps_lib* L = G->shards[i];
        CUDA_TRY(cudaStreamWaitEvent(sr, L->ev_done, 0));
        CUDA_TRY(cudaMemcpyPeerAsync(G->gbuf.as<char>() + i * blk, G->root, L->gout.p, L->device, blk_bytes, sr));
      }
    } else {  // NCCL: each shard sends its block on its own stream (after its scan), the root receives
      const NcclApi* api = nccl_api();
      if (!api) return fail(FPS_ECUDA, g_nccl_err);
      CUDA_TRY(cudaStreamWaitEvent(sr, G->shards[0]->ev_done, 0));
      NCCL_TRY(api, api->GroupStart());
      for (u32 i = 0; i < ng; ++i) {
        fps_lib* L = G->shards[i];
        api->Send(L->gout.p, blk_bytes, ncclUint8, 0, G->comms[i], L->stream);
        api->Recv(G->gbuf.as<char>() + i * blk, blk_bytes, ncclUint8, (int)i, G->comms[0], sr);
      }
      NCCL_TRY(api, api->GroupEnd());
    }
    for (u32 i = 0; i < ng; ++i) lists.keys[i] = reinterpret_cast<const u64*>(G->gbuf.as<char>() + i * blk);
  }
  for (u32 i = 0; i < ng; ++i) lists.cnt[i] = reinterpret_cast<const u32*>(reinterpret_cast<const char*>(lists.keys[i]) + (size_t)Q * k * 8);
  const u64 total = (u64)ng * Q * k + Q;
  const int blocks = (int)std::min<u64>((total + 255) / 256, 148ull * 8);
  fps::merge_lists_kernel<<<blocks, 256, 0, sr>>>(lists, ng, Q, k, out_keys, out_cnt);
  G->launches++;
  LAUNCH_CHECK("merge_lists_kernel");
  return FPS_OK;
}

enum { GRP_TOPK = 0, GRP_MIN = 1 };

// Every shard: queries in (from pinned host memory, or peer-copied from the
// root's d_q after the caller's stream), its own top-k into its result block,
// then ev_done. Then the root merges into out_keys / out_cnt on sr.
int group_topk_dev(fps_group* G, int what, const u64* h_q, const u64* d_q, u32 Q, u32 k, u64* out_keys,
                   u32* out_cnt, cudaStream_t sr) {
  int rc;
  const u32 rq = what == GRP_MIN ? 1u : Q;  // result rows per shard
  const size_t blk_bytes = (size_t)rq * k * 8 + (size_t)rq * 4;
  if (!h_q) {
    DeviceGuard g(G->root);
    if (!G->ev_in) CUDA_TRY(cudaEventCreateWithFlags(&G->ev_in, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(G->ev_in, sr));
  }
  for (fps_lib* L : G->shards) {
    DeviceGuard g(L->device);
    if ((rc = L->queries.ensure((size_t)Q * 24)) || (rc = L->gout.ensure(blk_align(blk_bytes)))) return rc;
    if (!L->ev_done) CUDA_TRY(cudaEventCreateWithFlags(&L->ev_done, cudaEventDisableTiming));
    if (h_q) {
      CUDA_TRY(cudaMemcpyAsync(L->queries.p, h_q, (size_t)Q * 24, cudaMemcpyHostToDevice, L->stream));
      // (a single host query: the plane scan sizes its ring to the query's plane list)
      L->pq_hint_np = (Q == 1 && what != GRP_MIN) ? pq_positions(h_q) : 0u;
    } else {
      CUDA_TRY(cudaStreamWaitEvent(L->stream, G->ev_in, 0));
      CUDA_TRY(cudaMemcpyPeerAsync(L->queries.p, L->device, d_q, G->root, (size_t)Q * 24, L->stream));
    }
    u64* bk = L->gout.as<u64>();
    u32* bc = reinterpret_cast<u32*>(L->gout.as<char>() + (size_t)rq * k * 8);
    rc = what == GRP_MIN ? topk_min_dev(L, L->queries.as<u64>(), Q, k, bk, bc, L->stream)
                         : topk_any(L, L->queries.as<u64>(), Q, k, bk, bc, L->stream);
    if (rc) {
      reset_state(L);
      return rc;
    }
    CUDA_TRY(cudaEventRecord(L->ev_done, L->stream));
  }
  DeviceGuard g(G->root);
  return group_merge(G, rq, k, blk_bytes, out_keys, out_cnt, sr);
}

int group_host_topk(fps_group* G, int what, const uint64_t* queries, u32 Q, u32 k, uint64_t* out_idx,
                    uint16_t* out_dist, uint32_t* out_cnt) {
  int rc;
  const u32 rq = what == GRP_MIN ? 1u : Q;
  fps_lib* L0 = G->shards[0];
  DeviceGuard g(G->root);
  if ((rc = G->hq.ensure((size_t)Q * 24)) || (rc = G->okeys.ensure((size_t)rq * k * 8)) ||
      (rc = G->ocnt.ensure((size_t)rq * 4)) || (rc = G->hout.ensure((size_t)rq * k * 8 + (size_t)rq * 4)))
    return rc;
  std::memcpy(G->hq.p, queries, (size_t)Q * 24);
  // the root shard's stream carries the merge and the result copy
  if ((rc = group_topk_dev(G, what, G->hq.as<u64>(), nullptr, Q, k, G->okeys.as<u64>(), G->ocnt.as<u32>(), L0->stream)))
    return rc;
  u64* hk = G->hout.as<u64>();
  u32* hc = reinterpret_cast<u32*>(G->hout.as<char>() + (size_t)rq * k * 8);
  CUDA_TRY(cudaMemcpyAsync(hk, G->okeys.p, (size_t)rq * k * 8, cudaMemcpyDeviceToHost, L0->stream));
  CUDA_TRY(cudaMemcpyAsync(hc, G->ocnt.p, (size_t)rq * 4, cudaMemcpyDeviceToHost, L0->stream));
  const cudaError_t e = cudaStreamSynchronize(L0->stream);
  if (e != cudaSuccess) return fail(FPS_ECUDA, std::string("group top-k: ") + cudaGetErrorString(e));
  unpack_topk(hk, hc, rq, k, out_idx, out_dist, out_cnt);
  return FPS_OK;
}

// Lock the group and every shard (in shard order) for one call.
struct GroupLock {
  std::unique_lock<std::mutex> g;
  std::vector<std::unique_lock<std::mutex>> s;
  explicit GroupLock(fps_group* G) : g(G->mu) {
    for (fps_lib* L : G->shards) s.emplace_back(L->mu);
  }
};

}  // namespace

extern "C" {

int fps_group_open(fps_lib* const* shards, uint32_t n_shards, int gather, fps_group** out) {
  if (!out) return fail(FPS_EINVAL, "out is null");
  *out = nullptr;
  if (!shards || n_shards == 0) return fail(FPS_EINVAL, "a group needs at least one shard");
  if (n_shards > (u32)fps::GROUP_MAX) return fail(FPS_EINVAL, "at most 32 shards per group");
  if (gather < FPS_GATHER_AUTO || gather > FPS_GATHER_COPY) return fail(FPS_EINVAL, "unknown gather mode");
  u64 next = 0;
  for (u32 i = 0; i < n_shards; ++i) {
    if (!shards[i]) return fail(FPS_EINVAL, "null shard handle");
    for (u32 j = 0; j < i; ++j)
      if (shards[j] == shards[i]) return fail(FPS_EINVAL, "a shard handle appears twice");
    if (i == 0) next = shards[0]->index_base;
    if (shards[i]->index_base != next)
      return fail(FPS_EINVAL, "shards must be contiguous: shard " + std::to_string(i) + " starts at index " +
                                  std::to_string(shards[i]->index_base) + ", expected " + std::to_string(next));
    next += shards[i]->n;
  }
  const int root = shards[0]->device;
  // resolve the gather mode
  bool distinct = true, peer_ok = true;
  for (u32 i = 0; i < n_shards; ++i) {
    for (u32 j = 0; j < i; ++j) distinct = distinct && shards[j]->device != shards[i]->device;
    if (shards[i]->device != root) {
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, root, shards[i]->device) != cudaSuccess) cudaGetLastError();
      peer_ok = peer_ok && can;
    }
  }
  if (gather == FPS_GATHER_AUTO) {
    const char* e = std::getenv("FPS_GATHER");
    const std::string m = e ? e : "";
    gather = m == "nccl" ? FPS_GATHER_NCCL : m == "copy" ? FPS_GATHER_COPY : m == "p2p" ? FPS_GATHER_P2P : 0;
    if (!gather) gather = peer_ok ? FPS_GATHER_P2P : FPS_GATHER_COPY;
  }
  if (gather == FPS_GATHER_P2P && !peer_ok) return fail(FPS_EINVAL, "peer access unavailable between shard devices");
  if (gather == FPS_GATHER_NCCL && !distinct)
    return fail(FPS_EINVAL, "NCCL gather needs one shard per device (shards share a device)");
  fps_group* G = new fps_group();
  G->shards.assign(shards, shards + n_shards);
  G->n = next - shards[0]->index_base;
  G->root = root;
  G->gather = gather;
  if (gather == FPS_GATHER_P2P) {
    DeviceGuard g(root);
    for (u32 i = 0; i < n_shards; ++i) {
      if (shards[i]->device == root) continue;
      const cudaError_t e = cudaDeviceEnablePeerAccess(shards[i]->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        delete G;
        return fail(FPS_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  }
  if (gather == FPS_GATHER_NCCL) {
    const NcclApi* api = nccl_api();
    if (!api) {
      delete G;
      return fail(FPS_ECUDA, g_nccl_err);
    }
    std::vector<int> devs(n_shards);
    for (u32 i = 0; i < n_shards; ++i) devs[i] = shards[i]->device;
    G->comms.resize(n_shards);
    const ncclResult_t r = api->CommInitAll(G->comms.data(), (int)n_shards, devs.data());
    if (r != ncclSuccess) {
      G->comms.clear();
      delete G;
      return fail(FPS_ECUDA, std::string("ncclCommInitAll: ") + api->GetErrorString(r));
    }
  }
  *out = G;
  return FPS_OK;
}

int fps_group_open_fps1(const char* const* paths, uint32_t n_paths, const int* devices, uint32_t n_devices, int gather,
                        uint64_t* cids, fps_group** out) {
  if (!out) return fail(FPS_EINVAL, "out is null");
  *out = nullptr;
  if (!devices || n_devices == 0) return fail(FPS_EINVAL, "at least one device");
  if (n_devices > (u32)fps::GROUP_MAX) return fail(FPS_EINVAL, "at most 32 shards per group");
  if (n_paths && !paths) return fail(FPS_EINVAL, "paths is null");
  // record count from the headers (each shard's loader validates them again)
  u64 total = 0;
  for (u32 f = 0; f < n_paths; ++f) {
    const std::string path = paths[f] ? paths[f] : "";
    FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) return fail(FPS_EIO, "shard " + path + ": " + std::strerror(errno));
    unsigned char h[16];
    const size_t got = std::fread(h, 1, 16, fp);
    std::fclose(fp);
    if (got < 16) return fail(FPS_EIO, "shard " + path + ": header is " + std::to_string(got) + " bytes, expected 16");
    u64 c = 0;
    for (int i = 0; i < 8; ++i) c |= (u64)h[8 + i] << (8 * i);
    total += c;
  }
  const std::vector<u64> sizes = split_sizes(total, n_devices);
  std::vector<fps_lib*> libs(n_devices, nullptr);
  std::vector<int> rcs(n_devices, FPS_OK);
  std::vector<std::string> errs(n_devices);
  std::vector<std::thread> th;
  u64 start = 0;
  // every device streams its own record slice concurrently
  for (u32 i = 0; i < n_devices; ++i) {
    th.emplace_back([&, i, start] {
      rcs[i] = fps_open_fps1(paths, n_paths, start, sizes[i], devices[i], cids ? cids + start : nullptr, &libs[i]);
      if (rcs[i]) errs[i] = g_err;
    });
    start += sizes[i];
  }
  for (auto& t : th) t.join();
  for (u32 i = 0; i < n_devices; ++i) {
    if (rcs[i]) {
      for (fps_lib* L : libs) fps_close(L);
      return fail(rcs[i], errs[i]);
    }
  }
  const int rc = fps_group_open(libs.data(), n_devices, gather, out);
  if (rc) {
    const std::string msg = g_err;
    for (fps_lib* L : libs) fps_close(L);
    return fail(rc, msg);
  }
  return FPS_OK;
}

int fps_group_close(fps_group* G) {
  if (!G) return FPS_OK;
  { std::lock_guard<std::mutex> lk(G->mu); }
  if (!G->comms.empty()) {
    if (const NcclApi* api = nccl_api())
      for (ncclComm_t c : G->comms) api->CommDestroy(c);
  }
  {
    DeviceGuard g(G->root);
    for (fps_lib* L : G->shards) {
      DeviceGuard gs(L->device);
      cudaStreamSynchronize(L->stream);
    }
    if (G->ev_in) cudaEventDestroy(G->ev_in);
    G->gbuf.release();
    G->okeys.release();
    G->ocnt.release();
    G->rout.release();
    G->hq.release();
    G->hout.release();
    G->hr[0].release();
    G->hr[1].release();
    G->hcount.release();
  }
  for (fps_lib* L : G->shards) fps_close(L);
  G->shards.clear();
  delete G;
  return FPS_OK;
}

int fps_group_info(const fps_group* G, uint64_t* n, uint32_t* n_shards, int* root_device, int* gather) {
  if (int rc = group_check(G)) return rc;
  if (n) *n = G->n;
  if (n_shards) *n_shards = (uint32_t)G->shards.size();
  if (root_device) *root_device = G->root;
  if (gather) *gather = G->gather;
  return FPS_OK;
}

int fps_group_shard(const fps_group* G, uint32_t i, fps_lib** shard) {
  if (int rc = group_check(G)) return rc;
  if (!shard || i >= G->shards.size()) return fail(FPS_EINVAL, "shard index out of range");
  *shard = G->shards[i];
  return FPS_OK;
}

uint64_t fps_group_launch_count(const fps_group* G) {
  if (!G) return 0;
  u64 s = G->launches.load();
  for (const fps_lib* L : G->shards) s += L->launches.load();
  return s;
}

int fps_group_topk(fps_group* G, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx,
                   uint16_t* out_dist, uint32_t* out_cnt) {
  if (int rc = group_check(G)) return rc;
  if (Q == 0) return FPS_OK;
  if (k == 0) return fail(FPS_EINVAL, "n must be >= 1");
  if (!queries || !out_cnt) return fail(FPS_EINVAL, "null argument");
  if (int rc = check_queries(queries, Q)) return rc;
  GroupLock lk(G);
  return group_host_topk(G, GRP_TOPK, queries, Q, k, out_idx, out_dist, out_cnt);
}

int fps_group_topk_min(fps_group* G, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx,
                       uint16_t* out_dist, uint32_t* out_cnt) {
  if (int rc = group_check(G)) return rc;
  if (Q == 0) return fail(FPS_EINVAL, "batch_search requires at least one query");
  if (k == 0) return fail(FPS_EINVAL, "n must be >= 1");
  if (!queries || !out_cnt) return fail(FPS_EINVAL, "null argument");
  if (int rc = check_queries(queries, Q)) return rc;
  GroupLock lk(G);
  return group_host_topk(G, GRP_MIN, queries, Q, k, out_idx, out_dist, out_cnt);
}

int fps_group_topk_prepare(fps_group* G, uint32_t Q, uint32_t k) {
  if (int rc = group_check(G)) return rc;
  for (fps_lib* L : G->shards) {
    if (int rc = fps_topk_prepare(L, Q, k)) return rc;
    std::lock_guard<std::mutex> lk(L->mu);
    DeviceGuard g(L->device);
    int rc;
    if ((rc = L->queries.ensure((size_t)Q * 24)) || (rc = L->gout.ensure(blk_align((size_t)Q * k * 12)))) return rc;
    if (!L->ev_done) CUDA_TRY(cudaEventCreateWithFlags(&L->ev_done, cudaEventDisableTiming));
  }
  std::lock_guard<std::mutex> lk(G->mu);
  DeviceGuard g(G->root);
  if (G->gather != FPS_GATHER_P2P)
    if (int rc = G->gbuf.ensure(blk_align((size_t)Q * k * 8 + (size_t)Q * 4) * G->shards.size())) return rc;
  return FPS_OK;
}

int fps_group_topk_async(fps_group* G, const uint64_t* d_queries, uint32_t Q, uint32_t k, uint64_t* d_keys,
                         uint32_t* d_cnt, void* stream) {
  if (int rc = group_check(G)) return rc;
  if (Q == 0 || k == 0) return fail(FPS_EINVAL, "Q and k must be >= 1");
  GroupLock lk(G);
  return group_topk_dev(G, GRP_TOPK, nullptr, (const u64*)d_queries, Q, k, (u64*)d_keys, d_cnt, (cudaStream_t)stream);
}

int fps_group_range_begin(fps_group* G, const uint64_t* queries, uint32_t Q, const uint8_t* radius, uint64_t* n_out) {
  if (int rc = group_check(G)) return rc;
  if (!n_out) return fail(FPS_EINVAL, "null output");
  *n_out = 0;
  if (Q > 65535) return fail(FPS_EINVAL, "at most 65535 queries per range call");
  if (Q && (!queries || !radius)) return fail(FPS_EINVAL, "null argument");
  if (int rc = check_queries(queries, Q)) return rc;
  GroupLock lk(G);
  G->range_pending = 0;
  if (Q == 0) return FPS_OK;
  int rc;
  const u32 ng = (u32)G->shards.size();
  {
    DeviceGuard g(G->root);
    if ((rc = G->hq.ensure((size_t)Q * 24 + Q)) || (rc = G->hcount.ensure(ng * 8 + 8))) return rc;
  }
  std::memcpy(G->hq.p, queries, (size_t)Q * 24);
  std::memcpy(G->hq.as<char>() + (size_t)Q * 24, radius, Q);
  u64* hcnt = G->hcount.as<u64>();
  std::vector<u64> caps(ng);
  // 1. every shard: queries in, range scan into its hit buffer, count out
  for (u32 i = 0; i < ng; ++i) {
    fps_lib* L = G->shards[i];
    DeviceGuard g(L->device);
    if ((rc = L->queries.ensure((size_t)Q * 24)) || (rc = L->radius.ensure(Q)) || (rc = L->rcount.ensure(8)) ||
        (rc = L->rkeys.ensure(std::max<size_t>(L->rkeys.bytes, (size_t)8 << 20))))
      return rc;
    if (!L->ev_done) CUDA_TRY(cudaEventCreateWithFlags(&L->ev_done, cudaEventDisableTiming));
    CUDA_TRY(cudaMemcpyAsync(L->queries.p, G->hq.p, (size_t)Q * 24, cudaMemcpyHostToDevice, L->stream));
    CUDA_TRY(cudaMemcpyAsync(L->radius.p, G->hq.as<char>() + (size_t)Q * 24, Q, cudaMemcpyHostToDevice, L->stream));
    CUDA_TRY(cudaMemsetAsync(L->rcount.p, 0, 8, L->stream));
    caps[i] = L->rkeys.bytes / 8;
    fps::ScanArgs a = base_args(L, L->queries.as<u64>(), Q);
    a.radius = L->radius.as<unsigned char>();
    a.out = L->rkeys.as<u64>();
    a.out_cnt = L->rcount.as<u64>();
    a.out_cap = caps[i];
    if ((rc = plain_dispatch<fps::MODE_RANGE>(L, a, L->stream))) return rc;
    CUDA_TRY(cudaMemcpyAsync(hcnt + i, L->rcount.p, 8, cudaMemcpyDeviceToHost, L->stream));
    CUDA_TRY(cudaEventRecord(L->ev_done, L->stream));
  }
  // 2. counts; a shard whose hits overflowed its buffer rescans with room; sort each run
  std::vector<u64> cnt(ng);
  u64 total = 0;
  for (u32 i = 0; i < ng; ++i) {
    fps_lib* L = G->shards[i];
    DeviceGuard g(L->device);
    CUDA_TRY(cudaEventSynchronize(L->ev_done));
    cnt[i] = hcnt[i];
    if (cnt[i] > caps[i] &&
        (rc = range_collect(L, L->queries.as<u64>(), Q, L->radius.as<unsigned char>(), &cnt[i], cnt[i] + cnt[i] / 8 + 1024)))
      return rc;
    if ((rc = sort_keys(L, L->rkeys.as<u64>(), cnt[i], L->stream))) return rc;
    CUDA_TRY(cudaEventRecord(L->ev_done, L->stream));
    total += cnt[i];
  }
  // 3. root: gather the sorted runs and merge them by rank
  DeviceGuard g(G->root);
  fps_lib* L0 = G->shards[0];
  cudaStream_t sr = L0->stream;
  if ((rc = G->rout.ensure(std::max<u64>(total, 1) * 8))) return rc;
  fps::ShardLists lists{};
  u64 off = 0;
  if (G->gather != FPS_GATHER_P2P && (rc = G->gbuf.ensure(std::max<u64>(total, 1) * 8))) return rc;
  const NcclApi* api = G->gather == FPS_GATHER_NCCL ? nccl_api() : nullptr;
  if (G->gather == FPS_GATHER_NCCL) {
    if (!api) return fail(FPS_ECUDA, g_nccl_err);
    CUDA_TRY(cudaStreamWaitEvent(sr, L0->ev_done, 0));
    NCCL_TRY(api, api->GroupStart());
  }
  for (u32 i = 0; i < ng; ++i) {
    fps_lib* L = G->shards[i];
    lists.len[i] = cnt[i];
    lists.off[i] = off;
    if (G->gather == FPS_GATHER_P2P) {
      CUDA_TRY(cudaStreamWaitEvent(sr, L->ev_done, 0));
      lists.keys[i] = L->rkeys.as<u64>();
    } else {
      u64* dst = G->gbuf.as<u64>() + off;
      lists.keys[i] = dst;
      if (cnt[i] == 0) {
      } else if (G->gather == FPS_GATHER_COPY) {
        CUDA_TRY(cudaStreamWaitEvent(sr, L->ev_done, 0));
        CUDA_TRY(cudaMemcpyPeerAsync(dst, G->root, L->rkeys.p, L->device, cnt[i] * 8, sr));
      } else {
        api->Send(L->rkeys.p, cnt[i] * 8, ncclUint8, 0, G->comms[i], L->stream);
        api->Recv(dst, cnt[i] * 8, ncclUint8, (int)i, G->comms[0], sr);
      }
    }
    off += cnt[i];
  }
  if (G->gather == FPS_GATHER_NCCL) NCCL_TRY(api, api->GroupEnd());
  if (total) {
    const int blocks = (int)std::min<u64>((total + 255) / 256, (u64)L0->sms * 8);
    fps::merge_runs_kernel<<<blocks, 256, 0, sr>>>(lists, ng, G->rout.as<u64>());
    G->launches++;
    LAUNCH_CHECK("merge_runs_kernel");
  }
  const cudaError_t e = cudaStreamSynchronize(sr);
  if (e != cudaSuccess) return fail(FPS_ECUDA, std::string("group range: ") + cudaGetErrorString(e));
  G->range_pending = total;
  *n_out = total;
  return FPS_OK;
}

int fps_group_range_fetch(fps_group* G, uint32_t* out_query, uint64_t* out_index, uint16_t* out_dist, uint64_t n) {
  if (int rc = group_check(G)) return rc;
  std::lock_guard<std::mutex> lk(G->mu);
  if (n != G->range_pending) return fail(FPS_EINVAL, "fps_group_range_fetch: n does not match fps_group_range_begin");
  if (n && (!out_query || !out_index || !out_dist)) return fail(FPS_EINVAL, "null argument");
  DeviceGuard g(G->root);
  const cudaError_t e = fetch_columns(G->shards[0]->stream, G->rout.as<u64>(), n, G->hr, out_query, out_index, out_dist);
  G->range_pending = 0;
  if (e != cudaSuccess) return fail(FPS_ECUDA, std::string("group range fetch: ") + cudaGetErrorString(e));
  return FPS_OK;
}

}  // extern "C"
