/*
 * fps.h — C ABI of libfpsgpu.so, the B200 (sm_100a) fingerprint-scan engine.
 *
 * Drop-in boundary for the reference fpscan search path
 * (/root/reference/pkg/src/fpscan/scan.py). The reference has no FFI: its
 * operator seam is `Kernel = Literal["packed","reference"]` (scan.py:35)
 * dispatched per 65,536-record block in `_scan_shard` (scan.py:180-193). This
 * ABI plugs in one level up, at `search` / `_search_multi` (scan.py:239-303),
 * with the library resident in HBM, because a per-block seam would be PCIe
 * bound. The Python shim (paper_1906_06170_b200/_native.py) binds it with
 * ctypes and maps status codes to the reference exception types.
 *
 * Conventions (all entry points):
 *  - plain pointers and sizes; no torch/CUDA types except `void* stream`
 *    (a cudaStream_t) on the *_async entry points;
 *  - return FPS_OK (0) or an FPS_E* status; fps_last_error() gives a
 *    thread-local message; nothing aborts the process;
 *  - a fingerprint is 3 little-endian u64 words, key j (1-based) at word
 *    (j-1)/64, bit (j-1)%64 (fingerprint.py:3-5). Distance = sum of
 *    popcount(a_w XOR b_w) over the three FULL words, exactly as the
 *    reference XORs the FPS1 record view (scan.py:137-143, :169);
 *  - results are ordered by (distance, index) ascending, index = global
 *    library index (the reference orders by (distance, cid), scan.py:55-56;
 *    identical when cid grows with index, e.g. cid = index + 1, synth.py:37);
 *  - a handle is bound to one CUDA device; calls on one handle are
 *    serialised by an internal mutex, so concurrent callers (the reference's
 *    ThreadPoolExecutor / JobQueue threads, scan.py:265, jobs.py:288) are safe.
 */
#ifndef FPS_H
#define FPS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPS_ABI_VERSION 1

enum fps_status {
  FPS_OK = 0,
  FPS_EINVAL = 1,     /* bad argument: ValueError (scan.py:82-88)            */
  FPS_ENOMEM = 2,     /* device or host allocation failed: MemoryError       */
  FPS_ECUDA = 3,      /* CUDA runtime error: ScanError                       */
  FPS_EPADDING = 4,   /* set bits above key 166: FingerprintError
                         (fingerprint.py:60-61)                              */
  FPS_ECANCELLED = 5, /* cancelled before launch: ScanCancelled (scan.py:190) */
  FPS_ENODEV = 6,     /* no CUDA device: RuntimeError                        */
  FPS_EIO = 7         /* shard file unreadable / bad header / truncated:
                         ScanError("shard <path>: ...") (scan.py:283-284,
                         libstore.py:202-212)                                */
};

/* Input layouts for fps_open. */
enum fps_layout {
  FPS_LAYOUT_ROWS3 = 0,  /* n x 3 u64, row-major (Fingerprint.words per row)    */
  FPS_LAYOUT_FPS1 = 1,   /* n x 32-byte FPS1 records: u64 cid, then the words
                            (libstore.py:5-16, :158-164; the (n,4) u64 view of
                            scan.py:169)                                       */
  FPS_LAYOUT_PLANES = 2  /* three consecutive planes of n u64 (w0[], w1[], w2[]) */
};

typedef struct fps_lib fps_lib;

int fps_version(void);
const char* fps_last_error(void);
int fps_device_count(int* count);

/* Library lifecycle. The handle owns all device memory until fps_close.
 * `words` is a borrowed host pointer valid for the duration of the call.
 * `index_base` is the global index of entry 0 (contiguous multi-GPU shards,
 * libstore.split_sizes semantics, libstore.py:174-179).
 * `check_padding`: nonzero -> FPS_EPADDING if any entry sets bits 166..191
 * (Fingerprint invariant). FPS1 files are scanned as stored (the reference
 * scan does not validate), so pass 0 for them. */
int fps_open(const uint64_t* words, uint64_t n, int layout, int device, uint64_t index_base, int check_padding,
             fps_lib** out);
/* Stream FPS1 shard files (libstore.py:5-16) straight into HBM: each file's
 * 16-byte header is validated (magic "FPS1", version 1, declared count, file
 * size — the checks of read_shard_header / _iter_blocks, libstore.py:202-212,
 * scan.py:166-168) before any device work, then records are read in chunks
 * into pinned buffers, copied asynchronously and transposed on the device
 * while the next chunk is read. Only the global record range [start,
 * start + count) of the concatenated shards is loaded (count = UINT64_MAX:
 * to the end), so each rank of a multi-GPU job streams just its slice.
 * cids (nullable, count entries) receives the records' CIDs. On FPS_EIO,
 * fps_last_error() names the shard path. */
int fps_open_fps1(const char* const* paths, uint32_t n_paths, uint64_t start, uint64_t count, int device,
                  uint64_t* cids, fps_lib** out);
/* Same, from three device planes already on `device` (copied). */
int fps_open_device(const uint64_t* d_w0, const uint64_t* d_w1, const uint64_t* d_w2, uint64_t n, int device,
                    uint64_t index_base, fps_lib** out);
/* Synthetic library generated on the device: key j set iff
 * u32(i, j) < thr[j-1] (or always if thr_all[j-1]); see csrc gen_kernel. */
int fps_open_generated(uint64_t n, uint64_t start, uint64_t seed_key, const uint32_t* thr166,
                       const uint8_t* thr_all166, int device, uint64_t index_base, fps_lib** out);
int fps_close(fps_lib* lib);
int fps_info(const fps_lib* lib, uint64_t* n, uint64_t* index_base, int* device);
/* HBM layout: tiles, each a small structure of arrays (w0[] | w1[] | word 2).
 * compact = 1 (the default whenever no entry sets bits 40.. of word 2, i.e.
 * every valid fingerprint): 256-entry tiles, word 2 as u32 (bits 0..31) + u8
 * (bits 32..39), 21 B per entry. compact = 0 (libraries with stray pad bits,
 * or FPS_LAYOUT=full): 128-entry tiles of three u64 sub-planes, 24 B/entry.
 * Derived copies built on first use are not counted here (fps_memory). */
int fps_layout(const fps_lib* lib, int* compact, uint64_t* bytes_per_entry);
/* Copy entries [start, start + count) back as count x 3 u64 rows (host). */
int fps_read_entries(fps_lib* lib, uint64_t start, uint64_t count, uint64_t* rows);
/* Overwrite entries idx[i] (local indices) with rows words[i] (host, m x 3). */
int fps_write_entries(fps_lib* lib, const uint64_t* idx, const uint64_t* words, uint64_t m);

/* Per-query top-k, host buffers (synchronous). queries: Q x 3. Outputs are
 * Q x k, row q holds out_cnt[q] = min(k, n) valid hits in (distance, index)
 * order; unused slots get index UINT64_MAX, distance 0xFFFF.
 * Replaces search (scan.py:290-303) for each query. k >= 1. */
int fps_topk(fps_lib* lib, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx,
             uint16_t* out_dist, uint32_t* out_cnt);

/* Min-over-queries top-k (the reference batch_search, scan.py:306-318):
 * each entry scores min_q distance; one (distance, index) top-k. */
int fps_topk_min(fps_lib* lib, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx,
                 uint16_t* out_dist, uint32_t* out_cnt);

/* Range search, host buffers: every (q, index, distance) with
 * distance <= radius[q] (radius has Q entries), sorted by (q, distance,
 * index). *out_keys is allocated by the library (free with fps_free); key =
 * (q << 48) | (distance << 40) | index. */
int fps_range(fps_lib* lib, const uint64_t* queries, uint32_t Q, const uint8_t* radius, uint64_t** out_keys,
              uint64_t* n_out);
void fps_free(void* p);
/* Range search in two calls, results straight into caller-owned columns
 * (no library-allocated buffer): fps_range_begin scans, sorts by (q,
 * distance, index) and leaves the n hits on the device; fps_range_fetch
 * copies them through a pinned double buffer and splits them into
 * query / index / distance columns of n entries. Same hits as fps_range. */
int fps_range_begin(fps_lib* lib, const uint64_t* queries, uint32_t Q, const uint8_t* radius, uint64_t* n_out);
int fps_range_fetch(fps_lib* lib, uint32_t* out_query, uint64_t* out_index, uint16_t* out_dist, uint64_t n);
/* Split n range keys into the three result columns (query, index, distance)
 * in one pass on the host -- the reference has no range op; this
 * builds the columns its RangeResult-style result needs without numpy
 * temporaries. Pure host code: callable without a GPU. */
void fps_range_unpack(const uint64_t* keys, uint64_t n, uint32_t* out_query, uint64_t* out_index,
                      uint16_t* out_dist);

/* ---- library builder (host only, no GPU) ---- */
/* 64-bit FNV-1a over n bytes, resumable: replaces libstore.fnv1a_64
 * (libstore.py:93-98). Start with value = 0xcbf29ce484222325. */
uint64_t fps_fnv1a64(const void* data, uint64_t n, uint64_t value);
/* FNV-1a of a file's bytes from `offset` to EOF (validate_manifest's record
 * region checksum, libstore.py:383-390). FPS_EIO if unreadable. */
int fps_fnv1a64_file(const char* path, uint64_t offset, uint64_t* out);
/* libstore.build_shards (libstore.py:243-272): parse `<CID>\t<bits>` lines
 * (parse_library_line, :136-155; parse_bitstring, fingerprint.py:112-134;
 * whitespace-only lines skipped but counted), pack FPS1 records and write
 * shard_count contiguous shards `out_dir/shard-NNN.fps` (split_sizes).
 * Input is either text_path (whole file, universal newlines like Python's
 * text mode) or the buffer text[0, len) cut into n_lines lines at
 * line_offsets[0..n_lines]. out_counts / out_checksums have shard_count
 * slots (record count, FNV-1a of the record region); *out_total = records.
 * A malformed line returns FPS_EINVAL with its 1-based number in *err_line
 * and its bytes at [*err_off, *err_off + *err_len) of the input, and writes
 * no file. threads <= 0: all hardware threads. */
int fps_build_shards(const char* text, uint64_t len, const uint64_t* line_offsets, uint64_t n_lines,
                     const char* text_path, uint32_t shard_count, const char* out_dir, int threads,
                     uint64_t* out_counts, uint64_t* out_checksums, uint64_t* out_total, uint64_t* err_line,
                     uint64_t* err_off, uint64_t* err_len);

/* ---- stream-ordered device API (benchmarks, CUDA graphs, multi-GPU) ---- */
/* Allocate scratch for (Q, k) so that fps_topk_async does not allocate. */
int fps_topk_prepare(fps_lib* lib, uint32_t Q, uint32_t k);
/* d_queries: Q x 3 on the device; out: d_keys Q x k of (distance << 40 |
 * index) keys (UINT64_MAX pads), d_cnt Q. k <= 1024: no host
 * synchronisation (graph-capturable; the tensor-core path decides its
 * overflow fallback on the device). k > 1024: the exact large-k path, which
 * synchronises (not capturable). The first call on a handle may build a
 * derived copy of the library (plane-major / bit-plane) synchronously. */
int fps_topk_async(fps_lib* lib, const uint64_t* d_queries, uint32_t Q, uint32_t k, uint64_t* d_keys,
                   uint32_t* d_cnt, void* stream);
/* Unsorted range hits into d_out (capacity cap), total count (may exceed cap:
 * then retry with a larger buffer) into *d_count (zeroed by the call). */
int fps_range_async(fps_lib* lib, const uint64_t* d_queries, uint32_t Q, const uint8_t* d_radius, uint64_t* d_out,
                    uint64_t cap, uint64_t* d_count, void* stream);
/* Sort n range keys ascending in place (device radix sort); uses scratch of
 * the handle (or a temporary allocation when lib is NULL). */
int fps_sort_keys(fps_lib* lib, uint64_t* d_keys, uint64_t n, void* stream);
/* Rank-0 merge of G per-shard top-k lists (merge_topk, scan.py:225-236):
 * d_in_keys G x Q x k (each row sorted, UINT64_MAX pads), d_in_cnt G x Q. */
int fps_merge_async(const uint64_t* d_in_keys, const uint32_t* d_in_cnt, uint32_t G, uint32_t Q, uint32_t k,
                    uint64_t* d_out_keys, uint32_t* d_out_cnt, void* stream);
/* Rank-0 merge of G <= 32 per-rank top-k blocks gathered into one buffer
 * (the torchrun gather of bench.py / distributed.gather_topk): block g starts
 * at d_packed + g * row_bytes and holds Q x k sorted u64 keys followed by Q
 * u32 counts -- the layout fps_topk_async writes when its key and count
 * pointers are taken from one such block -- so no repacking precedes the
 * merge (merge_topk, scan.py:225-236). */
int fps_merge_packed_async(const void* d_packed, uint64_t row_bytes, uint32_t G, uint32_t Q, uint32_t k,
                           uint64_t* d_out_keys, uint32_t* d_out_cnt, void* stream);
/* Rank-0 merge of G <= 32 sorted runs of unique range keys (one per shard,
 * the torchrun gather of bench.py / distributed.gather_range): run g is
 * d_runs[g][0 .. run_len[g]) on the device, run_len is a host array; the
 * union lands sorted in d_out by a merge by rank (no re-sort). Replaces the
 * reference's in-process union of shard results (merge_topk, scan.py:225-236)
 * for the range output, which the reference does not have. */
int fps_merge_runs_async(const uint64_t* const* d_runs, const uint64_t* run_len, uint32_t G, uint64_t* d_out,
                         void* stream);
/* Kernel family of the last scan on this handle (reporting / tests):
 * 1 single-query HBM scan, 2 multi-query POPC scan, 3 bit-sliced multi-query
 * scan, 4 large-k (histogram + range + sort) path, 5 single-query plane scan
 * (reads only the bit planes the query needs), 6 tensor-core multi-query scan
 * (tcgen05 int8 GEMM with the distance test folded in). */
int fps_last_kernel(const fps_lib* lib);
/* Operand kind of the last tensor-core scan on this handle (reporting / tests):
 * 0 none yet, 1 int8 (kind::i8, tiles expanded in the kernel), 2 block-scaled
 * fp4 expanded in the kernel (kind::mxf4), 3 block-scaled fp4 from the
 * library's fp4 operand copy (the default; FPS_MMA_KIND=i8|fp4|fp4x). */
int fps_last_mma_kind(const fps_lib* lib);
/* Optional hint for the stream-ordered single-query calls (fps_topk_async with
 * Q = 1), whose query lives on the device: the host copy of the query the next
 * calls will scan (3 words), so the plane scan can size its shared-memory ring
 * and warp count to the query's plane list (queries with more than 40 set or
 * clear keys otherwise run at half the warps). NULL forgets the hint. The
 * host-query entry points (fps_topk: scan.py:239-287) need no hint. */
int fps_query_hint(fps_lib* lib, const uint64_t* query);
/* Diagnostic (synchronises the device): 1 if the last tensor-core top-k had a
 * candidate list overflow its capacity, so its exact POPC fallback pass ran
 * (expected only for adversarial ties; the answer is exact either way). */
int fps_mma_overflowed(fps_lib* lib, int* flag);
/* HBM held by the handle: the tiled library, the derived copies built on
 * first use (plane-major copy of the single-query plane scan, bit-plane copy
 * of the multi-query kernels; ~21.75 and ~22.3 B per entry), and per-call
 * scratch; derived_build_ms = host time spent building derived copies. */
int fps_memory(const fps_lib* lib, uint64_t* library_bytes, uint64_t* derived_bytes, uint64_t* scratch_bytes,
               double* derived_build_ms);
/* Free the derived copies (rebuilt on next use) when HBM is needed elsewhere. */
int fps_release_derived(fps_lib* lib);
/* Number of kernels launched by this handle so far (evidence counter). */
uint64_t fps_launch_count(const fps_lib* lib);
/* Scan-kernel timing for roofline reporting: when enabled, every scan-kernel
 * launch is bracketed by CUDA events on its own stream; fps_timing_read
 * synchronises, returns the summed kernel time and launch count since the
 * last read, and resets. */
int fps_timing(fps_lib* lib, int enable);
int fps_timing_read(fps_lib* lib, double* total_ms, uint64_t* count);

/* ---- one library over several GPUs of one process ---- */
/* The reference fans a search out over contiguous, balanced shards inside one
 * process (scan.py:256-287, libstore.split_sizes libstore.py:174-179) and
 * merges per-shard top-k lists with merge_topk (scan.py:225-236). A group
 * binds contiguous shards (each an fps_lib on its own device) into one
 * library: every shard scans concurrently on its own stream, and the root
 * (shard 0's device) gathers and merges. Results are identical to one
 * fps_lib over the whole library. */
typedef struct fps_group fps_group;

enum fps_gather {
  FPS_GATHER_AUTO = 0, /* P2P when every shard device is peer-accessible from
                          the root, else COPY; env FPS_GATHER=p2p|nccl|copy    */
  FPS_GATHER_P2P = 1,  /* the merge kernel reads shard results from peer HBM
                          over NVLink: gather and merge in one kernel          */
  FPS_GATHER_NCCL = 2, /* grouped ncclSend/ncclRecv to the root, then merge
                          (libnccl.so.2 loaded at run time; distinct devices)  */
  FPS_GATHER_COPY = 3  /* cudaMemcpyPeerAsync to the root, then merge          */
};

/* Bind n_shards handles into a group. Shard i must start at global index
 * shards[0].index_base + sum of the earlier shards' sizes (contiguous). On
 * success the group owns the handles (fps_group_close closes them); on
 * failure they stay with the caller. At most 32 shards. */
int fps_group_open(fps_lib* const* shards, uint32_t n_shards, int gather, fps_group** out);
/* Stream FPS1 shard files into n_devices contiguous slices (split_sizes),
 * one per devices[i], all devices loading concurrently (fps_open_fps1 per
 * slice). cids (nullable) receives every record's CID in library order. */
int fps_group_open_fps1(const char* const* paths, uint32_t n_paths, const int* devices, uint32_t n_devices, int gather,
                        uint64_t* cids, fps_group** out);
int fps_group_close(fps_group* g);
int fps_group_info(const fps_group* g, uint64_t* n, uint32_t* n_shards, int* root_device, int* gather);
/* Borrowed handle of shard i (inspection: fps_last_kernel, fps_timing ...). */
int fps_group_shard(const fps_group* g, uint32_t i, fps_lib** shard);
uint64_t fps_group_launch_count(const fps_group* g);
/* Same contracts as fps_topk / fps_topk_min / fps_range_begin+fetch. */
int fps_group_topk(fps_group* g, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx,
                   uint16_t* out_dist, uint32_t* out_cnt);
int fps_group_topk_min(fps_group* g, const uint64_t* queries, uint32_t Q, uint32_t k, uint64_t* out_idx,
                       uint16_t* out_dist, uint32_t* out_cnt);
int fps_group_range_begin(fps_group* g, const uint64_t* queries, uint32_t Q, const uint8_t* radius, uint64_t* n_out);
int fps_group_range_fetch(fps_group* g, uint32_t* out_query, uint64_t* out_index, uint16_t* out_dist, uint64_t n);
/* Stream-ordered: d_queries, d_keys (Q x k) and d_cnt (Q) live on the root
 * device and `stream` is a root-device stream; the shards start after the
 * work already queued on it, and the merged keys are ready in stream order. */
int fps_group_topk_prepare(fps_group* g, uint32_t Q, uint32_t k);
int fps_group_topk_async(fps_group* g, const uint64_t* d_queries, uint32_t Q, uint32_t k, uint64_t* d_keys,
                         uint32_t* d_cnt, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FPS_H */
