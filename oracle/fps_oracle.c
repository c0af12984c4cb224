/*
 * fps_oracle.c — C restatement of the reference scan, TEST INFRASTRUCTURE ONLY.
 *
 * Used by tests/ (full-size parity) and bench.py's CPU baseline; never linked
 * or loaded by the product library. Semantics follow the reference fpscan:
 *   distance   = sum_w popcount(a_w XOR b_w) over three u64 words
 *                (fingerprint.py:151-158, scan.py:137-143 — full 64-bit words,
 *                exactly what the reference XORs from the FPS1 record view);
 *   top-k      = the k smallest (distance, index) pairs (scan.py:55-56,
 *                scan.py:91-126; cid order == index order for cid = index+1,
 *                synth.py:37), one independent search per query;
 *   range      = every (query, index, distance) with distance <= r_q, sorted by
 *                (query, distance, index) — no reference op;
 *   fnv1a_64   = libstore.py:93-98, for writing FPS1 shards + manifest.
 * Threads split the index range contiguously (libstore.split_sizes semantics,
 * libstore.py:174-179) and partial results are merged like merge_topk
 * (scan.py:225-236).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const uint64_t *w0, *w1, *w2;
  int64_t stride; /* in u64 units */
} planes_t;

static inline uint32_t dist_at(const planes_t* p, uint64_t i, const uint64_t* q) {
  int64_t o = (int64_t)i * p->stride;
  return (uint32_t)(__builtin_popcountll(p->w0[o] ^ q[0]) + __builtin_popcountll(p->w1[o] ^ q[1]) +
                    __builtin_popcountll(p->w2[o] ^ q[2]));
}

/* key = (d << 40) | index — index < 2^40 */
#define KEY(d, i) ((((uint64_t)(d)) << 40) | (uint64_t)(i))

/* bounded max-heap of keys */
static void heap_sift_down(uint64_t* h, uint32_t n, uint32_t i) {
  for (;;) {
    uint32_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && h[l] > h[m]) m = l;
    if (r < n && h[r] > h[m]) m = r;
    if (m == i) return;
    uint64_t t = h[i]; h[i] = h[m]; h[m] = t; i = m;
  }
}
static void heap_sift_up(uint64_t* h, uint32_t i) {
  while (i) {
    uint32_t p = (i - 1) / 2;
    if (h[p] >= h[i]) return;
    uint64_t t = h[i]; h[i] = h[p]; h[p] = t; i = p;
  }
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

typedef struct {
  planes_t p;
  uint64_t lo, hi;
  const uint64_t* q;
  uint32_t Q, k;
  uint64_t* heaps; /* Q * k */
  uint32_t* cnt;   /* Q */
} topk_job_t;

#define CHUNK 2048

static void* topk_worker(void* arg) {
  topk_job_t* j = (topk_job_t*)arg;
  for (uint32_t q = 0; q < j->Q; ++q) j->cnt[q] = 0;
  for (uint64_t c0 = j->lo; c0 < j->hi; c0 += CHUNK) {
    uint64_t c1 = c0 + CHUNK < j->hi ? c0 + CHUNK : j->hi;
    for (uint32_t q = 0; q < j->Q; ++q) {
      const uint64_t* qq = j->q + 3 * (uint64_t)q;
      uint64_t* h = j->heaps + (uint64_t)q * j->k;
      uint32_t n = j->cnt[q];
      for (uint64_t i = c0; i < c1; ++i) {
        uint64_t key = KEY(dist_at(&j->p, i, qq), i);
        if (n < j->k) { h[n] = key; heap_sift_up(h, n); ++n; }
        else if (key < h[0]) { h[0] = key; heap_sift_down(h, n, 0); }
      }
      j->cnt[q] = n;
    }
  }
  return NULL;
}

/* Exact per-query top-k. out_idx/out_d are Q*k; out_cnt[q] = min(k, n). */
int orc_topk(const uint64_t* w0, const uint64_t* w1, const uint64_t* w2, int64_t stride, uint64_t n,
             const uint64_t* queries, uint32_t Q, uint32_t k, int threads, uint64_t* out_idx,
             uint16_t* out_d, uint32_t* out_cnt) {
  if (k == 0) return -1;
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > n / CHUNK + 1) threads = (int)(n / CHUNK + 1);
  pthread_t* th = (pthread_t*)calloc(threads, sizeof(pthread_t));
  topk_job_t* jobs = (topk_job_t*)calloc(threads, sizeof(topk_job_t));
  uint64_t* heaps = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)threads * Q * k);
  uint32_t* cnts = (uint32_t*)calloc((size_t)threads * Q, sizeof(uint32_t));
  if (!th || !jobs || !heaps || !cnts) { free(th); free(jobs); free(heaps); free(cnts); return -2; }
  uint64_t base = n / threads, extra = n % threads, off = 0;
  for (int t = 0; t < threads; ++t) {
    uint64_t sz = base + ((uint64_t)t < extra ? 1 : 0);
    jobs[t].p.w0 = w0; jobs[t].p.w1 = w1; jobs[t].p.w2 = w2; jobs[t].p.stride = stride;
    jobs[t].lo = off; jobs[t].hi = off + sz; off += sz;
    jobs[t].q = queries; jobs[t].Q = Q; jobs[t].k = k;
    jobs[t].heaps = heaps + (size_t)t * Q * k; jobs[t].cnt = cnts + (size_t)t * Q;
    pthread_create(&th[t], NULL, topk_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  uint64_t* all = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)threads * k);
  for (uint32_t q = 0; q < Q; ++q) {
    uint32_t m = 0;
    for (int t = 0; t < threads; ++t) {
      memcpy(all + m, heaps + ((size_t)t * Q + q) * k, sizeof(uint64_t) * cnts[(size_t)t * Q + q]);
      m += cnts[(size_t)t * Q + q];
    }
    qsort(all, m, sizeof(uint64_t), cmp_u64);
    uint32_t r = m < k ? m : k;
    for (uint32_t i = 0; i < r; ++i) {
      out_idx[(size_t)q * k + i] = all[i] & ((1ull << 40) - 1);
      out_d[(size_t)q * k + i] = (uint16_t)(all[i] >> 40);
    }
    out_cnt[q] = r;
  }
  free(all); free(th); free(jobs); free(heaps); free(cnts);
  return 0;
}

typedef struct {
  planes_t p;
  uint64_t lo, hi;
  const uint64_t* q;
  uint32_t Q;
  const uint8_t* radius;
  uint64_t* hist; /* Q * 256, for the histogram job */
  uint64_t* keys; /* growable list of (q<<48 | d<<40 | idx) */
  uint64_t n, cap;
} range_job_t;

static void* range_worker(void* arg) {
  range_job_t* j = (range_job_t*)arg;
  for (uint64_t c0 = j->lo; c0 < j->hi; c0 += CHUNK) {
    uint64_t c1 = c0 + CHUNK < j->hi ? c0 + CHUNK : j->hi;
    for (uint32_t q = 0; q < j->Q; ++q) {
      const uint64_t* qq = j->q + 3 * (uint64_t)q;
      uint32_t r = j->radius[q];
      for (uint64_t i = c0; i < c1; ++i) {
        uint32_t d = dist_at(&j->p, i, qq);
        if (d <= r) {
          if (j->n == j->cap) {
            j->cap = j->cap ? 2 * j->cap : 1024;
            j->keys = (uint64_t*)realloc(j->keys, sizeof(uint64_t) * j->cap);
          }
          j->keys[j->n++] = ((uint64_t)q << 48) | KEY(d, i);
        }
      }
    }
  }
  return NULL;
}

/* Range search: returns malloc'd sorted keys (q<<48 | d<<40 | idx) via *out. */
int orc_range(const uint64_t* w0, const uint64_t* w1, const uint64_t* w2, int64_t stride, uint64_t n,
              const uint64_t* queries, uint32_t Q, const uint8_t* radius, int threads, uint64_t** out,
              uint64_t* n_out) {
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > n / CHUNK + 1) threads = (int)(n / CHUNK + 1);
  pthread_t* th = (pthread_t*)calloc(threads, sizeof(pthread_t));
  range_job_t* jobs = (range_job_t*)calloc(threads, sizeof(range_job_t));
  uint64_t base = n / threads, extra = n % threads, off = 0;
  for (int t = 0; t < threads; ++t) {
    uint64_t sz = base + ((uint64_t)t < extra ? 1 : 0);
    jobs[t].p.w0 = w0; jobs[t].p.w1 = w1; jobs[t].p.w2 = w2; jobs[t].p.stride = stride;
    jobs[t].lo = off; jobs[t].hi = off + sz; off += sz;
    jobs[t].q = queries; jobs[t].Q = Q; jobs[t].radius = radius;
    pthread_create(&th[t], NULL, range_worker, &jobs[t]);
  }
  uint64_t total = 0;
  for (int t = 0; t < threads; ++t) { pthread_join(th[t], NULL); total += jobs[t].n; }
  uint64_t* all = (uint64_t*)malloc(sizeof(uint64_t) * (total ? total : 1));
  uint64_t m = 0;
  for (int t = 0; t < threads; ++t) {
    if (jobs[t].n) memcpy(all + m, jobs[t].keys, sizeof(uint64_t) * jobs[t].n);
    m += jobs[t].n;
    free(jobs[t].keys);
  }
  qsort(all, m, sizeof(uint64_t), cmp_u64);
  *out = all;
  *n_out = m;
  free(th); free(jobs);
  return 0;
}

void orc_free(void* p) { free(p); }

/* 64-bit FNV-1a, resumable (libstore.py:93-98). */
uint64_t orc_fnv1a_64(const uint8_t* data, uint64_t len, uint64_t h) {
  for (uint64_t i = 0; i < len; ++i) h = (h ^ data[i]) * 0x100000001B3ull;
  return h;
}

/* Synthetic library generator — the C twin of generate_words (fps_oracle.py)
 * and of the device gen_kernel: entry i, key j (1-based) is set iff
 * u32(i, j) < thr[j-1] (or always when all[j-1]), u32 = half of
 * splitmix64(seed_key + (i*83 + c + 1) * golden), c = (j-1) >> 1. Input
 * preparation for the CPU baselines at paper scale (numpy takes minutes). */
typedef struct {
  uint64_t seed_key, start, lo, hi;
  const uint64_t* thr;
  uint64_t* out;
} gen_arg_t;

static void* gen_worker(void* arg) {
  gen_arg_t* a = (gen_arg_t*)arg;
  for (uint64_t r = a->lo; r < a->hi; ++r) {
    const uint64_t i = a->start + r;
    uint64_t w[3] = {0, 0, 0};
    for (uint64_t c = 0; c < 83; ++c) {
      uint64_t z = a->seed_key + (i * 83 + c + 1) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      const uint64_t j0 = 2 * c, j1 = 2 * c + 1;
      if ((z & 0xFFFFFFFFull) < a->thr[j0]) w[j0 >> 6] |= 1ull << (j0 & 63);
      if ((z >> 32) < a->thr[j1]) w[j1 >> 6] |= 1ull << (j1 & 63);
    }
    a->out[3 * r] = w[0];
    a->out[3 * r + 1] = w[1];
    a->out[3 * r + 2] = w[2];
  }
  return NULL;
}

/* thr: 166 thresholds in [0, 2^32] (2^32 = always set); out: count x 3 u64. */
int orc_generate(uint64_t seed_key, const uint64_t* thr, uint64_t start, uint64_t count, int threads,
                 uint64_t* out) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  gen_arg_t args[256];
  for (int t = 0; t < threads; ++t) {
    args[t].seed_key = seed_key;
    args[t].start = start;
    args[t].lo = count * (uint64_t)t / (uint64_t)threads;
    args[t].hi = count * (uint64_t)(t + 1) / (uint64_t)threads;
    args[t].thr = thr;
    args[t].out = out;
    if (pthread_create(&th[t], NULL, gen_worker, &args[t])) return 1;
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}
