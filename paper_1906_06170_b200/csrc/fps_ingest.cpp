// Native library builder: text lines -> FPS1 records -> shard files, plus the
// FNV-1a checksum -- SURVEY §8(f) rank 4. Host code (no GPU), multi-threaded.
//
// Reference behaviour restated here (/root/reference/pkg/src/fpscan):
//   * fnv1a_64 (libstore.py:93-98): h = (h ^ byte) * 0x100000001b3 mod 2^64,
//     offset basis 0xcbf29ce484222325, resumable.
//   * parse_library_line (libstore.py:136-155) + parse_bitstring
//     (fingerprint.py:112-134): `<CID><TAB><bits>`, trailing "\r\n" chars
//     stripped; CID = ASCII decimal digits in 1..2^64-1; bits = 166 '0'/'1'
//     chars (char i -> key i+1) or 167 with the first dropped.
//   * build_shards (libstore.py:243-272): whitespace-only lines skipped (but
//     counted for line numbers), records packed as u64 CID | 21 key bytes (key j
//     at byte (j-1)/8, bit (j-1)%8) | 3 zero bytes (libstore.py:158-164), split
//     contiguously (split_sizes, :174-179) into shard-NNN.fps files with a
//     16-byte header (:182-183), the record region FNV-1a checksummed.
//   * Text files are read like Python's text mode does (cli.py:69): universal
//     newlines, i.e. "\n", "\r\n" and a lone "\r" all end a line.
// A line the native parser rejects is reported by number and byte range; the
// Python layer re-parses just that line to raise the reference's exact
// exception (error path only).
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/fps.h"

void fps_set_last_error(const std::string& msg);  // fps_capi.cu

namespace {

constexpr uint64_t FNV_OFFSET = 0xcbf29ce484222325ull;
constexpr uint64_t FNV_PRIME = 0x100000001b3ull;
constexpr int NUM_KEYS = 166;
constexpr size_t REC = 32;


uint64_t fnv(const unsigned char* p, uint64_t n, uint64_t h) {
  for (uint64_t i = 0; i < n; ++i) h = (h ^ p[i]) * FNV_PRIME;
  return h;
}

// Python str.isspace() for one code point (the ASCII set plus the Unicode
// White_Space / bidi whitespace code points str.strip() removes).
bool py_space(uint32_t c) {
  if (c == 0x20 || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f)) return true;
  switch (c) {
    case 0x85: case 0xa0: case 0x1680: case 0x2028: case 0x2029: case 0x202f: case 0x205f: case 0x3000:
      return true;
    default:
      return c >= 0x2000 && c <= 0x200a;
  }
}

// 1 if [p, q) is empty or only whitespace code points (valid UTF-8 assumed for
// bytes >= 0x80; malformed sequences count as non-space).
bool blank(const unsigned char* p, const unsigned char* q) {
  while (p < q) {
    uint32_t c = *p;
    int n = 1;
    if (c >= 0x80) {
      if ((c & 0xe0) == 0xc0) { n = 2; c &= 0x1f; }
      else if ((c & 0xf0) == 0xe0) { n = 3; c &= 0x0f; }
      else if ((c & 0xf8) == 0xf0) { n = 4; c &= 0x07; }
      else return false;
      if (q - p < n) return false;
      for (int i = 1; i < n; ++i) {
        if ((p[i] & 0xc0) != 0x80) return false;
        c = (c << 6) | (p[i] & 0x3f);
      }
    }
    if (!py_space(c)) return false;
    p += n;
  }
  return true;
}

// Parse one line (terminator already removed, trailing '\r'/'\n' stripped).
// Returns 1 = record written, 0 = blank line, -1 = malformed.
int parse_line(const unsigned char* p, const unsigned char* q, unsigned char* rec) {
  while (q > p && (q[-1] == '\n' || q[-1] == '\r')) --q;  // line.rstrip("\r\n")
  if (blank(p, q)) return 0;
  const unsigned char* tab = static_cast<const unsigned char*>(std::memchr(p, '\t', (size_t)(q - p)));
  if (!tab || tab == p) return -1;
  uint64_t cid = 0;
  for (const unsigned char* c = p; c < tab; ++c) {
    if (*c < '0' || *c > '9') return -1;
    const uint64_t d = *c - '0';
    if (cid > (UINT64_MAX - d) / 10) return -1;  // > 2^64 - 1
    cid = cid * 10 + d;
  }
  if (cid == 0) return -1;
  const unsigned char* b = tab + 1;
  size_t len = (size_t)(q - b);
  if (len != NUM_KEYS && len != NUM_KEYS + 1) return -1;
  for (size_t i = 0; i < len; ++i)
    if (b[i] != '0' && b[i] != '1') return -1;
  if (len == NUM_KEYS + 1) ++b;  // the 167-char form drops its first char
  std::memset(rec, 0, REC);
  for (int i = 0; i < 8; ++i) rec[i] = (unsigned char)(cid >> (8 * i));
  unsigned char* fp = rec + 8;
  for (int i = 0; i < NUM_KEYS; ++i) fp[i >> 3] |= (unsigned char)((b[i] - '0') << (i & 7));
  return 1;
}

struct ChunkOut {
  std::vector<unsigned char> recs;
  uint64_t lines = 0;
  uint64_t err_line = 0;  // 1-based within the chunk, 0 = none
  uint64_t err_off = 0, err_len = 0;
};

// Split [text, text+len) into lines. Universal newlines when offs == nullptr,
// else the caller's line boundaries (line i = [offs[i], offs[i+1])).
void parse_chunk(const unsigned char* text, uint64_t lo, uint64_t hi, ChunkOut* out) {
  unsigned char rec[REC];
  uint64_t i = lo;
  while (i < hi) {
    uint64_t j = i;
    while (j < hi && text[j] != '\n' && text[j] != '\r') ++j;
    uint64_t next = j;
    if (j < hi) next = (text[j] == '\r' && j + 1 < hi && text[j + 1] == '\n') ? j + 2 : j + 1;
    ++out->lines;
    const int r = parse_line(text + i, text + j, rec);
    if (r < 0) {
      out->err_line = out->lines;
      out->err_off = i;
      out->err_len = j - i;
      return;
    }
    if (r > 0) out->recs.insert(out->recs.end(), rec, rec + REC);
    i = next;
  }
}

void parse_offsets(const unsigned char* text, const uint64_t* offs, uint64_t l0, uint64_t l1, ChunkOut* out) {
  unsigned char rec[REC];
  for (uint64_t l = l0; l < l1; ++l) {
    ++out->lines;
    const int r = parse_line(text + offs[l], text + offs[l + 1], rec);
    if (r < 0) {
      out->err_line = out->lines;
      out->err_off = offs[l];
      out->err_len = offs[l + 1] - offs[l];
      return;
    }
    if (r > 0) out->recs.insert(out->recs.end(), rec, rec + REC);
  }
}

int nthreads(int t) {
  if (t > 0) return t;
  const unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h, 64u));
}

// Parallel parse; on success *recs holds the FPS1 record region.
int parse_all(const unsigned char* text, uint64_t len, const uint64_t* offs, uint64_t n_lines, int threads,
              std::vector<unsigned char>* recs, uint64_t* lines_seen, uint64_t* err_line, uint64_t* err_off,
              uint64_t* err_len) {
  const int T = nthreads(threads);
  std::vector<ChunkOut> outs(T);
  std::vector<std::thread> pool;
  if (offs) {
    for (int t = 0; t < T; ++t) {
      const uint64_t l0 = n_lines * t / T, l1 = n_lines * (t + 1) / T;
      pool.emplace_back(parse_offsets, text, offs, l0, l1, &outs[t]);
    }
  } else {
    // chunk boundaries just after a line terminator ("\r\n" kept together)
    std::vector<uint64_t> cut(T + 1, len);
    cut[0] = 0;
    for (int t = 1; t < T; ++t) {
      uint64_t c = std::max(cut[t - 1], len * t / T);
      while (c < len && text[c] != '\n' && text[c] != '\r') ++c;
      if (c < len) c = (text[c] == '\r' && c + 1 < len && text[c + 1] == '\n') ? c + 2 : c + 1;
      cut[t] = c;
    }
    for (int t = 0; t < T; ++t) pool.emplace_back(parse_chunk, text, cut[t], cut[t + 1], &outs[t]);
  }
  for (auto& th : pool) th.join();
  uint64_t base = 0, total = 0;
  for (int t = 0; t < T; ++t) {
    if (outs[t].err_line) {
      *err_line = base + outs[t].err_line;
      *err_off = outs[t].err_off;
      *err_len = outs[t].err_len;
      *lines_seen = base + outs[t].lines;
      return FPS_EINVAL;
    }
    base += outs[t].lines;
    total += outs[t].recs.size();
  }
  *lines_seen = base;
  recs->resize(total);
  uint64_t at = 0;
  for (auto& o : outs) {
    if (!o.recs.empty()) std::memcpy(recs->data() + at, o.recs.data(), o.recs.size());
    at += o.recs.size();
  }
  return FPS_OK;
}

std::string shard_name(uint32_t i) {
  char b[32];
  std::snprintf(b, sizeof b, "shard-%03u.fps", i);
  return b;
}

// mkdir -p (the reference creates the output directory only after every line
// parsed, libstore.py:256).
bool mkdir_p(const std::string& dir) {
  std::string cur;
  size_t i = 0;
  while (i <= dir.size()) {
    const size_t j = dir.find('/', i);
    cur = dir.substr(0, j == std::string::npos ? dir.size() : j);
    if (!cur.empty() && ::mkdir(cur.c_str(), 0777) != 0 && errno != EEXIST) return false;
    if (j == std::string::npos) break;
    i = j + 1;
  }
  struct stat st;
  return ::stat(dir.c_str(), &st) == 0 && S_ISDIR(st.st_mode);
}

// Write shard_count contiguous shards (split_sizes) of the record region in
// parallel; checksums[i] = FNV-1a of shard i's record region.
int write_shards(const unsigned char* recs, uint64_t n, uint32_t shard_count, const char* out_dir,
                 uint64_t* counts, uint64_t* checksums) {
  if (shard_count < 1) {
    fps_set_last_error("shard_count must be >= 1");
    return FPS_EINVAL;
  }
  if (!mkdir_p(out_dir)) {
    fps_set_last_error(std::string("creating ") + out_dir + ": " + std::strerror(errno));
    return FPS_EIO;
  }
  std::vector<uint64_t> off(shard_count + 1, 0);
  const uint64_t base = n / shard_count, extra = n % shard_count;
  for (uint32_t i = 0; i < shard_count; ++i) {
    counts[i] = base + (i < extra ? 1 : 0);
    off[i + 1] = off[i] + counts[i];
  }
  std::vector<int> rc(shard_count, FPS_OK);
  std::vector<std::string> why(shard_count);
  auto work = [&](uint32_t i) {
    const std::string path = std::string(out_dir) + "/" + shard_name(i);
    const unsigned char* region = recs + off[i] * REC;
    const uint64_t bytes = counts[i] * REC;
    checksums[i] = fnv(region, bytes, FNV_OFFSET);
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) {
      rc[i] = FPS_EIO;
      why[i] = "writing " + path + ": " + std::strerror(errno);
      return;
    }
    unsigned char hdr[16] = {'F', 'P', 'S', '1', 1, 0, 0, 0};
    for (int b = 0; b < 8; ++b) hdr[8 + b] = (unsigned char)(counts[i] >> (8 * b));
    bool ok = std::fwrite(hdr, 1, 16, f) == 16;
    if (ok && bytes) ok = std::fwrite(region, 1, bytes, f) == bytes;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) {
      rc[i] = FPS_EIO;
      why[i] = "writing " + path + ": " + std::strerror(errno);
    }
  };
  const int T = std::min<int>(nthreads(0), (int)shard_count);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t]() {
      for (uint32_t i = t; i < shard_count; i += T) work(i);
    });
  for (auto& th : pool) th.join();
  for (uint32_t i = 0; i < shard_count; ++i)
    if (rc[i] != FPS_OK) {
      fps_set_last_error(why[i]);
      return rc[i];
    }
  return FPS_OK;
}

}  // namespace

extern "C" {

uint64_t fps_fnv1a64(const void* data, uint64_t n, uint64_t value) {
  return fnv(static_cast<const unsigned char*>(data), n, value);
}

int fps_fnv1a64_file(const char* path, uint64_t offset, uint64_t* out) {
  if (!path || !out) return FPS_EINVAL;
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    fps_set_last_error(std::string("reading ") + path + ": " + std::strerror(errno));
    return FPS_EIO;
  }
  if (offset && std::fseek(f, (long)offset, SEEK_SET) != 0) {
    std::fclose(f);
    fps_set_last_error(std::string("seeking ") + path);
    return FPS_EIO;
  }
  std::vector<unsigned char> buf(1 << 22);
  uint64_t h = FNV_OFFSET;
  size_t got;
  while ((got = std::fread(buf.data(), 1, buf.size(), f)) > 0) h = fnv(buf.data(), got, h);
  const bool err = std::ferror(f);
  std::fclose(f);
  if (err) {
    fps_set_last_error(std::string("reading ") + path);
    return FPS_EIO;
  }
  *out = h;
  return FPS_OK;
}

int fps_build_shards(const char* text, uint64_t len, const uint64_t* line_offsets, uint64_t n_lines,
                     const char* text_path, uint32_t shard_count, const char* out_dir, int threads,
                     uint64_t* out_counts, uint64_t* out_checksums, uint64_t* out_total, uint64_t* err_line,
                     uint64_t* err_off, uint64_t* err_len) {
  if (!out_dir || !out_counts || !out_checksums || !out_total || !err_line || !err_off || !err_len) return FPS_EINVAL;
  *err_line = *err_off = *err_len = *out_total = 0;
  if (shard_count < 1) {
    fps_set_last_error("shard_count must be >= 1");
    return FPS_EINVAL;
  }
  const unsigned char* src = reinterpret_cast<const unsigned char*>(text);
  void* map = nullptr;
  size_t map_len = 0;
  if (text_path) {  // whole text file, universal newlines
    const int fd = ::open(text_path, O_RDONLY);
    if (fd < 0) {
      fps_set_last_error(std::string("reading ") + text_path + ": " + std::strerror(errno));
      return FPS_EIO;
    }
    struct stat st;
    if (::fstat(fd, &st) != 0) {
      ::close(fd);
      fps_set_last_error(std::string("reading ") + text_path + ": " + std::strerror(errno));
      return FPS_EIO;
    }
    map_len = (size_t)st.st_size;
    if (map_len) {
      map = ::mmap(nullptr, map_len, PROT_READ, MAP_PRIVATE, fd, 0);
      if (map == MAP_FAILED) {
        ::close(fd);
        fps_set_last_error(std::string("mapping ") + text_path + ": " + std::strerror(errno));
        return FPS_EIO;
      }
      ::madvise(map, map_len, MADV_SEQUENTIAL);
    }
    ::close(fd);
    src = static_cast<const unsigned char*>(map);
    len = map_len;
    line_offsets = nullptr;
  }
  std::vector<unsigned char> recs;
  uint64_t seen = 0;
  int rc = parse_all(src, len, line_offsets, n_lines, threads, &recs, &seen, err_line, err_off, err_len);
  if (map) ::munmap(map, map_len);
  if (rc != FPS_OK) {
    fps_set_last_error("line " + std::to_string(*err_line) + ": malformed library line");
    return rc;
  }
  *out_total = recs.size() / REC;
  return write_shards(recs.data(), *out_total, shard_count, out_dir, out_counts, out_checksums);
}

}  // extern "C"
