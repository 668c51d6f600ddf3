// librdkv host side: error plumbing, FNV-1a (H1), .rdkv header codec and blob
// file I/O (H2).  Byte-for-byte compatible with the reference codec/store
// (codec.py, store.py); parity is pinned by tests/test_codec_native.py against
// the reference's own golden vectors.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/rdkv.h"

namespace rdkv {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

namespace {

constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001B3ull;
constexpr size_t kFixed = 16;  // magic(4) version(2) model_hash(8) doc_count(2)
constexpr size_t kTail = 30;   // token_count(4) layers kv_heads head_dim(2x3) elem_width(1) reserved(3) payload_len(8) checksum(8)

inline uint64_t fnv(const uint8_t* p, size_t n, uint64_t h) {
  // Serial chain: h = (h ^ b) * prime (mod 2^64).  Unrolled by 8 to keep the
  // loads off the critical path; the multiply chain itself is the floor.
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, p + i, 8);
#pragma GCC unroll 8
    for (int b = 0; b < 8; ++b) h = (h ^ ((w >> (8 * b)) & 0xFF)) * kFnvPrime;
  }
  for (; i < n; ++i) h = (h ^ p[i]) * kFnvPrime;
  return h;
}

template <typename T>
inline T load_le(const uint8_t* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));  // x86-64 / aarch64 hosts are little-endian
  return v;
}
template <typename T>
inline void store_le(uint8_t* p, T v) {
  std::memcpy(p, &v, sizeof(T));
}

// Mirrors KvBlobHeader.__post_init__ (codec.py:123-133) after decode_header's
// own checks (codec.py:244-266).
int decode_header_impl(const uint8_t* d, size_t len, rdkv_header* h, uint64_t* ids, size_t ids_cap,
                       size_t* hdr_len) {
  if (len < kFixed) return set_error(RDKV_ERR_TRUNCATED, "buffer too short for header: %zu bytes", len);
  if (std::memcmp(d, "RDKV", 4) != 0) return set_error(RDKV_ERR_BAD_MAGIC, "bad magic");
  const uint16_t version = load_le<uint16_t>(d + 4);
  if (version != 1) return set_error(RDKV_ERR_UNSUPPORTED_VERSION, "unsupported version %u", version);
  const uint64_t model_hash = load_le<uint64_t>(d + 6);
  const uint16_t doc_count = load_le<uint16_t>(d + 14);
  if (doc_count == 0) return set_error(RDKV_ERR_MALFORMED, "doc_count must be >= 1");
  const size_t hl = kFixed + 8 * (size_t)doc_count + kTail;
  if (len < hl) return set_error(RDKV_ERR_TRUNCATED, "buffer too short for %u doc ids", doc_count);
  const uint8_t* t = d + kFixed + 8 * (size_t)doc_count;
  if (t[11] | t[12] | t[13]) return set_error(RDKV_ERR_MALFORMED, "reserved bytes must be zero");
  rdkv_header x{};
  x.version = version;
  x.model_hash = model_hash;
  x.doc_count = doc_count;
  x.token_count = load_le<uint32_t>(t);
  x.layers = load_le<uint16_t>(t + 4);
  x.kv_heads = load_le<uint16_t>(t + 6);
  x.head_dim = load_le<uint16_t>(t + 8);
  x.elem_width = t[10];
  x.payload_len = load_le<uint64_t>(t + 14);
  x.checksum = load_le<uint64_t>(t + 22);
  if (x.token_count < 1) return set_error(RDKV_ERR_MALFORMED, "token_count must be >= 1");
  const unsigned __int128 expect = (unsigned __int128)2 * x.layers * x.kv_heads * x.head_dim *
                                   (unsigned __int128)x.token_count * x.elem_width;
  if (expect != (unsigned __int128)x.payload_len)
    return set_error(RDKV_ERR_MALFORMED, "payload_len %llu does not match dimensions",
                     (unsigned long long)x.payload_len);
  if (ids) {
    const size_t n = doc_count < ids_cap ? doc_count : ids_cap;
    for (size_t i = 0; i < n; ++i) ids[i] = load_le<uint64_t>(d + kFixed + 8 * i);
  }
  if (h) *h = x;
  if (hdr_len) *hdr_len = hl;
  return 0;
}

int check_impl(const uint8_t* d, size_t len, rdkv_header* h, uint64_t* ids, size_t ids_cap, size_t* poff) {
  rdkv_header x;
  size_t hl;
  int rc = decode_header_impl(d, len, &x, ids, ids_cap, &hl);
  if (rc) return rc;
  const unsigned __int128 end = (unsigned __int128)hl + x.payload_len;
  if ((unsigned __int128)len < end)
    return set_error(RDKV_ERR_TRUNCATED, "payload truncated: have %zu of %llu bytes", len - hl,
                     (unsigned long long)x.payload_len);
  if ((unsigned __int128)len > end)
    return set_error(RDKV_ERR_MALFORMED, "%llu trailing bytes after payload",
                     (unsigned long long)(len - (size_t)end));
  if (fnv(d + hl, x.payload_len, kFnvOffset) != x.checksum)
    return set_error(RDKV_ERR_CHECKSUM, "payload checksum mismatch");
  if (h) *h = x;
  if (poff) *poff = hl;
  return 0;
}

int write_all(int fd, const void* p, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  while (n) {
    ssize_t w = ::write(fd, b, n);
    if (w < 0) {
      if (errno == EINTR) continue;
      return -1;
    }
    b += w;
    n -= (size_t)w;
  }
  return 0;
}

int pread_all(int fd, uint8_t* b, size_t n, off_t off) {
  while (n) {
    ssize_t r = ::pread(fd, b, n, off);
    if (r < 0) {
      if (errno == EINTR) continue;
      return -1;
    }
    if (r == 0) return -2;  // file shrank under us
    b += r;
    n -= (size_t)r;
    off += r;
  }
  return 0;
}

// Whole-file read.  Cold multi-MiB blobs are read by several threads at once
// (contiguous 2-MiB-aligned ranges): a single buffered reader keeps one request
// in flight, several keep the NVMe queue busy.
int read_all(int fd, void* p, size_t n, size_t base = 0) {  // file bytes [base, base + n)
  constexpr size_t kPiece = 2u << 20;
  const size_t pieces = n / kPiece;
  const int threads = (int)std::min<size_t>(8, pieces);
  if (threads < 2) return pread_all(fd, static_cast<uint8_t*>(p), n, (off_t)base);
  const size_t per = (pieces + threads - 1) / threads * kPiece;
  std::vector<std::thread> pool;
  std::vector<int> rc(threads, 0);
  for (int t = 0; t < threads; ++t) {
    const size_t a = (size_t)t * per, b = t + 1 == threads ? n : std::min(n, a + per);  // last range takes the tail
    if (a >= b) break;
    pool.emplace_back([&, t, a, b] { rc[t] = pread_all(fd, static_cast<uint8_t*>(p) + a, b - a, (off_t)(base + a)); });
  }
  for (auto& th : pool) th.join();
  for (int r : rc)
    if (r) return r;
  return 0;
}

// O_DIRECT whole-file read into a 4096-aligned `p` (page cache bypassed): the same
// 2-MiB pieces on up to 8 threads; every request is block-aligned (the last one is
// rounded up and comes back short at EOF).  Returns 0, -1 (I/O error: errno), or
// -3 when the file system refuses O_DIRECT (caller falls back to buffered reads).
int io_threads() {
  static const int t = [] {
    const char* e = std::getenv("RDKV_IO_THREADS");  // A/B knob (default 8)
    const int v = e ? std::atoi(e) : 8;
    return v < 1 ? 1 : v > 64 ? 64 : v;
  }();
  return t;
}

int read_all_direct(int fd, void* p, size_t n, size_t base = 0) {  // file bytes [base, base + n)
  constexpr size_t kPiece = 2u << 20, kBlk = 4096;
  const size_t pieces = (n + kPiece - 1) / kPiece;
  const int threads = (int)std::min<size_t>((size_t)io_threads(), std::max<size_t>(1, pieces));
  const size_t per = (pieces + threads - 1) / threads * kPiece;
  std::vector<std::thread> pool;
  std::vector<int> rc(threads, 0);
  for (int t = 0; t < threads; ++t) {
    const size_t a = (size_t)t * per, b = std::min(n, a + per);
    if (a >= b) break;
    pool.emplace_back([&, t, a, b] {
      uint8_t* dst = static_cast<uint8_t*>(p) + a;
      size_t off = a;
      const size_t end = (b + kBlk - 1) / kBlk * kBlk;  // block-rounded request end
      while (off < b) {
        ssize_t r = ::pread(fd, dst, end - off, (off_t)(base + off));
        if (r < 0) {
          if (errno == EINTR) continue;
          rc[t] = errno == EINVAL ? -3 : -1;
          return;
        }
        if (r == 0) {  // EOF before b: the file shrank under us
          rc[t] = -1;
          return;
        }
        dst += r;
        off += (size_t)r;
        if ((size_t)r % kBlk && off < b) {  // a short unaligned read before the end: cannot continue direct
          rc[t] = -3;
          return;
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int r : rc)
    if (r) return r;
  return 0;
}

}  // namespace
}  // namespace rdkv

using namespace rdkv;

extern "C" {

int rdkv_abi_version(void) { return RDKV_ABI_VERSION; }

const char* rdkv_last_error(void) { return g_err; }

uint64_t rdkv_fnv1a64(const void* data, size_t len, uint64_t seed) {
  return fnv(static_cast<const uint8_t*>(data), len, seed);
}

void rdkv_fnv1a64_many(const void* const* bufs, const size_t* lens, size_t n, uint64_t* out, int threads) {
  if (threads <= 1 || n <= 1) {
    for (size_t i = 0; i < n; ++i) out[i] = fnv(static_cast<const uint8_t*>(bufs[i]), lens[i], kFnvOffset);
    return;
  }
  const size_t nt = (size_t)threads < n ? (size_t)threads : n;
  std::vector<std::thread> pool;
  for (size_t t = 0; t < nt; ++t)
    pool.emplace_back([=] {
      for (size_t i = t; i < n; i += nt) out[i] = fnv(static_cast<const uint8_t*>(bufs[i]), lens[i], kFnvOffset);
    });
  for (auto& th : pool) th.join();
}

size_t rdkv_header_size(uint32_t doc_count) { return kFixed + 8 * (size_t)doc_count + kTail; }

int64_t rdkv_header_encode(const rdkv_header* h, const uint64_t* ids, void* out, size_t cap) {
  if (!h || h->doc_count == 0) return set_error(RDKV_ERR_ARG, "doc_ids must be non-empty");
  const size_t n = rdkv_header_size(h->doc_count);
  if (cap < n) return set_error(RDKV_ERR_ARG, "output buffer too small (%zu < %zu)", cap, n);
  uint8_t* d = static_cast<uint8_t*>(out);
  std::memcpy(d, "RDKV", 4);
  store_le<uint16_t>(d + 4, 1);
  store_le<uint64_t>(d + 6, h->model_hash);
  store_le<uint16_t>(d + 14, h->doc_count);
  for (size_t i = 0; i < h->doc_count; ++i) store_le<uint64_t>(d + kFixed + 8 * i, ids[i]);
  uint8_t* t = d + kFixed + 8 * (size_t)h->doc_count;
  store_le<uint32_t>(t, h->token_count);
  store_le<uint16_t>(t + 4, h->layers);
  store_le<uint16_t>(t + 6, h->kv_heads);
  store_le<uint16_t>(t + 8, h->head_dim);
  t[10] = h->elem_width;
  t[11] = t[12] = t[13] = 0;
  store_le<uint64_t>(t + 14, h->payload_len);
  store_le<uint64_t>(t + 22, h->checksum);
  return (int64_t)n;
}

int rdkv_header_decode(const void* data, size_t len, rdkv_header* h, uint64_t* ids, size_t ids_cap,
                       size_t* header_len) {
  return decode_header_impl(static_cast<const uint8_t*>(data), len, h, ids, ids_cap, header_len);
}

int rdkv_blob_check(const void* data, size_t len, rdkv_header* h, uint64_t* ids, size_t ids_cap,
                    size_t* payload_off) {
  return check_impl(static_cast<const uint8_t*>(data), len, h, ids, ids_cap, payload_off);
}

int rdkv_blob_write(const char* tmp_path, const char* final_path, const void* header, size_t header_len,
                    const void* payload, size_t payload_len) {
  int fd = ::open(tmp_path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0) return set_error(RDKV_ERR_IO, "open %s: %s", tmp_path, strerror(errno));
  int bad = write_all(fd, header, header_len) || write_all(fd, payload, payload_len);
  const int err = errno;
  if (::close(fd) != 0 && !bad) bad = 1;
  if (bad || ::rename(tmp_path, final_path) != 0) {
    const int e2 = bad ? err : errno;
    ::unlink(tmp_path);
    return set_error(RDKV_ERR_IO, "write failed for %s: %s", final_path, strerror(e2));
  }
  return 0;
}

int64_t rdkv_file_size(const char* path) {
  struct stat st;
  if (::stat(path, &st) != 0) return set_error(RDKV_ERR_IO, "stat %s: %s", path, strerror(errno));
  return (int64_t)st.st_size;
}

int rdkv_blob_read(const char* path, void* buf, size_t cap, size_t align, int verify, rdkv_header* h,
                   uint64_t* ids, size_t ids_cap, size_t* file_off, size_t* payload_off) {
  if (align & (align - 1)) return set_error(RDKV_ERR_ARG, "align must be a power of two (or 0: O_DIRECT)");
  const bool direct = align == 0;
  int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return set_error(RDKV_ERR_IO, "open %s: %s", path, strerror(errno));
  struct stat st;
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    return set_error(RDKV_ERR_IO, "stat %s: %s", path, strerror(errno));
  }
  const size_t size = (size_t)st.st_size;
  // header length depends on doc_count (bytes 14..16); peek it first
  uint8_t head[kFixed];
  size_t hl = kFixed + kTail + 8;  // placeholder for short files
  if (size >= kFixed) {
    if (::pread(fd, head, kFixed, 0) != (ssize_t)kFixed) {
      ::close(fd);
      return set_error(RDKV_ERR_IO, "read %s: %s", path, strerror(errno));
    }
    hl = kFixed + 8 * (size_t)load_le<uint16_t>(head + 14) + kTail;
  }
  // pad so that the payload lands on an absolute `align` boundary; O_DIRECT (align 0):
  // the file's first byte on a 4096-byte boundary instead (block-aligned DMA targets)
  constexpr size_t kBlk = 4096;
  const uintptr_t b0 = reinterpret_cast<uintptr_t>(buf);
  const size_t pad = direct ? (kBlk - b0 % kBlk) % kBlk : (align - ((b0 + hl) % align)) % align;
  const size_t need = pad + (direct ? (size + kBlk - 1) / kBlk * kBlk : size);
  if (cap < need) {
    ::close(fd);
    return set_error(RDKV_ERR_ARG, "buffer too small for %s (%zu < %zu)", path, cap, need);
  }
  uint8_t* dst = static_cast<uint8_t*>(buf) + pad;
  int r = -3;
  if (direct) {
    const int dfd = ::open(path, O_RDONLY | O_CLOEXEC | O_DIRECT);
    if (dfd >= 0) {
      r = read_all_direct(dfd, dst, size);
      ::close(dfd);
    }
  }
  if (r == -3) r = read_all(fd, dst, size);  // buffered (or O_DIRECT refused by the file system)
  ::close(fd);
  if (r != 0) return set_error(RDKV_ERR_IO, "read %s failed", path);
  size_t poff = 0;
  const int rc = verify ? check_impl(dst, size, h, ids, ids_cap, &poff)
                        : decode_header_impl(dst, size, h, ids, ids_cap, &poff);
  if (rc) return rc;
  if (!verify) {
    rdkv_header x;
    decode_header_impl(dst, size, &x, nullptr, 0, nullptr);
    if (size < poff + x.payload_len) return set_error(RDKV_ERR_TRUNCATED, "payload truncated");
    if (size > poff + x.payload_len) return set_error(RDKV_ERR_MALFORMED, "trailing bytes after payload");
  }
  if (file_off) *file_off = pad;
  if (payload_off) *payload_off = pad + poff;
  return 0;
}

int64_t rdkv_file_read_range(const char* path, void* dst, size_t cap, uint64_t off, size_t len, int direct) {
  constexpr size_t kBlk = 4096;
  if (!dst || len == 0) return set_error(RDKV_ERR_ARG, "read_range: empty request");
  if (direct && ((reinterpret_cast<uintptr_t>(dst) | off) % kBlk))
    return set_error(RDKV_ERR_ARG, "read_range: O_DIRECT needs a 4096-aligned buffer and offset");
  int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return set_error(RDKV_ERR_IO, "open %s: %s", path, strerror(errno));
  struct stat st;
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    return set_error(RDKV_ERR_IO, "stat %s: %s", path, strerror(errno));
  }
  if (off >= (uint64_t)st.st_size) {
    ::close(fd);
    return 0;
  }
  const size_t n = std::min<uint64_t>(len, (uint64_t)st.st_size - off);
  const size_t need = direct ? (n + kBlk - 1) / kBlk * kBlk : n;  // bytes written into dst
  if (cap < need) {
    ::close(fd);
    return set_error(RDKV_ERR_ARG, "read_range: buffer too small (%zu < %zu)", cap, need);
  }
  int r = -3;
  if (direct) {
    const int dfd = ::open(path, O_RDONLY | O_CLOEXEC | O_DIRECT);
    if (dfd >= 0) {
      r = read_all_direct(dfd, dst, n, (size_t)off);
      ::close(dfd);
    }
  }
  if (r == -3) r = read_all(fd, dst, n, (size_t)off);
  ::close(fd);
  if (r != 0) return set_error(RDKV_ERR_IO, "read %s [%llu, +%zu) failed", path, (unsigned long long)off, n);
  return (int64_t)n;
}

int rdkv_drop_page_cache(const char* path) {
  int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return set_error(RDKV_ERR_IO, "open %s: %s", path, strerror(errno));
  ::fdatasync(fd);
  const int rc = ::posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);
  ::close(fd);
  return rc == 0 ? 0 : set_error(RDKV_ERR_IO, "fadvise %s: %s", path, strerror(rc));
}

}  // extern "C"
