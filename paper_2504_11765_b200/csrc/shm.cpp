// Node-local control plane shared by the instances of one node (one process per
// GPU): a POSIX shared-memory segment holding
//
//   * a key table: per KvKey (model_hash, file stem) a single-flight state word
//     (ABSENT -> REQUESTED -> GENERATING(owner) -> READY | FAILED) — the
//     cross-process form of SharedCacheService.get_or_generate's in-flight map
//     (reference service.py:87-127) — and an HBM-residency record (holder rank,
//     pool blocks, token count) with a pin count, so a peer can pull the blocks
//     over NVLink while the holder is barred from evicting them;
//   * bounded MPMC rings (Vyukov sequence-number cells): ring 0 is the central
//     query FIFO every idle instance pulls from (reference sim.py:403-409), ring
//     1 + r is rank r's generation-request queue (owner-partitioned precompute);
//   * a per-query state array (queued / dispatched / done) the queue monitor reads
//     to flag only queries still waiting (prefetch.py:63-72), and counters.
//
// Every word that is shared is a lock-free std::atomic (address-free on x86-64
// and aarch64), so the protocol works across processes without locks or futexes.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <new>
#include <thread>

#include "../../include/rdkv.h"

namespace rdkv {
int set_error(int code, const char* fmt, ...);
}
using rdkv::set_error;

namespace {

constexpr uint64_t kMagic = 0x52444B5653484D31ull;  // "RDKVSHM1"
constexpr uint32_t kVersion = 1;
constexpr uint64_t kTagBusy = 1;

struct alignas(64) Header {
  uint64_t magic;
  uint32_t version;
  int32_t world, table_slots, max_blocks, ring_slots, cell_bytes, n_rings, max_queries, n_counters;
  uint64_t slot_bytes, cell_stride, ring_bytes;
  uint64_t off_table, off_rings, off_qstate, off_counters, total_bytes;
  std::atomic<uint32_t> ready;
};

struct alignas(64) KeySlot {
  std::atomic<uint64_t> tag;     // 0 empty, 1 being claimed, else mix(mh, stem) | 2
  uint64_t mh, stem;
  std::atomic<uint32_t> state;   // RDKV_KEY_*
  std::atomic<int32_t> owner;    // rank generating / generated it
  std::atomic<uint64_t> res;     // [epoch:32][pins:16][holder+1:16]
  int32_t n_tokens, n_blocks;
  // int32_t blocks[max_blocks] follow (slot_bytes stride)
};

struct alignas(64) RingHdr {
  std::atomic<uint64_t> head;
  char pad0[56];
  std::atomic<uint64_t> tail;
  char pad1[56];
};

struct Cell {
  std::atomic<uint64_t> seq;
  uint32_t len;
  uint32_t pad;
  // uint8_t data[cell_bytes]
};

inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

inline uint64_t mix(uint64_t mh, uint64_t stem) {
  uint64_t z = mh ^ (stem * 0x9E3779B97F4A7C15ull) ^ (stem >> 29);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (z ^ (z >> 31)) | 2ull;  // never 0 (empty) or 1 (busy)
}

inline uint64_t res_pack(uint32_t epoch, uint32_t pins, uint32_t holder1) {
  return ((uint64_t)epoch << 32) | ((uint64_t)(pins & 0xFFFF) << 16) | (holder1 & 0xFFFF);
}
inline uint32_t res_epoch(uint64_t w) { return (uint32_t)(w >> 32); }
inline uint32_t res_pins(uint64_t w) { return (uint32_t)((w >> 16) & 0xFFFF); }
inline uint32_t res_holder1(uint64_t w) { return (uint32_t)(w & 0xFFFF); }

}  // namespace

struct rdkv_shm {
  Header* h = nullptr;
  uint8_t* base = nullptr;
  size_t bytes = 0;

  KeySlot* slot(int64_t i) const { return reinterpret_cast<KeySlot*>(base + h->off_table + (uint64_t)i * h->slot_bytes); }
  int32_t* blocks(KeySlot* s) const { return reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(s) + sizeof(KeySlot)); }
  RingHdr* ring(int r) const { return reinterpret_cast<RingHdr*>(base + h->off_rings + (uint64_t)r * h->ring_bytes); }
  Cell* cell(int r, uint64_t i) const {
    return reinterpret_cast<Cell*>(reinterpret_cast<uint8_t*>(ring(r)) + sizeof(RingHdr) + i * h->cell_stride);
  }
  std::atomic<uint8_t>* qstate() const { return reinterpret_cast<std::atomic<uint8_t>*>(base + h->off_qstate); }
  std::atomic<int64_t>* counters() const { return reinterpret_cast<std::atomic<int64_t>*>(base + h->off_counters); }

  // Find (or, with insert, claim) the slot of a key; nullptr if absent / table full.
  KeySlot* find(uint64_t mh, uint64_t stem, bool insert) const {
    const uint64_t tag = mix(mh, stem);
    const uint64_t mask = (uint64_t)h->table_slots - 1;
    for (uint64_t probe = 0; probe <= mask; ++probe) {
      KeySlot* s = slot((tag + probe) & mask);
      uint64_t t = s->tag.load(std::memory_order_acquire);
      if (t == 0) {
        if (!insert) return nullptr;
        uint64_t expect = 0;
        if (s->tag.compare_exchange_strong(expect, kTagBusy, std::memory_order_acq_rel)) {
          s->mh = mh;
          s->stem = stem;
          s->tag.store(tag, std::memory_order_release);
          return s;
        }
        t = expect;
      }
      while (t == kTagBusy) {  // another process is filling this slot's key
        std::this_thread::yield();
        t = s->tag.load(std::memory_order_acquire);
      }
      if (t == tag && s->mh == mh && s->stem == stem) return s;
    }
    return nullptr;
  }
};

extern "C" {

int rdkv_shm_open(const char* name, int create, int world, int table_slots, int max_blocks, int ring_slots,
                  int cell_bytes, int n_rings, int max_queries, int timeout_ms, rdkv_shm** out) {
  if (!name || !out) return set_error(RDKV_ERR_ARG, "shm_open: null argument");
  *out = nullptr;
  int fd = -1;
  size_t total = 0;
  if (create) {
    if (world < 1 || world > 0xFFFE || table_slots < 2 || (table_slots & (table_slots - 1)) || max_blocks < 1 ||
        ring_slots < 2 || (ring_slots & (ring_slots - 1)) || cell_bytes < 8 || n_rings < 1 || max_queries < 1)
      return set_error(RDKV_ERR_ARG, "shm_open: bad geometry");
    Header g{};
    g.world = world;
    g.table_slots = table_slots;
    g.max_blocks = max_blocks;
    g.ring_slots = ring_slots;
    g.cell_bytes = cell_bytes;
    g.n_rings = n_rings;
    g.max_queries = max_queries;
    g.n_counters = 64;
    g.slot_bytes = round_up(sizeof(KeySlot) + 4ull * max_blocks, 64);
    g.cell_stride = round_up(sizeof(Cell) + (uint64_t)cell_bytes, 64);
    g.ring_bytes = round_up(sizeof(RingHdr) + g.cell_stride * ring_slots, 4096);
    g.off_table = round_up(sizeof(Header), 4096);
    g.off_rings = round_up(g.off_table + g.slot_bytes * table_slots, 4096);
    g.off_qstate = g.off_rings + g.ring_bytes * n_rings;
    g.off_counters = round_up(g.off_qstate + (uint64_t)max_queries, 64);
    g.total_bytes = round_up(g.off_counters + 8ull * g.n_counters, 4096);
    total = g.total_bytes;
    shm_unlink(name);  // a stale segment of an earlier run is replaced
    fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) return set_error(RDKV_ERR_IO, "shm_open(%s): %s", name, strerror(errno));
    if (ftruncate(fd, (off_t)total) != 0) {
      int e = errno;
      close(fd);
      shm_unlink(name);
      return set_error(RDKV_ERR_IO, "ftruncate(%s): %s", name, strerror(e));
    }
    void* p = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return set_error(RDKV_ERR_IO, "mmap(%s): %s", name, strerror(errno));
    auto* s = new (std::nothrow) rdkv_shm;
    if (!s) {
      munmap(p, total);
      return set_error(RDKV_ERR_IO, "shm_open: out of memory");
    }
    s->base = static_cast<uint8_t*>(p);
    s->bytes = total;
    s->h = reinterpret_cast<Header*>(p);  // ftruncate zero-filled the segment: every atomic starts at 0
    std::memcpy(reinterpret_cast<void*>(s->h), &g, offsetof(Header, ready));
    for (int r = 0; r < n_rings; ++r)
      for (uint64_t i = 0; i < (uint64_t)ring_slots; ++i) s->cell(r, i)->seq.store(i, std::memory_order_relaxed);
    s->h->magic = kMagic;
    s->h->version = kVersion;
    s->h->ready.store(1, std::memory_order_release);
    *out = s;
    return 0;
  }
  // attach: wait for the creator to publish the segment
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms > 0 ? timeout_ms : 0);
  for (;;) {
    fd = shm_open(name, O_RDWR, 0600);
    if (fd >= 0) {
      struct stat st {};
      if (fstat(fd, &st) == 0 && (size_t)st.st_size >= sizeof(Header)) {
        void* p = mmap(nullptr, sizeof(Header), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        if (p != MAP_FAILED) {
          auto* hh = reinterpret_cast<Header*>(p);
          const bool ok = hh->ready.load(std::memory_order_acquire) == 1 && hh->magic == kMagic &&
                          hh->version == kVersion && (size_t)st.st_size >= hh->total_bytes;
          total = ok ? hh->total_bytes : 0;
          munmap(p, sizeof(Header));
          if (ok) break;
        }
      }
      close(fd);
      fd = -1;
    }
    if (std::chrono::steady_clock::now() >= deadline)
      return set_error(RDKV_ERR_IO, "shm attach(%s): segment not ready", name);
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
  void* p = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return set_error(RDKV_ERR_IO, "mmap(%s): %s", name, strerror(errno));
  auto* s = new (std::nothrow) rdkv_shm;
  if (!s) {
    munmap(p, total);
    return set_error(RDKV_ERR_IO, "shm attach: out of memory");
  }
  s->base = static_cast<uint8_t*>(p);
  s->bytes = total;
  s->h = reinterpret_cast<Header*>(p);
  *out = s;
  return 0;
}

void rdkv_shm_close(rdkv_shm* s) {
  if (!s) return;
  munmap(s->base, s->bytes);
  delete s;
}

int rdkv_shm_unlink(const char* name) {
  if (!name) return set_error(RDKV_ERR_ARG, "shm_unlink: null name");
  if (shm_unlink(name) != 0 && errno != ENOENT) return set_error(RDKV_ERR_IO, "shm_unlink(%s): %s", name, strerror(errno));
  return 0;
}

int rdkv_shm_world(const rdkv_shm* s) { return s ? s->h->world : set_error(RDKV_ERR_ARG, "shm: null"); }

// ---------------------------------------------------------------- single-flight state

int rdkv_shm_key_state(rdkv_shm* s, uint64_t mh, uint64_t stem, int* owner) {
  if (!s) return set_error(RDKV_ERR_ARG, "shm: null");
  KeySlot* k = s->find(mh, stem, false);
  if (owner) *owner = k ? k->owner.load(std::memory_order_acquire) : -1;
  return k ? (int)k->state.load(std::memory_order_acquire) : RDKV_KEY_ABSENT;
}

int rdkv_shm_key_cas(rdkv_shm* s, uint64_t mh, uint64_t stem, int expect, int desired, int owner) {
  if (!s || expect < 0 || desired < 0) return set_error(RDKV_ERR_ARG, "shm key_cas: bad arguments");
  KeySlot* k = s->find(mh, stem, true);
  if (!k) return set_error(RDKV_ERR_IO, "shm key table full (%d slots)", s->h->table_slots);
  uint32_t e = (uint32_t)expect;
  if (!k->state.compare_exchange_strong(e, (uint32_t)desired, std::memory_order_acq_rel)) return 0;
  if (owner >= 0) k->owner.store(owner, std::memory_order_release);
  return 1;
}

// ---------------------------------------------------------------- HBM residency directory

int rdkv_shm_res_publish(rdkv_shm* s, uint64_t mh, uint64_t stem, int rank, const int32_t* blocks, int n_blocks,
                         int n_tokens) {
  if (!s || !blocks || rank < 0 || rank >= s->h->world || n_blocks < 1 || n_blocks > s->h->max_blocks)
    return set_error(RDKV_ERR_ARG, "shm res_publish: bad arguments (n_blocks %d, max %d)", n_blocks, s->h->max_blocks);
  KeySlot* k = s->find(mh, stem, true);
  if (!k) return set_error(RDKV_ERR_IO, "shm key table full");
  uint64_t w = k->res.load(std::memory_order_acquire);
  if (res_holder1(w) != 0) return 0;  // someone holds it already
  // claim with a "publishing" marker (pins = 0xFFFF keeps readers out), fill, then open
  const uint64_t busy = res_pack(res_epoch(w), 0xFFFF, (uint32_t)rank + 1);
  if (!k->res.compare_exchange_strong(w, busy, std::memory_order_acq_rel)) return 0;
  std::memcpy(s->blocks(k), blocks, 4ull * n_blocks);
  k->n_blocks = n_blocks;
  k->n_tokens = n_tokens;
  k->res.store(res_pack(res_epoch(w) + 1, 0, (uint32_t)rank + 1), std::memory_order_release);
  return 1;
}

int rdkv_shm_res_pin(rdkv_shm* s, uint64_t mh, uint64_t stem, int* rank, int32_t* blocks, int cap, int* n_tokens) {
  if (!s) return set_error(RDKV_ERR_ARG, "shm: null");
  KeySlot* k = s->find(mh, stem, false);
  if (!k) return 0;
  uint64_t w = k->res.load(std::memory_order_acquire);
  for (;;) {
    if (res_holder1(w) == 0 || res_pins(w) >= 0xFFFE) return 0;  // absent, being published or retracted
    const uint64_t nw = res_pack(res_epoch(w), res_pins(w) + 1, res_holder1(w));
    if (k->res.compare_exchange_weak(w, nw, std::memory_order_acq_rel)) break;
  }
  const int n = k->n_blocks;
  if (n > cap) {
    k->res.fetch_sub(1ull << 16, std::memory_order_acq_rel);
    return set_error(RDKV_ERR_ARG, "shm res_pin: %d blocks > capacity %d", n, cap);
  }
  if (rank) *rank = (int)res_holder1(w) - 1;
  if (n_tokens) *n_tokens = k->n_tokens;
  if (blocks) std::memcpy(blocks, s->blocks(k), 4ull * n);
  return n;
}

int rdkv_shm_res_unpin(rdkv_shm* s, uint64_t mh, uint64_t stem) {
  if (!s) return set_error(RDKV_ERR_ARG, "shm: null");
  KeySlot* k = s->find(mh, stem, false);
  if (!k) return set_error(RDKV_ERR_ARG, "shm res_unpin: unknown key");
  uint64_t w = k->res.load(std::memory_order_acquire);
  for (;;) {
    if (res_pins(w) == 0 || res_pins(w) == 0xFFFF) return set_error(RDKV_ERR_ARG, "shm res_unpin: not pinned");
    const uint64_t nw = res_pack(res_epoch(w), res_pins(w) - 1, res_holder1(w));
    if (k->res.compare_exchange_weak(w, nw, std::memory_order_acq_rel)) return 0;
  }
}

int rdkv_shm_res_retract(rdkv_shm* s, uint64_t mh, uint64_t stem, int rank) {
  if (!s) return set_error(RDKV_ERR_ARG, "shm: null");
  KeySlot* k = s->find(mh, stem, false);
  if (!k) return 1;  // nothing published
  uint64_t w = k->res.load(std::memory_order_acquire);
  for (;;) {
    if (res_holder1(w) != (uint32_t)rank + 1) return 1;  // not ours: nothing to retract
    if (res_pins(w) != 0) return 0;                       // a peer is reading the blocks: keep them
    const uint64_t nw = res_pack(res_epoch(w) + 1, 0, 0);
    if (k->res.compare_exchange_weak(w, nw, std::memory_order_acq_rel)) return 1;
  }
}

int rdkv_shm_res_holder(rdkv_shm* s, uint64_t mh, uint64_t stem) {
  if (!s) return set_error(RDKV_ERR_ARG, "shm: null");
  KeySlot* k = s->find(mh, stem, false);
  if (!k) return -1;
  const uint64_t w = k->res.load(std::memory_order_acquire);
  return res_holder1(w) == 0 || res_pins(w) == 0xFFFF ? -1 : (int)res_holder1(w) - 1;
}

// ---------------------------------------------------------------- MPMC rings

int rdkv_shm_ring_push(rdkv_shm* s, int r, const void* data, int len) {
  if (!s || r < 0 || r >= s->h->n_rings || len < 0 || len > s->h->cell_bytes || (len && !data))
    return set_error(RDKV_ERR_ARG, "shm ring_push: bad arguments");
  RingHdr* rh = s->ring(r);
  const uint64_t mask = (uint64_t)s->h->ring_slots - 1;
  uint64_t pos = rh->tail.load(std::memory_order_relaxed);
  Cell* c;
  for (;;) {
    c = s->cell(r, pos & mask);
    const uint64_t seq = c->seq.load(std::memory_order_acquire);
    const int64_t dif = (int64_t)seq - (int64_t)pos;
    if (dif == 0) {
      if (rh->tail.compare_exchange_weak(pos, pos + 1, std::memory_order_relaxed)) break;
    } else if (dif < 0) {
      return 0;  // full
    } else {
      pos = rh->tail.load(std::memory_order_relaxed);
    }
  }
  c->len = (uint32_t)len;
  if (len) std::memcpy(reinterpret_cast<uint8_t*>(c) + sizeof(Cell), data, (size_t)len);
  c->seq.store(pos + 1, std::memory_order_release);
  return 1;
}

int rdkv_shm_ring_pop(rdkv_shm* s, int r, void* out, int cap) {
  if (!s || r < 0 || r >= s->h->n_rings || !out || cap < 0) return set_error(RDKV_ERR_ARG, "shm ring_pop: bad arguments");
  RingHdr* rh = s->ring(r);
  const uint64_t mask = (uint64_t)s->h->ring_slots - 1;
  uint64_t pos = rh->head.load(std::memory_order_relaxed);
  Cell* c;
  for (;;) {
    c = s->cell(r, pos & mask);
    const uint64_t seq = c->seq.load(std::memory_order_acquire);
    const int64_t dif = (int64_t)seq - (int64_t)(pos + 1);
    if (dif == 0) {
      if (rh->head.compare_exchange_weak(pos, pos + 1, std::memory_order_relaxed)) break;
    } else if (dif < 0) {
      return 0;  // empty
    } else {
      pos = rh->head.load(std::memory_order_relaxed);
    }
  }
  const int len = (int)c->len;
  const int n = len < cap ? len : cap;
  if (n) std::memcpy(out, reinterpret_cast<uint8_t*>(c) + sizeof(Cell), (size_t)n);
  c->seq.store(pos + mask + 1, std::memory_order_release);
  return len > cap ? set_error(RDKV_ERR_ARG, "shm ring_pop: record of %d bytes > buffer %d", len, cap) : (len ? len : 1);
}

int64_t rdkv_shm_ring_size(rdkv_shm* s, int r) {
  if (!s || r < 0 || r >= s->h->n_rings) return set_error(RDKV_ERR_ARG, "shm ring_size: bad arguments");
  RingHdr* rh = s->ring(r);
  return (int64_t)(rh->tail.load(std::memory_order_acquire) - rh->head.load(std::memory_order_acquire));
}

// ---------------------------------------------------------------- query states, counters

int rdkv_shm_qstate_cas(rdkv_shm* s, int q, int expect, int desired) {
  if (!s || q < 0 || q >= s->h->max_queries) return set_error(RDKV_ERR_ARG, "shm qstate: index %d out of range", q);
  uint8_t e = (uint8_t)expect;
  return s->qstate()[q].compare_exchange_strong(e, (uint8_t)desired, std::memory_order_acq_rel) ? 1 : 0;
}

int rdkv_shm_qstate(rdkv_shm* s, int q) {
  if (!s || q < 0 || q >= s->h->max_queries) return set_error(RDKV_ERR_ARG, "shm qstate: index %d out of range", q);
  return s->qstate()[q].load(std::memory_order_acquire);
}

int64_t rdkv_shm_counter_add(rdkv_shm* s, int i, int64_t delta) {
  if (!s || i < 0 || i >= s->h->n_counters) return set_error(RDKV_ERR_ARG, "shm counter: index %d", i);
  return s->counters()[i].fetch_add(delta, std::memory_order_acq_rel) + delta;
}

}  // extern "C"
