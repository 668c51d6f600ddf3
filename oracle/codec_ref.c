/*
 * codec_ref.c — plain-C restatement of the reference blob codec arithmetic
 * (TEST INFRASTRUCTURE; see oracle/__init__.py).  Independent of librdkv:
 * written from the reference's published algorithm, pinned by
 * tests/test_oracle.py against tests/golden/codec_golden.json which the
 * reference itself produced (tests/golden/make_golden.py).
 *
 *   oracle_fnv1a64          codec.fnv1a64            codec.py:64-69
 *   oracle_splitmix64       codec._splitmix64        codec.py:168-172
 *   oracle_synth_state      synth_blob seed chaining codec.py:206-210
 *   oracle_keystream        codec._keystream         codec.py:175-185
 *   oracle_encode_header    codec.encode header      codec.py:227-239 (+ layout :8-13, 35-36)
 */
#include <stdint.h>
#include <string.h>

#define FNV_OFF 0xCBF29CE484222325ULL
#define FNV_PRIME 0x100000001B3ULL
#define SM_G 0x9E3779B97F4A7C15ULL
#define SM_1 0xBF58476D1CE4E5B9ULL
#define SM_2 0x94D049BB133111EBULL

uint64_t oracle_fnv1a64(const uint8_t* p, uint64_t n, uint64_t h) {
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= FNV_PRIME;
  }
  return h;
}

uint64_t oracle_fnv_offset(void) { return FNV_OFF; }

uint64_t oracle_splitmix64(uint64_t x) {
  x += SM_G;
  x = (x ^ (x >> 30)) * SM_1;
  x = (x ^ (x >> 27)) * SM_2;
  return x ^ (x >> 31);
}

uint64_t oracle_synth_state(uint64_t seed, uint64_t model_hash, const uint64_t* ids, uint64_t n_ids,
                            uint64_t token_count) {
  uint64_t s = oracle_splitmix64(seed ^ model_hash);
  for (uint64_t i = 0; i < n_ids; ++i) s = oracle_splitmix64(s ^ ids[i]);
  return oracle_splitmix64(s ^ token_count);
}

/* word i (1-based) = mix(state + i*golden); little-endian bytes, truncated to n */
void oracle_keystream(uint64_t state, uint8_t* out, uint64_t n) {
  uint64_t words = (n + 7) / 8;
  for (uint64_t i = 1; i <= words; ++i) {
    uint64_t x = state + i * SM_G;
    x = (x ^ (x >> 30)) * SM_1;
    x = (x ^ (x >> 27)) * SM_2;
    x ^= x >> 31;
    for (int b = 0; b < 8; ++b) {
      uint64_t o = (i - 1) * 8 + (uint64_t)b;
      if (o < n) out[o] = (uint8_t)(x >> (8 * b));
    }
  }
}

static void put(uint8_t** p, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) (*p)[i] = (uint8_t)(v >> (8 * i));
  *p += bytes;
}

/* returns header length (16 + 8k + 30) */
uint64_t oracle_encode_header(uint8_t* out, uint64_t model_hash, const uint64_t* ids, uint16_t k,
                              uint32_t token_count, uint16_t layers, uint16_t kv_heads, uint16_t head_dim,
                              uint8_t elem_width, uint64_t payload_len, uint64_t checksum) {
  uint8_t* p = out;
  memcpy(p, "RDKV", 4);
  p += 4;
  put(&p, 1, 2);
  put(&p, model_hash, 8);
  put(&p, k, 2);
  for (uint16_t i = 0; i < k; ++i) put(&p, ids[i], 8);
  put(&p, token_count, 4);
  put(&p, layers, 2);
  put(&p, kv_heads, 2);
  put(&p, head_dim, 2);
  put(&p, elem_width, 1);
  put(&p, 0, 3);
  put(&p, payload_len, 8);
  put(&p, checksum, 8);
  return (uint64_t)(p - out);
}
