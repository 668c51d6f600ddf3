/*
 * rdkv.h — C ABI of librdkv, the B200-native Shared RAG-DCache hot path.
 *
 * The reference (`ragdcache`, /root/reference/pkg/src/ragdcache) is a pure-Python
 * package; its "FFI" for this path is the set of in-process Python calls listed
 * beside each entry point below.  The Python package `paper_2504_11765_b200`
 * binds these symbols with ctypes (GIL released during every call) and keeps the
 * reference's Python interfaces on top; INTEGRATION.md shows the binding a
 * maintainer would add to the reference itself.
 *
 * Conventions
 *   - Every status-returning function returns int32: 0 = ok, < 0 = error whose
 *     class maps 1:1 onto the reference exception hierarchy (see RDKV_ERR_*).
 *     rdkv_last_error() returns a thread-local message for the last failure.
 *   - No allocation on hot calls: device / pinned buffers are owned by the caller
 *     (PyTorch) and passed as plain pointers; `stream` is a cudaStream_t.
 *   - GPU calls are asynchronous on `stream` and reentrant per stream.
 */
#ifndef RDKV_H
#define RDKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RDKV_ABI_VERSION 1

#if defined(__GNUC__)
#define RDKV_API __attribute__((visibility("default")))
#else
#define RDKV_API
#endif

/* ----------------------------------------------------------------- status */
#define RDKV_OK 0
#define RDKV_ERR_BAD_MAGIC (-1)          /* codec.BadMagicError          codec.py:44  */
#define RDKV_ERR_UNSUPPORTED_VERSION (-2) /* codec.UnsupportedVersionError codec.py:48 */
#define RDKV_ERR_TRUNCATED (-3)          /* codec.TruncatedError         codec.py:52  */
#define RDKV_ERR_CHECKSUM (-4)           /* codec.ChecksumMismatchError  codec.py:56  */
#define RDKV_ERR_MALFORMED (-5)          /* codec.MalformedHeaderError   codec.py:60  */
#define RDKV_ERR_IO (-6)                 /* OSError on the store path    store.py:219, 268 */
#define RDKV_ERR_ARG (-7)                /* ValueError                                */
#define RDKV_ERR_CUDA (-8)               /* device failure (no reference analogue)    */

RDKV_API int rdkv_abi_version(void);
RDKV_API const char* rdkv_last_error(void);

/* ------------------------------------------------------- L0: blob codec (H1) */

/* 64-bit FNV-1a over `len` bytes starting from `seed` (pass 0xCBF29CE484222325
 * for the standard offset).  Replaces codec.fnv1a64 (codec.py:64-69). */
RDKV_API uint64_t rdkv_fnv1a64(const void* data, size_t len, uint64_t seed);

/* FNV-1a of n independent buffers on up to `threads` host threads (one serial
 * chain per buffer — the checksum itself cannot be split).  Used to hash the
 * k prefix blobs of one combination concurrently (prefetch.py:146-152). */
RDKV_API void rdkv_fnv1a64_many(const void* const* bufs, const size_t* lens, size_t n, uint64_t* out,
                       int threads);

/* FNV-1a of `len` bytes of DEVICE memory, computed in parallel on the GPU and
 * bit-exact with rdkv_fnv1a64: the low byte of the state is a 256-state
 * automaton (run from every start byte per 16-KiB chunk, then stitched), and
 * given it the 64-bit update is affine, so chunks compose.  The result lands in
 * *out_dev (device uint64) asynchronously on `stream`; `scratch` is device
 * memory of rdkv_fnv1a64_device_scratch(len) bytes.  Used for the payload
 * checksum of generated KV (codec.py:148/222) and of disk hits (codec.py:293),
 * which a single core computes at ~0.6 GB/s. */
RDKV_API size_t rdkv_fnv1a64_device_scratch(size_t len);
RDKV_API int rdkv_fnv1a64_device(const void* data, size_t len, uint64_t seed, void* scratch, size_t scratch_bytes,
                                 uint64_t* out_dev, void* stream);
/* The same in two steps for a payload still arriving (streamed disk hit): the
 * per-chunk automaton pass over the whole chunks of bytes [0, ready), from chunk
 * `chunk_begin` on — returns the next chunk to run (pass ready = len for the
 * rest) — then the stitch / affine / combine passes.  Same scratch, same result. */
RDKV_API int64_t rdkv_fnv1a64_device_partial(const void* data, size_t len, size_t ready, int64_t chunk_begin,
                                             void* scratch, size_t scratch_bytes, void* stream);
RDKV_API int rdkv_fnv1a64_device_finish(const void* data, size_t len, uint64_t seed, void* scratch,
                                        size_t scratch_bytes, uint64_t* out_dev, void* stream);

/* Fixed-width view of the .rdkv header (codec.py:8-13, 35-36, 110-137). */
typedef struct rdkv_header {
  uint64_t model_hash;
  uint64_t payload_len;
  uint64_t checksum;
  uint32_t token_count;
  uint16_t version;
  uint16_t doc_count;
  uint16_t layers;
  uint16_t kv_heads;
  uint16_t head_dim;
  uint8_t elem_width;
  uint8_t reserved_pad[3];
} rdkv_header;

/* Bytes of the encoded header for `doc_count` doc ids: 46 + 8*doc_count
 * (codec.header_size, codec.py:159-160). */
RDKV_API size_t rdkv_header_size(uint32_t doc_count);

/* Serialise a header (magic/version are written by the library) followed by
 * the doc ids into `out` (capacity `cap`).  codec.encode, header part
 * (codec.py:227-239).  Returns the number of bytes written or < 0. */
RDKV_API int64_t rdkv_header_encode(const rdkv_header* h, const uint64_t* doc_ids, void* out, size_t cap);

/* Parse and validate a header from the front of `data`; the doc ids are copied
 * into `doc_ids` (capacity `ids_cap`).  Same checks and error classes as
 * codec.decode_header (codec.py:242-279). */
RDKV_API int rdkv_header_decode(const void* data, size_t len, rdkv_header* h, uint64_t* doc_ids,
                       size_t ids_cap, size_t* header_len);

/* Full decode check of an encoded blob: header, truncation, trailing bytes and
 * the payload FNV-1a (codec.decode, codec.py:282-295). */
RDKV_API int rdkv_blob_check(const void* data, size_t len, rdkv_header* h, uint64_t* doc_ids,
                    size_t ids_cap, size_t* payload_off);

/* ------------------------------------------------ L1: blob file I/O (H2) */

/* Durable write: header + payload to `tmp_path`, then rename onto `final_path`
 * so readers never observe a partial blob (KvStore.put, store.py:215-223). */
RDKV_API int rdkv_blob_write(const char* tmp_path, const char* final_path, const void* header,
                    size_t header_len, const void* payload, size_t payload_len);

/* Size of a file in bytes, or < 0 (RDKV_ERR_IO). */
RDKV_API int64_t rdkv_file_size(const char* path);

/* Read a whole blob file into `buf` (capacity `cap`, normally pinned host
 * memory) placing the payload at an `align`-byte boundary (payload offset in
 * the file is 46+8k, never aligned), with parallel buffered preads.  align = 0:
 * O_DIRECT reads instead (page cache bypassed, block-aligned requests on up to
 * 8 threads): the file's first byte lands on a 4096-byte boundary, `cap` must
 * cover that pad plus the size rounded up to 4096, and file systems that refuse
 * O_DIRECT fall back to buffered reads.  With verify != 0 it runs the same
 * validation as rdkv_blob_check (KvStore.get disk path: store.py:266-267).
 * On success *file_off is where the file's first byte landed in `buf` and
 * *payload_off where the payload starts. */
RDKV_API int rdkv_blob_read(const char* path, void* buf, size_t cap, size_t align, int verify,
                   rdkv_header* h, uint64_t* doc_ids, size_t ids_cap, size_t* file_off,
                   size_t* payload_off);

/* Read file bytes [off, off + len) into `dst` (the part of a blob file a
 * streamed disk hit has not read yet; store.read_blob_file overlaps each
 * segment's H2D copy with the next segment's read).  direct != 0: O_DIRECT,
 * `dst` and `off` 4096-aligned, `cap` >= the bytes read rounded up to 4096 (buffered
 * fallback where the file system refuses O_DIRECT).  Returns the bytes read
 * (short only at end of file), or < 0. */
RDKV_API int64_t rdkv_file_read_range(const char* path, void* dst, size_t cap, uint64_t off, size_t len, int direct);

/* Drop a file's pages from the OS page cache (cold-read benchmarking). */
RDKV_API int rdkv_drop_page_cache(const char* path);

/* ------------------------------------------------------- K1: tcgen05 GEMM */

/* Epilogue selectors for rdkv_gemm_bf16. */
#define RDKV_EPI_STORE 0     /* D = A.B^T (bf16)                         */
#define RDKV_EPI_STORE_F32 1 /* D = A.B^T (fp32)                         */
#define RDKV_EPI_RESID 2     /* D = R + A.B^T (bf16)                     */
#define RDKV_EPI_SWIGLU 3    /* D = silu(gate) * up, [gate|up] blocks of 64 */

/* D[M,N] = A[M,K] . B[N,K]^T on the tcgen05 tensor cores (bf16 in, fp32
 * accumulate).  Building block of the document / query prefill; exposed for
 * tests and for callers that bring their own layers.  No reference analogue:
 * the reference models this work as prefill_work (costs.py:82-86). */
RDKV_API int rdkv_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                   const void* R, int64_t ldr, int M, int N, int K, int epilogue, void* stream);

/* -------------------------------------- document KV layout -> HBM (K3) */

/* One cached blob payload already resident in HBM (staged by an async H2D
 * copy from the pinned host tier, or fetched from a peer GPU). */
typedef struct rdkv_unpack_job {
  const void* src;      /* device payload [L][2][Hkv][n_tokens][dh], elem_width bytes each */
  int32_t n_tokens;     /* tokens of the blob (header token_count)                        */
  int32_t first_block;  /* index into block_table of the blob's first KV block            */
  int64_t reserved;
} rdkv_unpack_job;

/* Unpack n_jobs blob payloads into the paged KV pool
 *   pool: [L][2][Hkv][pool_slots][dh] bf16, token t of job j at slot
 *         block_table[first_block + t / block_size] * block_size + t % block_size.
 * Converts fp32 payloads (elem_width 4) to bf16.  Only layers [layer_begin,
 * layer_end) are moved, so a caller can stream layer by layer on a side stream
 * while the forward consumes earlier layers.  HBM-bound: 2 x payload bytes.  Replaces the payload materialisation of codec.decode
 * (codec.py:292) and the modeled load_time (costs.py:102-108). */
RDKV_API int rdkv_kv_unpack(const rdkv_unpack_job* jobs_dev, int n_jobs, int max_tokens,
                            const int32_t* block_table_dev, int block_size, void* pool_base,
                            int layers, int kv_heads, int head_dim, int64_t pool_slots,
                            int elem_width, int layer_begin, int layer_end, void* stream);

/* rdkv_kv_unpack for one tensor-parallel rank: the payloads hold src_kv_heads
 * heads (the full model's .rdkv layout) and heads [head_begin, head_begin +
 * kv_heads) are unpacked into a pool of kv_heads heads.  Each head is a
 * contiguous [n][dh] run per (layer, K|V) of the head-major payload, so a rank
 * moves exactly its share. */
RDKV_API int rdkv_kv_unpack_heads(const rdkv_unpack_job* jobs_dev, int n_jobs, int max_tokens,
                                  const int32_t* block_table_dev, int block_size, void* pool_base, int layers,
                                  int kv_heads, int head_dim, int64_t pool_slots, int elem_width, int layer_begin,
                                  int layer_end, int head_begin, int src_kv_heads, void* stream);

/* Layer-wise streaming of one batch's cached KV (host tier -> HBM -> pool) in one
 * call: for every layer l, the H2D copy of layer slice l of each (host_src[c],
 * dev_dst[c]) payload pair (copy_layers layers per copy, bytes_per_layer[c] each)
 * on h2d_stream, then on unpack_stream a wait for copied_events[l], the K3
 * unpack of layer l (rdkv_kv_unpack_heads semantics) and a record of
 * layer_events[l] — the events rdkv_batch.layer_ready hands to the forward.
 * n_copies = 0 unpacks device-resident payloads only.  Events must exist
 * (created/recorded once before). */
RDKV_API int rdkv_kv_stream_layers(const rdkv_unpack_job* jobs_dev, int n_jobs, int max_tokens,
                                   const int32_t* block_table_dev, int block_size, void* pool_base, int layers,
                                   int kv_heads, int head_dim, int64_t pool_slots, int elem_width, int head_begin,
                                   int src_kv_heads, int n_copies, void* const* host_src, void* const* dev_dst,
                                   const size_t* bytes_per_layer, int copy_layers, void* h2d_stream,
                                   void* unpack_stream, void* const* copied_events, void* const* layer_events);

/* Copy the first n_tokens slots of pool block src_block into dst_block, in every
 * (layer, K|V, head) plane: one strided DMA (cudaMemcpy2DAsync, L*2*Hkv rows).
 * Copy-on-write of a resident prefix's partial last block, so a query can append
 * its new tokens without touching the shared HBM-tier entry. */
RDKV_API int rdkv_kv_copy_block(void* pool_base, int layers, int kv_heads, int head_dim, int64_t pool_slots,
                                int block_size, int src_block, int dst_block, int n_tokens, void* stream);

/* --------------------------- multi-instance sharing: peer HBM tier (K3p) */

/* CUDA IPC handle (64 bytes) of the device allocation containing dev_ptr, and
 * dev_ptr's byte offset inside it, so a peer process can map this rank's KV
 * pool.  Replaces nothing in the reference: its instances share KV only via the
 * filesystem / TCP (store.py, service.py:143-414); SURVEY §8e. */
RDKV_API int rdkv_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out);
/* Map a peer's allocation (peer access enabled lazily); *base_out is its base. */
RDKV_API int rdkv_ipc_open(const void* handle, void** base_out);
RDKV_API int rdkv_ipc_close(void* base);

/* Strided device copy (cudaMemcpy2DAsync, any device to any device through UVA
 * / IPC mappings): one TP rank's KV heads into the gathered full-model payload
 * on the root rank ([L][2] rows of Hkv/T heads at a pitch of Hkv heads). */
RDKV_API int rdkv_memcpy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                            void* stream);

/* K3p: copy n_blocks KV blocks src_blocks[i] of pool src (possibly a peer's,
 * through rdkv_ipc_open) into dst_blocks[i] of the local pool dst, every
 * (layer, K|V, head) plane.  Pools are [L][2][Hkv][slots][dh] bf16; block
 * index arrays are device int32.  Bytes moved = payload of the blocks (NVLink
 * read + HBM write). */
RDKV_API int rdkv_kv_peer_gather(const void* src_pool, int64_t src_slots, const int32_t* src_blocks,
                                 void* dst_pool, int64_t dst_slots, const int32_t* dst_blocks, int n_blocks,
                                 int layers, int kv_heads, int head_dim, int block_size, void* stream);

/* ------------------- tensor parallelism inside an instance (C5, TP = 2..8) */

/* A TP group's communicator over NVLink peer memory.  Each rank allocates one
 * device buffer of rdkv_tp_comm_bytes(max_elems, size) bytes, ZEROED, exports it
 * (rdkv_ipc_handle) and maps every peer's (rdkv_ipc_open); bases[p] is rank p's
 * buffer as seen from this process (bases[rank] = the local one).  max_elems
 * bounds rows x hidden of one all-reduce.  The buffer holds flags, an epoch
 * counter and double-buffered receive slots [2][size][max_elems] bf16.  No
 * reference analogue: the reference models one device per instance
 * (costs.py:52-60); SURVEY §8e/§8f. */
typedef struct rdkv_tp_comm rdkv_tp_comm;
RDKV_API size_t rdkv_tp_comm_bytes(size_t max_elems, int size);
RDKV_API int rdkv_tp_comm_create(int rank, int size, void* const* bases, size_t max_elems, rdkv_tp_comm** out);
RDKV_API void rdkv_tp_comm_destroy(rdkv_tp_comm* comm);
/* Store a dense [rows][cols] bf16 partial into this rank's slot of parity `buf`
 * in every rank's buffer (P2P stores).  rdkv_forward does this from inside the
 * row-parallel GEMMs' epilogue instead; exposed for tests and custom layers. */
RDKV_API int rdkv_tp_push(rdkv_tp_comm* comm, const void* src, int rows, int cols, int buf, void* stream);
/* x[rows][cols] (ld ldx) += sum of the partials every rank pushed in parity
 * `buf`: publish / await the epoch over NVLink flags, reduce the local receive
 * slots in fp32 with the residual.  Every rank of the group calls it in the same
 * order; graph-capturable (epochs live in device memory). */
RDKV_API int rdkv_tp_reduce_resid(rdkv_tp_comm* comm, void* x, int64_t ldx, int rows, int cols, int buf,
                                  void* stream);

/* ------------------------------------------------ K2/K4: prefill attention */

/* Causal GQA attention of n_tokens new query rows over each sequence's cached
 * prefix plus its own new tokens (cached_prefill_work semantics, costs.py:89-99:
 * the token at position n_cached + i sees every position <= its own).
 *   q, o      [n_tokens][n_heads * head_dim] bf16 (q post-RoPE)
 *   kplane/vplane  one layer's K / V plane [kv_heads][kv_slots][head_dim] bf16,
 *             position p of sequence s at slot block_table[s*bt_stride + p/block_size]
 *             * block_size + p % block_size
 * impl 0 = tcgen05 kernel (block_size % 64 == 0 or bt_stride == 1), 1 = mma.sync
 * kernel (any block size), 2 = tcgen05 kernel on a stream-K schedule (148
 * persistent CTAs with equal KV-tile shares; grids of more than half a wave).
 * `scratch` (rdkv_attention_scratch_bytes) enables split-KV for grids too small
 * to fill the GPU and holds the stream-K partials.  The building block
 * rdkv_forward calls per layer; exposed for tests. */
RDKV_API int rdkv_attention(const void* q, int64_t ldq, void* o, int64_t ldo, const void* kplane,
                            const void* vplane, int64_t kv_slots, const int32_t* seq_start,
                            const int32_t* seq_new, const int32_t* seq_cached, const int32_t* block_table,
                            int bt_stride, int block_size, int n_seqs, int n_tokens, int max_new,
                            int max_ctx, int n_heads, int kv_heads, int head_dim, int impl, void* scratch,
                            size_t scratch_bytes, void* stream);
RDKV_API size_t rdkv_attention_scratch_bytes(int n_tokens, int n_heads, int head_dim);

/* ------------------------------------------ model: document / query prefill */

/* Llama-shaped decoder (RMSNorm, RoPE rotate-half, GQA, SwiGLU). */
typedef struct rdkv_model_desc {
  int32_t layers;
  int32_t hidden;
  int32_t n_heads;
  int32_t kv_heads;
  int32_t head_dim;
  int32_t ffn;
  int32_t vocab;
  int32_t max_pos;
  float rope_theta;
  float norm_eps;
  int32_t flags; /* RDKV_MODEL_* */
} rdkv_model_desc;

/* The attention / MLP RMSNorm gains are folded into the columns of w_qkv / w_gate_up
 * (W'[n][k] = W[n][k] * gain[k]); the gain vectors are then ignored.  Lets large
 * batches fuse the norms across GEMMs: the residual epilogues emit per-row sums of
 * squares and the consuming QKV / gate-up epilogues apply rsqrt(mean + eps). */
#define RDKV_MODEL_NORM_FOLDED 1

/* Weight pointers (device, 16-B aligned), in this order:
 *   [0]                 embedding       bf16 [vocab][hidden]
 *   per layer l (base 1 + 6l):
 *     +0 attn_norm      fp32 [hidden]
 *     +1 wqkv           bf16 [(n_heads + 2 kv_heads) head_dim][hidden]   (q | k | v rows)
 *     +2 wo             bf16 [hidden][n_heads head_dim]
 *     +3 mlp_norm       fp32 [hidden]
 *     +4 w_gate_up      bf16 [2 ffn][hidden], rows interleaved in blocks of 64: g0..63 u0..63 g64..
 *     +5 w_down         bf16 [hidden][ffn]
 *   [1 + 6L]            final_norm      fp32 [hidden]
 *   [2 + 6L]            lm_head         bf16 [vocab][hidden] (may alias the embedding)  */
#define RDKV_WEIGHTS_PER_LAYER 6

typedef struct rdkv_model rdkv_model;

RDKV_API int rdkv_model_create(const rdkv_model_desc* desc, const void* const* weights,
                               size_t n_weights, rdkv_model** out);
RDKV_API void rdkv_model_destroy(rdkv_model* model);

/* A batch of sequences, each = a cached prefix already in the KV pool plus
 * n_new new tokens (uncached documents then the query).  n_cached = 0 for
 * every sequence is the full-prompt prefill; a single sequence whose KV pool
 * is a blob payload (kv_slots = n, block_size = n, block_table = {0}) is
 * document-KV generation, written straight in the .rdkv payload layout. */
typedef struct rdkv_batch {
  int32_t n_seqs;              /* S                                                  */
  int32_t n_tokens;            /* T = sum of n_new                                   */
  int32_t max_new;             /* max n_new over sequences                           */
  int32_t block_size;          /* KV block size in tokens                            */
  int32_t bt_stride;           /* block-table entries per sequence                   */
  int32_t want_logits;         /* 1: last-row logits + argmax; 0: KV only            */
  const int32_t* tokens;       /* dev [T] new token ids, sequences back to back      */
  const int32_t* pos;          /* dev [T] position of each new token (n_cached + i)  */
  const int32_t* slot;         /* dev [T] KV-plane slot receiving each token's K/V   */
  const int32_t* seq_start;    /* dev [S] first row of each sequence in [0, T)       */
  const int32_t* seq_new;      /* dev [S]                                            */
  const int32_t* seq_cached;   /* dev [S] cached-prefix tokens                       */
  const int32_t* block_table;  /* dev [S * bt_stride]                                */
  const int32_t* last_row;     /* dev [S] row of each sequence's last token          */
  void* kv_base;               /* dev KV pool [L][2][Hkv][kv_slots][dh] bf16         */
  int64_t kv_slots;
  float* logits;               /* dev [S][vocab] fp32                                */
  int32_t* next_token;         /* dev [S] argmax (first token), may be NULL          */
  int32_t max_ctx;             /* max over sequences of n_cached + n_new (0: unknown;
                                  enables split-KV attention for small batches)      */
  void* const* layer_ready;     /* optional [layers] cudaEvent_t: layer l's attention
                                  waits for event l (layer-wise KV streaming)        */
  int32_t flags;               /* RDKV_BATCH_ROW_DETERMINISTIC: every row's arithmetic
                                  independent of the batch shape (no split-K GEMMs,
                                  no split-KV attention), so a prefix's KV is
                                  bit-identical to the same rows of a longer prefill */
} rdkv_batch;

#define RDKV_BATCH_ROW_DETERMINISTIC 1

/* Make the model one rank of a TP group: its descriptor / weights are this
 * rank's shard (n_heads, kv_heads, ffn divided by the group size; wqkv rows,
 * wo / w_down columns, w_gate_up blocks sliced accordingly) and rdkv_forward
 * all-reduces the attention-output and down projections over `comm` (NULL = off). */
RDKV_API int rdkv_model_set_tp(rdkv_model* model, rdkv_tp_comm* comm);

/* Device workspace needed by rdkv_forward for n_tokens / n_seqs. */
RDKV_API size_t rdkv_workspace_bytes(const rdkv_model* model, int n_tokens, int n_seqs);

/* Prefill a batch (K1 GEMMs + K2/K4 attention + K5 LM head) on `stream`.
 * Replaces synth_blob (codec.py:188-224) for document KV and ttft
 * (costs.py:121-144) / cached_prefill_work (costs.py:89-99) for queries. */
RDKV_API int rdkv_forward(rdkv_model* model, const rdkv_batch* batch, void* workspace,
                          size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------ measurement */

/* Kernel classes of rdkv_forward for per-class device timing. */
#define RDKV_PROF_QKV 0  /* K1 QKV GEMM (+ RoPE / KV-layout epilogue)        */
#define RDKV_PROF_ATTN 1 /* K2/K4 attention                                  */
#define RDKV_PROF_MISC 2 /* embedding gather, RMSNorm                         */
#define RDKV_PROF_HEAD 3 /* K5 LM-head GEMM + argmax                          */
#define RDKV_PROF_O 4    /* K1 attention-output GEMM (+ residual)            */
#define RDKV_PROF_GU 5   /* K1 gate/up GEMM (+ SwiGLU)                       */
#define RDKV_PROF_DOWN 6 /* K1 down GEMM (+ residual)                        */
#define RDKV_PROF_N 7

/* With on != 0, every kernel rdkv_forward launches is bracketed by CUDA events
 * on its stream.  Launch and algorithmic-FLOP counters run regardless. */
RDKV_API int rdkv_profile_enable(rdkv_model* model, int on);

/* Wait for the recorded launches and return, per class, the summed device
 * milliseconds (ms), kernel launches and GEMM FLOPs (2*M*N*K) since the last
 * collect; resets the counters.  Arrays hold RDKV_PROF_N entries. */
RDKV_API int rdkv_profile_collect(rdkv_model* model, double* ms, int64_t* launches, double* flops);

/* rdkv_gemm_bf16 with an explicit tile N (128 or 256; 0 = automatic) and an
 * optional fp32 scratch buffer enabling split-K for small-M shapes (the
 * partial sums are reduced in a fixed order: results are deterministic). */
RDKV_API int rdkv_gemm_bf16_ex(const void* A, int64_t lda, const void* B, int64_t ldb, void* D,
                               int64_t ldd, const void* R, int64_t ldr, int M, int N, int K,
                               int epilogue, int tile_n, void* scratch, size_t scratch_bytes,
                               void* stream);

/* ------------------------------------------------------------ node control plane (csrc/shm.cpp)
 *
 * One POSIX shared-memory segment per node, shared by the instances (one
 * process per GPU).  Replaces, across processes, what the reference keeps in
 * one Python process: the single-flight in-flight map of
 * SharedCacheService.get_or_generate (service.py:87-127), the central FIFO
 * every idle instance pulls from (sim.py:403-409) and the generator queue
 * (sim.py:297-332), plus the HBM-residency directory (holder rank + pool blocks
 * + pin count) that lets a peer pull a cached prefix over NVLink.
 * All shared words are lock-free atomics.  Keys are (model_hash, file stem)
 * (store.py:71-74). */
typedef struct rdkv_shm rdkv_shm;

#define RDKV_KEY_ABSENT 0     /* nobody asked for it                            */
#define RDKV_KEY_REQUESTED 1  /* queued on its owner's generation ring          */
#define RDKV_KEY_GENERATING 2 /* an owner is running generate() (single flight) */
#define RDKV_KEY_READY 3      /* generated: in the store and/or an HBM tier     */
#define RDKV_KEY_FAILED 4     /* generate() raised; waiters re-request          */

/* create != 0: make (replacing a stale one) and zero the segment; else attach,
 * waiting up to timeout_ms for the creator.  table_slots and ring_slots are
 * powers of two; cell_bytes is the largest ring record. */
RDKV_API int rdkv_shm_open(const char* name, int create, int world, int table_slots, int max_blocks,
                           int ring_slots, int cell_bytes, int n_rings, int max_queries, int timeout_ms,
                           rdkv_shm** out);
RDKV_API void rdkv_shm_close(rdkv_shm* shm);
RDKV_API int rdkv_shm_unlink(const char* name);
RDKV_API int rdkv_shm_world(const rdkv_shm* shm);

/* Single-flight state of a key (RDKV_KEY_*); *owner = the rank that moved it last. */
RDKV_API int rdkv_shm_key_state(rdkv_shm* shm, uint64_t model_hash, uint64_t stem, int* owner);
/* Atomic state transition expect -> desired (1 done, 0 state differed). */
RDKV_API int rdkv_shm_key_cas(rdkv_shm* shm, uint64_t model_hash, uint64_t stem, int expect, int desired,
                              int owner);

/* HBM residency: the holder publishes its pool blocks for a key (1 published,
 * 0 another rank holds it); a reader pins (returns the block count, 0 if not
 * resident), copies over NVLink, unpins; the holder may evict only after
 * retract succeeds (1 retracted or not held, 0 pinned by a reader). */
RDKV_API int rdkv_shm_res_publish(rdkv_shm* shm, uint64_t model_hash, uint64_t stem, int rank,
                                  const int32_t* blocks, int n_blocks, int n_tokens);
RDKV_API int rdkv_shm_res_pin(rdkv_shm* shm, uint64_t model_hash, uint64_t stem, int* rank, int32_t* blocks,
                              int cap, int* n_tokens);
RDKV_API int rdkv_shm_res_unpin(rdkv_shm* shm, uint64_t model_hash, uint64_t stem);
RDKV_API int rdkv_shm_res_retract(rdkv_shm* shm, uint64_t model_hash, uint64_t stem, int rank);
RDKV_API int rdkv_shm_res_holder(rdkv_shm* shm, uint64_t model_hash, uint64_t stem);

/* Bounded MPMC ring `ring`: push returns 1 (0 = full); pop returns the record
 * length (0 = empty). */
RDKV_API int rdkv_shm_ring_push(rdkv_shm* shm, int ring, const void* data, int len);
RDKV_API int rdkv_shm_ring_pop(rdkv_shm* shm, int ring, void* out, int cap);
RDKV_API int64_t rdkv_shm_ring_size(rdkv_shm* shm, int ring);

/* Per-query state byte (queued / dispatched / done) and 64 shared counters. */
RDKV_API int rdkv_shm_qstate_cas(rdkv_shm* shm, int query, int expect, int desired);
RDKV_API int rdkv_shm_qstate(rdkv_shm* shm, int query);
RDKV_API int64_t rdkv_shm_counter_add(rdkv_shm* shm, int index, int64_t delta);

#ifdef __cplusplus
}
#endif

#endif /* RDKV_H */
