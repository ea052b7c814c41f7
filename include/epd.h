/*
 * epd.h -- C ABI of the B200-native EPD encode-stage hot path.
 *
 * This is the drop-in boundary for the encode path of the EPD reference
 * simulator (`disaggsim`, /root/reference/pkg/src/disaggsim). The reference
 * has no FFI of its own: its encode worker, multimodal-token cache and stage
 * handoff are Python calls inside `engine._Sim`. Each group below names the
 * reference interface it stands behind (file:line, relative to
 * /root/reference/pkg/src/disaggsim/). Signatures use plain pointers, sizes and
 * opaque handles only; device pointers are caller-owned unless stated, and
 * `stream` is a cudaStream_t passed as void*. All work is asynchronous on
 * `stream`; nothing synchronises the host except where documented.
 *
 * Errors: every call returns an epd_status_t. The Python host maps each code
 * to the exception class the reference raises for the same condition.
 */
#ifndef EPD_H_
#define EPD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EPD_ABI_VERSION 1

typedef enum {
  EPD_OK = 0,
  EPD_ERR_VALUE = 1,       /* ValueError: irp_shard width<1 / patches<0 (engine.py:57-60),
                              negative counts (costs.py:85-86), bad shapes */
  EPD_ERR_RUNTIME = 2,     /* RuntimeError: cache misuse / overcommit (blocks.py:47-60) */
  EPD_ERR_CAPACITY = 4,    /* CapacityExceeded (simconfig.py:19-20): table or cache full */
  EPD_ERR_CUDA = 5,        /* RuntimeError carrying the CUDA error string */
  EPD_ERR_UNSUPPORTED = 6  /* ValueError: configuration outside what the kernels implement */
} epd_status_t;

int32_t epd_abi_version(void);
/* Message of the last failing call on this host thread ("" if none). */
const char* epd_last_error(void);

/* ------------------------------------------------------------------ routing
 * Replaces engine.irp_shard (engine.py:55-62): balanced partition of one
 * request's tiles across `width` encode workers; the first `patches % width`
 * workers get one extra tile. counts[width] is written.
 */
epd_status_t epd_irp_shard(int64_t patches, int32_t width, int64_t* counts);

/* Contiguous tile ranges implied by the shard order in engine._start_encode
 * (engine.py:589-602): worker k owns [first[k], first[k] + counts[k]). */
epd_status_t epd_irp_ranges(int64_t patches, int32_t width, int64_t* first, int64_t* counts);

/* ------------------------------------------------------------------ encoder
 * Replaces the modeled cost costs.encode_latency (costs.py:78-90) with the
 * real vision encoder + resampler/projector. One encoder per GPU process.
 */
typedef struct epd_encoder epd_encoder_t;

enum {
  EPD_FAMILY_SIGLIP_RESAMPLER = 1, /* MiniCPM-V 2.6: SigLIP ViT + 2D-sincos perceiver resampler */
  EPD_FAMILY_INTERNVIT_MLP = 2     /* InternVL2: InternViT (CLS, layer scale) + pixel shuffle + MLP */
};

typedef struct {
  int32_t family;
  int32_t image_size;  /* tile side in pixels (448) */
  int32_t patch_size;  /* 14 */
  int32_t channels;    /* 3 */
  int32_t hidden;      /* ViT width */
  int32_t layers;
  int32_t heads;
  int32_t mlp;         /* ViT MLP width */
  int32_t out_tokens;  /* MM tokens per tile (models.cfg tokens_per_patch) */
  int32_t out_dim;     /* MM token width (models.cfg hidden_dim) */
  int32_t out_heads;   /* resampler attention heads (family 1) */
  int32_t max_tiles;   /* workspace bound for one epd_encode_tiles call */
  float ln_eps;
  float mean[3];
  float std[3];
} epd_encoder_desc_t;

epd_status_t epd_encoder_create(const epd_encoder_desc_t* desc, int32_t device, epd_encoder_t** out);
void epd_encoder_destroy(epd_encoder_t* enc);
/* Canonical (framework-layout, fp32) weight schema; index order is stable. */
int32_t epd_encoder_num_weights(const epd_encoder_t* enc);
epd_status_t epd_encoder_weight_info(const epd_encoder_t* enc, int32_t index, const char** name,
                                     int32_t* ndim, int64_t* shape /* [4] */);
/* Host fp32 values for weight `index`; the library converts to bf16 and to
 * its own B200 layout (head padding, fused QKV, transposes) at finalize. */
epd_status_t epd_encoder_set_weight(epd_encoder_t* enc, int32_t index, const float* host_values,
                                    int64_t numel);
/* Uploads weights and precomputes weight-only constants. Synchronises. */
epd_status_t epd_encoder_finalize(epd_encoder_t* enc, void* stream);
/* tiles: device uint8 [n][S][S][C] (HWC); out: device bf16 [n][out_tokens][out_dim]. */
epd_status_t epd_encode_tiles(epd_encoder_t* enc, const uint8_t* tiles, int32_t n, void* out,
                              void* stream);
/* fp32 check mode (north star: <= 1e-4 vs the fp32 oracle). Call before
 * finalize; the library then also keeps fp32 twins of every weight image and
 * epd_encode_tiles_f32 runs the same pipeline (same layouts and fusions) on
 * fp32 CUDA cores. A verification path, not a serving path. */
epd_status_t epd_encoder_enable_fp32_check(epd_encoder_t* enc);
/* tiles: device uint8 [n][S][S][C]; out: device fp32 [n][out_tokens][out_dim]. */
epd_status_t epd_encode_tiles_f32(epd_encoder_t* enc, const uint8_t* tiles, int32_t n, float* out,
                                  void* stream);
/* Algorithmic FLOPs of one tile (roofline numerator). */
double epd_encoder_flops_per_tile(const epd_encoder_t* enc);
/* Kernel launches issued by one epd_encode_tiles call over n tiles. */
int32_t epd_encoder_launches(const epd_encoder_t* enc, int32_t n);
/* Replay each forward pass as one CUDA graph per chunk size (default on; the
 * graph reads/writes encoder-owned staging buffers). Off = direct launches. */
epd_status_t epd_encoder_set_graphs(epd_encoder_t* enc, int32_t on);
/* Per-launch CUDA-event profiling of subsequent encode calls (on = 1/0; uses
 * direct launches while on). */
epd_status_t epd_encoder_profile(epd_encoder_t* enc, int32_t on);
/* Drain the profile (synchronises on the last recorded event). Per kernel class
 * c in {0 patchify, 1 gemm, 2 attention, 3 layernorm, 4 other}: summed device
 * milliseconds, algorithmic FLOPs, algorithmic bytes and launch counts. */
epd_status_t epd_encoder_profile_read(epd_encoder_t* enc, double* ms, double* flops, double* bytes,
                                      int64_t* launches, int32_t nclass);
/* Per-launch view of the profile last drained by epd_encoder_profile_read, in
 * issue order: class, device ms, algorithmic FLOPs. Copies min(n, cap) records
 * and returns n (-1 for a null encoder). */
int32_t epd_encoder_profile_launches(const epd_encoder_t* enc, int32_t* cls, float* ms, double* flops,
                                     int32_t cap);

/* ------------------------------------------------------------------ MM-token cache
 * Stands behind blocks.BlockManager(CacheKind.MM) (blocks.py:14-61) as the
 * encode-side multimodal cache; adds the content-hash lookup the reference
 * lacks so repeated images skip encoding. Keys are 2 x u64 per record.
 */
typedef struct epd_mmcache epd_mmcache_t;

/* keys[n][2] <- content hash of n records of rec_bytes each (pitch rec_stride).
 * scratch: device buffer of >= 16*n bytes. The unkeyed form is the known-answer mode
 * (secret = 0); a serving cache keys the hash with a per-process random secret so
 * collisions cannot be forged offline. */
epd_status_t epd_hash_records(const void* data, int32_t n, int64_t rec_bytes, int64_t rec_stride,
                              uint64_t* keys, void* scratch, void* stream);
epd_status_t epd_hash_records_keyed(const void* data, int32_t n, int64_t rec_bytes, int64_t rec_stride,
                                    uint64_t secret0, uint64_t secret1, uint64_t* keys, void* scratch,
                                    void* stream);
/* Table with at least 2*capacity slots (power of two) + the device planner's LRU list, free
 * stack and entry keys. capacity <= 16384 entries. */
epd_status_t epd_mmcache_create(int64_t capacity, int32_t device, epd_mmcache_t** out);
void epd_mmcache_destroy(epd_mmcache_t* cache);
/* One request's cache plan, entirely on the device (one CTA): classify its n tiles (keys[n][2])
 * in tile order as hit (cached) / miss (first occurrence of an uncached key) / dup (repeat of an
 * earlier miss), refresh the hits' recency, evict least-recently-used entries not referenced by
 * the request, hand the misses entry ids from the LIFO free stack (the BlockManager discipline,
 * blocks.py:29-61) and insert them. Outputs (device): entries[n], kinds[n] (0/1/2),
 * miss_tiles[n] + miss_entries[n] (first counts[0] valid, tile order), victim_keys[n][2]
 * (first counts[3] valid, eviction order), counts[5] = misses, hits, dups, victims, status
 * (1: more distinct tiles than entries -- CapacityExceeded, nothing changed). n <= 4096.
 * The only value a host needs back is counts (the number of tiles to encode). */
epd_status_t epd_mmcache_plan(epd_mmcache_t* cache, const uint64_t* keys, int32_t n, int32_t* entries,
                              int32_t* kinds, int32_t* miss_tiles, int32_t* miss_entries, uint64_t* victim_keys,
                              int32_t* counts, void* stream);
/* Low-level table access (not mixed with epd_mmcache_plan on one cache):
 * entry[i] = value stored for keys[i] or -1; dup[i] = first j < i with the same
 * key among misses, else -1 (in-batch repeats). */
epd_status_t epd_mmcache_lookup(epd_mmcache_t* cache, const uint64_t* keys, int32_t n,
                                int32_t* entry, int32_t* dup, void* stream);
/* Insert absent, batch-unique keys with their entry ids. */
epd_status_t epd_mmcache_insert(epd_mmcache_t* cache, const uint64_t* keys, const int32_t* entries,
                                int32_t n, void* stream);
epd_status_t epd_mmcache_erase(epd_mmcache_t* cache, const uint64_t* keys, int32_t n, void* stream);
/* Empty the table and reset the planner (free stack 0, 1, 2, ... again). */
epd_status_t epd_mmcache_clear(epd_mmcache_t* cache, void* stream);
/* Synchronises `stream`; EPD_ERR_CAPACITY if any insert found no free slot. */
epd_status_t epd_mmcache_check(epd_mmcache_t* cache, void* stream);

/* ------------------------------------------------------------------ packing / handoff
 * MM-token packing (implicit in engine._send_ready_shards, engine.py:521-526):
 * dst[i] = src[index[i]] for records of rec_bytes (16-byte multiples). */
epd_status_t epd_gather_records(const void* src, const int32_t* index, int32_t n, int64_t rec_bytes,
                                void* dst, void* stream);
/* dst[index[i]] = src[i]. */
epd_status_t epd_scatter_records(const void* src, const int32_t* index, int32_t n, int64_t rec_bytes,
                                 void* dst, void* stream);
/* Paged KV handoff (engine._try_reserve_decode / _on_transfer_end("pd"),
 * engine.py:542-555, 436-439). The cache holds `segments` (= 2 x layers)
 * arrays of fixed-size blocks: block b of segment s starts at
 * cache + s*segment_stride + b*block_bytes. pack: out[i][s] = cache[s][ids[i]];
 * unpack: cache[s][ids[i]] = in[i][s]. */
epd_status_t epd_kv_pack(const void* cache, int32_t segments, int64_t segment_stride,
                         int64_t block_bytes, const int32_t* block_ids, int32_t nblocks, void* out,
                         void* stream);
epd_status_t epd_kv_unpack(const void* in, int32_t segments, int64_t segment_stride,
                           int64_t block_bytes, const int32_t* block_ids, int32_t nblocks, void* cache,
                           void* stream);

/* The same handoff without a staging buffer: dst[s][dst_ids[i]] = src[s][src_ids[i]] for
 * every segment s. dst_cache may be another GPU's pool mapped with epd_peer_open, in which
 * case this one kernel is the NVLink transfer (prefill pushes into the decode pool). */
epd_status_t epd_kv_move(const void* src_cache, int64_t src_segment_stride, void* dst_cache,
                         int64_t dst_segment_stride, int32_t segments, int64_t block_bytes, const int32_t* src_ids,
                         const int32_t* dst_ids, int32_t nblocks, void* stream);

/* Trace clock (trace.ShardRecord / RequestRecord times, trace.py:18-53): *slot = the GPU's
 * %globaltimer (ns) when the stream reaches this point. */
epd_status_t epd_timestamp(uint64_t* slot, void* stream);

/* ------------------------------------------------------------------ stage handoff over NCCL
 * The NCCL legs of the stage-handoff interface, so a non-Python host can
 * run them: the EP migration of MM tokens to the prefill rank (engine._send_ready_shards /
 * _schedule_transfer, engine.py:511-526; prefill starts once all shards landed,
 * _on_transfer_end("ep"), engine.py:424-435) and the PD migration of paged KV into the
 * blocks the decode instance reserved (_try_reserve_decode, engine.py:542-555;
 * _on_transfer_end("pd"), engine.py:436-439). NCCL is resolved at run time (the copy the
 * process already loaded, else libnccl.so.2, or $EPD_NCCL_LIB); without it these calls return
 * EPD_ERR_UNSUPPORTED. The unique id (EPD_COMM_ID_BYTES opaque bytes) is made on one rank
 * and broadcast by the host (e.g. through the torch.distributed store). */
#define EPD_COMM_ID_BYTES 128
typedef struct epd_comm epd_comm_t;
/* version = NCCL_VERSION_CODE of the loaded library (e.g. 22809 for 2.28.9). */
epd_status_t epd_comm_version(int32_t* version);
epd_status_t epd_comm_unique_id(uint8_t* id);
/* Collective over nranks processes (ncclCommInitRank on `device`). */
epd_status_t epd_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, epd_comm_t** comm);
void epd_comm_destroy(epd_comm_t* comm);
/* EP gather of one request of n_tiles tiles (tile_bytes each = tokens_per_patch x
 * mm_bytes_per_token, engine.py:524): rank k holds the shard epd_irp_ranges(n_tiles, nranks)
 * assigns it (irp_shard, engine.py:55-62) in `shard`; the root receives every shard into
 * packed[first_k * tile_bytes ...], i.e. request order whatever the arrival order. On the
 * root, `shard` may alias its own slice of `packed` (no copy) or be any other buffer. Called
 * by every rank of the communicator; ranks with an empty shard send nothing. */
epd_status_t epd_gather_tokens(epd_comm_t* comm, const void* shard, int64_t n_tiles, int64_t tile_bytes,
                               void* packed, int32_t root, void* stream);
/* Raw bytes between two ranks (stream-ordered ncclSend / ncclRecv); the group calls bracket
 * several of them into one NCCL group (e.g. a send to self and the matching receive). */
epd_status_t epd_comm_send(epd_comm_t* comm, const void* buf, int64_t bytes, int32_t peer, void* stream);
epd_status_t epd_comm_recv(epd_comm_t* comm, void* buf, int64_t bytes, int32_t peer, void* stream);
epd_status_t epd_comm_group_start(void);
epd_status_t epd_comm_group_end(void);
/* PD handoff: the prefill rank packs blocks block_ids[0..nblocks) of its paged cache
 * (geometry as epd_kv_pack) into `staging` (nblocks x segments x block_bytes) and sends it to
 * `peer`; the decode rank receives into its staging buffer and unpacks into the block ids it
 * reserved. Both sides must agree on nblocks (= blocks_needed(total_tokens), blocks.py:24-26)
 * before calling -- the host's reservation handshake (handoff.py). */
epd_status_t epd_kv_handoff_send(epd_comm_t* comm, const void* cache, int32_t segments, int64_t segment_stride,
                                 int64_t block_bytes, const int32_t* block_ids, int32_t nblocks, void* staging,
                                 int32_t peer, void* stream);
epd_status_t epd_kv_handoff_recv(epd_comm_t* comm, void* cache, int32_t segments, int64_t segment_stride,
                                 int64_t block_bytes, const int32_t* block_ids, int32_t nblocks, void* staging,
                                 int32_t peer, void* stream);

/* ------------------------------------------------------------------ EP gather over peer memory
 * The B200-native transport for the encode -> prefill MM-token transfer
 * (engine._send_ready_shards / _schedule_transfer, engine.py:511-526; arrival accounting
 * _on_transfer_end("ep"), engine.py:424-435). The prefill rank exports its packed-token
 * slots and per-rank flags with CUDA IPC; each encode rank maps them, stores its shard at
 * the shard's tile offset over NVLink (epd_peer_put) and raises its flag; the prefill
 * rank's stream waits on its local flags (epd_stream_wait_geq). Buffers shared this way
 * come from epd_peer_alloc (zero-filled, allocation base = the pointer). */
epd_status_t epd_peer_alloc(int64_t bytes, void** ptr);
epd_status_t epd_peer_free(void* ptr);
/* handle: 64 bytes (cudaIpcMemHandle_t) for a pointer returned by epd_peer_alloc. */
epd_status_t epd_peer_export(void* ptr, void* handle);
/* Map another process's exported allocation into this device's address space. */
epd_status_t epd_peer_open(const void* handle, void** ptr);
epd_status_t epd_peer_close(void* ptr);
/* dst[0:bytes] = src[0:bytes] (16-byte aligned; dst may be a peer mapping), then, when
 * flag is non-null, *flag = value once the bytes are visible system-wide. */
epd_status_t epd_peer_put(const void* src, void* dst, int64_t bytes, uint32_t* flag, uint32_t value,
                          void* stream);
/* *flag = value (release, system scope) after the stream's earlier work. */
epd_status_t epd_peer_signal(uint32_t* flag, uint32_t value, void* stream);
/* The stream's later work waits until *flag >= value (flag in this device's memory). */
epd_status_t epd_stream_wait_geq(const uint32_t* flag, uint32_t value, void* stream);

/* ------------------------------------------------------------------ kernel-level ops
 * The building blocks epd_encode_tiles is made of, exported for per-kernel
 * parity tests and profiling. All tensors are device bf16 unless stated.
 *
 * out[M,N] = act(A[M,K] W[N,K]^T + bias) ; if resid: out = resid[row % r_mod] + lscale * out
 * act: 0 none, 1 GELU (tanh approximation), 2 GELU (erf), 3 SwiGLU: W's rows alternate
 * 32-row gate / up groups and out[:, 32g + j] = silu(gate + b) * (up + b) for group g
 * (out has N/2 columns; no resid / lscale). bias/resid/lscale may be NULL.
 * bn: N tile (0 = auto, else 128/192/256). */
epd_status_t epd_linear_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M, int32_t N,
                             int32_t K, const void* bias, int32_t act, const void* resid, int32_t ldr,
                             int32_t r_mod, const void* lscale, void* out, int32_t ldo, int32_t bn,
                             void* stream);
/* GEMM tiling policy for subsequent launches in this process: 0 auto, else the cluster
 * size: 1 single-CTA tiles, 2 CTA pairs (tcgen05 cta_group::2), 4 two CTA pairs sharing
 * every B tile through TMA multicast. Results do not depend on the policy. */
epd_status_t epd_set_gemm_cta_group(int32_t policy);
/* Residual-stream update: h[M,N] (fp32, in place) += lscale * (A W^T + bias); lscale may be NULL.
 * The epilogue is a TMA reduce-add, so h is never read by the SMs. */
epd_status_t epd_linear_acc_f32(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M, int32_t N,
                                int32_t K, const void* bias, const void* lscale, float* h, int32_t ldh, int32_t bn,
                                void* stream);
/* The same, allowed to split K over up to max_split work items per output tile when the tiles
 * alone leave SMs idle (small M, long K: the LLM prefill's down / O projections). The splits
 * add into h in a fixed order, so results are run-to-run deterministic, but the split count
 * follows M: not batch invariant (the encoder path never splits). Split launches on one device
 * share a progress-counter buffer: issue them on one stream (or serialize them). */
epd_status_t epd_linear_acc_f32_split(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M,
                                      int32_t N, int32_t K, const void* bias, const void* lscale, float* h,
                                      int32_t ldh, int32_t bn, int32_t max_split, void* stream);
/* Projection straight into attention layouts: column n of A W^T + bias (+ resid[row % r_mod])
 * splits into section s = n / sec_cols, head h, dim d (head dim padded to Dp); row = b*T + t.
 * Section s writes out_s[((b*H + h)*T + t)*Dp + d], or, when bit s of trans_mask is set,
 * the keys-major out_s[((b*H + h)*Dp + d)*Tpad + t]. */
epd_status_t epd_linear_heads_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M,
                                   int32_t N, int32_t K, const void* bias, const void* resid, int32_t ldr,
                                   int32_t r_mod, int32_t H, int32_t Dp, int32_t T, int32_t Tpad,
                                   int32_t sec_cols, void* out0, void* out1, void* out2, int32_t trans_mask,
                                   void* stream);
/* O = softmax(Q K^T * scale) V per (batch, head); see csrc/kernels.h AttnParams.
 * q: [q_shared ? H : B*H][Tq][Dp], k and v: [B*H][Tk][Dp],
 * out[(b*Tq + i)*ldo + h*Dv + d]. Dp in {64, 80, 128}. */
/* Fused multi-head attention read in place from row-major projection outputs:
 *   Q: q[(b*Tq + t)*ldq + h*head_stride + d]  (EPD_ATTN_Q_SHARED: q[t*ldq + h*head_stride + d],
 *      one query set shared by every batch entry),
 *   K, V: k[(b*Tk + t)*ldk + (h / (H/kv_heads))*head_stride + d] (grouped K/V heads; kv_heads
 *      = 0 means H), V likewise with ldv,
 *   out[(b*Tq + t)*ldo + h*Dv + d], d < Dv.
 * EPD_ATTN_CAUSAL: query t sees keys <= t + (Tk - Tq). Dp (64, 80 or 128) is the MMA
 * width, Dv rounded up to 16; head_stride >= Dv. */
#define EPD_ATTN_Q_SHARED 1
#define EPD_ATTN_CAUSAL 2
epd_status_t epd_attention_bf16(const void* q, int32_t ldq, const void* k, int32_t ldk, const void* v,
                                int32_t ldv, void* out, int32_t ldo, int32_t B, int32_t H, int32_t kv_heads,
                                int32_t Tq, int32_t Tk, int32_t Dp, int32_t Dv, int32_t head_stride,
                                int32_t flags, float scale, void* stream);
epd_status_t epd_layernorm_bf16(const void* in, int32_t ld_in, void* out, int32_t ld_out, const void* gamma,
                                const void* beta, int32_t rows, int32_t D, float eps, void* stream);
/* Residual-stream LayerNorm: fp32 rows in, bf16 rows out (the encoder's pre-attention /
 * pre-MLP normalisation of its fp32 residual stream). */
epd_status_t epd_layernorm_f32_bf16(const float* in, int32_t ld_in, void* out, int32_t ld_out, const void* gamma,
                                    const void* beta, int32_t rows, int32_t D, float eps, void* stream);
/* uint8 HWC tiles [n][S][S][C] -> bf16 rows [n*rows_per_tile][Kpad], patch rows start at
 * row_offset within each tile's block; columns in (c, ky, kx) order, zero padded. */
epd_status_t epd_patchify_u8(const uint8_t* tiles, int32_t n, int32_t S, int32_t C, int32_t p, int32_t Kpad,
                             int32_t row_offset, int32_t rows_per_tile, const float* mean3, const float* std3,
                             void* out, void* stream);

/* ------------------------------------------------------------------ prefill consumer
 * the LLM prefill on the prefill GPU that consumes the packed MM
 * tokens (the reference models it as costs.prefill_latency, costs.py:93-99, and
 * _on_batch_end, engine.py:385-407). Decoder layers use epd_linear_* / epd_attention_bf16
 * (causal, grouped KV heads); these are the remaining pieces. */
/* fp32 rows -> RMSNorm (gamma) -> bf16 rows. */
epd_status_t epd_rmsnorm_f32_bf16(const float* in, int32_t ld_in, void* out, int32_t ld_out, const void* gamma,
                                  int32_t rows, int32_t D, float eps, void* stream);
/* In-place rotary embedding (rotate-half) on heads [0, nheads) of width hd starting at column
 * col0 of each bf16 row; position of row r = pos0 + r, angle = pos * theta^(-2i/hd).
 * cos_sin: NULL, or the table epd_rope_table built for the same rows / hd / pos0 / theta. */
epd_status_t epd_rope_bf16(void* x, int32_t ld, int32_t rows, int32_t col0, int32_t nheads, int32_t hd,
                           int32_t pos0, float theta, const float* cos_sin, void* stream);
/* cos_sin[r][i] = (cos, sin)(pos * theta^(-2i/hd)), pos = pos0 + r, i < hd/2: fp32 [rows][hd/2][2]. */
epd_status_t epd_rope_table(float* cos_sin, int32_t rows, int32_t hd, int32_t pos0, float theta, void* stream);
/* out[r][c] = silu(gu[r][c]) * gu[r][F + c]. */
epd_status_t epd_silu_mul_bf16(const void* gu, int32_t ld_in, void* out, int32_t ld_out, int32_t rows, int32_t F,
                               void* stream);
/* Prefill K/V rows into the paged KV pool (handoff.py layout [segments][blocks][block_size*row_elems]):
 * row t of K (src + t*ld_src) and V (src + t*ld_src + v_off) go to block block_ids[t/block_size],
 * slot t%block_size of segments seg0 and seg0+1. */
epd_status_t epd_kv_write_paged(const void* src, int32_t ld_src, int32_t v_off, int32_t rows, int32_t row_elems,
                                const int32_t* block_ids, int32_t block_size, void* pool, int64_t seg_elems,
                                int32_t seg0, void* stream);
/* dst[r][:D] = float(src[index[r]][:D]). */
epd_status_t epd_gather_rows_f32(const void* src, int32_t ld_src, const int32_t* index, int32_t rows, int32_t D,
                                 float* dst, int32_t ld_dst, void* stream);
/* *out = argmax(x[0:n]) (first index on ties). */
epd_status_t epd_argmax_bf16(const void* x, int32_t n, int32_t* out, void* stream);

/* ------------------------------------------------------------------ image tiling
 * SURVEY.md 8(f) item 3 (the step before the path; the reference only looks tile counts up,
 * models.py:138-143). out[n][S][S][C] uint8 = the cols x rows grid tiles (row-major) of the
 * image resized to (cols*S, rows*S), plus, when thumb, the whole image resized to S x S --
 * first when thumb_first (MiniCPM-V order) else last (InternVL order). Antialiased bilinear
 * (triangle filter widened by the downscale factor). cols*rows may be 0 (thumbnail only). */
epd_status_t epd_tile_image(const uint8_t* src, int32_t H, int32_t W, int32_t C, int32_t cols, int32_t rows,
                            int32_t thumb, int32_t thumb_first, int32_t S, uint8_t* out, void* stream);

/* ------------------------------------------------------------------ device block free list
 * blocks.BlockManager's free stack (blocks.py:29, 52, 61) in device
 * memory (int32 stack[total], int32 *top), stream-ordered. init: stack = total-1 .. 0, top =
 * total (ids 0, 1, 2, ... come out first). alloc: out[i] = stack[top-1-i], top -= need. free:
 * ids pushed in reverse, top += n (so they are handed out again in their original order).
 * Capacity / double-free checks are the caller's: the counts are host-known. */
epd_status_t epd_blocks_init(int32_t* stack, int32_t* top, int32_t total, void* stream);
epd_status_t epd_blocks_alloc(int32_t* stack, int32_t* top, int32_t need, int32_t* out_ids, void* stream);
epd_status_t epd_blocks_free(int32_t* stack, int32_t* top, const int32_t* ids, int32_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* EPD_H_ */
