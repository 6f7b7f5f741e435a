/*
 * sarathi.h — C ABI of libsarathi.so, the B200-native (sm_100a) hot path of SARATHI
 * (Agrawal et al., arXiv 2308.16369): the decode-maximal hybrid-batch transformer forward pass.
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn (section in parentheses).
 *
 * The problem the library solves (§4.3 "Decode-Maximal Batching"): one iteration runs
 * ONE prefill chunk (§4.2 "Chunked-prefills") together with up to B-1 single-token decodes of
 * other requests, fusing all linear operations over the p + d tokens into one matmul
 * each while attention runs separately per token kind.  KV caches are pre-allocated per
 * request for its maximum length and updated in place (§4.5).
 *
 * Conventions
 *  - Every function returning int returns SARATHI_OK (0) or a negative SARATHI_E* code; the
 *    thread-local message of the last failure is returned by sarathi_last_error().
 *  - On any error raised before device work is enqueued, library state is unchanged.
 *  - Host arrays passed in are owned by the caller and read synchronously during the call.
 *  - Device work is enqueued on the stream given in sarathi_dist.stream (NULL = legacy default
 *    stream); outputs are valid after the caller synchronises that stream.
 *  - One model handle serves one host thread (no internal locking).  One handle per GPU/process.
 *  - Under tensor parallelism (world > 1, Megatron column/row sharding, §2.3) every rank
 *    makes identical calls in the same order; integer metadata (schedules, block tables, slot
 *    mappings) is computed identically on every rank.
 */
#ifndef SARATHI_H_
#define SARATHI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------------------ */
#define SARATHI_OK 0
#define SARATHI_EINVAL (-1)       /* bad argument / configuration (e.g. heads % world != 0, T > cap) */
#define SARATHI_ENOKV (-2)        /* KV block reservation does not fit (admission failure)        */
#define SARATHI_EUNKNOWN_REQ (-3) /* request id not allocated                                      */
#define SARATHI_EDUP (-4)         /* request twice in one batch (incl. as prefill and decode)      */
#define SARATHI_EPOS (-5)         /* start_pos / position != the request's cached length           */
#define SARATHI_EOVERFLOW (-6)    /* would exceed the request's reserved max_tokens                */
#define SARATHI_ECUDA (-7)        /* CUDA runtime error (device state may be undefined)            */
#define SARATHI_ENCCL (-8)        /* NCCL error                                                    */
#define SARATHI_ESTATE (-9)       /* call out of order (e.g. run before alloc_kv)                  */

/* ---- model --------------------------------------------------------------------------------- */
typedef struct sarathi_model sarathi_model;

#define SARATHI_FFN_SWIGLU 0 /* gate, up, down (LLaMA)                                   */
#define SARATHI_FFN_GELU 1   /* ffn_ln1 + GELU-tanh + ffn_ln2 (Table, GPT-3) */

/* Logical (unsharded) decoder-only transformer, P:L193-203 (§2.1) with readings O-1..O-8. */
typedef struct {
  int32_t n_layers;   /* L                                                    */
  int32_t hidden;     /* H (embedding size)                           */
  int32_t n_heads;    /* query heads                                          */
  int32_t n_kv_heads; /* key/value heads (== n_heads for MHA; GQA otherwise)  */
  int32_t head_dim;   /* 64 or 128                                            */
  int32_t ffn_hidden; /* H2 ("second hidden dimension")               */
  int32_t vocab;      /* V                                                    */
  int32_t ffn_kind;   /* SARATHI_FFN_*                                        */
  float rms_eps;      /* RMSNorm epsilon (1e-5)                               */
  float rope_base;    /* RoPE base (10000)                                    */
  int32_t max_seq_len;          /* positions < max_seq_len (RoPE table size)  */
  int32_t max_tokens_per_batch; /* cap on T = p + d (workspace sizing)        */
} sarathi_model_config;

/* Process / device placement.  world == 1: no NCCL.  world > 1: nccl_unique_id points to the
 * 128-byte ncclUniqueId produced by sarathi_nccl_unique_id() on rank 0 and broadcast by the
 * caller (e.g. over a torch.distributed process group). */
typedef struct {
  int32_t rank;
  int32_t world;
  int32_t device;             /* CUDA device ordinal used by this handle               */
  const void* nccl_unique_id; /* 128 bytes, or NULL when world == 1 or local_group set */
  void* stream;               /* cudaStream_t all device work is enqueued on            */
  void* local_group;          /* sarathi_local_group* (world > 1 on ONE device), or NULL */
  int32_t pp_stage;           /* pipeline stage of this handle (0-based); 0 with pp_stages <= 1   */
  int32_t pp_stages;          /* pipeline stages (0 or 1 = no pipeline); stage s holds layers     */
                              /* [floor(L s / S), floor(L (s+1) / S)), the first also the         */
                              /* embedding, the last the final norm + LM head (NEXT-4)            */
} sarathi_dist;

/* Local tensor-parallel group: `world` (2..8) model handles created on the SAME device with
 * dist.local_group set, each driven by its own host thread making identical calls (SPMD), stand in
 * for one process per GPU.  Every world > 1 path of run_hybrid_batch runs unchanged (Megatron
 * shards, bf16 partials, all-reduce-add fused into RMSNorm, vocab-parallel LM head + all-gather);
 * only the two collectives are replaced: the all-reduce sums the ranks' bf16 partials in rank
 * order (fp32 accumulate, identical on every rank) and the all-gather copies peer buffers, both
 * ordered by CUDA events + a host barrier (timeout -> ENCCL; SARATHI_GROUP_TIMEOUT_S, default
 * 120 s).  With dist.stream == NULL each rank gets its own library-owned stream.  Destroy the group
 * after its models.  Used for on-one-GPU TP parity (§2.3). */
typedef struct sarathi_local_group sarathi_local_group;
int sarathi_local_group_create(int32_t world, int32_t device, sarathi_local_group** out);
void sarathi_local_group_destroy(sarathi_local_group* g);

/* Writes a fresh ncclUniqueId (128 bytes) to out.  Host only.  ENCCL if NCCL is unavailable. */
int sarathi_nccl_unique_id(void* out128);

/* Creates the model on dist->device with this rank's weight shards, either
 *  - host_tensors == NULL: generated ON DEVICE from the counter-based generator spec
 *    (synth/__init__.py header; seed = weight_seed), or
 *  - host_tensors != NULL: loaded from the caller's LOGICAL (unsharded) bf16 tensors in host memory
 *    (read during the call, not retained; weight_seed ignored), nn.Linear [out, in] row-major:
 *      host_tensors[9*l + 0..8] = layer l's  Wq [nq*hd, H], Wk [nkv*hd, H], Wv [nkv*hd, H],
 *                                 Wo [H, nq*hd], Wg [H2, H] (GELU: W1), Wu [H2, H] (GELU: NULL,
 *                                 unused), Wd [H, H2] (GELU: W2), g1 [H], g2 [H]
 *      host_tensors[9*L + 0..2]  = embedding [V, H], final norm gain [H], LM head [V, H]
 *    (the paper's real-model setting, §4.5: configs of real LLaMA/GPT models).
 *    The library takes this rank's Megatron shard (column/row/vocab-parallel, sarathi_shard_map),
 *    applies the packed row orders and the tile-major layout below; EINVAL if a needed pointer is NULL.
 * Weights are packed in kernel layout: per layer QKV [(nq+2nkv)/t*hd, H] (inside each head, row 32j+l is dim
 * 16j+l for l < 16 and dim hd/2+16j+l-16 otherwise: rotate-half partners share a warp), gate||up
 * interleaved in 16-row blocks [2*H2/t, H] (rows 32b..32b+15 gate features 16b.., the next 16 the
 * matching up features), O [H, nq*hd/t], down [H, H2/t]; embedding and final norm replicated; LM
 * head vocab-parallel [ceil(V/t), H].  Ownership: the library owns all device memory.
 * Errors: EINVAL (bad config / divisibility by world), ECUDA (allocation), ENCCL. */
int sarathi_init_model(const sarathi_model_config* cfg, const sarathi_dist* dist, uint64_t weight_seed,
                       const void* const* host_tensors, sarathi_model** out);

void sarathi_destroy(sarathi_model* m);

/* Allocates the paged KV pools: per layer K and V, bf16 [num_blocks][n_kv/t][block_size][hd].
 * block_size: 16, 32, 64 or 128 (each divides the 128-key tile of the tcgen05 prefill-attention
 * kernel, and the decode kernel's 2-stage K/V ring fits shared memory at head_dim 128).
 * Call once, after init, before any request.
 * Errors: EINVAL, ESTATE (already allocated), ECUDA (out of memory). */
int sarathi_alloc_kv(sarathi_model* m, int64_t num_blocks, int32_t block_size);

/* Bytes of KV cache one token occupies on this rank over all layers, m_kv (reading O-18). */
int sarathi_kv_bytes_per_token(const sarathi_model* m, int64_t* out);

/* Max batch B = floor((M_G - M_S) / (L * m_kv)) (§4.3) where M_G - M_S is the device
 * memory currently free minus reserve_bytes and L = tokens_per_request.  Host + cudaMemGetInfo. */
int sarathi_max_batch(const sarathi_model* m, int32_t tokens_per_request, int64_t reserve_bytes, int32_t* B_out);

/* Reserves ceil(max_tokens / block_size) KV blocks for req_id, lowest-free-block-first
 * (reading O-17), i.e. the paper's up-front pre-allocation.  cached length := 0.
 * Errors: EINVAL (max_tokens < 1 or > max_seq_len, or id in use), ENOKV, ESTATE. */
int sarathi_request_alloc(sarathi_model* m, int64_t req_id, int32_t max_tokens);
/* Releases the request's blocks.  EUNKNOWN_REQ. */
int sarathi_request_free(sarathi_model* m, int64_t req_id);
/* Current cached length (tokens whose K,V are in the cache).  EUNKNOWN_REQ. */
int sarathi_request_cached_len(const sarathi_model* m, int64_t req_id, int32_t* len_out);

/* One prefill chunk: token_ids[n_tokens] (host) at positions start_pos .. start_pos+n_tokens-1.
 * start_pos must equal the request's cached length (chunk j of §4.2). */
typedef struct {
  int64_t req_id;
  int32_t start_pos;
  int32_t n_tokens;
  const int32_t* token_ids;
} sarathi_prefill_chunk;

/* d single-token decodes of other requests (host arrays of length n).  positions[i] must equal
 * the cached length of req_ids[i]; each request at most once per batch. */
typedef struct {
  int32_t n;
  const int64_t* req_ids;
  const int32_t* token_ids;
  const int32_t* positions;
} sarathi_decode_set;

#define SARATHI_RETURN_ALL_ROWS 1 /* logits for all T rows (chunk rows then decodes) instead of R */
#define SARATHI_DUMP_LAYERS 2     /* keep every layer's residual for sarathi_debug_hidden        */
#define SARATHI_LOGITS_HOST 4     /* `logits` is pinned/pageable HOST memory: copy D2H + sync    */
#define SARATHI_NO_LOGITS 8       /* skip final norm + LM head (e.g. non-final prefill chunks)   */

/* Runs one hybrid batch (§4.3): token matrix = [chunk tokens (p) ; decode tokens (d)], T = p + d,
 * 1 <= T <= max_tokens_per_batch.  prefill may be NULL (decode-only batch, the paper's baseline
 * P:L26) and decodes may be NULL or n == 0 (prefill-only batch).
 * logits: fp32 [R][V] (device memory unless SARATHI_LOGITS_HOST), R = d + (prefill ? 1 : 0),
 *   row 0 = the chunk's LAST token, then decodes in decode-set order (reading O-11);
 *   with SARATHI_RETURN_ALL_ROWS, R = T rows in token-matrix order.
 * Effects: K,V of all T tokens appended in place; cached lengths advance by p (chunk) and 1
 *   (each decode).  Under TP the full [R][V] logits are produced on every rank.
 * Errors (state unchanged): EINVAL, EUNKNOWN_REQ, EDUP, EPOS, EOVERFLOW, ESTATE; ECUDA/ENCCL
 *   after enqueue (state undefined). */
int sarathi_run_hybrid_batch(sarathi_model* m, const sarathi_prefill_chunk* prefill, const sarathi_decode_set* decodes,
                             float* logits, int32_t flags);

/* Rolls a request back to new_len cached tokens (new_len <= current cached length); its later KV
 * slots are overwritten by subsequent appends.  Used to replay one fixed batch composition in
 * benchmarks.  EUNKNOWN_REQ, EINVAL. */
int sarathi_request_truncate(sarathi_model* m, int64_t req_id, int32_t new_len);

/* Pipeline parallelism (§3.2 / L1-19 §5.3): a stage > 0 takes
 * its input residual stream from the previous stage.  sarathi_stage_input: h_dev = fp32 [T][H]
 * device memory (the previous stage's sarathi_stage_output, or a copy of it on this device),
 * read by the next run_hybrid_batch (which must carry the same batch).  sarathi_stage_output:
 * this stage's residual stream after its last layer for the last batch (valid until the next run on
 * this handle; TP partials already added).  Stages before the last return no logits.  EINVAL. */
int sarathi_stage_input(sarathi_model* m, const float* h_dev);
int sarathi_stage_output(const sarathi_model* m, const float** h_dev, int32_t* T_out);

/* Bytes the last sarathi_run_hybrid_batch moved host->device (batch metadata: token ids, positions,
 * slots, block tables) and device->host (logits, only with SARATHI_LOGITS_HOST). */
int sarathi_last_io_bytes(const sarathi_model* m, int64_t* h2d, int64_t* d2h);

/* Per-op CUDA-event timers (SURVEY §5 tracing).  When enabled, every kernel group of
 * run_hybrid_batch is bracketed by events on the model stream; sarathi_op_times synchronises the
 * stream and returns the accumulated milliseconds and launch counts per op id since the last
 * reset (reset = 1 clears them after reading).  Op ids: SARATHI_OP_*. */
#define SARATHI_OP_EMBED 0
#define SARATHI_OP_RMSNORM 1
#define SARATHI_OP_GEMM_QKV 2
#define SARATHI_OP_PREFILL_ATTN 3
#define SARATHI_OP_DECODE_ATTN 4
#define SARATHI_OP_GEMM_O 5
#define SARATHI_OP_GEMM_GATE_UP 6
#define SARATHI_OP_GEMM_DOWN 7
#define SARATHI_OP_LM_HEAD 8
#define SARATHI_OP_ALLREDUCE 9
#define SARATHI_OP_OTHER 10
#define SARATHI_OP_GEMM_CHAIN 11
#define SARATHI_NUM_OPS 12
int sarathi_set_profiling(sarathi_model* m, int32_t enable);
int sarathi_op_times(sarathi_model* m, double* ms_out, int64_t* counts_out, int32_t n, int32_t reset);
/* Device spans of the profiled layer GEMMs (QKV, O, gate||up, down) and attention kernels (decode:
 * the main kernel after its grid dependency resolves, not the split combine; prefill: the tcgen05
 * kernel): first CTA start to last CTA end by the SM global timer, i.e. kernel time without launch
 * gaps or event overhead; same accumulate / reset / synchronise semantics as sarathi_op_times (ops
 * without spans read 0). */
int sarathi_op_kernel_times(sarathi_model* m, double* ms_out, int64_t* counts_out, int32_t n, int32_t reset);

/* ---- debug / parity hooks (host outputs, synchronise the stream) ------------------------ */
/* slot mapping of the last batch: out[T] with slot = table[pos / bs] * bs + pos % bs. */
int sarathi_debug_slot_mapping(const sarathi_model* m, int32_t* out, int32_t cap, int32_t* T_out);
/* block table of a request: out[n]. */
int sarathi_debug_block_table(const sarathi_model* m, int64_t req_id, int32_t* out, int32_t cap, int32_t* n_out);
/* residual stream h (fp32 [T][H]) after `layer` (0-based) of the last batch run with
 * SARATHI_DUMP_LAYERS; layer == -1 gives the embedding output (input of layer 0). */
int sarathi_debug_hidden(const sarathi_model* m, int32_t layer, float* host_out);
/* K and V (bf16 bits, [n][n_kv/t][hd] each) of positions pos0..pos0+n-1 of a request, layer l. */
int sarathi_debug_kv(const sarathi_model* m, int32_t layer, int64_t req_id, int32_t pos0, int32_t n,
                     uint16_t* host_k, uint16_t* host_v);
/* Copies `count` bf16 values (bits) of a packed weight tensor, starting at element `offset`, in
 * the packed ROW order of sarathi_init_model (QKV dims permuted inside heads, gate/up interleaved)
 * with the tile-major storage undone. 
 * tensor: 0 qkv, 1 o, 2 gate||up, 3 down, 4 g1, 5 g2 (per layer); 16 emb, 17 final gain, 18 lm head. */
int sarathi_debug_weight(const sarathi_model* m, int32_t layer, int32_t tensor, int64_t offset, int64_t count,
                         uint16_t* host_out);
/* Number of kernels this library launched since the handle was created (gpu_launches). */
int sarathi_launch_count(const sarathi_model* m, int64_t* out);

const char* sarathi_last_error(void);

/* Host-only view of this library's Megatron tensor-parallel sharding (§2.3): for
 * each row r of rank `rank`'s packed tensor (0 qkv, 1 o, 2 gate||up, 3 down, 16 embedding,
 * 18 LM head) of `layer`, the generator tensor id tau[r], fp32 scale[r] and the flat index base[r]
 * of element (r, 0) in the logical unsharded tensor (element (r, c) = base[r] + c).  rows/cols
 * receive the shard shape; tau/scale/base may be NULL (shape query).  No CUDA. */
int sarathi_shard_map(const sarathi_model_config* cfg, int32_t rank, int32_t world, int32_t layer, int32_t tensor,
                      int32_t* tau, float* scale, int64_t* base, int32_t cap, int32_t* rows, int32_t* cols);

/* ---- host-side scheduler (decode-maximal batching, §4.3) — no CUDA --------------------- */
/* Policy (reading O-16): FCFS admission by (arrival, id) while fewer than B requests run and the
 * full (P+D)-token KV reservation fits in the sched's own block allocator (lowest-free-first,
 * same algorithm as the model's); batch = <= 1 chunk of min(C_eff, P - done) from the oldest
 * running request with prefill left (tile_adjust 0: C; 1: the paper's C-(B-1); 2: the B200
 * token-quantum rule sarathi_chunk_advice(C, d, remaining) with d = this batch's decodes) + every
 * decode-phase request in admission order, at most B-1 with a chunk and B without.
 * SARATHI_POLICY_ORCA_BEST: C_eff = the full remaining prompt.
 * SARATHI_POLICY_REQUEST_LEVEL: cohorts; prompts as prefill-only batches, then decode-only. */
#define SARATHI_POLICY_SARATHI 0
#define SARATHI_POLICY_ORCA_BEST 1
#define SARATHI_POLICY_REQUEST_LEVEL 2

typedef struct sarathi_sched sarathi_sched;

typedef struct {
  int32_t iteration;
  int64_t prefill_req; /* -1 if no chunk */
  int32_t prefill_start;
  int32_t prefill_len;
  int32_t n_decodes;
  int32_t n_admitted; /* requests admitted while forming this plan (call request_alloc for them) */
} sarathi_plan;

int sarathi_sched_create(int32_t B, int32_t C, int32_t policy, int32_t tile_adjust, int64_t num_blocks,
                         int32_t block_size, sarathi_sched** out);
void sarathi_sched_destroy(sarathi_sched* s);
/* P >= 1, D >= 0.  EINVAL on duplicate id; ENOKV when ceil((P+D)/block_size) > num_blocks (the
 * request could never be admitted and, under strict FCFS, would block every later request). */
int sarathi_sched_submit(sarathi_sched* s, int64_t req_id, int32_t P, int32_t D, int32_t arrival_iter);
/* Forms the next plan.  Returns 1 with a plan, 0 if idle (nothing eligible this iteration; call
 * sarathi_sched_idle_step), <0 on error.  dec_req[cap], dec_pos[cap], admitted[cap] receive the
 * decode items and newly admitted ids (each at most B entries); EINVAL, with the scheduler
 * unchanged, if cap < B. */
int sarathi_sched_next(sarathi_sched* s, sarathi_plan* plan, int64_t* dec_req, int32_t* dec_pos, int64_t* admitted,
                       int32_t cap);
/* Marks the last plan as executed; finished[cap] receives requests that completed (free their KV;
 * at most B).  EINVAL, with the scheduler unchanged, if finished != NULL and cap < B. */
int sarathi_sched_complete(sarathi_sched* s, int64_t* finished, int32_t cap, int32_t* n_finished);
int sarathi_sched_idle_step(sarathi_sched* s);
int sarathi_sched_done(const sarathi_sched* s, int32_t* done);
int sarathi_sched_block_table(const sarathi_sched* s, int64_t req_id, int32_t* out, int32_t cap, int32_t* n_out);

/* Token tiling of the layer GEMMs for a T-token batch (host only): capacity = token columns the
 * tcgen05 GEMM computes (padding included), n_tiles token tiles, n_mma UMMAs per k-step (1 when a
 * tile holds <= 256 tokens).  n_tiles / n_mma may be NULL. */
int sarathi_token_capacity(int32_t T, int32_t* capacity, int32_t* n_tiles, int32_t* n_mma);
/* B200 chunk advisor (the §4.4 tile-quantization rule, on this GEMM's quanta):
 * with chunk C, d decodes in the batch and `remaining` prompt tokens: p = b - d when C + d overshoots
 * b in {256, 512} by at most C/8, else capacity(C + d) - d; clamped to [1, remaining].  Host only. */
int sarathi_chunk_advice(int32_t C, int32_t d, int32_t remaining, int32_t* p_out);
/* Layer-chain schedule (host only; the work list of the one-launch O -> FFN1 -> FFN2 -> next-QKV
 * GEMM chain, gemm_chain.cu).  Job j has pm_tiles[j] 256-row pair tiles and KB[j] k-blocks of 64;
 * split[j] != 0: a residual-add job (any k-range per segment), else whole tiles only; dep_shift[j]:
 * X k-block kb waits for the previous job's 128-row tile kb >> dep_shift (-1 none); e_done[j],
 * e_add, e_fin: epilogue latencies in k-block units.  Output: seg_off[pairs + 1] and segs[4 * n]
 * (job, pair tile, kb0, kb1) in per-pair execution order (cap = capacity of segs in segments),
 * *n_segs, *makespan (predicted, k-block units).  EINVAL on bad arguments or cap too small. */
int sarathi_chain_schedule(int32_t njobs, const int32_t* pm_tiles, const int32_t* KB, const int32_t* split,
                           const int32_t* dep_shift, const double* e_done, int32_t pairs, double e_add, double e_fin,
                           int32_t* seg_off, int32_t* segs, int32_t cap, int32_t* n_segs, double* makespan);

/* ---- kernel-level entry points (device pointers, caller's stream) for parity tests ------ */
/* out = X · Wᵀ on tcgen05: W bf16 [M][K] (K-major), X bf16 [N][K]; mode 0: out bf16 [N][M],
 * 1: out fp32 [N][M], 2: out fp32 += (residual add), 3: SiLU(gate)·up with gate/up interleaved in
 * 16-row blocks of W (rows 32b..32b+15 gate of features 16b.., next 16 rows their up) -> out bf16
 * [N][M/2], 4: GELU-tanh -> bf16.  K % 64 == 0, M % 8 == 0 (M % 128 == 0 for mode 3), N >= 1.
 * force_splits > 0 fixes the persistent stream-K grid size in CTA pairs (else one pair per 2 SMs).
 * mode | SARATHI_GEMM_W_PACKED: W is already in the tile-major layout of sarathi_op_pack_weight
 * (otherwise it is packed into a library-owned scratch buffer first, on the same stream). */
#define SARATHI_GEMM_W_PACKED 0x100
int sarathi_op_gemm(const void* W, const void* X, void* out, int32_t M, int32_t N, int32_t K, int32_t mode,
                    int32_t force_splits, void* stream);
/* Tile-major GEMM weight layout used by the library: out[ceil(rows/128)*128*cols] with element
 * (r, c) of the row-major W[rows][cols] at
 *     ((r/128)*(cols/64) + c/64)*8192 + (r%128)*64 + (((c%64)/8) ^ (r%8))*8 + c%8
 * (padding rows zero).  Each [128 x 64] tile is 16 KB contiguous and already in the tcgen05 K-major
 * SWIZZLE_128B shared-memory image, tiles ordered as a stream-K CTA consumes them, so one 1D bulk
 * copy (one request) moves a tile HBM -> SMEM.  cols % 64 == 0. */
int sarathi_op_pack_weight(const void* W, void* out, int32_t rows, int32_t cols, void* stream);
/* out[r] = bf16(RMSNorm(h[r]) * g), h fp32 [R][H], g bf16 [H]. */
int sarathi_op_rmsnorm(const float* h, const void* g, void* out, int32_t R, int32_t H, float eps, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SARATHI_H_ */
