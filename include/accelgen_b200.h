/*
 * accelgen_b200.h -- C ABI of the B200 mixed-batch forward (libaccelgen_b200.so).
 *
 * This library replaces ONE call in the reference: the simulated GPU step.  In the reference,
 * engine.step "advance[s] clock by iteration_time(S_f)" where iteration_time is
 * the linear stand-in  T_0 + T_pf * S_f / S_pf  (pkg/src/slosim/cost_model.py:101-109).  Here the
 * BatchPlan that AccelGen's policy packs is executed on the GPU instead:
 * embedding -> L x [LN, QKV(+paged KV append), mixed paged attention, out-proj(+TP all-reduce),
 * LN, FC1+ReLU, FC2(+TP all-reduce)] -> final LN on the logit rows -> LM head -> argmax.
 *
 * Conventions
 *   - Plain C types only; every device buffer is a raw pointer, every stream is a cudaStream_t
 *     passed as void*.  bf16 tensors are uint16-storage bfloat16, row-major.
 *   - Every function returns AG_OK (0) or an AG_E* code; ag_last_error() returns the message
 *     (thread-local).  The Python host maps AG_EINVAL -> ValidationError, AG_EALLOC ->
 *     AllocationError and AG_ECUDA / AG_EFAULT -> EngineFault (pkg/src/slosim/errors.py:16-32).
 *   - KV pool layout per layer and per K/V: [num_blocks][heads_local][block_size=32][head_dim=128]
 *     bf16; block ids are the physical ids assigned by the scheduler's BlockPool
 *     (the reference tracks counts only, pkg/src/slosim/kvc.py:42-45).
 */
#ifndef ACCELGEN_B200_H_
#define ACCELGEN_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define AG_API __attribute__((visibility("default")))
#else
#define AG_API
#endif

#define AG_OK 0
#define AG_EINVAL 1  /* bad argument / shape */
#define AG_ECUDA 2   /* CUDA runtime or launch error */
#define AG_EALLOC 3  /* capacity exceeded (tokens, sequences, workspace) */
#define AG_EFAULT 4  /* internal invariant violation (reference: EngineFault, errors.py:28-32) */
#define AG_ENCCL 5   /* NCCL error (tensor parallel) */
#define AG_ESTATE 6  /* call-order violation, e.g. a third asynchronous step (reference: StateError, errors.py:24) */

typedef struct ag_model ag_model; /* opaque */

/* Kernel classes of one forward, for ag_model_get_profile. */
enum {
  AG_K_EMBED = 0,
  AG_K_LAYERNORM,
  AG_K_QKV_GEMM,
  AG_K_ATTENTION,
  AG_K_OUT_GEMM,
  AG_K_FC1_GEMM,
  AG_K_FC2_GEMM,
  AG_K_LMHEAD_GEMM,
  AG_K_ARGMAX,
  AG_K_ALLREDUCE,
  AG_PROF_CLASSES
};

/* Model shape and capacities.  Mirrors the reference ModelProfile's shape fields
 * (cost_model.py:34-58: hidden_size, num_layers, bytes_per_element) plus the OPT architecture
 * constants the cost model folds away. */
typedef struct {
  int32_t hidden;          /* H (5120 for OPT-13B) */
  int32_t num_layers;      /* L */
  int32_t num_heads;       /* total heads; head_dim = hidden / num_heads must be 128 */
  int32_t ffn;             /* FC1 width (4H) */
  int32_t vocab;           /* V (50272) */
  int32_t pos_rows;        /* rows of the learned position table (incl. OPT offset 2) */
  int32_t tp_rank;
  int32_t tp_size;         /* 1, 2, 4, 8: heads, ffn and vocab must divide */
  int32_t num_blocks;      /* KV pool blocks (kvc_capacity_tokens // 32, kvc.py:47-50) */
  int32_t block_size;      /* 32 (kvc.py:16) */
  int32_t max_tokens;      /* max forward size S_f per step */
  int32_t max_seqs;        /* max sequences per step */
  int32_t max_blocks_per_seq; /* block-table row stride */
  float ln_eps;            /* 1e-5 */
} ag_model_config;

/* Per-layer weights (device pointers, bf16, nn.Linear layout [out, in]); this rank's shard. */
typedef struct {
  const void* ln1_g; const void* ln1_b;     /* [H] */
  const void* qkv_w; const void* qkv_b;     /* [3*Hl, H], [3*Hl]   (q | k | v, Hl = H/tp) */
  const void* out_w; const void* out_b;     /* [H, Hl], [H] */
  const void* ln2_g; const void* ln2_b;     /* [H] */
  const void* fc1_w; const void* fc1_b;     /* [F/tp, H], [F/tp] */
  const void* fc2_w; const void* fc2_b;     /* [H, F/tp], [H] */
} ag_layer_weights;

/* One iteration's packed BatchPlan (HOST pointers).  B sequences; sequence b contributes
 * q_b = cu_q[b+1]-cu_q[b] new tokens (a prompt chunk, or one decode token)
 * on top of ctx_len[b] tokens already in its KV blocks. */
typedef struct {
  int32_t num_tokens;           /* S_f = sum of chunk lengths */
  int32_t num_seqs;             /* B */
  int32_t num_logits;           /* rows that emit a token (final chunks + TG steps) */
  int32_t block_table_stride;   /* >= max blocks of any sequence, <= max_blocks_per_seq */
  const int32_t* token_ids;     /* [S_f] */
  const int32_t* positions;     /* [S_f] absolute positions (0-based) */
  const int32_t* cu_q;          /* [B+1] */
  const int32_t* ctx_len;       /* [B] */
  const int32_t* block_table;   /* [B, stride] physical block ids */
  const int32_t* slot_mapping;  /* [S_f] block*32+offset of each new token's KV slot */
  const int32_t* logit_rows;    /* [num_logits] token rows whose logits are needed */
} ag_step;

AG_API const char* ag_last_error(void);
AG_API int32_t ag_version(void);
AG_API int32_t ag_device_sm_count(void);

/* ---- model lifecycle (reference boundary: engine.step's clock advance) ---- */
/* Environment: AG_DETERMINISTIC=1 (read at create) disables the fp32-atomic split-K / stream-K
 * epilogues, so every result is bitwise reproducible run to run; AG_DEBUG_SYNC=1 synchronises and
 * checks after every launch of the forward; AG_PDL=0 launches the forward's kernels without
 * programmatic dependent launch (default on: a kernel's prologue and weight prefetch overlap its
 * predecessor's tail; AG_PDL_MASK=<bits> per launch class, see common.cuh). */
AG_API int32_t ag_model_create(const ag_model_config* cfg, ag_model** out);
AG_API void ag_model_destroy(ag_model* m);
AG_API int32_t ag_model_set_embeddings(ag_model* m, const void* tok_emb /*[V,H]*/, const void* pos_emb /*[pos_rows,H]*/,
                                const void* final_ln_g, const void* final_ln_b);
AG_API int32_t ag_model_set_layer(ag_model* m, int32_t layer, const ag_layer_weights* w);
AG_API int32_t ag_model_set_kv_cache(ag_model* m, int32_t layer, void* k_pool, void* v_pool);
/* Tensor parallel: rank 0 calls ag_nccl_get_unique_id, the 128 bytes are broadcast by the host,
 * then every rank calls ag_model_init_tp (NCCL communicator over NVLink, in-stream all-reduce). */
AG_API int32_t ag_nccl_get_unique_id(void* out_128_bytes);
AG_API int32_t ag_model_init_tp(ag_model* m, const void* unique_id_128_bytes);
/* Host collective backend (instead of ag_model_init_tp): every collective of the forward is copied
 * D2H into a pinned staging buffer, the stream is synchronised, and `fn` completes it in place on
 * that host buffer; the result is copied back H2D.  op AG_COLL_ALLREDUCE_SUM: `count` elements of
 * `dtype` summed over ranks in place.  op AG_COLL_ALLGATHER: the buffer holds tp_size slots of
 * `count` elements, this rank's slot (index tp_rank) filled; fn fills the others.  fn returns 0 on
 * success.  Used to run several TP ranks as processes sharing ONE GPU (NCCL refuses two ranks on a
 * device), so the sharded forward -- head-split attention, bias-after-reduce LayerNorm, the
 * vocab-parallel argmax merge -- is testable on a single B200; not a performance path. */
#define AG_COLL_ALLREDUCE_SUM 0
#define AG_COLL_ALLGATHER 1
#define AG_DT_BF16 0
#define AG_DT_F32 1
#define AG_DT_I32 2
typedef int32_t (*ag_host_collective_fn)(void* ctx, int32_t op, void* host_buf, int64_t count, int32_t dtype);
AG_API int32_t ag_model_init_tp_host(ag_model* m, ag_host_collective_fn fn, void* ctx);

/* Execute one BatchPlan.  Host metadata is packed into one pinned buffer, copied H2D on
 * `stream`, the forward runs, and next-token ids are copied back into out_tokens (host, int32
 * [num_logits]).  If logits_out (device, f32 [num_logits, vocab/tp]) is non-null the local logit
 * shard is also written (parity mode).  device_ms (optional) receives the CUDA-event time of the
 * forward alone (metadata already resident, before the D2H).  Synchronises `stream`. */
AG_API int32_t ag_model_forward(ag_model* m, const ag_step* step, int32_t* out_tokens, float* logits_out,
                         float* device_ms, void* stream);

/* Asynchronous steps (the host plans step k+1 while the GPU runs step k).  ag_model_submit validates
 * and stages the step like ag_model_forward, enqueues the forward and the D2H of its next-token ids on
 * `stream` and returns; at most two steps are in flight.  feed_pairs = n_feed (token index, logit row)
 * int32 pairs: decode token `token index` of this step takes the next-token id that the PREVIOUS
 * submitted step emits at `logit row` (autoregressive input resolved on the device, no host round
 * trip).  ag_model_wait completes the oldest step in flight: its ids into out_tokens (cap entries),
 * its CUDA-event forward time, and the time of its last kernel in ms after the ag_model_clock_ref
 * event (which records an event on `stream` and waits for it, so the host can map device completion
 * times onto its own clock).  Replaces the same clock advance as ag_model_forward. */
AG_API int32_t ag_model_submit(ag_model* m, const ag_step* step, const int32_t* feed_pairs, int32_t n_feed,
                               float* logits_out, void* stream);
AG_API int32_t ag_model_wait(ag_model* m, int32_t* out_tokens, int32_t cap, float* device_ms,
                             double* end_ms_since_ref);
AG_API int32_t ag_model_clock_ref(ag_model* m, void* stream);
AG_API int32_t ag_model_inflight(ag_model* m);

/* Same forward, asynchronous, with all metadata already packed in device memory by
 * ag_model_stage_step (used to time the kernels with inputs resident in HBM). */
AG_API int32_t ag_model_stage_step(ag_model* m, const ag_step* step, void* stream);
AG_API int32_t ag_model_forward_staged(ag_model* m, int32_t* out_tokens_dev, float* logits_out, void* stream);

/* Time every candidate (BLOCK_N, K-split) plan of the model's GEMM shapes (QKV, out, FC1, FC2,
 * LM head) over M buckets up to max_tokens on this GPU and keep the fastest; later forwards use
 * the table.  ~1 s at model load.  get_gemm_plans writes (kind, m_bucket, block_n, k_splits) rows. */
AG_API int32_t ag_model_autotune(ag_model* m, void* stream);
AG_API int32_t ag_model_get_gemm_plans(ag_model* m, int32_t* out_rows4, int32_t cap);
/* Install a plan table previously read with get_gemm_plans (same rows; replaces autotune). */
AG_API int32_t ag_model_set_gemm_plans(ag_model* m, const int32_t* rows4, int32_t n);

/* Per-kernel-class CUDA-event profiling of ag_model_forward (on = 1 resets the counters).
 * get_profile fills up to n entries per class: summed ms, algorithmic FLOPs and HBM bytes, launches. */
AG_API int32_t ag_model_set_profiling(ag_model* m, int32_t on);
AG_API int32_t ag_model_get_profile(ag_model* m, double* ms, double* flops, double* bytes, int64_t* counts, int32_t n);
/* Roofline accounting: with peaks set, every profiled launch adds
 * max(FLOPs / tensor peak, algorithmic bytes / HBM peak) to its class; get_roofline_ms returns the
 * per-class sums, so sum(roofline) / sum(measured) is the class's fraction of its roofline. */
AG_API int32_t ag_model_set_roofline_peaks(ag_model* m, double tensor_tflops, double hbm_gbs);
AG_API int32_t ag_model_get_roofline_ms(ag_model* m, double* roof_ms, int32_t n);
/* Kernel launches issued by the last forward (ours only; NCCL calls counted as AG_K_ALLREDUCE). */
AG_API int64_t ag_model_last_launches(ag_model* m);
/* Bytes of packed metadata (BatchPlan arrays + attention work list) copied H2D by the last step. */
AG_API int64_t ag_model_last_h2d_bytes(ag_model* m);

/* ---- individual kernels (device pointers), for parity tests and the profiler ---- */
/* D[M,N] = A[M,K] . W[N,K]^T (+bias[N]) (+residual[M,ldr]) (ReLU); bf16 out unless out_f32.
 * block_n in {0 (auto), 64, 128, 256}; k_splits 0 = auto (uses workspace, fp32 k_splits*M*N);
 * a_rows in {0/128, 64, 32}: activation rows staged per k-block (small-M variant needs M <= a_rows). */
AG_API int32_t ag_gemm_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, const void* bias,
                     const void* residual, int32_t ldr, int32_t relu, void* D, int32_t ldd, int32_t out_f32,
                     int32_t M, int32_t N, int32_t K, int32_t block_n, int32_t k_splits, int32_t a_rows,
                     void* workspace, int64_t workspace_bytes, void* stream);
/* Paged KV append: rows of k/v ([rows, heads*128], row stride ld) into their slots. */
AG_API int32_t ag_kv_append(const void* k, const void* v, int32_t ld, const int32_t* slot_mapping, int32_t rows,
                     int32_t heads, int32_t block_size, void* k_pool, void* v_pool, void* stream);
/* Mixed paged attention over B sequences (q already scaled by head_dim^-0.5).  cu_q/ctx_len are
 * given on both host (work-list construction) and device; pool_blocks = blocks in each pool. */
AG_API int32_t ag_paged_attention(const void* q, int32_t ldq, const void* k_pool, const void* v_pool,
                           int32_t pool_blocks, const int32_t* block_table_dev, int32_t bt_stride, const int32_t* cu_q_host,
                           const int32_t* ctx_len_host, const int32_t* cu_q_dev, const int32_t* ctx_len_dev,
                           int32_t num_seqs, int32_t heads, int32_t block_size, void* out, int32_t ldo,
                           void* workspace, int64_t workspace_bytes, void* stream);
AG_API int32_t ag_layernorm(void* x, const void* delta, const void* delta_bias, const int32_t* row_index,
                     const void* gamma, const void* beta, float eps, int32_t rows, int32_t hidden, void* out,
                     void* stream);
/* Llama-family variants (north_star kernel list; not on the OPT path, which uses LayerNorm and
 * learned positions): RMSNorm with optional in-place residual add, and rotary embedding in place
 * (rotate-half convention over the first rotary_dim dims of each head, angle pos * theta^(-2i/d)). */
AG_API int32_t ag_rmsnorm(void* x, const void* delta, const void* gamma, float eps, int32_t rows, int32_t hidden,
                   void* out, void* stream);
AG_API int32_t ag_rope(void* x, int32_t ld, const int32_t* positions, int32_t rows, int32_t heads, int32_t head_dim,
                int32_t rotary_dim, float theta, void* stream);
AG_API int32_t ag_embed_pos(const int32_t* ids, const int32_t* positions, const void* tok_emb, const void* pos_emb,
                     int32_t pos_offset, int32_t rows, int32_t hidden, int32_t vocab, int32_t pos_rows,
                     void* out, void* stream);
AG_API int32_t ag_argmax(const float* logits, int32_t rows, int32_t cols, int32_t ld, int32_t index_offset,
                  float* out_val, int32_t* out_idx, void* stream);
/* Preemption swap (reference BlockPool.preempt / demand_readmit, kvc.py:110-116,153-160):
 * gather blocks of one pool into a contiguous buffer (swap out) or scatter them back (swap in). */
AG_API int32_t ag_kv_swap_out(const void* pool, const int32_t* block_ids_dev, int32_t n_blocks, int64_t block_elems,
                       void* staging, void* stream);
AG_API int32_t ag_kv_swap_in(const void* staging, const int32_t* block_ids_dev, int32_t n_blocks, int64_t block_elems,
                      void* pool, void* stream);
/* The same over `planes` planes in one launch (every layer's K and V of a [L, 2, blocks, ...] pool):
 * plane p of the pool starts at p * pool_plane_elems, of the staging buffer at p * stage_plane_elems. */
AG_API int32_t ag_kv_swap_out_planes(const void* pool, int64_t pool_plane_elems, const int32_t* block_ids_dev,
                              int32_t n_blocks, int64_t block_elems, void* staging, int64_t stage_plane_elems,
                              int32_t planes, void* stream);
AG_API int32_t ag_kv_swap_in_planes(const void* staging, int64_t stage_plane_elems, const int32_t* block_ids_dev,
                             int32_t n_blocks, int64_t block_elems, void* pool, int64_t pool_plane_elems,
                             int32_t planes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ACCELGEN_B200_H_ */
