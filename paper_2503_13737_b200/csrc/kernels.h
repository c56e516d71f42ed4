// Internal (C++) declarations shared by the kernel translation units and the C-ABI layer.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ag {

// kEpiAtomicF32: every K split adds its fp32 tile into acc32 (red.global.add.v4.f32, no bias /
// residual / conversion here); the consumer (layernorm with an fp32 delta) finishes the epilogue
// and re-zeroes acc32.  Lets out-proj / FC2 split K across all SMs with no reduce launch.
enum EpiMode : int { kEpiPlain = 0, kEpiQkv = 1, kEpiAtomicF32 = 2 };

struct GemmEpilogue {
  int mode = kEpiPlain;
  const __nv_bfloat16* bias = nullptr;      // [N] or null
  const __nv_bfloat16* residual = nullptr;  // [M, ldr] or null (plain mode)
  int ldr = 0;
  int relu = 0;
  void* out = nullptr;  // bf16 (or f32 when out_f32) [M, ldc]; q output in QKV mode
  int ldc = 0;
  int out_f32 = 0;
  // QKV mode: columns [0,hq) -> q (scaled), [hq,2hq) -> K cache, [2hq,3hq) -> V cache
  int hq = 0;
  float q_scale = 1.0f;
  __nv_bfloat16* kcache = nullptr;  // [num_blocks, heads, block_size, head_dim]
  __nv_bfloat16* vcache = nullptr;
  const int32_t* slot_mapping = nullptr;  // [M]; <0 = skip
  int heads = 0;
  int head_dim = 128;
  int block_size = 32;
  float* acc32 = nullptr;  // [M, ldc] fp32 (kEpiAtomicF32)
  // Fused LayerNorm (TP=1; ln_out != null enables it; ln_bar: 2 words, zero-initialised, one per
  // model/stream).  Every CTA finishes rows blockIdx.x, +gridDim.x, ... of
  //   ln_x[r] = bf16(ln_x[r] + (ln_acc[r] + ln_bias));  ln_acc[r] = 0;  ln_out[r] = LN(ln_x[r]) * ln_g + ln_b
  // -- what launch_layernorm_acc does as its own launch.  Tail (ln_prologue = 0; kEpiAtomicF32 with
  // ln_acc = acc32): after this GEMM's reductions, behind a grid barrier.  Prologue (ln_prologue = 1):
  // before this GEMM loads any A tile (ln_out is its A operand; ln_acc holds the predecessor's
  // reductions), while its first weight stages are in flight.
  int ln_prologue = 0;
  float* ln_acc = nullptr;
  int ln_ld = 0;
  __nv_bfloat16* ln_x = nullptr;
  const __nv_bfloat16* ln_bias = nullptr;
  const __nv_bfloat16* ln_g = nullptr;
  const __nv_bfloat16* ln_b = nullptr;
  float ln_eps = 1e-5f;
  __nv_bfloat16* ln_out = nullptr;
  unsigned int* ln_bar = nullptr;
};

int make_tmap_kmajor(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld_elems,
                     int box_rows);
int num_sms();
int pick_block_n(int M, int N);
// k_splits > 1 writes fp32 partials to `partial` (k_splits * M * N floats) and a reduce kernel
// applies the epilogue; choose (bn, k_splits) with plan_gemm.
// am = activation rows loaded per stage (128; or 32/64 for the small-M variant, which needs M <= am
// and an A tensor map whose box has `am` rows).  am = 256 selects the CTA-pair kernel (256 x bn
// tiles, bn in {128, 256}): then ta's box has 128 rows and tb's box bn/2 rows.
cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int bn,
                        const GemmEpilogue& ep, int max_ctas, cudaStream_t stream, int k_splits = 1,
                        float* partial = nullptr, int am = 128);
// k_splits == kStreamK: stream-K over all SMs (1-CTA kernel, kEpiAtomicF32 epilogue only).
constexpr int kStreamK = 99;
struct GemmPlan {
  int bn;
  int k_splits;
  int am = 128;
};
GemmPlan plan_gemm(int M, int N, int K, int64_t partial_capacity_floats);
// CTAs launch_gemm starts for this plan (max_ctas = 0)
int gemm_grid(int M, int N, int K, int bn, int k_splits, int am);
// Apply `ep` to a stream-K fp32 accumulator acc[M, N] (atomically filled) and re-zero it.
cudaError_t launch_splitk_finish(float* acc, int M, int N, const GemmEpilogue& ep, cudaStream_t stream);

// embed: out[r] = tok_emb[ids[r]] + pos_emb[positions[r] + pos_offset]
cudaError_t launch_feed_tokens(int32_t* ids, const int32_t* pairs, int n, const int32_t* prev_out,
                               cudaStream_t stream);
cudaError_t launch_embed(const int32_t* ids, const int32_t* positions, const __nv_bfloat16* tok_emb,
                         const __nv_bfloat16* pos_emb, int pos_offset, int rows, int hidden,
                         int vocab, int max_pos_rows, __nv_bfloat16* out, cudaStream_t stream);

// layernorm over rows of x (optionally gathered through row_index), fp32 statistics.
// If delta != null: x[r] = x[r] + delta[r] (+ delta_bias) is written back first (residual add).
cudaError_t launch_layernorm(__nv_bfloat16* x, const __nv_bfloat16* delta,
                             const __nv_bfloat16* delta_bias, const int32_t* row_index,
                             const __nv_bfloat16* gamma, const __nv_bfloat16* beta, float eps,
                             int rows, int hidden, __nv_bfloat16* out, cudaStream_t stream);

// Same, with the residual delta in fp32 (a kEpiAtomicF32 GEMM's accumulator) plus bias: x[src] =
// bf16(x[src] + acc32[src] + bias) for the normalised rows; acc32 rows read are zeroed again.
cudaError_t launch_layernorm_acc(__nv_bfloat16* x, float* acc32, const __nv_bfloat16* delta_bias,
                                 const int32_t* row_index, const __nv_bfloat16* gamma, const __nv_bfloat16* beta,
                                 float eps, int rows, int hidden, __nv_bfloat16* out, cudaStream_t stream);

// RMSNorm over rows (hidden <= 5120), optional in-place residual add x += delta first.
cudaError_t launch_rmsnorm(__nv_bfloat16* x, const __nv_bfloat16* delta, const __nv_bfloat16* gamma, float eps,
                           int rows, int hidden, __nv_bfloat16* out, cudaStream_t stream);

// Rotary embedding in place on [rows, heads*head_dim] (rotate-half convention, first rotary_dim dims).
cudaError_t launch_rope(__nv_bfloat16* x, int ld, const int32_t* positions, int rows, int heads, int head_dim,
                        int rotary_dim, float theta, cudaStream_t stream);

// standalone paged KV append: k/v rows [rows, heads*head_dim] -> cache slots
cudaError_t launch_kv_append(const __nv_bfloat16* k, const __nv_bfloat16* v, int ld_src,
                             const int32_t* slot_mapping, int rows, int heads, int head_dim,
                             int block_size, __nv_bfloat16* kcache, __nv_bfloat16* vcache,
                             cudaStream_t stream);

// Work item of the mixed paged attention (host-built).
struct AttnItem {
  int32_t seq;        // sequence index
  int32_t q_start;    // first query row inside the sequence's q chunk
  int32_t q_rows;     // rows of this tile (<= 64)
  int32_t kv_start;   // first kv position (inclusive)
  int32_t kv_end;     // last kv position (exclusive), already clipped by causality
  int32_t part_row;   // >=0: row base into the split-KV partial buffers; -1: write final output
  int32_t pad0, pad1;
};

struct AttnCombine {  // one query row whose KV range was split
  int32_t tok_row;    // global token row
  int32_t q_rows;     // rows of the split piece: split s of this row is part_row first_part + s * q_rows
  int32_t first_part; // part_row of split 0
  int32_t n_splits;
};

struct AttnParams {
  const __nv_bfloat16* q;  // [S_f, heads*head_dim] (already scaled)
  int ldq;
  const __nv_bfloat16* kcache;
  const __nv_bfloat16* vcache;
  const int32_t* block_table;  // [B, bt_stride]
  int bt_stride;
  const int32_t* cu_q;     // [B+1]
  const int32_t* ctx_len;  // [B] cached prefix length before this step
  __nv_bfloat16* out;      // [S_f, heads*head_dim]
  int ldo;
  float* part_o;           // [P, heads, head_dim]
  float* part_ml;          // [P, heads, 2]
  int heads;
  int block_size;
};

// TMA maps of the tile path: q over [rows, heads*128] (box 64 x 128 rows), k/v over the pool
// viewed as [num_blocks*heads*32, 128] (box 64 x 32 rows = half a page row-block).
struct AttnTmaps {
  CUtensorMap q, k, v;
};
int attention_tile_rows();  // query rows per tcgen05 tile (128)
int attention_tile_kv();    // kv tokens per tile stage (128)
// items = [n_tile_items query tiles (tcgen05)] + [n_row_items single-row items (warp streaming)]
cudaError_t launch_attention(const AttnParams& p, const AttnTmaps& tm, const AttnItem* items, int n_tile_items,
                             int n_row_items, const AttnCombine* combines, int n_combines, cudaStream_t stream);

// argmax over rows of logits (f32), optional vocab offset; writes (value, index) pairs
cudaError_t launch_argmax(const float* logits, int rows, int cols, int ld, int index_offset,
                          float* out_val, int32_t* out_idx, cudaStream_t stream);

// merge per-rank (value,index) candidates [tp, rows] -> index [rows]
cudaError_t launch_argmax_merge(const float* vals, const int32_t* idx, int tp, int rows,
                                int32_t* out_idx, cudaStream_t stream);

// gather block rows: dst[i] = src[index[i]] (bf16 rows of width cols)
cudaError_t launch_gather_rows(const __nv_bfloat16* src, int ld_src, const int32_t* index, int rows,
                               int cols, __nv_bfloat16* dst, int ld_dst, cudaStream_t stream);

// KV block swap: gather=true copies pool[block_ids[i]] -> dst[i] (contiguous staging);
// gather=false copies src[i] -> dst[block_ids[i]] (staging back into the pool).  planes > 1 repeats it
// for plane p at element offsets p * pool_plane (pool) and p * stage_plane (staging): every layer's K and
// V in one launch.
cudaError_t launch_block_copy(const __nv_bfloat16* src, __nv_bfloat16* dst, const int32_t* block_ids,
                              int n_blocks, int64_t block_elems, bool gather, cudaStream_t stream, int planes = 1,
                              int64_t pool_plane = 0, int64_t stage_plane = 0);

// pseudo-random bf16 fill (autotune activations): scale * U[-1, 1), optionally ReLU'd
cudaError_t launch_fill_hash(__nv_bfloat16* x, int64_t n, uint32_t seed, float scale, bool relu,
                             cudaStream_t stream);

}  // namespace ag
