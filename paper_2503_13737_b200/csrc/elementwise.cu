// HBM-bound helper kernels of the mixed-batch forward: embedding gather, residual+LayerNorm,
// standalone paged KV append, row gather, vocab argmax (+ cross-rank merge), KV-block swap copies.
// All use 16-byte vector accesses with consecutive threads on consecutive addresses.
#include "common.cuh"
#include "kernels.h"

namespace ag {

namespace {

AG_DEVICE void bf16x8_to_f32(const uint4& w, float (&f)[8]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    float2 p = unpack_bf16x2(ws[h]);
    f[2 * h] = p.x;
    f[2 * h + 1] = p.y;
  }
}

AG_DEVICE uint4 f32_to_bf16x8(const float (&f)[8]) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                    pack_bf16x2(f[6], f[7]));
}

__global__ void embed_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ positions,
                             const __nv_bfloat16* __restrict__ tok_emb,
                             const __nv_bfloat16* __restrict__ pos_emb, int pos_offset, int rows,
                             int hidden, int vocab, int max_pos_rows, __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int vec_per_row = hidden / 8;
  const int64_t total = static_cast<int64_t>(rows) * vec_per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i - static_cast<int64_t>(r) * vec_per_row);
    int tok = ids[r];
    tok = tok < 0 ? 0 : (tok >= vocab ? vocab - 1 : tok);
    int pos = positions[r] + pos_offset;
    pos = pos < 0 ? 0 : (pos >= max_pos_rows ? max_pos_rows - 1 : pos);
    float a[8], b[8];
    bf16x8_to_f32(ld_global_nc_v4(tok_emb + static_cast<int64_t>(tok) * hidden + v * 8), a);
    bf16x8_to_f32(ld_global_nc_v4(pos_emb + static_cast<int64_t>(pos) * hidden + v * 8), b);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += b[j];
    *reinterpret_cast<uint4*>(out + static_cast<int64_t>(r) * hidden + v * 8) = f32_to_bf16x8(a);
  }
}

template <int kThreadsLN>
AG_DEVICE float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int i = 0; i < kThreadsLN / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

constexpr int kLNThreads = 128;
constexpr int kLNMaxVec = 12;  // hidden <= 12288

__global__ void __launch_bounds__(kLNThreads)
    layernorm_kernel(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                     const __nv_bfloat16* __restrict__ delta_bias, const int32_t* __restrict__ row_index,
                     const __nv_bfloat16* __restrict__ gamma, const __nv_bfloat16* __restrict__ beta,
                     float eps, int hidden, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();  // after the wait: an early norm never lets a third kernel in
  __shared__ float red[kLNThreads / 32];
  const int r = blockIdx.x;
  const int src = row_index ? row_index[r] : r;
  __nv_bfloat16* xr = x + static_cast<int64_t>(src) * hidden;
  const int nvec = hidden / 8;
  float vals[kLNMaxVec][8];
  float sum = 0.0f;
#pragma unroll
  for (int i = 0; i < kLNMaxVec; ++i) {
    const int idx = threadIdx.x + i * kLNThreads;
    if (idx < nvec) {
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(xr + idx * 8), vals[i]);
      if (delta != nullptr) {
        float d[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(delta + static_cast<int64_t>(src) * hidden + idx * 8), d);
        if (delta_bias != nullptr) {
          float bb[8];
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(delta_bias + idx * 8), bb);
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] += bb[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) vals[i][j] += d[j];
        const uint4 packed = f32_to_bf16x8(vals[i]);
        *reinterpret_cast<uint4*>(xr + idx * 8) = packed;  // updated residual stream
        bf16x8_to_f32(packed, vals[i]);                    // normalise the rounded value
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sum += vals[i][j];
    }
  }
  const float mean = block_sum<kLNThreads>(sum, red) / hidden;
  float sq = 0.0f;
#pragma unroll
  for (int i = 0; i < kLNMaxVec; ++i) {
    const int idx = threadIdx.x + i * kLNThreads;
    if (idx < nvec) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float c = vals[i][j] - mean;
        sq += c * c;
      }
    }
  }
  const float var = block_sum<kLNThreads>(sq, red) / hidden;
  const float rstd = rsqrtf(var + eps);
  __nv_bfloat16* orow = out + static_cast<int64_t>(r) * hidden;
#pragma unroll
  for (int i = 0; i < kLNMaxVec; ++i) {
    const int idx = threadIdx.x + i * kLNThreads;
    if (idx < nvec) {
      float g[8], b[8], y[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + idx * 8), g);
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(beta + idx * 8), b);
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = (vals[i][j] - mean) * rstd * g[j] + b[j];
      *reinterpret_cast<uint4*>(orow + idx * 8) = f32_to_bf16x8(y);
    }
  }
}

// Row-per-block LayerNorm with 2 vectors (16 values) per thread: hidden/16 threads (320 for OPT-13B)
// so the whole row is one load round trip and the per-thread work is tiny; two block reductions
// (warp shuffles + one smem exchange each).  For hidden <= 16384.
constexpr int kLNVpt = 2;
constexpr int kLNWarpVec = 20;  // RMSNorm warp-per-row capacity (hidden <= 5120)
constexpr int kLNWarpsPerBlock = 8;

AG_DEVICE float block_sum_dyn(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = 0.0f;
  for (int i = 0; i < nw; ++i) t += red[i];
  __syncthreads();
  return t;
}

template <typename DeltaT>
__global__ void __launch_bounds__(1024)
    layernorm_row_kernel(__nv_bfloat16* __restrict__ x, DeltaT* __restrict__ delta,
                         const __nv_bfloat16* __restrict__ delta_bias, const int32_t* __restrict__ row_index,
                         const __nv_bfloat16* __restrict__ gamma, const __nv_bfloat16* __restrict__ beta,
                         float eps, int hidden, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();  // after the wait: an early norm never lets a third kernel in
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int src = row_index ? row_index[r] : r;
  __nv_bfloat16* xr = x + static_cast<int64_t>(src) * hidden;
  const int nvec = hidden / 8;
  float v[kLNVpt][8];
  float sum = 0.0f;
#pragma unroll
  for (int i = 0; i < kLNVpt; ++i) {
    const int idx = threadIdx.x + i * blockDim.x;
    if (idx < nvec) {
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(xr + idx * 8), v[i]);
      if (delta != nullptr) {
        float d[8];
        if constexpr (sizeof(DeltaT) == 4) {  // fp32 split-K accumulator: read, then re-zero
          float4* d4 = reinterpret_cast<float4*>(delta + static_cast<int64_t>(src) * hidden + idx * 8);
          const float4 a = __ldcg(d4), b = __ldcg(d4 + 1);
          d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
          d4[0] = make_float4(0.f, 0.f, 0.f, 0.f);
          d4[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(delta + static_cast<int64_t>(src) * hidden + idx * 8), d);
        }
        if (delta_bias != nullptr) {
          float bb[8];
          bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(delta_bias) + idx), bb);
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] += bb[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i][j] += d[j];
        const uint4 packed = f32_to_bf16x8(v[i]);
        *reinterpret_cast<uint4*>(xr + idx * 8) = packed;  // updated residual stream
        bf16x8_to_f32(packed, v[i]);                       // normalise the rounded value
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sum += v[i][j];
    }
  }
  const float mean = block_sum_dyn(sum, red) / hidden;
  float sq = 0.0f;
#pragma unroll
  for (int i = 0; i < kLNVpt; ++i)
    if (threadIdx.x + i * blockDim.x < nvec)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float c = v[i][j] - mean;
        sq += c * c;
      }
  const float rstd = rsqrtf(block_sum_dyn(sq, red) / hidden + eps);
  __nv_bfloat16* orow = out + static_cast<int64_t>(r) * hidden;
#pragma unroll
  for (int i = 0; i < kLNVpt; ++i) {
    const int idx = threadIdx.x + i * blockDim.x;
    if (idx < nvec) {
      float g[8], b[8], y[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(gamma) + idx), g);
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(beta) + idx), b);
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = (v[i][j] - mean) * rstd * g[j] + b[j];
      *reinterpret_cast<uint4*>(orow + idx * 8) = f32_to_bf16x8(y);
    }
  }
}

// RMSNorm (Llama-family variants of the served model): warp per row, optional in-place residual add.
//   x[r] += delta[r] (rounded to bf16, written back);  out[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * gamma
__global__ void __launch_bounds__(kLNWarpsPerBlock * 32)
    rmsnorm_warp_kernel(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                        const __nv_bfloat16* __restrict__ gamma, float eps, int rows, int hidden,
                        __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();  // after the wait: an early norm never lets a third kernel in
  const int r = blockIdx.x * kLNWarpsPerBlock + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  __nv_bfloat16* xr = x + static_cast<int64_t>(r) * hidden;
  const int nvec = hidden / 8;
  float vals[kLNWarpVec][8];
  float sq = 0.0f;
#pragma unroll
  for (int i = 0; i < kLNWarpVec; ++i) {
    const int idx = lane + i * 32;
    if (idx < nvec) {
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(xr + idx * 8), vals[i]);
      if (delta != nullptr) {
        float d[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(delta + static_cast<int64_t>(r) * hidden + idx * 8), d);
#pragma unroll
        for (int j = 0; j < 8; ++j) vals[i][j] += d[j];
        const uint4 packed = f32_to_bf16x8(vals[i]);
        *reinterpret_cast<uint4*>(xr + idx * 8) = packed;
        bf16x8_to_f32(packed, vals[i]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sq += vals[i][j] * vals[i][j];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rstd = rsqrtf(sq / hidden + eps);
  __nv_bfloat16* orow = out + static_cast<int64_t>(r) * hidden;
#pragma unroll
  for (int i = 0; i < kLNWarpVec; ++i) {
    const int idx = lane + i * 32;
    if (idx < nvec) {
      float g[8], y[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(gamma) + idx), g);
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = vals[i][j] * rstd * g[j];
      *reinterpret_cast<uint4*>(orow + idx * 8) = f32_to_bf16x8(y);
    }
  }
}

// Rotary position embedding, in place on [rows, heads * head_dim] bf16 (q or k), rotate-half
// (GPT-NeoX / Llama) convention over the first rotary_dim dims of every head:
//   (x1, x2) <- (x1 cos - x2 sin, x2 cos + x1 sin),  angle = pos * theta^(-2i / rotary_dim).
// One thread per (row, head, pair of 2 x 4 dims): 8-B vector loads/stores of both halves.
__global__ void rope_kernel(__nv_bfloat16* __restrict__ x, int ld, const int32_t* __restrict__ positions, int rows,
                            int heads, int head_dim, int rotary_dim, float log2_theta) {
  pdl_trigger();
  pdl_wait();
  const int half = rotary_dim / 2;
  const int quads = half / 4;
  const int64_t total = static_cast<int64_t>(rows) * heads * quads;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int q4 = static_cast<int>(t % quads);
    const int64_t rh = t / quads;
    const int h = static_cast<int>(rh % heads);
    const int r = static_cast<int>(rh / heads);
    const float pos = static_cast<float>(positions[r]);
    __nv_bfloat16* base = x + static_cast<int64_t>(r) * ld + static_cast<int64_t>(h) * head_dim;
    uint2 a = *reinterpret_cast<const uint2*>(base + q4 * 4);
    uint2 b = *reinterpret_cast<const uint2*>(base + half + q4 * 4);
    float x1[4], x2[4];
    float2 f;
    f = unpack_bf16x2(a.x); x1[0] = f.x; x1[1] = f.y;
    f = unpack_bf16x2(a.y); x1[2] = f.x; x1[3] = f.y;
    f = unpack_bf16x2(b.x); x2[0] = f.x; x2[1] = f.y;
    f = unpack_bf16x2(b.y); x2[2] = f.x; x2[3] = f.y;
    float y1[4], y2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = q4 * 4 + j;
      const float inv_freq = exp2f(-log2_theta * (2.0f * i) / rotary_dim);
      float sn, cs;
      sincosf(pos * inv_freq, &sn, &cs);
      y1[j] = x1[j] * cs - x2[j] * sn;
      y2[j] = x2[j] * cs + x1[j] * sn;
    }
    *reinterpret_cast<uint2*>(base + q4 * 4) = make_uint2(pack_bf16x2(y1[0], y1[1]), pack_bf16x2(y1[2], y1[3]));
    *reinterpret_cast<uint2*>(base + half + q4 * 4) =
        make_uint2(pack_bf16x2(y2[0], y2[1]), pack_bf16x2(y2[2], y2[3]));
  }
}

__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                                 int ld_src, const int32_t* __restrict__ slot_mapping, int rows, int heads,
                                 int head_dim, int block_size, __nv_bfloat16* __restrict__ kcache,
                                 __nv_bfloat16* __restrict__ vcache) {
  pdl_trigger();
  pdl_wait();
  const int vec_per_row = heads * head_dim / 8;
  const int64_t total = static_cast<int64_t>(rows) * vec_per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vec_per_row);
    const int c = static_cast<int>(i - static_cast<int64_t>(r) * vec_per_row) * 8;
    const int slot = slot_mapping[r];
    if (slot < 0) continue;
    const int head = c / head_dim;
    const int d = c - head * head_dim;
    const int blk = slot / block_size;
    const int off = slot - blk * block_size;
    const int64_t dst = ((static_cast<int64_t>(blk) * heads + head) * block_size + off) * head_dim + d;
    *reinterpret_cast<uint4*>(kcache + dst) =
        ld_global_nc_v4(k + static_cast<int64_t>(r) * ld_src + c);
    *reinterpret_cast<uint4*>(vcache + dst) =
        ld_global_nc_v4(v + static_cast<int64_t>(r) * ld_src + c);
  }
}

__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ src, int ld_src,
                                   const int32_t* __restrict__ index, int rows, int cols,
                                   __nv_bfloat16* __restrict__ dst, int ld_dst) {
  pdl_trigger();
  pdl_wait();
  const int vec_per_row = cols / 8;
  const int64_t total = static_cast<int64_t>(rows) * vec_per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vec_per_row);
    const int c = static_cast<int>(i - static_cast<int64_t>(r) * vec_per_row) * 8;
    *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(r) * ld_dst + c) =
        *reinterpret_cast<const uint4*>(src + static_cast<int64_t>(index[r]) * ld_src + c);
  }
}

constexpr int kArgmaxThreads = 512;

AG_DEVICE void argmax_merge(float& v, int& i, float ov, int oi) {
  // larger value wins; ties go to the lower index (torch.argmax / numpy.argmax convention)
  if (ov > v || (ov == v && oi < i)) {
    v = ov;
    i = oi;
  }
}

__global__ void __launch_bounds__(kArgmaxThreads)
    argmax_kernel(const float* __restrict__ logits, int cols, int ld, int index_offset,
                  float* __restrict__ out_val, int32_t* __restrict__ out_idx) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sv[kArgmaxThreads / 32];
  __shared__ int si[kArgmaxThreads / 32];
  const float* row = logits + static_cast<int64_t>(blockIdx.x) * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  const int nvec = cols / 4;
  for (int c = threadIdx.x; c < nvec; c += kArgmaxThreads) {
    const float4 x = *reinterpret_cast<const float4*>(row + c * 4);
    argmax_merge(best, bi, x.x, c * 4);
    argmax_merge(best, bi, x.y, c * 4 + 1);
    argmax_merge(best, bi, x.z, c * 4 + 2);
    argmax_merge(best, bi, x.w, c * 4 + 3);
  }
  for (int c = nvec * 4 + threadIdx.x; c < cols; c += kArgmaxThreads) argmax_merge(best, bi, row[c], c);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    argmax_merge(best, bi, ov, oi);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = sv[0];
    int i = si[0];
    for (int k = 1; k < kArgmaxThreads / 32; ++k) argmax_merge(b, i, sv[k], si[k]);
    if (out_val) out_val[blockIdx.x] = b;
    out_idx[blockIdx.x] = i + index_offset;
  }
}

__global__ void argmax_merge_kernel(const float* __restrict__ vals, const int32_t* __restrict__ idx, int tp,
                                    int rows, int32_t* __restrict__ out_idx) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float b = vals[r];
  int i = idx[r];
  for (int k = 1; k < tp; ++k) argmax_merge(b, i, vals[k * rows + r], idx[k * rows + r]);
  out_idx[r] = i;
}

// Whole-block gather (swap out: pool -> staging) or scatter (swap in) over `planes` planes (layer x K/V):
// plane p of the pool starts at p * pool_plane elements, of the staging buffer at p * stage_plane.
__global__ void block_copy_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                  const int32_t* __restrict__ block_ids, int n_blocks, int64_t block_elems,
                                  int gather, int planes, int64_t pool_plane, int64_t stage_plane) {
  pdl_trigger();
  pdl_wait();
  const int64_t vec_per_block = block_elems / 8;
  const int64_t per_plane = vec_per_block * n_blocks;
  const int64_t total = per_plane * planes;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(i / per_plane);
    const int64_t j = i - p * per_plane;
    const int b = static_cast<int>(j / vec_per_block);
    const int64_t v = j - b * vec_per_block;
    const int64_t pool_off = p * pool_plane + static_cast<int64_t>(block_ids[b]) * block_elems + v * 8;
    const int64_t stage_off = p * stage_plane + static_cast<int64_t>(b) * block_elems + v * 8;
    if (gather)
      *reinterpret_cast<uint4*>(dst + stage_off) = *reinterpret_cast<const uint4*>(src + pool_off);
    else
      *reinterpret_cast<uint4*>(dst + pool_off) = *reinterpret_cast<const uint4*>(src + stage_off);
  }
}

// Deterministic pseudo-random bf16 fill: x = scale * u (or max(0, scale * u) with relu),
// u ~ U[-1, 1) from a hash of (seed, index).  Autotune inputs: timing GEMMs on zeroed activations
// underestimates their data-dependent power draw (and so overestimates clocks).
__global__ void fill_hash_kernel(__nv_bfloat16* __restrict__ x, int64_t n, uint32_t seed, float scale, int relu) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t h = static_cast<uint32_t>(i) * 0x9E3779B1u ^ static_cast<uint32_t>(i >> 32) * 0x85EBCA77u ^ seed;
    h ^= h >> 16;
    h *= 0x7FEB352Du;
    h ^= h >> 15;
    h *= 0x846CA68Bu;
    h ^= h >> 16;
    float v = scale * (static_cast<float>(h >> 8) * (2.0f / 16777216.0f) - 1.0f);
    if (relu) v = fmaxf(v, 0.0f);
    x[i] = __float2bfloat16(v);
  }
}

int grid_for(int64_t work_items, int threads) {
  int64_t g = (work_items + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

cudaError_t launch_fill_hash(__nv_bfloat16* x, int64_t n, uint32_t seed, float scale, bool relu,
                             cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  fill_hash_kernel<<<grid_for(n, 256), 256, 0, stream>>>(x, n, seed, scale, relu ? 1 : 0);
  return cudaGetLastError();
}

// decode inputs fed from the previous step's next-token ids without a host round trip (asynchronous
// steps, ag_model_submit): ids[pairs[2i]] = prev_out[pairs[2i+1]]
__global__ void feed_tokens_kernel(int32_t* __restrict__ ids, const int32_t* __restrict__ pairs, int n,
                                   const int32_t* __restrict__ prev_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[pairs[2 * i]] = prev_out[pairs[2 * i + 1]];
}

cudaError_t launch_feed_tokens(int32_t* ids, const int32_t* pairs, int n, const int32_t* prev_out,
                               cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  feed_tokens_kernel<<<(n + 255) / 256, 256, 0, stream>>>(ids, pairs, n, prev_out);
  return cudaGetLastError();
}

cudaError_t launch_embed(const int32_t* ids, const int32_t* positions, const __nv_bfloat16* tok_emb,
                         const __nv_bfloat16* pos_emb, int pos_offset, int rows, int hidden, int vocab,
                         int max_pos_rows, __nv_bfloat16* out, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int64_t work = static_cast<int64_t>(rows) * (hidden / 8);
  (void)launch_k(kPdlOther, embed_kernel, grid_for(work, 256), 256, 0, stream, ids, positions, tok_emb, pos_emb, pos_offset, rows,
                                                        hidden, vocab, max_pos_rows, out);
  return cudaGetLastError();
}

cudaError_t launch_layernorm(__nv_bfloat16* x, const __nv_bfloat16* delta, const __nv_bfloat16* delta_bias,
                             const int32_t* row_index, const __nv_bfloat16* gamma, const __nv_bfloat16* beta,
                             float eps, int rows, int hidden, __nv_bfloat16* out, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (hidden % 8 != 0 || hidden / 8 > kLNThreads * kLNMaxVec) return cudaErrorInvalidValue;
  if (hidden / 8 <= 1024 * kLNVpt) {
    const int threads = ((hidden / 8 + kLNVpt - 1) / kLNVpt + 31) / 32 * 32;
    (void)launch_k(kPdlNorm, layernorm_row_kernel<const __nv_bfloat16>, rows, threads, 0, stream, x, delta, delta_bias, row_index, gamma,
                                                                           beta, eps, hidden, out);
    return cudaGetLastError();
  }
  (void)launch_k(kPdlNorm, layernorm_kernel, rows, kLNThreads, 0, stream, x, delta, delta_bias, row_index, gamma, beta, eps, hidden,
                                                    out);
  return cudaGetLastError();
}

cudaError_t launch_layernorm_acc(__nv_bfloat16* x, float* acc32, const __nv_bfloat16* delta_bias,
                                 const int32_t* row_index, const __nv_bfloat16* gamma, const __nv_bfloat16* beta,
                                 float eps, int rows, int hidden, __nv_bfloat16* out, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (hidden % 8 != 0 || hidden / 8 > 1024 * kLNVpt || acc32 == nullptr) return cudaErrorInvalidValue;
  const int threads = ((hidden / 8 + kLNVpt - 1) / kLNVpt + 31) / 32 * 32;
  (void)launch_k(kPdlNorm, layernorm_row_kernel<float>, rows, threads, 0, stream, x, acc32, delta_bias, row_index, gamma, beta, eps, hidden,
                                                            out);
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm(__nv_bfloat16* x, const __nv_bfloat16* delta, const __nv_bfloat16* gamma, float eps,
                           int rows, int hidden, __nv_bfloat16* out, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (hidden % 8 != 0 || hidden / 8 > 32 * kLNWarpVec) return cudaErrorInvalidValue;
  (void)launch_k(kPdlNorm, rmsnorm_warp_kernel, (rows + kLNWarpsPerBlock - 1) / kLNWarpsPerBlock, kLNWarpsPerBlock * 32, 0, stream, 
      x, delta, gamma, eps, rows, hidden, out);
  return cudaGetLastError();
}

cudaError_t launch_rope(__nv_bfloat16* x, int ld, const int32_t* positions, int rows, int heads, int head_dim,
                        int rotary_dim, float theta, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (rotary_dim % 8 != 0 || rotary_dim > head_dim || ld % 4 != 0 || head_dim % 4 != 0 || theta <= 1.0f)
    return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(rows) * heads * (rotary_dim / 8);
  (void)launch_k(kPdlOther, rope_kernel, grid_for(work, 256), 256, 0, stream, x, ld, positions, rows, heads, head_dim, rotary_dim,
                                                        log2f(theta));
  return cudaGetLastError();
}

cudaError_t launch_kv_append(const __nv_bfloat16* k, const __nv_bfloat16* v, int ld_src,
                             const int32_t* slot_mapping, int rows, int heads, int head_dim, int block_size,
                             __nv_bfloat16* kcache, __nv_bfloat16* vcache, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (head_dim % 8 != 0 || ld_src % 8 != 0) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(rows) * heads * head_dim / 8;
  (void)launch_k(kPdlOther, kv_append_kernel, grid_for(work, 256), 256, 0, stream, k, v, ld_src, slot_mapping, rows, heads, head_dim,
                                                            block_size, kcache, vcache);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const __nv_bfloat16* src, int ld_src, const int32_t* index, int rows, int cols,
                               __nv_bfloat16* dst, int ld_dst, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int64_t work = static_cast<int64_t>(rows) * (cols / 8);
  (void)launch_k(kPdlOther, gather_rows_kernel, grid_for(work, 256), 256, 0, stream, src, ld_src, index, rows, cols, dst, ld_dst);
  return cudaGetLastError();
}

cudaError_t launch_argmax(const float* logits, int rows, int cols, int ld, int index_offset, float* out_val,
                          int32_t* out_idx, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (ld % 4 != 0) return cudaErrorInvalidValue;
  (void)launch_k(kPdlOther, argmax_kernel, rows, kArgmaxThreads, 0, stream, logits, cols, ld, index_offset, out_val, out_idx);
  return cudaGetLastError();
}

cudaError_t launch_argmax_merge(const float* vals, const int32_t* idx, int tp, int rows, int32_t* out_idx,
                                cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  (void)launch_k(kPdlOther, argmax_merge_kernel, (rows + 127) / 128, 128, 0, stream, vals, idx, tp, rows, out_idx);
  return cudaGetLastError();
}

cudaError_t launch_block_copy(const __nv_bfloat16* src, __nv_bfloat16* dst, const int32_t* block_ids,
                              int n_blocks, int64_t block_elems, bool gather, cudaStream_t stream, int planes,
                              int64_t pool_plane, int64_t stage_plane) {
  if (n_blocks <= 0 || planes <= 0) return cudaSuccess;
  if (block_elems % 8 != 0 || pool_plane % 8 != 0 || stage_plane % 8 != 0) return cudaErrorInvalidValue;
  const int64_t work = block_elems / 8 * n_blocks * planes;
  (void)launch_k(kPdlOther, block_copy_kernel, grid_for(work, 256), 256, 0, stream, src, dst, block_ids, n_blocks, block_elems,
                 gather ? 1 : 0, planes, pool_plane, stage_plane);
  return cudaGetLastError();
}

}  // namespace ag
