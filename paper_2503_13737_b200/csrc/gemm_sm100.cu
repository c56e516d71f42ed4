// Persistent warp-specialised tcgen05 GEMM for sm_100a:  D[M,N] = A[M,K] . B[N,K]^T  (+ epilogue)
//
// A = activations (tokens x hidden, K-major), B = nn.Linear weight [out, in] (K-major).
// Operands are staged by TMA (128 B swizzle) into a STAGES-deep shared-memory ring,
// one elected thread issues tcgen05.mma (M=128, N=BN, K=16) into a double-buffered TMEM
// accumulator, and four epilogue warps drain TMEM with tcgen05.ld while the next tile's
// MMAs run.  The epilogue fuses bias, ReLU, residual add, the OPT q-scaling and the
// paged KV append (QKV projection writes K/V straight into their cache slots).
//
// Warp roles (256 threads):  w0 TMA producer | w1 MMA issuer | w2 TMEM allocator |
//                            w3 idle | w4..w7 epilogue (TMEM lanes 0..127)
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace ag {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle row of bf16
constexpr int kThreads = 256;

// AM = activation rows TMA-loaded per stage.  AM < 128 is the small-M (weight streaming)
// variant: the M=128 UMMA still reads a 128-row A window, whose rows >= AM are stale smem that
// only feeds masked output rows, so ~4x more weight bytes fit in the ring.
template <int BN, int AM = 128>
struct GemmCfg {
  static constexpr int kABytes = AM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStagesFit = (200 * 1024) / kStageBytes;
  static constexpr int kStages = kStagesFit > 12 ? 12 : kStagesFit;
  // double-buffered accumulator; tcgen05.alloc takes a power of two >= 32 columns (BN=160 -> 512)
  static constexpr int kTmemCols = 2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512));
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + 256;
};

// Store W (a multiple of 8) consecutive bf16 values v[0..W) at dst.
template <int W>
AG_DEVICE void store_bf16(__nv_bfloat16* dst, const float* v) {
#pragma unroll
  for (int q = 0; q < W / 8; ++q)
    st_global_v4(dst + q * 8, pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]),
                 pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]));
}

// v[0..W) += W consecutive bf16 values at src.
template <int W>
AG_DEVICE void add_bf16(float* v, const __nv_bfloat16* src) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int q = 0; q < W / 8; ++q) {
    const uint4 w = s4[q];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 f = unpack_bf16x2(ws[h]);
      v[q * 8 + h * 2] += f.x;
      v[q * 8 + h * 2 + 1] += f.y;
    }
  }
}

// Fused epilogue of W consecutive accumulator columns [col0, col0 + W) of one output row: bias,
// then either the QKV split (q scaled -> q buffer; K/V -> their paged cache slots) or residual
// add / ReLU -> bf16 or f32 output.  W = 32 (one TMEM load per thread) or 8 (split-K reduce); a
// W-column group never straddles a head (head_dim % 32 == 0).
template <int W>
AG_DEVICE void epilogue_cols(const GemmEpilogue& ep, int row, int col0, float* v) {
  if (ep.bias != nullptr) add_bf16<W>(v, ep.bias + col0);
  if (ep.mode == kEpiQkv) {
    const int region = col0 / ep.hq;  // 0 = q, 1 = k, 2 = v
    if (region == 0) {
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] *= ep.q_scale;
      store_bf16<W>(reinterpret_cast<__nv_bfloat16*>(ep.out) + (size_t)row * ep.ldc + col0, v);
      return;
    }
    const int slot = ep.slot_mapping[row];
    if (slot < 0) return;  // padding token: no cache write
    const int within = col0 - region * ep.hq;
    const int head = within / ep.head_dim;
    const int d = within - head * ep.head_dim;
    const int blk = slot / ep.block_size;
    const int off = slot - blk * ep.block_size;
    __nv_bfloat16* cache = (region == 1) ? ep.kcache : ep.vcache;
    store_bf16<W>(cache + (((size_t)blk * ep.heads + head) * ep.block_size + off) * ep.head_dim + d, v);
    return;
  }
  if (ep.residual != nullptr) add_bf16<W>(v, ep.residual + (size_t)row * ep.ldr + col0);
  if (ep.relu) {
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] = fmaxf(v[j], 0.0f);
  }
  if (ep.out_f32) {
    float* dst = reinterpret_cast<float*>(ep.out) + (size_t)row * ep.ldc + col0;
#pragma unroll
    for (int q = 0; q < W / 4; ++q)
      st_global_v4(dst + q * 4, __float_as_uint(v[q * 4]), __float_as_uint(v[q * 4 + 1]),
                   __float_as_uint(v[q * 4 + 2]), __float_as_uint(v[q * 4 + 3]));
  } else {
    store_bf16<W>(reinterpret_cast<__nv_bfloat16*>(ep.out) + (size_t)row * ep.ldc + col0, v);
  }
}

AG_DEVICE void red_add_v4(float* dst, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

AG_DEVICE void epilogue_chunk(const GemmEpilogue& ep, int row, int col0, const uint32_t (&r)[32]) {
  if (ep.mode == kEpiAtomicF32) {
    float* dst = ep.acc32 + (size_t)row * ep.ldc + col0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      red_add_v4(dst + q * 4, __uint_as_float(r[q * 4]), __uint_as_float(r[q * 4 + 1]), __uint_as_float(r[q * 4 + 2]),
                 __uint_as_float(r[q * 4 + 3]));
    return;
  }
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  epilogue_cols<32>(ep, row, col0, v);
}

// ---------------------------------------------------------------- fused LayerNorm tail
// A TP=1 out-proj / FC2 whose K is split accumulates into the fp32 buffer acc32, and the residual
// add + bias + LayerNorm that consumes it used to be its own launch (launch_layernorm_acc): ~80 per
// OPT-13B forward, each paying a full launch gap because the norms cannot be launched early
// (profiles/r2/pdl_hang.md).  With ep.ln_out set, the GEMM's CTAs meet at a grid barrier once
// their reductions have drained and finish the rows themselves.

AG_DEVICE unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier.  Every CTA of these grids is co-resident: <= 1 CTA per SM (the operand ring
// takes ~200 KB of shared memory), grid <= SMs, and a PDL dependent is only launched once every CTA
// of this grid has executed griddepcontrol.launch_dependents -- i.e. is already resident -- so an
// early dependent can never hold the SM a straggler of this grid needs.  bar[0] counts arrivals,
// bar[1] is the generation; the last arriver resets the count before releasing the generation, and
// the next grid to use the barrier starts its tail only after this grid has completed.
AG_DEVICE void grid_barrier(unsigned* bar, unsigned ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire_u32(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == ctas - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire_u32(bar + 1) == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

AG_DEVICE float cta_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

constexpr int kLnMaxVec = 6;  // 8-column groups per thread: hidden <= 256 * 8 * 6 = 12288

AG_DEVICE void bf16x8_unpack(const uint4& w, float (&f)[8]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 p = unpack_bf16x2(ws[h]);
    f[2 * h] = p.x;
    f[2 * h + 1] = p.y;
  }
}

AG_DEVICE uint4 bf16x8_pack(const float (&f)[8]) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
}

// Rows blockIdx.x, +gridDim.x, ... of  x = bf16(x + (acc + bias)); acc = 0; out = LN(x) * g + b  -- the
// same rounding points as layernorm_row_kernel<float> (elementwise.cu), 256 threads per row (a row per
// warp instead was slower in-chain: 22.1 vs 20.8 ms on the median decode step -- too few loads in flight).
AG_DEVICE void ln_rows(const GemmEpilogue& ep, int M, int hidden) {
  __shared__ float red[kThreads / 32];
  const int nvec = hidden / 8;
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    __nv_bfloat16* xr = ep.ln_x + static_cast<int64_t>(r) * hidden;
    float4* ar = reinterpret_cast<float4*>(ep.ln_acc + static_cast<int64_t>(r) * ep.ln_ld);
    float v[kLnMaxVec][8];
    float sum = 0.0f;
#pragma unroll
    for (int i = 0; i < kLnMaxVec; ++i) {
      const int idx = threadIdx.x + i * kThreads;
      if (idx < nvec) {
        bf16x8_unpack(*reinterpret_cast<const uint4*>(xr + idx * 8), v[i]);
        const float4 a = __ldcg(ar + 2 * idx), b = __ldcg(ar + 2 * idx + 1);
        ar[2 * idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        ar[2 * idx + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
        float d[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        if (ep.ln_bias != nullptr) {
          float bb[8];
          bf16x8_unpack(__ldg(reinterpret_cast<const uint4*>(ep.ln_bias) + idx), bb);
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] += bb[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i][j] += d[j];
        const uint4 packed = bf16x8_pack(v[i]);
        *reinterpret_cast<uint4*>(xr + idx * 8) = packed;  // updated residual stream
        bf16x8_unpack(packed, v[i]);                       // normalise the rounded value
#pragma unroll
        for (int j = 0; j < 8; ++j) sum += v[i][j];
      }
    }
    const float mean = cta_sum(sum, red) / hidden;
    float sq = 0.0f;
#pragma unroll
    for (int i = 0; i < kLnMaxVec; ++i)
      if (threadIdx.x + i * kThreads < nvec)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float c = v[i][j] - mean;
          sq += c * c;
        }
    const float rstd = rsqrtf(cta_sum(sq, red) / hidden + ep.ln_eps);
    __nv_bfloat16* orow = ep.ln_out + static_cast<int64_t>(r) * hidden;
#pragma unroll
    for (int i = 0; i < kLnMaxVec; ++i) {
      const int idx = threadIdx.x + i * kThreads;
      if (idx < nvec) {
        float g[8], b[8], y[8];
        bf16x8_unpack(__ldg(reinterpret_cast<const uint4*>(ep.ln_g) + idx), g);
        bf16x8_unpack(__ldg(reinterpret_cast<const uint4*>(ep.ln_b) + idx), b);
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = (v[i][j] - mean) * rstd * g[j] + b[j];
        *reinterpret_cast<uint4*>(orow + idx * 8) = bf16x8_pack(y);
      }
    }
  }
}

// Fused LayerNorm prologue of the *consumer* GEMM (QKV after an atomic FC2, FC1 after an atomic
// out-proj): the predecessor left its fp32 reductions in ln_acc; this grid's CTAs -- resident, their
// first weight stages already in flight -- finish the rows into ln_out (= this GEMM's A operand), make the
// generic stores visible to the TMA (async proxy) and meet at a grid barrier before any A tile is loaded.
// Unlike the producer-side tail, the next GEMM's weight prefetch overlaps the norm.
AG_DEVICE void ln_prologue(const GemmEpilogue& ep, int M, int K) {
  pdl_wait();
  ln_rows(ep, M, K);
  asm volatile("fence.proxy.async.global;" ::: "memory");  // writer side: generic stores -> async proxy
  grid_barrier(ep.ln_bar, gridDim.x);
  asm volatile("fence.proxy.async.global;" ::: "memory");  // reader side: before this CTA's TMA loads of A
}

// Work decomposition shared by the three warp roles of the 1-CTA kernel.  Classic: unit t =
// (m_blk, k_split, n_blk), m fastest (concurrent CTAs share a weight tile), strided over CTAs.
// Stream-K (k_splits == kStreamK): CTA c takes the contiguous k-block range [c*U/G, (c+1)*U/G)
// of the flattened (n_blk, m_blk, kb) space, U = tiles x k-blocks, cut at tile boundaries into
// segments; every CTA streams the same number of weight k-blocks (no wave quantisation), and
// partial tiles meet in the atomic fp32 epilogue (kEpiAtomicF32 only).
struct SegIter {
  int num_m, num_kb, k_splits, kb_per, num_tiles, t, stride;
  long long u, u_end;
  bool streamk;
  AG_DEVICE SegIter(int M, int N, int K, int bm, int bn, int ks, int idx, int count) {
    num_m = (M + bm - 1) / bm;
    const int num_n = (N + bn - 1) / bn;
    num_kb = (K + kBK - 1) / kBK;
    streamk = ks == kStreamK;
    k_splits = streamk ? 1 : ks;
    kb_per = (num_kb + k_splits - 1) / k_splits;
    num_tiles = num_m * num_n * k_splits;
    t = idx;
    stride = count;
    const long long U = static_cast<long long>(num_m) * num_n * num_kb;
    u = U * idx / count;
    u_end = U * (idx + 1) / count;
  }
  AG_DEVICE bool next(int& m_blk, int& n_blk, int& ks_idx, int& kb0, int& kb1) {
    if (streamk) {
      if (u >= u_end) return false;
      const long long tile = u / num_kb;
      kb0 = static_cast<int>(u - tile * num_kb);
      kb1 = static_cast<int>(min(static_cast<long long>(num_kb), kb0 + (u_end - u)));
      m_blk = static_cast<int>(tile % num_m);
      n_blk = static_cast<int>(tile / num_m);
      ks_idx = 0;
      u += kb1 - kb0;
      return true;
    }
    if (t >= num_tiles) return false;
    m_blk = t % num_m;
    ks_idx = (t / num_m) % k_splits;
    n_blk = t / (num_m * k_splits);
    kb0 = ks_idx * kb_per;
    kb1 = min(num_kb, kb0 + kb_per);
    t += stride;
    return true;
  }
};

template <int BN, int AM>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_b, int M, int N, int K,
                        GemmEpilogue ep, int k_splits, float* __restrict__ partial) {
  using Cfg = GemmCfg<BN, AM>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (M + kBM - 1) / kBM;
  int m_blk, n_blk, ks, kb0, kb1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // dependents may launch only once this CTA holds its TMEM: an early dependent CTA on this SM
  // that allocated first would wait (griddepcontrol.wait) on us while we wait on its columns
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;

  // weights of a small-M GEMM are streamed once -> evict first (large M reuses a weight tile across
  // concurrent m-blocks)
  const uint64_t pol_w = num_m <= 2 ? policy_evict_first() : policy_evict_normal();
  // The weight k-blocks of the first S stages do not depend on the predecessor kernel: the producer
  // issues them before griddepcontrol.wait (and before a fused LayerNorm prologue), so the weight
  // stream starts while the predecessor drains.
  int pre = 0;
  if (warp == 0 && lane == 0) {
    SegIter ip(M, N, K, kBM, BN, k_splits, blockIdx.x, gridDim.x);
    while (pre < S && ip.next(m_blk, n_blk, ks, kb0, kb1))
      for (int kb = kb0; kb < kb1 && pre < S; ++kb, ++pre) {
        mbar_arrive_expect_tx(&full_bar[pre], Cfg::kStageBytes);
        tma_load_2d_hint(sB + pre * Cfg::kBBytes, &tmap_b, &full_bar[pre], kb * kBK, n_blk * BN, pol_w);
      }
  }
  if (ep.ln_out != nullptr && ep.ln_prologue) ln_prologue(ep, M, K);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      // activations are re-read by every N tile -> keep in L2
      const uint64_t pol_a = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      SegIter it(M, N, K, kBM, BN, k_splits, blockIdx.x, gridDim.x);
      pdl_wait();
      int g = 0;
      while (it.next(m_blk, n_blk, ks, kb0, kb1)) {
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          if (g < pre) {  // B already in flight on this stage's barrier
            tma_load_2d_hint(sA + stage * Cfg::kABytes, &tmap_a, &full_bar[stage], kb * kBK, m_blk * kBM, pol_a);
          } else {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
            tma_load_2d_hint(sA + stage * Cfg::kABytes, &tmap_a, &full_bar[stage], kb * kBK, m_blk * kBM, pol_a);
            tma_load_2d_hint(sB + stage * Cfg::kBBytes, &tmap_b, &full_bar[stage], kb * kBK, n_blk * BN, pol_w);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      SegIter it(M, N, K, kBM, BN, k_splits, blockIdx.x, gridDim.x);
      while (it.next(m_blk, n_blk, ks, kb0, kb1)) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * Cfg::kABytes));
          const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * Cfg::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // +32 bytes along K inside the swizzle atom == +2 in the (addr >> 4) field
            umma_bf16_ss(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> fused ops -> global
    const int ew = warp - 4;
    pdl_wait();  // the epilogue reads residuals and writes outputs the predecessor may still use
    int acc = 0;
    uint32_t acc_phase = 0;
    SegIter it(M, N, K, kBM, BN, k_splits, blockIdx.x, gridDim.x);
    while (it.next(m_blk, n_blk, ks, kb0, kb1)) {
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * kBM + ew * 32 + lane;
      const bool warp_live = m_blk * kBM + ew * 32 < M;  // whole warp beyond M: nothing to drain
#pragma unroll 1
      for (int c = 0; c < (warp_live ? BN / 32 : 0); ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int col0 = n_blk * BN + c * 32;
        if (row < M && col0 < N) {
          if (k_splits == 1 || ep.mode == kEpiAtomicF32) {
            epilogue_chunk(ep, row, col0, r);
          } else {  // fp32 partial of this K split; splitk_reduce_kernel applies the epilogue
            float* dst = partial + ((size_t)ks * M + row) * N + col0;
#pragma unroll
            for (int q = 0; q < 8; ++q) st_global_v4(dst + q * 4, r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    // Drain this thread's red.global.add before the CTA exits.  Without it, a kernel launched early
    // (PDL) behind this grid could sit in griddepcontrol.wait forever: the 40-layer OPT-13B forward
    // hung whenever the successor of an atomic-epilogue GEMM was early-launched, and completes with
    // the fence, at no measurable cost (profiles/r2/pdl_hang.md).
    if (ep.mode == kEpiAtomicF32) __threadfence();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
  if (ep.ln_out != nullptr && !ep.ln_prologue) {  // fused tail: every CTA's reductions have drained
    grid_barrier(ep.ln_bar, gridDim.x);
    ln_rows(ep, M, N);
  }
}

// ---------------------------------------------------------------- CTA-pair variant
// A cluster of two CTAs on one TPC computes a 256 x BN tile with tcgen05.mma.cta_group::2 (M=256):
// each CTA stages its own 128 activation rows and BN/2 weight rows per k-block, so a CTA moves
// (128 + BN/2) x 64 x 2 bytes through TMA per 128 x BN outputs instead of (128 + BN) x 64 x 2 --
// a third less L2->SMEM traffic at BN=256, which is what bounds the 1-CTA kernel at large M.
// The leader (rank 0) issues the MMAs; its commits multicast to both CTAs' barriers.  Each CTA's
// epilogue drains its own TMEM (rows 128*rank ..) exactly like the 1-CTA kernel.
template <int BN>
struct Gemm2Cfg {
  static constexpr int kABytes = 128 * kBK * 2;
  static constexpr int kBBytes = (BN / 2) * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStagesFit = (200 * 1024) / kStageBytes;
  static constexpr int kStages = kStagesFit > 10 ? 10 : kStagesFit;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + 256;
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                         int M, int N, int K, GemmEpilogue ep, int k_splits, float* __restrict__ partial) {
  using Cfg = Gemm2Cfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int num_pairs = gridDim.x >> 1;
  const int num_m = (M + 255) / 256;
  int m_blk, n_blk, ks, kb0, kb1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_cg2(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_trigger();  // after the TMEM allocation (see the 1-CTA kernel)
  const uint32_t tmem_base = *tmem_slot;

  const uint64_t pol_w = num_m <= 1 ? policy_evict_first() : policy_evict_normal();
  const uint32_t full0 = mapa_shared(smem_u32(&full_bar[0]), 0);
  int pre = 0;  // weight k-blocks issued before griddepcontrol.wait (see the 1-CTA kernel)
  if (warp == 0 && lane == 0) {
    SegIter ip(M, N, K, 256, BN, k_splits, pair, num_pairs);
    while (pre < S && ip.next(m_blk, n_blk, ks, kb0, kb1))
      for (int kb = kb0; kb < kb1 && pre < S; ++kb, ++pre) {
        if (rank == 0) mbar_arrive_expect_tx(&full_bar[pre], 2 * Cfg::kStageBytes);
        tma_load_2d_cg2(sB + pre * Cfg::kBBytes, &tmap_b, full0 + pre * 8, kb * kBK, n_blk * BN + rank * (BN / 2),
                        pol_w);
      }
  }
  if (ep.ln_out != nullptr && ep.ln_prologue) ln_prologue(ep, M, K);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs): own 128 A rows + own BN/2 B rows per k-block
      const uint64_t pol_a = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      SegIter it(M, N, K, 256, BN, k_splits, pair, num_pairs);
      pdl_wait();
      int g = 0;
      while (it.next(m_blk, n_blk, ks, kb0, kb1)) {
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const uint32_t fb = full0 + stage * 8;
          if (g >= pre) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
            tma_load_2d_cg2(sB + stage * Cfg::kBBytes, &tmap_b, fb, kb * kBK, n_blk * BN + rank * (BN / 2), pol_w);
          }
          tma_load_2d_cg2(sA + stage * Cfg::kABytes, &tmap_a, fb, kb * kBK, m_blk * 256 + rank * 128, pol_a);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: leader CTA only, one thread
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      SegIter it(M, N, K, 256, BN, k_splits, pair, num_pairs);
      while (it.next(m_blk, n_blk, ks, kb0, kb1)) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * Cfg::kABytes));
          const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * Cfg::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16_ss_cg2(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          umma_commit_cg2(&empty_bar[stage], 0x3);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_cg2(&tfull_bar[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): this CTA's 128 rows of the 256-row tile
    const int ew = warp - 4;
    pdl_wait();
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    SegIter it(M, N, K, 256, BN, k_splits, pair, num_pairs);
    while (it.next(m_blk, n_blk, ks, kb0, kb1)) {
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row0 = m_blk * 256 + static_cast<int>(rank) * 128 + ew * 32;
      const int row = row0 + lane;
      const bool warp_live = row0 < M;
#pragma unroll 1
      for (int c = 0; c < (warp_live ? BN / 32 : 0); ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int col0 = n_blk * BN + c * 32;
        if (row < M && col0 < N) {
          if (k_splits == 1 || ep.mode == kEpiAtomicF32) {
            epilogue_chunk(ep, row, col0, r);
          } else {
            float* dst = partial + ((size_t)ks * M + row) * N + col0;
#pragma unroll
            for (int q = 0; q < 8; ++q) st_global_v4(dst + q * 4, r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (ep.mode == kEpiAtomicF32) __threadfence();  // (see the 1-CTA kernel)
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, Cfg::kTmemCols);
  }
  if (ep.ln_out != nullptr && !ep.ln_prologue) {  // fused tail: every CTA's reductions have drained
    grid_barrier(ep.ln_bar, gridDim.x);
    ln_rows(ep, M, N);
  }
}

// Sum the K-split fp32 partials of 8 consecutive columns per thread and apply the fused epilogue
// (consecutive threads on consecutive 32-B column groups of a row: coalesced, 2 x splits loads in
// flight per thread).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ partial, int splits, int M,
                                                            int N, GemmEpilogue ep) {
  pdl_trigger();
  pdl_wait();
  const int groups = N / 8;
  const int64_t total = static_cast<int64_t>(M) * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / groups);
    const int col0 = static_cast<int>(i - static_cast<int64_t>(row) * groups) * 8;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
    const float* src = partial + (size_t)row * N + col0;
#pragma unroll 4
    for (int s = 0; s < splits; ++s) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(src + (size_t)s * M * N));
      const float4 b = __ldcg(reinterpret_cast<const float4*>(src + (size_t)s * M * N) + 1);
      acc[0] += a.x;
      acc[1] += a.y;
      acc[2] += a.z;
      acc[3] += a.w;
      acc[4] += b.x;
      acc[5] += b.y;
      acc[6] += b.z;
      acc[7] += b.w;
    }
    epilogue_cols<8>(ep, row, col0, acc);
  }
}

// Stream-K finish for GEMMs whose epilogue cannot be deferred to a consumer (QKV, FC1): the atomic
// fp32 accumulator acc[M, N] gets the fused epilogue (8 columns per thread) and is re-zeroed.
__global__ void __launch_bounds__(256) splitk_finish_kernel(float* __restrict__ acc, int M, int N, GemmEpilogue ep) {
  pdl_trigger();
  pdl_wait();
  const int groups = N / 8;
  const int64_t total = static_cast<int64_t>(M) * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / groups);
    const int col0 = static_cast<int>(i - static_cast<int64_t>(row) * groups) * 8;
    float4* src = reinterpret_cast<float4*>(acc + (size_t)row * N + col0);
    const float4 a = __ldcg(src), b = __ldcg(src + 1);
    src[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    src[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    epilogue_cols<8>(ep, row, col0, v);
  }
}

}  // namespace

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn g_encode = nullptr;

static bool load_encode_fn() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    return false;
  g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  return true;
}

int make_tmap_kmajor(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld_elems,
                     int box_rows) {
  if (!load_encode_fn()) return -1;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld_elems * 2) % 16 != 0) return -2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -3;
}

static int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

template <int BN, int AM = 128>
static cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                             const GemmEpilogue& ep, int k_splits, float* partial, int max_ctas,
                             cudaStream_t stream) {
  using Cfg = GemmCfg<BN, AM>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, AM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (k_splits == kStreamK && ep.mode != kEpiAtomicF32) return cudaErrorInvalidValue;
  const int64_t tiles = static_cast<int64_t>((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int64_t units = k_splits == kStreamK ? tiles * ((K + kBK - 1) / kBK) : tiles * k_splits;
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (units < grid) grid = static_cast<int>(units);
  const cudaError_t le = launch_k_ex(kPdlGemm, ep.ln_out != nullptr, gemm_bf16_tn_kernel<BN, AM>, grid, kThreads,
                                     Cfg::kSmemBytes, stream, ta, tb, M, N, K, ep, k_splits, partial);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = le;
  if (e != cudaSuccess || k_splits == 1 || ep.mode == kEpiAtomicF32) return e;
  const int64_t work = static_cast<int64_t>(M) * (N / 8);
  int rg = static_cast<int>(std::min<int64_t>((work + 255) / 256, static_cast<int64_t>(num_sms()) * 16));
  (void)launch_k(kPdlGemm, splitk_reduce_kernel, rg, 256, 0, stream, partial, k_splits, M, N, ep);
  return cudaGetLastError();
}

template <int BN>
static cudaError_t launch_bn2(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                              const GemmEpilogue& ep, int k_splits, float* partial, int max_ctas,
                              cudaStream_t stream) {
  using Cfg = Gemm2Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm2_bf16_tn_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t tiles = static_cast<int64_t>((M + 255) / 256) * ((N + BN - 1) / BN);
  const int64_t units = k_splits == kStreamK ? tiles * ((K + kBK - 1) / kBK) : tiles * k_splits;
  int grid = num_sms() & ~1;
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas & ~1;
  if (2 * units < grid) grid = static_cast<int>(2 * units);
  const cudaError_t le = launch_k_ex(kPdlGemm, ep.ln_out != nullptr, gemm2_bf16_tn_kernel<BN>, grid, kThreads,
                                     Cfg::kSmemBytes, stream, ta, tb, M, N, K, ep, k_splits, partial);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = le;
  if (e != cudaSuccess || k_splits == 1 || ep.mode == kEpiAtomicF32) return e;
  const int64_t work = static_cast<int64_t>(M) * (N / 8);
  int rg = static_cast<int>(std::min<int64_t>((work + 255) / 256, static_cast<int64_t>(num_sms()) * 16));
  (void)launch_k(kPdlGemm, splitk_reduce_kernel, rg, 256, 0, stream, partial, k_splits, M, N, ep);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int bn,
                        const GemmEpilogue& ep, int max_ctas, cudaStream_t stream, int k_splits, float* partial,
                        int am) {
  if (M <= 0) return cudaSuccess;
  if (ep.ln_out != nullptr) {
    const int hidden = ep.ln_prologue ? K : N;
    if ((!ep.ln_prologue && ep.mode != kEpiAtomicF32) || ep.ln_bar == nullptr || ep.ln_x == nullptr ||
        ep.ln_acc == nullptr || ep.ln_g == nullptr || ep.ln_b == nullptr || hidden % 8 != 0 ||
        hidden / 8 > kThreads * kLnMaxVec || ep.ln_ld % 4 != 0)
      return cudaErrorInvalidValue;
  }
  if (am == 256) {  // CTA pair: ta box = 128 rows, tb box = bn/2 rows
    if (k_splits == kStreamK && ep.mode != kEpiAtomicF32) return cudaErrorInvalidValue;
    if (k_splits > 1 && ep.mode != kEpiAtomicF32 && (partial == nullptr || N % 32 != 0)) return cudaErrorInvalidValue;
    if (bn == 256) return launch_bn2<256>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    if (bn == 128) return launch_bn2<128>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    return cudaErrorInvalidValue;
  }
  if (k_splits > 1 && ep.mode != kEpiAtomicF32 && (partial == nullptr || N % 32 != 0)) return cudaErrorInvalidValue;
  if (am != 128 && M > am) return cudaErrorInvalidValue;  // small-M variant needs one m-block
  if (am == 32) {
    if (bn == 256) return launch_bn<256, 32>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    if (bn == 160) return launch_bn<160, 32>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    if (bn == 64) return launch_bn<64, 32>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    return launch_bn<128, 32>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
  }
  if (am == 64) {
    if (bn == 256) return launch_bn<256, 64>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    if (bn == 160) return launch_bn<160, 64>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    if (bn == 64) return launch_bn<64, 64>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
    return launch_bn<128, 64>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
  }
  if (bn == 256) return launch_bn<256>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
  if (bn == 160) return launch_bn<160>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
  if (bn == 64) return launch_bn<64>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
  return launch_bn<128>(ta, tb, M, N, K, ep, k_splits, partial, max_ctas, stream);
}

int gemm_grid(int M, int N, int K, int bn, int k_splits, int am) {
  const int bm = am == 256 ? 256 : kBM;
  const int64_t tiles = static_cast<int64_t>((M + bm - 1) / bm) * ((N + bn - 1) / bn);
  const int64_t units = k_splits == kStreamK ? tiles * ((K + kBK - 1) / kBK) : tiles * k_splits;
  if (am == 256) return static_cast<int>(std::min<int64_t>(num_sms() & ~1, 2 * units));
  return static_cast<int>(std::min<int64_t>(num_sms(), units));
}

cudaError_t launch_splitk_finish(float* acc, int M, int N, const GemmEpilogue& ep, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (N % 8 != 0 || ep.mode == kEpiAtomicF32) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(M) * (N / 8);
  const int g = static_cast<int>(std::min<int64_t>((work + 255) / 256, static_cast<int64_t>(num_sms()) * 16));
  (void)launch_k(kPdlGemm, splitk_finish_kernel, g, 256, 0, stream, acc, M, N, ep);
  return cudaGetLastError();
}

GemmPlan plan_gemm(int M, int N, int K, int64_t partial_capacity_floats) {
  // Estimated makespan in "bytes streamed per SM": every unit loads (128 + BN) rows x 64 K per
  // k-block; units run in ceil(units / SMs) waves; a split adds an fp32 round trip through L2/HBM
  // spread over the whole chip, and every unit pays a fixed prologue.
  const int sms = num_sms();
  const int num_m = (M + kBM - 1) / kBM;
  const int num_kb = (K + kBK - 1) / kBK;
  GemmPlan best{256, 1};
  double best_cost = 1e300;
  for (int bn : {256, 128}) {
    if (bn == 256 && N % 256 != 0 && N > 256) continue;
    const int num_n = (N + bn - 1) / bn;
    for (int splits = 1; splits <= 16; ++splits) {
      const int kb_per = (num_kb + splits - 1) / splits;
      const int real_splits = (num_kb + kb_per - 1) / kb_per;
      if (real_splits != splits) continue;
      if (splits > 1 && (kb_per < 4 || static_cast<int64_t>(splits) * M * N > partial_capacity_floats)) break;
      const int64_t units = static_cast<int64_t>(num_m) * num_n * splits;
      const double waves = static_cast<double>((units + sms - 1) / sms);
      const double per_unit = kb_per * (128.0 + bn) * kBK * 2.0 + 96.0 * 1024.0;
      double cost = waves * per_unit;
      if (splits > 1) cost += static_cast<double>(M) * N * 4.0 * (splits + 1) / sms;
      if (cost < best_cost * 0.98) {
        best_cost = cost;
        best = {bn, splits};
      }
    }
  }
  return best;
}

int pick_block_n(int M, int N) {
  // Prefer the wider tile unless it leaves most SMs idle or N is not a multiple of 256.
  if (N % 256 != 0) return 128;
  const int tiles256 = ((M + kBM - 1) / kBM) * (N / 256);
  if (tiles256 < num_sms() / 2) return 128;
  return 256;
}

}  // namespace ag
