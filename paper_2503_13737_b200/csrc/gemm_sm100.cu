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

namespace ag {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle row of bf16
constexpr int kThreads = 256;

template <int BN>
struct GemmCfg {
  static constexpr int kStages = (BN == 256) ? 4 : 6;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + 256;
};

AG_DEVICE void epilogue_chunk(const GemmEpilogue& ep, int row, int col0, const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);

  if (ep.bias != nullptr) {
    const uint4* b4 = reinterpret_cast<const uint4*>(ep.bias + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w = __ldg(b4 + q);
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float2 f = unpack_bf16x2(ws[h]);
        v[q * 8 + h * 2] += f.x;
        v[q * 8 + h * 2 + 1] += f.y;
      }
    }
  }

  if (ep.mode == kEpiQkv) {
    const int region = col0 / ep.hq;  // 0 = q, 1 = k, 2 = v
    if (region == 0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= ep.q_scale;
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(ep.out) + (size_t)row * ep.ldc + col0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        st_global_v4(dst + q * 8, pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]),
                     pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]), pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]),
                     pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]));
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
    __nv_bfloat16* dst =
        cache + (((size_t)blk * ep.heads + head) * ep.block_size + off) * ep.head_dim + d;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      st_global_v4(dst + q * 8, pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]),
                   pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]), pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]),
                   pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]));
    return;
  }

  if (ep.residual != nullptr) {
    const uint4* r4 = reinterpret_cast<const uint4*>(ep.residual + (size_t)row * ep.ldr + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w = r4[q];
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float2 f = unpack_bf16x2(ws[h]);
        v[q * 8 + h * 2] += f.x;
        v[q * 8 + h * 2 + 1] += f.y;
      }
    }
  }
  if (ep.relu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
  }
  if (ep.out_f32) {
    float* dst = reinterpret_cast<float*>(ep.out) + (size_t)row * ep.ldc + col0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      st_global_v4(dst + q * 4, __float_as_uint(v[q * 4]), __float_as_uint(v[q * 4 + 1]),
                   __float_as_uint(v[q * 4 + 2]), __float_as_uint(v[q * 4 + 3]));
  } else {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(ep.out) + (size_t)row * ep.ldc + col0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      st_global_v4(dst + q * 8, pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]),
                   pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]), pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]),
                   pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]));
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_b, int M, int N, int K,
                        GemmEpilogue ep) {
  using Cfg = GemmCfg<BN>;
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
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + kBK - 1) / kBK;

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
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      const uint64_t pol_w = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m_blk = t % num_m;
        const int n_blk = t / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          tma_load_2d(sA + stage * Cfg::kABytes, &tmap_a, &full_bar[stage], kb * kBK, m_blk * kBM);
          tma_load_2d_hint(sB + stage * Cfg::kBBytes, &tmap_b, &full_bar[stage], kb * kBK, n_blk * BN,
                           pol_w);
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
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * Cfg::kABytes));
          const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * Cfg::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // +32 bytes along K inside the swizzle atom == +2 in the (addr >> 4) field
            umma_bf16_ss(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
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
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int m_blk = t % num_m;
      const int n_blk = t / num_m;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * kBM + ew * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int col0 = n_blk * BN + c * 32;
        if (row < M && col0 < N) epilogue_chunk(ep, row, col0, r);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
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

template <int BN>
static cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                             const GemmEpilogue& ep, int max_ctas, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (tiles < grid) grid = tiles;
  gemm_bf16_tn_kernel<BN><<<grid, kThreads, Cfg::kSmemBytes, stream>>>(ta, tb, M, N, K, ep);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int bn,
                        const GemmEpilogue& ep, int max_ctas, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (bn == 256) return launch_bn<256>(ta, tb, M, N, K, ep, max_ctas, stream);
  return launch_bn<128>(ta, tb, M, N, K, ep, max_ctas, stream);
}

int pick_block_n(int M, int N) {
  // Prefer the wider tile unless it leaves most SMs idle or N is not a multiple of 256.
  if (N % 256 != 0) return 128;
  const int tiles256 = ((M + kBM - 1) / kBM) * (N / 256);
  if (tiles256 < num_sms() / 2) return 128;
  return 256;
}

}  // namespace ag
