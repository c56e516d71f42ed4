// Mixed prefill+decode paged attention on sm_100a, one launch per layer.
//
// Work list (host-built in capi.cu build_attention_work), one launch, two CTA kinds:
//
//  * TILE CTAs (one per (query tile, head, KV split)): a prefill chunk's rows in tiles of 128.
//    TMA stages Q (128x128) once and K/V 128 tokens (four 32-token pages) per stage from the
//    paged pool into a 3-deep SW128 ring.  One thread issues tcgen05.mma:
//        S_j  = Q . K_j^T   (M=128, N=128, K=128)  -> TMEM (double-buffered, 2 x 128 columns)
//        O   += P_j . V_j   (A = P from TMEM, B = V MN-major)  -> TMEM (128 columns)
//    Four softmax warps own one query row per thread: tcgen05.ld the S row, causal/range mask,
//    online softmax in the exp2 domain with lazy O rescaling (only when the row max grows by
//    more than 2^8; the rescale is a tcgen05.ld/st round trip of the O row), tcgen05.st P as
//    packed bf16 pairs over the first 64 columns of the S buffer, signal the MMA warp.
//    Warp roles (192 threads): w0 TMA producer | w1 MMA issuer + TMEM owner | w2..w5 softmax.
//
//  * ROW CTAs (six (row, head, KV split) units per CTA, one per warp): decode tokens and rows
//    of tiny chunks.  Each warp streams its KV range page by page through its own 2-deep TMA ring
//    and runs QK^T / PV on mma.sync with the query as row 0 of the A tile -- this path is HBM-bound.
//
// Split-KV partial rows (O normalised, plus (m, l) in the log2 domain) are merged by
// attn_combine_kernel.  Causality: query row i of a chunk sits at position ctx_len + q_start + i.
#include "common.cuh"
#include "kernels.h"

namespace ag {
namespace {

constexpr int kHD = 128;
constexpr int kPage = 32;
constexpr int kRowBytes = kHD * 2;
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThresh = 8.0f;  // log2 units: P <= 2^8 between O rescales

// ---- tile path layout
constexpr int kTM = 128, kTN = 128;
constexpr int kSub = 128 * 64 * 2;                  // one [128 rows][64] bf16 SW128 sub-tile = 16 KB
constexpr int kQOff = 0;                            // Q: 2 sub-tiles (dims 0-63, 64-127)
constexpr int kKVOff = 2 * kSub;                    // stage s: K 2 sub-tiles, V 2 sub-tiles (64 KB)
constexpr int kStageBytes = 4 * kSub;
constexpr int kKVStages = 3;                        // P lives in TMEM, so three K/V stages fit
#ifndef AG_ATTN_SBUF
#define AG_ATTN_SBUF 3
#endif
constexpr int kSBuf = AG_ATTN_SBUF;                 // S/P buffers in TMEM (128 columns each)
constexpr uint32_t kOCol = kSBuf * 128;             // O accumulator columns
static_assert(kSBuf * 128 + 128 <= 512, "TMEM: S buffers + O must fit 512 columns");
constexpr int kBarOff = kKVOff + kKVStages * kStageBytes;  // 224 KB
constexpr int kTileSmem = kBarOff + 256;
// ---- row path layout (per warp): kRowStages pages of 32 tokens; a stage is
//   [K dims 0-63 | K dims 64-127 | V dims 0-63 | V dims 64-127], each 32 rows x 128 B, TMA SW128
constexpr int kRowStages = 2;
constexpr int kRowHalf = 32 * 64 * 2;                          // 4 KB
constexpr int kRowStageBytes = 4 * kRowHalf;                   // 16 KB
constexpr int kRowWarpBytes = kRowStages * kRowStageBytes;     // 32 KB per warp, 6 warps = 192 KB
constexpr int kRowBarOff = 6 * kRowWarpBytes;                  // + 6 warps x kRowStages mbarriers
constexpr int kRowSmem = kRowBarOff + 6 * kRowStages * 8;
constexpr int kSmemBytes = 1024 + (kTileSmem > kRowSmem ? kTileSmem : kRowSmem);

// 2^x on the SFU without the denormal range fix-up of exp2f (arguments here are <= 0).
AG_DEVICE float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

AG_DEVICE void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

AG_DEVICE void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
AG_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MN-major SW128 operand (V as the B of P.V): 64-element MN blocks `lbo` bytes apart, 8-row K
// groups 1024 B apart.
AG_DEVICE uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// D(TMEM) (+)= A(TMEM, K-major bf16 pairs per 32-bit column) . B(smem descriptor)
AG_DEVICE void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// ---------------------------------------------------------------- row (decode) path
AG_DEVICE void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
AG_DEVICE void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D += A(16x16, rows 1..15 zero here) . B(16x8), bf16 in, f32 accumulate
AG_DEVICE void mma_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// Byte offset of 16-B chunk cc (0..7) of row r inside a TMA SWIZZLE_128B [rows][64] bf16 box.
AG_DEVICE uint32_t sw128(int r, int cc) { return static_cast<uint32_t>(r * 128 + ((cc ^ (r & 7)) << 4)); }

// One warp streams one (query row, head, KV range) unit: TMA brings each 32-token page of K and V
// (the same SW128 boxes as the tile path) into a 2-deep ring; QK^T and PV run on mma.sync with the
// single query row as row 0 of the A operand (lanes 0-3 hold it), so a 32-token page costs 32
// ldmatrix + 64 mma per warp instead of ~1.6k CUDA-core instructions.  Online softmax in the exp2
// domain; lanes 0-3 own the row's running max, partial sums and O (C-fragment columns 2t, 2t+1).
AG_DEVICE void decode_row_warp(const AttnParams& p, const AttnTmaps& tm, const AttnItem& it, int head,
                               uint8_t* wsmem, uint64_t* bars) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int tok_row = p.cu_q[it.seq] + it.q_start;
  const int qpos = p.ctx_len[it.seq] + it.q_start;
  const int kv_lo = it.kv_start;
  const int kv_hi = min(it.kv_end, qpos + 1);
  const int pg0 = kv_lo / kPage;
  const int n_pages = kv_hi > kv_lo ? (kv_hi + kPage - 1) / kPage - pg0 : 0;
  const int32_t* bt = p.block_table + static_cast<int64_t>(it.seq) * p.bt_stride;
  const uint32_t sbase = smem_u32(wsmem);

  if (lane == 0) {
    for (int st = 0; st < kRowStages; ++st) mbar_init(&bars[st], 1);
    fence_barrier_init();
  }
  __syncwarp();
  auto issue = [&](int i) {  // lane 0: page pg0 + i into stage i % kRowStages
    const int st = i % kRowStages;
    const int row = (bt[pg0 + i] * p.heads + head) * kPage;
    uint8_t* dst = wsmem + st * kRowStageBytes;
    mbar_arrive_expect_tx(&bars[st], kRowStageBytes);
    tma_load_2d(dst, &tm.k, &bars[st], 0, row);
    tma_load_2d(dst + kRowHalf, &tm.k, &bars[st], 64, row);
    tma_load_2d(dst + 2 * kRowHalf, &tm.v, &bars[st], 0, row);
    tma_load_2d(dst + 3 * kRowHalf, &tm.v, &bars[st], 64, row);
  };
  if (lane == 0)
    for (int i = 0; i < min(kRowStages, n_pages); ++i) issue(i);

  // q row as the A operand: lanes 0-3 hold dims (16kk + 2t, +1) and (16kk + 8 + 2t, +1)
  uint32_t qa[8][2];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) qa[kk][0] = qa[kk][1] = 0u;
  if (g == 0) {
    const uint32_t* q32 = reinterpret_cast<const uint32_t*>(p.q + static_cast<int64_t>(tok_row) * p.ldq + head * kHD);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = q32[kk * 8 + t];
      qa[kk][1] = q32[kk * 8 + 4 + t];
    }
  }
  float o[16][4];
#pragma unroll
  for (int d = 0; d < 16; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
  float m = -INFINITY, lpart = 0.f;

  for (int i = 0; i < n_pages; ++i) {
    const int st = i % kRowStages;
    mbar_wait(&bars[st], (i / kRowStages) & 1);
    const uint32_t kb = sbase + st * kRowStageBytes;
    const uint32_t vb = kb + 2 * kRowHalf;
    // S = q . K^T for the page's 32 tokens: 4 n-tiles of 8 tokens x 8 k-steps
    float sc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
      const int r = 8 * j + (lane & 7);
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {  // 16-B chunks 4mm .. 4mm+3 = k-steps 2mm, 2mm+1
        const int cg = 4 * mm + (lane >> 3);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kb + (cg >> 3) * kRowHalf + sw128(r, cg & 7), b0, b1, b2, b3);
        mma_16816(sc[j], qa[2 * mm][0], qa[2 * mm][1], b0, b1);
        mma_16816(sc[j], qa[2 * mm + 1][0], qa[2 * mm + 1][1], b2, b3);
      }
    }
    // online softmax over the page (row 0 lives in lanes 0-3: tokens 8j + 2t, +1)
    const int tok0 = (pg0 + i) * kPage;
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = tok0 + 8 * j + 2 * t + e;
        const bool ok = g == 0 && tok >= kv_lo && tok < kv_hi;
        sc[j][e] = ok ? sc[j][e] * kLog2e : -INFINITY;
        mx = fmaxf(mx, sc[j][e]);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mnew = fmaxf(m, mx);
    const float mref = mnew == -INFINITY ? 0.f : mnew;
    const float alpha = ex2_ftz(m - mref);
    m = mnew;
    uint32_t pa[4];  // P as bf16x2 per n-tile (row 0 only)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float p0 = ex2_ftz(sc[j][0] - mref), p1 = ex2_ftz(sc[j][1] - mref);
      lpart = lpart * (j == 0 ? alpha : 1.f) + p0 + p1;
      pa[j] = pack_bf16x2(p0, p1);
    }
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      o[d][0] *= alpha;
      o[d][1] *= alpha;
    }
    // O += P . V: 2 k-steps of 16 tokens x 16 n-tiles of 8 dims (V loaded transposed)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int r = 16 * ks + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
      for (int d = 0; d < 16; d += 2) {
        const int cg = d + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vb + (cg >> 3) * kRowHalf + sw128(r, cg & 7), b0, b1, b2, b3);
        mma_16816(o[d], pa[2 * ks], pa[2 * ks + 1], b0, b1);
        mma_16816(o[d + 1], pa[2 * ks], pa[2 * ks + 1], b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0 && i + kRowStages < n_pages) {
      fence_async_smem();
      issue(i + kRowStages);
    }
  }
  float l = lpart + __shfl_xor_sync(0xffffffffu, lpart, 1);
  l += __shfl_xor_sync(0xffffffffu, l, 2);
  if (g != 0) return;
  const float inv = l > 0.f ? 1.f / l : 0.f;
  if (it.part_row < 0) {
    __nv_bfloat16* dst = p.out + static_cast<int64_t>(tok_row) * p.ldo + head * kHD + 2 * t;
#pragma unroll
    for (int d = 0; d < 16; ++d)
      *reinterpret_cast<uint32_t*>(dst + 8 * d) = pack_bf16x2(o[d][0] * inv, o[d][1] * inv);
  } else {
    const int64_t prow = static_cast<int64_t>(it.part_row) * p.heads + head;
    float* dst = p.part_o + prow * kHD + 2 * t;
#pragma unroll
    for (int d = 0; d < 16; ++d) *reinterpret_cast<float2*>(dst + 8 * d) = make_float2(o[d][0] * inv, o[d][1] * inv);
    if (t == 0) {
      p.part_ml[prow * 2] = m;
      p.part_ml[prow * 2 + 1] = l;
    }
  }
}

// ---------------------------------------------------------------- tile (tcgen05) path
struct TileBars {
  uint64_t q_full;
  uint64_t kv_full[kKVStages], kv_empty[kKVStages];
  uint64_t s_full[kSBuf], s_empty[kSBuf];
  uint64_t p_full[kSBuf], o_done[2];
  uint32_t tmem_base;
};

#ifdef AG_ATTN_SPIN_WAIT
#define AG_TILE_WAIT mbar_wait_spin
#else
#define AG_TILE_WAIT mbar_wait
#endif

#ifdef AG_ATTN_TIMELINE  // timing probe only: per-CTA globaltimer stamps (entry, setup, loop end, exit)
__device__ unsigned long long g_attn_tl[16384 * 16];
AG_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define AG_TL(slot, v) g_attn_tl[blockIdx.x * 16 + (slot)] = (v)
#define AG_CLK(var) const long long var = clock64()
#define AG_ACC(var, v) var += (v)
#else
#define AG_TL(slot, v)
#define AG_CLK(var)
#define AG_ACC(var, v)
#endif

AG_DEVICE void tile_tc(const AttnParams& p, const AttnTmaps& tm, const AttnItem& it, int head, uint8_t* smem) {
#ifdef AG_ATTN_TIMELINE
  if (threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    AG_TL(0, gtimer());
    AG_TL(5, smid);
  }
#endif
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  TileBars* bars = reinterpret_cast<TileBars*>(smem + kBarOff);
  const int q0 = p.cu_q[it.seq];
  const int tok_row0 = q0 + it.q_start;
  const int ctx = p.ctx_len[it.seq];
  // KV tiles of 128 tokens from kv_start (a multiple of 128) to the causal end of the tile
  const int kv_end = min(it.kv_end, ctx + it.q_start + it.q_rows);
  const int n_tiles = (kv_end - it.kv_start + kTN - 1) / kTN;
  const uint32_t sb = smem_u32(smem);

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    for (int i = 0; i < kKVStages; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    for (int i = 0; i < kSBuf; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_empty[i], 4);
      mbar_init(&bars->p_full[i], 4);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&bars->o_done[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
#ifdef AG_ATTN_TIMELINE
  if (threadIdx.x == 0) AG_TL(1, gtimer());
#endif
  pdl_trigger();  // only after the TMEM allocation (see gemm_bf16_tn_kernel)
  pdl_wait();     // Q, the paged K/V and the outputs belong to the predecessor kernels
  const uint32_t tmem = bars->tmem_base;  // S buffers [128 i, 128 i + 128), O [kOCol, kOCol + 128)

  if (warp == 0) {
    if (lane == 0 && n_tiles > 0) {
      tma_prefetch_desc(&tm.q);
      tma_prefetch_desc(&tm.k);
      tma_prefetch_desc(&tm.v);
      mbar_arrive_expect_tx(&bars->q_full, 2 * kSub);
      tma_load_2d(smem + kQOff, &tm.q, &bars->q_full, head * kHD, tok_row0);
      tma_load_2d(smem + kQOff + kSub, &tm.q, &bars->q_full, head * kHD + 64, tok_row0);
      const int32_t* bt = p.block_table + static_cast<int64_t>(it.seq) * p.bt_stride;
      const int last_page = (kv_end - 1) / kPage;
      long long c_ke = 0;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % kKVStages;
        AG_CLK(e0);
        mbar_wait(&bars->kv_empty[st], ((j / kKVStages) & 1) ^ 1);
        AG_CLK(e1);
        AG_ACC(c_ke, e1 - e0);
#ifdef AG_ATTN_PROBE_NOTMA  // timing probe only: K/V stages are not loaded (MMAs read stale smem)
        mbar_arrive(&bars->kv_full[st]);
        continue;
#endif
        mbar_arrive_expect_tx(&bars->kv_full[st], kStageBytes);
        uint8_t* kdst = smem + kKVOff + st * kStageBytes;
        uint8_t* vdst = kdst + 2 * kSub;
        for (int pg = 0; pg < 4; ++pg) {
          int page = (it.kv_start + j * kTN) / kPage + pg;
          page = page > last_page ? last_page : page;  // masked padding page
          const int row = (bt[page] * p.heads + head) * kPage;
          tma_load_2d(kdst + pg * 4096, &tm.k, &bars->kv_full[st], 0, row);
          tma_load_2d(kdst + kSub + pg * 4096, &tm.k, &bars->kv_full[st], 64, row);
          tma_load_2d(vdst + pg * 4096, &tm.v, &bars->kv_full[st], 0, row);
          tma_load_2d(vdst + kSub + pg * 4096, &tm.v, &bars->kv_full[st], 64, row);
        }
      }
      AG_TL(13, c_ke);
    }
  } else if (warp == 1) {
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(kTM, kTN);
      constexpr uint32_t idesc_o = umma_idesc_bf16(kTM, kHD) | (1u << 16);  // B (V) MN-major
      mbar_wait(&bars->q_full, 0);
      long long c_kv = 0, c_se = 0, c_pf = 0;
      auto issue_s = [&](int j) {
        const int st = j % kKVStages, sbuf = j % kSBuf;
        AG_CLK(k0);
        mbar_wait(&bars->kv_full[st], (j / kKVStages) & 1);
        AG_CLK(k1);
        mbar_wait(&bars->s_empty[sbuf], ((j / kSBuf) & 1) ^ 1);
        AG_CLK(k2);
        AG_ACC(c_kv, k1 - k0);
        AG_ACC(c_se, k2 - k1);
        tc_fence_after();
        const uint32_t kaddr = sb + kKVOff + st * kStageBytes;
#ifndef AG_ATTN_PROBE_NOS  // timing probe only: skip the S MMAs
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t a = umma_desc_sw128(sb + kQOff + (k >> 2) * kSub) + 2 * (k & 3);
          const uint64_t b = umma_desc_sw128(kaddr + (k >> 2) * kSub) + 2 * (k & 3);
          umma_bf16_ss(tmem + sbuf * 128, a, b, idesc_s, k > 0 ? 1u : 0u);
        }
#endif
        umma_commit(&bars->s_full[sbuf]);
      };
      // O += P_j . V_j with P_j (bf16, packed in columns 0-63 of its S buffer) as the TMEM A operand
      auto issue_pv = [&](int j) {
        const int pb = j % kSBuf, st = j % kKVStages;
        AG_CLK(p0);
        AG_TILE_WAIT(&bars->p_full[pb], (j / kSBuf) & 1);
        AG_CLK(p1);
        AG_ACC(c_pf, p1 - p0);
        tc_fence_after();
        const uint32_t ptmem = tmem + pb * 128;
        const uint32_t vaddr = sb + kKVOff + st * kStageBytes + 2 * kSub;
#ifndef AG_ATTN_PROBE_NOPV  // timing probe only: skip the P.V MMAs
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 tokens per MMA = 8 TMEM columns of packed bf16 pairs
          const uint64_t b = umma_desc_sw128_mn(vaddr + k * 2048, kSub);
          umma_bf16_ts(tmem + kOCol, ptmem + 8 * k, b, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        }
#endif
        umma_commit(&bars->o_done[j & 1]);
        umma_commit(&bars->kv_empty[st]);
      };
      if constexpr (kSBuf == 2) {  // S_{j+1} is queued before P_j is awaited
        issue_s(0);
        for (int j = 0; j < n_tiles; ++j) {
          if (j + 1 < n_tiles) issue_s(j + 1);
          issue_pv(j);
        }
      } else {  // S_{j+1}, S_{j+2} run ahead: the softmax never waits for S on the S -> P -> PV loop
        for (int j = 0; j < kSBuf - 1 && j < n_tiles; ++j) issue_s(j);
        for (int j = 0; j < n_tiles; ++j) {
          issue_pv(j);
          if (j + kSBuf - 1 < n_tiles) issue_s(j + kSBuf - 1);
        }
      }
      AG_TL(10, c_pf);
      AG_TL(11, c_kv);
      AG_TL(12, c_se);
    }
  } else {
    // ---------------- softmax / epilogue warps: one query row per thread
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    const bool row_ok = row < it.q_rows;
    const int qpos = ctx + it.q_start + row;
    float m_used = -INFINITY, l = 0.f;
    long long c_w = 0, c_ld = 0, c_mx = 0, c_ex = 0;
    for (int j = 0; j < n_tiles; ++j) {
      const int sbuf = j % kSBuf;
      AG_CLK(t0);
      AG_TILE_WAIT(&bars->s_full[sbuf], (j / kSBuf) & 1);
      tc_fence_after();
      AG_CLK(t1);
      AG_ACC(c_w, t1 - t0);
#ifdef AG_ATTN_PIPE_PROBE  // timing probe only: skip the softmax, keep the barrier protocol
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bars->s_empty[sbuf]);
        mbar_arrive(&bars->p_full[sbuf]);
      }
      continue;
#endif
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
#ifdef AG_ATTN_PROBE_NOLDS  // timing probe only: S not read from TMEM (synthetic scores)
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(0.01f * (lane ^ (c * 32 + i)) + 0.001f * j);
#else
        tmem_ld_32x32b_x32(tmem + lane_addr + sbuf * 128 + c * 32, r);
        tmem_ld_wait();
#endif
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->s_empty[sbuf]);
      AG_CLK(t2);
      AG_ACC(c_ld, t2 - t1);
      const int kbase = it.kv_start + j * kTN;
      // Only the tiles that cross a row's causal / range end need a mask (CTA-uniform test on
      // row 0, the row with the earliest end); rows past q_rows are never stored.
      if (kbase + kTN > min(kv_end, ctx + it.q_start + 1)) {
        const int lim = row_ok ? min(kv_end, qpos + 1) - kbase : 0;  // valid columns [0, lim)
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = c < lim ? s[c] : -INFINITY;
      }
      float m8[8];  // 8 independent max chains (a single 128-long fmax chain is latency-bound)
#pragma unroll
      for (int i = 0; i < 8; ++i) m8[i] = s[i];
#pragma unroll
      for (int c = 8; c < 128; ++c) m8[c & 7] = fmaxf(m8[c & 7], s[c]);
      float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      mx *= kLog2e;  // scores stay raw; the log2(e) scale is folded into the exponent's FMA
      // Lazy rescale: a row whose running max grew by more than 2^8 rescales l and its O row
      // (after every earlier P.V finished).  tcgen05.ld/st are .sync.aligned, so the decision to
      // touch TMEM is warp-uniform; rows that did not grow scale by 1.
      const bool grow = mx > m_used + kRescaleThresh;
      if (__any_sync(0xffffffffu, grow)) {
        const float alpha = grow ? ex2_ftz(m_used - mx) : 1.0f;  // 0 on a row's first visit
        if (__any_sync(0xffffffffu, grow && j > 0 && m_used != -INFINITY)) {
          mbar_wait(&bars->o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem + lane_addr + kOCol + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_addr + kOCol + c * 32, r);
          }
          tmem_st_wait();
          tc_fence_before();
        }
        if (grow) {
          l *= alpha;
          m_used = mx;
        }
      }
      const float mref = m_used == -INFINITY ? 0.f : m_used;
      AG_CLK(t3);
      AG_ACC(c_mx, t3 - t2);
      // P_j (bf16 pairs) -> columns 0-63 of this tile's S buffer; S_j is already in registers and
      // the MMA pipe runs P.V_j before the S_{j+2} that next overwrites the buffer (in-order issue)
      float rs2[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial row sums
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
#ifdef AG_ATTN_PROBE_NOEXP  // timing probe only: no MUFU (values are wrong)
          const float e0 = fmaf(s[half * 64 + 2 * i], kLog2e, -mref);
          const float e1 = fmaf(s[half * 64 + 2 * i + 1], kLog2e, -mref);
#else
          const float e0 = ex2_ftz(fmaf(s[half * 64 + 2 * i], kLog2e, -mref));
          const float e1 = ex2_ftz(fmaf(s[half * 64 + 2 * i + 1], kLog2e, -mref));
#endif
          rs2[i & 3] += e0 + e1;
          pk[i] = pack_bf16x2(e0, e1);
        }
        tmem_st_32x32b_x32(tmem + lane_addr + sbuf * 128 + half * 32, pk);
      }
      tmem_st_wait();
      l += (rs2[0] + rs2[1]) + (rs2[2] + rs2[3]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_full[sbuf]);
      AG_CLK(t4);
      AG_ACC(c_ex, t4 - t3);
    }
#ifdef AG_ATTN_TIMELINE
    if (threadIdx.x == 64) {
      AG_TL(2, gtimer());
      AG_TL(4, n_tiles);
      AG_TL(6, c_w);
      AG_TL(7, c_ld);
      AG_TL(8, c_mx);
      AG_TL(9, c_ex);
    }
#endif
    // epilogue: O row / l
    if (n_tiles > 0) {
      mbar_wait(&bars->o_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
      tc_fence_after();
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      if (n_tiles > 0) {
        tmem_ld_32x32b_x32(tmem + lane_addr + kOCol + c * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = 0u;
      }
      if (!row_ok) continue;
      if (it.part_row < 0) {
        __nv_bfloat16* dst = p.out + static_cast<int64_t>(tok_row0 + row) * p.ldo + head * kHD + c * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_global_v4(dst + q * 8, pack_bf16x2(__uint_as_float(r[q * 8]) * inv, __uint_as_float(r[q * 8 + 1]) * inv),
                       pack_bf16x2(__uint_as_float(r[q * 8 + 2]) * inv, __uint_as_float(r[q * 8 + 3]) * inv),
                       pack_bf16x2(__uint_as_float(r[q * 8 + 4]) * inv, __uint_as_float(r[q * 8 + 5]) * inv),
                       pack_bf16x2(__uint_as_float(r[q * 8 + 6]) * inv, __uint_as_float(r[q * 8 + 7]) * inv));
      } else {
        const int64_t prow = static_cast<int64_t>(it.part_row + row) * p.heads + head;
        float* dst = p.part_o + prow * kHD + c * 32;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_global_v4(dst + q * 4, __float_as_uint(__uint_as_float(r[q * 4]) * inv),
                       __float_as_uint(__uint_as_float(r[q * 4 + 1]) * inv),
                       __float_as_uint(__uint_as_float(r[q * 4 + 2]) * inv),
                       __float_as_uint(__uint_as_float(r[q * 4 + 3]) * inv));
        if (c == 0) {
          p.part_ml[prow * 2] = m_used;
          p.part_ml[prow * 2 + 1] = l;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef AG_ATTN_TIMELINE
  if (threadIdx.x == 0) AG_TL(3, gtimer());
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    mixed_attention_kernel(AttnParams p, const __grid_constant__ AttnTmaps tm, const AttnItem* __restrict__ items,
                           int n_tile_items, int n_row_items) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int n_tile_ctas = n_tile_items * p.heads;
  // The tile CTAs (tensor-bound) are spread evenly through the grid, tile i at block
  // floor(i * C / T), so they run concurrently with the HBM-bound decode-row CTAs from the first
  // wave on instead of occupying the SMs ahead of them.
  const long long C = gridDim.x, T = n_tile_ctas, b = blockIdx.x;
  const long long ti = T > 0 ? (b * T + C - 1) / C : 0;  // the only tile index that can sit at b
  if (ti < T && ti * C / T == b) {
    // head-major: the q tiles / splits of one head run side by side and share its K/V in L2
    const AttnItem it = items[ti % n_tile_items];
    tile_tc(p, tm, it, static_cast<int>(ti / n_tile_items), smem);
    return;
  }
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5;
  const int row_cta = static_cast<int>(b - (T > 0 ? ((b + 1) * T + C - 1) / C : 0));  // tiles at or before b
  const int u = row_cta * (kThreads / 32) + warp;
  if (u >= n_row_items * p.heads) return;
  const AttnItem itr = items[n_tile_items + u / p.heads];
  decode_row_warp(p, tm, itr, u % p.heads, smem + warp * kRowWarpBytes,
                  reinterpret_cast<uint64_t*>(smem + kRowBarOff) + warp * kRowStages);
}

// Merge split-KV partial rows: out = sum_s w_s O_s / sum_s w_s, w_s = l_s * 2^(m_s - M).
// One warp per (query row, head), four head dims per lane; splits of a row sit `q_rows` apart.
__global__ void __launch_bounds__(256) attn_combine_kernel(AttnParams p, const AttnCombine* __restrict__ combines,
                                                           int n_combines) {
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (unit >= n_combines * p.heads) return;
  const int lane = threadIdx.x & 31;
  const AttnCombine cb = combines[unit / p.heads];
  const int head = unit % p.heads;
  float mmax = -INFINITY;
  for (int sp = 0; sp < cb.n_splits; ++sp) {
    const int64_t prow = static_cast<int64_t>(cb.first_part + sp * cb.q_rows) * p.heads + head;
    mmax = fmaxf(mmax, p.part_ml[prow * 2]);
  }
  const float mref = mmax == -INFINITY ? 0.0f : mmax;
  float lsum = 0.0f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int sp = 0; sp < cb.n_splits; ++sp) {
    const int64_t prow = static_cast<int64_t>(cb.first_part + sp * cb.q_rows) * p.heads + head;
    const float w = p.part_ml[prow * 2 + 1] * exp2f(p.part_ml[prow * 2] - mref);
    const float4 o = *reinterpret_cast<const float4*>(p.part_o + prow * kHD + lane * 4);
    lsum += w;
    acc.x += w * o.x;
    acc.y += w * o.y;
    acc.z += w * o.z;
    acc.w += w * o.w;
  }
  const float inv = lsum > 0.0f ? 1.0f / lsum : 0.0f;
  __nv_bfloat16* dst = p.out + static_cast<int64_t>(cb.tok_row) * p.ldo + head * kHD + lane * 4;
  *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(acc.x * inv, acc.y * inv), pack_bf16x2(acc.z * inv, acc.w * inv));
}

}  // namespace

#ifdef AG_ATTN_TIMELINE
extern "C" __attribute__((visibility("default"))) int ag_debug_attn_timeline(void* dst, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(dst, g_attn_tl, sizeof(unsigned long long) * 16 * n));
}
#endif

int attention_tile_rows() { return kTM; }
int attention_tile_kv() { return kTN; }

cudaError_t launch_attention(const AttnParams& p, const AttnTmaps& tm, const AttnItem* items, int n_tile_items,
                             int n_row_items, const AttnCombine* combines, int n_combines, cudaStream_t stream) {
  if (p.block_size != kPage) return cudaErrorInvalidValue;
  if (n_tile_items + n_row_items > 0) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e =
          cudaFuncSetAttribute(mixed_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    const int ctas = n_tile_items * p.heads + (n_row_items * p.heads + kThreads / 32 - 1) / (kThreads / 32);
    (void)launch_k(kPdlAttn, mixed_attention_kernel, ctas, kThreads, kSmemBytes, stream, p, tm, items, n_tile_items, n_row_items);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (n_combines > 0) {
    const int units = n_combines * p.heads;
    (void)launch_k(kPdlAttn, attn_combine_kernel, (units + 7) / 8, 256, 0, stream, p, combines, n_combines);
    return cudaGetLastError();
  }
  return cudaSuccess;
}

}  // namespace ag
