// Mixed prefill+decode paged attention, one launch per layer.
//
// Work list (host-built, see capi.cu build_attention_work): every item is a query tile of one
// sequence (<= 64 rows of a prefill chunk, or <= 16 rows such as a single decode token) against
// a KV range [kv_start, kv_end) of that sequence's paged cache.  Long ranges are split across
// CTAs (split-KV); their partial (O, lse) rows are merged by attn_combine_kernel.
//
// grid = (items, heads), 128 threads.  KV is streamed 64 tokens (two 32-token pages) per stage
// through a double-buffered, XOR-swizzled shared-memory ring with cp.async; QK^T and PV run
// on mma.sync m16n8k16 (bf16 -> f32) with an online softmax in the exp2 domain.
//   prefill tile (q_rows > 16): warp w owns query rows 16w..16w+15 against all 64 stage tokens;
//   decode tile (q_rows <= 16): all warps share rows 0..15, warp w owns stage tokens 16w..16w+15,
//                               and the four partial softmax states are merged through smem.
// Causality: query row i of a chunk sits at position ctx_len + q_start + i and sees kv <= it.
#include "common.cuh"
#include "kernels.h"

namespace ag {
namespace {

constexpr int kHD = 128;         // head dim
constexpr int kPage = 32;        // tokens per KV block
constexpr int kStageTok = 64;    // tokens per pipeline stage
constexpr int kRowBytes = kHD * 2;
constexpr int kStageBytes = 2 * kStageTok * kRowBytes;  // K + V = 32 KB
constexpr int kStages = 2;
constexpr int kAttnThreads = 128;
constexpr int kDecHalf = 16;                              // tokens per decode ring slot (half page)
constexpr int kDecSlotBytes = 2 * kDecHalf * kRowBytes;   // K + V = 8 KB
constexpr int kDecStages = 3;
constexpr int kDecWarpBytes = kDecStages * kDecSlotBytes;  // 24 KB per warp
constexpr int kAttnSmem = 4 * kDecWarpBytes;               // 96 KB >= tile path 64 KB
constexpr float kLog2e = 1.4426950408889634f;

AG_DEVICE void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
AG_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
AG_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

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

AG_DEVICE void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte offset of (token, 16-byte chunk) inside a swizzled [64][128] bf16 tile
AG_DEVICE uint32_t swz(int token, int chunk) {
  return static_cast<uint32_t>(token * kRowBytes + ((chunk ^ (token & 7)) << 4));
}

struct Softmax2 {  // per-thread state for its two rows (g, g+8)
  float m[2];
  float l[2];
};

// One warp's pass over NT tokens [tok0, tok0+NT) of the current stage.
template <int NT>
AG_DEVICE void attend_stage(uint32_t sK, uint32_t sV, int tok0, const uint32_t (&qf)[8][4],
                            float (&o)[16][4], Softmax2& st, int stage_pos0, int kv_end,
                            const int (&qpos)[2]) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  constexpr int NTILE = NT / 8;
  float s[NTILE][4];
#pragma unroll
  for (int n = 0; n < NTILE; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.0f;

  // S = Q K^T
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
    for (int np = 0; np < NTILE / 2; ++np) {
      const int mat = lane >> 3, r = lane & 7;
      const int token = tok0 + np * 16 + r + 8 * (mat >> 1);
      const int chunk = 2 * ks + (mat & 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(sK + swz(token, chunk), b0, b1, b2, b3);
      mma_bf16(s[2 * np], qf[ks], b0, b1);
      mma_bf16(s[2 * np + 1], qf[ks], b2, b3);
    }
  }

  // mask + online softmax (log2 domain)
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int n = 0; n < NTILE; ++n) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = e >> 1;
      const int pos = stage_pos0 + tok0 + n * 8 + 2 * t + (e & 1);
      const bool ok = pos < kv_end && pos <= qpos[row];
      const float v = ok ? s[n][e] * kLog2e : -INFINITY;
      s[n][e] = v;
      mx[row] = fmaxf(mx[row], v);
    }
  }
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    mx[row] = fmaxf(mx[row], __shfl_xor_sync(0xffffffffu, mx[row], 1));
    mx[row] = fmaxf(mx[row], __shfl_xor_sync(0xffffffffu, mx[row], 2));
  }
  float alpha[2], mref[2], rs[2] = {0.0f, 0.0f};
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    const float mnew = fmaxf(st.m[row], mx[row]);
    mref[row] = (mnew == -INFINITY) ? 0.0f : mnew;
    alpha[row] = exp2f(st.m[row] - mref[row]);  // exp2(-inf) = 0 on the first visit
    st.m[row] = mnew;
  }
#pragma unroll
  for (int n = 0; n < NTILE; ++n) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float p = exp2f(s[n][e] - mref[e >> 1]);
      s[n][e] = p;
      rs[e >> 1] += p;
    }
  }
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    rs[row] += __shfl_xor_sync(0xffffffffu, rs[row], 1);
    rs[row] += __shfl_xor_sync(0xffffffffu, rs[row], 2);
    st.l[row] = st.l[row] * alpha[row] + rs[row];
  }
#pragma unroll
  for (int d = 0; d < 16; ++d) {
    o[d][0] *= alpha[0];
    o[d][1] *= alpha[0];
    o[d][2] *= alpha[1];
    o[d][3] *= alpha[1];
  }

  // O += P V
#pragma unroll
  for (int j = 0; j < NT / 16; ++j) {
    uint32_t a[4];
    a[0] = pack_bf16x2(s[2 * j][0], s[2 * j][1]);
    a[1] = pack_bf16x2(s[2 * j][2], s[2 * j][3]);
    a[2] = pack_bf16x2(s[2 * j + 1][0], s[2 * j + 1][1]);
    a[3] = pack_bf16x2(s[2 * j + 1][2], s[2 * j + 1][3]);
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      const int mat = lane >> 3, r = lane & 7;
      const int token = tok0 + 16 * j + r + 8 * (mat & 1);
      const int chunk = 2 * dp + (mat >> 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(sV + swz(token, chunk), b0, b1, b2, b3);
      mma_bf16(o[2 * dp], a, b0, b1);
      mma_bf16(o[2 * dp + 1], a, b2, b3);
    }
  }
}

// ---------------------------------------------------------------- single-row (decode) path
// One warp streams the KV range of one (sequence, head, split) through its own 3-slot cp.async
// ring of 16-token half pages (8 KB: K then V), independent of the other warps of the CTA.
//   QK^T: lanes 0-15 / 16-31 take token 2i / 2i+1 of a slot, 8 dims (one 16-B chunk) each, and
//         reduce over their 16 lanes -> every lane holds the score of its token pair member;
//   PV:   lane l owns output dims 4l..4l+3 and walks the slot's 16 tokens (coalesced 256-B rows).
AG_DEVICE void decode_row_warp(const AttnParams& p, const AttnItem& it, int head, uint8_t* wsmem) {
  const int lane = lane_id();
  const int q0 = p.cu_q[it.seq];
  const int tok_row = q0 + it.q_start;
  const int qpos = p.ctx_len[it.seq] + it.q_start;
  const int kv_end = min(it.kv_end, qpos + 1);
  const int chunk = lane & 15;
  // q chunk for the QK phase (pre-scaled by head_dim^-0.5 in the QKV epilogue), folded with log2e
  float qv[8];
  {
    const uint4 w = *reinterpret_cast<const uint4*>(p.q + static_cast<int64_t>(tok_row) * p.ldq + head * kHD + chunk * 8);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 f = unpack_bf16x2(ws[h]);
      qv[2 * h] = f.x * kLog2e;
      qv[2 * h + 1] = f.y * kLog2e;
    }
  }
  const int32_t* bt = p.block_table + static_cast<int64_t>(it.seq) * p.bt_stride;
  const int64_t page_elems = static_cast<int64_t>(p.heads) * kPage * kHD;
  const int64_t head_off = static_cast<int64_t>(head) * kPage * kHD;
  const int h0 = it.kv_start / kDecHalf;
  const int h1 = (kv_end + kDecHalf - 1) / kDecHalf;
  const uint32_t sbase = smem_u32(wsmem);

  auto issue = [&](int h, int slot) {
    const int page = (h * kDecHalf) / kPage;
    const int tok0 = (h * kDecHalf) % kPage;
    const int64_t base = static_cast<int64_t>(bt[page]) * page_elems + head_off + static_cast<int64_t>(tok0) * kHD;
    const uint32_t sk = sbase + slot * kDecSlotBytes;
    const uint32_t sv = sk + kDecHalf * kRowBytes;
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // 16 rows x 16 chunks = 256 x 16 B per tensor, 8 per lane
      const int id = lane + 32 * i;
      cp_async16(sk + id * 16, p.kcache + base + id * 8);
      cp_async16(sv + id * 16, p.vcache + base + id * 8);
    }
  };

  float o[4] = {0.f, 0.f, 0.f, 0.f};
  float m = -INFINITY, l = 0.f;
  int issued = h0;
  for (int k = 0; k < kDecStages - 1; ++k) {
    if (issued < h1) issue(issued, (issued - h0) % kDecStages);
    ++issued;
    cp_async_commit();
  }
  for (int h = h0; h < h1; ++h) {
    if (issued < h1) issue(issued, (issued - h0) % kDecStages);
    ++issued;
    cp_async_commit();
    cp_async_wait<kDecStages - 1>();
    __syncwarp();
    const int slot = (h - h0) % kDecStages;
    const uint8_t* sk = wsmem + slot * kDecSlotBytes;
    const uint8_t* sv = sk + kDecHalf * kRowBytes;
    // scores: lane keeps token (lane & 15)
    float s_mine = -INFINITY;
#pragma unroll
    for (int i = 0; i < kDecHalf / 2; ++i) {
      const int t = 2 * i + (lane >> 4);
      const uint4 w = *reinterpret_cast<const uint4*>(sk + t * kRowBytes + chunk * 16);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      float d = 0.f;
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        const float2 f = unpack_bf16x2(ws[hh]);
        d = fmaf(qv[2 * hh], f.x, d);
        d = fmaf(qv[2 * hh + 1], f.y, d);
      }
#pragma unroll
      for (int o2 = 8; o2 > 0; o2 >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o2);
      // lanes 0-15 now hold token 2i, lanes 16-31 token 2i+1; lane keeps token (lane & 15)
      const float other = __shfl_sync(0xffffffffu, d, (lane & 1) * 16);
      if ((lane & 15) >> 1 == i) s_mine = other;
    }
    const int pos = h * kDecHalf + (lane & 15);
    if (pos >= kv_end || pos < it.kv_start) s_mine = -INFINITY;
    float mx = s_mine;
#pragma unroll
    for (int o2 = 8; o2 > 0; o2 >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
    const float mnew = fmaxf(m, mx);
    const float mref = mnew == -INFINITY ? 0.f : mnew;
    const float alpha = exp2f(m - mref);
    const float pe = exp2f(s_mine - mref);
    float ps = pe;
#pragma unroll
    for (int o2 = 8; o2 > 0; o2 >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o2);
    l = l * alpha + ps;
    m = mnew;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] *= alpha;
#pragma unroll
    for (int t = 0; t < kDecHalf; ++t) {
      const float pt = __shfl_sync(0xffffffffu, pe, t);
      const uint2 w = *reinterpret_cast<const uint2*>(sv + t * kRowBytes + lane * 8);
      const float2 a = unpack_bf16x2(w.x), b = unpack_bf16x2(w.y);
      o[0] = fmaf(pt, a.x, o[0]);
      o[1] = fmaf(pt, a.y, o[1]);
      o[2] = fmaf(pt, b.x, o[2]);
      o[3] = fmaf(pt, b.y, o[3]);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  const float inv = l > 0.f ? 1.f / l : 0.f;
  if (it.part_row < 0) {
    __nv_bfloat16* dst = p.out + static_cast<int64_t>(tok_row) * p.ldo + head * kHD + lane * 4;
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(o[0] * inv, o[1] * inv), pack_bf16x2(o[2] * inv, o[3] * inv));
  } else {
    const int64_t prow = static_cast<int64_t>(it.part_row) * p.heads + head;
    *reinterpret_cast<float4*>(p.part_o + prow * kHD + lane * 4) = make_float4(o[0] * inv, o[1] * inv, o[2] * inv, o[3] * inv);
    if (lane == 0) {
      p.part_ml[prow * 2] = m;
      p.part_ml[prow * 2 + 1] = l;
    }
  }
}

__global__ void __launch_bounds__(kAttnThreads)
    mixed_attention_kernel(AttnParams p, const AttnItem* __restrict__ items, int n_tile_items, int n_row_items) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int n_tile_ctas = n_tile_items * p.heads;
  if (static_cast<int>(blockIdx.x) >= n_tile_ctas) {
    const int u = (blockIdx.x - n_tile_ctas) * 4 + warp;  // (item, head) unit of this warp
    if (u >= n_row_items * p.heads) return;
    const AttnItem itr = items[n_tile_items + u / p.heads];
    decode_row_warp(p, itr, u % p.heads, smem + warp * kDecWarpBytes);
    return;
  }
  const AttnItem it = items[blockIdx.x / p.heads];
  const int head = blockIdx.x % p.heads;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool decode_mode = it.q_rows <= 16;

  const int q0 = p.cu_q[it.seq];
  const int ctx = p.ctx_len[it.seq];
  const int row_off = decode_mode ? 0 : warp * 16;

  // query fragments (rows beyond q_rows are zero and fully masked)
  uint32_t qf[8][4];
  int qpos[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = row_off + g + 8 * h;
    qpos[h] = (r < it.q_rows) ? ctx + it.q_start + r : -1;
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = row_off + g + 8 * (e & 1);
      const int col = ks * 16 + 2 * t + 8 * (e >> 1);
      uint32_t v = 0;
      if (r < it.q_rows)
        v = *reinterpret_cast<const uint32_t*>(p.q + static_cast<int64_t>(q0 + it.q_start + r) * p.ldq +
                                               head * kHD + col);
      qf[ks][e] = v;
    }
  }

  float o[16][4];
#pragma unroll
  for (int d = 0; d < 16; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.0f;
  Softmax2 st;
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = 0.0f;

  const uint32_t smem_base = smem_u32(smem);
  const int n_stages = (it.kv_end - it.kv_start + kStageTok - 1) / kStageTok;
  const int last_page = (it.kv_end - 1) / kPage;
  const int32_t* bt = p.block_table + static_cast<int64_t>(it.seq) * p.bt_stride;
  const int64_t head_off = static_cast<int64_t>(head) * kPage * kHD;
  const int64_t page_elems = static_cast<int64_t>(p.heads) * kPage * kHD;

  auto load_stage = [&](int c, int buf) {
    const uint32_t sK = smem_base + buf * kStageBytes;
    const uint32_t sV = sK + kStageTok * kRowBytes;
    const int pos0 = it.kv_start + c * kStageTok;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int page = pos0 / kPage + j;
      page = page > last_page ? last_page : page;  // pad with a valid (masked) page
      const int64_t base = static_cast<int64_t>(bt[page]) * page_elems + head_off;
      const __nv_bfloat16* kp = p.kcache + base;
      const __nv_bfloat16* vp = p.vcache + base;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int id = threadIdx.x + i * kAttnThreads;  // 0..511 within the page
        const int tok = id >> 4, ch = id & 15;
        const uint32_t off = swz(j * kPage + tok, ch);
        cp_async16(sK + off, kp + tok * kHD + ch * 8);
        cp_async16(sV + off, vp + tok * kHD + ch * 8);
      }
    }
  };

  if (n_stages > 0) load_stage(0, 0);
  cp_async_commit();
  if (n_stages > 1) load_stage(1, 1);
  cp_async_commit();

  for (int c = 0; c < n_stages; ++c) {
    const int buf = c & 1;
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t sK = smem_base + buf * kStageBytes;
    const uint32_t sV = sK + kStageTok * kRowBytes;
    const int pos0 = it.kv_start + c * kStageTok;
    if (decode_mode)
      attend_stage<16>(sK, sV, warp * 16, qf, o, st, pos0, it.kv_end, qpos);
    else
      attend_stage<64>(sK, sV, 0, qf, o, st, pos0, it.kv_end, qpos);
    __syncthreads();
    if (c + 2 < n_stages) load_stage(c + 2, buf);
    cp_async_commit();
  }
  cp_async_wait<0>();

  const int tok_row0 = q0 + it.q_start;
  if (!decode_mode) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = row_off + g + 8 * h;
      if (r >= it.q_rows) continue;
      const float inv = st.l[h] > 0.0f ? 1.0f / st.l[h] : 0.0f;
      if (it.part_row < 0) {
        __nv_bfloat16* dst = p.out + static_cast<int64_t>(tok_row0 + r) * p.ldo + head * kHD;
#pragma unroll
        for (int d = 0; d < 16; ++d)
          *reinterpret_cast<uint32_t*>(dst + d * 8 + 2 * t) =
              pack_bf16x2(o[d][2 * h] * inv, o[d][2 * h + 1] * inv);
      } else {
        const int64_t prow = static_cast<int64_t>(it.part_row + r) * p.heads + head;
        float* dst = p.part_o + prow * kHD;
#pragma unroll
        for (int d = 0; d < 16; ++d)
          *reinterpret_cast<float2*>(dst + d * 8 + 2 * t) = make_float2(o[d][2 * h] * inv, o[d][2 * h + 1] * inv);
        if (t == 0) {
          p.part_ml[prow * 2] = st.m[h];
          p.part_ml[prow * 2 + 1] = st.l[h];
        }
      }
    }
    return;
  }

  // decode tile: merge the four warps' softmax states through shared memory
  float* so = reinterpret_cast<float*>(smem);          // [4][16][128]
  float* sm = so + 4 * 16 * kHD;                        // [4][16]
  float* sl = sm + 4 * 16;                              // [4][16]
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = g + 8 * h;
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      so[(warp * 16 + r) * kHD + d * 8 + 2 * t] = o[d][2 * h];
      so[(warp * 16 + r) * kHD + d * 8 + 2 * t + 1] = o[d][2 * h + 1];
    }
    if (t == 0) {
      sm[warp * 16 + r] = st.m[h];
      sl[warp * 16 + r] = st.l[h];
    }
  }
  __syncthreads();
  const int d = threadIdx.x;  // one output dim per thread
  for (int r = 0; r < it.q_rows; ++r) {
    float mmax = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) mmax = fmaxf(mmax, sm[w * 16 + r]);
    const float mref = mmax == -INFINITY ? 0.0f : mmax;
    float lsum = 0.0f, acc = 0.0f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float sc = exp2f(sm[w * 16 + r] - mref);
      lsum += sl[w * 16 + r] * sc;
      acc += so[(w * 16 + r) * kHD + d] * sc;
    }
    const float val = lsum > 0.0f ? acc / lsum : 0.0f;
    if (it.part_row < 0) {
      p.out[static_cast<int64_t>(tok_row0 + r) * p.ldo + head * kHD + d] = __float2bfloat16_rn(val);
    } else {
      const int64_t prow = static_cast<int64_t>(it.part_row + r) * p.heads + head;
      p.part_o[prow * kHD + d] = val;
      if (d == 0) {
        p.part_ml[prow * 2] = mmax;
        p.part_ml[prow * 2 + 1] = lsum;
      }
    }
  }
}

// Merge split-KV partial rows: out = sum_s w_s O_s / sum_s w_s, w_s = l_s * 2^(m_s - M).
__global__ void attn_combine_kernel(AttnParams p, const AttnCombine* __restrict__ combines) {
  const AttnCombine cb = combines[blockIdx.x];
  const int head = blockIdx.y;
  const int d = threadIdx.x;
  for (int r = 0; r < cb.q_rows; ++r) {
    float mmax = -INFINITY;
    for (int s = 0; s < cb.n_splits; ++s) {
      const int64_t prow = static_cast<int64_t>(cb.first_part + s * cb.q_rows + r) * p.heads + head;
      mmax = fmaxf(mmax, p.part_ml[prow * 2]);
    }
    const float mref = mmax == -INFINITY ? 0.0f : mmax;
    float lsum = 0.0f, acc = 0.0f;
    for (int s = 0; s < cb.n_splits; ++s) {
      const int64_t prow = static_cast<int64_t>(cb.first_part + s * cb.q_rows + r) * p.heads + head;
      const float w = p.part_ml[prow * 2 + 1] * exp2f(p.part_ml[prow * 2] - mref);
      lsum += w;
      acc += w * p.part_o[prow * kHD + d];
    }
    const float val = lsum > 0.0f ? acc / lsum : 0.0f;
    p.out[static_cast<int64_t>(cb.tok_row + r) * p.ldo + head * kHD + d] = __float2bfloat16_rn(val);
  }
}

}  // namespace

cudaError_t launch_attention(const AttnParams& p, const AttnItem* items, int n_tile_items, int n_row_items,
                             const AttnCombine* combines, int n_combines, cudaStream_t stream) {
  if (p.block_size != kPage) return cudaErrorInvalidValue;
  const int n_items = n_tile_items + n_row_items;
  if (n_items > 0) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(mixed_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kAttnSmem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    const int ctas = n_tile_items * p.heads + (n_row_items * p.heads + 3) / 4;
    mixed_attention_kernel<<<ctas, kAttnThreads, kAttnSmem, stream>>>(p, items, n_tile_items, n_row_items);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (n_combines > 0) {
    attn_combine_kernel<<<dim3(n_combines, p.heads), kHD, 0, stream>>>(p, combines);
    return cudaGetLastError();
  }
  return cudaSuccess;
}

}  // namespace ag
