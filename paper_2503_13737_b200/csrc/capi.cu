// C-ABI layer: model object, BatchPlan packing, the per-layer launch sequence and the
// standalone kernel entry points declared in include/accelgen_b200.h.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/accelgen_b200.h"
#include "kernels.h"

using ag::AttnCombine;
using ag::AttnItem;
using bf16 = __nv_bfloat16;

namespace {

thread_local std::string g_err;

int32_t fail(int32_t code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define AG_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(AG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
  } while (0)

#define AG_TRY(expr)                    \
  do {                                  \
    int32_t _r = (expr);                \
    if (_r != AG_OK) return _r;         \
  } while (0)

// ---------------------------------------------------------------- NCCL (dlopen'd)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
      api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
               api.GetErrorString;
    }
  }
  return api;
}

// ---------------------------------------------------------------- attention work list
struct AttnWork {
  std::vector<AttnItem> items;  // [tile items (q_rows > 1)] + [single-row items]
  std::vector<AttnCombine> combines;
  int n_tile = 0, n_row = 0;
  int part_rows = 0;
};

// Tile every sequence's new tokens: chunks of more than 16 rows become 128-row tcgen05 tiles;
// decode tokens and the rows of tiny chunks (<= 16 rows) become warp-level streaming items (one
// per row).  Long KV ranges are split (split-KV) so tiles give ~1 CTA/SM and rows ~24 warps/SM of
// work; tile splits are multiples of 128 tokens, row splits of 64; attn_combine_kernel merges.
void build_attention_work(const int32_t* cu_q, const int32_t* ctx_len, int B, int heads, int part_cap,
                          AttnWork& w) {
  w.items.clear();
  w.combines.clear();
  w.part_rows = 0;
  struct Piece {
    int seq, qs, rows, kv_hi;
  };
  const int TM = ag::attention_tile_rows(), TN = ag::attention_tile_kv();
  std::vector<Piece> tiles, rows1;
  double tile_work = 0.0, row_work = 0.0;
  for (int b = 0; b < B; ++b) {
    const int q = cu_q[b + 1] - cu_q[b];
    if (q <= 0) continue;
    if (q <= 16) {
      for (int r = 0; r < q; ++r) {
        rows1.push_back({b, r, 1, ctx_len[b] + r + 1});
        row_work += ctx_len[b] + r + 1;
      }
      continue;
    }
    for (int qs = 0; qs < q; qs += TM) {
      const int r = std::min(TM, q - qs);
      tiles.push_back({b, qs, r, ctx_len[b] + qs + r});
      tile_work += ctx_len[b] + qs + r;
    }
  }
  const int sms = ag::num_sms();
  auto emit = [&](const Piece& t, int n_split, int split, std::vector<AttnItem>& out) {
    if (n_split > 1 && w.part_rows + n_split * t.rows > part_cap) n_split = 1;
    if (n_split == 1) {
      out.push_back({t.seq, t.qs, t.rows, 0, t.kv_hi, -1, 0, 0});
      return;
    }
    const int base = w.part_rows;
    for (int s = 0; s < n_split; ++s) {
      const int a = s * split;
      out.push_back({t.seq, t.qs, t.rows, a, std::min(t.kv_hi, a + split), base + s * t.rows, 0, 0});
    }
    for (int r = 0; r < t.rows; ++r) w.combines.push_back({cu_q[t.seq] + t.qs + r, t.rows, base + r, n_split});
    w.part_rows += n_split * t.rows;
  };
  auto split_of = [](int kv_hi, double per_item, int min_len, int align, int& n_split, int& split) {
    n_split = static_cast<int>(std::ceil(kv_hi / per_item));
    n_split = std::max(1, std::min(n_split, (kv_hi + min_len - 1) / min_len));
    split = ((kv_hi + n_split - 1) / n_split + align - 1) / align * align;
    n_split = (kv_hi + split - 1) / split;
  };
  std::vector<AttnItem> tile_items, row_items;
  {
    const int desired = std::max(1, (sms + heads - 1) / heads);
    const double per_item = std::max(static_cast<double>(TN), tile_work / desired);
    for (const Piece& t : tiles) {
      int n, sp;
      split_of(t.kv_hi, per_item, 2 * TN, TN, n, sp);
      emit(t, n, sp, tile_items);
    }
  }
  {
    const int desired = std::max(1, (sms * 24 + heads - 1) / heads);
    const double per_item = std::max(512.0, row_work / desired);
    for (const Piece& t : rows1) {
      int n, sp;
      split_of(t.kv_hi, per_item, 512, 64, n, sp);
      emit(t, n, sp, row_items);
    }
  }
  // longest decode pieces first: the short ones fill the last wave instead of trailing it
  std::stable_sort(row_items.begin(), row_items.end(), [](const AttnItem& a, const AttnItem& b) {
    return a.kv_end - a.kv_start > b.kv_end - b.kv_start;
  });
  w.n_tile = static_cast<int>(tile_items.size());
  w.n_row = static_cast<int>(row_items.size());
  w.items = std::move(tile_items);
  w.items.insert(w.items.end(), row_items.begin(), row_items.end());
}

}  // namespace

// ---------------------------------------------------------------- model object
// A weight operand needs one tensor map per N-tile width (the TMA box must equal BLOCK_N).
struct WeightMap {
  CUtensorMap box64, box128, box160, box256;
  bool has256 = false, has160 = false;
  const CUtensorMap& box(int bn) const {
    return bn == 256 ? box256 : (bn == 160 ? box160 : (bn == 64 ? box64 : box128));
  }
};

// Activation operand maps for the three A-box heights (128 rows; 32/64 for small-M GEMMs).
struct ActMap {
  CUtensorMap box32, box64, box128;
  const CUtensorMap& box(int am) const { return am == 32 ? box32 : (am == 64 ? box64 : box128); }
};

// Autotuned (BLOCK_N, k_splits, A rows) per GEMM kind and M bucket (ag_model_autotune).
enum GemmKind { kGemmQkv = 0, kGemmOut, kGemmFc1, kGemmFc2, kGemmLm, kGemmKinds };
struct GemmTable {
  std::vector<int> m_bucket;                // ascending
  std::vector<ag::GemmPlan> plan[kGemmKinds];
  bool ready = false;
};

struct LayerState {
  ag_layer_weights w{};
  bf16* kpool = nullptr;
  bf16* vpool = nullptr;
  WeightMap tm_qkv, tm_out, tm_fc1, tm_fc2;
  CUtensorMap tm_kpool, tm_vpool;  // pool as [num_blocks*heads*32, 128], box 64 x 32
  bool ready = false;
};

struct ag_model {
  ag_model_config cfg{};
  int head_dim = 128, heads_l = 0, hq = 0, ffn_l = 0, vocab_l = 0, vocab_off = 0;
  int vocab_lp = 0;  // vocab_l padded to 32 columns (the GEMM epilogue stores 32-column chunks; TP=8: 6284)
  std::vector<LayerState> layers;
  const bf16* tok_emb = nullptr;
  const bf16* pos_emb = nullptr;
  const bf16* final_g = nullptr;
  const bf16* final_b = nullptr;
  // activations
  bf16 *resid = nullptr, *xln = nullptr, *qbuf = nullptr, *attn = nullptr, *ffn = nullptr, *proj = nullptr;
  bf16* lm_in = nullptr;
  float* logits = nullptr;
  float* cand_val = nullptr;
  int32_t* cand_idx = nullptr;
  float* gathered_val = nullptr;
  int32_t* gathered_idx = nullptr;
  int32_t* out_tok = nullptr;
  float *part_o = nullptr, *part_ml = nullptr;
  int part_cap = 0;
  float* splitk_ws = nullptr;
  float* acc32 = nullptr;  // fp32 [T, H] split-K accumulator of out-proj / FC2 at TP=1 (zero between uses)
  float* acc_big = nullptr;  // fp32 [T, max(3*hq, ffn)] stream-K accumulator of QKV / FC1 (zero between uses)
  int64_t acc_big_cols = 0;
  bool deterministic = false;  // AG_DETERMINISTIC=1: no fp32 atomics (split-K via the reduce kernel)
  // AG_FUSE_LN=1: the LayerNorm finishing a TP=1 atomic out-proj / FC2 runs in the consuming QKV / FC1
  // GEMM's prologue (or the atomic GEMM's tail) behind a grid barrier instead of its own launch
  bool fuse_ln = false;
  unsigned int* ln_bar = nullptr;
  int64_t splitk_cap = 0;
  GemmTable tune;
  // metadata: one pinned host buffer mirrored by one device buffer
  uint8_t* meta_host = nullptr;
  uint8_t* meta_dev = nullptr;
  size_t meta_cap = 0;
  int32_t* tok_host = nullptr;  // pinned D2H staging
  ActMap tm_xln, tm_attn, tm_ffn, tm_lm_in;
  CUtensorMap tm_qbuf;
  WeightMap tm_lm_w;
  // staged step
  int S = 0, B = 0, n_logit = 0, bt_stride = 0, n_items = 0, n_comb = 0, n_tile_items = 0, n_row_items = 0;
  const int32_t *d_ids = nullptr, *d_pos = nullptr, *d_cuq = nullptr, *d_ctx = nullptr, *d_bt = nullptr,
                *d_slot = nullptr, *d_lrows = nullptr;
  const AttnItem* d_items = nullptr;
  const AttnCombine* d_comb = nullptr;
  AttnWork work;
  ncclComm_t comm = nullptr;
  // host collective backend (ag_model_init_tp_host): collectives staged through pinned host memory
  // and completed by a host callback (one-GPU multi-process TP tests; no NCCL)
  ag_host_collective_fn host_coll = nullptr;
  void* host_coll_ctx = nullptr;
  uint8_t* coll_host = nullptr;
  size_t coll_host_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // asynchronous steps (ag_model_submit / ag_model_wait): two in-flight slots, each with its own pinned
  // metadata, next-token ids (device + pinned host), decode-feed pairs and events; the device metadata
  // buffer is shared (stream order: step k+1's H2D runs after step k's kernels)
  struct AsyncSlot {
    uint8_t* meta_host = nullptr;
    int32_t* out_tok = nullptr;
    int32_t* tok_host = nullptr;
    int32_t* feed_host = nullptr;
    cudaEvent_t start = nullptr, end = nullptr, done = nullptr;
    int n_logit = 0;
    bool active = false;
  } aslot[2];
  int32_t* feed_dev = nullptr;
  int64_t n_submit = 0, n_wait = 0;
  cudaEvent_t ev_ref = nullptr;
  // per-kernel-class profiling (CUDA events around every launch of one forward)
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_events;
  struct ProfRec {
    int cls;
    int ev;
    double flops, bytes;
  };
  std::vector<ProfRec> prof_pending;
  double prof_ms[AG_PROF_CLASSES] = {};
  double prof_flops[AG_PROF_CLASSES] = {};
  double prof_bytes[AG_PROF_CLASSES] = {};
  int64_t prof_count[AG_PROF_CLASSES] = {};
  // per-launch roofline time max(FLOPs / tensor peak, bytes / HBM peak), summed per class
  double prof_roof_ms[AG_PROF_CLASSES] = {};
  double peak_tflops = 0.0, peak_gbs = 0.0;
  int64_t launches_last = 0;
  int64_t h2d_last = 0;
  int64_t launches_total = 0;
  double attn_flops_step = 0.0, attn_bytes_step = 0.0;
};

namespace {

template <typename T>
int32_t dmalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) return fail(AG_EALLOC, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return AG_OK;
}

int32_t tmap(CUtensorMap* m, const void* ptr, int64_t rows, int64_t k, int box_rows, const char* what) {
  const int r = ag::make_tmap_kmajor(m, ptr, rows, k, k, box_rows);
  if (r != 0) return fail(AG_EINVAL, std::string("tensor map for ") + what + " failed (" + std::to_string(r) + ")");
  return AG_OK;
}

int32_t wmap(WeightMap* w, const void* ptr, int64_t rows, int64_t k, const char* what) {
  AG_TRY(tmap(&w->box64, ptr, rows, k, 64, what));
  AG_TRY(tmap(&w->box128, ptr, rows, k, 128, what));
  w->has256 = rows % 256 == 0;
  if (w->has256) AG_TRY(tmap(&w->box256, ptr, rows, k, 256, what));
  w->has160 = rows % 160 == 0;  // 160-wide tiles: FC1 (20480/160 = 128 tiles) fills the SMs at small M
  if (w->has160) AG_TRY(tmap(&w->box160, ptr, rows, k, 160, what));
  return AG_OK;
}

// GEMM against a weight: (N tile, K splits) from the autotuned table for this M bucket (or the
// analytic planner before autotune), then launch with the matching tensor map.
ag::GemmPlan pick_plan(const WeightMap& w, int M, int N, int K, int64_t splitk_cap, const GemmTable* tune, int kind) {
  ag::GemmPlan p{0, 0, 128};
  if (tune && tune->ready && kind >= 0) {
    for (size_t i = 0; i < tune->m_bucket.size(); ++i) {
      if (M <= tune->m_bucket[i] || i + 1 == tune->m_bucket.size()) {
        p = tune->plan[kind][i];
        break;
      }
    }
    if (p.k_splits != ag::kStreamK && static_cast<int64_t>(p.k_splits) * M * N > splitk_cap) p.k_splits = 1;
    if (p.am < 128 && M > p.am) p.am = 128;
  }
  if (p.bn == 0) p = ag::plan_gemm(M, N, K, splitk_cap);
  if (p.bn == 256 && !w.has256 && p.am != 256) p.bn = 128;
  if (p.bn == 160 && (!w.has160 || p.am == 256)) p.bn = 128;
  return p;
}

cudaError_t gemm_w(const ActMap& a, const WeightMap& w, int M, int N, int K, const ag::GemmEpilogue& ep,
                   cudaStream_t s, float* splitk_ws, int64_t splitk_cap, const GemmTable* tune = nullptr,
                   int kind = -1, const ag::GemmPlan* forced = nullptr) {
  ag::GemmPlan p{0, 0, 128};
  if (forced) {
    p = *forced;
    if (p.am == 256) return ag::launch_gemm(a.box(128), w.box(p.bn / 2), M, N, K, p.bn, ep, 0, s, p.k_splits, splitk_ws, 256);
    return ag::launch_gemm(a.box(p.am), w.box(p.bn), M, N, K, p.bn, ep, 0, s, p.k_splits, splitk_ws, p.am);
  }
  p = pick_plan(w, M, N, K, splitk_ws ? splitk_cap : 0, tune, kind);
  if (p.k_splits == ag::kStreamK && ep.mode != ag::kEpiAtomicF32) p.k_splits = 1;  // needs a deferred epilogue
  if (p.am == 256) return ag::launch_gemm(a.box(128), w.box(p.bn / 2), M, N, K, p.bn, ep, 0, s, p.k_splits, splitk_ws, 256);
  return ag::launch_gemm(a.box(p.am), w.box(p.bn), M, N, K, p.bn, ep, 0, s, p.k_splits, splitk_ws, p.am);
}

// QKV / FC1: a stream-K plan accumulates atomically into acc_big, then the finish kernel applies the
// real epilogue (bias, q scale + paged KV scatter, ReLU) and re-zeroes the accumulator.
cudaError_t gemm_planned(const ActMap& a, const WeightMap& w, int M, int N, int K, const ag::GemmEpilogue& ep,
                         const ag::GemmPlan& p, cudaStream_t s, float* splitk_ws, int64_t splitk_cap, float* acc_big) {
  if (p.k_splits != ag::kStreamK) return gemm_w(a, w, M, N, K, ep, s, splitk_ws, splitk_cap, nullptr, -1, &p);
  ag::GemmEpilogue ea = ep;  // keeps a fused LayerNorm prologue (the finish kernel ignores it)
  ea.mode = ag::kEpiAtomicF32;
  ea.acc32 = acc_big;
  ea.ldc = N;
  cudaError_t e = gemm_w(a, w, M, N, K, ea, s, splitk_ws, splitk_cap, nullptr, -1, &p);
  if (e != cudaSuccess) return e;
  return ag::launch_splitk_finish(acc_big, M, N, ep, s);
}

int32_t amap(ActMap* a, const void* ptr, int64_t rows, int64_t k, const char* what) {
  AG_TRY(tmap(&a->box32, ptr, rows, k, 32, what));
  AG_TRY(tmap(&a->box64, ptr, rows, k, 64, what));
  return tmap(&a->box128, ptr, rows, k, 128, what);
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int32_t check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return AG_OK;
  return fail(AG_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// Host backend: D2H into pinned staging, wait, the callback completes the collective in place on the
// host buffer, H2D back (stream-ordered, so the staging is free again once the next D2H is reached).
int32_t host_collective(ag_model* m, int32_t op, const void* src, void* dst, size_t count, size_t elem,
                        int32_t dtype, cudaStream_t s) {
  const size_t in_bytes = count * elem;
  const size_t out_bytes = op == AG_COLL_ALLGATHER ? in_bytes * m->cfg.tp_size : in_bytes;
  if (out_bytes > m->coll_host_cap) return fail(AG_EALLOC, "host collective staging too small");
  uint8_t* h = m->coll_host + (op == AG_COLL_ALLGATHER ? in_bytes * m->cfg.tp_rank : 0);
  AG_CUDA(cudaMemcpyAsync(h, src, in_bytes, cudaMemcpyDeviceToHost, s));
  AG_CUDA(cudaStreamSynchronize(s));
  const int32_t rc = m->host_coll(m->host_coll_ctx, op, m->coll_host, static_cast<int64_t>(count), dtype);
  if (rc != 0) return fail(AG_ENCCL, "host collective callback failed (" + std::to_string(rc) + ")");
  AG_CUDA(cudaMemcpyAsync(dst, m->coll_host, out_bytes, cudaMemcpyHostToDevice, s));
  return AG_OK;
}

int32_t allreduce_bf16(ag_model* m, bf16* buf, size_t count, cudaStream_t s) {
  if (m->cfg.tp_size == 1) return AG_OK;
  if (m->host_coll) return host_collective(m, AG_COLL_ALLREDUCE_SUM, buf, buf, count, 2, AG_DT_BF16, s);
  return check_nccl(nccl().AllReduce(buf, buf, count, ncclBfloat16, ncclSum, m->comm, s), "ncclAllReduce");
}

// per-rank (max, index) candidates of the vocab-parallel argmax -> every rank's candidates
int32_t allgather_cands(ag_model* m, int NL, cudaStream_t s) {
  if (m->host_coll) {
    AG_TRY(host_collective(m, AG_COLL_ALLGATHER, m->cand_val, m->gathered_val, NL, 4, AG_DT_F32, s));
    return host_collective(m, AG_COLL_ALLGATHER, m->cand_idx, m->gathered_idx, NL, 4, AG_DT_I32, s);
  }
  AG_TRY(check_nccl(nccl().AllGather(m->cand_val, m->gathered_val, NL, ncclFloat32, m->comm, s), "allgather"));
  return check_nccl(nccl().AllGather(m->cand_idx, m->gathered_idx, NL, ncclInt32, m->comm, s), "allgather");
}

// Event bracket around one launch of kernel class `cls` (algorithmic flops / bytes attached).
struct ProfScope {
  ag_model* m;
  int cls;
  cudaStream_t s;
  double flops, bytes;
  int ev = -1;
  ProfScope(ag_model* m_, int cls_, cudaStream_t s_, double f, double b) : m(m_), cls(cls_), s(s_), flops(f), bytes(b) {
    m->launches_last += 1;
    if (!m->prof_on) return;
    const size_t need = m->prof_pending.size() * 2 + 2;
    if (need > m->prof_events.size()) return;  // out of events: skip (counts stay exact)
    ev = static_cast<int>(m->prof_pending.size() * 2);
    cudaEventRecord(m->prof_events[ev], s);
  }
  ~ProfScope() {
    if (ev < 0) return;
    cudaEventRecord(m->prof_events[ev + 1], s);
    m->prof_pending.push_back({cls, ev, flops, bytes});
  }
};

void prof_harvest(ag_model* m) {
  for (const auto& r : m->prof_pending) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, m->prof_events[r.ev], m->prof_events[r.ev + 1]) == cudaSuccess) {
      m->prof_ms[r.cls] += ms;
      if (m->peak_tflops > 0.0 && m->peak_gbs > 0.0)
        m->prof_roof_ms[r.cls] += 1e3 * std::max(r.flops / (m->peak_tflops * 1e12), r.bytes / (m->peak_gbs * 1e9));
      m->prof_flops[r.cls] += r.flops;
      m->prof_bytes[r.cls] += r.bytes;
      m->prof_count[r.cls] += 1;
    }
  }
  m->prof_pending.clear();
}

// AG_DEBUG_SYNC=1: synchronise after every launch of the forward and name the failing kernel.
bool debug_sync() {
  static const bool on = [] {
    const char* e = std::getenv("AG_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}

int32_t dbg(cudaStream_t s, const char* what, int layer) {
  if (!debug_sync()) return AG_OK;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess)
    return fail(AG_ECUDA, std::string("AG_DEBUG_SYNC: ") + what + " (layer " + std::to_string(layer) + "): " +
                              cudaGetErrorString(e));
  return AG_OK;
}

double gemm_flops(int M, int N, int K) { return 2.0 * M * static_cast<double>(N) * K; }
double gemm_bytes(int M, int N, int K, int out_bytes) {
  return 2.0 * (static_cast<double>(M) * K + static_cast<double>(N) * K) + static_cast<double>(out_bytes) * M * N;
}

}  // namespace

extern "C" {

const char* ag_last_error(void) { return g_err.c_str(); }
int32_t ag_version(void) { return 1; }
int32_t ag_device_sm_count(void) { return ag::num_sms(); }

int32_t ag_model_create(const ag_model_config* cfg, ag_model** out) {
  if (!cfg || !out) return fail(AG_EINVAL, "null argument");
  const ag_model_config& c = *cfg;
  if (c.hidden <= 0 || c.num_layers <= 0 || c.num_heads <= 0 || c.hidden % c.num_heads != 0)
    return fail(AG_EINVAL, "bad hidden/num_heads");
  if (c.hidden / c.num_heads != 128) return fail(AG_EINVAL, "head_dim must be 128");
  if (c.tp_size < 1 || c.tp_rank < 0 || c.tp_rank >= c.tp_size) return fail(AG_EINVAL, "bad tp rank/size");
  if (c.num_heads % c.tp_size || c.ffn % c.tp_size || c.vocab % c.tp_size)
    return fail(AG_EINVAL, "heads, ffn and vocab must divide by tp_size");
  if (c.block_size != 32) return fail(AG_EINVAL, "block_size must be 32");
  if (c.max_tokens <= 0 || c.max_seqs <= 0 || c.max_blocks_per_seq <= 0 || c.num_blocks <= 0)
    return fail(AG_EINVAL, "capacities must be positive");
  if (c.hidden % 64 || (c.ffn / c.tp_size) % 64 || (c.vocab / c.tp_size) % 4)
    return fail(AG_EINVAL, "hidden, ffn/tp must be multiples of 64 and vocab/tp of 4");

  ag_model* m = new ag_model();
  m->cfg = c;
  m->heads_l = c.num_heads / c.tp_size;
  m->hq = m->heads_l * m->head_dim;
  m->ffn_l = c.ffn / c.tp_size;
  m->vocab_l = c.vocab / c.tp_size;
  m->vocab_off = c.tp_rank * m->vocab_l;
  m->vocab_lp = static_cast<int>(align_up(static_cast<size_t>(m->vocab_l), 32));
  m->layers.resize(c.num_layers);
  // activation rows are padded to a multiple of 128 so GEMM A-tiles never leave the buffer
  const size_t T = align_up(static_cast<size_t>(c.max_tokens), 128);
  const size_t Sq = align_up(static_cast<size_t>(c.max_seqs), 128);
  int32_t r = AG_OK;
  auto chk = [&](int32_t x) {
    if (r == AG_OK) r = x;
  };
  chk(dmalloc(&m->resid, T * c.hidden));
  chk(dmalloc(&m->xln, T * c.hidden));
  chk(dmalloc(&m->qbuf, T * m->hq));
  chk(dmalloc(&m->attn, T * m->hq));
  chk(dmalloc(&m->ffn, T * m->ffn_l));
  chk(dmalloc(&m->proj, T * c.hidden));
  chk(dmalloc(&m->lm_in, Sq * c.hidden));
  chk(dmalloc(&m->logits, Sq * m->vocab_lp));
  chk(dmalloc(&m->cand_val, Sq));
  chk(dmalloc(&m->cand_idx, Sq));
  chk(dmalloc(&m->gathered_val, Sq * c.tp_size));
  chk(dmalloc(&m->gathered_idx, Sq * c.tp_size));
  chk(dmalloc(&m->out_tok, Sq));
  m->part_cap = std::max(4096, c.max_tokens * 4);
  chk(dmalloc(&m->part_o, static_cast<size_t>(m->part_cap) * m->heads_l * m->head_dim));
  chk(dmalloc(&m->part_ml, static_cast<size_t>(m->part_cap) * m->heads_l * 2));
  m->splitk_cap = int64_t(32) << 20;  // fp32 K-split partials (128 MB)
  chk(dmalloc(&m->splitk_ws, static_cast<size_t>(m->splitk_cap)));
  chk(dmalloc(&m->acc32, T * c.hidden));
  m->acc_big_cols = std::max(3 * m->hq, m->ffn_l);
  {
    const char* e = std::getenv("AG_DETERMINISTIC");
    m->deterministic = e && e[0] == '1';
    // off by default: in-chain it gains <= 0.1 ms per decode step without the cooperative attribute, and
    // the cooperative launch that guarantees its grid barrier's co-residency costs +0.45 ms
    // (profiles/r2/fused_ln/README.md)
    const char* f = std::getenv("AG_FUSE_LN");
    m->fuse_ln = f && f[0] == '1';
  }
  chk(dmalloc(&m->ln_bar, 64));
  if (r == AG_OK && cudaMemset(m->ln_bar, 0, 64 * sizeof(unsigned int)) != cudaSuccess) r = fail(AG_ECUDA, "memset ln_bar");
  chk(dmalloc(&m->acc_big, T * m->acc_big_cols));
  if (r == AG_OK && cudaMemset(m->acc_big, 0, sizeof(float) * T * m->acc_big_cols) != cudaSuccess)
    r = fail(AG_ECUDA, "memset acc_big");
  if (r == AG_OK && cudaMemset(m->acc32, 0, sizeof(float) * T * c.hidden) != cudaSuccess)
    r = fail(AG_ECUDA, "memset acc32");
  // metadata capacity: token arrays, sequence arrays, block table, attention work list
  const size_t max_items = static_cast<size_t>(c.max_tokens) + c.max_seqs + 64 * static_cast<size_t>(ag::num_sms());
  m->meta_cap = align_up(4 * sizeof(int32_t) * T, 256) + align_up(2 * sizeof(int32_t) * (c.max_seqs + 1), 256) +
                align_up(sizeof(int32_t) * static_cast<size_t>(c.max_seqs) * c.max_blocks_per_seq, 256) +
                align_up(sizeof(AttnItem) * max_items, 256) + align_up(sizeof(AttnCombine) * max_items, 256) + 4096;
  if (r == AG_OK && cudaMallocHost(&m->meta_host, m->meta_cap) != cudaSuccess) r = fail(AG_EALLOC, "pinned alloc");
  chk(dmalloc(&m->meta_dev, m->meta_cap));
  if (r == AG_OK && cudaMallocHost(&m->tok_host, Sq * sizeof(int32_t)) != cudaSuccess) r = fail(AG_EALLOC, "pinned");
  if (r == AG_OK) {
    chk(amap(&m->tm_xln, m->xln, T, c.hidden, "xln"));
    chk(amap(&m->tm_attn, m->attn, T, m->hq, "attn"));
    chk(amap(&m->tm_ffn, m->ffn, T, m->ffn_l, "ffn"));
    chk(amap(&m->tm_lm_in, m->lm_in, Sq, c.hidden, "lm_in"));
    chk(tmap(&m->tm_qbuf, m->qbuf, T, m->hq, 128, "q buffer"));
  }
  if (r == AG_OK) {
    cudaEventCreate(&m->ev0);
    cudaEventCreate(&m->ev1);
  }
  if (r != AG_OK) {
    std::string keep = g_err;
    ag_model_destroy(m);
    g_err = keep;
    return r;
  }
  *out = m;
  return AG_OK;
}

void ag_model_destroy(ag_model* m) {
  if (!m) return;
  if (m->comm && nccl().ok) nccl().CommDestroy(m->comm);
  void* dev[] = {m->resid, m->xln, m->qbuf, m->attn, m->ffn, m->proj, m->lm_in, m->logits, m->cand_val,
                 m->cand_idx, m->gathered_val, m->gathered_idx, m->out_tok, m->part_o, m->part_ml, m->meta_dev,
                 m->splitk_ws, m->acc32, m->acc_big, m->ln_bar};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (m->aslot[0].meta_host) m->meta_host = m->aslot[0].meta_host;  // slot 1's buffer is freed below
  if (m->meta_host) cudaFreeHost(m->meta_host);
  if (m->coll_host) cudaFreeHost(m->coll_host);
  if (m->tok_host) cudaFreeHost(m->tok_host);
  if (m->ev0) cudaEventDestroy(m->ev0);
  if (m->ev1) cudaEventDestroy(m->ev1);
  for (int i = 1; i < 2; ++i) {  // slot 0 aliases meta_host / out_tok / tok_host
    if (m->aslot[i].meta_host) cudaFreeHost(m->aslot[i].meta_host);
    if (m->aslot[i].tok_host) cudaFreeHost(m->aslot[i].tok_host);
    if (m->aslot[i].out_tok) cudaFree(m->aslot[i].out_tok);
  }
  for (int i = 0; i < 2; ++i) {
    if (m->aslot[i].feed_host) cudaFreeHost(m->aslot[i].feed_host);
    for (cudaEvent_t e : {m->aslot[i].start, m->aslot[i].end, m->aslot[i].done})
      if (e) cudaEventDestroy(e);
  }
  if (m->feed_dev) cudaFree(m->feed_dev);
  if (m->ev_ref) cudaEventDestroy(m->ev_ref);
  delete m;
}

int32_t ag_model_set_embeddings(ag_model* m, const void* tok_emb, const void* pos_emb, const void* final_ln_g,
                                const void* final_ln_b) {
  if (!m || !tok_emb || !pos_emb || !final_ln_g || !final_ln_b) return fail(AG_EINVAL, "null argument");
  m->tok_emb = static_cast<const bf16*>(tok_emb);
  m->pos_emb = static_cast<const bf16*>(pos_emb);
  m->final_g = static_cast<const bf16*>(final_ln_g);
  m->final_b = static_cast<const bf16*>(final_ln_b);
  // tied LM head: this rank's vocab shard of the token embedding
  return wmap(&m->tm_lm_w, m->tok_emb + static_cast<size_t>(m->vocab_off) * m->cfg.hidden, m->vocab_l,
              m->cfg.hidden, "lm head");
}

int32_t ag_model_set_layer(ag_model* m, int32_t layer, const ag_layer_weights* w) {
  if (!m || !w || layer < 0 || layer >= m->cfg.num_layers) return fail(AG_EINVAL, "bad layer");
  const void* req[] = {w->ln1_g, w->ln1_b, w->qkv_w, w->qkv_b, w->out_w, w->out_b,
                       w->ln2_g, w->ln2_b, w->fc1_w, w->fc1_b, w->fc2_w, w->fc2_b};
  for (const void* p : req)
    if (!p) return fail(AG_EINVAL, "null weight pointer");
  LayerState& L = m->layers[layer];
  L.w = *w;
  const int H = m->cfg.hidden;
  AG_TRY(wmap(&L.tm_qkv, w->qkv_w, 3 * m->hq, H, "qkv_w"));
  AG_TRY(wmap(&L.tm_out, w->out_w, H, m->hq, "out_w"));
  AG_TRY(wmap(&L.tm_fc1, w->fc1_w, m->ffn_l, H, "fc1_w"));
  AG_TRY(wmap(&L.tm_fc2, w->fc2_w, H, m->ffn_l, "fc2_w"));
  L.ready = L.kpool != nullptr;
  return AG_OK;
}

int32_t ag_model_set_kv_cache(ag_model* m, int32_t layer, void* k_pool, void* v_pool) {
  if (!m || layer < 0 || layer >= m->cfg.num_layers || !k_pool || !v_pool) return fail(AG_EINVAL, "bad kv cache");
  m->layers[layer].kpool = static_cast<bf16*>(k_pool);
  m->layers[layer].vpool = static_cast<bf16*>(v_pool);
  const int64_t pool_rows = static_cast<int64_t>(m->cfg.num_blocks) * m->heads_l * m->cfg.block_size;
  AG_TRY(tmap(&m->layers[layer].tm_kpool, k_pool, pool_rows, m->head_dim, 32, "k pool"));
  AG_TRY(tmap(&m->layers[layer].tm_vpool, v_pool, pool_rows, m->head_dim, 32, "v pool"));
  m->layers[layer].ready = m->layers[layer].w.qkv_w != nullptr;
  return AG_OK;
}

int32_t ag_nccl_get_unique_id(void* out) {
  if (!out) return fail(AG_EINVAL, "null");
  if (!nccl().ok) return fail(AG_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  AG_TRY(check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId"));
  std::memcpy(out, &id, sizeof(id));
  return AG_OK;
}

int32_t ag_model_init_tp(ag_model* m, const void* uid) {
  if (!m || !uid) return fail(AG_EINVAL, "null");
  if (m->cfg.tp_size == 1) return AG_OK;
  if (!nccl().ok) return fail(AG_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  return check_nccl(nccl().CommInitRank(&m->comm, m->cfg.tp_size, id, m->cfg.tp_rank), "ncclCommInitRank");
}

int32_t ag_model_init_tp_host(ag_model* m, ag_host_collective_fn fn, void* ctx) {
  if (!m || !fn) return fail(AG_EINVAL, "null");
  if (m->cfg.tp_size == 1) return AG_OK;
  if (m->comm) return fail(AG_EINVAL, "NCCL communicator already initialised");
  const size_t T = align_up(static_cast<size_t>(m->cfg.max_tokens), 128);
  const size_t Sq = align_up(static_cast<size_t>(m->cfg.max_seqs), 128);
  m->coll_host_cap = std::max(T * m->cfg.hidden * sizeof(bf16), Sq * 4 * m->cfg.tp_size);
  if (cudaMallocHost(&m->coll_host, m->coll_host_cap) != cudaSuccess) return fail(AG_EALLOC, "pinned alloc");
  m->host_coll = fn;
  m->host_coll_ctx = ctx;
  return AG_OK;
}

int32_t ag_model_stage_step(ag_model* m, const ag_step* st, void* stream) {
  if (!m || !st) return fail(AG_EINVAL, "null argument");
  const ag_model_config& c = m->cfg;
  const int S = st->num_tokens, B = st->num_seqs, NL = st->num_logits, bts = st->block_table_stride;
  if (S < 0 || S > c.max_tokens) return fail(AG_EALLOC, "num_tokens exceeds max_tokens");
  if (B < 0 || B > c.max_seqs) return fail(AG_EALLOC, "num_seqs exceeds max_seqs");
  if (NL < 0 || NL > c.max_seqs) return fail(AG_EALLOC, "num_logits exceeds max_seqs");
  if (bts < 1 || bts > c.max_blocks_per_seq) return fail(AG_EALLOC, "block_table_stride out of range");
  for (int l = 0; l < c.num_layers; ++l)
    if (!m->layers[l].ready) return fail(AG_EINVAL, "layer " + std::to_string(l) + " weights/kv not set");
  if (!m->tok_emb) return fail(AG_EINVAL, "embeddings not set");
  if (S > 0 && (!st->token_ids || !st->positions || !st->slot_mapping))
    return fail(AG_EINVAL, "null token arrays");
  if (!st->cu_q || !st->ctx_len || (B > 0 && !st->block_table) || (NL > 0 && !st->logit_rows))
    return fail(AG_EINVAL, "null sequence arrays");
  // validate the plan against capacities (the reference's EngineFault conditions)
  if (st->cu_q[0] != 0 || st->cu_q[B] != S) return fail(AG_EFAULT, "cu_q must start at 0 and end at num_tokens");
  for (int b = 0; b < B; ++b) {
    const int q = st->cu_q[b + 1] - st->cu_q[b];
    if (q < 0) return fail(AG_EFAULT, "cu_q not monotone");
    const int kv = st->ctx_len[b] + q;
    if (st->ctx_len[b] < 0 || (kv + c.block_size - 1) / c.block_size > bts)
      return fail(AG_EFAULT, "sequence " + std::to_string(b) + " exceeds its block table");
    for (int j = 0; j < (kv + c.block_size - 1) / c.block_size; ++j) {
      const int blk = st->block_table[static_cast<size_t>(b) * bts + j];
      if (blk < 0 || blk >= c.num_blocks) return fail(AG_EFAULT, "block id out of range");
    }
  }
  for (int i = 0; i < S; ++i) {
    const int s = st->slot_mapping[i];
    if (s >= c.num_blocks * c.block_size) return fail(AG_EFAULT, "slot out of range");
    if (st->positions[i] + 2 >= c.pos_rows || st->positions[i] < 0)
      return fail(AG_EINVAL, "position beyond the position table");
  }
  for (int i = 0; i < NL; ++i)
    if (st->logit_rows[i] < 0 || st->logit_rows[i] >= S) return fail(AG_EINVAL, "logit row out of range");

  build_attention_work(st->cu_q, st->ctx_len, B, m->heads_l, m->part_cap, m->work);
  {
    // exact causal attention work: q_i new rows over p_i cached + causal triangle
    double fl = 0.0, by = 0.0;
    for (int b = 0; b < B; ++b) {
      const double q = st->cu_q[b + 1] - st->cu_q[b], p = st->ctx_len[b];
      fl += 4.0 * m->hq * (q * p + q * (q + 1) / 2.0);
      by += 2.0 * 2.0 * m->hq * (p + q) + 2.0 * 2.0 * m->hq * q;  // K+V read, q read + out write
    }
    m->attn_flops_step = fl;
    m->attn_bytes_step = by;
  }
  // pack
  uint8_t* h = m->meta_host;
  size_t off = 0;
  auto put = [&](const void* src, size_t bytes) -> size_t {
    const size_t at = off;
    if (bytes) std::memcpy(h + off, src, bytes);
    off = align_up(off + bytes, 256);
    return at;
  };
  const size_t o_ids = put(st->token_ids, sizeof(int32_t) * S);
  const size_t o_pos = put(st->positions, sizeof(int32_t) * S);
  const size_t o_slot = put(st->slot_mapping, sizeof(int32_t) * S);
  const size_t o_cuq = put(st->cu_q, sizeof(int32_t) * (B + 1));
  const size_t o_ctx = put(st->ctx_len, sizeof(int32_t) * B);
  const size_t o_bt = put(st->block_table, sizeof(int32_t) * static_cast<size_t>(B) * bts);
  const size_t o_lr = put(st->logit_rows, sizeof(int32_t) * NL);
  const size_t need = off + align_up(sizeof(AttnItem) * m->work.items.size(), 256) +
                      align_up(sizeof(AttnCombine) * m->work.combines.size(), 256);
  if (need > m->meta_cap) return fail(AG_EALLOC, "metadata exceeds staging capacity");
  const size_t o_items = put(m->work.items.data(), sizeof(AttnItem) * m->work.items.size());
  const size_t o_comb = put(m->work.combines.data(), sizeof(AttnCombine) * m->work.combines.size());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  AG_CUDA(cudaMemcpyAsync(m->meta_dev, m->meta_host, off, cudaMemcpyHostToDevice, s));
  m->h2d_last = static_cast<int64_t>(off);
  const uint8_t* d = m->meta_dev;
  m->d_ids = reinterpret_cast<const int32_t*>(d + o_ids);
  m->d_pos = reinterpret_cast<const int32_t*>(d + o_pos);
  m->d_slot = reinterpret_cast<const int32_t*>(d + o_slot);
  m->d_cuq = reinterpret_cast<const int32_t*>(d + o_cuq);
  m->d_ctx = reinterpret_cast<const int32_t*>(d + o_ctx);
  m->d_bt = reinterpret_cast<const int32_t*>(d + o_bt);
  m->d_lrows = reinterpret_cast<const int32_t*>(d + o_lr);
  m->d_items = reinterpret_cast<const AttnItem*>(d + o_items);
  m->d_comb = reinterpret_cast<const AttnCombine*>(d + o_comb);
  m->S = S;
  m->B = B;
  m->n_logit = NL;
  m->bt_stride = bts;
  m->n_items = static_cast<int>(m->work.items.size());
  m->n_tile_items = m->work.n_tile;
  m->n_row_items = m->work.n_row;
  m->n_comb = static_cast<int>(m->work.combines.size());
  return AG_OK;
}

int32_t ag_model_forward_staged(ag_model* m, int32_t* out_tokens_dev, float* logits_out, void* stream) {
  if (!m) return fail(AG_EINVAL, "null model");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const ag_model_config& c = m->cfg;
  const int S = m->S, H = c.hidden;
  const bool tp = c.tp_size > 1;
  const double bf = 2.0;
  m->launches_last = 0;
  const double ln_bytes = bf * 2.0 * S * H;
  bool final_acc = false;
  if (S > 0) {
    {
      ProfScope ps(m, AG_K_EMBED, s, 0.0, bf * 3.0 * S * H);
      AG_CUDA(ag::launch_embed(m->d_ids, m->d_pos, m->tok_emb, m->pos_emb, 2, S, H, c.vocab, c.pos_rows, m->resid, s));
    }
    const float qscale = 1.0f / std::sqrt(static_cast<float>(m->head_dim));
    // TP=1: an out-proj / FC2 plan that splits K accumulates into acc32 with fp32 reductions and the
    // next LayerNorm applies bias + residual (no reduce launch); else the GEMM epilogue does it
    auto atomic_plan = [&](const WeightMap& wm, int N, int K, int kind, ag::GemmPlan& p) {
      p = pick_plan(wm, S, N, K, m->splitk_cap, &m->tune, kind);
      if (m->deterministic && p.k_splits == ag::kStreamK) p.k_splits = 1;
      return !tp && p.k_splits > 1 && !m->deterministic;
    };
    bool acc_pending = false;
    bool ln1_done = false;  // the previous FC2's fused tail already wrote this layer's LN1 (xln)
    // fused LayerNorm tail on an atomic out-proj / FC2 (see ag::GemmEpilogue::ln_out)
    auto fuse_ln = [&](ag::GemmEpilogue& e, const void* bias, const void* g, const void* b) {
      e.ln_acc = m->acc32;
      e.ln_ld = H;
      e.ln_x = m->resid;
      e.ln_bias = static_cast<const bf16*>(bias);
      e.ln_g = static_cast<const bf16*>(g);
      e.ln_b = static_cast<const bf16*>(b);
      e.ln_eps = c.ln_eps;
      e.ln_out = m->xln;
      e.ln_bar = m->ln_bar;
    };
    // QKV / FC1 plans (the same for every layer at this S): a consumer whose grid covers the S rows
    // finishes the previous atomic out-proj / FC2's LayerNorm in its prologue (preferred: its weight
    // prefetch overlaps the norm); otherwise the atomic GEMM's own tail does when its grid covers them
    ag::GemmPlan pq = pick_plan(m->layers[0].tm_qkv, S, 3 * m->hq, H, m->splitk_cap, &m->tune, kGemmQkv);
    if (m->deterministic && pq.k_splits == ag::kStreamK) pq.k_splits = 1;
    ag::GemmPlan p1 = pick_plan(m->layers[0].tm_fc1, S, m->ffn_l, H, m->splitk_cap, &m->tune, kGemmFc1);
    if (m->deterministic && p1.k_splits == ag::kStreamK) p1.k_splits = 1;
    const bool qkv_prologue = m->fuse_ln && !tp && S <= ag::gemm_grid(S, 3 * m->hq, H, pq.bn, pq.k_splits, pq.am);
    const bool fc1_prologue = m->fuse_ln && !tp && S <= ag::gemm_grid(S, m->ffn_l, H, p1.bn, p1.k_splits, p1.am);
    for (int l = 0; l < c.num_layers; ++l) {
      const LayerState& L = m->layers[l];
      const ag_layer_weights& w = L.w;
      const bool ln1_in_qkv = acc_pending && qkv_prologue;
      if (!ln1_done && !ln1_in_qkv) {
        // LN1 (for TP the previous layer's FC2 all-reduce result + bias is folded in here)
        ProfScope ps(m, AG_K_LAYERNORM, s, 0.0, ((tp || acc_pending) && l > 0) ? 2.0 * ln_bytes : ln_bytes);
        if (acc_pending) {  // previous layer's FC2 was split-K into acc32: finish its epilogue here
          AG_CUDA(ag::launch_layernorm_acc(m->resid, m->acc32, static_cast<const bf16*>(m->layers[l - 1].w.fc2_b),
                                           nullptr, static_cast<const bf16*>(w.ln1_g), static_cast<const bf16*>(w.ln1_b),
                                           c.ln_eps, S, H, m->xln, s));
          acc_pending = false;
        } else if (tp && l > 0) {
          AG_CUDA(ag::launch_layernorm(m->resid, m->proj, static_cast<const bf16*>(m->layers[l - 1].w.fc2_b), nullptr,
                                       static_cast<const bf16*>(w.ln1_g), static_cast<const bf16*>(w.ln1_b), c.ln_eps,
                                       S, H, m->xln, s));
        } else {
          AG_CUDA(ag::launch_layernorm(m->resid, nullptr, nullptr, nullptr, static_cast<const bf16*>(w.ln1_g),
                                       static_cast<const bf16*>(w.ln1_b), c.ln_eps, S, H, m->xln, s));
        }
      }
      {
        // QKV projection: q -> qbuf (scaled), K/V -> paged cache slots (fused KV append)
        ag::GemmEpilogue ep;
        ep.mode = ag::kEpiQkv;
        ep.bias = static_cast<const bf16*>(w.qkv_b);
        ep.out = m->qbuf;
        ep.ldc = m->hq;
        ep.hq = m->hq;
        ep.q_scale = qscale;
        ep.kcache = L.kpool;
        ep.vcache = L.vpool;
        ep.slot_mapping = m->d_slot;
        ep.heads = m->heads_l;
        ep.head_dim = m->head_dim;
        ep.block_size = c.block_size;
        if (ln1_in_qkv) {  // the previous FC2's reductions + LN1, in this GEMM's prologue
          fuse_ln(ep, m->layers[l - 1].w.fc2_b, w.ln1_g, w.ln1_b);
          ep.ln_prologue = 1;
          acc_pending = false;
        }
        ProfScope ps(m, AG_K_QKV_GEMM, s, gemm_flops(S, 3 * m->hq, H),
                     gemm_bytes(S, 3 * m->hq, H, 2) + (ln1_in_qkv ? 2.0 * ln_bytes : 0.0));
        AG_CUDA(gemm_planned(m->tm_xln, L.tm_qkv, S, 3 * m->hq, H, ep, pq, s, m->splitk_ws, m->splitk_cap, m->acc_big));
        AG_TRY(dbg(s, "qkv_gemm", l));
      }
      {
        ag::AttnParams ap;
        ap.q = m->qbuf;
        ap.ldq = m->hq;
        ap.kcache = L.kpool;
        ap.vcache = L.vpool;
        ap.block_table = m->d_bt;
        ap.bt_stride = m->bt_stride;
        ap.cu_q = m->d_cuq;
        ap.ctx_len = m->d_ctx;
        ap.out = m->attn;
        ap.ldo = m->hq;
        ap.part_o = m->part_o;
        ap.part_ml = m->part_ml;
        ap.heads = m->heads_l;
        ap.block_size = c.block_size;
        ag::AttnTmaps atm;
        atm.q = m->tm_qbuf;
        atm.k = L.tm_kpool;
        atm.v = L.tm_vpool;
        ProfScope ps(m, AG_K_ATTENTION, s, m->attn_flops_step, m->attn_bytes_step);
        if (m->n_comb > 0) m->launches_last += 1;
        AG_CUDA(ag::launch_attention(ap, atm, m->d_items, m->n_tile_items, m->n_row_items, m->d_comb, m->n_comb, s));
        AG_TRY(dbg(s, "attention", l));
      }
      bool ln2_done = false;
      {
        // out-proj (+bias +residual when TP=1; partial sum + all-reduce when TP>1)
        ag::GemmEpilogue eo;
        eo.ldc = H;
        ag::GemmPlan po;
        const bool out_atomic = atomic_plan(L.tm_out, H, m->hq, kGemmOut, po);
        if (out_atomic) {
          eo.mode = ag::kEpiAtomicF32;
          eo.acc32 = m->acc32;
          if (m->fuse_ln && !fc1_prologue && S <= ag::gemm_grid(S, H, m->hq, po.bn, po.k_splits, po.am))
            fuse_ln(eo, w.out_b, w.ln2_g, w.ln2_b);
        } else if (!tp) {
          eo.bias = static_cast<const bf16*>(w.out_b);
          eo.residual = m->resid;
          eo.ldr = H;
          eo.out = m->resid;
        } else {
          eo.out = m->proj;
        }
        ProfScope ps(m, AG_K_OUT_GEMM, s, gemm_flops(S, H, m->hq),
                     gemm_bytes(S, H, m->hq, tp ? 2 : 4) + (eo.ln_out ? 2.0 * ln_bytes : 0.0));
        AG_CUDA(gemm_w(m->tm_attn, L.tm_out, S, H, m->hq, eo, s, m->splitk_ws, m->splitk_cap, &m->tune, kGemmOut,
                       &po));
        acc_pending = out_atomic && eo.ln_out == nullptr;
        ln2_done = eo.ln_out != nullptr;
        AG_TRY(dbg(s, "out_gemm", l));
      }
      if (tp) {
        {
          ProfScope ps(m, AG_K_ALLREDUCE, s, 0.0, bf * S * H);
          AG_TRY(allreduce_bf16(m, m->proj, static_cast<size_t>(S) * H, s));
        }
        ProfScope ps(m, AG_K_LAYERNORM, s, 0.0, 2.0 * ln_bytes);
        AG_CUDA(ag::launch_layernorm(m->resid, m->proj, static_cast<const bf16*>(w.out_b), nullptr,
                                     static_cast<const bf16*>(w.ln2_g), static_cast<const bf16*>(w.ln2_b), c.ln_eps, S,
                                     H, m->xln, s));
      } else if (acc_pending && fc1_prologue) {
        // LN2 runs in FC1's prologue (below)
      } else if (acc_pending) {
        ProfScope ps(m, AG_K_LAYERNORM, s, 0.0, 2.0 * ln_bytes);
        AG_CUDA(ag::launch_layernorm_acc(m->resid, m->acc32, static_cast<const bf16*>(w.out_b), nullptr,
                                         static_cast<const bf16*>(w.ln2_g), static_cast<const bf16*>(w.ln2_b), c.ln_eps,
                                         S, H, m->xln, s));
        acc_pending = false;
      } else if (ln2_done) {
        // LN2 was finished by the out-proj's fused tail
      } else {
        ProfScope ps(m, AG_K_LAYERNORM, s, 0.0, ln_bytes);
        AG_CUDA(ag::launch_layernorm(m->resid, nullptr, nullptr, nullptr, static_cast<const bf16*>(w.ln2_g),
                                     static_cast<const bf16*>(w.ln2_b), c.ln_eps, S, H, m->xln, s));
      }
      {
        ag::GemmEpilogue e1;
        e1.bias = static_cast<const bf16*>(w.fc1_b);
        e1.relu = 1;
        e1.out = m->ffn;
        e1.ldc = m->ffn_l;
        const bool ln2_in_fc1 = acc_pending && fc1_prologue;
        if (ln2_in_fc1) {  // the out-proj's reductions + LN2, in this GEMM's prologue
          fuse_ln(e1, w.out_b, w.ln2_g, w.ln2_b);
          e1.ln_prologue = 1;
          acc_pending = false;
        }
        ProfScope ps(m, AG_K_FC1_GEMM, s, gemm_flops(S, m->ffn_l, H),
                     gemm_bytes(S, m->ffn_l, H, 2) + (ln2_in_fc1 ? 2.0 * ln_bytes : 0.0));
        AG_CUDA(gemm_planned(m->tm_xln, L.tm_fc1, S, m->ffn_l, H, e1, p1, s, m->splitk_ws, m->splitk_cap, m->acc_big));
        AG_TRY(dbg(s, "fc1_gemm", l));
      }
      {
        ag::GemmEpilogue e2;
        e2.ldc = H;
        ag::GemmPlan p2;
        const bool fc2_atomic = atomic_plan(L.tm_fc2, H, m->ffn_l, kGemmFc2, p2);
        const bool fuse_next = fc2_atomic && m->fuse_ln && !qkv_prologue && l + 1 < c.num_layers &&
                               S <= ag::gemm_grid(S, H, m->ffn_l, p2.bn, p2.k_splits, p2.am);
        if (fc2_atomic) {
          e2.mode = ag::kEpiAtomicF32;
          e2.acc32 = m->acc32;
          if (fuse_next) {
            const ag_layer_weights& wn = m->layers[l + 1].w;
            fuse_ln(e2, w.fc2_b, wn.ln1_g, wn.ln1_b);
          }
        } else if (!tp) {
          e2.bias = static_cast<const bf16*>(w.fc2_b);
          e2.residual = m->resid;
          e2.ldr = H;
          e2.out = m->resid;
        } else {
          e2.out = m->proj;
        }
        ProfScope ps(m, AG_K_FC2_GEMM, s, gemm_flops(S, H, m->ffn_l),
                     gemm_bytes(S, H, m->ffn_l, tp ? 2 : 4) + (fuse_next ? 2.0 * ln_bytes : 0.0));
        AG_CUDA(gemm_w(m->tm_ffn, L.tm_fc2, S, H, m->ffn_l, e2, s, m->splitk_ws, m->splitk_cap, &m->tune, kGemmFc2,
                       &p2));
        acc_pending = fc2_atomic && !fuse_next;
        ln1_done = fuse_next;
        AG_TRY(dbg(s, "fc2_gemm", l));
      }
      if (tp) {
        ProfScope ps(m, AG_K_ALLREDUCE, s, 0.0, bf * S * H);
        AG_TRY(allreduce_bf16(m, m->proj, static_cast<size_t>(S) * H, s));
      }
    }
    if (acc_pending) {
      // last FC2 split K into acc32: the final LayerNorm (logit rows) applies bias + residual to the
      // rows it reads; every row of acc32 is re-zeroed for the next step
      final_acc = true;
    }
    if (tp) {  // fold the last FC2 all-reduce into the residual stream
      const ag_layer_weights& wl = m->layers[c.num_layers - 1].w;
      ProfScope ps(m, AG_K_LAYERNORM, s, 0.0, 2.0 * ln_bytes);
      AG_CUDA(ag::launch_layernorm(m->resid, m->proj, static_cast<const bf16*>(wl.fc2_b), nullptr, m->final_g,
                                   m->final_b, c.ln_eps, S, H, m->xln, s));
    }
  }
  const int NL = m->n_logit;
  if (NL > 0) {
    {
      // final LayerNorm only on the rows that emit a token (logit skip)
      ProfScope ps(m, AG_K_LAYERNORM, s, 0.0, bf * 2.0 * NL * H);
      if (final_acc)
        AG_CUDA(ag::launch_layernorm_acc(m->resid, m->acc32, static_cast<const bf16*>(m->layers[c.num_layers - 1].w.fc2_b),
                                         m->d_lrows, m->final_g, m->final_b, c.ln_eps, NL, H, m->lm_in, s));
      else
        AG_CUDA(ag::launch_layernorm(m->resid, nullptr, nullptr, m->d_lrows, m->final_g, m->final_b, c.ln_eps, NL, H,
                                     m->lm_in, s));
    }
    ag::GemmEpilogue el;
    // padded vocab shard (TP=8 of 50272 = 6284 columns): the LM head writes vocab_lp columns (the
    // weight map's out-of-range rows load as zeros) into the padded buffer, argmax reads vocab_l
    const bool direct = logits_out && m->vocab_lp == m->vocab_l;
    el.out = direct ? static_cast<void*>(logits_out) : static_cast<void*>(m->logits);
    el.ldc = m->vocab_lp;
    el.out_f32 = 1;
    float* lg = static_cast<float*>(el.out);
    {
      ProfScope ps(m, AG_K_LMHEAD_GEMM, s, gemm_flops(NL, m->vocab_l, H), gemm_bytes(NL, m->vocab_l, H, 4));
      AG_CUDA(gemm_w(m->tm_lm_in, m->tm_lm_w, NL, m->vocab_lp, H, el, s, m->splitk_ws, m->splitk_cap, &m->tune, kGemmLm));
      AG_TRY(dbg(s, "lm_head", -1));
    }
    if (!tp) {
      ProfScope ps(m, AG_K_ARGMAX, s, 0.0, 4.0 * NL * m->vocab_l);
      AG_CUDA(ag::launch_argmax(lg, NL, m->vocab_l, m->vocab_lp, 0, nullptr, out_tokens_dev, s));
    } else {
      {
        ProfScope ps(m, AG_K_ARGMAX, s, 0.0, 4.0 * NL * m->vocab_l);
        AG_CUDA(ag::launch_argmax(lg, NL, m->vocab_l, m->vocab_lp, m->vocab_off, m->cand_val, m->cand_idx, s));
      }
      {
        ProfScope ps(m, AG_K_ALLREDUCE, s, 0.0, 8.0 * NL * c.tp_size);
        AG_TRY(allgather_cands(m, NL, s));
      }
      ProfScope ps(m, AG_K_ARGMAX, s, 0.0, 8.0 * NL * c.tp_size);
      AG_CUDA(ag::launch_argmax_merge(m->gathered_val, m->gathered_idx, c.tp_size, NL, out_tokens_dev, s));
    }
    if (logits_out && !direct)
      AG_CUDA(cudaMemcpy2DAsync(logits_out, sizeof(float) * m->vocab_l, m->logits, sizeof(float) * m->vocab_lp,
                                sizeof(float) * m->vocab_l, NL, cudaMemcpyDeviceToDevice, s));
  }
  if (final_acc) AG_CUDA(cudaMemsetAsync(m->acc32, 0, sizeof(float) * static_cast<size_t>(S) * H, s));
  m->launches_total += m->launches_last;
  return AG_OK;
}

int32_t ag_model_set_profiling(ag_model* m, int32_t on) {
  if (!m) return fail(AG_EINVAL, "null model");
  m->prof_on = on != 0;
  m->prof_pending.clear();
  for (int i = 0; i < AG_PROF_CLASSES; ++i) {
    m->prof_ms[i] = m->prof_flops[i] = m->prof_bytes[i] = m->prof_roof_ms[i] = 0.0;
    m->prof_count[i] = 0;
  }
  if (m->prof_on && m->prof_events.empty()) {
    m->prof_events.resize(2 * (16 * static_cast<size_t>(m->cfg.num_layers) + 64));
    for (auto& e : m->prof_events) AG_CUDA(cudaEventCreate(&e));
  }
  return AG_OK;
}

int32_t ag_model_get_profile(ag_model* m, double* ms, double* flops, double* bytes, int64_t* counts, int32_t n) {
  if (!m) return fail(AG_EINVAL, "null model");
  for (int i = 0; i < std::min<int>(n, AG_PROF_CLASSES); ++i) {
    if (ms) ms[i] = m->prof_ms[i];
    if (flops) flops[i] = m->prof_flops[i];
    if (bytes) bytes[i] = m->prof_bytes[i];
    if (counts) counts[i] = m->prof_count[i];
  }
  return AG_OK;
}

int32_t ag_model_set_roofline_peaks(ag_model* m, double tensor_tflops, double hbm_gbs) {
  if (!m || tensor_tflops < 0.0 || hbm_gbs < 0.0) return fail(AG_EINVAL, "bad peaks");
  m->peak_tflops = tensor_tflops;
  m->peak_gbs = hbm_gbs;
  return AG_OK;
}

int32_t ag_model_get_roofline_ms(ag_model* m, double* roof_ms, int32_t n) {
  if (!m || !roof_ms) return fail(AG_EINVAL, "null argument");
  for (int i = 0; i < std::min<int>(n, AG_PROF_CLASSES); ++i) roof_ms[i] = m->prof_roof_ms[i];
  return AG_OK;
}

int32_t ag_model_autotune(ag_model* m, void* stream) {
  if (!m) return fail(AG_EINVAL, "null model");
  for (int l = 0; l < m->cfg.num_layers; ++l)
    if (!m->layers[l].ready) return fail(AG_EINVAL, "set weights before autotune");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const ag_model_config& c = m->cfg;
  const int H = c.hidden;
  GemmTable& t = m->tune;
  t.m_bucket.clear();
  for (int mb : {16, 32, 64, 128, 192, 256, 320, 384, 448, 512, 640, 768, 896, 1024, 1280, 1536, 2048, 3072, 4096,
                 6144, 8192, 12288, 16384})
    if (mb < c.max_tokens) t.m_bucket.push_back(mb);
  t.m_bucket.push_back(c.max_tokens);
  const size_t T = align_up(static_cast<size_t>(c.max_tokens), 128);
  // non-zero activations of the forward's magnitudes (LN output ~1, attention output ~0.1, ReLU'd
  // FC1): zeroed operands draw less power and would rank plans on optimistic clocks
  AG_CUDA(ag::launch_fill_hash(m->xln, static_cast<int64_t>(T) * H, 0x1234u, 1.7f, false, s));
  AG_CUDA(ag::launch_fill_hash(m->attn, static_cast<int64_t>(T) * m->hq, 0x2345u, 0.17f, false, s));
  AG_CUDA(ag::launch_fill_hash(m->ffn, static_cast<int64_t>(T) * m->ffn_l, 0x3456u, 1.7f, true, s));
  AG_CUDA(ag::launch_fill_hash(m->lm_in, static_cast<int64_t>(align_up(c.max_seqs, 128)) * H, 0x4567u, 1.7f, false, s));
  AG_CUDA(ag::launch_fill_hash(m->resid, static_cast<int64_t>(T) * H, 0x5678u, 1.7f, false, s));
  AG_CUDA(cudaMemsetAsync(m->acc32, 0, sizeof(float) * T * H, s));
  // Candidates are timed on the weights of successive layers (as in the forward), so weight tiles
  // come from HBM, not from an L2 that still holds the previous repetition's copy.
  struct Shape {
    const ActMap* a;
    std::vector<const WeightMap*> w;
    int N, K, mcap;
    void* out;
    int out_f32;
  } shapes[kGemmKinds] = {
      {&m->tm_xln, {}, 3 * m->hq, H, c.max_tokens, m->ffn, 0},
      {&m->tm_attn, {}, H, m->hq, c.max_tokens, m->ffn, 0},
      {&m->tm_xln, {}, m->ffn_l, H, c.max_tokens, m->ffn, 0},
      {&m->tm_ffn, {}, H, m->ffn_l, c.max_tokens, m->proj, 0},
      {&m->tm_lm_in, {&m->tm_lm_w}, m->vocab_lp, H, c.max_seqs, m->logits, 1},
  };
  for (const LayerState& L : m->layers) {
    shapes[kGemmQkv].w.push_back(&L.tm_qkv);
    shapes[kGemmOut].w.push_back(&L.tm_out);
    shapes[kGemmFc1].w.push_back(&L.tm_fc1);
    shapes[kGemmFc2].w.push_back(&L.tm_fc2);
  }
  std::vector<ag::GemmPlan> cands;
  for (int am : {256, 128, 64, 32})
    for (const ag::GemmPlan& q : {ag::GemmPlan{256, 1}, ag::GemmPlan{128, 1}, ag::GemmPlan{64, 1},
                                  ag::GemmPlan{256, 2}, ag::GemmPlan{128, 2}, ag::GemmPlan{64, 2},
                                  ag::GemmPlan{256, 3}, ag::GemmPlan{256, 4}, ag::GemmPlan{128, 4},
                                  ag::GemmPlan{64, 4}, ag::GemmPlan{256, 6}, ag::GemmPlan{128, 6},
                                  ag::GemmPlan{256, 8}, ag::GemmPlan{128, 8}})
      cands.push_back({q.bn, q.k_splits, am});
  for (int am : {128, 64, 32})  // stream-K (atomic fp32 epilogue; finished by LayerNorm or the finish kernel)
    for (int bn : {256, 128, 64}) cands.push_back({bn, ag::kStreamK, am});
  for (int am : {128, 64, 32})
    for (int ks : {1, 2}) cands.push_back({160, ks, am});
  cands.push_back({256, ag::kStreamK, 256});  // stream-K over CTA pairs
  cands.push_back({128, ag::kStreamK, 256});
  cudaEvent_t e0, e1;
  AG_CUDA(cudaEventCreate(&e0));
  AG_CUDA(cudaEventCreate(&e1));
  for (int k = 0; k < kGemmKinds; ++k) {
    t.plan[k].assign(t.m_bucket.size(), ag::GemmPlan{256, 1, 128});
    const Shape& sh = shapes[k];
    for (size_t b = 0; b < t.m_bucket.size(); ++b) {
      const int M = std::min(t.m_bucket[b], sh.mcap);
      float best = 1e30f;
      for (const ag::GemmPlan& p : cands) {
        ag::GemmEpilogue ep;
        ep.out = sh.out;
        ep.ldc = sh.N;
        ep.out_f32 = sh.out_f32;
        if (c.tp_size == 1 && (k == kGemmOut || k == kGemmFc2) && p.k_splits > 1) {
          ep.mode = ag::kEpiAtomicF32;  // as the forward runs split-K out-proj / FC2 at TP=1
          ep.acc32 = m->acc32;
        }
        const bool finish = p.k_splits == ag::kStreamK && (k == kGemmQkv || k == kGemmFc1);
        ag::GemmEpilogue ea;  // stream-K QKV / FC1: atomic accumulation, then the finish kernel
        ea.mode = ag::kEpiAtomicF32;
        ea.acc32 = m->acc_big;
        ea.ldc = sh.N;
        const ag::GemmEpilogue& eg = finish ? ea : ep;
        if (p.am == 256 && (p.bn == 64 || M <= 128)) continue;  // CTA pair: bn 128/256, M > 128
        if (p.bn == 256 && !sh.w[0]->has256 && p.am != 256) continue;
        if (p.bn == 160 && (!sh.w[0]->has160 || p.am == 256)) continue;
        if (p.am < 128 && M > p.am) continue;
        if (p.k_splits == ag::kStreamK) {
          if (k == kGemmLm || (p.am == 256 && M <= 128)) continue;
          if ((k == kGemmOut || k == kGemmFc2) && c.tp_size != 1) continue;
        } else {
          const int nkb = (sh.K + 63) / 64, per = (nkb + p.k_splits - 1) / p.k_splits;
          if ((nkb + per - 1) / per != p.k_splits || (p.k_splits > 1 && per < 2)) continue;
          if (static_cast<int64_t>(p.k_splits) * M * sh.N > m->splitk_cap) continue;
        }
        const int wbox = p.am == 256 ? p.bn / 2 : p.bn;
        const CUtensorMap& am = sh.a->box(p.am == 256 ? 128 : p.am);
        const int nw = static_cast<int>(sh.w.size());
        // TP=1 out-proj / FC2 are timed with the LayerNorm that consumes them, as in the forward: an
        // atomic plan leaves bias + residual + the fp32 accumulator's read-and-re-zero to
        // launch_layernorm_acc (12 B per element more than the direct epilogue's bf16 residual path)
        const bool with_ln = c.tp_size == 1 && (k == kGemmOut || k == kGemmFc2);
        const ag_layer_weights& w0 = m->layers[0].w;
        const bf16* bias_k = static_cast<const bf16*>(k == kGemmOut ? w0.out_b : w0.fc2_b);
        ag::GemmEpilogue ed = eg;
        if (with_ln && ed.mode != ag::kEpiAtomicF32) {
          ed.bias = bias_k;
          ed.residual = m->resid;
          ed.ldr = H;
          ed.out = m->resid;
        }
        const bool fused = with_ln && ed.mode == ag::kEpiAtomicF32 && m->fuse_ln &&
                           M <= ag::gemm_grid(M, sh.N, sh.K, p.bn, p.k_splits, p.am);
        if (fused) {  // the forward's fused LayerNorm tail (one launch)
          ed.ln_acc = m->acc32;
          ed.ln_ld = H;
          ed.ln_x = m->resid;
          ed.ln_bias = bias_k;
          ed.ln_g = static_cast<const bf16*>(w0.ln2_g);
          ed.ln_b = static_cast<const bf16*>(w0.ln2_b);
          ed.ln_eps = c.ln_eps;
          ed.ln_out = m->xln;
          ed.ln_bar = m->ln_bar;
        }
        auto one = [&](int rep) -> cudaError_t {
          cudaError_t e = ag::launch_gemm(am, sh.w[rep % nw]->box(wbox), M, sh.N, sh.K, p.bn, ed, 0, s, p.k_splits,
                                          m->splitk_ws, p.am);
          if (e != cudaSuccess) return e;
          if (finish) return ag::launch_splitk_finish(m->acc_big, M, sh.N, ep, s);
          if (!with_ln || fused) return cudaSuccess;
          const bf16* g = static_cast<const bf16*>(w0.ln2_g);
          const bf16* bb = static_cast<const bf16*>(w0.ln2_b);
          if (ed.mode == ag::kEpiAtomicF32)
            return ag::launch_layernorm_acc(m->resid, m->acc32, bias_k, nullptr, g, bb,
                                            c.ln_eps, M, H, m->xln, s);
          return ag::launch_layernorm(m->resid, nullptr, nullptr, nullptr, g, bb, c.ln_eps, M, H, m->xln, s);
        };
        AG_CUDA(one(nw - 1));
        const int iters = 8;
        AG_CUDA(cudaEventRecord(e0, s));
        for (int rep = 0; rep < iters; ++rep) AG_CUDA(one(rep));
        AG_CUDA(cudaEventRecord(e1, s));
        AG_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        AG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best * 0.985f) {  // prefer earlier (simpler) plans on near-ties
          best = ms;
          t.plan[k][b] = p;
        }
      }
      if (std::getenv("AG_AUTOTUNE_LOG"))
        std::fprintf(stderr, "{\"autotune\": %d, \"M\": %d, \"N\": %d, \"K\": %d, \"us\": %.2f, \"bn\": %d, \"ks\": %d, \"am\": %d}\n",
                     k, M, sh.N, sh.K, best * 1e3f / 8, t.plan[k][b].bn, t.plan[k][b].k_splits, t.plan[k][b].am);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  AG_CUDA(cudaMemsetAsync(m->acc32, 0, sizeof(float) * T * H, s));
  AG_CUDA(cudaStreamSynchronize(s));
  t.ready = true;
  return AG_OK;
}

int32_t ag_model_get_gemm_plans(ag_model* m, int32_t* out, int32_t cap) {
  // rows of (kind, m_bucket, block_n, k_splits); returns the row count
  if (!m || !m->tune.ready) return 0;
  int n = 0;
  for (int k = 0; k < kGemmKinds; ++k)
    for (size_t b = 0; b < m->tune.m_bucket.size(); ++b) {
      if (n < cap) {
        out[4 * n] = k;
        out[4 * n + 1] = m->tune.m_bucket[b];
        out[4 * n + 2] = m->tune.plan[k][b].bn;
        out[4 * n + 3] = m->tune.plan[k][b].k_splits + 100 * m->tune.plan[k][b].am;
      }
      ++n;
    }
  return n;
}

int32_t ag_model_set_gemm_plans(ag_model* m, const int32_t* rows, int32_t n) {
  if (!m || (n > 0 && !rows)) return fail(AG_EINVAL, "null argument");
  GemmTable t;
  for (int i = 0; i < n; ++i) {
    const int kind = rows[4 * i], mb = rows[4 * i + 1], bn = rows[4 * i + 2], ks = rows[4 * i + 3] % 100,
              am = rows[4 * i + 3] / 100;
    if (kind < 0 || kind >= kGemmKinds || mb <= 0 || (bn != 64 && bn != 128 && bn != 160 && bn != 256) || ks < 1 ||
        (am != 32 && am != 64 && am != 128 && am != 256))
      return fail(AG_EINVAL, "bad gemm plan row " + std::to_string(i));
    if (kind == 0) t.m_bucket.push_back(mb);
    t.plan[kind].push_back(ag::GemmPlan{bn, ks, am});
  }
  for (int k = 0; k < kGemmKinds; ++k)
    if (t.plan[k].size() != t.m_bucket.size()) return fail(AG_EINVAL, "plan table is not rectangular");
  t.ready = !t.m_bucket.empty();
  m->tune = t;
  return AG_OK;
}

int64_t ag_model_last_launches(ag_model* m) { return m ? m->launches_last : -1; }
int64_t ag_model_last_h2d_bytes(ag_model* m) { return m ? m->h2d_last : -1; }

int32_t ag_model_forward(ag_model* m, const ag_step* st, int32_t* out_tokens, float* logits_out, float* device_ms,
                         void* stream) {
  if (!m || !st) return fail(AG_EINVAL, "null argument");
  if (m->n_submit != m->n_wait) return fail(AG_ESTATE, "ag_model_forward with asynchronous steps in flight");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  AG_TRY(ag_model_stage_step(m, st, stream));
  AG_CUDA(cudaEventRecord(m->ev0, s));
  AG_TRY(ag_model_forward_staged(m, m->out_tok, logits_out, stream));
  AG_CUDA(cudaEventRecord(m->ev1, s));
  if (m->n_logit > 0)
    AG_CUDA(cudaMemcpyAsync(m->tok_host, m->out_tok, sizeof(int32_t) * m->n_logit, cudaMemcpyDeviceToHost, s));
  AG_CUDA(cudaStreamSynchronize(s));
  if (device_ms) AG_CUDA(cudaEventElapsedTime(device_ms, m->ev0, m->ev1));
  if (m->prof_on) prof_harvest(m);
  if (out_tokens && m->n_logit > 0) std::memcpy(out_tokens, m->tok_host, sizeof(int32_t) * m->n_logit);
  return AG_OK;
}

int32_t ag_model_clock_ref(ag_model* m, void* stream) {
  if (!m) return fail(AG_EINVAL, "null model");
  if (!m->ev_ref) AG_CUDA(cudaEventCreate(&m->ev_ref));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  AG_CUDA(cudaEventRecord(m->ev_ref, s));
  AG_CUDA(cudaEventSynchronize(m->ev_ref));
  return AG_OK;
}

int32_t ag_model_submit(ag_model* m, const ag_step* st, const int32_t* feed_pairs, int32_t n_feed, float* logits_out,
                        void* stream) {
  if (!m || !st) return fail(AG_EINVAL, "null argument");
  if (m->prof_on) return fail(AG_ESTATE, "per-kernel profiling needs the synchronous ag_model_forward");
  if (n_feed < 0 || n_feed > st->num_tokens || (n_feed > 0 && !feed_pairs)) return fail(AG_EINVAL, "bad feed");
  if (n_feed > 0 && m->n_submit == 0) return fail(AG_ESTATE, "decode feed without a previous step");
  const int k = static_cast<int>(m->n_submit & 1);
  ag_model::AsyncSlot& a = m->aslot[k];
  if (a.active) return fail(AG_ESTATE, "two asynchronous steps already in flight: ag_model_wait first");
  const ag_model_config& c = m->cfg;
  const size_t Sq = static_cast<size_t>(c.max_seqs);
  if (!a.start) {  // lazily: slot 0 aliases the synchronous path's buffers
    if (k == 0) {
      a.meta_host = m->meta_host;
      a.out_tok = m->out_tok;
      a.tok_host = m->tok_host;
    } else {
      if (cudaMallocHost(&a.meta_host, m->meta_cap) != cudaSuccess) return fail(AG_EALLOC, "pinned alloc");
      if (cudaMallocHost(&a.tok_host, Sq * sizeof(int32_t)) != cudaSuccess) return fail(AG_EALLOC, "pinned alloc");
      AG_CUDA(cudaMalloc(&a.out_tok, Sq * sizeof(int32_t)));
    }
    if (cudaMallocHost(&a.feed_host, 2 * sizeof(int32_t) * c.max_tokens) != cudaSuccess)
      return fail(AG_EALLOC, "pinned alloc");
    if (!m->feed_dev) AG_CUDA(cudaMalloc(&m->feed_dev, 2 * 2 * sizeof(int32_t) * c.max_tokens));
    AG_CUDA(cudaEventCreate(&a.start));
    AG_CUDA(cudaEventCreate(&a.end));
    AG_CUDA(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming));
  }
  for (int i = 0; i < n_feed; ++i) {
    const int dst = feed_pairs[2 * i], src = feed_pairs[2 * i + 1];
    if (dst < 0 || dst >= st->num_tokens || src < 0 || src >= m->aslot[k ^ 1].n_logit)
      return fail(AG_EINVAL, "decode feed pair out of range");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  m->meta_host = a.meta_host;
  AG_TRY(ag_model_stage_step(m, st, stream));
  if (n_feed > 0) {
    int32_t* fd = m->feed_dev + 2 * static_cast<size_t>(c.max_tokens) * k;
    std::memcpy(a.feed_host, feed_pairs, 2 * sizeof(int32_t) * n_feed);
    AG_CUDA(cudaMemcpyAsync(fd, a.feed_host, 2 * sizeof(int32_t) * n_feed, cudaMemcpyHostToDevice, s));
    AG_CUDA(ag::launch_feed_tokens(const_cast<int32_t*>(m->d_ids), fd, n_feed, m->aslot[k ^ 1].out_tok, s));
    m->h2d_last += 8 * n_feed;
  }
  AG_CUDA(cudaEventRecord(a.start, s));
  AG_TRY(ag_model_forward_staged(m, a.out_tok, logits_out, stream));
  AG_CUDA(cudaEventRecord(a.end, s));
  if (m->n_logit > 0)
    AG_CUDA(cudaMemcpyAsync(a.tok_host, a.out_tok, sizeof(int32_t) * m->n_logit, cudaMemcpyDeviceToHost, s));
  AG_CUDA(cudaEventRecord(a.done, s));
  a.n_logit = m->n_logit;
  a.active = true;
  ++m->n_submit;
  return AG_OK;
}

int32_t ag_model_wait(ag_model* m, int32_t* out_tokens, int32_t cap, float* device_ms, double* end_ms_since_ref) {
  if (!m) return fail(AG_EINVAL, "null model");
  if (m->n_wait == m->n_submit) return fail(AG_ESTATE, "no asynchronous step in flight");
  ag_model::AsyncSlot& a = m->aslot[m->n_wait & 1];
  AG_CUDA(cudaEventSynchronize(a.done));
  if (device_ms) AG_CUDA(cudaEventElapsedTime(device_ms, a.start, a.end));
  if (end_ms_since_ref) {
    float ms = -1.f;
    if (m->ev_ref) AG_CUDA(cudaEventElapsedTime(&ms, m->ev_ref, a.end));
    *end_ms_since_ref = ms;
  }
  if (out_tokens && a.n_logit > 0) {
    if (cap < a.n_logit) return fail(AG_EINVAL, "out_tokens too small");
    std::memcpy(out_tokens, a.tok_host, sizeof(int32_t) * a.n_logit);
  }
  a.active = false;
  ++m->n_wait;
  return AG_OK;
}

int32_t ag_model_inflight(ag_model* m) { return m ? static_cast<int32_t>(m->n_submit - m->n_wait) : -1; }

// ---------------------------------------------------------------- standalone kernels
int32_t ag_gemm_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, const void* bias, const void* residual,
                     int32_t ldr, int32_t relu, void* D, int32_t ldd, int32_t out_f32, int32_t M, int32_t N, int32_t K,
                     int32_t block_n, int32_t k_splits, int32_t a_rows, void* workspace, int64_t workspace_bytes,
                     void* stream) {
  if (a_rows == 0) a_rows = 128;
  if (a_rows != 32 && a_rows != 64 && a_rows != 128 && a_rows != 256)
    return fail(AG_EINVAL, "a_rows must be 32, 64, 128 or 256 (CTA pair)");
  if (a_rows < 128 && M > a_rows) return fail(AG_EINVAL, "a_rows < M");
  if (a_rows == 256 && block_n != 128 && block_n != 256) return fail(AG_EINVAL, "CTA pair needs block_n 128/256");
  if (!A || !W || !D) return fail(AG_EINVAL, "null pointer");
  if (M < 0 || N <= 0 || K <= 0 || N % 32 != 0 || K % 8 != 0) return fail(AG_EINVAL, "need N%32==0, K%8==0");
  const int64_t cap = workspace ? workspace_bytes / 4 : 0;
  if (block_n == 0 && k_splits == 0) {
    const ag::GemmPlan p = ag::plan_gemm(M, N, K, cap);
    block_n = p.bn;
    k_splits = p.k_splits;
  }
  if (block_n == 0) block_n = ag::pick_block_n(M, N);
  if (k_splits <= 0) k_splits = 1;
  if (k_splits > 1 && static_cast<int64_t>(k_splits) * M * N > cap)
    return fail(AG_EALLOC, "split-K workspace too small");
  {
    const int nkb = (K + 63) / 64, per = (nkb + k_splits - 1) / k_splits;
    if ((nkb + per - 1) / per != k_splits) return fail(AG_EINVAL, "k_splits leaves an empty K range");
  }
  if (block_n != 64 && block_n != 128 && block_n != 160 && block_n != 256)
    return fail(AG_EINVAL, "block_n must be 64, 128, 160 or 256");
  CUtensorMap ta, tb;
  int r = ag::make_tmap_kmajor(&ta, A, std::max<int64_t>(M, 1), K, lda, a_rows == 256 ? 128 : a_rows);
  if (r) return fail(AG_EINVAL, "tensor map A failed (alignment?)");
  r = ag::make_tmap_kmajor(&tb, W, N, K, ldw, a_rows == 256 ? block_n / 2 : block_n);
  if (r) return fail(AG_EINVAL, "tensor map W failed (alignment?)");
  ag::GemmEpilogue ep;
  ep.bias = static_cast<const bf16*>(bias);
  ep.residual = static_cast<const bf16*>(residual);
  ep.ldr = ldr;
  ep.relu = relu;
  ep.out = D;
  ep.ldc = ldd;
  ep.out_f32 = out_f32;
  AG_CUDA(ag::launch_gemm(ta, tb, M, N, K, block_n, ep, 0, static_cast<cudaStream_t>(stream), k_splits,
                          static_cast<float*>(workspace), a_rows));
  return AG_OK;
}

int32_t ag_kv_append(const void* k, const void* v, int32_t ld, const int32_t* slot_mapping, int32_t rows,
                     int32_t heads, int32_t block_size, void* k_pool, void* v_pool, void* stream) {
  if (!k || !v || !slot_mapping || !k_pool || !v_pool) return fail(AG_EINVAL, "null pointer");
  AG_CUDA(ag::launch_kv_append(static_cast<const bf16*>(k), static_cast<const bf16*>(v), ld, slot_mapping, rows, heads,
                               128, block_size, static_cast<bf16*>(k_pool), static_cast<bf16*>(v_pool),
                               static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_paged_attention(const void* q, int32_t ldq, const void* k_pool, const void* v_pool, int32_t pool_blocks,
                           const int32_t* block_table_dev, int32_t bt_stride, const int32_t* cu_q_host,
                           const int32_t* ctx_len_host, const int32_t* cu_q_dev, const int32_t* ctx_len_dev,
                           int32_t num_seqs, int32_t heads, int32_t block_size, void* out, int32_t ldo,
                           void* workspace, int64_t workspace_bytes, void* stream) {
  const int64_t q_rows_total = num_seqs > 0 ? cu_q_host[num_seqs] : 0;
  if (!q || !k_pool || !v_pool || !block_table_dev || !cu_q_host || !ctx_len_host || !out || !workspace)
    return fail(AG_EINVAL, "null pointer");
  if (block_size != 32) return fail(AG_EINVAL, "block_size must be 32");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // workspace: [items][combines][part_o][part_ml]
  const int64_t row_bytes = static_cast<int64_t>(heads) * (128 + 2) * 4;
  const int64_t meta_reserve = 1 << 20;
  if (workspace_bytes < meta_reserve + row_bytes * 64) return fail(AG_EALLOC, "workspace too small");
  const int part_cap = static_cast<int>((workspace_bytes - meta_reserve) / row_bytes);
  AttnWork w;
  build_attention_work(cu_q_host, ctx_len_host, num_seqs, heads, part_cap, w);
  const size_t ib = sizeof(AttnItem) * w.items.size(), cb = sizeof(AttnCombine) * w.combines.size();
  if (static_cast<int64_t>(align_up(ib, 256) + cb) > meta_reserve) return fail(AG_EALLOC, "too many attention items");
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  AG_CUDA(cudaMemcpyAsync(ws, w.items.data(), ib, cudaMemcpyHostToDevice, s));
  AG_CUDA(cudaMemcpyAsync(ws + align_up(ib, 256), w.combines.data(), cb, cudaMemcpyHostToDevice, s));
  ag::AttnParams ap;
  ap.q = static_cast<const bf16*>(q);
  ap.ldq = ldq;
  ap.kcache = static_cast<const bf16*>(k_pool);
  ap.vcache = static_cast<const bf16*>(v_pool);
  ap.block_table = block_table_dev;
  ap.bt_stride = bt_stride;
  ap.cu_q = cu_q_dev;
  ap.ctx_len = ctx_len_dev;
  ap.out = static_cast<bf16*>(out);
  ap.ldo = ldo;
  ap.part_o = reinterpret_cast<float*>(ws + meta_reserve);
  ap.part_ml = ap.part_o + static_cast<int64_t>(part_cap) * heads * 128;
  ap.heads = heads;
  ap.block_size = block_size;
  ag::AttnTmaps atm;
  {
    int64_t nblk = 0;
    // pool extent: highest block id referenced + 1 (host copy not available: use the workspace bound)
    nblk = pool_blocks;
    const int64_t pool_rows = nblk * heads * block_size;
    int r1 = ag::make_tmap_kmajor(&atm.q, q, std::max<int64_t>(q_rows_total, 1), 128 * heads, ldq, 128);
    int r2 = ag::make_tmap_kmajor(&atm.k, k_pool, pool_rows, 128, 128, 32);
    int r3 = ag::make_tmap_kmajor(&atm.v, v_pool, pool_rows, 128, 128, 32);
    if (r1 || r2 || r3) return fail(AG_EINVAL, "attention tensor maps failed (alignment?)");
  }
  AG_CUDA(ag::launch_attention(ap, atm, reinterpret_cast<const AttnItem*>(ws), w.n_tile, w.n_row,
                               reinterpret_cast<const AttnCombine*>(ws + align_up(ib, 256)),
                               static_cast<int>(w.combines.size()), s));
  // the host work vectors must outlive the async copies
  AG_CUDA(cudaStreamSynchronize(s));
  return AG_OK;
}

int32_t ag_layernorm(void* x, const void* delta, const void* delta_bias, const int32_t* row_index, const void* gamma,
                     const void* beta, float eps, int32_t rows, int32_t hidden, void* out, void* stream) {
  if (!x || !gamma || !beta || !out) return fail(AG_EINVAL, "null pointer");
  AG_CUDA(ag::launch_layernorm(static_cast<bf16*>(x), static_cast<const bf16*>(delta),
                               static_cast<const bf16*>(delta_bias), row_index, static_cast<const bf16*>(gamma),
                               static_cast<const bf16*>(beta), eps, rows, hidden, static_cast<bf16*>(out),
                               static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_rmsnorm(void* x, const void* delta, const void* gamma, float eps, int32_t rows, int32_t hidden, void* out,
                   void* stream) {
  if (!x || !gamma || !out) return fail(AG_EINVAL, "null pointer");
  if (hidden % 8 || hidden > 5120) return fail(AG_EINVAL, "hidden must be a multiple of 8 and <= 5120");
  AG_CUDA(ag::launch_rmsnorm(static_cast<bf16*>(x), static_cast<const bf16*>(delta), static_cast<const bf16*>(gamma),
                             eps, rows, hidden, static_cast<bf16*>(out), static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_rope(void* x, int32_t ld, const int32_t* positions, int32_t rows, int32_t heads, int32_t head_dim,
                int32_t rotary_dim, float theta, void* stream) {
  if (!x || !positions) return fail(AG_EINVAL, "null pointer");
  if (rotary_dim % 8 || rotary_dim > head_dim || ld % 4 || head_dim % 4 || theta <= 1.0f)
    return fail(AG_EINVAL, "rotary_dim must be a multiple of 8 <= head_dim, theta > 1");
  AG_CUDA(ag::launch_rope(static_cast<bf16*>(x), ld, positions, rows, heads, head_dim, rotary_dim, theta,
                          static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_embed_pos(const int32_t* ids, const int32_t* positions, const void* tok_emb, const void* pos_emb,
                     int32_t pos_offset, int32_t rows, int32_t hidden, int32_t vocab, int32_t pos_rows, void* out,
                     void* stream) {
  if (!ids || !positions || !tok_emb || !pos_emb || !out) return fail(AG_EINVAL, "null pointer");
  if (hidden % 8) return fail(AG_EINVAL, "hidden % 8 != 0");
  AG_CUDA(ag::launch_embed(ids, positions, static_cast<const bf16*>(tok_emb), static_cast<const bf16*>(pos_emb),
                           pos_offset, rows, hidden, vocab, pos_rows, static_cast<bf16*>(out),
                           static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_argmax(const float* logits, int32_t rows, int32_t cols, int32_t ld, int32_t index_offset, float* out_val,
                  int32_t* out_idx, void* stream) {
  if (!logits || !out_idx) return fail(AG_EINVAL, "null pointer");
  AG_CUDA(ag::launch_argmax(logits, rows, cols, ld, index_offset, out_val, out_idx, static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_kv_swap_out(const void* pool, const int32_t* block_ids_dev, int32_t n_blocks, int64_t block_elems,
                       void* staging, void* stream) {
  if (!pool || !block_ids_dev || !staging) return fail(AG_EINVAL, "null pointer");
  AG_CUDA(ag::launch_block_copy(static_cast<const bf16*>(pool), static_cast<bf16*>(staging), block_ids_dev, n_blocks,
                                block_elems, true, static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_kv_swap_in(const void* staging, const int32_t* block_ids_dev, int32_t n_blocks, int64_t block_elems,
                      void* pool, void* stream) {
  if (!pool || !block_ids_dev || !staging) return fail(AG_EINVAL, "null pointer");
  AG_CUDA(ag::launch_block_copy(static_cast<const bf16*>(staging), static_cast<bf16*>(pool), block_ids_dev, n_blocks,
                                block_elems, false, static_cast<cudaStream_t>(stream)));
  return AG_OK;
}

int32_t ag_kv_swap_out_planes(const void* pool, int64_t pool_plane_elems, const int32_t* block_ids_dev,
                              int32_t n_blocks, int64_t block_elems, void* staging, int64_t stage_plane_elems,
                              int32_t planes, void* stream) {
  if (!pool || !block_ids_dev || !staging) return fail(AG_EINVAL, "null pointer");
  if (planes < 1 || n_blocks < 0) return fail(AG_EINVAL, "planes >= 1, n_blocks >= 0");
  AG_CUDA(ag::launch_block_copy(static_cast<const bf16*>(pool), static_cast<bf16*>(staging), block_ids_dev, n_blocks,
                                block_elems, true, static_cast<cudaStream_t>(stream), planes, pool_plane_elems,
                                stage_plane_elems));
  return AG_OK;
}

int32_t ag_kv_swap_in_planes(const void* staging, int64_t stage_plane_elems, const int32_t* block_ids_dev,
                             int32_t n_blocks, int64_t block_elems, void* pool, int64_t pool_plane_elems,
                             int32_t planes, void* stream) {
  if (!pool || !block_ids_dev || !staging) return fail(AG_EINVAL, "null pointer");
  if (planes < 1 || n_blocks < 0) return fail(AG_EINVAL, "planes >= 1, n_blocks >= 0");
  AG_CUDA(ag::launch_block_copy(static_cast<const bf16*>(staging), static_cast<bf16*>(pool), block_ids_dev, n_blocks,
                                block_elems, false, static_cast<cudaStream_t>(stream), planes, pool_plane_elems,
                                stage_plane_elems));
  return AG_OK;
}

}  // extern "C"
