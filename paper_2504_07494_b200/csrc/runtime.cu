// Host runtime behind the C ABI (include/hc.h): unit-block pool allocator and block
// tables, append (a2), decode-call descriptor / split-K work list
// (a3) and launch sequencing of the reconstruction GEMM (a4), attention (a5) and
// combine (a6).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <queue>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/hc.h"
#include "internal.h"

using namespace hc;

namespace {

thread_local std::string g_err;

hc_status fail(hc_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
hc_status cuda_fail(cudaError_t e, const char* where) {
  return fail(HC_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr size_t kStagingBytes = 4u << 20;  // append descriptor staging inside storage
constexpr int kRing = 16;  // pinned host staging buffers: the host may run up to 16 calls ahead
                           // of the GPU (absorbs host-side stalls, e.g. NVML polling)
constexpr size_t kHeaderBytes = 128 + 128 * 80;  // zeroed each call: attention task counter (byte 0), GEMM
                                                 // tile counter (byte 64), 80 pair-progress lines

struct Req {
  int32_t mode = 0;
  int64_t n = 0;
  std::vector<int32_t> a;  // K blocks (KV) or X blocks (hidden)
  std::vector<int32_t> b;  // V blocks (KV)
};

struct Layout {  // storage layout
  size_t blocks_off, blocks_bytes;
  size_t wq_off;          // W_Q [d,d] directly in front of W_int, so [W_Q; W_int] is one [3d,d] operand
  size_t w_off, w_bytes;  // head-interleaved W_KV [2d,d]
  size_t bq_off;          // b_Q [d] fp32 directly in front of b_int
  size_t b_off, b_bytes;  // head-interleaved b_KV [2d] fp32
  size_t wo_off, bo_off;  // W_O [d,d], b_O [d] (when configured)
  size_t rope_off;        // RoPE inv_freq [dh/2] fp64 (when rope_theta > 0)
  size_t ln_off;          // LayerNorm gamma [d] then beta [d] fp32 (when ln_gamma != NULL)
  size_t stage_off, total;
  bool has_q, has_o, has_ln;
};

// K/V geometry (GQA, DESIGN R18): Hk K/V heads, K (or V) row width dk = Hk*dh, tokens per KV
// logical block Bkv, and whether K and V share one unit (packed: Bkv = B d / (2 dk)).
struct KvGeom {
  int32_t Hk = 0, dk = 0, Bkv = 0;
  bool packed = false;
  int64_t v_off = 0;   // elements from a V unit's base to its V rows
};
bool kv_geom(const hc_pool_config* c, KvGeom* g) {
  const int32_t Hk = c->n_kv_heads > 0 ? c->n_kv_heads : c->n_heads;
  if (Hk > c->n_heads || c->n_heads % Hk != 0 || c->n_kv_heads < 0) return false;
  g->Hk = Hk;
  g->dk = Hk * c->head_dim;
  if (Hk == c->n_heads) {   // multi-head: a K unit and a V unit per B tokens
    g->Bkv = c->block_size;
    g->packed = false;
    g->v_off = 0;
    return true;
  }
  if (c->d_model % (2 * g->dk) != 0) return false;
  g->Bkv = c->block_size * (c->d_model / (2 * g->dk));
  g->packed = true;
  g->v_off = (int64_t)Hk * g->Bkv * c->head_dim;
  return true;
}

bool layout_for(const hc_pool_config* c, Layout* L) {
  if (!c || c->d_model <= 0 || c->n_heads <= 0 || c->head_dim <= 0 || c->block_size <= 0 ||
      c->num_blocks <= 0 || (c->dtype != HC_BF16 && c->dtype != HC_F32))
    return false;
  if ((int64_t)c->n_heads * c->head_dim != c->d_model) return false;
  KvGeom kg;
  if (!kv_geom(c, &kg)) return false;
  const size_t e = c->dtype == HC_BF16 ? 2 : 4;
  const size_t d = (size_t)c->d_model, dk = (size_t)kg.dk;
  L->has_q = c->w_q != nullptr;
  L->has_o = c->w_o != nullptr;
  L->has_ln = c->ln_gamma != nullptr;
  L->blocks_off = 0;
  L->blocks_bytes = (size_t)c->num_blocks * c->block_size * d * e;
  L->wq_off = align_up(L->blocks_off + L->blocks_bytes, 1024);
  L->w_off = L->wq_off + (L->has_q ? d * d * e : 0);
  L->w_bytes = 2 * dk * d * e;
  L->bq_off = align_up(L->w_off + L->w_bytes, kAlign);
  L->b_off = L->bq_off + d * sizeof(float);
  L->b_bytes = 2 * dk * sizeof(float);
  size_t o = align_up(L->b_off + L->b_bytes, 1024);
  L->wo_off = L->bo_off = 0;
  if (L->has_o) {
    L->wo_off = o;
    L->bo_off = align_up(L->wo_off + d * d * e, kAlign);
    o = align_up(L->bo_off + d * sizeof(float), kAlign);
  }
  L->rope_off = 0;
  if (c->rope_theta > 0.f) {
    L->rope_off = o;
    o = align_up(o + (size_t)c->head_dim / 2 * sizeof(double), kAlign);
  }
  L->ln_off = 0;
  if (L->has_ln) {
    L->ln_off = o;
    o = align_up(o + 2 * d * sizeof(float), kAlign);
  }
  L->stage_off = align_up(o, kAlign);
  L->total = align_up(L->stage_off + kStagingBytes, kAlign);
  return true;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool make_tmap_2d(CUtensorMap* m, void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                  uint32_t box_outer) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// The library's only environment read: schedule / A-B knobs, once per hc_pool_create
// (see internal.h Tuning).  Unparsable values keep the default.
int env_int(const char* k, int dflt) {
  const char* v = std::getenv(k);
  if (!v || !*v) return dflt;
  char* end = nullptr;
  const long x = std::strtol(v, &end, 10);
  return (end && *end == 0) ? (int)x : dflt;
}
Tuning tuning_from_env() {
  Tuning t;
  t.fused = env_int("HC_FUSED", t.fused);
  t.epi_attend = env_int("HC_EPI_ATTEND", t.epi_attend);
  t.fused_cfg = env_int("HC_FUSED_CFG", t.fused_cfg);
  t.fused_nsub = env_int("HC_FUSED_NSUB", t.fused_nsub);
  t.group_n = env_int("HC_GROUP_N", t.group_n);
  t.sync_w = env_int("HC_SYNC_W", t.sync_w);
  t.group_m = env_int("HC_GROUP_M", t.group_m);
  t.l2_hint = env_int("HC_L2HINT", t.l2_hint);
  t.attn_tc = env_int("HC_ATTN_TC", t.attn_tc);
  t.gqa_scratch = env_int("HC_GQA_SCRATCH", t.gqa_scratch);
  t.block_runs = env_int("HC_BLOCK_RUNS", t.block_runs);
  t.tc_1sm = env_int("HC_TC_1SM", t.tc_1sm);
  t.tc_nsub = env_int("HC_TC_NSUB", t.tc_nsub);
  t.tc_stages = env_int("HC_TC_STAGES", t.tc_stages);
  t.attn_cfg = env_int("HC_ATTN_CFG", t.attn_cfg);
  t.prefill_tc = env_int("HC_PREFILL_TC", t.prefill_tc);
  t.prefill_cfg = env_int("HC_PREFILL_CFG", t.prefill_cfg);
  t.z_cfg = env_int("HC_Z_CFG", t.z_cfg);
  t.score_st = env_int("HC_SCORE_ST", t.score_st);
  t.qt_bn = env_int("HC_QT_BN", t.qt_bn);
  t.attn_sms = env_int("HC_ATTN_SMS", t.attn_sms);
  t.dyn_tiles = env_int("HC_DYN_TILES", t.dyn_tiles);
  t.epi_mma = env_int("HC_EPI_MMA", t.epi_mma);
#ifdef HC_DIAG
  t.diag_epi = env_int("HC_DIAG_EPI", 0);
  t.diag_box = env_int("HC_DIAG_BOX", 0);
  t.diag_attn = env_int("HC_DIAG_ATTN", 0);
#endif
  return t;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct Pinned {
  void* ptr = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
  bool captured = false;   // used by a call captured into a CUDA graph: the graph's memcpy node
                           // reads this buffer at every replay, so it leaves the rotation
};

// Decode-call plan: sizes and offsets inside the caller's workspace.
struct Plan {
  int32_t n_req = 0, n_splits = 0, n_hb = 0, split_blocks = 1, split_blocks_kv = 1;
  int32_t n_kv_splits = 0, n_hid_splits = 0;
  int64_t kv_tokens = 0;
  bool fused = false;                 // reconstruction + attention in one kernel (fused.cu)
  bool absorb = false;                // hidden requests through absorbed.cu (f4 (ii)), no splits
  bool attend = false;                // fused reconstruct-and-attend epilogue (no K/V scratch)
  bool tc = false;                    // tensor-core KV loop (attn_tc.cuh) for every attention task
  bool gqa_scratch = false;           // GQA: hidden K/V via scratch, attended by the tensor-core loop
  int32_t seg = 0;                    // attend: tokens per hidden partial (min(B, 32))
  size_t off_hreqblk = 0;             // attend: batch index of each hidden block's request
  int32_t n_h = 0, n_atiles = 0, Hp = 0;
  int32_t gemm_m_tiles = 0, gemm_n_tiles = 0;
  int64_t n_tab = 0;
  size_t off_reqs, off_splits, off_tabs, off_gather, off_hpos, off_kvsplit, off_hidsplit, off_tiledone, desc_bytes;
  size_t off_ml, off_acc, off_sk, off_sv, total;
  size_t off_hreq, off_hrow0, off_hntok, off_htile0, off_treq, off_tt0;   // absorb descriptor
  size_t off_qt, off_tml, off_pm, off_abml, off_z;                        // absorb workspace
};

}  // namespace

struct hc_pool {
  hc_pool_config cfg{};
  Layout L{};
  Tuning tune{};   // read once at create
  KvGeom kv{};     // K/V heads, row width, tokens per KV logical block (GQA, R18)
  size_t elem = 2;
  bool accounting = false;
  bool has_bias = false;
  char* storage = nullptr;
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_ids;
  std::unordered_map<int64_t, Req> reqs;
  CUtensorMap tmap_x{}, tmap_w{}, tmap_w_half{};
  CUtensorMap tmap_wqkv{}, tmap_wo{};   // [W_Q; W_int] and W_O with 128-row boxes (dense pair GEMMs)
  CUtensorMap tmap_x64{};               // pool rows, {64 x min(B,64)} boxes (absorbed Z GEMM)
  CUtensorMap tmap_kv{};                // pool as rows of dh elements, {64 x 16} boxes, 128-B swizzle (KV chunks)
  CUtensorMap tmap_x128{};              // pool rows, {64 x 128} boxes: runs of consecutive hidden blocks
  bool x128_ok = false;
  bool attn_tc_ok = false;              // tmap_kv built and attn_tc_supported
  bool tc_ok = false;
  bool dense_tc_ok = false;             // bf16 tcgen05 path for the current-token / output GEMMs
  int num_sms = 148;
  std::array<Pinned, kRing> ring{};
  int ring_next = 0;
  int32_t last_launches = 0;
  int32_t last_path = -1;
  int32_t last_cfg = 0;   // fused-kernel configuration of the last decode (see hc_last_kernel_config)
  bool profiling = false;
  std::vector<std::array<cudaEvent_t, 5>> prof_pending;
  std::vector<cudaEvent_t> ev_free;

  ~hc_pool() {
    for (auto& p : ring) {
      if (p.ev) {
        if (p.pending) cudaEventSynchronize(p.ev);
        cudaEventDestroy(p.ev);
      }
      if (p.ptr) cudaFreeHost(p.ptr);
    }
    for (auto& a : prof_pending)
      for (auto e : a) cudaEventDestroy(e);
    for (auto e : ev_free) cudaEventDestroy(e);
  }

  // pinned staging buffer of >= bytes; waits only if its previous copy is still queued
  Pinned* pinned(size_t bytes) {
    Pinned* p = nullptr;
    for (int i = 0; i < kRing && p == nullptr; ++i) {   // skip slots owned by captured graphs
      Pinned* c = &ring[ring_next];
      ring_next = (ring_next + 1) % kRing;
      if (!c->captured) p = c;
    }
    if (p == nullptr) return nullptr;
    if (p->pending) {
      cudaEventSynchronize(p->ev);
      p->pending = false;
    }
    if (p->cap < bytes) {
      // (Re)size the whole ring at once: cudaMallocHost / cudaFreeHost synchronise the
      // device, so growing one slot per call would stall the GPU on each of the next
      // kRing calls (measured: 30-80 ms gaps in the first timed steps).
      size_t cap = std::max<size_t>(bytes, 1 << 16);
      cap = align_up(cap + cap / 2, 4096);
      for (auto& r : ring) {
        if (r.captured) continue;
        if (r.pending) {
          cudaEventSynchronize(r.ev);
          r.pending = false;
        }
        if (r.cap >= cap) continue;
        if (r.ptr) cudaFreeHost(r.ptr);
        r.ptr = nullptr;
        r.cap = 0;
        if (cudaMallocHost(&r.ptr, cap) != cudaSuccess) {
          r.ptr = nullptr;
          return nullptr;
        }
        r.cap = cap;
      }
    }
    if (!p->ev) {   // events belong to the pool's device (callers hold a DeviceGuard; be safe anyway)
      DeviceGuard g(cfg.device);
      if (cudaEventCreateWithFlags(&p->ev, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    return p;
  }

  // After the H2D copy from `p` is enqueued on `s`: remember when the buffer is free again.
  // Under stream capture the copy becomes a graph node that re-reads the buffer at every
  // replay, so the slot is retired from the ring instead (kept until the pool is destroyed).
  void staged(Pinned* p, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
      p->captured = true;
      p->pending = false;
      return;
    }
    // a failed record leaves the slot free (never "pending" on an event that was not recorded);
    // the caller's next launch check reports the sticky error
    p->pending = cudaEventRecord(p->ev, s) == cudaSuccess;
  }

  cudaEvent_t get_event() {
    if (!ev_free.empty()) {
      cudaEvent_t e = ev_free.back();
      ev_free.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }

  int32_t split_tokens_auto(const std::vector<const Req*>& rs) const {
    const int B = cfg.block_size, H = cfg.n_heads;
    int spb = std::max(1, 512 / B);   // 512-token splits (256: +0.7% at cfg5 h=0; 1024 / 2048 within noise at
                                      // 1/64, 1/32 and cfg4: profiles/r02_split_size_ab.txt)
    const int64_t target = 4LL * num_sms * 6;  // ~4 tasks per resident warp
    while (spb > 1) {
      int64_t ns = 0;
      for (auto* r : rs) ns += cdiv(cdiv(r->n, B), spb);
      if (ns * H >= target) break;
      spb /= 2;
    }
    return spb;
  }

  Plan plan(const std::vector<const Req*>& rs) const {
    Plan P;
    const int B = cfg.block_size, H = cfg.n_heads, dh = cfg.head_dim;
    P.n_req = (int32_t)rs.size();
    P.split_blocks = cfg.split_tokens > 0 ? std::max(1, (int)cdiv(cfg.split_tokens, B)) : split_tokens_auto(rs);
    P.split_blocks_kv = std::max(1, P.split_blocks * B / kv.Bkv);   // same tokens per split in KV blocks
    P.absorb = (cfg.flags & HC_FLAG_ABSORB_HIDDEN) != 0;
    // GQA with HC_GQA_SCRATCH: rebuilt K/V go to scratch and the tensor-core KV loop attends a
    // whole query group per task instead of the attend epilogue serving G heads per K/V head
    // (auto for G >= 8: the attend epilogue's cost grows with G while the scratch round trip
    // does not — same-box A/B: Yi-6B (G 8) 1.27 vs 1.40-1.44 ms, LLaMA-3-8B (G 4) 2.54 vs 2.51 ms)
    // With the attend epilogue on mma.sync (HC_EPI_MMA, dh 128) the epilogue's cost no longer
    // grows with G and the attend path wins for G = 8 too (Yi-6B 1.24-1.25 vs 1.29-1.32 ms).
    const bool epi_mma_ok = tune.epi_mma != 0 && dh == 128;
    P.gqa_scratch = !P.absorb && tc_ok && attn_tc_ok && kv.Hk < H && tune.attn_tc != 0 &&
                    (tune.gqa_scratch == 1 || (tune.gqa_scratch < 0 && H / kv.Hk >= 8 && !epi_mma_ok));
    P.attend = !P.absorb && tc_ok && cfg.dtype == HC_BF16 && tune.epi_attend != 0 && recon_pair_mode(B, tune) &&
               !P.gqa_scratch;
    P.seg = std::min(B, 32);
    for (auto* r : rs) {
      const int64_t nb = cdiv(r->n, r->mode == HC_MODE_KV ? kv.Bkv : B);
      const int32_t ns = (int32_t)cdiv(nb, r->mode == HC_MODE_KV ? P.split_blocks_kv : P.split_blocks);
      if (r->mode == HC_MODE_KV) {
        P.n_splits += ns;
        P.n_tab += 2 * nb;
        P.n_kv_splits += ns;
        P.kv_tokens += r->n;
      } else {
        P.n_hb += (int32_t)nb;
        if (P.absorb) {
          ++P.n_h;
          P.n_atiles += (int32_t)cdiv(r->n, 128);
        } else if (P.attend) {
          P.n_splits += (int32_t)cdiv(r->n, P.seg);   // one partial per segment, in the GEMM epilogue
        } else {
          P.n_splits += ns;
          P.n_hid_splits += ns;
        }
      }
    }
    P.Hp = (int32_t)align_up((size_t)H, 16);
    // Tensor-core KV loop: for GQA groups by default (one task reads a K/V head once for its G
    // query heads); for multi-head its mma.sync compete with the fused GEMM's tcgen05 work for the
    // tensor pipe (same-box A/B: 1/64 -4%, 1/32 -2%), so the FHFMA SIMT loop stays the default.
    P.tc = attn_tc_ok && !(cfg.flags & HC_FLAG_GENERIC_ATTN) &&
           (P.attend || P.absorb || P.n_hb == 0 || P.gqa_scratch) &&
           (tune.attn_tc == 2 || (tune.attn_tc == 1 && kv.Hk < H));
    P.fused = !P.absorb && tc_ok && P.n_hb > 0 && tune.fused != 0 && !(cfg.flags & HC_FLAG_GENERIC_ATTN) &&
              fused_supported(cfg.d_model, kv.dk, cfg.head_dim, B);
    if (P.fused) {
      P.gemm_m_tiles = (int32_t)cdiv((int64_t)P.n_hb * B, fused_tile_m());
      P.gemm_n_tiles = 2 * kv.dk / fused_tile_n();
    }
    size_t o = kHeaderBytes;  // header: attention task counter, then GEMM pair-progress words
    P.off_reqs = o = align_up(o, 64);
    o += sizeof(ReqDesc) * P.n_req;
    P.off_splits = o = align_up(o, 64);
    o += sizeof(SplitDesc) * P.n_splits;
    P.off_tabs = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_tab;
    P.off_gather = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_hb;
    P.off_hpos = o = align_up(o, 64);
    o += (cfg.rope_theta > 0.f || P.attend) ? sizeof(int32_t) * P.n_hb : 0;
    P.off_hreqblk = o = align_up(o, 64);
    o += P.attend ? sizeof(int32_t) * P.n_hb : 0;
    P.off_kvsplit = o = align_up(o, 64);
    o += P.fused ? sizeof(int32_t) * P.n_kv_splits : 0;
    P.off_hidsplit = o = align_up(o, 64);
    o += P.fused ? sizeof(int32_t) * P.n_hid_splits : 0;
    P.off_tiledone = o = align_up(o, 64);
    o += P.fused ? sizeof(int32_t) * (size_t)P.gemm_m_tiles * P.gemm_n_tiles : 0;
    P.off_hreq = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_h;
    P.off_hrow0 = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_h;
    P.off_hntok = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_h;
    P.off_htile0 = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_h;
    P.off_treq = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_atiles;
    P.off_tt0 = o = align_up(o, 64);
    o += sizeof(int32_t) * P.n_atiles;
    P.desc_bytes = align_up(o, kAlign);
    const size_t n_tasks = (size_t)P.n_splits * H;
    P.off_ml = P.desc_bytes;
    P.off_acc = align_up(P.off_ml + n_tasks * 2 * sizeof(float), kAlign);
    const size_t scr = (P.absorb || P.attend) ? 0 : (size_t)P.n_hb * kv.Hk * B * dh * elem;
    P.off_sk = align_up(P.off_acc + n_tasks * dh * sizeof(float), 1024);
    P.off_sv = align_up(P.off_sk + scr, 1024);
    size_t e = align_up(P.off_sv + scr, kAlign);
    if (P.absorb) {
      const size_t rows = (size_t)P.n_hb * B, d = cfg.d_model;
      P.off_qt = e;
      e = align_up(e + (size_t)P.n_h * P.Hp * d * 2, kAlign);
      P.off_tml = e;
      e = align_up(e + (size_t)P.n_atiles * P.Hp * 2 * sizeof(float), kAlign);
      P.off_pm = e;
      e = align_up(e + rows * P.Hp * 2, kAlign);
      P.off_abml = e;
      e = align_up(e + (size_t)P.n_h * H * 3 * sizeof(float), kAlign);
      P.off_z = e;
      e = align_up(e + (size_t)P.n_h * H * d * 2, kAlign);
    }
    P.total = e;
    return P;
  }
};

// ======================================================================= C ABI
extern "C" {

const char* hc_last_error(void) { return g_err.c_str(); }
const char* hc_version(void) { return "hc 0.1 (sm_100a)"; }

size_t hc_pool_storage_bytes(const hc_pool_config* cfg) {
  Layout L;
  if (!layout_for(cfg, &L)) {
    g_err = "invalid pool config";
    return 0;
  }
  return L.total;
}

int64_t hc_units_needed(const hc_pool_config* cfg, int32_t mode, int64_t n_tokens) {
  Layout L;
  if (!layout_for(cfg, &L) || n_tokens < 0 || (mode != HC_MODE_KV && mode != HC_MODE_HIDDEN)) {
    g_err = "invalid config, mode or n_tokens";
    return -1;
  }
  if (mode == HC_MODE_HIDDEN) return cdiv(n_tokens, cfg->block_size);
  KvGeom kg;
  kv_geom(cfg, &kg);   // valid: layout_for checked it
  return cdiv(n_tokens, kg.Bkv) * (kg.packed ? 1 : 2);
}

hc_status hc_pool_create(const hc_pool_config* cfg, hc_pool** out) {
  if (!out) return fail(HC_E_INVALID, "out is null");
  *out = nullptr;
  Layout L;
  if (!layout_for(cfg, &L))
    return fail(HC_E_INVALID, "invalid pool config (d = H*dh, positive sizes, dtype; GQA: H % n_kv_heads == 0 and "
                              "d % (2 n_kv_heads dh) == 0)");
  const size_t e = cfg->dtype == HC_BF16 ? 2 : 4;
  if ((cfg->head_dim * e) % 16 != 0)
    return fail(HC_E_UNSUPPORTED, "head_dim * element size must be a multiple of 16 bytes");
  if (cfg->head_dim > 256) return fail(HC_E_UNSUPPORTED, "head_dim > 256");
  if (cfg->num_blocks > INT32_MAX || (int64_t)cfg->num_blocks * cfg->block_size > INT32_MAX)
    return fail(HC_E_UNSUPPORTED, "num_blocks * block_size must fit in int32");
  const bool accounting = (cfg->flags & HC_FLAG_ACCOUNTING_ONLY) != 0;
  KvGeom kg;
  kv_geom(cfg, &kg);   // valid: layout_for checked it (H % Hk == 0, d % (2 Hk dh) == 0 under GQA)
  if ((cfg->flags & HC_FLAG_ABSORB_HIDDEN) && kg.Hk != cfg->n_heads)
    return fail(HC_E_UNSUPPORTED, "HC_FLAG_ABSORB_HIDDEN needs multi-head attention (n_kv_heads = n_heads)");
  if (cfg->rope_theta < 0.f) return fail(HC_E_INVALID, "rope_theta < 0");
  if (cfg->ln_gamma && !(cfg->ln_eps >= 0.f)) return fail(HC_E_INVALID, "ln_eps < 0");
  if (cfg->rope_theta > 0.f &&
      (cfg->dtype != HC_BF16 || (cfg->flags & HC_FLAG_FORCE_SIMT) || cfg->head_dim % 64 != 0 ||
       !recon_tc_supported(cfg->d_model, kg.dk, cfg->head_dim, cfg->block_size) ||
       !dense_tc_supported(cfg->d_model) || !(cfg->block_size <= 128 || cfg->block_size % 256 == 0)))
    return fail(HC_E_UNSUPPORTED, "RoPE needs the bf16 tcgen05 path and head_dim % 64 == 0");
  if ((cfg->flags & HC_FLAG_ABSORB_HIDDEN) &&
      (cfg->rope_theta > 0.f || (cfg->flags & HC_FLAG_FORCE_SIMT) ||
       !absorb_supported(cfg->dtype, cfg->d_model, cfg->head_dim, cfg->n_heads, cfg->block_size) ||
       !recon_tc_supported(cfg->d_model, kg.dk, cfg->head_dim, cfg->block_size)))
    return fail(HC_E_UNSUPPORTED,
                "HC_FLAG_ABSORB_HIDDEN needs bf16, no RoPE, d % 128 == 0, head_dim % 16 == 0, head_dim <= 128, "
                "n_heads <= 128, block_size % 8 == 0 dividing or divisible by 128");
  if (!accounting) {
    if (!cfg->storage || cfg->storage_bytes < L.total)
      return fail(HC_E_INVALID, "storage null or smaller than hc_pool_storage_bytes()");
    if (reinterpret_cast<uintptr_t>(cfg->storage) % 1024 != 0)
      return fail(HC_E_INVALID, "storage must be 1024-byte aligned");
    if (!cfg->w_kv) return fail(HC_E_INVALID, "w_kv is null");
  }
  hc_pool* p = new hc_pool();
  p->cfg = *cfg;
  p->L = L;
  p->tune = tuning_from_env();
  p->kv = kg;
  p->elem = e;
  p->accounting = accounting;
  p->has_bias = cfg->b_kv != nullptr;
  for (int32_t i = 0; i < (int32_t)cfg->num_blocks; ++i) p->free_ids.push(i);
  if (!accounting) {
    DeviceGuard g(cfg->device);
    p->storage = static_cast<char*>(cfg->storage);
    cudaDeviceProp prop;
    cudaError_t err = cudaGetDeviceProperties(&prop, cfg->device);
    if (err != cudaSuccess) {
      delete p;
      return cuda_fail(err, "cudaGetDeviceProperties");
    }
    p->num_sms = prop.multiProcessorCount;
    err = cudaMemset(p->storage + L.blocks_off, 0, L.blocks_bytes);
    if (err == cudaSuccess)
      err = launch_relayout_w(cfg->w_kv, p->storage + L.w_off, cfg->b_kv, reinterpret_cast<float*>(p->storage + L.b_off),
                              cfg->d_model, kg.dk, cfg->head_dim, cfg->dtype, 0);
    const size_t dd = (size_t)cfg->d_model * cfg->d_model * e;
    const size_t dbytes = (size_t)cfg->d_model * sizeof(float);
    if (err == cudaSuccess && L.has_q) err = cudaMemcpy(p->storage + L.wq_off, cfg->w_q, dd, cudaMemcpyDeviceToDevice);
    if (err == cudaSuccess)
      err = cfg->b_q ? cudaMemcpy(p->storage + L.bq_off, cfg->b_q, dbytes, cudaMemcpyDeviceToDevice)
                     : cudaMemset(p->storage + L.bq_off, 0, dbytes);
    if (err == cudaSuccess && L.has_o) err = cudaMemcpy(p->storage + L.wo_off, cfg->w_o, dd, cudaMemcpyDeviceToDevice);
    if (err == cudaSuccess && L.has_o)
      err = cfg->b_o ? cudaMemcpy(p->storage + L.bo_off, cfg->b_o, dbytes, cudaMemcpyDeviceToDevice)
                     : cudaMemset(p->storage + L.bo_off, 0, dbytes);
    if (err == cudaSuccess && L.has_ln) {
      err = cudaMemcpy(p->storage + L.ln_off, cfg->ln_gamma, dbytes, cudaMemcpyDeviceToDevice);
      if (err == cudaSuccess)
        err = cfg->ln_beta ? cudaMemcpy(p->storage + L.ln_off + dbytes, cfg->ln_beta, dbytes, cudaMemcpyDeviceToDevice)
                           : cudaMemset(p->storage + L.ln_off + dbytes, 0, dbytes);
    }
    if (err == cudaSuccess && cfg->rope_theta > 0.f) {
      std::vector<double> inv(cfg->head_dim / 2);
      for (int c = 0; c < cfg->head_dim / 2; ++c)
        inv[c] = std::pow((double)cfg->rope_theta, -2.0 * c / cfg->head_dim);
      err = cudaMemcpy(p->storage + L.rope_off, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
    if (err == cudaSuccess) err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      delete p;
      return cuda_fail(err, "pool init");
    }
    p->dense_tc_ok = cfg->dtype == HC_BF16 && !(cfg->flags & HC_FLAG_FORCE_SIMT) && dense_tc_supported(cfg->d_model);
    if (p->dense_tc_ok) {
      bool ok = true;
      if (L.has_q)
        ok &= make_tmap_2d(&p->tmap_wqkv, p->storage + L.wq_off, (uint64_t)cfg->d_model,
                           (uint64_t)cfg->d_model + 2 * (uint64_t)kg.dk,
                           64, 128);
      if (L.has_o)
        ok &= make_tmap_2d(&p->tmap_wo, p->storage + L.wo_off, (uint64_t)cfg->d_model, (uint64_t)cfg->d_model, 64, 128);
      if (!ok) {
        delete p;
        return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed (projection weights)");
      }
    }
    if (cfg->dtype == HC_BF16 && !(cfg->flags & HC_FLAG_FORCE_SIMT) &&
        recon_tc_supported(cfg->d_model, kg.dk, cfg->head_dim, cfg->block_size)) {
      // -DHC_DIAG builds, HC_DIAG_BOX=1 (timing diagnostic, wrong results): 128-row A boxes as if dense
      const uint32_t rpb = p->tune.diag_box ? 128u : (uint32_t)std::min(cfg->block_size, 128);
      const bool ok1 = make_tmap_2d(&p->tmap_x, p->storage + L.blocks_off, (uint64_t)cfg->d_model,
                                    (uint64_t)cfg->num_blocks * cfg->block_size, 64, rpb);
      const bool ok2 = make_tmap_2d(&p->tmap_w, p->storage + L.w_off, (uint64_t)cfg->d_model,
                                    2 * (uint64_t)kg.dk, 64, 256);
      const bool ok3 = make_tmap_2d(&p->tmap_w_half, p->storage + L.w_off, (uint64_t)cfg->d_model,
                                    2 * (uint64_t)kg.dk, 64, 128);
      const bool ok4 = !(cfg->flags & HC_FLAG_ABSORB_HIDDEN) ||
                       make_tmap_2d(&p->tmap_x64, p->storage + L.blocks_off, (uint64_t)cfg->d_model,
                                    (uint64_t)cfg->num_blocks * cfg->block_size, 64, (uint32_t)std::min(cfg->block_size, 64));
      if (!ok1 || !ok2 || !ok3 || !ok4) {
        delete p;
        return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed");
      }
      p->tc_ok = true;
      // runs of consecutive hidden blocks as one 128-row box (B < 128)
      p->x128_ok = cfg->block_size < 128 && p->tune.block_runs != 0 &&
                   make_tmap_2d(&p->tmap_x128, p->storage + L.blocks_off, (uint64_t)cfg->d_model,
                                (uint64_t)cfg->num_blocks * cfg->block_size, 64, 128);
    }
    if (attn_tc_supported(cfg->dtype, cfg->head_dim, cfg->n_heads / kg.Hk, kg.Bkv) &&
        !(cfg->flags & HC_FLAG_FORCE_SIMT)) {
      // the pool viewed as rows of dh elements: a K (V) chunk of 16 tokens of one K/V head is
      // 16 consecutive rows (KV layout [Hk][Bkv][dh] per K / V region)
      p->attn_tc_ok = make_tmap_2d(&p->tmap_kv, p->storage + L.blocks_off, (uint64_t)cfg->head_dim,
                                   (uint64_t)cfg->num_blocks * cfg->block_size * cfg->d_model / cfg->head_dim, 64, 16);
    }
  }
  *out = p;
  return HC_OK;
}

void hc_pool_destroy(hc_pool* pool) {
  if (!pool) return;
  DeviceGuard g(pool->cfg.device);
  delete pool;
}

int64_t hc_pool_num_free(const hc_pool* pool) { return pool ? (int64_t)pool->free_ids.size() : -1; }

hc_status hc_request_info(const hc_pool* pool, int64_t id, int32_t* mode, int64_t* n_tokens, int64_t* n_units) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  auto it = pool->reqs.find(id);
  if (it == pool->reqs.end()) return fail(HC_E_UNKNOWN_REQ, "unknown request id");
  if (mode) *mode = it->second.mode;
  if (n_tokens) *n_tokens = it->second.n;
  if (n_units) *n_units = (int64_t)(it->second.a.size() + it->second.b.size());
  return HC_OK;
}

hc_status hc_request_blocks(const hc_pool* pool, int64_t id, int32_t kind, int32_t* out, int64_t cap,
                            int64_t* count) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  auto it = pool->reqs.find(id);
  if (it == pool->reqs.end()) return fail(HC_E_UNKNOWN_REQ, "unknown request id");
  const std::vector<int32_t>& v = kind == 0 ? it->second.a : it->second.b;
  if (count) *count = (int64_t)v.size();
  if (out)
    for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)v.size()); ++i) out[i] = v[i];
  return HC_OK;
}

hc_status hc_free(hc_pool* pool, int64_t id, int64_t* released) {
  if (released) *released = 0;
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  auto it = pool->reqs.find(id);
  if (it == pool->reqs.end()) return HC_OK;  // idempotent
  for (int32_t b : it->second.a) pool->free_ids.push(b);
  for (int32_t b : it->second.b) pool->free_ids.push(b);
  if (released) *released = (int64_t)(it->second.a.size() + it->second.b.size());
  pool->reqs.erase(it);
  return HC_OK;
}

// Upload the append descriptor(s) (chunked to the staging area) and launch the scatter.
static hc_status scatter_rows(hc_pool* pool, const std::vector<AppendReq>& ar, const std::vector<int32_t>& tabs,
                              const void* k, const void* v, const void* x, void* stream) {
  // ---- upload descriptor(s) and scatter (chunked to the staging area) ----
  DeviceGuard g(pool->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* staging = pool->storage + pool->L.stage_off;
  size_t i0 = 0;
  while (i0 < ar.size()) {
    // largest prefix [i0, i1) whose descriptor fits the staging area
    size_t i1 = i0, tab_lo = ar[i0].tab_off;
    size_t bytes_req = 0, bytes_tab = 0;
    int32_t rows = 0;
    while (i1 < ar.size()) {
      const size_t tab_hi = (i1 + 1 < ar.size()) ? ar[i1 + 1].tab_off : tabs.size();
      const size_t nb_req = align_up((i1 - i0 + 1) * sizeof(AppendReq), 64);
      const size_t nb_tab = (tab_hi - tab_lo) * sizeof(int32_t);
      if (i1 > i0 && nb_req + nb_tab > kStagingBytes / 2) break;
      bytes_req = nb_req;
      bytes_tab = nb_tab;
      rows = std::max(rows, ar[i1].n_tok);
      ++i1;
    }
    if (bytes_req + bytes_tab > kStagingBytes / 2) return fail(HC_E_UNSUPPORTED, "append descriptor too large");
    Pinned* pin = pool->pinned(bytes_req + bytes_tab);
    if (!pin) return fail(HC_E_CUDA, "pinned staging unavailable (cudaMallocHost failed, or all slots held by captured graphs)");
    AppendReq* hr = static_cast<AppendReq*>(pin->ptr);
    for (size_t i = i0; i < i1; ++i) {
      hr[i - i0] = ar[i];
      hr[i - i0].tab_off = (int32_t)(ar[i].tab_off - tab_lo);
    }
    std::memcpy(static_cast<char*>(pin->ptr) + bytes_req, tabs.data() + tab_lo, bytes_tab);
    cudaError_t err = cudaMemcpyAsync(staging, pin->ptr, bytes_req + bytes_tab, cudaMemcpyHostToDevice, s);
    if (err != cudaSuccess) return cuda_fail(err, "append descriptor upload");
    pool->staged(pin, s);
    AppendParams ap;
    ap.reqs = reinterpret_cast<const AppendReq*>(staging);
    ap.tabs = reinterpret_cast<const int32_t*>(staging + bytes_req);
    ap.k = k;
    ap.v = v;
    ap.x = x;
    ap.pool = pool->storage + pool->L.blocks_off;
    ap.n_req = (int32_t)(i1 - i0);
    ap.d = pool->cfg.d_model;
    ap.H = pool->cfg.n_heads;
    ap.dh = pool->cfg.head_dim;
    ap.B = pool->cfg.block_size;
    ap.dk = pool->kv.dk;
    ap.Bkv = pool->kv.Bkv;
    ap.v_off = pool->kv.v_off;
    err = launch_append(ap, pool->cfg.dtype, rows, s);
    if (err != cudaSuccess) return cuda_fail(err, "append kernel");
    ++pool->last_launches;
    i0 = i1;
  }
  return HC_OK;
}

// What validate_and_allocate changed, so a later failure in the same call can restore the
// pool exactly ("validation errors leave the pool unchanged", hc.h; a retry must not append
// the tokens twice).
struct AllocUndo {
  struct Entry {
    int64_t id;
    bool created;
    int64_t n;
    size_t na, nb;
  };
  std::vector<Entry> e;
  void rollback(hc_pool* pool) {
    for (auto it = e.rbegin(); it != e.rend(); ++it) {
      auto f = pool->reqs.find(it->id);
      if (f == pool->reqs.end()) continue;
      Req& r = f->second;
      for (size_t j = it->na; j < r.a.size(); ++j) pool->free_ids.push(r.a[j]);
      for (size_t j = it->nb; j < r.b.size(); ++j) pool->free_ids.push(r.b[j]);
      if (it->created) {
        pool->reqs.erase(f);
      } else {
        r.a.resize(it->na);
        r.b.resize(it->nb);
        r.n = it->n;
      }
    }
    e.clear();
  }
};

// Validation + all-or-nothing allocation shared by hc_append and hc_project_append.
// On success the requests' tables/lengths are extended and `ar`/`tabs` describe the new rows
// (row_off = running row index per mode, in call order; one entry per request with t > 0).
static hc_status validate_and_allocate(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                                       const int32_t* n_tokens, const void* k, const void* v, const void* x,
                                       std::vector<AppendReq>* ar, std::vector<int32_t>* tabs, int32_t* max_rows,
                                       AllocUndo* undo) {
  if (!req_ids || !modes || !n_tokens) return fail(HC_E_INVALID, "null id/mode/n_tokens array");
  const int B = pool->cfg.block_size;
  std::unordered_set<int64_t> seen;
  int64_t need = 0, kv_rows = 0, x_rows = 0;
  for (int32_t i = 0; i < n_req; ++i) {
    if (!seen.insert(req_ids[i]).second) return fail(HC_E_INVALID, "duplicate request id in append");
    if (modes[i] != HC_MODE_KV && modes[i] != HC_MODE_HIDDEN) return fail(HC_E_INVALID, "bad mode");
    if (n_tokens[i] < 0) return fail(HC_E_INVALID, "n_tokens < 0");
    int64_t n0 = 0;
    auto it = pool->reqs.find(req_ids[i]);
    if (it != pool->reqs.end()) {
      if (it->second.mode != modes[i])
        return fail(HC_E_MODE_MISMATCH, "request exists with the other cache mode (switch = free + re-append)");
      n0 = it->second.n;
    }
    if (n0 + n_tokens[i] > INT32_MAX) return fail(HC_E_INVALID, "context too long");
    const int Bm = modes[i] == HC_MODE_KV ? pool->kv.Bkv : B;
    const int64_t per = cdiv(n0 + n_tokens[i], Bm) - cdiv(n0, Bm);
    need += (modes[i] == HC_MODE_KV && !pool->kv.packed) ? 2 * per : per;
    (modes[i] == HC_MODE_KV ? kv_rows : x_rows) += n_tokens[i];
  }
  if (need > (int64_t)pool->free_ids.size()) return fail(HC_E_OOM, "not enough free blocks (all-or-nothing)");
  if (!pool->accounting && ((kv_rows > 0 && (!k || !v)) || (x_rows > 0 && !x)))
    return fail(HC_E_INVALID, "k/v or x is null while rows of that mode are appended");

  // ---- allocate (lowest free id first; K then V per logical block; call order) ----
  ar->reserve(n_req);
  int32_t kv_off = 0, x_off = 0;
  *max_rows = 0;
  for (int32_t i = 0; i < n_req; ++i) {
    const bool created = pool->reqs.find(req_ids[i]) == pool->reqs.end();
    Req& r = pool->reqs[req_ids[i]];
    undo->e.push_back({req_ids[i], created, r.n, r.a.size(), r.b.size()});
    if (r.n == 0 && r.a.empty()) r.mode = modes[i];
    const int64_t t = n_tokens[i];
    const int Bm = r.mode == HC_MODE_KV ? pool->kv.Bkv : B;   // tokens per logical block
    const bool two = r.mode == HC_MODE_KV && !pool->kv.packed;  // separate K and V units
    const int64_t new_lb = cdiv(r.n + t, Bm) - cdiv(r.n, Bm);
    for (int64_t j = 0; j < new_lb; ++j) {
      r.a.push_back(pool->free_ids.top());
      pool->free_ids.pop();
      if (two) {
        r.b.push_back(pool->free_ids.top());
        pool->free_ids.pop();
      }
    }
    if (t > 0) {
      AppendReq q{};
      q.mode = r.mode;
      q.start = (int32_t)r.n;
      q.n_tok = (int32_t)t;
      q.row_off = r.mode == HC_MODE_KV ? kv_off : x_off;
      q.tab_off = (int32_t)tabs->size();
      const int64_t lb0 = r.n / Bm, lb1 = (r.n + t - 1) / Bm;
      for (int64_t lb = lb0; lb <= lb1; ++lb) {
        tabs->push_back(r.a[lb]);
        if (r.mode == HC_MODE_KV) tabs->push_back(two ? r.b[lb] : r.a[lb]);   // (K unit, V unit)
      }
      ar->push_back(q);
      *max_rows = std::max<int32_t>(*max_rows, (int32_t)t);
      (r.mode == HC_MODE_KV ? kv_off : x_off) += (int32_t)t;
    }
    r.n += t;
  }
  return HC_OK;
}

hc_status hc_append(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                    const int32_t* n_tokens, const void* k, const void* v, const void* x, void* stream) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  pool->last_launches = 0;
  if (n_req < 0) return fail(HC_E_INVALID, "n_req < 0");
  if (n_req == 0) return HC_OK;
  std::vector<AppendReq> ar;
  std::vector<int32_t> tabs;
  int32_t max_rows = 0;
  AllocUndo undo;
  hc_status st = validate_and_allocate(pool, n_req, req_ids, modes, n_tokens, k, v, x, &ar, &tabs, &max_rows, &undo);
  if (st != HC_OK) return st;
  if (pool->accounting || ar.empty()) return HC_OK;
  st = scatter_rows(pool, ar, tabs, k, v, x, stream);
  if (st != HC_OK) undo.rollback(pool);
  return st;
}

static hc_status collect(const hc_pool* pool, int32_t n_req, const int64_t* ids, std::vector<const Req*>* rs) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  if (n_req < 0) return fail(HC_E_INVALID, "n_req < 0");
  if (n_req > 0 && !ids) return fail(HC_E_INVALID, "req_ids is null");
  std::unordered_set<int64_t> seen;
  rs->reserve(n_req);
  for (int32_t i = 0; i < n_req; ++i) {
    if (!seen.insert(ids[i]).second) return fail(HC_E_INVALID, "duplicate request id in decode batch");
    auto it = pool->reqs.find(ids[i]);
    if (it == pool->reqs.end()) return fail(HC_E_UNKNOWN_REQ, "unknown request id " + std::to_string(ids[i]));
    if (it->second.n < 1) return fail(HC_E_INVALID, "request has no cached token (append the current one first, P:135)");
    rs->push_back(&it->second);
  }
  return HC_OK;
}

size_t hc_workspace_size(const hc_pool* pool, int32_t n_req, const int64_t* req_ids) {
  std::vector<const Req*> rs;
  if (collect(pool, n_req, req_ids, &rs) != HC_OK) return 0;
  if (n_req == 0) return kAlign;
  return pool->plan(rs).total;
}

hc_status hc_decode_attention(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const void* q, float scale,
                              void* out, float* lse, void* workspace, size_t ws_bytes, void* stream) {
  if (pool) pool->last_launches = 0;
  std::vector<const Req*> rs;
  hc_status st = collect(pool, n_req, req_ids, &rs);
  if (st != HC_OK) return st;
  if (n_req == 0) return HC_OK;
  if (pool->accounting) return fail(HC_E_UNSUPPORTED, "accounting-only pool has no device storage");
  if (!q || !out || !workspace) return fail(HC_E_INVALID, "q/out/workspace is null");
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign != 0) return fail(HC_E_INVALID, "workspace must be 256-B aligned");
  const Plan P = pool->plan(rs);
  if (ws_bytes < P.total) return fail(HC_E_WORKSPACE, "workspace smaller than hc_workspace_size()");
  const int B = pool->cfg.block_size, H = pool->cfg.n_heads;
  DeviceGuard g(pool->cfg.device);   // before the staging slot: its event belongs to the pool's device

  // ---- descriptor (a3): requests, split-K work list, KV block tables, hidden gather list
  Pinned* pin = pool->pinned(P.desc_bytes);
  if (!pin) return fail(HC_E_CUDA, "pinned staging unavailable (cudaMallocHost failed, or all slots held by captured graphs)");
  char* h = static_cast<char*>(pin->ptr);
  std::memset(h, 0, kHeaderBytes);  // attention task counter and GEMM progress words = 0
  ReqDesc* rd = reinterpret_cast<ReqDesc*>(h + P.off_reqs);
  SplitDesc* sd = reinterpret_cast<SplitDesc*>(h + P.off_splits);
  int32_t* tab = reinterpret_cast<int32_t*>(h + P.off_tabs);
  int32_t* gat = reinterpret_cast<int32_t*>(h + P.off_gather);
  int32_t* kvs = reinterpret_cast<int32_t*>(h + P.off_kvsplit);
  const bool rope = pool->cfg.rope_theta > 0.f;
  int32_t* hpos = reinterpret_cast<int32_t*>(h + P.off_hpos);
  int32_t* hds = reinterpret_cast<int32_t*>(h + P.off_hidsplit);
  int32_t* ahreq = reinterpret_cast<int32_t*>(h + P.off_hreq);
  int32_t* ahrow0 = reinterpret_cast<int32_t*>(h + P.off_hrow0);
  int32_t* ahntok = reinterpret_cast<int32_t*>(h + P.off_hntok);
  int32_t* ahtile0 = reinterpret_cast<int32_t*>(h + P.off_htile0);
  int32_t* atreq = reinterpret_cast<int32_t*>(h + P.off_treq);
  int32_t* att0 = reinterpret_cast<int32_t*>(h + P.off_tt0);
  int32_t* hreqblk = reinterpret_cast<int32_t*>(h + P.off_hreqblk);
  int32_t n_split = 0, n_tab = 0, n_hb = 0, n_kvs = 0, n_hds = 0, n_ah = 0, n_at = 0;
  // attend mode: KV splits first (the attention kernels' tasks are exactly those), then one
  // split per hidden segment (written by the GEMM epilogue, read only by the combine)
  int32_t next_hid = P.n_kv_splits;
  if (P.fused) std::memset(h + P.off_tiledone, 0, P.desc_bytes - P.off_tiledone);
  const int Bkv = pool->kv.Bkv;
  const bool packed = pool->kv.packed;
  for (int32_t i = 0; i < n_req; ++i) {
    const Req& r = *rs[i];
    const int32_t nb = (int32_t)cdiv(r.n, r.mode == HC_MODE_KV ? Bkv : B);
    ReqDesc d{};
    d.mode = r.mode;
    d.n = (int32_t)r.n;
    d.split_begin = (P.attend && r.mode == HC_MODE_HIDDEN) ? next_hid : n_split;
    if (r.mode == HC_MODE_KV) {
      d.tab_off = n_tab;
      for (int32_t lb = 0; lb < nb; ++lb) {
        tab[n_tab++] = r.a[lb];
        tab[n_tab++] = packed ? r.a[lb] : r.b[lb];
      }
    } else {
      d.scratch_blk0 = n_hb;
      if (P.absorb) {
        ahreq[n_ah] = i;
        ahrow0[n_ah] = n_hb * B;
        ahntok[n_ah] = (int32_t)r.n;
        ahtile0[n_ah] = n_at;
        for (int32_t t0 = 0; t0 < r.n; t0 += 128) {
          atreq[n_at] = n_ah;
          att0[n_at++] = t0;
        }
        ++n_ah;
      }
      for (int32_t lb = 0; lb < nb; ++lb) {
        if (rope || P.attend) hpos[n_hb] = lb * B;
        if (P.attend) hreqblk[n_hb] = i;
        gat[n_hb++] = r.a[lb];
      }
    }
    if (P.attend && r.mode == HC_MODE_HIDDEN) {
      for (int64_t t0 = 0; t0 < r.n; t0 += P.seg) {
        SplitDesc s{};
        s.req = i;
        s.lb0 = (int32_t)(t0 / B);
        s.ntok = (int32_t)std::min<int64_t>(P.seg, r.n - t0);
        sd[next_hid++] = s;
      }
      d.split_count = next_hid - d.split_begin;
      rd[i] = d;
      continue;
    }
    const bool absorbed = P.absorb && r.mode == HC_MODE_HIDDEN;
    const int Bm = r.mode == HC_MODE_KV ? Bkv : B;
    const int sb = r.mode == HC_MODE_KV ? P.split_blocks_kv : P.split_blocks;
    for (int32_t lb = 0; lb < nb && !absorbed; lb += sb) {
      SplitDesc s{};
      s.req = i;
      s.lb0 = lb;
      const int64_t t0 = (int64_t)lb * Bm;
      s.ntok = (int32_t)std::min<int64_t>((int64_t)sb * Bm, r.n - t0);
      if (P.fused) (r.mode == HC_MODE_KV ? kvs[n_kvs++] : hds[n_hds++]) = n_split;
      sd[n_split++] = s;
    }
    d.split_count = n_split - d.split_begin;
    rd[i] = d;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::array<cudaEvent_t, 5> ev{};
  if (pool->profiling) {
    for (auto& e : ev) e = pool->get_event();
    cudaEventRecord(ev[0], s);
  }
  char* ws = static_cast<char*>(workspace);
  cudaError_t err = cudaMemcpyAsync(ws, h, P.desc_bytes, cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) return cuda_fail(err, "descriptor upload");
  pool->staged(pin, s);
  if (pool->profiling) cudaEventRecord(ev[1], s);

  char* blocks = pool->storage + pool->L.blocks_off;
  int launches = 0;
  // ---- a4 + a5: K/V reconstruction of hidden-mode requests, split-K attention
  ReconParams rp{};
  rp.gather = reinterpret_cast<const int32_t*>(ws + P.off_gather);
  rp.n_hblocks = P.n_hb;
  rp.pool = blocks;
  rp.w_int = pool->storage + pool->L.w_off;
  rp.b_int = pool->has_bias ? reinterpret_cast<const float*>(pool->storage + pool->L.b_off) : nullptr;
  rp.scr_k = ws + P.off_sk;
  rp.scr_v = ws + P.off_sv;
  rp.d = pool->cfg.d_model;
  rp.H = H;
  rp.Hk = pool->kv.Hk;
  rp.dk = pool->kv.dk;
  rp.dh = pool->cfg.head_dim;
  rp.B = B;
  rp.sync_counter = reinterpret_cast<int32_t*>(ws + 128);
  rp.tile_counter = reinterpret_cast<int32_t*>(ws + 64);   // header word, zeroed per call
  rp.hblk_pos = (rope || P.attend) ? reinterpret_cast<const int32_t*>(ws + P.off_hpos) : nullptr;
  rp.rope_inv = rope ? reinterpret_cast<const double*>(pool->storage + pool->L.rope_off) : nullptr;
  rp.epi_attend = P.attend;
  rp.hblk_req = reinterpret_cast<const int32_t*>(ws + P.off_hreqblk);
  rp.reqs = reinterpret_cast<const ReqDesc*>(ws + P.off_reqs);
  rp.q = q;
  rp.part_ml = reinterpret_cast<float*>(ws + P.off_ml);
  rp.part_acc = reinterpret_cast<float*>(ws + P.off_acc);
  rp.n_splits_all = P.n_splits;
  rp.scale_log2 = scale * 1.4426950408889634f;
  rp.seg = P.seg;
  rp.kv_tokens = P.kv_tokens;
  AttnParams ap{};
  ap.reqs = reinterpret_cast<const ReqDesc*>(ws + P.off_reqs);
  ap.splits = reinterpret_cast<const SplitDesc*>(ws + P.off_splits);
  ap.tables = reinterpret_cast<const int32_t*>(ws + P.off_tabs);
  ap.pool = blocks;
  ap.scr_k = ws + P.off_sk;
  ap.scr_v = ws + P.off_sv;
  ap.q = q;
  ap.part_ml = reinterpret_cast<float*>(ws + P.off_ml);
  ap.part_acc = reinterpret_cast<float*>(ws + P.off_acc);
  ap.n_splits_all = P.n_splits;
  ap.task_counter = reinterpret_cast<int32_t*>(ws);
  ap.th = P.tc ? pool->kv.Hk : H;   // tensor-core loop: one task per (split, K/V head) serves its G query heads
  ap.tc = P.tc ? 1 : 0;
  ap.n_tasks = (P.attend ? P.n_kv_splits : P.n_splits) * ap.th;   // attend: hidden partials come from the GEMM
  ap.H = H;
  ap.dh = pool->cfg.head_dim;
  ap.B = B;
  ap.d = pool->cfg.d_model;
  ap.Hk = pool->kv.Hk;
  ap.G = H / pool->kv.Hk;
  ap.Bkv = Bkv;
  ap.v_off = pool->kv.v_off;
  ap.scale_log2 = scale * 1.4426950408889634f;
  ap.diag = pool->tune.diag_attn;
  pool->last_path = P.absorb && P.n_h > 0 ? 3 : (P.fused ? 1 : (P.n_hb > 0 ? 0 : 2));
  pool->last_cfg = 0;
  // tensor-core KV loop over the rebuilt-K/V scratch (GQA scratch mode): rows of dh elements
  CUtensorMap tsk, tsv;
  const void *psk = nullptr, *psv = nullptr;
  if (P.tc && P.n_hb > 0 && !P.attend && !P.absorb) {
    const uint64_t rows = (uint64_t)P.n_hb * pool->kv.Hk * B;
    if (!make_tmap_2d(&tsk, ws + P.off_sk, (uint64_t)pool->cfg.head_dim, rows, 64, 16) ||
        !make_tmap_2d(&tsv, ws + P.off_sv, (uint64_t)pool->cfg.head_dim, rows, 64, 16))
      return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed (K/V scratch)");
    psk = &tsk;
    psv = &tsv;
  }
  if (P.absorb) {
    // f4 (ii): hidden requests never rebuild K/V; KV requests take the split-K path
    if (P.n_h > 0) {
      AbsorbParams bp{};
      bp.gather = rp.gather;
      bp.hreq = reinterpret_cast<const int32_t*>(ws + P.off_hreq);
      bp.hrow0 = reinterpret_cast<const int32_t*>(ws + P.off_hrow0);
      bp.hntok = reinterpret_cast<const int32_t*>(ws + P.off_hntok);
      bp.tile_req = reinterpret_cast<const int32_t*>(ws + P.off_treq);
      bp.tile_t0 = reinterpret_cast<const int32_t*>(ws + P.off_tt0);
      bp.htile0 = reinterpret_cast<const int32_t*>(ws + P.off_htile0);
      bp.pool = blocks;
      bp.q = q;
      bp.w_int = rp.w_int;
      bp.b_int = rp.b_int;
      bp.qt = reinterpret_cast<__nv_bfloat16*>(ws + P.off_qt);
      bp.tml = reinterpret_cast<float*>(ws + P.off_tml);
      bp.pm = reinterpret_cast<__nv_bfloat16*>(ws + P.off_pm);
      bp.ml = reinterpret_cast<float*>(ws + P.off_abml);
      bp.z = reinterpret_cast<__nv_bfloat16*>(ws + P.off_z);
      bp.out = out;
      bp.lse = lse;
      bp.n_h = P.n_h;
      bp.n_tiles = P.n_atiles;
      bp.H = H;
      bp.Hp = P.Hp;
      bp.dh = pool->cfg.head_dim;
      bp.d = pool->cfg.d_model;
      bp.B = B;
      bp.scale = scale;
      bp.scale_log2 = ap.scale_log2;
      bp.n_hb = P.n_hb;
      bp.rpb = std::min(B, 128);
      bp.rpb64 = std::min(B, 64);
      CUtensorMap tm_qt, tm_p, tm_w, tm_z;
      const uint64_t dd = (uint64_t)bp.d;
      if (!make_tmap_2d(&tm_qt, ws + P.off_qt, dd, (uint64_t)P.n_h * P.Hp, 64, (uint32_t)P.Hp) ||
          !make_tmap_2d(&tm_p, ws + P.off_pm, (uint64_t)P.Hp, (uint64_t)P.n_hb * B, 64, 64) ||
          !make_tmap_2d(&tm_w, pool->storage + pool->L.w_off, dd, 2 * dd, 64, (uint32_t)bp.dh) ||
          !make_tmap_2d(&tm_z, ws + P.off_z, dd, (uint64_t)H * P.n_h, 64, 128))
        return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed (absorbed path)");
      err = launch_absorbed(bp, &pool->tmap_x, &pool->tmap_x64, &tm_qt, &tm_p, &tm_w, &tm_z, &tm_w, pool->tune, s);
      if (err != cudaSuccess) return cuda_fail(err, "absorbed hidden attention");
      launches += absorb_launches();
    }
    if (pool->profiling) cudaEventRecord(ev[2], s);
    if (P.n_splits > 0) {
      err = launch_attn(ap, pool->cfg.dtype, (pool->cfg.flags & HC_FLAG_GENERIC_ATTN) != 0, pool->num_sms, pool->tune, s,
                      &pool->tmap_kv);
      if (err != cudaSuccess) return cuda_fail(err, "attention kernel");
      ++launches;
    }
    if (pool->profiling) cudaEventRecord(ev[3], s);
  } else if (P.fused) {
    ap.kv_split_ids = reinterpret_cast<const int32_t*>(ws + P.off_kvsplit);
    ap.hid_split_ids = reinterpret_cast<const int32_t*>(ws + P.off_hidsplit);
    ap.n_kv_tasks = P.n_kv_splits * ap.th;
    ap.n_hid_splits = P.n_hid_splits;
    err = launch_fused(rp, ap, &pool->tmap_x, &pool->tmap_w_half, reinterpret_cast<int32_t*>(ws + P.off_tiledone),
                       pool->num_sms, pool->tune, s, &pool->tmap_kv, &pool->last_cfg, psk, psv,
                       pool->x128_ok ? &pool->tmap_x128 : nullptr);
    if (err != cudaSuccess) return cuda_fail(err, "fused step kernel");
    ++launches;
    if (pool->profiling) {
      cudaEventRecord(ev[2], s);   // fused time is reported as the reconstruction slot
      cudaEventRecord(ev[3], s);
    }
  } else {
    if (P.n_hb > 0) {
      err = pool->tc_ok ? launch_recon_tc(rp, &pool->tmap_x, &pool->tmap_w, &pool->tmap_w_half, pool->num_sms, pool->tune, s,
                                          pool->x128_ok ? &pool->tmap_x128 : nullptr)
                        : launch_recon_simt(rp, pool->cfg.dtype, s);
      if (err != cudaSuccess) return cuda_fail(err, "reconstruction kernel");
      ++launches;
    }
    if (pool->profiling) cudaEventRecord(ev[2], s);
    err = launch_attn(ap, pool->cfg.dtype, (pool->cfg.flags & HC_FLAG_GENERIC_ATTN) != 0, pool->num_sms, pool->tune, s,
                      &pool->tmap_kv, psk, psv);
    if (err != cudaSuccess) return cuda_fail(err, "attention kernel");
    ++launches;
    if (pool->profiling) cudaEventRecord(ev[3], s);
  }
  // ---- a6: combine splits
  CombineParams cp;
  cp.reqs = ap.reqs;
  cp.part_ml = ap.part_ml;
  cp.part_acc = ap.part_acc;
  cp.n_splits = P.n_splits;
  cp.out = out;
  cp.lse = lse;
  cp.n_req = n_req;
  cp.H = H;
  cp.dh = pool->cfg.head_dim;
  cp.d = pool->cfg.d_model;
  err = launch_combine(cp, pool->cfg.dtype, s);
  if (err != cudaSuccess) return cuda_fail(err, "combine kernel");
  ++launches;
  if (pool->profiling) {
    cudaEventRecord(ev[4], s);
    pool->prof_pending.push_back(ev);
  }
  pool->last_launches = launches;
  return HC_OK;
}

// ============================================================ attention-module steps (f1)
static bool make_tmap_rows(CUtensorMap* m, const void* base, int rows, int d) {
  return make_tmap_2d(m, const_cast<void*>(base), (uint64_t)d, (uint64_t)rows, 64, 128);
}

static hc_status project_after_alloc(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const void* x, void* q_out,
                                     const std::vector<AppendReq>& ar, const std::vector<int32_t>& tabs, void* stream);

hc_status hc_project_append(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                            const void* x, void* q_out, void* stream) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  pool->last_launches = 0;
  if (n_req < 0) return fail(HC_E_INVALID, "n_req < 0");
  if (n_req == 0) return HC_OK;
  if (pool->accounting) return fail(HC_E_UNSUPPORTED, "accounting-only pool has no device storage");
  if (!pool->L.has_q) return fail(HC_E_UNSUPPORTED, "pool was created without w_q");
  if (!x || !q_out) return fail(HC_E_INVALID, "x / q_out is null");
  std::vector<int32_t> ones(n_req, 1);
  std::vector<AppendReq> ar;
  std::vector<int32_t> tabs;
  int32_t max_rows = 0;
  AllocUndo undo;
  // k/v rows come from the projection GEMM itself: pass x to satisfy the row-source check
  hc_status st = validate_and_allocate(pool, n_req, req_ids, modes, ones.data(), x, x, x, &ar, &tabs, &max_rows, &undo);
  if (st != HC_OK) return st;
  st = project_after_alloc(pool, n_req, req_ids, x, q_out, ar, tabs, stream);
  if (st != HC_OK) undo.rollback(pool);
  return st;
}

static hc_status project_after_alloc(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const void* x, void* q_out,
                                     const std::vector<AppendReq>& ar, const std::vector<int32_t>& tabs, void* stream) {
  const int B = pool->cfg.block_size, d = pool->cfg.d_model;
  hc_status st;
  // cache slot of each request's new token: KV rows are written by the GEMM epilogue,
  // hidden rows (x itself) by the append scatter
  std::vector<AppendReq> har;
  std::vector<int32_t> row_dst(4 * (size_t)n_req, 0);
  const int Bkv = pool->kv.Bkv;
  for (int32_t i = 0; i < n_req; ++i) {
    const Req& r = pool->reqs[req_ids[i]];
    const int64_t pos = r.n - 1, lb = pos / Bkv;
    row_dst[4 * i + 3] = (int32_t)pos;   // RoPE position of the new token
    if (r.mode == HC_MODE_KV) {
      row_dst[4 * i] = r.a[lb];
      row_dst[4 * i + 1] = pool->kv.packed ? r.a[lb] : r.b[lb];
      row_dst[4 * i + 2] = (int32_t)(pos - lb * Bkv);
    } else {
      row_dst[4 * i] = row_dst[4 * i + 1] = -1;
      AppendReq q = ar[i];   // one token per request: ar[i] is request i
      q.row_off = i;         // x row of request i
      har.push_back(q);
    }
  }
  DeviceGuard g(pool->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!har.empty()) {
    st = scatter_rows(pool, har, tabs, nullptr, nullptr, x, stream);
    if (st != HC_OK) return st;
  }
  const int launches = pool->last_launches;
  const size_t rd_bytes = row_dst.size() * sizeof(int32_t);
  if (rd_bytes > kStagingBytes / 2) return fail(HC_E_UNSUPPORTED, "batch too large for the staging area");
  char* rd_dev = pool->storage + pool->L.stage_off + kStagingBytes / 2;
  Pinned* pin = pool->pinned(rd_bytes);
  if (!pin) return fail(HC_E_CUDA, "pinned staging unavailable (cudaMallocHost failed, or all slots held by captured graphs)");
  std::memcpy(pin->ptr, row_dst.data(), rd_bytes);
  cudaError_t err = cudaMemcpyAsync(rd_dev, pin->ptr, rd_bytes, cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) return cuda_fail(err, "projection descriptor upload");
  pool->staged(pin, s);
  DenseParams dp{};
  dp.a = x;
  dp.w = pool->storage + pool->L.wq_off;
  dp.bias = reinterpret_cast<const float*>(pool->storage + pool->L.bq_off);   // [b_Q | b_int] (zeros if absent)
  dp.M = n_req;
  dp.N = d + 2 * pool->kv.dk;
  dp.K = d;
  dp.epi = 1;
  dp.out = q_out;
  dp.dk = pool->kv.dk;
  dp.Bkv = pool->kv.Bkv;
  dp.v_off = pool->kv.v_off;
  dp.pool = pool->storage + pool->L.blocks_off;
  dp.row_dst = reinterpret_cast<const int32_t*>(rd_dev);
  dp.rope_inv = pool->cfg.rope_theta > 0.f ? reinterpret_cast<const double*>(pool->storage + pool->L.rope_off) : nullptr;
  dp.d = d;
  dp.H = pool->cfg.n_heads;
  dp.dh = pool->cfg.head_dim;
  dp.B = B;
  if (pool->dense_tc_ok) {
    CUtensorMap ta;
    if (!make_tmap_rows(&ta, x, n_req, d)) return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed (x)");
    err = launch_dense_tc(dp, &ta, &pool->tmap_wqkv, pool->num_sms, s);
  } else {
    err = launch_dense_simt(dp, pool->cfg.dtype, s);
  }
  if (err != cudaSuccess) return cuda_fail(err, "projection kernel");
  pool->last_launches = launches + 1;
  return HC_OK;
}

hc_status hc_merge_partials(int32_t n_parts, int32_t n_rows, int32_t n_heads, int32_t head_dim, hc_dtype dtype,
                            const void* outs, const float* lses, void* out, float* lse, void* stream) {
  if (n_parts < 1 || n_rows < 0 || n_heads < 1 || head_dim < 1)
    return fail(HC_E_INVALID, "merge: n_parts >= 1, n_rows >= 0, n_heads >= 1, head_dim >= 1 required");
  if (dtype != HC_BF16 && dtype != HC_F32) return fail(HC_E_INVALID, "merge: unknown dtype");
  if (n_rows == 0) return HC_OK;
  if (!outs || !lses || !out) return fail(HC_E_INVALID, "merge: outs / lses / out is null");
  cudaError_t err = launch_merge(n_parts, n_rows, n_heads, head_dim, dtype == HC_F32 ? 1 : 0, outs, lses, out, lse,
                                 static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "merge kernel");
  return HC_OK;
}

hc_status hc_layer_norm(hc_pool* pool, int32_t n_rows, const void* x, void* u, void* stream) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  pool->last_launches = 0;
  if (n_rows < 0) return fail(HC_E_INVALID, "n_rows < 0");
  if (n_rows == 0) return HC_OK;
  if (pool->accounting) return fail(HC_E_UNSUPPORTED, "accounting-only pool has no device storage");
  if (!pool->L.has_ln) return fail(HC_E_UNSUPPORTED, "pool was created without ln_gamma");
  if (!x || !u) return fail(HC_E_INVALID, "x / u is null");
  DeviceGuard g(pool->cfg.device);
  const float* gb = reinterpret_cast<const float*>(pool->storage + pool->L.ln_off);
  cudaError_t err = launch_layer_norm(x, u, gb, gb + pool->cfg.d_model, pool->cfg.ln_eps, n_rows, pool->cfg.d_model,
                                      pool->cfg.dtype, static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "layer norm kernel");
  pool->last_launches = 1;
  return HC_OK;
}

hc_status hc_output_projection(hc_pool* pool, int32_t n_req, const void* o, void* y, void* stream) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  pool->last_launches = 0;
  if (n_req < 0) return fail(HC_E_INVALID, "n_req < 0");
  if (n_req == 0) return HC_OK;
  if (pool->accounting) return fail(HC_E_UNSUPPORTED, "accounting-only pool has no device storage");
  if (!pool->L.has_o) return fail(HC_E_UNSUPPORTED, "pool was created without w_o");
  if (!o || !y) return fail(HC_E_INVALID, "o / y is null");
  const int d = pool->cfg.d_model;
  DeviceGuard g(pool->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DenseParams dp{};
  dp.a = o;
  dp.w = pool->storage + pool->L.wo_off;
  dp.bias = reinterpret_cast<const float*>(pool->storage + pool->L.bo_off);
  dp.M = n_req;
  dp.N = d;
  dp.K = d;
  dp.epi = 2;
  dp.out = y;
  dp.d = d;
  dp.H = pool->cfg.n_heads;
  dp.dh = pool->cfg.head_dim;
  dp.B = pool->cfg.block_size;
  cudaError_t err;
  if (pool->dense_tc_ok) {
    CUtensorMap ta;
    if (!make_tmap_rows(&ta, o, n_req, d)) return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed (o)");
    err = launch_dense_tc(dp, &ta, &pool->tmap_wo, pool->num_sms, s);
  } else {
    err = launch_dense_simt(dp, pool->cfg.dtype, s);
  }
  if (err != cudaSuccess) return cuda_fail(err, "output projection kernel");
  pool->last_launches = 1;
  return HC_OK;
}

size_t hc_layer_workspace_size(const hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes) {
  if (!pool || n_req < 0 || (n_req > 0 && (!req_ids || !modes))) {
    g_err = "invalid arguments";
    return 0;
  }
  if (n_req == 0) return kAlign;
  std::vector<Req> tmp(n_req);
  std::vector<const Req*> rs(n_req);
  for (int32_t i = 0; i < n_req; ++i) {
    auto it = pool->reqs.find(req_ids[i]);
    tmp[i].mode = it != pool->reqs.end() ? it->second.mode : modes[i];
    tmp[i].n = (it != pool->reqs.end() ? it->second.n : 0) + 1;
    rs[i] = &tmp[i];
  }
  const size_t qa = align_up((size_t)n_req * pool->cfg.d_model * pool->elem, kAlign);
  return (pool->L.has_ln ? 3 : 2) * qa + pool->plan(rs).total;
}

hc_status hc_decode_layer(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                          const void* x, float scale, void* y, float* lse, void* workspace, size_t ws_bytes,
                          void* stream) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  if (n_req == 0) {
    pool->last_launches = 0;
    return HC_OK;
  }
  const size_t need = hc_layer_workspace_size(pool, n_req, req_ids, modes);
  if (need == 0) return fail(HC_E_INVALID, "invalid arguments");
  if (!workspace || ws_bytes < need) return fail(HC_E_WORKSPACE, "workspace smaller than hc_layer_workspace_size()");
  if (!y) return fail(HC_E_INVALID, "y is null");
  const size_t qa = align_up((size_t)n_req * pool->cfg.d_model * pool->elem, kAlign);
  char* ws = static_cast<char*>(workspace);
  // workspace: q | o | [u = LN(x)] | attention workspace
  const size_t pre = (pool->L.has_ln ? 3 : 2) * qa;
  int launches = 0;
  hc_status st;
  if (pool->L.has_ln) {
    st = hc_layer_norm(pool, n_req, x, ws + 2 * qa, stream);
    if (st != HC_OK) return st;
    x = ws + 2 * qa;
    launches = 1;
  }
  st = hc_project_append(pool, n_req, req_ids, modes, x, ws, stream);
  if (st != HC_OK) return st;
  launches += pool->last_launches;
  st = hc_decode_attention(pool, n_req, req_ids, ws, scale, ws + qa, lse, ws + pre, ws_bytes - pre, stream);
  if (st != HC_OK) return st;
  launches += pool->last_launches;
  st = hc_output_projection(pool, n_req, ws + qa, y, stream);
  if (st != HC_OK) return st;
  pool->last_launches = launches + pool->last_launches;
  return HC_OK;
}

// ============================================================ prefill / recompute (f3)
namespace {
struct PrefillPlan {
  int64_t rows = 0;
  int32_t n_qtiles = 0;
  size_t off_q, off_kv, off_o, off_u, off_rowdst, off_row0, off_treq, off_tq0, total;
};
// query rows per prefill attention tile: 128 on the tcgen05 kernel, 64 on the mma.sync one
bool prefill_uses_tc(const hc_pool* pool) {
  return pool->tune.prefill_tc != 0 && prefill_attn_mma_supported(pool->cfg.dtype, pool->cfg.head_dim) &&
         !(pool->cfg.flags & HC_FLAG_FORCE_SIMT);
}
int prefill_tile_rows(const hc_pool* pool) { return prefill_uses_tc(pool) ? prefill_attn_tc_rows(pool->tune) : 64; }

PrefillPlan prefill_plan(const hc_pool* pool, int32_t n_req, const int32_t* lens) {
  PrefillPlan P;
  const int tq = prefill_tile_rows(pool);
  for (int32_t i = 0; i < n_req; ++i) {
    P.rows += lens[i];
    P.n_qtiles += (int32_t)cdiv(lens[i], tq);
  }
  const size_t e = pool->elem, d = (size_t)pool->cfg.d_model;
  size_t o = 0;
  P.off_q = o;
  o = align_up(o + P.rows * d * e, kAlign);
  P.off_kv = o;
  o = align_up(o + P.rows * 2 * (size_t)pool->kv.dk * e, kAlign);
  P.off_o = o;
  o = align_up(o + P.rows * d * e, kAlign);
  P.off_u = o;   // LN(x) when the pool has a LayerNorm
  o = align_up(o + (pool->L.has_ln ? P.rows * d * e : 0), kAlign);
  P.off_rowdst = o;
  o = align_up(o + P.rows * 4 * sizeof(int32_t), kAlign);
  P.off_row0 = o;
  o = align_up(o + (n_req + 1) * sizeof(int32_t), kAlign);
  P.off_treq = o;
  o = align_up(o + P.n_qtiles * sizeof(int32_t), kAlign);
  P.off_tq0 = o;
  o = align_up(o + P.n_qtiles * sizeof(int32_t), kAlign);
  P.total = o;
  return P;
}
}  // namespace

size_t hc_prefill_workspace_size(const hc_pool* pool, int32_t n_req, const int32_t* lens) {
  if (!pool || n_req < 0 || (n_req > 0 && !lens)) {
    g_err = "invalid arguments";
    return 0;
  }
  for (int32_t i = 0; i < n_req; ++i)
    if (lens[i] < 1) {
      g_err = "lens must be >= 1";
      return 0;
    }
  return n_req == 0 ? kAlign : prefill_plan(pool, n_req, lens).total;
}

static hc_status prefill_after_alloc(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* lens,
                                     const void* x, float scale, void* y, void* workspace, const PrefillPlan& P,
                                     const std::vector<AppendReq>& ar, const std::vector<int32_t>& tabs, void* stream);

hc_status hc_prefill_layer(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                           const int32_t* lens, const void* x, float scale, void* y, void* workspace,
                           size_t ws_bytes, void* stream) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  pool->last_launches = 0;
  if (n_req < 0) return fail(HC_E_INVALID, "n_req < 0");
  if (n_req == 0) return HC_OK;
  if (pool->accounting) return fail(HC_E_UNSUPPORTED, "accounting-only pool has no device storage");
  if (!pool->L.has_q || !pool->L.has_o) return fail(HC_E_UNSUPPORTED, "pool was created without w_q / w_o");
  if (!req_ids || !modes || !lens || !x || !y || !workspace) return fail(HC_E_INVALID, "null argument");
  for (int32_t i = 0; i < n_req; ++i) {
    if (lens[i] < 1) return fail(HC_E_INVALID, "lens must be >= 1");
    auto it = pool->reqs.find(req_ids[i]);
    if (it != pool->reqs.end() && it->second.n > 0)
      return fail(HC_E_INVALID, "prefill needs new requests (cache-type switch: hc_free first)");
  }
  const PrefillPlan P = prefill_plan(pool, n_req, lens);
  if (ws_bytes < P.total) return fail(HC_E_WORKSPACE, "workspace smaller than hc_prefill_workspace_size()");
  std::vector<AppendReq> ar;
  std::vector<int32_t> tabs;
  int32_t max_rows = 0;
  AllocUndo undo;
  DeviceGuard g(pool->cfg.device);   // before the staging slot: its event belongs to the pool's device
  hc_status st = validate_and_allocate(pool, n_req, req_ids, modes, lens, x, x, x, &ar, &tabs, &max_rows, &undo);
  if (st != HC_OK) return st;
  st = prefill_after_alloc(pool, n_req, req_ids, lens, x, scale, y, workspace, P, ar, tabs, stream);
  if (st != HC_OK) undo.rollback(pool);
  return st;
}

static hc_status prefill_after_alloc(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* lens,
                                     const void* x, float scale, void* y, void* workspace, const PrefillPlan& P,
                                     const std::vector<AppendReq>& ar, const std::vector<int32_t>& tabs, void* stream) {
  const int B = pool->cfg.block_size, d = pool->cfg.d_model, H = pool->cfg.n_heads, dh = pool->cfg.head_dim;
  hc_status st;
  // host descriptor: per-row cache targets (KV rows), request row offsets, query tiles
  const size_t desc_bytes = P.total - P.off_rowdst;
  Pinned* pin = pool->pinned(desc_bytes);
  if (!pin) return fail(HC_E_CUDA, "pinned staging unavailable (cudaMallocHost failed, or all slots held by captured graphs)");
  char* hbase = static_cast<char*>(pin->ptr);
  std::memset(hbase, 0, desc_bytes);
  int32_t* rowdst = reinterpret_cast<int32_t*>(hbase);
  int32_t* row0 = reinterpret_cast<int32_t*>(hbase + (P.off_row0 - P.off_rowdst));
  int32_t* treq = reinterpret_cast<int32_t*>(hbase + (P.off_treq - P.off_rowdst));
  int32_t* tq0 = reinterpret_cast<int32_t*>(hbase + (P.off_tq0 - P.off_rowdst));
  std::vector<AppendReq> har;
  int64_t r = 0;
  int32_t nt = 0;
  for (int32_t i = 0; i < n_req; ++i) {
    const Req& q = pool->reqs[req_ids[i]];
    row0[i] = (int32_t)r;
    for (int32_t tkn = 0; tkn < lens[i]; ++tkn, ++r) {
      const int64_t lb = tkn / pool->kv.Bkv;
      rowdst[4 * r + 3] = tkn;           // RoPE position
      if (q.mode == HC_MODE_KV) {
        rowdst[4 * r] = q.a[lb];
        rowdst[4 * r + 1] = pool->kv.packed ? q.a[lb] : q.b[lb];
        rowdst[4 * r + 2] = (int32_t)(tkn - lb * pool->kv.Bkv);
      } else {
        rowdst[4 * r] = rowdst[4 * r + 1] = -1;
      }
    }
    for (int32_t t0 = 0; t0 < lens[i]; t0 += prefill_tile_rows(pool), ++nt) {
      treq[nt] = i;
      tq0[nt] = t0;
    }
    if (q.mode == HC_MODE_HIDDEN) {
      AppendReq a = ar[i];          // lens >= 1: ar[i] is request i
      a.row_off = row0[i];          // x rows of request i
      har.push_back(a);
    }
  }
  {  // causal work grows with the tile's position: launch the longest tiles first
    std::vector<std::pair<int32_t, int32_t>> tl(nt);
    for (int32_t k = 0; k < nt; ++k) tl[k] = {tq0[k], treq[k]};
    std::stable_sort(tl.begin(), tl.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    for (int32_t k = 0; k < nt; ++k) {
      tq0[k] = tl[k].first;
      treq[k] = tl[k].second;
    }
  }
  row0[n_req] = (int32_t)r;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  cudaError_t err = cudaMemcpyAsync(ws + P.off_rowdst, hbase, desc_bytes, cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) return cuda_fail(err, "prefill descriptor upload");
  pool->staged(pin, s);
  int launches = 0;
  if (pool->L.has_ln) {   // u = LN(x): the projections' input and what the hidden cache holds (R15)
    const float* gb = reinterpret_cast<const float*>(pool->storage + pool->L.ln_off);
    err = launch_layer_norm(x, ws + P.off_u, gb, gb + d, pool->cfg.ln_eps, (int32_t)P.rows, d, pool->cfg.dtype, s);
    if (err != cudaSuccess) return cuda_fail(err, "layer norm kernel");
    x = ws + P.off_u;
    ++launches;
  }
  if (!har.empty()) {
    st = scatter_rows(pool, har, tabs, nullptr, nullptr, x, stream);   // hidden mode: cache x itself
    if (st != HC_OK) return st;
    launches += pool->last_launches;
  }
  // q, k, v of every token; KV rows also land in the cache
  DenseParams dp{};
  dp.a = x;
  dp.w = pool->storage + pool->L.wq_off;
  dp.bias = reinterpret_cast<const float*>(pool->storage + pool->L.bq_off);
  dp.M = (int32_t)P.rows;
  dp.N = d + 2 * pool->kv.dk;
  dp.K = d;
  dp.epi = 1;
  dp.dk = pool->kv.dk;
  dp.Bkv = pool->kv.Bkv;
  dp.v_off = pool->kv.v_off;
  dp.out = ws + P.off_q;
  dp.pool = pool->storage + pool->L.blocks_off;
  dp.row_dst = reinterpret_cast<const int32_t*>(ws + P.off_rowdst);
  dp.kvbuf = ws + P.off_kv;
  dp.rope_inv = pool->cfg.rope_theta > 0.f ? reinterpret_cast<const double*>(pool->storage + pool->L.rope_off) : nullptr;
  dp.d = d;
  dp.H = H;
  dp.dh = dh;
  dp.B = B;
  if (pool->dense_tc_ok) {
    CUtensorMap ta;
    if (!make_tmap_rows(&ta, x, (int)P.rows, d)) return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed (x)");
    err = launch_dense_tc(dp, &ta, &pool->tmap_wqkv, pool->num_sms, s);
  } else {
    err = launch_dense_simt(dp, pool->cfg.dtype, s);
  }
  if (err != cudaSuccess) return cuda_fail(err, "prefill projection kernel");
  ++launches;
  PrefillAttnParams pa{};
  pa.q = ws + P.off_q;
  pa.kv = ws + P.off_kv;
  pa.o = ws + P.off_o;
  pa.row0 = reinterpret_cast<const int32_t*>(ws + P.off_row0);
  pa.tile_req = reinterpret_cast<const int32_t*>(ws + P.off_treq);
  pa.tile_q0 = reinterpret_cast<const int32_t*>(ws + P.off_tq0);
  pa.n_qtiles = P.n_qtiles;
  pa.H = H;
  pa.dh = dh;
  pa.d = d;
  pa.dk = pool->kv.dk;
  pa.G = H / pool->kv.Hk;
  pa.scale_log2 = scale * 1.4426950408889634f;
  if (prefill_uses_tc(pool)) {
    CUtensorMap tq, tkv;
    if (!make_tmap_2d(&tq, ws + P.off_q, (uint64_t)d, (uint64_t)P.rows, 64, 128) ||
        !make_tmap_2d(&tkv, ws + P.off_kv, 2 * (uint64_t)pool->kv.dk, (uint64_t)P.rows, 64,
                      (uint32_t)prefill_attn_tc_keys(pool->tune)))
      return fail(HC_E_CUDA, "cuTensorMapEncodeTiled failed (prefill attention)");
    err = launch_prefill_attn_tc(pa, &tq, &tkv, pool->tune, s);
  } else {
    err = launch_prefill_attn(pa, pool->cfg.dtype, s);
  }
  if (err != cudaSuccess) return cuda_fail(err, "prefill attention kernel");
  ++launches;
  st = hc_output_projection(pool, (int32_t)P.rows, ws + P.off_o, y, stream);
  if (st != HC_OK) return st;
  pool->last_launches = launches + 1;
  return HC_OK;
}

int32_t hc_last_launch_count(const hc_pool* pool) { return pool ? pool->last_launches : -1; }
int32_t hc_last_decode_path(const hc_pool* pool) { return pool ? pool->last_path : -1; }
int32_t hc_last_kernel_config(const hc_pool* pool) { return pool ? pool->last_cfg : -1; }

hc_status hc_set_profiling(hc_pool* pool, int32_t enable) {
  if (!pool) return fail(HC_E_INVALID, "pool is null");
  pool->profiling = enable != 0;
  return HC_OK;
}

hc_status hc_kernel_times(hc_pool* pool, float* ms4, int32_t* n_calls) {
  if (!pool || !ms4) return fail(HC_E_INVALID, "null argument");
  DeviceGuard g(pool->cfg.device);
  double acc[4] = {0, 0, 0, 0};
  for (auto& ev : pool->prof_pending) {
    cudaError_t err = cudaEventSynchronize(ev[4]);
    if (err != cudaSuccess) return cuda_fail(err, "cudaEventSynchronize");
    float t;
    const int pairs[4][2] = {{1, 2}, {2, 3}, {3, 4}, {0, 1}};
    for (int k = 0; k < 4; ++k) {
      cudaEventElapsedTime(&t, ev[pairs[k][0]], ev[pairs[k][1]]);
      acc[k] += t;
    }
    for (auto e : ev) pool->ev_free.push_back(e);
  }
  if (n_calls) *n_calls = (int32_t)pool->prof_pending.size();
  pool->prof_pending.clear();
  for (int k = 0; k < 4; ++k) ms4[k] = (float)acc[k];
  return HC_OK;
}

}  // extern "C"
