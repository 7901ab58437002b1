// Internal types shared by the host runtime (runtime.cu) and the kernels.
// Not part of the C ABI.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace hc {

// Schedule / A-B knobs of the kernels.  Read ONCE from the environment when a pool is created
// (runtime.cu tuning_from_env, the library's only getenv site) and fixed for the pool's life;
// the defaults are the measured-best configuration.  None of them changes
// what is computed — only tile order, pipeline depth or which equivalent kernel runs.  The
// timing diagnostics that DO change results (HC_DIAG_*) exist only in a -DHC_DIAG build.
struct Tuning {
  int fused = -1;        // HC_FUSED: 0 = two-kernel path, else the fused step kernel when supported
  int epi_attend = 1;    // HC_EPI_ATTEND: 0 = rebuilt K/V into scratch + attention kernel
  int fused_cfg = 0;     // HC_FUSED_CFG: {GEMM stages, attention warps, stages} of the fused kernel; 0 = auto
  int fused_nsub = 0;    // HC_FUSED_NSUB: fused GEMM tile 256 x 256*nsub (1 or 2); 0 = auto (1 for GQA)
  int group_n = 4;       // HC_GROUP_N: n-tiles per raster group of the fused kernel
  int sync_w = -1;       // HC_SYNC_W: partner k-lockstep window (-1: kernel default, 0 off)
  int group_m = -2;      // HC_GROUP_M: raster of the stand-alone reconstruction GEMM
  int l2_hint = 0;       // HC_L2HINT: L2 policy of the GEMM operand loads (pair_gemm.cuh TcArgs)
  int block_runs = 0;    // HC_BLOCK_RUNS: 1 = runs of consecutive hidden blocks as one 128-row TMA box
                         // (off: at cfg4 with request-by-request fills it lifted the tensor pipe to 93% but
                         // raised L2/DRAM traffic 309 -> 418 / 46 -> 81 GB and the capped clock fell 10%)
  int gqa_scratch = -1;  // HC_GQA_SCRATCH: GQA hidden requests via rebuilt K/V scratch + the tensor-core KV loop
                         // (-1 auto: for groups of >= 8 query heads; 0 never; 1 always)
  int attn_tc = 1;       // HC_ATTN_TC: KV attention on mma.sync (attn_tc.cuh): 0 never, 1 GQA only, 2 always
  int tc_1sm = 0;        // HC_TC_1SM: 1-SM tcgen05 reconstruction kernel instead of CTA pairs
  int tc_nsub = 0;       // HC_TC_NSUB: 1 = 256-wide pair tiles
  int tc_stages = 4;     // HC_TC_STAGES (3 or 4)
  int attn_cfg = 0;      // HC_ATTN_CFG: warps x stages of the stand-alone attention kernel
  int prefill_tc = 1;    // HC_PREFILL_TC: 0 = mma.sync prefill attention
  int prefill_cfg = 1;   // HC_PREFILL_CFG: 1, 2 or 128 (prefill_attn.cu)
  int z_cfg = 1282;      // HC_Z_CFG (absorbed variant)
  int score_st = 2;      // HC_SCORE_ST (absorbed variant)
  int qt_bn = 128;       // HC_QT_BN (absorbed variant)
  int epi_mma = 1;       // HC_EPI_MMA: attend epilogue on mma.sync (attend_tile_mma): 0 off, 1 GQA, 2 always
  int dyn_tiles = 1;     // HC_DYN_TILES: fused kernel takes GEMM tiles from a global counter (0: static stride)
  int attn_sms = 0;      // HC_ATTN_SMS: stand-alone attention kernel on at most this many SMs (measurement)
  int diag_epi = 0;      // -DHC_DIAG builds only: HC_DIAG_EPI (wrong outputs, timing only)
  int diag_box = 0;      // -DHC_DIAG builds only: HC_DIAG_BOX (wrong outputs, timing only)
  int diag_attn = 0;     // -DHC_DIAG builds only: HC_DIAG_ATTN (wrong outputs, timing only)
};

// Per-request entry of the decode-call descriptor (uploaded once per call).
struct ReqDesc {
  int32_t mode;          // 0 KV, 1 hidden (beta_i)
  int32_t n;             // cached tokens incl. the current one
  int32_t tab_off;       // KV: offset of (K,V) block-id pairs in the flat table
  int32_t scratch_blk0;  // hidden: first scratch block of the rebuilt K/V
  int32_t split_begin;   // first split of this request
  int32_t split_count;
  int32_t pad0, pad1;
};

// A split-K unit: tokens [lb0*B, lb0*B + ntok) of request `req`.
struct SplitDesc {
  int32_t req;
  int32_t lb0;   // first logical block
  int32_t ntok;  // tokens in this split (>= 1)
  int32_t pad;
};

struct AttnParams {
  const ReqDesc* reqs;
  const SplitDesc* splits;
  const int32_t* tables;  // KV (K id, V id) pairs per logical block
  const void* pool;       // unit blocks; KV block layout [H][B][dh]
  const void* scr_k;      // rebuilt K of hidden requests, [hblock][H][B][dh]
  const void* scr_v;
  const void* q;          // [n_req, d]
  float* part_ml;         // [H][n_splits_all][2]: running max (log2 domain), sum
  float* part_acc;        // [H][n_splits_all][dh]: unnormalised sum_j p_j v_j (head-major, so a
                          // (request, head)'s splits are contiguous for the combine)
  int32_t n_splits_all;   // splits in the call (partial index = head * n_splits_all + split)
  int32_t* task_counter;  // zero on entry (part of the uploaded descriptor)
  int32_t n_tasks;        // n_splits * H; task = split * H + head
  int32_t H, dh, B, d;    // B: hidden block (and scratch) tokens
  // KV-mode layout (GQA, R18): query head h reads K/V head h / G of Hk; a KV logical block
  // holds Bkv tokens, K at unit(tab K) + hk*Bkv*dh, V at unit(tab V) + v_off + hk*Bkv*dh
  // (multi-head: Hk = H, G = 1, Bkv = B, v_off = 0; GQA: K and V share one unit)
  int32_t Hk, G, Bkv;
  int64_t v_off;
  float scale_log2;       // scale * log2(e)
  // ---- fused step kernel only: KV tasks first, then hidden tasks in GEMM n-tile order
  const int32_t* kv_split_ids;   // splits of KV-mode requests
  const int32_t* hid_split_ids;  // splits of hidden-mode requests, in scratch (GEMM row) order
  int32_t n_kv_tasks;            // (#KV splits) * H
  int32_t n_hid_splits;
  const int32_t* tile_done;      // [gemm_m_tiles][gemm_n_tiles] finished epilogue warps (8 = ready)
  int32_t gemm_n_tiles, gemm_tile_m, gemm_tile_n;
  int32_t tile_target;           // finished epilogue warps per GEMM tile (8, or 16 with extra epilogue warps)
  int32_t th;                    // heads per split in the task numbering: H (SIMT loop) or Hk (tensor-core loop)
  int32_t tc;                    // 1: every task is a KV-mode split and runs attn_tc.cuh (task = split * Hk + kvhead)
  int32_t diag;                  // -DHC_DIAG builds only (HC_DIAG_ATTN): 1 skip the math, 2 read block 0 only
};

struct CombineParams {
  const ReqDesc* reqs;
  const float* part_ml;   // [H][n_splits][2]
  const float* part_acc;  // [H][n_splits][dh]
  int32_t n_splits;
  void* out;   // [n_req, d]
  float* lse;  // nullable [n_req, H]
  int32_t n_req, H, dh, d;
};

struct ReconParams {
  const int32_t* gather;  // pool block id of each hidden block (in scratch order)
  int32_t n_hblocks;      // hidden blocks; GEMM rows M = n_hblocks * B
  const void* pool;
  const void* w_int;      // head-interleaved W_KV copy, [2d, d]: row h*2dh + kv*dh + c
  const float* b_int;     // nullable, same interleaving
  void* scr_k;            // [hblock][Hk][B][dh]
  void* scr_v;
  int32_t d, H, dh, B;
  int32_t Hk, dk;         // K/V heads and K (or V) row width Hk*dh (GEMM N = 2 dk; GQA, R18)
  int32_t* sync_counter;  // >= 32*num_sms zeroed ints (pair progress words)
  int32_t* tile_counter;  // one zeroed int: dynamic GEMM tile schedule of the fused kernel
  const int32_t* hblk_pos;  // token position of row 0 of each hidden block (RoPE / attend; nullable)
  const double* rope_inv;   // RoPE: inv_freq table [dh/2] (nullable = no RoPE)
  // ---- fused reconstruct-and-attend (epi_attend): the GEMM epilogue turns each segment of
  // `seg` tokens x head into a flash-decoding partial; rebuilt K/V never reach memory
  bool epi_attend;
  const int32_t* hblk_req;  // batch index of each hidden block's request
  const ReqDesc* reqs;      // n, split_begin of every request
  const void* q;            // [n_req, d]
  float* part_ml;
  float* part_acc;
  int32_t n_splits_all;     // partial index = head * n_splits_all + split
  float scale_log2;
  int32_t seg;              // tokens per partial: min(B, 32)
  int64_t kv_tokens;        // KV-mode tokens attended in this call (fused-kernel configuration choice)
};
bool recon_pair_mode(int B, const Tuning& t);   // the CTA-pair GEMM serves this block size (else the 1-SM kernel)

struct AppendReq {
  int32_t mode;
  int32_t start;    // tokens already cached
  int32_t n_tok;    // rows appended
  int32_t row_off;  // first source row in k/v (KV) or x (hidden)
  int32_t tab_off;  // block ids covering logical blocks [start/B, (start+n_tok-1)/B];
                    // KV: (K,V) pairs, hidden: single ids
  int32_t pad0, pad1, pad2;
};

struct AppendParams {
  const AppendReq* reqs;
  const int32_t* tabs;
  const void* k;          // [rows, dk]
  const void* v;
  const void* x;          // [rows, d]
  void* pool;
  int32_t n_req, d, H, dh, B;
  int32_t dk, Bkv;        // KV row width and tokens per KV logical block (AttnParams)
  int64_t v_off;
};

// Dense projection GEMM for the current-token q/k/v map and the output map (NEXT row f1):
// C = A W^T (+ bias), A [M, K] row-major, W [N, K] row-major.
struct DenseParams {
  const void* a;           // [M, K], pool dtype
  const void* w;           // [N, K] (SIMT path; the tcgen05 path reads it through a tensor map)
  const float* bias;       // nullable [N]
  int32_t M, N, K;
  int32_t epi;             // 1: project (q | head-interleaved K||V -> cache slot), 2: dense C
  void* out;               // epi 1: q [M, d]; epi 2: C [M, N]
  void* pool;              // epi 1: unit blocks
  const int32_t* row_dst;  // epi 1: per row {K block, V block, slot, 0}; K block < 0 = hidden row
  int32_t d, H, dh, B;
  int32_t dk, Bkv;         // epi 1: K/V row width, tokens per KV logical block (GQA, R18)
  int64_t v_off;           // epi 1: V rows' offset inside the V unit (GQA: K and V share a unit)
  void* kvbuf;             // epi 1 (prefill): also each row's head-interleaved K||V, [M, 2dk]
  const double* rope_inv;  // epi 1: rotate q and k at row_dst[4r+3] (nullable = no RoPE)
};

// dtype: 0 bf16, 1 fp32
cudaError_t launch_append(const AppendParams& p, int dtype, int max_rows, cudaStream_t s);
cudaError_t launch_relayout_w(const void* w, void* w_int, const float* b, float* b_int, int d,
                              int dk, int dh, int dtype, cudaStream_t s);
cudaError_t launch_recon_simt(const ReconParams& p, int dtype, cudaStream_t s);
// tmap_w: W_int with 256-row boxes (1-SM kernel); tmap_w_half: 128-row boxes (CTA-pair kernel)
cudaError_t launch_recon_tc(const ReconParams& p, const void* tmap_x, const void* tmap_w,
                            const void* tmap_w_half, int num_sms, const Tuning& t, cudaStream_t s,
                            const void* tmap_x128 = nullptr);
bool recon_tc_supported(int d, int dk, int dh, int B);
bool dense_tc_supported(int d);
// tmap_a: A with {64 x 128} boxes; tmap_w: W with {64 x 128} boxes
cudaError_t launch_dense_tc(const DenseParams& p, const void* tmap_a, const void* tmap_w, int num_sms, cudaStream_t s);
cudaError_t launch_dense_simt(const DenseParams& p, int dtype, cudaStream_t s);
cudaError_t launch_attn(const AttnParams& p, int dtype, bool generic, int num_sms, const Tuning& t, cudaStream_t s,
                        const void* tmap_kv = nullptr, const void* tmap_scr_k = nullptr,
                        const void* tmap_scr_v = nullptr);
// tensor-core KV attention (attn_tc.cuh) serves this shape: bf16, dh 64/128, G <= 8, Bkv % 16 == 0
bool attn_tc_supported(int dtype, int dh, int G, int Bkv);
bool attn_pipe_supported(int dtype, int dh, int B);
// Fused step: reconstruction GEMM (CTA pairs, 256x512 tiles) and split-K attention warps in
// one persistent kernel; hidden tasks wait on per-tile completion counters.
bool fused_supported(int d, int dk, int dh, int B);
int fused_tile_m();
int fused_tile_n();
cudaError_t launch_fused(const ReconParams& rp, AttnParams ap, const void* tmap_x, const void* tmap_w_half,
                         int32_t* tile_done, int num_sms, const Tuning& t, cudaStream_t s,
                         const void* tmap_kv = nullptr, int* cfg_out = nullptr, const void* tmap_scr_k = nullptr,
                         const void* tmap_scr_v = nullptr, const void* tmap_x128 = nullptr);
cudaError_t launch_combine(const CombineParams& p, int dtype, cudaStream_t s);
cudaError_t launch_merge(int n_parts, int n_rows, int H, int dh, int dtype, const void* outs, const float* lses,
                         void* out, float* lse, cudaStream_t s);
// u = (x - mean) / sqrt(var + eps) * gamma + beta per row of d (pre-attention LayerNorm, R15)
cudaError_t launch_layer_norm(const void* x, void* u, const float* gamma, const float* beta, float eps, int rows,
                              int d, int dtype, cudaStream_t s);

// Causal self-attention over each request's new tokens (prefill / recompute, NEXT row f3).
struct PrefillAttnParams {
  const void* q;            // [R, d] (R = sum of lens), heads = dh-column slices
  const void* kv;           // [R, 2dk], head-interleaved K_hk || V_hk per row (hk = h / G)
  void* o;                  // [R, d]
  const int32_t* row0;      // [n_req + 1] first row of each request (prefix sums of lens)
  const int32_t* tile_req;  // [n_qtiles] request of each 64-row query tile
  const int32_t* tile_q0;   // [n_qtiles] first query row (within its request) of each tile
  int32_t n_qtiles, H, dh, d;
  int32_t dk, G;            // K/V row width and query heads per K/V head (GQA, R18)
  float scale_log2;
};
cudaError_t launch_prefill_attn(const PrefillAttnParams& p, int dtype, cudaStream_t s);
bool prefill_attn_mma_supported(int dtype, int dh);
// tcgen05 version (128-query tiles; tile_q0 multiples of 128): tmap_q over q [R, d] and
// tmap_kv over kv [R, 2d], both {64 x 128} boxes.  HC_PREFILL_TC=0 selects the mma.sync kernel.
int prefill_attn_tc_keys(const Tuning& t);   // keys per tile (tmap_kv box rows)
int prefill_attn_tc_rows(const Tuning& t);   // query rows per CTA (tile_q0 step): 128 or 256
cudaError_t launch_prefill_attn_tc(const PrefillAttnParams& p, const void* tmap_q, const void* tmap_kv,
                                   const Tuning& t, cudaStream_t s);

// Absorbed hidden-cache attention (NEXT row f4 (ii), opt-in, absorbed.cu).  Hidden request
// r (0..n_h-1) owns gathered rows [hrow0[r], hrow0[r] + hntok[r]) (row g*B + t = slot t of
// pool block gather[g]); its tokens are split into 128-row score tiles (tile_req, tile_t0).
struct AbsorbParams {
  const int32_t* gather;   // pool block id of each hidden block (request order)
  const int32_t* hreq;     // [n_h] batch index of each hidden request
  const int32_t* hrow0;    // [n_h] first gathered row
  const int32_t* hntok;    // [n_h] cached tokens
  const int32_t* tile_req; // [n_tiles]
  const int32_t* tile_t0;  // [n_tiles] (128-token tiles)
  const int32_t* htile0;   // [n_h] first score tile of each hidden request
  const void* pool;
  const void* q;           // [n_req, d]
  const void* w_int;       // head-interleaved W_KV: row h*2dh + kv*dh + c
  const float* b_int;      // nullable, same interleaving
  __nv_bfloat16* qt;       // [n_h][Hp][d]  q~ = W_K,h^T q_h (rows H..Hp-1 zero)
  __nv_bfloat16* pm;       // [rows][Hp]    2^(scaled score - m_t), m_t = its tile's max
  float* tml;              // [n_tiles][Hp][2] tile max m_t (log2 domain), tile sum l_t
  float* ml;               // [n_h][H][3]   m (log2 domain), l, q_h . b_K,h
  __nv_bfloat16* z;        // [H][n_h][d]   sum_j 2^(s_j - m) x_j (head-major: K5's A operand)
  void* out;               // [n_req, d]
  float* lse;              // nullable [n_req, H]
  int32_t n_h, n_tiles, H, Hp, dh, d, B;
  int32_t n_hb;            // gathered hidden blocks
  int32_t rpb, rpb64;      // rows per TMA box of the pool tensor maps: min(B,128), min(B,64)
  float scale, scale_log2;
};
bool absorb_supported(int dtype, int d, int dh, int H, int B);
int absorb_launches();
// tmap_x / tmap_x64: pool rows with {64 x min(B,128)} / {64 x min(B,64)} boxes; tmap_qt:
// q~ [n_h*Hp, d] with {64 x Hp} boxes; tmap_p: P [rows, Hp] with {64 x 64} boxes; tmap_wk:
// W_int [2d, d] with {64 x dh} boxes (W_K,h rows, MN-major use) ; tmap_z: Z [H*n_h, d]
// with {64 x 128} boxes; tmap_wv: W_int with {64 x dh} boxes (W_V,h rows).
cudaError_t launch_absorbed(const AbsorbParams& p, const void* tmap_x, const void* tmap_x64, const void* tmap_qt,
                            const void* tmap_p, const void* tmap_wk, const void* tmap_z, const void* tmap_wv,
                            const Tuning& t, cudaStream_t s);

}  // namespace hc
