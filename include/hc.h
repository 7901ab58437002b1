/*
 * hc.h — C ABI of the B200-native hybrid-cache decode-attention library (libhc.so).
 *
 * The method (Apt-Serve, arXiv 2504.07494; citations are /root/reference/PAPER.md line
 * numbers "P:n" and SPEC.md lines "S:n"): every request i of a decode batch keeps,
 * per layer, EITHER a KV cache (beta_i = 0) OR a hidden cache of the layer's input
 * hidden states x_j (beta_i = 1; "Opportunity I", half the memory).
 * One decode step of one attention layer computes, per request and head h,
 *     hidden mode:  k_j = W_K x_j (+b_K),  v_j = W_V x_j (+b_V)   for all cached j  (Eq. 1)
 *     a_j = softmax_j(scale * q_h . k_{j,h})                                           (Eq. 2)
 *     out_{i,h} = sum_j a_j v_{j,h}         (Eq. 3 before W_o; v_i typo = v_j)
 * over all n_i cached tokens INCLUDING the current one ("attending to ... itself").
 * Cache storage is one unified pool of fixed-size blocks holding K, V or X vectors of
 * B consecutive tokens of one request (§4.3; Fig. 6).
 *
 * Conventions
 *  - Every call returns hc_status (HC_OK == 0) and never throws; hc_last_error() gives a
 *    thread-local message for the last non-OK status.
 *  - Validation errors are synchronous and leave the pool unchanged.  Launch failures
 *    return HC_E_CUDA (device state then undefined for that call).
 *  - One pool = one device.  Calls on a pool must be serialised by the caller (one host
 *    thread at a time) and their device work must be ordered (pass the same stream, or
 *    order the streams); device work is asynchronous on `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream).
 *  - The caller owns ALL device memory (pool storage, weights, q, out, lse, workspace);
 *    the library borrows the pointers.  It owns only host metadata (free list, block
 *    tables, a small ring of pinned staging buffers) — no hidden cudaMalloc.
 *  - Element type of K/V/X/q/out/W is the pool dtype (bf16 or fp32); bias and lse are fp32.
 */
#ifndef HC_H_
#define HC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HC_OK = 0,
  HC_E_INVALID = 1,        /* bad argument: null pointer, n_req < 0, duplicate ids, n_i = 0 ... */
  HC_E_OOM = 2,            /* not enough free unit blocks (append is all-or-nothing) */
  HC_E_UNKNOWN_REQ = 3,    /* decode of an id the pool has never seen / has freed */
  HC_E_MODE_MISMATCH = 4,  /* append with the other mode; switching = hc_free + re-append */
  HC_E_CUDA = 5,           /* a CUDA runtime call or launch failed */
  HC_E_UNSUPPORTED = 6,    /* shape / dtype combination not implemented */
  HC_E_WORKSPACE = 7       /* workspace too small (see hc_workspace_size) */
} hc_status;

typedef enum { HC_MODE_KV = 0, HC_MODE_HIDDEN = 1 } hc_mode; /* beta_i = 0 / 1 */
typedef enum { HC_BF16 = 0, HC_F32 = 1 } hc_dtype;

/* hc_pool_config.flags */
#define HC_FLAG_ACCOUNTING_ONLY 0x1 /* host allocator only: storage/w_kv may be NULL, no device
                                       work; hc_decode_attention returns HC_E_UNSUPPORTED */
#define HC_FLAG_FORCE_SIMT 0x2      /* rebuild K/V with the SIMT GEMM even in bf16 (cross-check) */
#define HC_FLAG_GENERIC_ATTN 0x4    /* use the generic (unpipelined) attention kernel */
#define HC_FLAG_ABSORB_HIDDEN 0x8   /* NON-PAPER variant: hidden-mode
                                       requests attend through q~ = W_K,h^T q_h and
                                       o_h = W_V,h (sum_j a_j x_j) + b_V,h instead of rebuilding
                                       K/V; same Eq. 2-3 by associativity.  bf16,
                                       no RoPE, d % 128 == 0, head_dim % 16 == 0, <= 128,
                                       n_heads <= 128; else hc_pool_create -> HC_E_UNSUPPORTED */

typedef struct hc_pool hc_pool;

typedef struct {
  int32_t d_model;       /* d = n_heads * head_dim */
  int32_t n_heads;       /* H; heads are contiguous head_dim-column slices of d (DESIGN R1) */
  int32_t head_dim;      /* dh */
  int32_t block_size;    /* B tokens per unit block (paper: fixed, unstated; default 16, R7) */
  int64_t num_blocks;    /* unit blocks in the pool (each B*d elements) */
  int32_t dtype;         /* hc_dtype */
  int32_t flags;         /* HC_FLAG_* */
  void* storage;         /* device buffer of hc_pool_storage_bytes() bytes, borrowed */
  size_t storage_bytes;
  const void* w_kv;      /* device [2 Dk, d] row-major, rows = W_K (Dk rows) then W_V; k = W_K x;
                            Dk = n_kv_heads * head_dim (= d for multi-head attention).
                            Copied once at create into head-interleaved order inside storage;
                            may be freed after create. */
  const float* b_kv;     /* nullable device [2 Dk] fp32 bias (b_K then b_V); copied at create */
  int32_t device;        /* CUDA device ordinal the storage lives on */
  int32_t split_tokens;  /* split-K chunk in tokens (multiple of B); 0 = automatic */
  /* Optional rest of the attention module (NEXT row f1; all nullable, copied at create):
   * w_q [d, d] (q = W_Q x, Eq. 1), b_q [d] fp32; w_o [d, d] (the output map of Eq. 3),
   * b_o [d] fp32.  Required by hc_project_append / hc_output_projection / hc_decode_layer. */
  const void* w_q;
  const float* b_q;
  const void* w_o;
  const float* b_o;
  /* Rotary position embedding (NEXT row f4; LLaMA/Yi-style models): 0 = none (OPT,
   * absolute positions before layer 1).  > 0: base theta of the NeoX "rotate_half" RoPE;
   * rebuilt K rows are rotated at their token positions in the reconstruction epilogue, and
   * hc_project_append / hc_prefill_layer rotate q and k at the new tokens' positions.
   * Callers of hc_decode_attention pass q already rotated.  Requires the bf16 tcgen05 path
   * and head_dim % 64 == 0 (HC_E_UNSUPPORTED otherwise). */
  float rope_theta;
  /* Optional pre-attention LayerNorm of the layer input (OPT; the
   * paper's Eq. 1 multiplies the layer input directly and specifies none, DESIGN R4/R15):
   * ln_gamma nullable device [d] fp32 (NULL = no LayerNorm), ln_beta nullable device [d]
   * fp32 (NULL = 0), ln_eps.  Copied at create.  With it, hc_decode_layer and
   * hc_prefill_layer normalise x before the projections, and the hidden cache holds the
   * normalised vector u = LN(x) — the exact vector Eq. 1 multiplies — so reconstruction
   * needs no extra work (DESIGN R15). */
  const float* ln_gamma;
  const float* ln_beta;
  float ln_eps;
  /* Grouped-query attention (NEXT row f4 (i): the LLaMA-3 / Yi models of §6.6; DESIGN
   * R18): n_kv_heads = Hk key/value heads, query head h attends K/V head h / (H / Hk).
   * 0 or n_heads = multi-head (Eq. 2-3 per head as written).  With Hk < H a KV-mode token
   * holds 2 Dk = 2 Hk dh values (< d): one unit block then stores the K and the V rows of
   * Bkv = B d / (2 Dk) tokens ([Hk][Bkv][dh] K, then the same for V), so KV takes ONE unit
   * per Bkv tokens while hidden takes one per B — under GQA the hidden cache is the larger
   * one.  Requires H % Hk == 0 and d % (2 Dk) == 0; not with HC_FLAG_ABSORB_HIDDEN. */
  int32_t n_kv_heads;
} hc_pool_config;

/* Bytes of device storage a pool with this config needs: the unit blocks, the
 * head-interleaved W_KV copy, the bias copy and the append staging area (256-B aligned).
 * Returns 0 for an invalid config. */
size_t hc_pool_storage_bytes(const hc_pool_config* cfg);

/* Unit blocks a request of n_tokens tokens occupies in `mode` under this config (the
 * allocation rule of hc_append: KV takes a K and a V unit per B tokens, hidden one unit per
 * B tokens; under GQA KV takes one unit per Bkv tokens, see n_kv_heads).  For sizing pools.  Returns -1 for an invalid config/mode or
 * n_tokens < 0.  Host only. */
int64_t hc_units_needed(const hc_pool_config* cfg, int32_t mode, int64_t n_tokens);

/* Create a pool ("unified block-wise memory pool").  Zero-fills the block
 * region (so padding rows of a partly filled block are finite), copies W_KV / b_KV into
 * storage, and builds TMA descriptors.  Synchronous w.r.t. the device (cudaDeviceSynchronize
 * on cfg->device).  Errors: HC_E_INVALID (null / inconsistent sizes, storage too small),
 * HC_E_UNSUPPORTED (shape not implemented), HC_E_CUDA. */
hc_status hc_pool_create(const hc_pool_config* cfg, hc_pool** out);

/* Destroy; does not free caller-owned device memory.  NULL is a no-op. */
void hc_pool_destroy(hc_pool* pool);

/* Append tokens (hidden-cache I/O; cache-map creation/extension).
 * For each of the n_req DISTINCT requests, n_tokens[i] >= 0 new tokens are appended at
 * the end of its cache in mode modes[i] (a new id is created with that mode).  Rows are
 * device buffers packed in request order: `k`, `v` hold [sum over KV-mode requests of
 * n_tokens, Dk]; `x` holds [sum over hidden-mode requests of n_tokens, d] (token-major,
 * row-major).  Either of k/v or x may be NULL if no request of that mode is present.
 * Block allocation: SPEC memory-pool contract — unit blocks, KV takes a K and a V block
 * per B tokens, hidden one, new blocks only when the last is full,
 * lowest free id first, K before V per logical block, requests in call order,
 * ALL-OR-NOTHING over the whole call.  Errors: HC_E_INVALID, HC_E_OOM,
 * HC_E_MODE_MISMATCH (pool unchanged), HC_E_CUDA.  Asynchronous on `stream`; host
 * buffers k/v/x are NOT accepted. */
hc_status hc_append(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                    const int32_t* n_tokens, const void* k, const void* v, const void* x,
                    void* stream);

/* Discard a request's cache (cache-type switch = discard + recompute).
 * Unknown ids are an idempotent no-op.  *released_units (nullable) = unit blocks freed. */
hc_status hc_free(hc_pool* pool, int64_t req_id, int64_t* released_units);

/* Workspace bytes hc_decode_attention needs for this batch (descriptor, split partials,
 * reconstructed-K/V scratch).  Returns 0 on invalid input (see hc_last_error). */
size_t hc_workspace_size(const hc_pool* pool, int32_t n_req, const int64_t* req_ids);

/* One decode-step attention layer over the hybrid cache (Eq. 1-3).
 *   req_ids  host [n_req], distinct, known, each with n_i >= 1 (current token appended).
 *   q        device [n_req, d] pool dtype, row i = query of req_ids[i].
 *   scale    softmax scale (Eq. 2 uses 1/sqrt(d) for one head; multi-head 1/sqrt(dh), R1).
 *   out      device [n_req, d] pool dtype: concat_h sum_j a_j v_{j,h} (pre-W_o).
 *   lse      nullable device [n_req, H] fp32: log sum_j exp(scale q_h.k_j) (natural log).
 *   workspace device, >= hc_workspace_size() bytes, 256-B aligned.
 * Hidden-mode K/V are rebuilt by a tcgen05 GEMM (bf16 in, fp32 accumulate in TMEM) whose
 * epilogue attends them straight from TMEM (fp32, never stored; HC_EPI_ATTEND=0 restores
 * the bf16 scratch path), while KV-mode requests stream through the same persistent
 * kernel's split-K flash-decoding warps; a split combine then writes out and lse.  n_req = 0 is HC_OK and launches nothing.  Errors: HC_E_INVALID,
 * HC_E_UNKNOWN_REQ, HC_E_WORKSPACE, HC_E_UNSUPPORTED, HC_E_CUDA.
 * CUDA graphs: the call may be stream-captured (relaxed capture mode).  The descriptor is
 * built on the host at capture time and its pinned staging buffer is retired from the
 * runtime's 16-slot ring, so every replay recomputes exactly the captured batch (same
 * ids, tables, q/out/lse/workspace pointers) until hc_pool_destroy; appends after the
 * capture are not seen by replays.  HC_E_CUDA once all 16 slots are held by captures. */
hc_status hc_decode_attention(hc_pool* pool, int32_t n_req, const int64_t* req_ids,
                              const void* q, float scale, void* out, float* lse,
                              void* workspace, size_t ws_bytes, void* stream);

/* ---- the rest of the attention module (NEXT row f1) --------------------------------- */
/* Current-token projections and cache append for one decode step: Eq. 1 for the new token
 * fused with the block-wise cache write (the paper's I/O kernel).
 *   x      device [n_req, d]: layer input of each request's current token.
 *   q_out  device [n_req, d]: q = W_Q x (+ b_Q), for every request.
 * KV-mode requests: k = W_K x (+b_K), v = W_V x (+b_V) are written by the GEMM epilogue
 * straight into the request's cache slot (one [H][B][dh] row per head).  Hidden-mode
 * requests: x itself is appended (their K/V are rebuilt at attention time).  Each
 * request gains one token; allocation, modes and errors as hc_append (new ids allowed).
 * Needs the pool's w_q.  Asynchronous on `stream`. */
hc_status hc_project_append(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                            const void* x, void* q_out, void* stream);
/* u = LN(x) with the pool's ln_gamma / ln_beta / ln_eps (population variance over d,
 * fp32 statistics): x, u device [n_rows, d] pool dtype (may alias).  HC_E_UNSUPPORTED if
 * the pool has no LayerNorm.  hc_project_append takes the normalised input. */
hc_status hc_layer_norm(hc_pool* pool, int32_t n_rows, const void* x, void* u, void* stream);
/* Cross-partition merge (SURVEY §8(e) phase 2; Eq. 2-3 over a union of token ranges).
 * A request whose tokens are split over n_parts partitions (e.g. ranks that each hold part
 * of a long request's blocks and each ran hc_decode_attention on their part) has per-part
 * results out_p (normalised within the part) and lse_p (natural log).  This writes
 *   lse = log sum_p e^{lse_p},  out = sum_p e^{lse_p - lse} out_p.
 *   outs  device [n_parts][n_rows][n_heads * head_dim], dtype (the gathered part outputs)
 *   lses  device [n_parts][n_rows][n_heads] fp32; -inf marks an empty part (weight 0)
 *   out   device [n_rows][n_heads * head_dim] dtype;  lse nullable device [n_rows][n_heads]
 * A row whose parts are all empty gets out = 0, lse = -inf.  No pool: buffers are the
 * caller's.  Errors: HC_E_INVALID (sizes, dtype, null pointers), HC_E_CUDA.  Asynchronous
 * on `stream`. */
hc_status hc_merge_partials(int32_t n_parts, int32_t n_rows, int32_t n_heads, int32_t head_dim, hc_dtype dtype,
                            const void* outs, const float* lses, void* out, float* lse, void* stream);
/* y = W_O o (+ b_O): the output map of Eq. 3.  o, y device [n_req, d]. */
hc_status hc_output_projection(hc_pool* pool, int32_t n_req, const void* o, void* y, void* stream);
/* One attention layer for one decode step: [hc_layer_norm,] hc_project_append,
 * hc_decode_attention, hc_output_projection in sequence.  `workspace` >= hc_layer_workspace_size() bytes,
 * sized for the batch AFTER the current token is appended (unknown ids count as n = 1).
 * lse (nullable) as hc_decode_attention. */
size_t hc_layer_workspace_size(const hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes);
hc_status hc_decode_layer(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                          const void* x, float scale, void* y, float* lse, void* workspace, size_t ws_bytes,
                          void* stream);

/* Prefill (or recompute after preemption / a cache-type switch: P:297 fn) of one
 * attention layer for NEW requests (unknown ids or ids with 0 cached tokens).
 *   lens  host [n_req], >= 1 tokens per request; x device [sum lens, d], rows packed in
 *         request order (the layer inputs of the prompt tokens, or of prompt + generated
 *         tokens for a recompute).
 * Projects q, k, v for every token (Eq. 1) in one tcgen05 GEMM whose epilogue also writes
 * the cache (KV mode: k, v rows; hidden mode: x rows are appended), runs causal attention
 * over each request's tokens (Eq. 2-3 with j <= i) and the output map:
 *   y device [sum lens, d] = W_O o (+ b_O).
 * Needs w_q and w_o.  workspace >= hc_prefill_workspace_size().  Errors as hc_append, plus
 * HC_E_INVALID for a request that already holds tokens. */
size_t hc_prefill_workspace_size(const hc_pool* pool, int32_t n_req, const int32_t* lens);
hc_status hc_prefill_layer(hc_pool* pool, int32_t n_req, const int64_t* req_ids, const int32_t* modes,
                           const int32_t* lens, const void* x, float scale, void* y, void* workspace,
                           size_t ws_bytes, void* stream);

/* ---- adaptive scheduler (host only; NEXT row f2; §4.2, §5) ---- */
typedef struct {
  double rho;            /* seconds of extra projection time per memory unit (Eq. 6, t = rho m) */
  double total_units;    /* M~: pool capacity in memory units */
  double ttft_slo;       /* seconds; a waiting request with p > ttft_slo has violated its SLO (<= 0: never) */
  double tbt_slo;        /* seconds; a running request with p > tbt_slo has violated its SLO (<= 0: never) */
  int32_t fallback;      /* SLO-aware fallback: 0 = near-zero constant eps, 1 = decay factor */
  double eps;            /* near-zero value (default 1e-6 s) */
  double decay;          /* decay factor (0.4 in §6.5) */
  int32_t hybrid;        /* 1: hidden cache allowed; 0: KV-only ablation */
  int32_t block_size;    /* memory unit granularity: a KV request of L tokens needs 2*ceil(L/B) units (B=1: tokens) */
} hc_sched_config;

typedef struct {
  int64_t id;
  int32_t running;         /* 1: in the running queue R^e (decode phase, cache resident); 0: waiting W^e */
  int32_t has_token;       /* has received an output token (pending time since the last token) */
  double arrival_time;     /* seconds */
  double last_token_time;  /* seconds (used when has_token) */
  int64_t seq_len;         /* tokens cached (running) or to prefill (waiting: prompt + generated, P:297 fn) */
} hc_sched_request;

typedef struct {
  int32_t iter_type;       /* 0 decode, 1 prefill, -1 idle (both queues empty) */
  int32_t n_candidates;    /* |U^e| */
  double budget;           /* M^e (Eq. 7 right-hand side) */
  double objective;        /* sum_i g_i alpha_i (Definition 1) */
  double memory_used;      /* sum_i (1 - beta_i/2) m_i alpha_i */
} hc_sched_result;

/* One scheduling decision for iteration e at time `now`.  Tracks p_i and m_i
 * (m_i = KV units of seq_len + 1, the token produced this iteration), picks the
 * iteration type by the larger cumulative pending time (ties -> decode), the candidate set
 * U^e and budget M^e, values g_i = p_i - beta_i (|W|+|R|) rho m_i (Eq. 5-6) with the
 * SLO fallback applied to p_i, then the marginal-gain greedy (hidden / upgrade /
 * direct-KV stages, refinement when p/m < 2 N rho; ties theta desc, delta-m asc, request id asc)
 * compared against the best single feasible assignment (KV or hidden; R14).
 * alpha[i], beta[i] (n each, host) receive the decision for every input request (0 for
 * requests outside U^e); g (nullable) receives each candidate's value at its decided beta.
 * Pure host computation; errors: HC_E_INVALID. */
hc_status hc_schedule(const hc_sched_config* cfg, int32_t n, const hc_sched_request* reqs, double now,
                      int32_t* alpha, int32_t* beta, double* g, hc_sched_result* result);
/* Least-squares slope through the origin, rho = sum m t / sum m^2 (the "approximately 30
 * seconds" pre-serving fit of Eq. 6).  Returns -1 if n < 1 or all m are 0. */
double hc_calibrate_rho(int32_t n, const double* m, const double* t);

/* ---- introspection (host-side, no device work) ------------------------------------ */
int64_t hc_pool_num_free(const hc_pool* pool);
/* mode (hc_mode), cached tokens and unit blocks of a request; HC_E_UNKNOWN_REQ if absent */
hc_status hc_request_info(const hc_pool* pool, int64_t req_id, int32_t* mode, int64_t* n_tokens,
                          int64_t* n_units);
/* block ids of a request's cache map: kind 0 = K (or X for hidden; under GQA the
 * unit holding K and V), 1 = V (empty under GQA).
 * Writes min(count, cap) ids to out; *count = list length. */
hc_status hc_request_blocks(const hc_pool* pool, int64_t req_id, int32_t kind, int32_t* out,
                            int64_t cap, int64_t* count);

/* ---- measurement hooks --------------------------------------------------------------- */
/* Kernels launched by the last hc_decode_attention / hc_append call on this pool. */
int32_t hc_last_launch_count(const hc_pool* pool);
/* Kernel path of the last hc_decode_attention: 0 = reconstruction GEMM + attention kernels,
 * 1 = fused step kernel (GEMM and attention warps in one launch), 2 = attention only (no
 * hidden-mode request), 3 = absorbed hidden attention (HC_FLAG_ABSORB_HIDDEN), -1 = none. */
int32_t hc_last_decode_path(const hc_pool* pool);
/* Fused step kernel configuration of the last hc_decode_attention (path 1): decimal digits
 * {GEMM stages, attention warps, attention stages[, extra epilogue warps]} — 352, 282, 342,
 * 3424, 3224 (10000 + cfg for 256-wide tiles); 0 when no fused kernel ran. */
int32_t hc_last_kernel_config(const hc_pool* pool);
/* When enabled, hc_decode_attention records CUDA events around each of its kernels on
 * the stream it launches them on.  hc_kernel_times() synchronises on all events recorded
 * since the previous read and returns, summed over those calls, the milliseconds of
 * [0] reconstruction GEMM, [1] attention, [2] combine, [3] descriptor upload, plus the
 * number of calls in *n_calls; then it clears the record. */
hc_status hc_set_profiling(hc_pool* pool, int32_t enable);
hc_status hc_kernel_times(hc_pool* pool, float* ms4, int32_t* n_calls);

const char* hc_last_error(void);
const char* hc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HC_H_ */
