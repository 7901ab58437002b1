// CTA-pair (cta_group::2) tcgen05 reconstruction GEMM roles, shared by the stand-alone
// reconstruction kernel (recon_tc.cu) and the fused step kernel (fused.cu).
//
//   [K || V] = X W_KV^T (+ b)        Eq. 1 applied to every cached x_j
//
// A CTA pair computes a 256 x (256*NSUB) tile.  CTA rank r loads A rows [r*128, r*128+128)
// of the 256-row M tile (one TMA box per hidden block: the block-wise hidden cache IS the
// A operand) and, for each 256-wide N sub-tile j, W_int rows [j*256 + r*128, +128); the
// leader issues M=256 N=256 K=16 UMMAs that read both CTAs' smem; each CTA's TMEM holds its
// own 128 rows x 256*NSUB fp32 columns.  Warp roles (192 threads):
//   warp 0  TMA producer (both CTAs; bytes counted on the leader's full barrier)
//   warp 1  TMEM allocator (both CTAs) and single-thread MMA issuer (leader only)
//   warps 2-5  epilogue: tcgen05.ld -> (+bias) -> bf16 RNE -> scratch [hblock][H][B][dh]
// Schedule: n-major raster (2 n-tiles per group) — pairs p and p^1 of a wave share an A
// panel, every wave shares the group's W panels — plus a partner k-progress lockstep that
// keeps p and p^1 within `sync_w` k-steps so the second reader of A hits in L2.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace hc {
namespace pg {

constexpr int BK = 64, BN = 256, P_BM = 256;
constexpr int P_A_BYTES = 128 * BK * 2;   // this CTA's half of A: 16 KiB
constexpr int P_B_BYTES = 128 * BK * 2;   // this CTA's half of one 256-wide B sub-tile: 16 KiB
constexpr int TMEM_COLS = 512;
constexpr int GEMM_THREADS = 192;
constexpr int kMaxSyncPairs = 80;         // progress words reserved in the workspace header

struct TcArgs {
  const int32_t* gather;
  int32_t n_hblocks, M, B, rows_per_box;
  int32_t runs;             // 1: fetch runs of consecutive pool blocks as one 128-row box (tmap_x128)
  int32_t m_tiles, n_tiles, k_iters;
  int32_t H, dh, d;         // H: K/V heads of the GEMM's K||V columns (= query heads unless GQA)
  int32_t grp;              // query heads per K/V head (GQA, R18; 1 = multi-head)
  int32_t dk, Bkv;          // EPI_PROJECT: K/V row width, tokens per KV logical block
  int64_t v_off;            // EPI_PROJECT: V rows' offset inside their unit (GQA: K, V share one)
  __nv_bfloat16* scr_k;
  __nv_bfloat16* scr_v;
  const float* bias;
  int32_t group_m;      // raster group (m-tiles sweeping all n-tiles); < 0: n-major, -group_m n-tiles
  int32_t l2_hint;      // 0 none, 1 A evict_last + W evict_first, 2 the reverse, 3 A normal + W evict_last
  int32_t* sync;        // zeroed per-pair progress words (stride 32 ints), nullptr = off
  int32_t sync_w;       // partner lockstep window in k-steps
  int32_t* tile_done;   // nullable: per (m-tile, n-tile) count of finished epilogue warps (8 = ready)
  // ---- epilogue routing (EPI_* below) and dense-A mode
  int32_t epi;          // EPI_SCRATCH (reconstruction), EPI_PROJECT (q + KV-cache write), EPI_DENSE
  int32_t n_total;      // output columns (EPI_DENSE / EPI_PROJECT), = n_tiles * TILE_N
  __nv_bfloat16* out;   // EPI_DENSE: [M, n_total];  EPI_PROJECT: q [M, d]
  __nv_bfloat16* pool;  // EPI_PROJECT: unit blocks
  const int32_t* row_dst;  // EPI_PROJECT: per row {K block, V block, slot} (K block < 0: hidden row)
  __nv_bfloat16* kvbuf;    // EPI_PROJECT (prefill): also every row's head-interleaved K||V, [M, 2d]
  // RoPE (NEXT row f4): rotate K (and q) columns at each row's token position
  const double* rope_inv;  // nullable: inv_freq[c] = theta^(-2c/dh), c < dh/2
  const int32_t* row_pos;  // EPI_SCRATCH / EPI_ATTEND: position of row 0 of each hidden block (lb * B)
  // EPI_ATTEND (fused reconstruct-and-attend)
  const int32_t* hblk_req;  // batch index of each hidden block's request
  const ReqDesc* reqs;
  const __nv_bfloat16* q;   // [n_req, d]
  float* part_ml;           // [H*grp][n_splits_all][2]  (query heads)
  float* part_acc;          // [H*grp][n_splits_all][dh]
  int32_t n_splits_all;
  float scale_log2;
  int32_t seg;              // tokens per partial (8, 16 or 32; segments never straddle a block)
  int32_t epi_split;        // epilogue warps per TMEM lane quarter (1, or 2 with the fused kernel's extra
                            // epilogue warps: each takes every other head / column chunk)
  int32_t diag;             // -DHC_DIAG builds only (HC_DIAG_EPI): timing diagnostics with wrong outputs
  int32_t* tile_counter;    // nullable: zeroed per launch; tiles handed out dynamically (see pair_roles)
  int32_t epi_mma;          // EPI_ATTEND on mma.sync (attend_tile_mma): dh = 128, no RoPE, seg 16 or 32
};

// Epilogue modes.  gather == nullptr means dense A rows (row = m index, no block gather).
constexpr int EPI_SCRATCH = 0;   // [K||V] rows -> scratch blocks [hblock][H][B][dh]
constexpr int EPI_PROJECT = 1;   // cols [0,d): q row; cols [d,3d) (head-interleaved K||V) -> cache slot
constexpr int EPI_DENSE = 2;     // plain row-major C
constexpr int EPI_ATTEND = 3;    // [K||V] rows -> per-(segment, head) flash-decoding partials

template <int NSUB, int NSTAGE>
struct PairCfg {
  static constexpr int STAGE_BYTES = P_A_BYTES + NSUB * P_B_BYTES;
  static constexpr int STAGES = NSTAGE;
  static constexpr int NACC = 2 / NSUB;   // accumulator buffers in the 512 TMEM columns
  static constexpr int TILE_N = 256 * NSUB;
  static constexpr int REGION_BYTES = STAGES * STAGE_BYTES + 512;   // stages + barriers (1024-aligned base)
};

__device__ __forceinline__ void tile_coords_p(int t, int m_tiles, int n_tiles, int group_m, int& mt, int& nt) {
  if (group_m < 0) {  // n-major raster: -group_m n-tiles sweep all m-tiles
    const int gn = -group_m;
    const int per_group = gn * m_tiles;
    const int g = t / per_group;
    const int first_n = g * gn;
    const int gsize = min(gn, n_tiles - first_n);
    const int r = t - g * per_group;
    nt = first_n + r % gsize;
    mt = r / gsize;
    return;
  }
  const int per_group = group_m * n_tiles;
  const int g = t / per_group;
  const int first_m = g * group_m;
  const int gsize = min(group_m, m_tiles - first_m);
  const int r = t - g * per_group;
  mt = first_m + r % gsize;
  nt = r / gsize;
}

__device__ __forceinline__ void st_relaxed(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_relaxed(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int32_t* p, int32_t v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- epilogue helpers ------------------------------------------------------------------
__device__ __forceinline__ void load_chunk(uint32_t taddr, const float* bias, int n, float (&f)[32]) {
  uint32_t v[32];
  ptx::tmem_ld_32x32b_x32(taddr, v);
  ptx::tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
  if (bias) {
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] += __ldg(bias + n + j);
  }
}

// Rotate 32 (x, y) pairs = columns (c, c + dh/2) by angle pos * inv_freq[c] (NeoX / LLaMA
// "rotate_half" convention).  The angle is reduced modulo 2 pi in fp64 so long positions
// keep full fp32 accuracy in the sine and cosine.
__device__ __forceinline__ void rope_rotate(float (&x)[32], float (&y)[32], int pos, const double* inv) {
  constexpr double kTwoPi = 6.283185307179586476925286766559;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double ang = (double)pos * __ldg(inv + j);
    const double k = rint(ang * (1.0 / kTwoPi));
    const float th = (float)fma(-k, kTwoPi, ang);
    float sn, cs;
    __sincosf(th, &sn, &cs);
    const float x0 = x[j], y0 = y[j];
    x[j] = x0 * cs - y0 * sn;
    y[j] = y0 * cs + x0 * sn;
  }
}

__device__ __forceinline__ void store_chunk(const TcArgs& a, int n, const float (&f)[32], int grow, int g, int r,
                                            const int4& dst_info) {
  __nv_bfloat16* dst = nullptr;
  __nv_bfloat16* dst2 = nullptr;
  if (a.epi == EPI_SCRATCH) {
    const int h = n / (2 * a.dh), rem = n - h * 2 * a.dh, kv = rem / a.dh, c0 = rem - kv * a.dh;
    dst = (kv ? a.scr_v : a.scr_k) + (((size_t)g * a.H + h) * a.B + r) * a.dh + c0;
  } else if (a.epi == EPI_DENSE) {
    dst = a.out + (size_t)grow * a.n_total + n;
  } else {  // EPI_PROJECT
    if (n < a.d) {
      dst = a.out + (size_t)grow * a.d + n;
    } else {
      const int m = n - a.d;
      if (dst_info.x >= 0) {
        const int h = m / (2 * a.dh), rem = m - h * 2 * a.dh, kv = rem / a.dh, c0 = rem - kv * a.dh;
        const int blk = kv ? dst_info.y : dst_info.x;
        dst = a.pool + (size_t)blk * a.B * a.d + (kv ? a.v_off : 0) + (size_t)h * a.Bkv * a.dh +
              (size_t)dst_info.z * a.dh + c0;
      }
      if (a.kvbuf) dst2 = a.kvbuf + (size_t)grow * 2 * a.dk + m;
    }
  }
  if (dst == nullptr && dst2 == nullptr) return;
  uint4 pk[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    pk[j] = make_uint4(pack_bf16(f[8 * j], f[8 * j + 1]), pack_bf16(f[8 * j + 2], f[8 * j + 3]),
                       pack_bf16(f[8 * j + 4], f[8 * j + 5]), pack_bf16(f[8 * j + 6], f[8 * j + 7]));
  if (dst != nullptr) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int j = 0; j < 4; ++j) d4[j] = pk[j];
  }
  if (dst2 != nullptr) {
    uint4* d4 = reinterpret_cast<uint4*>(dst2);
#pragma unroll
    for (int j = 0; j < 4; ++j) d4[j] = pk[j];
  }
}


// ---- EPI_ATTEND: fused reconstruct-and-attend -------------------------------------------
constexpr unsigned kFull = 0xffffffffu;

// Butterfly reduce-scatter over the S lanes of a segment: on return lane i (= lane % S)
// holds in x[0 .. 32/S) the segment sums of columns [i*32/S, (i+1)*32/S) of its chunk.
template <int OFF, int CNT>
struct SegReduceScatter {
  static __device__ __forceinline__ void run(float* x, int lane) {
    constexpr int HALF = CNT / 2;
    const bool up = (lane & OFF) != 0;
#pragma unroll
    for (int i = 0; i < HALF; ++i) {
      const float send = up ? x[i] : x[i + HALF];
      const float keep = up ? x[i + HALF] : x[i];
      x[i] = keep + __shfl_xor_sync(kFull, send, OFF);
    }
    SegReduceScatter<OFF / 2, HALF>::run(x, lane);
  }
};
template <int CNT>
struct SegReduceScatter<0, CNT> {
  static __device__ __forceinline__ void run(float*, int) {}
};

// q chunk (32 bf16) for a dot with a TMEM chunk: loaded BEFORE the tcgen05.ld so the L1/L2
// latency overlaps the TMEM load; four independent FMA chains (chain length 8, not 32).
__device__ __forceinline__ void load_q32(const __nv_bfloat16* q, uint4 (&u)[4]) {
  const uint4* q4 = reinterpret_cast<const uint4*>(q);
#pragma unroll
  for (int j = 0; j < 4; ++j) u[j] = __ldg(q4 + j);
}
__device__ __forceinline__ float dot32_q(const float (&f)[32], const uint4 (&u)[4]) {
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u[j]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 v = __bfloat1622float2(b[e]);
      s[e] = fmaf(f[8 * j + 2 * e], v.x, s[e]);
      s[e] = fmaf(f[8 * j + 2 * e + 1], v.y, s[e]);
    }
  }
  return (s[0] + s[1]) + (s[2] + s[3]);
}

// One pair tile's rows -> partials.  Thread = GEMM row (a token of a hidden block); the
// tile's columns are HT = TILE_N / (2 dh) K/V heads of K_hk || V_hk, each serving grp query
// heads (GQA, R18).  Per query head: s = scale * q_h . k (bias and RoPE applied to k in
// registers), segment max / sum over the S lanes of the segment, and the segment's
// sum_j p_j v_j by a butterfly reduce-scatter; lane i of the segment writes dims
// [i*32/S, (i+1)*32/S) of every 32-column chunk.  Rows past M and tokens past n get p = 0;
// a segment that starts past n writes nothing.
template <int S, int TILE_N, int NSPLIT = 1>
__device__ __forceinline__ void attend_tile(const TcArgs& a, uint32_t tacc, int nt, int grow, int lane, int sub) {
  const bool valid = grow < a.M;
  int req = 0, tok = 0, n = 0;
  if (valid) {
    const int g = grow / a.B;
    req = a.hblk_req[g];
    tok = a.row_pos[g] + (grow - g * a.B);
    n = a.reqs[req].n;
  }
  const bool live = valid && tok < n;
  const int tok0 = tok - (lane & (S - 1));   // first token of this lane's segment
  const bool seg_live = valid && tok0 < n;
  const int split = valid ? a.reqs[req].split_begin + tok0 / S : 0;
  const int dh = a.dh, HT = TILE_N / (2 * dh);
#pragma unroll 1
  for (int jg = sub; jg < HT * a.grp; jg += NSPLIT) {
    const int j = jg / a.grp;                     // K/V head of the tile
    const int h = (nt * HT + j) * a.grp + (jg - j * a.grp);   // query head
    const int nk = nt * TILE_N + j * 2 * dh;      // interleaved column of K_hk (bias index)
    const uint32_t tk = tacc + j * 2 * dh;
    const __nv_bfloat16* qh = a.q + (size_t)req * a.d + h * dh;
    float s = 0.f;
    if (a.rope_inv != nullptr) {
#pragma unroll 1
      for (int c0 = 0; c0 < dh / 2; c0 += 32) {
        uint4 qa[4], qb[4];
        load_q32(qh + c0, qa);
        load_q32(qh + c0 + dh / 2, qb);
        float f[32], f2[32];
        load_chunk(tk + c0, a.bias, nk + c0, f);
        load_chunk(tk + c0 + dh / 2, a.bias, nk + c0 + dh / 2, f2);
        rope_rotate(f, f2, tok, a.rope_inv + c0);
        s += dot32_q(f, qa) + dot32_q(f2, qb);
      }
    } else {
#pragma unroll 1
      for (int c0 = 0; c0 < dh; c0 += 32) {
        uint4 qa[4];
        load_q32(qh + c0, qa);
        float f[32];
        load_chunk(tk + c0, a.bias, nk + c0, f);
        s += dot32_q(f, qa);
      }
    }
    s = live ? s * a.scale_log2 : -INFINITY;
    float m = s;
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
    const float p = live ? exp2f(s - m) : 0.f;
    float l = p;
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
    const size_t task = (size_t)h * a.n_splits_all + split;   // head-major partial index
#pragma unroll 1
    for (int c0 = 0; c0 < dh; c0 += 32) {
      float f[32];
      load_chunk(tk + dh + c0, a.bias, nk + dh + c0, f);
#pragma unroll
      for (int e = 0; e < 32; ++e) f[e] *= p;
      SegReduceScatter<S / 2, 32>::run(f, lane);
      if (seg_live) {
        float* dst = a.part_acc + task * dh + c0 + (lane & (S - 1)) * (32 / S);
        if constexpr (S == 32) {
          dst[0] = f[0];
        } else if constexpr (S == 16) {
          *reinterpret_cast<float2*>(dst) = make_float2(f[0], f[1]);
        } else {
          *reinterpret_cast<float4*>(dst) = make_float4(f[0], f[1], f[2], f[3]);
        }
      }
    }
    if (seg_live && (lane & (S - 1)) == 0) {
      a.part_ml[2 * task] = m;
      a.part_ml[2 * task + 1] = l;
    }
  }
}

// GQA, grp even: the query heads of a K/V head are taken two at a time — every K and V
// chunk comes out of TMEM once per pair, and the two heads' dot products, softmax shuffles
// and Σ p·v reduce-scatters are independent chains the scheduler interleaves (the epilogue
// of a GQA tile is latency-bound: the per-head loop runs them back to back).
template <int S, int TILE_N, int NSPLIT>
__device__ __forceinline__ void attend_tile_gqa2(const TcArgs& a, uint32_t tacc, int nt, int grow, int lane, int sub) {
  const bool valid = grow < a.M;
  int req = 0, tok = 0, n = 0;
  if (valid) {
    const int g = grow / a.B;
    req = a.hblk_req[g];
    tok = a.row_pos[g] + (grow - g * a.B);
    n = a.reqs[req].n;
  }
  const bool live = valid && tok < n;
  const int tok0 = tok - (lane & (S - 1));
  const bool seg_live = valid && tok0 < n;
  const int split = valid ? a.reqs[req].split_begin + tok0 / S : 0;
  const int dh = a.dh, HT = TILE_N / (2 * dh);
#pragma unroll 1
  for (int jg = 2 * sub; jg < HT * a.grp; jg += 2 * NSPLIT) {
    const int j = jg / a.grp;
    const int h = (nt * HT + j) * a.grp + (jg - j * a.grp);   // query heads h, h + 1
    const int nk = nt * TILE_N + j * 2 * dh;
    const uint32_t tk = tacc + j * 2 * dh;
    const __nv_bfloat16* qh0 = a.q + (size_t)req * a.d + (size_t)h * dh;
    const __nv_bfloat16* qh1 = qh0 + dh;
    float s0 = 0.f, s1 = 0.f;
    if (a.rope_inv != nullptr) {
#pragma unroll 1
      for (int c0 = 0; c0 < dh / 2; c0 += 32) {
        uint4 qa0[4], qb0[4], qa1[4], qb1[4];
        load_q32(qh0 + c0, qa0);
        load_q32(qh0 + c0 + dh / 2, qb0);
        load_q32(qh1 + c0, qa1);
        load_q32(qh1 + c0 + dh / 2, qb1);
        float f[32], f2[32];
        load_chunk(tk + c0, a.bias, nk + c0, f);
        load_chunk(tk + c0 + dh / 2, a.bias, nk + c0 + dh / 2, f2);
        rope_rotate(f, f2, tok, a.rope_inv + c0);
        s0 += dot32_q(f, qa0) + dot32_q(f2, qb0);
        s1 += dot32_q(f, qa1) + dot32_q(f2, qb1);
      }
    } else {
#pragma unroll 1
      for (int c0 = 0; c0 < dh; c0 += 32) {
        uint4 qa0[4], qa1[4];
        load_q32(qh0 + c0, qa0);
        load_q32(qh1 + c0, qa1);
        float f[32];
        load_chunk(tk + c0, a.bias, nk + c0, f);
        s0 += dot32_q(f, qa0);
        s1 += dot32_q(f, qa1);
      }
    }
    s0 = live ? s0 * a.scale_log2 : -INFINITY;
    s1 = live ? s1 * a.scale_log2 : -INFINITY;
    float m0 = s0, m1 = s1;
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) {
      m0 = fmaxf(m0, __shfl_xor_sync(kFull, m0, o));
      m1 = fmaxf(m1, __shfl_xor_sync(kFull, m1, o));
    }
    const float p0 = live ? exp2f(s0 - m0) : 0.f, p1 = live ? exp2f(s1 - m1) : 0.f;
    float l0 = p0, l1 = p1;
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) {
      l0 += __shfl_xor_sync(kFull, l0, o);
      l1 += __shfl_xor_sync(kFull, l1, o);
    }
    const size_t task0 = (size_t)h * a.n_splits_all + split, task1 = task0 + a.n_splits_all;
#pragma unroll 1
    for (int c0 = 0; c0 < dh; c0 += 32) {
      float v[32];
      load_chunk(tk + dh + c0, a.bias, nk + dh + c0, v);
      float f0[32], f1[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        f0[e] = v[e] * p0;
        f1[e] = v[e] * p1;
      }
      SegReduceScatter<S / 2, 32>::run(f0, lane);
      SegReduceScatter<S / 2, 32>::run(f1, lane);
      if (seg_live) {
        const int off = c0 + (lane & (S - 1)) * (32 / S);
        float* d0 = a.part_acc + task0 * dh + off;
        float* d1 = a.part_acc + task1 * dh + off;
        if constexpr (S == 32) {
          d0[0] = f0[0];
          d1[0] = f1[0];
        } else if constexpr (S == 16) {
          *reinterpret_cast<float2*>(d0) = make_float2(f0[0], f0[1]);
          *reinterpret_cast<float2*>(d1) = make_float2(f1[0], f1[1]);
        } else {
          *reinterpret_cast<float4*>(d0) = make_float4(f0[0], f0[1], f0[2], f0[3]);
          *reinterpret_cast<float4*>(d1) = make_float4(f1[0], f1[1], f1[2], f1[3]);
        }
      }
    }
    if (seg_live && (lane & (S - 1)) == 0) {
      a.part_ml[2 * task0] = m0;
      a.part_ml[2 * task0 + 1] = l0;
      a.part_ml[2 * task1] = m1;
      a.part_ml[2 * task1 + 1] = l1;
    }
  }
}

// Attend epilogue on mma.sync (dh = 128; default for GQA).  Per 16 rows (tokens) of
// the warp's TMEM lane quarter and per K/V head of the tile:
//   S = K Q^T   m16n8k16 over dh: the K rows come out of a tcgen05.ld.16x256b load already in
//               the A-fragment order (+ bias, split into bf16 hi + lo terms: two MMAs, scores as
//               accurate as the fp32 path); Q^T of the segment's request (its G <= 8 query
//               heads) is the B operand
//   softmax per query head over the segment's tokens (3 shuffle levels), p rounded to bf16
//   O = P^T V   P^T re-laid from the score fragment by 4 shuffles + prmt (A operand, rows =
//               query heads); V's B fragments are the 16x256b load transposed by movmatrix
// A segment (S tokens, never straddling a block) becomes one (m, l, acc[dh]) partial per query
// head, as in attend_tile.  V is rounded to bf16 here (the per-row path keeps fp32).
template <int S, int TILE_N, int NSPLIT>
__device__ __forceinline__ void attend_tile_mma(const TcArgs& a, uint32_t tq, int nt, int row0, int lane, int sub) {
  constexpr int DH = 128;
  constexpr int HT = TILE_N / (2 * DH);
  constexpr int NG = S / 16;   // 16-row groups per segment
  static_assert(S == 16 || S == 32, "segments of 16 or 32 tokens");
  const int g = lane >> 2, t = lane & 3;
  const int G = a.grp;
  const uint32_t sel = (g & 1) ? 0x7632u : 0x5410u;
  const int srcA = 4 * (2 * t) + (g >> 1), srcB = 4 * (2 * t + 1) + (g >> 1);
#pragma unroll 1
  for (int j = sub; j < HT; j += NSPLIT) {
    const int hk = nt * HT + j;
    const int nk = nt * TILE_N + j * 2 * DH;   // bias column of K_hk; V_hk at + DH
    const uint32_t tk = tq + j * 2 * DH;
#pragma unroll 1
    for (int sg = 0; sg < 32 / S; ++sg) {
      const int r_seg = row0 + sg * S;   // first row of the segment (warp-uniform)
      if (r_seg >= a.M) continue;
      const int blk = r_seg / a.B;
      const int req = a.hblk_req[blk];
      const int tok0 = a.row_pos[blk] + (r_seg - blk * a.B);
      const int n = a.reqs[req].n;
      if (tok0 >= n) continue;   // a segment past n writes nothing
      const bool qv = g < G;
      const __nv_bfloat16* qh = a.q + (size_t)req * a.d + (size_t)(hk * G + (qv ? g : 0)) * DH;
      uint32_t qb[8][2];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qb[kk][0] = qv ? __ldg(reinterpret_cast<const uint32_t*>(qh + 16 * kk + 2 * t)) : 0u;
        qb[kk][1] = qv ? __ldg(reinterpret_cast<const uint32_t*>(qh + 16 * kk + 8 + 2 * t)) : 0u;
      }
      // ---- scores
      float sc[NG][4];
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) {
        sc[gi][0] = sc[gi][1] = sc[gi][2] = sc[gi][3] = 0.f;
        const uint32_t tg = tk + ((uint32_t)(16 * (sg * NG + gi)) << 16);
        // slices kk and kk + 4 hold columns c and c + 64 = the RoPE partners (dh = 128)
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {   // 4 k-slices per TMEM wait
          uint32_t r[4][8];
          const int ks[4] = {2 * kb, 2 * kb + 1, 2 * kb + 4, 2 * kb + 5};
#pragma unroll
          for (int i = 0; i < 4; ++i) ptx::tmem_ld_16x256b_x2(tg + 16 * ks[i], r[i]);
          ptx::tmem_ld_wait();
          float x[4][8];   // fp32 K (+ bias): x[i][2e + h] = row (e & 1 ? g + 8 : g), col 16 ks[i] + 2t + h (+ 8 if e >= 2)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 b0 = make_float2(0.f, 0.f), b1 = b0;
            if (a.bias) {
              b0 = __ldg(reinterpret_cast<const float2*>(a.bias + nk + 16 * ks[i] + 2 * t));
              b1 = __ldg(reinterpret_cast<const float2*>(a.bias + nk + 16 * ks[i] + 8 + 2 * t));
            }
            x[i][0] = __uint_as_float(r[i][0]) + b0.x;   // row g,   col 2t
            x[i][1] = __uint_as_float(r[i][1]) + b0.y;   // row g,   col 2t+1
            x[i][2] = __uint_as_float(r[i][2]) + b0.x;   // row g+8, col 2t
            x[i][3] = __uint_as_float(r[i][3]) + b0.y;   // row g+8, col 2t+1
            x[i][4] = __uint_as_float(r[i][4]) + b1.x;   // row g,   col 2t+8
            x[i][5] = __uint_as_float(r[i][5]) + b1.y;
            x[i][6] = __uint_as_float(r[i][6]) + b1.x;   // row g+8, col 2t+8
            x[i][7] = __uint_as_float(r[i][7]) + b1.y;
          }
          if (a.rope_inv != nullptr) {   // rotate (c, c + 64) by pos * inv_freq[c] (rope_rotate's convention)
            constexpr double kTwoPi = 6.283185307179586476925286766559;
            const int pos0 = tok0 + gi * 16 + g;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int c = 16 * ks[i] + 2 * t + (e & 1) + (e >= 4 ? 8 : 0);
                const int pos = pos0 + ((e >> 1) & 1) * 8;
                const double ang = (double)pos * __ldg(a.rope_inv + c);
                const double kq = rint(ang * (1.0 / kTwoPi));
                float sn, cs;
                __sincosf((float)fma(-kq, kTwoPi, ang), &sn, &cs);
                const float x0 = x[i][e], y0 = x[i + 2][e];
                x[i][e] = x0 * cs - y0 * sn;
                x[i + 2][e] = y0 * cs + x0 * sn;
              }
            }
          }
          // k = k_hi + k_lo (two bf16 terms: ~16 mantissa bits), so q.k keeps fp32-level
          // accuracy — the softmax exponentiates score errors (peaky scores)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float x0 = x[i][2 * e], x1 = x[i][2 * e + 1];
              hi[e] = pack_bf16(x0, x1);
              lo[e] = pack_bf16(x0 - __uint_as_float(hi[e] << 16), x1 - __uint_as_float(hi[e] & 0xffff0000u));
            }
            ptx::mma_bf16_16816(sc[gi], hi[0], hi[1], hi[2], hi[3], qb[ks[i]][0], qb[ks[i]][1]);
            ptx::mma_bf16_16816(sc[gi], lo[0], lo[1], lo[2], lo[3], qb[ks[i]][0], qb[ks[i]][1]);
          }
        }
      }
      // ---- mask, scale, per-query-head max over the segment's tokens
      const bool cv0 = 2 * t < G, cv1 = 2 * t + 1 < G;
      float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = gi * 16 + g + (e >= 2 ? 8 : 0);
          const bool ok = (tok0 + row < n) && (r_seg + row < a.M) && ((e & 1) ? cv1 : cv0);
          sc[gi][e] = ok ? sc[gi][e] * a.scale_log2 : -INFINITY;
        }
        m0 = fmaxf(m0, fmaxf(sc[gi][0], sc[gi][2]));
        m1 = fmaxf(m1, fmaxf(sc[gi][1], sc[gi][3]));
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        m0 = fmaxf(m0, __shfl_xor_sync(kFull, m0, o));
        m1 = fmaxf(m1, __shfl_xor_sync(kFull, m1, o));
      }
      // ---- p (rounded once to bf16: the weight P^T V uses and the one l sums)
      float l0 = 0.f, l1 = 0.f;
      uint32_t pk[NG][2];
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) {
        float pv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float mm = (e & 1) ? m1 : m0;
          pv[e] = sc[gi][e] == -INFINITY ? 0.f : __bfloat162float(__float2bfloat16_rn(exp2f(sc[gi][e] - mm)));
        }
        l0 += pv[0] + pv[2];
        l1 += pv[1] + pv[3];
        pk[gi][0] = pack_bf16(pv[0], pv[1]);
        pk[gi][1] = pack_bf16(pv[2], pv[3]);
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(kFull, l0, o);
        l1 += __shfl_xor_sync(kFull, l1, o);
      }
      // ---- O = P^T V over the segment's 16-token groups, 64 output dims at a time
      uint32_t pa[NG][2];
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) {
        const uint32_t X = __shfl_sync(kFull, pk[gi][0], srcA), Y = __shfl_sync(kFull, pk[gi][0], srcB);
        const uint32_t Z = __shfl_sync(kFull, pk[gi][1], srcA), W = __shfl_sync(kFull, pk[gi][1], srcB);
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(pa[gi][0]) : "r"(X), "r"(Y), "r"(sel));
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(pa[gi][1]) : "r"(Z), "r"(W), "r"(sel));
      }
      const float mA = __shfl_sync(kFull, m0, g >> 1), mB = __shfl_sync(kFull, m1, g >> 1);
      const float lA = __shfl_sync(kFull, l0, g >> 1), lB = __shfl_sync(kFull, l1, g >> 1);
      const int split = a.reqs[req].split_begin + tok0 / S;
      const size_t task = (size_t)(hk * G + (qv ? g : 0)) * a.n_splits_all + split;   // head-major partial index
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        float o[8][4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.f;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
          const uint32_t tg = tk + DH + half * 64 + ((uint32_t)(16 * (sg * NG + gi)) << 16);
          uint32_t rv[4][8];
#pragma unroll
          for (int c2 = 0; c2 < 4; ++c2) ptx::tmem_ld_16x256b_x2(tg + 16 * c2, rv[c2]);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 4; ++c2) {
            const uint32_t (&r)[8] = rv[c2];
            float2 b0 = make_float2(0.f, 0.f), b1 = b0;
            if (a.bias) {
              const float* bv = a.bias + nk + DH + half * 64 + 16 * c2 + 2 * t;
              b0 = __ldg(reinterpret_cast<const float2*>(bv));
              b1 = __ldg(reinterpret_cast<const float2*>(bv + 8));
            }
            const uint32_t u0 = pack_bf16(__uint_as_float(r[0]) + b0.x, __uint_as_float(r[1]) + b0.y);
            const uint32_t u1 = pack_bf16(__uint_as_float(r[2]) + b0.x, __uint_as_float(r[3]) + b0.y);
            const uint32_t u2 = pack_bf16(__uint_as_float(r[4]) + b1.x, __uint_as_float(r[5]) + b1.y);
            const uint32_t u3 = pack_bf16(__uint_as_float(r[6]) + b1.x, __uint_as_float(r[7]) + b1.y);
            ptx::mma_bf16_16816(o[2 * c2], pa[gi][0], 0u, pa[gi][1], 0u, ptx::movmatrix_trans(u0),
                                ptx::movmatrix_trans(u1));
            ptx::mma_bf16_16816(o[2 * c2 + 1], pa[gi][0], 0u, pa[gi][1], 0u, ptx::movmatrix_trans(u2),
                                ptx::movmatrix_trans(u3));
          }
        }
        // ---- emit: lane (g, t) holds O[query head g][dims half*64 + 8 nb + 2t, + 1]
        if (qv) {
          float* dst = a.part_acc + task * DH + half * 64 + 2 * t;
#pragma unroll
          for (int nb = 0; nb < 8; ++nb) *reinterpret_cast<float2*>(dst + 8 * nb) = make_float2(o[nb][0], o[nb][1]);
        }
      }
      if (qv && t == 0) {
        a.part_ml[2 * task] = (g & 1) ? mB : mA;
        a.part_ml[2 * task + 1] = (g & 1) ? lB : lA;
      }
    }
  }
}

struct PairSmem {
  uint8_t* stages;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t* tmem_slot;
  int32_t* prow;   // 16 gathered pool rows of the producer's current tile
  // dynamic tile queue (TcArgs::tile_counter): the leader's producer grabs tile ids and hands
  // them to every role of both CTAs through TQ slots
  int32_t* tq;
  uint64_t* tq_full;
  uint64_t* tq_empty;
};
constexpr int TQ = 4;

template <int NSUB, int NSTAGE>
__device__ __forceinline__ PairSmem pair_carve(uint8_t* base /*1024-aligned*/) {
  using PC = PairCfg<NSUB, NSTAGE>;
  PairSmem s;
  s.stages = base;
  s.full = reinterpret_cast<uint64_t*>(base + PC::STAGES * PC::STAGE_BYTES);
  s.empty = s.full + PC::STAGES;
  s.tfull = s.empty + PC::STAGES;
  s.tempty = s.tfull + 2;
  s.tmem_slot = reinterpret_cast<uint32_t*>(s.tempty + 2);
  s.prow = reinterpret_cast<int32_t*>(s.tempty + 4);
  uint8_t* bar_base = base + PC::STAGES * PC::STAGE_BYTES;   // 512 B of barriers / control
  static_assert(16 * NSTAGE + 112 <= 256, "pair barrier block");
  s.tq = reinterpret_cast<int32_t*>(bar_base + 256);
  s.tq_full = reinterpret_cast<uint64_t*>(bar_base + 256 + 16);
  s.tq_empty = s.tq_full + TQ;
  return s;
}

// Barrier init (warp 0) and pair TMEM allocation (warp 1, both CTAs).  The caller must then
// run tc_fence_before; cluster_sync; tc_fence_after before reading *tmem_slot.
template <int NSUB, int NSTAGE, int EPI_SPLIT = 1>
__device__ __forceinline__ void pair_setup(const PairSmem& s, int warp, int lane, const CUtensorMap* tmx,
                                           const CUtensorMap* tmw) {
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(tmx);
    ptx::prefetch_tmap(tmw);
    for (int i = 0; i < NSTAGE; ++i) {
      ptx::mbar_init(&s.full[i], 1);
      ptx::mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s.tfull[i], 1);
      ptx::mbar_init(&s.tempty[i], 8 * EPI_SPLIT);   // 4 (or 8) epilogue warps x 2 CTAs (used on the leader)
    }
    for (int i = 0; i < TQ; ++i) {
      ptx::mbar_init(&s.tq_full[i], 1);
      // released by every reader of the slot (used on the leader): the epilogue warps of both
      // CTAs, the partner's producer and the MMA issuer
      ptx::mbar_init(&s.tq_empty[i], 8 * EPI_SPLIT + 2);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_cg2<TMEM_COLS>(s.tmem_slot);
}

// Roles of warps 0..5 (+ 4 extra epilogue warps 6..9 when ESPLIT == 2).  Call with
// warp < 6 (or < 10) only.  GQA2: compile the paired-query-head GQA epilogue in.
template <int NSUB, int NSTAGE, int ESPLIT = 1, bool GQA2 = false>
__device__ __forceinline__ void pair_roles(const PairSmem& s, int warp, int lane, const CUtensorMap* tmap_x,
                                           const CUtensorMap* tmap_w, const TcArgs& a, uint32_t tmem_base,
                                           const CUtensorMap* tmap_x128 = nullptr) {
  using PC = PairCfg<NSUB, NSTAGE>;
  constexpr int STAGES_ = PC::STAGES, NACC = PC::NACC;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int n_tiles_total = a.m_tiles * a.n_tiles;
  // Tile schedule.  Static: pair p takes tiles p, p + n_pairs, ...  Dynamic (a.tile_counter):
  // the leader's producer takes the next tile id from a global counter when it starts a tile
  // and publishes it in the TQ-slot queue to the partner's producer (st.shared::cluster +
  // remote arrive), the MMA issuer and the epilogue warps of both CTAs; a tile id
  // >= n_tiles_total ends every role.  Consecutive ids (the tiles that share an A panel in the
  // n-major raster) then start at about the same time on whichever pairs are free, so the
  // pairs that read an A panel stay together instead of drifting apart over hundreds of
  // waves, and the panel is read from DRAM about once.
  const bool dyn = a.tile_counter != nullptr;
  int q_it = 0;   // queue slots consumed by this role
  // consumer side of the queue (partner producer, MMA issuer, epilogue warps; the caller
  // arrives on the leader's empty barrier after reading)
  auto q_read = [&](int& t) -> uint32_t {
    const int slot = q_it & (TQ - 1);
    const uint32_t ph = (uint32_t)(q_it / TQ) & 1u;
    ++q_it;
    ptx::mbar_wait_cluster(&s.tq_full[slot], ph);
    t = *reinterpret_cast<volatile int32_t*>(&s.tq[slot]);
    return ptx::mapa(ptx::smem_u32(&s.tq_empty[slot]), 0);   // the leader's empty barrier
  };

  if (warp == 0) {
    // ================= TMA producer (both CTAs) =================
    if (lane == 0) {
      // l2_hint: 1 A evict_last + W evict_first, 2 the reverse, 3 A normal + W evict_last
      const uint64_t pol_a = a.l2_hint == 2   ? ptx::policy_evict_first()
                             : a.l2_hint == 3 ? ptx::policy_evict_normal()
                                              : ptx::policy_evict_last();
      const uint64_t pol_b = a.l2_hint == 1 ? ptx::policy_evict_first() : ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int my_step = 0;
      const bool sync_on = a.sync != nullptr && leader && (pair ^ 1) < n_pairs;
      const int nbox = 128 / a.rows_per_box;
      const int box_bytes = a.rows_per_box * BK * 2;
      // Runs of consecutive pool blocks (a request appended in one go gets consecutive ids,
      // lowest free first) are fetched as ONE 128-row box instead of 128/B gathered ones: the
      // smem image is identical (the 128-B swizzle repeats every 8 rows).
      const bool runs_ok = tmap_x128 != nullptr && a.gather != nullptr && nbox > 1;
      for (int t = pair;; t += n_pairs) {
        if (dyn) {
          if (leader) {
            const int slot = q_it & (TQ - 1);
            const uint32_t ph = (uint32_t)(q_it / TQ) & 1u;
            ++q_it;
            ptx::mbar_wait(&s.tq_empty[slot], ph ^ 1);
            t = atomicAdd(a.tile_counter, 1);
            if (t > n_tiles_total) t = n_tiles_total;
            s.tq[slot] = t;
            ptx::st_shared_cluster_u32(ptx::mapa(ptx::smem_u32(&s.tq[slot]), 1), (uint32_t)t);
            ptx::mbar_arrive(&s.tq_full[slot]);
            ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&s.tq_full[slot]), 1));
          } else {
            const uint32_t e = q_read(t);
            ptx::mbar_arrive_cluster(e);
          }
        }
        if (t >= n_tiles_total) break;
        int mt, nt;
        tile_coords_p(t, a.m_tiles, a.n_tiles, a.group_m, mt, nt);
        for (int i = 0; i < nbox; ++i) {
          const int grow = mt * P_BM + (int)rank * 128 + i * a.rows_per_box;
          if (a.gather == nullptr) {
            s.prow[i] = grow;   // dense A (rows past M are zero-filled by TMA and discarded)
          } else {
            const int g = grow / a.B;
            s.prow[i] = g < a.n_hblocks ? a.gather[g] * a.B + (grow - g * a.B) : 0;
#ifdef HC_DIAG
            if (a.diag == 3 && i > 0) s.prow[i] = s.prow[0] + i * a.rows_per_box;   // timing diagnostic
#endif
          }
        }
        bool one_box = runs_ok;
        for (int i = 1; i < nbox && one_box; ++i) one_box = s.prow[i] == s.prow[0] + i * a.rows_per_box;
        if (one_box) {   // and the first box's block must be a real one (rows past M gather block 0)
          const int g0 = (mt * P_BM + (int)rank * 128) / a.B;
          one_box = g0 + nbox * a.rows_per_box / a.B <= a.n_hblocks;
        }
        const int wrow = nt * PC::TILE_N + (int)rank * 128;
        for (int kb = 0; kb < a.k_iters; ++kb) {
          if (sync_on && (my_step & 7) == 0) {
            // partner lockstep: pairs p and p^1 share the A panel; keep them within sync_w
            // k-steps so the second reader hits in L2.
            st_relaxed(a.sync + 32 * pair, my_step);
            if (my_step > a.sync_w) {
              const long long t0 = clock64();
              while (ld_relaxed(a.sync + 32 * (pair ^ 1)) < my_step - a.sync_w) {
                if (clock64() - t0 > (1ll << 34)) __trap();
              }
            }
          }
          ptx::mbar_wait(&s.empty[stage], phase ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&s.full[stage], 2 * PC::STAGE_BYTES);
          uint8_t* dA = s.stages + stage * PC::STAGE_BYTES;
          uint8_t* dB = dA + P_A_BYTES;
          if (one_box) {
            ptx::tma_load_2d_cg2(dA, tmap_x128, kb * BK, s.prow[0], &s.full[stage]);
#pragma unroll
            for (int j = 0; j < NSUB; ++j)
              ptx::tma_load_2d_cg2(dB + j * P_B_BYTES, tmap_w, kb * BK, wrow + j * 256, &s.full[stage]);
          } else if (a.l2_hint == 0) {
            for (int i = 0; i < nbox; ++i)
              ptx::tma_load_2d_cg2(dA + i * box_bytes, tmap_x, kb * BK, s.prow[i], &s.full[stage]);
#pragma unroll
            for (int j = 0; j < NSUB; ++j)
              ptx::tma_load_2d_cg2(dB + j * P_B_BYTES, tmap_w, kb * BK, wrow + j * 256, &s.full[stage]);
          } else {
            for (int i = 0; i < nbox; ++i)
              ptx::tma_load_2d_cg2_hint(dA + i * box_bytes, tmap_x, kb * BK, s.prow[i], &s.full[stage], pol_a);
#pragma unroll
            for (int j = 0; j < NSUB; ++j)
              ptx::tma_load_2d_cg2_hint(dB + j * P_B_BYTES, tmap_w, kb * BK, wrow + j * 256, &s.full[stage], pol_b);
          }
          ++my_step;
          if (++stage == STAGES_) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (sync_on) st_relaxed(a.sync + 32 * pair, 0x7fffffff);  // done: never hold the partner
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA only) =================
    if (leader && lane == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc_bf16_f32(P_BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair;; t += n_pairs, ++it) {
        if (dyn) ptx::mbar_arrive_cluster(q_read(t));
        if (t >= n_tiles_total) break;
        const int acc = it % NACC;
        const uint32_t acc_phase = (it / NACC) & 1;
        ptx::mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * PC::TILE_N;
        for (int kb = 0; kb < a.k_iters; ++kb) {
          ptx::mbar_wait(&s.full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(s.stages + stage * PC::STAGE_BYTES);
          const uint32_t b_addr = a_addr + P_A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = ptx::umma_desc_k_sw128(a_addr + k * 32);
#pragma unroll
            for (int j = 0; j < NSUB; ++j) {
              const uint64_t bd = ptx::umma_desc_k_sw128(b_addr + j * P_B_BYTES + k * 32);
              ptx::umma_f16_ss_cg2(d_tmem + j * 256, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          ptx::umma_commit_cg2_mc(&s.empty[stage], 0x3);
          if (++stage == STAGES_) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit_cg2_mc(&s.tfull[acc], 0x3);
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue (warps 2..5, and 6..9 with epi_split 2, of both CTAs) ==========
    const int q = warp & 3;
    const int esub = ESPLIT > 1 ? (warp - 2) >> 2 : 0;   // ESPLIT 2: every other head / column chunk
    const int row_in_tile = (int)rank * 128 + q * 32 + lane;
    const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&s.tempty[0]), 0);
    int it = 0;
    for (int t = pair;; t += n_pairs, ++it) {
      if (dyn) {
        const uint32_t e = q_read(t);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(e);
      }
      if (t >= n_tiles_total) break;
      int mt, nt;
      tile_coords_p(t, a.m_tiles, a.n_tiles, a.group_m, mt, nt);
      const int acc = it % NACC;
      const uint32_t acc_phase = (it / NACC) & 1;
      ptx::mbar_wait(&s.tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int grow = mt * P_BM + row_in_tile;
      if (a.epi == EPI_ATTEND) {
#ifdef HC_DIAG
        if (a.diag == 1 || a.diag == 2) {   // timing diagnostics (wrong outputs; -DHC_DIAG builds only)
          if (a.diag == 2) {   // read the whole accumulator from TMEM, skip the math
            float f[32], sum = 0.f;
            for (int c = 0; c < PC::TILE_N / 32; ++c) {
              load_chunk(tmem_base + ((uint32_t)(q * 32) << 16) + acc * PC::TILE_N + c * 32, nullptr, 0, f);
#pragma unroll
              for (int j = 0; j < 32; ++j) sum += f[j];
            }
            if (sum == 12345.f) a.part_ml[0] = sum;
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
          continue;
        }
#endif
        const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * PC::TILE_N;
        bool done = false;
        if (a.epi_mma) {   // mma.sync attend epilogue (the runtime checked dh = 128)
          const int row0 = mt * P_BM + (int)rank * 128 + q * 32;
          if (a.seg == 16) attend_tile_mma<16, PC::TILE_N, ESPLIT>(a, tacc, nt, row0, lane, esub);
          else attend_tile_mma<32, PC::TILE_N, ESPLIT>(a, tacc, nt, row0, lane, esub);
          done = true;
        }
        if constexpr (GQA2) {
          if (!done && a.grp % 2 == 0) {   // GQA: query heads two at a time
            if (a.seg == 8) attend_tile_gqa2<8, PC::TILE_N, ESPLIT>(a, tacc, nt, grow, lane, esub);
            else if (a.seg == 16) attend_tile_gqa2<16, PC::TILE_N, ESPLIT>(a, tacc, nt, grow, lane, esub);
            else attend_tile_gqa2<32, PC::TILE_N, ESPLIT>(a, tacc, nt, grow, lane, esub);
            done = true;
          }
        }
        if (!done) {
          if (a.seg == 8)
            attend_tile<8, PC::TILE_N, ESPLIT>(a, tacc, nt, grow, lane, esub);
          else if (a.seg == 16)
            attend_tile<16, PC::TILE_N, ESPLIT>(a, tacc, nt, grow, lane, esub);
          else
            attend_tile<32, PC::TILE_N, ESPLIT>(a, tacc, nt, grow, lane, esub);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
        continue;
      }
      const bool valid = grow < a.M;
      const int g = grow / a.B, r = grow - g * a.B;
      int4 dst_info = make_int4(-1, -1, 0, 0);
      if (a.epi == EPI_PROJECT && valid) dst_info = *reinterpret_cast<const int4*>(a.row_dst + 4 * grow);
      const int pos = a.rope_inv == nullptr ? 0
                      : (a.epi == EPI_SCRATCH ? (valid ? a.row_pos[g] + r : 0) : dst_info.w);
#pragma unroll 1
      for (int c = esub; c < PC::TILE_N / 32; c += ESPLIT) {   // (RoPE partners c, c + dh/64 share parity)
        const int n = nt * PC::TILE_N + c * 32;
        // RoPE pairs columns (c0, c0 + dh/2) of a rotated head segment (K; and q in EPI_PROJECT)
        int seg_c0 = -1;   // column within the rotated head segment, or -1
        if (a.rope_inv != nullptr && a.epi != EPI_DENSE) {
          const int m = (a.epi == EPI_PROJECT) ? n - a.d : n;
          if (a.epi == EPI_PROJECT && n < a.d) {
            seg_c0 = n % a.dh;                                   // q
          } else {
            const int rem = m % (2 * a.dh);
            if (rem < a.dh) seg_c0 = rem;                        // K half of K_h || V_h
          }
        }
        if (seg_c0 >= a.dh / 2) continue;   // written together with its partner chunk
        float f[32], f2[32];
        load_chunk(tmem_base + ((uint32_t)(q * 32) << 16) + acc * PC::TILE_N + c * 32, a.bias, n, f);
        if (seg_c0 >= 0) {
          const int half = a.dh / 2;
          load_chunk(tmem_base + ((uint32_t)(q * 32) << 16) + acc * PC::TILE_N + c * 32 + half, a.bias, n + half, f2);
          rope_rotate(f, f2, pos, a.rope_inv + seg_c0);
        }
        if (!valid) continue;
        store_chunk(a, n, f, grow, g, r, dst_info);
        if (seg_c0 >= 0) store_chunk(a, n + a.dh / 2, f2, grow, g, r, dst_info);
      }
      ptx::tc_fence_before();
      if (a.tile_done) __threadfence();   // this warp's rows are globally visible before the count
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
        if (a.tile_done) red_release_add(a.tile_done + mt * a.n_tiles + nt, 1);
      }
    }
  }
}

template <int NSUB, int NSTAGE>
__device__ __forceinline__ void pair_teardown(int warp, uint32_t tmem_base) {
  if (warp == 1) ptx::tmem_dealloc_cg2<TMEM_COLS>(tmem_base);
}

}  // namespace pg
}  // namespace hc
