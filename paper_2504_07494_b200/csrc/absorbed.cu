// Absorbed hidden-cache attention (NEXT row f4 (ii); a NON-PAPER variant, opt-in through
// HC_FLAG_ABSORB_HIDDEN).  For hidden-mode requests the paper rebuilds K = X W_K^T and
// V = X W_V^T every step (4 d^2 FLOPs per cached token).  Associativity gives
// the same Eq. 2-3 without the rebuild, per head h:
//     q~_h = W_K,h^T q_h                      (d values, once per request)
//     s_j  = scale (q~_h . x_j + q_h . b_K,h)  (the bias term is a per-head constant: it
//                                              cancels in the softmax and only shifts lse)
//     z_h  = sum_j a_j x_j,   o_h = W_V,h z_h + b_V,h       (sum_j a_j = 1)
// so a hidden token costs two reads of x (4d bytes, like the K and V rows of a KV token)
// plus O(d H) FLOPs, and the per-call work is two weight reads (W_K, W_V) — the path is
// HBM-bound instead of tensor-bound.  Five kernels, all bf16 in / fp32 accumulate on
// warp-level MMA (mma.sync.m16n8k16 + ldmatrix; the contractions are memory-bound):
//   K1 qt_kernel     q~[r][h][:]  = W_K,h^T q_{r,h}            (per head: [n_h x dh][dh x d])
//   K2 score_kernel  S[row][h]    = x_row . q~[r(row)][h]       (gathered hidden rows x H)
//   K3 stats_kernel  per (r,h): m, l over the request's tokens; P[row][h] = 2^(s - m) (bf16)
//   K4 z_kernel      Z[r][h][:]   = sum_rows P[row][h] x_row     (per request: [H x n][n x d])
//   K5 wv_kernel     out[r][h*dh:] = W_V,h Z[r][h] / l + b_V,h;  lse
#include <cuda_bf16.h>

#include "internal.h"

namespace hc {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp16_zfill(void* dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;   // src-size 0: the 16 bytes are zero-filled
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(dst)), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
__device__ __forceinline__ void ldsm4t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// 64-element (128 B) swizzled rows: 16-byte chunk c (0..7) of row r at chunk c ^ (r & 7)
__device__ __forceinline__ uint32_t sw64(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// ------------------------------------------------------------------ K1: q~ = W_K,h^T q_h
// CTA: 64 hidden requests x 128 columns of d, one head; K = dh (<= 128, multiple of 16).
// A = q rows [64 x dh] (row-major, K contiguous), B = W_K,h [dh x 128] (row-major K x N ->
// ldmatrix.trans).  4 warps x 16 rows.
__global__ void __launch_bounds__(128) qt_kernel(const AbsorbParams p) {
  __shared__ __align__(128) uint8_t sA[64 * 256];      // 64 rows x dh(<=128) bf16, as 2 x 64-wide halves
  __shared__ __align__(128) uint8_t sB[128 * 256];     // dh rows x 128 cols bf16, as 2 x 64-wide halves
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * 128, h = blockIdx.y, r0 = blockIdx.z * 64;
  const int dh = p.dh, d = p.d;
  const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(p.q);
  const __nv_bfloat16* w = static_cast<const __nv_bfloat16*>(p.w_int);
  // A: rows r0.., columns [h*dh, h*dh+dh) of q; half k of 64 columns each
  for (int i = tid; i < 64 * (dh / 8); i += 128) {
    const int r = i / (dh / 8), c = i % (dh / 8);
    const int rr = r0 + r;
    const bool ok = rr < p.n_h;
    const int req = ok ? p.hreq[rr] : 0;
    cp16_zfill(sA + (c >> 3) * (64 * 128) + sw64(r, c & 7), q + (size_t)req * d + h * dh + c * 8, ok);
  }
  // B: W_K,h rows k = 0..dh-1 (W_int row h*2dh + k), columns n0..n0+127
  for (int i = tid; i < dh * 16; i += 128) {
    const int k = i >> 4, c = i & 15;
    cp16(sB + (c >> 3) * (128 * 128) + sw64(k, c & 7), w + (size_t)(h * 2 * dh + k) * d + n0 + c * 8);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  float acc[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const int mat = lane >> 3, rr = lane & 7;
  for (int ks = 0; ks < dh / 16; ++ks) {
    uint32_t a0, a1, a2, a3;
    {
      const int row = warp * 16 + ((mat & 1) << 3) + rr, chunk = 2 * ks + (mat >> 1);
      ldsm4(saddr(sA) + (chunk >> 3) * (64 * 128) + sw64(row, chunk & 7), a0, a1, a2, a3);
    }
#pragma unroll
    for (int nj = 0; nj < 8; ++nj) {   // 16 columns per ldmatrix.x4.trans
      const int krow = ks * 16 + ((mat & 1) << 3) + rr, chunk = 2 * nj + (mat >> 1);
      uint32_t b0, b1, b2, b3;
      ldsm4t(saddr(sB) + (chunk >> 3) * (128 * 128) + sw64(krow, chunk & 7), b0, b1, b2, b3);
      mma(acc[2 * nj], a0, a1, a2, a3, b0, b1);
      mma(acc[2 * nj + 1], a0, a1, a2, a3, b2, b3);
    }
  }
  const int g = lane >> 2, t4 = lane & 3;
  __nv_bfloat16* qt = p.qt;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = n0 + j * 8 + 2 * t4;
    const int ra = r0 + warp * 16 + g, rb = ra + 8;
    if (ra < p.n_h) *reinterpret_cast<uint32_t*>(qt + ((size_t)ra * p.H + h) * d + col) = pk(acc[j][0], acc[j][1]);
    if (rb < p.n_h) *reinterpret_cast<uint32_t*>(qt + ((size_t)rb * p.H + h) * d + col) = pk(acc[j][2], acc[j][3]);
  }
}

// ------------------------------------------------------------------ K2: S = X q~^T
// CTA: 64 gathered rows of ONE hidden request x Hp (<= 128) heads, K loop over d in 64s.
// A = X rows (gathered from pool blocks), B = q~[r] [Hp x d] (rows = heads, K contiguous).
__global__ void __launch_bounds__(128) score_kernel(const AbsorbParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int ST = 2;
  uint8_t* sA = sm;                       // ST x [64 x 64]
  uint8_t* sB = sm + ST * 64 * 128;       // ST x [Hp x 64]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = p.tile_req[blockIdx.x], t0 = p.tile_t0[blockIdx.x];
  const int Hp = p.Hp, d = p.d, B = p.B, H = p.H;
  const int row_base = p.hrow0[r];        // first gathered row of request r
  const int ntok = p.hntok[r];
  const __nv_bfloat16* pool = static_cast<const __nv_bfloat16*>(p.pool);
  const __nv_bfloat16* qt = p.qt + (size_t)r * H * d;
  auto load = [&](int kc, int buf) {
    uint8_t* a = sA + buf * 64 * 128;
    uint8_t* b = sB + buf * Hp * 128;
    for (int i = tid; i < 64 * 8; i += 128) {
      const int row = i >> 3, c = i & 7;
      const int t = min(t0 + row, ntok - 1);
      const int grow = row_base + t, g = grow / B;
      cp16(a + sw64(row, c), pool + ((size_t)p.gather[g] * B + (grow - g * B)) * d + kc * 64 + c * 8);
    }
    for (int i = tid; i < Hp * 8; i += 128) {
      const int hh = i >> 3, c = i & 7;
      cp16_zfill(b + sw64(hh, c), qt + (size_t)min(hh, H - 1) * d + kc * 64 + c * 8, hh < H);
    }
  };
  const int NT = Hp / 8;   // n-tiles of 8 heads
  float acc[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const int KC = d / 64;
  load(0, 0);
  cp_commit();
  const int mat = lane >> 3, rr = lane & 7;
  for (int kc = 0; kc < KC; ++kc) {
    if (kc + 1 < KC) load(kc + 1, (kc + 1) & 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const uint32_t a_s = saddr(sA + (kc & 1) * 64 * 128), b_s = saddr(sB + (kc & 1) * Hp * 128);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t a0, a1, a2, a3;
      ldsm4(a_s + sw64(warp * 16 + ((mat & 1) << 3) + rr, 2 * ks + (mat >> 1)), a0, a1, a2, a3);
#pragma unroll
      for (int nj = 0; nj < 8; ++nj) {
        if (2 * nj < NT) {
          uint32_t b0, b1, b2, b3;
          ldsm4(b_s + sw64(nj * 16 + ((mat >> 1) << 3) + rr, 2 * ks + (mat & 1)), b0, b1, b2, b3);
          mma(acc[2 * nj], a0, a1, a2, a3, b0, b1);
          if (2 * nj + 1 < NT) mma(acc[2 * nj + 1], a0, a1, a2, a3, b2, b3);
        }
      }
    }
    __syncthreads();
  }
  const int g = lane >> 2, t4 = lane & 3;
  const int ta = t0 + warp * 16 + g, tb = ta + 8;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j >= NT) break;
    const int col = j * 8 + 2 * t4;
    if (ta < ntok) *reinterpret_cast<float2*>(p.s + (size_t)(row_base + ta) * Hp + col) = make_float2(acc[j][0], acc[j][1]);
    if (tb < ntok) *reinterpret_cast<float2*>(p.s + (size_t)(row_base + tb) * Hp + col) = make_float2(acc[j][2], acc[j][3]);
  }
}

// ------------------------------------------------------------------ K3: softmax statistics
// One warp per (hidden request, head): m = max_j s_j, l = sum_j 2^(s_j - m) (log2 domain,
// scores scaled by scale*log2 e); P[row][h] = 2^(s - m) in bf16 for the request's rows
// (padding rows of the last block get P = 0); the key-bias constant q_h . b_K,h.
__global__ void __launch_bounds__(128) stats_kernel(const AbsorbParams p) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= p.n_h * p.H) return;
  const int r = w / p.H, h = w - r * p.H;
  const int base = p.hrow0[r], ntok = p.hntok[r], Hp = p.Hp;
  float m = -INFINITY;
  for (int t = lane; t < ntok; t += 32) m = fmaxf(m, p.s[(size_t)(base + t) * Hp + h] * p.scale_log2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
  float l = 0.f;
  for (int t = lane; t < ntok; t += 32) {
    const float e = exp2f(p.s[(size_t)(base + t) * Hp + h] * p.scale_log2 - m);
    l += e;
    p.pm[(size_t)(base + t) * Hp + h] = __float2bfloat16_rn(e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(FULL, l, o);
  float c = 0.f;
  if (p.b_int) {   // q_h . b_K,h
    const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(p.q) + (size_t)p.hreq[r] * p.d + h * p.dh;
    for (int e = lane; e < p.dh; e += 32) c += __bfloat162float(q[e]) * p.b_int[h * 2 * p.dh + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
  }
  if (lane == 0) {
    p.ml[3 * (size_t)w] = m;
    p.ml[3 * (size_t)w + 1] = l;
    p.ml[3 * (size_t)w + 2] = c;
  }
}

// ------------------------------------------------------------------ K4: Z = P^T X
// CTA: one hidden request x 128 columns of d; M = Hp heads (<= 128), K loop over the
// request's rows in 64s.  A = P^T (P tile [64 rows x Hp] -> ldmatrix.trans), B = X tile
// [64 rows x 128 cols] (row-major K x N -> ldmatrix.trans).  4 warps split N (32 each).
__global__ void __launch_bounds__(128) z_kernel(const AbsorbParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int ST = 2;
  const int Hp = p.Hp;
  const int PH = (Hp + 63) / 64;                  // 64-column halves of the P tile
  uint8_t* sP = sm;                               // ST x [PH halves x 64 rows x 64 cols]
  uint8_t* sX = sm + ST * PH * 64 * 128;          // ST x [64 rows x 128 cols] as 2 halves
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * 128, r = blockIdx.y;
  const int d = p.d, B = p.B, H = p.H;
  const int base = p.hrow0[r], ntok = p.hntok[r];
  const __nv_bfloat16* pool = static_cast<const __nv_bfloat16*>(p.pool);
  // rows >= ntok are zero-filled in both operands (slots past n in the last block are
  // never written by hc_append and may hold anything)
  auto load = [&](int t0, int buf) {
    uint8_t* ps = sP + buf * PH * 64 * 128;
    uint8_t* xs = sX + buf * 64 * 256;
    for (int i = tid; i < 64 * (Hp / 8); i += 128) {
      const int row = i / (Hp / 8), c = i % (Hp / 8);
      const bool ok = t0 + row < ntok;
      cp16_zfill(ps + (c >> 3) * (64 * 128) + sw64(row, c & 7),
                 p.pm + (size_t)(base + (ok ? t0 + row : 0)) * Hp + c * 8, ok);
    }
    for (int i = tid; i < 64 * 16; i += 128) {
      const int row = i >> 4, c = i & 15;
      const bool ok = t0 + row < ntok;
      const int grow = base + (ok ? t0 + row : 0), g = grow / B;
      cp16_zfill(xs + (c >> 3) * (64 * 128) + sw64(row, c & 7),
                 pool + ((size_t)p.gather[g] * B + (grow - g * B)) * d + n0 + c * 8, ok);
    }
  };
  const int MT = Hp / 16;
  float acc[8][4][4];   // [m-tile (<= 8)][n-tile (4 x 8 cols)][frag]
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0.f;
  const int nkt = (ntok + 63) / 64;
  load(0, 0);
  cp_commit();
  const int mat = lane >> 3, rr = lane & 7;
  for (int kt = 0; kt < nkt; ++kt) {
    if (kt + 1 < nkt) load((kt + 1) * 64, (kt + 1) & 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const uint32_t p_s = saddr(sP + (kt & 1) * PH * 64 * 128), x_s = saddr(sX + (kt & 1) * 64 * 256);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {   // 16 rows (K) per step
      // B fragments for this warp's 32 columns: 2 x ldmatrix.x4.trans (16 cols each)
      uint32_t b[4][2];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        const int col_chunk = (warp * 32 + nb * 16) / 8 + (mat >> 1);
        const int krow = ks * 16 + ((mat & 1) << 3) + rr;
        uint32_t b0, b1, b2, b3;
        ldsm4t(x_s + (col_chunk >> 3) * (64 * 128) + sw64(krow, col_chunk & 7), b0, b1, b2, b3);
        b[2 * nb][0] = b0;
        b[2 * nb][1] = b1;
        b[2 * nb + 1][0] = b2;
        b[2 * nb + 1][1] = b3;
      }
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        if (mi >= MT) break;
        // A = P^T rows (heads) mi*16.., k = rows ks*16..: transpose of the [row x head] tile
        uint32_t a0, a1, a2, a3;
        const int head_chunk = mi * 2 + (mat >> 1);   // 8 heads per chunk
        const int krow = ks * 16 + ((mat & 1) << 3) + rr;
        ldsm4t(p_s + (head_chunk >> 3) * (64 * 128) + sw64(krow, head_chunk & 7), a0, a1, a2, a3);
        // ldmatrix.trans order: m0 (heads 0-7, k 0-7), m1 (heads 0-7, k 8-15), m2 (heads 8-15, k 0-7),
        // m3 (heads 8-15, k 8-15) -> A fragment {a0: m0, a1: m2, a2: m1, a3: m3}
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) mma(acc[mi][nt], a0, a2, a1, a3, b[nt][0], b[nt][1]);
      }
    }
    __syncthreads();
  }
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 8; ++mi) {
    if (mi >= MT) break;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int col = n0 + warp * 32 + nt * 8 + 2 * t4;
      const int ha = mi * 16 + g, hb = ha + 8;
      if (ha < H) *reinterpret_cast<uint32_t*>(p.z + ((size_t)r * H + ha) * d + col) = pk(acc[mi][nt][0], acc[mi][nt][1]);
      if (hb < H) *reinterpret_cast<uint32_t*>(p.z + ((size_t)r * H + hb) * d + col) = pk(acc[mi][nt][2], acc[mi][nt][3]);
    }
  }
}

// ------------------------------------------------------------------ K5: o = W_V,h z / l + b_V
// CTA: 64 hidden requests x dh outputs of one head, K loop over d in 64s.  A = Z[r][h]
// rows (K contiguous), B = W_V,h [dh x d] rows (N x K, K contiguous -> non-trans).
__global__ void __launch_bounds__(128) wv_kernel(const AbsorbParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int ST = 2;
  const int dh = p.dh, d = p.d, H = p.H;
  uint8_t* sA = sm;                        // ST x [64 x 64]
  uint8_t* sB = sm + ST * 64 * 128;        // ST x [dh x 64]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.x, r0 = blockIdx.y * 64;
  const __nv_bfloat16* w = static_cast<const __nv_bfloat16*>(p.w_int);
  auto load = [&](int kc, int buf) {
    uint8_t* a = sA + buf * 64 * 128;
    uint8_t* b = sB + buf * dh * 128;
    for (int i = tid; i < 64 * 8; i += 128) {
      const int row = i >> 3, c = i & 7;
      const bool ok = r0 + row < p.n_h;
      cp16_zfill(a + sw64(row, c), p.z + ((size_t)(ok ? r0 + row : 0) * H + h) * d + kc * 64 + c * 8, ok);
    }
    for (int i = tid; i < dh * 8; i += 128) {
      const int e = i >> 3, c = i & 7;
      cp16(b + sw64(e, c), w + (size_t)(h * 2 * dh + dh + e) * d + kc * 64 + c * 8);
    }
  };
  const int NT = dh / 8;
  float acc[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const int KC = d / 64;
  load(0, 0);
  cp_commit();
  const int mat = lane >> 3, rr = lane & 7;
  for (int kc = 0; kc < KC; ++kc) {
    if (kc + 1 < KC) load(kc + 1, (kc + 1) & 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const uint32_t a_s = saddr(sA + (kc & 1) * 64 * 128), b_s = saddr(sB + (kc & 1) * dh * 128);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t a0, a1, a2, a3;
      ldsm4(a_s + sw64(warp * 16 + ((mat & 1) << 3) + rr, 2 * ks + (mat >> 1)), a0, a1, a2, a3);
#pragma unroll
      for (int nj = 0; nj < 8; ++nj) {
        if (2 * nj < NT) {
          uint32_t b0, b1, b2, b3;
          ldsm4(b_s + sw64(nj * 16 + ((mat >> 1) << 3) + rr, 2 * ks + (mat & 1)), b0, b1, b2, b3);
          mma(acc[2 * nj], a0, a1, a2, a3, b0, b1);
          mma(acc[2 * nj + 1], a0, a1, a2, a3, b2, b3);
        }
      }
    }
    __syncthreads();
  }
  const int g = lane >> 2, t4 = lane & 3;
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int r = r0 + warp * 16 + g + 8 * hr;
    if (r >= p.n_h) continue;
    const float* ml = p.ml + 3 * ((size_t)r * H + h);
    const float inv = 1.f / ml[1];
    const int req = p.hreq[r];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= NT) break;
      const int e = j * 8 + 2 * t4;
      float v0 = acc[j][2 * hr] * inv, v1 = acc[j][2 * hr + 1] * inv;
      if (p.b_int) {
        v0 += p.b_int[h * 2 * dh + dh + e];
        v1 += p.b_int[h * 2 * dh + dh + e + 1];
      }
      *reinterpret_cast<uint32_t*>(out + (size_t)req * d + h * dh + e) = pk(v0, v1);
    }
    if (t4 == 0 && p.lse) p.lse[(size_t)req * H + h] = (ml[0] + log2f(ml[1])) * 0.69314718055994531f + p.scale * ml[2];
  }
}

}  // namespace

bool absorb_supported(int dtype, int d, int dh, int H) {
  return dtype == 0 && d % 128 == 0 && dh % 16 == 0 && dh <= 128 && H <= 128;
}

cudaError_t launch_absorbed(const AbsorbParams& p, cudaStream_t s) {
  if (p.n_h <= 0) return cudaSuccess;
  cudaError_t e;
  qt_kernel<<<dim3(p.d / 128, p.H, (p.n_h + 63) / 64), 128, 0, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int smem2 = 2 * 64 * 128 + 2 * p.Hp * 128;
  score_kernel<<<p.n_tiles, 128, smem2, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  stats_kernel<<<(p.n_h * p.H + 3) / 4, 128, 0, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int smem4 = 2 * ((p.Hp + 63) / 64) * 64 * 128 + 2 * 64 * 256;
  static const cudaError_t attr = cudaFuncSetAttribute(z_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 2 * 64 * 128 + 2 * 64 * 256);
  if (attr != cudaSuccess) return attr;
  z_kernel<<<dim3(p.d / 128, p.n_h), 128, smem4, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int smem5 = 2 * 64 * 128 + 2 * p.dh * 128;
  wv_kernel<<<dim3(p.H, (p.n_h + 63) / 64), 128, smem5, s>>>(p);
  return cudaGetLastError();
}

}  // namespace hc
