// Absorbed hidden-cache attention (NEXT row f4 (ii); a NON-PAPER variant, opt-in through
// HC_FLAG_ABSORB_HIDDEN).  For hidden-mode requests the paper rebuilds K = X W_K^T and
// V = X W_V^T every step (4 d^2 FLOPs per cached token).  Associativity gives
// the same Eq. 2-3 without the rebuild, per head h:
//     q~_h = W_K,h^T q_h                      (d values, once per request)
//     s_j  = scale (q~_h . x_j + q_h . b_K,h)  (the bias term is a per-head constant: it
//                                              cancels in the softmax and only shifts lse)
//     z_h  = sum_j a_j x_j,   o_h = W_V,h z_h + b_V,h       (sum_j a_j = 1)
// so a hidden token costs two reads of x (4d bytes, like the K and V rows of a KV token)
// plus 4 Hp d FLOPs, and the per-call work is two weight reads (W_K, W_V) — the path is
// HBM-bound instead of tensor-bound.  Five kernels, bf16 in / fp32 accumulate:
//   K1 qt_tc_kernel    q~[r][h][:] = W_K,h^T q_{r,h} (per head [n_h x dh][dh x d], tcgen05,
//                      W_K,h as an MN-major operand); q_h . b_K,h
//   K2 score_tc_kernel per 128-token tile of request r (tcgen05): s = x . q~[r][h]; tile max
//                      m_t[h], P[row][h] = 2^(scaled s - m_t) (bf16), l_t[h] = sum P
//   K3 rescale_kernel  m[h] = max_t m_t, P *= 2^(m_t - m), l = sum_t 2^(m_t - m) l_t
//   K4 z_tc_kernel     Z[r][h][:] = sum_rows P[row][h] x_row (tcgen05, MN-major operands)
//   K5 wv_tc_kernel    out[r][h*dh:] = W_V,h Z[h][r] / l + b_V,h;  lse (tcgen05)
// x is read exactly twice (K2, K4), straight from the pool blocks through TMA.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

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
__device__ __forceinline__ uint32_t pk(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// 64-element (128 B) swizzled rows: 16-byte chunk c (0..7) of row r at chunk c ^ (r & 7)
__device__ __forceinline__ uint32_t sw64(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// ------------------------------------------------------------------ K2: scores on tcgen05
// CTA: one 128-token tile of one hidden request.  S[128 x Hp] = X_tile q~[r]^T with
// tcgen05.mma M=128 N=Hp K=16 (both operands K-major SWIZZLE_128B, A = the request's pool
// blocks as TMA boxes — no gather copy — B = q~[r] rows), fp32 accumulators in TMEM.
// Warp 0: TMA producer; warp 1: TMEM allocator + MMA issuer; warps 2-5: epilogue (thread =
// token row): scaled scores -> smem (column-major), per-head tile max m_t and l_t =
// sum 2^(s - m_t) by column scans, P = 2^(s - m_t) bf16 rows (0 for the padding slots of
// the request's last block).
constexpr int SC_STAGE = 32768;   // 16 KiB A + <= 16 KiB B per stage
constexpr int TC_THREADS = 192;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t a = ptx::smem_u32(p);
  return p + ((1024 - (a & 1023)) & 1023);
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int SC_ST>
__global__ void __launch_bounds__(TC_THREADS, SC_ST == 2 ? 3 : 2)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_qt,
                    const AbsorbParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  // stages, then (after the MMAs retire) the [Hp][129] fp32 score staging of the epilogue
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + max(SC_ST * SC_STAGE, 128 * 129 * 4));
  uint64_t* empty = full + SC_ST;
  uint64_t* tfull = empty + SC_ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* m_s = reinterpret_cast<float*>(tmem_slot + 4);   // [128]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, r = p.tile_req[tile], t0 = p.tile_t0[tile];
  const int ntok = p.hntok[r], row_base = p.hrow0[r], Hp = p.Hp, B = p.B;
  const int KC = p.d / 64;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    ptx::prefetch_tmap(&tmap_qt);
    for (int s = 0; s < SC_ST; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<128>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      const int rpb = p.rpb, nbox = 128 / rpb;
      int prow[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        prow[i] = 0;
        if (i < nbox) {
          const int grow = row_base + t0 + i * rpb, g = grow / B;
          if (g < p.n_hb) prow[i] = p.gather[g] * B + (grow - g * B);
        }
      }
      const uint32_t bytes = 128 * 128 + Hp * 128;
      int stage = 0;
      uint32_t phase = 0;
      for (int kc = 0; kc < KC; ++kc) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], bytes);
        uint8_t* a = smem + stage * SC_STAGE;
        for (int i = 0; i < nbox; ++i) ptx::tma_load_2d(a + i * rpb * 128, &tmap_x, kc * 64, prow[i], &full[stage]);
        ptx::tma_load_2d(a + 16384, &tmap_qt, kc * 64, r * Hp, &full[stage]);
        if (++stage == SC_ST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16_f32(128, Hp);
      int stage = 0;
      uint32_t phase = 0;
      for (int kc = 0; kc < KC; ++kc) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a = ptx::smem_u32(smem + stage * SC_STAGE), b = a + 16384;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          ptx::umma_f16_ss(tmem, ptx::umma_desc_k_sw128(a + k * 32), ptx::umma_desc_k_sw128(b + k * 32), idesc,
                           (kc | k) != 0 ? 1u : 0u);
        ptx::umma_commit(&empty[stage]);
        if (++stage == SC_ST) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::umma_commit(tfull);
    }
    __syncwarp();
  } else {
    // ---- epilogue: thread = token row of the tile (TMEM lane quadrant = warp & 3)
    const int q = warp & 3, row = q * 32 + lane;
    const int nvalid = min(128, ntok - t0);
    const int padded = (ntok + B - 1) / B * B;
    const bool valid = row < nvalid, keep = t0 + row < padded;
    ptx::mbar_wait(tfull, 0);
    ptx::tc_fence_after();
    float* S = reinterpret_cast<float*>(smem);   // [Hp][129] column-major (all MMAs retired)
    const float sl = p.scale_log2;
    for (int c = 0; c < Hp; c += 32) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c + j < Hp) S[(c + j) * 129 + row] = __uint_as_float(v[j]) * sl;
    }
    epi_bar();
    const int h = row;   // column scan: thread h owns head h
    if (h < Hp) {
      const float* col = S + h * 129;
      float m = -INFINITY;
      for (int i = 0; i < nvalid; ++i) m = fmaxf(m, col[i]);
      float l = 0.f;
      for (int i = 0; i < nvalid; ++i) l += exp2f(col[i] - m);
      m_s[h] = m;
      p.tml[2 * ((size_t)tile * Hp + h)] = m;
      p.tml[2 * ((size_t)tile * Hp + h) + 1] = l;
    }
    epi_bar();
    if (keep) {
      uint4* dst = reinterpret_cast<uint4*>(p.pm + (size_t)(row_base + t0 + row) * Hp);
      for (int c8 = 0; c8 < Hp / 8; ++c8) {
        float e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = valid ? exp2f(S[(c8 * 8 + j) * 129 + row] - m_s[c8 * 8 + j]) : 0.f;
        dst[c8] = make_uint4(pk(e[0], e[1]), pk(e[2], e[3]), pk(e[4], e[5]), pk(e[6], e[7]));
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<128>(tmem);
}

// ------------------------------------------------------------------ K3: request max, P rescale
// CTA per 128-token tile: m = max over the request's tiles, P *= 2^(m_t - m); the request's
// first tile also publishes m and l = sum_t 2^(m_t - m) l_t.
__global__ void __launch_bounds__(128) rescale_kernel(const AbsorbParams p) {
  __shared__ float f_s[128];
  const int tid = threadIdx.x, tile = blockIdx.x;
  const int r = p.tile_req[tile], t0 = p.tile_t0[tile], ntok = p.hntok[r], tile0 = p.htile0[r];
  const int Hp = p.Hp, H = p.H, B = p.B;
  const int nt = (ntok + 127) / 128;
  if (tid < Hp) {
    float m = -INFINITY;
    for (int k = 0; k < nt; ++k) m = fmaxf(m, p.tml[2 * ((size_t)(tile0 + k) * Hp + tid)]);
    f_s[tid] = exp2f(p.tml[2 * ((size_t)tile * Hp + tid)] - m);
    if (tile == tile0 && tid < H) {
      float l = 0.f;
      for (int k = 0; k < nt; ++k) {
        const float* t = p.tml + 2 * ((size_t)(tile0 + k) * Hp + tid);
        l += exp2f(t[0] - m) * t[1];
      }
      p.ml[3 * ((size_t)r * H + tid)] = m;
      p.ml[3 * ((size_t)r * H + tid) + 1] = l;
    }
  }
  __syncthreads();
  const int padded = (ntok + B - 1) / B * B;
  const int nrows = min(128, padded - t0), c8n = Hp / 8;
  uint4* P = reinterpret_cast<uint4*>(p.pm + (size_t)(p.hrow0[r] + t0) * Hp);
  for (int i = tid; i < nrows * c8n; i += 128) {
    const int c8 = i % c8n;
    uint4 v = P[i];
    __nv_bfloat162* e = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(e[j]);
      e[j] = __floats2bfloat162_rn(f.x * f_s[c8 * 8 + 2 * j], f.y * f_s[c8 * 8 + 2 * j + 1]);
    }
    P[i] = v;
  }
}

// ------------------------------------------------------------------ K4: Z = P^T X on tcgen05
// CTA: one hidden request x 128 columns of d.  D[128 heads x 128 cols] += P^T X over the
// request's 64-token k-blocks; A = P^T and B = X are both MN-major (P rows [token][Hp] and X
// rows [token][d] as stored), SWIZZLE_128B, loaded by TMA (P: 2 boxes of 64 heads x 64
// tokens, heads >= Hp zero-filled out of bounds; X: the request's pool blocks, 64-column
// boxes).  Token rows past n in the last k-block are zeroed in smem by the MMA warp (pool
// slots past n are never written; rows past the request's blocks belong to the next one).
// Epilogue: thread = head, Z row slice -> bf16.
template <int BN, int ST>
__global__ void __launch_bounds__(TC_THREADS, BN * ST <= 256 ? 3 : (BN == 128 ? 2 : 1))
    z_tc_kernel(const __grid_constant__ CUtensorMap tmap_x64, const __grid_constant__ CUtensorMap tmap_p,
                const AbsorbParams p) {
  constexpr int Z_ST = ST, Z_STAGE = 16384 + BN * 128, NCH = BN / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Z_ST * Z_STAGE);
  uint64_t* empty = full + Z_ST;
  uint64_t* tfull = empty + Z_ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, r = blockIdx.y;
  const int ntok = p.hntok[r], base = p.hrow0[r], B = p.B, H = p.H, d = p.d;
  const int nkb = (ntok + 63) / 64;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_x64);
    ptx::prefetch_tmap(&tmap_p);
    for (int s = 0; s < Z_ST; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      const int rpb = p.rpb64, nbox = 64 / rpb;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], Z_STAGE);
        uint8_t* a = smem + stage * Z_STAGE;
        uint8_t* b = a + 16384;
        ptx::tma_load_2d(a, &tmap_p, 0, base + kb * 64, &full[stage]);
        ptx::tma_load_2d(a + 8192, &tmap_p, 64, base + kb * 64, &full[stage]);
        for (int i = 0; i < nbox; ++i) {
          const int grow = base + kb * 64 + i * rpb, g = grow / B;
          const int prow = g < p.n_hb ? p.gather[g] * B + (grow - g * B) : 0;
#pragma unroll
          for (int j = 0; j < NCH; ++j)
            ptx::tma_load_2d(b + j * 8192 + i * rpb * 128, &tmap_x64, n0 + 64 * j, prow, &full[stage]);
        }
        if (++stage == Z_ST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // (a = P^T: M = heads, MN-major, 64-head chunks 8 KiB apart; b = X: N = columns)
    const uint32_t idesc = ptx::umma_idesc_bf16_f32(128, BN) | (1u << 15) | (1u << 16);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      ptx::mbar_wait(&full[stage], phase);
      uint8_t* a = smem + stage * Z_STAGE;
      const int valid = ntok - kb * 64;
      if (valid < 64) {   // zero X rows [valid, 64) of every 64-column chunk
        const int per = (64 - valid) * 8;
        for (int i = lane; i < NCH * per; i += 32) {
          const int ch = i / per, rem = i - ch * per;
          *reinterpret_cast<uint4*>(a + 16384 + ch * 8192 + (valid + (rem >> 3)) * 128 + (rem & 7) * 16) =
              make_uint4(0, 0, 0, 0);
        }
        ptx::fence_proxy_async_smem();
      }
      __syncwarp();
      if (lane == 0) {
        ptx::tc_fence_after();
        const uint32_t aa = ptx::smem_u32(a), bb = aa + 16384;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          ptx::umma_f16_ss(tmem, ptx::umma_desc_mn_sw128(aa + k * 2048, 8192), ptx::umma_desc_mn_sw128(bb + k * 2048, 8192),
                           idesc, (kb | k) != 0 ? 1u : 0u);
        ptx::umma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == Z_ST) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (lane == 0) ptx::umma_commit(tfull);
    __syncwarp();
  } else {
    const int q = warp & 3, h = q * 32 + lane;
    ptx::mbar_wait(tfull, 0);
    ptx::tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
      ptx::tmem_ld_wait();
      if (h < H) {
        uint4* dst = reinterpret_cast<uint4*>(p.z + ((size_t)h * p.n_h + r) * d + n0 + c);   // [H][n_h][d]
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_uint4(pk(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1])),
                              pk(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                              pk(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                              pk(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<BN>(tmem);
}

// ------------------------------------------------------------------ K1: q~ = W_K,h^T q_h on tcgen05
// CTA: 128 hidden requests x 256 columns of d, one head.  D[128 x 256] = A[128 x dh] B[dh x 256]:
// A = the requests' q_h rows, gathered by the 4 epilogue warps with cp.async straight into
// the K-major SWIZZLE_128B layout; B = W_K,h rows (dh x 256 columns, MN-major) by TMA.
// The blockIdx.x == 0 CTAs also store c = q_h . b_K,h (the score shift that only moves lse).
template <int DH, int BN>
__global__ void __launch_bounds__(TC_THREADS, BN == 128 ? 3 : 2)
    qt_tc_kernel(const __grid_constant__ CUtensorMap tmap_wk, const AbsorbParams p) {
  constexpr int NCH = DH / 64, A_BYTES = NCH * 128 * 128, B_BYTES = DH * BN * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + B_BYTES);
  uint64_t* a_full = bars;      // 128 gather threads
  uint64_t* b_full = bars + 1;  // TMA
  uint64_t* tfull = bars + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, h = blockIdx.y, r0 = blockIdx.z * 128;
  const int d = p.d, Hp = p.Hp;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_wk);
    ptx::mbar_init(a_full, 128);
    ptx::mbar_init(b_full, 1);
    ptx::mbar_init(tfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(p.q);
  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(b_full, B_BYTES);
      for (int j = 0; j < BN / 64; ++j)   // W_K,h rows h*2dh .. +dh, 64-column boxes
        ptx::tma_load_2d(sB + j * DH * 128, &tmap_wk, n0 + 64 * j, h * 2 * DH, b_full);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // A K-major; B MN-major (bit 16), 64-column chunks DH*128 bytes apart
      const uint32_t idesc = ptx::umma_idesc_bf16_f32(128, BN) | (1u << 16);
      ptx::mbar_wait(a_full, 0);
      ptx::mbar_wait(b_full, 0);
      ptx::tc_fence_after();
      const uint32_t aa = ptx::smem_u32(sA), bb = ptx::smem_u32(sB);
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk)
        ptx::umma_f16_ss(tmem, ptx::umma_desc_k_sw128(aa + (kk >> 2) * (128 * 128) + (kk & 3) * 32),
                         ptx::umma_desc_mn_sw128(bb + kk * 2048, DH * 128), idesc, kk != 0 ? 1u : 0u);
      ptx::umma_commit(tfull);
    }
    __syncwarp();
  } else {
    const int q4 = warp & 3, row = q4 * 32 + lane, r = r0 + row;
    const bool ok = r < p.n_h;
    const int req = ok ? p.hreq[r] : 0;
    // gather: this thread's request row, DH/8 16-byte chunks, swizzled
#pragma unroll
    for (int c = 0; c < DH / 8; ++c)
      cp16_zfill(sA + (c >> 3) * (128 * 128) + sw64(row, c & 7), q + (size_t)req * d + h * DH + c * 8, ok);
    cp_commit();
    cp_wait<0>();
    ptx::fence_proxy_async_smem();
    ptx::mbar_arrive(a_full);
    if (blockIdx.x == 0 && ok) {   // c = q_h . b_K,h
      float cb = 0.f;
      if (p.b_int) {
        const __nv_bfloat16* qr = q + (size_t)req * d + h * DH;
        for (int e = 0; e < DH; ++e) cb += __bfloat162float(qr[e]) * p.b_int[h * 2 * DH + e];
      }
      p.ml[3 * ((size_t)r * p.H + h) + 2] = cb;
    }
    ptx::mbar_wait(tfull, 0);
    ptx::tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(q4 * 32) << 16) + c, v);
      ptx::tmem_ld_wait();
      if (ok) {
        uint4* dst = reinterpret_cast<uint4*>(p.qt + ((size_t)r * Hp + h) * d + n0 + c);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_uint4(pk(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1])),
                              pk(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                              pk(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                              pk(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<BN>(tmem);
}

// ------------------------------------------------------------------ K5: o = W_V,h z / l + b_V on tcgen05
// CTA: one head x 128 hidden requests.  D[128 x dh] = Z_h [128 x d] W_V,h^T, both operands
// K-major by TMA (Z is head-major [H][n_h][d], so a head's rows are one block), 6-stage
// ring over d.  Epilogue: thread = request row: o = D / l + b_V, and lse.
template <int DH>
__global__ void __launch_bounds__(TC_THREADS, 1)
    wv_tc_kernel(const __grid_constant__ CUtensorMap tmap_z, const __grid_constant__ CUtensorMap tmap_wv,
                 const AbsorbParams p) {
  constexpr int ST = 6, A_BYTES = 128 * 128, STAGE = A_BYTES + DH * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x, r0 = blockIdx.y * 128, H = p.H, d = p.d;
  const int KC = d / 64;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_z);
    ptx::prefetch_tmap(&tmap_wv);
    for (int i = 0; i < ST; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<(DH < 32 ? 32 : DH)>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kc = 0; kc < KC; ++kc) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], STAGE);
        uint8_t* a = smem + stage * STAGE;
        ptx::tma_load_2d(a, &tmap_z, kc * 64, h * p.n_h + r0, &full[stage]);
        ptx::tma_load_2d(a + A_BYTES, &tmap_wv, kc * 64, h * 2 * DH + DH, &full[stage]);
        if (++stage == ST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc_bf16_f32(128, DH);
      int stage = 0;
      uint32_t phase = 0;
      for (int kc = 0; kc < KC; ++kc) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a = ptx::smem_u32(smem + stage * STAGE), b = a + A_BYTES;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          ptx::umma_f16_ss(tmem, ptx::umma_desc_k_sw128(a + k * 32), ptx::umma_desc_k_sw128(b + k * 32), idesc,
                           (kc | k) != 0 ? 1u : 0u);
        ptx::umma_commit(&empty[stage]);
        if (++stage == ST) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::umma_commit(tfull);
    }
    __syncwarp();
  } else {
    const int q4 = warp & 3, r = r0 + q4 * 32 + lane;
    ptx::mbar_wait(tfull, 0);
    ptx::tc_fence_after();
    const bool ok = r < p.n_h;
    const float* ml = p.ml + 3 * ((size_t)(ok ? r : 0) * H + h);
    const float inv = ok ? 1.f / ml[1] : 0.f;
    const int req = ok ? p.hreq[r] : 0;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out) + (size_t)req * d + h * DH;
#pragma unroll 1
    for (int c = 0; c < DH; c += 32) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(q4 * 32) << 16) + c, v);
      ptx::tmem_ld_wait();
      if (ok) {
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
          f[j] = __uint_as_float(v[j]) * inv + (p.b_int ? p.b_int[h * 2 * DH + DH + c + j] : 0.f);
        uint4* dst = reinterpret_cast<uint4*>(out + c);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_uint4(pk(f[8 * j], f[8 * j + 1]), pk(f[8 * j + 2], f[8 * j + 3]), pk(f[8 * j + 4], f[8 * j + 5]),
                              pk(f[8 * j + 6], f[8 * j + 7]));
      }
    }
    if (ok && p.lse) p.lse[(size_t)req * H + h] = (ml[0] + log2f(ml[1])) * 0.69314718055994531f + p.scale * ml[2];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<(DH < 32 ? 32 : DH)>(tmem);
}

}  // namespace

bool absorb_supported(int dtype, int d, int dh, int H, int B) {
  return dtype == 0 && d % 128 == 0 && dh % 16 == 0 && dh <= 128 && H <= 128 && B % 8 == 0 &&
         (128 % B == 0 || B % 128 == 0);
}

int absorb_launches() { return 5; }

template <int BN, int ST>
static cudaError_t launch_z(const AbsorbParams& p, const CUtensorMap& tx, const CUtensorMap& tp, cudaStream_t s) {
  constexpr int smem = 1024 + ST * (16384 + BN * 128) + 256;
  static const cudaError_t attr =
      cudaFuncSetAttribute(z_tc_kernel<BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (attr != cudaSuccess) return attr;
  z_tc_kernel<BN, ST><<<dim3(p.d / BN, p.n_h), TC_THREADS, smem, s>>>(tx, tp, p);
  return cudaGetLastError();
}

template <int DH, int BN>
static cudaError_t launch_qt(const AbsorbParams& p, const CUtensorMap& twk, cudaStream_t s) {
  constexpr int smem = 1024 + (DH / 64) * 128 * 128 + DH * BN * 2 + 256;
  static const cudaError_t attr =
      cudaFuncSetAttribute(qt_tc_kernel<DH, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (attr != cudaSuccess) return attr;
  qt_tc_kernel<DH, BN><<<dim3(p.d / BN, p.H, (p.n_h + 127) / 128), TC_THREADS, smem, s>>>(twk, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || p.Hp == p.H) return e;
  // padding heads H..Hp-1 of q~ are zero rows (the score GEMM's B operand is Hp rows wide)
  const size_t row = (size_t)p.d * 2;
  return cudaMemset2DAsync(p.qt + (size_t)p.H * p.d, p.Hp * row, 0, (size_t)(p.Hp - p.H) * row, p.n_h, s);
}

template <int DH>
static cudaError_t launch_wv(const AbsorbParams& p, const CUtensorMap& tz, const CUtensorMap& twv, cudaStream_t s) {
  constexpr int smem = 1024 + 6 * (128 * 128 + DH * 128) + 256;
  static const cudaError_t attr =
      cudaFuncSetAttribute(wv_tc_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (attr != cudaSuccess) return attr;
  wv_tc_kernel<DH><<<dim3(p.H, (p.n_h + 127) / 128), TC_THREADS, smem, s>>>(tz, twv, p);
  return cudaGetLastError();
}

cudaError_t launch_absorbed(const AbsorbParams& p, const void* tmap_x, const void* tmap_x64, const void* tmap_qt,
                            const void* tmap_p, const void* tmap_wk, const void* tmap_z, const void* tmap_wv,
                            const Tuning& t, cudaStream_t s) {
  if (p.n_h <= 0) return cudaSuccess;
  constexpr int smem_tc = 1024 + 3 * 32768 + 256 + 512;
  const int zcfg = t.z_cfg;     // Z GEMM tile width x pipeline depth (default 128x2: 3 CTAs per SM)
  const int sst = t.score_st;   // score GEMM stages: 2 (3 CTAs/SM, default) or 3
  constexpr int smem_s2 = 1024 + 128 * 129 * 4 + 256 + 512;
  static const cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(score_tc_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(score_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s2);
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  cudaError_t e;
  const CUtensorMap& twk = *static_cast<const CUtensorMap*>(tmap_wk);
  const int qbn = t.qt_bn == 256 ? 256 : 128;   // q~ GEMM tile width (128 also serves d % 256 != 0)
  if (qbn == 256 && p.d % 256 == 0)
    e = p.dh == 128 ? launch_qt<128, 256>(p, twk, s) : launch_qt<64, 256>(p, twk, s);
  else
    e = p.dh == 128 ? launch_qt<128, 128>(p, twk, s) : launch_qt<64, 128>(p, twk, s);
  if (e != cudaSuccess) return e;
  if (sst == 2)
    score_tc_kernel<2><<<p.n_tiles, TC_THREADS, smem_s2, s>>>(*static_cast<const CUtensorMap*>(tmap_x),
                                                              *static_cast<const CUtensorMap*>(tmap_qt), p);
  else
    score_tc_kernel<3><<<p.n_tiles, TC_THREADS, smem_tc, s>>>(*static_cast<const CUtensorMap*>(tmap_x),
                                                              *static_cast<const CUtensorMap*>(tmap_qt), p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  rescale_kernel<<<p.n_tiles, 128, 0, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const CUtensorMap& tx = *static_cast<const CUtensorMap*>(tmap_x64);
  const CUtensorMap& tp = *static_cast<const CUtensorMap*>(tmap_p);
  if (zcfg == 2564 && p.d % 256 == 0)
    e = launch_z<256, 4>(p, tx, tp, s);
  else if (zcfg == 1283)
    e = launch_z<128, 3>(p, tx, tp, s);
  else
    e = launch_z<128, 2>(p, tx, tp, s);
  if (e != cudaSuccess) return e;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const CUtensorMap& tz = *static_cast<const CUtensorMap*>(tmap_z);
  const CUtensorMap& twv = *static_cast<const CUtensorMap*>(tmap_wv);
  return p.dh == 128 ? launch_wv<128>(p, tz, twv, s) : launch_wv<64>(p, tz, twv, s);
}

}  // namespace hc
