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
//   K1 qt_kernel       q~[r][h][:] = W_K,h^T q_{r,h} (per head [n_h x dh][dh x d], warp MMA);
//                      q_h . b_K,h
//   K2 score_tc_kernel per 128-token tile of request r (tcgen05): s = x . q~[r][h]; tile max
//                      m_t[h], P[row][h] = 2^(scaled s - m_t) (bf16), l_t[h] = sum P
//   K3 rescale_kernel  m[h] = max_t m_t, P *= 2^(m_t - m), l = sum_t 2^(m_t - m) l_t
//   K4 z_tc_kernel     Z[r][h][:] = sum_rows P[row][h] x_row (tcgen05, MN-major operands)
//   K5 wv_kernel       out[r][h*dh:] = W_V,h Z[r][h] / l + b_V,h;  lse (warp MMA)
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
  const int dh = p.dh, d = p.d, Hp = p.Hp;
  if (h >= p.H) {   // padding heads of q~ (rows H..Hp-1 of each request) are zero
    for (int i = threadIdx.x; i < 64 * 16; i += 128) {
      const int rr = r0 + (i >> 4);
      if (rr < p.n_h) reinterpret_cast<uint4*>(p.qt + ((size_t)rr * Hp + h) * d + n0)[i & 15] = make_uint4(0, 0, 0, 0);
    }
    return;
  }
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
  if (blockIdx.x == 0 && tid < 64 && r0 + tid < p.n_h) {   // c = q_h . b_K,h (shifts lse only)
    float c = 0.f;
    if (p.b_int) {
      const __nv_bfloat16* qr = q + (size_t)p.hreq[r0 + tid] * d + h * dh;
      for (int e = 0; e < dh; ++e) c += __bfloat162float(qr[e]) * p.b_int[h * 2 * dh + e];
    }
    p.ml[3 * ((size_t)(r0 + tid) * p.H + h) + 2] = c;
  }
  const int g = lane >> 2, t4 = lane & 3;
  __nv_bfloat16* qt = p.qt;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = n0 + j * 8 + 2 * t4;
    const int ra = r0 + warp * 16 + g, rb = ra + 8;
    if (ra < p.n_h) *reinterpret_cast<uint32_t*>(qt + ((size_t)ra * Hp + h) * d + col) = pk(acc[j][0], acc[j][1]);
    if (rb < p.n_h) *reinterpret_cast<uint32_t*>(qt + ((size_t)rb * Hp + h) * d + col) = pk(acc[j][2], acc[j][3]);
  }
}

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
        uint4* dst = reinterpret_cast<uint4*>(p.z + ((size_t)r * H + h) * d + n0 + c);
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

// ------------------------------------------------------------------ K5: o = W_V,h z / l + b_V
constexpr int kST = 4;   // cp.async pipeline depth of K5
// CTA: 64 hidden requests x dh outputs of one head, K loop over d in 64s.  A = Z[r][h]
// rows (K contiguous), B = W_V,h [dh x d] rows (N x K, K contiguous -> non-trans).
__global__ void __launch_bounds__(128) wv_kernel(const AbsorbParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int dh = p.dh, d = p.d, H = p.H;
  const int stage_bytes = 64 * 128 + dh * 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.x, r0 = blockIdx.y * 64;
  const __nv_bfloat16* w = static_cast<const __nv_bfloat16*>(p.w_int);
  auto load = [&](int kc, int st) {
    uint8_t* a = sm + st * stage_bytes;
    uint8_t* b = a + 64 * 128;
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
#pragma unroll
  for (int st = 0; st < kST - 1; ++st) {
    if (st < KC) load(st, st);
    cp_commit();
  }
  const int mat = lane >> 3, rr = lane & 7;
  for (int kc = 0; kc < KC; ++kc) {
    cp_wait<kST - 2>();
    __syncthreads();
    const uint32_t a_s = saddr(sm + (kc % kST) * stage_bytes), b_s = a_s + 64 * 128;
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
    const int nk = kc + kST - 1;
    if (nk < KC) load(nk, nk % kST);
    cp_commit();
  }
  cp_wait<0>();
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

cudaError_t launch_absorbed(const AbsorbParams& p, const void* tmap_x, const void* tmap_x64, const void* tmap_qt,
                            const void* tmap_p, cudaStream_t s) {
  if (p.n_h <= 0) return cudaSuccess;
  constexpr int smem_tc = 1024 + 3 * 32768 + 256 + 512;
  static const int zcfg = [] {   // Z GEMM tile width x pipeline depth (A/B knob; default 128x2: 3 CTAs per SM)
    const char* e = std::getenv("HC_Z_CFG");
    return e ? std::atoi(e) : 1282;
  }();
  static const int sst = [] {
    const char* e = std::getenv("HC_SCORE_ST");   // A/B knob: 2 stages (3 CTAs/SM, default) or 3
    return e ? std::atoi(e) : 2;
  }();
  constexpr int smem_s2 = 1024 + 128 * 129 * 4 + 256 + 512;
  static const cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(score_tc_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(score_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s2);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(wv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kST * (64 * 128 + 128 * 128));
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  cudaError_t e;
  qt_kernel<<<dim3(p.d / 128, p.Hp, (p.n_h + 63) / 64), 128, 0, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
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
  const int smem5 = kST * (64 * 128 + p.dh * 128);
  wv_kernel<<<dim3(p.H, (p.n_h + 63) / 64), 128, smem5, s>>>(p);
  return cudaGetLastError();
}

}  // namespace hc
