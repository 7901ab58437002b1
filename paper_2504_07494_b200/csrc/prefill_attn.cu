// Causal self-attention over each request's new tokens: the prefill / recompute path
// (NEXT row f3; P:180-182 prefill, P:297 fn recompute after preemption, P:392 after a
// cache-type switch).  Eq. 2-3 with the causal index range j <= i.
//
// prefill_attn_mma_kernel (bf16, dh 64/128): FlashAttention-2 style — a CTA of 4 warps owns
// 64 query rows of one (request, head); K/V tiles of 64 tokens stream through a
// cp.async double buffer in XOR-swizzled shared memory; S = Q K^T and O += P V run on
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate) with ldmatrix fragment loads; online
// softmax in exp2 with the scale folded in; the S accumulator is re-packed in registers as
// the A operand of P V.  (First version of this row: the sm_80-style tensor-core path;
// a tcgen05/TMEM version is the next step.)
// prefill_attn_tc_kernel (bf16, dh 64/128, default): the same computation on tcgen05 —
// see the kernel's comment.  prefill_attn_mma_kernel stays as the cross-check path
// (HC_PREFILL_TC=0).
// prefill_attn_simt_kernel: one warp per (query row, head), any dtype / dh (fp32 mode).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace hc {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int QT = 64, KT = 64;   // query rows per CTA, keys per tile

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Swizzled tile of R rows x DH bf16: 16-byte chunk c of row r lives at chunk c ^ (r & 7).
template <int DH>
__device__ __forceinline__ uint32_t swz(int r, int chunk) {
  return (uint32_t)(r * DH * 2 + ((chunk ^ (r & 7)) << 4));
}

template <int DH>
__global__ void __launch_bounds__(128) prefill_attn_mma_kernel(const PrefillAttnParams p) {
  constexpr int CH = DH / 8;         // 16-byte chunks per row
  constexpr int KS = DH / 16;        // k-steps of Q K^T
  constexpr int NO = DH / 8;         // n-tiles of the O accumulator
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* sQ = sm;
  uint8_t* sK = sm + QT * DH * 2;              // 2 buffers
  uint8_t* sV = sK + 2 * KT * DH * 2;          // 2 buffers
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y;
  const int req = p.tile_req[blockIdx.x], q0 = p.tile_q0[blockIdx.x];
  const int row0 = p.row0[req], L = p.row0[req + 1] - row0;
  const int d = p.d;
  const __nv_bfloat16* Q = static_cast<const __nv_bfloat16*>(p.q);
  const __nv_bfloat16* KV = static_cast<const __nv_bfloat16*>(p.kv);

  auto load_q = [&]() {
    for (int i = tid; i < QT * CH; i += 128) {
      const int r = i / CH, c = i - r * CH;
      const int tok = min(q0 + r, L - 1);
      cp_async16(sQ + swz<DH>(r, c), Q + (size_t)(row0 + tok) * d + h * DH + c * 8);
    }
  };
  auto load_kv = [&](int t, int buf) {
    uint8_t* k = sK + buf * KT * DH * 2;
    uint8_t* v = sV + buf * KT * DH * 2;
    for (int i = tid; i < KT * CH; i += 128) {
      const int r = i / CH, c = i - r * CH;
      const int tok = min(t * KT + r, L - 1);
      const __nv_bfloat16* src = KV + (size_t)(row0 + tok) * 2 * p.dk + (h / p.G) * 2 * DH + c * 8;
      cp_async16(k + swz<DH>(r, c), src);
      cp_async16(v + swz<DH>(r, c), src + DH);
    }
  };
  const int n_kv_tiles = (min(q0 + QT, L) + KT - 1) / KT;   // causal: keys up to the tile's last query
  load_q();
  load_kv(0, 0);
  cp_commit();

  // per-warp state: 16 query rows (g = lane/4: rows g and g+8 of the warp's 16)
  uint32_t qa[KS][4];
  float o[NO][4];
#pragma unroll
  for (int i = 0; i < NO; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int g = lane >> 2, t4 = lane & 3;
  const int qr0 = q0 + warp * 16 + g, qr1 = qr0 + 8;   // query token indices of this lane's rows

  for (int t = 0; t < n_kv_tiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < n_kv_tiles) load_kv(t + 1, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int mat = lane >> 3, r = lane & 7;
        const int row = warp * 16 + ((mat & 1) << 3) + r, chunk = 2 * ks + (mat >> 1);
        ldsm_x4(smem_addr(sQ) + swz<DH>(row, chunk), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
      }
    }
    const uint32_t kbase = smem_addr(sK + buf * KT * DH * 2), vbase = smem_addr(sV + buf * KT * DH * 2);
    // ---- S = Q K^T (16 x 64 per warp)
    float s[KT / 8][4];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int nj = 0; nj < KT / 16; ++nj) {
        const int mat = lane >> 3, r = lane & 7;
        const int krow = nj * 16 + ((mat >> 1) << 3) + r, chunk = 2 * ks + (mat & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kbase + swz<DH>(krow, chunk), b0, b1, b2, b3);
        mma_bf16(s[2 * nj], qa[ks], b0, b1);
        mma_bf16(s[2 * nj + 1], qa[ks], b2, b3);
      }
    }
    // ---- scale, causal / length mask, online softmax (rows qr0, qr1)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
      const int kc = t * KT + j * 8 + 2 * t4;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int kj = kc + e;
        s[j][e] = (kj <= qr0 && kj < L) ? s[j][e] * p.scale_log2 : -INFINITY;
        s[j][2 + e] = (kj <= qr1 && kj < L) ? s[j][2 + e] * p.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[j][e]);
        mx1 = fmaxf(mx1, s[j][2 + e]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(FULL, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(FULL, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(FULL, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(FULL, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    // rows with no valid key yet (only possible for padding rows) keep a finite reference
    const float r0 = mn0 == -INFINITY ? 0.f : mn0, r1 = mn1 == -INFINITY ? 0.f : mn1;
    const float al0 = ex2(m0 - r0), al1 = ex2(m1 - r1);
    float ps0 = 0.f, ps1 = 0.f;
    uint32_t pa[KT / 16][4];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
      const float p00 = ex2(s[j][0] - r0), p01 = ex2(s[j][1] - r0);
      const float p10 = ex2(s[j][2] - r1), p11 = ex2(s[j][3] - r1);
      ps0 += p00 + p01;
      ps1 += p10 + p11;
      // C fragment of n-tile j -> A fragment of k-step j/2 (keys 16*(j/2) .. +15)
      pa[j >> 1][(j & 1) * 2 + 0] = pack2(p00, p01);
      pa[j >> 1][(j & 1) * 2 + 1] = pack2(p10, p11);
    }
    l0 = l0 * al0 + ps0;
    l1 = l1 * al1 + ps1;
    m0 = mn0;
    m1 = mn1;
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      o[i][0] *= al0;
      o[i][1] *= al0;
      o[i][2] *= al1;
      o[i][3] *= al1;
    }
    // ---- O += P V
#pragma unroll
    for (int kk = 0; kk < KT / 16; ++kk) {
      // A fragment order for m16n8k16: {row g k0-7, row g+8 k0-7, row g k8-15, row g+8 k8-15}
      const uint32_t a[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
#pragma unroll
      for (int nd = 0; nd < DH / 16; ++nd) {
        const int mat = lane >> 3, r = lane & 7;
        const int vrow = kk * 16 + ((mat & 1) << 3) + r, chunk = 2 * nd + (mat >> 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vbase + swz<DH>(vrow, chunk), b0, b1, b2, b3);
        mma_bf16(o[2 * nd], a, b0, b1);
        mma_bf16(o[2 * nd + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  // ---- finalize: row sums across the 4 lanes of a row, normalise, store bf16
  l0 += __shfl_xor_sync(FULL, l0, 1);
  l0 += __shfl_xor_sync(FULL, l0, 2);
  l1 += __shfl_xor_sync(FULL, l1, 1);
  l1 += __shfl_xor_sync(FULL, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  __nv_bfloat16* O = static_cast<__nv_bfloat16*>(p.o);
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    const int col = h * DH + i * 8 + 2 * t4;
    if (qr0 < L)
      *reinterpret_cast<uint32_t*>(O + (size_t)(row0 + qr0) * d + col) = pack2(o[i][0] * inv0, o[i][1] * inv0);
    if (qr1 < L)
      *reinterpret_cast<uint32_t*>(O + (size_t)(row0 + qr1) * d + col) = pack2(o[i][2] * inv1, o[i][3] * inv1);
  }
}


// ------------------------------------------------------------------ tcgen05 / TMEM version
// CTA = 128 query rows of one (request, head); 6 warps:
//   warp 0     TMA producer: Q tile once, then K and V tiles of 128 keys (64-column boxes of
//              the head's K_h || V_h slices of the projection output), 2-stage ring.
//   warp 1     TMEM allocator + MMA issuer: S_j = Q K_j^T (M=128, N=128 keys, K=dh; both
//              operands K-major) into one of two TMEM S buffers, issued one tile ahead so it
//              overlaps the softmax of the previous tile; O += P_j V_j (M=128, N=dh, K=128
//              keys; P from shared memory K-major, V as stored = MN-major) into TMEM.
//   warps 2-5  softmax, thread = query row (TMEM lane): tcgen05.ld the S row, causal and
//              length mask, exp2 with the scale folded in, P row -> swizzled smem (bf16).
//              Lazy rescaling (the reference max only moves when a row max exceeds it by
//              more than 2^8): O rows are rescaled in TMEM (ld / scale / st) only then;
//              P <= 2^8 in bf16 is exact enough and l is fp32.  Epilogue: O / l -> bf16.
// TMEM: S0 cols [0,128), S1 [128,256), O [256, 256+dh).
// NQ = query tiles of 128 rows per CTA sharing every K/V tile (NQ = 2: FlashAttention-4
// style pair of softmax warpgroups that ping-pong on the tensor core); ST = K/V stages.
template <int DH, int BK, int NQ, int ST>
__global__ void __launch_bounds__(64 + 128 * NQ, (BK == 64 && NQ == 1) ? 2 : 1)
    prefill_attn_tc_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_kv,
                           const PrefillAttnParams p) {
  constexpr int BM = 128, NCH = DH / 64, NPC = BK / 64;
  constexpr int QCH = 128 * 128;                   // Q / P chunk: 128 rows x 64 columns (16 KiB)
  constexpr int KCH = BK * 128;                    // K / V chunk: BK rows x 64 columns
  constexpr int Q_OFF = 0, K_OFF = NQ * NCH * QCH, V_OFF = K_OFF + ST * NCH * KCH;
  constexpr int P_OFF = V_OFF + ST * NCH * KCH, BAR_OFF = P_OFF + NQ * NPC * QCH;
  // TMEM per query tile: S buffers [0, 2 BK), O [2 BK, 2 BK + DH); tiles TCOLS apart
  constexpr uint32_t O_COL = 2 * BK, TCOLS = (2 * BK + DH <= 256) ? 256 : 512;
  constexpr uint32_t TMEM_ALLOC = NQ * TCOLS;
  static_assert(TMEM_ALLOC <= 512, "TMEM");
  constexpr float kRescale = 8.f;                  // log2 headroom before O is rescaled
  // no alignment slack (two CTAs per SM need every KiB): the dynamic window is 1024-aligned
  // when the kernel has no static shared memory; trap otherwise rather than overflow
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem) & 1023) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;                    // [ST]
  uint64_t* kv_empty = kv_full + ST;               // [ST]
  uint64_t* s_full = kv_empty + ST;                // [NQ][2]
  uint64_t* s_free = s_full + 2 * NQ;              // [NQ][2]
  uint64_t* p_full = s_free + 2 * NQ;              // [NQ]
  uint64_t* o_done = p_full + NQ;                  // [NQ]
  uint64_t* o_final = o_done + NQ;                 // [NQ]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + NQ);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y;
  const int req = p.tile_req[blockIdx.x], q0 = p.tile_q0[blockIdx.x];
  const int row0 = p.row0[req], L = p.row0[req + 1] - row0;
  // key tiles each query tile needs (causal: up to its last query); 0 = tile past L
  int ntq[NQ];
#pragma unroll
  for (int qt = 0; qt < NQ; ++qt)
    ntq[qt] = q0 + qt * BM < L ? (min(q0 + (qt + 1) * BM, L) + BK - 1) / BK : 0;
  const int nt = ntq[0] > ntq[NQ - 1] ? ntq[0] : ntq[NQ - 1];
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_q);
    ptx::prefetch_tmap(&tmap_kv);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < ST; ++i) {
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2 * NQ; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 128);
    }
    for (int i = 0; i < NQ; ++i) {
      ptx::mbar_init(&p_full[i], 128);
      ptx::mbar_init(&o_done[i], 1);
      ptx::mbar_init(&o_final[i], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_ALLOC>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(q_full, NQ * NCH * QCH);
      for (int qt = 0; qt < NQ; ++qt)
        for (int c = 0; c < NCH; ++c)
          ptx::tma_load_2d(smem + Q_OFF + (qt * NCH + c) * QCH, &tmap_q, h * DH + c * 64, row0 + q0 + qt * BM, q_full);
      for (int t = 0; t < nt; ++t) {
        const int st = t % ST;
        ptx::mbar_wait(&kv_empty[st], ((t / ST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[st], 2 * NCH * KCH);
        for (int c = 0; c < NCH; ++c) {
          ptx::tma_load_2d(smem + K_OFF + (st * NCH + c) * KCH, &tmap_kv, (h / p.G) * 2 * DH + c * 64,
                           row0 + t * BK, &kv_full[st]);
          ptx::tma_load_2d(smem + V_OFF + (st * NCH + c) * KCH, &tmap_kv, (h / p.G) * 2 * DH + DH + c * 64,
                           row0 + t * BK, &kv_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = ptx::umma_idesc_bf16_f32(BM, BK);
      constexpr uint32_t idesc_o = ptx::umma_idesc_bf16_f32(BM, DH) | (1u << 16);   // B (V) MN-major
      auto issue_s = [&](int qt, int t) {
        const int st = t % ST, b = t & 1;
        ptx::mbar_wait(&kv_full[st], (t / ST) & 1);
        ptx::mbar_wait(&s_free[2 * qt + b], ((t >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t sq = ptx::smem_u32(smem + Q_OFF + qt * NCH * QCH);
        const uint32_t sk = ptx::smem_u32(smem + K_OFF + st * NCH * KCH);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          ptx::umma_f16_ss(tmem + qt * TCOLS + b * BK, ptx::umma_desc_k_sw128(sq + (kk >> 2) * QCH + (kk & 3) * 32),
                           ptx::umma_desc_k_sw128(sk + (kk >> 2) * KCH + (kk & 3) * 32), idesc_s, kk != 0 ? 1u : 0u);
        ptx::umma_commit(&s_full[2 * qt + b]);
      };
      ptx::mbar_wait(q_full, 0);
      for (int qt = 0; qt < NQ; ++qt)
        if (ntq[qt] > 0) issue_s(qt, 0);
      for (int t = 0; t < nt; ++t) {
        for (int qt = 0; qt < NQ; ++qt)
          if (t + 1 < ntq[qt]) issue_s(qt, t + 1);
        const uint32_t sv = ptx::smem_u32(smem + V_OFF + (t % ST) * NCH * KCH);
        for (int qt = 0; qt < NQ; ++qt) {
          if (t >= ntq[qt]) continue;
          ptx::mbar_wait(&p_full[qt], t & 1);
          ptx::tc_fence_after();
          const uint32_t sp = ptx::smem_u32(smem + P_OFF + qt * NPC * QCH);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            ptx::umma_f16_ss(tmem + qt * TCOLS + O_COL, ptx::umma_desc_k_sw128(sp + (kk >> 2) * QCH + (kk & 3) * 32),
                             ptx::umma_desc_mn_sw128(sv + kk * 2048, KCH), idesc_o, (t | kk) != 0 ? 1u : 0u);
          ptx::umma_commit(&o_done[qt]);
        }
        ptx::umma_commit(&kv_empty[t % ST]);
      }
      for (int qt = 0; qt < NQ; ++qt) ptx::umma_commit(&o_final[qt]);
    }
    __syncwarp();
  } else {
    const int qt = (warp - 2) >> 2;                // query tile of this softmax warpgroup
    const int quad = warp & 3, row = quad * 32 + lane;
    const int qi = q0 + qt * BM + row;             // query token index (>= L: padding row)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tq = tmem + qt * TCOLS, tmem_o = tq + O_COL;
    const float sl = p.scale_log2;
    float m_ref = -INFINITY, l = 0.f;
    uint8_t* sP = smem + P_OFF + qt * NPC * QCH;
    const int my_nt = ntq[qt];
    for (int t = 0; t < my_nt; ++t) {
      const int b = t & 1;
      ptx::mbar_wait(&s_full[2 * qt + b], (t >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t v[BK / 32][32];
#pragma unroll
      for (int c = 0; c < BK / 32; ++c) ptx::tmem_ld_32x32b_x32(tq + lane_off + b * BK + c * 32, v[c]);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&s_free[2 * qt + b]);
      // keys k0 + j valid iff k0 + j <= qi and < L
      const int lim = min(qi, L - 1) - t * BK;     // last valid j (may be >= BK-1 or < 0)
      float sv[BK];
#pragma unroll
      for (int c = 0; c < BK / 32; ++c)
#pragma unroll
        for (int j = 0; j < 32; ++j) sv[c * 32 + j] = __uint_as_float(v[c][j]) * sl;
      if (lim < BK - 1) {   // diagonal / last tile: mask
#pragma unroll
        for (int j = 0; j < BK; ++j)
          if (j > lim) sv[j] = -INFINITY;
      }
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};   // 4 independent chains
#pragma unroll
      for (int j = 0; j < BK; ++j) mx4[j & 3] = fmaxf(mx4[j & 3], sv[j]);
      const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      float scale_o = 1.f;
      if (t == 0) {
        m_ref = mx;
      } else if (mx > m_ref + kRescale) {
        scale_o = ex2(m_ref - mx);
        l *= scale_o;
        m_ref = mx;
      }
      float ps4[4] = {0.f, 0.f, 0.f, 0.f};
      uint32_t pk[BK / 2];
#pragma unroll
      for (int j = 0; j < BK; j += 2) {
        const float e0 = ex2(sv[j] - m_ref), e1 = ex2(sv[j + 1] - m_ref);   // ex2(-inf) = 0
        ps4[(j >> 1) & 3] += e0 + e1;
        pk[j / 2] = pack2(e0, e1);
      }
      l += (ps4[0] + ps4[1]) + (ps4[2] + ps4[3]);
      if (t > 0) {
        ptx::mbar_wait(&o_done[qt], (t - 1) & 1);  // PV_{t-1} retired: P buffer free, O stable
        ptx::tc_fence_after();
        if (scale_o != 1.f) {
#pragma unroll 1
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(tmem_o + lane_off + c * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * scale_o);
            ptx::tmem_st_32x32b_x32(tmem_o + lane_off + c * 32, o);
          }
          ptx::tmem_st_wait();
        }
      }
      // P row -> K-major SWIZZLE_128B tile: chunk (8 keys) c of row r at (c ^ (r & 7)) within
      // its 64-key chunk
#pragma unroll
      for (int c = 0; c < BK / 8; ++c) {
        uint4* dst = reinterpret_cast<uint4*>(sP + (c >> 3) * QCH + row * 128 + (((c & 7) ^ (row & 7)) << 4));
        *dst = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&p_full[qt]);
    }
    if (my_nt > 0) {
      ptx::mbar_wait(&o_final[qt], 0);
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      __nv_bfloat16* O = static_cast<__nv_bfloat16*>(p.o);
#pragma unroll 1
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        ptx::tmem_ld_32x32b_x32(tmem_o + lane_off + c * 32, o);
        ptx::tmem_ld_wait();
        if (qi < L) {
          uint4* dst = reinterpret_cast<uint4*>(O + (size_t)(row0 + qi) * p.d + h * DH + c * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j] = make_uint4(pack2(__uint_as_float(o[8 * j]) * inv, __uint_as_float(o[8 * j + 1]) * inv),
                                pack2(__uint_as_float(o[8 * j + 2]) * inv, __uint_as_float(o[8 * j + 3]) * inv),
                                pack2(__uint_as_float(o[8 * j + 4]) * inv, __uint_as_float(o[8 * j + 5]) * inv),
                                pack2(__uint_as_float(o[8 * j + 6]) * inv, __uint_as_float(o[8 * j + 7]) * inv));
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<TMEM_ALLOC>(tmem);
}

// ------------------------------------------------------------------ SIMT fallback
template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void stf(T* p, float v);
template <>
__device__ __forceinline__ void stf<float>(float* p, float v) {
  *p = v;
}
template <>
__device__ __forceinline__ void stf<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

// one warp per (query row of a tile, head); grid (n_qtiles, H), 4 warps loop over the tile's rows
template <typename T>
__global__ void __launch_bounds__(128) prefill_attn_simt_kernel(const PrefillAttnParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y, DH = p.dh, d = p.d;
  const int req = p.tile_req[blockIdx.x], q0 = p.tile_q0[blockIdx.x];
  const int row0 = p.row0[req], L = p.row0[req + 1] - row0;
  const T* Q = static_cast<const T*>(p.q);
  const T* KV = static_cast<const T*>(p.kv);
  T* O = static_cast<T*>(p.o);
  __shared__ float qs[4][256];
  for (int qi = q0 + warp; qi < min(q0 + QT, L); qi += 4) {
    for (int c = lane; c < DH; c += 32) qs[warp][c] = ldf(Q + (size_t)(row0 + qi) * d + h * DH + c) * p.scale_log2;
    __syncwarp();
    float m = -INFINITY, l = 0.f, acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j0 = 0; j0 <= qi; j0 += 32) {
      const int j = j0 + lane;
      float sc = -INFINITY;
      if (j <= qi) {
        const T* kr = KV + (size_t)(row0 + j) * 2 * p.dk + (h / p.G) * 2 * DH;
        float a = 0.f;
        for (int c = 0; c < DH; ++c) a += qs[warp][c] * ldf(kr + c);
        sc = a;
      }
      float mx = sc;
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
      const float mn = fmaxf(m, mx);
      const float pj = j <= qi ? exp2f(sc - mn) : 0.f;
      const float al = exp2f(m - mn);
      float ps = pj;
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(FULL, ps, o);
      l = l * al + ps;
      for (int i = 0; i < 8; ++i) acc[i] *= al;
      const int cnt = min(32, qi + 1 - j0);
      for (int jj = 0; jj < cnt; ++jj) {
        const float pw = __shfl_sync(FULL, pj, jj);
        const T* vr = KV + (size_t)(row0 + j0 + jj) * 2 * p.dk + (h / p.G) * 2 * DH + DH;
        for (int i = 0; i < 8; ++i) {
          const int c = lane + 32 * i;
          if (c < DH) acc[i] += pw * ldf(vr + c);
        }
      }
      m = mn;
    }
    for (int i = 0; i < 8; ++i) {
      const int c = lane + 32 * i;
      if (c < DH) stf(O + (size_t)(row0 + qi) * d + h * DH + c, acc[i] / l);
    }
    __syncwarp();
  }
}

}  // namespace

bool prefill_attn_mma_supported(int dtype, int dh) { return dtype == 0 && (dh == 128 || dh == 64); }

// Configuration of the tcgen05 prefill kernel (A/B knob HC_PREFILL_CFG): 1 = one query tile
// per CTA, 64-key tiles, 2 K/V stages, two CTAs per SM (default, fastest measured);
// 2 = two query tiles per CTA sharing 3 K/V stages (FA4-style pair of softmax warpgroups);
// 128 = one query tile, 128-key tiles.
static int prefill_attn_tc_cfg(const Tuning& t) {
  const int v = t.prefill_cfg;
  return (v == 2 || v == 128) ? v : 1;
}
int prefill_attn_tc_keys(const Tuning& t) { return prefill_attn_tc_cfg(t) == 128 ? 128 : 64; }
int prefill_attn_tc_rows(const Tuning& t) { return prefill_attn_tc_cfg(t) == 2 ? 256 : 128; }

template <int DH, int BK, int NQ, int ST>
static cudaError_t launch_tc(const PrefillAttnParams& p, const CUtensorMap& tq, const CUtensorMap& tkv,
                             cudaStream_t s) {
  constexpr int NCH = DH / 64;
  constexpr int smem = NQ * NCH * 128 * 128 + 2 * ST * NCH * BK * 128 + NQ * (BK / 64) * 128 * 128 + 256;
  static const cudaError_t a =
      cudaFuncSetAttribute(prefill_attn_tc_kernel<DH, BK, NQ, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (a != cudaSuccess) return a;
  prefill_attn_tc_kernel<DH, BK, NQ, ST><<<dim3(p.n_qtiles, p.H), 64 + 128 * NQ, smem, s>>>(tq, tkv, p);
  return cudaGetLastError();
}

cudaError_t launch_prefill_attn_tc(const PrefillAttnParams& p, const void* tmap_q, const void* tmap_kv,
                                   const Tuning& t, cudaStream_t s) {
  if (p.n_qtiles <= 0) return cudaSuccess;
  const CUtensorMap& tq = *static_cast<const CUtensorMap*>(tmap_q);
  const CUtensorMap& tkv = *static_cast<const CUtensorMap*>(tmap_kv);
  const int cfg = prefill_attn_tc_cfg(t);
  if (p.dh == 128) {
    if (cfg == 128) return launch_tc<128, 128, 1, 2>(p, tq, tkv, s);
    if (cfg == 1) return launch_tc<128, 64, 1, 2>(p, tq, tkv, s);
    return launch_tc<128, 64, 2, 3>(p, tq, tkv, s);
  }
  if (p.dh == 64) {
    if (cfg == 128) return launch_tc<64, 128, 1, 2>(p, tq, tkv, s);
    if (cfg == 1) return launch_tc<64, 64, 1, 2>(p, tq, tkv, s);
    return launch_tc<64, 64, 2, 3>(p, tq, tkv, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_prefill_attn(const PrefillAttnParams& p, int dtype, cudaStream_t s) {
  if (p.n_qtiles <= 0) return cudaSuccess;
  dim3 grid(p.n_qtiles, p.H);
  if (prefill_attn_mma_supported(dtype, p.dh)) {
    if (p.dh == 128) {
      constexpr int smem = (QT + 4 * KT) * 128 * 2;
      cudaError_t e = cudaFuncSetAttribute(prefill_attn_mma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem);
      if (e != cudaSuccess) return e;
      prefill_attn_mma_kernel<128><<<grid, 128, smem, s>>>(p);
    } else {
      constexpr int smem = (QT + 4 * KT) * 64 * 2;
      prefill_attn_mma_kernel<64><<<grid, 128, smem, s>>>(p);
    }
    return cudaGetLastError();
  }
  if (p.dh > 256) return cudaErrorInvalidValue;
  if (dtype == 1)
    prefill_attn_simt_kernel<float><<<grid, 128, 0, s>>>(p);
  else
    prefill_attn_simt_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace hc
