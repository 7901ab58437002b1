// Split-K flash-decoding attention warp loop, shared by the stand-alone
// attention kernel (attention.cu) and the fused step kernel (fused.cu).
//
// Eq. 2-3 for one decode query per request, per (split, head) task, as an
// online softmax: running max m (log2 domain, q pre-scaled by scale*log2 e), running sum l,
// unnormalised acc = sum_j 2^(s_j - m) v_j.  KV-mode requests read K/V unit blocks of the
// pool through their block table; hidden-mode requests read the K/V the
// reconstruction GEMM rebuilt from scratch in the same [H][B][dh] layout.
// Scores are masked by token index (j < n_i); padding rows get p = 0 (and are finite).
// Lane 0 issues 1-D bulk copies (TMA engine) of a 16-token K chunk and V chunk (4 KiB each
// at dh=128: a head's rows of a block are contiguous) into shared memory; all lanes
// compute from shared memory: each lane dots 8 dims of a row (128-bit LDS), a butterfly
// transpose-reduce leaves one complete score per lane pair.  The products run as
// mixed-precision FMAs (fma.rn.f32.bf16 = FHFMA: bf16 x bf16, fp32 accumulate) straight
// on the stored bf16 words, so no element is converted: q.k is exact per product as before,
// and Σ p v takes p rounded once to bf16 (l sums the same rounded p, so the weights stay
// normalised).  One instruction per element instead of a convert + an FMA.
#pragma once
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace hc {
namespace ap {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// a0 += q.lo * k.lo, a1 += q.hi * k.hi (bf16 products, fp32 accumulation; FHFMA.BF16)
__device__ __forceinline__ void dot2_bf16(float& a0, float& a1, uint32_t q, uint32_t k) {
  asm("{\n .reg .b16 ql, qh, kl, kh;\n mov.b32 {ql, qh}, %2;\n mov.b32 {kl, kh}, %3;\n"
      " fma.rn.f32.bf16 %0, ql, kl, %0;\n fma.rn.f32.bf16 %1, qh, kh, %1;\n}"
      : "+f"(a0), "+f"(a1)
      : "r"(q), "r"(k));
}
// a0 += p * v.lo, a1 += p * v.hi (p a bf16 scalar)
__device__ __forceinline__ void axpy2_bf16(float& a0, float& a1, uint16_t p, uint32_t v) {
  asm("{\n .reg .b16 vl, vh;\n mov.b32 {vl, vh}, %3;\n"
      " fma.rn.f32.bf16 %0, %2, vl, %0;\n fma.rn.f32.bf16 %1, %2, vh, %1;\n}"
      : "+f"(a0), "+f"(a1)
      : "h"(p), "r"(v));
}
__device__ __forceinline__ uint16_t bf16_bits(float x) {
  __nv_bfloat16 b = __float2bfloat16_rn(x);
  return *reinterpret_cast<uint16_t*>(&b);
}
__device__ __forceinline__ float bf16_val(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

__device__ __forceinline__ void bf16x4_to_f32(uint2 u, float (&f)[4]) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
}

// Butterfly transpose-reduce: NV partial sums per lane over groups of 2*OFF lanes;
// afterwards v[0] of each lane holds a complete sum for one of the NV rows.
template <int NV, int OFF>
struct Bfly {
  static __device__ __forceinline__ void run(float* v, int lane, int& idx) {
    if constexpr (OFF == 0) {
      return;
    } else if constexpr (NV == 1) {
      v[0] += __shfl_xor_sync(FULL, v[0], OFF);
      Bfly<1, OFF / 2>::run(v, lane, idx);
    } else {
      const bool hi = (lane & OFF) != 0;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        const float send = hi ? v[i] : v[i + NV / 2];
        const float keep = hi ? v[i + NV / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(FULL, send, OFF);
      }
      if (hi) idx += NV / 2;
      Bfly<NV / 2, OFF / 2>::run(v, lane, idx);
    }
  }
};

// QREG: q_h is loaded into registers at the producer (one 16-byte vector per lane) instead
// of riding in every stage, so a stage is exactly K chunk + V chunk — the fused kernel uses
// the saved smem for a fifth attention warp.
template <int DH, int NST, bool QREG = false>
struct PipeCfg {
  static constexpr int TOK = 16;                      // tokens per chunk
  static constexpr int CHUNK = TOK * DH * 2;          // bytes of one K (or V) chunk
  static constexpr int QB = QREG ? 0 : DH * 2;        // bytes of q_h staged per stage
  static constexpr int STAGE = 2 * CHUNK + QB;        // multiple of 16 bytes
  static_assert(STAGE % 16 == 0, "stage alignment");
  static constexpr int WARP_BYTES = (NST * STAGE + NST * 8 + NST * 16 + TOK * 4 + 127) / 128 * 128;
};

__device__ __forceinline__ void bf16x8_to_f32(uint4 u, float (&f)[8]) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xffff0000u);
}

// Task maps: which (split, head) the t-th task of the atomic counter is, and whether the
// producer must wait before reading its K/V.
struct DirectTaskMap {   // stand-alone attention: all K/V already in memory, task = split*H + head
  int n_tasks, H;
  __device__ __forceinline__ void map(int t, int& split, int& head) const {
    split = t / H;
    head = t - split * H;
  }
  __device__ __forceinline__ void wait_ready(int, int, const SplitDesc&, const ReqDesc&, int) const {}
};

// One warp's attention loop: a private NST-stage ring of bulk copies (K chunk, V chunk, q_h)
// on mbarriers, fed from a global task counter; the ring flows across task boundaries.
// wb: this warp's smem region of PipeCfg<DH,NST>::WARP_BYTES bytes (16-B aligned).
template <int DH, int NST, class TaskMap, bool QREG = false>
__device__ __forceinline__ void attn_warp_run(const AttnParams& p, uint8_t* wb, int lane, const TaskMap& tm) {
  using C = PipeCfg<DH, NST, QREG>;
  static_assert(!QREG || NST <= 3, "register q slots: at most 3 stages");
  constexpr int TOK = C::TOK;
  constexpr int LPR = DH / 8;      // lanes per row (each lane: 8 dims = 16 bytes)
  constexpr int RPI = 32 / LPR;    // rows per 128-bit load instruction
  constexpr int NV = TOK / RPI;    // rows (partial dot products) per lane per chunk
  uint8_t* stage_base = wb;
  // per-warp layout: NST stages (16-B multiples) | meta[NST] int4 | bars[NST] | pbuf[16]
  int4* meta = reinterpret_cast<int4*>(wb + NST * C::STAGE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wb + NST * C::STAGE + NST * 16);
  float* pbuf = reinterpret_cast<float*>(wb + NST * C::STAGE + NST * 16 + NST * 8);

  if (lane == 0) {
    for (int s = 0; s < NST; ++s) ptx::mbar_init(&bars[s], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();

  const int H = p.H, B = p.B, d = p.d;
  const size_t blk_elems = (size_t)B * d;          // one unit block
  const size_t head_elems = (size_t)B * DH;        // one head of one hidden/scratch block
  const size_t kv_head_elems = (size_t)p.Bkv * DH; // one head of one KV logical block
  const __nv_bfloat16* pool = static_cast<const __nv_bfloat16*>(p.pool);
  const __nv_bfloat16* scr_k = static_cast<const __nv_bfloat16*>(p.scr_k);
  const __nv_bfloat16* scr_v = static_cast<const __nv_bfloat16*>(p.scr_v);
  const __nv_bfloat16* qg = static_cast<const __nv_bfloat16*>(p.q);

  // ---- producer state (warp-uniform) ----
  auto grab = [&]() -> int {
    int t = 0;
    if (lane == 0) t = atomicAdd(p.task_counter, 1);
    return __shfl_sync(FULL, t, 0);
  };
  int ptask = grab();
  int pchunk = 0;
  int pnch = 0;
  int plb = 0, prow = 0, phk = 0;   // logical block and row of the next chunk (kept incrementally: no divisions)
  SplitDesc psp{};
  ReqDesc prq{};
  int phead = 0;
  int psplit = 0;
  auto load_task = [&](int t) {
    if (t < p.n_tasks) {
      tm.map(t, psplit, phead);
      psp = p.splits[psplit];
      prq = p.reqs[psp.req];
      pnch = (psp.ntok + TOK - 1) / TOK;
      plb = psp.lb0;
      prow = 0;
      phk = phead / p.G;
      tm.wait_ready(psplit, phead, psp, prq, lane);
    }
  };
  load_task(ptask);
  uint4 qr0 = make_uint4(0, 0, 0, 0), qr1 = qr0, qr2 = qr0;   // QREG: q_h slot per stage

  // issue the next chunk of the producer stream into `stage`; false when no work is left
  auto produce = [&](int stage) -> bool {
    if (ptask >= p.n_tasks) return false;
    const int Bm = prq.mode == 0 ? p.Bkv : B;     // tokens per logical block of this mode
    const int lb = plb, row = prow;               // (lb0 * Bm + pchunk * TOK) as (block, row); Bm % TOK == 0
    const int hk = phk;                           // K/V head of this query head (GQA, R18)
    const int rem = psp.ntok - pchunk * TOK;
    const int nvalid = rem < TOK ? rem : TOK;
    const bool first = pchunk == 0, last = pchunk == pnch - 1;
    if (lane == 0) {
      const __nv_bfloat16 *ksrc, *vsrc;
      if (prq.mode == 0) {
        int kb = p.tables[prq.tab_off + 2 * lb];
        int vb = p.tables[prq.tab_off + 2 * lb + 1];
#ifdef HC_DIAG
        if (p.diag == 2) kb = vb = 0;   // timing diagnostic: every chunk from one L2-resident block
#endif
        ksrc = pool + (size_t)kb * blk_elems + hk * kv_head_elems + (size_t)row * DH;
        vsrc = pool + (size_t)vb * blk_elems + p.v_off + hk * kv_head_elems + (size_t)row * DH;
      } else {
        const size_t off = ((size_t)(prq.scratch_blk0 + lb) * p.Hk + hk) * head_elems + (size_t)row * DH;
        ksrc = scr_k + off;
        vsrc = scr_v + off;
      }
      meta[stage] = make_int4(psplit * H + phead, pchunk, nvalid, (first ? 1 : 0) | (last ? 2 : 0));
      uint8_t* sb = stage_base + stage * C::STAGE;
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive_expect_tx(&bars[stage], 2 * C::CHUNK + (first ? C::QB : 0));
      ptx::bulk_g2s(sb, ksrc, C::CHUNK, &bars[stage]);
      ptx::bulk_g2s(sb + C::CHUNK, vsrc, C::CHUNK, &bars[stage]);
      if (!QREG && first)
        ptx::bulk_g2s(sb + 2 * C::CHUNK, qg + (size_t)psp.req * d + phead * DH, C::QB, &bars[stage]);
    }
    if (QREG && first) {   // every lane: its 8 dims of q_h (consumed when this stage is)
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(qg + (size_t)psp.req * d + phead * DH) + lane % LPR);
      if (stage == 0) qr0 = v;
      else if (stage == 1) qr1 = v;
      else qr2 = v;
    }
    prow += TOK;
    if (prow >= Bm) {
      prow -= Bm;
      ++plb;
    }
    if (++pchunk == pnch) {
      ptask = grab();
      pchunk = 0;
      load_task(ptask);
    }
    return true;
  };

  int in_flight = 0;
#pragma unroll 1
  for (int s = 0; s < NST; ++s)
    if (produce(s)) ++in_flight;
  __syncwarp();

  const int lr = lane % LPR;   // this lane's 16-byte column slot (dims 8*lr .. 8*lr+7)
  const int lg = lane / LPR;   // this lane's row group
  uint16_t* pbuf16 = reinterpret_cast<uint16_t*>(pbuf);
  uint4 qw = make_uint4(0, 0, 0, 0);   // this lane's 8 dims of q_h, bf16 as stored
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  float m_run = -INFINITY, l_lane = 0.f;   // l kept per lane (rows this lane owns), reduced per task
  int cstage = 0;
  uint32_t cphase = 0;

#pragma unroll 1
  while (in_flight > 0) {
    const int4 mt = meta[cstage];
    ptx::mbar_wait(&bars[cstage], cphase);
    const uint8_t* sb = stage_base + cstage * C::STAGE;
#ifdef HC_DIAG
    if (p.diag == 1) {   // timing diagnostic: stream the chunks, skip the math (wrong outputs)
      __syncwarp();
      --in_flight;
      if (produce(cstage)) ++in_flight;
      __syncwarp();
      if (++cstage == NST) {
        cstage = 0;
        cphase ^= 1u;
      }
      continue;
    }
#endif
    if (mt.w & 1) {  // first chunk of a task: fresh state, load q_h (bf16 words as stored)
      if constexpr (QREG)
        qw = cstage == 0 ? qr0 : (cstage == 1 ? qr1 : qr2);
      else
        qw = reinterpret_cast<const uint4*>(sb + 2 * C::CHUNK)[lr];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
      m_run = -INFINITY;
      l_lane = 0.f;
    }
    // ---- scores: lane dots 8 dims of NV rows, butterfly leaves one full score per lane pair
    const uint4* ks = reinterpret_cast<const uint4*>(sb);
    float part[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const uint4 kw = ks[(i * RPI + lg) * LPR + lr];
      float a0 = 0.f, a1 = 0.f;
      dot2_bf16(a0, a1, qw.x, kw.x);
      dot2_bf16(a0, a1, qw.y, kw.y);
      dot2_bf16(a0, a1, qw.z, kw.z);
      dot2_bf16(a0, a1, qw.w, kw.w);
      part[i] = a0 + a1;
    }
    int idx = 0;
    Bfly<NV, LPR / 2>::run(part, lane, idx);
    const int row = idx * RPI + lg;
    const bool valid = row < mt.z;
    const float s = valid ? part[0] * p.scale_log2 : -INFINITY;
    // lanes 2k and 2k+1 hold the same score: the max over the warp needs 4 levels, not 5
    float smax = s;
#pragma unroll
    for (int o = 16; o > 1; o >>= 1) smax = fmaxf(smax, __shfl_xor_sync(FULL, smax, o));
    const float m_new = fmaxf(m_run, smax);
    const uint16_t pj16 = bf16_bits(valid ? fast_exp2(s - m_new) : 0.f);   // the weight Σ p v uses
    const float pj = bf16_val(pj16);
    const float alpha = fast_exp2(m_run - m_new);   // 0 when m_run = -inf
    if ((lane & 1) == 0) {
      pbuf16[row] = pj16;
      l_lane = l_lane * alpha + pj;
    } else {
      l_lane *= alpha;
    }
    m_run = m_new;
    __syncwarp();
    // ---- acc = alpha * acc + sum_j p_j v_j (padding rows have p_j = 0 and finite v_j)
    const uint4* vs = reinterpret_cast<const uint4*>(sb + C::CHUNK);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] *= alpha;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int r = i * RPI + lg;
      const uint4 vw = vs[r * LPR + lr];
      const uint16_t pr = pbuf16[r];
      axpy2_bf16(acc[0], acc[1], pr, vw.x);
      axpy2_bf16(acc[2], acc[3], pr, vw.y);
      axpy2_bf16(acc[4], acc[5], pr, vw.z);
      axpy2_bf16(acc[6], acc[7], pr, vw.w);
    }
    if (mt.w & 2) {  // last chunk of the task: emit the partial (m, l, acc)
      float a[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = acc[c];
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] += __shfl_xor_sync(FULL, a[c], o);
      const float l_tot = warp_sum(l_lane);
      const int task = mt.x;   // split * H + head -> head-major partial index
      const size_t pidx = (size_t)(task % p.H) * p.n_splits_all + task / p.H;
      if (lane < LPR) {
        float4* dst = reinterpret_cast<float4*>(p.part_acc + pidx * DH) + 2 * lane;
        dst[0] = make_float4(a[0], a[1], a[2], a[3]);
        dst[1] = make_float4(a[4], a[5], a[6], a[7]);
      }
      if (lane == 0) {
        p.part_ml[2 * pidx] = m_run;
        p.part_ml[2 * pidx + 1] = l_tot;
      }
    }
    __syncwarp();
    --in_flight;
    if (produce(cstage)) ++in_flight;
    __syncwarp();
    if (++cstage == NST) {
      cstage = 0;
      cphase ^= 1u;
    }
  }
}


}  // namespace ap
}  // namespace hc
