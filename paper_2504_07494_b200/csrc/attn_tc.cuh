// Split-K flash-decoding over KV-mode blocks on the tensor cores:
// the KV attention warp loop of the fused step kernel and of the stand-alone attention
// kernel when every task reads the pool (KV-mode requests; hidden partials come from the
// GEMM's attend epilogue).
//
// Eq. 2-3 for the NQ <= 8 query heads that share one K/V head (GQA group, R18;
// NQ = 1 for multi-head), one (split, K/V head) task at a time, as an online softmax in the
// log2 domain.  Per 16-token chunk:
//   scores  S[16 tok x 8 q] = K[16 x dh] . Q^T[dh x 8]      mma.sync m16n8k16, bf16 in, fp32 acc
//   softmax per query column (lazy rescale: the reference max moves only when a score
//           exceeds it by more than 8, so p <= 2^8 — exact enough in bf16; l in fp32)
//   output  O^T[dh x 8] += V^T[dh x 16 tok] . P^T[16 tok x 8 q]   (fp32 accumulators stay in
//           the mma's C registers, no per-chunk rescale)
// The chunks arrive by TMA (2-D tensor map over the pool viewed as rows of dh elements,
// 64-column boxes, 128-B swizzle) into a per-warp ring on mbarriers, so ldmatrix reads
// them conflict-free.  Against the SIMT loop (attn_pipe.cuh) this issues ~80 instead of
// ~320 warp instructions per 8-KiB chunk: the attention warps leave the issue slots to the
// GEMM's attend epilogue in the fused kernel, and a GQA group's K/V is read once.
#pragma once
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace hc {
namespace at {

constexpr unsigned FULL = 0xffffffffu;
constexpr float kRescaleLog2 = 8.f;   // lazy-rescale headroom: p <= 2^8

template <int DH, int NST>
struct TcCfg {
  static constexpr int TOK = 16;                 // tokens per chunk (never straddles a block)
  static constexpr int NB = DH / 64;             // 128-B swizzled boxes per 16-row K (or V) chunk
  static constexpr int BOX = TOK * 128;          // 2 KiB
  static constexpr int CHUNK = NB * BOX;         // K (or V) chunk
  static constexpr int STAGE = 2 * CHUNK;        // K then V; multiple of 1024 (swizzle atom)
  static constexpr int STAGES_BYTES = NST * STAGE;
  static constexpr int CTRL_BYTES = NST * 32;    // per warp: meta int4 + mbarrier per stage
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One warp's loop.  stages: NST * STAGE bytes, 1024-aligned; ctrl: CTRL_BYTES, 16-aligned.
// Tasks t = split * Hk + kvhead from the task map; every task is a KV-mode split.
// Hidden-mode tasks (the fused kernel's scratch path: the GEMM epilogue wrote rebuilt K and V
// as [hblock][Hk][B][dh]) read through tmap_scr_k / tmap_scr_v (rows of dh elements) after
// the task map's wait_ready (the tiles that wrote them are done).
template <int DH, int NST, class TaskMap>
__device__ __forceinline__ void attn_warp_run_tc(const AttnParams& p, const CUtensorMap* tmap, uint8_t* stages,
                                                 uint8_t* ctrl, int lane, const TaskMap& tm,
                                                 const CUtensorMap* tmap_scr_k = nullptr,
                                                 const CUtensorMap* tmap_scr_v = nullptr) {
  using C = TcCfg<DH, NST>;
  constexpr int TOK = C::TOK;
  constexpr int KS = DH / 16;       // k-slices of the score mma, m-slices of the output mma
  int4* meta = reinterpret_cast<int4*>(ctrl);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ctrl + NST * 16);
  if (lane == 0) {
    for (int s = 0; s < NST; ++s) ptx::mbar_init(&bars[s], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();

  const int G = p.G, NQ = G;        // query heads per task (<= 8, checked by the host)
  const int64_t rows_per_unit = (int64_t)p.B * p.d / DH;   // pool rows of DH elements per unit block
  const int64_t v_rows = p.v_off / DH;
  const __nv_bfloat16* qg = static_cast<const __nv_bfloat16*>(p.q);

  // ---- producer (lane 0 issues; state warp-uniform)
  auto grab = [&]() -> int {
    int t = 0;
    if (lane == 0) t = atomicAdd(p.task_counter, 1);
    return __shfl_sync(FULL, t, 0);
  };
  int ptask = grab(), pchunk = 0, pnch = 0, psplit = 0, phk = 0;
  int plb = 0, prow = 0;   // logical block and row of the next chunk (kept incrementally: no divisions)
  SplitDesc psp{};
  ReqDesc prq{};
  auto load_task = [&](int t) {
    if (t < p.n_tasks) {
      tm.map(t, psplit, phk);
      psp = p.splits[psplit];
      prq = p.reqs[psp.req];
      pnch = (psp.ntok + TOK - 1) / TOK;
      plb = psp.lb0;
      prow = 0;
      tm.wait_ready(psplit, phk, psp, prq, lane);
    }
  };
  load_task(ptask);
  auto produce = [&](int stage) -> bool {
    if (ptask >= p.n_tasks) return false;
    const bool hid = prq.mode != 0;
    const int Bm = hid ? p.B : p.Bkv;
    const int lb = plb, row = prow;   // (lb0 * Bm + pchunk * TOK) as (block, row); Bm % TOK == 0
    const int rem = psp.ntok - pchunk * TOK;
    const bool first = pchunk == 0, last = pchunk == pnch - 1;
    if (lane == 0) {
      int rk, rv;
      const CUtensorMap *tk = tmap, *tv = tmap;
      if (!hid) {
        const int kb = p.tables[prq.tab_off + 2 * lb], vb = p.tables[prq.tab_off + 2 * lb + 1];
        rk = (int)(kb * rows_per_unit + (int64_t)phk * p.Bkv + row);
        rv = (int)(vb * rows_per_unit + v_rows + (int64_t)phk * p.Bkv + row);
      } else {   // scratch [hblock][Hk][B][dh]
        rk = rv = (int)(((int64_t)(prq.scratch_blk0 + lb) * p.Hk + phk) * p.B + row);
        tk = tmap_scr_k;
        tv = tmap_scr_v;
      }
      meta[stage] = make_int4(psplit, phk, rem < TOK ? rem : TOK, (first ? 1 : 0) | (last ? 2 : 0) | (psp.req << 2));
      uint8_t* sb = stages + stage * C::STAGE;
      ptx::fence_proxy_async_smem();   // the warp's ldmatrix reads of this stage precede the TMA writes
      ptx::mbar_arrive_expect_tx(&bars[stage], C::STAGE);
#pragma unroll
      for (int b = 0; b < C::NB; ++b) {
        ptx::tma_load_2d(sb + b * C::BOX, tk, b * 64, rk, &bars[stage]);
        ptx::tma_load_2d(sb + C::CHUNK + b * C::BOX, tv, b * 64, rv, &bars[stage]);
      }
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

  // ---- consumer: fragment coordinates
  const int g = lane >> 2, t = lane & 3;
  // ldmatrix row addresses (byte offsets inside a K or V chunk, before the box / slice part)
  const int mi = lane >> 3;
  const int ka_row = (lane & 7) + (mi & 1) * 8, ka_chk = mi >> 1;   // K as A (non-trans)
  const int va_row = (lane & 7) + (mi >> 1) * 8, va_chk = mi & 1;   // V^T as A (trans)
  const int q0 = 2 * t, q1 = 2 * t + 1;                              // this lane's score/output columns
  const bool qv0 = q0 < NQ, qv1 = q1 < NQ;
  const uint32_t sel = (g & 1) ? 0x7632u : 0x5410u;                 // P transpose: half g&1
  const int srcA = 4 * (2 * t) + (g >> 1), srcB = 4 * (2 * t + 1) + (g >> 1);

  uint32_t qb[KS][2];
  float acc[KS][4];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  int cstage = 0;
  uint32_t cphase = 0;

#pragma unroll 1
  while (in_flight > 0) {
    const int4 mt = meta[cstage];
    if (mt.w & 1) {   // first chunk of a task: q fragments of the group's query heads, fresh state
      const int req = mt.w >> 2;
      const bool qlive = g < NQ;
      const __nv_bfloat16* qh = qg + (size_t)req * p.d + (size_t)(mt.y * G + (qlive ? g : 0)) * DH;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        qb[kk][0] = qlive ? __ldg(reinterpret_cast<const uint32_t*>(qh + kk * 16 + 2 * t)) : 0u;
        qb[kk][1] = qlive ? __ldg(reinterpret_cast<const uint32_t*>(qh + kk * 16 + 8 + 2 * t)) : 0u;
      }
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) acc[kk][0] = acc[kk][1] = acc[kk][2] = acc[kk][3] = 0.f;
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
    }
    ptx::mbar_wait(&bars[cstage], cphase);
    const uint32_t sK = ptx::smem_u32(stages + cstage * C::STAGE);
    const uint32_t sV = sK + C::CHUNK;
    // ---- S = K Q^T
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      uint32_t a[4];
      const int chk = (kk & 3) * 2 + ka_chk;
      ldsm_x4(sK + (kk >> 2) * C::BOX + ka_row * 128 + ((chk ^ (ka_row & 7)) << 4), a);
      mma16816(s, a, qb[kk][0], qb[kk][1]);
    }
    // s[0]: (tok g, q0)  s[1]: (tok g, q1)  s[2]: (tok g+8, q0)  s[3]: (tok g+8, q1)
    const int nvalid = mt.z;
    const bool tv0 = g < nvalid, tv1 = g + 8 < nvalid;
    s[0] = (tv0 && qv0) ? s[0] * p.scale_log2 : -INFINITY;
    s[1] = (tv0 && qv1) ? s[1] * p.scale_log2 : -INFINITY;
    s[2] = (tv1 && qv0) ? s[2] * p.scale_log2 : -INFINITY;
    s[3] = (tv1 && qv1) ? s[3] * p.scale_log2 : -INFINITY;
    float x0 = fmaxf(s[0], s[2]), x1 = fmaxf(s[1], s[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      x0 = fmaxf(x0, __shfl_xor_sync(FULL, x0, o));
      x1 = fmaxf(x1, __shfl_xor_sync(FULL, x1, o));
    }
    // lazy rescale: move the reference only when a score exceeds it by more than 2^8
    const bool r0 = qv0 && x0 > m0 + kRescaleLog2, r1 = qv1 && x1 > m1 + kRescaleLog2;
    if (__any_sync(FULL, r0 || r1)) {
      const float n0 = r0 ? x0 : m0, n1 = r1 ? x1 : m1;
      const float a0 = r0 ? ex2(m0 - n0) : 1.f, a1 = r1 ? ex2(m1 - n1) : 1.f;   // 0 when m was -inf
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        acc[kk][0] *= a0;
        acc[kk][1] *= a1;
        acc[kk][2] *= a0;
        acc[kk][3] *= a1;
      }
      l0 *= a0;
      l1 *= a1;
      m0 = n0;
      m1 = n1;
    }
    const float p0 = qv0 ? ex2(s[0] - m0) : 0.f, p1 = qv1 ? ex2(s[1] - m1) : 0.f;
    const float p2 = qv0 ? ex2(s[2] - m0) : 0.f, p3 = qv1 ? ex2(s[3] - m1) : 0.f;
    l0 += p0 + p2;
    l1 += p1 + p3;
    // ---- P^T as the B operand: lane (g, t) needs p[q=g][tok 2t, 2t+1] and [2t+8, 2t+9]
    const uint32_t P01 = pack_bf16x2(p0, p1), P23 = pack_bf16x2(p2, p3);
    const uint32_t X = __shfl_sync(FULL, P01, srcA), Y = __shfl_sync(FULL, P01, srcB);
    const uint32_t Z = __shfl_sync(FULL, P23, srcA), W = __shfl_sync(FULL, P23, srcB);
    const uint32_t b0 = prmt(X, Y, sel), b1 = prmt(Z, W, sel);
    // ---- O^T += V^T P^T
#pragma unroll
    for (int ms = 0; ms < KS; ++ms) {
      uint32_t a[4];
      const int chk = (ms & 3) * 2 + va_chk;
      ldsm_x4_t(sV + (ms >> 2) * C::BOX + va_row * 128 + ((chk ^ (va_row & 7)) << 4), a);
      mma16816(acc[ms], a, b0, b1);
    }
    if (mt.w & 2) {   // last chunk of the task: (m, l, acc) of every query head of the group
      float L0 = l0, L1 = l1;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        L0 += __shfl_xor_sync(FULL, L0, o);
        L1 += __shfl_xor_sync(FULL, L1, o);
      }
      const int split = mt.x, hk = mt.y;
      if (qv0) {
        const size_t pidx = (size_t)(hk * G + q0) * p.n_splits_all + split;
        float* dst = p.part_acc + pidx * DH;
#pragma unroll
        for (int ms = 0; ms < KS; ++ms) {
          dst[ms * 16 + g] = acc[ms][0];
          dst[ms * 16 + g + 8] = acc[ms][2];
        }
        if (g == 0) {
          p.part_ml[2 * pidx] = m0;
          p.part_ml[2 * pidx + 1] = L0;
        }
      }
      if (qv1) {
        const size_t pidx = (size_t)(hk * G + q1) * p.n_splits_all + split;
        float* dst = p.part_acc + pidx * DH;
#pragma unroll
        for (int ms = 0; ms < KS; ++ms) {
          dst[ms * 16 + g] = acc[ms][1];
          dst[ms * 16 + g + 8] = acc[ms][3];
        }
        if (g == 0) {
          p.part_ml[2 * pidx] = m1;
          p.part_ml[2 * pidx + 1] = L1;
        }
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

}  // namespace at
}  // namespace hc
