// Split-K flash-decoding attention over the hybrid cache.
//
// Eq. 2-3 of the paper for one decode query per request, computed per
// (split, head) task as an online softmax: running max m (log2 domain, q pre-scaled by
// scale*log2 e), running sum l, unnormalised acc = sum_j 2^(s_j - m) v_j.  KV-mode
// requests read K/V unit blocks of the pool through their block table;
// hidden-mode requests read the K/V the reconstruction GEMM just rebuilt from
// scratch, in the same [H][B][dh] block layout, so one pass covers both modes.
// Masking is by token index (j < n_i), never by multiplying padding by zero.
//
// attn_pipe_kernel (bf16, dh in {64,128}, B % 16 == 0) is the hot kernel: persistent,
// one warp = one task at a time, tasks handed out by an atomic counter.  Each warp runs a
// private NST-stage ring: lane 0 issues 1-D bulk copies (cp.async.bulk, TMA engine) of a
// 16-token K chunk and V chunk (4 KiB each at dh=128: a head's rows of a block are
// contiguous) into shared memory, completion counted on an mbarrier; all lanes compute
// from shared memory.  The ring flows across task boundaries, so HBM traffic never
// drains between tasks.  Scores: each lane dots 4 dims (one 8-byte LDS per row), then a
// butterfly transpose-reduce leaves one full score per lane pair (1 shuffle per row).
//
// attn_generic_kernel (any dtype / dh <= 256 / B) is the simple unpipelined version used
// for fp32 mode and shapes the pipe kernel does not cover.
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace hc {

namespace {

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

template <int DH, int NW, int NST>
struct PipeCfg {
  static constexpr int TOK = 16;                      // tokens per chunk
  static constexpr int CHUNK = TOK * DH * 2;          // bytes of one K (or V) chunk
  static constexpr int QB = DH * 2;                   // bytes of q_h
  static constexpr int STAGE = 2 * CHUNK + QB;        // multiple of 16 bytes
  static_assert(STAGE % 16 == 0, "stage alignment");
  static constexpr int WARP_BYTES = (NST * STAGE + NST * 8 + NST * 16 + TOK * 4 + 127) / 128 * 128;
  static constexpr int SMEM = NW * WARP_BYTES;
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

template <int DH, int NW, int NST>
__global__ void __launch_bounds__(NW * 32, 1) attn_pipe_kernel(const AttnParams p) {
  using C = PipeCfg<DH, NW, NST>;
  constexpr int TOK = C::TOK;
  constexpr int LPR = DH / 8;      // lanes per row (each lane: 8 dims = 16 bytes)
  constexpr int RPI = 32 / LPR;    // rows per 128-bit load instruction
  constexpr int NV = TOK / RPI;    // rows (partial dot products) per lane per chunk
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wb = smem + warp * C::WARP_BYTES;
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
  const size_t head_elems = (size_t)B * DH;        // one head of one block
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
  SplitDesc psp{};
  ReqDesc prq{};
  int phead = 0;
  auto load_task = [&](int t) {
    if (t < p.n_tasks) {
      const int s = t / H;
      phead = t - s * H;
      psp = p.splits[s];
      prq = p.reqs[psp.req];
      pnch = (psp.ntok + TOK - 1) / TOK;
    }
  };
  load_task(ptask);

  // issue the next chunk of the producer stream into `stage`; false when no work is left
  auto produce = [&](int stage) -> bool {
    if (ptask >= p.n_tasks) return false;
    const int tok = psp.lb0 * B + pchunk * TOK;   // token index within the request
    const int lb = tok / B, row = tok - lb * B;
    const int rem = psp.ntok - pchunk * TOK;
    const int nvalid = rem < TOK ? rem : TOK;
    const bool first = pchunk == 0, last = pchunk == pnch - 1;
    if (lane == 0) {
      const __nv_bfloat16 *ksrc, *vsrc;
      if (prq.mode == 0) {
        const int kb = p.tables[prq.tab_off + 2 * lb];
        const int vb = p.tables[prq.tab_off + 2 * lb + 1];
        ksrc = pool + (size_t)kb * blk_elems + phead * head_elems + (size_t)row * DH;
        vsrc = pool + (size_t)vb * blk_elems + phead * head_elems + (size_t)row * DH;
      } else {
        const size_t off = ((size_t)(prq.scratch_blk0 + lb) * H + phead) * head_elems + (size_t)row * DH;
        ksrc = scr_k + off;
        vsrc = scr_v + off;
      }
      meta[stage] = make_int4(ptask, pchunk, nvalid, (first ? 1 : 0) | (last ? 2 : 0));
      uint8_t* sb = stage_base + stage * C::STAGE;
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive_expect_tx(&bars[stage], 2 * C::CHUNK + (first ? C::QB : 0));
      ptx::bulk_g2s(sb, ksrc, C::CHUNK, &bars[stage]);
      ptx::bulk_g2s(sb + C::CHUNK, vsrc, C::CHUNK, &bars[stage]);
      if (first)
        ptx::bulk_g2s(sb + 2 * C::CHUNK, qg + (size_t)psp.req * d + phead * DH, C::QB, &bars[stage]);
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
  float qf[8], acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) qf[i] = acc[i] = 0.f;
  float m_run = -INFINITY, l_lane = 0.f;   // l kept per lane (rows this lane owns), reduced per task
  int cstage = 0;
  uint32_t cphase = 0;

#pragma unroll 1
  while (in_flight > 0) {
    const int4 mt = meta[cstage];
    ptx::mbar_wait(&bars[cstage], cphase);
    const uint8_t* sb = stage_base + cstage * C::STAGE;
    if (mt.w & 1) {  // first chunk of a task: fresh state, load q_h (pre-scaled by scale*log2 e)
      bf16x8_to_f32(reinterpret_cast<const uint4*>(sb + 2 * C::CHUNK)[lr], qf);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        qf[i] *= p.scale_log2;
        acc[i] = 0.f;
      }
      m_run = -INFINITY;
      l_lane = 0.f;
    }
    // ---- scores: lane dots 8 dims of NV rows, butterfly leaves one full score per lane pair
    const uint4* ks = reinterpret_cast<const uint4*>(sb);
    float part[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float kf[8];
      bf16x8_to_f32(ks[(i * RPI + lg) * LPR + lr], kf);
      float a0 = qf[0] * kf[0], a1 = qf[1] * kf[1];
      a0 = fmaf(qf[2], kf[2], a0);
      a1 = fmaf(qf[3], kf[3], a1);
      a0 = fmaf(qf[4], kf[4], a0);
      a1 = fmaf(qf[5], kf[5], a1);
      a0 = fmaf(qf[6], kf[6], a0);
      a1 = fmaf(qf[7], kf[7], a1);
      part[i] = a0 + a1;
    }
    int idx = 0;
    Bfly<NV, LPR / 2>::run(part, lane, idx);
    const int row = idx * RPI + lg;
    const bool valid = row < mt.z;
    const float s = valid ? part[0] : -INFINITY;
    const float m_new = fmaxf(m_run, warp_max(s));
    const float pj = valid ? fast_exp2(s - m_new) : 0.f;
    const float alpha = fast_exp2(m_run - m_new);   // 0 when m_run = -inf
    if ((lane & 1) == 0) {
      pbuf[row] = pj;
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
      float vf[8];
      bf16x8_to_f32(vs[r * LPR + lr], vf);
      const float pr = pbuf[r];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fmaf(pr, vf[c], acc[c]);
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
      const int task = mt.x;
      if (lane < LPR) {
        float4* dst = reinterpret_cast<float4*>(p.part_acc + (size_t)task * DH) + 2 * lane;
        dst[0] = make_float4(a[0], a[1], a[2], a[3]);
        dst[1] = make_float4(a[4], a[5], a[6], a[7]);
      }
      if (lane == 0) {
        p.part_ml[2 * (size_t)task] = m_run;
        p.part_ml[2 * (size_t)task + 1] = l_tot;
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

// ------------------------------------------------------------------ generic kernel
template <typename T>
__device__ __forceinline__ float ld_f(const T* p);
template <>
__device__ __forceinline__ float ld_f<float>(const float* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

template <typename T, int MAXC>
__global__ void __launch_bounds__(128) attn_generic_kernel(const AttnParams p) {
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  __shared__ float qs[4][256];
  float* q_s = qs[threadIdx.x >> 5];
  const int H = p.H, B = p.B, d = p.d, DH = p.dh;
  const T* pool = static_cast<const T*>(p.pool);
  const T* scr_k = static_cast<const T*>(p.scr_k);
  const T* scr_v = static_cast<const T*>(p.scr_v);
  const T* qg = static_cast<const T*>(p.q);
  for (int task = wid; task < p.n_tasks; task += nwarps) {
    const int s = task / H, h = task - s * H;
    const SplitDesc sp = p.splits[s];
    const ReqDesc rq = p.reqs[sp.req];
    for (int c = lane; c < DH; c += 32) q_s[c] = ld_f(qg + (size_t)sp.req * d + h * DH + c) * p.scale_log2;
    __syncwarp();
    auto row_ptr = [&](int t, bool is_v) -> const T* {
      const int tok = sp.lb0 * B + t;
      const int lb = tok / B, row = tok - lb * B;
      if (rq.mode == 0) {
        const int blk = p.tables[rq.tab_off + 2 * lb + (is_v ? 1 : 0)];
        return pool + (size_t)blk * B * d + (size_t)h * B * DH + (size_t)row * DH;
      }
      return (is_v ? scr_v : scr_k) + (((size_t)(rq.scratch_blk0 + lb) * H + h) * B + row) * DH;
    };
    float m = -INFINITY, l = 0.f, acc[MAXC];
#pragma unroll
    for (int i = 0; i < MAXC; ++i) acc[i] = 0.f;
    for (int t0 = 0; t0 < sp.ntok; t0 += 32) {
      const int t = t0 + lane;
      const bool valid = t < sp.ntok;
      float sc = -INFINITY;
      if (valid) {
        const T* kr = row_ptr(t, false);
        float a = 0.f;
        for (int c = 0; c < DH; ++c) a += q_s[c] * ld_f(kr + c);
        sc = a;
      }
      const float m_new = fmaxf(m, warp_max(sc));
      const float pj = valid ? exp2f(sc - m_new) : 0.f;
      const float alpha = exp2f(m - m_new);
      l = l * alpha + warp_sum(pj);
#pragma unroll
      for (int i = 0; i < MAXC; ++i) acc[i] *= alpha;
      const int cnt = min(32, sp.ntok - t0);
      for (int jj = 0; jj < cnt; ++jj) {
        const float pw = __shfl_sync(FULL, pj, jj);
        const T* vr = row_ptr(t0 + jj, true);
#pragma unroll
        for (int i = 0; i < MAXC; ++i) {
          const int c = lane + 32 * i;
          if (c < DH) acc[i] += pw * ld_f(vr + c);
        }
      }
      m = m_new;
    }
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int c = lane + 32 * i;
      if (c < DH) p.part_acc[(size_t)task * DH + c] = acc[i];
    }
    if (lane == 0) {
      p.part_ml[2 * (size_t)task] = m;
      p.part_ml[2 * (size_t)task + 1] = l;
    }
    __syncwarp();
  }
}

template <int DH, int NW, int NST>
cudaError_t launch_pipe(const AttnParams& p, int num_sms, cudaStream_t s) {
  using C = PipeCfg<DH, NW, NST>;
  auto k = attn_pipe_kernel<DH, NW, NST>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const int max_ctas = (p.n_tasks + NW - 1) / NW;
  const int grid = max_ctas < num_sms ? max_ctas : num_sms;
  k<<<grid, NW * 32, C::SMEM, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

bool attn_pipe_supported(int dtype, int dh, int B) {
  return dtype == 0 && (dh == 128 || dh == 64) && B % 16 == 0;
}

cudaError_t launch_attn(const AttnParams& p, int dtype, bool generic, int num_sms, cudaStream_t s) {
  if (p.n_tasks <= 0) return cudaSuccess;
  if (!generic && attn_pipe_supported(dtype, p.dh, p.B)) {
    static const int cfg = [] { const char* v = std::getenv("HC_ATTN_CFG"); return v ? std::atoi(v) : 0; }();
    if (p.dh == 128) {
      if (cfg == 1) return launch_pipe<128, 6, 4>(p, num_sms, s);
      if (cfg == 2) return launch_pipe<128, 4, 6>(p, num_sms, s);
      return launch_pipe<128, 8, 3>(p, num_sms, s);
    }
    return launch_pipe<64, 8, 5>(p, num_sms, s);
  }
  if (p.dh > 256) return cudaErrorInvalidValue;
  const int threads = 128;
  int blocks = (p.n_tasks + 3) / 4;
  if (blocks > num_sms * 16) blocks = num_sms * 16;
  if (dtype == 1)
    attn_generic_kernel<float, 8><<<blocks, threads, 0, s>>>(p);
  else
    attn_generic_kernel<__nv_bfloat16, 8><<<blocks, threads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace hc
