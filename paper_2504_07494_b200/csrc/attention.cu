// Split-K flash-decoding attention over the hybrid cache: the
// stand-alone persistent kernel around ap::attn_warp_run (attn_pipe.cuh; bf16, dh 64/128,
// B % 16 == 0), and attn_generic_kernel — the simple unpipelined version for fp32 mode and
// shapes the pipe kernel does not cover.
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdlib>

#include <cuda.h>

#include "attn_pipe.cuh"
#include "attn_tc.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace hc {

namespace {

using ap::FULL;
using ap::warp_max;
using ap::warp_sum;

// Every task a KV-mode (split, K/V head): the tensor-core loop (attn_tc.cuh), NW warps per CTA.
template <int DH, int NW, int NST>
__global__ void __launch_bounds__(NW * 32, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap tmap_kv,
                                                             const __grid_constant__ CUtensorMap tmap_sk,
                                                             const __grid_constant__ CUtensorMap tmap_sv,
                                                             const AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_tc[];
  using C = at::TcCfg<DH, NST>;
  const uint32_t base_u32 = ptx::smem_u32(smem_tc);
  uint8_t* smem = smem_tc + ((1024 - (base_u32 & 1023)) & 1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ap::DirectTaskMap tm{p.n_tasks, p.th};
  at::attn_warp_run_tc<DH, NST>(p, &tmap_kv, smem + warp * C::STAGES_BYTES,
                                smem + NW * C::STAGES_BYTES + warp * C::CTRL_BYTES, lane, tm, &tmap_sk, &tmap_sv);
}

template <int DH, int NW, int NST>
__global__ void __launch_bounds__(NW * 32, 1) attn_pipe_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ap::DirectTaskMap tm{p.n_tasks, p.H};
  ap::attn_warp_run<DH, NST>(p, smem + warp * ap::PipeCfg<DH, NST>::WARP_BYTES, lane, tm);
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
    const int hk = h / p.G;   // this query head's K/V head (GQA, R18)
    auto row_ptr = [&](int t, bool is_v) -> const T* {
      if (rq.mode == 0) {
        const int tok = sp.lb0 * p.Bkv + t;
        const int lb = tok / p.Bkv, row = tok - lb * p.Bkv;
        const int blk = p.tables[rq.tab_off + 2 * lb + (is_v ? 1 : 0)];
        return pool + (size_t)blk * B * d + (is_v ? p.v_off : 0) + (size_t)hk * p.Bkv * DH + (size_t)row * DH;
      }
      const int tok = sp.lb0 * B + t;
      const int lb = tok / B, row = tok - lb * B;
      return (is_v ? scr_v : scr_k) + (((size_t)(rq.scratch_blk0 + lb) * p.Hk + hk) * B + row) * DH;
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
    const size_t pidx = (size_t)(task % p.H) * p.n_splits_all + task / p.H;   // head-major
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int c = lane + 32 * i;
      if (c < DH) p.part_acc[pidx * DH + c] = acc[i];
    }
    if (lane == 0) {
      p.part_ml[2 * pidx] = m;
      p.part_ml[2 * pidx + 1] = l;
    }
    __syncwarp();
  }
}

template <int DH, int NW, int NST>
cudaError_t launch_pipe(const AttnParams& p, int num_sms, cudaStream_t s) {
  constexpr int smem = NW * ap::PipeCfg<DH, NST>::WARP_BYTES;
  auto k = attn_pipe_kernel<DH, NW, NST>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int max_ctas = (p.n_tasks + NW - 1) / NW;
  const int grid = max_ctas < num_sms ? max_ctas : num_sms;
  k<<<grid, NW * 32, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

bool attn_pipe_supported(int dtype, int dh, int B) {
  return dtype == 0 && (dh == 128 || dh == 64) && B % 16 == 0;
}
bool attn_tc_supported(int dtype, int dh, int G, int Bkv) {
  return dtype == 0 && (dh == 128 || dh == 64) && G >= 1 && G <= 8 && Bkv % 16 == 0;
}

template <int DH, int NW, int NST>
static cudaError_t launch_tc(const AttnParams& p, const void* tmap, const void* tsk, const void* tsv, int num_sms,
                             cudaStream_t s) {
  using C = at::TcCfg<DH, NST>;
  constexpr int smem = 1024 + NW * (C::STAGES_BYTES + C::CTRL_BYTES);
  auto k = attn_tc_kernel<DH, NW, NST>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int max_ctas = (p.n_tasks + NW - 1) / NW;
  const int grid = max_ctas < num_sms ? max_ctas : num_sms;
  k<<<grid, NW * 32, smem, s>>>(*static_cast<const CUtensorMap*>(tmap),
                                *static_cast<const CUtensorMap*>(tsk ? tsk : tmap),
                                *static_cast<const CUtensorMap*>(tsv ? tsv : tmap), p);
  return cudaGetLastError();
}

cudaError_t launch_attn(const AttnParams& p, int dtype, bool generic, int num_sms, const Tuning& t, cudaStream_t s,
                        const void* tmap_kv, const void* tmap_scr_k, const void* tmap_scr_v) {
  if (p.n_tasks <= 0) return cudaSuccess;
  if (t.attn_sms > 0 && t.attn_sms < num_sms) num_sms = t.attn_sms;   // measurement knob (per-SM KV rate)
  if (p.tc) {   // tensor-core loop (the runtime checked attn_tc_supported)
    if (p.dh == 128) return launch_tc<128, 8, 3>(p, tmap_kv, tmap_scr_k, tmap_scr_v, num_sms, s);
    return launch_tc<64, 8, 5>(p, tmap_kv, tmap_scr_k, tmap_scr_v, num_sms, s);
  }
  if (!generic && attn_pipe_supported(dtype, p.dh, p.B)) {
    const int cfg = t.attn_cfg;
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
