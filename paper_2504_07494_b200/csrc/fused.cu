// Fused decode step (SURVEY §3.2 "[s1] reconstruction concurrent with [s2] KV attention",
// hard part 4): one persistent kernel per SM running
//   warps 0-5   the CTA-pair tcgen05 reconstruction GEMM (pair_gemm.cuh, 3-stage ring), and
//   warps 6..   NA split-K attention warps (attn_pipe.cuh) on a shared task counter.
// Attention tasks are ordered KV-mode first (their K/V are in the pool: they stream from HBM
// while the tensor cores rebuild hidden K/V), then hidden-mode tasks in the GEMM's n-tile
// order.  Before reading a hidden task's K/V a warp waits until every GEMM tile covering its
// rows and head has been written: each of the 8 epilogue warps of a pair tile fences its
// stores and adds 1 to the tile's counter (release); the attention warp acquires 8, then
// fences the async proxy before its bulk copies.  The two workloads use different units —
// tensor pipes + L2 for the GEMM, HBM + LSU for the KV stream — so near the KV/hidden
// crossover the step approaches max(T_gemm, T_attn) instead of their sum.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>

#include "attn_pipe.cuh"
#include "attn_tc.cuh"
#include "internal.h"
#include "pair_gemm.cuh"
#include "ptx.cuh"

namespace hc {
namespace {

#ifdef HC_TIMELINE
// Diagnostic build only: per-CTA globaltimer stamps of the last fused launch —
// [0] start, [1] GEMM warps drained, [2] last attention warp done, [3] attention tasks taken
// (global counter) when this CTA's GEMM drained, [4] first attention warp done.
__device__ unsigned long long g_timeline[512][5];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

constexpr int kNsubMax = 2;
constexpr bool kLateJoin = true;
using PC = pg::PairCfg<kNsubMax, 3>;   // widest tile (256 x 512); NSUB = 1 runs 256 x 256 tiles

struct FusedTaskMap {
  const AttnParams* p;
  __device__ __forceinline__ void map(int t, int& split, int& head) const {
    const int H = p->th;   // heads per split in the task numbering (Hk for the tensor-core loop)
    if (t < p->n_kv_tasks) {
      const int ks = t / H;
      split = p->kv_split_ids[ks];
      head = t - ks * H;
      return;
    }
    // heads per GEMM n-tile in the task numbering (K/V heads for the tensor-core loop)
    const int hpt = p->gemm_tile_n / (2 * p->dh) * (p->tc ? 1 : p->G);
    const int u = t - p->n_kv_tasks;
    const int per_nt = p->n_hid_splits * hpt;
    const int nt = u / per_nt;
    const int r = u - nt * per_nt;
    split = p->hid_split_ids[r / hpt];
    head = nt * hpt + r % hpt;
  }
  __device__ __forceinline__ void wait_ready(int /*split*/, int head, const SplitDesc& sp, const ReqDesc& rq,
                                             int lane) const {
    if (rq.mode != 1) return;
    if (lane == 0) {
      const int B = p->B;
      const int g0 = rq.scratch_blk0 + sp.lb0;
      const int nblk = (sp.ntok + B - 1) / B;
      const int mt0 = (g0 * B) / p->gemm_tile_m, mt1 = ((g0 + nblk) * B - 1) / p->gemm_tile_m;
      const int nt = (p->tc ? head : head / p->G) * 2 * p->dh / p->gemm_tile_n;
      const long long t0 = clock64();
      for (int mt = mt0; mt <= mt1; ++mt) {
        const int32_t* f = p->tile_done + mt * p->gemm_n_tiles + nt;
        while (pg::ld_acquire(f) < p->tile_target) {
          __nanosleep(256);
          if (clock64() - t0 > (1ll << 35)) __trap();
        }
      }
      // K/V were written by generic stores; the bulk copies read through the async proxy.
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncwarp();
  }
};

// Shared-memory plan of the attention part: TC = the tensor-core KV loop (attn_tc.cuh), whose
// stages must be 1024-aligned (128-B swizzle atoms) with the per-warp control words apart.
template <int GS, int NA, int NSTA, bool QR, bool TC, int NS>
struct FusedSmem {
  using PC = pg::PairCfg<NS, GS>;
  using TCC = at::TcCfg<128, NSTA>;
  using TCJ = at::TcCfg<128, 2>;   // joiners: 2-stage rings in the freed GEMM stage buffers
  static constexpr int kJoinBytes = TC ? TCJ::STAGES_BYTES : ap::PipeCfg<128, 2, QR>::WARP_BYTES;
  static constexpr int kJoin = (GS * PC::STAGE_BYTES / kJoinBytes) < 6 ? (GS * PC::STAGE_BYTES / kJoinBytes) : 6;
  static constexpr int ATTN_OFF = TC ? (PC::REGION_BYTES + 1023) / 1024 * 1024 : PC::REGION_BYTES;
  static constexpr int WARP_BYTES = TC ? TCC::STAGES_BYTES : ap::PipeCfg<128, NSTA, QR>::WARP_BYTES;
  static constexpr int CTRL_OFF = ATTN_OFF + NA * WARP_BYTES;
  static constexpr int TOTAL = CTRL_OFF + (TC ? (NA + 6) * TCC::CTRL_BYTES : 0);
};

// EW: extra epilogue warps (0 or 4): with 4, two warps per TMEM lane quarter split each
// tile's epilogue (every other head / column chunk) — for GQA, whose attend epilogue serves
// G query heads per rebuilt K/V head and otherwise idles the tensor cores.
template <int GS, int NA, int NSTA, bool QR, bool TC, int NS, int EW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pg::GEMM_THREADS + 32 * (NA + EW), 1)
    fused_step_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                      const __grid_constant__ CUtensorMap tmap_kv, const __grid_constant__ CUtensorMap tmap_sk,
                      const __grid_constant__ CUtensorMap tmap_sv, const __grid_constant__ CUtensorMap tmap_x128,
                      const pg::TcArgs a, const AttnParams p) {
  constexpr int kGemmStages = GS;
  using FS = FusedSmem<GS, NA, NSTA, QR, TC, NS>;
  constexpr int kJoin = FS::kJoin;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
  const pg::PairSmem ps = pg::pair_carve<NS, kGemmStages>(smem);
  uint8_t* attn_base = smem + FS::ATTN_OFF;
  uint8_t* ctrl_base = smem + FS::CTRL_OFF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kGemmWarps = pg::GEMM_THREADS / 32 + EW;
  pg::pair_setup<NS, kGemmStages, EW ? 2 : 1>(ps, warp, lane, &tmap_x, &tmap_w);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *ps.tmem_slot;
#ifdef HC_TIMELINE
  if (threadIdx.x == 0) {
    g_timeline[blockIdx.x][0] = gtimer();
    g_timeline[blockIdx.x][2] = 0;
    g_timeline[blockIdx.x][4] = ~0ull;
  }
#endif
  if (warp < kGemmWarps) {
    pg::pair_roles<NS, kGemmStages, EW ? 2 : 1, (EW > 0)>(ps, warp, lane, &tmap_x, &tmap_w, a, tmem_base,
                                                         a.runs ? &tmap_x128 : nullptr);
#ifdef HC_TIMELINE
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kGemmWarps) : "memory");
    if (threadIdx.x == 0) {
      g_timeline[blockIdx.x][1] = gtimer();
      g_timeline[blockIdx.x][3] = (unsigned long long)*(volatile int32_t*)p.task_counter;
    }
#endif
    if (p.n_tasks > 0 && kLateJoin) {
      // This CTA's GEMM has drained (the epilogue consumed the last tile, so the leader's
      // UMMAs no longer read these stages): its 6 warps join the attention pool, each with a
      // 2-stage ring carved from the freed GEMM stage buffers.
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kGemmWarps) : "memory");
      ptx::fence_proxy_async_smem();
      if (warp < kJoin) {
        const FusedTaskMap tm{&p};
        if constexpr (TC)
          at::attn_warp_run_tc<128, 2>(p, &tmap_kv, ps.stages + warp * FS::kJoinBytes,
                                       ctrl_base + (NA + warp) * at::TcCfg<128, NSTA>::CTRL_BYTES, lane, tm,
                                       &tmap_sk, &tmap_sv);
        else
          ap::attn_warp_run<128, 2, FusedTaskMap, QR>(p, ps.stages + warp * FS::kJoinBytes, lane, tm);
      }
    }
  } else {
    const FusedTaskMap tm{&p};
    const int aw = warp - kGemmWarps;
    if constexpr (TC)
      at::attn_warp_run_tc<128, NSTA>(p, &tmap_kv, attn_base + aw * FS::WARP_BYTES,
                                      ctrl_base + aw * at::TcCfg<128, NSTA>::CTRL_BYTES, lane, tm, &tmap_sk, &tmap_sv);
    else
      ap::attn_warp_run<128, NSTA, FusedTaskMap, QR>(p, attn_base + aw * FS::WARP_BYTES, lane, tm);
#ifdef HC_TIMELINE
    if (lane == 0) {
      const unsigned long long t = gtimer();
      atomicMax(&g_timeline[blockIdx.x][2], t);
      atomicMin(&g_timeline[blockIdx.x][4], t);
    }
#endif
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  pg::pair_teardown<NS, kGemmStages>(warp, tmem_base);
}

template <int GS, int NA, int NSTA, bool QR, bool TC, int NS, int EW>
cudaError_t launch_cfg1(const pg::TcArgs& a0, const AttnParams& p0, const void* tmx, const void* tmw,
                        const void* tmkv, const void* const* tms, int num_sms, cudaStream_t s) {
  constexpr int smem = 1024 + FusedSmem<GS, NA, NSTA, QR, TC, NS>::TOTAL;
  static_assert(smem <= 232448, "fused kernel exceeds 227 KiB of shared memory");
  auto k = fused_step_kernel<GS, NA, NSTA, QR, TC, NS, EW>;
  pg::TcArgs a = a0;
  AttnParams p = p0;
  a.epi_split = EW ? 2 : 1;
  p.tile_target = 8 * a.epi_split;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int pairs = num_sms / 2;
  k<<<2 * pairs, pg::GEMM_THREADS + 32 * (NA + EW), smem, s>>>(*static_cast<const CUtensorMap*>(tmx),
                                                        *static_cast<const CUtensorMap*>(tmw),
                                                        *static_cast<const CUtensorMap*>(tmkv ? tmkv : tmx),
                                                        *static_cast<const CUtensorMap*>(tms[0] ? tms[0] : tmx),
                                                        *static_cast<const CUtensorMap*>(tms[1] ? tms[1] : tmx),
                                                        *static_cast<const CUtensorMap*>(tms[2] ? tms[2] : tmx), a, p);
  return cudaGetLastError();
}
template <int GS, int NA, int NSTA, bool QR, int NS = 2, int EW = 0>
cudaError_t launch_cfg(const pg::TcArgs& a, const AttnParams& p, const void* tmx, const void* tmw, const void* tmkv,
                       const void* const* tms, int num_sms, cudaStream_t s) {
  if (p.tc) return launch_cfg1<GS, NA, NSTA, QR, true, NS, EW>(a, p, tmx, tmw, tmkv, tms, num_sms, s);
  return launch_cfg1<GS, NA, NSTA, QR, false, NS, EW>(a, p, tmx, tmw, tmkv, tms, num_sms, s);
}

}  // namespace

bool fused_supported(int d, int dk, int dh, int B) {
  return dh == 128 && dk % dh == 0 && d % 64 == 0 && (2 * dk) % 256 == 0 && B % 16 == 0 &&
         B >= 16 && (B <= 128 || B % 256 == 0) && (B & (B - 1)) == 0;
}
int fused_tile_m() { return pg::P_BM; }
int fused_tile_n() { return 256; }   // the narrowest tile (NSUB = 1): sizes per-tile arrays for either

cudaError_t launch_fused(const ReconParams& rp, AttnParams ap_, const void* tmap_x, const void* tmap_w_half,
                         int32_t* tile_done, int num_sms, const Tuning& t, cudaStream_t s, const void* tmap_kv,
                         int* cfg_out, const void* tmap_scr_k, const void* tmap_scr_v, const void* tmap_x128) {
  const void* tms[3] = {tmap_scr_k, tmap_scr_v, tmap_x128};
  pg::TcArgs a{};
  a.gather = rp.gather;
  a.n_hblocks = rp.n_hblocks;
  a.B = rp.B;
  a.M = rp.n_hblocks * rp.B;
  a.rows_per_box = (rp.B < 128 && !t.diag_box) ? rp.B : 128;
  a.runs = (tmap_x128 != nullptr && a.rows_per_box < 128) ? 1 : 0;
  a.m_tiles = (a.M + pg::P_BM - 1) / pg::P_BM;
  // Tile width: 256 x 512 pair tiles (NSUB = 2; one 512-column accumulator) whenever 2 dk is a
  // multiple of 512; 256 x 256 tiles with two accumulators (NSUB = 1) otherwise.  Measured on
  // GQA (where the attend epilogue serves G query heads per rebuilt K/V head) the second
  // accumulator does not pay for the halved operand reuse: LLaMA-3-8B 3.26 vs 2.75 ms, cfg4
  // 64.5 vs 40.9 ms.
  const int nsub = t.fused_nsub ? t.fused_nsub : ((2 * rp.dk) % 512 != 0 ? 1 : 2);
  const int tile_n = 256 * nsub;
  a.n_tiles = 2 * rp.dk / tile_n;
  a.k_iters = rp.d / pg::BK;
  a.H = rp.Hk;
  a.grp = rp.H / rp.Hk;
  a.dk = rp.dk;
  a.dh = rp.dh;
  a.d = rp.d;
  a.scr_k = static_cast<__nv_bfloat16*>(rp.scr_k);
  a.scr_v = static_cast<__nv_bfloat16*>(rp.scr_v);
  a.bias = rp.b_int;
  a.rope_inv = rp.rope_inv;
  a.row_pos = rp.hblk_pos;
  // n-major raster, 4 n-tiles per group: four pairs of a wave share each A panel (same-box
  // A/B vs 2: cfg4 -2.5%, cfg5 1/32 -2..-4%)
  // (HC_GROUP_N = -g: m-major groups of g m-tiles sweeping all n-tiles instead)
  a.group_m = t.group_n <= -1 ? -t.group_n : -(t.group_n >= 1 ? t.group_n : 4);
  a.l2_hint = t.l2_hint;
  // Partner lockstep off by default in the fused kernel: with the attend epilogue, tiles of
  // partner pairs finish at different times and the spin costs more than the L2 reuse buys
  // (same-box A/B: cfg4 -2.5%, cfg3 -2%, cfg2 -1%, crossover neutral).
  // HC_SYNC_W=<w> re-enables it with window w (the stand-alone GEMM keeps w = 8).
  a.sync_w = t.sync_w > 0 ? t.sync_w : 0;
  a.sync = (a.sync_w > 0 && num_sms / 2 <= pg::kMaxSyncPairs) ? rp.sync_counter : nullptr;
  // Dynamic tile schedule (pair_gemm.cuh pair_roles): the pairs that share an A panel start its
  // tiles together instead of drifting apart; the partner lockstep assumes the static stride.
  a.tile_counter = t.dyn_tiles ? rp.tile_counter : nullptr;
  if (a.tile_counter) a.sync = nullptr;
  if (rp.epi_attend) {   // hidden rows become partials in the GEMM epilogue: no hidden tasks
    a.epi = pg::EPI_ATTEND;
    a.hblk_req = rp.hblk_req;
    a.reqs = rp.reqs;
    a.q = static_cast<const __nv_bfloat16*>(rp.q);
    a.part_ml = rp.part_ml;
    a.part_acc = rp.part_acc;
    a.n_splits_all = rp.n_splits_all;
    a.scale_log2 = rp.scale_log2;
    a.seg = rp.seg;
    tile_done = nullptr;
    a.diag = t.diag_epi;
    // the attend epilogue on mma.sync (pair_gemm.cuh attend_tile_mma): dh = 128
    a.epi_mma = (rp.dh == 128 && (rp.seg == 16 || rp.seg == 32) &&
                 (t.epi_mma == 2 || (t.epi_mma == 1 && rp.H > rp.Hk))) ? 1 : 0;
  }
  a.epi_split = 1;
  ap_.tile_target = 8;
  a.tile_done = tile_done;
  ap_.tile_done = tile_done;
  ap_.gemm_n_tiles = a.n_tiles;
  ap_.gemm_tile_m = pg::P_BM;
  ap_.gemm_tile_n = tile_n;
  // 3-stage GEMM ring + 5 attention warps x 2 stages with q_h in registers (the stages carry
  // only K and V chunks, which frees the smem for the fifth warp: more KV bytes in flight
  // next to the GEMM; crossover 1/64-1/32 -1.5..-7% on cool boxes, neutral elsewhere).
  // Measured earlier (q staged): {3,4,2} best of {3,3,3}, {2,6,2}, {2,4,3} — two GEMM stages
  // starve the tensor cores.
  // When the rebuild is small next to the KV stream (est. GEMM time < half the KV time,
  // e.g. 1/64 of OPT-66B requests hidden), a 2-stage GEMM ring and 8 attention warps
  // stream KV faster (-4% at 1/64); from 1/32 up the 2-stage ring starves the tensor cores
  // (+15..+25%), so the default stays <3,5,2>.
  const double t_gemm = 4.0 * rp.d * (double)rp.dk * a.M / 1.3e15;
  const double t_kv = (double)rp.kv_tokens * 4.0 * rp.dk / 6.5e12;
  if (nsub == 1) {   // 256 x 256 tiles: 32-KiB stages, 4 of them (the same bytes in flight as 3 x 48)
    const int cfg = t.fused_cfg ? t.fused_cfg : (t_gemm < 0.5 * t_kv ? 382 : 452);
    if (cfg_out) *cfg_out = 10000 + cfg;
    if (cfg == 382) return launch_cfg<3, 8, 2, true, 1>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
    return launch_cfg<4, 5, 2, true, 1>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
  }
  // GQA: the tensor-core KV loop drains the KV stream early, so 2 attention warps suffice and
  // 4 extra epilogue warps split the G-query-head attend epilogue (cfg 3224)
  // GEMM-dominated batches (KV stream < 5% of the rebuild, or none) and GQA with the attend
  // epilogue: 2 attention warps + 8 epilogue warps (cfg 3224: 12 warps keep 168 registers per
  // thread; with 3-4 attention warps ptxas drops to 128 and spills).  Same-box A/B against
  // <3,5,2>: cfg4 40.8 vs 41.2 ms (tensor pipe 88 vs 86%), cfg2 1.020 vs 1.040 ms, cfg3
  // 3.62-3.67 vs 3.64-3.70 ms, all-hidden -0.7%; wherever the KV stream matters (cfg5
  // 1/64..1/4) the attention warps win (+4% and more), so those batches keep <3,5,2> / <2,8,2>.
  const bool epi_heavy = t_kv < 0.05 * t_gemm;
  const int cfg = t.fused_cfg ? t.fused_cfg
                              : (((rp.H > rp.Hk && rp.epi_attend) || epi_heavy) ? 3224
                                                                                 : (t_gemm < 0.5 * t_kv ? 282 : 352));
  if (cfg_out) *cfg_out = cfg;
  if (cfg == 3224) return launch_cfg<3, 2, 2, true, 2, 4>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
  if (cfg == 3424) return launch_cfg<3, 4, 2, true, 2, 4>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
  if (cfg == 3324) return launch_cfg<3, 3, 2, true, 2, 4>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
  if (cfg == 342) return launch_cfg<3, 4, 2, true>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
  if (cfg == 282) return launch_cfg<2, 8, 2, true>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
  return launch_cfg<3, 5, 2, true>(a, ap_, tmap_x, tmap_w_half, tmap_kv, tms, num_sms, s);
}

}  // namespace hc

#ifdef HC_TIMELINE
// Diagnostic build only (not in hc.h): copy the per-CTA stamps of the last fused launch.
extern "C" int hc_debug_timeline(unsigned long long* host, int n_ctas) {
  if (n_ctas > 512) n_ctas = 512;
  return (int)cudaMemcpyFromSymbol(host, hc::g_timeline, sizeof(unsigned long long) * 5 * n_ctas);
}
#endif
