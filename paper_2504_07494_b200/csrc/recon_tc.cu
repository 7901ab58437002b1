// tcgen05 / TMEM / TMA K/V reconstruction GEMM for sm_100a.
//
//   [K || V] = X W_KV^T (+ b)                       Eq. 1 on every cached x_j
//
// M = rows of the gathered hidden blocks (sum over hidden requests of ceil(n_i/B)*B),
// N = 2d, K = d.  The hidden cache's "extra linear transformation cost" (t = rho m,
// P:308-311) is exactly this contraction: 4 d^2 FLOPs per cached hidden token, so it
// runs on the 5th-generation tensor cores.
//
// Design (one CTA per SM, persistent, warp-specialised, 192 threads):
//   warp 0      TMA producer.  A tile = 128 gathered rows x 64 k: 128/min(B,128) boxes of
//               [min(B,128) rows x 64] bf16, one per hidden block (the block-wise hidden
//               cache is the A operand — no gather copy), SWIZZLE_128B.  B tile = 256 rows
//               of the head-interleaved W_KV (K_h || V_h for 128-wide heads) x 64 k.
//               4-stage smem ring (48 KiB/stage), full/empty mbarriers.
//   warp 1      TMEM allocator + single-thread MMA issuer: tcgen05.mma.cta_group::1
//               kind::f16, M=128 N=256 K=16, fp32 accumulators in TMEM, two accumulator
//               buffers (2 x 256 columns) so the epilogue of tile i overlaps tile i+1.
//               tcgen05.commit releases smem stages / signals the epilogue.
//   warps 2-5   epilogue: tcgen05.ld 32x32b.x32 (thread = one output row), + bias,
//               RNE to bf16, store K_h and V_h rows into scratch blocks [hblock][H][B][dh].
// Tile order: grouped rasterisation (GROUP_M m-tiles sweep all n-tiles) so a wave of 148
// tiles shares A and W_KV tiles in L2 (W_KV is 340 MB at OPT-66B, larger than L2).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>

#include "internal.h"
#include "pair_gemm.cuh"
#include "ptx.cuh"

namespace hc {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;      // 16 KiB
constexpr int B_BYTES = BN * BK * 2;      // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 192;
constexpr int GROUP_M = 16;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/;

__device__ __forceinline__ void tile_coords(int t, int m_tiles, int n_tiles, int& mt, int& nt) {
  const int per_group = GROUP_M * n_tiles;
  const int g = t / per_group;
  const int first_m = g * GROUP_M;
  const int gsize = min(GROUP_M, m_tiles - first_m);
  const int r = t - g * per_group;
  mt = first_m + r % gsize;
  nt = r / gsize;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    recon_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                    const pg::TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
  uint8_t* sA = smem;                              // STAGES x 16 KiB
  uint8_t* sB = smem + STAGES * A_BYTES;           // STAGES x 32 KiB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_total = a.m_tiles * a.n_tiles;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    ptx::prefetch_tmap(&tmap_w);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int nbox = BM / a.rows_per_box;
      const int box_bytes = a.rows_per_box * BK * 2;
      for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
        int mt, nt;
        tile_coords(t, a.m_tiles, a.n_tiles, mt, nt);
        // physical pool rows of this m-tile's boxes (gathered hidden blocks)
        int prow[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          prow[i] = 0;
          if (i < nbox) {
            const int grow = mt * BM + i * a.rows_per_box;
            const int g = grow / a.B;
            if (g < a.n_hblocks) prow[i] = a.gather[g] * a.B + (grow - g * a.B);
          }
        }
        for (int kb = 0; kb < a.k_iters; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          uint8_t* dA = sA + stage * A_BYTES;
          for (int i = 0; i < nbox; ++i)
            ptx::tma_load_2d(dA + i * box_bytes, &tmap_x, kb * BK, prow[i], &full[stage]);
          ptx::tma_load_2d(sB + stage * B_BYTES, &tmap_w, kb * BK, nt * BN, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc_bf16_f32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < a.k_iters; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + stage * A_BYTES);
          const uint32_t b_addr = ptx::smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = ptx::umma_desc_k_sw128(a_addr + k * 32);
            const uint64_t bd = ptx::umma_desc_k_sw128(b_addr + k * 32);
            ptx::umma_f16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue (warps 2..5) =================
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int row_in_tile = q * 32 + lane;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
      int mt, nt;
      tile_coords(t, a.m_tiles, a.n_tiles, mt, nt);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int grow = mt * BM + row_in_tile;
      const bool valid = grow < a.M;
      const int g = grow / a.B, r = grow - g * a.B;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
        ptx::tmem_ld_wait();
        const int n = nt * BN + c * 32;            // interleaved output column
        const int h = n / (2 * a.dh), rem = n - h * 2 * a.dh, kv = rem / a.dh, c0 = rem - kv * a.dh;
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        if (a.bias) {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] += __ldg(a.bias + n + j);
        }
        if (valid) {
          __nv_bfloat16* dst = (kv ? a.scr_v : a.scr_k) + (((size_t)g * a.H + h) * a.B + r) * a.dh + c0;
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            d4[j] = make_uint4(pg::pack_bf16(f[8 * j], f[8 * j + 1]), pg::pack_bf16(f[8 * j + 2], f[8 * j + 3]),
                               pg::pack_bf16(f[8 * j + 4], f[8 * j + 5]), pg::pack_bf16(f[8 * j + 6], f[8 * j + 7]));
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
}


// ------------------------------------------------------------------------------------
// CTA-pair kernel: the roles live in pair_gemm.cuh (shared with the fused step kernel).
template <int NSUB, int NSTAGE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pg::GEMM_THREADS, 1)
    recon_tc2_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                     const __grid_constant__ CUtensorMap tmap_x128, const pg::TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
  const pg::PairSmem ps = pg::pair_carve<NSUB, NSTAGE>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pg::pair_setup<NSUB, NSTAGE>(ps, warp, lane, &tmap_x, &tmap_w);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *ps.tmem_slot;
  pg::pair_roles<NSUB, NSTAGE>(ps, warp, lane, &tmap_x, &tmap_w, a, tmem_base, a.runs ? &tmap_x128 : nullptr);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  pg::pair_teardown<NSUB, NSTAGE>(warp, tmem_base);
}

template <int NSUB, int NSTAGE>
cudaError_t launch_pair(pg::TcArgs a, const void* tmap_x, const void* tmap_w_half, int num_sms, cudaStream_t s,
                        const void* tmap_x128 = nullptr) {
  a.runs = (tmap_x128 != nullptr && a.gather != nullptr && a.rows_per_box < 128) ? 1 : 0;
  using PC = pg::PairCfg<NSUB, NSTAGE>;
  constexpr int smem = 1024 + PC::REGION_BYTES;
  a.m_tiles = (a.M + pg::P_BM - 1) / pg::P_BM;
  a.n_tiles = (a.n_total > 0 ? a.n_total : 2 * a.dk) / PC::TILE_N;   // reconstruction: N = 2 dk (K || V)
  cudaError_t e = cudaFuncSetAttribute(recon_tc2_kernel<NSUB, NSTAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int tiles = a.m_tiles * a.n_tiles;
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  if (pairs > pg::kMaxSyncPairs) a.sync = nullptr;
  recon_tc2_kernel<NSUB, NSTAGE><<<2 * pairs, pg::GEMM_THREADS, smem, s>>>(
      *static_cast<const CUtensorMap*>(tmap_x), *static_cast<const CUtensorMap*>(tmap_w_half),
      *static_cast<const CUtensorMap*>(tmap_x128 ? tmap_x128 : tmap_x), a);
  return cudaGetLastError();
}

}  // namespace

bool dense_tc_supported(int d) { return d % 256 == 0; }

bool recon_pair_mode(int B, const Tuning& t) { return (B <= 128 || B % 256 == 0) && t.tc_1sm == 0; }

cudaError_t launch_dense_tc(const DenseParams& p, const void* tmap_a, const void* tmap_w, int num_sms, cudaStream_t s) {
  if (p.M <= 0) return cudaSuccess;
  pg::TcArgs a{};
  a.gather = nullptr;   // dense A rows
  a.M = p.M;
  a.B = p.B;
  a.rows_per_box = 128;
  a.k_iters = p.K / BK;
  a.H = p.dk / p.dh;
  a.grp = 1;
  a.dh = p.dh;
  a.d = p.d;
  a.dk = p.dk;
  a.Bkv = p.Bkv;
  a.v_off = p.v_off;
  a.bias = p.bias;
  a.group_m = -2;
  a.epi = p.epi;
  a.n_total = p.N;
  a.out = static_cast<__nv_bfloat16*>(p.out);
  a.pool = static_cast<__nv_bfloat16*>(p.pool);
  a.row_dst = p.row_dst;
  a.kvbuf = static_cast<__nv_bfloat16*>(p.kvbuf);
  a.rope_inv = p.rope_inv;
  if (p.N % 512 == 0) return launch_pair<2, 4>(a, tmap_a, tmap_w, num_sms, s);
  return launch_pair<1, 6>(a, tmap_a, tmap_w, num_sms, s);
}

bool recon_tc_supported(int d, int dk, int dh, int B) {
  if (d % BK != 0 || dk % dh != 0) return false;
  if ((2 * dh) > BN || BN % (2 * dh) != 0 || dh % 32 != 0) return false;
  if ((2 * dk) % BN != 0) return false;
  if (B < 8 || (B & (B - 1)) != 0) return false;  // power of two >= 8: boxes are whole swizzle atoms
  if (B > BM && B % BM != 0) return false;
  return true;
}

cudaError_t launch_recon_tc(const ReconParams& p, const void* tmap_x, const void* tmap_w,
                            const void* tmap_w_half, int num_sms, const Tuning& t, cudaStream_t s,
                            const void* tmap_x128) {
  if (p.n_hblocks <= 0) return cudaSuccess;
  pg::TcArgs a{};
  a.gather = p.gather;
  a.n_hblocks = p.n_hblocks;
  a.B = p.B;
  a.M = p.n_hblocks * p.B;
  a.rows_per_box = p.B < BM ? p.B : BM;
  a.m_tiles = (a.M + BM - 1) / BM;
  a.n_tiles = 2 * p.dk / BN;
  a.k_iters = p.d / BK;
  a.H = p.Hk;
  a.grp = p.H / p.Hk;
  a.dk = p.dk;
  a.dh = p.dh;
  a.d = p.d;
  a.scr_k = static_cast<__nv_bfloat16*>(p.scr_k);
  a.scr_v = static_cast<__nv_bfloat16*>(p.scr_v);
  a.bias = p.b_int;
  a.rope_inv = p.rope_inv;
  a.row_pos = p.hblk_pos;
  if (p.epi_attend) {   // fused reconstruct-and-attend: partials instead of scratch K/V
    a.epi = pg::EPI_ATTEND;
    a.hblk_req = p.hblk_req;
    a.reqs = p.reqs;
    a.q = static_cast<const __nv_bfloat16*>(p.q);
    a.part_ml = p.part_ml;
    a.part_acc = p.part_acc;
    a.n_splits_all = p.n_splits_all;
    a.scale_log2 = p.scale_log2;
    a.seg = p.seg;
  }
  // Default schedule: n-major raster with 2 n-tiles per group, so pairs p and p^1 of a wave
  // share one A panel and every wave shares the group's W panels; the partner lockstep
  // makes the shared A panel hit in L2 (measured: DRAM reads 190 GB -> ~60 GB at OPT-66B).
  a.group_m = t.group_m != 0 ? t.group_m : -2;
  a.l2_hint = t.l2_hint;
  a.sync_w = t.sync_w >= 0 ? t.sync_w : 8;
  a.sync = (a.sync_w > 0 && a.group_m == -2) ? p.sync_counter : nullptr;
  const bool pair_mode = recon_pair_mode(p.B, t) || p.rope_inv || p.epi_attend;
  if (pair_mode) {
    const bool can2 = (2 * p.dk) % 512 == 0;
    if (can2 && t.tc_nsub != 1) {
      if (t.tc_stages == 3) return launch_pair<2, 3>(a, tmap_x, tmap_w_half, num_sms, s, tmap_x128);
      return launch_pair<2, 4>(a, tmap_x, tmap_w_half, num_sms, s, tmap_x128);
    }
    return launch_pair<1, 6>(a, tmap_x, tmap_w_half, num_sms, s, tmap_x128);
  }
  cudaError_t e = cudaFuncSetAttribute(recon_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles = a.m_tiles * a.n_tiles;
  const int grid = tiles < num_sms ? tiles : num_sms;
  recon_tc_kernel<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(*static_cast<const CUtensorMap*>(tmap_x),
                                                      *static_cast<const CUtensorMap*>(tmap_w), a);
  return cudaGetLastError();
}

}  // namespace hc
