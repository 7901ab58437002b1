// Cache append, weight re-layout, split combine (row a6).
#include <cuda_bf16.h>

#include "internal.h"

namespace hc {

namespace {

// Block-wise cache write, "fusing reshaping with read/write": each appended row
// goes to (table[pos / Bb], pos % Bb).  KV rows are scattered head-major ([Hk][Bkv][dh] per
// K (V) region, so a head's rows of a block are contiguous for the attention reads; under
// GQA the V region sits v_off elements into the same unit); hidden rows are stored
// row-major ([B][d], the GEMM's gathered A operand).
// 16-byte vectors; grid.y = request of the call, grid.x strides over its rows.
template <typename T>
__global__ void __launch_bounds__(256) append_kernel(const AppendParams p) {
  const AppendReq rq = p.reqs[blockIdx.y];
  constexpr int VE = 16 / sizeof(T);   // elements per vector
  const int d = p.d, B = p.B, dh = p.dh, dk = p.dk;
  const int Bb = rq.mode == 0 ? p.Bkv : B;   // tokens per logical block of this mode
  T* pool = static_cast<T*>(p.pool);
  const int lb_first = rq.start / Bb;
  for (int r = blockIdx.x; r < rq.n_tok; r += gridDim.x) {
    const int pos = rq.start + r;
    const int lb = pos / Bb - lb_first, row = pos % Bb;
    if (rq.mode == 0) {
      const size_t src_row = (size_t)(rq.row_off + r) * dk;
      const int kb = p.tabs[rq.tab_off + 2 * lb], vb = p.tabs[rq.tab_off + 2 * lb + 1];
      const uint4* ks = reinterpret_cast<const uint4*>(static_cast<const T*>(p.k) + src_row);
      const uint4* vs = reinterpret_cast<const uint4*>(static_cast<const T*>(p.v) + src_row);
      for (int e = threadIdx.x; e < dk / VE; e += blockDim.x) {
        const int col = e * VE, h = col / dh, c = col - h * dh;
        const size_t off = (size_t)h * Bb * dh + (size_t)row * dh + c;
        *reinterpret_cast<uint4*>(pool + (size_t)kb * B * d + off) = ks[e];
        *reinterpret_cast<uint4*>(pool + (size_t)vb * B * d + p.v_off + off) = vs[e];
      }
    } else {
      const size_t src_row = (size_t)(rq.row_off + r) * d;
      const int nvec = d / VE;
      const int xb = p.tabs[rq.tab_off + lb];
      const uint4* xs = reinterpret_cast<const uint4*>(static_cast<const T*>(p.x) + src_row);
      uint4* dst = reinterpret_cast<uint4*>(pool + (size_t)xb * B * d + (size_t)row * d);
      for (int e = threadIdx.x; e < nvec; e += blockDim.x) dst[e] = xs[e];
    }
  }
}

// W_int[h*2dh + kv*dh + c, :] = W_KV[kv*dk + h*dh + c, :]  (and the bias likewise; h runs
// over the Hk K/V heads, dk = Hk*dh): one N=256 GEMM tile of the head-interleaved weight
// then yields K_h || V_h directly.
template <typename T>
__global__ void __launch_bounds__(256) relayout_kernel(const T* __restrict__ w, T* __restrict__ wi,
                                                       const float* __restrict__ b, float* __restrict__ bi,
                                                       int d, int dk, int dh) {
  const int dst = blockIdx.x;   // 0 .. 2dk-1
  const int h = dst / (2 * dh), rem = dst - h * 2 * dh, kv = rem / dh, c = rem - kv * dh;
  const int src = kv * dk + h * dh + c;
  constexpr int VE = 16 / sizeof(T);
  const uint4* s = reinterpret_cast<const uint4*>(w + (size_t)src * d);
  uint4* o = reinterpret_cast<uint4*>(wi + (size_t)dst * d);
  for (int e = threadIdx.x; e < d / VE; e += blockDim.x) o[e] = s[e];
  if (threadIdx.x == 0 && bi != nullptr) bi[dst] = b ? b[src] : 0.f;
}

template <typename T>
__device__ __forceinline__ void st_out(T* p, float v);
template <>
__device__ __forceinline__ void st_out<float>(float* p, float v) {
  *p = v;
}
template <>
__device__ __forceinline__ void st_out<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

// Split combine: M = max_s m_s, L = sum_s 2^(m_s-M) l_s, out = sum_s 2^(m_s-M) acc_s / L,
// lse = (M + log2 L) ln 2 (scores were kept in log2 units).  One CTA (256 threads) per
// (request, head): block reductions for M and L, the split weights 2^(m_s - M) staged in
// shared memory chunk by chunk, then 256/dh groups of threads each accumulate every output
// dimension over an interleaved subset of the splits (partials are head-major, so the
// splits of one (request, head) are contiguous), reduced through shared memory.
template <typename T>
__global__ void __launch_bounds__(256) combine_kernel(const CombineParams p) {
  constexpr int NT = 256, kChunk = 512;
  __shared__ float w_s[kChunk];
  __shared__ float red[NT / 32];
  __shared__ float part[NT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = blockIdx.x / p.H, h = blockIdx.x - r * p.H;
  const ReqDesc rq = p.reqs[r];
  if (rq.split_count == 0) return;   // absorbed hidden request: written by wv_kernel
  const int H = p.H, dh = p.dh, cnt = rq.split_count;
  const size_t base_idx = (size_t)h * p.n_splits + rq.split_begin;   // head-major: splits contiguous
  const float* ml = p.part_ml + 2 * base_idx;                         // split s at ml[2 s]
  auto block_reduce = [&](float v, bool is_max) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float u = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmaxf(v, u) : v + u;
    }
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = red[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) t = is_max ? fmaxf(t, red[w]) : t + red[w];
    __syncthreads();
    return t;
  };
  float M = -INFINITY;
  for (int s = tid; s < cnt; s += NT) M = fmaxf(M, ml[2 * s]);
  M = block_reduce(M, true);
  float L = 0.f;
  for (int s = tid; s < cnt; s += NT) L += exp2f(ml[2 * s] - M) * ml[2 * s + 1];
  L = block_reduce(L, false);
  const float inv = 1.f / L;
  // thread -> (split group, dimension): G = NT / dh groups take interleaved splits
  const int G = NT / dh, grp = tid / dh, c = tid - grp * dh;
  const float* acc = p.part_acc + base_idx * dh;   // split s at s dh
  float o = 0.f;
  for (int base = 0; base < cnt; base += kChunk) {
    const int n = min(kChunk, cnt - base);
    __syncthreads();
    for (int s = tid; s < n; s += NT) w_s[s] = exp2f(ml[2 * (base + s)] - M);
    __syncthreads();
    if (grp < G) {
      const float* a0 = acc + (size_t)base * dh + c;
#pragma unroll 4
      for (int s = grp; s < n; s += G) o = fmaf(w_s[s], a0[(size_t)s * dh], o);
    }
  }
  part[tid] = o;
  __syncthreads();
  T* out = static_cast<T*>(p.out) + (size_t)r * p.d + h * dh;
  for (int cc = tid; cc < dh; cc += NT) {
    float t = 0.f;
    for (int g = 0; g < G; ++g) t += part[g * dh + cc];
    st_out<T>(out + cc, t * inv);
  }
  if (tid == 0 && p.lse) p.lse[(size_t)r * H + h] = (M + log2f(L)) * 0.69314718055994531f;
}

}  // namespace

cudaError_t launch_append(const AppendParams& p, int dtype, int max_rows, cudaStream_t s) {
  if (p.n_req <= 0 || max_rows <= 0) return cudaSuccess;
  dim3 grid(max_rows < 1024 ? max_rows : 1024, p.n_req);
  if (dtype == 1)
    append_kernel<float><<<grid, 256, 0, s>>>(p);
  else
    append_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_relayout_w(const void* w, void* w_int, const float* b, float* b_int, int d, int dk,
                              int dh, int dtype, cudaStream_t s) {
  if (dtype == 1)
    relayout_kernel<float><<<2 * dk, 256, 0, s>>>(static_cast<const float*>(w), static_cast<float*>(w_int),
                                                  b, b_int, d, dk, dh);
  else
    relayout_kernel<__nv_bfloat16><<<2 * dk, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(w),
                                                          static_cast<__nv_bfloat16*>(w_int), b, b_int, d, dk, dh);
  return cudaGetLastError();
}

cudaError_t launch_combine(const CombineParams& p, int dtype, cudaStream_t s) {
  const int blocks = p.n_req * p.H;   // one CTA per (request, head)
  if (blocks <= 0) return cudaSuccess;
  if (p.dh > 256) return cudaErrorInvalidValue;
  if (dtype == 1)
    combine_kernel<float><<<blocks, 256, 0, s>>>(p);
  else
    combine_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ pre-attention LayerNorm
// One CTA (256 threads) per row: two passes over the row (mean, then the centred second
// moment — the population variance, as torch.nn.LayerNorm), fp32 statistics.
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// ------------------------------------------------------------------ cross-partition merge
// SURVEY §8(e) phase 2: a request whose token range is split over P partitions (e.g. ranks
// that each hold part of a long hidden request's blocks) has P partial results, out_p
// normalised over its own range and lse_p = log sum over that range.  Over the union
// (Eq. 2-3): LSE = log sum_p e^{lse_p}, out = sum_p e^{lse_p - LSE} out_p.  A part with
// lse_p = -inf (empty range) weighs 0; a row with no token anywhere gets out = 0,
// lse = -inf.  One CTA per (row, head), threads over dh.
template <typename T>
__global__ void __launch_bounds__(128) merge_kernel(int n_parts, int n_rows, int H, int dh, const T* outs,
                                                    const float* lses, T* out, float* lse) {
  const int r = blockIdx.x / H, h = blockIdx.x - r * H;
  float M = -INFINITY;
  for (int q = 0; q < n_parts; ++q) M = fmaxf(M, lses[((size_t)q * n_rows + r) * H + h]);
  float L = 0.f;
  if (M != -INFINITY)
    for (int q = 0; q < n_parts; ++q) L += expf(lses[((size_t)q * n_rows + r) * H + h] - M);
  const float inv = L > 0.f ? 1.f / L : 0.f;
  for (int c = threadIdx.x; c < dh; c += blockDim.x) {
    float acc = 0.f;
    if (M != -INFINITY) {
      for (int q = 0; q < n_parts; ++q) {
        const float lq = lses[((size_t)q * n_rows + r) * H + h];
        if (lq == -INFINITY) continue;   // empty part: its out is never read (0 * NaN = NaN)
        acc = fmaf(expf(lq - M), to_f(outs[(((size_t)q * n_rows + r) * H + h) * dh + c]), acc);
      }
    }
    out[((size_t)r * H + h) * dh + c] = from_f<T>(acc * inv);
  }
  if (lse != nullptr && threadIdx.x == 0) lse[(size_t)r * H + h] = M == -INFINITY ? M : M + logf(L);
}

cudaError_t launch_merge(int n_parts, int n_rows, int H, int dh, int dtype, const void* outs, const float* lses,
                         void* out, float* lse, cudaStream_t s) {
  if (n_rows == 0) return cudaSuccess;
  const int blocks = n_rows * H;
  if (dtype == 1)
    merge_kernel<float><<<blocks, 128, 0, s>>>(n_parts, n_rows, H, dh, static_cast<const float*>(outs), lses,
                                               static_cast<float*>(out), lse);
  else
    merge_kernel<__nv_bfloat16><<<blocks, 128, 0, s>>>(n_parts, n_rows, H, dh,
                                                       static_cast<const __nv_bfloat16*>(outs), lses,
                                                       static_cast<__nv_bfloat16*>(out), lse);
  return cudaGetLastError();
}


// x and u may alias (each element is read before it is overwritten by the same thread)
template <typename T>
__global__ void __launch_bounds__(256) layer_norm_kernel(const T* x, T* u,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ beta, float eps, int d) {
  __shared__ float red[8];
  const size_t row = blockIdx.x;
  const T* xr = x + row * d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto block_sum = [&](float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w];
    return t;
  };
  float s = 0.f;
  for (int c = tid; c < d; c += 256) s += to_f(xr[c]);
  const float mean = block_sum(s) / d;
  float q = 0.f;
  for (int c = tid; c < d; c += 256) {
    const float t = to_f(xr[c]) - mean;
    q += t * t;
  }
  const float rstd = rsqrtf(block_sum(q) / d + eps);
  T* ur = u + row * d;
  for (int c = tid; c < d; c += 256) ur[c] = from_f<T>((to_f(xr[c]) - mean) * rstd * gamma[c] + beta[c]);
}

cudaError_t launch_layer_norm(const void* x, void* u, const float* gamma, const float* beta, float eps, int rows,
                              int d, int dtype, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (dtype == 1)
    layer_norm_kernel<float><<<rows, 256, 0, s>>>(static_cast<const float*>(x), static_cast<float*>(u), gamma, beta,
                                                  eps, d);
  else
    layer_norm_kernel<__nv_bfloat16><<<rows, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                          static_cast<__nv_bfloat16*>(u), gamma, beta, eps, d);
  return cudaGetLastError();
}

}  // namespace hc
