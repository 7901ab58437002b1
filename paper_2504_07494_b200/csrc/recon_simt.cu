// SIMT K/V reconstruction (SURVEY §8 row a4, fp32 mode and the bf16 cross-check path).
//
// [K || V] = X_hat W_KV^T (+ b), Eq. 1, for every cached hidden token
// (P:269-271).  Rows of X are gathered from the request's hidden blocks (row-major
// [B][d] unit blocks); the result is written to scratch in the attention kernel's
// [hblock][H][B][dh] block layout.  64x64 output tile per CTA, 4x4 per thread, fp32
// accumulation, one rounding to the storage type (RNE) at the end.
#include <cuda_bf16.h>

#include "internal.h"

namespace hc {
namespace {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
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

template <typename T>
__global__ void __launch_bounds__(256) recon_simt_kernel(const ReconParams p) {
  constexpr int TM = 64, TN = 64, TK = 16;
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
  const int d = p.d, B = p.B, M = p.n_hblocks * B, N = 2 * p.dk;
  const T* pool = static_cast<const T*>(p.pool);
  const T* w = static_cast<const T*>(p.w_int);
  float acc[4][4] = {};
  // loader mapping: 256 threads x 4 elements = 64 rows x 16 k
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  const int gm = m0 + lr;
  const T* arow = nullptr;
  if (gm < M) {
    const int g = gm / B, r = gm - g * B;
    arow = pool + ((size_t)p.gather[g] * B + r) * d;
  }
  const int gn = n0 + lr;
  const T* brow = gn < N ? w + (size_t)gn * d : nullptr;
  for (int k0 = 0; k0 < d; k0 += TK) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + lk + j;
      As[lk + j][lr] = (arow && k < d) ? to_f(arow[k]) : 0.f;
      Bs[lk + j][lr] = (brow && k < d) ? to_f(brow[k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        b[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int H = p.Hk, dh = p.dh;   // scratch [hblock][Hk][B][dh]
  T* sk = static_cast<T*>(p.scr_k);
  T* sv = static_cast<T*>(p.scr_v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm2 = m0 + ty * 4 + i;
    if (gm2 >= M) continue;
    const int g = gm2 / B, r = gm2 - g * B;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      const int h = n / (2 * dh), rem = n - h * 2 * dh, kv = rem / dh, c = rem - kv * dh;
      float v = acc[i][j];
      if (p.b_int) v += p.b_int[n];
      T* dst = (kv ? sv : sk) + (((size_t)g * H + h) * B + r) * dh + c;
      *dst = from_f<T>(v);
    }
  }
}

// Dense C = A W^T (+ bias) with the projection epilogues (see DenseParams).
template <typename T>
__global__ void __launch_bounds__(256) dense_simt_kernel(const DenseParams p) {
  constexpr int TM = 64, TN = 64, TK = 16;
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
  const int K = p.K, M = p.M, N = p.N;
  const T* A = static_cast<const T*>(p.a);
  const T* W = static_cast<const T*>(p.w);
  float acc[4][4] = {};
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  const T* arow = (m0 + lr) < M ? A + (size_t)(m0 + lr) * K : nullptr;
  const T* brow = (n0 + lr) < N ? W + (size_t)(n0 + lr) * K : nullptr;
  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + lk + j;
      As[lk + j][lr] = (arow && k < K) ? to_f(arow[k]) : 0.f;
      Bs[lk + j][lr] = (brow && k < K) ? to_f(brow[k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        b[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  T* out = static_cast<T*>(p.out);
  T* pool = static_cast<T*>(p.pool);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (p.bias) v += p.bias[n];
      if (p.epi == 2) {
        out[(size_t)row * N + n] = from_f<T>(v);
      } else if (n < p.d) {
        out[(size_t)row * p.d + n] = from_f<T>(v);
      } else {
        const int m = n - p.d;
        if (p.kvbuf) static_cast<T*>(p.kvbuf)[(size_t)row * 2 * p.dk + m] = from_f<T>(v);
        const int4 di = reinterpret_cast<const int4*>(p.row_dst)[row];
        if (di.x < 0) continue;
        const int h = m / (2 * p.dh), rem = m - h * 2 * p.dh, kv = rem / p.dh, c = rem - kv * p.dh;
        const int blk = kv ? di.y : di.x;
        pool[(size_t)blk * p.B * p.d + (kv ? p.v_off : 0) + (size_t)h * p.Bkv * p.dh + (size_t)di.z * p.dh + c] =
            from_f<T>(v);
      }
    }
  }
}

}  // namespace

cudaError_t launch_dense_simt(const DenseParams& p, int dtype, cudaStream_t s) {
  if (p.M <= 0) return cudaSuccess;
  dim3 grid((p.M + 63) / 64, (p.N + 63) / 64);
  if (dtype == 1)
    dense_simt_kernel<float><<<grid, 256, 0, s>>>(p);
  else
    dense_simt_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_recon_simt(const ReconParams& p, int dtype, cudaStream_t s) {
  if (p.n_hblocks <= 0) return cudaSuccess;
  const int M = p.n_hblocks * p.B, N = 2 * p.dk;
  dim3 grid((M + 63) / 64, (N + 63) / 64);
  if (dtype == 1)
    recon_simt_kernel<float><<<grid, 256, 0, s>>>(p);
  else
    recon_simt_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace hc
