// Measurement tool (not part of libhc): L2 -> SM and HBM -> SM streaming bandwidth with
// 1-D bulk copies (cp.async.bulk, the TMA engine's path) into a per-CTA smem ring, one
// persistent CTA per SM.  Used to put a number on the on-chip operand fabric that the
// reconstruction GEMM and the KV stream share at the hidden/KV crossover.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2504_07494_b200/csrc \
//        scripts/l2_fabric_bw.cu -o /tmp/l2bw && /tmp/l2bw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "ptx.cuh"

using namespace hc;

template <int CHUNK, int NST>
__global__ void __launch_bounds__(32, 1) stream_kernel(const uint8_t* buf, size_t buf_bytes, long long per_cta,
                                                       unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * CHUNK);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const size_t n_chunks = buf_bytes / CHUNK;
  // each CTA walks the buffer from its own offset with a large odd stride: at any time the
  // 148 CTAs read different lines, every line is read by every CTA over the run
  size_t c = (size_t)blockIdx.x * 7919 % n_chunks;
  const long long iters = per_cta / CHUNK;
  uint32_t acc = 0;
  for (long long it = 0; it < iters; ++it) {
    const int st = (int)(it % NST);
    if (it >= NST) {
      ptx::mbar_wait(&full[st], (uint32_t)(((it / NST) - 1) & 1));
      acc += smem[st * CHUNK + (it & 127)];
    }
    ptx::mbar_arrive_expect_tx(&full[st], CHUNK);
    ptx::bulk_g2s(smem + st * CHUNK, buf + c * CHUNK, CHUNK, &full[st]);
    c += 131;
    if (c >= n_chunks) c -= n_chunks;
  }
  for (long long it = iters; it < iters + NST; ++it) {
    const int st = (int)(it % NST);
    if (it >= NST) ptx::mbar_wait(&full[st], (uint32_t)(((it / NST) - 1) & 1));
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  constexpr int CHUNK = 16384, NST = 8;
  const int smem = NST * CHUNK + 8 * NST;
  cudaFuncSetAttribute(stream_kernel<CHUNK, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const size_t sizes[] = {size_t(32) << 20, size_t(64) << 20, size_t(96) << 20, size_t(4) << 30};
  for (size_t bytes : sizes) {
    uint8_t* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
    cudaMemset(buf, 1, bytes);
    const long long per_cta = 256ll << 20;   // 256 MiB per CTA -> 37.9 GB over 148 SMs
    for (int rep = 0; rep < 2; ++rep) stream_kernel<CHUNK, NST><<<sms, 32, smem>>>(buf, bytes, per_cta, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int rep = 0; rep < reps; ++rep) stream_kernel<CHUNK, NST><<<sms, 32, smem>>>(buf, bytes, per_cta, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tb = (double)per_cta * sms * reps / (ms * 1e-3) / 1e12;
    printf("{\"buffer_MiB\": %zu, \"chunk\": %d, \"stages\": %d, \"ctas\": %d, \"TBps\": %.3f, \"err\": \"%s\"}\n",
           bytes >> 20, CHUNK, NST, sms, tb, cudaGetErrorString(cudaGetLastError()));
    cudaFree(buf);
  }
  return 0;
}
