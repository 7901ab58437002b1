// Measurement tool (not part of libhc): how much HBM bandwidth k SMs can pull with 1-D bulk
// copies into a smem ring of R bytes, optionally running an L2 bulk prefetch PF chunks ahead of
// the copies (bytes in flight without smem).  Question it answers: can a minority of SMs stream
// the KV half of a crossover batch while the rest run the reconstruction GEMM (spatial split,
// DESIGN.md §7)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2504_07494_b200/csrc \
//        scripts/kv_sm_bw.cu -o /tmp/kvbw && /tmp/kvbw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "ptx.cuh"

using namespace hc;

// W producer warps per CTA (lane 0 of each issues), each with its own ring of NST chunks.
__global__ void __launch_bounds__(512, 1) stream_kernel(const uint8_t* buf, size_t n_chunks, int chunk, int nst,
                                                        int pf, long long per_warp_chunks,
                                                        unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint8_t* ring = smem + (size_t)w * nst * chunk;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nw * nst * chunk) + w * nst;
  if (lane == 0) {
    for (int i = 0; i < nst; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  if (lane != 0) return;
  // each warp walks a contiguous stretch (like a KV split of one head), CTAs far apart
  const size_t gw = (size_t)blockIdx.x * nw + w;
  size_t c0 = (gw * (size_t)per_warp_chunks * 2654435761ull) % n_chunks;
  uint32_t acc = 0;
  // 32-bit stage/phase counters and a wrapping pointer: no 64-bit divisions in the issue loop
  const uint8_t* src = buf + c0 * chunk;
  const uint8_t* end = buf + n_chunks * (size_t)chunk;
  int st = 0;
  uint32_t ph = 0;
  const int n = (int)per_warp_chunks;
  for (int it = 0; it < n; ++it) {
    if (it >= nst) {
      ptx::mbar_wait(&full[st], ph ^ 1);
      acc += ring[st * chunk + (it & 127)];
    }
    ptx::mbar_arrive_expect_tx(&full[st], chunk);
    ptx::bulk_g2s(ring + st * chunk, src, chunk, &full[st]);
    src += chunk;
    if (src >= end) src = buf;
    if (++st == nst) {
      st = 0;
      ph ^= 1;
    }
  }
  for (int k = 0; k < nst; ++k) {   // drain the last nst fills (never-filled stages pass at once)
    ptx::mbar_wait(&full[st], ph ^ 1);
    if (++st == nst) {
      st = 0;
      ph ^= 1;
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const size_t big = size_t(8) << 30;
  uint8_t* buf;
  if (cudaMalloc(&buf, big) != cudaSuccess) return 1;
  cudaMemset(buf, 1, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // Sweep: op size, buffer (L2-resident 32 MiB or 8 GiB from HBM), issuing warps, stages per
  // warp (ops in flight per SM = warps x stages), CTAs (one per SM).
  struct Cfg { int chunk, nw, nst; };
  const Cfg cfgs[] = {{2048, 1, 16}, {2048, 2, 16}, {2048, 4, 16}, {2048, 8, 8}, {2048, 16, 4}, {2048, 16, 6},
                      {4096, 1, 16}, {4096, 4, 8}, {4096, 8, 4}, {4096, 16, 3},
                      {8192, 1, 16}, {8192, 4, 4}, {8192, 8, 2}, {8192, 8, 3},
                      {16384, 4, 2}, {16384, 8, 1}};
  for (size_t bytes : {size_t(32) << 20, big}) {
    for (int ctas : {32, 148}) {
      for (const Cfg& c : cfgs) {
        const size_t n_chunks = bytes / c.chunk;
        const int smem = c.nw * c.nst * c.chunk + c.nw * c.nst * 8;
        if (smem > 227 * 1024) continue;
        const long long per_warp = (1ll << 30) / c.chunk / ((long long)ctas * c.nw);
        stream_kernel<<<ctas, 32 * c.nw, smem>>>(buf, n_chunks, c.chunk, c.nst, 0, per_warp, sink);
        cudaEventRecord(e0);
        stream_kernel<<<ctas, 32 * c.nw, smem>>>(buf, n_chunks, c.chunk, c.nst, 0, per_warp, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double moved = (double)per_warp * c.chunk * ctas * c.nw;
        const double ops = (double)per_warp * ctas * c.nw;
        printf("{\"buf_MiB\": %zu, \"chunk\": %d, \"ctas\": %d, \"warps\": %d, \"stages\": %d, \"inflight_ops\": %d, "
               "\"GBps_per_sm\": %.1f, \"Mops_per_sm\": %.2f, \"err\": \"%s\"}\n",
               bytes >> 20, c.chunk, ctas, c.nw, c.nst, c.nw * c.nst, moved / (ms * 1e-3) / 1e9 / ctas,
               ops / (ms * 1e-3) / 1e6 / ctas, cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
      }
    }
  }
  return 0;
}
