// Minimal reproducer for the one racecheck hazard class compute-sanitizer reports on the
// CTA-pair kernels: a cluster of 2 CTAs where warp 1 of EACH CTA runs the
// collective tcgen05.alloc.cta_group::2 (it writes the allocated TMEM address into a
// shared-memory slot of its own CTA), then every thread reads the slot after a cluster
// barrier — the same sequence as pair_setup()/pair_teardown() in pair_gemm.cuh, with no
// other shared-memory traffic.  Each slot has exactly one writer (the alloc of its CTA) and
// all reads follow barrier.cluster, so there is no race; racecheck still reports the write
// by the alloc against the later reads (it does not model tcgen05.alloc's shared-memory
// write as ordered by the barrier).  Variant 1 adds a fence.proxy.async.shared::cta and a
// __syncthreads() between the alloc and the barrier — racecheck's verdict is reported for both.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_slot_race scripts/tmem_slot_race.cu
//   compute-sanitizer --tool racecheck /tmp/tmem_slot_race
#include <cstdio>
#include <cstdint>

__global__ void __cluster_dims__(2, 1, 1) pair_alloc_kernel(int variant, uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (variant == 1) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot;   // every thread reads the slot its CTA's alloc wrote
  if (threadIdx.x == 0) out[blockIdx.x] = t;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(t));
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 2 * sizeof(uint32_t));
  for (int v = 0; v < 2; ++v) {
    pair_alloc_kernel<<<2, 128>>>(v, out);
    cudaError_t e = cudaDeviceSynchronize();
    uint32_t h[2];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("variant %d: %s, tmem addr cta0=0x%x cta1=0x%x\n", v, cudaGetErrorString(e), h[0], h[1]);
  }
  return 0;
}
