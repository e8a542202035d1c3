// Bisect the per-iteration cost of a single-warp issue loop (B200): which piece of the conv
// mainloop's control flow costs hundreds of cycles per k-block?  One CTA of 256 threads; warp 1
// runs 64 iterations of a loop body built from the selected pieces; others wait at bar.sync.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scratch/loop_bisect tools/loop_bisect.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\tselp.u32 %0, 1, 0, q;\n\t}" : "=r"(p));
  return p != 0;
}

__global__ void k(int pieces, int nst, unsigned long long *out) {
  __shared__ __align__(8) unsigned long long bar[16];
  __shared__ long long itc[65];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 2 && (pieces & 64)) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  int acc = 0;
  if (warp == 1) {
    for (int i = 0; i < 65; ++i) {
      if (threadIdx.x == 32) itc[i] = clock64();
      int s = i;
      if (pieces & 1) { s = i % nst; acc += i / nst; }
      if (pieces & 8) {   // try_wait on a barrier phase that never completes (parity 1 of a fresh barrier = the
        // preceding phase, which counts as complete)
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar[s & 15])), "r"(1u) : "memory");
        acc += ok;
      }
      if (pieces & 16) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (pieces & 2) {
        if (elect_one()) acc += s;
      }
      if (pieces & 32) {
        if (elect_one()) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[8 + (s & 7)])) : "memory");
      }
      if (pieces & 4) __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = (unsigned long long)(itc[64] - itc[0]);
    out[1] = acc;
  }
  if (warp == 2 && (pieces & 64)) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem_base));
}

int main() {
  unsigned long long *out;
  cudaMallocManaged(&out, 16);
  int list[] = {0, 1, 2, 4, 6, 8, 16, 32, 7, 15, 31, 63, 64, 64 | 16, 127};
  for (int pieces : list) {
    k<<<1, 256>>>(pieces, 6, out);
    cudaDeviceSynchronize();
    k<<<1, 256>>>(pieces, 6, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    printf("pieces %3d (div %d elect %d syncwarp %d trywait %d tcfence %d arrive %d tmem %d): %.1f cyc/iter\n", pieces,
           pieces & 1, !!(pieces & 2), !!(pieces & 4), !!(pieces & 8), !!(pieces & 16), !!(pieces & 32), !!(pieces & 64),
           out[0] / 64.0);
  }
  return 0;
}
