// Which kernel feature limits executor CTAs per SM?  Occupancy of small kernels with one feature
// each (B200).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scratch/occ_probe tools/occ_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void k_plain(int *o) { if (o) o[threadIdx.x] = threadIdx.x; }
__global__ void k_tmem(int *o) {
  __shared__ uint32_t base;
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (o) o[threadIdx.x] = base;
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(base));
}
__global__ void k_mma(int *o, uint64_t a, uint64_t b, uint32_t t) {
  if (threadIdx.x == 0 && o)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(t), "l"(a), "l"(b), "r"(0u), "r"(0u));
}
__global__ void k_smid(int *o) {
  uint32_t v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  if (o) o[threadIdx.x] = v;
}
// co-residency in practice: each CTA allocates 128 TMEM columns, records SM id and its time window
__global__ void k_window(unsigned long long *o, long long spin_ns) {
  __shared__ uint32_t base;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while ((long long)(t1 - t0) < spin_ns);
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base));
  if (threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    o[blockIdx.x * 3] = sm; o[blockIdx.x * 3 + 1] = t0; o[blockIdx.x * 3 + 2] = t1;
  }
}
template <typename K> void rep(const char *n, K k, int thr, int dyn) {
  int occ = -1;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, thr, dyn);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  printf("%-8s thr %d dyn %d: occ %d (%s) regs %d smem %zu\n", n, thr, dyn, occ, cudaGetErrorString(e), fa.numRegs, fa.sharedSizeBytes);
}
int main() {
  rep("plain", k_plain, 128, 0);
  rep("tmem", k_tmem, 128, 0);
  rep("mma", k_mma, 128, 0);
  rep("smid", k_smid, 128, 0);
  rep("plain", k_plain, 128, 100 * 1024);
  unsigned long long *o;
  cudaMallocManaged(&o, 296 * 3 * 8);
  k_window<<<296, 128>>>(o, 200000);
  cudaError_t e = cudaDeviceSynchronize();
  printf("window launch: %s\n", cudaGetErrorString(e));
  unsigned long long tmin = ~0ull, tmax = 0;
  int overl = 0;
  for (int i = 0; i < 296; ++i) { if (o[i*3+1] < tmin) tmin = o[i*3+1]; if (o[i*3+2] > tmax) tmax = o[i*3+2]; }
  for (int i = 0; i < 296; ++i)
    for (int j = i + 1; j < 296; ++j)
      if (o[i*3] == o[j*3] && o[i*3+1] < o[j*3+2] && o[j*3+1] < o[i*3+2]) ++overl;
  printf("296 CTAs x 200 us: span %.1f us, overlapping same-SM pairs %d\n", (tmax - tmin) / 1e3, overl);
  return 0;
}
