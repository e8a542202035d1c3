// Device latency microbenchmarks on B200 (cycles via clock64, ns via %globaltimer).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_lat(int *buf, int *flag, unsigned long long *out) {
  // single thread: dependent-chain L2 load latency, atomic RTT, red.release cost, gtimer steps
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  volatile int *vb = buf;
  int idx = 0;
  for (int i = 0; i < 64; ++i) idx = buf[idx];  // warm
  long long c0 = clock64();
  for (int i = 0; i < 256; ++i) {
    int v;
    asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(v) : "l"(buf + idx));
    idx = v;
  }
  long long c1 = clock64();
  out[0] = (c1 - c0) / 256;  // L2 hit latency (cycles)
  c0 = clock64();
  int acc = 0;
  for (int i = 0; i < 64; ++i) acc += atomicAdd(flag, 1);
  c1 = clock64();
  out[1] = (c1 - c0) / 64;  // atomicAdd with return (cycles)
  c0 = clock64();
  for (int i = 0; i < 64; ++i) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(flag + 32) : "memory");
  c1 = clock64();
  out[2] = (c1 - c0) / 64;  // red.release (cycles, back to back)
  c0 = clock64();
  for (int i = 0; i < 64; ++i) {
    buf[1024 + i] = i;
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(flag + 32) : "memory");
  }
  c1 = clock64();
  out[3] = (c1 - c0) / 64;  // store + red.release
  c0 = clock64();
  for (int i = 0; i < 64; ++i) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag + 64) : "memory");
    acc += v;
  }
  c1 = clock64();
  out[4] = (c1 - c0) / 64;  // ld.acquire (cycles)
  c0 = clock64();
  for (int i = 0; i < 64; ++i) __threadfence();
  c1 = clock64();
  out[5] = (c1 - c0) / 64;  // __threadfence
  // globaltimer resolution: distinct consecutive values
  unsigned long long t0 = gt(), t1 = t0, minstep = ~0ull;
  for (int i = 0; i < 100000; ++i) {
    unsigned long long t = gt();
    if (t != t1) {
      if (t - t1 < minstep) minstep = t - t1;
      t1 = t;
    }
  }
  out[6] = minstep;
  long long cc0 = clock64();
  unsigned long long g0 = gt();
  while (gt() - g0 < 100000) {
  }
  long long cc1 = clock64();
  out[7] = (cc1 - cc0);  // cycles per 100 us -> clock MHz = out[7] / 100
  out[8] = acc + vb[0];
}

__global__ void k_bar(unsigned long long *out) {
  __shared__ int s;
  long long c0 = clock64();
  for (int i = 0; i < 256; ++i) {
    if (threadIdx.x == 0) s = i;
    __syncthreads();
  }
  long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[9] = (c1 - c0) / 256;
}

__global__ void k_gridbar(unsigned *cnt, unsigned *gen, unsigned long long *out, int iters) {
  __shared__ int ok;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g;
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
      unsigned arrived = atomicAdd(cnt, 1u);
      if (arrived == gridDim.x - 1) {
        atomicExch(cnt, 0u);
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
      } else {
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
        } while (v == g);
      }
      ok = 1;
    }
    __syncthreads();
  }
  long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[10] = (c1 - c0) / iters;
}

// ---- single-CTA L2 read pattern: each thread issues NL independent 16-byte ld.global.cg loads ----
template <int NL>
__global__ void k_l2read(const uint4 *src, unsigned long long *out, int stride_elems) {
  const int t = threadIdx.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  __syncthreads();
  long long c0 = clock64();
  uint4 v[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i)
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w)
                 : "l"(src + (size_t)i * stride_elems + t));
#pragma unroll
  for (int i = 0; i < NL; ++i) { acc.x ^= v[i].x; acc.y ^= v[i].y; }
  __syncthreads();
  long long c1 = clock64();
  if (t == 0) out[blockIdx.x] = c1 - c0;
  if (acc.x == 0x12345 && acc.y == 7) out[100] = 1;
}

int main() {
  int *buf, *flag;
  unsigned *cnt;
  unsigned long long *out;
  cudaMalloc(&buf, 1 << 20);
  cudaMalloc(&flag, 4096);
  cudaMalloc(&cnt, 64);
  cudaMallocManaged(&out, 256);
  cudaMemset(flag, 0, 4096);
  cudaMemset(cnt, 0, 64);
  int h[2048];
  for (int i = 0; i < 2048; ++i) h[i] = (i * 97 + 13) % 1024;
  cudaMemcpy(buf, h, sizeof h, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    k_lat<<<1, 32>>>(buf, flag, out);
    k_bar<<<1, 256>>>(out);
    void *args[] = {&cnt, &cnt, &out, nullptr};
    unsigned *gen = cnt + 8;
    int iters = 200;
    void *a2[] = {&cnt, &gen, &out, &iters};
    cudaLaunchCooperativeKernel((void *)k_gridbar, 148, 256, a2, 0, 0);
    cudaDeviceSynchronize();
  }
  {
    uint4 *big;
    cudaMalloc(&big, 64 << 20);
    cudaMemset(big, 1, 64 << 20);
    for (int rep = 0; rep < 2; ++rep) {
      k_l2read<1><<<1, 256>>>(big, out, 256);
      cudaDeviceSynchronize();
      unsigned long long c1 = out[0];
      k_l2read<18><<<1, 256>>>(big, out, 256);
      cudaDeviceSynchronize();
      unsigned long long c18 = out[0];
      k_l2read<18><<<148, 256>>>(big, out, 256);
      cudaDeviceSynchronize();
      unsigned long long c18all = out[0];
      printf("1 CTA x 256 thr: 1 load/thr %llu cyc (4 KB); 18 loads/thr %llu cyc (72 KB -> %.1f B/cyc); 148 CTAs same data: %llu cyc\n",
             c1, c18, 73728.0 / c18, c18all);
    }
  }
  printf("L2 hit (ld.cg) %llu cyc | atomicAdd RTT %llu | red.release %llu | st+red.release %llu | ld.acquire %llu | threadfence %llu\n",
         out[0], out[1], out[2], out[3], out[4], out[5]);
  printf("globaltimer min step %llu ns | SM clock ~%llu MHz | __syncthreads(256) %llu cyc | grid barrier(148) %llu cyc\n",
         out[6], out[7] / 100, out[9], out[10]);
  return 0;
}

