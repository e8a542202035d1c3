#include <cstdio>
__global__ void k(unsigned long long *out) {
  unsigned long long t, s = 0;
  long long c0 = clock64();
  for (int i = 0; i < 100; ++i) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); s += t; }
  long long c1 = clock64();
  unsigned v = 0;
  for (int i = 0; i < 100; ++i) { unsigned x; asm volatile("mov.u32 %0, %%clock;" : "=r"(x)); v += x; }
  long long c2 = clock64();
  if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = c2 - c1; out[2] = s + v; }
}
int main() {
  unsigned long long *o; cudaMallocManaged(&o, 64);
  for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o); cudaDeviceSynchronize(); printf("globaltimer: %.1f cyc/read, clock: %.1f cyc/read\n", o[0] / 100.0, o[1] / 100.0); }
}
