// TMA load microbenchmark: one CTA, thread 0 issues NB 2-D box loads {64 bf16, ROWS} from an
// L2-resident matrix (row pitch PITCH bytes), each completing on its own mbarrier; time from the
// first issue until all have landed (clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool GMEM>
__global__ void k_tma4t(const __grid_constant__ CUtensorMap pmap, const CUtensorMap *gmap, int nb, int boxbytes,
                        unsigned long long *out) {
  const void *mp = GMEM ? (const void *)gmap : (const void *)&pmap;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) unsigned long long bars[16];
  uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long c0 = clock64();
    for (int i = 0; i < nb; ++i) {
      uint32_t bar = smem_u32(&bars[i]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(boxbytes));
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
              smem_u32(base + i * ((boxbytes + 1023) / 1024) * 1024)),
          "l"(mp), "r"(64 * i), "r"(0), "r"(0), "r"(0), "r"(bar)
          : "memory");
    }
    long long c1 = clock64();
    for (int i = 0; i < nb; ++i) {
      uint32_t bar = smem_u32(&bars[i]), ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok)
                     : "r"(bar), "r"(0));
    }
    long long c2 = clock64();
    out[0] = c1 - c0;
    out[1] = c2 - c0;
  }
}

__global__ void k_tma4(const __grid_constant__ CUtensorMap map, int nb, int boxbytes, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) unsigned long long bars[16];
  uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int rep = 0; rep < 2; ++rep) {
      long long c0 = clock64();
      for (int i = 0; i < nb; ++i) {
        uint32_t bar = smem_u32(&bars[i]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(boxbytes));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                smem_u32(base + i * ((boxbytes + 1023) / 1024) * 1024)),
            "l"(&map), "r"(64 * i), "r"(0), "r"(0), "r"(0), "r"(bar)
            : "memory");
      }
      long long c1 = clock64();
      for (int i = 0; i < nb; ++i) {
        uint32_t bar = smem_u32(&bars[i]), ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                       : "=r"(ok)
                       : "r"(bar), "r"(rep & 1));
      }
      long long c2 = clock64();
      out[2 * rep] = c1 - c0;
      out[2 * rep + 1] = c2 - c0;
    }
  }
}

__global__ void k_tma(const __grid_constant__ CUtensorMap map, int nb, int rows, int rows_step, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) unsigned long long bars[16];
  uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int rep = 0; rep < 3; ++rep) {
      long long c0 = clock64();
      for (int i = 0; i < nb; ++i) {
        uint32_t bar = smem_u32(&bars[i]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rows * 128));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(base + i * rows * 128)),
            "l"(&map), "r"(64 * (i + rep * 16)), "r"(0), "r"(bar)
            : "memory");
      }
      for (int i = 0; i < nb; ++i) {
        uint32_t bar = smem_u32(&bars[i]), ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                       : "=r"(ok)
                       : "r"(bar), "r"(rep & 1));
      }
      long long c1 = clock64();
      out[rep] = c1 - c0;
    }
  }
}

int main() {
  const int K = 8192;  // elements per row -> covers 64 * 48 boxes along K
  for (int pitch_mul : {1, 15}) {   // row pitch = K*2 bytes; pitch_mul unused placeholder
    (void)pitch_mul;
  }
  int rows_list[] = {32, 49, 126, 128};
  int nb_list[] = {1, 4, 12};
  for (int rows : rows_list) {
    const int R = 256;
    void *buf;
    cudaMalloc(&buf, (size_t)R * K * 2);
    cudaMemset(buf, 0, (size_t)R * K * 2);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    unsigned long long *out;
    cudaMallocManaged(&out, 64);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int nb : nb_list) {
      if (nb * rows * 128 > 190 * 1024) continue;
      k_tma<<<1, 32, 200 * 1024>>>(map, nb, rows, 0, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      printf("rows %3d boxes %2d: %6llu %6llu %6llu cycles (warm rep %.1f cyc/box, %.1f B/cyc)\n", rows, nb,
             out[0], out[1], out[2], (double)out[2] / nb, (double)nb * rows * 128 / out[2]);
    }
    cudaFree(buf);
  }
  // 4-D activation box like the conv A operand: {64 ch, 7 w, 7 h, 1 n} of a [1][7][7][C] tensor
  for (int C : {960, 1024, 256}) {
    void *buf;
    cudaMalloc(&buf, (size_t)49 * C * 2);
    cudaMemset(buf, 0, (size_t)49 * C * 2);
    CUtensorMap map;
    cuuint64_t dims[4] = {(cuuint64_t)C, 7, 7, 1};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)7 * C * 2, (cuuint64_t)49 * C * 2};
    cuuint32_t box[4] = {64, 7, 7, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode4 failed %d\n", (int)r); return 1; }
    unsigned long long *out;
    cudaMallocManaged(&out, 64);
    cudaFuncSetAttribute(k_tma4, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int nb = C / 64 < 12 ? C / 64 : 12;
    k_tma4<<<1, 32, 200 * 1024>>>(map, nb, 49 * 128, out);
    cudaDeviceSynchronize();
    printf("4-D box {64,7,7,1} of C=%d: %d boxes: issue %llu cyc, all landed %llu cyc (rep2: %llu / %llu)\n", C, nb,
           out[0], out[1], out[2], out[3]);
    CUtensorMap *gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &map, sizeof map, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_tma4t<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_tma4t<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
      k_tma4t<true><<<1, 32, 200 * 1024>>>(map, gm, nb, 49 * 128, out);
      cudaDeviceSynchronize();
      unsigned long long gi = out[0], gl = out[1];
      k_tma4t<false><<<1, 32, 200 * 1024>>>(map, gm, nb, 49 * 128, out);
      cudaDeviceSynchronize();
      printf("   map in global memory: issue %llu landed %llu | param: issue %llu landed %llu\n", gi, gl, out[0], out[1]);
    }
    // same bytes as a 2-D box {64, 49} of [49][C]
    cuuint64_t d2[2] = {(cuuint64_t)C, 49};
    cuuint64_t s2[1] = {(cuuint64_t)C * 2};
    cuuint32_t b2[2] = {64, 49};
    cuuint32_t e2[2] = {1, 1};
    CUtensorMap m2;
    cuTensorMapEncodeTiled(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k_tma<<<1, 32, 200 * 1024>>>(m2, nb, 49, 0, out);
    cudaDeviceSynchronize();
    printf("   2-D box {64,49}: %llu cycles all landed (rep0)\n", out[0]);
    cudaFree(buf);
  }
  return 0;
}
