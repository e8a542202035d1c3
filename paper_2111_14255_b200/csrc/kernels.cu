// Device code of libmt.so for sm_100a (B200).
//
//  * executor_kernel  -- the persistent stage executor: one cooperative launch,
//    one CTA per SM; per stage every CTA pulls work tiles from its home tenant's operator queue
//    (runtime-aware SM partition, a3) and, when that queue is empty or blocked, from the other
//    tenants (round-robin, the device analogue of the paper's BFS issue); an op's tiles
//    start only when its producers are complete ("operators in one stream can only be launched
//    sequentially", P:289 -- relaxed to true data dependencies); a grid barrier ends each stage
//    ("all operators in the same stage must all finish so as to step into the next stage").
//  * tile functions   -- conv as implicit GEMM on tcgen05 (UMMA 128xBNx16, bf16 in, fp32 in TMEM)
//    with a fused scale/shift/residual/activation epilogue (a5); depthwise conv (a6); pools,
//    elementwise, input pack (a7); FC GEMV (a8).  The SAME tile functions run in the executor
//    and in the one-launch-per-op baselines, so outputs are bit-identical across all schedules.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "kernels.h"
#include "mt_types.h"

namespace MT_NS {

typedef __nv_bfloat16 bf16;

// ------------------------------------------------------------------------------------------
// shared-memory map of a CTA (1024-aligned base)
// ------------------------------------------------------------------------------------------
static constexpr int PIPE_BYTES = MT_PIPE_BYTES;   // conv pipeline ring (stage geometry per op)
static constexpr int TMEM_COLS = 256;   // accumulator of one 128 x 256 tile

struct CtaShared {
  unsigned long long bar_full[MT_MAXST];     // TMA: stage loaded (expect_tx)
  unsigned long long bar_empty[MT_MAXST];    // stage consumed by the MMAs (tcgen05.commit)
  unsigned long long bar_accf;
  uint32_t tmem_base;
  int op, tile, last, ok, home, ten;
  int vcta;                   // index into the home table: blockIdx.x, or (2 CTAs/SM) slot * #SMs + SM
  int smem_cap;               // bytes of dynamic shared memory this kernel has (staging budget)
  int tracing;                // mt_set_trace on: extra producer stamps
  unsigned long long t_pick, t_pick_next, t_deps, t_mma, t_run, t_first, t_lastmma, t_aissue;
  unsigned long long t_kb[4], t_is[1];
  int *xrel;   // extra counter released with the tile (split-K partial arrival)
  int cur[MT_MAXT], end[MT_MAXT], beg[MT_MAXT];
  uint32_t complete[64];      // bitset of ops observed fully complete (global op id < 2048)
  int16_t gate[MT_GATE_OPS];  // claim-ahead gate op of each op (-1 none; claim_depth != 0)
  float esc[256], esh[256];   // epilogue scale / shift of the current conv tile's columns
  OpDesc d;
};
static constexpr int SMEM_BYTES = 1024 + PIPE_BYTES;   // + static __shared__ CtaShared

// Every conv tile drains its pipeline (waits for the accumulator), so each tile starts with all
// stages free; only the mbarrier phase parities persist between tiles.
struct PipeState {
  uint32_t eph;        // bit s: parity of the next completion of empty[s]
  uint32_t fph;        // bit s: parity of the next completion of full[s]
  uint32_t acc_phase;  // parity of the accumulator-ready barrier
};

// ------------------------------------------------------------------------------------------
// PTX helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int *p) {   // heuristic reads: no ordering needed
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_u(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(int *p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// release pattern (PTX memory model): one gpu-scope fence followed by relaxed reds -- every red
// publishes the writes ordered before the fence, at the cost of a single MEMBAR.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_add(int *p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, uint64_t tmap, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, uint64_t tmap, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// generic-proxy global writes (epilogue stores, input pack) of other CTAs, acquired through the
// dependency counters, are read here by TMA (async proxy): order the acquire before the bulk
// tensor loads (consumer side) and the stores before the release (producer side)
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// waiting warps that are not on the tile's critical issue path back off between probes so they
// do not take issue slots from the TMA-producer / MMA lanes
__device__ __forceinline__ void mbar_wait_backoff(uint32_t bar, uint32_t parity) {
  // try_wait with a suspend-time hint: the warp is parked by the hardware until the phase
  // completes (or the hint elapses) -- no issue slots taken, no oversleeping
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(1000000u)
        : "memory");
  }
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, fp32 accumulate), one CTA
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
// 32 lanes x 32 bit x 8 columns: thread i of the warp gets TMEM lane (base lane + i), 8 columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float *v) {
  uint32_t r0, r1, r2, r3, r4, r5, r6, r7;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
      : "r"(taddr)
      : "memory");
  v[0] = __uint_as_float(r0); v[1] = __uint_as_float(r1); v[2] = __uint_as_float(r2);
  v[3] = __uint_as_float(r3); v[4] = __uint_as_float(r4); v[5] = __uint_as_float(r5);
  v[6] = __uint_as_float(r6); v[7] = __uint_as_float(r7);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 lanes x 32 bit x 32 columns in one load (one wait for 32 accumulator columns)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, 8-row atoms of 1024 B
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);      // start address
  d |= (uint64_t)(16 >> 4) << 16;              // leading byte offset (ignored for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;            // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;                      // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}
// UMMA descriptor, K-major, no swizzle ("interleave"): 8-row x 16-byte core matrices, lbo = byte
// distance between the two 16-byte K chunks of one MMA, sbo = distance between 8-row groups
__device__ __forceinline__ uint64_t sdesc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;   // layout type 0 = SWIZZLE_NONE
}
// instruction descriptor kind::f16: D f32, A/B bf16, both K-major, M = 128, N = n
__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(MT_BM >> 4) << 24);
}

// ------------------------------------------------------------------------------------------
// element helpers: 8 channels at a time (16 B of bf16, 32 B of fp32)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void ld8_cg(const bf16 *p, float *v) {  // activations: L2 only
  uint4 u;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void ld8_cg(const float *p, float *v) {
  float4 a, b;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p));
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(p + 4));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
// raw (unconverted) 8-channel vectors: 4 registers for bf16, 8 for fp32
template <typename T> struct Raw8;
template <> struct Raw8<bf16> { uint4 u; };
template <> struct Raw8<float> { float4 a, b; };
__device__ __forceinline__ uint32_t raw_word(const Raw8<bf16> &r) { return r.u.x; }
__device__ __forceinline__ uint32_t raw_word(const Raw8<float> &r) { return __float_as_uint(r.a.x); }
__shared__ unsigned long long sh_t_first_dw, sh_t_load_dw;   // trace stamps (dw tiles)
__device__ __forceinline__ void ldraw_cg(const bf16 *p, Raw8<bf16> &r) {
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.u.x), "=r"(r.u.y), "=r"(r.u.z), "=r"(r.u.w) : "l"(p));
}
__device__ __forceinline__ void ldraw_cg(const float *p, Raw8<float> &r) {
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w) : "l"(p));
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.b.x), "=f"(r.b.y), "=f"(r.b.z), "=f"(r.b.w) : "l"(p + 4));
}
__device__ __forceinline__ Raw8<bf16> ldraw_nc(const bf16 *p) {
  Raw8<bf16> r;
  r.u = __ldg(reinterpret_cast<const uint4 *>(p));
  return r;
}
__device__ __forceinline__ Raw8<float> ldraw_nc(const float *p) {
  Raw8<float> r;
  r.a = __ldg(reinterpret_cast<const float4 *>(p));
  r.b = __ldg(reinterpret_cast<const float4 *>(p + 4));
  return r;
}
__device__ __forceinline__ Raw8<bf16> ldraw_gen(const bf16 *p) {   // generic: smem or global
  Raw8<bf16> r;
  r.u = *reinterpret_cast<const uint4 *>(p);
  return r;
}
__device__ __forceinline__ Raw8<float> ldraw_gen(const float *p) {
  Raw8<float> r;
  r.a = reinterpret_cast<const float4 *>(p)[0];
  r.b = reinterpret_cast<const float4 *>(p)[1];
  return r;
}
__device__ __forceinline__ void zero_raw(Raw8<bf16> &r) { r.u = make_uint4(0, 0, 0, 0); }
__device__ __forceinline__ void zero_raw(Raw8<float> &r) { r.a = r.b = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void cvt8(const Raw8<bf16> &r, float *v) {
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&r.u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void cvt8(const Raw8<float> &r, float *v) {
  v[0] = r.a.x; v[1] = r.a.y; v[2] = r.a.z; v[3] = r.a.w; v[4] = r.b.x; v[5] = r.b.y; v[6] = r.b.z; v[7] = r.b.w;
}
__device__ __forceinline__ void ld8_nc(const bf16 *p, float *v) {  // immutable weights
  uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void ld8_nc(const float *p, float *v) {
  float4 a = __ldg(reinterpret_cast<const float4 *>(p)), b = __ldg(reinterpret_cast<const float4 *>(p + 4));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8(bf16 *p, const float *v) {
  uint4 u;
  __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4 *>(p) = u;
}
__device__ __forceinline__ void st8(float *p, const float *v) {
  reinterpret_cast<float4 *>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4 *>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ float ld1_cg(const bf16 *p) {
  unsigned short u;
  asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(u) : "l"(p));
  return __bfloat162float(__ushort_as_bfloat16(u));
}
__device__ __forceinline__ float ld1_cg(const float *p) { return __ldcg(p); }
__device__ __forceinline__ void st1(bf16 *p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ void st1(float *p, float v) { *p = v; }

// branch-free clamp: none = [-inf, inf], ReLU = [0, inf], ReLU6 = [0, 6] (bounds are loop
// invariant at every call site, so an unrolled epilogue is two FMNMX per value)
__device__ __forceinline__ float act_f(float y, int act) {
  const float lo = act ? 0.f : -INFINITY, hi = act == 2 ? 6.f : INFINITY;
  return fminf(fmaxf(y, lo), hi);
}

template <typename T>
__device__ __forceinline__ const T *in_ptr(const RunArgs &a, const OpDesc &d) {
  return (d.flags & OPF_GRAPH_IN) ? reinterpret_cast<const T *>(a.packed[d.tenant])
                                  : reinterpret_cast<const T *>(d.in);
}

// store 8 output channels [c0, c0+8) of output pixel `pix` (row of N*Ho*Wo); nvalid <= 8
template <typename T>
__device__ __forceinline__ void store_out8(const RunArgs &a, const OpDesc &d, int64_t pix, int c0,
                                           const float *v, int nvalid) {
  if (d.flags & OPF_OUT) {
    float *o = a.outputs[d.tenant] + pix * d.Co + c0;
    for (int e = 0; e < nvalid; ++e) o[e] = v[e];
  } else {
    T *o = reinterpret_cast<T *>(d.out) + pix * d.out_cs + d.out_co + c0;
    if (nvalid == 8) st8(o, v);
    else
      for (int e = 0; e < nvalid; ++e) st1(o + e, v[e]);
  }
}

// ------------------------------------------------------------------------------------------
// a5: conv implicit GEMM on tcgen05.  GEMM view M = N*Ho*Wo (pixels), N = Cout, K = kh*kw*C
// (K order (r, s, c), c fastest, matching NHWC).  A = im2col rows gathered with cp.async
// (zero-fill for padding / tails), B = packed weights [Cout_pad][Kpad].  Both staged in a
// MT_STAGES-deep ring of 128B-swizzled K-major tiles; one thread issues UMMA 128 x BN x 16 and
// commits to per-stage mbarriers; the accumulator lives in TMEM and is drained by all 8 warps.
// Deterministic split-K: fp32 partials in workspace, the last-arriving CTA sums them in split
// order 0..S-1 and runs the epilogue.
// ------------------------------------------------------------------------------------------
struct ConvTile {
  int tmn, ks, mt, m0, n0, kb0, nk;
  int img, ho0, wo0;   // TMA path: image, first output row and first column of the M tile
};
__device__ __forceinline__ ConvTile conv_tile_coords(const OpDesc &d, int tile) {
  ConvTile c;
  const int S = d.splits;
  c.tmn = tile / S;
  c.ks = tile - c.tmn * S;
  c.mt = c.tmn / d.tiles_n;
  const int nt = c.tmn - c.mt * d.tiles_n;
  c.m0 = c.mt * MT_BM;
  c.n0 = nt * d.bn;
  c.kb0 = c.ks * d.kb_per_split;
  c.nk = min(d.nkb, c.kb0 + d.kb_per_split) - c.kb0;
  if (d.tma == 1 || d.tma == 2) {
    const int rg = c.mt / d.nseg, seg = c.mt - rg * d.nseg;
    c.img = rg / d.blk_tpi;
    c.ho0 = (rg - c.img * d.blk_tpi) * d.blk_rows;
    c.wo0 = seg * d.seg_w;
  } else {
    c.img = 0;
    c.ho0 = 0;
    c.wo0 = 0;
  }
  return c;
}
// output pixel of accumulator row r (TMEM lane), or -1 if the row is padding
__device__ __forceinline__ int conv_row_pixel(const OpDesc &d, const ConvTile &c, int r) {
  if (d.tma == 3) return c.m0 + r < d.Co ? c.m0 + r : -1;   // tensor-core FC: row = output feature
  if (d.tma) {
    const int hl = r / d.seg_w;
    const int ho = c.ho0 + hl, wo = c.wo0 + (r - hl * d.seg_w);
    if (hl >= d.blk_rows || ho >= d.Ho || wo >= d.Wo) return -1;
    return (c.img * d.Ho + ho) * d.Wo + wo;
  }
  const int m = c.m0 + r;
  return m < d.M ? m : -1;
}

// parity helpers: k-block i of a tile uses stage i % nst; its j-th use (j = i / nst) of the stage
// within the tile completes the stage's barriers with parity (start parity ^ (j & 1))
__device__ __forceinline__ uint32_t stage_par(uint32_t bits, int s, int j) { return ((bits >> s) & 1u) ^ (uint32_t)(j & 1); }

// Work that needs no producer data, issued BEFORE the tile waits for its dependencies so the weight
// stream overlaps the wait: the weight (B) tiles of the first min(nk, nst) k-blocks and the
// epilogue constants.  TMA path: thread 0 arms each stage's full barrier for A+B bytes and issues
// B; A follows once the producers are complete.  cp.async path: one commit group per k-block.
__device__ void conv_tc_prefetch(const OpDesc &d, int tile, uint8_t *smem, CtaShared &sh,
                                 const PipeState &ps) {
  const int tid = threadIdx.x;
  const ConvTile ct = conv_tile_coords(d, tile);
  const bf16 *Wt = reinterpret_cast<const bf16 *>(d.w);
  const uint32_t s0 = smem_u32(smem);
  if (d.tma) {
    if (tid == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(d.tmap_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(d.tmap_b) : "memory");
      const uint32_t bar_full0 = smem_u32(&sh.bar_full[0]);
      const int kg = d.kg;
      const uint32_t txb = (uint32_t)(d.a_bytes + d.bn * 128);
      // ring stage i holds k-blocks [i*kg, min(nk, (i+1)*kg)) as kg consecutive sub-blocks
      for (int i = 0, kb = 0; i < d.nst && kb < ct.nk; ++i) {
        const int g = min(kg, ct.nk - kb);
        const uint32_t bar = bar_full0 + 8 * i;
        mbar_expect_tx(bar, txb * (uint32_t)g);
        for (int u = 0; u < g; ++u, ++kb) {
          const uint32_t sub = s0 + (uint32_t)(kb * d.st_bytes);
          if (d.tma == 3)   // FC: the weights are the A (M = features) operand
            tma_load_2d(sub, d.tmap_a, bar, (ct.kb0 + kb) * MT_BK, ct.m0);
          else
            tma_load_2d(sub + d.st_boff, d.tmap_b, bar, (ct.kb0 + kb) * MT_BK, ct.n0);
        }
      }
    }
  } else {
    const int c = tid & 7;
    for (int i = 0; i < MT_STAGES; ++i) {
      if (i < ct.nk) {
        const int kb = ct.kb0 + i;
        const uint32_t sb = s0 + i * d.st_bytes + d.st_boff;
        for (int row = tid >> 3; row < d.bn; row += MT_NTHREADS / 8) {
          const bf16 *src = Wt + (int64_t)(ct.n0 + row) * d.Kpad + kb * MT_BK + c * 8;
          cp_async16(sb + row * 128 + ((c ^ (row & 7)) << 4), src, true);
        }
      }
      cp_async_commit();
    }
  }
  if (d.tma == 3) {   // FC: per-row (feature) constants.  No L2 prefetch of the rest of the weight
    if (tid < MT_BM) {  // stream: it is read once and would evict the other tenants' working sets
      const int o = ct.m0 + tid;
      sh.esc[tid] = o < d.Co ? __ldg(reinterpret_cast<const float *>(d.scale) + o) : 0.f;
      sh.esh[tid] = o < d.Co ? __ldg(reinterpret_cast<const float *>(d.shift) + o) : 0.f;
    }
    return;
  }
  for (int c = tid; c < d.bn; c += MT_NTHREADS) {   // bn may exceed the CTA (2 CTAs/SM: 128 threads)
    const int n = ct.n0 + c;
    sh.esc[c] = n < d.Co ? __ldg(reinterpret_cast<const float *>(d.scale) + n) : 0.f;
    sh.esh[c] = n < d.Co ? __ldg(reinterpret_cast<const float *>(d.shift) + n) : 0.f;
  }
  // the rest of this split's weight rows -> L2 (one bulk prefetch per row)
  const int kpre = d.tma ? d.nst * d.kg : MT_STAGES;   // k-blocks whose weights are already requested
  if (ct.nk > kpre)
    for (int row = tid; row < d.bn; row += MT_NTHREADS)
      prefetch_l2_bulk(Wt + (int64_t)(ct.n0 + row) * d.Kpad + (ct.kb0 + kpre) * MT_BK,
                       (uint32_t)(ct.nk - kpre) * MT_BK * 2);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\tselp.u32 %0, 1, 0, q;\n\t}" : "=r"(p));
  return p != 0;
}

// TMA mainloop.  Warp 0 = producer (A boxes, and B beyond the prefetched stages), warp 1 = MMA
// issuer (UMMA 128 x bn x 16 from a sub-block's two tiles; commit frees the ring stage).  A ring
// stage holds KG (1 or 2) consecutive k-blocks (sub-blocks st_bytes apart) behind one full / empty
// barrier pair, so the per-stage chain of single-thread latencies (barrier probe, expect_tx or
// commit, warp reconvergence, ~250 ns; tools/kb_pipe.cu) is paid once per KG k-blocks.  KG is a
// template parameter with the sub-block loop unrolled: a runtime-trip-count inner loop measured 10 %
// slower end to end (the issue state leaves the uniform datapath), and so did one 4-slot body
// predicated by a runtime kg (kg = 1 ops paid for the dead slots).  A tile's tail stage holds
// g <= KG k-blocks.  Both loops run warp-wide with one elected lane issuing; everyone else waits
// for the accumulator.
template <int KG>
__device__ __forceinline__ void conv_tc_mainloop_tma(const OpDesc &d, const ConvTile &ct, uint8_t *smem,
                                                     CtaShared &sh, const PipeState &ps) {
  const int warp = threadIdx.x >> 5;
  const uint32_t s0 = smem_u32(smem);
  const uint32_t bar_full0 = smem_u32(&sh.bar_full[0]);
  const uint32_t bar_empty0 = smem_u32(&sh.bar_empty[0]);
  const uint32_t bar_accf = smem_u32(&sh.bar_accf);
  const int nst = d.nst, nk = ct.nk, st_bytes = d.st_bytes, st_boff = d.st_boff;
  const int nsq = KG == 1 ? nk : (nk + KG - 1) / KG;   // ring stages this tile fills
  if (warp == 0) {
    const uint32_t txb = (uint32_t)(d.a_bytes + d.bn * 128);
    const uint64_t tmap_a = d.tmap_a, tmap_b = d.tmap_b;
    const int kb0 = ct.kb0, cblks = d.cblks, kw = d.kw, pw = d.pw, n0 = ct.n0, img = ct.img;
    const int small = d.tma == 2, ntap = d.kh * d.kw, fc = d.tma == 3, m0 = ct.m0;
    int tap = kb0 / cblks, cb = kb0 - tap * cblks;
    int rr = tap / kw, ss = tap - rr * kw;
    const int hbase = ct.ho0 * d.sh - d.ph, wbase = ct.wo0 * d.sw - pw;
    const uint32_t eph = ps.eph;
    int s = 0, j = 0, kb = kb0;
    uint32_t st = s0;
    fence_proxy_async_global();   // dependencies acquired (generic proxy) -> TMA reads (async proxy)
    for (int q = 0; q < nsq; ++q) {
      if (j > 0) mbar_wait(bar_empty0 + 8 * s, ((eph >> s) & 1u) ^ (uint32_t)((j - 1) & 1));
      const int g = KG == 1 ? 1 : min(KG, kb0 + nk - kb);
      if (elect_one()) {
        const uint32_t bar = bar_full0 + 8 * s;
        if (j > 0) mbar_expect_tx(bar, KG == 1 ? txb : txb * (uint32_t)g);
        int c2 = cb, s2 = ss, r2 = rr;
#pragma unroll
        for (int u = 0; u < KG; ++u) {
          if (KG == 1 || u < g) {
            const uint32_t sub = st + (uint32_t)(u * st_bytes);
            const int kbu = kb + u;
            if (fc) {   // FC: weights (A slot) prefetched for the first nst stages; input -> B slot
              if (j > 0) tma_load_2d(sub, tmap_a, bar, kbu * MT_BK, m0);
              tma_load_2d(sub + st_boff, tmap_b, bar, kbu * MT_BK, n0);
            } else {
              if (j > 0) tma_load_2d(sub + st_boff, tmap_b, bar, kbu * MT_BK, n0);
              if (small) {   // 8 taps x 8 channels: one 16-byte-row box per tap, 2 KB apart
                int t8 = kbu * 8;
                for (int tt = 0; tt < 8; ++tt, ++t8) {
                  const int ra = t8 / kw, sa = t8 - ra * kw;
                  const bool v = t8 < ntap;   // missing taps: an out-of-range box is zero-filled
                  tma_load_4d(sub + tt * 2048, tmap_a, bar, 0, v ? wbase + sa : -(1 << 20), v ? hbase + ra : 0, img);
                }
              } else {
                tma_load_4d(sub, tmap_a, bar, c2 * 64, wbase + s2, hbase + r2, img);
              }
            }
            if (KG > 1 && ++c2 == cblks) {
              c2 = 0;
              if (++s2 == kw) { s2 = 0; ++r2; }
            }
          }
        }
        if (sh.tracing && (q == 0 || q == nsq - 1)) {   // producer issue stamps (trace only)
          if (q == 0) sh.t_is[0] = gtimer();
          if (q == nsq - 1) sh.t_aissue = gtimer();
        }
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < KG; ++u) {
        if (KG == 1 || u < g) {
          if (++cb == cblks) {
            cb = 0;
            if (++ss == kw) { ss = 0; ++rr; }
          }
        }
      }
      kb += g;
      st += (uint32_t)(KG * st_bytes);
      if (++s == nst) { s = 0; ++j; st = s0; }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16(d.bn);
    const uint32_t tmem = sh.tmem_base;
    const uint32_t fph = ps.fph;
    const bool small = d.tma == 2;
    // descriptors of stage 0; a sub-block advances the start-address field by st_bytes/16, a ring
    // stage by KG*st_bytes/16, one MMA K step by 32 B (SW128: +2) or 2 x 2 KB (no swizzle: +256)
    const uint64_t ad0 = small ? sdesc_noswz(s0, 2048, 128) : sdesc_sw128(s0);
    const uint64_t bd0 = sdesc_sw128(s0 + st_boff);
    const uint64_t a_k = small ? 256 : 2, sub16 = (uint64_t)(st_bytes >> 4), stg16 = (uint64_t)KG * sub16;
    uint64_t ad = ad0, bd = bd0;
    int s = 0, j = 0, kb = 0;
    for (int q = 0; q < nsq; ++q) {
      mbar_wait(bar_full0 + 8 * s, ((fph >> s) & 1u) ^ (uint32_t)(j & 1));
      tc_fence_after();
      const int g = KG == 1 ? 1 : min(KG, nk - kb);
      if (elect_one()) {
        if (q == 0) sh.t_first = gtimer();
#pragma unroll
        for (int u = 0; u < KG; ++u) {
          if (KG == 1 || u < g) {
            const uint64_t a = ad + u * sub16, b = bd + u * sub16;
            tc_mma(tmem, a, b, idesc, (kb + u) > 0 ? 1u : 0u);
            tc_mma(tmem, a + a_k, b + 2, idesc, 1u);
            tc_mma(tmem, a + 2 * a_k, b + 4, idesc, 1u);
            tc_mma(tmem, a + 3 * a_k, b + 6, idesc, 1u);
          }
        }
        // the empty barrier only tracks reuse within the tile: a stage's last use is covered by
        // the accumulator commit, so no mbarrier phase completes without a waiter (synccheck)
        if (q + nst < nsq) tc_commit(bar_empty0 + 8 * s);
      }
      __syncwarp();
      kb += g;
      ad += stg16;
      bd += stg16;
      if (++s == nst) { s = 0; ++j; ad = ad0; bd = bd0; }
    }
    if (elect_one()) {
      tc_commit(bar_accf);
      sh.t_lastmma = gtimer();
    }
    __syncwarp();
  }
}

// cp.async mainloop (small-channel convs, e.g. the 3->8-padded stems): all threads gather im2col
// rows, commit groups: MT_STAGES B-prefetch groups (conv_tc_prefetch) precede the loop's groups;
// group NS + j holds A (and, for j >= NS, B) of k-block j, so wait_group<NS-1> at iteration
// i = j + NS - 1 completes both the prefetched B of k-block j and its A.
__device__ __forceinline__ void conv_tc_mainloop_cpasync(const RunArgs &a, const OpDesc &d, const ConvTile &ct,
                                                         uint8_t *smem, CtaShared &sh, const PipeState &ps) {
  const int tid = threadIdx.x;
  const int m0 = ct.m0, n0 = ct.n0, kb0 = ct.kb0, nk = ct.nk;
  const bf16 *X = in_ptr<bf16>(a, d);
  const bf16 *Wt = reinterpret_cast<const bf16 *>(d.w);
  const int HoWo = d.Ho * d.Wo;
  const int c = tid & 7;
  constexpr int RP = MT_NTHREADS / 8, NP = MT_BM / RP;   // rows per pass, passes per tile
  int pbase[NP], hb[NP], wb[NP];
  bool rv[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int m = m0 + (tid >> 3) + RP * i;
    rv[i] = m < d.M;
    const int mm = rv[i] ? m : 0;
    const int n = mm / HoWo, rem = mm - n * HoWo;
    const int ho = rem / d.Wo, wo = rem - ho * d.Wo;
    pbase[i] = n * d.H * d.W;
    hb[i] = ho * d.sh - d.ph;
    wb[i] = wo * d.sw - d.pw;
  }
  const uint32_t s0 = smem_u32(smem);
  const uint32_t idesc = idesc_bf16(d.bn);
  const uint32_t tmem = sh.tmem_base;
  const uint32_t bar_empty0 = smem_u32(&sh.bar_empty[0]);
  const uint32_t bar_accf = smem_u32(&sh.bar_accf);
  for (int i = 0; i < nk + MT_STAGES - 1; ++i) {
    if (i < nk) {
      const int s = i % MT_STAGES, jj = i / MT_STAGES;
      if (jj > 0) mbar_wait(bar_empty0 + 8 * s, stage_par(ps.eph, s, jj - 1));
      const int kb = kb0 + i;
      const int k = kb * MT_BK + c * 8;
      const bool kv = k < d.K;
      const int tap = kv ? k / d.C : 0;
      const int ci = k - tap * d.C;
      const int rr = tap / d.kw, ss = tap - rr * d.kw;
      const uint32_t sa = s0 + s * d.st_bytes;
#pragma unroll
      for (int i2 = 0; i2 < NP; ++i2) {
        const int row = (tid >> 3) + RP * i2;
        const int hi = hb[i2] + rr, wi = wb[i2] + ss;
        const bool valid = kv && rv[i2] && hi >= 0 && hi < d.H && wi >= 0 && wi < d.W;
        const bf16 *src = valid ? X + (int64_t)(pbase[i2] + hi * d.W + wi) * d.in_cs + d.in_co + ci : X;
        cp_async16(sa + row * 128 + ((c ^ (row & 7)) << 4), src, valid);
      }
      if (jj > 0) {
        const uint32_t sb = sa + d.st_boff;
        for (int row = tid >> 3; row < d.bn; row += RP) {
          const bf16 *src = Wt + (int64_t)(n0 + row) * d.Kpad + kb * MT_BK + c * 8;
          cp_async16(sb + row * 128 + ((c ^ (row & 7)) << 4), src, true);
        }
      }
    }
    cp_async_commit();
    const int j = i - (MT_STAGES - 1);
    if (j >= 0) {
      cp_async_wait<MT_STAGES - 1>();
      fence_proxy_async();  // make the cp.async smem writes visible to the tensor core (async proxy)
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const int s = j % MT_STAGES;
        const uint32_t ab = s0 + s * d.st_bytes, bb = ab + d.st_boff;
#pragma unroll
        for (int kk = 0; kk < MT_BK / 16; ++kk)
          tc_mma(tmem, sdesc_sw128(ab + kk * 32), sdesc_sw128(bb + kk * 32), idesc,
                 (j > 0 || kk > 0) ? 1u : 0u);
        if (j + MT_STAGES < nk) tc_commit(bar_empty0 + 8 * s);   // frees the stage for its reuse
        if (j == nk - 1) tc_commit(bar_accf);  // accumulator complete
      }
    }
  }
  cp_async_wait<0>();
}

// residual of output pixel m, channels n..n+7 (zeros past Co or without a residual)
__device__ __forceinline__ void conv_residual8(const OpDesc &d, int m, int n, float *r) {
#pragma unroll
  for (int e = 0; e < 8; ++e) r[e] = 0.f;
  if (d.flags & OPF_RES) {
    const int nvalid = min(8, d.Co - n);
    const bf16 *rp = reinterpret_cast<const bf16 *>(d.res) + (int64_t)m * d.res_cs + d.res_co + n;
    if (nvalid == 8) {
      ld8_cg(rp, r);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = e < nvalid ? ld1_cg(rp + e) : 0.f;   // static indices
    }
  }
}
__device__ __forceinline__ void conv_epilogue_store(const RunArgs &a, const OpDesc &d, const CtaShared &sh,
                                                    int m, int n0, int col, float *v, const float *r) {
  const int n = n0 + col;
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = act_f(fmaf(v[e], sh.esc[col + e], sh.esh[col + e]) + r[e], d.act);
  store_out8<bf16>(a, d, m, n, v, min(8, d.Co - n));
}
__device__ __forceinline__ void conv_epilogue_vals(const RunArgs &a, const OpDesc &d, const CtaShared &sh,
                                                   int m, int n0, int col, float *v) {
  float r[8];
  conv_residual8(d, m, n0 + col, r);
  conv_epilogue_store(a, d, sh, m, n0, col, v, r);
}

// tensor-core FC epilogue: accumulator row r = output feature o, 8 columns = batch images b..b+7
__device__ __forceinline__ void fc_tc_store(const RunArgs &a, const OpDesc &d, const CtaShared &sh, int r, int o,
                                            int b, const float *v) {
  const float sc = sh.esc[r], sf = sh.esh[r];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    if (b + e < d.N) {
      const float y = act_f(fmaf(v[e], sc, sf), d.act);
      if (d.flags & OPF_OUT) a.outputs[d.tenant][(int64_t)(b + e) * d.Co + o] = y;
      else st1(reinterpret_cast<bf16 *>(d.out) + (int64_t)(b + e) * d.out_cs + d.out_co + o, y);
    }
  }
}

// split-K reduce tile (tmn, rc): waits for the S partials of (M,N) tile tmn, sums columns
// [rc*32, rc*32+32) of its valid rows in split order 0..S-1 (float4 over 4 rows), stages the sums
// in shared memory and runs the fused epilogue.  The last of the rc reduce tiles resets the
// arrival counter (S compute + rc reduce arrivals) for the next run.
__device__ void conv_reduce_tile(const RunArgs &a, const OpDesc &d, int rtile, uint8_t *smem, CtaShared &sh,
                                 bool wait_splits) {
  const int tid = threadIdx.x;
  const int S = d.splits;
  const int tmn = rtile / d.rc, rc = rtile - (rtile / d.rc) * d.rc;
  const ConvTile ct = conv_tile_coords(d, tmn * S);
  int *cnt = a.splitcnt + d.cnt_off + tmn;
  if (tid == 0) {
    if (wait_splits) {
      const unsigned long long t0 = gtimer();
      unsigned spins = 0;
      while (ld_acquire(cnt) < S) {
        if ((++spins & 255) == 0 && gtimer() - t0 > a.timeout_ns) { atomicExch(&a.ctl->error, 3u); break; }
        __nanosleep(20);
      }
    }
  }
  // valid accumulator rows form a prefix of the 128 TMEM lanes
  int nv;
  if (d.tma == 3) nv = min(MT_BM, d.Co - ct.m0);
  else if (d.tma) nv = d.nseg > 1 ? min(d.seg_w, d.Wo - ct.wo0) : min(d.blk_rows, d.Ho - ct.ho0) * d.Wo;
  else nv = min(MT_BM, d.M - ct.m0);
  const int c0 = rc * 32;
  const int ncol = min(32, d.bn - c0);
  if (d.tma == 3) {
    if (tid < MT_BM) {
      const int o = ct.m0 + tid;
      sh.esc[tid] = o < d.Co ? __ldg(reinterpret_cast<const float *>(d.scale) + o) : 0.f;
      sh.esh[tid] = o < d.Co ? __ldg(reinterpret_cast<const float *>(d.shift) + o) : 0.f;
    }
  } else if (tid < ncol) {
    const int n = ct.n0 + c0 + tid;
    sh.esc[c0 + tid] = n < d.Co ? __ldg(reinterpret_cast<const float *>(d.scale) + n) : 0.f;
    sh.esh[c0 + tid] = n < d.Co ? __ldg(reinterpret_cast<const float *>(d.shift) + n) : 0.f;
  }
  __syncthreads();
  const int nv4 = (nv + 3) >> 2;
  const float *ws = reinterpret_cast<const float *>(d.ws);
  float *red = reinterpret_cast<float *>(smem);   // [32 cols][128 rows]
  const int64_t sstride = (int64_t)d.bn * MT_BM;
  for (int it = tid; it < ncol * nv4; it += MT_NTHREADS) {
    const int col = it / nv4, r4 = it - col * nv4;
    const float4 *p = reinterpret_cast<const float4 *>(ws + ((int64_t)tmn * S * d.bn + c0 + col) * MT_BM) + r4;
    float4 acc = __ldcg(p);
    int s2 = 1;
    for (; s2 + 3 < S; s2 += 4) {
      const float4 p1 = __ldcg(p + (s2 * sstride) / 4), p2 = __ldcg(p + ((s2 + 1) * sstride) / 4);
      const float4 p3 = __ldcg(p + ((s2 + 2) * sstride) / 4), p4 = __ldcg(p + ((s2 + 3) * sstride) / 4);
      acc.x = (((acc.x + p1.x) + p2.x) + p3.x) + p4.x;
      acc.y = (((acc.y + p1.y) + p2.y) + p3.y) + p4.y;
      acc.z = (((acc.z + p1.z) + p2.z) + p3.z) + p4.z;
      acc.w = (((acc.w + p1.w) + p2.w) + p3.w) + p4.w;
    }
    for (; s2 < S; ++s2) {
      const float4 p1 = __ldcg(p + (s2 * sstride) / 4);
      acc.x += p1.x; acc.y += p1.y; acc.z += p1.z; acc.w += p1.w;
    }
    reinterpret_cast<float4 *>(red + col * MT_BM)[r4] = acc;
  }
  __syncthreads();
  for (int it = tid; it < nv * (ncol / 8); it += MT_NTHREADS) {
    const int r = it % nv, ch = it / nv;
    const int m = conv_row_pixel(d, ct, r);
    const int col = c0 + ch * 8;
    if (m >= 0 && ct.n0 + col < (d.tma == 3 ? d.N : d.Co)) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = red[(ch * 8 + e) * MT_BM + r];
      if (d.tma == 3) fc_tc_store(a, d, sh, r, m, ct.n0 + col, v);
      else conv_epilogue_vals(a, d, sh, m, ct.n0, col, v);
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int old = atomicAdd(cnt, 1);
    if (old == S + d.rc - 1) atomicExch(cnt, 0);   // every arrival of this run is in
  }
}

__device__ void conv_tc_tile(const RunArgs &a, const OpDesc &d, int tile, uint8_t *smem,
                             CtaShared &sh, PipeState &ps) {
  if (d.splits > 1 && tile >= d.tiles_m * d.tiles_n * d.splits) {
    conv_reduce_tile(a, d, tile - d.tiles_m * d.tiles_n * d.splits, smem, sh, true);
    return;
  }
  const int tid = threadIdx.x;
  const int S = d.splits;
  const ConvTile ct = conv_tile_coords(d, tile);
  const int tmn = ct.tmn, ks = ct.ks, n0 = ct.n0;
  const uint32_t bar_accf = smem_u32(&sh.bar_accf);
  if (d.tma) {
    if (d.kg == 2) conv_tc_mainloop_tma<2>(d, ct, smem, sh, ps);
    else conv_tc_mainloop_tma<1>(d, ct, smem, sh, ps);
  }
  else conv_tc_mainloop_cpasync(a, d, ct, smem, sh, ps);
  {   // ring stage s was used u = ceil((nsq - s) / nst) times: full completed u times, empty u - 1
    const int nst = d.tma ? d.nst : MT_STAGES;
    const int nsq = d.tma ? (ct.nk + d.kg - 1) / d.kg : ct.nk;   // ring stages filled by this tile
    for (int st = 0; st < nst && st < nsq; ++st) {
      const int u1 = (nsq - 1 - st) / nst;   // u - 1
      if (u1 & 1) ps.eph ^= 1u << st;
      if (d.tma && (u1 & 1) == 0) ps.fph ^= 1u << st;
    }
  }
  if (tid < 64) mbar_wait(bar_accf, ps.acc_phase);
  else mbar_wait_backoff(bar_accf, ps.acc_phase);
  ps.acc_phase ^= 1;
  tc_fence_after();
  if (tid == 0) sh.t_mma = gtimer();

  // epilogue: warp w drains TMEM lanes 32*(w&3).. and column half (w>>2)
  const int warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, half = warp >> 2;   // 2 CTAs/SM: 4 warps, each drains all columns
  const int r = 32 * q + lane;
  const int m = conv_row_pixel(d, ct, r);
  const int hcols = d.bn / (MT_NTHREADS / 128);
  const uint32_t tl = sh.tmem_base + ((uint32_t)(32 * q) << 16);
  const bool stamp = a.trace != nullptr && (tid == 0 || tid == MT_NTHREADS - 1);
  if (stamp) sh.t_kb[tid == 0 ? 0 : 2] = gtimer();   // epilogue start (warp 0 / warp 7)
  if (S == 1) {
    if (hcols >= 32) {
      for (int cb = half * hcols; cb < (half + 1) * hcols; cb += 32) {
        // residual of these 32 columns requested before the TMEM drain (hides its L2 latency)
        uint4 rr[4] = {};
        const bool okrow = m >= 0;
        if ((d.flags & OPF_RES) && okrow && n0 + cb + 32 <= d.Co) {
          const bf16 *rp = reinterpret_cast<const bf16 *>(d.res) + (int64_t)m * d.res_cs + d.res_co + n0 + cb;
#pragma unroll
          for (int j = 0; j < 4; ++j) rr[j] = __ldcg(reinterpret_cast<const uint4 *>(rp) + j);
        }
        float v[32];
        tmem_ld32(tl + cb, v);
        if (okrow) {
          if ((d.flags & OPF_RES) && n0 + cb + 32 <= d.Co) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float rf[8];
              Raw8<bf16> raw;
              raw.u = rr[j];
              cvt8(raw, rf);
              float y[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                y[e] = act_f(fmaf(v[j * 8 + e], sh.esc[cb + j * 8 + e], sh.esh[cb + j * 8 + e]) + rf[e], d.act);
              store_out8<bf16>(a, d, m, n0 + cb + j * 8, y, 8);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (n0 + cb + j * 8 < d.Co) conv_epilogue_vals(a, d, sh, m, n0, cb + j * 8, v + j * 8);
          }
        }
      }
    } else if (hcols == 16 && d.tma != 3 && n0 + half * 16 + 16 <= d.Co) {
      // bn = 32, both 8-column groups valid: the residual (packed bf16) is requested before the
      // TMEM drain and both groups come out of one TMEM load + wait
      const int c0 = half * 16;
      uint4 rr[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
      if ((d.flags & OPF_RES) && m >= 0) {
        const bf16 *rp = reinterpret_cast<const bf16 *>(d.res) + (int64_t)m * d.res_cs + d.res_co + n0 + c0;
        rr[0] = __ldcg(reinterpret_cast<const uint4 *>(rp));
        rr[1] = __ldcg(reinterpret_cast<const uint4 *>(rp) + 1);
      }
      float v[16];
      tmem_ld16(tl + c0, v);
      if (m >= 0) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          Raw8<bf16> raw;
          raw.u = rr[j];
          float rf[8];
          cvt8(raw, rf);
          conv_epilogue_store(a, d, sh, m, n0, c0 + 8 * j, v + 8 * j, rf);
        }
      }
    } else {
      for (int col = half * hcols; col < (half + 1) * hcols; col += 8) {
        float v[8];
        tmem_ld8(tl + col, v);
        if (d.tma == 3) {
          if (m >= 0 && n0 + col < d.N) fc_tc_store(a, d, sh, r, m, n0 + col, v);
        } else if (m >= 0 && n0 + col < d.Co) {
          conv_epilogue_vals(a, d, sh, m, n0, col, v);
        }
      }
    }
  } else {
    // split-K part: fp32 partial tile -> workspace [tmn*S + ks][bn][128] (valid rows/cols only);
    // the reduce tiles of this (M,N) tile sum the S partials in split order (deterministic)
    float *ws = reinterpret_cast<float *>(d.ws);
    if (hcols >= 32) {
      for (int cb = half * hcols; cb < (half + 1) * hcols; cb += 32) {
        float v[32];
        tmem_ld32(tl + cb, v);
        float *p = ws + ((int64_t)(tmn * S + ks) * d.bn + cb) * MT_BM + r;
        if (m >= 0)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (n0 + cb + e < d.Co) __stcg(p + e * MT_BM, v[e]);
      }
    } else {
      for (int col = half * hcols; col < (half + 1) * hcols; col += 8) {
        float v[8];
        tmem_ld8(tl + col, v);
        float *p = ws + ((int64_t)(tmn * S + ks) * d.bn + col) * MT_BM + r;
        if (m >= 0 && n0 + col < (d.tma == 3 ? d.N : d.Co))
#pragma unroll
          for (int e = 0; e < 8; ++e) __stcg(p + e * MT_BM, v[e]);
      }
    }
    // published together with the tile's completion in run_stage (one fence for all counters)
    if (tid == 0) sh.xrel = a.splitcnt + d.cnt_off + tmn;
  }
  if (stamp) sh.t_kb[tid == 0 ? 1 : 3] = gtimer();   // stores issued (warp 0 / warp 7)
  tc_fence_before();
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// fp32 path (config 1, 1e-4 parity): implicit GEMM on CUDA cores, 64 x 64 tile, 4x4 per thread
// ------------------------------------------------------------------------------------------
template <typename T>
__device__ void conv_simt_tile(const RunArgs &a, const OpDesc &d, int tile, uint8_t *smem) {
  // double-buffered K-blocks: As[2][BK][BM], Bs[2][BK][BN]; the gathers of K-block j+1 are in
  // flight while K-block j's FMAs run.  A thread loads k = k0 + (tid & 15) for the four rows /
  // output channels p0 + 16 i; the per-row gather bases are computed once per tile.  Same FMA
  // order as a single-buffered loop (bit-identical results).
  float *As = reinterpret_cast<float *>(smem);
  float *Bs = As + 2 * MT_SIMT_BK * MT_SIMT_BM;
  const int tid = threadIdx.x;
  const int mt = tile / d.tiles_n, nt = tile - (tile / d.tiles_n) * d.tiles_n;
  const int m0 = mt * MT_SIMT_BM, n0 = nt * MT_SIMT_BN;
  const T *X = in_ptr<T>(a, d);
  const float *Wt = reinterpret_cast<const float *>(d.w);
  const int HoWo = d.Ho * d.Wo;
  const int ty = tid >> 4, tx = tid & 15;
  const int kk = tid & 15, p0 = tid >> 4;
  int hb[4], wb[4], base[4];
  bool rv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + p0 + 16 * i;
    rv[i] = m < d.M;
    const int mm = rv[i] ? m : 0;
    const int n = mm / HoWo, rem = mm - n * HoWo;
    const int ho = rem / d.Wo, wo = rem - ho * d.Wo;
    base[i] = n * d.H;
    hb[i] = ho * d.sh - d.ph;
    wb[i] = wo * d.sw - d.pw;
  }
  float ra[4], rb[4];
  auto load = [&](int k0) {
    const int k = k0 + kk;
    const bool kv = k < d.K;
    const int tap = kv ? k / d.C : 0, ci = k - tap * d.C;
    const int rr = tap / d.kw, ss = tap - rr * d.kw;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int hi = hb[i] + rr, wi = wb[i] + ss;
      ra[i] = (kv && rv[i] && hi >= 0 && hi < d.H && wi >= 0 && wi < d.W)
                  ? ld1_cg(X + ((int64_t)(base[i] + hi) * d.W + wi) * d.in_cs + d.in_co + ci)
                  : 0.f;
      const int co = n0 + p0 + 16 * i;
      rb[i] = (kv && co < d.Co) ? __ldg(Wt + (int64_t)co * d.K + k) : 0.f;
    }
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  load(0);
  int buf = 0;
  for (int k0 = 0; k0 < d.K; k0 += MT_SIMT_BK) {
    float *Ab = As + buf * MT_SIMT_BK * MT_SIMT_BM, *Bb = Bs + buf * MT_SIMT_BK * MT_SIMT_BN;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      Ab[kk * MT_SIMT_BM + p0 + 16 * i] = ra[i];
      Bb[kk * MT_SIMT_BN + p0 + 16 * i] = rb[i];
    }
    __syncthreads();
    if (k0 + MT_SIMT_BK < d.K) load(k0 + MT_SIMT_BK);
#pragma unroll
    for (int k2 = 0; k2 < MT_SIMT_BK; ++k2) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = Ab[k2 * MT_SIMT_BM + ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bb[k2 * MT_SIMT_BN + tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    buf ^= 1;
  }
  __syncthreads();
  const float *sc = reinterpret_cast<const float *>(d.scale);
  const float *sf = reinterpret_cast<const float *>(d.shift);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= d.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= d.Co) continue;
      float y = fmaf(acc[i][j], __ldg(sc + n), __ldg(sf + n));
      if (d.flags & OPF_RES) y += ld1_cg(reinterpret_cast<const T *>(d.res) + (int64_t)m * d.res_cs + d.res_co + n);
      y = act_f(y, d.act);
      if (d.flags & OPF_OUT) a.outputs[d.tenant][(int64_t)m * d.Co + n] = y;
      else st1(reinterpret_cast<T *>(d.out) + (int64_t)m * d.out_cs + d.out_co + n, y);
    }
  }
}

// ------------------------------------------------------------------------------------------
// a6: depthwise conv (+ folded BN + act); item = (output pixel, 8-channel group)
// ------------------------------------------------------------------------------------------
template <typename T, int KH, int KW>
__device__ __forceinline__ void dw_item(const RunArgs &a, const OpDesc &d, const T *X, const float *Wt,
                                        int64_t pix, int g) {
  const int n = (int)(pix / (d.Ho * d.Wo));
  const int rem = (int)(pix - (int64_t)n * d.Ho * d.Wo);
  const int ho = rem / d.Wo, wo = rem - ho * d.Wo;
  const int kh = KH > 0 ? KH : d.kh, kw = KW > 0 ? KW : d.kw;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  constexpr int NT = (KH > 0 && KW > 0) ? KH * KW : 1;
  if constexpr (NT > 1) {
    Raw8<T> xr[NT];
    // issue every tap's load first (memory-level parallelism), out-of-window taps read zeros
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int hi = ho * d.sh - d.ph + t / KW, wi = wo * d.sw - d.pw + t % KW;
      if (hi >= 0 && hi < d.H && wi >= 0 && wi < d.W)
        ldraw_cg(X + ((int64_t)(n * d.H + hi) * d.W + wi) * d.in_cs + d.in_co + g * 8, xr[t]);
      else
        zero_raw(xr[t]);
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      float w[8], x[8];
      ld8_nc(Wt + (int64_t)t * d.C + g * 8, w);
      cvt8(xr[t], x);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fmaf(x[q], w[q], acc[q]);
    }
  } else {
    for (int r = 0; r < kh; ++r) {
      const int hi = ho * d.sh - d.ph + r;
      if (hi < 0 || hi >= d.H) continue;
      for (int s = 0; s < kw; ++s) {
        const int wi = wo * d.sw - d.pw + s;
        if (wi < 0 || wi >= d.W) continue;
        float x[8], w[8];
        ld8_cg(X + ((int64_t)(n * d.H + hi) * d.W + wi) * d.in_cs + d.in_co + g * 8, x);
        ld8_nc(Wt + (int64_t)(r * kw + s) * d.C + g * 8, w);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fmaf(x[q], w[q], acc[q]);
      }
    }
  }
  const float *sc = reinterpret_cast<const float *>(d.scale);
  const float *sf = reinterpret_cast<const float *>(d.shift);
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = act_f(fmaf(acc[q], __ldg(sc + g * 8 + q), __ldg(sf + g * 8 + q)), d.act);
  store_out8<T>(a, d, pix, g * 8, acc, 8);
}

__device__ __forceinline__ bool dw3_staged(const OpDesc &d, int cap) {
  return d.kh == 3 && d.kw == 3 && d.sh == d.sw && (d.sh == 1 || d.sh == 2) && d.pix_tile % d.Wo == 0 &&
         11 * d.C * 4 <= cap;
}
__device__ __forceinline__ bool fc_staged(const OpDesc &d, int cap) {
  const int64_t b = (int64_t)MT_FC_ROWS * d.K * (d.prec == 1 ? 4 : 2);
  return b <= 96 * 1024 && b <= cap;
}
// packed fp32x2 FMA (sm_100 FFMA2): per lane identical to fmaf, so results are unchanged
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)),
        "l"(*reinterpret_cast<unsigned long long *>(&c)));
  return *reinterpret_cast<float2 *>(&r);
}
__device__ __forceinline__ void cvt8x2(const Raw8<bf16> &r, float2 *v) {
  const uint32_t *u = reinterpret_cast<const uint32_t *>(&r.u);
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = make_float2(__uint_as_float(u[i] << 16), __uint_as_float(u[i] & 0xFFFF0000u));
}
__device__ __forceinline__ void cvt8x2(const Raw8<float> &r, float2 *v) {
  v[0] = make_float2(r.a.x, r.a.y); v[1] = make_float2(r.a.z, r.a.w);
  v[2] = make_float2(r.b.x, r.b.y); v[3] = make_float2(r.b.z, r.b.w);
}
__device__ __forceinline__ Raw8<bf16> ldraw_cg_pred(const bf16 *p, bool ok) {
  Raw8<bf16> r;
  r.u = ok ? __ldcg(reinterpret_cast<const uint4 *>(p)) : make_uint4(0, 0, 0, 0);
  return r;
}
__device__ __forceinline__ Raw8<float> ldraw_cg_pred(const float *p, bool ok) {
  Raw8<float> r;
  r.a = ok ? __ldcg(reinterpret_cast<const float4 *>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
  r.b = ok ? __ldcg(reinterpret_cast<const float4 *>(p) + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
  return r;
}

// 3x3 depthwise, row-run form: a thread computes RUN consecutive outputs of one row for one
// 8-channel group; each kernel row's (RUN-1)*S+3 input columns are loaded and converted once and
// reused by the neighbouring outputs; weights (fp32, [9][C]) stay in registers; packed FFMA2.
// A tile = whole output rows (pix_tile = rows * Wo); item = (row, run segment, channel group),
// channel group fastest for coalescing.
template <typename T, int S, int RUN>
__device__ void dw3_tile(const RunArgs &a, const OpDesc &d, int tile, const uint8_t *smem) {
  constexpr int NC = (RUN - 1) * S + 3;
  const T *X = in_ptr<T>(a, d);
  cp_async_wait<0>();   // weights / scale / shift staged by tile_prefetch during the dependency wait
  __syncthreads();
  if (threadIdx.x == 0) sh_t_first_dw = gtimer();
  const float *Wt = reinterpret_cast<const float *>(smem);
  const float *sc = Wt + 9 * d.C;
  const float *sf = Wt + 10 * d.C;
  const int cg = d.C >> 3;
  const int nseg = (d.Wo + RUN - 1) / RUN;
  const int rows = d.pix_tile / d.Wo;
  const int row0 = tile * rows;
  const int nrows = min(rows, d.N * d.Ho - row0);
  const int items = nrows * nseg * cg;
  const int H = d.H, W = d.W, cs = d.in_cs;
  for (int it = threadIdx.x; it < items; it += MT_NTHREADS) {
    const int g = it % cg;
    const int rs = it / cg;
    const int seg = rs % nseg;
    const int gr = row0 + rs / nseg;            // global output row (n*Ho + ho)
    const int n = gr / d.Ho, ho = gr - n * d.Ho;
    const int wo0 = seg * RUN;
    const int wi0 = wo0 * S - d.pw;
    const T *xrow = X + (int64_t)n * H * W * cs + d.in_co + g * 8;
    float2 acc[RUN][4];
#pragma unroll
    for (int o = 0; o < RUN; ++o)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[o][q] = make_float2(0.f, 0.f);
    // rolling two-row window: rows 0 and 1 are loaded up front, row 2 into row 0's registers once
    // row 0 is consumed (two thirds of the registers of loading all three rows, which set the
    // executor's register peak); taps are still accumulated in (r, s) order
    Raw8<T> xa[NC], xb[NC];
    auto load_row = [&](int r, Raw8<T> *dst) {
      const int hi = ho * S - d.ph + r;
      const bool rok = hi >= 0 && hi < H;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int wi = wi0 + c;
        dst[c] = ldraw_cg_pred(xrow + (int64_t)(hi * W + wi) * cs, rok && wi >= 0 && wi < W);
      }
    };
    auto mac_row = [&](int r, const Raw8<T> *src) {
      float2 w2[3][4];   // this kernel row's 3 taps (fp32 weights, [9][C])
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const float4 lo = reinterpret_cast<const float4 *>(Wt + (r * 3 + t) * d.C + g * 8)[0];
        const float4 hi = reinterpret_cast<const float4 *>(Wt + (r * 3 + t) * d.C + g * 8)[1];
        w2[t][0] = make_float2(lo.x, lo.y); w2[t][1] = make_float2(lo.z, lo.w);
        w2[t][2] = make_float2(hi.x, hi.y); w2[t][3] = make_float2(hi.z, hi.w);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        float2 x[4];
        cvt8x2(src[c], x);
#pragma unroll
        for (int s2 = 0; s2 < 3; ++s2) {
          // column c feeds output o when o*S + s2 == c
          if ((c - s2) >= 0 && (c - s2) % S == 0 && (c - s2) / S < RUN) {
            const int o = (c - s2) / S;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[o][q] = ffma2(x[q], w2[s2][q], acc[o][q]);
          }
        }
      }
    };
    load_row(0, xa);
    load_row(1, xb);
    if (threadIdx.x == 0 && it == 0) { const uint32_t u = raw_word(xb[NC - 1]); sh_t_load_dw = gtimer() + (u == 0x7fff1234u); }
    mac_row(0, xa);
    load_row(2, xa);
    mac_row(1, xb);
    mac_row(2, xa);
    float2 sc2[4], sf2[4];
    {
      const float4 a0 = reinterpret_cast<const float4 *>(sc + g * 8)[0];
      const float4 a1 = reinterpret_cast<const float4 *>(sc + g * 8)[1];
      const float4 b0 = reinterpret_cast<const float4 *>(sf + g * 8)[0];
      const float4 b1 = reinterpret_cast<const float4 *>(sf + g * 8)[1];
      sc2[0] = make_float2(a0.x, a0.y); sc2[1] = make_float2(a0.z, a0.w);
      sc2[2] = make_float2(a1.x, a1.y); sc2[3] = make_float2(a1.z, a1.w);
      sf2[0] = make_float2(b0.x, b0.y); sf2[1] = make_float2(b0.z, b0.w);
      sf2[2] = make_float2(b1.x, b1.y); sf2[3] = make_float2(b1.z, b1.w);
    }
#pragma unroll
    for (int o = 0; o < RUN; ++o) {
      if (wo0 + o < d.Wo) {
        float y[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 t = ffma2(acc[o][q], sc2[q], sf2[q]);
          y[2 * q] = act_f(t.x, d.act);
          y[2 * q + 1] = act_f(t.y, d.act);
        }
        store_out8<T>(a, d, (int64_t)gr * d.Wo + wo0 + o, g * 8, y, 8);
      }
    }
  }
}

template <typename T>
__device__ void dw_tile(const RunArgs &a, const OpDesc &d, int tile, const uint8_t *smem, int cap) {
  if (dw3_staged(d, cap)) {
    // fp32 storage: shorter runs (an fp32 8-channel vector is 8 registers, bf16's is 4); the
    // per-output tap order is the same for every run length, so results do not depend on it
    constexpr int R1 = sizeof(T) == 4 ? 2 : 4, R2 = sizeof(T) == 4 ? 1 : 2;
    if (d.sh == 1) dw3_tile<T, 1, R1>(a, d, tile, smem);
    else dw3_tile<T, 2, R2>(a, d, tile, smem);
    return;
  }
  const T *X = in_ptr<T>(a, d);
  const float *Wt = reinterpret_cast<const float *>(d.w);
  const int cg = d.C >> 3;
  const int p0 = tile * d.pix_tile;
  const int np = min(d.pix_tile, d.N * d.Ho * d.Wo - p0);
  for (int it = threadIdx.x; it < np * cg; it += MT_NTHREADS) {
    const int pix = p0 + it / cg;
    const int g = it % cg;
    dw_item<T, 0, 0>(a, d, X, Wt, pix, g);
  }
}

// ------------------------------------------------------------------------------------------
// a7: max / avg pooling (PyTorch window semantics: padding, ceil_mode, count_include_pad)
// ------------------------------------------------------------------------------------------
template <typename T, int K>
__device__ __forceinline__ void pool_item(const RunArgs &a, const OpDesc &d, const T *X, int64_t pix, int g) {
  const bool is_max = d.kind == 4;
  const int n = (int)(pix / (d.Ho * d.Wo));
  const int rem = (int)(pix - (int64_t)n * d.Ho * d.Wo);
  const int ho = rem / d.Wo, wo = rem - ho * d.Wo;
  const int hs = ho * d.sh - d.ph, ws = wo * d.sw - d.pw;
  const int he = min(hs + d.kh, d.H + d.ph), we = min(ws + d.kw, d.W + d.pw);
  int div = (he - hs) * (we - ws);
  const int h0 = max(hs, 0), h1 = min(he, d.H), w0 = max(ws, 0), w1 = min(we, d.W);
  if (!d.cip) div = (h1 - h0) * (w1 - w0);
  float acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = is_max ? -INFINITY : 0.f;
  if constexpr (K > 0) {
    Raw8<T> xr[K * K];
    bool v[K * K];
#pragma unroll
    for (int t = 0; t < K * K; ++t) {
      const int hi = h0 + t / K, wi = w0 + t % K;
      v[t] = hi < h1 && wi < w1;
      if (v[t]) ldraw_cg(X + ((int64_t)(n * d.H + hi) * d.W + wi) * d.in_cs + d.in_co + g * 8, xr[t]);
    }
#pragma unroll
    for (int t = 0; t < K * K; ++t)
      if (v[t]) {
        float x[8];
        cvt8(xr[t], x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = is_max ? fmaxf(acc[q], x[q]) : acc[q] + x[q];
      }
  } else {
    for (int hi = h0; hi < h1; ++hi)
      for (int wi = w0; wi < w1; ++wi) {
        float x[8];
        ld8_cg(X + ((int64_t)(n * d.H + hi) * d.W + wi) * d.in_cs + d.in_co + g * 8, x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = is_max ? fmaxf(acc[q], x[q]) : acc[q] + x[q];
      }
  }
  if (!is_max) {
    const float inv = 1.f / (float)div;
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = acc[q] * inv;
  }
  store_out8<T>(a, d, pix, g * 8, acc, 8);
}

template <typename T>
__device__ void pool_tile(const RunArgs &a, const OpDesc &d, int tile) {
  const T *X = in_ptr<T>(a, d);
  const int cg = d.C >> 3;
  const int64_t p0 = (int64_t)tile * d.pix_tile;
  const int64_t np = min((int64_t)d.pix_tile, (int64_t)d.N * d.Ho * d.Wo - p0);
  for (int it = threadIdx.x; it < np * cg; it += MT_NTHREADS) {
    const int64_t pix = p0 + it / cg;
    const int g = it - (it / cg) * cg;
    if (d.kh <= 2 && d.kw <= 2) pool_item<T, 2>(a, d, X, pix, g);
    else if (d.kh <= 3 && d.kw <= 3) pool_item<T, 3>(a, d, X, pix, g);
    else pool_item<T, 0>(a, d, X, pix, g);
  }
}

// global average pool: tile = (n, 32 channel groups); thread = (group, pixel lane of 8); each
// lane sums pixels p = lane, lane+8, ... then lanes are combined in a fixed tree (deterministic)
template <typename T>
__device__ void gap_tile(const RunArgs &a, const OpDesc &d, int tile, uint8_t *smem) {
  const T *X = in_ptr<T>(a, d);
  const int cg = d.C >> 3;
  const int tiles_c = (cg + MT_GAP_G - 1) / MT_GAP_G;
  const int n = tile / tiles_c, g0 = (tile - n * tiles_c) * MT_GAP_G;
  const int g = g0 + (threadIdx.x >> 3), lane = threadIdx.x & 7;
  const int HW = d.H * d.W;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (g < cg) {
    const T *p = X + (int64_t)n * HW * d.in_cs + d.in_co + g * 8;
    int i = lane;
    for (; i + 24 < HW; i += 32) {   // 4 independent loads in flight per thread
      float x0[8], x1[8], x2[8], x3[8];
      ld8_cg(p + (int64_t)i * d.in_cs, x0);
      ld8_cg(p + (int64_t)(i + 8) * d.in_cs, x1);
      ld8_cg(p + (int64_t)(i + 16) * d.in_cs, x2);
      ld8_cg(p + (int64_t)(i + 24) * d.in_cs, x3);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += ((x0[q] + x1[q]) + (x2[q] + x3[q]));
    }
    for (; i < HW; i += 8) {
      float x[8];
      ld8_cg(p + (int64_t)i * d.in_cs, x);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += x[q];
    }
  }
  float *red = reinterpret_cast<float *>(smem);   // [MT_NTHREADS][8]
#pragma unroll
  for (int q = 0; q < 8; ++q) red[threadIdx.x * 8 + q] = acc[q];
  __syncthreads();
  if (lane == 0 && g < cg) {
    float s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float *r = red + threadIdx.x * 8 + q;
      s[q] = ((r[0] + r[8]) + (r[16] + r[24])) + ((r[32] + r[40]) + (r[48] + r[56]));
    }
    const float inv = 1.f / (float)HW;
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] *= inv;
    store_out8<T>(a, d, n, g * 8, s, 8);
  }
}

// ------------------------------------------------------------------------------------------
// a8: FC (GEMV at b=1, skinny GEMM up to 8 columns per pass): one warp per output row, 16-byte
// weight loads, lane-strided partial sums reduced by a fixed xor-shuffle tree (deterministic)
// ------------------------------------------------------------------------------------------
template <typename T, int NB>
__device__ __forceinline__ void fc_rows(const OpDesc &d, const T *X, const T *Wr, int b0, int nb, int lane,
                                        float *acc) {
  const int K8 = d.K >> 3;
  constexpr int U = NB == 1 ? 8 : 2;   // 16-byte weight loads in flight per lane
  int k8 = lane;
  for (; k8 + 32 * (U - 1) < K8; k8 += 32 * U) {
    Raw8<T> wr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) wr[u] = ldraw_gen(Wr + (int64_t)(k8 + 32 * u) * 8);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float w[8];
      cvt8(wr[u], w);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (NB == 1 || b < nb) {
          float x[8];
          ld8_cg(X + (int64_t)(b0 + b) * d.K + (int64_t)(k8 + 32 * u) * 8, x);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[b] = fmaf(w[q], x[q], acc[b]);
        }
      }
    }
  }
  for (; k8 < K8; k8 += 32) {
    float w[8];
    cvt8(ldraw_gen(Wr + (int64_t)k8 * 8), w);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (NB == 1 || b < nb) {
        float x[8];
        ld8_cg(X + (int64_t)(b0 + b) * d.K + (int64_t)k8 * 8, x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[b] = fmaf(w[q], x[q], acc[b]);
      }
    }
  }
}

template <typename T>
__device__ void fc_tile(const RunArgs &a, const OpDesc &d, int tile, const uint8_t *smem, int cap) {
  const bool staged = fc_staged(d, cap);
  if (staged) {   // weight rows staged by tile_prefetch during the dependency wait
    cp_async_wait<0>();
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = (int)(tile % ((d.Co + MT_FC_ROWS - 1) / MT_FC_ROWS));
  const int bb = (int)(tile / ((d.Co + MT_FC_ROWS - 1) / MT_FC_ROWS));
  const int o = rb * MT_FC_ROWS + warp;
  if (o >= d.Co) return;
  const int b0 = bb * MT_FC_BATCH;
  const int nb = min(MT_FC_BATCH, d.N - b0);
  const T *X = in_ptr<T>(a, d);
  const T *Wr = staged ? reinterpret_cast<const T *>(smem) + (int64_t)warp * d.K
                       : reinterpret_cast<const T *>(d.w) + (int64_t)o * d.K;
  float acc[MT_FC_BATCH];
#pragma unroll
  for (int b = 0; b < MT_FC_BATCH; ++b) acc[b] = 0.f;
  if (nb == 1) fc_rows<T, 1>(d, X, Wr, b0, 1, lane, acc);
  else fc_rows<T, MT_FC_BATCH>(d, X, Wr, b0, nb, lane, acc);
#pragma unroll
  for (int b = 0; b < MT_FC_BATCH; ++b) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], off);
  }
  if (lane == 0) {
    const float sc = __ldg(reinterpret_cast<const float *>(d.scale) + o);
    const float sf = __ldg(reinterpret_cast<const float *>(d.shift) + o);
    for (int b = 0; b < nb; ++b) {
      const float y = act_f(fmaf(acc[b], sc, sf), d.act);
      if (d.flags & OPF_OUT) a.outputs[d.tenant][(int64_t)(b0 + b) * d.Co + o] = y;
      else st1(reinterpret_cast<T *>(d.out) + (int64_t)(b0 + b) * d.out_cs + d.out_co + o, y);
    }
  }
}

// ADD (sum of inputs) / BN (affine) / RELU, + act
template <typename T>
__device__ void elt_tile(const RunArgs &a, const OpDesc &d, int tile) {
  const int cg = d.Co >> 3;
  const int64_t p0 = (int64_t)tile * d.pix_tile;
  const int64_t np = min((int64_t)d.pix_tile, (int64_t)d.N * d.Ho * d.Wo - p0);
  for (int it = threadIdx.x; it < np * cg; it += MT_NTHREADS) {
    const int64_t pix = p0 + it / cg;
    const int g = it - (it / cg) * cg;
    float y[8];
    if (d.kind == 8) {  // ADD
      for (int q = 0; q < 8; ++q) y[q] = 0.f;
      for (int i = 0; i < d.n_in; ++i) {
        const T *p = d.ins[i] ? reinterpret_cast<const T *>(d.ins[i]) : reinterpret_cast<const T *>(a.packed[d.tenant]);
        float x[8];
        ld8_cg(p + pix * d.ins_cs[i] + d.ins_co[i] + g * 8, x);
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] += x[q];
      }
    } else {
      ld8_cg(in_ptr<T>(a, d) + pix * d.in_cs + d.in_co + g * 8, y);
      if (d.kind == 2) {  // BN
        const float *sc = reinterpret_cast<const float *>(d.scale);
        const float *sf = reinterpret_cast<const float *>(d.shift);
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] = fmaf(y[q], __ldg(sc + g * 8 + q), __ldg(sf + g * 8 + q));
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = act_f(y[q], d.act);
    store_out8<T>(a, d, pix, g * 8, y, 8);
  }
}

// a7: input pack NCHW fp32 -> NHWC (bf16 or fp32), channels zero-padded to cpad (the
// shared input is packed once per distinct pointer)
template <typename T>
__device__ void pack_pixels(const RunArgs &a, int t, int64_t first, int64_t stride) {
  const int N = a.in_n[t], C = a.in_c[t], H = a.in_h[t], W = a.in_w[t], cp = a.in_cpad[t];
  const int64_t HW = (int64_t)H * W, total = (int64_t)N * HW;
  const float *src = a.inputs[t];
  T *dst = reinterpret_cast<T *>(a.packed[t]);
  for (int64_t p = first; p < total; p += stride) {
    const int64_t n = p / HW, hw = p - n * HW;
    for (int c0 = 0; c0 < cp; c0 += 8) {
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (c0 + q < C) ? __ldg(src + (n * C + c0 + q) * HW + hw) : 0.f;
      st8(dst + p * cp + c0, v);
    }
  }
}

// ------------------------------------------------------------------------------------------
// tile dispatch (shared by the executor and the per-op baseline kernels)
// ------------------------------------------------------------------------------------------
// F32 = false: the kernel instantiation for mixes whose tenants all store bf16 -- the fp32 tile
// variants (config 1 only) are compiled out, which keeps the persistent kernel's code (and its
// instruction-cache footprint) smaller
template <bool F32>
__device__ void run_tile(const RunArgs &a, const OpDesc &d, int tile, uint8_t *smem, CtaShared &sh,
                         PipeState &ps) {
  const bool f32 = F32 && d.prec == 1;
  switch (d.tk) {
    case TK_CONV_TC: conv_tc_tile(a, d, tile, smem, sh, ps); return;
    case TK_CONV_SIMT:
      if constexpr (F32) {
        if (f32) conv_simt_tile<float>(a, d, tile, smem);
        else conv_simt_tile<bf16>(a, d, tile, smem);
      }
      break;
    case TK_DW: if (f32) dw_tile<float>(a, d, tile, smem, sh.smem_cap); else dw_tile<bf16>(a, d, tile, smem, sh.smem_cap); break;
    case TK_POOL: if (f32) pool_tile<float>(a, d, tile); else pool_tile<bf16>(a, d, tile); break;
    case TK_GAP: if (f32) gap_tile<float>(a, d, tile, smem); else gap_tile<bf16>(a, d, tile, smem); break;
    case TK_FC: if (f32) fc_tile<float>(a, d, tile, smem, sh.smem_cap); else fc_tile<bf16>(a, d, tile, smem, sh.smem_cap); break;
    case TK_ELT: if (f32) elt_tile<float>(a, d, tile); else elt_tile<bf16>(a, d, tile); break;
    default: break;
  }
  __syncthreads();
}

// output pixel range [p0, p1) of a tile (pixel = n*Ho*Wo + ho*Wo + wo; FC/GAP: batch index)
__device__ __forceinline__ void tile_out_range(const OpDesc &d, int tile, int64_t &p0, int64_t &p1) {
  const int64_t npix = (int64_t)d.N * d.Ho * d.Wo;
  switch (d.tk) {
    case TK_CONV_TC:
      if (d.splits > 1 && tile >= d.tiles_m * d.tiles_n * d.splits)   // reduce tile -> its (M,N) tile
        tile = ((tile - d.tiles_m * d.tiles_n * d.splits) / d.rc) * d.splits;
      if (d.tma == 3) {   // FC: batch images [n0, n0 + bn)
        p0 = (int64_t)(((tile / d.splits) % d.tiles_n) * d.bn);
        p1 = min((int64_t)d.N, p0 + d.bn);
        return;
      }
      if (d.tma) {
        const int mt = (tile / d.splits) / d.tiles_n, rg = mt / d.nseg, seg = mt - rg * d.nseg;
        const int img = rg / d.blk_tpi, ho0 = (rg - img * d.blk_tpi) * d.blk_rows;
        p0 = ((int64_t)img * d.Ho + ho0) * d.Wo + seg * d.seg_w;
        p1 = d.nseg > 1 ? p0 + min(d.seg_w, d.Wo - seg * d.seg_w)
                        : ((int64_t)img * d.Ho + min(d.Ho, ho0 + d.blk_rows)) * d.Wo;
      } else {
        p0 = (int64_t)((tile / d.splits) / d.tiles_n) * MT_BM;
        p1 = p0 + MT_BM;
      }
      break;
    case TK_CONV_SIMT: p0 = (int64_t)(tile / d.tiles_n) * MT_SIMT_BM; p1 = p0 + MT_SIMT_BM; break;
    case TK_GAP: p0 = tile / ((d.Co / 8 + MT_GAP_G - 1) / MT_GAP_G); p1 = p0 + 1; break;
    case TK_FC: p0 = (int64_t)(tile / ((d.Co + MT_FC_ROWS - 1) / MT_FC_ROWS)) * MT_FC_BATCH; p1 = p0 + MT_FC_BATCH; break;
    default: p0 = (int64_t)tile * d.pix_tile; p1 = p0 + d.pix_tile; break;
  }
  if (p1 > npix) p1 = npix;
}
// input pixel range [i0, i1) the tile reads (receptive field, whole rows, clamped)
__device__ __forceinline__ void tile_in_range(const OpDesc &d, int64_t p0, int64_t p1, int64_t &i0, int64_t &i1) {
  const int64_t HW = (int64_t)d.H * d.W;
  if (d.tk == TK_ELT) { i0 = p0; i1 = p1; return; }
  if (d.tk == TK_GAP) { i0 = p0 * HW; i1 = p1 * HW; return; }
  if (d.tk == TK_FC || (d.tk == TK_CONV_TC && d.tma == 3)) { i0 = p0 * HW; i1 = p1 * HW; return; }
  const int HoWo = d.Ho * d.Wo;
  const int na = (int)(p0 / HoWo), nb = (int)((p1 - 1) / HoWo);
  const int hoa = (int)((p0 - (int64_t)na * HoWo) / d.Wo), hob = (int)((p1 - 1 - (int64_t)nb * HoWo) / d.Wo);
  const int ha = max(0, min(d.H - 1, hoa * d.sh - d.ph));
  const int hb = max(0, min(d.H - 1, hob * d.sh - d.ph + d.kh - 1));
  i0 = (int64_t)na * HW + (int64_t)ha * d.W;
  i1 = (int64_t)nb * HW + (int64_t)(hb + 1) * d.W;
}
// completion block a finished tile contributes to (-1: none, e.g. a non-final split-K part)
__device__ __forceinline__ int tile_block(const OpDesc &d, int tile, const CtaShared &sh) {
  switch (d.tk) {
    case TK_CONV_TC: {   // block = M tile (TMA: row group, i.e. all column segments of it)
      if (d.tma == 3) {    // FC: block = batch tile
        const int nct = d.tiles_m * d.tiles_n * d.splits;
        if (d.splits == 1) return tile % d.tiles_n;
        return tile >= nct ? ((tile - nct) / d.rc) % d.tiles_n : -1;
      }
      const int ns = d.tma ? d.nseg : 1;
      if (d.splits == 1) return tile / d.tiles_n / ns;
      const int nct = d.tiles_m * d.tiles_n * d.splits;
      return tile >= nct ? ((tile - nct) / d.rc) / d.tiles_n / ns : -1;   // only reduce tiles complete
    }
    case TK_CONV_SIMT: return tile / d.tiles_n;
    case TK_GAP: return tile / ((d.Co / 8 + MT_GAP_G - 1) / MT_GAP_G);
    case TK_FC: return tile / ((d.Co + MT_FC_ROWS - 1) / MT_FC_ROWS);
    default: return tile;
  }
}

// work that needs no producer data: issued before the dependency wait so it overlaps it
// copy n16 16-byte chunks global -> shared with cp.async (completion waited in the tile)
__device__ __forceinline__ void stage_smem(uint32_t dst, const void *src, int n16) {
  for (int i = threadIdx.x; i < n16; i += MT_NTHREADS)
    cp_async16(dst + i * 16, reinterpret_cast<const char *>(src) + (int64_t)i * 16, true);
}

__device__ void tile_prefetch(const OpDesc &d, int tile, uint8_t *smem, CtaShared &sh, const PipeState &ps) {
  if (d.tk == TK_DW && dw3_staged(d, sh.smem_cap)) {   // [9][C] fp32 weights, scale[C], shift[C]
    const uint32_t s0 = smem_u32(smem);
    stage_smem(s0, reinterpret_cast<const void *>(d.w), 9 * d.C * 4 / 16);
    stage_smem(s0 + 9 * d.C * 4, reinterpret_cast<const void *>(d.scale), d.C * 4 / 16);
    stage_smem(s0 + 10 * d.C * 4, reinterpret_cast<const void *>(d.shift), d.C * 4 / 16);
    cp_async_commit();
    return;
  }
  if (d.tk == TK_FC && fc_staged(d, sh.smem_cap)) {     // the tile's weight rows
    const int rb = (int)(tile % ((d.Co + MT_FC_ROWS - 1) / MT_FC_ROWS));
    const int rows = min(MT_FC_ROWS, d.Co - rb * MT_FC_ROWS);
    const int eb = d.prec == 1 ? 4 : 2;
    stage_smem(smem_u32(smem), reinterpret_cast<const char *>(d.w) + (int64_t)rb * MT_FC_ROWS * d.K * eb,
               (int)((int64_t)rows * d.K * eb / 16));
    cp_async_commit();
    return;
  }
  if (d.tk == TK_CONV_TC) {
    if (d.splits > 1 && tile >= d.tiles_m * d.tiles_n * d.splits) return;   // reduce tile
    conv_tc_prefetch(d, tile, smem, sh, ps);
  } else if (d.tk == TK_FC) {
    const int rb = (int)(tile % ((d.Co + MT_FC_ROWS - 1) / MT_FC_ROWS));
    const int o = rb * MT_FC_ROWS + (threadIdx.x >> 5);
    if ((threadIdx.x & 31) == 0 && o < d.Co) {
      const int eb = d.prec == 1 ? 4 : 2;
      const char *row = reinterpret_cast<const char *>(d.w) + (int64_t)o * d.K * eb;
      const int64_t bytes = (int64_t)d.K * eb;
      for (int64_t off = 0; off < bytes; off += 65536)
        prefetch_l2_bulk(row + off, (uint32_t)(bytes - off < 65536 ? bytes - off : 65536));
    }
  }
}

__device__ __forceinline__ void load_desc(CtaShared &sh, const OpDesc *src) {
  const int *s = reinterpret_cast<const int *>(src);
  int *d = reinterpret_cast<int *>(&sh.d);
  for (int i = threadIdx.x; i < (int)(sizeof(OpDesc) / 4); i += blockDim.x) d[i] = __ldg(s + i);
}

__device__ __forceinline__ uint8_t *smem_base() {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  return reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
}

__device__ void cta_setup(CtaShared &sh, bool need_tmem) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    sh.xrel = nullptr;
    for (int s = 0; s < MT_MAXST; ++s) {
      mbar_init(smem_u32(&sh.bar_empty[s]), 1);
      mbar_init(smem_u32(&sh.bar_full[s]), 1);
    }
    mbar_init(smem_u32(&sh.bar_accf), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (need_tmem && (tid >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sh.tmem_base)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

__device__ void cta_teardown(CtaShared &sh, bool need_tmem) {
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (need_tmem && (threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sh.tmem_base), "r"(TMEM_COLS)
                 : "memory");
}

// ------------------------------------------------------------------------------------------
// grid barrier (sense via a generation counter; all CTAs co-resident by cooperative launch)
// ------------------------------------------------------------------------------------------
__device__ bool grid_barrier(const RunArgs &a, CtaShared &sh) {
  __syncthreads();
  if (threadIdx.x == 0) {
    CtlBlock *ctl = a.ctl;
    const unsigned gen = ld_acquire_u(&ctl->bar_gen);
    __threadfence();
    const unsigned arrived = atomicAdd(&ctl->bar_count, 1u);
    int ok = 1;
    if (arrived == gridDim.x - 1) {
      atomicExch(&ctl->bar_count, 0u);
      __threadfence();
      st_release_u(&ctl->bar_gen, gen + 1);
    } else {
      const unsigned long long t0 = gtimer();
      while (ld_acquire_u(&ctl->bar_gen) == gen) {
        if (ld_acquire_u(&ctl->error)) { ok = 0; break; }
        if (gtimer() - t0 > a.timeout_ns) {
          atomicExch(&ctl->error, 1u);
          ok = 0;
          break;
        }
        __nanosleep(32);
      }
    }
    sh.ok = ok;
  }
  __syncthreads();
  return sh.ok != 0;
}

// debug trace record: op, tile, smid/cta, pick, deps-satisfied, mainloop-done, end timestamps
__device__ __forceinline__ void trace_tile(const RunArgs &a, const CtaShared &sh, int op, int tile) {
  if (!a.trace) return;
  const unsigned i = atomicAdd(&a.ctl->trace_count, 1u);
  if ((int)i >= a.trace_cap) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  unsigned long long *e = a.trace + (size_t)i * 16;
  e[0] = ((unsigned long long)(unsigned)tile << 32) | (unsigned)op;
  e[1] = ((unsigned long long)blockIdx.x << 32) | smid;
  e[2] = sh.t_pick;
  e[3] = sh.t_deps;
  e[4] = sh.t_mma;
  e[5] = sh.t_run + (unsigned long long)sh.last;   // after the release
  e[6] = (unsigned long long)sh.home;
  e[7] = sh.t_run;
  e[8] = sh.t_first;      // MMA thread: first stage landed
  e[9] = sh.t_lastmma;    // MMA thread: last MMA issued
  e[10] = sh.t_aissue;    // producer: last A box issued
  e[11] = sh.t_kb[0]; e[12] = sh.t_kb[1]; e[13] = sh.t_kb[2]; e[14] = sh.t_kb[3];   // epilogue phases (TC)
  if (!sh.t_kb[0]) { e[11] = sh_t_first_dw; e[12] = sh_t_load_dw; }                    // dw: staged, loads back
  e[15] = sh.t_is[0];     // producer: 4th A box issued
}

// One stage.  Claim-then-wait: thread 0 claims the next unclaimed tile of the first op of its
// home tenant's slice that still has unclaimed tiles (then of the other tenants, round-robin,
// when stealing), i.e. one atomic per pick; tiles are claimed in op order per tenant, so every
// dependency of a claimed tile is itself claimed by a running CTA and the wait always ends
// (all CTAs co-resident).  While the dependencies finish, the tile's weights are already
// streamed into shared memory / L2 (tile_prefetch).
template <bool F32>
__device__ bool run_stage(const RunArgs &a, int s, uint8_t *smem, CtaShared &sh, PipeState &ps) {
  const int T = a.n_tenants;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int t = 0; t < T; ++t) {
      sh.beg[t] = sh.cur[t] = a.rng[(s * T + t) * 2];
      sh.end[t] = a.rng[(s * T + t) * 2 + 1];
    }
    sh.home = a.home[(size_t)s * gridDim.x + sh.vcta];
  }
  __syncthreads();
  while (true) {
    // thread 32 picks the next tile while thread 0 is still releasing the previous one
    if (tid == 32) {
      int op = -1, tile = 0, ten = -1;
      // visiting order: home tenant first; then (steal 1) round-robin or (steal 2) the tenant with
      // the most unclaimed ops of its slice first (critical-path-first list scheduling)
      // (selection on the fly, no local array: ties go to the earlier tenant in round-robin order)
      unsigned visited = 0;
      bool blocked = false;   // claim_depth: some tenant has unclaimed tiles not yet claimable
      for (int q = 0; q < T && op < 0; ++q) {
        if (!a.steal && q > 0) break;
        int t = sh.home + q;
        if (t >= T) t -= T;
        if (q > 0 && a.steal == 2) {
          int best = -1, bestr = -1;
          for (int k = 1; k < T; ++k) {
            int c = sh.home + k;
            if (c >= T) c -= T;
            const int rem = sh.end[c] - sh.cur[c];
            if (!((visited >> c) & 1u) && rem > bestr) { bestr = rem; best = c; }
          }
          t = best;
        }
        visited |= 1u << t;
        while (sh.cur[t] < sh.end[t]) {
          const int o = sh.cur[t];
          if (a.claim_depth != 0) {
            // bounded claim-ahead: op o is claimable once its gate op (host table, staged in
            // shared memory: an ancestor at DAG distance D, or op o - |D|) is complete, so CTAs do
            // not park on tiles far down a latency-bound chain while other tenants have ready
            // work.  Relaxed read: a claiming heuristic; the tile's own dependency wait
            // (acquire) orders its data reads.
            const int x = sh.gate[o];
            bool cpl = x < 0 || ((sh.complete[x >> 5] >> (x & 31)) & 1u);
            if (!cpl && ld_relaxed(a.done + x) >= __ldg(&a.ops[x].tiles)) {
              cpl = true;
              atomicOr(&sh.complete[x >> 5], 1u << (x & 31));
            }
            if (!cpl) { blocked = true; break; }
          }
          const int k = atomicAdd(a.claim + o, 1);
          if (k < __ldg(&a.ops[o].tiles)) { op = o; tile = k; ten = t; break; }
          // every tile of o is claimed: publish that and jump to the furthest frontier any CTA
          // has seen for this tenant (one atomic instead of one failed claim per op when a CTA
          // catches up on a tenant it has not served, e.g. when stealing or at the stage end)
          const int g = atomicMax(&a.ctl->gcur[t], o + 1);
          sh.cur[t] = max(o + 1, g);
        }
      }
      if (op < 0 && blocked) {   // work remains but none is claimable yet: retry shortly
        op = -2;
        if (ld_acquire_u(&a.ctl->error)) op = -3;
        __nanosleep(100);
      }
      sh.op = op;
      sh.tile = tile;
      sh.ten = ten;
      sh.t_pick_next = gtimer();
    }
    __syncthreads();
    const int op = sh.op;
    const int my_tile = sh.tile;
    if (op == -2) continue;
    if (op == -3) return false;
    if (op < 0) return true;
    if (tid == 0) {
      sh.t_pick = sh.t_pick_next;
      sh.t_mma = sh.t_first = sh.t_lastmma = sh.t_aissue = 0;
      sh.t_kb[0] = sh.t_kb[1] = sh.t_kb[2] = sh.t_kb[3] = sh.t_is[0] = 0;
      sh_t_first_dw = sh_t_load_dw = 0;
    }
    load_desc(sh, a.ops + op);
    __syncthreads();
    tile_prefetch(sh.d, sh.tile, smem, sh, ps);
    if (tid < 32) {
      // wait for exactly the producer pixel blocks this tile reads (tile-level dataflow between
      // consecutive ops of a tenant).  Warp 0 polls in parallel: lane k checks whether dependency
      // k is complete as a whole (cached per CTA), then, per incomplete dependency, the lanes poll
      // its blocks together -- one L2 round trip when everything is already there.
      const int lane = tid;
      const OpDesc &d = sh.d;
      int ok = 1;
      bool incomplete = false;
      if (lane < d.n_dep) {
        const int dep = d.deps[lane];
        const bool cached = dep < 2048 && ((sh.complete[dep >> 5] >> (dep & 31)) & 1u);
        if (!cached) {
          if (ld_acquire(a.done + dep) >= __ldg(&a.ops[dep].tiles)) {
            if (dep < 2048) atomicOr(&sh.complete[dep >> 5], 1u << (dep & 31));
          } else {
            incomplete = true;
          }
        }
      }
      unsigned todo = __ballot_sync(0xffffffffu, incomplete);
      if (todo) {
        int64_t p0, p1, i0, i1;
        tile_out_range(d, sh.tile, p0, p1);
        tile_in_range(d, p0, p1, i0, i1);
        bool need_in = true, need_res = true;
        if (d.tk == TK_CONV_TC && d.splits > 1) {
          const bool red_tile = sh.tile >= d.tiles_m * d.tiles_n * d.splits;
          need_in = !red_tile;   // compute parts read the input only,
          need_res = red_tile;   // reduce tiles (epilogue) the residual only
        }
        const unsigned long long t0 = gtimer();
        unsigned spins = 0;
        while (todo) {
          const int k = __ffs(todo) - 1;
          todo &= todo - 1;
          const int dep = d.deps[k];
          const OpDesc *pd = a.ops + dep;
          int64_t lo = INT64_MAX, hi = 0;
          if ((d.dep_kind[k] & 1) && need_in) { lo = i0; hi = i1; }
          if ((d.dep_kind[k] & 2) && need_res) { lo = min(lo, p0); hi = max(hi, p1); }
          if (hi <= lo) continue;
          const int need = __ldg(&pd->blk_need), off = __ldg(&pd->blk_off), nbk = __ldg(&pd->nblk);
          int b0, b1;
          const int br = __ldg(&pd->blk_rows);
          if (br > 0) {   // producer blocks are whole-row M tiles: block = n * tpi + ho / rows
            const int pWo = __ldg(&pd->Wo), pHoWo = __ldg(&pd->Ho) * pWo, tpi = __ldg(&pd->blk_tpi);
            const int na = (int)(lo / pHoWo), nb2 = (int)((hi - 1) / pHoWo);
            b0 = na * tpi + (int)((lo - (int64_t)na * pHoWo) / pWo) / br;
            b1 = nb2 * tpi + (int)((hi - 1 - (int64_t)nb2 * pHoWo) / pWo) / br;
          } else {
            const int pb = __ldg(&pd->pix_blk);
            b0 = (int)(lo / pb);
            b1 = (int)((hi - 1) / pb);
          }
          b1 = min(nbk - 1, b1);
          for (int b = b0 + lane; b <= b1 && ok; b += 32) {
            while (ld_acquire(a.blkcnt + off + b) < need) {
              if ((++spins & 255) == 0) {
                if (ld_acquire_u(&a.ctl->error)) { ok = 0; break; }
                if (gtimer() - t0 > a.timeout_ns) { atomicExch(&a.ctl->error, 2u); ok = 0; break; }
              }
              __nanosleep(20);
            }
          }
        }
      }
      ok = __all_sync(0xffffffffu, ok);
      if (lane == 0) {
        sh.ok = ok;
        sh.t_deps = gtimer();
      }
    }
    __syncthreads();
    if (!sh.ok) { cp_async_wait<0>(); return false; }
    run_tile<F32>(a, sh.d, my_tile, smem, sh, ps);
    if (tid == 0) {   // publish: this tile's outputs are visible (release)
      sh.t_run = gtimer();
      const int b = tile_block(sh.d, my_tile, sh);
      const int boff = sh.d.blk_off;
      fence_proxy_async_global();   // the tile's generic stores, before the release, for TMA readers
      fence_acq_rel_gpu();
      if (sh.xrel) { red_relaxed_add(sh.xrel, 1); sh.xrel = nullptr; }
      if (b >= 0) red_relaxed_add(a.blkcnt + boff + b, 1);
      red_relaxed_add(a.done + op, 1);
      if (a.trace) {
        sh.last = (int)(gtimer() - sh.t_run);
        trace_tile(a, sh, op, my_tile);
      }
    }
  }
}

__device__ __forceinline__ uint32_t sm_id() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}

template <bool F32>
__global__ void __launch_bounds__(MT_NTHREADS, MT_CTAS_PER_SM) executor_kernel(RunArgs a) {
  uint8_t *smem = smem_base();
  __shared__ __align__(16) CtaShared sh;
  PipeState ps{0u, 0u, 0u};
  if (threadIdx.x < 64) sh.complete[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    sh.smem_cap = PIPE_BYTES;
    sh.tracing = a.trace != nullptr;
    sh.vcta = blockIdx.x;
#ifdef MT_CR
    // f4 co-residency: the home table is laid out per (slot, SM) so the host can pair tenants of
    // different kinds on one SM; the slot is this CTA's arrival order on its SM
    const uint32_t sm = sm_id();
    const int nsm = gridDim.x / 2;
    const int slot = sm < 256 ? atomicAdd(&a.ctl->smslot[sm], 1) : 2;
    if (slot < 2 && (int)sm < nsm) sh.vcta = slot * nsm + (int)sm;
    else atomicExch(&a.ctl->error, 4u);   // SM ids outside [0, #SMs): no (slot, SM) home layout
#endif
  }
  if (a.claim_depth != 0)
    for (int i = threadIdx.x; i < a.n_ops; i += blockDim.x) sh.gate[i] = (int16_t)__ldg(a.gates + i);
  cta_setup(sh, true);
  bool ok = grid_barrier(a, sh);
  if (ok) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.ts) a.ts[0] = gtimer();
    // prologue: pack every distinct graph input (grid-stride over all threads)
    const int64_t first = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int q = 0; q < a.n_pack; ++q) {
      const int t = a.pack_tenant[q];
      if (a.in_prec[t] == 1) pack_pixels<float>(a, t, first, stride);
      else pack_pixels<bf16>(a, t, first, stride);
    }
    fence_proxy_async_global();   // packed input (generic stores) is read by the stems' TMA
    ok = grid_barrier(a, sh);
    if (ok && blockIdx.x == 0 && threadIdx.x == 0 && a.ts && a.ts_full) a.ts[2] = gtimer();
  }
  for (int s = 0; ok && s < a.n_stages; ++s) {
    ok = run_stage<F32>(a, s, smem, sh, ps);
    if (ok) ok = grid_barrier(a, sh);
    if (ok && blockIdx.x == 0 && threadIdx.x == 0 && a.ts && a.ts_full) a.ts[3 + s] = gtimer();
  }
  if (ok) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.ts) a.ts[1] = gtimer();
  }
  if (ok && !a.no_reset) {
    // all tiles of the run are complete: reset the claim / done counters for the next launch
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_ops; i += gridDim.x * blockDim.x) {
      a.claim[i] = 0;
      a.done[i] = 0;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_blk; i += gridDim.x * blockDim.x)
      a.blkcnt[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x < MT_MAXT) a.ctl->gcur[threadIdx.x] = 0;
  }
#ifdef MT_CR
  if (threadIdx.x == 0) {
    const uint32_t sm = sm_id();
    if (sm < 256) atomicSub(&a.ctl->smslot[sm], 1);
  }
#endif
  cta_teardown(sh, true);
}

// baseline: tiles [t0, t1) of one op, grid-strided.  Split-K ops are issued as two launches
// (partials, then the reduce tiles), so no tile of a non-cooperative launch waits on another
// CTA of the same launch.
template <bool F32>
__global__ void __launch_bounds__(MT_NTHREADS, 1) op_kernel(RunArgs a, int op, int t0, int t1) {
  uint8_t *smem = smem_base();
  __shared__ __align__(16) CtaShared sh;
  PipeState ps{0u, 0u, 0u};
  load_desc(sh, a.ops + op);
  if (threadIdx.x == 0) { sh.smem_cap = PIPE_BYTES; sh.tracing = a.trace != nullptr; }
  const bool tc = __ldg(&a.ops[op].tk) == TK_CONV_TC;
  cta_setup(sh, tc);
  for (int t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
    if (threadIdx.x == 0) { sh.t_pick = gtimer(); sh.t_mma = 0; sh.home = -1; }
    tile_prefetch(sh.d, t, smem, sh, ps);
    if (threadIdx.x == 0) sh.t_deps = gtimer();
    __syncthreads();
    run_tile<F32>(a, sh.d, t, smem, sh, ps);
    if (threadIdx.x == 0 && sh.xrel) {   // split-K partial arrival (the reduce launch checks it)
      fence_acq_rel_gpu();
      red_relaxed_add(sh.xrel, 1);
      sh.xrel = nullptr;
    }
    if (threadIdx.x == 0) trace_tile(a, sh, op, t);
  }
  cta_teardown(sh, tc);
}

// small-smem variant for non-tensor-core ops so several op kernels can share an SM
static constexpr int SMALL_SMEM = 47 * 1024;   // <= 48 KB: no opt-in needed; 46 KB usable after alignment
template <bool F32>
__global__ void __launch_bounds__(MT_NTHREADS) op_kernel_small(RunArgs a, int op) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(16) CtaShared sh;
  PipeState ps{0u, 0u, 0u};
  load_desc(sh, a.ops + op);
  if (threadIdx.x == 0) { sh.smem_cap = SMALL_SMEM - 1024; sh.xrel = nullptr; sh.tracing = a.trace != nullptr; }
  __syncthreads();
  for (int t = blockIdx.x; t < sh.d.tiles; t += gridDim.x) {
    if (threadIdx.x == 0) { sh.t_pick = gtimer(); sh.t_mma = 0; sh.home = -1; }
    tile_prefetch(sh.d, t, smem, sh, ps);
    if (threadIdx.x == 0) sh.t_deps = gtimer();
    __syncthreads();
    run_tile<F32>(a, sh.d, t, smem, sh, ps);
    if (threadIdx.x == 0) trace_tile(a, sh, op, t);
  }
}

__global__ void pack_kernel(RunArgs a, int t) {
  const int64_t first = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (a.in_prec[t] == 1) pack_pixels<float>(a, t, first, stride);
  else pack_pixels<bf16>(a, t, first, stride);
}

// bind-time weight repack from the caller's fp32 PyTorch layouts
__global__ void weight_pack_kernel(int mode, const float *src, void *dst, OpDesc d, int cin_real) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (mode == 1 || mode == 2) {  // conv [Cout][Cin][kh][kw] -> [rows][K] with K = (r, s, c)
    const int rows = mode == 1 ? d.tiles_n * d.bn : d.Co;
    const int ld = mode == 1 ? d.Kpad : d.K;
    const int64_t total = (int64_t)rows * ld;
    for (int64_t i = tid; i < total; i += stride) {
      const int row = (int)(i / ld), k = (int)(i - (int64_t)row * ld);
      float v = 0.f;
      if (row < d.Co && k < d.K) {
        const int tap = k / d.C, ci = k - tap * d.C;
        const int r = tap / d.kw, s = tap - r * d.kw;
        if (ci < cin_real) v = src[(((int64_t)row * cin_real + ci) * d.kh + r) * d.kw + s];
      }
      if (mode == 1) reinterpret_cast<bf16 *>(dst)[i] = __float2bfloat16_rn(v);
      else reinterpret_cast<float *>(dst)[i] = v;
    }
  } else if (mode == 5) {  // conv for the TMA mainloop: K = (tap, 64-channel blocks), zero padded
    const int rows = d.tiles_n * d.bn;
    const int ld = d.Kpad, per_tap = d.cblks * 64;
    const int64_t total = (int64_t)rows * ld;
    for (int64_t i = tid; i < total; i += stride) {
      const int row = (int)(i / ld), k = (int)(i - (int64_t)row * ld);
      const int tap = k / per_tap, ci = k - tap * per_tap;
      const int r = tap / d.kw, s2 = tap - r * d.kw;
      float v = 0.f;
      if (row < d.Co && ci < cin_real) v = src[(((int64_t)row * cin_real + ci) * d.kh + r) * d.kw + s2];
      reinterpret_cast<bf16 *>(dst)[i] = __float2bfloat16_rn(v);
    }
  } else if (mode == 3) {  // depthwise [C][1][kh][kw] -> [kh*kw][C]
    const int64_t total = (int64_t)d.kh * d.kw * d.C;
    for (int64_t i = tid; i < total; i += stride) {
      const int tap = (int)(i / d.C), ch = (int)(i - (int64_t)tap * d.C);
      const float v = src[(int64_t)ch * d.kh * d.kw + tap];
      // bf16 graphs: the weight value is rounded to bf16 (as every conv weight), stored as fp32
      reinterpret_cast<float *>(dst)[i] = d.prec == 0 ? __bfloat162float(__float2bfloat16_rn(v)) : v;
    }
  } else if (mode == 4) {  // FC [out][C*H*W] (NCHW flatten) -> [out][H*W*C] (NHWC flatten)
    const int64_t total = (int64_t)d.Co * d.K;
    const int HW = d.H * d.W;
    for (int64_t i = tid; i < total; i += stride) {
      const int row = (int)(i / d.K), k = (int)(i - (int64_t)row * d.K);
      const int pix = k / d.C, ci = k - pix * d.C;
      float v = 0.f;
      if (ci < cin_real) v = src[(int64_t)row * cin_real * HW + (int64_t)ci * HW + pix];
      if (d.prec == 0) reinterpret_cast<bf16 *>(dst)[i] = __float2bfloat16_rn(v);
      else reinterpret_cast<float *>(dst)[i] = v;
    }
  }
}

// ------------------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------------------
size_t executor_smem_bytes() { return SMEM_BYTES; }

static cudaError_t set_attrs() {
  static bool done = false;
  if (done) return cudaSuccess;
  for (auto f : {executor_kernel<true>, executor_kernel<false>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    // the whole unified L1/shared array as shared memory (2 CTAs/SM need 2 x ~107 KB)
    e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e;
  for (auto f : {op_kernel<true>, op_kernel<false>}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  for (auto f : {op_kernel_small<true>, op_kernel_small<false>}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM);
    if (e != cudaSuccess) return e;
  }
  done = true;
  return cudaSuccess;
}

cudaError_t executor_occupancy(int *bps) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
#ifdef MT_CR
  // the runtime's occupancy calculator reports 1 CTA/SM for every kernel containing tcgen05
  // instructions (tools/occ_probe.cu: even a 4-register kernel), while the hardware runs two per
  // SM (same probe: 296 CTAs allocating TMEM, 148 same-SM pairs overlapping).  Count the resources
  // instead: registers (allocated per thread in multiples of 8) and shared memory.
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, executor_kernel<false>);
  if (e != cudaSuccess) return e;
  int dev = 0, smem_sm = 0, regs_sm = 0, resv = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  const int by_regs = regs_sm / (((fa.numRegs + 7) / 8 * 8) * MT_NTHREADS);
  const int by_smem = smem_sm / ((int)fa.sharedSizeBytes + SMEM_BYTES + resv);
  *bps = by_regs < by_smem ? by_regs : by_smem;
  return cudaSuccess;
#else
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, executor_kernel<false>, MT_NTHREADS, SMEM_BYTES);
#endif
}

// resource summary of the bf16 executor (diagnostics of the co-residency check)
int executor_resources(char *buf, int n) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, executor_kernel<false>) != cudaSuccess) return 0;
  int dev = 0, smem_sm = 0, regs_sm = 0, smem_blk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&smem_blk, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  int o1 = -1, o2 = -1, o3 = -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, executor_kernel<false>, MT_NTHREADS, 80 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, executor_kernel<false>, MT_NTHREADS, 32 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, executor_kernel<false>, MT_NTHREADS, 0);
  return snprintf(buf, n, "regs %d static smem %zu dyn %d (max dyn %d) local %zu; SM: smem %d regs %d reserved/blk %d; "
                  "occ at 80K/32K/0 dyn: %d %d %d",
                  fa.numRegs, fa.sharedSizeBytes, SMEM_BYTES, fa.maxDynamicSharedSizeBytes, fa.localSizeBytes, smem_sm,
                  regs_sm, smem_blk, o1, o2, o3);
}

cudaError_t launch_executor(const RunArgs &a, int grid, cudaStream_t s) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&a};
  bool f32 = false;
  for (int t = 0; t < a.n_tenants; ++t) f32 |= a.in_prec[t] == 1;
#ifdef MT_CR
  // 2 CTAs/SM: cudaLaunchCooperativeKernel applies the calculator's 1-CTA/SM limit to tcgen05 kernels
  // (see executor_occupancy), so this build launches normally; the grid fits the GPU by the resource
  // count, and a CTA that could not become resident would end the run by the grid-barrier timeout
  // (MT_ERR_INTERNAL), never hang it
  (void)args;
  if (f32) executor_kernel<true><<<grid, MT_NTHREADS, SMEM_BYTES, s>>>(a);
  else executor_kernel<false><<<grid, MT_NTHREADS, SMEM_BYTES, s>>>(a);
  return cudaGetLastError();
#else
  return cudaLaunchCooperativeKernel(f32 ? (void *)executor_kernel<true> : (void *)executor_kernel<false>,
                                     dim3(grid), dim3(MT_NTHREADS), args, SMEM_BYTES, s);
#endif
}

cudaError_t launch_op(const RunArgs &a, const OpDesc &d, int op, int max_grid, cudaStream_t s) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  if (d.tk == TK_CONV_TC) {
    const int nc = d.splits > 1 ? d.tiles_m * d.tiles_n * d.splits : d.tiles;   // compute tiles
    for (int part = 0; part < 2; ++part) {
      const int t0 = part ? nc : 0, t1 = part ? d.tiles : nc;
      if (t1 <= t0) continue;
      const int grid = t1 - t0 < max_grid ? t1 - t0 : max_grid;
      if (d.prec == 1) op_kernel<true><<<grid, MT_NTHREADS, SMEM_BYTES, s>>>(a, op, t0, t1);
      else op_kernel<false><<<grid, MT_NTHREADS, SMEM_BYTES, s>>>(a, op, t0, t1);
    }
  } else {
    const int cap = 4 * max_grid;
    const int grid = d.tiles < cap ? d.tiles : cap;
    if (d.prec == 1) op_kernel_small<true><<<grid, MT_NTHREADS, SMALL_SMEM, s>>>(a, op);
    else op_kernel_small<false><<<grid, MT_NTHREADS, SMALL_SMEM, s>>>(a, op);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack(const RunArgs &a, int t, cudaStream_t s) {
  const int64_t pix = (int64_t)a.in_n[t] * a.in_h[t] * a.in_w[t];
  int grid = (int)((pix + 255) / 256);
  if (grid > 1184) grid = 1184;
  pack_kernel<<<grid, 256, 0, s>>>(a, t);
  return cudaGetLastError();
}

cudaError_t launch_weight_pack(int mode, const float *src, void *dst, const OpDesc &d, int cin_real,
                               cudaStream_t s) {
  weight_pack_kernel<<<1184, 256, 0, s>>>(mode, src, dst, d, cin_real);
  return cudaGetLastError();
}

}  // namespace MT_NS
