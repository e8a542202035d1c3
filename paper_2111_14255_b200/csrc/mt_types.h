// Plan structures shared by the host plan compiler (plan.cpp) and the device code (kernels.cu).
// Plain-old-data only: uploaded to device memory as-is.
#pragma once
#include <stdint.h>

#define MT_MAXT 16        // max tenants (== MT_MAX_TENANTS)
#define MT_MAXIN 8        // max inputs of one op (== MT_MAX_INPUTS)
#define MT_MAXDEP 9       // inputs + residual
// Device-code configuration.  kernels.cu is compiled twice:
//  * default: one 256-thread CTA per SM with a 192 KB conv ring (namespace mtk);
//  * MT_CR (kernels_cr.cu, MT_OPT_CTAS_PER_SM = 2): two co-resident 128-thread CTAs per SM, each
//    with a 96 KB ring, 255 registers per thread (2 x 128 x 256 = the whole register file) and 256
//    TMEM columns (namespace mtk_cr).
// The host plans with the values of the configuration the context runs (mt_ctx::dev).
#define MT_PIPE_BYTES_1 (192 * 1024)   // ring of the 1-CTA-per-SM configuration (host planning)
#ifndef MT_PIPE_BYTES_2
#define MT_PIPE_BYTES_2 (96 * 1024)    // ring of the 2-CTA-per-SM configuration
#endif
#ifdef MT_CR
#define MT_NTHREADS 128   // threads per CTA of every kernel
#define MT_PIPE_BYTES MT_PIPE_BYTES_2  // shared-memory ring of the conv pipeline
#define MT_CTAS_PER_SM 2
#define MT_NS mtk_cr
#else
#define MT_NTHREADS 256
#define MT_PIPE_BYTES MT_PIPE_BYTES_1
#define MT_CTAS_PER_SM 1
#define MT_NS mtk
#endif
#define MT_STAGES 4       // smem pipeline depth of the cp.async conv mainloop (32 KB stages)
#define MT_MAXST 12       // max pipeline depth of the TMA conv mainloop (stage = A box + B box)
#define MT_BM 128         // tcgen05 conv tile rows (output pixels), UMMA M
#define MT_BK 64          // K per pipeline stage (one 128-byte swizzle atom of bf16)
#define MT_SIMT_BM 64     // SIMT conv tile
#define MT_SIMT_BN 64
#define MT_SIMT_BK 16
#define MT_EW_PER_THREAD 2   // 8-channel vectors per thread in pointwise tiles
#define MT_FC_ROWS (MT_NTHREADS / 32)   // FC output rows per tile (one per warp)
#define MT_GAP_G (MT_NTHREADS / 8)      // GAP: 8-channel groups per tile (8 threads each)
#define MT_FC_BATCH 8        // FC batch columns per pass
#define MT_GATE_OPS 2048     // bounded claim-ahead: gate table staged in shared memory (ops)

enum mt_tile_kind {
  TK_NONE = 0,
  TK_CONV_TC = 1,   // bf16 implicit GEMM on tcgen05 (UMMA 128 x BN x 16, fp32 accum in TMEM)
  TK_CONV_SIMT = 2, // fp32-accumulating implicit GEMM on CUDA cores (fp32 graphs)
  TK_DW = 3,        // depthwise conv on CUDA cores
  TK_POOL = 4,      // max / avg pooling
  TK_GAP = 5,       // global average pooling
  TK_FC = 6,        // GEMV / skinny GEMM (weight streaming)
  TK_ELT = 7        // ADD / BN / RELU
};

enum mt_op_flags {
  OPF_OUT = 1,          // final op: writes fp32 into the caller's output buffer
  OPF_RES = 2,          // fused residual
  OPF_GRAPH_IN = 4,     // reads the (packed) graph input of its tenant
};

struct OpDesc {
  int32_t kind, tk, tenant, prec;   // prec: 0 bf16, 1 fp32 storage
  int32_t flags, act, n_in, n_dep;
  int32_t N, H, W, C;               // input: batch, height, width, channels (stored, padded)
  int32_t Ho, Wo, Co, groups;
  int32_t kh, kw, sh, sw;
  int32_t ph, pw, ceil_mode, cip;
  int32_t in_cs, in_co, out_cs, out_co;
  int32_t res_cs, res_co, ins_cs[MT_MAXIN], ins_co[MT_MAXIN];
  int32_t deps[MT_MAXDEP];          // global op ids this op reads
  int32_t dep_kind[MT_MAXDEP];      // bit 0: read as input, bit 1: read as residual
  // completion tracking: output pixels (N*Ho*Wo, FC/GAP: batch index) are split into blocks of
  // pix_blk; block b of this op is complete when blkcnt[blk_off + b] == blk_need
  int32_t pix_blk, blk_need, nblk, blk_off;
  int32_t pix_tile;                 // pointwise tiles: output pixels per tile
  int32_t blk_rows;                 // >0: blocks are whole-row M-tiles (TMA conv): block of pixel p =
                                    //     n * blk_tpi + ho / blk_rows
  int32_t blk_tpi;                  // tiles (blocks) per image for blk_rows > 0
  int32_t nseg, seg_w;              // TMA: an output row wider than 128 is split into nseg column
                                    //     segments of seg_w pixels (one M tile each, blk_rows = 1);
                                    //     the nseg segment tiles of a row complete one block
  int32_t tma;                      // 1: TMA mainloop (whole-row M tiles, K-block = tap x 64 ch)
  int32_t cblks;                    // TMA: 64-channel blocks per tap
  int32_t a_bytes;                  // TMA: bytes of one A box (rows * Wo * 128)
  int32_t rc;                       // split-K: reduce tiles per (M,N) tile (32 columns each); the op's
                                    // tiles are [tmn*splits compute tiles][tmn*rc reduce tiles]
  int32_t nst;                      // conv pipeline: ring stages; bytes of one k-block's (A box + B box)
  int32_t st_bytes, st_boff, kg;    // sub-block, offset of B in it; kg = k-blocks per ring stage (one
                                    // full/empty barrier pair, expect_tx and commit per kg k-blocks)
  int32_t M, K, Kpad, nkb;          // GEMM view (conv / FC)
  int32_t bn, tiles_m, tiles_n, splits;
  int32_t kb_per_split, tiles, cnt_off, pad0;
  uint64_t in, res, out, w, scale, shift, ws;   // device addresses (filled at bind)
  uint64_t ins[MT_MAXIN];                        // ADD inputs
  uint64_t tmap_a, tmap_b;                       // TMA: device addresses of CUtensorMaps
};

// Device-side control block in the workspace (counters are zero between runs).
struct CtlBlock {
  unsigned int bar_count;
  unsigned int bar_gen;
  unsigned int error;        // nonzero: a spin timed out / invariant broken
  unsigned int trace_count;  // entries written to the trace buffer
  unsigned long long err_info;
  int gcur[MT_MAXT];         // per tenant: every op below is fully claimed (monotonic hint; reset per run)
  int smslot[256];           // 2 CTAs/SM: CTAs resident on SM i so far (slot counter; back to 0 at exit)
};

struct RunArgs {
  const OpDesc *ops;
  const int32_t *rng;        // [S][T][2] global op ids (begin, end)
  const uint8_t *home;       // [S][grid] home tenant of each CTA
  int32_t n_stages, n_tenants, steal, n_pack;
  int32_t claim_depth;       // 0: claim any tile of the slice; D: only ops whose gate ops are complete
  const int32_t *gates;      // [n_ops]: gate op of each op (-1 none), host table for claim_depth
  int32_t *claim;            // [n_ops] tile claim counters
  int32_t *done;             // [n_ops] completed-tile counters
  int32_t *blkcnt;           // [total blocks] completed-tile counters per output pixel block
  int32_t *splitcnt;         // split-K arrival counters
  CtlBlock *ctl;
  unsigned long long *ts;    // [n_stages + 2] %globaltimer stamps (or NULL)
  unsigned long long timeout_ns;
  int32_t n_ops, ts_full;
  int32_t no_reset;           // stage-split launches before the last: keep claim/done/block counters
  int32_t n_blk, trace_cap;
  unsigned long long *trace; // [trace_cap][8] per-tile records (debug; NULL = off)     // ts_full: 1 = all stage stamps, 0 = start/end only
  const float *inputs[MT_MAXT];     // per tenant user input (NCHW fp32)
  float *outputs[MT_MAXT];          // per tenant user output (fp32)
  uint64_t packed[MT_MAXT];         // per tenant packed-input buffer (NHWC, C padded)
  int32_t pack_tenant[MT_MAXT];     // tenants whose input is packed in the prologue
  int32_t in_n[MT_MAXT], in_c[MT_MAXT], in_h[MT_MAXT], in_w[MT_MAXT], in_cpad[MT_MAXT], in_prec[MT_MAXT];
};
