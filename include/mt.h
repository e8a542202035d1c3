/*
 * mt.h -- C ABI of the B200 multi-tenant stage-schedule executor (libmt.so).
 *
 * Implements the computation the scheduler of Yu et al., "Automated Runtime-Aware Scheduling
 * for Multi-Tenant DNN Inference on GPU" (arXiv 2111.14255, /root/reference/PAPER.md) speeds
 * up: executing a multi-tenant schedule.  Citations P:n are PAPER.md line numbers.
 *
 *   problem   N independent DNN models sharing one input; objective = latency "from the
 *             earliest starting time of the tasks to the latest ending time"
 *   IR        each model = one operator sequence (Eq.1); pointers split it
 *             (Eq.3); a stage = one slice per model, possibly empty ("None",
 *             Eq.4/5); "all operators in the same stage must all finish so as to
 *             step into the next stage"; schedule = ordered stage list (Eq.6,
 *             P:334-341); pointer matrix rho[N][P] -> schedule via T(G, rho) (Eq.8)
 *   cost      "profile the latency by multiple runs" (Alg.1 L8); "the averaged latency
 *             is then used as the cost"; infeasible candidates are "filtered out"
 *
 * Conventions (readings R1-R4): operators are 0-based; a slice is a half-open range
 * [begin, end) and begin == end is the paper's "None"; pointer p = barrier after op p, so
 * slice k of tenant i is [rho_i[k-1], rho_i[k]) with rho_i[-1] = 0, rho_i[P] = L_i; every
 * row of rho has the same P (P+1 stages); an all-empty stage is infeasible.
 *
 * Ownership: the caller owns every device buffer (weights, scale/shift, inputs, outputs and the
 * workspace, all allocated e.g. by torch).  The library copies host arrays before returning,
 * never frees caller memory and allocates only host-side plan state and CUDA events/streams.
 * Weights/scale/shift pointers are borrowed from mt_load_graphs until mt_destroy or the next
 * mt_load_graphs; weights are repacked into the workspace by mt_bind_workspace.
 *
 * Errors: every call returns mt_status.  MT_ERR_VALIDATION carries mt_error_info (the first
 * violation, stage-major then tenant-minor scan).  A failed mt_set_schedule* leaves the
 * previous schedule active.  Device-side spin timeouts return MT_ERR_INTERNAL.
 * MT_ERR_REFUSED = the cooperative grid cannot be co-resident.  A context is not thread-safe.
 */
#ifndef MT_H_
#define MT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mt_ctx mt_ctx;

typedef enum {
  MT_OK = 0,
  MT_ERR_INTERNAL = 1,   /* device timeout / broken invariant                         */
  MT_ERR_VALIDATION = 2, /* infeasible schedule; see mt_last_error_info        */
  MT_ERR_REFUSED = 3,    /* cooperative grid not co-resident, or no device             */
  MT_ERR_CUDA = 4,       /* a CUDA runtime call failed (message in mt_last_error)      */
  MT_ERR_ARG = 5,        /* bad argument / unsupported graph                           */
  MT_ERR_STATE = 6       /* call out of order (e.g. run before bind / schedule)        */
} mt_status;

/* schedule-IR violation codes (mt_error_info.code); identical to oracle/ir.py */
typedef enum {
  MT_E_OK = 0,
  MT_E_SHAPE = 1,       /* wrong number of tenants / rows, or zero stages           */
  MT_E_RANGE = 2,       /* begin < 0, end > L_i or begin > end                       */
  MT_E_NONCONTIG = 3,   /* begin != previous end of that tenant (gap / overlap)      */
  MT_E_EMPTY_STAGE = 4, /* every slice of a stage is empty                           */
  MT_E_INCOMPLETE = 5,  /* a tenant's last end != L_i                                */
  MT_E_ROW_ORDER = 6,   /* pointer row decreasing                                    */
  MT_E_ROW_RANGE = 7    /* pointer outside [0, L_i]                                  */
} mt_ir_error;

typedef struct {
  int32_t code, stage, tenant, op; /* -1 where not applicable */
} mt_error_info;

/* operator kinds of a tenant graph (the paper's conv/bn/relu/pooling...) */
typedef enum {
  MT_CONV = 1,            /* conv -> y*scale+shift (+residual) -> act; groups 1 or depthwise */
  MT_BN = 2,              /* y = act(x*scale + shift)                                        */
  MT_RELU = 3,            /* y = act(x)                                                      */
  MT_MAXPOOL = 4,         /* kh x kw window, stride, padding, ceil_mode                      */
  MT_AVGPOOL = 5,         /* + count_include_pad                                             */
  MT_GLOBAL_AVGPOOL = 6,  /* mean over H x W                                                 */
  MT_FC = 7,              /* y = act(scale * (W x) + shift), x = NCHW flatten of the input   */
  MT_ADD = 8              /* y = act(sum of inputs)                                          */
} mt_op_kind;

typedef enum { MT_ACT_NONE = 0, MT_ACT_RELU = 1, MT_ACT_RELU6 = 2 } mt_act;
typedef enum { MT_PREC_BF16 = 0, MT_PREC_FP32 = 1 } mt_precision;

#define MT_MAX_INPUTS 8
#define MT_MAX_TENANTS 16

typedef struct {
  int32_t kind;                    /* mt_op_kind                                          */
  int32_t n_inputs;                /* 1..MT_MAX_INPUTS                                    */
  int32_t inputs[MT_MAX_INPUTS];   /* node ids < own id, -1 = the graph input. n_inputs>1: */
                                   /* channel concat (CONV/POOLs/FC) or sum (ADD)          */
  int32_t out_c, out_h, out_w;     /* checked against shape inference                    */
  int32_t kh, kw, sh, sw, ph, pw;  /* window / stride / padding (CONV, pools)            */
  int32_t groups;                  /* CONV: 1 or == in_c == out_c (depthwise)             */
  int32_t ceil_mode, count_include_pad;
  int32_t act;                     /* mt_act                                               */
  int32_t residual;                /* CONV: node id added before act, or -1               */
  const float *weight;             /* DEVICE fp32. CONV [Cout][Cin/groups][kh][kw];        */
                                   /* FC [out][in], in = NCHW flatten index of the input   */
  const float *scale, *shift;      /* DEVICE fp32 [out_c] (CONV/BN/FC), else NULL          */
} mt_node;

typedef struct {
  int32_t n_nodes;
  const mt_node *nodes;            /* host array, copied by mt_load_graphs                 */
  int32_t batch, in_c, in_h, in_w; /* graph input NCHW fp32 [batch][in_c][in_h][in_w]      */
  int32_t precision;               /* mt_precision: activation storage; bf16 convs run on  */
                                   /* tcgen05 tensor cores with fp32 accumulation          */
} mt_graph;

/* options for mt_set_option */
typedef enum {
  MT_OPT_STEAL = 1,        /* 0: strict per-tenant SM partition; 1: when its home tenant's  */
                           /* slice is fully claimed a CTA helps the others, round-robin;   */
                           /* 2 (default): ... the tenant with most unclaimed ops first     */
  MT_OPT_NUM_SMS = 2,      /* host-only contexts: SM count used for the partition (148)    */
  MT_OPT_TIMEOUT_MS = 3,   /* device spin timeout (default 2000 ms)                         */
  MT_OPT_CTAS_PER_SM = 4,  /* 1 (default): one 256-thread executor CTA per SM, 192 KB conv  */
                           /* ring.  2: heterogeneous co-residency:  */
                           /* two 128-thread CTAs per SM (96 KB ring, 256 TMEM columns      */
                           /* each); slot 0 of every SM serves the stage's SM partition from */
                           /* the most to the least compute-intense tenant, slot 1 the same  */
                           /* list reversed, pairing compute- and memory-bound slices on one */
                           /* SM.  Plans depend on it: set before mt_load_graphs           */
                           /* (MT_ERR_STATE after); bf16 tenants only (MT_ERR_REFUSED at     */
                           /* load for fp32); MT_ERR_REFUSED if the build does not fit.     */
  MT_OPT_PARTITION = 5,    /* SM partition rule per stage (a3; R16 / R16b):       */
                           /* 0 (default): n_t proportional to the slice's roofline time    */
                           /*    (north star); 1: latency-balanced -- minimise max_t E_t,   */
                           /*    E_t(n) = sum over the slice's work items ceil(tiles/n)*ns  */
                           /*    (mt_op_work); 2: work/span, E_t(n) = ceil(W_t/n) + S_t.    */
                           /*    Setting it re-plans the active schedule.                   */
  MT_OPT_CLAIM_DEPTH = 6,  /* 0 (default): a CTA may claim any tile of its tenant's slice     */
                           /* (claim-then-wait).  D > 0: a tile of op o is claimable only   */
                           /* once o's ancestors at DAG distance D are complete; D < 0: once */
                           /* op o-|D| of the same tenant is complete (bounded claim-ahead: */
                           /* CTAs blocked everywhere retry instead of parking on a tile)   */
  MT_OPT_STAGE_SPLIT = 7   /* 1: mt_run / mt_run_async launch the executor once per stage (the */
                           /* kernel boundary replaces the grid barrier) so a profiler       */
                           /* attributes counters per stage; debug/profiling only (launch    */
                           /* gaps between stages); 0 (default): one cooperative launch      */
} mt_option;

/* execution modes of mt_run_baseline: the same tile functions launched one kernel per op */
typedef enum {
  MT_BASE_SEQ = 1,          /* one stream, tenant-major op order ("CuDNN-Seq" analogue)   */
  MT_BASE_MS_DFS = 2,       /* one stream per tenant, issued stream by stream     */
  MT_BASE_MS_BFS = 3,       /* one stream per tenant, round-robin issue           */
  MT_BASE_SEQ_GRAPH = 4,    /* SEQ captured in a CUDA graph                                */
  MT_BASE_MS_GRAPH = 5,     /* MS_BFS captured in a CUDA graph                             */
  MT_BASE_STAGE_EVENTS = 6  /* the paper's mechanism: per-tenant streams, BFS issue of each */
                            /* stage's ops, cross-stream event barrier after every stage   */
} mt_base_mode;

/* device >= 0: CUDA device ordinal.  device == -1: host-only plan context (IR, validation,
 * stage assignment, SM partition; no CUDA call is ever made). */
mt_status mt_create(int device, mt_ctx **out);
mt_status mt_destroy(mt_ctx *ctx);
mt_status mt_set_option(mt_ctx *ctx, int32_t option, int64_t value);

/* Ingest N tenant DAGs (a1).  Checks topological order (inputs < own id), shape inference
 * against out_c/out_h/out_w, concat groupings (a producer may belong to one concat group
 * only), channel counts of consumed tensors (multiples of 8).  Node order = the model's
 * operator sequence (Eq.1).  Invalidates any bound workspace and schedule. */
mt_status mt_load_graphs(mt_ctx *ctx, int32_t n_tenants, const mt_graph *graphs);
mt_status mt_op_count(mt_ctx *ctx, int32_t tenant, int32_t *n_ops);
/* algorithmic FLOPs (2*MACs of conv/FC) and bytes (inputs+weights+residual+output at the
 * storage element size) of one op -- the roofline / SM-partition inputs (SURVEY d.4) */
mt_status mt_op_cost(mt_ctx *ctx, int32_t tenant, int32_t op, int64_t *flops, int64_t *bytes);
/* number of work tiles an op is split into (shape-only, identical for every schedule) */
mt_status mt_op_tiles(mt_ctx *ctx, int32_t tenant, int32_t op, int32_t *tiles);
/* How an op is executed (introspection for tests and tuning; shape + mix only, identical for
 * every schedule).  plan[MT_PLAN_LEN] receives: [0] kernel kind (MT_PLAN_KIND_*), [1] operand
 * path of a tensor-core op (0 cp.async im2col, 1 TMA im2col, 2 TMA 8-channel stem, 3 TMA FC),
 * [2] N tile (bn), [3] split-K factor, [4] M tiles, [5] N tiles, [6] pipeline stages,
 * [7] total tiles (compute + split-K reduce), [8] column segments per output row. */
#define MT_PLAN_LEN 9
#define MT_PLAN_KIND_CONV_TC 0
#define MT_PLAN_KIND_CONV_SIMT 1
#define MT_PLAN_KIND_DW 2
#define MT_PLAN_KIND_POOL 3
#define MT_PLAN_KIND_GAP 4
#define MT_PLAN_KIND_FC 5
#define MT_PLAN_KIND_ELT 6
mt_status mt_op_plan(mt_ctx *ctx, int32_t tenant, int32_t op, int32_t *plan);
/* Latency model of one op (input of the MT_OPT_PARTITION = 1 rule; shape + mix only):
 * tiles[2] = compute tiles, split-K reduce tiles (0 without split-K); ns[2] = estimated
 * nanoseconds of one tile of each (calibrated on device traces).
 * Host arrays of 2 elements, written on MT_OK; MT_ERR_STATE before mt_load_graphs. */
mt_status mt_op_work(mt_ctx *ctx, int32_t tenant, int32_t op, int32_t *tiles, int64_t *ns);

/* Device workspace: packed weights, activations, split-K partials, counters, plans. */
mt_status mt_workspace_size(mt_ctx *ctx, size_t *bytes);
/* dev_ptr: caller-allocated device memory >= mt_workspace_size, 256-byte aligned.  Repacks
 * the weights (synchronously) and zeroes the counters. */
mt_status mt_bind_workspace(mt_ctx *ctx, void *dev_ptr, size_t bytes);

/* Schedule tau in stage form (Eq.6): ranges[S][N][2] = (begin, end) per stage and tenant. */
mt_status mt_set_schedule(mt_ctx *ctx, int32_t n_stages, const int32_t *ranges);
/* Schedule in pointer form rho[N][P] (Eq.8); builds tau = T(G, rho) and sets it. */
mt_status mt_set_schedule_pointers(mt_ctx *ctx, int32_t P, const int32_t *rho);
mt_status mt_num_stages(mt_ctx *ctx, int32_t *n_stages);
/* copy of the active stage table: ranges[S][N][2] */
mt_status mt_get_schedule(mt_ctx *ctx, int32_t *ranges);
/* stage_of[concat_i L_i]: stage index of op j of tenant i */
mt_status mt_stage_assignment(mt_ctx *ctx, int32_t *stage_of);
/* sms[S][N]: CTAs whose home queue is tenant i in stage s (runtime-aware partition, a3;
 * rule chosen by MT_OPT_PARTITION; every active tenant >= 1, inactive 0, sum = #SMs) */
mt_status mt_sm_partition(mt_ctx *ctx, int32_t *sms);
/* *grid = executor CTAs per launch (#SMs x MT_OPT_CTAS_PER_SM); homes[S][grid] (may be NULL to
 * query the grid): the home tenant of every CTA per stage.  1 CTA/SM: CTA index; 2 CTAs/SM: index
 * slot * #SMs + SM id, slot 0 listing the partition from the most to the least compute-intense
 * tenant (FLOP/byte of the stage slice), slot 1 the same list reversed (f4 pairing). */
mt_status mt_stage_homes(mt_ctx *ctx, int32_t *grid, int32_t *homes);

/* Run the active schedule once on the persistent stage executor (one launch: cooperative with 1
 * CTA/SM; with MT_OPT_CTAS_PER_SM = 2 a normal launch of a grid whose co-residency was checked by
 * resource count at mt_set_option -- a CTA that could not become resident ends the run through the
 * grid-barrier timeout with MT_ERR_INTERNAL).
 * inputs[N]: DEVICE fp32 NCHW graph inputs (may alias: the shared input of P:240).
 * outputs[N]: DEVICE fp32 [batch][out_c*out_h*out_w] (NHWC flatten; [batch][classes]).
 * stage_us[S] (host, may be NULL): device time of each stage (%globaltimer deltas).
 * total_us (host, may be NULL): makespan, first stage start -> last barrier,
 * including the input-pack prologue.  stream: cudaStream_t (NULL = legacy default).
 * Synchronous: returns after the run completed. */
mt_status mt_run(mt_ctx *ctx, const float *const *inputs, float *const *outputs,
                 float *stage_us, float *total_us, void *stream);
/* Same, asynchronous: enqueue only (no timing read-back, no sync). */
mt_status mt_run_async(mt_ctx *ctx, const float *const *inputs, float *const *outputs,
                       void *stream);
/* End-to-end variant with HOST buffers: copies inputs (pinned or pageable host memory,
 * identical pointers copied once) to device staging in the workspace, runs, copies outputs
 * back.  Synchronous. */
mt_status mt_run_host(mt_ctx *ctx, const float *const *host_inputs, float *const *host_outputs,
                      float *total_us, void *stream);

/* Baselines: the same tile functions launched one kernel per op (mt_base_mode).  total_us =
 * cudaEvent makespan.  STAGE_EVENTS uses the active schedule.  Synchronous. */
mt_status mt_run_baseline(mt_ctx *ctx, int32_t mode, const float *const *inputs,
                          float *const *outputs, float *total_us, void *stream);

/* Profile candidate schedules (a10, Alg.1 L7-L9): for each candidate, `warmup` untimed and
 * `iters` timed runs of the executor; lat_us[c] = mean device makespan of the timed runs.
 * status[c] = MT_OK, or MT_ERR_VALIDATION with lat_us[c] = NaN (filtered out).
 * Stage form: cand_nstages[n], cand_ranges = concatenation of [S_c][N][2] blocks.
 * The active schedule is left unchanged.  Synchronous. */
mt_status mt_profile_batch(mt_ctx *ctx, int32_t n_cand, const int32_t *cand_nstages,
                           const int32_t *cand_ranges, const float *const *inputs,
                           float *const *outputs, int32_t warmup, int32_t iters,
                           float *lat_us, int32_t *status, void *stream);
/* Pointer form: cand_P[n], cand_rho = concatenation of [N][P_c] blocks. */
mt_status mt_profile_batch_pointers(mt_ctx *ctx, int32_t n_cand, const int32_t *cand_P,
                                    const int32_t *cand_rho, const float *const *inputs,
                                    float *const *outputs, int32_t warmup, int32_t iters,
                                    float *lat_us, int32_t *status, void *stream);

/* Analytic schedule-cost estimate: a cheap PRE-FILTER for candidate schedules,
 * never the cost itself -- the paper rejects modeling-based costs as inaccurate and profiles
 * (P:433-441); candidates that survive the filter are profiled with mt_profile_batch*.  Model
 * (the contention form of SPEC.md cost_model S:229-239 plus a fixed per-op dependent-hop latency,
 * DESIGN.md reading R19): per op j, roof_j = max(F_j/peak_flops, B_j/mem_bw) with F, B from
 * mt_op_cost; an op is compute-bound iff F_j/peak_flops >= B_j/mem_bw.  Per stage:
 *   chain_i = sum over tenant i's slice of (roof_j + op_latency_us)
 *   compute = (sum F of compute-bound ops / peak_flops) * (1 + c_compute * max(0, n_c - 1) / max_concurrency)
 *   memory  = (sum B of memory-bound ops / mem_bw)     * (1 + c_memory  * max(0, n_m - 1) / max_concurrency)
 *   stage   = max(compute, memory, max_i chain_i) + sync_us
 * (n_c / n_m = tenants whose slice holds a compute- / memory-bound op); est = sum of stages, us.
 * Host-only: works on a host-only context (no GPU).  Pointer form as mt_profile_batch_pointers;
 * status[c] = MT_OK or MT_ERR_VALIDATION (est_us[c] = NaN). */
typedef struct mt_cost_params {
  double peak_flops;       /* FLOP/s */
  double mem_bw;           /* bytes/s */
  double op_latency_us;    /* fixed latency of one dependent op hop */
  double sync_us;          /* per-stage barrier */
  double c_compute, c_memory;
  int32_t max_concurrency; /* >= 1 */
} mt_cost_params;
mt_status mt_estimate_batch_pointers(mt_ctx *ctx, const mt_cost_params *params, int32_t n_cand,
                                     const int32_t *cand_P, const int32_t *cand_rho, double *est_us,
                                     int32_t *status);

/* Debug: copy op `op` of tenant `tenant`'s activation (NHWC, storage precision, channels
 * [0, out_c) of its row) from the last run to host.  bytes must equal
 * batch*out_h*out_w*out_c*elem.  The graph's final op has no activation buffer. */
mt_status mt_get_activation(mt_ctx *ctx, int32_t tenant, int32_t op, void *host_dst,
                            size_t bytes);

/* Debug tracing: when enabled, every executed tile appends one record of 16 uint64 to
 * the caller's DEVICE buffer: [0] op | tile << 32 (global op id), [1] smid | cta << 32,
 * [2] claim time, [3] dependencies satisfied, [4] tensor-core mainloop done (0 if none),
 * [5] tile end (after the release), [6] home tenant of the CTA (-1 in baselines), [7] tile body
 * done (before the release), [8] first pipeline stage landed, [9] last MMA issued, [10] last
 * A box issued (TMA convs; else 0), [11..15] 0; times are %globaltimer ns.
 * capacity = records; 0 / NULL disables.  Resets the record counter. */
mt_status mt_set_trace(mt_ctx *ctx, void *dev_buf, int64_t capacity);
mt_status mt_trace_count(mt_ctx *ctx, int64_t *n_records);

mt_status mt_last_error_info(mt_ctx *ctx, mt_error_info *info);
const char *mt_last_error(mt_ctx *ctx);
/* static build/version string */
const char *mt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MT_H_ */
