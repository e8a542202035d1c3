// libmt.so host runtime: C ABI (include/mt.h), graph ingest (a1), tile plans + stage plans (a3),
// workspace layout, executor / baseline / profiling launches (a4, a9, a10).
#include <cuda.h>  // CUtensorMap types only; the driver is reached via cudaGetDriverEntryPoint
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <map>
#include <string>
#include <limits>
#include <vector>

#include "kernels.h"
#include "plan.h"

using namespace mt;

static const int64_t BW_GBS = 8000;        // spec HBM GB/s (north star "8 TB/s")
static const int64_t TC_GFLOPS = 2250000;  // spec dense bf16 GFLOP/s (2.25 PFLOP/s)
// per-SM TMA operand bandwidth of the conv cost model, bytes per microsecond (calibrated on
// executor traces, tools/kb_rate.py).  Plans depend only on the op's shape
// and the mix's tenant count -- no environment input.
static constexpr double TMA_BPUS = 160000.0;
static const int64_t MT_HOP_NS = 2000;   // partition mode 2: dependency hop between ops (traces)
static constexpr int BN_MIN = 32;        // narrowest N tile the cost model considers
// K-blocks per ring stage of the TMA conv mainloop.  The producer and MMA-issuer loops run on one
// thread each, and per ring stage they pay a dependent chain of barrier probe, expect_tx / commit
// and descriptor moves of ~250 ns (tools/kb_pipe.cu, tools/loop_bisect.cu) -- more than the TMA
// transfer or the UMMAs of one 64-wide k-block at batch-1 tile sizes.  Grouping kg k-blocks under
// one barrier pair amortises that chain; kg = 2 is taken when it still leaves MT_KG_MIN_NST stages
// in the ring (kg = 4 measured the same end to end; each kg is one more mainloop instantiation).
// Only the pipeline's granularity changes: the UMMAs and their order are the same, so outputs are
// bit-identical for every kg.
#ifndef MT_KG_MIN_NST
#define MT_KG_MIN_NST 3
#endif
#ifndef MT_KG_MAX
#define MT_KG_MAX 2   // the device mainloop is instantiated for kg = 1 and 2
#endif
// The UMMA reads all 128 rows (16 KB) of an A sub-block even when the box holds fewer output
// pixels (e.g. 25 at 5x5): the rows past the box are discarded by the epilogue, but the read must
// stay inside the ring, so the last sub-block needs (16 KB - A region) bytes of slack behind it.
#ifndef MT_CR_PAIR
#define MT_CR_PAIR 1   // 2 CTAs/SM: slot 1 lists the partition reversed (0: same order, ablation)
#endif
#ifndef MT_KB_OVH
#define MT_KB_OVH 0.0   // cost model: us of issue-chain latency per ring stage (divided over its kg k-blocks)
#endif
static int ring_slack(int st_boff) { return std::max(0, MT_BM * 128 - st_boff); }
static int kgroup(int pipe, int st_bytes, int st_boff, int kb_per_split) {
  // the co-resident configuration's 96 KB ring groups down to 2 stages (same box: c4 b1 689 ->
  // 675 us, c3 639 -> 624 us; c4b8 unchanged); the 192 KB ring keeps >= 3 (2 measured neutral or
  // slower there)
  const int min_nst = pipe <= MT_PIPE_BYTES_2 ? 2 : MT_KG_MIN_NST;
  for (int kg = MT_KG_MAX; kg > 1; kg >>= 1)
    if (kb_per_split >= 2 * kg && (pipe - ring_slack(st_boff)) / (kg * st_bytes) >= min_nst) return kg;
  return 1;
}
static int ring_stages(int pipe, int st_bytes, int st_boff, int kg) {
  return std::min(MT_MAXST, (pipe - ring_slack(st_boff)) / (kg * st_bytes));
}

struct mt_ctx {
  int device = -1;
  bool host_only = true;
  int n_sms = 148;
  int grid = 148;
  int steal = 2;
  int claim_depth = 0; // MT_OPT_CLAIM_DEPTH
  int stage_split = 0; // MT_OPT_STAGE_SPLIT
  int partition = 0;   // MT_OPT_PARTITION: 0 roofline-proportional, 1 latency-balanced, 2 work/span
  int cps = 1;         // MT_OPT_CTAS_PER_SM: 1 (mtk build) or 2 (co-resident mtk_cr build, f4)
  // device-code configuration the plans are made for (mt_types.h)
  int nthreads() const { return cps == 2 ? 128 : 256; }
  int pipe_bytes() const { return cps == 2 ? MT_PIPE_BYTES_2 : MT_PIPE_BYTES_1; }
  int64_t timeout_ms = 2000;
  bool loaded = false, bound = false, has_sched = false;
  std::vector<Tenant> T;
  std::vector<HostOp> ops;
  std::vector<Buf> bufs;
  std::vector<WPack> wpacks;
  int64_t weight_bytes = 0, act_bytes = 0, partial_bytes = 0;
  int total_split_cnt = 0;
  int total_blocks = 0;
  int sum_L = 0;
  Layout lay;
  char *ws = nullptr;
  size_t ws_bytes = 0;
  Schedule sched;
  Err err;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t streams[MT_MAXT] = {};
  cudaEvent_t tev[MT_MAXT] = {};
  // cached CUDA graphs of the graph baselines (keyed by mode; invalidated on pointer change)
  cudaGraphExec_t gexec[8] = {};
  const float *g_in[8][MT_MAXT] = {};
  unsigned long long *trace = nullptr;
  int64_t trace_cap = 0;
  float *g_out[8][MT_MAXT] = {};
};

// launch interface of the device build a context plans for (1 or 2 CTAs per SM)
static cudaError_t k_executor(const mt_ctx *c, const RunArgs &a, int grid, cudaStream_t s) {
  return c->cps == 2 ? mtk_cr::launch_executor(a, grid, s) : mtk::launch_executor(a, grid, s);
}
static cudaError_t k_op(const mt_ctx *c, const RunArgs &a, const OpDesc &d, int op, int max_grid, cudaStream_t s) {
  return c->cps == 2 ? mtk_cr::launch_op(a, d, op, max_grid, s) : mtk::launch_op(a, d, op, max_grid, s);
}
static cudaError_t k_pack(const mt_ctx *c, const RunArgs &a, int t, cudaStream_t s) {
  return c->cps == 2 ? mtk_cr::launch_pack(a, t, s) : mtk::launch_pack(a, t, s);
}

// cached baseline graphs capture RunArgs (workspace, trace buffer, timeout): drop them whenever
// one of those changes
static void drop_graphs(mt_ctx *c) {
  for (auto &g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}

static mt_status fail(mt_ctx *c, mt_status st, const std::string &msg) {
  if (c) {
    c->err.st = st;
    c->err.msg = msg;
  }
  return st;
}
#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(c, MT_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }

static int pool_out(int size, int k, int s, int p, int ceil_mode) {
  if (ceil_mode) {
    int o = (int)cdiv(size + 2 * p - k, s) + 1;
    if ((int64_t)(o - 1) * s >= size + p) --o;
    return o;
  }
  return (size + 2 * p - k) / s + 1;
}

// ------------------------------------------------------------------------------------------
// graph ingest (a1)
// ------------------------------------------------------------------------------------------
namespace {
struct Shape { int c, h, w; };
}

static mt_status load_tenant(mt_ctx *c, int t, std::vector<std::vector<int>> &groups_members,
                             std::vector<int> &group_of_global, std::vector<Shape> &shapes) {
  Tenant &tn = c->T[t];
  const mt_graph &g = tn.g;
  const int L = tn.L;
  char buf[256];
  auto bad = [&](int j, const char *why) {
    snprintf(buf, sizeof buf, "tenant %d op %d: %s", t, j, why);
    return fail(c, MT_ERR_ARG, buf);
  };
  shapes.assign(L, Shape{0, 0, 0});
  auto shp = [&](int i) -> Shape { return i == -1 ? Shape{g.in_c, g.in_h, g.in_w} : shapes[i]; };
  for (int j = 0; j < L; ++j) {
    const mt_node &n = tn.nodes[j];
    if (n.n_inputs < 1 || n.n_inputs > MT_MAX_INPUTS) return bad(j, "n_inputs out of range");
    for (int q = 0; q < n.n_inputs; ++q)
      if (n.inputs[q] < -1 || n.inputs[q] >= j) return bad(j, "input id not topological");
    if (n.kind == MT_CONV && n.residual >= j) return bad(j, "residual id not topological");
    if (n.kind != MT_CONV && n.residual != -1) return bad(j, "residual only on CONV");
    // concatenated input shape
    Shape in = shp(n.inputs[0]);
    if (n.kind == MT_ADD) {
      for (int q = 1; q < n.n_inputs; ++q) {
        Shape s = shp(n.inputs[q]);
        if (s.c != in.c || s.h != in.h || s.w != in.w) return bad(j, "ADD input shapes differ");
      }
    } else {
      for (int q = 1; q < n.n_inputs; ++q) {
        Shape s = shp(n.inputs[q]);
        if (s.h != in.h || s.w != in.w) return bad(j, "concat spatial mismatch");
        in.c += s.c;
      }
    }
    Shape o{0, 0, 0};
    switch (n.kind) {
      case MT_CONV: {
        if (n.kh < 1 || n.kw < 1 || n.sh < 1 || n.sw < 1 || n.ph < 0 || n.pw < 0) return bad(j, "bad conv geometry");
        if (!(n.groups == 1 || (n.groups == in.c && n.out_c == in.c))) return bad(j, "only groups=1 or depthwise");
        if (!n.weight || !n.scale || !n.shift) return bad(j, "CONV needs weight/scale/shift");
        if (n.act < 0 || n.act > 2) return bad(j, "bad act");
        o = Shape{n.out_c, (in.h + 2 * n.ph - n.kh) / n.sh + 1, (in.w + 2 * n.pw - n.kw) / n.sw + 1};
        if (in.h + 2 * n.ph < n.kh || in.w + 2 * n.pw < n.kw) return bad(j, "kernel larger than input");
        break;
      }
      case MT_MAXPOOL:
      case MT_AVGPOOL: {
        if (n.kh < 1 || n.kw < 1 || n.sh < 1 || n.sw < 1 || n.ph < 0 || n.pw < 0) return bad(j, "bad pool geometry");
        if (2 * n.ph > n.kh || 2 * n.pw > n.kw) return bad(j, "pad > kernel/2");
        if (in.h + 2 * n.ph < n.kh || in.w + 2 * n.pw < n.kw) return bad(j, "window larger than input");
        o = Shape{in.c, pool_out(in.h, n.kh, n.sh, n.ph, n.ceil_mode), pool_out(in.w, n.kw, n.sw, n.pw, n.ceil_mode)};
        break;
      }
      case MT_GLOBAL_AVGPOOL: o = Shape{in.c, 1, 1}; break;
      case MT_FC:
        if (!n.weight || !n.scale || !n.shift) return bad(j, "FC needs weight/scale/shift");
        o = Shape{n.out_c, 1, 1};
        break;
      case MT_ADD:
      case MT_RELU: o = in; break;
      case MT_BN:
        if (!n.scale || !n.shift) return bad(j, "BN needs scale/shift");
        o = in;
        break;
      default: return bad(j, "unknown op kind");
    }
    if (o.c < 1 || o.h < 1 || o.w < 1) return bad(j, "empty output");
    if (o.c != n.out_c || o.h != n.out_h || o.w != n.out_w) return bad(j, "out shape disagrees with shape inference");
    if (n.kind == MT_CONV && n.residual >= 0) {
      Shape r = shapes[n.residual];
      if (r.c != o.c || r.h != o.h || r.w != o.w) return bad(j, "residual shape mismatch");
    }
    if ((n.kind == MT_ADD || n.kind == MT_BN || n.kind == MT_RELU || n.kind == MT_MAXPOOL ||
         n.kind == MT_AVGPOOL || n.kind == MT_GLOBAL_AVGPOOL || (n.kind == MT_CONV && n.groups > 1)) &&
        in.c % 8 != 0)
      return bad(j, "channel count of a pointwise/pool/depthwise input must be a multiple of 8");
    shapes[j] = o;
    // concat groups (channel concat of a multi-input CONV/POOL/FC consumer)
    if (n.kind != MT_ADD && n.n_inputs > 1) {
      std::vector<int> mem(n.inputs, n.inputs + n.n_inputs);
      for (int q = 0; q < n.n_inputs; ++q) {
        if (mem[q] == -1) return bad(j, "graph input cannot be concatenated");
        for (int r = 0; r < q; ++r)
          if (mem[r] == mem[q]) return bad(j, "duplicate concat member");
      }
      const int gb = tn.op_base;
      int existing = group_of_global[gb + mem[0]];
      if (existing >= 0 && groups_members[existing] == mem) continue;  // same group again
      for (int q = 0; q < n.n_inputs; ++q)
        if (group_of_global[gb + mem[q]] >= 0) return bad(j, "producer in two different concat groups");
      const int gid = (int)groups_members.size();
      groups_members.push_back(mem);
      for (int q = 0; q < n.n_inputs; ++q) group_of_global[gb + mem[q]] = gid;
    }
  }
  return MT_OK;
}

static mt_status plan_graphs(mt_ctx *c) {
  const int NT = (int)c->T.size();
  // cost model: SMs per op (shape + mix only)
  // workers (CTAs) an op's tiles spread over: the mix's share of the grid (2 CTAs/SM: twice the
  // workers -- same box, calibrated knobs: c4 b1 674 -> 622 us, c3 624 -> 549 us)
  const int wk = c->cps;
  const int sm_avail = std::min(148 * wk, std::max(24 * wk, 148 * wk / std::max(NT, 1)));
  int total = 0;
  for (auto &tn : c->T) { tn.op_base = total; total += tn.L; }
  c->sum_L = total;
  c->ops.assign(total, HostOp{});
  c->bufs.clear();
  c->wpacks.clear();
  std::vector<std::vector<int>> gmem;          // tenant-local member ids per group
  std::vector<int> gten;                       // tenant of group
  std::vector<int> group_of(total, -1);
  std::vector<std::vector<Shape>> shapes(NT);
  for (int t = 0; t < NT; ++t) {
    size_t g0 = gmem.size();
    mt_status st = load_tenant(c, t, gmem, group_of, shapes[t]);
    if (st != MT_OK) return st;
    for (size_t q = g0; q < gmem.size(); ++q) gten.push_back(t);
  }
  // ---- consumed-channel checks + buffers ----------------------------------------------
  std::vector<int> consumed(total, 0);
  for (int t = 0; t < NT; ++t)
    for (int j = 0; j < c->T[t].L; ++j) {
      const mt_node &n = c->T[t].nodes[j];
      for (int q = 0; q < n.n_inputs; ++q)
        if (n.inputs[q] >= 0) consumed[c->T[t].op_base + n.inputs[q]] = 1;
      if (n.kind == MT_CONV && n.residual >= 0) consumed[c->T[t].op_base + n.residual] = 1;
    }
  std::vector<TensorView> view(total);
  int64_t act = 0;
  auto new_buf = [&](int64_t bytes, int C) {
    Buf b;
    b.off = act;
    b.bytes = bytes;
    b.C = C;
    act += rup(bytes, 256);
    c->bufs.push_back(b);
    return (int)c->bufs.size() - 1;
  };
  for (size_t gi = 0; gi < gmem.size(); ++gi) {
    const int t = gten[gi];
    const Tenant &tn = c->T[t];
    const int eb = tn.g.precision == MT_PREC_BF16 ? 2 : 4;
    int Ctot = 0;
    for (int m : gmem[gi]) Ctot += shapes[t][m].c;
    const Shape s0 = shapes[t][gmem[gi][0]];
    int b = new_buf((int64_t)tn.g.batch * s0.h * s0.w * Ctot * eb, Ctot);
    int off = 0;
    for (int m : gmem[gi]) {
      if (m == tn.L - 1) return fail(c, MT_ERR_ARG, "final op cannot be a concat member");
      view[tn.op_base + m] = TensorView{b, Ctot, off, shapes[t][m].c, false};
      off += shapes[t][m].c;
    }
  }
  for (int t = 0; t < NT; ++t) {
    const Tenant &tn = c->T[t];
    const int eb = tn.g.precision == MT_PREC_BF16 ? 2 : 4;
    for (int j = 0; j < tn.L; ++j) {
      const int gid = tn.op_base + j;
      const Shape s = shapes[t][j];
      if (consumed[gid] && s.c % 8 != 0) {
        char m[160];
        snprintf(m, sizeof m, "tenant %d op %d: consumed tensor channels %d not a multiple of 8", t, j, s.c);
        return fail(c, MT_ERR_ARG, m);
      }
      if (group_of[gid] >= 0) continue;
      if (j == tn.L - 1) { view[gid] = TensorView{-1, s.c, 0, s.c, false}; continue; }
      int b = new_buf((int64_t)tn.g.batch * s.h * s.w * s.c * eb, s.c);
      view[gid] = TensorView{b, s.c, 0, s.c, false};
    }
  }
  c->act_bytes = act;
  // ---- per-op descriptors, tiles, costs, weight packing --------------------------------
  int64_t wbytes = 0, pbytes = 0;
  int split_cnt = 0;
  for (int t = 0; t < NT; ++t) {
    Tenant &tn = c->T[t];
    const mt_graph &g = tn.g;
    const bool bf16 = g.precision == MT_PREC_BF16;
    const int eb = bf16 ? 2 : 4;
    for (int j = 0; j < tn.L; ++j) {
      const mt_node &n = tn.nodes[j];
      const int gid = tn.op_base + j;
      HostOp &h = c->ops[gid];
      OpDesc &d = h.d;
      memset(&d, 0, sizeof d);
      d.kind = n.kind;
      d.tenant = t;
      d.prec = g.precision;
      d.act = n.act;
      d.groups = n.groups;
      d.kh = n.kh; d.kw = n.kw; d.sh = n.sh; d.sw = n.sw; d.ph = n.ph; d.pw = n.pw;
      d.ceil_mode = n.ceil_mode;
      d.cip = n.count_include_pad;
      d.N = g.batch;
      // input view
      auto in_view = [&](int i) -> TensorView {
        if (i == -1) return TensorView{-1, tn.cpad, 0, tn.cpad, true};
        return view[tn.op_base + i];
      };
      TensorView iv;
      if (n.kind != MT_ADD && n.n_inputs > 1) {
        TensorView m0 = view[tn.op_base + n.inputs[0]];
        int Ctot = 0;
        for (int q = 0; q < n.n_inputs; ++q) Ctot += shapes[t][n.inputs[q]].c;
        iv = TensorView{m0.buf, m0.cs, 0, Ctot, false};
      } else {
        iv = in_view(n.inputs[0]);
      }
      h.in[0] = iv;
      h.n_in = n.kind == MT_ADD ? n.n_inputs : 1;
      d.n_in = h.n_in;
      if (n.kind == MT_ADD)
        for (int q = 0; q < n.n_inputs; ++q) {
          h.in[q] = in_view(n.inputs[q]);
          d.ins_cs[q] = h.in[q].cs;
          d.ins_co[q] = h.in[q].co;
        }
      const Shape ins = n.inputs[0] == -1 ? Shape{g.in_c, g.in_h, g.in_w} : shapes[t][n.inputs[0]];
      d.H = ins.h;
      d.W = ins.w;
      d.C = iv.C;
      d.in_cs = iv.cs;
      d.in_co = iv.co;
      if (iv.graph_in) d.flags |= OPF_GRAPH_IN;
      if (iv.graph_in && n.kind != MT_CONV && n.kind != MT_FC && g.in_c % 8 != 0)
        return fail(c, MT_ERR_ARG, "only CONV/FC may read a graph input whose channels are not a multiple of 8");
      if (iv.graph_in && n.kind == MT_CONV && n.groups > 1)
        return fail(c, MT_ERR_ARG, "depthwise conv on the graph input is unsupported");
      const Shape os = shapes[t][j];
      d.Ho = os.h; d.Wo = os.w; d.Co = os.c;
      h.out = view[gid];
      d.out_cs = h.out.cs;
      d.out_co = h.out.co;
      if (j == tn.L - 1) d.flags |= OPF_OUT;
      if (n.kind == MT_CONV && n.residual >= 0) {
        h.res = view[tn.op_base + n.residual];
        d.flags |= OPF_RES;
        d.res_cs = h.res.cs;
        d.res_co = h.res.co;
      }
      // dependencies: every producer op this op reads (global ids)
      d.n_dep = 0;
      auto add_dep = [&](int gid_dep, int kind) {
        for (int r = 0; r < d.n_dep; ++r)
          if (d.deps[r] == gid_dep) { d.dep_kind[r] |= kind; return; }
        d.deps[d.n_dep] = gid_dep;
        d.dep_kind[d.n_dep++] = kind;
      };
      for (int q = 0; q < n.n_inputs; ++q)
        if (n.inputs[q] >= 0) add_dep(tn.op_base + n.inputs[q], 1);
      if (n.kind == MT_CONV && n.residual >= 0) add_dep(tn.op_base + n.residual, 2);
      h.scale = n.scale;
      h.shift = n.shift;
      // --- algorithmic cost (SURVEY d.4 B_op), identical to oracle/ir.py op_cost ---
      {
        int64_t in_el = 0;
        int cin_real = 0;
        for (int q = 0; q < n.n_inputs; ++q) {
          Shape s = n.inputs[q] == -1 ? Shape{g.in_c, g.in_h, g.in_w} : shapes[t][n.inputs[q]];
          in_el += (int64_t)g.batch * s.c * s.h * s.w;
          cin_real += s.c;
        }
        const int64_t out_el = (int64_t)g.batch * os.c * os.h * os.w;
        int64_t F = 0, wel = 0;
        if (n.kind == MT_CONV) {
          F = 2 * out_el * (int64_t)(cin_real / n.groups) * n.kh * n.kw;
          wel = (int64_t)os.c * (cin_real / n.groups) * n.kh * n.kw;
        } else if (n.kind == MT_FC) {
          const int64_t kin = (int64_t)cin_real * ins.h * ins.w;
          F = 2 * (int64_t)g.batch * kin * os.c;
          wel = kin * os.c;
        }
        const int64_t res_el = (n.kind == MT_CONV && n.residual >= 0) ? out_el : 0;
        h.flops = F;
        h.bytes = (in_el + wel + res_el + out_el) * eb;
      }
      // --- tile plan (shape only: identical for every schedule, §7 hard part 4) ---
      const int cin_real = (iv.graph_in ? g.in_c : iv.C);
      WPack wp;
      wp.op = gid;
      wp.src = n.weight;
      switch (n.kind) {
        case MT_CONV:
          if (n.groups > 1) {
            d.tk = TK_DW;
            if (n.kh == 3 && n.kw == 3 && n.sh == n.sw && (n.sh == 1 || n.sh == 2)) {
              // whole output rows per tile (row-run kernel): ~MT_NTHREADS*1.5 items per tile
              const int run = n.sh == 1 ? 4 : 2;
              const int64_t per_row = cdiv(os.w, run) * (os.c / 8);
              const int rows = (int)std::max<int64_t>(1, c->nthreads() / per_row);
              d.pix_tile = rows * os.w;
            } else {
              d.pix_tile = (int)std::max<int64_t>(1, (c->nthreads() * MT_EW_PER_THREAD) / (os.c / 8));
            }
            d.tiles = (int)cdiv((int64_t)g.batch * os.h * os.w, d.pix_tile);
            wp.mode = 3;
            wp.bytes = (int64_t)n.kh * n.kw * os.c * 4;   // fp32 (tiny; saves conversions)
          } else if (bf16) {
            d.tk = TK_CONV_TC;
            d.M = g.batch * os.h * os.w;
            d.bn = os.c <= 16 ? 16 : os.c <= 32 ? 32 : os.c <= 64 ? 64 : os.c <= 128 ? 128 : 256;   // refined below
            d.tiles_n = (int)cdiv(os.c, d.bn);
            // TMA mainloop: whole output rows per M tile; a K-block is one tap x 64 channels, loaded
            // as one 4-D box {64 ch, Wo*sw, R*sh, 1} with element strides {1, sw, sh, 1}
            // rows wider than 128 pixels: nseg column segments of seg_w pixels, one row per tile
            const int nseg = (int)cdiv(std::max(os.w, 1), 128);
            const int seg_w = (int)cdiv(std::max(os.w, 1), nseg);
            const int Rrows = std::min(os.h, 128 / seg_w);
            const bool geo_ok = seg_w * n.sw <= 256 && Rrows >= 1 && Rrows * n.sh <= 256;
            if (!iv.graph_in && d.C >= 16 && geo_ok) {
              d.tma = 1;
              d.cblks = (int)cdiv(d.C, 64);
              d.nkb = n.kh * n.kw * d.cblks;
              d.Kpad = d.nkb * MT_BK;
              d.K = d.Kpad;
              d.a_bytes = Rrows * seg_w * 128;
            } else if (d.C == 8 && geo_ok && (!iv.graph_in || g.in_c <= 8)) {
              // 8-channel input (the padded 3-channel stems): one 16-byte-row box per filter tap,
              // 8 taps per K-block, canonical no-swizzle K-major layout
              d.tma = 2;
              d.cblks = 1;
              d.K = n.kh * n.kw * 8;
              d.Kpad = (int)rup(d.K, MT_BK);
              d.nkb = d.Kpad / MT_BK;
              d.a_bytes = 8 * Rrows * seg_w * 16;
              if (iv.graph_in) tn.tma_input = true;
            }
            if (d.tma) {
              d.nseg = nseg;
              d.seg_w = seg_w;
              d.blk_rows = Rrows;
              d.blk_tpi = (int)cdiv(os.h, Rrows);
              d.tiles_m = g.batch * d.blk_tpi * nseg;
            } else {
              d.K = n.kh * n.kw * d.C;
              d.Kpad = (int)rup(d.K, MT_BK);
              d.nkb = d.Kpad / MT_BK;
              d.tiles_m = (int)cdiv(d.M, MT_BM);
            }
            // (bn, splits) from a latency model of one op (shape-only, so outputs are schedule-
            // invariant), calibrated on executor traces: a tile streams its
            // A box + B box per k-block at ~160 B/ns per SM (TMA) or pays the MMA time, whichever is
            // larger; ~2.6 us of fixed cost per tile (dependency -> first data, epilogue); a split
            // adds a dependent reduce hop (~4 us fixed + the partials at ~50 B/ns per reduce tile);
            // SMs available to the op: the GPU shared evenly by the mix's tenants (>= 37).
            int best_bn = d.bn, splits = 1;
            {
              double best = 1e30;
              const int bn_max = d.tma == 1 ? d.bn : std::min(d.bn, 128);   // 256-wide N tiles: TMA path only
              const double a_kb = d.tma ? (double)d.a_bytes : 16384.0;   // bytes of A per k-block
              const double rows = d.tma ? (double)d.blk_rows * d.seg_w : 128.0;
              const int bn_min = BN_MIN;
              for (int bn = bn_max; bn >= bn_min || bn == bn_max; bn >>= 1) {
                const int64_t tn = cdiv(os.c, bn), tmn_c = (int64_t)d.tiles_m * tn;
                const int boff = d.tma == 2 ? 16 * 1024 : (int)rup(d.a_bytes, 1024);
                for (int sp = 1; sp <= 12; ++sp) {
                  if (sp > 1 && d.nkb / sp < 2) break;
                  const int64_t kbps = cdiv(d.nkb, sp);
                  const int kgb = d.tma ? kgroup(c->pipe_bytes(), boff + (int)rup(bn * 128, 1024), boff, (int)kbps) : 1;
                  const double t_kb = std::max(0.13 * bn / 128.0, (a_kb + bn * 128.0) / TMA_BPUS) + MT_KB_OVH / kgb;
                  const int64_t waves = cdiv(tmn_c * sp, sm_avail);
                  double t = waves * (1.3 + kbps * t_kb + (sp == 1 ? 1.3 + 0.01 * bn : 0.6));
                  if (sp > 1) {
                    const int rcn = std::max(1, bn / 32);
                    t += 4.0 + cdiv(tmn_c * rcn, sm_avail) * (sp * rows * 32 * 4 / 50000.0);
                  }
                  if (t < best * 0.97) { best = t; best_bn = bn; splits = sp; }
                }
                if (bn <= bn_min) break;
              }
            }
            d.bn = best_bn;
            d.tiles_n = (int)cdiv(os.c, d.bn);
            const int tmn = d.tiles_m * d.tiles_n;
            d.kb_per_split = (int)cdiv(d.nkb, splits);
            d.splits = (int)cdiv(d.nkb, d.kb_per_split);
            d.rc = d.splits > 1 ? std::max(1, d.bn / 32) : 0;
            if (d.tma) {   // pipeline depth from the real box sizes (SW128 needs 1 KB alignment)
              d.st_boff = d.tma == 2 ? 16 * 1024 : (int)rup(d.a_bytes, 1024);
              d.st_bytes = d.st_boff + (int)rup(d.bn * 128, 1024);
              d.kg = kgroup(c->pipe_bytes(), d.st_bytes, d.st_boff, d.kb_per_split);
              d.nst = ring_stages(c->pipe_bytes(), d.st_bytes, d.st_boff, d.kg);
            } else {
              d.st_boff = 16 * 1024;
              d.st_bytes = 32 * 1024;
              d.kg = 1;
              d.nst = MT_STAGES;
            }
            d.tiles = tmn * d.splits + tmn * d.rc;
            wp.mode = d.tma == 1 ? 5 : 1;
            wp.bytes = (int64_t)d.tiles_n * d.bn * d.Kpad * 2;
            if (d.splits > 1) {
              d.cnt_off = split_cnt;
              split_cnt += tmn;
              h.ws_off = pbytes;
              h.ws_bytes = (int64_t)tmn * d.splits * MT_BM * d.bn * 4;
              pbytes += rup(h.ws_bytes, 256);
            }
          } else {
            d.tk = TK_CONV_SIMT;
            d.M = g.batch * os.h * os.w;
            d.K = n.kh * n.kw * d.C;
            d.tiles_m = (int)cdiv(d.M, MT_SIMT_BM);
            d.tiles_n = (int)cdiv(os.c, MT_SIMT_BN);
            d.splits = 1;
            d.tiles = d.tiles_m * d.tiles_n;
            wp.mode = 2;
            wp.bytes = (int64_t)os.c * d.K * 4;
          }
          break;
        case MT_MAXPOOL:
        case MT_AVGPOOL:
          d.tk = TK_POOL;
          d.pix_tile = (int)std::max<int64_t>(1, (c->nthreads() * MT_EW_PER_THREAD) / (os.c / 8));
          d.tiles = (int)cdiv((int64_t)g.batch * os.h * os.w, d.pix_tile);
          break;
        case MT_GLOBAL_AVGPOOL:
          d.tk = TK_GAP;
          d.tiles = (int)(g.batch * cdiv(os.c / 8, c->nthreads() / 8));
          break;
        case MT_FC:
          d.tk = TK_FC;
          if (!(iv.graph_in || (iv.cs == iv.C && iv.co == 0)))
            return fail(c, MT_ERR_ARG, "FC input must be a contiguous tensor");
          d.K = ins.h * ins.w * d.C;
          if (bf16 && !iv.graph_in && d.K % 8 == 0 &&
              (g.batch > 1 || (int64_t)os.c * d.K * 2 >= ((int64_t)8 << 20))) {
            // tensor-core FC (swap-AB): D[128 features][bn batch] = W[128][K] . X[bn][K]^T on
            // tcgen05, W and X streamed by TMA (2-D boxes, SW128), split-K over the SMs; used when
            // the weight stream is large (bandwidth-bound GEMV) or the batch makes CUDA-core FMAs
            // the bottleneck.  DESIGN.md section 5.
            d.tma = 3;
            d.tk = TK_CONV_TC;
            d.kh = d.kw = 1;
            d.cblks = 1;
            d.nseg = 1;
            d.M = os.c;
            d.bn = g.batch <= 16 ? 16 : 32;
            d.tiles_n = (int)cdiv(g.batch, d.bn);
            d.tiles_m = (int)cdiv(os.c, MT_BM);
            d.nkb = (int)cdiv(d.K, MT_BK);
            d.Kpad = d.nkb * MT_BK;
            d.a_bytes = MT_BM * 128;
            const int64_t tmn = (int64_t)d.tiles_m * d.tiles_n;
            // one wave: every compute tile of the op can be resident at once (148 SMs)
            const int want = (int)std::max<int64_t>(1, std::min<int64_t>(d.nkb / 8, 148 / tmn));
            d.kb_per_split = (int)cdiv(d.nkb, want);
            d.splits = (int)cdiv(d.nkb, d.kb_per_split);
            d.rc = d.splits > 1 ? 1 : 0;
            d.st_boff = d.a_bytes;
            d.st_bytes = d.st_boff + (int)rup(d.bn * 128, 1024);
            d.kg = kgroup(c->pipe_bytes(), d.st_bytes, d.st_boff, d.kb_per_split);
            d.nst = ring_stages(c->pipe_bytes(), d.st_bytes, d.st_boff, d.kg);
            d.tiles = (int)(tmn * d.splits + tmn * d.rc);
            if (d.splits > 1) {
              d.cnt_off = split_cnt;
              split_cnt += (int)tmn;
              h.ws_off = pbytes;
              h.ws_bytes = tmn * d.splits * MT_BM * d.bn * 4;
              pbytes += rup(h.ws_bytes, 256);
            }
            wp.mode = 4;
            wp.bytes = (int64_t)os.c * d.K * eb;
            break;
          }
          d.tiles = (int)(cdiv(os.c, c->nthreads() / 32) * cdiv(g.batch, MT_FC_BATCH));
          wp.mode = 4;
          wp.bytes = (int64_t)os.c * d.K * eb;
          break;
        default:
          d.tk = TK_ELT;
          d.pix_tile = (int)std::max<int64_t>(1, (c->nthreads() * MT_EW_PER_THREAD) / (os.c / 8));
          d.tiles = (int)cdiv((int64_t)g.batch * os.h * os.w, d.pix_tile);
          break;
      }
      (void)cin_real;
      if (wp.mode) {
        wp.dst_off = wbytes;
        h.w_off = wbytes;
        wbytes += rup(wp.bytes, 256);
        c->wpacks.push_back(wp);
      }
      if (d.tiles < 1) d.tiles = 1;
    }
  }
  int64_t nblk_total = 0;
  for (auto &h : c->ops) {
    OpDesc &d = h.d;
    const int64_t npix = (int64_t)d.N * d.Ho * d.Wo;
    switch (d.tk) {
      case TK_CONV_TC:   // (blk_rows for TMA); split-K: the reduce tiles complete the block
        if (d.tma == 3) {   // tensor-core FC: block = one batch tile (bn images), all feature tiles
          d.pix_blk = d.bn;
          d.blk_need = d.tiles_m * (d.splits > 1 ? d.rc : 1);
          break;
        }
        d.pix_blk = MT_BM;
        d.blk_need = d.tiles_n * (d.splits > 1 ? d.rc : 1) * (d.tma ? d.nseg : 1);
        break;
      case TK_CONV_SIMT: d.pix_blk = MT_SIMT_BM; d.blk_need = d.tiles_n; break;
      case TK_GAP: d.pix_blk = 1; d.blk_need = (int)cdiv(d.Co / 8, c->nthreads() / 8); break;
      case TK_FC: d.pix_blk = MT_FC_BATCH; d.blk_need = (int)cdiv(d.Co, c->nthreads() / 32); break;
      default: d.pix_blk = d.pix_tile; d.blk_need = 1; break;
    }
    d.nblk = d.blk_rows > 0 ? d.N * d.blk_tpi : (int)cdiv(npix, d.pix_blk);
    d.blk_off = (int)nblk_total;
    nblk_total += d.nblk;
  }
  c->total_blocks = (int)nblk_total;
  // ---- latency model of every op (partition input, R16b): tiles x ns per tile ----
  // Same calibration as the (bn, splits) choice above: per k-block max(MMA, A+B bytes at ~160 B/ns
  // per SM), ~2.6 us fixed per tile; split-K reduce tiles read their partials at ~50 B/ns; the
  // memory-bound kinds ~2.6 us fixed + their bytes per tile at ~50 B/ns.
  for (auto &h : c->ops) {
    const OpDesc &d = h.d;
    double us0 = 0.0, us1 = 0.0;
    int64_t t0 = d.tiles, t1 = 0;
    if (d.tk == TK_CONV_TC) {
      const double a_kb = d.tma ? (double)d.a_bytes : 16384.0;
      const double rows = d.tma == 3 ? 128.0 : d.tma ? (double)d.blk_rows * d.seg_w : 128.0;
      const double t_kb = std::max(0.13 * d.bn / 128.0, (a_kb + d.bn * 128.0) / TMA_BPUS) +
                          MT_KB_OVH / std::max(1, (int)d.kg);
      const int64_t tmn = (int64_t)d.tiles_m * d.tiles_n;
      t0 = tmn * d.splits;
      us0 = 1.3 + d.kb_per_split * t_kb + (d.splits == 1 ? 1.3 + 0.01 * d.bn : 0.6);
      if (d.splits > 1) {
        t1 = tmn * d.rc;
        us1 = 2.6 + d.splits * rows * 32 * 4 / 50000.0;
      }
    } else if (d.tk == TK_CONV_SIMT) {
      us0 = 3.0 + 2.0 * MT_SIMT_BM * MT_SIMT_BN * d.K / 50000.0;
    } else {
      us0 = 2.6 + (double)h.bytes / std::max(1, d.tiles) / 50000.0;
    }
    h.work_tiles[0] = (int32_t)t0;
    h.work_ns[0] = (int64_t)llround(us0 * 1000.0);
    h.work_tiles[1] = (int32_t)t1;
    h.work_ns[1] = t1 ? (int64_t)llround(us1 * 1000.0) : 0;
  }
  c->weight_bytes = wbytes;
  c->partial_bytes = pbytes;
  c->total_split_cnt = split_cnt;
  // ---- workspace layout ------------------------------------------------------------------
  Layout &L = c->lay;
  L = Layout{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (size_t)rup((int64_t)bytes, 256);
    return o;
  };
  const int S_max = std::max(c->sum_L, 1);
  L.ctl = take(sizeof(CtlBlock));
  L.claim = take(sizeof(int32_t) * total);
  L.done = take(sizeof(int32_t) * total);
  L.blk = take(sizeof(int32_t) * std::max(c->total_blocks, 1));
  L.splitcnt = take(sizeof(int32_t) * std::max(split_cnt, 1));
  L.counters_bytes = off;
  L.gates = take(sizeof(int32_t) * total);   // outside the counters: error recovery zeroes those
  L.ops = take(sizeof(OpDesc) * total);
  L.tmaps = take((size_t)256 * total);
  L.sched_rng = take(sizeof(int32_t) * S_max * NT * 2);
  L.sched_home = take((size_t)S_max * c->grid);
  L.prof_area_bytes = 8u << 20;
  L.prof_area = take(L.prof_area_bytes);
  L.prof_ts_bytes = 1u << 20;
  L.prof_ts = take(L.prof_ts_bytes);
  L.run_ts = take(sizeof(unsigned long long) * 4 * (S_max + 1));   // stage-split: 4 stamps per launch
  L.packed_off.resize(NT);
  L.stage_in_off.resize(NT);
  L.stage_out_off.resize(NT);
  for (int t = 0; t < NT; ++t) {
    const mt_graph &g = c->T[t].g;
    const int eb = g.precision == MT_PREC_BF16 ? 2 : 4;
    L.packed_off[t] = take((size_t)g.batch * g.in_h * g.in_w * c->T[t].cpad * eb);
  }
  for (int t = 0; t < NT; ++t) {
    const mt_graph &g = c->T[t].g;
    L.stage_in_off[t] = take((size_t)g.batch * g.in_c * g.in_h * g.in_w * 4);
    const mt_node &last = c->T[t].nodes.back();
    L.stage_out_off[t] = take((size_t)g.batch * last.out_c * last.out_h * last.out_w * 4);
  }
  L.weights = take(wbytes);
  L.acts = take(act);
  L.partials = take(pbytes);
  L.total = off;
  return MT_OK;
}

// ------------------------------------------------------------------------------------------
// schedule -> stage plan (a2/a3)
// ------------------------------------------------------------------------------------------
static std::vector<int> lengths(mt_ctx *c) {
  std::vector<int> L;
  for (auto &t : c->T) L.push_back(t.L);
  return L;
}

// Gate op of every op for claim depth D (R20), -1 = none.  D > 0: the newest (largest
// id) of o's ancestors at DAG distance exactly D (layer D of a breadth-first walk up the dependency
// edges; older members of the layer complete first).  D < 0: op o - |D| of the same tenant.  No
// gate when o is closer than |D| to the graph input.  Any ancestor keeps claiming deadlock-free.
static std::vector<int32_t> gate_table(mt_ctx *c, int D) {
  const int n = (int)c->ops.size();
  std::vector<int32_t> g((size_t)n, -1);
  if (D == 0) return g;
  for (int o = 0; o < n; ++o) {
    if (D < 0) {
      if (o + D >= c->T[c->ops[o].d.tenant].op_base) g[o] = o + D;
      continue;
    }
    std::vector<int> layer{o};
    for (int k = 1; k <= D && !layer.empty(); ++k) {
      std::vector<int> nx;
      for (int x : layer) {
        const OpDesc &d = c->ops[x].d;
        for (int r = 0; r < d.n_dep; ++r)
          if (std::find(nx.begin(), nx.end(), d.deps[r]) == nx.end()) nx.push_back(d.deps[r]);
      }
      layer = nx;
    }
    for (int x : layer) g[o] = std::max(g[o], x);
  }
  return g;
}

static mt_status upload_gates(mt_ctx *c) {
  if (c->host_only || !c->bound) return MT_OK;
  std::vector<int32_t> g = gate_table(c, c->claim_depth);
  CK(cudaMemcpy(c->ws + c->lay.gates, g.data(), g.size() * 4, cudaMemcpyHostToDevice));
  return MT_OK;
}

static void build_stage_plan(mt_ctx *c, Schedule &s) {
  const int N = (int)c->T.size();
  s.sms.assign((size_t)s.S * N, 0);
  s.home.assign((size_t)s.S * c->grid, 0);
  for (int k = 0; k < s.S; ++k) {
    std::vector<bool> active(N, false);
    std::vector<__int128> w(N, 0);
    std::vector<int64_t> caps(N, 0);   // a3 tile cap: most tiles of one op of the slice
    for (int t = 0; t < N; ++t) {
      const int b = s.ranges[(k * N + t) * 2], e = s.ranges[(k * N + t) * 2 + 1];
      if (b == e) continue;
      active[t] = true;
      for (int j = b; j < e; ++j) {
        const HostOp &h = c->ops[c->T[t].op_base + j];
        const __int128 a = (__int128)h.flops * BW_GBS, bb = (__int128)h.bytes * TC_GFLOPS;
        w[t] += a > bb ? a : bb;
        caps[t] = std::max<int64_t>(caps[t], h.d.tiles);
      }
    }
    std::vector<int> n;
    if (c->partition >= 1) {
      std::vector<std::vector<std::pair<int64_t, int64_t>>> items(N);
      for (int t = 0; t < N; ++t) {
        if (!active[t]) continue;
        for (int j = s.ranges[(k * N + t) * 2]; j < s.ranges[(k * N + t) * 2 + 1]; ++j) {
          const HostOp &h = c->ops[c->T[t].op_base + j];
          for (int q = 0; q < 2; ++q)
            if (h.work_tiles[q] > 0) items[t].push_back({h.work_tiles[q], h.work_ns[q]});
        }
      }
      n = sm_partition_balanced(active, items, c->n_sms, c->partition, MT_HOP_NS);
    } else {
      n = sm_partition(active, w, c->n_sms, &caps);
    }
    int cta = 0;
    for (int t = 0; t < N; ++t) s.sms[k * N + t] = n[t];
    if (c->cps == 2) {
      // f4 heterogeneous co-residency: the CTA in slot 0 of SM i serves the i-th entry of the SM
      // partition listed from the most to the least compute-intense tenant (FLOP per byte of the
      // stage slice), the CTA in slot 1 the list reversed -- so the two CTAs of an SM pair a
      // compute-bound slice with a memory-bound one where the mix has both
      std::vector<int> order;
      for (int t = 0; t < N; ++t)
        if (n[t] > 0) order.push_back(t);
      std::vector<double> inten(N, 0.0);
      for (int t : order) {
        double F = 0.0, B = 0.0;
        for (int j = s.ranges[(k * N + t) * 2]; j < s.ranges[(k * N + t) * 2 + 1]; ++j) {
          F += (double)c->ops[c->T[t].op_base + j].flops;
          B += (double)c->ops[c->T[t].op_base + j].bytes;
        }
        inten[t] = F / std::max(B, 1.0);
      }
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return inten[x] > inten[y]; });
      std::vector<int> list;
      for (int t : order)
        for (int q = 0; q < n[t]; ++q) list.push_back(t);
      const int nsm = c->grid / 2;
      for (int i = 0; i < nsm && i < (int)list.size(); ++i) {
        s.home[(size_t)k * c->grid + i] = (uint8_t)list[i];
        s.home[(size_t)k * c->grid + nsm + i] = (uint8_t)list[MT_CR_PAIR ? list.size() - 1 - i : i];
      }
      cta = c->grid;
    }
    for (int t = 0; t < N && cta < c->grid; ++t)
      for (int q = 0; q < n[t] && cta < c->grid; ++q) s.home[(size_t)k * c->grid + cta++] = (uint8_t)t;
    // grid larger than n_sms (never with 1 CTA/SM): spread the rest round-robin
    int t0 = 0;
    while (cta < c->grid) {
      while (!active[t0 % N]) ++t0;
      s.home[(size_t)k * c->grid + cta++] = (uint8_t)(t0 % N);
      ++t0;
    }
  }
}

static void to_global_ranges(mt_ctx *c, const Schedule &s, int32_t *dst) {
  const int N = (int)c->T.size();
  for (int k = 0; k < s.S; ++k)
    for (int t = 0; t < N; ++t) {
      dst[(k * N + t) * 2] = s.ranges[(k * N + t) * 2] + c->T[t].op_base;
      dst[(k * N + t) * 2 + 1] = s.ranges[(k * N + t) * 2 + 1] + c->T[t].op_base;
    }
}

static mt_status apply_schedule(mt_ctx *c, Schedule &s) {
  build_stage_plan(c, s);
  if (!c->host_only && c->bound) {
    std::vector<int32_t> g((size_t)s.S * c->T.size() * 2);
    to_global_ranges(c, s, g.data());
    CK(cudaMemcpy(c->ws + c->lay.sched_rng, g.data(), g.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->ws + c->lay.sched_home, s.home.data(), s.home.size(), cudaMemcpyHostToDevice));
  }
  c->sched = s;
  c->has_sched = true;
  return MT_OK;
}

// ------------------------------------------------------------------------------------------
// run-time argument block
// ------------------------------------------------------------------------------------------
static RunArgs base_args(mt_ctx *c, const float *const *inputs, float *const *outputs) {
  RunArgs a;
  memset(&a, 0, sizeof a);
  const int N = (int)c->T.size();
  a.ops = (const OpDesc *)(c->ws + c->lay.ops);
  a.rng = (const int32_t *)(c->ws + c->lay.sched_rng);
  a.home = (const uint8_t *)(c->ws + c->lay.sched_home);
  a.n_stages = c->has_sched ? c->sched.S : 0;
  a.n_tenants = N;
  a.steal = c->steal;
  a.claim_depth = (int)c->ops.size() <= MT_GATE_OPS ? c->claim_depth : 0;
  a.gates = (const int32_t *)(c->ws + c->lay.gates);
  a.claim = (int32_t *)(c->ws + c->lay.claim);
  a.done = (int32_t *)(c->ws + c->lay.done);
  a.blkcnt = (int32_t *)(c->ws + c->lay.blk);
  a.n_blk = c->total_blocks;
  a.splitcnt = (int32_t *)(c->ws + c->lay.splitcnt);
  a.ctl = (CtlBlock *)(c->ws + c->lay.ctl);
  a.ts = (unsigned long long *)(c->ws + c->lay.run_ts);
  a.ts_full = 1;
  a.timeout_ns = (unsigned long long)c->timeout_ms * 1000000ull;
  a.n_ops = (int)c->ops.size();
  a.n_pack = 0;
  a.trace = c->trace;
  a.trace_cap = (int32_t)c->trace_cap;
  for (int t = 0; t < N; ++t) {
    const mt_graph &g = c->T[t].g;
    a.inputs[t] = inputs ? inputs[t] : nullptr;
    a.outputs[t] = outputs ? outputs[t] : nullptr;
    a.in_n[t] = g.batch; a.in_c[t] = g.in_c; a.in_h[t] = g.in_h; a.in_w[t] = g.in_w;
    a.in_cpad[t] = c->T[t].cpad;
    a.in_prec[t] = g.precision;
    // shared input: pack once per distinct (pointer, shape, precision)
    int src = t;
    for (int u = 0; u < t && !c->T[t].tma_input; ++u) {
      const mt_graph &h = c->T[u].g;
      if (inputs && inputs[u] == inputs[t] && h.batch == g.batch && h.in_c == g.in_c &&
          h.in_h == g.in_h && h.in_w == g.in_w && h.precision == g.precision) { src = u; break; }
    }
    a.packed[t] = (uint64_t)(c->ws + c->lay.packed_off[src]);
    if (src == t) a.pack_tenant[a.n_pack++] = t;
  }
  return a;
}

static mt_status check_ready(mt_ctx *c, bool need_sched) {
  if (!c) return MT_ERR_ARG;
  if (c->host_only) return fail(c, MT_ERR_STATE, "host-only context cannot run");
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (!c->bound) return fail(c, MT_ERR_STATE, "workspace not bound");
  if (need_sched && !c->has_sched) return fail(c, MT_ERR_STATE, "no schedule set");
  return MT_OK;
}

static mt_status check_device_error(mt_ctx *c) {
  CtlBlock cb;
  CK(cudaMemcpy(&cb, c->ws + c->lay.ctl, sizeof cb, cudaMemcpyDeviceToHost));
  if (cb.error) {
    char m[200];
    snprintf(m, sizeof m, "device timeout/invariant failure (code %u, info %llx); counters reset",
             cb.error, cb.err_info);
    cudaMemset(c->ws, 0, c->lay.counters_bytes);
    cudaDeviceSynchronize();
    return fail(c, MT_ERR_INTERNAL, m);
  }
  return MT_OK;
}

// ------------------------------------------------------------------------------------------
// TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point)
// ------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                      const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                      const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled_t)p;
  }
  return fn;
}

// A: activations NHWC viewed as 4-D {C, W, H, N} (channel slice of a possibly concatenated
// buffer); box {64, Wo*sw, R*sh, 1} with traversal strides {1, sw, sh, 1} = the im2col rows of one
// tap for R whole output rows; out-of-range coordinates (padding) are zero-filled by the TMA unit.
// B: packed weights {Kpad, Cout_pad}, box {64, bn}.  Both 128-byte swizzled (UMMA SW128 K-major).
static mt_status make_conv_tmaps(mt_ctx *c, const OpDesc &o, const HostOp &h, char *ma_dev, char *mb_dev) {
  PFN_encodeTiled_t enc = encode_fn();
  if (!enc) return fail(c, MT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  alignas(64) CUtensorMap ma, mb;
  const cuuint64_t es = 2;
  if (o.tma == 3) {   // tensor-core FC: A = packed weights {K, Co} box {64, 128}; B = input {K, N} box {64, bn}
    cuuint64_t adim[2] = {(cuuint64_t)o.K, (cuuint64_t)o.Co}, astr[1] = {(cuuint64_t)o.K * es};
    cuuint64_t bdim[2] = {(cuuint64_t)o.K, (cuuint64_t)o.N}, bstr[1] = {(cuuint64_t)o.K * es};
    cuuint32_t abox[2] = {64, (cuuint32_t)MT_BM}, bbox[2] = {64, (cuuint32_t)o.bn}, one[2] = {1, 1};
    CUresult r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)o.w, adim, astr, abox, one,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, MT_ERR_CUDA, "FC tensor map A encode failed");
    r = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)(o.in + (uint64_t)o.in_co * es), bdim, bstr, bbox, one,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, MT_ERR_CUDA, "FC tensor map B encode failed");
    CK(cudaMemcpy(ma_dev, &ma, sizeof ma, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(mb_dev, &mb, sizeof mb, cudaMemcpyHostToDevice));
    return MT_OK;
  }
  cuuint64_t gdim[4] = {(cuuint64_t)o.C, (cuuint64_t)o.W, (cuuint64_t)o.H, (cuuint64_t)o.N};
  cuuint64_t gstr[3] = {(cuuint64_t)o.in_cs * es, (cuuint64_t)o.W * o.in_cs * es,
                        (cuuint64_t)o.H * o.W * o.in_cs * es};
  const bool small = o.tma == 2;   // 8-channel rows of 16 bytes, no swizzle
  cuuint32_t box[4] = {small ? 8u : 64u, (cuuint32_t)(o.seg_w * o.sw), (cuuint32_t)(o.blk_rows * o.sh), 1};
  cuuint32_t estr[4] = {1, (cuuint32_t)o.sw, (cuuint32_t)o.sh, 1};
  void *base = (o.flags & OPF_GRAPH_IN) ? (void *)(c->ws + c->lay.packed_off[o.tenant])
                                        : (void *)(o.in + (uint64_t)o.in_co * es);
  CUresult r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, gdim, gstr, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, small ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char m[160];
    snprintf(m, sizeof m, "tensor map A (op %d) encode failed: %d", (int)(&h - c->ops.data()), (int)r);
    return fail(c, MT_ERR_CUDA, m);
  }
  cuuint64_t bdim[2] = {(cuuint64_t)o.Kpad, (cuuint64_t)o.tiles_n * o.bn};
  cuuint64_t bstr[1] = {(cuuint64_t)o.Kpad * es};
  cuuint32_t bbox[2] = {64, (cuuint32_t)o.bn};
  cuuint32_t bes[2] = {1, 1};
  r = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)o.w, bdim, bstr, bbox, bes,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, MT_ERR_CUDA, "tensor map B encode failed");
  CK(cudaMemcpy(ma_dev, &ma, sizeof ma, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(mb_dev, &mb, sizeof mb, cudaMemcpyHostToDevice));
  return MT_OK;
}

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
extern "C" {

const char *mt_version(void) { return "mt-b200 0.1 (sm_100a, tcgen05 implicit-GEMM conv, persistent stage executor)"; }

mt_status mt_create(int device, mt_ctx **out) {
  if (!out) return MT_ERR_ARG;
  *out = nullptr;
  mt_ctx *c = new mt_ctx();
  c->device = device;
  c->host_only = device < 0;
  if (!c->host_only) {
    if (cudaSetDevice(device) != cudaSuccess) {
      delete c;
      return MT_ERR_REFUSED;
    }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
      delete c;
      return MT_ERR_REFUSED;
    }
    int bps = 0;
    if (mtk::executor_occupancy(&bps) != cudaSuccess || bps < 1) {
      delete c;
      return MT_ERR_REFUSED;
    }
    c->n_sms = sms;
    c->grid = sms;  // one persistent CTA per SM (smem sized for the conv pipeline)
    cudaEventCreate(&c->ev0);
    cudaEventCreate(&c->ev1);
    for (int t = 0; t < MT_MAXT; ++t) {
      cudaStreamCreateWithFlags(&c->streams[t], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&c->tev[t], cudaEventDisableTiming);
    }
  }
  *out = c;
  return MT_OK;
}

mt_status mt_destroy(mt_ctx *c) {
  if (!c) return MT_ERR_ARG;
  if (!c->host_only) {
    cudaDeviceSynchronize();
    for (auto &g : c->gexec)
      if (g) cudaGraphExecDestroy(g);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (int t = 0; t < MT_MAXT; ++t) {
      if (c->streams[t]) cudaStreamDestroy(c->streams[t]);
      if (c->tev[t]) cudaEventDestroy(c->tev[t]);
    }
  }
  delete c;
  return MT_OK;
}

mt_status mt_set_option(mt_ctx *c, int32_t option, int64_t value) {
  if (!c) return MT_ERR_ARG;
  switch (option) {
    case MT_OPT_STEAL:
      if (value < 0 || value > 2) return fail(c, MT_ERR_ARG, "steal must be 0, 1 or 2");
      c->steal = (int)value;
      return MT_OK;
    case MT_OPT_NUM_SMS:
      if (!c->host_only) return fail(c, MT_ERR_STATE, "NUM_SMS only settable on host-only contexts");
      if (value < 1 || value > 4096) return fail(c, MT_ERR_ARG, "bad NUM_SMS");
      if (c->loaded && value < (int64_t)c->T.size()) return fail(c, MT_ERR_ARG, "NUM_SMS < tenants");
      c->n_sms = (int)value;
      c->grid = (int)value * c->cps;
      if (c->has_sched) build_stage_plan(c, c->sched);
      return MT_OK;
    case MT_OPT_TIMEOUT_MS:
      if (value < 1) return fail(c, MT_ERR_ARG, "bad timeout");
      c->timeout_ms = value;
      drop_graphs(c);
      return MT_OK;
    case MT_OPT_CTAS_PER_SM: {   // f4: 2 co-resident CTAs per SM (plans depend on it: set before loading)
      if (value != 1 && value != 2) return fail(c, MT_ERR_ARG, "CTAs per SM must be 1 or 2");
      if (c->loaded) return fail(c, MT_ERR_STATE, "set CTAs per SM before mt_load_graphs");
      if (!c->host_only) {
        int bps = 0;
        cudaError_t e = value == 2 ? mtk_cr::executor_occupancy(&bps) : mtk::executor_occupancy(&bps);
        if (e != cudaSuccess || bps < value) {
          char m[400], r[256] = "";
          if (value == 2) mtk_cr::executor_resources(r, sizeof r);
          snprintf(m, sizeof m, "executor does not fit %d CTAs per SM (occupancy %d, %s; %s)", (int)value, bps,
                   cudaGetErrorString(e), r);
          return fail(c, MT_ERR_REFUSED, m);
        }
      }
      c->cps = (int)value;
      c->grid = c->n_sms * c->cps;
      return MT_OK;
    }
    case MT_OPT_CLAIM_DEPTH:
      if (value < -(1 << 20) || value > 1 << 20) return fail(c, MT_ERR_ARG, "bad claim depth");
      if (value != 0 && c->loaded && (int)c->ops.size() > MT_GATE_OPS)
        return fail(c, MT_ERR_ARG, "claim depth needs <= 2048 ops in the mix");
      c->claim_depth = (int)value;
      return upload_gates(c);
    case MT_OPT_STAGE_SPLIT:
      if (value < 0 || value > 1) return fail(c, MT_ERR_ARG, "stage split must be 0 or 1");
      c->stage_split = (int)value;
      return MT_OK;
    case MT_OPT_PARTITION:
      if (value < 0 || value > 2) return fail(c, MT_ERR_ARG, "partition must be 0, 1 or 2");
      c->partition = (int)value;
      if (c->has_sched) {
        Schedule s = c->sched;
        return apply_schedule(c, s);
      }
      return MT_OK;
  }
  return fail(c, MT_ERR_ARG, "unknown option");
}

mt_status mt_load_graphs(mt_ctx *c, int32_t n, const mt_graph *graphs) {
  if (!c) return MT_ERR_ARG;
  if (n < 1 || n > MT_MAX_TENANTS || !graphs) return fail(c, MT_ERR_ARG, "n_tenants out of range");
  if (n > c->n_sms) return fail(c, MT_ERR_ARG, "more tenants than SMs");
  if (!c->host_only) cudaDeviceSynchronize();
  drop_graphs(c);
  c->loaded = c->bound = c->has_sched = false;
  c->T.assign(n, Tenant{});
  for (int t = 0; t < n; ++t) {
    const mt_graph &g = graphs[t];
    if (g.n_nodes < 1 || !g.nodes) return fail(c, MT_ERR_ARG, "empty graph");
    if (g.batch < 1 || g.in_c < 1 || g.in_h < 1 || g.in_w < 1) return fail(c, MT_ERR_ARG, "bad input shape");
    if (g.precision != MT_PREC_BF16 && g.precision != MT_PREC_FP32) return fail(c, MT_ERR_ARG, "bad precision");
    if (c->cps == 2 && g.precision == MT_PREC_FP32)   // the fp32 SIMT conv tile assumes 256 threads
      return fail(c, MT_ERR_REFUSED, "2 CTAs per SM: bf16 tenants only");
    c->T[t].g = g;
    c->T[t].nodes.assign(g.nodes, g.nodes + g.n_nodes);
    c->T[t].g.nodes = nullptr;
    c->T[t].L = g.n_nodes;
    c->T[t].cpad = (int)rup(g.in_c, 8);
  }
  mt_status st = plan_graphs(c);
  if (st != MT_OK) { c->T.clear(); c->ops.clear(); return st; }
  c->loaded = true;
  return MT_OK;
}

mt_status mt_op_count(mt_ctx *c, int32_t t, int32_t *n) {
  if (!c || !n) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (t < 0 || t >= (int)c->T.size()) return fail(c, MT_ERR_ARG, "bad tenant");
  *n = c->T[t].L;
  return MT_OK;
}

mt_status mt_op_cost(mt_ctx *c, int32_t t, int32_t op, int64_t *flops, int64_t *bytes) {
  if (!c) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (t < 0 || t >= (int)c->T.size() || op < 0 || op >= c->T[t].L) return fail(c, MT_ERR_ARG, "bad op");
  const HostOp &h = c->ops[c->T[t].op_base + op];
  if (flops) *flops = h.flops;
  if (bytes) *bytes = h.bytes;
  return MT_OK;
}

mt_status mt_op_tiles(mt_ctx *c, int32_t t, int32_t op, int32_t *tiles) {
  if (!c || !tiles) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (t < 0 || t >= (int)c->T.size() || op < 0 || op >= c->T[t].L) return fail(c, MT_ERR_ARG, "bad op");
  *tiles = c->ops[c->T[t].op_base + op].d.tiles;
  return MT_OK;
}

mt_status mt_op_plan(mt_ctx *c, int32_t t, int32_t op, int32_t *plan) {
  if (!c || !plan) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (t < 0 || t >= (int)c->T.size() || op < 0 || op >= c->T[t].L) return fail(c, MT_ERR_ARG, "bad op");
  const OpDesc &d = c->ops[c->T[t].op_base + op].d;
  int kind = MT_PLAN_KIND_ELT;
  switch (d.tk) {
    case TK_CONV_TC: kind = MT_PLAN_KIND_CONV_TC; break;
    case TK_CONV_SIMT: kind = MT_PLAN_KIND_CONV_SIMT; break;
    case TK_DW: kind = MT_PLAN_KIND_DW; break;
    case TK_POOL: kind = MT_PLAN_KIND_POOL; break;
    case TK_GAP: kind = MT_PLAN_KIND_GAP; break;
    case TK_FC: kind = MT_PLAN_KIND_FC; break;
    default: break;
  }
  const bool tc = d.tk == TK_CONV_TC;
  const int32_t v[MT_PLAN_LEN] = {kind, tc ? d.tma : 0, tc ? d.bn : 0, tc ? d.splits : 1, tc ? d.tiles_m : 0,
                                  tc ? d.tiles_n : 0, tc ? (d.tma ? d.nst : MT_STAGES) : 0, d.tiles,
                                  tc && d.tma ? d.nseg : 1};
  for (int i = 0; i < MT_PLAN_LEN; ++i) plan[i] = v[i];
  return MT_OK;
}

mt_status mt_op_work(mt_ctx *c, int32_t t, int32_t op, int32_t *tiles, int64_t *ns) {
  if (!c || !tiles || !ns) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (t < 0 || t >= (int)c->T.size() || op < 0 || op >= c->T[t].L) return fail(c, MT_ERR_ARG, "bad op");
  const HostOp &h = c->ops[c->T[t].op_base + op];
  for (int q = 0; q < 2; ++q) {
    tiles[q] = h.work_tiles[q];
    ns[q] = h.work_ns[q];
  }
  return MT_OK;
}

mt_status mt_workspace_size(mt_ctx *c, size_t *bytes) {
  if (!c || !bytes) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  *bytes = c->lay.total;
  return MT_OK;
}

mt_status mt_bind_workspace(mt_ctx *c, void *dev, size_t bytes) {
  if (!c) return MT_ERR_ARG;
  if (c->host_only) return fail(c, MT_ERR_STATE, "host-only context has no workspace");
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (!dev || bytes < c->lay.total || ((uintptr_t)dev & 255)) return fail(c, MT_ERR_ARG, "workspace too small or misaligned");
  drop_graphs(c);
  c->ws = (char *)dev;
  c->ws_bytes = bytes;
  const Layout &L = c->lay;
  // device addresses into the op descriptors
  std::vector<OpDesc> d(c->ops.size());
  for (size_t i = 0; i < c->ops.size(); ++i) {
    HostOp &h = c->ops[i];
    OpDesc o = h.d;
    auto addr = [&](const TensorView &v) -> uint64_t {
      if (v.graph_in || v.buf < 0) return 0;
      return (uint64_t)(c->ws + L.acts + c->bufs[v.buf].off);
    };
    o.in = addr(h.in[0]);
    for (int q = 0; q < h.n_in && o.kind == MT_ADD; ++q) o.ins[q] = addr(h.in[q]);
    o.out = addr(h.out);
    o.res = (o.flags & OPF_RES) ? addr(h.res) : 0;
    o.w = h.w_off >= 0 ? (uint64_t)(c->ws + L.weights + h.w_off) : 0;
    o.ws = h.ws_off >= 0 ? (uint64_t)(c->ws + L.partials + h.ws_off) : 0;
    o.scale = (uint64_t)h.scale;
    o.shift = (uint64_t)h.shift;
    if (o.tma) {
      char *ma = c->ws + L.tmaps + 256 * i, *mb = ma + 128;
      mt_status st = make_conv_tmaps(c, o, h, ma, mb);
      if (st != MT_OK) return st;
      o.tmap_a = (uint64_t)ma;
      o.tmap_b = (uint64_t)mb;
    }
    h.d = o;
    d[i] = o;
  }
  CK(cudaMemset(c->ws, 0, L.counters_bytes));
  CK(cudaMemcpy(c->ws + L.ops, d.data(), sizeof(OpDesc) * d.size(), cudaMemcpyHostToDevice));
  for (const WPack &wp : c->wpacks) {
    const HostOp &h = c->ops[wp.op];
    const Tenant &tn = c->T[h.d.tenant];
    const int cin_real = h.in[0].graph_in ? tn.g.in_c : h.d.C;
    CK(cudaMemset(c->ws + L.weights + wp.dst_off, 0, wp.bytes));
    CK(mtk::launch_weight_pack(wp.mode, wp.src, c->ws + L.weights + wp.dst_off, h.d, cin_real, 0));
  }
  CK(cudaDeviceSynchronize());
  c->bound = true;
  if (upload_gates(c) != MT_OK) return c->err.st;
  if (c->has_sched) return apply_schedule(c, c->sched);
  return MT_OK;
}

mt_status mt_set_schedule(mt_ctx *c, int32_t S, const int32_t *ranges) {
  if (!c) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (S < 0 || (S > 0 && !ranges)) return fail(c, MT_ERR_ARG, "bad ranges");
  std::vector<int> L = lengths(c);
  mt_error_info e = S > 0 ? validate(L, S, ranges) : mt_error_info{MT_E_SHAPE, -1, -1, -1};
  if (e.code != MT_E_OK) {
    c->err.info = e;
    return fail(c, MT_ERR_VALIDATION, "infeasible schedule");
  }
  Schedule s;
  s.S = S;
  s.ranges.assign(ranges, ranges + (size_t)S * L.size() * 2);
  return apply_schedule(c, s);
}

mt_status mt_set_schedule_pointers(mt_ctx *c, int32_t P, const int32_t *rho) {
  if (!c) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (P < 0 || (P > 0 && !rho)) return fail(c, MT_ERR_ARG, "bad rho");
  std::vector<int> L = lengths(c);
  Schedule s;
  mt_error_info e = pointers_to_ranges(L, P, rho, s.ranges);
  if (e.code != MT_E_OK) {
    c->err.info = e;
    return fail(c, MT_ERR_VALIDATION, "infeasible pointer matrix");
  }
  s.S = P + 1;
  return apply_schedule(c, s);
}

mt_status mt_num_stages(mt_ctx *c, int32_t *S) {
  if (!c || !S) return MT_ERR_ARG;
  if (!c->has_sched) return fail(c, MT_ERR_STATE, "no schedule set");
  *S = c->sched.S;
  return MT_OK;
}

mt_status mt_get_schedule(mt_ctx *c, int32_t *ranges) {
  if (!c || !ranges) return MT_ERR_ARG;
  if (!c->has_sched) return fail(c, MT_ERR_STATE, "no schedule set");
  memcpy(ranges, c->sched.ranges.data(), c->sched.ranges.size() * 4);
  return MT_OK;
}

mt_status mt_stage_assignment(mt_ctx *c, int32_t *stage_of) {
  if (!c || !stage_of) return MT_ERR_ARG;
  if (!c->has_sched) return fail(c, MT_ERR_STATE, "no schedule set");
  const int N = (int)c->T.size();
  for (int k = 0; k < c->sched.S; ++k)
    for (int t = 0; t < N; ++t)
      for (int j = c->sched.ranges[(k * N + t) * 2]; j < c->sched.ranges[(k * N + t) * 2 + 1]; ++j)
        stage_of[c->T[t].op_base + j] = k;
  return MT_OK;
}

mt_status mt_sm_partition(mt_ctx *c, int32_t *sms) {
  if (!c || !sms) return MT_ERR_ARG;
  if (!c->has_sched) return fail(c, MT_ERR_STATE, "no schedule set");
  memcpy(sms, c->sched.sms.data(), c->sched.sms.size() * 4);
  return MT_OK;
}

mt_status mt_stage_homes(mt_ctx *c, int32_t *grid, int32_t *homes) {
  if (!c || !grid) return MT_ERR_ARG;
  *grid = c->grid;
  if (!homes) return MT_OK;
  if (!c->has_sched) return fail(c, MT_ERR_STATE, "no schedule set");
  for (size_t i = 0; i < c->sched.home.size(); ++i) homes[i] = c->sched.home[i];
  return MT_OK;
}

mt_status mt_run_async(mt_ctx *c, const float *const *inputs, float *const *outputs, void *stream) {
  mt_status st = check_ready(c, true);
  if (st != MT_OK) return st;
  if (!inputs || !outputs) return fail(c, MT_ERR_ARG, "null inputs/outputs");
  RunArgs a = base_args(c, inputs, outputs);
  if (!c->stage_split) {
    CK(k_executor(c, a, c->grid, (cudaStream_t)stream));
    return MT_OK;
  }
  // debug/profiling mode (SURVEY d.5): one launch per stage -- the kernel boundary is the stage
  // barrier, so ncu attributes counters to stages; launch k stamps ts[4k .. 4k+3]
  const int S = c->sched.S, N = (int)c->T.size();
  unsigned long long *ts = (unsigned long long *)(c->ws + c->lay.run_ts);
  for (int k = 0; k < S; ++k) {
    RunArgs b = a;
    b.rng = a.rng + (size_t)k * N * 2;
    b.home = a.home + (size_t)k * c->grid;
    b.n_stages = 1;
    if (k > 0) b.n_pack = 0;
    b.no_reset = k < S - 1;
    b.ts = ts + 4 * k;
    b.ts_full = 1;
    CK(k_executor(c, b, c->grid, (cudaStream_t)stream));
  }
  return MT_OK;
}

mt_status mt_run(mt_ctx *c, const float *const *inputs, float *const *outputs, float *stage_us,
                 float *total_us, void *stream) {
  mt_status st = mt_run_async(c, inputs, outputs, stream);
  if (st != MT_OK) return st;
  const int S = c->sched.S;
  std::vector<unsigned long long> ts(c->stage_split ? 4 * S : S + 3);
  CK(cudaMemcpyAsync(ts.data(), c->ws + c->lay.run_ts, ts.size() * 8, cudaMemcpyDeviceToHost,
                     (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  st = check_device_error(c);
  if (st != MT_OK) return st;
  if (c->stage_split) {   // per launch k: [0] start, [1] end, [2] after the pack, [3] stage end
    if (total_us) *total_us = (float)((double)(ts[4 * (S - 1) + 1] - ts[0]) * 1e-3);
    if (stage_us)
      for (int k = 0; k < S; ++k) stage_us[k] = (float)((double)(ts[4 * k + 3] - ts[4 * k + 2]) * 1e-3);
    return MT_OK;
  }
  if (total_us) *total_us = (float)((double)(ts[1] - ts[0]) * 1e-3);
  if (stage_us)
    for (int k = 0; k < S; ++k) stage_us[k] = (float)((double)(ts[3 + k] - ts[2 + k]) * 1e-3);
  return MT_OK;
}

mt_status mt_run_host(mt_ctx *c, const float *const *hin, float *const *hout, float *total_us,
                      void *stream) {
  mt_status st = check_ready(c, true);
  if (st != MT_OK) return st;
  if (!hin || !hout) return fail(c, MT_ERR_ARG, "null inputs/outputs");
  cudaStream_t s = (cudaStream_t)stream;
  const int N = (int)c->T.size();
  const float *din[MT_MAXT];
  float *dout[MT_MAXT];
  CK(cudaEventRecord(c->ev0, s));
  for (int t = 0; t < N; ++t) {
    const mt_graph &g = c->T[t].g;
    int src = t;
    for (int u = 0; u < t; ++u)
      if (hin[u] == hin[t]) { src = u; break; }
    din[t] = (const float *)(c->ws + c->lay.stage_in_off[src]);
    dout[t] = (float *)(c->ws + c->lay.stage_out_off[t]);
    if (src == t)
      CK(cudaMemcpyAsync((void *)din[t], hin[t], (size_t)g.batch * g.in_c * g.in_h * g.in_w * 4,
                         cudaMemcpyHostToDevice, s));
  }
  RunArgs a = base_args(c, din, dout);
  CK(k_executor(c, a, c->grid, s));
  for (int t = 0; t < N; ++t) {
    const mt_node &last = c->T[t].nodes.back();
    CK(cudaMemcpyAsync(hout[t], dout[t], (size_t)c->T[t].g.batch * last.out_c * last.out_h * last.out_w * 4,
                       cudaMemcpyDeviceToHost, s));
  }
  CK(cudaEventRecord(c->ev1, s));
  CK(cudaEventSynchronize(c->ev1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  if (total_us) *total_us = ms * 1000.f;
  return check_device_error(c);
}

// ---- baselines: one launch per op, same tile functions (SURVEY d.2) -----------------------
static mt_status issue_op(mt_ctx *c, const RunArgs &a, int gid, cudaStream_t s) {
  CK(k_op(c, a, c->ops[gid].d, gid, c->n_sms, s));
  return MT_OK;
}

static mt_status issue_baseline(mt_ctx *c, int mode, const RunArgs &a, cudaStream_t main) {
  const int N = (int)c->T.size();
  mt_status st;
  auto pack_needed = [&](int t) {
    for (int q = 0; q < a.n_pack; ++q)
      if (a.pack_tenant[q] == t) return true;
    return false;
  };
  if (mode == MT_BASE_SEQ || mode == MT_BASE_SEQ_GRAPH) {
    for (int t = 0; t < N; ++t)
      if (pack_needed(t)) CK(k_pack(c, a, t, main));
    for (int t = 0; t < N; ++t)
      for (int j = 0; j < c->T[t].L; ++j)
        if ((st = issue_op(c, a, c->T[t].op_base + j, main)) != MT_OK) return st;
    return MT_OK;
  }
  // fork: every tenant stream waits for the main stream
  CK(cudaEventRecord(c->tev[0], main));
  for (int t = 0; t < N; ++t) CK(cudaStreamWaitEvent(c->streams[t], c->tev[0], 0));
  // packing first (a shared input is packed once; its readers wait for it)
  for (int t = 0; t < N; ++t)
    if (pack_needed(t)) CK(k_pack(c, a, t, c->streams[t]));
  std::vector<cudaEvent_t> packed_ev(N, nullptr);
  for (int t = 0; t < N; ++t) {
    int src = t;
    for (int q = 0; q < a.n_pack; ++q)
      if (a.packed[t] == a.packed[a.pack_tenant[q]]) src = a.pack_tenant[q];
    if (src != t) {
      CK(cudaEventRecord(c->tev[src], c->streams[src]));
      CK(cudaStreamWaitEvent(c->streams[t], c->tev[src], 0));
    }
  }
  if (mode == MT_BASE_MS_DFS) {
    for (int t = 0; t < N; ++t)
      for (int j = 0; j < c->T[t].L; ++j)
        if ((st = issue_op(c, a, c->T[t].op_base + j, c->streams[t])) != MT_OK) return st;
  } else if (mode == MT_BASE_MS_BFS || mode == MT_BASE_MS_GRAPH) {
    int maxL = 0;
    for (int t = 0; t < N; ++t) maxL = std::max(maxL, c->T[t].L);
    for (int j = 0; j < maxL; ++j)
      for (int t = 0; t < N; ++t)
        if (j < c->T[t].L)
          if ((st = issue_op(c, a, c->T[t].op_base + j, c->streams[t])) != MT_OK) return st;
  } else if (mode == MT_BASE_STAGE_EVENTS) {
    const Schedule &s = c->sched;
    for (int k = 0; k < s.S; ++k) {
      int maxlen = 0;
      for (int t = 0; t < N; ++t)
        maxlen = std::max(maxlen, s.ranges[(k * N + t) * 2 + 1] - s.ranges[(k * N + t) * 2]);
      for (int q = 0; q < maxlen; ++q)  // BFS issue within the stage
        for (int t = 0; t < N; ++t) {
          const int b = s.ranges[(k * N + t) * 2], e = s.ranges[(k * N + t) * 2 + 1];
          if (b + q < e)
            if ((st = issue_op(c, a, c->T[t].op_base + b + q, c->streams[t])) != MT_OK) return st;
        }
      if (k + 1 < s.S) {  // stage barrier: every stream waits for every stream
        for (int t = 0; t < N; ++t) CK(cudaEventRecord(c->tev[t], c->streams[t]));
        for (int t = 0; t < N; ++t)
          for (int u = 0; u < N; ++u)
            if (u != t) CK(cudaStreamWaitEvent(c->streams[t], c->tev[u], 0));
      }
    }
  } else {
    return fail(c, MT_ERR_ARG, "unknown baseline mode");
  }
  // join
  for (int t = 0; t < N; ++t) {
    CK(cudaEventRecord(c->tev[t], c->streams[t]));
    CK(cudaStreamWaitEvent(main, c->tev[t], 0));
  }
  return MT_OK;
}

mt_status mt_run_baseline(mt_ctx *c, int32_t mode, const float *const *inputs,
                          float *const *outputs, float *total_us, void *stream) {
  mt_status st = check_ready(c, mode == MT_BASE_STAGE_EVENTS);
  if (st != MT_OK) return st;
  if (!inputs || !outputs) return fail(c, MT_ERR_ARG, "null inputs/outputs");
  if (mode < MT_BASE_SEQ || mode > MT_BASE_STAGE_EVENTS) return fail(c, MT_ERR_ARG, "bad mode");
  cudaStream_t s = (cudaStream_t)stream;
  const int N = (int)c->T.size();
  RunArgs a = base_args(c, inputs, outputs);
  if (mode == MT_BASE_SEQ_GRAPH || mode == MT_BASE_MS_GRAPH) {
    bool same = c->gexec[mode] != nullptr;
    for (int t = 0; t < N && same; ++t) same = c->g_in[mode][t] == inputs[t] && c->g_out[mode][t] == outputs[t];
    if (!same) {
      if (c->gexec[mode]) { cudaGraphExecDestroy(c->gexec[mode]); c->gexec[mode] = nullptr; }
      cudaStream_t cap;
      CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      st = issue_baseline(c, mode, a, cap);
      cudaGraph_t graph;
      cudaError_t e = cudaStreamEndCapture(cap, &graph);
      cudaStreamDestroy(cap);
      if (st != MT_OK) return st;
      if (e != cudaSuccess) return fail(c, MT_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(e));
      CK(cudaGraphInstantiate(&c->gexec[mode], graph, 0));
      cudaGraphDestroy(graph);
      for (int t = 0; t < N; ++t) { c->g_in[mode][t] = inputs[t]; c->g_out[mode][t] = outputs[t]; }
    }
    CK(cudaEventRecord(c->ev0, s));
    CK(cudaGraphLaunch(c->gexec[mode], s));
    CK(cudaEventRecord(c->ev1, s));
  } else {
    CK(cudaEventRecord(c->ev0, s));
    st = issue_baseline(c, mode, a, s);
    if (st != MT_OK) return st;
    CK(cudaEventRecord(c->ev1, s));
  }
  CK(cudaEventSynchronize(c->ev1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  if (total_us) *total_us = ms * 1000.f;
  return check_device_error(c);   // a device timeout fails this call and is cleared here
}

// ---- profiling (a10) ---------------------------------------------------------------------
static mt_status profile_impl(mt_ctx *c, int32_t n, const std::vector<Schedule> &cands,
                              const std::vector<int> &valid, const float *const *inputs,
                              float *const *outputs, int32_t warmup, int32_t iters, float *lat_us,
                              int32_t *status, cudaStream_t s) {
  const int N = (int)c->T.size();
  const int runs = warmup + iters;
  const size_t ts_slots = c->lay.prof_ts_bytes / 16;
  if (runs < 1 || (size_t)runs > ts_slots) return fail(c, MT_ERR_ARG, "warmup+iters out of range");
  RunArgs base = base_args(c, inputs, outputs);
  int i = 0;
  while (i < n) {
    // pack as many candidates as fit into the profile area / timestamp area
    size_t used = 0, run_slot = 0;
    std::vector<std::pair<int, std::pair<size_t, size_t>>> chunk;  // cand, (rng off, home off)
    std::vector<char> host(c->lay.prof_area_bytes);
    int j = i;
    for (; j < n; ++j) {
      if (!valid[j]) continue;
      const Schedule &sc = cands[j];
      const size_t rb = (size_t)sc.S * N * 2 * 4, hb = (size_t)sc.S * c->grid;
      const size_t need = rup(rb, 256) + rup(hb, 256);
      if (used + need > c->lay.prof_area_bytes || (run_slot + runs) > ts_slots) break;
      to_global_ranges(c, sc, (int32_t *)(host.data() + used));
      memcpy(host.data() + used + rup(rb, 256), sc.home.data(), hb);
      chunk.push_back({j, {used, used + rup(rb, 256)}});
      used += need;
      run_slot += runs;
    }
    if (chunk.empty() && j < n) return fail(c, MT_ERR_ARG, "candidate schedule too large for the profile area");
    if (!chunk.empty()) {
      CK(cudaMemcpyAsync(c->ws + c->lay.prof_area, host.data(), used, cudaMemcpyHostToDevice, s));
      size_t slot = 0;
      for (auto &ch : chunk) {
        RunArgs a = base;
        a.rng = (const int32_t *)(c->ws + c->lay.prof_area + ch.second.first);
        a.home = (const uint8_t *)(c->ws + c->lay.prof_area + ch.second.second);
        a.n_stages = cands[ch.first].S;
        a.ts_full = 0;
        for (int r = 0; r < runs; ++r, ++slot) {
          a.ts = (unsigned long long *)(c->ws + c->lay.prof_ts + slot * 16);
          CK(k_executor(c, a, c->grid, s));
        }
      }
      std::vector<unsigned long long> ts(slot * 2);
      CK(cudaMemcpyAsync(ts.data(), c->ws + c->lay.prof_ts, ts.size() * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      mt_status st = check_device_error(c);
      if (st != MT_OK) return st;
      slot = 0;
      for (auto &ch : chunk) {
        double sum = 0;
        for (int r = 0; r < runs; ++r, ++slot)
          if (r >= warmup) sum += (double)(ts[slot * 2 + 1] - ts[slot * 2]) * 1e-3;
        lat_us[ch.first] = (float)(sum / iters);
        status[ch.first] = MT_OK;
      }
    }
    i = j;
  }
  for (int k = 0; k < n; ++k)
    if (!valid[k]) { lat_us[k] = NAN; status[k] = MT_ERR_VALIDATION; }
  return MT_OK;
}

mt_status mt_profile_batch(mt_ctx *c, int32_t n, const int32_t *cand_nstages, const int32_t *cand_ranges,
                           const float *const *inputs, float *const *outputs, int32_t warmup,
                           int32_t iters, float *lat_us, int32_t *status, void *stream) {
  mt_status st = check_ready(c, false);
  if (st != MT_OK) return st;
  if (n < 0 || (n > 0 && (!cand_nstages || !cand_ranges || !lat_us || !status)) || iters < 1 || warmup < 0)
    return fail(c, MT_ERR_ARG, "bad profile arguments");
  std::vector<int> L = lengths(c);
  const int N = (int)L.size();
  std::vector<Schedule> cands(n);
  std::vector<int> valid(n, 0);
  size_t off = 0;
  for (int k = 0; k < n; ++k) {
    const int S = cand_nstages[k];
    if (S < 1) continue;
    const int32_t *r = cand_ranges + off;
    off += (size_t)S * N * 2;
    if (validate(L, S, r).code != MT_E_OK) continue;
    cands[k].S = S;
    cands[k].ranges.assign(r, r + (size_t)S * N * 2);
    build_stage_plan(c, cands[k]);
    valid[k] = 1;
  }
  return profile_impl(c, n, cands, valid, inputs, outputs, warmup, iters, lat_us, status, (cudaStream_t)stream);
}

mt_status mt_profile_batch_pointers(mt_ctx *c, int32_t n, const int32_t *cand_P, const int32_t *cand_rho,
                                    const float *const *inputs, float *const *outputs, int32_t warmup,
                                    int32_t iters, float *lat_us, int32_t *status, void *stream) {
  mt_status st = check_ready(c, false);
  if (st != MT_OK) return st;
  if (n < 0 || (n > 0 && (!cand_P || !cand_rho || !lat_us || !status)) || iters < 1 || warmup < 0)
    return fail(c, MT_ERR_ARG, "bad profile arguments");
  std::vector<int> L = lengths(c);
  const int N = (int)L.size();
  std::vector<Schedule> cands(n);
  std::vector<int> valid(n, 0);
  size_t off = 0;
  for (int k = 0; k < n; ++k) {
    const int P = cand_P[k];
    if (P < 0) continue;
    const int32_t *rho = cand_rho + off;
    off += (size_t)N * P;
    if (pointers_to_ranges(L, P, rho, cands[k].ranges).code != MT_E_OK) continue;
    cands[k].S = P + 1;
    build_stage_plan(c, cands[k]);
    valid[k] = 1;
  }
  return profile_impl(c, n, cands, valid, inputs, outputs, warmup, iters, lat_us, status, (cudaStream_t)stream);
}

mt_status mt_estimate_batch_pointers(mt_ctx *c, const mt_cost_params *p, int32_t n, const int32_t *cand_P,
                                     const int32_t *cand_rho, double *est_us, int32_t *status) {
  if (!c || !p) return MT_ERR_ARG;
  if (!c->loaded) return fail(c, MT_ERR_STATE, "no graphs loaded");
  if (n < 0 || (n > 0 && (!cand_P || !cand_rho || !est_us || !status)) || !(p->peak_flops > 0) ||
      !(p->mem_bw > 0) || p->max_concurrency < 1)
    return fail(c, MT_ERR_ARG, "bad estimate arguments");
  std::vector<int> L = lengths(c);
  const int N = (int)L.size();
  std::vector<std::vector<double>> F(N), B(N);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < L[i]; ++j) {
      const HostOp &h = c->ops[c->T[i].op_base + j];
      F[i].push_back((double)h.flops);
      B[i].push_back((double)h.bytes);
    }
  size_t off = 0;
  std::vector<int32_t> ranges;
  for (int k = 0; k < n; ++k) {
    const int P = cand_P[k];
    est_us[k] = std::numeric_limits<double>::quiet_NaN();
    status[k] = MT_ERR_VALIDATION;
    if (P < 0) continue;
    const int32_t *rho = cand_rho + off;
    off += (size_t)N * P;
    if (pointers_to_ranges(L, P, rho, ranges).code != MT_E_OK) continue;
    est_us[k] = estimate_schedule(F, B, P + 1, ranges.data(), *p);
    status[k] = MT_OK;
  }
  return MT_OK;
}

mt_status mt_get_activation(mt_ctx *c, int32_t t, int32_t op, void *host, size_t bytes) {
  mt_status st = check_ready(c, false);
  if (st != MT_OK) return st;
  if (t < 0 || t >= (int)c->T.size() || op < 0 || op >= c->T[t].L || !host) return fail(c, MT_ERR_ARG, "bad op");
  const HostOp &h = c->ops[c->T[t].op_base + op];
  if (h.out.buf < 0) return fail(c, MT_ERR_ARG, "final op has no activation buffer");
  const int eb = h.d.prec == MT_PREC_BF16 ? 2 : 4;
  const size_t rows = (size_t)h.d.N * h.d.Ho * h.d.Wo;
  if (bytes != rows * h.d.Co * eb) return fail(c, MT_ERR_ARG, "bytes mismatch");
  const char *src = c->ws + c->lay.acts + c->bufs[h.out.buf].off + (size_t)h.out.co * eb;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy2D(host, (size_t)h.d.Co * eb, src, (size_t)h.out.cs * eb, (size_t)h.d.Co * eb, rows,
                  cudaMemcpyDeviceToHost));
  return MT_OK;
}

mt_status mt_set_trace(mt_ctx *c, void *dev, int64_t capacity) {
  mt_status st = check_ready(c, false);
  if (st != MT_OK) return st;
  if (capacity < 0 || capacity > (1 << 30) || (capacity > 0 && !dev)) return fail(c, MT_ERR_ARG, "bad trace buffer");
  drop_graphs(c);
  c->trace = capacity > 0 ? (unsigned long long *)dev : nullptr;
  c->trace_cap = capacity;
  CK(cudaMemset(c->ws + c->lay.ctl + offsetof(CtlBlock, trace_count), 0, sizeof(unsigned)));
  return MT_OK;
}

mt_status mt_trace_count(mt_ctx *c, int64_t *n) {
  mt_status st = check_ready(c, false);
  if (st != MT_OK) return st;
  if (!n) return fail(c, MT_ERR_ARG, "null");
  unsigned v = 0;
  CK(cudaMemcpy(&v, c->ws + c->lay.ctl + offsetof(CtlBlock, trace_count), sizeof v, cudaMemcpyDeviceToHost));
  *n = v;
  return MT_OK;
}

mt_status mt_last_error_info(mt_ctx *c, mt_error_info *info) {
  if (!c || !info) return MT_ERR_ARG;
  *info = c->err.info;
  return MT_OK;
}

const char *mt_last_error(mt_ctx *c) { return c ? c->err.msg.c_str() : "null context"; }

}  // extern "C"
