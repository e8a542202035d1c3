// Host plan compiler: graph ingest (a1), schedule IR (a2), stage plan (a3), workspace layout.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/mt.h"
#include "mt_types.h"

namespace mt {

struct Tenant {
  mt_graph g{};
  std::vector<mt_node> nodes;
  int L = 0;          // number of ops
  int op_base = 0;    // global id of op 0
  int cpad = 8;       // stored channels of the packed graph input
  bool tma_input = false;   // a TMA conv reads the packed input: keep the tenant's own pack slot
};

struct Buf {          // one activation buffer (NHWC), possibly shared by a concat group
  int64_t off = 0;    // byte offset in the activation arena
  int64_t bytes = 0;
  int C = 0;          // channel stride
};

struct TensorView { int buf = -1; int cs = 0; int co = 0; int C = 0; bool graph_in = false; };

struct WPack {        // one weight repack job executed at bind
  int op = -1;
  int mode = 0;       // 1 conv TC bf16, 2 conv SIMT fp32, 3 dw, 4 fc
  const float *src = nullptr;
  int64_t dst_off = 0;  // in weight arena
  int64_t bytes = 0;
};

struct HostOp {
  OpDesc d{};
  int64_t flops = 0, bytes = 0;     // algorithmic cost (SURVEY d.4)
  int32_t work_tiles[2] = {0, 0};   // latency model (R16b): compute tiles, reduce tiles
  int64_t work_ns[2] = {0, 0};      // ... and the estimated ns of one tile of each
  TensorView out, res;
  TensorView in[MT_MAXIN];
  int n_in = 0;
  int64_t w_off = -1, ws_off = -1, ws_bytes = 0;
  const float *scale = nullptr, *shift = nullptr;
  int out_buf = -1;                 // -1: final op (user output)
};

struct Schedule {
  int S = 0;
  std::vector<int32_t> ranges;      // [S][N][2], tenant-local op indices
  std::vector<int32_t> sms;         // [S][N]
  std::vector<uint8_t> home;        // [S][grid]
};

struct Layout {
  size_t gates = 0;   // [n_ops]: claim-ahead gate op (-1 none), MT_OPT_CLAIM_DEPTH
  size_t ctl = 0, claim = 0, done = 0, blk = 0, splitcnt = 0, ops = 0, tmaps = 0, sched_rng = 0, sched_home = 0,
         prof_area = 0, prof_ts = 0, run_ts = 0, packed = 0, stage_in = 0, stage_out = 0,
         weights = 0, acts = 0, partials = 0, total = 0;
  size_t prof_area_bytes = 0, prof_ts_bytes = 0;
  std::vector<size_t> packed_off, stage_in_off, stage_out_off;
  size_t counters_bytes = 0;
};

// status + error message helper
struct Err {
  mt_status st = MT_OK;
  std::string msg;
  mt_error_info info{0, -1, -1, -1};
};

// ---- schedule IR (pure functions; mirror oracle/ir.py semantics bit for bit) --------------
mt_error_info validate(const std::vector<int> &L, int S, const int32_t *ranges);
// T(G, rho): returns info (code MT_E_OK on success) and fills ranges [P+1][N][2]
mt_error_info pointers_to_ranges(const std::vector<int> &L, int P, const int32_t *rho,
                                 std::vector<int32_t> &ranges);
std::vector<int> sm_partition(const std::vector<bool> &active,
                              const std::vector<__int128> &w, int n_sms,
                              const std::vector<int64_t> *caps = nullptr);
// latency-balanced partition: items[t] = (tiles, ns per tile) of each op of tenant t's slice
std::vector<int> sm_partition_balanced(const std::vector<bool> &active,
                                       const std::vector<std::vector<std::pair<int64_t, int64_t>>> &items,
                                       int n_sms, int mode, int64_t hop_ns);
// analytic pre-filter cost of one valid schedule (ranges [S][N][2]); flops/bytes per tenant op
double estimate_schedule(const std::vector<std::vector<double>> &flops,
                         const std::vector<std::vector<double>> &bytes, int S, const int32_t *ranges,
                         const mt_cost_params &p);

}  // namespace mt
