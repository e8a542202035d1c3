// Schedule IR (a2) and runtime-aware SM partition (a3) -- pure host functions.
//
// These restate the paper's IR (§3.2): Eq.3 pointer split, Eq.4/5 stages
// with possibly empty ("None") slices, Eq.6 schedule, Eq.8 T(G, rho)
// (P:386-393).  Semantics must equal oracle/ir.py bit for bit (tests/test_ir_parity.py); the
// two implementations share no code.
#include "plan.h"

#include <algorithm>

namespace mt {

static mt_error_info E(int code, int s, int t, int op) { return mt_error_info{code, s, t, op}; }

// First violation, scanning stages k = 0..S-1, tenants i = 0..N-1 (R1-R4).
mt_error_info validate(const std::vector<int> &L, int S, const int32_t *r) {
  const int N = (int)L.size();
  if (S < 1) return E(MT_E_SHAPE, -1, -1, -1);
  std::vector<int> pos(N, 0);
  for (int k = 0; k < S; ++k) {
    bool all_empty = true;
    for (int i = 0; i < N; ++i) {
      const int b = r[(k * N + i) * 2 + 0], e = r[(k * N + i) * 2 + 1];
      if (b < 0 || e > L[i] || b > e) return E(MT_E_RANGE, k, i, b);
      if (b != pos[i]) return E(MT_E_NONCONTIG, k, i, pos[i]);
      if (e > b) all_empty = false;
      pos[i] = e;
    }
    if (all_empty) return E(MT_E_EMPTY_STAGE, k, -1, -1);
  }
  for (int i = 0; i < N; ++i)
    if (pos[i] != L[i]) return E(MT_E_INCOMPLETE, S, i, pos[i]);
  return E(MT_E_OK, -1, -1, -1);
}

// tau = T(G, rho): stage k slice of tenant i = [rho_i[k-1], rho_i[k]), rho_i[-1] = 0,
// rho_i[P] = L_i (Eq.3: (3,5,7) on 10 ops -> [1..3],[4,5],[6,7],[8..10]).
mt_error_info pointers_to_ranges(const std::vector<int> &L, int P, const int32_t *rho,
                                 std::vector<int32_t> &ranges) {
  const int N = (int)L.size();
  if (P < 0) return E(MT_E_SHAPE, -1, -1, -1);
  for (int i = 0; i < N; ++i) {
    int prev = 0;
    for (int k = 0; k < P; ++k) {
      const int p = rho[i * P + k];
      if (p < 0 || p > L[i]) return E(MT_E_ROW_RANGE, k, i, p);
      if (p < prev) return E(MT_E_ROW_ORDER, k, i, p);
      prev = p;
    }
  }
  const int S = P + 1;
  ranges.assign((size_t)S * N * 2, 0);
  for (int k = 0; k < S; ++k)
    for (int i = 0; i < N; ++i) {
      ranges[(k * N + i) * 2 + 0] = k == 0 ? 0 : rho[i * P + k - 1];
      ranges[(k * N + i) * 2 + 1] = k == P ? L[i] : rho[i * P + k];
    }
  return validate(L, S, ranges.data());
}

// n_t proportional to w_t by largest remainder; every active tenant gets >= 1 CTA; ties in the
// remainder go to the lower tenant index; inactive tenants get 0; all weights 0 -> equal.
static std::vector<int> lr_split(const std::vector<bool> &active, const std::vector<__int128> &w,
                                 int n_sms) {
  const int N = (int)active.size();
  std::vector<int> out(N, 0);
  int A = 0;
  __int128 W = 0;
  for (int t = 0; t < N; ++t)
    if (active[t]) { ++A; W += w[t]; }
  if (A == 0) return out;
  std::vector<__int128> ww(N, 0);
  for (int t = 0; t < N; ++t) ww[t] = active[t] ? (W == 0 ? (__int128)1 : w[t]) : 0;
  if (W == 0) W = A;
  const __int128 R = n_sms - A;
  std::vector<__int128> rem(N, 0);
  __int128 used = 0;
  for (int t = 0; t < N; ++t) {
    if (!active[t]) continue;
    const __int128 q = R * ww[t] / W;
    rem[t] = R * ww[t] % W;
    out[t] = 1 + (int)q;
    used += q;
  }
  int left = (int)(R - used);
  std::vector<int> order;
  for (int t = 0; t < N; ++t)
    if (active[t]) order.push_back(t);
  // stable selection: descending remainder, ascending index
  for (int a = 0; a < (int)order.size(); ++a)
    for (int b = a + 1; b < (int)order.size(); ++b) {
      const int x = order[a], y = order[b];
      if (rem[y] > rem[x] || (rem[y] == rem[x] && y < x)) { order[a] = y; order[b] = x; }
    }
  for (int k = 0; k < left && k < (int)order.size(); ++k) out[order[k]] += 1;
  return out;
}

// SURVEY §8(a) a3 tile cap: n_t <= cap_t (the most tiles of one op of the slice: more CTAs cannot
// run in parallel on the slice), the excess redistributed.  Water-filling: split over the free
// tenants U (initially every active one) with lr_split; the tenants of U over their cap are fixed
// at the cap and leave U; repeat with the SMs left.  If every tenant of U is over its cap the
// last split stands (the GPU cannot be filled within the caps; the excess stays proportional).
std::vector<int> sm_partition(const std::vector<bool> &active, const std::vector<__int128> &w,
                              int n_sms, const std::vector<int64_t> *caps) {
  std::vector<int> out = lr_split(active, w, n_sms);
  if (!caps) return out;
  const int N = (int)active.size();
  std::vector<bool> U = active;
  int budget = n_sms;
  while (true) {
    std::vector<int> part = lr_split(U, w, budget);
    int nu = 0, nover = 0;
    for (int t = 0; t < N; ++t)
      if (U[t]) { ++nu; nover += part[t] > (*caps)[t]; }
    if (nu == 0) break;
    if (nover == 0 || nover == nu) {
      for (int t = 0; t < N; ++t)
        if (U[t]) out[t] = part[t];
      break;
    }
    for (int t = 0; t < N; ++t)
      if (U[t] && part[t] > (*caps)[t]) {
        out[t] = (int)(*caps)[t];
        budget -= out[t];
        U[t] = false;
      }
  }
  return out;
}

// Latency-balanced partition (reading R16b).  Tenant t's slice is a list of work items
// (tiles, ns per tile); with n CTAs its estimated time is E_t(n) = sum ceil(tiles / n) * ns
// (a tenant's ops run one after another, each in ceil(tiles / n) waves).  Every active tenant
// starts with one CTA; each remaining CTA goes to the tenant with the largest E_t among those
// with n_t < cap_t (cap = most tiles of one item; more CTAs than that cannot shorten the slice),
// ties to the lower index; once every tenant is capped, to the largest E_t regardless.  Greedy
// "feed the current maximum" minimises max_t E_t exactly (each E_t is non-increasing in n).
// mode 2 (work/span, Brent): E_t(n) = ceil(W_t / n) + S_t with W_t = sum tiles * ns (busy time)
// and S_t = sum (ns + hop_ns) (the chain's latency floor: consecutive ops overlap as a wavefront,
// so a tenant is either throughput-bound on its n CTAs or latency-bound on its chain).
static int64_t est_time(const std::vector<std::pair<int64_t, int64_t>> &items, int n, int mode,
                        int64_t hop_ns) {
  int64_t e = 0;
  if (mode == 2) {
    int64_t w = 0;
    for (const auto &it : items) {
      w += it.first * it.second;
      e += it.second + hop_ns;
    }
    return e + (w + n - 1) / n;
  }
  for (const auto &it : items) e += (it.first + n - 1) / n * it.second;
  return e;
}

std::vector<int> sm_partition_balanced(const std::vector<bool> &active,
                                       const std::vector<std::vector<std::pair<int64_t, int64_t>>> &items,
                                       int n_sms, int mode, int64_t hop_ns) {
  const int N = (int)active.size();
  std::vector<int> out(N, 0);
  std::vector<int64_t> E(N, 0), cap(N, 0);
  int A = 0;
  for (int t = 0; t < N; ++t) {
    if (!active[t]) continue;
    ++A;
    out[t] = 1;
    for (const auto &it : items[t]) cap[t] = std::max(cap[t], it.first);
    E[t] = est_time(items[t], 1, mode, hop_ns);
  }
  if (A == 0) return out;
  for (int left = n_sms - A; left > 0; --left) {
    int best = -1;
    for (int pass = 0; pass < 2 && best < 0; ++pass)
      for (int t = 0; t < N; ++t) {
        if (!active[t] || (pass == 0 && out[t] >= cap[t])) continue;
        if (best < 0 || E[t] > E[best]) best = t;
      }
    out[best] += 1;
    E[best] = est_time(items[best], out[best], mode, hop_ns);
  }
  return out;
}

// Pre-filter estimate (include/mt.h mt_estimate_batch_pointers; reading R19).
double estimate_schedule(const std::vector<std::vector<double>> &flops,
                         const std::vector<std::vector<double>> &bytes, int S, const int32_t *ranges,
                         const mt_cost_params &p) {
  const int N = (int)flops.size();
  const double us = 1e6;
  double total = 0.0;
  for (int k = 0; k < S; ++k) {
    double C = 0.0, M = 0.0, chain_max = 0.0;
    int n_c = 0, n_m = 0;
    for (int i = 0; i < N; ++i) {
      const int a = ranges[(k * N + i) * 2], b = ranges[(k * N + i) * 2 + 1];
      double chain = 0.0;
      bool has_c = false, has_m = false;
      for (int j = a; j < b; ++j) {
        const double tc = flops[i][j] / p.peak_flops * us, tm = bytes[i][j] / p.mem_bw * us;
        chain += std::max(tc, tm) + p.op_latency_us;
        if (tc >= tm) { C += flops[i][j]; has_c = true; }
        else { M += bytes[i][j]; has_m = true; }
      }
      n_c += has_c;
      n_m += has_m;
      chain_max = std::max(chain_max, chain);
    }
    const double mc = (double)std::max(1, p.max_concurrency);
    const double compute = C / p.peak_flops * us * (1.0 + p.c_compute * std::max(0, n_c - 1) / mc);
    const double memory = M / p.mem_bw * us * (1.0 + p.c_memory * std::max(0, n_m - 1) / mc);
    total += std::max(std::max(compute, memory), chain_max) + p.sync_us;
  }
  return total;
}

}  // namespace mt
