// (4) Event-level schedule replay on the host CPU, one thread per commodity.
//
// Restates collsched.simulator.simulate (pkg/src/collsched/simulator.py:
// 58-208, with _check_capacity :211-223 and _check_switch_rest :226-235) for
// copy / no-copy switches: the emitted event list itself is replayed, not the
// flows it came from. Events are ordered by (epoch, str(source), str(src),
// str(dst), chunk) with a stable sort (the reference's sorted()); each
// (source, chunk) commodity's holdings depend only on its own events, so the
// causality replay runs one commodity per task in parallel, with the same
// floating-point operations in the same order as the reference. Capacity
// loads are summed per (edge, epoch) in the global sorted order and checked
// per window; deliveries are accumulated per demanded entry in (arrival,
// fraction) order. The host wrapper (simulate.py) computes the per-edge
// window, budget and delay with the reference's exact rational arithmetic
// and formats the violations.

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdint>
#include <numeric>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace {

constexpr double kWhole = 1.0 - 1e-9;  // simulator.py:22

struct SwRec {
  int64_t usable;
  double qty, used;
  bool whole;
};

struct FracRec {
  int64_t usable;
  double qty;
};

struct CommodityOut {
  std::vector<int64_t> causality;                      // original event ids
  std::vector<std::array<int64_t, 2>> sw_rest;         // (switch node, usable epoch)
};

struct Sim {
  const teccl_sim_desc* d;
  int64_t n;
  const int32_t *src, *dst, *edge, *epoch, *source, *chunk;
  const double* frac;
  std::vector<int64_t> order;                 // sorted event ids
  // commodities: (source node, chunk) -> id
  std::vector<int64_t> comm_of_event;         // per sorted position
  std::vector<std::vector<int64_t>> comm_events;  // sorted positions per commodity
  std::vector<int32_t> comm_source, comm_chunk;
  std::vector<uint8_t> comm_demanded;
  // demanded entries of each commodity: (dst node, entry id)
  std::vector<std::vector<std::pair<int32_t, int64_t>>> comm_entries;
  std::vector<std::vector<std::pair<int64_t, double>>> deliveries;  // per entry
};

inline uint64_t key2(int64_t a, int64_t b) { return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b; }

void replay_commodity(Sim& S, int64_t c, CommodityOut& out) {
  const teccl_sim_desc& d = *S.d;
  const double tol = d.tolerance;
  const bool no_copy = d.switch_mode == 1;
  const int32_t s = S.comm_source[c], ch = S.comm_chunk[c];
  (void)ch;
  // holdings of this commodity
  std::unordered_map<int32_t, int64_t> copy_from;               // node -> first epoch a whole copy is usable
  std::unordered_map<int32_t, std::vector<FracRec>> frac_pool;  // node -> fractional arrivals (insertion order)
  std::unordered_map<int32_t, size_t> frac_live;                // node -> first not-exhausted record
  std::vector<SwRec> sw;                                        // switch arrivals (insertion order)
  std::vector<int32_t> sw_node;
  std::unordered_map<uint64_t, std::vector<int32_t>> sw_at;     // (node, usable) -> records
  if (S.comm_demanded[c]) copy_from[s] = 0;
  const auto& ents = S.comm_entries[c];

  auto draw = [&](int32_t node, int64_t k, double qty) -> bool {
    if (d.node_is_switch[node]) {
      auto it = sw_at.find(key2(node, k));
      if (it == sw_at.end()) return qty <= tol;  // no records: remaining = qty
      const std::vector<int32_t>& recs = it->second;
      if (!no_copy)
        for (int32_t r : recs)
          if (sw[r].whole) {
            sw[r].used += qty;
            return true;
          }
      double remaining = qty;
      for (int32_t r : recs) {
        const double fr = sw[r].qty - sw[r].used;
        if (fr > tol) {
          const double take = std::min(fr, remaining);
          sw[r].used += take;
          remaining -= take;
          if (remaining <= tol) return true;
        }
      }
      return remaining <= tol;
    }
    auto cf = copy_from.find(node);
    if (cf != copy_from.end() && cf->second <= k) return true;
    double remaining = qty;
    auto fp = frac_pool.find(node);
    if (fp != frac_pool.end()) {
      std::vector<FracRec>& recs = fp->second;
      size_t& live = frac_live[node];
      while (live < recs.size() && !(recs[live].qty > tol)) ++live;  // exhausted records stay exhausted
      for (size_t i = live; i < recs.size(); ++i) {
        FracRec& r = recs[i];
        if (r.usable <= k && r.qty > tol) {
          const double take = std::min(r.qty, remaining);
          r.qty -= take;
          remaining -= take;
          if (remaining <= tol) return true;
        }
      }
    }
    return remaining <= tol;
  };

  for (int64_t pos : S.comm_events[c]) {
    const int64_t e = S.order[pos];
    const int32_t from = S.src[e], to = S.dst[e];
    const int64_t k = S.epoch[e];
    const double q = S.frac[e];
    if (!draw(from, k, q)) out.causality.push_back(e);
    const int64_t arr = k + d.edge_delta[S.edge[e]];
    // register_arrival (simulator.py:119-131)
    if (d.node_is_switch[to]) {
      sw.push_back(SwRec{arr + 1, q, 0.0, q >= kWhole});
      sw_node.push_back(to);
      sw_at[key2(to, arr + 1)].push_back((int32_t)sw.size() - 1);
    } else if (q >= kWhole) {
      auto cf = copy_from.find(to);
      if (cf == copy_from.end() || arr + 1 < cf->second) copy_from[to] = arr + 1;
    } else {
      frac_pool[to].push_back(FracRec{arr + 1, q});
    }
    for (const auto& en : ents)
      if (en.first == to) S.deliveries[en.second].push_back({arr, q});
  }
  // switch rest (simulator.py:226-235), records in insertion order
  for (size_t r = 0; r < sw.size(); ++r) {
    const SwRec& R = sw[r];
    bool bad;
    if (no_copy || !R.whole) bad = R.qty - R.used > tol;
    else bad = R.used == 0.0;
    if (bad) out.sw_rest.push_back({sw_node[r], R.usable});
  }
}

struct SimResult {
  std::vector<int64_t> causality;                   // original event ids, replay order
  std::vector<std::array<int64_t, 2>> capacity;     // (edge, epoch)
  std::vector<std::array<int64_t, 4>> sw_rest;      // (source, chunk, switch, usable)
  std::vector<int32_t> entry_done;                  // per entry: completion epoch or -1
};

}  // namespace

extern "C" int teccl_simulate(const teccl_sim_desc* d, int64_t n_events, const int32_t* ev_source,
                              const int32_t* ev_chunk, const int32_t* ev_src, const int32_t* ev_dst,
                              const int32_t* ev_edge, const int32_t* ev_epoch, const double* ev_frac,
                              const int32_t* source_rank, const int32_t* node_rank, int32_t threads,
                              void** out, int64_t* counts4) {
  if (!d || !out || !counts4 || n_events < 0 || (n_events > 0 && (!ev_source || !ev_chunk || !ev_src ||
      !ev_dst || !ev_edge || !ev_epoch || !ev_frac)) || !source_rank || !node_rank) {
    teccl::set_error("teccl_simulate: null argument");
    return TECCL_EINVAL;
  }
  if (d->switch_mode != 0 && d->switch_mode != 1) {
    teccl::set_error("teccl_simulate: switch_mode must be 0 (copy) or 1 (no-copy)");
    return TECCL_EINVAL;
  }
  for (int64_t e = 0; e < n_events; ++e)
    if (ev_edge[e] < 0 || ev_edge[e] >= d->num_edges || ev_epoch[e] < 0) {
      teccl::set_error("teccl_simulate: event with a bad edge or a negative epoch");
      return TECCL_EINVAL;
    }
  Sim S;
  S.d = d;
  S.n = n_events;
  S.src = ev_src; S.dst = ev_dst; S.edge = ev_edge; S.epoch = ev_epoch;
  S.source = ev_source; S.chunk = ev_chunk; S.frac = ev_frac;
  // stable sort by (epoch, str(source), str(src), str(dst), chunk) (simulator.py:94-95)
  S.order.resize(n_events);
  std::iota(S.order.begin(), S.order.end(), 0);
  std::stable_sort(S.order.begin(), S.order.end(), [&](int64_t a, int64_t b) {
    if (ev_epoch[a] != ev_epoch[b]) return ev_epoch[a] < ev_epoch[b];
    const int32_t sa = source_rank[ev_source[a]], sb = source_rank[ev_source[b]];
    if (sa != sb) return sa < sb;
    const int32_t ra = node_rank[ev_src[a]], rb = node_rank[ev_src[b]];
    if (ra != rb) return ra < rb;
    const int32_t da = node_rank[ev_dst[a]], db = node_rank[ev_dst[b]];
    if (da != db) return da < db;
    return ev_chunk[a] < ev_chunk[b];
  });
  // commodities: demanded ones first (entry order), then any others events mention
  std::unordered_map<uint64_t, int64_t> cid;
  auto comm = [&](int32_t s, int32_t c) -> int64_t {
    auto it = cid.find(key2(s, c));
    if (it != cid.end()) return it->second;
    const int64_t id = (int64_t)S.comm_source.size();
    cid[key2(s, c)] = id;
    S.comm_source.push_back(s);
    S.comm_chunk.push_back(c);
    S.comm_demanded.push_back(0);
    S.comm_entries.emplace_back();
    S.comm_events.emplace_back();
    return id;
  };
  S.deliveries.resize(d->num_entries);
  for (int64_t i = 0; i < d->num_entries; ++i) {
    const int64_t c = comm(d->entry_source[i], d->entry_chunk[i]);
    S.comm_demanded[c] = 1;
    S.comm_entries[c].push_back({d->entry_dst[i], i});
  }
  for (int64_t pos = 0; pos < n_events; ++pos) {
    const int64_t e = S.order[pos];
    S.comm_events[comm(ev_source[e], ev_chunk[e])].push_back(pos);
  }
  const int64_t nc = (int64_t)S.comm_source.size();
  std::vector<CommodityOut> co(nc);
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, nc));
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (int64_t c; (c = next.fetch_add(1)) < nc;) replay_commodity(S, c, co[c]);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();

  SimResult* R = new SimResult();
  // causality violations in replay order (merge the commodities' lists by sorted position)
  {
    std::vector<std::pair<int64_t, int64_t>> pos;  // (sorted position, event)
    std::vector<int64_t> rank(n_events);
    for (int64_t p = 0; p < n_events; ++p) rank[S.order[p]] = p;
    for (const auto& o : co)
      for (int64_t e : o.causality) pos.push_back({rank[e], e});
    std::sort(pos.begin(), pos.end());
    for (const auto& pe : pos) R->causality.push_back(pe.second);
  }
  // capacity per (edge, window) (simulator.py:211-223)
  int64_t max_epoch = -1;
  for (int64_t e = 0; e < n_events; ++e) max_epoch = std::max<int64_t>(max_epoch, ev_epoch[e]);
  if (max_epoch >= 0) {
    const int64_t KE = max_epoch + 1;
    std::vector<double> load((size_t)d->num_edges * KE, 0.0);
    for (int64_t p = 0; p < n_events; ++p) {
      const int64_t e = S.order[p];
      load[(size_t)ev_edge[e] * KE + ev_epoch[e]] += ev_frac[e];
    }
    const double tol = d->tolerance;
    for (int32_t ed = 0; ed < d->num_edges; ++ed) {
      const int64_t w = d->edge_window[ed];
      const double budget = d->edge_budget[ed];
      const double* L = load.data() + (size_t)ed * KE;
      for (int64_t k = 0; k < KE; ++k) {
        double total = 0.0;
        for (int64_t k2 = k - w + 1; k2 <= k; ++k2) total += (k2 >= 0) ? L[k2] : 0.0;
        if (total > budget * (1 + tol) + tol) R->capacity.push_back({ed, k});
      }
    }
  }
  for (int64_t c = 0; c < nc; ++c)
    for (const auto& r : co[c].sw_rest) R->sw_rest.push_back({S.comm_source[c], S.comm_chunk[c], r[0], r[1]});
  // per-entry completion: deliveries in (arrival, fraction) order (simulator.py:176-189)
  R->entry_done.assign(d->num_entries, -1);
  for (int64_t i = 0; i < d->num_entries; ++i) {
    auto& got = S.deliveries[i];
    std::sort(got.begin(), got.end());
    double acc = 0.0;
    for (const auto& g : got) {
      acc += g.second;
      if (acc >= 1.0 - d->tolerance) {
        R->entry_done[i] = (int32_t)g.first;
        break;
      }
    }
  }
  counts4[0] = (int64_t)R->causality.size();
  counts4[1] = (int64_t)R->capacity.size();
  counts4[2] = (int64_t)R->sw_rest.size();
  counts4[3] = d->num_entries;
  *out = R;
  return TECCL_OK;
}

// causality[n0] (event ids), capacity[2*n1] (edge, epoch), sw_rest[4*n2]
// (source, chunk, switch, usable), entry_done[n3]; frees the handle.
extern "C" int teccl_simulate_fetch(void* handle, int64_t* causality, int64_t* capacity, int64_t* sw_rest,
                                    int32_t* entry_done) {
  SimResult* R = (SimResult*)handle;
  if (!R) {
    teccl::set_error("teccl_simulate_fetch: null handle");
    return TECCL_EINVAL;
  }
  if (causality) std::copy(R->causality.begin(), R->causality.end(), causality);
  if (capacity)
    for (size_t i = 0; i < R->capacity.size(); ++i) {
      capacity[2 * i] = R->capacity[i][0];
      capacity[2 * i + 1] = R->capacity[i][1];
    }
  if (sw_rest)
    for (size_t i = 0; i < R->sw_rest.size(); ++i)
      for (int q = 0; q < 4; ++q) sw_rest[4 * i + q] = R->sw_rest[i][q];
  if (entry_done) std::copy(R->entry_done.begin(), R->entry_done.end(), entry_done);
  delete R;
  return TECCL_OK;
}
