// Rate -> schedule decomposition on the host CPU, one thread per source.
//
// Restates collsched.lp.lp_rates_to_schedule (pkg/src/collsched/lp.py:156-301)
// over dense per-source arrays: reads are served earliest first; each is
// traced backwards -- a positive buffer carries the chunk one epoch back,
// otherwise the first in-edge (senders in str() order) whose send lands in
// this epoch -- to the source's epoch-0 pool; the bottleneck is peeled off
// every arc; events are sorted by (epoch, str(source), str(src), str(dst),
// chunk) and equal keys merged by summing in that order. Sources are
// independent commodities, so they are decomposed in parallel; the Python
// restatement in schedule.py defines the semantics and the tests pin both to
// the reference's event lists.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {

struct Ev {
  int32_t src_slot, chunk, edge, epoch;
  double frac;
};

struct Job {
  // problem
  int Nn, E, S, P, K, G;
  const uint8_t* is_sw;
  const int32_t *esrc, *edst, *edelta, *snode;
  const int32_t *in_ptr, *in_edges;          // in-edges per node, str(sender) order
  const int32_t *pair_src, *pair_dst;
  const int32_t *pair_chunk_ptr, *pair_chunks, *pair_order;
  const double* x;
  double tol, need_tol;
  std::vector<int> gpu_of;
  int64_t SB;
};

// returns false (and an error string) on a conservation residue
bool run_source(const Job& J, int s, std::vector<Ev>& out, std::string& err) {
  const int K = J.K, E = J.E;
  const double* xs = J.x + (int64_t)s * J.SB;
  std::vector<double> F(xs, xs + (int64_t)E * K);                 // F[e*K + k]
  std::vector<double> B(xs + (int64_t)E * K, xs + J.SB);           // B[g*(K+1) + k]
  const int snode = J.snode[s];
  const double tol = J.tol;
  struct Arc { int kind, a, b; };
  std::vector<Arc> arcs;
  std::vector<double> rres(K);
  for (int oi = 0; oi < J.P; ++oi) {
    const int p = J.pair_order[oi];
    if (J.pair_src[p] != s) continue;
    const double* rd = J.x + (int64_t)J.S * J.SB + (int64_t)p * 2 * K;
    for (int k = 0; k < K; ++k) rres[k] = rd[2 * k];
    const int dst = J.pair_dst[p];
    int cursor = 0;
    for (int ci = J.pair_chunk_ptr[p]; ci < J.pair_chunk_ptr[p + 1]; ++ci) {
      const int chunk = J.pair_chunks[ci];
      double need = 1.0;
      int guard = 0;
      while (need > J.need_tol) {
        if (++guard > 10000) { err = "path peeling did not converge"; return false; }
        while (cursor < K && !(rres[cursor] > tol)) ++cursor;
        if (cursor >= K) {
          err = "conservation residue: chunk " + std::to_string(chunk) + " short by " +
                std::to_string(need);
          return false;
        }
        const int k_read = cursor;
        const double amount = std::min(need, rres[k_read]);
        // backward trace (lp.py:244-269)
        arcs.clear();
        int node = dst, k = k_read;
        bool dead = false;
        while (true) {
          if (node == snode && k == 0) break;
          const int g = J.gpu_of[node];
          if (g >= 0 && B[(int64_t)g * (K + 1) + k] > tol) {
            arcs.push_back({0, g, k});
            if (--k < 0) { err = "buffer traces past epoch 0"; return false; }
            continue;
          }
          int found = -1, ft = 0;
          for (int j = J.in_ptr[node]; j < J.in_ptr[node + 1]; ++j) {
            const int e = J.in_edges[j];
            const int tt = k - J.edelta[e];
            if (tt >= 0 && F[(int64_t)e * K + tt] > tol) { found = e; ft = tt; break; }
          }
          if (found < 0) { dead = true; break; }
          arcs.push_back({1, found, ft});
          if (ft == 0) {
            if (J.esrc[found] != snode) dead = true;
            break;
          }
          node = J.esrc[found];
          k = ft - 1;
        }
        double got = 0.0;
        if (!dead) {
          double bottleneck = amount;
          for (const Arc& a : arcs)
            bottleneck = std::min(bottleneck, a.kind == 0 ? B[(int64_t)a.a * (K + 1) + a.b]
                                                          : F[(int64_t)a.a * K + a.b]);
          if (bottleneck > tol) {
            got = bottleneck;
            for (const Arc& a : arcs) {
              double& v = a.kind == 0 ? B[(int64_t)a.a * (K + 1) + a.b] : F[(int64_t)a.a * K + a.b];
              v -= bottleneck;
              if (v <= tol) v = 0.0;
              if (a.kind == 1) out.push_back({s, chunk, a.a, a.b, bottleneck});
            }
          }
        }
        if (got <= tol) {
          err = "conservation residue: no backing path for read at epoch " + std::to_string(k_read);
          return false;
        }
        rres[k_read] -= got;
        if (rres[k_read] <= tol) rres[k_read] = 0.0;
        need -= got;
      }
    }
  }
  return true;
}

struct EventList {
  std::vector<Ev> ev;
};

}  // namespace

using namespace teccl;

extern "C" int teccl_schedule_te(const teccl_te_desc* desc, const double* x, double tol,
                                 double need_tol, const int32_t* in_ptr, const int32_t* in_edges,
                                 const int32_t* pair_chunk_ptr, const int32_t* pair_chunks,
                                 const int32_t* pair_order, const int32_t* source_rank,
                                 const int32_t* node_rank, int32_t threads, void** out,
                                 int64_t* n_events) {
  if (!desc || !x || !in_ptr || !in_edges || !pair_chunk_ptr || !pair_chunks || !pair_order ||
      !source_rank || !node_rank || !out || !n_events) {
    set_error("null argument");
    return TECCL_EINVAL;
  }
  Job J;
  J.Nn = desc->num_nodes; J.E = desc->num_edges; J.S = desc->num_sources;
  J.P = desc->num_pairs; J.K = desc->K;
  J.is_sw = desc->node_is_switch; J.esrc = desc->edge_src; J.edst = desc->edge_dst;
  J.edelta = desc->edge_delta; J.snode = desc->source_node;
  J.in_ptr = in_ptr; J.in_edges = in_edges;
  J.pair_src = desc->pair_source; J.pair_dst = desc->pair_dst;
  J.pair_chunk_ptr = pair_chunk_ptr; J.pair_chunks = pair_chunks; J.pair_order = pair_order;
  J.x = x; J.tol = tol; J.need_tol = need_tol;
  J.gpu_of.assign(J.Nn, -1);
  int G = 0;
  for (int n = 0; n < J.Nn; ++n)
    if (!J.is_sw[n]) J.gpu_of[n] = G++;
  J.G = G;
  J.SB = (int64_t)J.E * J.K + (int64_t)G * (J.K + 1);

  // key order of the reference's event list: (epoch, str(source), str(src),
  // str(dst), chunk), stable in generation order; equal keys are merged by
  // summing in that order. Every key carries its source, so each source's
  // list is sorted and merged in its own thread, and the global order is a
  // merge of the per-source lists by (epoch, source rank).
  auto key_less = [&](const Ev& a, const Ev& b) {
    if (a.epoch != b.epoch) return a.epoch < b.epoch;
    const int sa = source_rank[a.src_slot], sb = source_rank[b.src_slot];
    if (sa != sb) return sa < sb;
    const int ia = node_rank[J.esrc[a.edge]], ib = node_rank[J.esrc[b.edge]];
    if (ia != ib) return ia < ib;
    const int da = node_rank[J.edst[a.edge]], db = node_rank[J.edst[b.edge]];
    if (da != db) return da < db;
    return a.chunk < b.chunk;
  };
  auto sort_merge = [&](std::vector<Ev>& v) {
    std::stable_sort(v.begin(), v.end(), key_less);
    size_t w = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      if (w > 0) {
        Ev& m = v[w - 1];
        const Ev& e = v[i];
        if (m.src_slot == e.src_slot && m.chunk == e.chunk && m.edge == e.edge && m.epoch == e.epoch) {
          m.frac += e.frac;
          continue;
        }
      }
      v[w++] = v[i];
    }
    v.resize(w);
  };
  std::vector<std::vector<Ev>> per(J.S);
  std::vector<std::string> errs(J.S);
  std::vector<char> ok(J.S, 1);
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, J.S));
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; ++w)
    pool.emplace_back([&, w]() {
      for (int s = w; s < J.S; s += nt) {
        ok[s] = run_source(J, s, per[s], errs[s]);
        if (ok[s]) sort_merge(per[s]);
      }
    });
  for (auto& t : pool) t.join();
  for (int s = 0; s < J.S; ++s)
    if (!ok[s]) { set_error(errs[s]); return TECCL_EINVAL; }

  auto* L = new EventList();
  size_t total = 0;
  for (auto& v : per) total += v.size();
  L->ev.reserve(total);
  std::vector<int> by_rank(J.S);
  for (int s = 0; s < J.S; ++s) by_rank[s] = s;
  std::stable_sort(by_rank.begin(), by_rank.end(),
                   [&](int a, int b) { return source_rank[a] < source_rank[b]; });
  std::vector<size_t> pos(J.S, 0);
  for (int k = 0; k < J.K; ++k)
    for (int s : by_rank) {
      const std::vector<Ev>& v = per[s];
      size_t& i = pos[s];
      while (i < v.size() && v[i].epoch == k) L->ev.push_back(v[i++]);
    }
  if (L->ev.size() != total) {
    delete L;
    set_error("schedule event outside the horizon");
    return TECCL_EINVAL;
  }
  *out = L;
  *n_events = (int64_t)L->ev.size();
  return TECCL_OK;
}

extern "C" int teccl_schedule_fetch(void* handle, int32_t* src_slot, int32_t* chunk, int32_t* edge,
                                    int32_t* epoch, double* frac) {
  if (!handle) { set_error("null handle"); return TECCL_EINVAL; }
  auto* L = (EventList*)handle;
  for (size_t i = 0; i < L->ev.size(); ++i) {
    const Ev& e = L->ev[i];
    if (src_slot) src_slot[i] = e.src_slot;
    if (chunk) chunk[i] = e.chunk;
    if (edge) edge[i] = e.edge;
    if (epoch) epoch[i] = e.epoch;
    if (frac) frac[i] = e.frac;
  }
  delete L;
  return TECCL_OK;
}
