// Weight residency under an HBM budget (PAPER.md:180
// "pipelined load", P:399 co-location, P:1057 pin list).
//
// When the unique (merged) weights do not fit gemel_options.weight_budget_bytes,
// a pinned set stays resident and the rest stream every step from pinned host
// memory into a ring of slots at the end of the weight arena, on a copy stream
// one launch ahead of the compute stream:
//   * resident set: the fewest streamed bytes per step (an unmerged workload over
//     budget is copy-bound, PAPER.md:191 / 1068), subject to pinned + ring <= budget
//     where the ring keeps >= 2x the largest swapped tensor; among equal sizes,
//     weights shared by >= 2 models and earlier first use stay first;
//   * GEMM launches are split so the swapped bytes first read by one launch fit
//     half the ring (the other half fills for the next launch);
//   * ring slots are a circular FIFO in copy order; a copy waits for the last
//     launch reading any earlier tensor whose slot it overwrites.
// The schedule is static: slots, and hence the tensor maps of swapped weights,
// are fixed at plan time and the whole step (copies included) is one CUDA graph.
#include <algorithm>
#include <functional>
#include <set>

#include "internal.h"

namespace gemel {

int plan_swap(Ctx* c, const std::function<void(Launch&, int)>& gemm_cost) {
  c->pinned_bytes = c->ring_bytes = c->swap_bytes = 0;
  c->swap_order.clear();
  const int ndw = int(c->dweights.size());
  for (auto& w : c->dweights) {
    w.swapped = false;
    w.first_launch = w.last_launch = w.wait_launch = w.copy_order = -1;
  }
  const uint64_t budget = c->opt.weight_budget_bytes;
  uint64_t epi = 0, total = 0;
  for (auto& g : c->nodes)
    if (g.kind == NK_GEMM) epi += 2 * align_up(uint64_t(g.Cout) * 4, 256);
    else if (g.kind == NK_MISC && g.misc == MISC_L2NORM) epi += align_up(uint64_t(g.Cout) * 4, 256);
  for (auto& w : c->dweights) total += align_up(w.bytes, 256);
  if (budget == 0 || total + epi <= budget) {
    c->pinned_bytes = total;
    return GEMEL_OK;
  }
  if (budget <= epi) return set_err(c, GEMEL_E_NOMEM, "plan: weight budget below the resident epilogue vectors");
  const uint64_t avail = budget - epi;

  // first use (launch, position) and the models reading each weight
  std::vector<int64_t> first_rank(ndw, INT64_MAX);
  std::vector<std::set<int>> models(ndw);
  int64_t rank = 0;
  for (auto& L : c->launches) {
    if (L.kind != NK_GEMM) continue;
    for (int pid : L.items) {
      const int wk = c->problems[pid].wkey;
      first_rank[wk] = std::min(first_rank[wk], rank++);
      for (int nid : c->problems[pid].members) models[wk].insert(c->nodes[nid].model);
    }
  }
  // Resident set with the fewest streamed bytes (the step is copy-bound once anything
  // streams): for every candidate size m of the largest streamed tensor, tensors
  // larger than m must stay resident, the ring takes 2m, and the rest of the budget
  // is filled by a max-bytes subset of the tensors <= m -- exact subset enumeration
  // when <= 20 candidates remain, first-fit decreasing beyond.  The all-resident
  // case was handled above.  Ties keep the first candidate (largest m).
  std::vector<uint64_t> sz(ndw);
  for (int i = 0; i < ndw; ++i) sz[i] = align_up(c->dweights[i].bytes, 256);
  std::vector<uint64_t> cands(sz.begin(), sz.end());
  std::sort(cands.begin(), cands.end(), std::greater<uint64_t>());
  cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
  std::vector<char> pin(ndw, 0), best_pin;
  uint64_t best_stream = UINT64_MAX, pinned = 0;
  std::vector<int> order(ndw);
  for (int i = 0; i < ndw; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {   // size desc, then shared / first use
    if (sz[a] != sz[b]) return sz[a] > sz[b];
    const bool sa = models[a].size() > 1, sb = models[b].size() > 1;
    if (sa != sb) return sa;
    return first_rank[a] < first_rank[b];
  });
  for (uint64_t m : cands) {
    if (2 * m > avail) continue;
    uint64_t must = 0;
    std::vector<int> rest;
    for (int i : order) {
      if (sz[i] > m) must += sz[i];
      else rest.push_back(i);
    }
    if (must + 2 * m > avail) continue;
    const uint64_t cap = avail - 2 * m - must;
    std::vector<char> p(ndw, 0);
    for (int i = 0; i < ndw; ++i) p[i] = sz[i] > m;
    uint64_t got = 0;
    if (rest.size() <= 20) {
      uint32_t best_mask = 0;
      for (uint32_t mask = 0; mask < (1u << rest.size()); ++mask) {
        uint64_t b = 0;
        for (size_t j = 0; j < rest.size(); ++j)
          if (mask >> j & 1) b += sz[rest[j]];
        if (b <= cap && b > got) { got = b; best_mask = mask; }
      }
      for (size_t j = 0; j < rest.size(); ++j) p[rest[j]] = (best_mask >> j & 1) ? 1 : 0;
    } else {
      for (int i : rest)
        if (got + sz[i] <= cap) { p[i] = 1; got += sz[i]; }
    }
    uint64_t streamed = 0;
    for (int i = 0; i < ndw; ++i)
      if (!p[i]) streamed += c->dweights[i].bytes;
    if (streamed < best_stream) {
      best_stream = streamed;
      best_pin = p;
      pinned = must + got;
    }
  }
  if (best_pin.empty()) return set_err(c, GEMEL_E_NOMEM, "plan: weight budget too small for a double-buffered swap ring");
  pin = best_pin;
  auto max_unpinned = [&]() {
    uint64_t mx = 0;
    for (int i = 0; i < ndw; ++i)
      if (!pin[i]) mx = std::max(mx, sz[i]);
    return mx;
  };
  const uint64_t ring = (avail - pinned) / 256 * 256;
  const uint64_t big = max_unpinned();
  if (big == 0) {
    c->pinned_bytes = pinned;
    return GEMEL_OK;
  }
  if (ring < 2 * big) return set_err(c, GEMEL_E_NOMEM, "plan: weight budget too small for a double-buffered swap ring");
  for (int i = 0; i < ndw; ++i) c->dweights[i].swapped = !pin[i];

  // split GEMM launches: swapped bytes first read by one launch <= ring / 2
  std::vector<Launch> out;
  std::vector<char> seen(ndw, 0);
  for (auto& L : c->launches) {
    if (L.kind != NK_GEMM) {
      out.push_back(L);
      continue;
    }
    auto fresh = [&](int level) {
      Launch n;
      n.kind = NK_GEMM;
      n.stem = L.stem;
      n.level = level;
      return n;
    };
    Launch cur = fresh(L.level);
    uint64_t cur_bytes = 0;
    for (int pid : L.items) {
      const int wk = c->problems[pid].wkey;
      const uint64_t add = (c->dweights[wk].swapped && !seen[wk]) ? align_up(c->dweights[wk].bytes, 256) : 0;
      if (!cur.items.empty() && cur_bytes + add > ring / 2) {
        out.push_back(cur);
        cur = fresh(c->problems[pid].level);
        cur_bytes = 0;
      }
      cur.items.push_back(pid);
      gemm_cost(cur, pid);
      cur_bytes += add;
      seen[wk] = 1;
    }
    out.push_back(cur);
  }
  c->launches.swap(out);

  // lifetimes, copy order, ring slots, copy waits
  for (size_t li = 0; li < c->launches.size(); ++li) {
    const Launch& L = c->launches[li];
    if (L.kind != NK_GEMM) continue;
    for (int pid : L.items) {
      DevWeight& w = c->dweights[c->problems[pid].wkey];
      if (w.first_launch < 0) w.first_launch = int(li);
      w.last_launch = int(li);
    }
  }
  for (int i = 0; i < ndw; ++i)
    if (c->dweights[i].swapped) c->swap_order.push_back(i);
  std::stable_sort(c->swap_order.begin(), c->swap_order.end(), [&](int a, int b) {
    return c->dweights[a].first_launch != c->dweights[b].first_launch
               ? c->dweights[a].first_launch < c->dweights[b].first_launch
               : first_rank[a] < first_rank[b];
  });
  uint64_t p = 0;
  for (size_t k = 0; k < c->swap_order.size(); ++k) {
    DevWeight& u = c->dweights[c->swap_order[k]];
    const uint64_t b = align_up(u.bytes, 256);
    if (p + b > ring) p = 0;
    u.offset = p;   // slot within the ring; the arena layout adds the ring base
    u.copy_order = int(k);
    p += b;
    for (size_t j = 0; j < k; ++j) {
      const DevWeight& w = c->dweights[c->swap_order[j]];
      const uint64_t wb = align_up(w.bytes, 256);
      if (w.offset < u.offset + b && u.offset < w.offset + wb) u.wait_launch = std::max(u.wait_launch, w.last_launch);
    }
    if (u.wait_launch >= u.first_launch)
      return set_err(c, GEMEL_E_NOMEM, "plan: swap ring too small (a slot is still read by the launch that needs it)");
    c->swap_bytes += u.bytes;
  }
  c->pinned_bytes = pinned;
  c->ring_bytes = ring;
  return GEMEL_OK;
}

}  // namespace gemel
