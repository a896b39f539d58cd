// orchestrator.cpp — see orchestrator.hpp.
#include "orchestrator.hpp"

#include <algorithm>

namespace spray {

std::vector<LocalCandidate> orient_candidates(const Topology& g, const std::vector<Reach>& entries,
                                              const std::string& backend, Direction dir, const Segment& src,
                                              const Segment& dst) {
  // The scheduling side is the initiator: the source for WRITE, the destination for READ.
  const bool write = dir == Direction::kWrite;
  const std::string& local_node = write ? src.node : dst.node;
  const std::string& remote_node = write ? dst.node : src.node;
  const auto& remote_rails = g.rails_on(remote_node, backend);
  auto position = [&](RailIndex r, const std::string& node) -> size_t {
    const auto& v = g.rails_on(node, backend);
    auto it = std::find(v.begin(), v.end(), r);
    return it == v.end() ? 0 : size_t(it - v.begin());
  };
  std::vector<LocalCandidate> out;
  for (const Reach& e : entries) {
    if (e.backend != backend) continue;
    if (write ? !e.write_ok : !e.read_ok) continue;
    const RailIndex local = write ? e.local : e.remote;
    const RailIndex remote = write ? e.remote : e.local;
    // the 1:1 topology-aligned partner: same position modulo the remote rail count
    bool aff = local == remote;
    if (!aff) aff = !remote_rails.empty() && position(local, local_node) % remote_rails.size() == position(remote, remote_node);
    auto it = std::find_if(out.begin(), out.end(), [&](const LocalCandidate& c) { return c.local == local; });
    if (it == out.end()) {
      out.push_back(LocalCandidate{local, {}});
      it = out.end() - 1;
    }
    it->pairs.push_back(PairOption{remote, e.tier, aff});
  }
  std::sort(out.begin(), out.end(),
            [&](const LocalCandidate& a, const LocalCandidate& b) { return g.rail(a.local).id < g.rail(b.local).id; });
  return out;
}

std::vector<Route> build_plan(const Topology& g, const Segment& src, const Segment& dst, Direction dir,
                              const double penalties[3], const std::vector<Capabilities>& caps) {
  auto schedulable = [&](int t) { return t >= 1 && t <= 3 && penalties[t - 1] > 0.0; };
  const auto entries = reachable(g, src, dst, caps);
  std::vector<std::string> seen;
  for (const Reach& e : entries)
    if (std::find(seen.begin(), seen.end(), e.backend) == seen.end()) seen.push_back(e.backend);
  std::vector<Route> routes;
  for (const std::string& b : seen) {
    Route r;
    r.backend = b;
    r.candidates = orient_candidates(g, entries, b, dir, src, dst);
    if (r.candidates.empty()) continue;
    bool any = false;
    int best = 4;
    for (const LocalCandidate& c : r.candidates)
      for (const PairOption& p : c.pairs) {
        any = any || schedulable(p.tier);
        best = std::min(best, p.tier);
      }
    if (!any) continue;
    r.best_tier = best;
    routes.push_back(std::move(r));
  }
  if (routes.empty())
    throw NoRouteError("NoRoute: no backend chain connects '" + src.id + "' -> '" + dst.id + "'");
  std::stable_sort(routes.begin(), routes.end(), [](const Route& a, const Route& b) {
    if (a.best_tier != b.best_tier) return a.best_tier < b.best_tier;
    return a.backend < b.backend;
  });
  return routes;
}

void append_stream(std::vector<int32_t>& out, const std::vector<LocalCandidate>& set) {
  out.push_back(static_cast<int32_t>(set.size()));
  for (const LocalCandidate& c : set) {
    out.push_back(static_cast<int32_t>(c.local));
    out.push_back(static_cast<int32_t>(c.pairs.size()));
    for (const PairOption& p : c.pairs) {
      out.push_back(static_cast<int32_t>(p.remote));
      out.push_back(p.tier);
      out.push_back(p.affinity ? 1 : 0);
    }
  }
}

}  // namespace spray
