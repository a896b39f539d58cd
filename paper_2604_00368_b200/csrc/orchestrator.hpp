// orchestrator.hpp — route planning for one transfer (orchestrator.hpp:61-81 contract).
//
// Direct routes only: one per backend that reaches the endpoints, each carrying the
// candidate list choose_rail iterates, oriented to the initiator and sorted by local
// rail id exactly as orient_candidates does (orchestrator.cpp:39-81), routes ranked by
// (best tier, backend) (orchestrator.cpp:239-243). Staged synthesis through host pools
// (orchestrator.cpp:120-234) is not part of this data plane: every B200 endpoint pair
// has a direct path (SM/CE over UVA), so a missing route is a NoRouteError.
#pragma once
#include <string>
#include <vector>

#include "fabric.hpp"

namespace spray {

struct PairOption {
  RailIndex remote = kNoRail;
  int tier = 3;
  bool affinity = false;
};
struct LocalCandidate {
  RailIndex local = kNoRail;
  std::vector<PairOption> pairs;
};
struct Route {
  std::string backend;
  int best_tier = 3;
  std::vector<LocalCandidate> candidates;
};

// penalties[t-1] <= 0 marks tier t unschedulable.
std::vector<Route> build_plan(const Topology& g, const Segment& src, const Segment& dst, Direction dir,
                              const double penalties[3], const std::vector<Capabilities>& caps);

std::vector<LocalCandidate> orient_candidates(const Topology& g, const std::vector<Reach>& entries,
                                              const std::string& backend, Direction dir, const Segment& src,
                                              const Segment& dst);

// Flattened candidate stream (include/spray_b200.h) of one set.
void append_stream(std::vector<int32_t>& out, const std::vector<LocalCandidate>& set);

}  // namespace spray
