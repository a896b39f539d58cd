// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver around the UNMODIFIED reference library, compiled from the
// sources where they lie under /root/reference/proj by oracle/Makefile into
// oracle/_ref/libspray_ref.so. It exposes the reference's own SliceScheduler,
// ResilienceManager, Orchestrator, SimBackend and Engine to ctypes so that
//   * tests/golden/make_golden.py can record reference outputs as fixtures, and
//   * bench.py --impl reference can time the reference CPU path on the host cores.
// Nothing in paper_2604_00368_b200/ links or loads this file.

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "spray/bench.hpp"
#include "spray/engine.hpp"
#include "spray/memory_backend.hpp"
#include "spray/orchestrator.hpp"
#include "spray/resilience.hpp"
#include "spray/scheduler.hpp"
#include "spray/sim_backend.hpp"
#include "spray/telemetry.hpp"

#include "../include/spray_b200.h"

using namespace spray;

namespace {

thread_local std::string g_err;

SchedulerConfig to_ref(const spray_sched_config* c) {
  SchedulerConfig s;
  s.min_slice_size = c->min_slice_size;
  s.max_slices_per_transfer = c->max_slices_per_transfer;
  s.tolerance = c->tolerance;
  s.penalties.tier1 = c->penalty[0] > 0 ? std::optional<double>(c->penalty[0]) : std::nullopt;
  s.penalties.tier2 = c->penalty[1] > 0 ? std::optional<double>(c->penalty[1]) : std::nullopt;
  s.penalties.tier3 = c->penalty[2] > 0 ? std::optional<double>(c->penalty[2]) : std::nullopt;
  s.ewma_alpha = c->ewma_alpha;
  s.reset_interval = c->reset_interval_ns;
  s.policy = c->policy == SPRAY_POLICY_RR ? Policy::kRoundRobin
             : c->policy == SPRAY_POLICY_HASH ? Policy::kHash : Policy::kTelemetry;
  s.beta0_init_s = c->beta0_init_s;
  s.beta1_init = c->beta1_init;
  s.feedback_clamp = c->feedback_clamp;
  s.diffusion_weight = c->diffusion_weight;
  return s;
}

ResilienceConfig to_ref(const spray_resilience_config* c) {
  ResilienceConfig r;
  if (!c) return r;
  r.failure_threshold = c->failure_threshold;
  r.degradation_ratio = c->degradation_ratio;
  r.degradation_events = c->degradation_events;
  r.degradation_min_t_obs_s = c->degradation_min_t_obs_s;
  r.probe_successes_needed = c->probe_successes_needed;
  r.probe_bytes = c->probe_bytes;
  r.probe_interval = c->probe_interval_ns;
  r.probe_backoff_mult = c->probe_backoff_mult;
  r.probe_backoff_cap = c->probe_backoff_cap;
  r.max_attempts = c->max_attempts;
  r.slice_timeout = c->slice_timeout_ns;
  return r;
}

std::vector<std::vector<LocalCandidate>> parse_sets(const int32_t* st, size_t len) {
  std::vector<std::vector<LocalCandidate>> out;
  size_t i = 0;
  const int32_t ns = st[i++];
  for (int32_t k = 0; k < ns; ++k) {
    std::vector<LocalCandidate> set;
    const int32_t nl = st[i++];
    for (int32_t l = 0; l < nl; ++l) {
      LocalCandidate c;
      c.local = static_cast<RailIndex>(st[i++]);
      const int32_t np = st[i++];
      for (int32_t q = 0; q < np; ++q) {
        PairOption p;
        p.remote = static_cast<RailIndex>(st[i++]);
        p.tier = st[i++];
        p.affinity = st[i++] != 0;
        c.pairs.push_back(p);
      }
      set.push_back(std::move(c));
    }
    out.push_back(std::move(set));
  }
  if (i > len) throw std::runtime_error("candidate stream overrun");
  return out;
}

Medium medium_of(int m) {
  return m == SPRAY_MEDIUM_DEVICE ? Medium::kDeviceMemoryEmulated
         : m == SPRAY_MEDIUM_FILE ? Medium::kFile : Medium::kHostMemory;
}

BackendCapabilities caps_of(const spray_backend_caps& c) {
  BackendCapabilities b;
  b.id = c.id;
  for (int s = 0; s < 3; ++s)
    for (int d = 0; d < 3; ++d)
      if (c.media_pairs_mask & (1u << (s * 3 + d))) b.media_pairs.push_back({medium_of(s), medium_of(d)});
  b.supports_read = c.supports_read;
  b.supports_write = c.supports_write;
  b.cross_node = c.cross_node;
  b.same_node = c.same_node;
  return b;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_decompose(uint64_t total, uint64_t min_slice, uint32_t max_slices, uint64_t* off,
                  uint64_t* len, uint64_t cap, uint64_t* n) {
  SchedulerConfig cfg;
  cfg.min_slice_size = min_slice;
  cfg.max_slices_per_transfer = max_slices;
  auto v = SliceScheduler::decompose(total, cfg);
  *n = v.size();
  for (size_t i = 0; i < v.size() && i < cap; ++i) {
    off[i] = v[i].first;
    len[i] = v[i].second;
  }
  return 0;
}

// Rails of a topology in index order: bandwidth, tier, rank of id in sorted order,
// and the ids joined by '\n'.
int ref_rails(const char* topo, double* bw, int32_t* tier, uint32_t* id_rank, uint32_t cap,
              uint32_t* n, char* ids, size_t ids_cap) {
  try {
    TopologyGraph g = load_topology(topo);
    *n = static_cast<uint32_t>(g.rail_count());
    std::vector<std::pair<std::string, uint32_t>> order;
    std::string joined;
    for (uint32_t i = 0; i < g.rail_count(); ++i) {
      if (i < cap) {
        bw[i] = g.rail(i).bandwidth_bps;
        tier[i] = g.tier(i);
      }
      order.emplace_back(g.rail(i).id, i);
      joined += g.rail(i).id + "\n";
    }
    std::sort(order.begin(), order.end());
    for (uint32_t k = 0; k < order.size(); ++k)
      if (order[k].second < cap) id_rank[order[k].second] = k;
    std::snprintf(ids, ids_cap, "%s", joined.c_str());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Candidate stream for the active (first-ranked) direct route the reference
// Orchestrator builds for src -> dst (orchestrator.cpp:98-245). Returns 0, or
// -4 NoRoute / -1 config error.
int ref_build_candidates(const char* topo, const spray_backend_caps* caps, uint32_t n_caps,
                         const char* src_node, int src_medium, const char* src_device,
                         const char* dst_node, int dst_medium, const char* dst_device, int dir,
                         const spray_sched_config* sc, int32_t* stream, size_t cap, size_t* len,
                         char* backend_out, size_t backend_cap, uint32_t* n_routes) {
  try {
    TopologyGraph g = load_topology(topo);
    SegmentRegistry reg(&g);
    std::vector<std::byte> dummy(64);
    SegmentDescriptor s;
    s.id = "src";
    s.medium = medium_of(src_medium);
    s.node = src_node;
    s.device = src_device ? src_device : "";
    s.buffers = {BufferDesc{0, 64, dummy.data()}};
    SegmentDescriptor d = s;
    d.id = "dst";
    d.medium = medium_of(dst_medium);
    d.node = dst_node;
    d.device = dst_device ? dst_device : "";
    auto sp = reg.register_segment(s);
    auto dp = reg.register_segment(d);
    std::vector<BackendCapabilities> bc;
    for (uint32_t i = 0; i < n_caps; ++i) bc.push_back(caps_of(caps[i]));
    Orchestrator orch(&g, &reg, bc);
    SchedulerConfig cfg = to_ref(sc);
    auto plan = orch.build_plan(*sp, *dp, dir == SPRAY_READ ? Direction::kRead : Direction::kWrite,
                                cfg.penalties);
    *n_routes = static_cast<uint32_t>(plan->routes.size());
    const Route& r = plan->active_route();
    std::vector<int32_t> out;
    out.push_back(1);
    if (!r.direct) {
      g_err = "staged route";
      return -2;
    }
    out.push_back(static_cast<int32_t>(r.candidates.size()));
    for (const LocalCandidate& c : r.candidates) {
      out.push_back(static_cast<int32_t>(c.local));
      out.push_back(static_cast<int32_t>(c.pairs.size()));
      for (const PairOption& p : c.pairs) {
        out.push_back(static_cast<int32_t>(p.remote));
        out.push_back(p.tier);
        out.push_back(p.affinity ? 1 : 0);
      }
    }
    *len = out.size();
    for (size_t i = 0; i < out.size() && i < cap; ++i) stream[i] = out[i];
    std::snprintf(backend_out, backend_cap, "%s", r.backend.c_str());
    return 0;
  } catch (const NoRouteError& e) {
    g_err = e.what();
    return -4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Trace replay through the reference SliceScheduler + ResilienceManager with the
// event semantics documented in include/spray_b200.h.
int ref_replay(const char* topo, const spray_sched_config* sc, const spray_resilience_config* rc,
               const int32_t* cand_stream, size_t cand_len, const spray_trace_event* ev, size_t n,
               spray_decision* dec, size_t dcap, size_t* n_dec, uint64_t* expect_fail,
               int64_t* queued_out, double* beta_out, int32_t* health_out) {
  try {
    TopologyGraph g = load_topology(topo);
    // omega > 0: a board is attached (trace semantics, spray_b200.h BOARD event). A
    // BOARD(rail, G) event makes global_queued(rail) == G exactly: this instance
    // publishes its own queues (publish_to_board, which also sets the time hint) and an
    // external instance publishes the remainder G - own.
    GlobalLoadBoard board(10 * kMilli);
    const bool with_board = sc->diffusion_weight > 0.0;
    SliceScheduler sched(&g, to_ref(sc), with_board ? &board : nullptr, "engine0");
    Telemetry tel(&g, 10 * kMilli, false);
    ResilienceManager res(&g, &sched, &tel, to_ref(rc));
    auto sets = parse_sets(cand_stream, cand_len);
    size_t nd = 0;
    uint64_t bad = 0;
    for (size_t i = 0; i < n; ++i) {
      const spray_trace_event& e = ev[i];
      switch (e.kind) {
        case SPRAY_EV_DECIDE: {
          spray_decision d{};
          auto pick = sched.choose_rail(e.len, e.offset, sets.at(e.rail));
          if (pick) {
            d.local = pick->local;
            d.remote = pick->remote;
            d.tier = pick->tier;
            d.ok = 1;
            d.predicted_s = pick->predicted_s;
            d.x_norm = pick->x_norm;
          } else {
            d.local = d.remote = 0xffffffffu;
          }
          if (nd < dcap) dec[nd] = d;
          ++nd;
          break;
        }
        case SPRAY_EV_COMPLETE: {
          const int status = static_cast<int>((e.flags >> 8) & 0xff);
          const SliceStatus st = status == 0 ? SliceStatus::kOk
                                 : status == 1 ? SliceStatus::kFailed : SliceStatus::kTimeout;
          const double t_s = to_seconds(e.t_ns);
          sched.release(e.rail, e.len);
          res.observe(e.rail, e.remote == 0xffffffffu ? kNoRail : e.remote, st, t_s,
                      (e.flags & SPRAY_EVF_MODEL) ? e.predicted : 0.0, e.now_ns);
          if (st == SliceStatus::kOk && (e.flags & SPRAY_EVF_MODEL) &&
              !(e.flags & SPRAY_EVF_CANCELLED) && e.x_norm > 0.0)
            sched.feedback(e.rail, t_s, e.x_norm);
          break;
        }
        case SPRAY_EV_CHARGE: sched.charge(e.rail, e.len); break;
        case SPRAY_EV_RELEASE: sched.release(e.rail, e.len); break;
        case SPRAY_EV_HEALTH: sched.set_health(e.rail, static_cast<RailHealthState>(e.flags)); break;
        case SPRAY_EV_RESET: sched.periodic_reset(e.t_ns); break;
        case SPRAY_EV_RESET_RAIL: sched.reset_rail(e.rail, e.t_ns); break;
        case SPRAY_EV_EXPECT_HEALTH:
          if (static_cast<uint32_t>(sched.health(e.rail)) != e.flags) ++bad;
          break;
        case SPRAY_EV_DUE_PROBES: (void)res.due_probes(e.t_ns); break;
        case SPRAY_EV_BOARD: {
          if (!with_board) break;
          sched.publish_to_board(e.now_ns);
          board.publish("ext", e.rail, static_cast<int64_t>(e.len) - sched.queued_bytes(e.rail), e.now_ns);
          break;
        }
        case SPRAY_EV_PROBE_DONE: {
          const int status = static_cast<int>((e.flags >> 8) & 0xff);
          sched.release(e.rail, e.len);
          res.observe_probe(e.rail, status == 0 ? SliceStatus::kOk : status == 1 ? SliceStatus::kFailed
                                                                                   : SliceStatus::kTimeout,
                            e.now_ns);
          break;
        }
        default: g_err = "bad event kind"; return -1;
      }
    }
    *n_dec = nd;
    *expect_fail = bad;
    for (RailIndex i = 0; i < g.rail_count(); ++i) {
      if (queued_out) queued_out[i] = sched.queued_bytes(i);
      if (beta_out) {
        beta_out[2 * i] = sched.beta0(i);
        beta_out[2 * i + 1] = sched.beta1(i);
      }
      if (health_out) health_out[i] = static_cast<int32_t>(sched.health(i));
    }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// SimBackend service-time arithmetic through the reference class itself
// (test_backends.cpp:95-120 pattern): one slice of `len` on rail 0 posted at t=0.
int ref_sim_one(const char* topo, uint64_t len, double degrade, uint64_t* done_ns) {
  try {
    TopologyGraph g = load_topology(topo);
    SegmentRegistry reg(&g);
    VirtualClock clk;
    SimBackend sim(&g, &reg, &clk, SimBackendOptions{});
    if (degrade != 1.0) {
      FaultSchedule fs;
      FaultEntry f;
      f.rail = g.rail(0).id;
      f.effect = FaultEffect::kDegrade;
      f.start = 0;
      f.end = 1000 * kSecond;
      f.factor = degrade;
      fs.entries.push_back(f);
      sim.set_fault_schedule(fs);
    }
    std::vector<std::byte> a(len), b(len);
    SegmentDescriptor s{"s", Medium::kHostMemory, g.rail(0).node, {BufferDesc{0, len, a.data()}}, "", ""};
    std::string other = g.nodes().back().id;
    SegmentDescriptor d{"d", Medium::kHostMemory, other, {BufferDesc{0, len, b.data()}}, "", ""};
    reg.register_segment(s);
    reg.register_segment(d);
    SliceWorkRequest r;
    r.slice = 1;
    r.src_segment = "s";
    r.dst_segment = "d";
    r.length = len;
    r.local_rail = 0;
    r.remote_rail = static_cast<RailIndex>(g.rail_count() - 1);
    std::vector<SliceWorkRequest> v{r};
    sim.post_slices(v);
    *done_ns = *sim.next_event_time();
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// Config 1 bytes oracle: the reference Engine with the sim backend in virtual time
// moves `nbytes` of the bench payload (bench.cpp:99) from node a to node b. Reports
// delivered-byte checksums and per-rail bytes_ok.
int ref_engine_sim_transfer(const char* topo, uint64_t nbytes, uint64_t seed, uint8_t* dst_copy,
                            uint64_t* bytes_ok, uint32_t cap) {
  try {
    EngineOptions eo;
    eo.topology_json = topo;
    eo.backends = {"sim"};
    eo.seed = seed;
    Engine eng(std::move(eo));
    eng.start();
    std::vector<std::byte> src(nbytes), dst(nbytes);
    Rng rng(seed ^ 0x517cc1b727220a95ULL);
    uint64_t i = 0;
    for (; i + 8 <= nbytes; i += 8) {
      uint64_t v = rng.next_u64();
      std::memcpy(src.data() + i, &v, 8);
    }
    for (; i < nbytes; ++i) src[i] = static_cast<std::byte>(rng.next_u64());
    const auto& nodes = eng.graph().nodes();
    SegmentDescriptor s{"bench/src", Medium::kHostMemory, nodes.front().id, {BufferDesc{0, nbytes, src.data()}}, "", ""};
    SegmentDescriptor d{"bench/dst", Medium::kHostMemory, nodes.back().id, {BufferDesc{0, nbytes, dst.data()}}, "", ""};
    eng.register_segment(s);
    eng.register_segment(d);
    BatchId b = eng.allocate_batch();
    eng.submit_transfer(b, TransferRequest{"bench/src", 0, "bench/dst", 0, nbytes, Direction::kWrite});
    BatchStatus st = eng.await_batch(b);
    if (st.state != BatchState::kComplete) {
      g_err = "batch not complete";
      return -1;
    }
    std::memcpy(dst_copy, dst.data(), nbytes);
    auto snap = eng.telemetry().snapshot();
    for (uint32_t r = 0; r < snap.rails.size() && r < cap; ++r) bytes_ok[r] = snap.rails[r].bytes_ok;
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// CPU baseline: the reference Engine, real clock, memory backend, `workers` worker
// threads, moving n_blocks x block bytes host->host as individual transfers of one
// batch (a KV-block batch), block table = seeded permutation over a pool. Returns
// the best wall time in seconds over `iters` batches (allocate -> submit -> await).
double ref_cpu_kv_batch(uint32_t rails, uint32_t workers, uint64_t block, uint32_t n_blocks,
                        uint64_t seed, int iters, uint64_t* checksum_ok) {
  try {
    std::string topo = "{\"nodes\":[{\"id\":\"a\",\"devices\":[{\"id\":\"a.mem\",\"kind\":\"host_memory\"}]},"
                       "{\"id\":\"b\",\"devices\":[{\"id\":\"b.mem\",\"kind\":\"host_memory\"}]}],\"rails\":[";
    for (uint32_t n = 0; n < 2; ++n)
      for (uint32_t r = 0; r < rails; ++r) {
        if (n || r) topo += ",";
        const char* node = n ? "b" : "a";
        topo += std::string("{\"id\":\"") + node + ".r" + std::to_string(r) + "\",\"node\":\"" + node +
                "\",\"bandwidth_bytes_per_sec\":1e10,\"affinity\":\"direct\",\"backend\":\"memory\"}";
      }
    topo += "]}";
    EngineOptions eo;
    eo.topology_json = topo;
    eo.backends = {"memory"};
    eo.clock_mode = ClockMode::kReal;
    eo.workers = workers;
    eo.stats = true;
    Engine eng(std::move(eo));
    eng.start();
    const uint64_t pool = block * n_blocks;
    std::vector<std::byte> src(pool), dst(pool);
    Rng rng(seed);
    for (uint64_t i = 0; i + 8 <= pool; i += 8) {
      uint64_t v = rng.next_u64();
      std::memcpy(src.data() + i, &v, 8);
    }
    std::vector<uint32_t> perm(n_blocks);
    for (uint32_t i = 0; i < n_blocks; ++i) perm[i] = i;
    for (uint32_t i = n_blocks; i > 1; --i) std::swap(perm[i - 1], perm[rng.next_below(i)]);
    SegmentDescriptor s{"kv/hbm", Medium::kHostMemory, "a", {BufferDesc{0, pool, src.data()}}, "", ""};
    SegmentDescriptor d{"kv/host", Medium::kHostMemory, "b", {BufferDesc{0, pool, dst.data()}}, "", ""};
    eng.register_segment(s);
    eng.register_segment(d);
    double best = 1e30;
    for (int it = 0; it < iters; ++it) {
      auto t0 = std::chrono::steady_clock::now();
      BatchId b = eng.allocate_batch();
      for (uint32_t k = 0; k < n_blocks; ++k)
        eng.submit_transfer(b, TransferRequest{"kv/hbm", uint64_t(k) * block, "kv/host",
                                               uint64_t(perm[k]) * block, block, Direction::kWrite});
      BatchStatus st = eng.await_batch(b);
      auto t1 = std::chrono::steady_clock::now();
      if (st.state != BatchState::kComplete) {
        g_err = "cpu baseline batch failed";
        return -1.0;
      }
      eng.free_batch(b);
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    uint64_t ok = 1;
    for (uint32_t k = 0; k < n_blocks && ok; ++k)
      ok = std::memcmp(src.data() + uint64_t(k) * block, dst.data() + uint64_t(perm[k]) * block, block) == 0;
    *checksum_ok = ok;
    eng.stop();
    return best;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1.0;
  }
}

}  // extern "C"
