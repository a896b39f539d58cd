// engine.cpp — host side of the B200 spray engine (see engine.hpp).
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <deque>
#include <cstring>
#include <immintrin.h>
#include <set>
#include <tuple>

namespace spray_launch {
size_t engine_smem_bytes();
cudaError_t launch_engine(const spray_dev::EngineDev& E, int grid, int block, cudaStream_t st);
cudaError_t launch_epoch(uint64_t* out, cudaStream_t st);
cudaError_t launch_relay_forward(const spray_dev::EngineDev& E, uint32_t r, int grid, cudaStream_t st);
cudaError_t launch_hold(const uint32_t* flag, cudaStream_t st);
cudaError_t preload_kernels();
}  // namespace spray_launch

namespace spray {

using namespace spray_dev;

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)

void default_sched_config(spray_sched_config* c) {  // scheduler.hpp:44-58
  c->min_slice_size = 64 * 1024;
  c->max_slices_per_transfer = 4096;
  c->policy = SPRAY_POLICY_TELEMETRY;
  c->tolerance = 0.05;
  c->penalty[0] = 1.0;
  c->penalty[1] = 3.0;
  c->penalty[2] = 0.0;  // tier 3 unschedulable
  c->ewma_alpha = 0.2;
  c->reset_interval_ns = 30ull * 1000000000ull;
  c->beta0_init_s = 0.0;
  c->beta1_init = 1.0;
  c->feedback_clamp = 5.0;
  c->diffusion_weight = 0.0;  // scheduler.hpp:51
}

void default_resilience_config(spray_resilience_config* c) {  // resilience.hpp:17-28
  std::memset(c, 0, sizeof(*c));
  c->failure_threshold = 3;
  c->degradation_ratio = 4.0;
  c->degradation_events = 8;
  c->degradation_min_t_obs_s = 1e-3;
  c->probe_successes_needed = 2;
  c->probe_bytes = 4096;
  c->probe_interval_ns = 1000000000ull;
  c->probe_backoff_mult = 1.0;
  c->probe_backoff_cap = 3;
  c->max_attempts = 4;
  c->slice_timeout_ns = 2000000000ull;  // real clock default (engine.cpp:78-79)
}

static void reject_unknown(const Json& j, std::initializer_list<const char*> known, const char* scope) {
  for (const auto& kv : j.obj) {
    bool ok = false;
    for (const char* k : known) ok = ok || kv.first == k;
    if (!ok) throw ConfigError(std::string("engine config: unknown key '") + kv.first + "' in " + scope);
  }
}

// SchedulerConfig::validate (scheduler.cpp:34-61)
static void validate(const spray_sched_config& c, double omega) {
  if (c.min_slice_size < 4096) throw ConfigError("min slice size must be >= 4096");
  if (c.max_slices_per_transfer == 0) throw ConfigError("max slices must be >= 1");
  if (!(c.tolerance > 0.0)) throw ConfigError("tolerance must be > 0");
  if (c.ewma_alpha <= 0.0 || c.ewma_alpha > 1.0) throw ConfigError("alpha must be in (0, 1]");
  if (omega < 0.0 || omega > 1.0) throw ConfigError("diffusion weight must be in [0, 1]");
  double prev = 0.0;
  for (int t = 0; t < 3; ++t) {
    if (!(c.penalty[t] > 0.0)) {
      for (int u = t + 1; u < 3; ++u)
        if (c.penalty[u] > 0.0) throw ConfigError("tier penalties must be non-decreasing");
      break;
    }
    if (c.penalty[t] < prev) throw ConfigError("tier penalties must be non-decreasing");
    prev = c.penalty[t];
  }
}

static void validate(const spray_resilience_config& c) {  // resilience.cpp:6-14
  if (c.failure_threshold < 1) throw ConfigError("failure threshold must be >= 1");
  if (c.degradation_ratio <= 1.0) throw ConfigError("degradation ratio must be > 1");
  if (c.degradation_events < 1) throw ConfigError("degradation events must be >= 1");
  if (c.probe_successes_needed < 1) throw ConfigError("probe successes must be >= 1");
  if (c.probe_bytes == 0) throw ConfigError("probe bytes must be > 0");
  if (c.max_attempts < 1) throw ConfigError("max attempts must be >= 1");
  if (c.probe_backoff_mult < 1.0) throw ConfigError("probe backoff mult must be >= 1");
}

EngineOptions engine_options_from_json(const std::string& text) {
  EngineOptions eo;
  default_sched_config(&eo.sched);
  default_resilience_config(&eo.res);
  if (text.empty()) return eo;
  Json j;
  try {
    j = Json::parse(text);
  } catch (const JsonError& e) {
    throw ConfigError(std::string("engine config parse error: ") + e.what());
  }
  try {
    reject_unknown(j, {"topology_file", "topology", "backends", "workers", "clock", "scheduler", "resilience",
                       "staging", "burst", "ring_capacity", "stats", "stats_window_ms", "seed", "sim", "memory",
                       "instance_id", "b200"},
                   "root");
    if (j.contains("stats_window_ms")) {  // Telemetry window (engine.cpp:1186-1197 key set)
      const double ms = j.at("stats_window_ms").as_number();
      if (!(ms >= 0.001)) throw ConfigError("stats_window_ms must be >= 0.001");
      eo.window_ns = static_cast<uint64_t>(ms * 1e6);
    }
    if (j.contains("backends")) {
      eo.backends.clear();
      for (const Json& b : j.at("backends").arr) eo.backends.push_back(b.as_string());
    }
    if (j.contains("clock") && j.at("clock").as_string() != "real")
      throw ConfigError("engine config: the B200 engine runs on the device clock (clock must be real)");
    if (j.contains("scheduler")) {
      const Json& s = j.at("scheduler");
      reject_unknown(s, {"min_slice_size", "max_slices_per_transfer", "tolerance", "tier1_penalty", "tier2_penalty",
                         "tier3_penalty", "ewma_alpha", "reset_interval_ms", "diffusion_weight", "policy",
                         "feedback_clamp"},
                     "scheduler");
      spray_sched_config& c = eo.sched;
      c.min_slice_size = static_cast<uint64_t>(s.number_or("min_slice_size", double(c.min_slice_size)));
      c.max_slices_per_transfer =
          static_cast<uint32_t>(s.number_or("max_slices_per_transfer", double(c.max_slices_per_transfer)));
      c.tolerance = s.number_or("tolerance", c.tolerance);
      const char* keys[3] = {"tier1_penalty", "tier2_penalty", "tier3_penalty"};
      for (int t = 0; t < 3; ++t)
        if (s.contains(keys[t])) c.penalty[t] = s.at(keys[t]).is_null() ? 0.0 : s.at(keys[t]).as_number();
      c.ewma_alpha = s.number_or("ewma_alpha", c.ewma_alpha);
      if (s.contains("reset_interval_ms"))
        c.reset_interval_ns = static_cast<uint64_t>(s.at("reset_interval_ms").as_number() * 1e6);
      eo.diffusion_weight = s.number_or("diffusion_weight", 0.0);
      c.diffusion_weight = eo.diffusion_weight;
      if (s.contains("policy")) {
        const std::string p = s.at("policy").as_string();
        if (p == "telemetry") c.policy = SPRAY_POLICY_TELEMETRY;
        else if (p == "rr" || p == "round_robin") c.policy = SPRAY_POLICY_RR;
        else if (p == "hash") c.policy = SPRAY_POLICY_HASH;
        else throw ConfigError("engine config: unknown policy");
      }
      c.feedback_clamp = s.number_or("feedback_clamp", c.feedback_clamp);
    }
    if (j.contains("resilience")) {
      const Json& r = j.at("resilience");
      reject_unknown(r, {"failure_threshold", "degradation_ratio", "degradation_events", "degradation_min_t_obs_ms",
                         "probe_successes", "probe_bytes", "probe_interval_ms", "probe_backoff_mult",
                         "probe_backoff_cap", "max_attempts", "slice_timeout_ms"},
                     "resilience");
      spray_resilience_config& c = eo.res;
      c.failure_threshold = static_cast<int32_t>(r.number_or("failure_threshold", c.failure_threshold));
      c.degradation_ratio = r.number_or("degradation_ratio", c.degradation_ratio);
      c.degradation_events = static_cast<int32_t>(r.number_or("degradation_events", c.degradation_events));
      if (r.contains("degradation_min_t_obs_ms"))
        c.degradation_min_t_obs_s = r.at("degradation_min_t_obs_ms").as_number() * 1e-3;
      c.probe_successes_needed = static_cast<int32_t>(r.number_or("probe_successes", c.probe_successes_needed));
      c.probe_bytes = static_cast<uint64_t>(r.number_or("probe_bytes", double(c.probe_bytes)));
      if (r.contains("probe_interval_ms"))
        c.probe_interval_ns = static_cast<uint64_t>(r.at("probe_interval_ms").as_number() * 1e6);
      c.probe_backoff_mult = r.number_or("probe_backoff_mult", c.probe_backoff_mult);
      c.probe_backoff_cap = static_cast<int32_t>(r.number_or("probe_backoff_cap", c.probe_backoff_cap));
      c.max_attempts = static_cast<uint32_t>(r.number_or("max_attempts", c.max_attempts));
      if (r.contains("slice_timeout_ms"))
        c.slice_timeout_ns = static_cast<uint64_t>(r.at("slice_timeout_ms").as_number() * 1e6);
    }
    if (j.contains("b200")) {
      const Json& b = j.at("b200");
      reject_unknown(b, {"grid", "block", "chunk_bytes", "idle_exit_ms", "slice_capacity", "work_capacity",
                         "sub_capacity", "batch_slots", "gate_timeout_ms", "post_window", "fence_batch", "diag",
                         "no_peer", "staged_routes", "worker_fence", "copy", "fence", "bulk_stages"},
                     "b200");
      eo.post_window = static_cast<uint32_t>(b.number_or("post_window", eo.post_window));
      eo.fence_batch = static_cast<uint32_t>(b.number_or("fence_batch", eo.fence_batch));
      if (b.contains("diag")) eo.diag = b.at("diag").as_bool();
      if (b.contains("worker_fence")) {
        const std::string wf = b.at("worker_fence").as_string();
        if (wf != "sys" && wf != "gpu") throw ConfigError("b200.worker_fence must be sys or gpu");
        eo.worker_fence_sys = wf == "sys";
      }
      eo.bulk_stages = static_cast<uint32_t>(b.number_or("bulk_stages", eo.bulk_stages));
      if (eo.bulk_stages < 2 || eo.bulk_stages > 7) throw ConfigError("b200.bulk_stages must be in [2, 7]");
      if (b.contains("fence")) {
        const std::string fe = b.at("fence").as_string();
        if (fe != "release" && fe != "sc") throw ConfigError("b200.fence must be release or sc");
        eo.fence_release = fe == "release";
      }
      if (b.contains("copy")) {
        const std::string cp = b.at("copy").as_string();
        if (cp != "bulk" && cp != "ldg") throw ConfigError("b200.copy must be bulk or ldg");
        eo.copy_bulk = cp == "bulk";
      }
      if (b.contains("staged_routes")) eo.staged_routes = b.at("staged_routes").as_bool();
      if (b.contains("no_peer"))
        for (const Json& g : b.at("no_peer").arr) eo.no_peer.push_back(static_cast<int>(g.as_number()));
      if (eo.fence_batch < 1 || eo.fence_batch > 4) throw ConfigError("b200.fence_batch must be in [1, 4]");
      if (b.contains("gate_timeout_ms"))
        eo.gate_timeout_ns = static_cast<uint64_t>(b.at("gate_timeout_ms").as_number() * 1e6);
      eo.grid = static_cast<int>(b.number_or("grid", eo.grid));
      eo.block = static_cast<int>(b.number_or("block", eo.block));
      eo.chunk_bytes = static_cast<uint64_t>(b.number_or("chunk_bytes", double(eo.chunk_bytes)));
      if (b.contains("idle_exit_ms")) eo.idle_exit_ns = static_cast<uint64_t>(b.at("idle_exit_ms").as_number() * 1e6);
      eo.slice_capacity = static_cast<uint32_t>(b.number_or("slice_capacity", eo.slice_capacity));
      eo.work_capacity = static_cast<uint64_t>(b.number_or("work_capacity", double(eo.work_capacity)));
      eo.sub_capacity = static_cast<uint64_t>(b.number_or("sub_capacity", double(eo.sub_capacity)));
      eo.batch_slots = static_cast<uint32_t>(b.number_or("batch_slots", eo.batch_slots));
      if (eo.block % 32 || eo.block < 256 || eo.block > 1024) throw ConfigError("b200.block must be a multiple of 32 in [256, 1024]");
      if (eo.slice_capacity == 0 || eo.slice_capacity > (1u << 28))
        throw ConfigError("b200.slice_capacity must be in [1, 2^28]");
      if (eo.chunk_bytes < 4096 || (eo.chunk_bytes & (eo.chunk_bytes - 1)) || eo.chunk_bytes > (1ull << 31))
        throw ConfigError("b200.chunk_bytes must be a power of two in [4096, 2^31]");
    }
  } catch (const JsonError& e) {
    throw ConfigError(std::string("engine config: ") + e.what());
  }
  return eo;
}

// ------------------------------------------------------------------ construction

Engine::Engine(EngineOptions opts, const std::string& topology_json, int device)
    : opts_(std::move(opts)), topo_(Topology::parse(topology_json)), device_(device) {
  validate(opts_.sched, opts_.diffusion_weight);
  validate(opts_.res);
  synthesize_staged_routes();
  if (opts_.backends.empty()) throw ConfigError("engine: no backends configured");
  for (const std::string& b : opts_.backends) caps_.push_back(Capabilities::preset(b));
  if (topo_.rail_count() > size_t(kMaxRails)) throw ConfigError("topology: more than 64 rails per engine");
  for (RailIndex i = 0; i < topo_.rail_count(); ++i) {
    const RailDecl& r = topo_.rail(i);
    if (r.executor == 2 && r.via < 0)
      throw ConfigError("rail '" + r.id + "': relay executor needs \"via\" (the relay GPU ordinal)");
    if (r.executor == 1) {
      has_ce_ = true;
      if (r.ce_index >= 8) throw ConfigError("rail '" + r.id + "': ce_index must be < 8");
    }
  }
  // A single-GPU host-staging fabric: one node with device memory (no peer HBM paths)
  // and every SM rail serving pinned host memory.
  uint32_t n_sm = 0, n_sm_host = 0, n_dev_nodes = 0;
  for (const NodeDecl& n : topo_.nodes()) {
    bool dev = false;
    for (const DeviceDecl& d : n.devices) dev = dev || d.kind == DeviceKind::kDeviceMemory;
    n_dev_nodes += dev ? 1 : 0;
  }
  for (RailIndex i = 0; i < topo_.rail_count(); ++i) {
    if (topo_.rail(i).executor != 0) continue;
    ++n_sm;
    bool host = false;
    for (const NodeDecl& n : topo_.nodes())
      for (const DeviceDecl& d : n.devices)
        if (d.kind == DeviceKind::kHostMemory && topo_.tier_from_device(d.id, i)) host = true;
    if (host) ++n_sm_host;
  }
  host_only_sm_ = n_dev_nodes == 1 && n_sm > 0 && n_sm_host == n_sm;
  slot_busy_.assign(opts_.batch_slots, 0);
}

// Staged-route synthesis (orchestrator.cpp:120-234, engine.cpp:465-610): a GPU node this
// engine's GPU has no peer access to (cudaDeviceCanAccessPeer, or b200.no_peer) cannot be
// reached by direct rails. With b200.staged_routes (default on) the engine declares a
// host-staged relay rail pair towards it (<own node>.st<K>, <K's node>.st<K>): hop 1 stores
// into a bounded pinned-host pool, a forwarder on GPU K drains it into K's HBM. Planning
// then routes transfers into K over that rail only (set_for), and keeps it out of every
// route a direct rail can serve.
void Engine::synthesize_staged_routes() {
  std::string own;
  for (const NodeDecl& nd : topo_.nodes())
    if (topo_.node_gpu(nd.id) == device_) own = nd.id;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    cudaGetLastError();
    ndev = 0;
  }
  std::vector<std::pair<std::string, int>> far;
  for (const NodeDecl& nd : topo_.nodes()) {
    const int g = topo_.node_gpu(nd.id);
    if (g < 0 || g == device_) continue;
    bool peer = true;
    if (std::find(opts_.no_peer.begin(), opts_.no_peer.end(), g) != opts_.no_peer.end()) {
      peer = false;
    } else if (g < ndev && device_ < ndev) {
      int ok = 1;
      if (cudaDeviceCanAccessPeer(&ok, device_, g) != cudaSuccess) cudaGetLastError(), ok = 1;
      peer = ok != 0;
    }
    if (!peer) {
      no_peer_gpus_.insert(g);
      far.emplace_back(nd.id, g);
    }
  }
  if (!opts_.staged_routes || own.empty()) return;
  for (const auto& [node, g] : far) {
    const std::string tag = ".st" + std::to_string(g);
    if (topo_.rail_index(own + tag)) continue;  // declared by the application
    RailDecl a;
    a.id = own + tag;
    a.node = own;
    a.backend = "cuda";
    a.bandwidth = 55e9;  // a pinned-host pool: one PCIe Gen5 x16 crossing each way
    a.tier = 1;
    a.executor = 2;
    a.gpu = device_;
    a.via = g < ndev ? g : device_;  // (test boxes with fewer GPUs: the forwarder runs here)
    a.host_staged = true;
    topo_.add_rail(a);
    RailDecl b = a;
    b.id = node + tag;
    b.node = node;
    b.gpu = g;
    if (!topo_.rail_index(b.id)) topo_.add_rail(b);
  }
}

Engine::~Engine() {
  try {
    stop();
  } catch (...) {
  }
  if (!wedged_) free_device();
}

void Engine::alloc_device() {
  CK(cudaSetDevice(device_));
  CK(spray_launch::preload_kernels());  // no lazy load may wait behind the persistent kernel
  CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
  auto host = [&](size_t bytes) -> void* {
    void* p = nullptr;
    CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(p, 0, bytes);
    return p;
  };
  auto dev = [&](size_t bytes) -> void* {
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMemsetAsync(p, 0, bytes, copy_stream_));
    dev_allocs_.push_back(p);
    return p;
  };
  auto dptr = [&](void* h) -> void* {
    void* d = nullptr;
    CK(cudaHostGetDevicePointer(&d, h, 0));
    return d;
  };
  const uint32_t nr = rail_count();
  ctl_ = static_cast<Control*>(host(sizeof(Control)));
  ring_ = static_cast<Intent*>(host(sizeof(Intent) * opts_.sub_capacity));
  bmirror_ = static_cast<BatchDev*>(host(sizeof(BatchDev) * opts_.batch_slots));
  faults_ = static_cast<FaultDev*>(host(sizeof(FaultDev) * kMaxRails));
  rmirror_ = static_cast<RailState*>(host(sizeof(RailState) * kMaxRails));
  const uint64_t xc_cap = 1 << 16;
  ce_ring_ = static_cast<CeOrder*>(host(sizeof(CeOrder) * 8 * ce_cap));
  xc_ring_ = static_cast<Completion*>(host(sizeof(Completion) * xc_cap));

  E_ = EngineDev{};
  E_.ctl = static_cast<Control*>(dptr(ctl_));
  E_.sub_ring = static_cast<Intent*>(dptr(ring_));
  E_.sub_cap = opts_.sub_capacity;
  E_.batches = static_cast<BatchDev*>(dptr(bmirror_));
  E_.n_batch_slots = opts_.batch_slots;
  E_.batches_hbm = static_cast<BatchDev*>(dev(sizeof(BatchDev) * opts_.batch_slots));
  E_.faults = static_cast<FaultDev*>(dptr(faults_));
  E_.rail_mirror = static_cast<RailState*>(dptr(rmirror_));
  E_.ce_ring = static_cast<CeOrder*>(dptr(ce_ring_));
  E_.ce_cap = ce_cap;
  E_.xc_ring = static_cast<Completion*>(dptr(xc_ring_));
  E_.xc_cap = xc_cap;

  // rails
  std::vector<RailDesc> rd(nr);
  std::vector<RailState> rs(nr);
  const auto ranks = topo_.id_ranks();
  std::vector<std::tuple<uint32_t, int, bool>> relay_rails;  // (relay index, via GPU, host staged)
  for (uint32_t i = 0; i < nr; ++i) {
    const RailDecl& r = topo_.rail(i);
    rd[i] = RailDesc{};
    // posting window (SimBackend inflight_window, sim_backend.cpp:81): units in flight per
    // rail. SM / relay rails: a copy warp holds up to fence_batch counted-late chunks plus its
    // prefetched ticket, so twice (fence_batch + 1) chunks per warp keep one rail alone
    // saturating every warp with work queued (tools/gpu/run_c3.sh: 2 x warps throttles the
    // KV batch by 7% at fence_batch 4); CE rails: orders, at most half the proxy ring (the
    // ring can then never overrun the proxy)
    {
      const uint32_t warps = static_cast<uint32_t>(std::max(1, launch_grid() - 1)) * (opts_.block / 32);
      uint32_t w = opts_.post_window ? opts_.post_window
                                     : (r.executor == 1 ? 2048u : std::max(64u, 2 * (opts_.fence_batch + 1) * warps));
      // host-staged relays: the staging pool's slots (the forwarder's PCIe reads take
      // hundreds of µs under load, so the whole pool is kept in flight)
      if (r.host_staged && !opts_.post_window) w = 2048;
      rd[i].window = r.executor == 1 ? std::min<uint32_t>(w, ce_cap / 2) : w;
    }
    rd[i].bandwidth = r.bandwidth;
    rd[i].base_tier = r.tier;
    rd[i].id_rank = ranks[i];
    rd[i].executor = r.executor;
    rd[i].gpu = r.gpu;
    rd[i].via = r.via;
    rd[i].ce_index = r.ce_index;
    if (r.executor == 2) {
      if (relay_rails.size() >= size_t(kMaxRelays)) throw ConfigError("more than 8 relay rails");
      rd[i].ce_index = static_cast<uint32_t>(relay_rails.size());
      relay_rails.emplace_back(rd[i].ce_index, r.via, r.host_staged);
    }
    // probe counterparts (resilience.cpp:17-44): same-backend rails on other nodes, the
    // 1:1 affinity partner first, nodes in id order; node-local backends probe themselves
    {
      const auto& own = topo_.rails_on(r.node, r.backend);
      size_t my_pos = 0;
      for (size_t k = 0; k < own.size(); ++k)
        if (own[k] == i) my_pos = k;
      std::vector<std::string> others;
      for (const NodeDecl& n : topo_.nodes())
        if (n.id != r.node && !topo_.rails_on(n.id, r.backend).empty()) others.push_back(n.id);
      std::sort(others.begin(), others.end());
      std::vector<uint32_t> ps;
      for (const std::string& n : others) {
        const auto& theirs = topo_.rails_on(n, r.backend);
        const uint32_t first = theirs[my_pos % theirs.size()];
        ps.push_back(first);
        for (uint32_t t : theirs)
          if (t != first) ps.push_back(t);
      }
      if (ps.empty()) ps.push_back(i);
      rd[i].n_partners = static_cast<uint8_t>(std::min<size_t>(ps.size(), 15));
      for (size_t k = 0; k < rd[i].n_partners; ++k) rd[i].partners[k] = static_cast<uint8_t>(ps[k]);
    }
    rs[i] = RailState{};
    rs[i].beta0 = opts_.sched.beta0_init_s;  // scheduler.cpp:87-90
    rs[i].beta1 = opts_.sched.beta1_init;
    rs[i].health = kHealthy;
  }
  void* rails_d = dev(sizeof(RailDesc) * kMaxRails);
  void* state_d = dev(sizeof(RailState) * kMaxRails);
  CK(cudaMemcpyAsync(rails_d, rd.data(), sizeof(RailDesc) * nr, cudaMemcpyHostToDevice, copy_stream_));
  CK(cudaMemcpyAsync(state_d, rs.data(), sizeof(RailState) * nr, cudaMemcpyHostToDevice, copy_stream_));
  std::memcpy(rmirror_, rs.data(), sizeof(RailState) * nr);
  E_.rails = static_cast<RailDesc*>(rails_d);
  E_.n_rails = nr;
  E_.rail_state = static_cast<RailState*>(state_d);
  E_.sets = static_cast<CandSet*>(dev(sizeof(CandSet) * opts_.max_sets));
  E_.n_sets = 0;
  E_.n_slices = opts_.slice_capacity;
  E_.slices = static_cast<Slice*>(dev(sizeof(Slice) * opts_.slice_capacity));
  E_.free_slices = static_cast<uint64_t*>(dev(sizeof(uint64_t) * opts_.slice_capacity));
  {
    // (slot | base << 32): every slot starts with a zero chunk-counter base
    std::vector<uint64_t> fl(opts_.slice_capacity);
    for (uint32_t i = 0; i < opts_.slice_capacity; ++i) fl[i] = opts_.slice_capacity - 1 - i;
    CK(cudaMemcpyAsync(E_.free_slices, fl.data(), fl.size() * 8, cudaMemcpyHostToDevice, copy_stream_));
    CK(cudaStreamSynchronize(copy_stream_));
  }
  E_.slot_ctr = static_cast<unsigned long long*>(dev(sizeof(unsigned long long) * opts_.slice_capacity));
  E_.deadline = static_cast<unsigned long long*>(dev(sizeof(unsigned long long) * opts_.slice_capacity));
  E_.pending = static_cast<uint32_t*>(dev(sizeof(uint32_t) * opts_.slice_capacity * std::max<size_t>(1, nr)));
  E_.pend_pos = static_cast<uint64_t*>(dev(sizeof(uint64_t) * 2 * kMaxRails));
  E_.slice_timeout_ns = opts_.res.slice_timeout_ns;
  E_.fence_batch = opts_.fence_batch;
  E_.diag = opts_.diag ? 1u : 0u;
  E_.worker_fence_sys = opts_.worker_fence_sys ? 1u : 0u;
  E_.copy_bulk = opts_.copy_bulk ? 1u : 0u;
  E_.fence_release = opts_.fence_release ? 1u : 0u;
  E_.bulk_stages = opts_.bulk_stages;
  // the deadline scan runs ~8 times per timeout (the reference's wheel has 10 ms buckets,
  // engine.cpp:18), bounded to [0.2, 10] ms
  E_.timeout_scan_ns = std::min<uint64_t>(10'000'000, std::max<uint64_t>(200'000, opts_.res.slice_timeout_ns / 8));
  E_.faults_hbm = static_cast<FaultDev*>(dev(sizeof(FaultDev) * kMaxRails));
  E_.faults_any = static_cast<uint32_t*>(dev(sizeof(uint32_t)));
  E_.any_failed = static_cast<uint32_t*>(dev(sizeof(uint32_t)));
  E_.next_free = static_cast<unsigned long long*>(dev(sizeof(unsigned long long) * kMaxRails));
  {  // telemetry windows: every cell starts empty (window = ~0)
    const size_t tb = sizeof(TeleCell) * kTeleWindows * std::max<size_t>(1, topo_.rail_count());
    E_.tele = static_cast<TeleCell*>(dev(tb));
    CK(cudaMemset(E_.tele, 0xff, tb));
    E_.window_ns = opts_.window_ns;
  }
  E_.exit_flag = static_cast<uint32_t*>(dev(sizeof(uint32_t)));
  E_.board_hbm = static_cast<int64_t*>(dev(sizeof(int64_t) * kMaxRails));
  E_.board = nullptr;
  E_.omega = 0.0;  // until a board is attached (scheduler.cpp:110: no board, local queue only)
  E_.has_ce = has_ce_ ? 1u : 0u;
  E_.work_cap = opts_.work_capacity;
  E_.work = static_cast<WorkItem*>(dev(sizeof(WorkItem) * opts_.work_capacity));
  E_.work_head = static_cast<unsigned long long*>(dev(sizeof(unsigned long long)));
  E_.comp_cap = std::max<uint64_t>(2ull * opts_.slice_capacity, 1024);
  E_.comp = static_cast<uint64_t*>(dev(sizeof(uint64_t) * E_.comp_cap));
  E_.comp_tail = static_cast<unsigned long long*>(dev(sizeof(unsigned long long)));
  E_.parked_cap = opts_.slice_capacity;
  E_.parked = static_cast<uint32_t*>(dev(sizeof(uint32_t) * opts_.slice_capacity));
  E_.persist = static_cast<uint64_t*>(dev(sizeof(uint64_t) * kPNum));
  {
    uint64_t p[kPNum] = {0};
    p[kPFreeTop] = opts_.slice_capacity;
    CK(cudaMemcpyAsync(E_.persist, p, sizeof(p), cudaMemcpyHostToDevice, copy_stream_));
  }
  E_.trace_ev = nullptr;
  E_.trace_dec = nullptr;
  E_.trace_cap = 0;
  // constants
  E_.tolerance = opts_.sched.tolerance;
  for (int t = 0; t < 3; ++t) E_.penalty[t] = opts_.sched.penalty[t];
  E_.alpha = opts_.sched.ewma_alpha;
  E_.beta0_init = opts_.sched.beta0_init_s;
  E_.beta1_init = opts_.sched.beta1_init;
  E_.clamp = opts_.sched.feedback_clamp;
  E_.reset_interval = opts_.sched.reset_interval_ns;
  E_.min_slice = opts_.sched.min_slice_size;
  E_.max_slices = opts_.sched.max_slices_per_transfer;
  E_.policy = static_cast<uint32_t>(opts_.sched.policy);
  E_.failure_threshold = opts_.res.failure_threshold;
  E_.degradation_events = opts_.res.degradation_events;
  E_.probe_successes = opts_.res.probe_successes_needed;
  E_.degradation_ratio = opts_.res.degradation_ratio;
  E_.degradation_min_t = opts_.res.degradation_min_t_obs_s;
  E_.max_attempts = opts_.res.max_attempts;
  E_.probe_interval = opts_.res.probe_interval_ns;
  E_.probe_bytes = std::min<uint64_t>(opts_.res.probe_bytes, 1ull << 20);
  E_.probe_backoff_mult = opts_.res.probe_backoff_mult;
  E_.probe_backoff_cap = opts_.res.probe_backoff_cap;
  E_.scratch = reinterpret_cast<uint64_t>(dev(2 * E_.probe_bytes));
  E_.chunk_bytes = opts_.chunk_bytes;
  E_.gate_timeout_ns = opts_.gate_timeout_ns;
  E_.n_gates = 0;
  E_.chunk_shift = 0;
  while ((1ull << E_.chunk_shift) < opts_.chunk_bytes) ++E_.chunk_shift;
  // engine epoch on the device clock
  uint64_t* ep = static_cast<uint64_t*>(dev(sizeof(uint64_t)));
  CK(spray_launch::launch_epoch(ep, copy_stream_));
  CK(cudaMemcpyAsync(&E_.epoch, ep, sizeof(uint64_t), cudaMemcpyDeviceToHost, copy_stream_));
  CK(cudaStreamSynchronize(copy_stream_));
  ctl_->epoch = E_.epoch;
  ctl_->idle_exit_ns = opts_.idle_exit_ns;
  for (const auto& rr : relay_rails) setup_relay(std::get<0>(rr), std::get<1>(rr), std::get<2>(rr));
  E_.n_relays = static_cast<uint32_t>(relay_rails.size());
  E_.has_staged = 0;
  for (const auto& rr : relay_rails) E_.has_staged |= std::get<2>(rr) ? 1u : 0u;
  if (has_ce_) {
    ce_streams_.resize(8);
    for (auto& s : ce_streams_) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
}

// A relay rail's state: staging slots, descriptors and the exit generation in the relay
// GPU's HBM (hop 2 reads them locally), the slot-free rounds and the ticket counter here
// (hop 1 polls them locally). Peer access: this GPU <-> via both ways (staging stores,
// completion atomics), via -> every other GPU it can reach (hop-2 destinations).
void Engine::setup_relay(uint32_t idx, int via, bool host_staged) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (via >= n) throw ConfigError("relay rail: via GPU " + std::to_string(via) + " does not exist");
  auto enable = [](int peer) {
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
    cudaGetLastError();
  };
  if (!host_staged) {  // device staging: hop 1 stores into K's HBM, hop 2 counts in ours
    int a = 1, b = 1;
    if (via != device_) {
      CK(cudaDeviceCanAccessPeer(&a, device_, via));
      CK(cudaDeviceCanAccessPeer(&b, via, device_));
    }
    if (!a || !b) throw ConfigError("relay rail: no peer access between GPU " + std::to_string(device_) + " and " +
                                    std::to_string(via) + " (declare it \"staging\": \"host\")");
    CK(cudaSetDevice(device_));
    if (via != device_) enable(via);
    CK(cudaSetDevice(via));
    for (int j = 0; j < n; ++j) {
      int ok = 0;
      if (j != via && cudaDeviceCanAccessPeer(&ok, via, j) == cudaSuccess && ok) enable(j);
    }
  }
  CK(cudaSetDevice(via));
  CK(spray_launch::preload_kernels());  // the forwarder launches on `via` while engines run
  RelayHost h;
  h.via = via;
  CK(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
  constexpr uint32_t kSlots = 2048;  // power of two: 64 MiB of 32 KiB granules (engine.hpp:56-58's pool)
  RelayDev R{};
  R.n_slots = kSlots;
  R.via = static_cast<uint32_t>(via);
  R.host_staged = host_staged ? 1u : 0u;
  auto on_via = [&](size_t bytes) -> void* {
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMemset(p, 0, bytes));
    h.via_allocs.push_back(p);
    return p;
  };
  auto pinned = [&](size_t bytes) -> void* {  // mapped pinned host memory both GPUs address
    void* p = nullptr;
    CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(p, 0, bytes);
    h.host_allocs.push_back(p);
    void* d = nullptr;
    CK(cudaHostGetDevicePointer(&d, p, 0));
    return d;
  };
  R.head = static_cast<unsigned long long*>(on_via(sizeof(unsigned long long)));
  if (host_staged) {
    R.staging = static_cast<uint8_t*>(pinned(size_t(kSlots) << E_.chunk_shift));
    R.desc = static_cast<RelayDesc*>(pinned(sizeof(RelayDesc) * kSlots));
    R.exit_gen = static_cast<uint32_t*>(pinned(sizeof(uint32_t)));
    R.seq = static_cast<uint32_t*>(pinned(sizeof(uint32_t) * kSlots));
    R.done_stamp = static_cast<uint64_t*>(pinned(sizeof(uint64_t) * kSlots));
  } else {
    R.staging = static_cast<uint8_t*>(on_via(size_t(kSlots) << E_.chunk_shift));
    R.desc = static_cast<RelayDesc*>(on_via(sizeof(RelayDesc) * kSlots));
    R.exit_gen = static_cast<uint32_t*>(on_via(sizeof(uint32_t)));
  }
  CK(cudaSetDevice(device_));
  void* p = nullptr;
  if (!host_staged) {
    CK(cudaMalloc(&p, sizeof(uint32_t) * kSlots));
    CK(cudaMemset(p, 0, sizeof(uint32_t) * kSlots));
    dev_allocs_.push_back(p);
    R.seq = static_cast<uint32_t*>(p);
  } else {
    CK(cudaMalloc(&p, sizeof(unsigned long long)));
    CK(cudaMemset(p, 0, sizeof(unsigned long long)));
    dev_allocs_.push_back(p);
    R.consumed = static_cast<unsigned long long*>(p);
    CK(cudaMalloc(&p, sizeof(RelayDone) * kSlots));
    CK(cudaMemset(p, 0, sizeof(RelayDone) * kSlots));
    dev_allocs_.push_back(p);
    R.done = static_cast<RelayDone*>(p);
    CK(cudaMalloc(&p, sizeof(uint32_t)));
    CK(cudaMemset(p, 0, sizeof(uint32_t)));
    dev_allocs_.push_back(p);
    R.writers = static_cast<uint32_t*>(p);
  }
  CK(cudaMalloc(&p, sizeof(unsigned long long)));
  CK(cudaMemset(p, 0, sizeof(unsigned long long)));
  dev_allocs_.push_back(p);
  R.tail = static_cast<unsigned long long*>(p);
  E_.relays[idx] = R;
  if (relays_.size() <= idx) relays_.resize(idx + 1);
  relays_[idx] = std::move(h);
}

// Every forwarder of the previous launch has returned (each exits once the engine kernel
// has published its exit generation).
void Engine::sync_relays() {
  for (RelayHost& h : relays_)
    if (h.stream) CK(cudaStreamSynchronize(h.stream));
}

void Engine::free_device() {
  for (RelayHost& h : relays_) {
    cudaSetDevice(h.via);
    if (h.stream) cudaStreamSynchronize(h.stream), cudaStreamDestroy(h.stream);
    for (void* p : h.via_allocs) cudaFree(p);
    for (void* p : h.host_allocs) cudaFreeHost(p);
  }
  relays_.clear();
  cudaSetDevice(device_);
  for (void* p : dev_allocs_) cudaFree(p);
  dev_allocs_.clear();
  for (void* p : {static_cast<void*>(ctl_), static_cast<void*>(ring_), static_cast<void*>(bmirror_),
                  static_cast<void*>(faults_), static_cast<void*>(rmirror_), static_cast<void*>(ce_ring_),
                  static_cast<void*>(xc_ring_)})
    if (p) cudaFreeHost(p);
  ctl_ = nullptr;
  ring_ = nullptr;
  bmirror_ = nullptr;
  faults_ = nullptr;
  rmirror_ = nullptr;
  ce_ring_ = nullptr;
  xc_ring_ = nullptr;
  for (auto& kv : segs_)
    for (void* p : kv.second.registered) cudaHostUnregister(p);
  if (board_registered_) cudaHostUnregister(board_registered_), board_registered_ = nullptr;
  if (hold_) cudaFreeHost(const_cast<uint32_t*>(hold_)), hold_ = nullptr, hold_dev_ = nullptr;
  if (stage_host_) cudaFreeHost(stage_host_), stage_host_ = nullptr;
  for (auto& d : stage_dev_) d = nullptr;  // freed with dev_allocs_
  for (auto& s : ce_streams_)
    if (s) cudaStreamDestroy(s);
  ce_streams_.clear();
  if (stream_) cudaStreamDestroy(stream_);
  if (copy_stream_) cudaStreamDestroy(copy_stream_);
  stream_ = copy_stream_ = nullptr;
}

void Engine::start() {
  std::lock_guard<std::mutex> lk(mu_);
  if (started_) return;
  alloc_device();
  started_ = true;
  if (has_ce_) {
    ce_run_ = true;
    xc_reserve_ = ctl_->xc_head;
    uint32_t used = 0;  // one proxy thread per CE stream a rail uses: cudaMemcpyAsync calls in parallel
    for (RailIndex i = 0; i < topo_.rail_count(); ++i)
      if (topo_.rail(i).executor == 1) used |= 1u << (topo_.rail(i).ce_index & 7);
    for (int k = 0; k < 8; ++k)
      if (used & (1u << k)) ce_threads_.emplace_back([this, k] { ce_proxy_loop(k); });
  }
}

void Engine::stop() {
  std::lock_guard<std::mutex> lk(mu_);
  if (!started_) return;
  ctl_->stop = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  // bounded: a kernel that never observes the stop word leaves the engine wedged (its
  // memory is then leaked rather than freed under a running kernel) and says so
  auto drain = [&](cudaStream_t s) {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q != cudaErrorNotReady) return true;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20)) return false;
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  };
  bool ok = drain(stream_);
  for (RelayHost& h : relays_)
    if (h.stream) ok = drain(h.stream) && ok;
  if (has_ce_) {
    ce_run_ = false;
    for (auto& t : ce_threads_)
      if (t.joinable()) t.join();
    ce_threads_.clear();
  }
  started_ = false;
  if (!ok) {
    wedged_ = true;
    throw EngineError("engine kernel did not stop within 20 s");
  }
  ctl_->stop = 0;
  ctl_->state = 0;
}

// ------------------------------------------------------------------ kernel lifecycle

int Engine::launch_grid() {
  int grid = opts_.grid;
  if (grid <= 0) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
    grid = sms;
    // Every SM rail stages through pinned host memory: 48 worker CTAs (384 warps) already
    // saturate a Gen5 x16 root in each direction, while more writers only deepen the
    // posted-write backlog that every fence and L2 access then waits behind
    // (profiles/pcie_peak.json: 1184 writers -> 72 us fences, 21 us L2 reads).
    if (host_only_sm_) grid = std::min(grid, 1 + kHostLinkCtas);
    // this GPU relays for others: leave 16 SMs to the forwarders (64 CTAs, 4 per SM)
    for (RailIndex i = 0; i < topo_.rail_count(); ++i)
      if (topo_.rail(i).executor == 2 && topo_.rail(i).via == device_) grid = std::min(grid, sms - 16);
  }
  return grid;
}

void Engine::launch() {
  CK(cudaSetDevice(device_));
  const int grid = launch_grid();
  ctl_->stop = 0;
  ctl_->drain = drain_ ? 1u : 0u;
  ctl_->state = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  sync_relays();
  E_.launch_gen = ++launch_gen_;
  {  // the device-written words this launch resumes from (no kernel is resident now)
    LaunchSnap& sn = E_.snap;
    sn.sub_head = ctl_->sub_head;
    sn.bulk_done = ctl_->bulk_done;
    sn.xc_head = ctl_->xc_head;
    for (int k = 0; k < 8; ++k) sn.ce_tail[k] = ctl_->ce_tail[k];
    sn.idle_exit_ns = ctl_->idle_exit_ns;
    sn.bytes_dispatched = ctl_->bytes_dispatched;
    sn.bytes_terminated = ctl_->bytes_terminated;
    sn.batches_failed = ctl_->batches_failed;
    sn.heal_fault_start = ctl_->heal_fault_start;
    sn.heal_first_ok = ctl_->heal_first_ok;
    sn.failed_attempts = ctl_->failed_attempts;
    sn.retried_ok = ctl_->retried_ok;
    sn.trace_n = ctl_->trace_n;
    sn.trace_dn = ctl_->trace_dn;
    sn.drain = ctl_->drain;
    sn.trace_on = ctl_->trace_on;
  }
  CK(spray_launch::launch_engine(E_, grid, opts_.block, stream_));
  bool local_relay = false;
  for (const RelayHost& h : relays_) local_relay |= h.via == device_;
  if (local_relay) {  // forwarders beside the engine start only once every engine CTA has
    const auto t0 = std::chrono::steady_clock::now();
    while (ctl_->resident_gen != E_.launch_gen) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5))
        throw EngineError("engine kernel not resident after 5 s");
      _mm_pause();
    }
  }
  for (uint32_t r = 0; r < relays_.size(); ++r) {  // hop 2 on each relay GPU
    CK(cudaSetDevice(relays_[r].via));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, relays_[r].via));
    // beside this engine: the SMs launch_grid() left free, two forwarder CTAs each
    if (relays_[r].via == device_) sms = std::max(2, 2 * (sms - grid));
    CK(cudaMemsetAsync(E_.relays[r].head, 0, sizeof(unsigned long long), relays_[r].stream));
    CK(spray_launch::launch_relay_forward(E_, r, sms, relays_[r].stream));
  }
  if (!relays_.empty()) CK(cudaSetDevice(device_));
}

bool Engine::running_kernel() { return ctl_ && ctl_->state != 0; }

// EXITING handshake (spray_kernel.cu scheduler exit): the device publishes EXITING,
// fences and re-checks the ring; the host publishes the tail, fences and reads state.
void Engine::ensure_running() {
  std::atomic_thread_fence(std::memory_order_seq_cst);
  uint32_t st = ctl_->state;
  if (st == 1) return;
  while (st == 2) {
    _mm_pause();
    st = ctl_->state;
  }
  if (st == 1) return;
  CK(cudaStreamSynchronize(stream_));  // previous launch fully drained
  launch();
}

void Engine::set_drain(bool on) {
  std::lock_guard<std::mutex> lk(mu_);
  drain_ = on;
  if (ctl_) ctl_->drain = on ? 1u : 0u;
}

// ------------------------------------------------------------------ segments

void Engine::register_segment(const spray_segment_desc& d) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!d.id || !*d.id) throw ConfigError("segment id must be non-empty");
  const std::string node = d.node ? d.node : "";
  if (!topo_.node(node)) throw ConfigError(std::string("segment '") + d.id + "': unknown node '" + node + "'");
  if (d.n_buffers == 0 || !d.buffers) throw ConfigError(std::string("segment '") + d.id + "': no buffers");
  if (d.medium == SPRAY_MEDIUM_FILE)
    throw ConfigError(std::string("segment '") + d.id + "': file media are not served by the B200 data plane");
  SegRec rec;
  rec.seg.id = d.id;
  rec.seg.medium = d.medium == SPRAY_MEDIUM_DEVICE ? Medium::kDevice : Medium::kHost;
  rec.seg.node = node;
  rec.seg.id_hash = hash128(rec.seg.id);
  for (uint32_t i = 0; i < d.n_buffers; ++i)
    rec.seg.buffers.push_back(Buffer{d.buffers[i].offset, d.buffers[i].length, d.buffers[i].data, 0});
  std::sort(rec.seg.buffers.begin(), rec.seg.buffers.end(),
            [](const Buffer& a, const Buffer& b) { return a.offset < b.offset; });
  for (size_t i = 0; i + 1 < rec.seg.buffers.size(); ++i)
    if (rec.seg.buffers[i].offset + rec.seg.buffers[i].length > rec.seg.buffers[i + 1].offset)
      throw ConfigError(std::string("segment '") + d.id + "': OverlappingBuffers");
  for (const Buffer& b : rec.seg.buffers) {
    if (b.length == 0) throw ConfigError(std::string("segment '") + d.id + "': zero-length buffer");
    if (!b.data) throw ConfigError(std::string("segment '") + d.id + "': null buffer");
  }
  if (d.device && *d.device) {
    if (!topo_.find_device(node, d.device))
      throw ConfigError(std::string("segment '") + d.id + "': unknown device '" + d.device + "'");
    rec.seg.device = d.device;
  } else if (const DeviceDecl* dd = topo_.first_device_of_kind(
                 node, rec.seg.medium == Medium::kDevice ? DeviceKind::kDeviceMemory : DeviceKind::kHostMemory)) {
    rec.seg.device = dd->id;
  }
  if (segs_.count(rec.seg.id)) throw ConfigError("duplicate segment id '" + rec.seg.id + "'");
  segs_.emplace(rec.seg.id, std::move(rec));
}

// Device-usable addresses: pinned host buffers through their mapped alias (registering
// pageable ones), peer HBM after enabling peer access. Done lazily, on the first
// transfer that touches the segment, so registration itself stays host-only.
void Engine::translate(SegRec& s) {
  if (s.translated) return;
  CK(cudaSetDevice(device_));
  for (Buffer& b : s.seg.buffers) {
    if (s.seg.medium == Medium::kHost) {
      void* dp = nullptr;
      if (cudaHostGetDevicePointer(&dp, b.data, 0) != cudaSuccess) {
        cudaGetLastError();
        CK(cudaHostRegister(b.data, b.length, cudaHostRegisterMapped | cudaHostRegisterPortable));
        s.registered.push_back(b.data);
        CK(cudaHostGetDevicePointer(&dp, b.data, 0));
      }
      b.dev_addr = reinterpret_cast<uint64_t>(dp);
    } else {
      cudaPointerAttributes a{};
      CK(cudaPointerGetAttributes(&a, b.data));
      if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
        throw ConfigError("segment '" + s.seg.id + "': device medium buffer is not device memory");
      if (a.device != device_) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      }
      b.dev_addr = reinterpret_cast<uint64_t>(b.data);
    }
  }
  s.translated = true;
}

// ------------------------------------------------------------------ planning

uint32_t Engine::set_for(const Segment& src, const Segment& dst, Direction dir) {
  const std::string key = src.id + '\x1f' + dst.id + '\x1f' + (dir == Direction::kWrite ? 'w' : 'r');
  auto it = set_cache_.find(key);
  if (it != set_cache_.end()) return it->second;
  CK(cudaSetDevice(device_));
  auto routes = build_plan(topo_, src, dst, dir, opts_.sched.penalty, caps_);  // throws NoRouteError
  // The plan's routes in order (one per backend chain, build_plan's order). The first is
  // the active route; each set names the next, which a slice moves to once its attempts
  // on a route are exhausted (substitute_or_fail, engine.cpp:676-683).
  std::vector<Route> plan;
  for (size_t k = 0; k < routes.size(); ++k) {
    Route r = routes[k];
    if (k == 0) {
      filter_staged(r, src, dst);  // throws NoRouteError for the active route
    } else {
      try {
        filter_staged(r, src, dst);
      } catch (const NoRouteError&) {
        continue;
      }
    }
    plan.push_back(std::move(r));
  }
  if (sets_.size() + plan.size() > opts_.max_sets) throw EngineError("candidate-set table full");
  const uint32_t first = static_cast<uint32_t>(sets_.size());
  for (size_t k = 0; k < plan.size(); ++k)
    add_set(plan[k], k + 1 < plan.size() ? first + static_cast<uint32_t>(k + 1) : kNoSet);
  set_cache_.emplace(key, first);
  return first;
}

uint32_t Engine::add_set(const Route& r, uint32_t next) {
  if (r.candidates.size() > size_t(kMaxLocals)) throw ConfigError("route has more than 32 local rails");
  CandSet cs{};
  cs.next_set = next;
  cs.n_locals = static_cast<uint32_t>(r.candidates.size());
  for (size_t l = 0; l < r.candidates.size(); ++l) {
    const LocalCandidate& c = r.candidates[l];
    if (c.pairs.size() > size_t(kMaxPairs)) throw ConfigError("more than 16 remote options for one rail");
    cs.local[l] = c.local;
    cs.n_pairs[l] = static_cast<uint32_t>(c.pairs.size());
    for (size_t p = 0; p < c.pairs.size(); ++p) {
      cs.pair_remote[l][p] = c.pairs[p].remote;
      cs.pair_tier[l][p] = c.pairs[p].tier;
      cs.pair_aff[l][p] = c.pairs[p].affinity ? 1 : 0;
    }
  }
  const uint32_t id = static_cast<uint32_t>(sets_.size());
  if (started_) {
    CK(cudaMemcpyAsync(const_cast<CandSet*>(E_.sets) + id, &cs, sizeof(cs), cudaMemcpyHostToDevice, copy_stream_));
    CK(cudaStreamSynchronize(copy_stream_));
  }
  sets_.push_back(r.candidates);
  return id;
}

std::vector<int32_t> Engine::plan_candidates(const std::string& s, const std::string& d, int dir,
                                             std::string* backend) {
  std::lock_guard<std::mutex> lk(mu_);
  auto si = segs_.find(s), di = segs_.find(d);
  if (si == segs_.end() || di == segs_.end()) throw EngineError("unknown segment id");
  auto routes = build_plan(topo_, si->second.seg, di->second.seg, dir == SPRAY_READ ? Direction::kRead : Direction::kWrite,
                           opts_.sched.penalty, caps_);
  Route r = routes.front();
  filter_staged(r, si->second.seg, di->second.seg);
  if (backend) *backend = r.backend;
  std::vector<int32_t> out{1};
  append_stream(out, r.candidates);
  return out;
}

// Staged routes only where no direct route exists (orchestrator.cpp:120-122): into a GPU
// without peer access, keep just the host-staged relay rails; everywhere else, drop them.
// A staged route starts at this engine's GPU: moving out of a GPU without peer access
// needs an engine there.
void Engine::filter_staged(Route& r, const Segment& src, const Segment& dst) const {
  auto far = [&](const Segment& s) {
    return s.medium == Medium::kDevice && no_peer_gpus_.count(topo_.node_gpu(s.node)) != 0;
  };
  if (far(src))
    throw NoRouteError("NoRoute: '" + src.id + "' is on a GPU without peer access; staged routes start at GPU " +
                       std::to_string(device_));
  const bool staged = far(dst);
  std::vector<LocalCandidate> keep;
  for (const LocalCandidate& c : r.candidates)
    if (topo_.rail(c.local).host_staged == staged) keep.push_back(c);
  if (keep.empty())
    throw NoRouteError(staged ? "NoRoute: no staged route into '" + dst.id + "' (b200.staged_routes off)"
                              : "NoRoute: no direct rail connects '" + src.id + "' -> '" + dst.id + "'");
  r.candidates = std::move(keep);
}

uint64_t Engine::decompose_count(uint64_t len) const {  // scheduler.cpp:94-106
  uint64_t n = len / opts_.sched.min_slice_size;
  if (n == 0) n = 1;
  if (n > opts_.sched.max_slices_per_transfer) n = opts_.sched.max_slices_per_transfer;
  const uint64_t size = (len + n - 1) / n;
  return (len + size - 1) / size;
}

// ------------------------------------------------------------------ telemetry export

// LatencyHistogram::percentile_us (telemetry.cpp:28-44)
static double percentile_us(const uint32_t* h, double q) {
  uint64_t n = 0;
  for (int b = 0; b < 48; ++b) n += h[b];
  if (n == 0) return 0.0;
  uint64_t rank = static_cast<uint64_t>(std::ceil(q * static_cast<double>(n)));
  if (rank == 0) rank = 1;
  uint64_t seen = 0;
  for (int b = 0; b < 48; ++b) {
    seen += h[b];
    if (seen >= rank) return std::exp2((static_cast<double>(b) + 0.5) / 2.0);
  }
  return std::exp2(48.0 / 2.0);
}

static const char* health_name(uint32_t h) {  // health_state_name (scheduler.cpp)
  return h == kHealthy ? "healthy" : h == kExcluded ? "excluded" : "probing";
}

// TelemetrySnapshot::to_csv (telemetry.cpp:123-158) from the device window cells: the same
// columns, one row per (window, rail) over the windows the ring still holds, health and
// queue carried forward through untouched windows.
std::string Engine::telemetry_csv() {
  std::string out =
      "window_start_ms,rail_id,bytes_ok,bytes_failed,queue_depth_bytes,p50_us,p99_us,health_state,throughput_gbps\n";
  if (!started_) return out;
  CK(cudaSetDevice(device_));
  const size_t nr = topo_.rail_count();
  std::vector<TeleCell> cells(nr * kTeleWindows);
  CK(cudaMemcpyAsync(cells.data(), E_.tele, cells.size() * sizeof(TeleCell), cudaMemcpyDeviceToHost, copy_stream_));
  CK(cudaStreamSynchronize(copy_stream_));
  uint64_t last = 0;
  bool any = false;
  for (const TeleCell& c : cells)
    if (c.window != ~0ull && c.touched) last = std::max(last, c.window), any = true;
  if (!any) return out;
  const uint64_t first = last >= kTeleWindows - 1 ? last - (kTeleWindows - 1) : 0;
  const double window_s = static_cast<double>(opts_.window_ns) * 1e-9;
  char line[320];
  std::vector<uint32_t> health(nr, kHealthy);
  std::vector<int64_t> queue(nr, 0);
  for (uint64_t w = first; w <= last; ++w) {
    for (size_t r = 0; r < nr; ++r) {
      const TeleCell& c = cells[r * kTeleWindows + (w % kTeleWindows)];
      const bool hit = c.window == w && c.touched;
      if (hit) {
        health[r] = c.health_close;
        queue[r] = c.queue_close;
      }
      static const uint32_t kZero[48] = {};
      const uint32_t* h = hit ? c.hist : kZero;
      const uint64_t ok = hit ? c.bytes_ok : 0, failed = hit ? c.bytes_failed : 0;
      std::snprintf(line, sizeof(line), "%llu,%s,%llu,%llu,%lld,%.3f,%.3f,%s,%.6f\n",
                    static_cast<unsigned long long>(w * (opts_.window_ns / 1000000ull)), topo_.rail(r).id.c_str(),
                    static_cast<unsigned long long>(ok), static_cast<unsigned long long>(failed),
                    static_cast<long long>(queue[r]), percentile_us(h, 0.50), percentile_us(h, 0.99),
                    health_name(health[r]), static_cast<double>(ok) * 8.0 / window_s / 1e9);
      out += line;
    }
  }
  return out;
}

// ------------------------------------------------------------------ global load board

size_t board_bytes(uint32_t n_slots) { return sizeof(BoardSlot) * n_slots; }

void Engine::attach_board(void* board, uint32_t n_slots, uint32_t slot, uint64_t period_ns) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!started_) throw EngineError("engine not started");
  if (!board) throw ConfigError("load board: null board");
  if (n_slots == 0 || slot >= n_slots) throw ConfigError("load board: slot out of range");
  if (period_ns == 0) throw ConfigError("load board: publish period must be > 0");
  if (E_.board) throw EngineError("load board: already attached");
  for (const auto& kv : batches_) {
    volatile BatchDev* m = &bmirror_[kv.second.slot];
    if (m->failed_id != kv.second.id && m->done - kv.second.base < kv.second.submitted)
      throw EngineError("load board: attach while no batch is in flight");
  }
  CK(cudaSetDevice(device_));
  void* dp = nullptr;
  if (cudaHostGetDevicePointer(&dp, board, 0) != cudaSuccess) {  // not pinned yet: map it
    cudaGetLastError();
    CK(cudaHostRegister(board, board_bytes(n_slots), cudaHostRegisterMapped | cudaHostRegisterPortable));
    board_registered_ = board;
    CK(cudaHostGetDevicePointer(&dp, board, 0));
  }
  // the running kernel holds the previous EngineDev: let it exit, the next launch has the board
  if (ctl_->state != 0) {
    ctl_->stop = 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    CK(cudaStreamSynchronize(stream_));
    ctl_->stop = 0;
    ctl_->state = 0;
  }
  E_.board = static_cast<BoardSlot*>(dp);
  E_.board_slots = n_slots;
  E_.board_slot = slot;
  E_.board_period = period_ns;
  E_.omega = opts_.diffusion_weight;
}

// ------------------------------------------------------------------ dataflow gates

// logical_bytes != 0 makes a ring gate (the staged route's bounded staging pool,
// reference engine.hpp:56-58 / engine.cpp:465-610): the segment's single buffer is the
// physical ring, intents address a logical window of logical_bytes that wraps onto it, and
// `credits` (one uint32 per granule, zeroed, shared by both ends) carries the consumer's
// drained laps back to the producer.
void Engine::gate_segment(const std::string& seg_id, uint32_t role, void* flags, void* credits,
                          uint64_t logical_bytes) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!started_) throw EngineError("engine not started");
  if (role != kGateConsume && role != kGateProduce) throw ConfigError("gate role must be consume (1) or produce (2)");
  if (!flags) throw ConfigError("gate: flags array is null");
  if (has_ce_) throw ConfigError("dataflow gates are served by SM rails only (the fabric has copy-engine rails)");
  if (E_.n_gates >= uint32_t(kMaxGates)) throw ConfigError("too many gated segments (max 4)");
  auto it = segs_.find(seg_id);
  if (it == segs_.end()) throw EngineError("unknown segment id");
  SegRec& s = it->second;
  if (s.seg.buffers.size() != 1) throw ConfigError("gate: the segment must have exactly one buffer");
  translate(s);
  for (const auto& kv : batches_) {
    volatile BatchDev* m = &bmirror_[kv.second.slot];
    if (m->failed_id != kv.second.id && m->done - kv.second.base < kv.second.submitted)
      throw EngineError("gate: register gates while no batch is in flight");
  }
  // the running kernel holds the previous EngineDev: let it exit, the next launch has the gate
  if (ctl_->state != 0) {
    ctl_->stop = 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    CK(cudaStreamSynchronize(stream_));
    ctl_->stop = 0;
    ctl_->state = 0;
  }
  Buffer& bf = s.seg.buffers.front();
  const uint64_t granules = (bf.length + opts_.chunk_bytes - 1) / opts_.chunk_bytes;
  if (logical_bytes) {
    if (!credits) throw ConfigError("ring gate: credits array is null");
    if (bf.offset != 0 || bf.length % opts_.chunk_bytes)
      throw ConfigError("ring gate: the ring buffer must start at offset 0 and be a multiple of b200.chunk_bytes");
    if (logical_bytes < bf.length) throw ConfigError("ring gate: logical_bytes is smaller than the ring");
    if (logical_bytes / bf.length >= (1ull << 32)) throw ConfigError("ring gate: too many laps");
    if (E_.n_relays) throw ConfigError("ring gates are served by direct SM rails only (the fabric has relay rails)");
  }
  if (logical_bytes >= (1ull << 56)) throw ConfigError("ring gate: logical_bytes must stay below 2^56");
  GateDev g{};
  g.lo = bf.dev_addr;
  if (logical_bytes) {
    // the logical window gets a tagged virtual base of its own (bit 63 + the gate index):
    // it can never alias a real allocation, and only this engine's workers, which wrap it
    // onto the ring before touching memory, ever see it
    g.phys = bf.dev_addr;
    g.lo = (1ull << 63) | (uint64_t(E_.n_gates + 1) << 56);
  }
  g.hi = g.lo + (logical_bytes ? logical_bytes : bf.length);
  g.flags = static_cast<uint32_t*>(flags);
  g.role = role;
  g.ring = logical_bytes ? bf.length : 0;
  g.ngran = static_cast<uint32_t>(granules);
  {  // this engine's own per-granule counters (consumed or produced), zeroed
    CK(cudaSetDevice(device_));
    void* p = nullptr;
    CK(cudaMalloc(&p, granules * sizeof(uint32_t)));
    CK(cudaMemset(p, 0, granules * sizeof(uint32_t)));
    dev_allocs_.push_back(p);
    if (role == kGateConsume) g.consumed = static_cast<uint32_t*>(p);
    else g.produced = static_cast<uint32_t*>(p);
  }
  // flags may be mapped pinned host memory (a staged route through the host): use the
  // device alias of such a pointer
  {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, flags) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      g.flags = static_cast<uint32_t*>(pa.devicePointer);
    cudaGetLastError();
  }
  if (logical_bytes) {
    g.credits = static_cast<uint32_t*>(credits);
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, credits) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      g.credits = static_cast<uint32_t*>(pa.devicePointer);
    cudaGetLastError();
    s.ring = bf.length;
    bf.length = logical_bytes;  // intents address the logical window; workers wrap onto the ring
    bf.dev_addr = g.lo;
  }
  E_.gates[E_.n_gates++] = g;
  s.gated = true;
}

// ------------------------------------------------------------------ batches

Engine::BatchRec& Engine::batch_ref(uint64_t id) {
  auto it = batches_.find(id);
  if (it == batches_.end()) throw EngineError("unknown batch");
  return it->second;
}

uint64_t Engine::allocate_batch() {
  std::lock_guard<std::mutex> lk(mu_);
  return allocate_batch_locked();
}

uint64_t Engine::allocate_batch_locked() {
  if (!started_) throw EngineError("engine not started");
  // the slot of the batch freed last (if it completed) first: its delivered counter is
  // still in the scheduler's counter cache, so the batch's first completion does not wait
  // on an HBM read of a cold slot; otherwise round robin
  const int64_t hint = last_freed_;
  last_freed_ = -1;
  for (uint32_t k = 0; k <= opts_.batch_slots; ++k) {
    const uint32_t slot = (hint >= 0 && k == 0) ? static_cast<uint32_t>(hint) : (next_slot_ + k) % opts_.batch_slots;
    if (slot_busy_[slot]) continue;
    slot_busy_[slot] = 1;
    if (!(hint >= 0 && k == 0)) next_slot_ = slot + 1;
    BatchRec b;
    b.id = next_batch_++;
    b.slot = slot;
    b.base = reinterpret_cast<volatile BatchDev*>(bmirror_)[slot].done;
    batches_.emplace(b.id, b);
    return b.id;
  }
  throw EngineError("no free batch slot (free completed batches)");
}

static spray_batch_status_t status_of(uint64_t submitted, uint64_t done, bool failed) {
  spray_batch_status_t st{};
  st.remaining = submitted > done ? submitted - done : 0;
  if (failed) {
    st.state = SPRAY_BATCH_FAILED;
    std::snprintf(st.failure_reason, sizeof(st.failure_reason), "AllRoutesExhausted");
  } else {
    st.state = st.remaining > 0 ? SPRAY_BATCH_IN_FLIGHT : SPRAY_BATCH_COMPLETE;
  }
  return st;
}

spray_batch_status_t Engine::batch_status(uint64_t batch) {
  std::lock_guard<std::mutex> lk(mu_);
  BatchRec& b = batch_ref(batch);
  volatile BatchDev* m = &bmirror_[b.slot];
  const uint64_t failed_id = m->failed_id;
  const uint64_t done = m->done - b.base;
  return status_of(b.submitted, done, failed_id == b.id);
}

spray_batch_status_t Engine::await_batch(uint64_t batch, uint64_t limit_ns) {
  const auto t0 = std::chrono::steady_clock::now();
  uint32_t spins = 0;
  for (;;) {
    spray_batch_status_t st = batch_status(batch);
    if (st.state != SPRAY_BATCH_IN_FLIGHT) return st;
    const uint64_t el = static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
    if (el > limit_ns) return st;
    if (++spins < 2000) _mm_pause();
    else std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

void Engine::free_batch(uint64_t batch) {
  std::lock_guard<std::mutex> lk(mu_);
  free_batch_locked(batch);
}

void Engine::free_batch_locked(uint64_t batch) {
  BatchRec& b = batch_ref(batch);
  volatile BatchDev* m = &bmirror_[b.slot];
  const bool failed = m->failed_id == b.id;
  const uint64_t done = m->done - b.base;
  if (!failed && b.submitted > 0 && done < b.submitted) throw EngineError("cannot free an in-flight batch");
  slot_busy_[b.slot] = 0;
  if (!failed) last_freed_ = b.slot;  // a failed batch's slot may still see late completions
  batches_.erase(batch);
}

// ------------------------------------------------------------------ submit

Engine::SegRec& Engine::seg_lookup(const char* name, const char*& cname, SegRec*& crec) {
  if (!name) name = "";
  if (crec && std::strcmp(cname, name) == 0) return *crec;
  auto it = segs_.find(name);
  if (it == segs_.end()) throw EngineError("unknown segment id");
  crec = &it->second;
  cname = it->second.seg.id.c_str();
  return it->second;
}

Intent Engine::make_intent(uint64_t batch, const spray_transfer_request& req, uint64_t* n_slices, LookupCache* lc) {
  if (!started_) throw EngineError("engine not started");
  LookupCache local;
  LookupCache& c = lc ? *lc : local;
  if (!c.batch || c.batch_id != batch) {
    c.batch = &batch_ref(batch);
    c.batch_id = batch;
    // batch state is checked once per submit call: its own earlier intents may already
    // have completed on the device while the host builds the rest
    BatchRec& b = *c.batch;
    volatile BatchDev* m = &bmirror_[b.slot];
    if (m->failed_id == b.id) throw EngineError("batch already failed");
    if (b.submitted > 0 && m->done - b.base >= b.submitted) throw EngineError("batch already complete");
  }
  BatchRec& b = *c.batch;
  SegRec& ss = seg_lookup(req.src_segment, c.src_name, c.src);
  SegRec& ds = seg_lookup(req.dst_segment, c.dst_name, c.dst);
  if (req.length == 0) throw InvalidRangeError("zero-length transfer");
  if (!ss.seg.covering(req.src_offset, req.length))
    throw InvalidRangeError("source range not covered by one registered buffer");
  if (!ds.seg.covering(req.dst_offset, req.length))
    throw InvalidRangeError("destination range not covered by one registered buffer");
  const Direction dir = req.direction == SPRAY_READ ? Direction::kRead : Direction::kWrite;
  if ((ss.ring && req.length > ss.ring) || (ds.ring && req.length > ds.ring))
    throw InvalidRangeError("ring-gated segment: a transfer may not exceed the ring");
  if (ss.gated || ds.gated) {  // gated segments: every chunk is exactly one granule
    const uint64_t cb = opts_.chunk_bytes;
    uint64_t nsl = req.length / opts_.sched.min_slice_size;
    if (nsl == 0) nsl = 1;
    if (nsl > opts_.sched.max_slices_per_transfer) nsl = opts_.sched.max_slices_per_transfer;
    const uint64_t size = (req.length + nsl - 1) / nsl;
    if (req.src_offset % cb || req.dst_offset % cb || (nsl > 1 && size % cb))
      throw InvalidRangeError("gated segment: offsets and slice sizes must be multiples of b200.chunk_bytes");
  }
  if (c.set_src != &ss || c.set_dst != &ds || c.set_dir != static_cast<int>(dir)) {
    c.set = set_for(ss.seg, ds.seg, dir);  // throws NoRouteError
    c.set_src = &ss;
    c.set_dst = &ds;
    c.set_dir = static_cast<int>(dir);
  }
  translate(ss);
  translate(ds);
  const Buffer* sb = ss.seg.covering(req.src_offset, req.length);
  const Buffer* db = ds.seg.covering(req.dst_offset, req.length);
  Intent in{};
  in.batch_id = b.id;
  in.src = sb->dev_addr + (req.src_offset - sb->offset);
  in.dst = db->dev_addr + (req.dst_offset - db->offset);
  in.len = req.length;
  in.hash_offset = req.src_offset;
  in.transfer_id = next_transfer_++;
  in.set_id = c.set;
  in.batch_slot = b.slot;
  in.flags = 0;
  *n_slices = decompose_count(req.length);
  return in;
}

void Engine::publish(const Intent* in, size_t n) {
  const uint64_t cap = opts_.sub_capacity;
  for (size_t i = 0; i < n; ++i) {
    while (sub_tail_ - ctl_->sub_head >= cap) {
      // ring full: make what is there visible and let the device drain it
      std::atomic_thread_fence(std::memory_order_release);
      ctl_->sub_tail = sub_tail_;
      ensure_running();
      _mm_pause();
    }
    ring_[sub_tail_ % cap] = in[i];
    ++sub_tail_;
  }
  std::atomic_thread_fence(std::memory_order_release);
  ctl_->sub_tail = sub_tail_;
  ensure_running();
}

uint64_t Engine::submit_transfer(uint64_t batch, const spray_transfer_request& req) {
  std::lock_guard<std::mutex> lk(mu_);
  uint64_t n = 0;
  Intent in = make_intent(batch, req, &n);
  batch_ref(batch).submitted += n;
  publish(&in, 1);
  return in.transfer_id;
}

// Intents are published in groups as they are built, so the device starts on the head of
// a large batch while the host is still translating its tail (order is unchanged).
size_t Engine::submit_transfers(uint64_t batch, const spray_transfer_request* reqs, size_t n, uint64_t* ids) {
  std::lock_guard<std::mutex> lk(mu_);
  if (n >= kStageMin) return submit_staged_locked(batch, reqs, n, ids);
  constexpr size_t kGroup = 256;
  Intent v[kGroup];
  size_t nv = 0, done = 0;
  LookupCache lc;
  try {
    for (; done < n; ++done) {
      uint64_t k = 0;
      v[nv] = make_intent(batch, reqs[done], &k, &lc);
      lc.batch->submitted += k;
      if (ids) ids[done] = v[nv].transfer_id;
      if (++nv == kGroup) {
        publish(v, nv);
        nv = 0;
      }
    }
  } catch (...) {
    if (nv) publish(v, nv);
    throw;
  }
  if (nv) publish(v, nv);
  return done;
}

// A large submission goes to the device as bulk intent arrays in HBM (one copy-engine copy
// and one ring entry per kStageCap intents, so the device starts on the first piece while
// the host builds the next) instead of through the mapped ring: the
// HOSTRX warp's reads of host memory queue behind every write the engine has posted to the
// PCIe root, so under a host-bound batch the ring is fetched at the pace of that backlog.
// kStageAreas device areas rotate; an area is refilled only after INGRESS has finished the bulk
// array it last held (the device's bulk_done counter). Order and accounting are those of
// the ring path.
size_t Engine::submit_staged_locked(uint64_t batch, const spray_transfer_request* reqs, size_t n, uint64_t* ids) {
  CK(cudaSetDevice(device_));
  if (!stage_host_) {
    void* h = nullptr;
    CK(cudaHostAlloc(&h, sizeof(Intent) * kStageCap * kStageAreas, cudaHostAllocPortable));
    stage_host_ = static_cast<Intent*>(h);
    for (Intent*& d : stage_dev_) {
      void* p = nullptr;
      CK(cudaMalloc(&p, sizeof(Intent) * kStageCap));
      dev_allocs_.push_back(p);
      d = static_cast<Intent*>(p);
    }
  }
  LookupCache lc;
  size_t done = 0;
  for (uint32_t piece = 0; done < n; ++piece) {
    const size_t k = std::min(kStageCap, n - done);
    const uint32_t a = static_cast<uint32_t>(bulk_pub_ % kStageAreas);
    Intent* hs = stage_host_ + size_t(a) * kStageCap;
    const auto t0 = std::chrono::steady_clock::now();
    while (stage_use_[a] && ctl_->bulk_done < stage_use_[a]) {  // INGRESS still reads it
      ensure_running();
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
        throw EngineError("staged submit: bulk array not consumed within 60 s");
      _mm_pause();
    }
    size_t built = 0;
    try {
      for (; built < k; ++built) {
        uint64_t sl = 0;
        hs[built] = make_intent(batch, reqs[done + built], &sl, &lc);
        lc.batch->submitted += sl;
        if (ids) ids[done + built] = hs[built].transfer_id;
      }
    } catch (...) {
      // what was built so far still goes out, as the ring path would have published it
      if (built) {
        CK(cudaMemcpyAsync(stage_dev_[a], hs, sizeof(Intent) * built, cudaMemcpyHostToDevice, copy_stream_));
        CK(cudaStreamSynchronize(copy_stream_));
        Intent bulk{};
        bulk.batch_id = lc.batch->id;
        bulk.src = reinterpret_cast<uint64_t>(stage_dev_[a]);
        bulk.len = built;
        bulk.batch_slot = lc.batch->slot;
        bulk.flags = kIntentBulk;
        stage_use_[a] = ++bulk_pub_;
        publish(&bulk, 1);
      }
      throw;
    }
    CK(cudaMemcpyAsync(stage_dev_[a], hs, sizeof(Intent) * k, cudaMemcpyHostToDevice, copy_stream_));
    CK(cudaStreamSynchronize(copy_stream_));
    Intent bulk{};
    bulk.batch_id = lc.batch->id;
    bulk.src = reinterpret_cast<uint64_t>(stage_dev_[a]);
    bulk.len = k;
    bulk.batch_slot = lc.batch->slot;
    bulk.flags = kIntentBulk;
    stage_use_[a] = ++bulk_pub_;
    publish(&bulk, 1);
    done += k;
  }
  return done;
}

// Plans and validates n requests exactly like submit_transfer (through a scratch batch), under
// the engine lock, and returns the intents for a device-resident submission.
std::vector<Intent> Engine::prepare(const spray_transfer_request* reqs, size_t n, uint64_t* slices) {
  std::lock_guard<std::mutex> lk(mu_);
  const uint64_t b = allocate_batch_locked();
  std::vector<Intent> v(n);
  uint64_t total = 0;
  try {
    LookupCache lc;
    for (size_t i = 0; i < n; ++i) {
      uint64_t k = 0;
      v[i] = make_intent(b, reqs[i], &k, &lc);
      total += k;
    }
  } catch (...) {
    free_batch_locked(b);
    throw;
  }
  free_batch_locked(b);
  *slices = total;
  return v;
}

void Engine::submit_device_intents(uint64_t batch, const void* dev_intents, uint64_t n, uint64_t total_slices) {
  std::lock_guard<std::mutex> lk(mu_);
  BatchRec& b = batch_ref(batch);
  b.submitted += total_slices;
  Intent bulk{};
  bulk.batch_id = b.id;
  bulk.src = reinterpret_cast<uint64_t>(dev_intents);
  bulk.len = n;
  bulk.batch_slot = b.slot;
  bulk.flags = kIntentBulk;
  ++bulk_pub_;
  publish(&bulk, 1);
}

// Prepared (device-resident) intents, timed: the caller guarantees no launch is resident
// and the stream is idle. The bulk descriptor is published first; then the stream is held
// on a mapped flag while the bracket (event, launch, event) is enqueued, and released, so
// the events time the engine kernel and not the host's launch latency.
float Engine::run_device_intents_timed(uint64_t batch, const void* dev_intents, uint64_t n, uint64_t total_slices) {
  std::lock_guard<std::mutex> lk(mu_);
  if (ctl_->state != 0) throw EngineError("timed run: a launch is still resident");
  BatchRec& b = batch_ref(batch);
  b.submitted += total_slices;
  Intent bulk{};
  bulk.batch_id = b.id;
  bulk.src = reinterpret_cast<uint64_t>(dev_intents);
  bulk.len = n;
  bulk.batch_slot = b.slot;
  bulk.flags = kIntentBulk;
  ++bulk_pub_;
  ring_[sub_tail_ % opts_.sub_capacity] = bulk;
  ++sub_tail_;
  std::atomic_thread_fence(std::memory_order_release);
  ctl_->sub_tail = sub_tail_;
  CK(cudaSetDevice(device_));
  if (!hold_) {
    void* h = nullptr;
    void* d = nullptr;
    CK(cudaHostAlloc(&h, sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer(&d, h, 0));
    hold_ = static_cast<volatile uint32_t*>(h);
    hold_dev_ = static_cast<uint32_t*>(d);
  }
  *hold_ = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  cudaEvent_t a, z;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&z));
  CK(spray_launch::launch_hold(hold_dev_, stream_));
  CK(cudaEventRecord(a, stream_));
  launch();
  CK(cudaEventRecord(z, stream_));
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *hold_ = 1;
  CK(cudaEventSynchronize(z));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, a, z));
  cudaEventDestroy(a);
  cudaEventDestroy(z);
  return ms;
}

// ------------------------------------------------------------------ introspection

void Engine::rail_stats(uint32_t rail, spray_rail_stats* out) {
  if (rail >= rail_count()) throw EngineError("bad rail index");
  std::memset(out, 0, sizeof(*out));
  if (!rmirror_) return;
  // the scheduler writes its rail states to HBM whenever it goes quiet (and at exit), so a
  // caller that saw a batch complete reads stats that include its completions
  RailState s;
  CK(cudaSetDevice(device_));
  CK(cudaMemcpyAsync(&s, &E_.rail_state[rail], sizeof(s), cudaMemcpyDeviceToHost, copy_stream_));
  CK(cudaStreamSynchronize(copy_stream_));
  out->bytes_posted = s.bytes_posted;
  out->bytes_ok = s.bytes_ok;
  out->bytes_failed = s.bytes_failed;
  out->queue_depth = s.queued;
  out->beta0 = s.beta0;
  out->beta1 = s.beta1;
  out->health = static_cast<int32_t>(s.health);
  std::memcpy(out->latency_hist, s.hist, sizeof(s.hist));
}

void Engine::counters(uint64_t* d, uint64_t* t, uint64_t* f) {
  if (!ctl_) {
    *d = *t = *f = 0;
    return;
  }
  *d = ctl_->bytes_dispatched;
  *t = ctl_->bytes_terminated;
  *f = ctl_->batches_failed;
}

// One FaultEntry (backend.hpp:79-86) applied to the live fabric; FaultSchedule::validate's
// rules: a non-empty interval, a positive degrade factor, a non-negative jitter bound. An
// entry replaces the rail's previous entry of the same effect.
void Engine::inject_fault(const std::string& rail, int effect, uint64_t start, uint64_t end, double factor,
                          double jitter_us) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!started_) throw EngineError("engine not started");
  auto r = topo_.rail_index(rail);
  if (!r) throw ConfigError("fault schedule references unknown rail '" + rail + "'");
  if (end <= start) throw ConfigError("fault interval must be non-empty");
  if (effect < 0 || effect > 3) throw ConfigError("unknown fault effect");
  if (effect == kFxDegrade && !(factor > 0.0 && factor <= 1.0)) throw ConfigError("degrade factor must be in (0, 1]");
  if (effect == kFxJitter && !(jitter_us >= 0.0)) throw ConfigError("jitter_us must be >= 0");
  volatile FaultDev* f = &faults_[*r];
  const uint32_t bit = 1u << effect;
  f->active = f->active & ~bit;  // retract the effect while its words change
  std::atomic_thread_fence(std::memory_order_seq_cst);
  f->start[effect] = start;
  f->end[effect] = end;
  if (effect == kFxDegrade) f->factor = factor;
  if (effect == kFxJitter) f->jitter_us = jitter_us;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  f->active = f->active | bit;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  ctl_->fault_epoch = ctl_->fault_epoch + 1;
  ctl_->heal_fault_start = 0;
  ctl_->heal_first_ok = 0;
}

void Engine::clear_faults() {
  std::lock_guard<std::mutex> lk(mu_);
  if (!faults_) return;
  for (int i = 0; i < kMaxRails; ++i) faults_[i].active = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  ctl_->fault_epoch = ctl_->fault_epoch + 1;
}

uint64_t Engine::now_ns() { return ctl_ ? ctl_->device_now : 0; }

void Engine::debug_words(uint64_t* out, size_t n) {
  std::vector<uint64_t> v;
  if (ctl_) {
    v = {sub_tail_, ctl_->sub_tail, ctl_->sub_head, ctl_->state, ctl_->device_now, ctl_->bytes_dispatched,
         ctl_->bytes_terminated, ctl_->failed_attempts, ctl_->retried_ok, ctl_->trace_n,
         static_cast<uint64_t>(cudaStreamQuery(stream_)), ctl_->prof_loops, ctl_->prof_comp_ns,
         ctl_->prof_sub_ns, ctl_->prof_ctl_ns, ctl_->prof_n_comp, ctl_->prof_n_dec};
    for (int q = 0; q < 16; ++q) v.push_back(static_cast<uint64_t>(ctl_->prof_x[q]));
    v.push_back(static_cast<uint64_t>(ctl_->ce_tail[0]));
    v.push_back(static_cast<uint64_t>(ctl_->ce_head[0]));
    v.push_back(static_cast<uint64_t>(ctl_->xc_tail));
    v.push_back(static_cast<uint64_t>(ctl_->xc_head));
    for (int q = 0; q < 8; ++q) v.push_back(static_cast<uint64_t>(ctl_->tl[q]));  // words 37..44
    // words 45..60: device diagnostic words (Control::dbg), 61: this launch's generation
    for (int q = 0; q < 16; ++q) v.push_back(static_cast<uint64_t>(ctl_->dbg[q]));
    v.push_back(E_.launch_gen);
    for (int q = 0; q < 8; ++q) v.push_back(static_cast<uint64_t>(ctl_->lat[q]));  // words 62..69
    for (int q = 0; q < 8; ++q) v.push_back(static_cast<uint64_t>(ctl_->lat_w[q]));  // words 70..77
    for (int q = 0; q < 8; ++q) v.push_back(static_cast<uint64_t>(ctl_->prof_y[q]));  // words 78..85
    for (int q = 0; q < 8; ++q) v.push_back(static_cast<uint64_t>(ctl_->prof_z[q]));  // words 86..93
    for (int q = 0; q < 8; ++q) v.push_back(static_cast<uint64_t>(ctl_->lat_s[q]));  // words 94..101
  }
  for (size_t i = 0; i < n; ++i) out[i] = i < v.size() ? v[i] : 0;
}

void Engine::heal_stats(uint64_t* fs, uint64_t* ok, uint64_t* fa, uint64_t* ro) {
  *fs = ctl_ ? ctl_->heal_fault_start : 0;
  *ok = ctl_ ? ctl_->heal_first_ok : 0;
  *fa = ctl_ ? ctl_->failed_attempts : 0;
  *ro = ctl_ ? ctl_->retried_ok : 0;
}

// ------------------------------------------------------------------ trace

void Engine::trace_enable(size_t cap) {
  CK(cudaSetDevice(device_));
  std::lock_guard<std::mutex> lk(mu_);
  if (!started_) throw EngineError("engine not started");
  ctl_->stop = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  CK(cudaStreamSynchronize(stream_));
  ctl_->stop = 0;
  ctl_->state = 0;
  void* ev = nullptr;
  void* dc = nullptr;
  CK(cudaMalloc(&ev, cap * sizeof(spray_trace_event)));
  CK(cudaMalloc(&dc, cap * sizeof(spray_decision)));
  dev_allocs_.push_back(ev);
  dev_allocs_.push_back(dc);
  E_.trace_ev = static_cast<uint8_t*>(ev);
  E_.trace_dec = static_cast<uint8_t*>(dc);
  E_.trace_cap = cap;
  trace_cap_ = cap;
  ctl_->trace_n = 0;
  ctl_->trace_dn = 0;
  ctl_->trace_on = 1;
}

void Engine::trace_fetch(spray_trace_event* ev, size_t cap, size_t* n, spray_decision* dec, size_t dcap, size_t* nd) {
  CK(cudaSetDevice(device_));
  std::lock_guard<std::mutex> lk(mu_);
  if (!started_ || !trace_cap_) throw EngineError("tracing not enabled");
  // quiesce the kernel so the trace is complete and stable
  ctl_->stop = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  CK(cudaStreamSynchronize(stream_));
  ctl_->stop = 0;
  ctl_->state = 0;
  const uint64_t tn = std::min<uint64_t>(uint64_t(ctl_->trace_n), uint64_t(trace_cap_));
  const uint64_t tdn = std::min<uint64_t>(uint64_t(ctl_->trace_dn), uint64_t(trace_cap_));
  *n = ctl_->trace_n;
  *nd = ctl_->trace_dn;
  if (ev) CK(cudaMemcpy(ev, E_.trace_ev, std::min<uint64_t>(tn, cap) * sizeof(spray_trace_event), cudaMemcpyDeviceToHost));
  if (dec) CK(cudaMemcpy(dec, E_.trace_dec, std::min<uint64_t>(tdn, dcap) * sizeof(spray_decision), cudaMemcpyDeviceToHost));
}

std::vector<int32_t> Engine::trace_candidates() {
  std::lock_guard<std::mutex> lk(mu_);
  std::vector<int32_t> out{static_cast<int32_t>(sets_.size())};
  for (const auto& s : sets_) append_stream(out, s);
  return out;
}

// ------------------------------------------------------------------ CE proxy
// Copy-engine rails: the device publishes CeOrders into a mapped ring; this thread
// issues one cudaMemcpyAsync per order on the rail's side stream, and posts the
// completion into the mapped external-completion ring the device scheduler drains.
// CE rails: the device publishes copy orders per CE stream; one thread per stream issues
// them with cudaMemcpyAsync in order, records one event per group of orders taken in a
// pass, and completes a group when its event fires (a stream's copies finish in issue
// order, so only the oldest group is ever queried). Completions go to the shared
// completion ring: a slot is reserved atomically, and its stamp (written last) publishes
// it to the device (HOSTRX reads the stamped prefix).
void Engine::ce_proxy_loop(int k) {
  cudaSetDevice(device_);
  struct Group {
    cudaEvent_t ev;
    std::vector<CeOrder> orders;
  };
  std::deque<Group> fifo;
  std::vector<cudaEvent_t> pool;
  uint64_t head = ctl_->ce_head[k];
  // fault words of a rail the proxy honours (host view of the same FaultEntry words)
  auto fault_at = [&](uint32_t rail, uint32_t effect, uint64_t now) {
    if (rail >= kMaxRails) return false;
    const volatile FaultDev* f = &faults_[rail];
    return ((f->active >> effect) & 1u) && f->start[effect] <= now && now < f->end[effect];
  };
  auto post = [&](const CeOrder& o, uint32_t status) {
    // DROP_COMPLETION (sim_backend.cpp:118-121, 139): the bytes landed, the event is lost; the
    // device's deadline scan times the attempt out
    const uint64_t now = ctl_->device_now;
    if (status == kStOk && (fault_at(o.rail, kFxDrop, now) || fault_at(o.remote, kFxDrop, now))) return;
    const uint64_t pos = xc_reserve_.fetch_add(1);
    while (pos - ctl_->xc_head >= E_.xc_cap) _mm_pause();
    volatile Completion* c = &xc_ring_[pos % E_.xc_cap];
    c->slice = o.slice;
    c->gen = o.gen;
    c->status = status;
    c->rail = o.rail;
    std::atomic_thread_fence(std::memory_order_release);
    c->stamp = static_cast<uint32_t>(pos + 1);
  };
  // Orders are issued as strided runs: a host call costs ~4 us whatever its size
  // (tools/ce_issue_peak.cu: 64 KiB per call caps a copy engine at 13 GB/s, 256 KiB at
  // 64 GB/s), so consecutive orders of equal length whose source and destination advance
  // by constant pitches go out as ONE copy: 1D when both pitches equal the length (a
  // contiguous run), else one cudaMemcpy2DAsync (rows = slices; the copy engines move
  // pitch-linear rows natively). Completions stay per order, reported when the group's
  // event fires.
  constexpr int kMaxGroup = 1024;  // orders taken per pass (one completion event per pass)
  struct Run {
    uint64_t src = 0, dst = 0, len = 0, spitch = 0, dpitch = 0, rows = 0;
  } run;
  auto flush = [&] {
    if (!run.rows) return;
    void* d = reinterpret_cast<void*>(run.dst);
    const void* sp = reinterpret_cast<const void*>(run.src);
    if (run.rows == 1 || (run.spitch == run.len && run.dpitch == run.len))
      cudaMemcpyAsync(d, sp, run.len * run.rows, cudaMemcpyDefault, ce_streams_[k]);
    else
      cudaMemcpy2DAsync(d, run.dpitch, sp, run.spitch, run.len, run.rows, cudaMemcpyDefault, ce_streams_[k]);
    run.rows = 0;
  };
  auto extend = [&](const CeOrder& o) {
    constexpr uint64_t kMaxPitch = 1ull << 30;  // well inside cudaDevAttrMaxPitch
    if (run.rows && o.len == run.len) {
      if (run.rows == 1) {
        const uint64_t sp = o.src - run.src, dp = o.dst - run.dst;  // wraps when negative: rejected below
        if (o.src > run.src && o.dst > run.dst && sp >= o.len && dp >= o.len && sp <= kMaxPitch && dp <= kMaxPitch) {
          run.spitch = sp, run.dpitch = dp, run.rows = 2;
          return;
        }
      } else if (o.src == run.src + run.rows * run.spitch && o.dst == run.dst + run.rows * run.dpitch) {
        ++run.rows;
        return;
      }
    }
    flush();
    run.src = o.src, run.dst = o.dst, run.len = o.len, run.rows = 1;
  };
  while (ce_run_.load()) {
    bool any = false;
    Group g;
    g.ev = nullptr;
    while (head < ctl_->ce_tail[k] && g.orders.size() < size_t(kMaxGroup)) {
      volatile CeOrder* vo = &ce_ring_[k * E_.ce_cap + (head % E_.ce_cap)];
      if (vo->stamp != head + 1) break;
      CeOrder o;
      o.src = vo->src; o.dst = vo->dst; o.len = vo->len; o.slice = vo->slice; o.gen = vo->gen;
      o.rail = vo->rail; o.remote = vo->remote; o.stamp = vo->stamp;
      ++head;
      any = true;
      const uint64_t now = ctl_->device_now;
      if (fault_at(o.rail, kFxDown, now) || fault_at(o.remote, kFxDown, now)) {
        post(o, kStFailed);
        continue;
      }
      extend(o);
      g.orders.push_back(o);
    }
    flush();
    ctl_->ce_head[k] = head;
    if (!g.orders.empty()) {
      if (pool.empty()) {
        cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming);
      } else {
        g.ev = pool.back();
        pool.pop_back();
      }
      cudaEventRecord(g.ev, ce_streams_[k]);
      fifo.push_back(std::move(g));
    }
    while (!fifo.empty()) {
      Group& h = fifo.front();
      const cudaError_t q = cudaEventQuery(h.ev);
      if (q == cudaErrorNotReady) break;
      for (const CeOrder& o : h.orders) post(o, q == cudaSuccess ? kStOk : kStFailed);
      pool.push_back(h.ev);
      fifo.pop_front();
      any = true;
    }
    if (!any) std::this_thread::sleep_for(std::chrono::microseconds(5));
  }
  for (auto& h : fifo) cudaEventSynchronize(h.ev), pool.push_back(h.ev);
  for (auto e : pool) cudaEventDestroy(e);
}

}  // namespace spray
