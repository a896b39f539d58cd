// capi.cpp — the extern "C" boundary (include/spray_b200.h). C++ exceptions never
// cross it: each entry maps the reference exception class to its SPRAY_E* code and
// keeps the message in a thread-local buffer (spray_last_error).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <thread>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/spray_b200.h"
#include "dev_types.cuh"
#include "engine.hpp"

namespace spray_launch {
size_t engine_smem_bytes();
cudaError_t launch_engine(const spray_dev::EngineDev& E, int grid, int block, cudaStream_t st);
cudaError_t launch_replay(const spray_dev::EngineDev& E, const spray_trace_event* ev, uint64_t n, spray_decision* dec,
                          uint64_t dcap, unsigned long long* out, spray_dev::RailState* final_state, cudaStream_t st);
cudaError_t launch_fill(void* p, uint64_t n, uint64_t seed, cudaStream_t st);
cudaError_t launch_checksum(const void* p, uint64_t n, unsigned long long* out, cudaStream_t st);
cudaError_t launch_group_copy(const void* descs, uint32_t n, uint64_t total_chunks, uint64_t chunk, int grid,
                              cudaStream_t st);
}  // namespace spray_launch

using namespace spray;
using spray_dev::Intent;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    g_err.clear();
    f();
    return SPRAY_OK;
  } catch (const NoRouteError& e) {
    g_err = e.what();
    return SPRAY_ENOROUTE;
  } catch (const InvalidRangeError& e) {
    g_err = e.what();
    return SPRAY_EINVALID_RANGE;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return SPRAY_ECONFIG;
  } catch (const EngineError& e) {
    g_err = e.what();
    return SPRAY_EENGINE;
  } catch (const CudaError& e) {
    g_err = e.what();
    return SPRAY_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SPRAY_EENGINE;
  }
}

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)
}  // namespace

struct spray_engine {
  Engine* eng;
};

struct spray_prepared {
  spray_engine* owner = nullptr;
  void* dev = nullptr;
  uint64_t n = 0;
  uint64_t slices = 0;
};

extern "C" {

const char* spray_last_error(void) { return g_err.c_str(); }
uint32_t spray_abi_version(void) { return SPRAY_ABI_VERSION; }
void spray_sched_config_default(spray_sched_config* c) { default_sched_config(c); }
void spray_resilience_config_default(spray_resilience_config* c) { default_resilience_config(c); }

// ------------------------------------------------------------------ engine
int spray_engine_create(const char* config_json, const char* topology_json, int device, spray_engine** out) {
  return guard([&] {
    if (!topology_json) throw ConfigError("engine: no topology given");
    EngineOptions eo = engine_options_from_json(config_json ? config_json : "");
    *out = new spray_engine{new Engine(std::move(eo), topology_json, device)};
  });
}

void spray_engine_destroy(spray_engine* e) {
  if (!e) return;
  delete e->eng;
  delete e;
}

int spray_engine_start(spray_engine* e) { return guard([&] { e->eng->start(); }); }
int spray_engine_stop(spray_engine* e) { return guard([&] { e->eng->stop(); }); }
int spray_register_segment(spray_engine* e, const spray_segment_desc* d) {
  return guard([&] { e->eng->register_segment(*d); });
}
int spray_allocate_batch(spray_engine* e, uint64_t* out) { return guard([&] { *out = e->eng->allocate_batch(); }); }
int spray_submit_transfer(spray_engine* e, uint64_t batch, const spray_transfer_request* req, uint64_t* id) {
  return guard([&] {
    const uint64_t t = e->eng->submit_transfer(batch, *req);
    if (id) *id = t;
  });
}
int spray_submit_transfers(spray_engine* e, uint64_t batch, const spray_transfer_request* reqs, size_t n,
                           uint64_t* ids, size_t* n_done) {
  if (n_done) *n_done = 0;
  return guard([&] {
    const size_t k = e->eng->submit_transfers(batch, reqs, n, ids);
    if (n_done) *n_done = k;
  });
}
int spray_batch_status(spray_engine* e, uint64_t batch, spray_batch_status_t* out) {
  return guard([&] { *out = e->eng->batch_status(batch); });
}
int spray_await_batch(spray_engine* e, uint64_t batch, uint64_t limit_ns, spray_batch_status_t* out) {
  return guard([&] { *out = e->eng->await_batch(batch, limit_ns); });
}
int spray_free_batch(spray_engine* e, uint64_t batch) { return guard([&] { e->eng->free_batch(batch); }); }

// Batch latency as a C++ application sees it (bench.cpp:156-157, 213-215: submit -> batch
// terminal): n_batches rounds of allocate_batch, submit_transfers(per_batch requests, cycling
// through reqs), await_batch, free_batch, one batch in flight, through the same public calls
// as above. lat_ns[i] = steady-clock nanoseconds of round i.
int spray_batch_latency(spray_engine* e, const spray_transfer_request* reqs, size_t n_reqs, size_t per_batch,
                        size_t n_batches, uint64_t* lat_ns) {
  return guard([&] {
    if (per_batch == 0 || per_batch > n_reqs) throw ConfigError("batch_latency: per_batch must be in [1, n_reqs]");
    const size_t groups = n_reqs / per_batch;
    for (size_t i = 0; i < n_batches; ++i) {
      const spray_transfer_request* g = reqs + (i % groups) * per_batch;
      const auto t0 = std::chrono::steady_clock::now();
      const uint64_t b = e->eng->allocate_batch();
      e->eng->submit_transfers(b, g, per_batch, nullptr);
      const spray_batch_status_t st = e->eng->await_batch(b, 60'000'000'000ull);
      if (st.state != SPRAY_BATCH_COMPLETE) throw EngineError("batch_latency: batch did not complete");
      e->eng->free_batch(b);
      lat_ns[i] = static_cast<uint64_t>(
          std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
    }
  });
}

int spray_rail_count(spray_engine* e, uint32_t* n) { return guard([&] { *n = e->eng->rail_count(); }); }
int spray_rail_id(spray_engine* e, uint32_t rail, char* buf, size_t cap) {
  return guard([&] {
    if (rail >= e->eng->rail_count()) throw EngineError("bad rail index");
    std::snprintf(buf, cap, "%s", e->eng->topology().rail(rail).id.c_str());
  });
}
int spray_rail_stats_get(spray_engine* e, uint32_t rail, spray_rail_stats* out) {
  return guard([&] { e->eng->rail_stats(rail, out); });
}
int spray_engine_counters(spray_engine* e, uint64_t* d, uint64_t* t, uint64_t* f) {
  return guard([&] { e->eng->counters(d, t, f); });
}
int spray_inject_fault(spray_engine* e, const char* rail, int32_t effect, uint64_t start, uint64_t end, double factor) {
  return guard([&] {
    e->eng->inject_fault(rail ? rail : "", effect, start, end, effect == SPRAY_FAULT_JITTER ? 1.0 : factor,
                         effect == SPRAY_FAULT_JITTER ? factor : 0.0);
  });
}

int spray_inject_fault_entry(spray_engine* e, const spray_fault_entry* f) {
  return guard([&] {
    if (!f) throw ConfigError("null fault entry");
    e->eng->inject_fault(f->rail_id ? f->rail_id : "", f->effect, f->start_ns, f->end_ns, f->factor, f->jitter_us);
  });
}
int spray_clear_faults(spray_engine* e) { return guard([&] { e->eng->clear_faults(); }); }
uint64_t spray_engine_now_ns(spray_engine* e) { return e->eng->now_ns(); }
int spray_heal_stats(spray_engine* e, uint64_t* fs, uint64_t* ok, uint64_t* fa, uint64_t* ro) {
  return guard([&] { e->eng->heal_stats(fs, ok, fa, ro); });
}

int spray_gate_segment(spray_engine* e, const char* segment_id, int role, void* flags) {
  return guard([&] { e->eng->gate_segment(segment_id ? segment_id : "", static_cast<uint32_t>(role), flags); });
}

int spray_gate_ring(spray_engine* e, const char* segment_id, int role, void* flags, void* credits,
                    uint64_t logical_bytes) {
  if (!logical_bytes) return SPRAY_ECONFIG;
  return guard([&] {
    e->eng->gate_segment(segment_id ? segment_id : "", static_cast<uint32_t>(role), flags, credits, logical_bytes);
  });
}

int spray_telemetry_csv(spray_engine* e, char* buf, size_t cap, size_t* len) {
  return guard([&] {
    const std::string s = e->eng->telemetry_csv();
    if (len) *len = s.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

size_t spray_board_bytes(uint32_t n_slots) { return spray::board_bytes(n_slots); }
int spray_engine_attach_board(spray_engine* e, void* board, uint32_t n_slots, uint32_t slot, uint64_t period_ns) {
  return guard([&] { e->eng->attach_board(board, n_slots, slot, period_ns); });
}
int spray_engine_chunk_bytes(spray_engine* e, uint64_t* out) {
  return guard([&] { *out = e->eng->chunk_bytes(); });
}

int spray_engine_debug(spray_engine* e, uint64_t* out, size_t n) {
  return guard([&] { e->eng->debug_words(out, n); });
}

int spray_trace_enable(spray_engine* e, size_t cap) { return guard([&] { e->eng->trace_enable(cap); }); }
int spray_trace_fetch(spray_engine* e, spray_trace_event* ev, size_t cap, size_t* n, spray_decision* dec, size_t dcap,
                      size_t* nd) {
  return guard([&] { e->eng->trace_fetch(ev, cap, n, dec, dcap, nd); });
}
int spray_trace_candidates(spray_engine* e, int32_t* stream, size_t cap, size_t* len) {
  return guard([&] {
    auto v = e->eng->trace_candidates();
    *len = v.size();
    if (stream) std::memcpy(stream, v.data(), std::min(cap, v.size()) * sizeof(int32_t));
  });
}
int spray_plan_candidates(spray_engine* e, const char* src, const char* dst, int32_t direction, int32_t* stream,
                          size_t cap, size_t* len, char* backend, size_t bcap) {
  return guard([&] {
    std::string b;
    auto v = e->eng->plan_candidates(src ? src : "", dst ? dst : "", direction, &b);
    *len = v.size();
    if (stream) std::memcpy(stream, v.data(), std::min(cap, v.size()) * sizeof(int32_t));
    if (backend) std::snprintf(backend, bcap, "%s", b.c_str());
  });
}

// ------------------------------------------------------------------ prepared (device-resident) batches
int spray_prepare_transfers(spray_engine* e, const spray_transfer_request* reqs, size_t n, spray_prepared** out) {
  return guard([&] {
    CK(cudaSetDevice(e->eng->device()));  // callers may be on any thread / current device
    uint64_t slices = 0;
    const std::vector<Intent> v = e->eng->prepare(reqs, n, &slices);  // under the engine lock
    auto* p = new spray_prepared;
    p->owner = e;
    p->n = n;
    p->slices = slices;
    CK(cudaMalloc(&p->dev, std::max<size_t>(1, n) * sizeof(Intent)));
    CK(cudaMemcpy(p->dev, v.data(), n * sizeof(Intent), cudaMemcpyHostToDevice));
    *out = p;
  });
}

int spray_run_prepared(spray_engine* e, uint64_t batch, spray_prepared* p, float* kernel_ms) {
  return guard([&] {
    if (p->owner != e) throw EngineError("prepared set belongs to another engine");
    Engine& g = *e->eng;
    CK(cudaSetDevice(g.device()));  // events below belong to the engine's device
    struct DrainGuard {  // drain mode is off again however the run ends
      Engine& g;
      explicit DrainGuard(Engine& e) : g(e) { g.set_drain(true); }
      ~DrainGuard() { g.set_drain(false); }
    } drain(g);
    // make sure no launch is resident, so this one is bracketed alone
    while (g.running_kernel()) std::this_thread::sleep_for(std::chrono::microseconds(50));
    CK(cudaStreamSynchronize(g.stream()));
    const float ms = g.run_device_intents_timed(batch, p->dev, p->n, p->slices);  // one drain-mode launch
    if (kernel_ms) *kernel_ms = ms;
  });
}

void spray_prepared_free(spray_prepared* p) {
  if (!p) return;
  if (p->dev) cudaFree(p->dev);
  delete p;
}

// ------------------------------------------------------------------ replay (device decision function)
int spray_replay_device(int device, const spray_sched_config* sc, const spray_resilience_config* rc, uint32_t n_rails,
                        const double* bandwidth, const int32_t* base_tier, const uint32_t* id_rank,
                        const int32_t* cand, size_t cand_len, const spray_trace_event* events, size_t n_events,
                        spray_decision* dec_out, size_t dcap, size_t* n_dec, uint64_t* expect_failures) {
  using namespace spray_dev;
  return guard([&] {
    if (n_rails > uint32_t(kMaxRails)) throw ConfigError("more than 64 rails");
    CK(cudaSetDevice(device));
    // candidate sets
    std::vector<CandSet> sets;
    size_t i = 0;
    const int32_t ns = cand_len ? cand[i++] : 0;
    for (int32_t k = 0; k < ns; ++k) {
      CandSet cs{};
      cs.n_locals = static_cast<uint32_t>(cand[i++]);
      if (cs.n_locals > uint32_t(kMaxLocals)) throw ConfigError("more than 32 locals in a candidate set");
      for (uint32_t l = 0; l < cs.n_locals; ++l) {
        cs.local[l] = static_cast<uint32_t>(cand[i++]);
        cs.n_pairs[l] = static_cast<uint32_t>(cand[i++]);
        if (cs.n_pairs[l] > uint32_t(kMaxPairs)) throw ConfigError("more than 16 pairs");
        for (uint32_t p = 0; p < cs.n_pairs[l]; ++p) {
          cs.pair_remote[l][p] = static_cast<uint32_t>(cand[i++]);
          cs.pair_tier[l][p] = cand[i++];
          cs.pair_aff[l][p] = static_cast<uint8_t>(cand[i++] != 0);
        }
      }
      sets.push_back(cs);
    }
    if (i > cand_len) throw ConfigError("candidate stream overrun");
    std::vector<RailDesc> rd(n_rails);
    std::vector<RailState> rs(n_rails);
    for (uint32_t r = 0; r < n_rails; ++r) {
      rd[r] = RailDesc{};
      rd[r].bandwidth = bandwidth[r];
      rd[r].base_tier = base_tier[r];
      rd[r].id_rank = id_rank ? id_rank[r] : r;
      rs[r] = RailState{};
      rs[r].beta0 = sc->beta0_init_s;
      rs[r].beta1 = sc->beta1_init;
    }
    std::vector<void*> allocs;
    auto dev = [&](size_t bytes) {
      void* p = nullptr;
      CK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
      allocs.push_back(p);
      return p;
    };
    try {
      EngineDev E{};
      E.rails = static_cast<RailDesc*>(dev(sizeof(RailDesc) * n_rails));
      E.rail_state = static_cast<RailState*>(dev(sizeof(RailState) * n_rails));
      E.sets = static_cast<CandSet*>(dev(sizeof(CandSet) * sets.size()));
      E.n_rails = n_rails;
      E.n_sets = static_cast<uint32_t>(sets.size());
      E.tolerance = sc->tolerance;
      for (int t = 0; t < 3; ++t) E.penalty[t] = sc->penalty[t];
      E.alpha = sc->ewma_alpha;
      E.beta0_init = sc->beta0_init_s;
      E.beta1_init = sc->beta1_init;
      E.clamp = sc->feedback_clamp;
      E.omega = sc->diffusion_weight;  // trace semantics: omega > 0 <=> a board is attached
      E.reset_interval = sc->reset_interval_ns;
      E.policy = static_cast<uint32_t>(sc->policy);
      E.failure_threshold = rc->failure_threshold;
      E.degradation_events = rc->degradation_events;
      E.degradation_ratio = rc->degradation_ratio;
      E.degradation_min_t = rc->degradation_min_t_obs_s;
      E.probe_successes = rc->probe_successes_needed;
      E.probe_interval = rc->probe_interval_ns;
      E.probe_backoff_mult = rc->probe_backoff_mult;
      E.probe_backoff_cap = rc->probe_backoff_cap;
      CK(cudaMemcpy(const_cast<RailDesc*>(E.rails), rd.data(), sizeof(RailDesc) * n_rails, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(E.rail_state, rs.data(), sizeof(RailState) * n_rails, cudaMemcpyHostToDevice));
      if (!sets.empty())
        CK(cudaMemcpy(const_cast<CandSet*>(E.sets), sets.data(), sizeof(CandSet) * sets.size(), cudaMemcpyHostToDevice));
      auto* ev = static_cast<spray_trace_event*>(dev(sizeof(spray_trace_event) * n_events));
      CK(cudaMemcpy(ev, events, sizeof(spray_trace_event) * n_events, cudaMemcpyHostToDevice));
      auto* dd = static_cast<spray_decision*>(dev(sizeof(spray_decision) * std::max<size_t>(dcap, 1)));
      auto* out = static_cast<unsigned long long*>(dev(2 * sizeof(unsigned long long)));
      auto* fin = static_cast<RailState*>(dev(sizeof(RailState) * n_rails));
      CK(spray_launch::launch_replay(E, ev, n_events, dd, dcap, out, fin, 0));
      CK(cudaStreamSynchronize(0));
      unsigned long long o[2];
      CK(cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost));
      *n_dec = o[0];
      if (expect_failures) *expect_failures = o[1];
      if (dec_out && dcap) CK(cudaMemcpy(dec_out, dd, sizeof(spray_decision) * std::min<uint64_t>(dcap, o[0]), cudaMemcpyDeviceToHost));
    } catch (...) {
      for (void* p : allocs) cudaFree(p);
      throw;
    }
    for (void* p : allocs) cudaFree(p);
  });
}

// ------------------------------------------------------------------ utilities
int spray_fill_splitmix(int device, void* ptr, uint64_t n, uint64_t seed) {
  return guard([&] {
    CK(cudaSetDevice(device));
    CK(spray_launch::launch_fill(ptr, n, seed, 0));
    CK(cudaStreamSynchronize(0));  // not the device: a persistent engine kernel may be resident
  });
}

int spray_checksum(int device, const void* ptr, uint64_t n, uint64_t* out) {
  return guard([&] {
    CK(cudaSetDevice(device));
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, sizeof(unsigned long long)));
    cudaMemset(d, 0, sizeof(unsigned long long));
    cudaError_t e = spray_launch::launch_checksum(ptr, n, d, 0);
    unsigned long long v = 0;
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e == cudaSuccess) e = cudaMemcpy(&v, d, sizeof(v), cudaMemcpyDeviceToHost);
    cudaFree(d);
    CK(e);
    *out = v ^ n;
  });
}

int spray_host_alloc(uint64_t n, void** out) {
  return guard([&] { CK(cudaHostAlloc(out, n, cudaHostAllocMapped | cudaHostAllocPortable)); });
}
int spray_host_free(void* p) { return guard([&] { CK(cudaFreeHost(p)); }); }

// NUMA node of a GPU's PCIe root: /sys/bus/pci/devices/<bus id>/numa_node (-1: unknown or
// a single-node host).
static int numa_node_of(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  std::string id(bus);
  for (char& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  std::FILE* f = std::fopen(("/sys/bus/pci/devices/" + id + "/numa_node").c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (std::fscanf(f, "%d", &node) != 1) node = -1;
  std::fclose(f);
  return node;
}

static std::mutex g_numa_mu;
static std::map<void*, size_t> g_numa_allocs;

int spray_device_numa_node(int device, int32_t* node) {
  return guard([&] { *node = numa_node_of(device); });
}

// Pinned host memory on the GPU's own NUMA node: anonymous pages bound there with mbind
// (MPOL_BIND, strict) and faulted in before cudaHostRegister pins and maps them, so the
// PCIe root's DMA and the SM copies never cross the socket interconnect. Falls back to
// first-touch placement when the node is unknown.
int spray_host_alloc_numa(int device, uint64_t n, void** out, int32_t* node_out) {
  return guard([&] {
    if (n == 0) throw ConfigError("host_alloc_numa: zero bytes");
    const size_t len = (n + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
    void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) throw EngineError("host_alloc_numa: mmap failed");
    const int node = numa_node_of(device);
    int bound = -1;
    if (node >= 0 && node < 1024) {
      unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
      mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
      constexpr int kMpolBind = 2, kMfStrict = 1, kMfMove = 2;
      if (syscall(SYS_mbind, p, len, kMpolBind, mask, 1024ul, kMfStrict | kMfMove) == 0) bound = node;
    }
    std::memset(p, 0, len);  // fault every page in on the bound node
    const cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      munmap(p, len);
      CK(e);
    }
    {
      std::lock_guard<std::mutex> lk(g_numa_mu);
      g_numa_allocs[p] = len;
    }
    *out = p;
    if (node_out) *node_out = bound;
  });
}

int spray_host_free_numa(void* p) {
  return guard([&] {
    size_t len = 0;
    {
      std::lock_guard<std::mutex> lk(g_numa_mu);
      auto it = g_numa_allocs.find(p);
      if (it == g_numa_allocs.end()) throw EngineError("host_free_numa: not a spray_host_alloc_numa pointer");
      len = it->second;
      g_numa_allocs.erase(it);
    }
    CK(cudaHostUnregister(p));
    munmap(p, len);
  });
}

int spray_rr_copy(int device, const uint64_t* src, const uint64_t* dst, const uint64_t* len, size_t n, int streams,
                  double* ms_out) {
  return guard([&] {
    if (streams < 1 || streams > 64) throw ConfigError("rr_copy: streams must be in [1, 64]");
    CK(cudaSetDevice(device));
    std::vector<cudaStream_t> st(static_cast<size_t>(streams));
    for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaDeviceSynchronize());
    const auto t0 = std::chrono::steady_clock::now();
    for (size_t i = 0; i < n; ++i)
      CK(cudaMemcpyAsync(reinterpret_cast<void*>(dst[i]), reinterpret_cast<const void*>(src[i]), len[i],
                         cudaMemcpyDefault, st[i % st.size()]));
    for (auto& s : st) CK(cudaStreamSynchronize(s));
    const auto t1 = std::chrono::steady_clock::now();
    for (auto& s : st) cudaStreamDestroy(s);
    *ms_out = std::chrono::duration<double, std::milli>(t1 - t0).count();
  });
}

// The allocation base of a device pointer: cuMemGetAddressRange through the runtime's
// driver entry point (no link-time dependency on libcuda).
static uint64_t alloc_base(void* ptr) {
  using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw EngineError("cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<Fn>(f);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
    throw InvalidRangeError("ipc export: pointer is not inside a device allocation");
  return base;
}

static std::mutex g_ipc_mu;
static std::map<uint64_t, std::pair<uint64_t, int>> g_ipc_open;  // returned ptr -> (mapped base, refs)

int spray_ipc_export(int device, void* ptr, uint8_t handle_out[SPRAY_IPC_HANDLE_BYTES]) {
  return guard([&] {
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ptr));
    static_assert(sizeof(h) == 64, "ipc handle is 64 B");
    const uint64_t off = reinterpret_cast<uint64_t>(ptr) - alloc_base(ptr);
    std::memcpy(handle_out, &h, 64);
    std::memcpy(handle_out + 64, &off, 8);
  });
}
int spray_ipc_open(int device, const uint8_t handle[SPRAY_IPC_HANDLE_BYTES], void** ptr_out) {
  return guard([&] {
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    uint64_t off = 0;
    std::memcpy(&h, handle, 64);
    std::memcpy(&off, handle + 64, 8);
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    const uint64_t p = reinterpret_cast<uint64_t>(base) + off;
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto& e = g_ipc_open[p];
    e.first = reinterpret_cast<uint64_t>(base);
    ++e.second;
    *ptr_out = reinterpret_cast<void*>(p);
  });
}
int spray_ipc_close(void* ptr) {
  return guard([&] {
    uint64_t base = reinterpret_cast<uint64_t>(ptr);
    {
      std::lock_guard<std::mutex> lk(g_ipc_mu);
      auto it = g_ipc_open.find(base);
      if (it != g_ipc_open.end()) {
        base = it->second.first;
        if (--it->second.second == 0) g_ipc_open.erase(it);
      }
    }
    CK(cudaIpcCloseMemHandle(reinterpret_cast<void*>(base)));
  });
}

}  // extern "C"

// ------------------------------------------------------------------ backend (plugin mode)
// TransportBackend (backend.hpp:49-72) over CUDA: each post_slices group becomes one
// group_copy_kernel launch whose descriptors sit in mapped pinned memory; completions
// are reported per slice, in order, when the group's event fires.
struct spray_backend {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool started = false;
  bool fatal = false;
  uint32_t window = 64;  // in-flight slices per backend (sim_backend.hpp:18 analogue)
  struct Seg {
    Medium medium;
    std::vector<Buffer> bufs;
  };
  std::map<std::pair<uint64_t, uint64_t>, Seg> segs;
  struct Group {
    cudaEvent_t ev;
    std::vector<spray_cqe> cqes;
    void* descs;
    std::chrono::steady_clock::time_point t0;
  };
  std::deque<Group> groups;
  std::deque<spray_cqe> ready;
  uint32_t inflight = 0;
  std::mutex mu;
};

extern "C" {

int spray_backend_open(int device, spray_backend** out) {
  return guard([&] {
    auto* b = new spray_backend;
    b->device = device;
    *out = b;
  });
}

void spray_backend_close(spray_backend* b) {
  if (!b) return;
  spray_backend_stop(b);
  delete b;
}

int spray_backend_start(spray_backend* b) {
  return guard([&] {
    if (b->started) return;
    CK(cudaSetDevice(b->device));
    CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
    b->started = true;
  });
}

int spray_backend_stop(spray_backend* b) {
  return guard([&] {
    if (!b->started) return;
    cudaStreamSynchronize(b->stream);
    for (auto& g : b->groups) {
      cudaEventDestroy(g.ev);
      cudaFreeHost(g.descs);
    }
    b->groups.clear();
    cudaStreamDestroy(b->stream);
    b->started = false;
  });
}

int spray_backend_capabilities(spray_backend*, spray_backend_caps* out) {
  std::memset(out, 0, sizeof(*out));
  std::snprintf(out->id, sizeof(out->id), "cuda");
  out->media_pairs_mask = (1u << 0) | (1u << 1) | (1u << 3) | (1u << 4);
  out->supports_read = out->supports_write = 1;
  out->cross_node = out->same_node = 1;
  out->max_post_size = 1ull << 30;
  out->batched_posting = 1;
  return SPRAY_OK;
}

int spray_backend_attach_segment(spray_backend* b, const spray_segment_desc* d, uint8_t* blob, size_t cap,
                                 size_t* blob_len) {
  if (d->medium == SPRAY_MEDIUM_FILE) {
    g_err = "cuda backend: file media are not served";
    return SPRAY_ECAPABILITY;
  }
  return guard([&] {
    CK(cudaSetDevice(b->device));
    spray_backend::Seg s;
    s.medium = d->medium == SPRAY_MEDIUM_DEVICE ? Medium::kDevice : Medium::kHost;
    for (uint32_t i = 0; i < d->n_buffers; ++i) {
      Buffer buf{d->buffers[i].offset, d->buffers[i].length, d->buffers[i].data, 0};
      if (s.medium == Medium::kHost) {
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, buf.data, 0) != cudaSuccess) {
          cudaGetLastError();
          CK(cudaHostRegister(buf.data, buf.length, cudaHostRegisterMapped | cudaHostRegisterPortable));
          CK(cudaHostGetDevicePointer(&dp, buf.data, 0));
        }
        buf.dev_addr = reinterpret_cast<uint64_t>(dp);
      } else {
        buf.dev_addr = reinterpret_cast<uint64_t>(buf.data);
      }
      s.bufs.push_back(buf);
    }
    std::sort(s.bufs.begin(), s.bufs.end(), [](const Buffer& x, const Buffer& y) { return x.offset < y.offset; });
    const Hash128 h = hash128(d->id);
    std::lock_guard<std::mutex> lk(b->mu);
    b->segs[{h.lo, h.hi}] = std::move(s);
    const std::string tag = std::string("cuda:") + d->id;
    if (blob_len) *blob_len = tag.size();
    if (blob) std::memcpy(blob, tag.data(), std::min(cap, tag.size()));
  });
}

static uint64_t resolve(const spray_backend::Seg& s, uint64_t off, uint64_t len) {
  for (const Buffer& b : s.bufs) {
    if (off >= b.offset && off + len <= b.offset + b.length) return b.dev_addr + (off - b.offset);
    if (b.offset > off) break;
  }
  return 0;
}

int spray_backend_post(spray_backend* b, const spray_slice_wr* reqs, size_t n, size_t* accepted) {
  *accepted = 0;
  if (b->fatal) {
    g_err = "backend latched fatal";
    return SPRAY_EFATAL;
  }
  return guard([&] {
    if (!b->started) throw EngineError("backend not started");
    std::lock_guard<std::mutex> lk(b->mu);
    const size_t room = b->inflight >= b->window ? 0 : b->window - b->inflight;
    const size_t take = std::min(room, n);  // the rejected suffix is backpressure (backend.hpp:42-43)
    if (take == 0) return;
    struct GD {
      uint64_t src, dst, len, first_chunk;
    };
    void* hd = nullptr;
    CK(cudaHostAlloc(&hd, take * sizeof(GD), cudaHostAllocMapped | cudaHostAllocPortable));
    GD* gd = static_cast<GD*>(hd);
    spray_backend::Group g;
    g.descs = hd;
    const uint64_t chunk = 128 << 10;
    uint64_t chunks = 0;
    for (size_t i = 0; i < take; ++i) {
      const spray_slice_wr& r = reqs[i];
      auto si = b->segs.find({r.src_seg_lo, r.src_seg_hi});
      auto di = b->segs.find({r.dst_seg_lo, r.dst_seg_hi});
      if (si == b->segs.end() || di == b->segs.end()) {
        cudaFreeHost(hd);
        throw EngineError("cuda: unknown segment");
      }
      const uint64_t s = resolve(si->second, r.src_offset, r.length);
      const uint64_t d = resolve(di->second, r.dst_offset, r.length);
      if (!s || !d) {
        cudaFreeHost(hd);
        throw EngineError("cuda: slice range not covered by one buffer");
      }
      gd[i] = GD{s, d, r.length, chunks};
      chunks += (r.length + chunk - 1) / chunk;
      spray_cqe c{};
      c.slice = r.slice;
      c.batch = r.batch;
      c.status = SPRAY_SLICE_OK;
      c.rail = r.local_rail;
      c.bytes = r.length;
      g.cqes.push_back(c);
    }
    void* dd = nullptr;
    CK(cudaHostGetDevicePointer(&dd, hd, 0));
    CK(cudaSetDevice(b->device));
    CK(spray_launch::launch_group_copy(dd, static_cast<uint32_t>(take), chunks, chunk, 148 * 4, b->stream));
    CK(cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming));
    CK(cudaEventRecord(g.ev, b->stream));
    g.t0 = std::chrono::steady_clock::now();
    b->inflight += static_cast<uint32_t>(take);
    b->groups.push_back(std::move(g));
    *accepted = take;
  });
}

int spray_backend_poll(spray_backend* b, spray_cqe* out, size_t max, size_t* n) {
  *n = 0;
  return guard([&] {
    std::lock_guard<std::mutex> lk(b->mu);
    while (!b->groups.empty()) {
      spray_backend::Group& g = b->groups.front();
      const cudaError_t q = cudaEventQuery(g.ev);
      if (q == cudaErrorNotReady) break;
      const auto t1 = std::chrono::steady_clock::now();
      const uint64_t ns = static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - g.t0).count());
      for (spray_cqe& c : g.cqes) {
        c.t_obs_ns = ns > 0 ? ns : 1;
        if (q != cudaSuccess) {
          c.status = SPRAY_SLICE_FAILED;
          c.bytes = 0;
        }
        b->ready.push_back(c);
      }
      b->inflight -= static_cast<uint32_t>(g.cqes.size());
      cudaEventDestroy(g.ev);
      cudaFreeHost(g.descs);
      b->groups.pop_front();
    }
    while (*n < max && !b->ready.empty()) {
      out[(*n)++] = b->ready.front();
      b->ready.pop_front();
    }
  });
}

int spray_backend_fatal(spray_backend* b) { return b->fatal ? 1 : 0; }
int spray_backend_latch_fatal(spray_backend* b) {
  b->fatal = true;
  return SPRAY_OK;
}

}  // extern "C"
