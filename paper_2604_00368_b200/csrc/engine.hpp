// engine.hpp — host side of the B200 spray engine.
//
// Public surface = the reference Engine's batch API (proj/include/spray/engine.hpp:90-131).
// The host does only what must happen on the application's thread: validate the
// request, plan the route (candidate list, cached per (src, dst, direction)), resolve
// device-usable addresses and publish a 64-B intent into the mapped submission ring.
// Slicing, rail choice, copies, completion accounting, retries and health all run in
// the persistent device kernel (spray_kernel.cu). Batch status is read from mapped
// host counters the device writes: polling a batch never touches the GPU.
#pragma once
#include <atomic>
#include <cstdint>
#include <map>
#include <set>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/spray_b200.h"
#include "dev_types.cuh"
#include "fabric.hpp"
#include "orchestrator.hpp"

namespace spray {

struct EngineOptions {
  std::vector<std::string> backends = {"cuda"};
  spray_sched_config sched{};
  spray_resilience_config res{};
  double diffusion_weight = 0.0;
  // B200 execution parameters ("b200" section of the config document)
  int grid = 0;                 // 0 = one CTA per SM
  int block = 256;
  uint64_t chunk_bytes = 32 << 10;  // finer granules shorten the tail: C2 1 GiB 619 -> 653 GB/s (32 KiB), flat at 4 GiB
  uint64_t idle_exit_ns = 20'000'000;
  uint32_t slice_capacity = 1u << 17;
  uint64_t work_capacity = 1ull << 21;
  uint64_t sub_capacity = 1ull << 16;
  uint32_t batch_slots = 1u << 16;
  uint32_t max_sets = 1024;
  uint64_t gate_timeout_ns = 10'000'000'000ull;  // dataflow gate wait before an attempt fails
  uint64_t window_ns = 10'000'000;              // telemetry window (stats_window_ms)
  uint32_t fence_batch = 2;                      // chunks a copy warp copies per system fence when
                                                 // its next chunk is already queued (1 = every chunk)
  bool diag = false;                             // per-stage timeline words (Control::lat)
  bool worker_fence_sys = false;                 // copy warps fence at GPU scope before counting a chunk; PUBLISH's
                                                 // system fence before the host-visible words is cumulative over them
  bool fence_release = false;                    // system fences as fence.release.sys (else fence.sc.sys)
  uint32_t bulk_stages = 4;                      // shared-memory stages per copy warp (4 KiB each)
  bool copy_bulk = true;                         // copy warps move chunks with bulk copies (TMA) through
                                                 // shared memory (else 16-deep vector loads/stores)
  bool staged_routes = true;                     // synthesize host-staged routes to GPUs without peer access
  std::vector<int> no_peer;                      // GPUs treated as lacking peer access (testing / policy)
  uint32_t post_window = 0;                      // units in flight per rail (0: 2 x worker warps for
                                                 // SM/relay rails, 2048 orders for CE rails)
};

// engine_options_from_json (engine.cpp:1199-1307): unknown keys rejected.
EngineOptions engine_options_from_json(const std::string& text);
void default_sched_config(spray_sched_config* c);
size_t board_bytes(uint32_t n_slots);  // spray_board_bytes
void default_resilience_config(spray_resilience_config* c);

class Engine {
 public:
  Engine(EngineOptions opts, const std::string& topology_json, int device);
  ~Engine();

  void start();
  void stop();
  void register_segment(const spray_segment_desc& desc);
  uint64_t allocate_batch();
  uint64_t submit_transfer(uint64_t batch, const spray_transfer_request& req);
  size_t submit_transfers(uint64_t batch, const spray_transfer_request* reqs, size_t n, uint64_t* ids);
  spray_batch_status_t batch_status(uint64_t batch);
  spray_batch_status_t await_batch(uint64_t batch, uint64_t limit_ns);
  void free_batch(uint64_t batch);

  // Device-resident submission (bench / device producers): `dev_intents` is an HBM
  // array of n Intent records built with make_intent(). Counts n transfers into batch.
  struct BatchRec;
  struct SegRec;
  // Lookups reused across the requests of one submit call (consecutive requests usually
  // name the same segments and route).
  struct LookupCache {
    uint64_t batch_id = 0;
    BatchRec* batch = nullptr;
    const char *src_name = nullptr, *dst_name = nullptr;
    SegRec *src = nullptr, *dst = nullptr;
    const SegRec *set_src = nullptr, *set_dst = nullptr;
    int set_dir = -1;
    uint32_t set = 0;
  };
  spray_dev::Intent make_intent(uint64_t batch, const spray_transfer_request& req, uint64_t* n_slices,
                                LookupCache* lc = nullptr);
  void submit_device_intents(uint64_t batch, const void* dev_intents, uint64_t n, uint64_t total_slices);
  std::vector<spray_dev::Intent> prepare(const spray_transfer_request* reqs, size_t n, uint64_t* slices);
  void set_drain(bool on);
  cudaStream_t stream() const { return stream_; }
  bool running_kernel();

  const Topology& topology() const { return topo_; }
  uint32_t rail_count() const { return static_cast<uint32_t>(topo_.rail_count()); }
  void rail_stats(uint32_t rail, spray_rail_stats* out);
  void counters(uint64_t* dispatched, uint64_t* terminated, uint64_t* failed);
  void inject_fault(const std::string& rail, int effect, uint64_t start, uint64_t end, double factor,
                    double jitter_us = 0.0);
  void clear_faults();
  uint64_t now_ns();
  void heal_stats(uint64_t* fs, uint64_t* ok, uint64_t* fa, uint64_t* ro);

  void trace_enable(size_t cap);
  void trace_fetch(spray_trace_event* ev, size_t cap, size_t* n, spray_decision* dec, size_t dcap, size_t* nd);
  std::vector<int32_t> trace_candidates();
  // Candidate stream of the route the engine would use (host planning only).
  std::vector<int32_t> plan_candidates(const std::string& src, const std::string& dst, int dir,
                                       std::string* backend);

  int device() const { return device_; }
  uint64_t chunk_bytes() const { return opts_.chunk_bytes; }
  // Dataflow gate on a registered single-buffer segment (role kGateConsume/kGateProduce);
  // `flags` = one uint32 counter per chunk_bytes granule, device memory reachable from this
  // GPU (the producer's and the consumer's engines share it).
  void gate_segment(const std::string& seg_id, uint32_t role, void* flags, void* credits = nullptr,
                    uint64_t logical_bytes = 0);
  // GlobalLoadBoard (scheduler.hpp:66-90): publish/blend through a shared host board
  void attach_board(void* board, uint32_t n_slots, uint32_t slot, uint64_t period_ns);
  // prepared intents in one drain-mode launch, timed by CUDA events around the kernel only
  float run_device_intents_timed(uint64_t batch, const void* dev_intents, uint64_t n, uint64_t total_slices);
  // TelemetrySnapshot::to_csv columns from the device's per-rail window cells.
  std::string telemetry_csv();
  // Diagnostic snapshot: host/device ring positions, kernel state, counters, stream status.
  void debug_words(uint64_t* out, size_t n);

  struct BatchRec {
    uint64_t id = 0;
    uint32_t slot = 0;
    uint64_t base = 0;       // device done-counter value when the batch was allocated
    uint64_t submitted = 0;  // slices submitted (decompose counts)
  };
  struct SegRec {
    Segment seg;
    bool translated = false;
    bool gated = false;             // a dataflow gate covers this segment
    uint64_t ring = 0;              // ring gate: physical bytes behind the logical window
    std::vector<void*> registered;  // host buffers we cudaHostRegister'ed
  };

 private:

  void alloc_device();
  void free_device();
  void launch();
  int launch_grid();
  void ensure_running();
  uint32_t set_for(const Segment& src, const Segment& dst, Direction dir);
  uint32_t add_set(const Route& r, uint32_t next);  // one route's candidate set, chained to the plan's next
  void translate(SegRec& s);
  void publish(const spray_dev::Intent* in, size_t n);
  SegRec& seg_lookup(const char* name, const char*& cname, SegRec*& crec);
  void ce_proxy_loop(int k);
  BatchRec& batch_ref(uint64_t id);
  uint64_t allocate_batch_locked();
  void free_batch_locked(uint64_t batch);
  uint64_t decompose_count(uint64_t len) const;
  void synthesize_staged_routes();
  void filter_staged(Route& r, const Segment& src, const Segment& dst) const;
  std::set<int> no_peer_gpus_;

  EngineOptions opts_;
  Topology topo_;
  int device_;
  std::vector<Capabilities> caps_;
  std::mutex mu_;
  std::map<std::string, SegRec> segs_;
  std::map<uint64_t, BatchRec> batches_;
  std::vector<uint8_t> slot_busy_;
  uint64_t next_batch_ = 1, next_transfer_ = 1;
  uint32_t next_slot_ = 0;
  int64_t last_freed_ = -1;  // slot of the last batch freed after completing (allocated first)
  std::map<std::string, uint32_t> set_cache_;
  std::vector<std::vector<LocalCandidate>> sets_;
  bool started_ = false;
  bool wedged_ = false;  // stop() timed out: device memory is left to process teardown

  // device resources
  cudaStream_t stream_ = nullptr, copy_stream_ = nullptr;
  spray_dev::EngineDev E_{};
  spray_dev::Control* ctl_ = nullptr;        // mapped host
  spray_dev::Intent* ring_ = nullptr;        // mapped host
  spray_dev::BatchDev* bmirror_ = nullptr;   // mapped host
  spray_dev::FaultDev* faults_ = nullptr;    // mapped host
  spray_dev::RailState* rmirror_ = nullptr;  // mapped host
  spray_dev::CeOrder* ce_ring_ = nullptr;    // mapped host
  spray_dev::Completion* xc_ring_ = nullptr; // mapped host
  std::vector<void*> dev_allocs_;
  uint64_t sub_tail_ = 0;
  size_t trace_cap_ = 0;
  bool drain_ = false;

  // CE proxy
  std::vector<std::thread> ce_threads_;
  std::atomic<bool> ce_run_{false};
  std::atomic<uint64_t> xc_reserve_{0};  // next CE completion ring position (proxy threads)
  std::vector<cudaStream_t> ce_streams_;
  bool has_ce_ = false;

  // 2-hop relay rails: state on the relay GPU, one forwarder kernel per relay and launch
  struct RelayHost {
    int via = -1;
    cudaStream_t stream = nullptr;    // on the relay GPU
    std::vector<void*> via_allocs;    // staging, descriptors, exit generation
    std::vector<void*> host_allocs;   // host-staged relays: the pinned pool and its rings
  };
  std::vector<RelayHost> relays_;
  void* board_registered_ = nullptr;  // host board this engine registered (unregistered on free)
  volatile uint32_t* hold_ = nullptr;  // mapped flag of the timed-run stream hold
  uint32_t* hold_dev_ = nullptr;
  // large submissions are staged through HBM as bulk intent arrays (submit_staged_locked)
  static constexpr size_t kStageMin = 1024, kStageCap = 1024;  // intents (per piece / area)
  static constexpr uint32_t kStageAreas = 8;
  spray_dev::Intent* stage_host_ = nullptr;      // pinned, kStageAreas x kStageCap intents
  spray_dev::Intent* stage_dev_[kStageAreas] = {};
  uint64_t stage_use_[kStageAreas] = {};  // bulk index of each area's last use (1-based)
  uint64_t bulk_pub_ = 0;             // bulk entries this engine has published
  size_t submit_staged_locked(uint64_t batch, const spray_transfer_request* reqs, size_t n, uint64_t* ids);
  uint32_t launch_gen_ = 0;
  void setup_relay(uint32_t idx, int via, bool host_staged);
  void sync_relays();
  bool host_only_sm_ = false;  // every SM rail stages through pinned host memory
  static constexpr int kHostLinkCtas = 48;
  static constexpr uint64_t ce_cap = 4096;  // CE orders per proxy stream ring
};

}  // namespace spray
