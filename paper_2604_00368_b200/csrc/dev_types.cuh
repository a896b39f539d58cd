// dev_types.cuh — POD layout shared by the host engine (C++) and the persistent
// sm_100a spray kernel. Everything the device touches lives in one of three places:
//   * HBM (cudaMalloc): slice table, SM work ring, completion ring, candidate tables,
//     trace buffers, per-engine flags — hot, written and read only by the GPU;
//   * mapped pinned host memory (cudaHostAlloc Mapped): the submission ring the host
//     produces into, batch counters the host polls, the CE proxy rings and the stats
//     mirror — the host<->device boundary, no cudaMemcpy on it;
//   * shared memory of CTA 0: the scheduler warp's working copy of the per-rail cost
//     state (scheduler.hpp:158-168), single-owner, so decisions need no atomics.
#pragma once
#include <stdint.h>

namespace spray_dev {

constexpr int kMaxRails = 64;          // per engine (one GPU's fabric view)
constexpr int kMaxLocals = 32;         // candidates per set: one scheduler lane each
constexpr int kMaxPairs = 16;          // remote options per candidate
constexpr uint32_t kNoRail = 0xffffffffu;

enum : uint32_t { kHealthy = 0, kExcluded = 1, kProbing = 2 };
enum : uint32_t { kExecSM = 0, kExecCE = 1, kExecRelay = 2 };
enum : uint32_t { kStOk = 0, kStFailed = 1, kStTimeout = 2 };

// Per-rail immutable description (uploaded at start).
struct RailDesc {
  double bandwidth;       // B_d, bytes/s (fabric.hpp:68)
  int32_t base_tier;      // 1..3
  uint32_t id_rank;       // rank of the rail id string: map_remote/dispatch_retry tie-break
  uint32_t executor;      // kExec*
  int32_t gpu;            // owning GPU ordinal (-1 for host-side rails)
  int32_t via;            // relay GPU (relay rails)
  uint32_t ce_index;      // CE proxy stream index (CE rails); relay index (relay rails)
  uint8_t n_partners;     // probe counterparts, affinity partner first (resilience.cpp:17-44)
  uint8_t partners[15];
  uint32_t window;        // posting window: units (chunks; CE orders) in flight on the rail
                          // (SimBackend inflight_window, sim_backend.cpp:81; engine.cpp:884-948)
  uint32_t pad_w;
};

// Scheduler cost state (scheduler.hpp:158-168) + resilience record (resilience.hpp:68-76)
// + telemetry counters (telemetry.hpp:88-98). Lives in CTA-0 shared memory while the
// kernel runs; written back to HBM when it exits and mirrored to host periodically.
struct RailState {
  double beta0, beta1, min_obs;
  int64_t queued;
  uint64_t last_reset;
  uint32_t health;
  uint32_t has_obs;
  int32_t consec_failures;
  int32_t degradation_count;
  int32_t backoff;
  int32_t probe_streak;
  uint32_t probe_inflight;
  uint32_t beta_epoch;     // bumped whenever beta0/beta1/min_obs change other than by adopting
                           // the FEEDBACK warp's chain result (its stale-result check)
  uint64_t next_probe, excluded_at;
  uint64_t bytes_posted, bytes_ok, bytes_failed;
  uint32_t hist[48];
};

constexpr uint32_t kNoSet = 0xffffffffu;
// Candidate set (orchestrator.cpp:39-81 output), flattened for the device.
struct alignas(16) CandSet {
  uint32_t n_locals;
  uint32_t next_set;  // the plan's next route (TransferPlan::advance_past_backend), kNoSet if none
  uint32_t local[kMaxLocals];
  uint32_t n_pairs[kMaxLocals];
  uint32_t pair_remote[kMaxLocals][kMaxPairs];
  int32_t pair_tier[kMaxLocals][kMaxPairs];
  uint8_t pair_aff[kMaxLocals][kMaxPairs];
};

// One transfer intent (TransferRequest after planning), 64 B, in the submission ring.
// flags bit0 = BULK: src points at an array of `len` Intent records in HBM that inherit
// this record's batch.
struct Intent {
  uint64_t batch_id;
  uint64_t src;           // device-usable address of src_offset (BULK: HBM Intent array)
  uint64_t dst;           // device-usable address of dst_offset
  uint64_t len;           // bytes (BULK: number of intents in the array)
  uint64_t hash_offset;   // absolute source offset (hash policy input, engine.cpp:387)
  uint64_t transfer_id;
  uint32_t set_id;
  uint32_t batch_slot;
  uint32_t flags;
  uint32_t pad_;
};
static_assert(sizeof(Intent) == 64, "intent is one 64-B line");
constexpr uint32_t kIntentBulk = 1u;

// Slice record (engine.hpp:135-161 SliceRec, device form), in HBM. 128 B.
struct Slice {
  uint64_t src, dst, len;
  uint64_t dispatched_at;
  double predicted, x_norm;
  uint64_t batch_id;
  uint64_t hash_offset;
  uint32_t local, remote;
  uint32_t attempt;
  uint32_t batch_slot;
  uint32_t set_id;
  uint32_t model;          // 1 = dispatched by the cost model
  uint32_t target;         // units (chunks; 1 for a CE order) of the current attempt
  uint32_t n_failed_pairs;
  uint8_t failed_local[4], failed_remote[4];  // burned pairs (engine.cpp:765-767)
  uint32_t kind;           // kSliceData or kSliceProbe (engine.hpp:133 SliceKind)
  uint32_t gen;            // attempt generation of the slot's counter (last issued attempt)
  uint8_t pad_[16];
};
constexpr uint32_t kSliceData = 0, kSliceProbe = 2;
static_assert(sizeof(Slice) == 128, "slice record is 128 B");

// SM work item: one chunk, self-contained so a worker never reads the slice record to
// copy. `stamp` = ring position + 1 publishes it. 48 B.
struct WorkItem {
  uint64_t src, dst;
  uint32_t len;
  uint32_t slice;
  uint32_t target;         // units of the attempt: its slot counter closes at this count
  uint16_t rail, remote;   // fault words to honour (remote 0xffff = none)
  uint32_t gen;            // attempt generation (slot counter high word)
  uint32_t pad_;
  uint32_t stamp;
  uint32_t pad2_;
};
static_assert(sizeof(WorkItem) == 48, "work item is 48 B");
static_assert(offsetof(WorkItem, len) == 16 && offsetof(WorkItem, rail) == 28 && offsetof(WorkItem, remote) == 30 &&
                  offsetof(WorkItem, gen) == 32 && offsetof(WorkItem, stamp) == 40,
              "EGRESS writes work items as two 16-byte vectors + the generation word");

// Per-slot attempt counter (HBM, one 64-bit word per slice slot): the exactly-once rule of
// process_completion (engine.cpp:792-797: an event for an attempt that is no longer
// outstanding is stale) on the device. high 32 bits = the attempt generation EGRESS armed it
// with; bits 29..0 = units of that attempt delivered; FAIL = some unit failed; CLOSED = the
// attempt's terminal event is decided. Units count only while the generation matches and
// the word is open, so a late unit of a timed-out attempt never counts for its retry, and
// exactly one of {the last unit, the timeout scanner} closes an attempt and posts its
// completion word.
constexpr uint64_t kCtrClosed = 1ull << 31, kCtrFail = 1ull << 30, kCtrCount = (1ull << 30) - 1;

// Posting deadline of the outstanding attempt of a slot (worker_timeout_phase analog,
// engine.cpp:953-956, 996-1022): bits 47..0 = (engine ns >> 10) after which the attempt
// times out, bits 63..48 = low 16 bits of its generation; 0 = none.
constexpr uint64_t kDlMask = (1ull << 48) - 1;

// Device completion word: one 8-byte store carries slice, status and the publication
// stamp, so a reader validates and reads it in a single access (no acquire fence).
__host__ __device__ inline uint64_t pack_completion(uint32_t slice, uint32_t status, uint32_t stamp) {
  return ((uint64_t)stamp << 32) | ((uint64_t)(status & 0xfu) << 28) | (slice & 0x0fffffffu);
}

// Completion record posted by the CE proxy on the host (mapped ring). 32 B.
struct Completion {
  uint32_t slice;
  uint32_t gen;            // attempt generation of the order
  uint32_t status;
  uint32_t rail;
  uint64_t t_done;         // engine clock at completion
  uint32_t stamp;
  uint32_t pad_;
};

// CE work order to the host proxy (mapped host ring), 48 B.
struct CeOrder {
  uint64_t src, dst, len;
  uint32_t slice, gen;     // slot and attempt generation (echoed in the Completion)
  uint32_t rail, remote;   // fault words the proxy honours (remote 0xffffffff = none)
  uint64_t stamp;
};

// Per-batch counters. Slots are reused across batches: `done` is monotonic over the
// slot's lifetime (the host keeps the value at allocation as the batch's base) and
// `failed_id` names the batch id that failed (AllRoutesExhausted): no reset is needed.
struct BatchDev {
  uint64_t done;           // slices delivered through this slot (finish_logical count)
  uint64_t failed_id;      // batch id that failed terminally in this slot (0 = none)
  uint64_t owner;          // HBM copy only: newest batch id whose slices used this slot;
                           // a completion of an older batch id is from a freed failed batch
  uint64_t pad_;
};

// Fault words per rail: one FaultEntry (backend.hpp:74-94) per effect, as the reference
// schedule allows one interval per (rail, effect) (FaultSchedule::validate).
enum : uint32_t { kFxDown = 0, kFxDegrade = 1, kFxJitter = 2, kFxDrop = 3 };
struct FaultDev {
  uint64_t start[4], end[4];  // engine ns, per effect
  double factor;              // degrade: bandwidth multiplier
  double jitter_us;           // jitter: uniform added delay bound (FaultEntry::jitter_us)
  uint32_t active;            // bit e: effect e scheduled (written last)
  uint32_t pad_;
};

// The host<->device control block (mapped host memory). The first 32 bytes are the
// host->device words the scheduler polls; it reads them in one round trip.
struct alignas(64) Control {
  volatile uint64_t sub_tail;        // host: intents published
  volatile uint32_t stop;            // host: request exit
  volatile uint32_t drain;           // host: exit when idle (bench timing mode)
  volatile uint32_t fault_epoch;     // host: bumped whenever a fault word changes
  volatile uint32_t trace_on;
  volatile uint64_t idle_exit_ns;
  // device -> host
  volatile uint64_t sub_head;        // intents consumed
  volatile uint64_t bulk_done;       // bulk intent arrays fully read by the device (in order)
  volatile uint32_t state;           // 0 exited, 1 running, 2 exiting
  volatile uint32_t pad0_;
  volatile uint64_t device_now;      // engine clock (ns since epoch) seen by the scheduler
  volatile uint64_t epoch;           // globaltimer value of engine time 0
  volatile uint64_t bytes_dispatched, bytes_terminated;
  volatile uint64_t batches_failed;
  volatile uint64_t heal_fault_start, heal_first_ok, failed_attempts, retried_ok;
  volatile uint64_t ce_tail[8];      // device: CE orders produced per CE stream
  volatile uint64_t ce_head[8];      // host: CE orders consumed
  volatile uint64_t xc_tail;         // host: external completions produced (CE proxy)
  volatile uint64_t xc_head;         // device: consumed
  volatile uint64_t trace_n, trace_dn;
  volatile uint64_t error;           // sticky device-side error code (0 = none)
  // scheduler profile (globaltimer ns): loops, time in completions / submissions / control
  volatile uint64_t prof_loops, prof_comp_ns, prof_sub_ns, prof_ctl_ns, prof_n_comp, prof_n_dec;
  volatile uint64_t prof_x[16];      // fine-grained scheduler phase clocks (SM cycles) and counts
  // per-launch timeline (engine ns): 0 scheduler start, 1 first work items stamped,
  // 2 first decision, 3 last decision, 4 first completion applied, 5 last completion
  // applied, 6 scheduler exit
  volatile uint64_t tl[8];
  volatile uint64_t lat_w[8];        // b200.diag: a copy warp's last chunk (picked up, copied,
                                     // fenced, counted) and COMPLETE's word seen / record read
  volatile uint64_t lat[8];          // b200.diag: engine ns of the last pass of each pipeline stage
                                     // (HOSTRX fetch, INGRESS block, STATE decide, EGRESS post,
                                     // PUBLISH stamp, COMPLETE gather, STATE apply, PUBLISH done)
  volatile uint64_t dbg[16];         // diagnostic words (relay 0: hop-1 / hop-2 tickets, slots 0-3's
                                     // free rounds and descriptor stamps, exit generation)
  volatile uint64_t prof_y[8];       // decision phases (cycles): table, broadcast, lane-0 loop,
                                     // its decisions, its blocks, hand-back, warp-path decisions
  volatile uint64_t prof_z[8];       // FEEDBACK warp: chain cycles, completions, entries
  volatile uint64_t lat_s[8];        // b200.diag: STATE sub-steps (block seen, slots, set, -, completion seen, FEEDBACK done)
  volatile uint32_t resident_gen;    // launch generation whose every engine CTA is resident
};

// Telemetry window cell (telemetry.hpp:37-44 WindowCell), one per rail per window in an
// HBM ring of kTeleWindows windows: the STATE warp updates it at every completion.
constexpr uint32_t kTeleWindows = 1024;
struct TeleCell {
  uint64_t window;          // absolute window index (engine ns / window_ns); ~0 = empty
  uint64_t bytes_ok, bytes_failed;
  int64_t queue_close;
  uint32_t health_close, touched;
  uint32_t hist[48];        // OK service times, LatencyHistogram buckets
};

// Dataflow gate on one segment (forwarding, relays, broadcast chains; SURVEY.md §8(e):
// GPU k re-emits slices it received). Per granule (= chunk_bytes) of [lo, hi):
//   CONSUME: this engine's workers read a granule only once flags[g] > consumed[g];
//            consumed[g] (this engine's HBM) advances when a slice reading it completes OK.
//   PRODUCE: when a slice writing the granule completes OK, flags[g] (any GPU) advances,
//            after a system fence (PUBLISH warp).
enum : uint32_t { kGateConsume = 1, kGateProduce = 2 };
constexpr int kMaxGates = 4;
//   Ring gates (ring != 0; the staged route's bounded staging pool, engine.hpp:56-58):
//   the segment's logical window [lo, hi) wraps onto its physical buffer [phys, phys + ring),
//   lap = (addr - lo) / ring. A CONSUME read of lap k waits for flags[g] >= k + 1 and,
//   when it completes OK, stores its lap count into credits[g]; a PRODUCE write of lap k waits for
//   credits[g] >= k (the consumer drained lap k - 1 of the granule).
struct GateDev {
  uint64_t lo, hi;         // device-usable address range of the segment (logical for a ring)
  uint32_t* flags;         // per-granule counters (written by the producing engine)
  uint32_t* consumed;      // per-granule consumption counters (CONSUME only, local HBM)
  uint32_t* produced;      // per-granule production counters (PRODUCE only, local HBM): the
                           // flag is written as a plain value, so it may live in any memory
                           // this GPU can store to (peer HBM, mapped pinned host memory)
  uint32_t* credits;       // ring only: per-granule drained laps (CONSUME adds, PRODUCE waits)
  uint64_t ring;           // physical bytes of a ring gate, 0 for a plain gate
  uint64_t phys;           // ring only: device address of the physical buffer; lo is a tagged
                           // virtual base (bit 63 set) that no real allocation can alias
  uint32_t role;
  uint32_t ngran;          // granules of the physical buffer
};

// 2-hop relay rail (executor "relay", via GPU K). Hop 1: this engine's copy workers move a
// chunk into a staging slot in K's HBM and publish a descriptor there; hop 2: a forwarder
// kernel running on K's SMs moves it to the destination and does the chunk's completion
// accounting in this engine's counters (peer atomics), so to the scheduler a relay chunk
// completes like any other chunk. Tickets restart at 0 every launch (the prologue clears
// `tail` and `seq`, the host clears `head` on K's stream); descriptor stamps carry the
// launch generation.
constexpr int kMaxRelays = 8;
struct RelayDesc {  // 32 B, in K's HBM: written by the hop-1 worker, read by the forwarder
  uint64_t dst;
  uint32_t len, slice, target, gen;  // target = units of the attempt, gen = its generation
  uint64_t stamp;   // (launch_gen << 32) | (ticket + 1), release-stored last
};
// Host-staged relay (the staged route, engine.cpp:465-610: D2H into a bounded pinned-host
// pool, H2D out of it, pipelined; needs no peer access): staging, descriptors, slot rounds,
// the exit generation and a ticket-indexed completion ring live in mapped pinned host
// memory. The forwarder on K cannot touch this engine's counters, so it posts each forwarded
// chunk into `done[ticket % n_slots]` (stamped last); HOSTRX drains that ring in ticket order
// into COMPLETE, like copy-engine completions, and publishes `consumed` (this GPU's HBM),
// which hop 1 checks before reusing a ring position.
struct RelayDone {
  uint32_t slice, gen, target, pad_;  // target: units | drop flag (bit 31)
  uint64_t stamp;                     // (launch_gen << 32) | (ticket + 1), release-stored last
  uint64_t pad2_;
};
struct RelayDev {
  uint8_t* staging;             // K's HBM (host-staged: pinned host): n_slots x chunk_bytes
  RelayDesc* desc;              // K's HBM (host-staged: pinned host): n_slots descriptors
  uint32_t* exit_gen;           // K's HBM (host-staged: pinned host): launch generation on exit
  uint32_t* seq;                // this GPU's HBM (host-staged: pinned host): per-slot free round
  unsigned long long* tail;     // this GPU's HBM: hop-1 ticket counter (workers)
  unsigned long long* head;     // K's HBM: hop-2 ticket counter (forwarder warps)
  RelayDone* done;              // host-staged only: this GPU's HBM, hop 1's record of each slot's
                                //   chunk (slice, generation, units); stamp unused
  uint64_t* done_stamp;         // host-staged only: pinned host, per slot: (launch_gen << 32) |
                                //   (ticket + 1) once the forwarder has drained the slot
  unsigned long long* consumed; // host-staged only: this GPU's HBM, done records HOSTRX drained
  uint32_t* writers;            // host-staged only: this GPU's HBM, hop-1 warps writing the pool now
  uint32_t n_slots, via;        // power of two; relay GPU ordinal
  uint32_t host_staged, pad_;
};

// GlobalLoadBoard slot (scheduler.hpp:66-90) in caller-owned shared host memory: one per
// engine instance; `heartbeat` = GPU global timer at the slot's last publish.
struct BoardSlot {
  uint64_t heartbeat;
  uint64_t pad_;
  int64_t queued[kMaxRails];
};

// The device-written control-block words a launch resumes from, snapshotted by the host
// at launch (no kernel is resident then): reading them from mapped host memory at kernel
// start cost one PCIe round trip each on the scheduler's critical path.
struct LaunchSnap {
  uint64_t sub_head, bulk_done, xc_head, ce_tail[8], idle_exit_ns;
  uint64_t bytes_dispatched, bytes_terminated, batches_failed;
  uint64_t heal_fault_start, heal_first_ok, failed_attempts, retried_ok, trace_n, trace_dn;
  uint32_t drain, trace_on;
};

// Everything the kernel needs, passed by value.
struct EngineDev {
  Control* ctl;                      // mapped host
  Intent* sub_ring; uint64_t sub_cap;  // mapped host
  BatchDev* batches; uint32_t n_batch_slots;  // mapped host mirror (device writes, host reads)
  BatchDev* batches_hbm;             // HBM: the scheduler's own copy
  FaultDev* faults;                  // mapped host, per rail (host writes)
  RailState* rail_mirror;            // mapped host, per rail (stats mirror)
  CeOrder* ce_ring; uint64_t ce_cap; // mapped host, [8][ce_cap]
  Completion* xc_ring; uint64_t xc_cap;  // mapped host (CE proxy completions)

  const RailDesc* rails; uint32_t n_rails;     // HBM
  RailState* rail_state;                       // HBM (persisted between launches)
  const CandSet* sets; uint32_t n_sets;        // HBM
  Slice* slices; uint32_t n_slices;            // HBM
  uint64_t* free_slices;                       // HBM stack of (slot | last attempt generation << 32)
  unsigned long long* slot_ctr;                // HBM per-slot attempt counters (see kCtrClosed)
  unsigned long long* deadline;                // HBM per-slot posting deadline (see kDlMask)
  uint32_t* pending;                           // HBM [n_rails][n_slices]: decided, not yet posted
  uint64_t* pend_pos;                          // HBM [2][kMaxRails]: pending head / tail per rail
  WorkItem* work; uint64_t work_cap;           // HBM MPMC ring
  unsigned long long* work_head;               // HBM ticket counter (workers)
  uint64_t* comp; uint64_t comp_cap;           // HBM MPSC ring of packed completion words
  unsigned long long* comp_tail;               // HBM ticket counter (workers)
  uint32_t* parked; uint32_t parked_cap;       // HBM
  uint8_t* trace_ev; uint8_t* trace_dec; uint64_t trace_cap;  // HBM (spray_trace_event / spray_decision)
  uint64_t* persist;                           // HBM: scheduler scalars persisted across launches
  FaultDev* faults_hbm;                        // HBM mirror of the fault words (workers read)
  uint32_t* faults_any;                        // HBM: 1 while any fault word is active (HOSTRX)
  uint32_t* any_failed;                        // HBM: 1 once any batch failed (COMPLETE's cancel check)
  unsigned long long* next_free;               // HBM degrade FIFO server per rail
  uint32_t* exit_flag;                         // HBM: scheduler -> workers

  // scheduler constants (spray_sched_config / spray_resilience_config, device form)
  double tolerance, penalty[3], alpha, beta0_init, beta1_init, clamp;
  uint64_t reset_interval, min_slice;
  uint32_t max_slices, policy;
  int32_t failure_threshold, degradation_events, probe_successes;
  double degradation_ratio, degradation_min_t;
  uint32_t max_attempts;
  uint32_t has_ce;                             // poll the CE proxy completion ring
  uint32_t has_staged;                         // host-staged relays: poll their done rings
  uint64_t slice_timeout_ns;                   // ResilienceConfig::slice_timeout (0 = none)
  uint32_t fence_batch;                        // chunks a copy warp moves per system fence (1..4)
  uint32_t diag;                               // write the per-stage timeline words (Control::lat)
  uint32_t worker_fence_sys;                   // copy warps fence at system scope (else GPU scope)
  uint32_t copy_bulk;                          // copy warps use the bulk-copy (TMA) pipeline
  uint32_t fence_release;                      // system fences as fence.release.sys (b200.fence)
  uint32_t bulk_stages;                        // shared-memory stages per copy warp (2..7)
  uint64_t timeout_scan_ns;                    // deadline scan period of the TIMER warp
  uint64_t probe_interval, probe_bytes;        // resilience.hpp:23-26
  double probe_backoff_mult;
  int32_t probe_backoff_cap, pad_pb_;
  uint64_t scratch;                            // HBM probe scratch (2 x probe_bytes)
  uint64_t chunk_bytes;                        // SM work granule (power of two)
  uint32_t chunk_shift;                        // log2(chunk_bytes)
  uint32_t n_gates;                            // dataflow gates (0: none, the common case)
  uint64_t epoch;                              // globaltimer at engine time 0
  uint64_t gate_timeout_ns;                    // a consumer gives up on a granule after this
  GateDev gates[kMaxGates];
  TeleCell* tele;                              // HBM [n_rails][kTeleWindows] telemetry windows
  uint64_t window_ns;                          // telemetry window (stats_window_ms, default 10 ms)
  RelayDev relays[kMaxRelays];                 // relay rails (RailDesc::ce_index = relay index)
  uint32_t n_relays;
  uint32_t launch_gen;                         // bumped by the host on every launch
  double omega;                                // diffusion weight (0 unless a board is attached)
  BoardSlot* board;                            // mapped host: the load board (null = none)
  int64_t* board_hbm;                          // HBM: the adopted global view, kept across launches
  uint32_t board_slots, board_slot;
  uint64_t board_period;                       // publish period, ns (staleness = 3 periods)
  LaunchSnap snap;                             // control-block words at launch (host snapshot)
};

// scalars persisted in EngineDev::persist between launches
enum : int { kPRr = 0, kPWorkTail = 1, kPCompHead = 2, kPFreeTop = 3, kPParked = 4,
             kPLastReset = 5, kPOutChunks = 6, kPOutSlices = 7, kPSlotHwm = 8,
             kPResident = 9, kPNum = 16 };

}  // namespace spray_dev
