/*
 * spray_b200.h — C-ABI of the B200-native slice-spraying data plane.
 *
 * Two entry surfaces, both plain C (no C++ types, no torch types, no exceptions):
 *
 *  1. ENGINE (fused mode). The application-facing declarative intent API of the
 *     reference `spray::Engine` (proj/include/spray/engine.hpp:90-131), with slice
 *     decomposition, rail choice, copy execution, completion accounting and
 *     self-healing all running inside one persistent sm_100a kernel per GPU.
 *
 *  2. BACKEND (plugin mode). The reference's fabric plugin boundary
 *     `spray::TransportBackend` (proj/include/spray/backend.hpp:49-72): a CUDA
 *     transport the reference engine would instantiate by name in
 *     `Engine::load_backends` (proj/src/engine.cpp:116-140) and drive slice by slice.
 *
 * plus the replay entry used for slice-plan parity (the device decision function run
 * over a recorded telemetry trace, proj/src/scheduler.cpp:138-230 semantics).
 *
 * Error model (reference: proj/include/spray/common.hpp:31-41, engine.hpp:28-31,
 * orchestrator.hpp:20-23): API-contract violations return a negative SPRAY_E* code
 * naming the reference exception class; `spray_last_error()` holds the message
 * (thread-local). Datapath faults never produce an error code: they surface only as
 * batch state, exactly like the reference.
 */
#ifndef SPRAY_B200_H
#define SPRAY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPRAY_ABI_VERSION 1u

/* ------------------------------------------------------------------ errors */
enum spray_status {
  SPRAY_OK = 0,
  SPRAY_ECONFIG = -1,       /* spray::ConfigError        (common.hpp:33-36) */
  SPRAY_EENGINE = -2,       /* spray::EngineError        (common.hpp:38-41) */
  SPRAY_EINVALID_RANGE = -3,/* spray::InvalidRangeError  (engine.hpp:28-31) */
  SPRAY_ENOROUTE = -4,      /* spray::NoRouteError       (orchestrator.hpp:20-23) */
  SPRAY_ECUDA = -5,         /* CUDA runtime failure (no reference analogue; never a fallback) */
  SPRAY_EFATAL = -6,        /* PostResult.fatal (backend.hpp:44-47): backend latched fatal */
  SPRAY_ECAPABILITY = -7    /* capability mismatch: a programming error (backend.hpp:56-57) */
};

/* Message of the last failing call on this thread ("" when none). */
const char* spray_last_error(void);
uint32_t spray_abi_version(void);

/* ------------------------------------------------------------------ enums */
/* spray::Direction (common.hpp:27) */
enum spray_direction { SPRAY_READ = 0, SPRAY_WRITE = 1 };
/* spray::Medium (common.hpp:29). DEVICE is real HBM here, not emulated. */
enum spray_medium { SPRAY_MEDIUM_HOST = 0, SPRAY_MEDIUM_DEVICE = 1, SPRAY_MEDIUM_FILE = 2 };
/* spray::SliceStatus (backend.hpp:29) */
enum spray_slice_status { SPRAY_SLICE_OK = 0, SPRAY_SLICE_FAILED = 1, SPRAY_SLICE_TIMEOUT = 2 };
/* spray::BatchState (engine.hpp:35) */
enum spray_batch_state { SPRAY_BATCH_IN_FLIGHT = 0, SPRAY_BATCH_COMPLETE = 1, SPRAY_BATCH_FAILED = 2 };
/* spray::RailHealthState (scheduler.hpp:63) */
enum spray_health { SPRAY_HEALTHY = 0, SPRAY_EXCLUDED = 1, SPRAY_PROBING = 2 };
/* spray::Policy (scheduler.hpp:23) */
enum spray_policy { SPRAY_POLICY_TELEMETRY = 0, SPRAY_POLICY_RR = 1, SPRAY_POLICY_HASH = 2 };
/* spray::FaultEffect (backend.hpp:74) */
enum spray_fault_effect {
  SPRAY_FAULT_DOWN = 0, SPRAY_FAULT_DEGRADE = 1, SPRAY_FAULT_JITTER = 2, SPRAY_FAULT_DROP_COMPLETION = 3
};
/* How a rail's bytes move on B200 (no reference analogue: the reference's rails are
 * simulated). Chosen per rail by the topology document's "executor" key. */
enum spray_executor {
  SPRAY_EXEC_SM = 0,     /* SM warps, 128-bit ld/st over UVA: local HBM, NVLink peer, mapped host */
  SPRAY_EXEC_CE = 1,     /* copy engine: cudaMemcpyAsync on a side stream, driven by a host proxy */
  SPRAY_EXEC_RELAY = 2   /* 2-hop through an intermediate GPU's staging buffer */
};

/* ------------------------------------------------------------------ engine types */
/* spray::BufferDesc (fabric.hpp:128-132). `data` is a device pointer for DEVICE
 * segments and a pinned host pointer (cudaHostAlloc / cudaHostRegister) for HOST. */
typedef struct spray_buffer_desc {
  uint64_t offset;
  uint64_t length;
  void* data;
} spray_buffer_desc;

/* spray::SegmentDescriptor (fabric.hpp:134-141). */
typedef struct spray_segment_desc {
  const char* id;
  int32_t medium;            /* enum spray_medium */
  const char* node;
  const spray_buffer_desc* buffers;
  uint32_t n_buffers;
  const char* device;        /* optional explicit topology device binding ("" or NULL = first of kind) */
} spray_segment_desc;

/* spray::TransferRequest (engine.hpp:73-80). */
typedef struct spray_transfer_request {
  const char* src_segment;
  uint64_t src_offset;
  const char* dst_segment;
  uint64_t dst_offset;
  uint64_t length;
  int32_t direction;         /* enum spray_direction */
} spray_transfer_request;

/* spray::BatchStatus (engine.hpp:39-43). */
typedef struct spray_batch_status {
  int32_t state;             /* enum spray_batch_state */
  uint64_t remaining;
  char failure_reason[64];
} spray_batch_status_t;

/* Per-rail counters (telemetry.hpp:53-61 RailStatsView, without windows). */
typedef struct spray_rail_stats {
  uint64_t bytes_posted;
  uint64_t bytes_ok;
  uint64_t bytes_failed;
  int64_t queue_depth;       /* scheduler queued bytes A_d */
  double beta0, beta1;       /* cost-model state (scheduler.hpp:158-168) */
  int32_t health;            /* enum spray_health */
  uint32_t latency_hist[48]; /* LatencyHistogram buckets (telemetry.hpp:23-35) */
} spray_rail_stats;

typedef struct spray_engine spray_engine;

/* Engine(EngineOptions) (engine.cpp:71-112). `config_json` is the documented engine
 * config document (README "Engine config document"; unknown keys rejected,
 * engine.cpp:1186-1197) and may be NULL for defaults; `topology_json` is the
 * topology document (fabric.cpp:157-210) extended with per-rail "executor",
 * "gpu" and "via" keys. `device` is the CUDA ordinal this engine drives. */
int spray_engine_create(const char* config_json, const char* topology_json, int device,
                        spray_engine** out);
void spray_engine_destroy(spray_engine* e);
int spray_engine_start(spray_engine* e);    /* Engine::start (engine.cpp:142-154) */
int spray_engine_stop(spray_engine* e);     /* Engine::stop  (engine.cpp:156-163) */

/* Engine::register_segment (engine.cpp:222-224 -> fabric.cpp:261-304). */
int spray_register_segment(spray_engine* e, const spray_segment_desc* desc);

/* Engine::allocate_batch / submit_transfer / batch_status / free_batch / await_batch
 * (engine.cpp:228-332, 1141-1158). submit returns before any data moves. */
int spray_allocate_batch(spray_engine* e, uint64_t* batch_out);
int spray_submit_transfer(spray_engine* e, uint64_t batch, const spray_transfer_request* req,
                          uint64_t* transfer_id_out);
/* Vectorised submit: n calls of submit_transfer in order, one lock acquisition and
 * one publication to the device submission ring. Stops at the first failing
 * request; *n_done says how many were accepted. */
int spray_submit_transfers(spray_engine* e, uint64_t batch, const spray_transfer_request* reqs,
                           size_t n, uint64_t* transfer_ids_out, size_t* n_done);
int spray_batch_status(spray_engine* e, uint64_t batch, spray_batch_status_t* out);
int spray_await_batch(spray_engine* e, uint64_t batch, uint64_t limit_ns, spray_batch_status_t* out);
int spray_free_batch(spray_engine* e, uint64_t batch);
/* Batch latency through the calls above, as a C++ caller sees it (bench.cpp:156-157,
 * 213-215: submit -> batch terminal): n_batches rounds of allocate / submit_transfers
 * (per_batch requests, cycling through reqs) / await / free, one batch in flight;
 * lat_ns[i] = the round's steady-clock nanoseconds. Measurement helper, not data path. */
int spray_batch_latency(spray_engine* e, const spray_transfer_request* reqs, size_t n_reqs, size_t per_batch,
                        size_t n_batches, uint64_t* lat_ns);

/* Introspection. */
int spray_rail_count(spray_engine* e, uint32_t* n);
int spray_rail_id(spray_engine* e, uint32_t rail, char* buf, size_t cap);
int spray_rail_stats_get(spray_engine* e, uint32_t rail, spray_rail_stats* out);
/* bytes_dispatched / bytes_terminated (engine.hpp:127-128): equal at quiescence. */
int spray_engine_counters(spray_engine* e, uint64_t* bytes_dispatched, uint64_t* bytes_terminated,
                          uint64_t* batches_failed);

/* FaultSchedule entry (backend.hpp:74-94) applied to the live device fabric.
 * Times are engine-relative nanoseconds (spray_engine_now_ns). A DOWN fault aborts
 * in-flight slices with a partial prefix write and fails new ones
 * (sim_backend.cpp:100-112 semantics). */
int spray_inject_fault(spray_engine* e, const char* rail_id, int32_t effect, uint64_t start_ns,
                       uint64_t end_ns, double factor);
/* spray::FaultEntry (backend.hpp:79-86) in full: effect DOWN / DEGRADE (factor in (0, 1]) /
 * JITTER (uniform added delay in [0, jitter_us) per copy unit, sim_backend.cpp:52-63) /
 * DROP_COMPLETION (the bytes land, the completion is lost; the attempt times out after
 * resilience.slice_timeout_ms and is retried, engine.cpp:996-1022). An entry replaces the
 * rail's previous entry of the same effect (FaultSchedule::validate forbids overlaps per
 * (rail, effect)). spray_inject_fault(e, r, JITTER, s, t, f) is this call with jitter_us = f. */
typedef struct spray_fault_entry {
  const char* rail_id;
  int32_t effect;            /* enum spray_fault_effect */
  uint64_t start_ns, end_ns; /* engine clock (spray_engine_now_ns) */
  double factor;             /* degrade: effective bandwidth multiplier */
  double jitter_us;          /* jitter: added uniform delay bound */
} spray_fault_entry;
int spray_inject_fault_entry(spray_engine* e, const spray_fault_entry* entry);
int spray_clear_faults(spray_engine* e);
uint64_t spray_engine_now_ns(spray_engine* e);

/* Diagnostic snapshot (ring positions, kernel state, counters, stream status). Word map
 * (engine.cpp Engine::debug_words): 0-16 host/ring positions, state, device clock, byte
 * counters, trace count, stream status, scheduler loop counters; 17-32 STATE phase clocks;
 * 33-36 CE / completion ring positions; 37-44 per-launch timeline; 45-60 diagnostic words
 * (b200.diag: relay tickets, host-staged drain and forwarder timings); 61 launch
 * generation; 62-69 pipeline stage stamps; 70-77 copy-warp stamps; 78-85 decision-phase
 * split; 86-93 FEEDBACK chain and decision-path counters; 94-101 STATE sub-step stamps. */
int spray_engine_debug(spray_engine* e, uint64_t* out, size_t n);

/* Heal timing of the most recent DOWN fault: fault start -> first retried slice OK,
 * in device-clock nanoseconds (0 when not observed). */
int spray_heal_stats(spray_engine* e, uint64_t* fault_start_ns, uint64_t* first_reroute_ok_ns,
                     uint64_t* failed_attempts, uint64_t* retried_ok);

/* Dataflow gates: how a GPU re-emits slices it received (relay paths, broadcast chains;
 * the exchange step of SURVEY.md §8(e)). `flags` is one uint32 counter per chunk_bytes
 * granule of the (single-buffer) segment, in device memory reachable from this GPU and
 * shared by the producing and the consuming engine (zero-initialised by the caller).
 *   PRODUCE (2): a slice this engine writes into the segment advances the counters of
 *                its granules when it completes OK (after a system fence).
 *   CONSUME (1): this engine's copies out of the segment wait, granule by granule,
 *                until the producer has delivered it (gate_timeout_ms, then the attempt
 *                fails and is retried). Offsets and slice sizes on a gated segment must
 *                be multiples of chunk_bytes. SM rails only. Register while idle. */
enum { SPRAY_GATE_CONSUME = 1, SPRAY_GATE_PRODUCE = 2 };
int spray_gate_segment(spray_engine* e, const char* segment_id, int role, void* flags);
/* Ring gate: the staged route's bounded staging pool (reference engine.hpp:56-58, 4 MiB
 * chunks x depth 4 per 64 MiB pool; staged_* in engine.cpp:465-610). The segment's single
 * buffer (offset 0, a multiple of chunk_bytes) is a ring; intents address a logical window
 * of `logical_bytes` that wraps onto it (lap = offset / ring bytes), so a transfer of any
 * size streams through a fixed pool, one transfer per intent at most the ring's size.
 * `flags` as above; `credits` is one uint32 per granule (zeroed, reachable by both engines):
 *   CONSUME: a read of lap k waits for flags >= k + 1; completing OK adds 1 to credits.
 *   PRODUCE: a write of lap k waits for credits >= k (the consumer drained lap k - 1).
 * Direct SM rails only. Register while idle. logical_bytes == 0 -> SPRAY_ECONFIG. */
int spray_gate_ring(spray_engine* e, const char* segment_id, int role, void* flags, void* credits,
                    uint64_t logical_bytes);
int spray_engine_chunk_bytes(spray_engine* e, uint64_t* out);

/* TelemetrySnapshot::to_csv (telemetry.cpp:123-158): one row per (window, rail),
 * columns window_start_ms,rail_id,bytes_ok,bytes_failed,queue_depth_bytes,p50_us,p99_us,
 * health_state,throughput_gbps, from the device's per-rail window cells (the last 1024
 * windows of stats_window_ms, default 10 ms). Writes at most cap-1 bytes + NUL; *len gets
 * the full length. */
int spray_telemetry_csv(spray_engine* e, char* buf, size_t cap, size_t* len);

/* Device-resident submission (intents built once, kept in HBM, reused by many batches).
 * prepare: validates and plans every request exactly like submit_transfer and stages the
 * resulting intents in HBM. run: submits them all into `batch` as one bulk record and
 * runs the engine kernel in drain mode: one launch, bracketed by CUDA events on the
 * engine's stream, that exits when the batch is delivered; *kernel_ms is its duration.
 * Any running launch of the engine is stopped first. */
typedef struct spray_prepared spray_prepared;
int spray_prepare_transfers(spray_engine* e, const spray_transfer_request* reqs, size_t n,
                            spray_prepared** out);
int spray_run_prepared(spray_engine* e, uint64_t batch, spray_prepared* p, float* kernel_ms);
void spray_prepared_free(spray_prepared* p);

/* Multi-process peer segments: export a device pointer as an IPC handle and open a peer's
 * handle in this process (the returned pointer can be registered as a DEVICE segment on
 * the peer's node). The handle is the CUDA IPC handle of the allocation that contains
 * `ptr` (64 B) followed by ptr's byte offset inside it (8 B, little endian): pointers
 * handed out by sub-allocating pools (e.g. PyTorch's caching allocator) map to the same
 * bytes in the importing process. spray_ipc_close takes the pointer spray_ipc_open
 * returned. */
#define SPRAY_IPC_HANDLE_BYTES 72
int spray_ipc_export(int device, void* ptr, uint8_t handle_out[SPRAY_IPC_HANDLE_BYTES]);
int spray_ipc_open(int device, const uint8_t handle[SPRAY_IPC_HANDLE_BYTES], void** ptr_out);
int spray_ipc_close(void* ptr);

/* GlobalLoadBoard (scheduler.hpp:66-90, scheduler.cpp:63-79): engines publish their
 * per-rail queued bytes into slots of a shared board every `period_ns` (control phase,
 * engine.cpp:1090-1093), and blend the board's fresh entries (heartbeat within 3 periods)
 * into their effective queue with scheduler.diffusion_weight. The board is caller-owned,
 * zeroed host memory of spray_board_bytes(n_slots) bytes (pinned or pageable: the engine
 * maps it; share it across processes with shared memory); `slot` is this engine's
 * instance. Heartbeats are GPU global-timer nanoseconds, common to the GPUs of a host.
 * Attach while no batch is in flight. */
size_t spray_board_bytes(uint32_t n_slots);
int spray_engine_attach_board(spray_engine* e, void* board, uint32_t n_slots, uint32_t slot, uint64_t period_ns);

/* Host planning only (no GPU work): the candidate stream of the route the engine would
 * use for src -> dst (orchestrator.cpp:98-245 + 39-81), and the backend serving it. */
int spray_plan_candidates(spray_engine* e, const char* src_segment, const char* dst_segment,
                          int32_t direction, int32_t* stream, size_t cap, size_t* len,
                          char* backend, size_t backend_cap);

/* ------------------------------------------------------------------ trace / replay */
/* One scheduler-state event. A live engine records, in the exact order its device
 * scheduler applied them, every event that changes cost-model or health state; the
 * same stream replayed through the reference SliceScheduler/ResilienceManager (or the
 * oracle) must reproduce every decision bit for bit. Semantics per kind:
 *   DECIDE(set=rail, len, offset)       choose_rail(len, offset, candidate set)       (scheduler.cpp:138-195)
 *   COMPLETE(local=rail, remote, len, status, t_ns, flags, predicted, x_norm, now=aux)
 *        release(local,len); observe(local, remote, status, to_seconds(t_ns),
 *        flags&MODEL ? predicted : 0, now); if status==OK && flags&MODEL && !(flags&CANCELLED)
 *        && x_norm>0: feedback(local, to_seconds(t_ns), x_norm)          (engine.cpp:792-851)
 *   CHARGE(rail, len) / RELEASE(rail, len)                                (scheduler.cpp:197-206)
 *   HEALTH(rail, state=flags)          set_health                          (scheduler.hpp:136-138)
 *   RESET(now=t_ns)                    periodic_reset(now)                 (scheduler.cpp:232-240)
 *   RESET_RAIL(rail, now=t_ns)         reset_rail                          (scheduler.cpp:242-247)
 *   EXPECT_HEALTH(rail, state=flags)   assertion: health(rail) == state
 *   DUE_PROBES(now=t_ns)               due_probes(now): excluded rails whose timer
 *                                      elapsed go to PROBING       (resilience.cpp:129-153)
 *   PROBE_DONE(rail, len, status, now=now_ns)  release(rail,len); observe_probe(rail,
 *                                      status, now)                (resilience.cpp:100-121)
 *   BOARD(rail, len=(int64) global queued bytes, now=now_ns)  the load board's
 *                                      global_queued(rail) seen by every later
 *                                      effective_queued(rail) until the next BOARD event
 *                                      of the rail (scheduler.cpp:63-79, 108-114, 249-254)
 */
enum spray_trace_kind {
  SPRAY_EV_DECIDE = 1, SPRAY_EV_COMPLETE = 2, SPRAY_EV_CHARGE = 3, SPRAY_EV_RELEASE = 4,
  SPRAY_EV_HEALTH = 5, SPRAY_EV_RESET = 6, SPRAY_EV_RESET_RAIL = 7, SPRAY_EV_EXPECT_HEALTH = 8,
  SPRAY_EV_DUE_PROBES = 9, SPRAY_EV_PROBE_DONE = 10, SPRAY_EV_BOARD = 11
};
#define SPRAY_EVF_MODEL 0x1u
#define SPRAY_EVF_CANCELLED 0x2u

typedef struct spray_trace_event {  /* 64 bytes */
  uint32_t kind;
  uint32_t rail;      /* DECIDE: candidate-set index; else the (local) rail */
  uint32_t remote;    /* COMPLETE: remote rail (0xffffffff = none) */
  uint32_t flags;     /* COMPLETE: SPRAY_EVF_* | status << 8; HEALTH/EXPECT_HEALTH: the state */
  uint64_t len;
  uint64_t offset;    /* DECIDE: offset fed to the hash policy */
  uint64_t t_ns;      /* COMPLETE: observed time since the decision; RESET/RESET_RAIL: now */
  uint64_t now_ns;    /* COMPLETE: engine clock when the completion was applied */
  double predicted;   /* COMPLETE: t_hat at dispatch */
  double x_norm;      /* COMPLETE: x at dispatch */
} spray_trace_event;

/* spray::DispatchChoice (scheduler.hpp:98-104) plus an eligibility flag. */
typedef struct spray_decision {  /* 32 bytes */
  uint32_t local;
  uint32_t remote;
  int32_t tier;
  uint32_t ok;        /* 0 = NoEligibleDevice (choose_rail returned nullopt) */
  double predicted_s;
  double x_norm;
} spray_decision;

/* Scheduler constants (spray::SchedulerConfig, scheduler.hpp:44-60). A tier penalty
 * <= 0 encodes the reference's disengaged optional (tier unschedulable). */
typedef struct spray_sched_config {
  uint64_t min_slice_size;
  uint32_t max_slices_per_transfer;
  int32_t policy;            /* enum spray_policy */
  double tolerance;
  double penalty[3];         /* tiers 1..3 */
  double ewma_alpha;
  uint64_t reset_interval_ns;
  double beta0_init_s;
  double beta1_init;
  double feedback_clamp;
  double diffusion_weight;   /* omega (scheduler.hpp:51): blend of the global load board;
                                0 disables it, as does the absence of a board */
} spray_sched_config;

/* Resilience constants (spray::ResilienceConfig, resilience.hpp:17-31). */
typedef struct spray_resilience_config {
  int32_t failure_threshold;
  int32_t degradation_events;
  double degradation_ratio;
  double degradation_min_t_obs_s;
  int32_t probe_successes_needed;
  int32_t probe_backoff_cap;
  uint64_t probe_bytes;
  uint64_t probe_interval_ns;
  double probe_backoff_mult;
  uint32_t max_attempts;
  uint32_t pad_;
  uint64_t slice_timeout_ns;
} spray_resilience_config;

void spray_sched_config_default(spray_sched_config* c);
void spray_resilience_config_default(spray_resilience_config* c);

/* Candidate sets are flattened int32 streams:
 *   [n_sets, { n_locals, { local, n_pairs, { remote, tier, affinity }* }* }*]
 * in exactly the order orient_candidates produces (orchestrator.cpp:39-81). */

/* Runs the DEVICE decision function (the same code the live engine's scheduler warp
 * executes) over `events`, on GPU `device`. Rails are described by bandwidth, base
 * tier and the rank of their id string in sorted order (map_remote's id tie-break,
 * scheduler.cpp:124-136). decisions_out gets one entry per DECIDE event;
 * *expect_failures counts EXPECT_HEALTH mismatches. */
int spray_replay_device(int device, const spray_sched_config* sc, const spray_resilience_config* rc,
                        uint32_t n_rails, const double* bandwidth, const int32_t* base_tier,
                        const uint32_t* id_rank, const int32_t* cand_stream, size_t cand_len,
                        const spray_trace_event* events, size_t n_events,
                        spray_decision* decisions_out, size_t decisions_cap, size_t* n_decisions,
                        uint64_t* expect_failures);

/* Recorded live trace of an engine (events in application order + the decisions the
 * device made for each DECIDE), and the candidate sets those events index. */
int spray_trace_enable(spray_engine* e, size_t capacity_events);
int spray_trace_fetch(spray_engine* e, spray_trace_event* events, size_t cap, size_t* n_events,
                      spray_decision* decisions, size_t dcap, size_t* n_decisions);
int spray_trace_candidates(spray_engine* e, int32_t* stream, size_t cap, size_t* len);

/* ------------------------------------------------------------------ backend (plugin) */
/* spray::SliceWorkRequest (backend.hpp:15-27) as an 88-byte POD: segment ids become
 * their Hash128 (common.hpp:111-120), as on the reference TCP wire. */
typedef struct spray_slice_wr {  /* 88 bytes */
  uint64_t slice;
  uint64_t batch;
  uint64_t src_seg_lo, src_seg_hi;
  uint64_t src_offset;
  uint64_t dst_seg_lo, dst_seg_hi;
  uint64_t dst_offset;   /* absolute; re-execution is byte-idempotent (backend.hpp:21) */
  uint64_t length;
  int32_t direction;     /* enum spray_direction */
  uint32_t local_rail;
  uint32_t remote_rail;
  uint32_t attempt;
} spray_slice_wr;

/* spray::CompletionEvent (backend.hpp:33-40). */
typedef struct spray_cqe {  /* 40 bytes */
  uint64_t slice;
  uint64_t batch;
  int32_t status;     /* enum spray_slice_status */
  uint32_t rail;
  uint64_t t_obs_ns;
  uint64_t bytes;
} spray_cqe;

/* spray::BackendCapabilities (fabric.hpp:207-221). */
typedef struct spray_backend_caps {
  char id[32];
  uint32_t media_pairs_mask;  /* bit (src*3+dst) set when (src,dst) medium pair is covered */
  uint8_t supports_read, supports_write, cross_node, same_node;
  uint64_t max_post_size;
  uint8_t batched_posting;
  uint8_t pad_[7];
} spray_backend_caps;

typedef struct spray_backend spray_backend;

int spray_backend_open(int device, spray_backend** out);
void spray_backend_close(spray_backend* b);
int spray_backend_start(spray_backend* b);                 /* TransportBackend::start */
int spray_backend_stop(spray_backend* b);                  /* TransportBackend::stop  */
int spray_backend_capabilities(spray_backend* b, spray_backend_caps* out);
/* attach_segment_metadata (backend.hpp:65-68): registers (id hash -> buffers). Returns
 * SPRAY_OK and writes a metadata blob, or SPRAY_ECAPABILITY when the medium is not served. */
int spray_backend_attach_segment(spray_backend* b, const spray_segment_desc* desc,
                                 uint8_t* blob_out, size_t blob_cap, size_t* blob_len);
/* post_slices (backend.hpp:55-58): accepted = prefix count; a rejected suffix is
 * backpressure. Returns SPRAY_EFATAL with *accepted = 0 once latched fatal. */
int spray_backend_post(spray_backend* b, const spray_slice_wr* reqs, size_t n, size_t* accepted);
/* poll_completions (backend.hpp:60-61): never blocks; single consumer. */
int spray_backend_poll(spray_backend* b, spray_cqe* out, size_t max, size_t* n);
int spray_backend_fatal(spray_backend* b);                 /* 1 when latched */
int spray_backend_latch_fatal(spray_backend* b);           /* MemoryBackend::latch_fatal analogue */

/* ------------------------------------------------------------------ utilities */
/* Device-side splitmix64 fill matching the reference payload generator
 * (common.hpp:81-97 driven as in bench.cpp:59-67): byte i of the stream is byte
 * (i mod 8) of the (i/8)-th next_u64() of Rng(seed), tail bytes take the low byte of
 * one further draw each. Works on device or mapped-host pointers. */
int spray_fill_splitmix(int device, void* ptr, uint64_t n, uint64_t seed);
/* 64-bit order-sensitive checksum computed on the GPU: sum over little-endian 8-byte
 * words w_i (zero-padded tail) of splitmix64_mix(w_i + (i+1)*0x9e3779b97f4a7c15), xor n.
 * Identical to the oracle's so_checksum. */
int spray_checksum(int device, const void* ptr, uint64_t n, uint64_t* out);
/* Pinned, device-mapped host allocation (cudaHostAlloc Portable|Mapped). */
int spray_host_alloc(uint64_t n, void** out);
int spray_host_free(void* p);
/* NUMA node of a GPU's PCIe root (-1 when the host reports none). */
int spray_device_numa_node(int device, int32_t* node);
/* Pinned, device-mapped host memory placed on `device`'s NUMA node (mbind + first touch,
 * then cudaHostRegister Mapped|Portable): the pinned-host staging pool of one PCIe root.
 * *node_out = the node the pages are bound to (-1: not bound, first-touch placement). */
int spray_host_alloc_numa(int device, uint64_t n, void** out, int32_t* node_out);
int spray_host_free_numa(void* p);

/* State-blind striping baseline (the Policy::kRoundRobin analog a25,
 * scheduler.cpp:175-177): copy n (src[i], dst[i], len[i]) ranges with one
 * cudaMemcpyAsync each, round-robin over `streams` copy streams on `device`, then
 * synchronize. Writes the wall time in milliseconds. Not part of the drop-in path. */
int spray_rr_copy(int device, const uint64_t* src, const uint64_t* dst, const uint64_t* len, size_t n,
                  int streams, double* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* SPRAY_B200_H */
