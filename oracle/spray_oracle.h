/*
 * spray_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's slice-spraying control arithmetic, used as
 * the CPU checker for the CUDA product path. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this. The product
 * (paper_2604_00368_b200/) never links, loads or calls it.
 *
 * Parity is pinned: tests/golden/ holds vectors produced by the reference itself
 * (oracle/_ref, built from /root/reference/proj/src by oracle/Makefile, driven by
 * oracle/ref_harness.cpp and tests/golden/make_golden.py) and the reference's own
 * known-answer tests (proj/tests/test_scheduler.cpp, test_backends.cpp,
 * test_resilience.cpp). Every function cites the reference lines it restates.
 *
 * FP64 operation order follows the reference exactly; compile with
 * -ffp-contract=off (the reference is built for baseline x86-64: no FMA).
 */
#ifndef SPRAY_ORACLE_H
#define SPRAY_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/spray_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SO_MAX_RAILS 256

/* common.hpp:81-97 */
uint64_t so_splitmix_next(uint64_t* state);
/* bench.cpp:59-67 fill_pattern */
void so_fill_pattern(uint8_t* p, uint64_t n, uint64_t seed);
/* common.hpp:101-120 */
uint64_t so_fnv1a64(const void* data, size_t len, uint64_t basis);
void so_hash128(const char* s, size_t len, uint64_t out[2]);
/* Position-keyed 64-bit checksum shared with the device (spray_checksum). */
uint64_t so_checksum(const uint8_t* p, uint64_t n);

/* scheduler.cpp:94-106. Returns the slice count; writes at most `cap` pieces. */
uint64_t so_decompose(uint64_t total, uint64_t min_slice, uint32_t max_slices, uint64_t* off,
                      uint64_t* len, uint64_t cap);

/* scheduler.cpp:34-61 SchedulerConfig::validate; 0 ok, -1 invalid. */
int so_sched_config_validate(const spray_sched_config* c);

typedef struct so_rail {       /* scheduler.hpp:158-168 RailCostState */
  double bandwidth;
  int base_tier;
  int64_t queued;
  double beta0, beta1, min_obs_s;
  int has_obs;
  uint64_t last_reset;
  int health;
} so_rail;

typedef struct so_res_rail {   /* resilience.hpp:68-76 RailRec */
  int consec_failures, degradation_count, backoff, probe_streak, probe_inflight;
  uint64_t next_probe, excluded_at;
} so_res_rail;

typedef struct so_pair { uint32_t remote; int32_t tier; int32_t affinity; } so_pair;
typedef struct so_cand { uint32_t local; uint32_t n_pairs; const so_pair* pairs; } so_cand;
typedef struct so_cset { uint32_t n; so_cand* cands; } so_cset;

typedef struct so_sched {
  spray_sched_config cfg;
  spray_resilience_config rcfg;
  uint32_t n_rails;
  so_rail rails[SO_MAX_RAILS];
  so_res_rail res[SO_MAX_RAILS];
  uint32_t id_rank[SO_MAX_RAILS];
  uint64_t rr_cursor;
  uint64_t exclusions;
  int64_t board_g[SO_MAX_RAILS];  /* GlobalLoadBoard::global_queued(rail) (BOARD events) */
} so_sched;

void so_sched_init(so_sched* s, const spray_sched_config* sc, const spray_resilience_config* rc,
                   uint32_t n_rails, const double* bw, const int32_t* tier, const uint32_t* id_rank);
double so_predict_completion_s(const so_sched* s, uint32_t rail, uint64_t len); /* 116-122 */
/* scheduler.cpp:124-136; returns index into pairs or -1 */
int so_map_remote(const so_sched* s, const so_pair* pairs, uint32_t n);
/* scheduler.cpp:138-195; returns 1 with *out filled, 0 = NoEligibleDevice */
int so_choose_rail(so_sched* s, uint64_t len, uint64_t offset, const so_cset* cs, spray_decision* out);
void so_charge(so_sched* s, uint32_t rail, uint64_t len);    /* 197-201 */
void so_release(so_sched* s, uint32_t rail, uint64_t len);   /* 203-209 */
void so_feedback(so_sched* s, uint32_t rail, double t_obs_s, double x_norm); /* 208-230 */
void so_periodic_reset(so_sched* s, uint64_t now);           /* 232-240 */
void so_reset_rail(so_sched* s, uint32_t rail, uint64_t now);/* 242-247 */
/* resilience.cpp:71-98 observe (exclusion at 137-148) */
void so_observe(so_sched* s, uint32_t local, uint32_t remote, int status, double t_obs_s,
                double predicted_s, uint64_t now);

/* resilience.cpp:100-121, 220-244 */
void so_observe_probe(so_sched* s, uint32_t rail, int status, uint64_t now);
void so_due_probes(so_sched* s, uint64_t now);

/* Parse a flattened candidate stream (spray_b200.h). Returns number of sets or -1.
 * Storage for cands/pairs is carved from the caller's arrays. */
int so_parse_candidates(const int32_t* stream, size_t len, so_cset* sets, uint32_t max_sets,
                        so_cand* cand_store, uint32_t max_cands, so_pair* pair_store,
                        uint32_t max_pairs);

/* Trace replay with the semantics documented in spray_b200.h. Returns 0 or -1 on a
 * malformed trace. */
int so_replay(so_sched* s, const so_cset* sets, uint32_t n_sets, const spray_trace_event* ev,
              size_t n, spray_decision* dec, size_t dcap, size_t* n_dec, uint64_t* expect_fail);

/* Convenience entry for ctypes: init + parse + replay in one call. */
int so_replay_flat(const spray_sched_config* sc, const spray_resilience_config* rc,
                   uint32_t n_rails, const double* bw, const int32_t* tier, const uint32_t* id_rank,
                   const int32_t* cand_stream, size_t cand_len, const spray_trace_event* ev,
                   size_t n, spray_decision* dec, size_t dcap, size_t* n_dec, uint64_t* expect_fail,
                   int64_t* queued_out, double* beta_out /* 2 per rail */, int32_t* health_out);

/* Incremental form (used by trace generators): a scheduler state that persists across
 * so_state_step calls. */
typedef struct so_state so_state;
so_state* so_state_new(const spray_sched_config* sc, const spray_resilience_config* rc,
                       uint32_t n_rails, const double* bw, const int32_t* tier, const uint32_t* id_rank,
                       const int32_t* cand_stream, size_t cand_len);
void so_state_free(so_state* st);
int so_state_step(so_state* st, const spray_trace_event* ev, size_t n, spray_decision* dec,
                  size_t dcap, size_t* n_dec, uint64_t* expect_fail, int64_t* queued_out,
                  double* beta_out, int32_t* health_out);

/* LatencyHistogram::bucket_for (telemetry.cpp:10-19) */
int so_hist_bucket(uint64_t t_ns);

/* sim_backend.cpp:83-93: modelled completion of one slice posted at `now` on a rail
 * free at `next_free` (no jitter, no faults) */
uint64_t so_sim_done_ns(uint64_t now, uint64_t next_free, uint64_t len, double bw,
                        double service_factor, double degrade, double latency_us);
/* sim_backend.cpp:104-112: bytes written by an attempt aborted by a down fault */
uint64_t so_sim_partial_bytes(uint64_t len, uint64_t start, uint64_t done, uint64_t down_start);

#ifdef __cplusplus
}
#endif
#endif
