/*
 * spray_oracle.c — TEST INFRASTRUCTURE ONLY (see spray_oracle.h).
 * Plain-C restatement of the reference control arithmetic; pinned by
 * tests/golden/ (reference outputs) and the reference's own KATs.
 */
#include "spray_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------- primitives */

/* common.hpp:84-89 Rng::next_u64 */
uint64_t so_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* bench.cpp:59-67 fill_pattern: 8-byte little-endian words, then one draw per tail byte */
void so_fill_pattern(uint8_t* p, uint64_t n, uint64_t seed) {
  uint64_t st = seed, i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t v = so_splitmix_next(&st);
    memcpy(p + i, &v, 8);
  }
  for (; i < n; ++i) p[i] = (uint8_t)so_splitmix_next(&st);
}

/* common.hpp:101-109 */
uint64_t so_fnv1a64(const void* data, size_t len, uint64_t basis) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = basis;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* common.hpp:117-120 */
void so_hash128(const char* s, size_t len, uint64_t out[2]) {
  out[0] = so_fnv1a64(s, len, 0xcbf29ce484222325ULL);
  out[1] = so_fnv1a64(s, len, 0x84222325cbf29ce4ULL);
}

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* checksum = sum_i mix64(w_i + (i+1)*golden) over little-endian 8-byte words, the
 * zero-padded tail word included; order-sensitive through the word index. */
uint64_t so_checksum(const uint8_t* p, uint64_t n) {
  uint64_t acc = 0, i = 0, w;
  for (; (i + 1) * 8 <= n; ++i) {
    memcpy(&w, p + i * 8, 8);
    acc += mix64(w + (i + 1) * 0x9e3779b97f4a7c15ULL);
  }
  if (i * 8 < n) {
    w = 0;
    memcpy(&w, p + i * 8, (size_t)(n - i * 8));
    acc += mix64(w + (i + 1) * 0x9e3779b97f4a7c15ULL);
  }
  return acc ^ n;
}

/* ------------------------------------------------------------- scheduler */

/* scheduler.cpp:94-106 */
uint64_t so_decompose(uint64_t total, uint64_t min_slice, uint32_t max_slices, uint64_t* off,
                      uint64_t* len, uint64_t cap) {
  if (total == 0) return 0;
  uint64_t n = total / min_slice;
  if (n == 0) n = 1;
  if (n > max_slices) n = max_slices;
  const uint64_t size = (total + n - 1) / n;
  uint64_t k = 0;
  for (uint64_t o = 0; o < total; o += size, ++k) {
    if (k < cap) {
      off[k] = o;
      len[k] = size < total - o ? size : total - o;
    }
  }
  return k;
}

static int pen_ok(const spray_sched_config* c, int tier) {
  return tier >= 1 && tier <= 3 && c->penalty[tier - 1] > 0.0;
}

/* scheduler.cpp:34-61 */
int so_sched_config_validate(const spray_sched_config* c) {
  if (c->min_slice_size < 4096) return -1;
  if (c->max_slices_per_transfer == 0) return -1;
  if (!(c->tolerance > 0.0)) return -1;
  if (c->ewma_alpha <= 0.0 || c->ewma_alpha > 1.0) return -1;
  if (c->diffusion_weight < 0.0 || c->diffusion_weight > 1.0) return -1; /* scheduler.cpp:39-40 */
  double prev = 0.0;
  for (int t = 1; t <= 3; ++t) {
    if (!pen_ok(c, t)) {
      for (int u = t + 1; u <= 3; ++u)
        if (pen_ok(c, u)) return -1;
      break;
    }
    if (c->penalty[t - 1] < prev) return -1;
    prev = c->penalty[t - 1];
  }
  return 0;
}

void so_sched_init(so_sched* s, const spray_sched_config* sc, const spray_resilience_config* rc,
                   uint32_t n_rails, const double* bw, const int32_t* tier, const uint32_t* id_rank) {
  memset(s, 0, sizeof(*s));
  s->cfg = *sc;
  if (rc) s->rcfg = *rc;
  s->n_rails = n_rails;
  for (uint32_t i = 0; i < n_rails; ++i) {
    s->rails[i].bandwidth = bw[i];
    s->rails[i].base_tier = tier[i];
    s->rails[i].beta0 = sc->beta0_init_s;   /* scheduler.cpp:87-90 */
    s->rails[i].beta1 = sc->beta1_init;
    s->rails[i].health = SPRAY_HEALTHY;
    s->id_rank[i] = id_rank ? id_rank[i] : i;
  }
}

/* scheduler.cpp:108-114 effective_queued: the local queue, blended with the board's
 * global view (the last BOARD event of the rail; 0 before the first) when omega > 0.
 * Trace semantics: omega > 0 means a board is attached. */
static double so_effective_queued(const so_sched* s, uint32_t rail) {
  const double local = (double)s->rails[rail].queued;
  if (!(s->cfg.diffusion_weight > 0.0)) return local;  /* omega > 0 <=> a board is attached */
  const double global = (double)s->board_g[rail];
  return (1.0 - s->cfg.diffusion_weight) * local + s->cfg.diffusion_weight * global;
}

/* scheduler.cpp:116-122 */
double so_predict_completion_s(const so_sched* s, uint32_t rail, uint64_t len) {
  const so_rail* st = &s->rails[rail];
  const double a = so_effective_queued(s, rail);
  return st->beta0 + st->beta1 * ((a + (double)len) / st->bandwidth);
}

/* scheduler.cpp:124-136 */
int so_map_remote(const so_sched* s, const so_pair* pairs, uint32_t n) {
  int best = -1;
  for (uint32_t i = 0; i < n; ++i) {
    const so_pair* p = &pairs[i];
    if (s->rails[p->remote].health != SPRAY_HEALTHY) continue;
    if (!pen_ok(&s->cfg, p->tier)) continue;
    if (p->affinity) return (int)i;
    if (best < 0 || p->tier < pairs[best].tier ||
        (p->tier == pairs[best].tier && s->id_rank[p->remote] < s->id_rank[pairs[best].remote]))
      best = (int)i;
  }
  return best;
}

/* scheduler.cpp:138-195 */
int so_choose_rail(so_sched* s, uint64_t len, uint64_t offset, const so_cset* cs, spray_decision* out) {
  struct scored { uint32_t local, remote; int tier; double score, predicted, x; };
  struct scored el[SO_MAX_RAILS];
  uint32_t ne = 0;
  for (uint32_t i = 0; i < cs->n; ++i) {
    const so_cand* c = &cs->cands[i];
    if (s->rails[c->local].health != SPRAY_HEALTHY) continue;
    int pi = so_map_remote(s, c->pairs, c->n_pairs);
    if (pi < 0) continue;
    const so_pair* p = &c->pairs[pi];
    if (!pen_ok(&s->cfg, p->tier)) continue;
    const double penalty = s->cfg.penalty[p->tier - 1];
    const so_rail* st = &s->rails[c->local];
    const double x = (so_effective_queued(s, c->local) + (double)len) / st->bandwidth;
    const double predicted = st->beta0 + st->beta1 * x;
    el[ne].local = c->local;
    el[ne].remote = p->remote;
    el[ne].tier = p->tier;
    el[ne].score = penalty * predicted;
    el[ne].predicted = predicted;
    el[ne].x = x;
    ++ne;
  }
  if (ne == 0) return 0;
  uint32_t pick = 0;
  if (s->cfg.policy == SPRAY_POLICY_TELEMETRY) {
    double s_min = el[0].score;
    for (uint32_t i = 0; i < ne; ++i) s_min = (el[i].score < s_min) ? el[i].score : s_min; /* std::min */
    uint32_t win[SO_MAX_RAILS], nw = 0;
    const double bound = (1.0 + s->cfg.tolerance) * s_min;
    for (uint32_t i = 0; i < ne; ++i)
      if (el[i].score <= bound) win[nw++] = i;
    pick = win[s->rr_cursor++ % nw];
  } else if (s->cfg.policy == SPRAY_POLICY_RR) {
    pick = (uint32_t)(s->rr_cursor++ % ne);
  } else {
    pick = (uint32_t)(mix64(offset) % ne);
  }
  s->rails[el[pick].local].queued += (int64_t)len;
  out->local = el[pick].local;
  out->remote = el[pick].remote;
  out->tier = el[pick].tier;
  out->ok = 1;
  out->predicted_s = el[pick].predicted;
  out->x_norm = el[pick].x;
  return 1;
}

void so_charge(so_sched* s, uint32_t rail, uint64_t len) { s->rails[rail].queued += (int64_t)len; }
void so_release(so_sched* s, uint32_t rail, uint64_t len) { s->rails[rail].queued -= (int64_t)len; }

/* std::max / std::min / std::clamp as libstdc++ 13 defines them */
static double cxx_max(double a, double b) { return (a < b) ? b : a; }
static double cxx_min(double a, double b) { return (b < a) ? b : a; }

/* scheduler.cpp:208-230 */
void so_feedback(so_sched* s, uint32_t rail, double t_obs_s, double x_norm) {
  if (x_norm <= 0.0) return;
  so_rail* st = &s->rails[rail];
  const double alpha = s->cfg.ewma_alpha;
  const double b0 = st->beta0;
  const double b1 = st->beta1;
  const double residual = cxx_max(0.0, t_obs_s - b1 * x_norm);
  double floor_obs = residual;
  if (st->has_obs) floor_obs = cxx_min(st->min_obs_s, residual);
  st->min_obs_s = floor_obs;
  st->has_obs = 1;
  st->beta0 = (1.0 - alpha) * b0 + alpha * floor_obs;
  double ratio = (t_obs_s - b0) / x_norm;
  const double lo = cxx_max(1e-9, b1 / s->cfg.feedback_clamp);
  const double hi = b1 * s->cfg.feedback_clamp;
  ratio = cxx_min(cxx_max(ratio, lo), hi);
  st->beta1 = (1.0 - alpha) * b1 + alpha * ratio;
}

/* scheduler.cpp:242-247 */
void so_reset_rail(so_sched* s, uint32_t rail, uint64_t now) {
  so_rail* st = &s->rails[rail];
  st->beta0 = s->cfg.beta0_init_s;
  st->beta1 = s->cfg.beta1_init;
  st->has_obs = 0;
  st->min_obs_s = 0.0;
  st->last_reset = now;
}

/* scheduler.cpp:232-240 */
void so_periodic_reset(so_sched* s, uint64_t now) {
  for (uint32_t i = 0; i < s->n_rails; ++i) {
    const uint64_t last = s->rails[i].last_reset;
    if (now >= last && now - last >= s->cfg.reset_interval_ns) so_reset_rail(s, i, now);
  }
}

/* ------------------------------------------------------------- resilience */

static uint64_t backoff_interval(const so_sched* s, int level) { /* resilience.cpp:123-127 */
  double mult = 1.0;
  for (int i = 0; i < level; ++i) mult *= s->rcfg.probe_backoff_mult;
  return (uint64_t)((double)s->rcfg.probe_interval_ns * mult);
}

static void so_exclude(so_sched* s, uint32_t rail, uint64_t now) { /* resilience.cpp:46-57 */
  if (s->rails[rail].health == SPRAY_EXCLUDED) return;
  s->rails[rail].health = SPRAY_EXCLUDED;
  so_res_rail* r = &s->res[rail];
  r->excluded_at = now;
  r->probe_streak = 0;
  r->backoff = 0;
  r->next_probe = now + backoff_interval(s, 0);
  s->exclusions++;
}

/* resilience.cpp:71-98 */
void so_observe(so_sched* s, uint32_t local, uint32_t remote, int status, double t_obs_s,
                double predicted_s, uint64_t now) {
  if (status != SPRAY_SLICE_OK) {
    uint32_t rr[2] = {local, remote};
    int n = (remote != 0xffffffffu && remote != local) ? 2 : 1;
    for (int k = 0; k < n; ++k) {
      uint32_t r = rr[k];
      if (s->rails[r].health != SPRAY_HEALTHY) continue;
      s->res[r].consec_failures++;
      if (s->res[r].consec_failures >= s->rcfg.failure_threshold) so_exclude(s, r, now);
    }
    return;
  }
  s->res[local].consec_failures = 0;
  if (remote != 0xffffffffu && remote != local) s->res[remote].consec_failures = 0;
  if (s->rails[local].health == SPRAY_HEALTHY && predicted_s > 0.0) {
    so_res_rail* rec = &s->res[local];
    if (t_obs_s >= s->rcfg.degradation_min_t_obs_s &&
        t_obs_s / predicted_s > s->rcfg.degradation_ratio) {
      rec->degradation_count++;
      if (rec->degradation_count >= s->rcfg.degradation_events) so_exclude(s, local, now);
    } else {
      rec->degradation_count = 0;
    }
  }
}

/* resilience.cpp:59-69 reintegrate */
static void so_reintegrate(so_sched* s, uint32_t rail, uint64_t now) {
  s->rails[rail].health = SPRAY_HEALTHY;
  so_reset_rail(s, rail, now);
  so_res_rail* r = &s->res[rail];
  r->consec_failures = 0;
  r->degradation_count = 0;
  r->probe_streak = 0;
  r->backoff = 0;
}

/* resilience.cpp:100-121 observe_probe */
void so_observe_probe(so_sched* s, uint32_t rail, int status, uint64_t now) {
  so_res_rail* r = &s->res[rail];
  r->probe_inflight = 0;
  if (s->rails[rail].health == SPRAY_HEALTHY) return;
  if (status == SPRAY_SLICE_OK) {
    r->probe_streak++;
    if (r->probe_streak >= s->rcfg.probe_successes_needed)
      so_reintegrate(s, rail, now);
    else
      r->next_probe = now;
  } else {
    if (s->rails[rail].health != SPRAY_EXCLUDED) s->rails[rail].health = SPRAY_EXCLUDED;
    r->probe_streak = 0;
    r->backoff = r->backoff + 1 < s->rcfg.probe_backoff_cap ? r->backoff + 1 : s->rcfg.probe_backoff_cap;
    r->next_probe = now + backoff_interval(s, r->backoff);
  }
}

/* resilience.cpp:129-153 due_probes (the partner choice does not touch scheduler state) */
void so_due_probes(so_sched* s, uint64_t now) {
  for (uint32_t i = 0; i < s->n_rails; ++i) {
    const int h = s->rails[i].health;
    if (h == SPRAY_HEALTHY) continue;
    if (s->res[i].probe_inflight) continue;
    if (s->res[i].next_probe > now) continue;
    s->res[i].probe_inflight = 1;
    if (h == SPRAY_EXCLUDED) s->rails[i].health = SPRAY_PROBING;
  }
}

/* ------------------------------------------------------------- replay */

int so_parse_candidates(const int32_t* st, size_t len, so_cset* sets, uint32_t max_sets,
                        so_cand* cs, uint32_t max_c, so_pair* ps, uint32_t max_p) {
  size_t i = 0;
  uint32_t nc = 0, np = 0;
  if (len < 1) return -1;
  const int32_t n_sets = st[i++];
  if (n_sets < 0 || (uint32_t)n_sets > max_sets) return -1;
  for (int32_t k = 0; k < n_sets; ++k) {
    if (i >= len) return -1;
    const int32_t nl = st[i++];
    if (nl < 0 || nc + (uint32_t)nl > max_c) return -1;
    sets[k].n = (uint32_t)nl;
    sets[k].cands = &cs[nc];
    for (int32_t l = 0; l < nl; ++l) {
      if (i + 2 > len) return -1;
      so_cand* c = &cs[nc++];
      c->local = (uint32_t)st[i++];
      const int32_t npair = st[i++];
      if (npair < 0 || np + (uint32_t)npair > max_p || i + 3 * (size_t)npair > len) return -1;
      c->n_pairs = (uint32_t)npair;
      c->pairs = &ps[np];
      for (int32_t q = 0; q < npair; ++q) {
        ps[np].remote = (uint32_t)st[i++];
        ps[np].tier = st[i++];
        ps[np].affinity = st[i++];
        ++np;
      }
    }
  }
  return n_sets;
}

static double to_seconds(uint64_t t) { return (double)t * 1e-9; } /* common.hpp:20 */

int so_replay(so_sched* s, const so_cset* sets, uint32_t n_sets, const spray_trace_event* ev,
              size_t n, spray_decision* dec, size_t dcap, size_t* n_dec, uint64_t* expect_fail) {
  size_t nd = 0;
  uint64_t bad = 0;
  for (size_t i = 0; i < n; ++i) {
    const spray_trace_event* e = &ev[i];
    switch (e->kind) {
      case SPRAY_EV_DECIDE: {
        spray_decision d;
        memset(&d, 0, sizeof d);
        if (e->rail >= n_sets) return -1;
        if (!so_choose_rail(s, e->len, e->offset, &sets[e->rail], &d)) {
          d.local = d.remote = 0xffffffffu;
          d.ok = 0;
        }
        if (nd < dcap) dec[nd] = d;
        ++nd;
        break;
      }
      case SPRAY_EV_COMPLETE: {
        const int status = (int)((e->flags >> 8) & 0xff);
        const double t_s = to_seconds(e->t_ns);
        so_release(s, e->rail, e->len);
        so_observe(s, e->rail, e->remote, status, t_s,
                   (e->flags & SPRAY_EVF_MODEL) ? e->predicted : 0.0, e->now_ns);
        if (status == SPRAY_SLICE_OK && (e->flags & SPRAY_EVF_MODEL) &&
            !(e->flags & SPRAY_EVF_CANCELLED) && e->x_norm > 0.0)
          so_feedback(s, e->rail, t_s, e->x_norm);
        break;
      }
      case SPRAY_EV_CHARGE: so_charge(s, e->rail, e->len); break;
      case SPRAY_EV_RELEASE: so_release(s, e->rail, e->len); break;
      case SPRAY_EV_HEALTH: s->rails[e->rail].health = (int)e->flags; break;
      case SPRAY_EV_RESET: so_periodic_reset(s, e->t_ns); break;
      case SPRAY_EV_RESET_RAIL: so_reset_rail(s, e->rail, e->t_ns); break;
      case SPRAY_EV_EXPECT_HEALTH:
        if (s->rails[e->rail].health != (int)e->flags) ++bad;
        break;
      case SPRAY_EV_DUE_PROBES: so_due_probes(s, e->t_ns); break;
      case SPRAY_EV_BOARD: s->board_g[e->rail] = (int64_t)e->len; break;
      case SPRAY_EV_PROBE_DONE:
        so_release(s, e->rail, e->len);
        so_observe_probe(s, e->rail, (int)((e->flags >> 8) & 0xff), e->now_ns);
        break;
      default: return -1;
    }
  }
  if (n_dec) *n_dec = nd;
  if (expect_fail) *expect_fail = bad;
  return 0;
}

#define SO_MAX_SETS 4096
#define SO_MAX_CANDS 65536
#define SO_MAX_PAIRS 262144

struct so_state {
  so_sched s;
  int n_sets;
  so_cset sets[SO_MAX_SETS];
  so_cand cands[SO_MAX_CANDS];
  so_pair pairs[SO_MAX_PAIRS];
};

so_state* so_state_new(const spray_sched_config* sc, const spray_resilience_config* rc,
                       uint32_t n_rails, const double* bw, const int32_t* tier, const uint32_t* id_rank,
                       const int32_t* cand_stream, size_t cand_len) {
  if (n_rails > SO_MAX_RAILS) return NULL;
  so_state* st = (so_state*)calloc(1, sizeof(so_state));
  if (!st) return NULL;
  so_sched_init(&st->s, sc, rc, n_rails, bw, tier, id_rank);
  st->n_sets = so_parse_candidates(cand_stream, cand_len, st->sets, SO_MAX_SETS, st->cands,
                                   SO_MAX_CANDS, st->pairs, SO_MAX_PAIRS);
  if (st->n_sets < 0) {
    free(st);
    return NULL;
  }
  return st;
}

void so_state_free(so_state* st) { free(st); }

int so_state_step(so_state* st, const spray_trace_event* ev, size_t n, spray_decision* dec,
                  size_t dcap, size_t* n_dec, uint64_t* expect_fail, int64_t* queued_out,
                  double* beta_out, int32_t* health_out) {
  int rc2 = so_replay(&st->s, st->sets, (uint32_t)st->n_sets, ev, n, dec, dcap, n_dec, expect_fail);
  for (uint32_t i = 0; i < st->s.n_rails; ++i) {
    if (queued_out) queued_out[i] = st->s.rails[i].queued;
    if (beta_out) {
      beta_out[2 * i] = st->s.rails[i].beta0;
      beta_out[2 * i + 1] = st->s.rails[i].beta1;
    }
    if (health_out) health_out[i] = st->s.rails[i].health;
  }
  return rc2;
}

int so_replay_flat(const spray_sched_config* sc, const spray_resilience_config* rc,
                   uint32_t n_rails, const double* bw, const int32_t* tier, const uint32_t* id_rank,
                   const int32_t* cand_stream, size_t cand_len, const spray_trace_event* ev,
                   size_t n, spray_decision* dec, size_t dcap, size_t* n_dec, uint64_t* expect_fail,
                   int64_t* queued_out, double* beta_out, int32_t* health_out) {
  so_state* st = so_state_new(sc, rc, n_rails, bw, tier, id_rank, cand_stream, cand_len);
  if (!st) return -1;
  int r = so_state_step(st, ev, n, dec, dcap, n_dec, expect_fail, queued_out, beta_out, health_out);
  so_state_free(st);
  return r;
}

/* ------------------------------------------------------------- telemetry / sim */

/* telemetry.cpp:10-19 */
int so_hist_bucket(uint64_t t) {
  const uint64_t us = t / 1000;
  if (us < 2) return 0;
  const int k = 63 - __builtin_clzll(us);
  const uint64_t kSqrt2 = 0xb504f333f9de6485ULL;
  const int b = 2 * k + ((us << (63 - k)) >= kSqrt2 ? 1 : 0);
  return b < 48 ? b : 47;
}

static uint64_t from_seconds(double s) { return (uint64_t)(s * 1e9); } /* common.hpp:21 */

/* sim_backend.cpp:83-93 */
uint64_t so_sim_done_ns(uint64_t now, uint64_t next_free, uint64_t len, double bw,
                        double service_factor, double degrade, double latency_us) {
  const uint64_t start = now > next_free ? now : next_free;
  double factor = service_factor;
  factor *= degrade;
  const double service_s = (double)len / (bw * factor);
  return start + from_seconds(latency_us * 1e-6) + from_seconds(service_s) + from_seconds(0.0 * 1e-6);
}

/* sim_backend.cpp:104-112 */
uint64_t so_sim_partial_bytes(uint64_t len, uint64_t start, uint64_t done, uint64_t down_start) {
  if (down_start <= start) return 0;
  const double frac = (double)(down_start - start) / (double)(done - start);
  return (uint64_t)((double)len * frac);
}
