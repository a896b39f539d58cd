"""The C oracle (oracle/spray_oracle.c) pinned against the reference: golden vectors
recorded from the reference library (tests/golden/, made by make_golden.py) and the
reference's own known-answer tests (proj/tests/test_scheduler.cpp, test_backends.cpp,
test_telemetry.cpp). CPU only."""
import os

import numpy as np
import pytest

from oracle.oracle import (EVENT_DTYPE, EV_BOARD, EV_CHARGE, EV_COMPLETE, EV_DECIDE, EV_EXPECT, EV_HEALTH, EV_RELEASE,
                           EV_RESET, EVF_MODEL, CState, ResConfig, SchedConfig, ref_available, res_config,
                           sched_config)


def ev(kind, rail=0, **kw):
    e = np.zeros(1, EVENT_DTYPE)
    e["kind"] = kind
    e["rail"] = rail
    for k, v in kw.items():
        e[k] = v
    return e


def cat(*evs):
    return np.concatenate(evs)


def one_set(locals_pairs):
    """[(local, [(remote, tier, aff), ...]), ...] -> single-set candidate stream."""
    out = [1, len(locals_pairs)]
    for l, pairs in locals_pairs:
        out += [l, len(pairs)]
        for r, t, a in pairs:
            out += [r, t, a]
    return np.array(out, np.int32)


# ------------------------------------------------------------------ decompose
def test_decompose_kats(co):
    # test_scheduler.cpp:62-98
    off, ln = co.decompose(1 << 20)
    assert len(off) == 16 and (ln == 65536).all()
    off, ln = co.decompose(10 * 1024)
    assert len(off) == 1 and off[0] == 0 and ln[0] == 10 * 1024
    off, ln = co.decompose(1 << 30)
    assert len(off) == 4096 and (ln == 262144).all()
    rng = np.random.default_rng(11)
    for total in rng.integers(1, 1 << 28, 300):
        off, ln = co.decompose(int(total))
        assert 1 <= len(off) <= 4096
        assert off[0] == 0 and int(ln.sum()) == total
        assert (off[1:] == np.cumsum(ln)[:-1]).all()
        if len(off) > 1:
            assert (ln[:-1] >= 65536).all()
    assert co.decompose(0)[0].size == 0


def test_decompose_golden(co, golden_dir):
    rows = np.load(os.path.join(golden_dir, "decompose.npy"))
    for total, mn, mx, n, first, last, last_off in rows:
        off, ln = co.decompose(int(total), int(mn), int(mx))
        assert (len(off), int(ln[0]), int(ln[-1]), int(off[-1])) == (n, first, last, last_off)


# ------------------------------------------------------------------ replay vs reference goldens
def _cases(golden_dir):
    z = np.load(os.path.join(golden_dir, "replay.npz"))
    return z, sorted({k.split("__")[0] for k in z.files})


def test_replay_matches_reference_goldens(co, golden_dir):
    z, cases = _cases(golden_dir)
    assert len(cases) >= 20
    n_dec = n_excl = 0
    for c in cases:
        sc = SchedConfig.from_buffer_copy(z[c + "__sc"].tobytes())
        rc = ResConfig.from_buffer_copy(z[c + "__rc"].tobytes())
        out = co.replay(sc, rc, z[c + "__bw"], z[c + "__tier"], z[c + "__rank"], z[c + "__stream"],
                        z[c + "__events"])
        assert out["decisions"].tobytes() == z[c + "__decisions"].tobytes(), c
        assert (out["queued"] == z[c + "__queued"]).all(), c
        assert out["beta"].tobytes() == z[c + "__beta"].tobytes(), c
        assert (out["health"] == z[c + "__health"]).all(), c
        assert out["expect_failures"] == int(z[c + "__expect_failures"]) == 0, c
        n_dec += len(out["decisions"])
        n_excl += int((z[c + "__health"] != 0).sum())
    assert n_dec > 15000


def test_c1_plan_golden(co, golden_dir):
    """Config 1: 64 MiB over 2 sim rails per node decides 1024 x 64 KiB slices that
    alternate a.r0->b.r0 / a.r1->b.r1 (512 each), exactly as the reference."""
    z = np.load(os.path.join(golden_dir, "c1.npz"))
    off, ln = co.decompose(64 << 20)
    events = np.zeros(len(off), EVENT_DTYPE)
    events["kind"] = EV_DECIDE
    events["len"] = ln
    events["offset"] = off
    out = co.replay(sched_config(), res_config(), [1e9] * 4, [1] * 4, [0, 1, 2, 3], z["stream"], events)
    g = z["decisions"]
    assert out["decisions"].tobytes() == g.tobytes()
    assert np.bincount(g["local"]).tolist() == [512, 512]
    assert (g["local"][::2] == 0).all() and (g["local"][1::2] == 1).all()


# ------------------------------------------------------------------ scheduler KATs (test_scheduler.cpp)
def _two_rail(tier2=True):
    # local rails 0 (tier 1) and 1 (tier 2 or 1), remotes 2 and 3, bandwidth 100
    stream = one_set([(0, [(2, 1, 1)]), (1, [(3, 2 if tier2 else 1, 1)])])
    return [100.0] * 4, [1, 2 if tier2 else 1, 1, 2 if tier2 else 1], [0, 1, 2, 3], stream


def test_tier1_preferred_at_equal_load(co):
    bw, tier, rank, stream = _two_rail()
    out = co.replay(sched_config(), res_config(), bw, tier, rank, stream, ev(EV_DECIDE, 0, len=10))
    assert out["decisions"][0]["local"] == 0 and out["queued"][0] == 10


def test_spillover_to_idle_tier2(co):
    bw, tier, rank, stream = _two_rail()
    out = co.replay(sched_config(), res_config(), bw, tier, rank, stream,
                    cat(ev(EV_CHARGE, 0, len=500), ev(EV_DECIDE, 0, len=100)))
    assert out["decisions"][0]["local"] == 1


def test_no_eligible_device(co):
    bw, tier, rank, stream = _two_rail()
    out = co.replay(sched_config(), res_config(), bw, tier, rank, stream,
                    cat(ev(EV_HEALTH, 0, flags=1), ev(EV_HEALTH, 1, flags=1), ev(EV_DECIDE, 0, len=10)))
    assert out["decisions"][0]["ok"] == 0


def test_round_robin_alternation(co):
    bw, tier, rank, stream = _two_rail(tier2=False)
    evs = []
    for _ in range(4):
        evs += [ev(EV_DECIDE, 0, len=10)]
    dec = []
    st = CState(co, sched_config(), res_config(), bw, tier, rank, stream)
    for e in evs:
        d, q, *_ = st.step(e)
        dec.append(int(d[0]["local"]))
        st.step(ev(EV_RELEASE, dec[-1], len=10))
    assert dec[0] != dec[1] and dec[0] == dec[2] and dec[1] == dec[3]


def test_spillover_grid_matches_brute_force(co):
    # test_scheduler.cpp:218-243: tier-2 chosen exactly when A1 + L > P2 (A2 + L)
    bw, tier, rank, stream = _two_rail()
    sc = sched_config(tolerance=1e-9)
    for a1 in range(0, 2001, 100):
        for a2 in range(0, 601, 37):
            out = co.replay(sc, res_config(), bw, tier, rank, stream,
                            cat(ev(EV_CHARGE, 0, len=a1), ev(EV_CHARGE, 1, len=a2), ev(EV_DECIDE, 0, len=64)))
            s1, s2 = a1 + 64, 3.0 * (a2 + 64)
            if s1 != s2:
                assert out["decisions"][0]["local"] == (1 if s2 < s1 else 0)


def test_window_invariant_10k(co):
    # acceptance.cpp:149-215: chosen score <= (1 + gamma) * min score
    rng = np.random.default_rng(7)
    bw = [5e8 + 2.5e8 * i for i in range(8)] + [1e9] * 8
    tier = [1 if i < 4 else 2 for i in range(8)] + [1] * 8
    stream = one_set([(i, [(8 + i, tier[i], 1)]) for i in range(8)])
    st = CState(co, sched_config(), res_config(), bw, tier, list(range(16)), stream)
    q = np.zeros(8, np.int64)
    for n in range(2000):
        for i in range(8):
            want = int(rng.integers(0, 1 << 22))
            if want > q[i]:
                st.step(ev(EV_CHARGE, i, len=want - int(q[i])))
            else:
                st.step(ev(EV_RELEASE, i, len=int(q[i]) - want))
            q[i] = want
        L = int(rng.integers(1, 1 << 20))
        d, queued, beta, *_ = st.step(ev(EV_DECIDE, 0, len=L, offset=L))
        pick = int(d[0]["local"])
        scores = []
        for i in range(8):
            qq = float(queued[i]) - (L if i == pick else 0)
            t = beta[i][0] + beta[i][1] * ((qq + L) / bw[i])
            scores.append((1.0 if tier[i] == 1 else 3.0) * t)
        assert scores[pick] <= 1.05 * min(scores) * (1 + 1e-12)
        q[pick] += L


def test_ewma_kats(co):
    # test_scheduler.cpp:277-307 (rail 0, B = 1000)
    stream = one_set([(0, [(1, 1, 1)])])
    bw, tier, rank = [1000.0, 1000.0], [1, 1], [0, 1]
    x = 0.1

    def complete(t_s):
        return cat(ev(EV_CHARGE, 0, len=100),
                   ev(EV_COMPLETE, 0, remote=1, len=100, flags=EVF_MODEL, t_ns=int(round(t_s * 1e9)), x_norm=x,
                      predicted=x))
    fixed = co.replay(sched_config(), res_config(), bw, tier, rank, stream, cat(*[complete(x) for _ in range(50)]))
    assert abs(fixed["beta"][0][1] - 1.0) < 0.05
    deg = co.replay(sched_config(), res_config(degradation_ratio=1e9), bw, tier, rank, stream,
                    cat(*[complete(4 * x) for _ in range(20)]))
    b0, b1 = deg["beta"][0]
    assert abs((b0 + b1 * 0.1) - 0.4) <= 0.1 * 0.4
    base = co.replay(sched_config(), res_config(), bw, tier, rank, stream, cat(*[complete(x) for _ in range(30)]))
    out = co.replay(sched_config(), res_config(), bw, tier, rank, stream,
                    cat(*([complete(x) for _ in range(30)] + [complete(10 * x)])))
    before = base["beta"][0][0] + base["beta"][0][1] * 0.1
    after = out["beta"][0][0] + out["beta"][0][1] * 0.1
    assert before < after <= 2.0 * before


def test_periodic_reset(co):
    # test_scheduler.cpp:309-328
    stream = one_set([(0, [(1, 1, 1)])])
    comp = [cat(ev(EV_CHARGE, 0, len=100),
                ev(EV_COMPLETE, 0, remote=1, len=100, flags=EVF_MODEL, t_ns=400_000_000, x_norm=0.1, predicted=0.1))
            for _ in range(10)]
    base = cat(ev(EV_CHARGE, 0, len=777), *comp)
    before = co.replay(sched_config(), res_config(degradation_ratio=1e9), [1000.0] * 2, [1, 1], [0, 1], stream,
                       cat(base, ev(EV_RESET, t_ns=10_000_000_000)))
    assert before["beta"][0][1] > 1.5
    after = co.replay(sched_config(), res_config(degradation_ratio=1e9), [1000.0] * 2, [1, 1], [0, 1], stream,
                      cat(base, ev(EV_RESET, t_ns=30_000_000_000)))
    assert after["beta"][0][1] == 1.0 and after["beta"][0][0] == 0.0 and after["queued"][0] == 777


def test_resilience_exclusion_kats(co):
    # test_resilience.cpp:46-77: 3 consecutive failures exclude both ends; 8 slow OKs
    stream = one_set([(0, [(1, 1, 1)])])

    def fail():
        return cat(ev(EV_CHARGE, 0, len=10), ev(EV_COMPLETE, 0, remote=1, len=10, flags=(1 << 8), t_ns=1000))
    out = co.replay(sched_config(), res_config(), [1e9] * 2, [1, 1], [0, 1], stream,
                    cat(fail(), fail(), ev(EV_EXPECT, 0, flags=0), fail(), ev(EV_EXPECT, 0, flags=1),
                        ev(EV_EXPECT, 1, flags=1)))
    assert out["expect_failures"] == 0

    def slow():  # t_obs 10 ms vs predicted 1 ms: ratio 10 > 4
        return cat(ev(EV_CHARGE, 0, len=10),
                   ev(EV_COMPLETE, 0, remote=1, len=10, flags=EVF_MODEL, t_ns=10_000_000, predicted=1e-3, x_norm=1e-3))
    out = co.replay(sched_config(), res_config(), [1e9] * 2, [1, 1], [0, 1], stream,
                    cat(*[slow() for _ in range(7)], ev(EV_EXPECT, 0, flags=0), slow(), ev(EV_EXPECT, 0, flags=1)))
    assert out["expect_failures"] == 0


def test_config_validation(co):
    import ctypes as C
    ok = sched_config()
    assert co.lib.so_sched_config_validate(C.byref(ok)) == 0
    for kw in (dict(min_slice=1024), dict(alpha=0.0), dict(tolerance=0.0), dict(penalties=(1.0, 0.0, 5.0))):
        assert co.lib.so_sched_config_validate(C.byref(sched_config(**kw))) == -1


# ------------------------------------------------------------------ sim backend / telemetry KATs
def test_sim_service_kats(co, golden_dir):
    # test_backends.cpp:95-120: 1 MiB at 2^30 B/s + 10 us = 986562 ns; degrade 0.25 -> 3906250 + latency
    assert co.lib.so_sim_done_ns(0, 0, 1 << 20, float(1 << 30), 1.0, 1.0, 10.0) == 986562
    for ln, deg_milli, done in np.load(os.path.join(golden_dir, "sim.npy")):
        assert co.lib.so_sim_done_ns(0, 0, int(ln), float(1 << 30), 1.0, deg_milli / 1000.0, 10.0) == done


def test_partial_write_prefix(co):
    # sim_backend.cpp:104-112: bytes proportional to progress before the down start
    assert co.lib.so_sim_partial_bytes(1000, 0, 1000, 250) == 250
    assert co.lib.so_sim_partial_bytes(1000, 100, 1100, 50) == 0


def test_histogram_buckets(co):
    # telemetry.cpp:10-19 / test_telemetry.cpp:33-41
    assert co.lib.so_hist_bucket(0) == 0 and co.lib.so_hist_bucket(1999) == 0
    assert co.lib.so_hist_bucket(2000) == 2
    assert co.lib.so_hist_bucket(3000) == 3
    assert co.lib.so_hist_bucket(1 << 60) == 47


def test_fill_pattern_is_reference_rng(co):
    a = co.fill(19, 42)
    st = [42]

    def nxt():
        st[0] = (st[0] + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = st[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)
    exp = list(nxt().to_bytes(8, "little")) + list(nxt().to_bytes(8, "little")) + [nxt() & 0xFF for _ in range(3)]
    assert a.tolist() == exp


def test_checksum_is_order_sensitive(co):
    a = co.fill(4099, 3)
    b = a.copy()
    b[[0, 8]] = b[[8, 0]]
    assert co.checksum(a) != co.checksum(b)
    assert co.checksum(a) == co.checksum(a.copy())


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_c_oracle_vs_reference_fresh_traces(co):
    """Fresh random traces (not the committed ones) through both checkers."""
    import spraygen
    from oracle.oracle import RefOracle, caps
    ref = RefOracle()
    rng = np.random.default_rng(99)
    for _ in range(6):
        topo = spraygen.random_doc(rng)
        sc = sched_config(policy=int(rng.integers(0, 3)))
        rc = res_config()
        bw, tier, rank, _ids = ref.rails(topo)
        try:
            s = ref.candidates(topo, [caps("sim", **spraygen.SIM_CAPS)], ("a", 0, ""), ("b", 0, ""), 1, sc)[0]
        except RuntimeError:
            continue
        stream = spraygen.stream_concat([s])
        events = spraygen.random_trace(rng, CState(co, sc, rc, bw, tier, rank, stream), 1, len(bw), bw, 800)
        a = ref.replay(topo, sc, rc, stream, events, len(bw))
        b = co.replay(sc, rc, bw, tier, rank, stream, events)
        assert a["decisions"].tobytes() == b["decisions"].tobytes()
        assert a["beta"].tobytes() == b["beta"].tobytes()


# ------------------------------------------------------------------ global load board
def test_load_board_blends_into_effective_queue(co):
    """test_scheduler.cpp:389-403: another instance reports rail 0 loaded (100000 B), so
    with omega 0.5 the decision steers to rail 1; without the board (omega 0) it does not.
    The BOARD event carries global_queued(rail) = own published + others."""
    bw, tier, rank, stream = _two_rail(tier2=False)
    bw = [1000.0] * 4
    trace = cat(ev(EV_BOARD, 0, len=100000), ev(EV_BOARD, 1, len=0), ev(EV_DECIDE, 0, len=100))
    on = co.replay(sched_config(omega=0.5), res_config(), bw, tier, rank, stream, trace)
    off = co.replay(sched_config(omega=0.0), res_config(), bw, tier, rank, stream, trace)
    assert on["decisions"][0]["local"] == 1
    assert off["decisions"][0]["local"] == 0
    # x = ((1 - w) * local + w * global + L) / B for the picked rail (global 0 there)
    assert on["decisions"][0]["x_norm"] == (0.5 * 0.0 + 0.5 * 0.0 + 100.0) / 1000.0
    if ref_available():
        import spraygen
        from oracle.oracle import RefOracle
        ref = RefOracle()
        topo = spraygen.two_node_doc(2, 1000.0)
        a = ref.replay(topo, sched_config(omega=0.5), res_config(), stream, trace, 4)
        assert a["decisions"].tobytes() == on["decisions"].tobytes()


def test_load_board_golden_cases_depend_on_the_board(co, golden_dir):
    """The omega > 0 goldens are not vacuous: for a board refresh, replaying the prefix
    that ends with the decisions after it, with that one refresh's global queues zeroed,
    decides differently. (Before that refresh both replays see the same board, so each
    prefix stays a consistent trace.)"""
    z, cases = _cases(golden_dir)
    n_board = n_diff = 0
    for c in cases:
        sc = SchedConfig.from_buffer_copy(z[c + "__sc"].tobytes())
        if not sc.diffusion_weight > 0:
            continue
        n_board += 1
        ev_ = z[c + "__events"]
        rc = ResConfig.from_buffer_copy(z[c + "__rc"].tobytes())
        args = (z[c + "__bw"], z[c + "__tier"], z[c + "__rank"], z[c + "__stream"])
        kinds = ev_["kind"]
        starts = [i for i in np.nonzero(kinds == EV_BOARD)[0] if i == 0 or kinds[i - 1] != EV_BOARD]
        for b in starts:
            k = int(b)
            while k < len(ev_) and kinds[k] == EV_BOARD:
                k += 1
            end = k
            while end < len(ev_) and kinds[end] in (EV_DECIDE, EV_CHARGE, EV_RELEASE):
                end += 1
            pre = ev_[:end].copy()
            on = co.replay(sc, rc, *args, pre)
            assert on["decisions"].tobytes() == z[c + "__decisions"][:len(on["decisions"])].tobytes()
            pre["len"][b:k] = 0
            off = co.replay(sc, rc, *args, pre)
            if off["decisions"].tobytes() != on["decisions"].tobytes():
                n_diff += 1
                break
    assert n_board >= 6 and n_diff >= n_board - 1
