"""Host logic of the product through its C-ABI (no GPU work): symbol exports, route
planning vs reference goldens, configuration/registration errors mirroring the
reference's exception classes."""
import json
import os
import re

import numpy as np
import pytest

import paper_2604_00368_b200 as sp
from paper_2604_00368_b200 import _lib, fabrics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "spray_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(spray_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) > 40
    for n in sorted(names):
        assert hasattr(_lib.lib, n), n
    assert set(_lib.EXPORTED) <= names
    assert _lib.lib.spray_abi_version() == 1


def _engine(topo, cfg):
    e = sp.Engine(topo, json.dumps(cfg))
    e.register_segment(sp.SegmentDescriptor("src", sp.Medium.HOST, "a", [sp.BufferDesc(0, 1 << 20, 0x1000)]))
    e.register_segment(sp.SegmentDescriptor("dst", sp.Medium.HOST, "b", [sp.BufferDesc(0, 1 << 20, 0x2000)]))
    return e


@pytest.mark.parametrize("fabric", ["uniform8", "skewed8", "tiered"])
@pytest.mark.parametrize("backend", ["sim", "memory"])
@pytest.mark.parametrize("direction", [0, 1])
def test_plan_candidates_match_reference(golden_dir, fabric, backend, direction):
    z = np.load(os.path.join(golden_dir, "orchestrator.npz"))
    topo = z[f"doc_{fabric}"].tobytes().decode()
    golden = z[f"{fabric}_X_{direction}_X_{'sim' if backend == 'sim' else 'mem'}"]
    e = _engine(topo, {"backends": [backend]})
    if golden[0] == -1:
        with pytest.raises(sp.NoRouteError):
            e.plan_candidates("src", "dst", sp.Direction(direction))
    else:
        s, b = e.plan_candidates("src", "dst", sp.Direction(direction))
        assert b == backend
        assert np.array_equal(s, golden)


def test_c1_candidates_match_reference(golden_dir):
    z = np.load(os.path.join(golden_dir, "c1.npz"))
    topo = z["topo"].tobytes().decode()
    e = _engine(topo, {"backends": ["sim"]})
    s, _ = e.plan_candidates("src", "dst")
    assert np.array_equal(s, z["stream"])


def test_kv_fabric_routes_host_only_over_pcie_rails():
    topo = fabrics.kv_offload(0, sm_rails=2, ce_rails=1)
    e = sp.Engine(topo, None)
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, 1 << 20, 0x1000)]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, "g0", [sp.BufferDesc(0, 1 << 20, 0x2000)]))
    s, b = e.plan_candidates("hbm", "host")
    assert b == "cuda"
    assert s[1] == 3  # three locals, each paired with itself (same node)
    assert {e.rail_id(i) for i in range(e.rail_count())} == {"g0.pcie0", "g0.pcie1", "g0.ce0"}


@pytest.mark.parametrize("cfg,msg", [
    ({"bogus": 1}, "unknown key"),
    ({"scheduler": {"tolerance": 0}}, "tolerance"),
    ({"scheduler": {"ewma_alpha": 0}}, "alpha"),
    ({"scheduler": {"min_slice_size": 1024}}, "min slice"),
    ({"scheduler": {"tier2_penalty": None, "tier3_penalty": 5}}, "non-decreasing"),
    ({"scheduler": {"policy": "nope"}}, "policy"),
    ({"resilience": {"failure_threshold": 0}}, "failure threshold"),
    ({"clock": "virtual"}, "clock"),
    ({"b200": {"chunk_bytes": 12345}}, "power of two"),
    ({"scheduler": {"diffusion_weight": 1.5}}, "diffusion"),  # scheduler.cpp:39-40
])
def test_config_errors(cfg, msg):
    with pytest.raises(sp.ConfigError, match=msg):
        sp.Engine(fabrics.two_node(2), json.dumps(cfg))


@pytest.mark.parametrize("doc,msg", [
    ({"nodes": [{"id": "a"}], "rails": [{"id": "r", "node": "a", "bandwidth_bytes_per_sec": 0, "affinity": "direct"}]},
     "NonPositiveBandwidth"),
    ({"nodes": [{"id": "a"}], "rails": [{"id": "r", "node": "x", "bandwidth_bytes_per_sec": 1, "affinity": "direct"}]},
     "dangling node"),
    ({"nodes": [{"id": "a"}], "rails": [{"id": "r", "node": "a", "bandwidth_bytes_per_sec": 1, "affinity": "direct"},
                                         {"id": "r", "node": "a", "bandwidth_bytes_per_sec": 1, "affinity": "direct"}]},
     "duplicate rail"),
    ({"nodes": [{"id": "a"}]}, "missing required"),
    ({"nodes": [{"id": "a"}], "rails": [{"id": "r", "node": "a", "bandwidth_bytes_per_sec": 1, "affinity": "far"}]},
     "affinity"),
])
def test_topology_errors(doc, msg):
    with pytest.raises(sp.ConfigError, match=msg):
        sp.Engine(json.dumps(doc), None)


def test_segment_registration_errors():
    e = sp.Engine(fabrics.two_node(2), None)
    ok = sp.SegmentDescriptor("s", sp.Medium.HOST, "a", [sp.BufferDesc(0, 100, 0x1000)])
    e.register_segment(ok)
    with pytest.raises(sp.ConfigError, match="duplicate"):
        e.register_segment(ok)
    with pytest.raises(sp.ConfigError, match="OverlappingBuffers"):
        e.register_segment(sp.SegmentDescriptor("o", sp.Medium.HOST, "a",
                                                [sp.BufferDesc(0, 100, 0x1000), sp.BufferDesc(50, 100, 0x3000)]))
    with pytest.raises(sp.ConfigError, match="zero-length"):
        e.register_segment(sp.SegmentDescriptor("z", sp.Medium.HOST, "a", [sp.BufferDesc(0, 0, 0x1000)]))
    with pytest.raises(sp.ConfigError, match="unknown node"):
        e.register_segment(sp.SegmentDescriptor("n", sp.Medium.HOST, "zz", [sp.BufferDesc(0, 10, 0x1000)]))
    with pytest.raises(sp.ConfigError, match="no buffers"):
        e.register_segment(sp.SegmentDescriptor("n2", sp.Medium.HOST, "a", []))


def test_api_contract_before_start():
    e = sp.Engine(fabrics.two_node(2), None)
    with pytest.raises(sp.EngineError, match="not started"):
        e.allocate_batch()


def test_hash128_matches_reference_construction():
    from oracle.oracle import COracle
    import ctypes as C
    co = COracle()
    out = (C.c_uint64 * 2)()
    co.lib.so_hash128(b"kv/block0", 9, out)
    assert sp.hash128("kv/block0") == (out[0], out[1])


def test_relay_rails_plan_as_spillover_tier():
    """2-hop relay rails (executor "relay", via GPU K) are ordinary rails to the planner:
    the direct SM pair first (tier 1), the relay pair behind it at tier 2 (the reference's
    spillover tier, P = 3), like with like by position (orchestrator.cpp:59-67)."""
    topo = fabrics.peer_fabric([0, 1], sm_rails=1, relay_via=[2])
    e = sp.Engine(topo, json.dumps({}))
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, 1 << 20, 0x1000)]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, 1 << 20, 0x2000)]))
    s, b = e.plan_candidates("s", "d")
    ids = {e.rail_id(r): r for r in range(e.rail_count())}
    # stream: 1 set, n locals, then per local: rail, n pairs, (remote, tier, affinity)...
    n_loc = s[1]
    locs, k = {}, 2
    for _ in range(n_loc):
        rail, npair = s[k], s[k + 1]
        locs[rail] = [tuple(s[k + 2 + 3 * p:k + 5 + 3 * p]) for p in range(npair)]
        k += 2 + 3 * npair
    assert set(locs) == {ids["g0.nvl0"], ids["g0.rl2"]}
    tiers = {r: {p[0]: p[1] for p in v} for r, v in locs.items()}
    assert tiers[ids["g0.rl2"]][ids["g1.rl2"]] == 2
    assert tiers[ids["g0.nvl0"]][ids["g1.nvl0"]] == 1


def test_relay_rail_without_via_is_a_config_error():
    topo = json.loads(fabrics.peer_fabric([0, 1], sm_rails=1, relay_via=[2]))
    for r in topo["rails"]:
        r.pop("via", None)
    with pytest.raises(sp.ConfigError):
        sp.Engine(json.dumps(topo), json.dumps({}))


def _locals(e, s):
    locs, k = [], 2
    for _ in range(s[1]):
        locs.append(e.rail_id(s[k]))
        k += 2 + 3 * s[k + 1]
    return locs


def test_staged_route_synthesized_for_gpu_without_peer_access():
    """Staged-route synthesis (orchestrator.cpp:120-234): with GPU 1 lacking peer access
    (b200.no_peer), the engine on GPU 0 declares a host-staged relay rail pair towards it
    and routes g0 -> g1 over that rail alone; a host destination keeps the direct rails
    (staged only where no direct route exists); a transfer starting on GPU 1 has no route
    from this engine."""
    topo = fabrics.peer_fabric([0, 1], sm_rails=1)
    e = sp.Engine(topo, json.dumps({"b200": {"no_peer": [1]}}), 0)
    ids = [e.rail_id(r) for r in range(e.rail_count())]
    assert "g0.st1" in ids and "g1.st1" in ids
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, 1 << 20, 0x1000)]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, 1 << 20, 0x2000)]))
    e.register_segment(sp.SegmentDescriptor("h", sp.Medium.HOST, "g0", [sp.BufferDesc(0, 1 << 20, 0x3000)]))
    s, _ = e.plan_candidates("s", "d")
    assert _locals(e, s) == ["g0.st1"]
    s, _ = e.plan_candidates("s", "h")
    assert "g0.st1" not in _locals(e, s) and "g0.nvl0" in _locals(e, s)
    with pytest.raises(sp.NoRouteError):
        e.plan_candidates("d", "s")


def test_staged_routes_off_leaves_no_route():
    topo = fabrics.peer_fabric([0, 1], sm_rails=1)
    e = sp.Engine(topo, json.dumps({"b200": {"no_peer": [1], "staged_routes": False}}), 0)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, 1 << 20, 0x1000)]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, 1 << 20, 0x2000)]))
    with pytest.raises(sp.NoRouteError):
        e.plan_candidates("s", "d")


def test_host_staging_is_for_relay_rails():
    topo = json.loads(fabrics.peer_fabric([0, 1], sm_rails=1))
    topo["rails"][0]["staging"] = "host"
    with pytest.raises(sp.ConfigError):
        sp.Engine(json.dumps(topo), json.dumps({}))
