"""Canonical B200 fabric documents, in the reference's topology format
(proj/src/fabric.cpp:157-210) plus the per-rail "executor" key.

Appendix-A mapping: node = GPU ordinal (with its host memory), rail = a
physical path declared with its bandwidth B_d and tier. The same rail-id set is declared
on every GPU so the 1:1 affinity pairing (orchestrator.cpp:59-67) pairs like with like.
"""
from __future__ import annotations

import json
from typing import Dict, List, Optional

PCIE5_X16 = 55e9      # measured pinned H2D/D2H on this pool's B200 (cudaMemcpy, 256 MiB)
NVLINK5 = 770e9       # measured peer copy per direction (B200_PROFILING.md)
HBM_COPY = 3.2e12     # delivered bytes/s of a local HBM->HBM copy (measured peak / 2)


def _node(g: int, host: bool = True) -> Dict:
    devs = [{"id": f"g{g}.hbm", "kind": "device_memory"}]
    if host:
        devs.append({"id": f"g{g}.host", "kind": "host_memory"})
    return {"id": f"g{g}", "devices": devs}


def kv_offload(gpu: int = 0, sm_rails: int = 1, ce_rails: int = 0, bw_sm: float = PCIE5_X16,
               bw_ce: float = PCIE5_X16, relay_via: Optional[List[int]] = None, bw_relay: float = PCIE5_X16) -> str:
    """HiCache-style KV offload on one GPU (config 3): HBM <-> pinned host over the GPU's
    PCIe root. Host memory links only to the PCIe rails; HBM links to all. `relay_via` adds
    one 2-hop rail per listed GPU K (g.rlK): hop 1 over NVLink into K's HBM, hop 2 by K's
    SMs over K's own PCIe root, so the host staging spans several roots."""
    rails, links = [], []
    for v in relay_via or []:
        rails.append({"id": f"g{gpu}.rl{v}", "node": f"g{gpu}", "bandwidth_bytes_per_sec": bw_relay,
                      "affinity": "direct", "backend": "cuda", "executor": "relay", "via": v, "gpu": gpu})
    for i in range(sm_rails):
        rails.append({"id": f"g{gpu}.pcie{i}", "node": f"g{gpu}", "bandwidth_bytes_per_sec": bw_sm,
                      "affinity": "direct", "backend": "cuda", "executor": "sm"})
    for i in range(ce_rails):
        rails.append({"id": f"g{gpu}.ce{i}", "node": f"g{gpu}", "bandwidth_bytes_per_sec": bw_ce,
                      "affinity": "direct", "backend": "cuda", "executor": "ce", "ce_index": i})
    for r in rails:
        links.append({"device": f"g{gpu}.host", "rail": r["id"]})
        links.append({"device": f"g{gpu}.hbm", "rail": r["id"]})
    return json.dumps({"nodes": [_node(gpu)], "rails": rails, "links": links})


def peer_fabric(gpus: List[int], sm_rails: int = 1, ce_rails: int = 0, bw_sm: float = NVLINK5,
                bw_ce: float = NVLINK5, extra: Optional[List[Dict]] = None, relay_via: Optional[List[int]] = None,
                relay_affinity: str = "same_socket", bw_relay: float = NVLINK5) -> str:
    """NVLink fabric: one node per GPU, each with `sm_rails` SM peer-store rails (tier 1),
    `ce_rails` copy-engine rails and one 2-hop relay rail per GPU in `relay_via` (tier 2 by
    default: the reference's spillover tier), identical ids on every GPU (gK.nvlI / gK.ceI /
    gK.rlV) so the affinity pairing pairs like with like."""
    rails = []
    for g in gpus:
        for v in relay_via or []:
            rails.append({"id": f"g{g}.rl{v}", "node": f"g{g}", "bandwidth_bytes_per_sec": bw_relay,
                          "affinity": relay_affinity, "backend": "cuda", "executor": "relay", "via": v, "gpu": g})
        for i in range(sm_rails):
            rails.append({"id": f"g{g}.nvl{i}", "node": f"g{g}", "bandwidth_bytes_per_sec": bw_sm,
                          "affinity": "direct", "backend": "cuda", "executor": "sm", "gpu": g})
        for i in range(ce_rails):
            rails.append({"id": f"g{g}.ce{i}", "node": f"g{g}", "bandwidth_bytes_per_sec": bw_ce,
                          "affinity": "direct", "backend": "cuda", "executor": "ce", "ce_index": i, "gpu": g})
    rails += extra or []
    return json.dumps({"nodes": [_node(g) for g in gpus], "rails": rails})


def two_node(rails_per_node: int, bw=1e9, backend: str = "cuda", affinities=None) -> str:
    """Reference-style 2-node fabric (nodes a/b, rails a.rK/b.rK); used for plan parity
    with the reference's own fabrics (fabrics/uniform8.json shape)."""
    nodes = [{"id": n, "devices": [{"id": f"{n}.mem", "kind": "host_memory"},
                                    {"id": f"{n}.dev", "kind": "device_memory"}]} for n in ("a", "b")]
    rails = []
    for n in ("a", "b"):
        for i in range(rails_per_node):
            b = bw[i] if isinstance(bw, (list, tuple)) else bw
            rails.append({"id": f"{n}.r{i}", "node": n, "bandwidth_bytes_per_sec": float(b),
                          "affinity": affinities[i] if affinities else "direct", "backend": backend})
    return json.dumps({"nodes": nodes, "rails": rails})
