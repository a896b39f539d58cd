// fabric.hpp — declarative fabric model of the B200 data plane.
//
// Mirrors the reference's topology document and planning vocabulary
// (proj/include/spray/fabric.hpp:22-241, proj/src/fabric.cpp:46-366) so the same JSON
// describes both the reference's simulated rails and the B200 paths, and so the
// candidate lists the scheduler sees are ordered exactly as the reference orders them.
// B200 extensions per rail: "executor" (sm | ce | relay), "gpu", "via", "ce_index".
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"

namespace spray {

// Error classes of the reference (common.hpp:31-41, engine.hpp:28-31,
// orchestrator.hpp:20-23); the C-ABI maps each to its SPRAY_E* code.
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct EngineError : std::runtime_error {
  explicit EngineError(const std::string& w) : std::runtime_error(w) {}
};
struct InvalidRangeError : EngineError {
  explicit InvalidRangeError(const std::string& w) : EngineError(w) {}
};
struct NoRouteError : EngineError {
  explicit NoRouteError(const std::string& w) : EngineError(w) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

enum class Medium { kHost = 0, kDevice = 1, kFile = 2 };
enum class Direction { kRead = 0, kWrite = 1 };
enum class DeviceKind { kHostMemory, kDeviceMemory, kFileStore };

using RailIndex = uint32_t;
constexpr RailIndex kNoRail = 0xffffffffu;

uint64_t fnv1a64(const void* data, size_t len, uint64_t basis = 0xcbf29ce484222325ULL);
struct Hash128 {
  uint64_t lo = 0, hi = 0;
  bool operator==(const Hash128& o) const { return lo == o.lo && hi == o.hi; }
};
Hash128 hash128(const std::string& s);  // common.hpp:117-120

struct DeviceDecl {
  std::string id;
  DeviceKind kind = DeviceKind::kHostMemory;
};
struct NodeDecl {
  std::string id;
  std::vector<DeviceDecl> devices;
};
struct RailDecl {
  std::string id, node, backend;
  double bandwidth = 0.0;  // B_d, bytes/s
  int tier = 1;            // affinity class: 1 direct, 2 same_socket, 3 cross_socket
  uint32_t executor = 0;   // 0 sm, 1 ce, 2 relay
  int gpu = -1, via = -1;
  uint32_t ce_index = 0;
  bool host_staged = false;  // relay through a bounded pinned-host pool ("staging": "host"):
                             // the staged route of engine.cpp:465-610, no peer access needed
};

class Topology {
 public:
  static Topology parse(const std::string& json_text);  // fabric.cpp:157-210 format

  size_t rail_count() const { return rails_.size(); }
  const RailDecl& rail(RailIndex i) const { return rails_[i]; }
  std::optional<RailIndex> rail_index(const std::string& id) const;
  const std::vector<NodeDecl>& nodes() const { return nodes_; }
  const NodeDecl* node(const std::string& id) const;
  // Rails of one backend on one node, sorted by rail id (the affinity index order).
  const std::vector<RailIndex>& rails_on(const std::string& node, const std::string& backend) const;
  // Tier of `rail` as seen from `device` (link override / nullopt if unlinked).
  std::optional<int> tier_from_device(const std::string& device, RailIndex rail) const;
  const DeviceDecl* find_device(const std::string& node, const std::string& id) const;
  const DeviceDecl* first_device_of_kind(const std::string& node, DeviceKind kind) const;
  // Rank of each rail's id string in sorted order (string-order tie-breaks on device).
  std::vector<uint32_t> id_ranks() const;
  // Appends a rail (staged-route synthesis): linked at tier `tier` to every device of its
  // node that has explicit links, indices rebuilt.
  RailIndex add_rail(const RailDecl& r);
  // GPU ordinal a node's rails declare ("gpu" key), -1 if none.
  int node_gpu(const std::string& node) const;

 private:
  std::vector<NodeDecl> nodes_;
  std::vector<RailDecl> rails_;
  std::map<std::string, RailIndex> by_id_;
  std::map<std::pair<std::string, std::string>, std::vector<RailIndex>> by_node_backend_;
  std::map<std::string, std::map<RailIndex, int>> links_;  // device -> rail -> tier
  std::vector<RailIndex> empty_;
};

struct Buffer {
  uint64_t offset = 0, length = 0;
  void* data = nullptr;     // as registered (host pointer for host media)
  uint64_t dev_addr = 0;    // address the GPU uses for the same bytes (UVA / mapped)
};

struct Segment {
  std::string id;
  Medium medium = Medium::kHost;
  std::string node, device;
  Hash128 id_hash;
  std::vector<Buffer> buffers;  // sorted by offset, non-overlapping
  // The buffer containing [off, off+len) entirely, or null (fabric.cpp:220-237).
  const Buffer* covering(uint64_t off, uint64_t len) const;
};

// What a backend declares about itself (fabric.hpp:207-221).
struct Capabilities {
  std::string id;
  uint32_t media_mask = 0;  // bit (src*3+dst)
  bool read = true, write = true, cross_node = true, same_node = true;
  bool covers(Medium s, Medium d) const { return media_mask & (1u << (int(s) * 3 + int(d))); }
  static Capabilities preset(const std::string& name);  // "cuda" | "sim" | "memory"
};

struct Reach {
  RailIndex local = kNoRail, remote = kNoRail;
  int tier = 3;
  bool read_ok = false, write_ok = false;
  std::string backend;
};

// reachable_rails (fabric.cpp:325-366): every (src-side, dst-side) rail pair a backend
// can serve, sorted by (tier, backend, local id, remote id).
std::vector<Reach> reachable(const Topology& g, const Segment& src, const Segment& dst,
                             const std::vector<Capabilities>& caps);

}  // namespace spray
