// fabric.cpp — topology parsing, segment coverage, reachability (see fabric.hpp).
#include "fabric.hpp"

#include <algorithm>

namespace spray {

uint64_t fnv1a64(const void* data, size_t len, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < len; ++i) h = (h ^ p[i]) * 0x100000001b3ULL;
  return h;
}

Hash128 hash128(const std::string& s) {
  return Hash128{fnv1a64(s.data(), s.size()), fnv1a64(s.data(), s.size(), 0x84222325cbf29ce4ULL)};
}

static int tier_of_name(const std::string& s) {
  if (s == "direct") return 1;
  if (s == "same_socket") return 2;
  if (s == "cross_socket") return 3;
  return 0;
}

Topology Topology::parse(const std::string& text) {
  Json doc;
  try {
    doc = Json::parse(text);
  } catch (const JsonError& e) {
    throw ConfigError(std::string("topology parse error: ") + e.what());
  }
  if (!doc.is_object() || !doc.contains("nodes") || !doc.contains("rails"))
    throw ConfigError("topology: missing required sections 'nodes' and 'rails'");
  Topology t;
  try {
    for (const Json& jn : doc.at("nodes").arr) {
      NodeDecl n;
      n.id = jn.at("id").as_string();
      if (jn.contains("devices")) {
        for (const Json& jd : jn.at("devices").arr) {
          DeviceDecl d;
          d.id = jd.at("id").as_string();
          const std::string k = jd.at("kind").as_string();
          if (k == "host_memory") d.kind = DeviceKind::kHostMemory;
          else if (k == "device_memory") d.kind = DeviceKind::kDeviceMemory;
          else if (k == "file_store") d.kind = DeviceKind::kFileStore;
          else throw ConfigError("unknown device kind in node '" + n.id + "'");
          n.devices.push_back(d);
        }
      }
      t.nodes_.push_back(std::move(n));
    }
    for (const Json& jr : doc.at("rails").arr) {
      RailDecl r;
      r.id = jr.at("id").as_string();
      r.node = jr.at("node").as_string();
      r.bandwidth = jr.at("bandwidth_bytes_per_sec").as_number();
      r.tier = tier_of_name(jr.at("affinity").as_string());
      if (!r.tier) throw ConfigError("rail '" + r.id + "': unknown affinity");
      r.backend = jr.string_or("backend", "sim");
      const std::string ex = jr.string_or("executor", "sm");
      if (ex == "sm") r.executor = 0;
      else if (ex == "ce") r.executor = 1;
      else if (ex == "relay") r.executor = 2;
      else throw ConfigError("rail '" + r.id + "': unknown executor '" + ex + "'");
      r.gpu = static_cast<int>(jr.number_or("gpu", -1));
      r.via = static_cast<int>(jr.number_or("via", -1));
      r.ce_index = static_cast<uint32_t>(jr.number_or("ce_index", 0));
      const std::string stg = jr.string_or("staging", "device");
      if (stg != "device" && stg != "host") throw ConfigError("rail '" + r.id + "': staging must be device or host");
      r.host_staged = stg == "host";
      if (r.host_staged && r.executor != 2) throw ConfigError("rail '" + r.id + "': host staging is for relay rails");
      t.rails_.push_back(std::move(r));
    }
  } catch (const JsonError& e) {
    throw ConfigError(std::string("topology: ") + e.what());
  }
  // validation (fabric.cpp:46-76 semantics)
  for (RailIndex i = 0; i < t.rails_.size(); ++i) {
    const RailDecl& r = t.rails_[i];
    if (!(r.bandwidth > 0.0)) throw ConfigError("rail '" + r.id + "': NonPositiveBandwidth");
    if (!t.node(r.node)) throw ConfigError("rail '" + r.id + "': dangling node reference '" + r.node + "'");
    if (!t.by_id_.emplace(r.id, i).second) throw ConfigError("duplicate rail id '" + r.id + "'");
  }
  for (RailIndex i = 0; i < t.rails_.size(); ++i) t.by_node_backend_[{t.rails_[i].node, t.rails_[i].backend}].push_back(i);
  for (auto& kv : t.by_node_backend_)
    std::sort(kv.second.begin(), kv.second.end(),
              [&](RailIndex a, RailIndex b) { return t.rails_[a].id < t.rails_[b].id; });
  if (doc.contains("links")) {
    for (const Json& jl : doc.at("links").arr) {
      const std::string dev = jl.at("device").as_string();
      const std::string rid = jl.at("rail").as_string();
      auto ri = t.rail_index(rid);
      if (!ri) throw ConfigError("link: dangling rail reference '" + rid + "'");
      bool found = false;
      for (const NodeDecl& n : t.nodes_)
        for (const DeviceDecl& d : n.devices)
          if (d.id == dev) found = true;
      if (!found) throw ConfigError("link: dangling device reference '" + dev + "'");
      int tier = t.rails_[*ri].tier;
      if (jl.contains("affinity")) {
        tier = tier_of_name(jl.at("affinity").as_string());
        if (!tier) throw ConfigError("link: unknown affinity");
      }
      t.links_[dev][*ri] = tier;
    }
  }
  return t;
}

std::optional<RailIndex> Topology::rail_index(const std::string& id) const {
  auto it = by_id_.find(id);
  if (it == by_id_.end()) return std::nullopt;
  return it->second;
}

const NodeDecl* Topology::node(const std::string& id) const {
  for (const NodeDecl& n : nodes_)
    if (n.id == id) return &n;
  return nullptr;
}

const std::vector<RailIndex>& Topology::rails_on(const std::string& node, const std::string& backend) const {
  auto it = by_node_backend_.find({node, backend});
  return it == by_node_backend_.end() ? empty_ : it->second;
}

std::optional<int> Topology::tier_from_device(const std::string& device, RailIndex rail) const {
  auto it = links_.find(device);
  if (it == links_.end()) return rails_[rail].tier;
  auto jt = it->second.find(rail);
  if (jt == it->second.end()) return std::nullopt;
  return jt->second;
}

const DeviceDecl* Topology::find_device(const std::string& node_id, const std::string& id) const {
  const NodeDecl* n = node(node_id);
  if (!n) return nullptr;
  for (const DeviceDecl& d : n->devices)
    if (d.id == id) return &d;
  return nullptr;
}

const DeviceDecl* Topology::first_device_of_kind(const std::string& node_id, DeviceKind kind) const {
  const NodeDecl* n = node(node_id);
  if (!n) return nullptr;
  for (const DeviceDecl& d : n->devices)
    if (d.kind == kind) return &d;
  return nullptr;
}

RailIndex Topology::add_rail(const RailDecl& r) {
  if (!node(r.node)) throw ConfigError("rail '" + r.id + "': dangling node reference '" + r.node + "'");
  const RailIndex i = static_cast<RailIndex>(rails_.size());
  if (!by_id_.emplace(r.id, i).second) throw ConfigError("duplicate rail id '" + r.id + "'");
  rails_.push_back(r);
  auto& v = by_node_backend_[{r.node, r.backend}];
  v.push_back(i);
  std::sort(v.begin(), v.end(), [&](RailIndex a, RailIndex b) { return rails_[a].id < rails_[b].id; });
  for (const DeviceDecl& d : node(r.node)->devices) {
    auto it = links_.find(d.id);
    if (it != links_.end()) it->second[i] = r.tier;
  }
  return i;
}

int Topology::node_gpu(const std::string& n) const {
  for (const RailDecl& r : rails_)
    if (r.node == n && r.gpu >= 0) return r.gpu;
  return -1;
}

std::vector<uint32_t> Topology::id_ranks() const {
  std::vector<uint32_t> ranks(rails_.size());
  uint32_t k = 0;
  for (const auto& kv : by_id_) ranks[kv.second] = k++;  // std::map iterates in id order
  return ranks;
}

const Buffer* Segment::covering(uint64_t off, uint64_t len) const {
  if (len == 0) return nullptr;
  for (const Buffer& b : buffers) {
    if (off >= b.offset && off + len <= b.offset + b.length) return &b;
    if (b.offset > off) break;
  }
  return nullptr;
}

Capabilities Capabilities::preset(const std::string& name) {
  Capabilities c;
  c.id = name;
  const uint32_t hh = 1u << 0, hd = 1u << 1, dh = 1u << 3, dd = 1u << 4;
  if (name == "sim") {  // sim_backend.cpp:9-25
    c.media_mask = hh | hd | dh | dd;
    c.cross_node = true;
    c.same_node = false;
  } else if (name == "memory") {  // memory_backend.cpp:8-19
    c.media_mask = hh | hd | dh | dd;
    c.cross_node = true;
    c.same_node = true;
  } else if (name == "cuda") {  // this backend: every host/HBM pair, within and across nodes
    c.media_mask = hh | hd | dh | dd;
    c.cross_node = true;
    c.same_node = true;
  } else {
    throw ConfigError("unknown backend '" + name + "'");
  }
  return c;
}

std::vector<Reach> reachable(const Topology& g, const Segment& src, const Segment& dst,
                             const std::vector<Capabilities>& caps) {
  std::vector<Reach> out;
  const bool same_node = src.node == dst.node;
  for (const Capabilities& cap : caps) {
    if (!cap.covers(src.medium, dst.medium)) continue;
    if (!cap.read && !cap.write) continue;
    if (same_node ? !cap.same_node : !cap.cross_node) continue;
    const auto& lr = g.rails_on(src.node, cap.id);
    const auto& rr = g.rails_on(dst.node, cap.id);
    auto emit = [&](RailIndex l, RailIndex r) {
      auto lt = g.tier_from_device(src.device, l);
      auto rt = g.tier_from_device(dst.device, r);
      if (!lt || !rt) return;
      out.push_back(Reach{l, r, std::max(*lt, *rt), cap.read, cap.write, cap.id});
    };
    if (same_node) {
      for (RailIndex r : lr) emit(r, r);
    } else {
      for (RailIndex l : lr)
        for (RailIndex r : rr) emit(l, r);
    }
  }
  std::sort(out.begin(), out.end(), [&](const Reach& a, const Reach& b) {
    if (a.tier != b.tier) return a.tier < b.tier;
    if (a.backend != b.backend) return a.backend < b.backend;
    if (g.rail(a.local).id != g.rail(b.local).id) return g.rail(a.local).id < g.rail(b.local).id;
    return g.rail(a.remote).id < g.rail(b.remote).id;
  });
  return out;
}

}  // namespace spray
