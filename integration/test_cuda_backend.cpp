// test_cuda_backend.cpp — the reference-side "cuda" TransportBackend driven through the
// reference's own contract, in the style of proj/tests/test_backends.cpp:262-300
// (MemoryBackend: inline copy, one CQE per request, fatal latch), on a B200.
//
// Built by integration/Makefile against the reference headers + the unmodified reference
// library (oracle/_ref/libspray_ref.so) + libspray_b200.so; run by
// tests/test_gpu_integration.py. Exit code 0 = every check passed.
//
//  1. capabilities translate to BackendCapabilities (fabric.hpp:207-221)
//  2. attach_segment_metadata through a reference SegmentRegistry provider
//     (fabric.cpp:294-298): blobs for host and device segments, none for a file segment
//  3. post_slices/poll_completions: HBM->HBM, HBM->pinned host, host->HBM, bit-exact,
//     exactly one CompletionEvent per accepted request, t_obs > 0, bytes = length
//  4. backpressure: a post beyond the in-flight window accepts a prefix (backend.hpp:42-43)
//  5. capability mismatch (unregistered segment) throws EngineError (backend.hpp:55-57)
//  6. fatal latch: {accepted 0, fatal}, fatal() (memory_backend.cpp:23-26)
//  7. plugin mode end to end: the reference SliceScheduler decomposes a 64 MiB transfer
//     (config 1: 1024 x 64 KiB over 2 rails), decides every slice (choose_rail), the CUDA
//     backend moves it in per-rail groups of <= 32 (worker_post_phase burst,
//     engine.cpp:884), completions release + feed back (engine.cpp:800, 833-834);
//     delivered bytes equal the source (checksum), every slice completes exactly once.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "cuda_backend.hpp"
#include "spray/scheduler.hpp"

using namespace spray;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                             \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(c)) {                                                              \
      ++g_fail;                                                              \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                                        \
  } while (0)

static const char* kFabric = R"({
  "nodes": [
    {"id": "a", "devices": [{"id": "a.mem", "kind": "host_memory"}, {"id": "a.dev", "kind": "device_memory"}]},
    {"id": "b", "devices": [{"id": "b.mem", "kind": "host_memory"}, {"id": "b.dev", "kind": "device_memory"}]}
  ],
  "rails": [
    {"id": "a.r0", "node": "a", "bandwidth_bytes_per_sec": 1e9, "affinity": "direct", "backend": "cuda"},
    {"id": "a.r1", "node": "a", "bandwidth_bytes_per_sec": 1e9, "affinity": "direct", "backend": "cuda"},
    {"id": "b.r0", "node": "b", "bandwidth_bytes_per_sec": 1e9, "affinity": "direct", "backend": "cuda"},
    {"id": "b.r1", "node": "b", "bandwidth_bytes_per_sec": 1e9, "affinity": "direct", "backend": "cuda"}
  ]
})";

static void* dev_alloc(size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, n) != cudaSuccess) {
    std::fprintf(stderr, "cudaMalloc failed\n");
    std::exit(2);
  }
  cudaMemset(p, 0, n);
  return p;
}
static uint64_t sum(const void* p, uint64_t n) {
  uint64_t v = 0;
  if (spray_checksum(0, p, n, &v) != SPRAY_OK) std::fprintf(stderr, "checksum: %s\n", spray_last_error());
  return v;
}
static SegmentDescriptor seg(const std::string& id, Medium m, const std::string& node, void* p, Bytes n) {
  SegmentDescriptor d;
  d.id = id;
  d.medium = m;
  d.node = node;
  d.buffers = {BufferDesc{0, n, static_cast<std::byte*>(p)}};
  return d;
}
static std::vector<CompletionEvent> drain(CudaBackend& be, size_t want) {
  std::vector<CompletionEvent> out;
  for (int spin = 0; out.size() < want && spin < 2000000; ++spin) {
    auto ev = be.poll_completions(64);
    out.insert(out.end(), ev.begin(), ev.end());
  }
  return out;
}

int main() {
  cudaSetDevice(0);
  TopologyGraph graph = load_topology(kFabric);
  SegmentRegistry registry(&graph);
  WallClock clock;
  CudaBackend cuda(&registry, &clock, 0);
  registry.add_provider(MetadataProvider{
      "cuda", [&cuda](const SegmentDescriptor& d) { return cuda.attach_segment_metadata(d); }});
  cuda.start();

  // 1. capabilities
  const BackendCapabilities& caps = cuda.capabilities();
  CHECK(caps.id == "cuda");
  CHECK(caps.covers(Medium::kHostMemory, Medium::kHostMemory));
  CHECK(caps.covers(Medium::kDeviceMemoryEmulated, Medium::kDeviceMemoryEmulated));
  CHECK(caps.covers(Medium::kHostMemory, Medium::kDeviceMemoryEmulated));
  CHECK(caps.covers(Medium::kDeviceMemoryEmulated, Medium::kHostMemory));
  CHECK(!caps.covers(Medium::kFile, Medium::kHostMemory));
  CHECK(caps.supports_read && caps.supports_write && caps.cross_node && caps.same_node);

  // 2. segments (device memory is real HBM here; host memory pinned and mapped)
  const Bytes n = 64ull << 20;
  void* src = dev_alloc(n);
  void* dst = dev_alloc(n);
  void* host = nullptr;
  spray_host_alloc(n, &host);
  std::memset(host, 0, n);
  spray_fill_splitmix(0, src, n, 1 ^ 0x517cc1b727220a95ULL);  // bench.cpp:99 payload, seed 1
  auto s_src = registry.register_segment(seg("src", Medium::kDeviceMemoryEmulated, "a", src, n));
  auto s_dst = registry.register_segment(seg("dst", Medium::kDeviceMemoryEmulated, "b", dst, n));
  auto s_host = registry.register_segment(seg("host", Medium::kHostMemory, "b", host, n));
  CHECK(s_src->metadata_for("cuda") != nullptr);
  CHECK(s_host->metadata_for("cuda") != nullptr);
  {
    const auto* m = s_dst->metadata_for("cuda");
    CHECK(m && std::string(reinterpret_cast<const char*>(m->data()), m->size()) == "cuda:dst");
  }
  {
    SegmentDescriptor f;
    f.id = "file0";
    f.medium = Medium::kFile;
    f.node = "a";
    f.file_path = "/tmp/none";
    f.buffers = {BufferDesc{0, 4096, nullptr}};
    CHECK(!cuda.attach_segment_metadata(f).has_value());
  }

  // 3. three media pairs, bit-exact, one CQE each (requests of one post are unordered, so
  // the host->HBM leg is posted after the HBM->host leg it reads has completed)
  {
    std::vector<SliceWorkRequest> r(3);
    r[0] = SliceWorkRequest{1, 7, "src", 0, "dst", 0, 1 << 20, Direction::kWrite, 0, 2, 0};
    r[1] = SliceWorkRequest{2, 7, "src", 1 << 20, "host", 1 << 20, 1 << 20, Direction::kWrite, 1, 3, 0};
    r[2] = SliceWorkRequest{3, 7, "host", 1 << 20, "dst", 2 << 20, 1 << 20, Direction::kWrite, 1, 3, 0};
    auto res = cuda.post_slices(std::span<const SliceWorkRequest>(r).first(2));
    CHECK(res.accepted == 2 && !res.fatal);
    auto ev = drain(cuda, 2);
    res = cuda.post_slices(std::span<const SliceWorkRequest>(r).subspan(2));
    CHECK(res.accepted == 1 && !res.fatal);
    auto ev2 = drain(cuda, 1);
    ev.insert(ev.end(), ev2.begin(), ev2.end());
    CHECK(ev.size() == 3);
    std::set<SliceId> seen;
    for (const auto& e : ev) {
      CHECK(e.status == SliceStatus::kOk);
      CHECK(e.t_obs > 0);
      CHECK(e.bytes == (1u << 20));
      CHECK(e.batch == 7);
      seen.insert(e.slice);
    }
    CHECK(seen == (std::set<SliceId>{1, 2, 3}));
    CHECK(sum(dst, 1 << 20) == sum(src, 1 << 20));
    CHECK(sum(static_cast<char*>(dst) + (2 << 20), 1 << 20) == sum(static_cast<char*>(src) + (1 << 20), 1 << 20));
  }

  // 4. backpressure: the window (64 in flight) accepts a prefix of 100
  {
    std::vector<SliceWorkRequest> r;
    for (int i = 0; i < 100; ++i)
      r.push_back(SliceWorkRequest{uint64_t(100 + i), 8, "src", Bytes(i) << 16, "dst", Bytes(i) << 16, 65536,
                                   Direction::kWrite, 0, 2, 0});
    auto res = cuda.post_slices(r);
    CHECK(res.accepted > 0 && res.accepted < r.size() && !res.fatal);
    size_t posted = res.accepted;
    size_t done = 0;
    for (int spin = 0; posted < r.size() && spin < 2000000; ++spin) {  // the rejected suffix, re-posted
      done += cuda.poll_completions(64).size();
      auto rr = cuda.post_slices(std::span<const SliceWorkRequest>(r).subspan(posted));
      posted += rr.accepted;
    }
    CHECK(posted == r.size());
    done += drain(cuda, r.size() - done).size();
    CHECK(done == r.size());
  }

  // 5. a request the backend cannot serve is a programming error
  {
    std::vector<SliceWorkRequest> r{SliceWorkRequest{500, 9, "nowhere", 0, "dst", 0, 4096, Direction::kWrite, 0, 2, 0}};
    bool threw = false;
    try {
      cuda.post_slices(r);
    } catch (const EngineError&) {
      threw = true;
    }
    CHECK(threw);
  }

  // 7. plugin mode end to end: reference scheduler, B200 copies (config 1)
  {
    cudaMemset(dst, 0, n);
    cudaDeviceSynchronize();
    SchedulerConfig cfg;
    SliceScheduler sched(&graph, cfg);
    const RailIndex a0 = *graph.rail_index("a.r0"), a1 = *graph.rail_index("a.r1");
    const RailIndex b0 = *graph.rail_index("b.r0"), b1 = *graph.rail_index("b.r1");
    std::vector<LocalCandidate> cands(2);
    cands[0].local = a0;
    cands[0].pairs = {PairOption{b0, 1, true}, PairOption{b1, 1, false}};
    cands[1].local = a1;
    cands[1].pairs = {PairOption{b1, 1, true}, PairOption{b0, 1, false}};
    const auto pieces = SliceScheduler::decompose(n, cfg);
    CHECK(pieces.size() == 1024);
    struct Rec {
      Bytes off, len;
      DispatchChoice ch;
      bool done = false;
    };
    std::vector<Rec> recs;
    std::map<RailIndex, std::vector<size_t>> pending;
    for (const auto& [off, len] : pieces) {
      auto ch = sched.choose_rail(len, off, cands);
      CHECK(ch.has_value());
      recs.push_back(Rec{off, len, *ch});
      pending[ch->local].push_back(recs.size() - 1);
    }
    size_t completed = 0, dup = 0;
    std::map<RailIndex, size_t> per_rail;
    for (int spin = 0; completed < recs.size() && spin < 20000000; ++spin) {
      for (auto& [rail, q] : pending) {  // one grouped post per rail per round, burst <= 32
        if (q.empty()) continue;
        std::vector<SliceWorkRequest> g;
        for (size_t k = 0; k < q.size() && g.size() < 32; ++k) {
          const Rec& r = recs[q[k]];
          g.push_back(SliceWorkRequest{q[k], 1, "src", r.off, "dst", r.off, r.len, Direction::kWrite, r.ch.local,
                                       r.ch.remote, 0});
        }
        const auto res = cuda.post_slices(g);
        q.erase(q.begin(), q.begin() + static_cast<std::ptrdiff_t>(res.accepted));
      }
      for (const CompletionEvent& e : cuda.poll_completions(32)) {
        Rec& r = recs[e.slice];
        if (r.done) ++dup;
        r.done = true;
        ++completed;
        ++per_rail[r.ch.local];
        sched.release(r.ch.local, r.len);
        if (e.status == SliceStatus::kOk && r.ch.x_norm > 0.0) sched.feedback(r.ch.local, to_seconds(e.t_obs), r.ch.x_norm);
      }
    }
    CHECK(completed == recs.size());
    CHECK(dup == 0);
    CHECK(per_rail[a0] > 0 && per_rail[a1] > 0);
    CHECK(sched.queued_bytes(a0) == 0 && sched.queued_bytes(a1) == 0);
    CHECK(sum(dst, n) == sum(src, n));
  }

  // 6. fatal latch
  {
    cuda.latch_fatal();
    std::vector<SliceWorkRequest> r{SliceWorkRequest{900, 9, "src", 0, "dst", 0, 4096, Direction::kWrite, 0, 2, 0}};
    auto res = cuda.post_slices(r);
    CHECK(res.accepted == 0 && res.fatal);
    CHECK(cuda.fatal());
  }

  cuda.stop();
  cudaFree(src);
  cudaFree(dst);
  spray_host_free(host);
  std::printf("cuda backend plugin: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
