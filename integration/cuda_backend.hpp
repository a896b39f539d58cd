// cuda_backend.hpp — the reference-side plugin: a `"cuda"` spray::TransportBackend
// (proj/include/spray/backend.hpp:49-72) over the B200 C-ABI (include/spray_b200.h).
//
// This is the file a reference maintainer adds next to proj/src/backends/*.cpp; the only
// other change on their side is one branch in Engine::load_backends (proj/src/engine.cpp:
// 116-140):   } else if (name == "cuda") { b = std::make_unique<CudaBackend>(registry_.get(),
//                                                                            clock_.get(), 0); }
// It compiles against the reference's own headers and links the reference library and
// libspray_b200.so (integration/Makefile). The reference keeps scheduling, retries and
// health; every posted group of slices becomes one B200 copy launch.
#pragma once

#include <optional>
#include <span>
#include <vector>

#include "spray/backend.hpp"
#include "spray/fabric.hpp"
#include "spray_b200.h"

namespace spray {

class CudaBackend final : public TransportBackend {
 public:
  // `registry` is the engine's (non-owning, as memory_backend.hpp:31); `clock` stamps
  // nothing here (the B200 side measures t_obs itself) but keeps the constructor shape of
  // the reference's backends.
  CudaBackend(SegmentRegistry* registry, const Clock* clock, int device);
  ~CudaBackend() override;
  CudaBackend(const CudaBackend&) = delete;
  CudaBackend& operator=(const CudaBackend&) = delete;

  const BackendCapabilities& capabilities() const override { return caps_; }
  PostResult post_slices(std::span<const SliceWorkRequest> requests) override;
  std::vector<CompletionEvent> poll_completions(std::size_t max) override;
  bool fatal() const override;
  std::optional<std::vector<std::byte>> attach_segment_metadata(const SegmentDescriptor& desc) override;
  void start() override;
  void stop() override;

  // MemoryBackend::latch_fatal analogue (memory_backend.hpp), for tests.
  void latch_fatal();

 private:
  SegmentRegistry* registry_;
  const Clock* clock_;
  spray_backend* b_ = nullptr;
  BackendCapabilities caps_;
};

}  // namespace spray
