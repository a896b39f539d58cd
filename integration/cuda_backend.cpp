// cuda_backend.cpp — see cuda_backend.hpp. Translates the reference's TransportBackend
// contract onto spray_backend_* (include/spray_b200.h):
//   * SliceWorkRequest (backend.hpp:15-27) -> 88-byte spray_slice_wr, segment ids as their
//     Hash128 (common.hpp:111-120, the TCP wire's construction);
//   * PostResult (backend.hpp:44-47): accepted = prefix, a rejected suffix is backpressure,
//     SPRAY_EFATAL -> {0, fatal}; a capability mismatch is a programming error and throws
//     EngineError (backend.hpp:55-57, memory_backend.cpp:31-32);
//   * CompletionEvent (backend.hpp:33-40) <- spray_cqe, exactly one per accepted request;
//   * attach_segment_metadata (backend.hpp:65-68): registers the segment's buffers with the
//     B200 side; nullopt when the medium is not served (file media).
#include "cuda_backend.hpp"

#include <cstring>
#include <string>

namespace spray {

namespace {
Medium medium_of(uint32_t bit_index) { return static_cast<Medium>(bit_index); }
}  // namespace

CudaBackend::CudaBackend(SegmentRegistry* registry, const Clock* clock, int device)
    : registry_(registry), clock_(clock) {
  if (spray_backend_open(device, &b_) != SPRAY_OK) throw ConfigError(spray_last_error());
  spray_backend_caps c{};
  spray_backend_capabilities(b_, &c);
  caps_.id = c.id;
  // media_pairs_mask bit (src * 3 + dst), src/dst in spray_medium order = spray::Medium order
  for (uint32_t s = 0; s < 3; ++s)
    for (uint32_t d = 0; d < 3; ++d)
      if (c.media_pairs_mask & (1u << (s * 3 + d))) caps_.media_pairs.emplace_back(medium_of(s), medium_of(d));
  caps_.supports_read = c.supports_read != 0;
  caps_.supports_write = c.supports_write != 0;
  caps_.cross_node = c.cross_node != 0;
  caps_.same_node = c.same_node != 0;
  caps_.max_post_size = c.max_post_size;
  caps_.batched_posting = c.batched_posting != 0;
}

CudaBackend::~CudaBackend() { spray_backend_close(b_); }

void CudaBackend::start() {
  if (spray_backend_start(b_) != SPRAY_OK) throw EngineError(spray_last_error());
}

void CudaBackend::stop() { spray_backend_stop(b_); }

bool CudaBackend::fatal() const { return spray_backend_fatal(b_) != 0; }

void CudaBackend::latch_fatal() { spray_backend_latch_fatal(b_); }

std::optional<std::vector<std::byte>> CudaBackend::attach_segment_metadata(const SegmentDescriptor& desc) {
  std::vector<spray_buffer_desc> bufs;
  for (const BufferDesc& b : desc.buffers) bufs.push_back(spray_buffer_desc{b.offset, b.length, b.data});
  spray_segment_desc d{};
  d.id = desc.id.c_str();
  d.medium = desc.medium == Medium::kHostMemory ? SPRAY_MEDIUM_HOST
             : desc.medium == Medium::kFile     ? SPRAY_MEDIUM_FILE
                                                : SPRAY_MEDIUM_DEVICE;
  d.node = desc.node.c_str();
  d.buffers = bufs.data();
  d.n_buffers = static_cast<uint32_t>(bufs.size());
  d.device = desc.device.c_str();
  uint8_t blob[256];
  size_t len = 0;
  const int rc = spray_backend_attach_segment(b_, &d, blob, sizeof(blob), &len);
  if (rc == SPRAY_ECAPABILITY) return std::nullopt;  // medium not served by this backend
  if (rc != SPRAY_OK) throw EngineError(spray_last_error());
  std::vector<std::byte> out(std::min(len, sizeof(blob)));
  std::memcpy(out.data(), blob, out.size());
  return out;
}

PostResult CudaBackend::post_slices(std::span<const SliceWorkRequest> reqs) {
  std::vector<spray_slice_wr> wr(reqs.size());
  for (std::size_t i = 0; i < reqs.size(); ++i) {
    const SliceWorkRequest& r = reqs[i];
    const Hash128 s = hash128(r.src_segment), d = hash128(r.dst_segment);
    wr[i] = spray_slice_wr{r.slice, r.batch, s.lo, s.hi, r.src_offset, d.lo, d.hi, r.dst_offset, r.length,
                           r.direction == Direction::kRead ? SPRAY_READ : SPRAY_WRITE, r.local_rail,
                           r.remote_rail, r.attempt};
  }
  std::size_t accepted = 0;
  const int rc = spray_backend_post(b_, wr.data(), wr.size(), &accepted);
  if (rc == SPRAY_EFATAL) return PostResult{0, true};
  if (rc != SPRAY_OK) throw EngineError(spray_last_error());  // capability mismatch / bad request
  return PostResult{accepted, false};
}

std::vector<CompletionEvent> CudaBackend::poll_completions(std::size_t max) {
  std::vector<spray_cqe> c(max);
  std::size_t n = 0;
  if (max && spray_backend_poll(b_, c.data(), max, &n) != SPRAY_OK) throw EngineError(spray_last_error());
  std::vector<CompletionEvent> out(n);
  for (std::size_t i = 0; i < n; ++i) {
    out[i].slice = c[i].slice;
    out[i].batch = c[i].batch;
    out[i].status = c[i].status == SPRAY_SLICE_OK       ? SliceStatus::kOk
                    : c[i].status == SPRAY_SLICE_FAILED ? SliceStatus::kFailed
                                                        : SliceStatus::kTimeout;
    out[i].rail = c[i].rail;
    out[i].t_obs = c[i].t_obs_ns;
    out[i].bytes = c[i].bytes;
  }
  return out;
}

}  // namespace spray
