// NVLink peer-copy ceilings GPU0 -> GPU1 for the three ways the engine could move a slice:
// SM 128-bit loads/stores (the worker path), TMA bulk copies staged through shared memory
// (cp.async.bulk global->shared->global), and the copy engines (cudaMemcpyPeerAsync).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o peer_peak tools/peer_peak.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

struct V4 { uint32_t a, b, c, d; };

__global__ void __launch_bounds__(256) lsu_copy(V4* __restrict__ dst, const V4* __restrict__ src, uint64_t n,
                                                uint32_t chunk_v4) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = warp; c < n / chunk_v4; c += nwarps) {
    const V4* s = src + c * chunk_v4;
    V4* d = dst + c * chunk_v4;
    for (uint32_t i = lane; i < chunk_v4; i += 8 * 32) {
      V4 r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = s[i + u * 32];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + i + u * 32), "r"(r[u].a),
                     "r"(r[u].b), "r"(r[u].c), "r"(r[u].d)
                     : "memory");
    }
  }
}

// one elected lane per warp moves kPiece-byte pieces global->shared->global, kBuf deep
template <int kBuf>
__global__ void __launch_bounds__(128) tma_copy(uint8_t* dst, const uint8_t* src, uint64_t nbytes, uint32_t chunk,
                                                uint32_t piece) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[4][kBuf];
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = smem + (size_t)w * kBuf * piece;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (lane != 0) return;
  for (int b = 0; b < kBuf; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[w][b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[kBuf] = {};
  const uint32_t per = chunk / piece;
  for (uint64_t c = warp; c < nbytes / chunk; c += nwarps) {
    const uint8_t* s = src + c * chunk;
    uint8_t* d = dst + c * chunk;
    auto load = [&](uint32_t p) {
      const uint32_t b = p % kBuf;
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[w][b]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(piece) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(buf + (size_t)b * piece)),
                   "l"(s + (uint64_t)p * piece), "r"(piece), "r"(bar)
                   : "memory");
    };
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    for (uint32_t p = 0; p < per && p < (uint32_t)kBuf - 1; ++p) load(p);
    for (uint32_t p = 0; p < per; ++p) {
      const uint32_t b = p % kBuf;
      if (p + kBuf - 1 < per) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBuf - 2) : "memory");
        load(p + kBuf - 1);
      }
      uint32_t done = 0;
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[w][b]);
      while (!done)
        asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                     : "=r"(done) : "r"(bar), "r"(phase[b]) : "memory");
      phase[b] ^= 1;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + (uint64_t)p * piece),
                   "r"((uint32_t)__cvta_generic_to_shared(buf + (size_t)b * piece)), "r"(piece)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static float ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int main(int argc, char** argv) {
  const uint64_t bytes = (argc > 1 ? strtoull(argv[1], nullptr, 0) : (1ull << 30));
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  void *src, *dst;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&dst, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 7, bytes));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto best_of = [&](auto&& launch) {
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(a, st));
      launch();
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
      best = std::min(best, ms_between(a, b));
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  const double ce = best_of([&] { CK(cudaMemcpyPeerAsync(dst, 1, src, 0, bytes, st)); });
  std::printf("copy engine  %.1f GB/s\n", ce);
  for (int g : {sms, 2 * sms, 4 * sms}) {
    const double v = best_of([&] { lsu_copy<<<g, 256, 0, st>>>((V4*)dst, (const V4*)src, bytes / 16, (128u << 10) / 16); });
    std::printf("lsu  ctas=%4d %.1f GB/s\n", g, v);
  }
  for (uint32_t piece : {8192u, 16384u}) {
    const size_t smem = 4 * 3 * piece;  // 4 warps x 3 buffers
    CK(cudaFuncSetAttribute(tma_copy<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int g : {sms, 2 * sms}) {
      const double v = best_of([&] { tma_copy<3><<<g, 128, smem, st>>>((uint8_t*)dst, (const uint8_t*)src, bytes, 128u << 10, piece); });
      std::printf("tma  ctas=%4d (4 warps) piece=%5u x3 %.1f GB/s\n", g, piece, v);
    }
  }
  return 0;
}
