// Push vs pull over NVLink: the same 128-bit copy loop run on the SOURCE GPU (loads local,
// stores into peer HBM: the engine's WRITE path) or on the DESTINATION GPU (loads from
// peer HBM, stores local: a READ-direction transfer scheduled by the receiver), and both
// ends splitting the bytes (half pushed, half pulled). Also the copy engine for reference.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o peer_pull tools/peer_pull.cu
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

// warp-per-chunk copy, 8 x 16 B in flight per lane; U = unroll depth
template <int U>
__global__ void __launch_bounds__(256) copy_kernel(V4* __restrict__ dst, const V4* __restrict__ src, uint64_t n_v4,
                                                   uint32_t chunk_v4) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = warp; c < n_v4 / chunk_v4; c += nwarps) {
    const V4* s = src + c * chunk_v4;
    V4* d = dst + c * chunk_v4;
    for (uint32_t i = lane; i < chunk_v4; i += U * 32) {
      V4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[u].a), "=r"(r[u].b), "=r"(r[u].c), "=r"(r[u].d) : "l"(s + i + u * 32));
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + i + u * 32), "r"(r[u].a),
                     "r"(r[u].b), "r"(r[u].c), "r"(r[u].d)
                     : "memory");
    }
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t sizes[] = {1ull << 30, 4ull << 30};
  uint8_t *a, *b;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a, sizes[1]));
  CK(cudaMemset(a, 7, sizes[1]));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&b, sizes[1]));
  cudaStream_t s0, s1;
  CK(cudaSetDevice(0));
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaSetDevice(1));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, f0, f1;
  CK(cudaSetDevice(0));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaSetDevice(1));
  CK(cudaEventCreate(&f0));
  CK(cudaEventCreate(&f1));
  const uint32_t chunk = 32768 / 16;
  std::printf("{\n");
  for (uint64_t sz : sizes) {
    const uint64_t nv = sz / 16;
    for (int mode = 0; mode < 4; ++mode) {
      for (int ctas_per_sm : {1, 2, 4}) {
        const int grid = sms * ctas_per_sm;
        float best = 1e9f;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaSetDevice(0));
          CK(cudaDeviceSynchronize());
          CK(cudaSetDevice(1));
          CK(cudaDeviceSynchronize());
          float ms = 0.f;
          if (mode == 0) {  // push: GPU0 kernel stores into GPU1
            CK(cudaSetDevice(0));
            CK(cudaEventRecord(e0, s0));
            copy_kernel<8><<<grid, 256, 0, s0>>>((V4*)b, (const V4*)a, nv, chunk);
            CK(cudaEventRecord(e1, s0));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
          } else if (mode == 1) {  // pull: GPU1 kernel loads from GPU0
            CK(cudaSetDevice(1));
            CK(cudaEventRecord(f0, s1));
            copy_kernel<8><<<grid, 256, 0, s1>>>((V4*)b, (const V4*)a, nv, chunk);
            CK(cudaEventRecord(f1, s1));
            CK(cudaEventSynchronize(f1));
            CK(cudaEventElapsedTime(&ms, f0, f1));
          } else if (mode == 2) {  // half pushed by GPU0, half pulled by GPU1
            CK(cudaSetDevice(0));
            CK(cudaEventRecord(e0, s0));
            copy_kernel<8><<<grid, 256, 0, s0>>>((V4*)b, (const V4*)a, nv / 2, chunk);
            CK(cudaSetDevice(1));
            copy_kernel<8><<<grid, 256, 0, s1>>>((V4*)b + nv / 2, (const V4*)a + nv / 2, nv / 2, chunk);
            CK(cudaEventRecord(f1, s1));
            CK(cudaSetDevice(0));
            CK(cudaStreamWaitEvent(s0, f1, 0));
            CK(cudaEventRecord(e1, s0));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
          } else {  // copy engine
            if (ctas_per_sm != 1) break;
            CK(cudaSetDevice(0));
            CK(cudaEventRecord(e0, s0));
            CK(cudaMemcpyPeerAsync(b, 1, a, 0, sz, s0));
            CK(cudaEventRecord(e1, s0));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
          }
          CK(cudaGetLastError());
          if (ms > 0) best = std::min(best, ms);
        }
        if (best < 1e8f) {
          const char* nm[] = {"push", "pull", "push_half_pull_half", "copy_engine"};
          std::printf("  \"%s_%lluMiB_%dcta\": %.1f,\n", nm[mode], (unsigned long long)(sz >> 20), ctas_per_sm,
                      sz / (best * 1e-3) / 1e9);
        }
      }
    }
  }
  std::printf("  \"unit\": \"GB/s\"\n}\n");
  return 0;
}
