// Host-link ceiling probe: what the HBM <-> pinned-host path of one B200 delivers to
// (a) the copy engines (cudaMemcpyAsync) and (b) SM load/store copies into mapped pinned
// memory (the engine's copy-worker path), each direction alone and both at once. Also the
// latency of a GPU-scope fence and of a host-memory read while the link is saturated.
// Output: one JSON object on stdout (profiles/pcie_peak.json keeps a copy).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pcie_peak tools/pcie_peak.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
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

// grid-stride 16-byte copy, 8 loads in flight per lane
__global__ void __launch_bounds__(256) sm_copy(V4* __restrict__ dst, const V4* __restrict__ src, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    V4 r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) r[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[i + u * stride] = r[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
  __threadfence_system();
}

// warp-per-chunk copy (the engine worker's access pattern): each warp moves whole
// contiguous chunks; fence = 1 adds a system fence after every chunk (completion publish)
__global__ void __launch_bounds__(256) chunk_copy(V4* __restrict__ dst, const V4* __restrict__ src, uint64_t n,
                                                  uint32_t chunk_v4, int fence) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nch = n / chunk_v4;
  for (uint64_t c = warp; c < nch; c += nwarps) {
    const V4* s = src + c * chunk_v4;
    V4* d = dst + c * chunk_v4;
    for (uint32_t i = lane; i < chunk_v4; i += 8 * 32) {
      V4 r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = s[i + u * 32];
      if (fence & 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + i + u * 32), "r"(r[u].a),
                       "r"(r[u].b), "r"(r[u].c), "r"(r[u].d)
                       : "memory");
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) d[i + u * 32] = r[u];
      }
    }
    if (fence & 1) __threadfence_system();
  }
}

// warp-per-chunk copy through shared memory with bulk-async (TMA) copies: lane 0 moves
// kPiece-byte pieces global->shared (mbarrier completion) and shared->global (bulk group),
// double buffered per warp
constexpr uint32_t kPiece = 8192;
__global__ void __launch_bounds__(256) tma_copy(uint8_t* dst, const uint8_t* src, uint64_t nbytes, uint32_t chunk) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[8][2];
  const uint32_t warp_in = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = smem + warp_in * 2 * kPiece;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (lane == 0) {
    for (int b = 0; b < 2; ++b) {
      const uint32_t a = (uint32_t)__cvta_generic_to_shared(&bars[warp_in][b]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (lane != 0) return;
  uint32_t phase[2] = {0, 0};
  const uint64_t nch = nbytes / chunk;
  const uint32_t per = chunk / kPiece;
  for (uint64_t c = warp; c < nch; c += nwarps) {
    const uint8_t* s = src + c * chunk;
    uint8_t* d = dst + c * chunk;
    auto load = [&](uint32_t p) {
      const uint32_t b = p & 1;
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp_in][b]);
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf + b * kPiece);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kPiece) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb),
                   "l"(s + (uint64_t)p * kPiece), "r"(kPiece), "r"(bar)
                   : "memory");
    };
    // buffer 0 is free once the previous chunk's stores have read it
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    load(0);
    for (uint32_t p = 0; p < per; ++p) {
      const uint32_t b = p & 1;
      if (p + 1 < per) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // buffer b^1 free
        load(p + 1);
      }
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp_in][b]);
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
            : "=r"(done) : "r"(bar), "r"(phase[b]) : "memory");
      phase[b] ^= 1;
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf + b * kPiece);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + (uint64_t)p * kPiece),
                   "r"(sb), "r"(kPiece)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// one thread: fence latency and L2 (HBM-resident) read latency, sampled while a copy runs
__global__ void probe_l2(const volatile uint64_t* dev_word, uint64_t* out, int iters) {
  long long f = 0, r = 0;
  uint64_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    long long t0 = clock64();
    __threadfence();
    long long t1 = clock64();
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(dev_word + (i & 7) * 64) : "memory");
    acc += v;
    asm volatile("" ::"l"(acc));
    long long t2 = clock64();
    f += t1 - t0;
    r += t2 - t1;
    __nanosleep(5000);
  }
  out[0] = (uint64_t)f;
  out[1] = (uint64_t)r;
  out[2] = acc;
}

// one thread: time fences and host-word reads while other kernels load the link
__global__ void probe_latency(const volatile uint64_t* host_word, uint64_t* out, int iters) {
  long long f = 0, r = 0, q = 0;
  uint64_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    long long t0 = clock64();
    __threadfence();
    long long t1 = clock64();
    acc += *host_word;
    long long t2 = clock64();
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    long long t3 = clock64();
    f += t1 - t0;
    r += t2 - t1;
    q += t3 - t2;
    __nanosleep(2000);
  }
  out[0] = (uint64_t)f;
  out[1] = (uint64_t)r;
  out[2] = acc;
  out[3] = (uint64_t)q;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int main() {
  const uint64_t bytes = 512ull << 20;
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  void *d0, *d1, *h0, *h1, *hw;
  CK(cudaMalloc(&d0, bytes));
  CK(cudaMalloc(&d1, bytes));
  CK(cudaHostAlloc(&h0, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h1, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&hw, 4096, cudaHostAllocMapped));
  CK(cudaMemset(d0, 1, bytes));
  CK(cudaMemset(d1, 2, bytes));
  void *h0d, *h1d, *hwd;
  CK(cudaHostGetDevicePointer(&h0d, h0, 0));
  CK(cudaHostGetDevicePointer(&h1d, h1, 0));
  CK(cudaHostGetDevicePointer(&hwd, hw, 0));
  uint64_t* dout;
  CK(cudaMalloc(&dout, 64));
  cudaStream_t s0, s1, s2;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a0, a1, b0, b1;
  CK(cudaEventCreate(&a0));
  CK(cudaEventCreate(&a1));
  CK(cudaEventCreate(&b0));
  CK(cudaEventCreate(&b1));
  const uint64_t nv = bytes / 16;
  const int reps = 3;
  double best[6] = {0, 0, 0, 0, 0, 0};
  for (int rep = 0; rep < reps; ++rep) {
    // CE D2H, CE H2D, CE both
    CK(cudaEventRecord(a0, s0));
    CK(cudaMemcpyAsync(h0, d0, bytes, cudaMemcpyDeviceToHost, s0));
    CK(cudaEventRecord(a1, s0));
    CK(cudaStreamSynchronize(s0));
    double g = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    if (g > best[0]) best[0] = g;
    CK(cudaEventRecord(a0, s0));
    CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s0));
    CK(cudaEventRecord(a1, s0));
    CK(cudaStreamSynchronize(s0));
    g = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    if (g > best[1]) best[1] = g;
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a0, s0));
    CK(cudaStreamWaitEvent(s1, a0, 0));
    CK(cudaMemcpyAsync(h0, d0, bytes, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1));
    CK(cudaEventRecord(b1, s1));
    CK(cudaStreamWaitEvent(s0, b1, 0));
    CK(cudaEventRecord(a1, s0));
    CK(cudaStreamSynchronize(s0));
    g = 2.0 * bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    if (g > best[2]) best[2] = g;
    // SM D2H, SM H2D, SM both (two concurrent kernels, half the SMs each)
    const int grid = sms * 4;
    CK(cudaEventRecord(a0, s0));
    sm_copy<<<grid, 256, 0, s0>>>((V4*)h0d, (const V4*)d0, nv);
    CK(cudaEventRecord(a1, s0));
    CK(cudaStreamSynchronize(s0));
    g = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    if (g > best[3]) best[3] = g;
    CK(cudaEventRecord(a0, s0));
    sm_copy<<<grid, 256, 0, s0>>>((V4*)d1, (const V4*)h1d, nv);
    CK(cudaEventRecord(a1, s0));
    CK(cudaStreamSynchronize(s0));
    g = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    if (g > best[4]) best[4] = g;
    CK(cudaEventRecord(a0, s0));
    CK(cudaStreamWaitEvent(s1, a0, 0));
    sm_copy<<<grid / 2, 256, 0, s0>>>((V4*)h0d, (const V4*)d0, nv);
    sm_copy<<<grid / 2, 256, 0, s1>>>((V4*)d1, (const V4*)h1d, nv);
    CK(cudaEventRecord(b1, s1));
    CK(cudaStreamWaitEvent(s0, b1, 0));
    CK(cudaEventRecord(a1, s0));
    CK(cudaStreamSynchronize(s0));
    g = 2.0 * bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    if (g > best[5]) best[5] = g;
  }
  // warp-per-chunk copies, 64 KiB chunks, without / with a system fence per chunk
  double chunked[4][3] = {};
  const uint32_t cv = (64u << 10) / 16;
  for (int fence = 0; fence < 4; ++fence)
    for (int rep = 0; rep < reps; ++rep) {
      const int grid = sms;
      CK(cudaEventRecord(a0, s0));
      chunk_copy<<<grid, 256, 0, s0>>>((V4*)h0d, (const V4*)d0, nv, cv, fence);
      CK(cudaEventRecord(a1, s0));
      CK(cudaStreamSynchronize(s0));
      double g = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
      if (g > chunked[fence][0]) chunked[fence][0] = g;
      CK(cudaEventRecord(a0, s0));
      chunk_copy<<<grid, 256, 0, s0>>>((V4*)d1, (const V4*)h1d, nv, cv, fence);
      CK(cudaEventRecord(a1, s0));
      CK(cudaStreamSynchronize(s0));
      g = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
      if (g > chunked[fence][1]) chunked[fence][1] = g;
      CK(cudaEventRecord(a0, s0));
      CK(cudaStreamWaitEvent(s1, a0, 0));
      chunk_copy<<<grid / 2, 256, 0, s0>>>((V4*)h0d, (const V4*)d0, nv, cv, fence);
      chunk_copy<<<grid / 2, 256, 0, s1>>>((V4*)d1, (const V4*)h1d, nv, cv, fence);
      CK(cudaEventRecord(b1, s1));
      CK(cudaStreamWaitEvent(s0, b1, 0));
      CK(cudaEventRecord(a1, s0));
      CK(cudaStreamSynchronize(s0));
      g = 2.0 * bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
      if (g > chunked[fence][2]) chunked[fence][2] = g;
    }
  for (int f = 0; f < 4; ++f)
    std::fprintf(stderr, "chunked fence=%d asm=%d d2h %.2f h2d %.2f both %.2f\n", f & 1, f >> 1, chunked[f][0],
                 chunked[f][1], chunked[f][2]);
  // bulk-async (TMA) staged copies, 64 KiB chunks
  {
    const size_t smem = 8 * 2 * kPiece;
    CK(cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int g : {16, 32, 48, 74, 148}) {
      double best3[3] = {0, 0, 0};
      for (int rep = 0; rep < reps; ++rep) {
        CK(cudaEventRecord(a0, s0));
        tma_copy<<<g, 256, smem, s0>>>((uint8_t*)h0d, (const uint8_t*)d0, bytes, 64u << 10);
        CK(cudaEventRecord(a1, s0));
        CK(cudaStreamSynchronize(s0));
        best3[0] = std::max(best3[0], bytes / (time_ms(a0, a1) * 1e-3) / 1e9);
        CK(cudaEventRecord(a0, s0));
        tma_copy<<<g, 256, smem, s0>>>((uint8_t*)d1, (const uint8_t*)h1d, bytes, 64u << 10);
        CK(cudaEventRecord(a1, s0));
        CK(cudaStreamSynchronize(s0));
        best3[1] = std::max(best3[1], bytes / (time_ms(a0, a1) * 1e-3) / 1e9);
        CK(cudaEventRecord(a0, s0));
        CK(cudaStreamWaitEvent(s1, a0, 0));
        tma_copy<<<g, 256, smem, s0>>>((uint8_t*)h0d, (const uint8_t*)d0, bytes, 64u << 10);
        tma_copy<<<g, 256, smem, s1>>>((uint8_t*)d1, (const uint8_t*)h1d, bytes, 64u << 10);
        CK(cudaEventRecord(b1, s1));
        CK(cudaStreamWaitEvent(s0, b1, 0));
        CK(cudaEventRecord(a1, s0));
        CK(cudaStreamSynchronize(s0));
        best3[2] = std::max(best3[2], 2.0 * bytes / (time_ms(a0, a1) * 1e-3) / 1e9);
      }
      std::fprintf(stderr, "tma ctas=%d d2h %.2f h2d %.2f both(2 kernels x %d ctas) %.2f\n", g, best3[0], best3[1], g,
                   best3[2]);
    }
  }
  // copy engines fed one 64 KiB block per call from one host thread (the CE proxy's
  // pattern): issue rate and throughput, one direction and both (alternating streams)
  {
    const uint64_t blk = 64 << 10, nb = bytes / blk;
    for (int both = 0; both < 2; ++both) {
      double best_g = 0, best_us = 1e9;
      for (int rep = 0; rep < reps; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a0, s0));
        CK(cudaStreamWaitEvent(s1, a0, 0));
        const auto t0 = std::chrono::steady_clock::now();
        for (uint64_t i = 0; i < nb; ++i) {
          const uint64_t j = (i * 2654435761ull) % nb;  // scattered host blocks
          CK(cudaMemcpyAsync((uint8_t*)h0 + j * blk, (uint8_t*)d0 + i * blk, blk, cudaMemcpyDeviceToHost, s0));
          if (both)
            CK(cudaMemcpyAsync((uint8_t*)d1 + i * blk, (uint8_t*)h1 + j * blk, blk, cudaMemcpyHostToDevice, s1));
        }
        const auto t1 = std::chrono::steady_clock::now();
        CK(cudaEventRecord(b1, s1));
        CK(cudaStreamWaitEvent(s0, b1, 0));
        CK(cudaEventRecord(a1, s0));
        CK(cudaStreamSynchronize(s0));
        const double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / (nb * (both ? 2 : 1));
        best_us = std::min(best_us, us);
        best_g = std::max(best_g, (both ? 2.0 : 1.0) * bytes / (time_ms(a0, a1) * 1e-3) / 1e9);
      }
      std::fprintf(stderr, "ce per-block %s: %.2f GB/s, %.2f us per cudaMemcpyAsync call\n", both ? "both" : "d2h",
                   best_g, best_us);
    }
  }
  // LSU copies with the same CTA counts, both directions concurrently
  for (int g : {16, 32, 48, 74}) {
    double bb = 0;
    for (int rep = 0; rep < reps; ++rep) {
      CK(cudaEventRecord(a0, s0));
      CK(cudaStreamWaitEvent(s1, a0, 0));
      chunk_copy<<<g, 256, 0, s0>>>((V4*)h0d, (const V4*)d0, nv, cv, 3);
      chunk_copy<<<g, 256, 0, s1>>>((V4*)d1, (const V4*)h1d, nv, cv, 3);
      CK(cudaEventRecord(b1, s1));
      CK(cudaStreamWaitEvent(s0, b1, 0));
      CK(cudaEventRecord(a1, s0));
      CK(cudaStreamSynchronize(s0));
      bb = std::max(bb, 2.0 * bytes / (time_ms(a0, a1) * 1e-3) / 1e9);
    }
    std::fprintf(stderr, "lsu both(2 kernels x %d ctas) %.2f\n", g, bb);
  }
  // D2H writer-count sweep: throughput vs the fence / L2-read latency it imposes
  for (int g : {2, 4, 8, 16, 32, 74, 148}) {
    const int iters = 100;
    CK(cudaEventRecord(a0, s0));
    chunk_copy<<<g, 256, 0, s0>>>((V4*)h0d, (const V4*)d0, nv, cv, 3);
    CK(cudaEventRecord(a1, s0));
    probe_l2<<<1, 32, 0, s2>>>((const volatile uint64_t*)d1, dout, iters);
    CK(cudaDeviceSynchronize());
    uint64_t o[3];
    CK(cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost));
    const double gbs = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    std::fprintf(stderr, "d2h ctas=%d warps=%d %.2f GB/s  fence %.2f us  l2 read %.2f us\n", g, g * 8, gbs,
                 o[0] / (double)iters / (clk * 1e-3), o[1] / (double)iters / (clk * 1e-3));
  }
  for (int g : {2, 4, 8, 16, 32, 74, 148}) {
    const int iters = 100;
    CK(cudaEventRecord(a0, s0));
    chunk_copy<<<g, 256, 0, s0>>>((V4*)d1, (const V4*)h1d, nv, cv, 3);
    CK(cudaEventRecord(a1, s0));
    probe_l2<<<1, 32, 0, s2>>>((const volatile uint64_t*)d0, dout, iters);
    CK(cudaDeviceSynchronize());
    uint64_t o[3];
    CK(cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost));
    const double gbs = bytes / (time_ms(a0, a1) * 1e-3) / 1e9;
    std::fprintf(stderr, "h2d ctas=%d warps=%d %.2f GB/s  fence %.2f us  l2 read %.2f us\n", g, g * 8, gbs,
                 o[0] / (double)iters / (clk * 1e-3), o[1] / (double)iters / (clk * 1e-3));
  }
  // latency of a fence / a host read: idle, then under SM copy load in both directions
  uint64_t lat[2][3];
  const int iters = 200;
  for (int loaded = 0; loaded < 2; ++loaded) {
    if (loaded) {
      chunk_copy<<<(sms - 2) / 2, 256, 0, s0>>>((V4*)h0d, (const V4*)d0, nv, cv, 1);
      chunk_copy<<<(sms - 2) / 2, 256, 0, s1>>>((V4*)d1, (const V4*)h1d, nv, cv, 1);
    }
    probe_latency<<<1, 1, 0, s2>>>((const volatile uint64_t*)hwd, dout, iters);
    CK(cudaDeviceSynchronize());
    uint64_t o[4];
    CK(cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost));
    lat[loaded][0] = o[0];
    lat[loaded][1] = o[1];
    lat[loaded][2] = o[3];
  }
  const double ghz = clk * 1e-6;
  std::printf(
      "{\"bytes\": %llu, \"sms\": %d, \"ce_d2h_gbs\": %.2f, \"ce_h2d_gbs\": %.2f, \"ce_both_gbs\": %.2f, "
      "\"sm_d2h_gbs\": %.2f, \"sm_h2d_gbs\": %.2f, \"sm_both_gbs\": %.2f, "
      "\"fence_us_idle\": %.3f, \"host_read_us_idle\": %.3f, \"fence_us_loaded\": %.3f, \"host_read_us_loaded\": %.3f, "
      "\"fence_acq_rel_us_idle\": %.3f, \"fence_acq_rel_us_loaded\": %.3f, "
      "\"clock_ghz_attr\": %.3f}\n",
      (unsigned long long)bytes, sms, best[0], best[1], best[2], best[3], best[4], best[5],
      lat[0][0] / (double)iters / ghz / 1e3, lat[0][1] / (double)iters / ghz / 1e3,
      lat[1][0] / (double)iters / ghz / 1e3, lat[1][1] / (double)iters / ghz / 1e3,
      lat[0][2] / (double)iters / ghz / 1e3, lat[1][2] / (double)iters / ghz / 1e3, ghz);
  return 0;
}
