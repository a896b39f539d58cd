// Copy-engine batch probe: can one cudaMemcpyBatchAsync call carry a whole KV block table
// (4096 x 64 KiB, random block order) to the copy engines at link rate, where one
// cudaMemcpyAsync per block costs ~4 us of host time (profiles/ce_issue_peak_r01.json)?
// Measures offload (HBM -> pinned host), reload (pinned host -> HBM) and both at once on
// two streams, for per-block cudaMemcpyAsync and for cudaMemcpyBatchAsync, plus the host
// time of the submit call itself. Output: one JSON object on stdout.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ce_batch_probe tools/ce_batch_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

using clk = std::chrono::steady_clock;

struct Table {
  std::vector<void*> dst, src;
  std::vector<size_t> size;
};

static Table make_table(char* dst_pool, const char* src_pool, size_t blocks, size_t bs, uint64_t seed) {
  std::vector<size_t> a(blocks), b(blocks);
  std::iota(a.begin(), a.end(), 0);
  std::iota(b.begin(), b.end(), 0);
  std::mt19937_64 g(seed);
  std::shuffle(a.begin(), a.end(), g);
  std::shuffle(b.begin(), b.end(), g);
  Table t;
  for (size_t i = 0; i < blocks; ++i) {
    t.dst.push_back(dst_pool + a[i] * bs);
    t.src.push_back(const_cast<char*>(src_pool) + b[i] * bs);
    t.size.push_back(bs);
  }
  return t;
}

// issue one table on one stream; returns host microseconds spent in the issue call(s)
static double issue(const Table& t, cudaStream_t s, bool batch, size_t chunk) {
  auto h0 = clk::now();
  if (!batch) {
    for (size_t i = 0; i < t.dst.size(); ++i)
      CK(cudaMemcpyAsync(t.dst[i], t.src[i], t.size[i], cudaMemcpyDefault, s));
  } else {
    cudaMemcpyAttributes attr{};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    size_t idx0 = 0;
    for (size_t off = 0; off < t.dst.size(); off += chunk) {
      size_t n = std::min(chunk, t.dst.size() - off);
      size_t fail = SIZE_MAX;
      CK(cudaMemcpyBatchAsync(const_cast<void**>(t.dst.data() + off), const_cast<void**>(t.src.data() + off),
                              const_cast<size_t*>(t.size.data() + off), n, &attr, &idx0, 1, &fail, s));
    }
  }
  return std::chrono::duration<double, std::micro>(clk::now() - h0).count();
}

int main(int argc, char** argv) {
  const size_t blocks = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 4096;
  const size_t bs = (argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 64) << 10;
  const int reps = 5;
  const size_t pool = blocks * bs;
  char *dev_a, *dev_b, *host_a, *host_b;
  CK(cudaMalloc(&dev_a, pool));
  CK(cudaMalloc(&dev_b, pool));
  CK(cudaHostAlloc(&host_a, pool, cudaHostAllocDefault));
  CK(cudaHostAlloc(&host_b, pool, cudaHostAllocDefault));
  CK(cudaMemset(dev_a, 0x5a, pool));
  std::fill(host_b, host_b + pool, (char)0x3c);
  Table off = make_table(host_a, dev_a, blocks, bs, 1);  // offload HBM -> host
  Table rel = make_table(dev_b, host_b, blocks, bs, 2);  // reload host -> HBM
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));

  std::printf("{\"blocks\": %zu, \"block_bytes\": %zu", blocks, bs);
  const size_t chunks[] = {blocks, 256, 32};
  for (int mode = 0; mode < 4; ++mode) {     // 0 per-call, 1..3 batch with chunk sizes
    const bool batch = mode > 0;
    const size_t chunk = batch ? chunks[mode - 1] : 0;
    for (int dir = 0; dir < 3; ++dir) {      // 0 offload, 1 reload, 2 both
      double best = 0, issue_us = 0;
      for (int r = 0; r < reps + 1; ++r) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, s0));
        CK(cudaStreamWaitEvent(s1, e0));
        double us = 0;
        if (dir != 1) us += issue(off, s0, batch, chunk);
        if (dir != 0) us += issue(rel, s1, batch, chunk);
        CK(cudaEventRecord(e1, s0));
        CK(cudaEventRecord(e2, s1));
        CK(cudaDeviceSynchronize());
        float m1 = 0, m2 = 0;
        CK(cudaEventElapsedTime(&m1, e0, e1));
        CK(cudaEventElapsedTime(&m2, e0, e2));
        const double ms = std::max(m1, m2);
        const double bytes = (dir == 2 ? 2.0 : 1.0) * pool;
        const double gbs = bytes / (ms * 1e6);
        if (r > 0 && gbs > best) { best = gbs; issue_us = us; }
      }
      static const char* dn[] = {"offload", "reload", "both"};
      if (batch)
        std::printf(", \"batch%zu_%s_gbs\": %.2f, \"batch%zu_%s_issue_us\": %.1f", chunk, dn[dir], best, chunk, dn[dir], issue_us);
      else
        std::printf(", \"percall_%s_gbs\": %.2f, \"percall_%s_issue_us\": %.1f", dn[dir], best, dn[dir], issue_us);
    }
  }
  // correctness spot check of the last reload: every destination block holds 0x3c
  std::vector<char> chk(bs);
  CK(cudaMemcpy(chk.data(), rel.dst[blocks / 2], bs, cudaMemcpyDeviceToHost));
  const bool ok = std::all_of(chk.begin(), chk.end(), [](char c) { return c == (char)0x3c; });
  std::printf(", \"reload_bytes_ok\": %s}\n", ok ? "true" : "false");
  return 0;
}
