// Copy-engine issue-rate probe: how fast can host threads drive the copy engines with
// many small slices (one cudaMemcpyAsync per slice, 1..8 issuing threads, or one
// cudaMemcpy2DAsync per strided run), and does a copy-engine rail add bandwidth beside an
// SM copy rail (the spray question)?
//   single GPU: 4096 x 64 KiB blocks HBM <-> pinned host through a random block table
//   two GPUs  : 4096 x 256 KiB slices GPU0 -> GPU1 (C2 shape), same questions over NVLink
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ce_issue_peak tools/ce_issue_peak.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

struct V4 { uint32_t a, b, c, d; };

// warp-per-block copy through a block table (the engine worker's access pattern)
__global__ void __launch_bounds__(256) table_copy(uint8_t* dst, const uint8_t* src, const uint32_t* dtab,
                                                  const uint32_t* stab, uint32_t nblk, uint32_t blk) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nv = blk / 16;
  for (uint32_t c = warp; c < nblk; c += nwarps) {
    const V4* s = reinterpret_cast<const V4*>(src + (uint64_t)stab[c] * blk);
    V4* d = reinterpret_cast<V4*>(dst + (uint64_t)dtab[c] * blk);
    for (uint32_t i = lane; i < nv; i += 8 * 32) {
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

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Job {
  std::vector<void*> dst, src;
  std::vector<size_t> len;
};

// issue the job per call from `threads` host threads, thread t taking every t-th copy on
// its own stream; returns issue seconds
static std::vector<cudaStream_t> g_streams;
static double issue(const Job& j, cudaStream_t s, int threads) {
  const double t0 = now_s();
  const size_t n = j.dst.size();
  if (threads <= 1) {
    for (size_t i = 0; i < n; ++i) CK(cudaMemcpyAsync(j.dst[i], j.src[i], j.len[i], cudaMemcpyDefault, s));
  } else {
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t)
      ts.emplace_back([&, t] {
        for (size_t i = t; i < n; i += threads)
          CK(cudaMemcpyAsync(j.dst[i], j.src[i], j.len[i], cudaMemcpyDefault, g_streams[t]));
      });
    for (auto& x : ts) x.join();
    for (int t = 0; t < threads; ++t) CK(cudaStreamSynchronize(g_streams[t]));
  }
  return now_s() - t0;
}

static Job table_job(uint8_t* dst, const uint8_t* src, const std::vector<uint32_t>& dt, const std::vector<uint32_t>& st,
                     size_t blk) {
  Job j;
  for (size_t i = 0; i < dt.size(); ++i) {
    j.dst.push_back(dst + (size_t)dt[i] * blk);
    j.src.push_back(const_cast<uint8_t*>(src) + (size_t)st[i] * blk);
    j.len.push_back(blk);
  }
  return j;
}

int main(int argc, char** argv) {
  int ngpu = 0;
  CK(cudaGetDeviceCount(&ngpu));
  const size_t blk = 64 << 10;
  const uint32_t nb = 4096;
  const size_t pool = blk * nb;
  CK(cudaSetDevice(0));
  uint8_t *hbm, *hbm2, *host, *host2;
  CK(cudaMalloc(&hbm, pool));
  CK(cudaMalloc(&hbm2, pool));
  CK(cudaHostAlloc(&host, pool, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc(&host2, pool, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaMemset(hbm, 1, pool));
  std::memset(host2, 2, pool);
  std::vector<uint32_t> id(nb), p1(nb), p2(nb);
  for (uint32_t i = 0; i < nb; ++i) id[i] = p1[i] = p2[i] = i;
  std::mt19937 rng(7);
  std::shuffle(p1.begin(), p1.end(), rng);
  std::shuffle(p2.begin(), p2.end(), rng);
  uint32_t *did, *dp1, *dp2;
  CK(cudaMalloc(&did, nb * 4));
  CK(cudaMalloc(&dp1, nb * 4));
  CK(cudaMalloc(&dp2, nb * 4));
  CK(cudaMemcpy(did, id.data(), nb * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dp1, p1.data(), nb * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dp2, p2.data(), nb * 4, cudaMemcpyHostToDevice));
  uint8_t *mh, *mh2;
  CK(cudaHostGetDevicePointer((void**)&mh, host, 0));
  CK(cudaHostGetDevicePointer((void**)&mh2, host2, 0));

  cudaStream_t s1, s2, s3;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  for (int t = 0; t < 8; ++t) {
    cudaStream_t x;
    CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    g_streams.push_back(x);
  }
  const Job d2h = table_job(host, hbm, p1, id, blk);   // offload: hbm[i] -> host[p1[i]]
  const Job h2d = table_job(hbm2, host2, id, p2, blk);  // reload: host2[p2[i]] -> hbm2[i]

  auto gbs = [](double bytes, double s) { return bytes / s / 1e9; };
  std::printf("{\n");
  // 1) one direction, one thread
  for (int batch : {1, 2, 4, 8}) {
    for (int dir = 0; dir < 2; ++dir) {
      const Job& j = dir ? h2d : d2h;
      issue(j, s1, batch);
      CK(cudaStreamSynchronize(s1));
      double best = 1e9, ibest = 1e9;
      for (int r = 0; r < 3; ++r) {
        const double t0 = now_s();
        const double it = issue(j, s1, batch);
        CK(cudaStreamSynchronize(s1));
        best = std::min(best, now_s() - t0);
        ibest = std::min(ibest, it);
      }
      std::printf("  \"ce_%s_threads%d\": {\"gbs\": %.2f, \"issue_us_per_copy\": %.3f},\n", dir ? "h2d" : "d2h", batch,
                  gbs(pool, best), ibest / nb * 1e6);
    }
  }
  // 2) both directions on copy engines, two threads
  for (int batch : {1}) {
    double best = 1e9;
    for (int r = 0; r < 3; ++r) {
      CK(cudaDeviceSynchronize());
      const double t0 = now_s();
      std::thread t([&] { issue(h2d, s2, batch); });
      issue(d2h, s1, batch);
      t.join();
      CK(cudaStreamSynchronize(s1));
      CK(cudaStreamSynchronize(s2));
      best = std::min(best, now_s() - t0);
    }
    std::printf("  \"ce_both_threads%d_gbs\": %.2f,\n", batch, gbs(2.0 * pool, best));
  }
  // 3) hybrid: SM kernel one direction (48 CTAs), CE batch the other; and SM both
  for (int mode = 0; mode < 3; ++mode) {
    double best = 1e9;
    for (int r = 0; r < 4; ++r) {
      CK(cudaDeviceSynchronize());
      const double t0 = now_s();
      if (mode == 0) {  // SM d2h + CE h2d
        table_copy<<<48, 256, 0, s3>>>(mh, hbm, dp1, did, nb, blk);
        issue(h2d, s1, 4);
      } else if (mode == 1) {  // SM h2d + CE d2h
        table_copy<<<48, 256, 0, s3>>>(hbm2, mh2, did, dp2, nb, blk);
        issue(d2h, s1, 4);
      } else {  // SM both (two kernels)
        table_copy<<<24, 256, 0, s3>>>(mh, hbm, dp1, did, nb, blk);
        table_copy<<<24, 256, 0, s1>>>(hbm2, mh2, did, dp2, nb, blk);
      }
      CK(cudaStreamSynchronize(s1));
      CK(cudaStreamSynchronize(s3));
      best = std::min(best, now_s() - t0);
    }
    const char* nm[] = {"sm_d2h_ce_h2d", "sm_h2d_ce_d2h", "sm_both"};
    std::printf("  \"hybrid_%s_gbs\": %.2f,\n", nm[mode], gbs(2.0 * pool, best));
  }
  // 4) NVLink: GPU0 -> GPU1, 4096 x 256 KiB, CE per call / batched, SM, SM + CE split
  if (ngpu >= 2) {
    const size_t sl = 256 << 10;
    const size_t big = sl * nb;
    uint8_t *a, *b;
    CK(cudaMalloc(&a, big));
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&b, big));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaMemset(a, 3, big));
    Job pj = table_job(b, a, id, id, sl);
    for (int batch : {1, 2, 4}) {
      double best = 1e9, ib = 1e9;
      for (int r = 0; r < 4; ++r) {
        CK(cudaDeviceSynchronize());
        const double t0 = now_s();
        ib = std::min(ib, issue(pj, s1, batch));
        CK(cudaStreamSynchronize(s1));
        best = std::min(best, now_s() - t0);
      }
      std::printf("  \"peer_ce_threads%d\": {\"gbs\": %.2f, \"issue_us_per_copy\": %.3f},\n", batch, gbs(big, best),
                  ib / nb * 1e6);
    }
    // CE alone on half the slices: every other slice as 2D copies of R rows, or
    // contiguous runs of K slices as 1D copies
    for (int rows : {16, 64, 2048}) {
      double best = 1e9;
      for (int r = 0; r < 4; ++r) {
        CK(cudaDeviceSynchronize());
        const double t0 = now_s();
        for (uint32_t i = 0; i < nb; i += 2 * rows)
          CK(cudaMemcpy2DAsync(b + i * sl, 2 * sl, a + i * sl, 2 * sl, sl, std::min<uint32_t>(rows, (nb - i) / 2),
                               cudaMemcpyDefault, s1));
        CK(cudaStreamSynchronize(s1));
        best = std::min(best, now_s() - t0);
      }
      std::printf("  \"peer_ce_2d_stride2_rows%d_gbs\": %.2f,\n", rows, gbs(big / 2, best));
    }
    for (int run : {8, 32, 128}) {
      double best = 1e9;
      for (int r = 0; r < 4; ++r) {
        CK(cudaDeviceSynchronize());
        const double t0 = now_s();
        for (uint32_t i = 0; i < nb; i += 2 * run)
          CK(cudaMemcpyAsync(b + i * sl, a + i * sl, run * sl, cudaMemcpyDefault, s1));
        CK(cudaStreamSynchronize(s1));
        best = std::min(best, now_s() - t0);
      }
      std::printf("  \"peer_ce_1d_run%d_gbs\": %.2f,\n", run, gbs(big / 2, best));
    }
    // SM + CE: CE takes the first f/32 slices of every 32 (one 1D copy each run), SM the rest
    for (int frac_ce : {0, 4, 8, 12, 16, 32}) {
      std::vector<uint32_t> sm_ids;
      for (uint32_t i = 0; i < nb; ++i)
        if ((i % 32) >= (uint32_t)frac_ce) sm_ids.push_back(i);
      uint32_t* dsm;
      CK(cudaMalloc(&dsm, std::max<size_t>(1, sm_ids.size()) * 4));
      if (!sm_ids.empty()) CK(cudaMemcpy(dsm, sm_ids.data(), sm_ids.size() * 4, cudaMemcpyHostToDevice));
      double best = 1e9;
      for (int r = 0; r < 4; ++r) {
        CK(cudaDeviceSynchronize());
        const double t0 = now_s();
        if (!sm_ids.empty()) table_copy<<<148 * 2, 256, 0, s3>>>(b, a, dsm, dsm, sm_ids.size(), sl);
        CK(cudaGetLastError());
        if (frac_ce)
          for (uint32_t i = 0; i < nb; i += 32) CK(cudaMemcpyAsync(b + i * sl, a + i * sl, frac_ce * sl, cudaMemcpyDefault, s1));
        CK(cudaStreamSynchronize(s1));
        CK(cudaStreamSynchronize(s3));
        best = std::min(best, now_s() - t0);
      }
      std::printf("  \"peer_sm_plus_ce_%d_of_32_gbs\": %.2f,\n", frac_ce, gbs(big, best));
      CK(cudaFree(dsm));
    }
  }
  std::printf("  \"gpus\": %d\n}\n", ngpu);
  return 0;
}
