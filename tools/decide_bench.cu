// decide_bench.cu — cycles per serial multi-candidate decision (choose_rail's telemetry
// window + round robin, scheduler.cpp:156-173) in two shapes:
//   V1 warp: lane per candidate, warp min-reduction (REDUX on the double bit pattern),
//      ballot of the window, round-robin index (the engine's decide_block loop);
//   V2 lane: one lane holds every candidate's score (n <= 8), min / window / pick in
//      registers, no warp collectives.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o decide_bench tools/decide_bench.cu
#include <cstdio>
#include <cstdint>
#define FULL 0xffffffffu

__device__ __forceinline__ double warp_min_pos(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const uint32_t hi = (uint32_t)(b >> 32), lo = (uint32_t)b;
  const uint32_t mhi = __reduce_min_sync(FULL, hi);
  const uint32_t mlo = __reduce_min_sync(FULL, hi == mhi ? lo : 0xffffffffu);
  return __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
}
__device__ __forceinline__ int nth_set_bit(uint32_t m, uint32_t k) {
  for (uint32_t i = 0; i < k; ++i) m &= m - 1;
  return __ffs(m) - 1;
}

__global__ void v1(int n, int iters, const double* bw, double* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  const bool elig = lane < n;
  double b0 = 0.0, b1 = 1.0, pen = 1.0, w = elig ? bw[lane] : 1.0;
  int64_t q = 0;
  const uint64_t l = 65536;
  uint64_t rr = 0;
  const double inf = __longlong_as_double(0x7ff0000000000000LL), onept = 1.05;
  double acc = 0;
  const long long t0 = clock64();
  for (int j = 0; j < iters; ++j) {
    double score = inf, x = 0, pred = 0;
    if (elig) {
      x = __ddiv_rn(__dadd_rn(__ll2double_rn(q), __ull2double_rn(l)), w);
      pred = __dadd_rn(b0, __dmul_rn(b1, x));
      score = __dmul_rn(pen, pred);
    }
    const double bound = __dmul_rn(onept, warp_min_pos(score));
    const uint32_t wm = __ballot_sync(FULL, elig && score <= bound);
    const uint32_t nw = __popc(wm);
    const int pick = nw == 1 ? __ffs(wm) - 1 : nth_set_bit(wm, (uint32_t)rr % nw);
    rr++;
    if (lane == pick) { q += l; acc += x; }
  }
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
  out[lane] = acc;
}

// one lane, n <= 8 candidates in registers
__global__ void v2(int n, int iters, const double* bw, double* out, long long* cyc) {
  if (threadIdx.x != 0) return;
  double s[8], x[8], w[8];
  int64_t q[8];
  for (int i = 0; i < 8; ++i) { w[i] = i < n ? bw[i] : 1.0; q[i] = 0; }
  const uint64_t l = 65536;
  const double b0 = 0.0, b1 = 1.0, pen = 1.0, onept = 1.05;
  uint64_t rr = 0;
  double acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = __ddiv_rn(__dadd_rn(__ll2double_rn(q[i]), __ull2double_rn(l)), w[i]);
    s[i] = __dmul_rn(pen, __dadd_rn(b0, __dmul_rn(b1, x[i])));
  }
  const long long t0 = clock64();
  for (int j = 0; j < iters; ++j) {
    double smin = s[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) if (i < n && s[i] < smin) smin = s[i];
    const double bound = __dmul_rn(onept, smin);
    uint32_t wm = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) if (i < n && s[i] <= bound) wm |= 1u << i;
    const uint32_t nw = __popc(wm);
    const int pick = nw == 1 ? __ffs(wm) - 1 : nth_set_bit(wm, (uint32_t)rr % nw);
    rr++;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i == pick) {
        acc += x[i];
        q[i] += l;
        x[i] = __ddiv_rn(__dadd_rn(__ll2double_rn(q[i]), __ull2double_rn(l)), w[i]);
        s[i] = __dmul_rn(pen, __dadd_rn(b0, __dmul_rn(b1, x[i])));
      }
  }
  const long long t1 = clock64();
  *cyc = t1 - t0;
  out[0] = acc;
}

int main() {
  double* bw; double* out; long long* cyc;
  cudaMalloc(&bw, 64 * 8); cudaMalloc(&out, 64 * 8); cudaMalloc(&cyc, 8);
  double h[32];
  for (int i = 0; i < 32; ++i) h[i] = 8e11 / (1 + (i & 1));
  cudaMemcpy(bw, h, sizeof(h), cudaMemcpyHostToDevice);
  const int iters = 4096;
  for (int n : {2, 4, 8}) {
    long long c1 = 0, c2 = 0;
    v1<<<1, 32>>>(n, iters, bw, out, cyc); cudaDeviceSynchronize();
    v1<<<1, 32>>>(n, iters, bw, out, cyc); cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
    v2<<<1, 32>>>(n, iters, bw, out, cyc); cudaDeviceSynchronize();
    v2<<<1, 32>>>(n, iters, bw, out, cyc); cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"candidates\": %d, \"warp_cycles_per_decision\": %.1f, \"lane_cycles_per_decision\": %.1f}\n", n,
           (double)c1 / iters, (double)c2 / iters);
  }
  return 0;
}
