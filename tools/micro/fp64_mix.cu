// FP64 pipe microbenchmarks on B200: throughput of DFMA / DMUL / DADD / DSETP+FSEL streams and
// the latency of a dependent DFMA chain. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -fmad=false -o fp64_mix fp64_mix.cu ; run on one GPU.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void k_tput(int iters, double* sink) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double m = 0.999999, c = 1e-7;
  double be = 1e300;
  int best = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (KIND == 0) a[k] = __fma_rn(a[k], m, c);
      if (KIND == 1) a[k] = __dmul_rn(a[k], m);
      if (KIND == 2) a[k] = __dadd_rn(a[k], c);
      if (KIND == 3) {  // the K2 argmin tail: compare + select per value
        a[k] = __dmul_rn(a[k], m);
        const bool t = a[k] < be;
        be = t ? a[k] : be;
        best = t ? i : best;
      }
      if (KIND == 4) {  // independent compares (no chain): DMUL + DSETP + int add
        a[k] = __dmul_rn(a[k], m);
        best += a[k] < c * k ? 1 : 0;
      }
      if (KIND == 5) {  // the argmin tail with a 64-bit integer compare of the bit patterns
        a[k] = __dmul_rn(a[k], m);
        const long long x = __double_as_longlong(a[k]), y = __double_as_longlong(be);
        const bool t = x < y;
        be = t ? a[k] : be;
        best = t ? i : best;
      }
      if (KIND == 6) {  // half the values through the chain
        a[k] = __dmul_rn(a[k], m);
        if (k & 1) { const bool t = a[k] < be; be = t ? a[k] : be; best = t ? i : best; }
        else { const bool t = a[k] < c; best += t; }
      }
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678 || best == -7) sink[0] = s + be;
}

__global__ void k_lat(int iters, double* sink) {
  double a = threadIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) a = __fma_rn(a, 0.999999, 1e-7);
  if (a == 12345.678) sink[0] = a;
}

template <class K>
float time_it(K k, int blocks, int threads, int iters, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<blocks, threads>>>(64, sink);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  const double n_ops = double(blocks) * threads * iters * 8;
  const char* names[] = {"DFMA", "DMUL", "DADD", "DMUL+DSETP+2xSEL", "DMUL+DSETP indep", "DMUL+ISETP64 chain", "half chain"};
  float ms[7] = {time_it(k_tput<0>, blocks, threads, iters, sink), time_it(k_tput<1>, blocks, threads, iters, sink),
                 time_it(k_tput<2>, blocks, threads, iters, sink), time_it(k_tput<3>, blocks, threads, iters, sink),
                 time_it(k_tput<4>, blocks, threads, iters, sink), time_it(k_tput<5>, blocks, threads, iters, sink),
                 time_it(k_tput<6>, blocks, threads, iters, sink)};
  for (int k = 0; k < 7; ++k)
    printf("%-18s %.3f ms  %.3e ops/s  %.2f lane-ops/SM/clk(at %d MHz)\n", names[k], ms[k],
           n_ops / (ms[k] * 1e-3), n_ops / (ms[k] * 1e-3) / sms / (clk * 1e3), clk / 1000);
  const int li = 1 << 16;
  float lm = time_it(k_lat, 1, 32, li, sink);
  printf("DFMA dependent latency: %.2f cycles (at %d MHz)\n", lm * 1e-3 * clk * 1e3 / li, clk / 1000);
  return 0;
}
