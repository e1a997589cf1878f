// fp64_peak.cu -- measured FP64 roof of this B200 ("B200
// FP64 peak: not measured ... builder must microbenchmark").
//
// Throughput: every thread runs 8 independent dependency chains of one FP64
// op (DFMA, DADD or DMUL) for a fixed number of iterations; grid = 148 SMs x
// 8 CTAs x 256 threads.  Timed with CUDA events over >= 1 s of work, best of
// 3.  Reported as warp-level instructions per clock per SM and as lane
// operations per second (a DFMA counts as one instruction, two flops).
// Latency: one warp, one dependent chain (cycles per dependent op, clock64).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp64_peak fp64_peak.cu
//   ./fp64_peak > profiles/fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;

template <int OP>
__global__ void k_tput(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) {
        if (OP == 0) x[c] = fma(x[c], a, b);
        else if (OP == 1) x[c] = x[c] + b;
        else x[c] = x[c] * a;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[blockIdx.x] = s;  // keeps the chains alive
}

template <int OP>
__global__ void k_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = 1.0 + 1e-3 * threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = fma(x, a, b);
      else if (OP == 1) x = x + b;
      else x = x * a;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

template <int OP>
void run(const char* name, int sms, int clock_khz, bool last) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, sizeof(long long));
  const int ctas = sms * 8, thr = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 1000;
  float ms = 0.f;
  // grow the work until one launch takes >= 1 s
  for (;;) {
    cudaEventRecord(e0);
    k_tput<OP><<<ctas, thr>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms >= 1000.f || iters > (1 << 26)) break;
    iters = (int)(iters * (ms > 1.f ? 1100.0 / ms : 16.0));
  }
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    k_tput<OP><<<ctas, thr>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double lane_ops = (double)ctas * thr * iters * 16.0 * CHAINS;
  double ops_per_s = lane_ops / (best * 1e-3);
  double warp_inst_per_clk_sm = ops_per_s / 32.0 / sms / (clock_khz * 1e3);
  // latency: one warp
  const int liters = 1 << 14;
  k_lat<OP><<<1, 32>>>(out, cyc, liters, 0.999999, 1e-9);
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  double lat = (double)c / (liters * 16.0);
  printf("    \"%s\": {\"lane_ops_per_s\": %.4e, \"warp_inst_per_clk_per_sm\": %.3f, "
         "\"dependent_latency_cycles\": %.2f, \"ms\": %.1f, \"iters\": %d}%s\n",
         name, ops_per_s, warp_inst_per_clk_sm, lat, best, iters, last ? "" : ",");
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int dev = 0, sms = 0, khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  printf("{\n  \"device\": \"%s\", \"sms\": %d, \"max_sm_clock_mhz\": %.0f,\n  \"ops\": {\n", p.name,
         sms, khz / 1e3);
  run<0>("DFMA", sms, khz, false);
  run<1>("DADD", sms, khz, false);
  run<2>("DMUL", sms, khz, true);
  printf("  },\n  \"note\": \"throughput at the clock the GPU ran (boost may be below max); "
         "lane ops = per-thread FP64 instructions (a DFMA is 2 flops)\"\n}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
