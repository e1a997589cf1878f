// PCIe probe (developer tool): host<->device bandwidth of the paths the
// host-buffer step uses -- copy-engine H2D / D2H of pinned memory and a
// kernel's zero-copy stores into mapped pinned memory (8 B and 16 B per
// thread, whole rows like k_step's write-through) -- so the e2e line can be
// read against what this box's link delivers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pcie_probe tools/pcie_probe.cu
//   tools/pcie_probe [MiB]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));           \
      std::exit(1);                                                           \
    }                                                                         \
  } while (0)

__global__ void k_store8(const double* __restrict__ src, double* dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_store16(const double2* __restrict__ src, double2* dst, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// tile-shaped stores like k_step's write-through: 32-double row segments of
// 32 x 16 tiles, a fraction `every` of the tiles
__global__ void k_store_tiles(const double* __restrict__ src, double* dst, int nx, int ny,
                              int every) {
  const int tiles_x = nx / 32, tiles = tiles_x * (ny / 16);
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    if (t % every) continue;
    const int i0 = (t % tiles_x) * 32, j0 = (t / tiles_x) * 16;
    for (int c = threadIdx.x; c < 512; c += blockDim.x) {
      const size_t k = (size_t)(i0 + c % 32) + (size_t)(j0 + c / 32) * nx;
      dst[k] = src[k];
    }
  }
}

static float timed(cudaStream_t s, cudaEvent_t a, cudaEvent_t b, int reps, auto&& f) {
  f();
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(a, s));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main(int argc, char** argv) {
  size_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 2048;
  size_t bytes = mib << 20, n = bytes / 8;
  double *d, *h, *hd;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(d, 0, bytes));
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const double gb = bytes / 1e9;
  auto rep = [&](const char* what, float ms, double g) {
    std::printf("{\"path\": \"%s\", \"GB\": %.3f, \"ms\": %.3f, \"GB_s\": %.2f}\n", what, g, ms,
                g / (ms * 1e-3));
  };
  rep("h2d_memcpy", timed(s, a, b, 3, [&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s)); }), gb);
  rep("d2h_memcpy", timed(s, a, b, 3, [&] { CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s)); }), gb);
  for (int per : {2, 4, 8}) {
    char name[64];
    std::snprintf(name, sizeof name, "zero_copy_store8_%dxSM", per);
    rep(name, timed(s, a, b, 3, [&] { k_store8<<<sms * per, 256, 0, s>>>(d, hd, n); }), gb);
  }
  rep("zero_copy_store16_4xSM",
      timed(s, a, b, 3, [&] { k_store16<<<sms * 4, 256, 0, s>>>((const double2*)d, (double2*)hd, n / 2); }), gb);
  // tile-shaped write-through over a 16384-wide grid
  const int nx = 16384, ny = (int)(n / nx) / 16 * 16;
  for (int every : {1, 3}) {
    char name[64];
    std::snprintf(name, sizeof name, "zero_copy_tiles_1of%d", every);
    const double g = (double)nx * ny * 8 / every / 1e9;
    rep(name, timed(s, a, b, 3, [&] { k_store_tiles<<<sms * 4, 256, 0, s>>>(d, hd, nx, ny, every); }), g);
  }
  // zero-copy loads (k_ingest_hu's path): device reads of mapped pinned memory
  for (int per : {4, 8}) {
    char name[64];
    std::snprintf(name, sizeof name, "zero_copy_load8_%dxSM", per);
    rep(name, timed(s, a, b, 3, [&] { k_store8<<<sms * per, 256, 0, s>>>(hd, d, n); }), gb);
  }
  rep("zero_copy_load16_8xSM",
      timed(s, a, b, 3, [&] { k_store16<<<sms * 8, 256, 0, s>>>((const double2*)hd, (double2*)d, n / 2); }), gb);
  for (int every : {1, 3}) {
    char name[64];
    std::snprintf(name, sizeof name, "zero_copy_load_tiles_1of%d", every);
    const double g = (double)nx * ny * 8 / every / 1e9;
    rep(name, timed(s, a, b, 3, [&] { k_store_tiles<<<sms * 8, 256, 0, s>>>(hd, d, nx, ny, every); }), g);
  }
  // concurrent H2D (copy engine) + zero-copy stores: does the link run both directions at once?
  cudaStream_t s2;
  CK(cudaStreamCreate(&s2));
  double* d2;
  CK(cudaMalloc(&d2, bytes));
  double* h2;
  CK(cudaHostAlloc(&h2, bytes, cudaHostAllocDefault));
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a, s));
  CK(cudaMemcpyAsync(d2, h2, bytes, cudaMemcpyHostToDevice, s2));
  k_store8<<<sms * 4, 256, 0, s>>>(d, hd, n);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  rep("duplex_h2d_plus_zero_copy_store8", ms, 2 * gb);
  return 0;
}
