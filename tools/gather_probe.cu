// Random 8-byte gather throughput on one B200, per SM per clock.
//
// The C3/C5 kernels are bound by their x gathers (uniform offsets over
// +-32767: every gather its own 32-byte sector).  This probe measures what a
// gather costs from each place x could live:
//   global   x window (W doubles) in HBM/L2, ld.global (L1 allocating)
//   global.cg  same, L1 bypassed (L2 only)
//   smem     x window of 8192 doubles (64 KiB) in the CTA's shared memory
//   dsmem    x spread over a cluster's shared memories (mapa + ld.shared::cluster)
// each with all 32 lanes active or only `active` lanes (the tiled kernel's
// lane occupancy).  Output: one line per case, gathers per SM per clock
// (cycles from clock64 inside the kernel, max over CTAs).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

constexpr int kIters = 4096;
constexpr int kSmemElems = 8192;

__device__ __forceinline__ uint32_t xs(uint32_t& s) {
  s ^= s << 13;
  s ^= s >> 17;
  s ^= s << 5;
  return s;
}

__device__ __forceinline__ double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// mode 0 global (ldg), 1 global.cg, 2 smem
template <int MODE>
__global__ void gather_kernel(const double* __restrict__ x, uint32_t mask, int active,
                              unsigned long long* cycles, double* sink) {
  extern __shared__ double sx[];
  if (MODE == 2) {
    for (int i = threadIdx.x; i < kSmemElems; i += blockDim.x) sx[i] = x[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  uint32_t s = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  double acc = 0.0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (lane < active) {
#pragma unroll 8
    for (int it = 0; it < kIters; ++it) {
      const uint32_t i = xs(s) & mask;
      if (MODE == 0) acc += __ldg(x + i);
      else if (MODE == 1) acc += ld_cg(x + i);
      else acc += sx[i & (kSmemElems - 1)];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 12345.678) sink[0] = acc;
}

__global__ void dsmem_kernel(const double* __restrict__ x, int active, unsigned long long* cycles,
                             double* sink) {
  extern __shared__ double sx[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < kSmemElems; i += blockDim.x) sx[i] = x[i];
  cl.sync();
  const int lane = threadIdx.x & 31;
  const unsigned nr = cl.num_blocks();
  uint32_t s = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  double acc = 0.0;
  const unsigned long long t0 = clock64();
  if (lane < active) {
#pragma unroll 8
    for (int it = 0; it < kIters / 4; ++it) {
      const uint32_t h = xs(s);
      const double* p = cl.map_shared_rank(sx + (h & (kSmemElems - 1)), (h >> 16) % nr);
      acc += *p;
    }
  }
  const unsigned long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t nx = size_t(1) << 22;  // 32 MiB of x (L2-resident)
  double* x;
  cudaMalloc(&x, nx * sizeof(double));
  std::vector<double> h(nx);
  for (size_t i = 0; i < nx; ++i) h[i] = 1.0 + 1e-9 * double(i);
  cudaMemcpy(x, h.data(), nx * sizeof(double), cudaMemcpyHostToDevice);
  unsigned long long* cyc;
  double* sink;
  const int threads = 1024;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms * 8);
  cudaMalloc(&sink, 8);
  auto report = [&](const char* name, int active, int ctas, int iters) {
    std::vector<unsigned long long> c(ctas);
    cudaMemcpy(c.data(), cyc, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    const double per_sm = double(ctas) / sms * (threads / 32) * active * double(iters);
    printf("%-26s active=%2d  gathers/SM/clk = %6.2f   (cycles %llu)\n", name, active,
           per_sm / double(mx), mx);
  };
  cudaFuncSetAttribute(gather_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemElems * 8);
  cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemElems * 8);
  for (int active : {32, 12}) {
    for (uint32_t win : {1u << 16, 1u << 22}) {  // 512 KiB window, 32 MiB window
      char nm[64];
      gather_kernel<0><<<sms, threads>>>(x, win - 1, active, cyc, sink);
      cudaDeviceSynchronize();
      snprintf(nm, sizeof nm, "global ldg win=%uK", win / 1024 * 8);
      report(nm, active, sms, kIters);
      gather_kernel<1><<<sms, threads>>>(x, win - 1, active, cyc, sink);
      cudaDeviceSynchronize();
      snprintf(nm, sizeof nm, "global .cg win=%uK", win / 1024 * 8);
      report(nm, active, sms, kIters);
    }
    gather_kernel<2><<<sms, threads, kSmemElems * 8>>>(x, kSmemElems - 1, active, cyc, sink);
    cudaDeviceSynchronize();
    report("smem 64K", active, sms, kIters);
    for (int csz : {2, 4, 8}) {
      cudaLaunchConfig_t cfg = {};
      const int ctas = (sms / csz) * csz;
      cfg.gridDim = dim3(ctas);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = kSmemElems * 8;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, dsmem_kernel, (const double*)x, active, cyc, sink);
      cudaError_t e2 = cudaDeviceSynchronize();
      if (e != cudaSuccess || e2 != cudaSuccess) {
        printf("dsmem cluster %d: %s / %s\n", csz, cudaGetErrorString(e), cudaGetErrorString(e2));
        cudaGetLastError();
        continue;
      }
      char nm[64];
      snprintf(nm, sizeof nm, "dsmem cluster=%d", csz);
      report(nm, active, ctas, kIters / 4);
    }
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d  clock attr %d kHz\n", sms, clk);
  return 0;
}
