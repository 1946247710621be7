// Host<->device transfer of frame-sized buffers on the B200 box: DMA copies (cudaMemcpyAsync
// from / to pinned memory) vs zero-copy kernels (SMs reading / writing mapped pinned memory
// with 16-byte coalesced accesses).  Device time per transfer from CUDA events, median of 50.
#include <algorithm>
#include <cstdint>
#include <chrono>
#include <cstring>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

template <typename F>
float med(F f, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> v;
  for (int i = 0; i < 60; ++i) {
    cudaEventRecord(a, s);
    f();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 10) v.push_back(ms * 1e3f);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  const size_t maxb = 16 << 20;
  uint8_t *h, *d;
  cudaHostAlloc(&h, maxb, cudaHostAllocMapped);
  cudaMalloc(&d, maxb);
  uint8_t* hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  for (size_t n : {32768ul, 262144ul, 786432ul, 1048576ul, 4194304ul, 16777216ul}) {
    const float h2d = med([&] { cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s); }, s);
    const float d2h = med([&] { cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s); }, s);
    const size_t n16 = n / 16;
    float zr[3], zw[3];
    const int grids[3] = {148, 296, 592};
    for (int g = 0; g < 3; ++g) {
      zr[g] = med([&] { zc_read<<<grids[g], 256, 0, s>>>((const uint4*)hd, (uint4*)d, n16); }, s);
      zw[g] = med([&] { zc_read<<<grids[g], 256, 0, s>>>((const uint4*)d, (uint4*)hd, n16); }, s);
    }
    printf("%8zu B: DMA H2D %7.1f us (%5.1f GB/s)  D2H %7.1f us (%5.1f GB/s) | zero-copy read %6.1f/%6.1f/%6.1f us  write %6.1f/%6.1f/%6.1f us (148/296/592 CTAs)\n",
           n, h2d, n / h2d / 1e3, d2h, n / d2h / 1e3, zr[0], zr[1], zr[2], zw[0], zw[1], zw[2]);
  }
  // two back-to-back H2D copies (rgb + mask) vs one merged copy
  const float two = med([&] {
    cudaMemcpyAsync(d, h, 786432, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d + 786432, h + 786432, 262144, cudaMemcpyHostToDevice, s);
  }, s);
  printf("rgb + mask as two H2D copies: %.1f us\n", two);
  // the same after the CPU has just written the pinned source (dirty in the CPU caches), and
  // after writing it with non-temporal stores
  std::vector<uint8_t> src(1 << 20, 7);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    std::vector<float> v;
    for (int i = 0; i < 60; ++i) {
      if (mode == 0) {
        memcpy(h, src.data(), 1 << 20);
      } else {
        for (size_t o = 0; o < (1 << 20); o += 16)
          __builtin_ia32_movntdq((__attribute__((vector_size(16))) long long*)(h + o),
                                 *(__attribute__((vector_size(16))) long long*)(src.data() + o));
        __builtin_ia32_sfence();
      }
      cudaEventRecord(a, s);
      cudaMemcpyAsync(d, h, 1 << 20, cudaMemcpyHostToDevice, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 10) v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    printf("1 MB H2D right after the CPU wrote the source (%s): %.1f us\n",
           mode ? "non-temporal stores" : "memcpy", v[v.size() / 2]);
  }
  // D2H into a pinned buffer the CPU has just read (lines cached) vs flushed
  std::vector<uint8_t> sink(1 << 20);
  for (int mode = 0; mode < 3; ++mode) {
    std::vector<float> v;
    for (int i = 0; i < 60; ++i) {
      if (mode == 1) memcpy(sink.data(), h, 786432);
      if (mode == 2) {
        memcpy(sink.data(), h, 786432);
        for (size_t o = 0; o < 786432; o += 64) __builtin_ia32_clflushopt(h + o);
        __builtin_ia32_sfence();
      }
      cudaEventRecord(a, s);
      cudaMemcpyAsync(h, d, 786432, cudaMemcpyDeviceToHost, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 10) v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    printf("768 KB D2H, destination %s: %.1f us\n",
           mode == 0 ? "untouched" : (mode == 1 ? "just read by the CPU" : "read then clflushopt"),
           v[v.size() / 2]);
  }
  // CPU side: one thread copying 1 MB pageable -> pinned, memcpy vs streaming stores
  for (int mode = 0; mode < 2; ++mode) {
    std::vector<double> v;
    for (int i = 0; i < 60; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      if (mode == 0) {
        memcpy(h, src.data(), 1 << 20);
      } else {
        for (size_t o = 0; o < (1 << 20); o += 16)
          __builtin_ia32_movntdq((__attribute__((vector_size(16))) long long*)(h + o),
                                 *(__attribute__((vector_size(16))) long long*)(src.data() + o));
        __builtin_ia32_sfence();
      }
      v.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(v.begin(), v.end());
    printf("CPU 1 MB copy into pinned (1 thread, %s): %.1f us\n", mode ? "streaming" : "memcpy", v[v.size() / 2]);
  }
  return 0;
}
