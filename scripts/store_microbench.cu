// Global store throughput on B200 for the decoder raster (fp16 NHWC, 128 B per pixel):
// (a) contiguous pixels, (b) Vec2Patch pattern: each warp instruction stores 4 whole
// 128-B pixel rows 8 pixels (1 KB) apart.  33.5 MB raster, grid = 2 x SMs x 4 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_microbench store_microbench.cu
#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(128) st(uint4* out, size_t n_px) {
  const int lane = threadIdx.x & 31;
  const size_t warps = (size_t)gridDim.x * 4;
  const size_t w = (size_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const uint4 v = make_uint4(lane, 1, 2, 3);
  // each warp instruction: 4 pixels x 8 chunks
  for (size_t g = w; g < n_px / 4; g += warps) {
    size_t px;
    if (MODE == 0) px = g * 4 + (lane >> 3);                               // contiguous
    else {                                                                 // stride 8 px
      const size_t blk = g / 8, ph = g % 8;                                // 32 px = 4 x 8
      px = (blk * 32 + (lane >> 3) * 8 + ph);
    }
    out[px * 8 + (lane & 7)] = v;
  }
}

int main() {
  const size_t n_px = 512 * 512;
  uint4* out;
  cudaMalloc(&out, n_px * 128);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    const int mult = mode < 2 ? 2 : 16;               // CTAs of 4 warps per SM
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode % 2 == 0) st<0><<<mult * sms, 128>>>(out, n_px);
      else st<1><<<mult * sms, 128>>>(out, n_px);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("%s, %2d warps/SM: %.2f us, %.1f GB/s\n", mode % 2 ? "stride-8 pixels" : "contiguous",
               4 * mult, ms * 1e3,
               n_px * 128 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
