// Softmax-sweep microbenchmark for the tcgen05 attention design on B200 (sm_100a).
//
// Reproduces the per-score instruction mix of attention_tc.cu's softmax warps (one FFMA,
// one exp2, half an F2FP pack, half an FMNMX3 per score, 64 scores per row block held in
// registers) and reports exp2/clk/SM for 1..4 warps per SM sub-partition, with a fraction
// of the exp2s evaluated on the FMA pipe by a degree-3 polynomial (MUFU offload).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/softmax_microbench softmax_microbench.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 2048;
constexpr int KB = 64;

__device__ unsigned long long g_cycles;
__device__ uint32_t g_sink;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float r = __fadd_rn(x, 12582912.f);
  const float j = __fadd_rn(r, -12582912.f);
  const float f = __fsub_rn(x, j);
  float p = fmaf(f, 0.05517161f, 0.24261111f);
  p = fmaf(f, p, 0.69326097f);
  p = fmaf(f, p, 0.99992806f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(r) << 23));
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// POLY_EVERY: element pairs c with (c % POLY_EVERY) == POLY_EVERY-1 use the polynomial
// (0 = none).  Per 32 pairs: POLY_EVERY 4 -> 25%, 8 -> 12.5%.
template <int POLY_EVERY>
__global__ void sweep_bench(float seed) {
  float s[KB];
#pragma unroll
  for (int i = 0; i < KB; ++i) s[i] = seed * (float)((threadIdx.x * 7 + i * 13) % 97) * 0.05f;
  uint32_t acc = 0;
  float mx = -1e30f, base = 1.0f;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
    float m4[4] = {mx, mx, mx, mx};
#pragma unroll
    for (int c = 0; c < KB / 2; ++c) {
      const float s0 = s[2 * c], s1 = s[2 * c + 1];
      m4[c & 3] = fmaxf(m4[c & 3], fmaxf(s0, s1));
      const float x0 = fmaf(s0, 0.36067376f, -base), x1 = fmaf(s1, 0.36067376f, -base);
      float e0, e1;
      if (POLY_EVERY && (c % (POLY_EVERY ? POLY_EVERY : 1)) == (POLY_EVERY ? POLY_EVERY : 1) - 1) {
        e0 = ex2_poly(x0);
        e1 = ex2_poly(x1);
      } else {
        e0 = ex2(x0);
        e1 = ex2(x1);
      }
      acc ^= pack(e0, e1);
    }
    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    base += 1e-7f * (float)(acc & 1);   // loop-carried, keeps the sweep live
  }
  const long long t1 = clock64();
  if (acc == 0x12345678u && mx == 3.f) g_sink = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) g_cycles = (unsigned long long)(t1 - t0);
}

template <int P>
void run(const char* name, int sms) {
  for (int warps : {4, 8, 12, 16}) {
    sweep_bench<P><<<sms, warps * 32>>>(1.0f);
    sweep_bench<P><<<sms, warps * 32>>>(1.0f);
    cudaDeviceSynchronize();
    unsigned long long cyc;
    cudaMemcpyFromSymbol(&cyc, g_cycles, sizeof(cyc));
    const double exps = (double)ITERS * KB * warps * 32;
    printf("%-14s warps/SM=%2d  %6.2f exp2/clk/SM  (%6.1f clk per 64-score row-block/warp)\n",
           name, warps, exps / (double)cyc, (double)cyc / ITERS);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("mufu-only", sms);
  run<8>("poly 1/8", sms);
  run<4>("poly 1/4", sms);
  run<3>("poly 1/3", sms);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
