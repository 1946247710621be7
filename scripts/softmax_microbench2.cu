// Softmax-sweep ceiling on B200 (sm_100a): the per-score instruction mix of the attention
// softmax warps as shipped (FFMA2 scale-and-shift of score pairs, ex2.approx on MUFU for
// most pairs, a packed degree-3 polynomial exp2 on the FMA pipe for 1 pair in POLY_EVERY,
// fp16x2 pack, running max) with the scores already in registers -- no TMEM, no MMA, no
// barriers.  Reports scores/clk/SM for 4..24 warps per SM, so the attention kernel's
// achieved rate can be read against what the pipes allow.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/softmax_microbench2 softmax_microbench2.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 1024;
constexpr int KB = 64;

__device__ unsigned long long g_cycles;
__device__ uint32_t g_sink;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return make_float2(a, b);
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  const float2 xv = f2_unpack(x2);
  const uint64_t x = f2_pack(fmaxf(xv.x, -125.f), fmaxf(xv.y, -125.f));
  const uint64_t r = f2_add(x, f2_pack(12582912.f, 12582912.f));
  const uint64_t j = f2_add(r, f2_pack(-12582912.f, -12582912.f));
  const uint64_t f = f2_fma(j, f2_pack(-1.f, -1.f), x);
  uint64_t p = f2_fma(f, f2_pack(0.05517161f, 0.05517161f), f2_pack(0.24261111f, 0.24261111f));
  p = f2_fma(f, p, f2_pack(0.69326097f, 0.69326097f));
  p = f2_fma(f, p, f2_pack(0.99992806f, 0.99992806f));
  const float2 pv = f2_unpack(p), rv = f2_unpack(r);
  return f2_pack(__int_as_float(__float_as_int(pv.x) + (__float_as_int(rv.x) << 23)),
                 __int_as_float(__float_as_int(pv.y) + (__float_as_int(rv.y) << 23)));
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// MAXMODE 0: no max, 1: fmaxf(m, fmaxf(s0, s1)), 2: three-input max
template <int POLY_EVERY, int MAXMODE>
__global__ void sweep_bench(float seed, uint32_t* out) {
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
    const uint64_t sl2 = f2_pack(0.36067376f, 0.36067376f), nb = f2_pack(-base, -base);
    uint32_t pk[KB / 2];
#pragma unroll
    for (int c = 0; c < KB / 2; ++c) {
      const float s0 = s[2 * c], s1 = s[2 * c + 1];
      if (MAXMODE == 1) m4[c & 3] = fmaxf(m4[c & 3], fmaxf(s0, s1));
      if (MAXMODE == 2) m4[c & 3] = max3(m4[c & 3], s0, s1);
      const float2 xv = f2_unpack(f2_fma(f2_pack(s0, s1), sl2, nb));
      if (POLY_EVERY && (c % (POLY_EVERY ? POLY_EVERY : 1)) == (POLY_EVERY ? POLY_EVERY : 1) - 1) {
        const float2 e = f2_unpack(ex2_poly2(f2_pack(xv.x, xv.y)));
        pk[c] = pack(e.x, e.y);
      } else {
        pk[c] = pack(ex2(xv.x), ex2(xv.y));
      }
    }
#pragma unroll
    for (int c = 0; c < KB / 2; ++c) acc += pk[c];
    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    base += 1e-7f * (float)(acc & 1);   // loop-carried, keeps the sweep live
#pragma unroll
    for (int i = 0; i < KB; ++i) s[i] = __uint_as_float(__float_as_uint(s[i]) ^ (acc & 1));
  }
  const long long t1 = clock64();
  if (acc == 0x12345678u && mx == 3.f) *out = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) g_cycles = (unsigned long long)(t1 - t0);
}

template <int P, int M>
void run(const char* name, int sms, uint32_t* out) {
  for (int warps : {4, 8, 12, 16, 24}) {
    sweep_bench<P, M><<<sms, warps * 32>>>(1.0f, out);
    sweep_bench<P, M><<<sms, warps * 32>>>(1.0f, out);
    cudaDeviceSynchronize();
    unsigned long long cyc;
    cudaMemcpyFromSymbol(&cyc, g_cycles, sizeof(cyc));
    const double exps = (double)ITERS * KB * warps * 32;
    printf("%-24s warps/SM=%2d  %6.2f scores/clk/SM  (%6.1f clk per 64-score row block)\n",
           name, warps, exps / (double)cyc, (double)cyc / ITERS);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  cudaMalloc(&out, 4);
  run<0, 1>("mufu-only, max", sms, out);
  run<3, 1>("poly 1/3, max (shipped)", sms, out);
  run<3, 0>("poly 1/3, no max", sms, out);
  run<3, 2>("poly 1/3, max3", sms, out);
  run<2, 2>("poly 1/2, max3", sms, out);
  run<4, 2>("poly 1/4, max3", sms, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
