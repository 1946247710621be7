// Pipe-throughput microbenchmark for the attention design on B200 (sm_100a):
// MUFU ex2 (f32, f16x2), fp32->fp16x2 pack (F2FP), FFMA, HMMA m16n8k16.  Reports
// operations per SM per clock (clock64 inside the kernel, all SMs busy).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_microbench pipe_microbench.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 4096;
constexpr int ILP = 8;

__device__ unsigned long long g_cycles;
__device__ float g_sink;

template <int KIND>
__global__ void bench(float seed) {
  float x[ILP];
  uint32_t hx[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { x[i] = seed * (i + 1) * 1e-3f; hx[i] = 0x3c003c00u + i; }
  float acc[4] = {0, 0, 0, 0};
  uint32_t a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
  float c[ILP][4] = {};
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (KIND == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      } else if (KIND == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(hx[i]));
      } else if (KIND == 2) {
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) % ILP]));
        hx[i] ^= r;
      } else if (KIND == 3) {
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x[i]));
      } else if (KIND == 5) {
        asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      } else if (KIND == 6) {
        asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      } else if (KIND == 4) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(hx[0]), "r"(hx[1]));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i] + (float)hx[i] + c[i][0] + acc[0];
  if (s == 12345.f) g_sink = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) g_cycles = (unsigned long long)(t1 - t0);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"ex2.f32", "ex2.f16x2", "cvt.f16x2.f32", "ffma", "hmma.m16n8k16",
                         "rcp.approx.f32", "rsqrt.approx.f32"};
  for (int kind = 0; kind < 7; ++kind) {
    for (int warps : {8, 16, 32}) {
      void (*k)(float) = kind == 0 ? bench<0> : kind == 1 ? bench<1> : kind == 2 ? bench<2>
                       : kind == 3 ? bench<3> : kind == 4 ? bench<4> : kind == 5 ? bench<5>
                       : bench<6>;
      k<<<sms, warps * 32>>>(1.0f);
      k<<<sms, warps * 32>>>(1.0f);
      cudaDeviceSynchronize();
      unsigned long long cyc;
      cudaMemcpyFromSymbol(&cyc, g_cycles, sizeof(cyc));
      const double ops = (double)ITERS * ILP * warps * 32;     // per SM (one CTA per SM)
      double per_clk = ops / (double)cyc;
      const char* unit = "lane-ops/clk/SM";
      if (kind == 4) { per_clk = per_clk / 32 * 4096; unit = "flop/clk/SM"; }
      printf("%-16s warps/SM=%2d  %10.2f %s  (cycles %llu)\n", names[kind], warps, per_clk, unit, cyc);
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
