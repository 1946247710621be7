// TMEM read / write bandwidth on B200 (sm_100a): tcgen05.ld / tcgen05.st 32x32b.x32 in a
// loop by W warps per CTA (1 CTA per SM, all SMs), bytes per SM per clock (clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_microbench tmem_microbench.cu
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 2048;

__device__ unsigned long long g_cycles;
__device__ uint32_t g_sink;

template <int MODE>   // 0 = ld x32 + wait, 1 = st x32 + wait, 2 = two lds then one wait
__global__ void __launch_bounds__(512, 1) bench() {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tbase_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t taddr = tbase_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(32 * ((warp >> 2) & 7));
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = i;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 1) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n"
                   :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    } else {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(taddr + 256 * (it & 1)));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicMax(&g_cycles, (unsigned long long)(t1 - t0));
  if (acc == 0x12345678) g_sink = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tbase_s) : "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16}) {
      unsigned long long zero = 0;
      cudaMemcpyToSymbol(g_cycles, &zero, sizeof(zero));
      if (mode == 0) bench<0><<<sms, 32 * warps>>>();
      else bench<1><<<sms, 32 * warps>>>();
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long cyc = 0;
      cudaMemcpyFromSymbol(&cyc, g_cycles, sizeof(cyc));
      const double bytes = (double)ITERS * warps * 32 * 32 * 4;   // per SM
      printf("%s x32 warps=%2d: %.1f B/clk/SM (%s)\n", mode ? "tcgen05.st" : "tcgen05.ld",
             warps, bytes / cyc, cudaGetErrorString(e));
    }
  return 0;
}
