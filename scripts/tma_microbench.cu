// TMA halo-load throughput on B200: 4-D boxes {64 ch, 130 px, R rows, 1} (fp16 NHWC raster,
// 128B swizzle, the decoder's halo) from an L2-resident raster, one CTA per SM, `inflight`
// boxes outstanding.  Reports bytes per SM per clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_microbench tma_microbench.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

__device__ unsigned long long g_cyc;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R>
__global__ void __launch_bounds__(32, 1) tma_bench(const __grid_constant__ CUtensorMap m, int boxes, int inflight, int H) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[8];
  constexpr int BOX = 130 * 128 * R;
  constexpr int STRIDE = (BOX + 1023) & ~1023;
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  for (int b = 0; b < boxes; ++b) {
    const int s = b % inflight;
    if (b >= inflight) {   // wait for the box that used this slot
      const uint32_t ph = ((b / inflight) - 1) & 1;
      uint32_t ok = 0;
      while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[s])), "r"(BOX) : "memory");
    const int x = ((blockIdx.x * 7 + b) % 4) * 128 - 1, y = ((blockIdx.x * 13 + b * 3) % (H / R)) * R - 1;
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                 :: "r"(sa(buf + s * STRIDE)), "l"(&m), "r"(sa(&bar[s])), "r"(0), "r"(x), "r"(y), "r"(0) : "memory");
  }
  for (int b = boxes - inflight; b < boxes; ++b) {
    const int s = b % inflight;
    const uint32_t ph = (b / inflight) & 1;
    uint32_t ok = 0;
    while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
  }
  const long long t1 = clock64();
  atomicMax(&g_cyc, (unsigned long long)(t1 - t0));
}

int main() {
  const int W = 512, H = 512;
  void* raster;
  cudaMalloc(&raster, (size_t)W * H * 128);
  cudaMemset(raster, 0, (size_t)W * H * 128);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, int R, int inflight) {
    CUtensorMap m;
    cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, 1};
    cuuint64_t str[3] = {128, (cuuint64_t)W * 128, (cuuint64_t)H * W * 128};
    cuuint32_t box[4] = {64, 130, (cuuint32_t)R, 1}, es[4] = {1, 1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, raster, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int boxbytes = 130 * 128 * R, stride = (boxbytes + 1023) & ~1023;
    const int smem = stride * inflight + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int boxes = 64;
    unsigned long long z = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpyToSymbol(g_cyc, &z, sizeof(z));
      kern<<<sms, 32, smem>>>(m, boxes, inflight, H);
      cudaDeviceSynchronize();
    }
    unsigned long long cyc;
    cudaMemcpyFromSymbol(&cyc, g_cyc, sizeof(cyc));
    printf("box R=%d (%6d B) inflight=%d: %6.1f B/clk/SM  (%s)\n", R, boxbytes, inflight,
           (double)boxes * boxbytes / cyc, cudaGetErrorString(cudaGetLastError()));
  };
  run(tma_bench<1>, 1, 2); run(tma_bench<1>, 1, 4); run(tma_bench<1>, 1, 8);
  run(tma_bench<4>, 4, 2); run(tma_bench<4>, 4, 3);
  run(tma_bench<6>, 6, 2);
  return 0;
}
