// Occupancy probe: CTAs per SM the runtime reports for 192-thread kernels at several
// register caps, with and without a max-shared carveout (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>
template <int R>
__global__ void __maxnreg__(R) k_reg(float* p, int n) {
  float acc[40];
#pragma unroll
  for (int i = 0; i < 40; ++i) acc[i] = p[threadIdx.x + i * n];
  for (int j = 0; j < n; ++j)
#pragma unroll
    for (int i = 0; i < 40; ++i) acc[i] = acc[i] * acc[(i + j) % 40] + 1.f;
  float s = 0;
#pragma unroll
  for (int i = 0; i < 40; ++i) s += acc[i];
  p[threadIdx.x] = s;
}
template <int R>
void probe(int smem) {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k_reg<R>);
  cudaFuncSetAttribute(k_reg<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int n0 = -1, n1 = -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n0, k_reg<R>, 192, smem);
  cudaFuncSetAttribute(k_reg<R>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n1, k_reg<R>, 192, smem);
  printf("maxnreg %d (used %d) smem %d: %d CTAs/SM default carveout, %d max carveout, err %d\n", R,
         fa.numRegs, smem, n0, n1, (int)cudaGetLastError());
}
int main() {
  for (int smem : {0, 30720}) {
    probe<80>(smem); probe<96>(smem); probe<104>(smem); probe<112>(smem); probe<128>(smem); probe<168>(smem);
  }
  return 0;
}
