// Global write throughput on B200 for a 33.5 MB raster: SM stores (st.global.v4, full
// 128-B lines) vs bulk copies from shared memory (cp.async.bulk.global.shared::cta, 4-16 KB
// per copy, the TMA store path).  Grid = SMs x CTAs/SM, each CTA owns a contiguous slice.
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

__global__ void __launch_bounds__(256) st_v4(uint4* out, size_t n16) {
  const size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const size_t b = blockIdx.x * per, e = min(n16, b + per);
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = b + threadIdx.x; i < e; i += blockDim.x) out[i] = v;
}

template <int CHUNK>
__global__ void __launch_bounds__(128) st_bulk(uint8_t* out, size_t nbytes) {
  extern __shared__ __align__(128) uint8_t buf[];
  for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(buf)[i] = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  const size_t nch = nbytes / CHUNK;
  const size_t per = (nch + gridDim.x - 1) / gridDim.x;
  const size_t b = blockIdx.x * per, e = min(nch, b + per);
  if (threadIdx.x == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
    for (size_t c = b; c < e; ++c) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                   :: "l"(out + c * CHUNK), "r"(s), "n"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;\n" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> v;
  for (int i = 0; i < 30; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 5) v.push_back(ms * 1e3f);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  const size_t nbytes = 512ull * 512 * 128;
  uint8_t* out;
  cudaMalloc(&out, nbytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {2, 4, 8}) {
    const float t = timeit([&] { st_v4<<<sms * per_sm, 256>>>((uint4*)out, nbytes / 16); });
    printf("st.global.v4   %d CTAs/SM x 256 thr: %7.2f us  %7.1f GB/s\n", per_sm, t, nbytes / t / 1e3);
  }
  cudaFuncSetAttribute(st_bulk<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  for (int per_sm : {1, 2, 4, 8}) {
    float t = timeit([&] { st_bulk<4096><<<sms * per_sm, 128, 4096>>>(out, nbytes); });
    printf("bulk 4 KB      %d CTAs/SM:           %7.2f us  %7.1f GB/s\n", per_sm, t, nbytes / t / 1e3);
    t = timeit([&] { st_bulk<16384><<<sms * per_sm, 128, 16384>>>(out, nbytes); });
    printf("bulk 16 KB     %d CTAs/SM:           %7.2f us  %7.1f GB/s\n", per_sm, t, nbytes / t / 1e3);
  }
  printf("err %d\n", (int)cudaGetLastError());
  return 0;
}
