// tcgen05.mma throughput vs N on B200 (sm_100a): one CTA per SM, one elected thread issues
// ITERS kind::f16 MMAs M=128 x N x K=16 (both operands in shared memory, K-major, A
// 128B-swizzled, B no-swizzle core matrices as in the decoder) into one TMEM accumulator,
// commits once and waits.  Reports cycles per MMA and flop/clk/SM for N = 32..256.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2509_10466_b200/csrc -o bin/umma_microbench umma_microbench.cu
#include <cstdio>

#include "tc.cuh"

using namespace dr;

constexpr int ITERS = 4096;

// MODE 0: A SW128 SBO 1024, one B; 1: A SBO 1280 with row offsets (the decoder's token
// tile); 2: MODE 1 + B rotating over 4 slots + a commit every 4 MMAs (the decoder's tap loop)
DR_DEV uint64_t sdesc_sw128_sbo(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}
// MODE 6: MODE 2 + 16 more warps spinning on an mbarrier until the MMAs are done;
// MODE 4: MODE 2 + warp 1 streaming 8 KB bulk copies global -> smem meanwhile (the tap
// ring); MODE 5: MODE 2 + an mbarrier wait and tcgen05 fence before every tap
template <int N, int MODE = 0>
__global__ void __launch_bounds__(640, 1) umma_bench(unsigned long long* out, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = base;                       // 180 rows x 128 B (SW128)
  uint8_t* b = base + 180 * 128 + 1024 - (180 * 128) % 1024;   // 4 x [k-chunk 8][N][16 B]
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tmem;
  for (int i = threadIdx.x; i < (int)((b - base) + 4 * 8 * N * 16) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;          // fp16 1.0 pairs
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&bar2, 1);
    tc::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tmem);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t d = tmem;
  __shared__ uint64_t lbar;
  if ((MODE == 4 || MODE == 8) && threadIdx.x == 32) {
    tc::mbar_init(&lbar, 1);
    tc::fence_barrier_init();
    uint8_t* dst = b + 4 * 8 * N * 16;
    // MODE 4: one 8 KB tap per 4 MMAs x 4; MODE 8: 8 KB per MMA (the N = 256 decoder rate)
    for (int k = 0; k < (MODE == 8 ? ITERS : ITERS / 16); ++k) {
      tc::mbar_arrive_expect_tx(&lbar, 8192);
      tc::bulk_load(dst, gsrc + (size_t)(k % 144) * 8192, 8192, &lbar);
      tc::mbar_wait(&lbar, (uint32_t)k & 1u);
    }
  }
  __shared__ uint64_t rbar[8];
  if (MODE == 10 && threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) tc::mbar_init(&rbar[i], 1);
    tc::fence_barrier_init();
  }
  if (MODE == 9 && threadIdx.x == 32) {             // 8 KB per MMA, 8 copies in flight
    for (int i = 0; i < 8; ++i) tc::mbar_init(&rbar[i], 1);
    tc::fence_barrier_init();
    uint8_t* dst = b + 4 * 8 * N * 16;              // 8 slots of 8 KB after the B ring
    for (int k = 0; k < ITERS; ++k) {
      const int sl = k & 7;
      if (k >= 8) tc::mbar_wait(&rbar[sl], (uint32_t)((k >> 3) - 1) & 1u);
      tc::mbar_arrive_expect_tx(&rbar[sl], 8192);
      tc::bulk_load(dst + sl * 8192, gsrc + (size_t)(k % 144) * 8192, 8192, &rbar[sl]);
    }
    for (int sl = 0; sl < 8; ++sl) tc::mbar_wait(&rbar[sl], (uint32_t)((ITERS >> 3) - 1) & 1u);
  }
  __shared__ uint64_t done;
  if (threadIdx.x == 0) { tc::mbar_init(&done, 1); tc::fence_barrier_init(); }
  __syncthreads();
  if (MODE == 6 && threadIdx.x >= 128) tc::mbar_wait(&done, 0);     // spinning warps
  if (MODE == 7 && threadIdx.x >= 32 && threadIdx.x < 64) {          // TS MMAs meanwhile
    const uint64_t bd2 = tc::sdesc(tc::smem_u32(b), 32 * 16, 128);
    for (int i = 0; i < ITERS / 4; ++i)
      tc::mma_ts_f16_warp(d + 384, d + 256 + (uint32_t)(8 * (i & 3)), bd2, tc::idesc_f16(128, 32), i != 0);
  }
  if (threadIdx.x < 32) {
    const uint64_t ad = MODE == 0 ? tc::sdesc_sw128(tc::smem_u32(a), 0) : sdesc_sw128_sbo(tc::smem_u32(a), 1280);
    const uint64_t bd = tc::sdesc(tc::smem_u32(b), N * 16, 128);
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    const int offs[4] = {0, 1, 10, 11};
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
      const int tap = (i >> 2) & 3, ks = i & 3;
      const uint64_t aa = MODE == 0 ? ad + (uint64_t)(ks * 2) : ad + (uint64_t)(offs[tap] * 8 + ks * 2);
      if (MODE == 11) {                                   // wait + fence before EVERY MMA
        tc::mbar_wait(&bar2, 0u ^ 1u);
        tc::fence_after();
      }
      if (MODE == 5 && ks == 0) {
        tc::mbar_wait(&bar2, 0u ^ 1u);                 // a completed phase: returns at once
        tc::fence_after();
      }
      const uint64_t bb = (MODE >= 2) ? bd + (uint64_t)(tap * (8 * N) + ks * 2 * N) : bd + (uint64_t)(ks * 2 * N);
      if (MODE == 3)   // A from TMEM (fp16 pairs in columns 128.., 8 per K-step), B from smem
        tc::mma_ts_f16_warp(d, d + 128 + (uint32_t)(8 * ks), bb, idesc, i != 0);
      else
        tc::mma_f16_warp(d, aa, bb, idesc, i != 0);
      if (MODE >= 2 && MODE != 3 && MODE != 10 && ks == 3) tc::mma_commit_warp(&bar2);
      if (MODE == 10) tc::mma_commit_warp(&rbar[i & 7]);   // a commit after every MMA
    }
    tc::mma_commit_warp(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    if (threadIdx.x == 0) tc::mbar_arrive(&done);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(d);
}

template <int N, int MODE = 0>
void run(int sms, unsigned long long* d_out) {
  const int smem = 180 * 128 + 1024 + 4 * 8 * N * 16 + (MODE == 9 ? 8 * 8192 : 8192) + 2048;
  if (smem > 227 * 1024) { printf("mode %d N=%d: smem %d too large\n", MODE, N, smem); return; }
  cudaFuncSetAttribute(umma_bench<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  static uint8_t* gsrc = nullptr;
  if (!gsrc) { cudaMalloc(&gsrc, 144 * 8192); cudaMemset(gsrc, 0, 144 * 8192); }
  const int thr = MODE == 6 ? 640 : 128;  // (MODE 9: warp 1 streams the copies)  // (MODE 7: warp 1 issues the TS MMAs)
  umma_bench<N, MODE><<<sms, thr, smem>>>(d_out, gsrc);
  umma_bench<N, MODE><<<sms, thr, smem>>>(d_out, gsrc);
  cudaDeviceSynchronize();
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  const double per = (double)cyc / ITERS;
  printf("mode %d M=128 N=%3d K=16: %7.1f cycles per MMA, %7.0f flop/clk/SM\n", MODE, N, per, 2.0 * 128 * N * 16 / per);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 8);
  run<32>(sms, d_out);
  run<64>(sms, d_out);
  run<128>(sms, d_out);
  run<256>(sms, d_out);
  run<64, 1>(sms, d_out);
  run<64, 2>(sms, d_out);
  run<128, 1>(sms, d_out);
  run<128, 2>(sms, d_out);
  run<32, 3>(sms, d_out);
  run<64, 3>(sms, d_out);
  run<64, 4>(sms, d_out);
  run<64, 6>(sms, d_out);
  run<64, 7>(sms, d_out);
  run<256, 1>(sms, d_out);
  run<256, 2>(sms, d_out);
  run<256, 4>(sms, d_out);
  run<256, 8>(sms, d_out);
  run<128, 8>(sms, d_out);
  run<256, 9>(sms, d_out);
  run<128, 9>(sms, d_out);
  run<64, 9>(sms, d_out);
  run<256, 10>(sms, d_out);
  run<256, 5>(sms, d_out);
  run<256, 11>(sms, d_out);
  run<128, 10>(sms, d_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
