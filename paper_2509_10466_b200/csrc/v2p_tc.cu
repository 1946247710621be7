// Vec2Patch on the 5th-gen tensor cores: ConvTranspose2d(64, 64, k=10, stride=8) over the
// token grid + crop offset 1 (reference dstt.py:198-221), written as an NHWC fp16 raster.
//
// Output-stationary phase GEMM.  Canvas pixel (8i+py, 8j+px) (raster pixel (y,x) = canvas
// - 1) is the sum over the 1, 2 or 4 tokens whose 10x10 kernel covers it:
//   token (i,j)     through tap (py,   px)
//   token (i,j-1)   through tap (py,   px+8)   if px < 2
//   token (i-1,j)   through tap (py+8, px)     if py < 2
//   token (i-1,j-1) through tap (py+8, px+8)   if both
// Tokens are stored on a zero-padded (R+2) x (Cc+2) grid (position (i+1, j+1)), so for a
// run of 128 consecutive padded positions the four neighbour sets are the same run shifted
// by 0, -1, -(Cc+2), -(Cc+3) rows: one TMA window (128B-swizzled, 128 B = one token per
// row) serves every term as a descriptor offset.  A CTA = (128 positions, one py, frame):
// the 8 output phases px accumulate in 4 rotating 64-column TMEM buffers, and the 10 or 20
// 8 KB tap images stream through a 4-slot smem ring in consumption order, so a CTA needs
// ~100 KB of smem and 256 TMEM columns: two CTAs per SM, one wave for a 512^2 frame.  Warp
// 0 loads, warp 1 issues the MMAs, warps 2-5 run the epilogue (bias, fp16, transposed
// through smem so 8 lanes store one pixel's 128 B), overlapping the next phases' MMAs.
#include <cuda.h>

#include "kernels.h"
#include "tc.cuh"

namespace dr {

namespace {

constexpr int M = 128;
constexpr int THREADS = 192;
constexpr int TAP_BYTES = 64 * 64 * 2;                 // [k-chunk 8][co 64][8 ci] fp16
constexpr int WIN_CHUNKS = 3;                          // window <= 384 rows (Cc <= 253)
constexpr int NSLOT = 4;                               // tap ring
constexpr int NBUF = 4;                                // TMEM phase buffers (64 columns)

struct __align__(1024) V2pSmem {
  uint8_t win[WIN_CHUNKS][M * 128];                    // token window, 128B-swizzled rows
  uint8_t w[NSLOT][TAP_BYTES];
  uint8_t stage[4][32 * 128];                          // per epilogue warp: 32 pixels x 128 B
  uint64_t win_full, w_full[NSLOT], w_empty[NSLOT], tmem_full[8], tmem_empty[NBUF];
  uint32_t tmem_base;
  float bias[64];                                      // epilogue bias (smem, not registers)
};

// Diagnostic build only (-DDR_TRACE): clock64 stamps per CTA (scripts/v2p_trace.py).
// Slots: 0 entry, 1 TMEM allocated, 2 window landed (MMA warp), 3+px MMAs of phase px
// issued, 11+px epilogue (warp 2) done with phase px, 19 exit.
#ifdef DR_TRACE
__device__ unsigned long long g_v2p_trace[4096 * 20];
#define VT(slot) do { unsigned long long c_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_) :: "memory"); \
    const int b_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);                      \
    if (b_ < 4096) g_v2p_trace[b_ * 20 + (slot)] = c_; } while (0)
#else
#define VT(slot) do {} while (0)
#endif

// The taps of phase px in consumption order: (tap image index, token-window row offset).
// Image index a*10 + b = kernel tap (a, b); window offsets for terms (i,j), (i,j-1),
// (i-1,j), (i-1,j-1) are PC+1, PC, 1, 0.
DR_DEV int phase_taps(int py, int px, int PC, int* img, int* off) {
  int n = 0;
  img[n] = py * 10 + px; off[n++] = PC + 1;
  if (px < 2) { img[n] = py * 10 + px + 8; off[n++] = PC; }
  if (py < 2) { img[n] = (py + 8) * 10 + px; off[n++] = 1; }
  if (py < 2 && px < 2) { img[n] = (py + 8) * 10 + px + 8; off[n++] = 0; }
  return n;
}

__global__ void __launch_bounds__(THREADS, 2)
v2p_tc_kernel(const __grid_constant__ CUtensorMap tok, V2pArgs a) {
  extern __shared__ uint8_t smem_raw[];
  V2pSmem& sm = *reinterpret_cast<V2pSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P0 = blockIdx.x * M, py = blockIdx.y, f = blockIdx.z;
  const int PC = a.Cc + 2;                              // padded row length
  const int NP = (a.R + 2) * PC;
  const int win_rows = M + PC + 1;
  const int n_chunks = (win_rows + M - 1) / M;

  if (threadIdx.x == 0) VT(0);
  pdl_trigger();
  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.win_full, 1);
    for (int i = 0; i < NSLOT; ++i) {
      tc::mbar_init(&sm.w_full[i], 1);
      tc::mbar_init(&sm.w_empty[i], 1);
    }
    for (int i = 0; i < 8; ++i) tc::mbar_init(&sm.tmem_full[i], 1);
    for (int i = 0; i < NBUF; ++i) tc::mbar_init(&sm.tmem_empty[i], 4);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tok);
    // the first NSLOT taps are constant: stream them before waiting on the predecessor
    int k = 0;
    for (int px = 0; px < 8 && k < NSLOT; ++px) {
      int img[4], off[4];
      const int n = phase_taps(py, px, PC, img, off);
      for (int t = 0; t < n && k < NSLOT; ++t, ++k) {
        tc::mbar_arrive_expect_tx(&sm.w_full[k], TAP_BYTES);
        tc::bulk_load(sm.w[k], reinterpret_cast<const uint8_t*>(a.w) + (size_t)img[t] * TAP_BYTES,
                      TAP_BYTES, &sm.w_full[k]);
      }
    }
  }
  pdl_wait();                    // predecessor complete: its outputs and its TMEM are free
  if (warp == 1) tc::tmem_alloc<64 * NBUF>(&sm.tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = sm.tmem_base;
  if (threadIdx.x == 0) VT(1);

  if (warp == 0) {
    if (lane == 0) {                                   // ------------------- loads
      tc::mbar_arrive_expect_tx(&sm.win_full, n_chunks * M * 128);
      for (int c = 0; c < n_chunks; ++c)
        tc::tma_load_3d(sm.win[c], &tok, &sm.win_full, 0, P0 - (PC + 1) + c * M, f);
      int k = 0;                                       // tap ring, taps NSLOT.. of the CTA
      for (int px = 0; px < 8; ++px) {
        int img[4], off[4];
        const int n = phase_taps(py, px, PC, img, off);
        for (int t = 0; t < n; ++t, ++k) {
          if (k < NSLOT) continue;                     // issued in the prologue
          const int sl = k % NSLOT;
          tc::mbar_wait(&sm.w_empty[sl], (uint32_t)(k / NSLOT - 1) & 1u);
          tc::mbar_arrive_expect_tx(&sm.w_full[sl], TAP_BYTES);
          tc::bulk_load(sm.w[sl], reinterpret_cast<const uint8_t*>(a.w) + (size_t)img[t] * TAP_BYTES,
                        TAP_BYTES, &sm.w_full[sl]);
        }
      }
    }
  } else if (warp == 1) {
    {                                                  // ------------------- MMA issue
      constexpr uint32_t idesc = tc::idesc_f16(128, 64);   // (whole warp, elected lane)
      tc::mbar_wait(&sm.win_full, 0);
      tc::fence_after();
      if (lane == 0) VT(2);
      // base descriptors; per-MMA offsets in 16-byte units (row = 8, k-step = 2)
      const uint64_t a0 = tc::sdesc_sw128(tc::smem_u32(sm.win[0]), 0);
      const uint64_t b0 = tc::sdesc(tc::smem_u32(sm.w[0]), 1024, 128);
      int k = 0;
#pragma unroll 1
      for (int px = 0; px < 8; ++px) {
        const int buf = px & (NBUF - 1);
        if (px >= NBUF) tc::mbar_wait(&sm.tmem_empty[buf], 0);   // epilogue drained px-4
        const uint32_t d = tbase + (uint32_t)(buf * 64);
        int img[4], off[4];
        const int n = phase_taps(py, px, PC, img, off);
        for (int t = 0; t < n; ++t) {
          const int sl = (k + t) % NSLOT;
          tc::mbar_wait(&sm.w_full[sl], (uint32_t)((k + t) / NSLOT) & 1u);
          tc::fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc::mma_f16_warp(d, a0 + (uint64_t)(off[t] * 8 + ks * 2),
                             b0 + (uint64_t)(sl * (TAP_BYTES / 16) + ks * 128), idesc,
                             (t | ks) != 0);
        }
        for (int t = 0; t < n; ++t) tc::mma_commit_warp(&sm.w_empty[(k + t) % NSLOT]);
        k += n;
        tc::mma_commit_warp(&sm.tmem_full[px]);
        if (lane == 0) VT(3 + px);
      }
    }
  } else {                                             // ------------------- epilogue
    const int q = warp & 3;
    // pixel slots this lane stores (slot 4*it + lane/8 of the warp's 32 positions): raster
    // row and x base of each, precomputed once for the 8 phases
    int ys[8], xb[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int Pp = P0 + 32 * q + 4 * it + (lane >> 3);
      const int ip = Pp / PC, jp = Pp - ip * PC;
      const int yp = 8 * (ip - 1) + py - 1;
      const bool ok = Pp < NP && yp >= 0 && yp < a.H && jp >= 1;
      ys[it] = ok ? yp : -1;
      xb[it] = 8 * (jp - 1) - 1;
    }
    // bias via shared memory (broadcast reads): 64 registers back for the epilogue
    if (warp == 2) {
      sm.bias[lane] = __ldg(a.bias + lane);
      sm.bias[32 + lane] = __ldg(a.bias + 32 + lane);
    }
    asm volatile("bar.sync 2, 128;\n" ::: "memory");          // the 4 epilogue warps
    const float* bias = sm.bias;
#pragma unroll 1
    for (int px = 0; px < 8; ++px) {
      tc::mbar_wait(&sm.tmem_full[px], 0);
      tc::fence_after();
      uint32_t v[64];
      const uint32_t taddr = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)((px & (NBUF - 1)) * 64);
#pragma unroll
      for (int j = 0; j < 4; ++j) tc::tmem_ld16(taddr + 16 * j, v + 16 * j);
      tc::tmem_wait_ld();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.tmem_empty[px & (NBUF - 1)]);
      // bias + fp16 in registers, transpose through the warp's staging buffer (chunk c of
      // pixel slot p at p*128 + ((c ^ (p & 7)) << 4)), then 8 lanes per pixel write its
      // 128 B: each store instruction covers 4 whole lines instead of 32 half-sectors
      uint8_t* st = sm.stage[q];
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = c8 * 8 + 2 * e;
          const float u0 = __uint_as_float(v[c]) + bias[c], u1 = __uint_as_float(v[c + 1]) + bias[c + 1];
          pk[e] = pack_half2(u0, u1);
        }
        *reinterpret_cast<uint4*>(st + lane * 128 + ((c8 ^ (lane & 7)) << 4)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int pp = 4 * it + (lane >> 3), c8 = lane & 7;
        const int yp = ys[it], xp = xb[it] + px;
        if (yp >= 0 && xp >= 0 && xp < a.W) {
          const uint4 val = *reinterpret_cast<const uint4*>(st + pp * 128 + ((c8 ^ (pp & 7)) << 4));
          reinterpret_cast<uint4*>(a.raster + (((size_t)f * a.H + yp) * a.W + xp) * 64)[c8] = val;
        }
      }
      __syncwarp();
      if (warp == 2 && lane == 0) VT(11 + px);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) VT(19);
  if (warp == 1) tc::tmem_dealloc<64 * NBUF>(tbase);
}

}  // namespace

size_t v2p_tc_weight_bytes() { return (size_t)100 * TAP_BYTES; }

void launch_v2p_tc(const CUtensorMap& tok, const V2pArgs& a, cudaStream_t s) {
  static unsigned long long init = 0;
  const int smem = (int)sizeof(V2pSmem) + 1024;
  once_per_device(init, [&] {
    cudaFuncSetAttribute(v2p_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  const int NP = (a.R + 2) * (a.Cc + 2);
  dim3 grid((NP + M - 1) / M, 8, a.frames);
  launch_pdl(v2p_tc_kernel, grid, dim3(THREADS), smem, s, tok, a);
}

}  // namespace dr

#ifdef DR_TRACE
extern "C" int dr_debug_v2p_trace(unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  const int k = n < 4096 * 20 ? n : 4096 * 20;
  cudaMemcpyFromSymbol(host, dr::g_v2p_trace, (size_t)k * sizeof(unsigned long long));
  return k;
}
#endif
