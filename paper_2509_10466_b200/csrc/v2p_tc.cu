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
// 8 output phases px accumulate in 8 x 64 TMEM columns (the whole TMEM), 10 or 20 taps
// of 8 KB weights sit in smem.  Warp 0 TMA, warp 1 MMA issue, warps 2-5 epilogue (bias,
// fp16, transposed through smem so 8 lanes store one pixel's 128 B), with a TMEM barrier
// per phase so stores overlap MMAs.
#include <cuda.h>

#include "kernels.h"
#include "tc.cuh"

namespace dr {

namespace {

constexpr int M = 128;
constexpr int THREADS = 192;
constexpr int TAP_BYTES = 64 * 64 * 2;                 // [k-chunk 8][co 64][8 ci] fp16
constexpr int WIN_CHUNKS = 3;                          // window <= 384 rows (Cc <= 253)

struct __align__(1024) V2pSmem {
  uint8_t win[WIN_CHUNKS][M * 128];                    // token window, 128B-swizzled rows
  uint8_t w[20][TAP_BYTES];
  uint8_t stage[4][32 * 128];                          // per epilogue warp: 32 pixels x 128 B
  uint64_t win_full, w_full, tmem_full[8];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(THREADS, 1)
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
  const int n_taps = py < 2 ? 20 : 10;

  pdl_trigger();
  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.win_full, 1);
    tc::mbar_init(&sm.w_full, 1);
    for (int i = 0; i < 8; ++i) tc::mbar_init(&sm.tmem_full[i], 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tok);
    tc::mbar_arrive_expect_tx(&sm.w_full, n_taps * TAP_BYTES);   // constant: pre-wait
    const uint8_t* w0 = reinterpret_cast<const uint8_t*>(a.w) + (size_t)(py * 10) * TAP_BYTES;
    for (int t = 0; t < 10; ++t) tc::bulk_load(sm.w[t], w0 + (size_t)t * TAP_BYTES, TAP_BYTES, &sm.w_full);
    if (py < 2) {
      const uint8_t* w1 = reinterpret_cast<const uint8_t*>(a.w) + (size_t)((py + 8) * 10) * TAP_BYTES;
      for (int t = 0; t < 10; ++t)
        tc::bulk_load(sm.w[10 + t], w1 + (size_t)t * TAP_BYTES, TAP_BYTES, &sm.w_full);
    }
  }
  pdl_wait();                    // predecessor complete: its outputs and its TMEM are free
  if (warp == 1) tc::tmem_alloc<512>(&sm.tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {                                   // ------------------- loads
      tc::mbar_arrive_expect_tx(&sm.win_full, n_chunks * M * 128);
      for (int c = 0; c < n_chunks; ++c)
        tc::tma_load_3d(sm.win[c], &tok, &sm.win_full, 0, P0 - (PC + 1) + c * M, f);
    }
  } else if (warp == 1) {
    {                                                  // ------------------- MMA issue
      constexpr uint32_t idesc = tc::idesc_f16(128, 64);   // (whole warp, elected lane)
      tc::mbar_wait(&sm.win_full, 0);
      tc::mbar_wait(&sm.w_full, 0);
      tc::fence_after();
      // base descriptors; per-MMA offsets in 16-byte units (row = 8, k-step = 2)
      const uint64_t a0 = tc::sdesc_sw128(tc::smem_u32(sm.win[0]), 0);
      const uint64_t b0 = tc::sdesc(tc::smem_u32(sm.w[0]), 1024, 128);
      auto term = [&](uint32_t d, int tap, int off, bool first) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc::mma_f16_warp(d, a0 + (uint64_t)(off * 8 + ks * 2),
                           b0 + (uint64_t)(tap * (TAP_BYTES / 16) + ks * 128), idesc,
                           !(first && ks == 0));
      };
#pragma unroll 1
      for (int px = 0; px < 8; ++px) {
        const uint32_t d = tbase + (uint32_t)(px * 64);
        term(d, px, PC + 1, true);                                  // (i, j)
        if (px < 2) term(d, px + 8, PC, false);                     // (i, j-1)
        if (py < 2) term(d, 10 + px, 1, false);                     // (i-1, j)
        if (py < 2 && px < 2) term(d, 18 + px, 0, false);           // (i-1, j-1)
        tc::mma_commit_warp(&sm.tmem_full[px]);
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
    float bias[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) bias[c] = __ldg(a.bias + c);
#pragma unroll 1
    for (int px = 0; px < 8; ++px) {
      tc::mbar_wait(&sm.tmem_full[px], 0);
      tc::fence_after();
      uint32_t v[64];
      const uint32_t taddr = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(px * 64);
#pragma unroll
      for (int j = 0; j < 4; ++j) tc::tmem_ld16(taddr + 16 * j, v + 16 * j);
      tc::tmem_wait_ld();
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
          pk[e] = pack_half2(__uint_as_float(v[c]) + bias[c], __uint_as_float(v[c + 1]) + bias[c + 1]);
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
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tbase);
}

}  // namespace

size_t v2p_tc_weight_bytes() { return (size_t)100 * TAP_BYTES; }

void launch_v2p_tc(const CUtensorMap& tok, const V2pArgs& a, cudaStream_t s) {
  static bool init = false;
  const int smem = (int)sizeof(V2pSmem) + 1024;
  if (!init) {
    cudaFuncSetAttribute(v2p_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  const int NP = (a.R + 2) * (a.Cc + 2);
  dim3 grid((NP + M - 1) / M, 8, a.frames);
  launch_pdl(v2p_tc_kernel, grid, dim3(THREADS), smem, s, tok, a);
}

}  // namespace dr
