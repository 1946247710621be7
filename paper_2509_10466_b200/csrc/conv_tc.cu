// 3x3 convolutions of the decoder on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
//   decode.0  Conv2d(64, 64, 3, pad 1) + LeakyReLU(0.2)          dstt.py:241-242
//   decode.2  Conv2d(64, 3, 3, pad 1), (tanh+1)/2, u8 conversion, non-finite guard and
//             the alpha composite                               dstt.py:243, :267, :322-325;
//                                                               base.py:87-88
//             -- as a tap-expanded GEMM (dec2_te_kernel below)
//
// Implicit GEMM, M = 128 pixels of one output row, N = output channels (64, or 16 with
// 3 real for decode.2), K = 9 taps x 64 input channels.  A persistent CTA owns the whole
// fp16 weight image in smem (one bulk copy) and walks TR-row x 128-pixel tiles:
//   warp 0      TMA: the (TR+2) x 130-pixel x 64-channel input halo of the next tile, one
//               box, 128B-swizzled K-major rows (128 B = one pixel); off-image rows and
//               columns are zero-filled by TMA = the conv's zero padding
//   warp 1      one thread issues TR x 9 x 4 tcgen05.mma (128 x N x 16) per tile into a
//               double-buffered TMEM accumulator; tap (dy,dx) is just a descriptor offset
//   warps 2-9   epilogue (two warps per TMEM lane quarter, alternate rows): tcgen05.ld
//               (lane = pixel), bias (registers) + activation, stores; decode.2
//               prefetches alpha / rgb of the next tile before waiting on the accumulator
// Double-buffered halo and TMEM let TMA, MMA and the epilogue overlap.  decode.0 uses
// 2-row tiles (74 KB of weights + 2 x 65 KB halo), decode.2 4-row tiles (1.5x halo reuse).
#include <cuda.h>
#include <math.h>

#include "kernels.h"
#include "tc.cuh"

namespace dr {

#ifdef DR_TRACE
void conv_trace_snapshot(cudaStream_t s, int n_cta);
#endif

namespace {

constexpr int TX = 128;                     // pixels per MMA (M)
constexpr int HX = TX + 2;                  // halo width
constexpr int THREADS = 320;                // TMA warp, MMA warp, 8 epilogue warps
// The tap (dy,dx) A operand starts (r+dy)*130+dx pixel rows into a 1024-byte aligned
// swizzled halo.  Measured on B200: the MMA unit applies the 128B XOR swizzle on absolute
// smem address bits (like TMA), so such row-shifted descriptors need base_offset 0
// (tests/test_gpu_ops.py pins this; base_offset = row & 7 produces garbage).

template <int N, int TR>
struct __align__(1024) ConvSmem {
  static constexpr int HALO_BYTES = (TR + 2) * HX * 128;    // [row][px][64 ch] fp16
  static constexpr int HALO_STRIDE = (HALO_BYTES + 1023) & ~1023;   // keep 1024 alignment
  uint8_t halo[2][HALO_STRIDE];
  uint8_t w[9 * 8 * N * 16];                 // [tap][k-chunk][co][8 ci] fp16
  // decode.0 store staging: per epilogue warp 16 pixels x 128 B (transpose for full-line
  // coalesced stores: 8 lanes write one pixel's 128 B, one instruction = 4 whole lines)
  uint8_t stage[N == 64 ? 8 : 1][N == 64 ? 16 * 128 : 16];
  uint64_t halo_full[2], halo_empty[2], tmem_full[2], tmem_empty[2], w_full;
  uint32_t tmem_base;
};

template <int N, int TR>
constexpr uint32_t tmem_cols() {
  return 2 * TR * N <= 32 ? 32 : (2 * TR * N <= 64 ? 64 : (2 * TR * N <= 128 ? 128 : (2 * TR * N <= 256 ? 256 : 512)));
}

// Diagnostic build only (-DDR_TRACE): per-CTA clock64 stamps, scripts/conv_trace.py.
// Slots: 0 entry, 1 weights in smem (MMA warp), 2 exit; tile i (< 16): 3+5i TMA issued,
// 4+5i halo landed (MMA warp), 5+5i MMAs committed, 6+5i accumulator ready (epilogue
// warp 2), 7+5i epilogue warp 2 done.
#ifdef DR_TRACE
constexpr int CT_SLOTS = 128;
__device__ unsigned long long g_conv_trace[256 * CT_SLOTS];
DR_DEV unsigned long long ct_timer() {    // SM cycle counter: exact within a CTA
  return (unsigned long long)clock64();
}
#define CT_AT(slot) do { if (blockIdx.x < 256 && (slot) < CT_SLOTS) \
    g_conv_trace[blockIdx.x * CT_SLOTS + (slot)] = ct_timer(); } while (0)
#else
#define CT_AT(slot) do {} while (0)
#endif

template <int N, int TR>
__global__ void __launch_bounds__(THREADS, 1)
conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tin, ConvTcArgs a) {
  using Smem = ConvSmem<N, TR>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr uint32_t COLS = tmem_cols<N, TR>();
  constexpr uint32_t WBYTES = 9 * 8 * N * 16;
  constexpr int HALO_BYTES = Smem::HALO_BYTES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_x = (a.W + TX - 1) / TX, tiles_y = (a.H + TR - 1) / TR;
  const int n_tiles = a.frames * tiles_y * tiles_x;

  if (threadIdx.x == 0) CT_AT(0);
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&sm.halo_full[b], 1);
      tc::mbar_init(&sm.halo_empty[b], 1);
      tc::mbar_init(&sm.tmem_full[b], 1);
      tc::mbar_init(&sm.tmem_empty[b], 8);
    }
    tc::mbar_init(&sm.w_full, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tin);
    tc::mbar_arrive_expect_tx(&sm.w_full, WBYTES);
    for (uint32_t off = 0; off < WBYTES; off += 16384) {   // constant: before the wait
      const uint32_t n = WBYTES - off < 16384 ? WBYTES - off : 16384;
      tc::bulk_load(sm.w + off, reinterpret_cast<const uint8_t*>(a.w) + off, n, &sm.w_full);
    }
  }
  pdl_wait();                    // predecessor complete: its outputs and its TMEM are free
  if (warp == 1) tc::tmem_alloc<COLS>(&sm.tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {                                     // ---------------- TMA producer
      int i = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int buf = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        const int tx = t % tiles_x, rest = t / tiles_x;
        const int ty = rest % tiles_y, f = rest / tiles_y;
        tc::mbar_wait(&sm.halo_empty[buf], ph ^ 1);
        if (i < 16) CT_AT(3 + 5 * i);
        tc::mbar_arrive_expect_tx(&sm.halo_full[buf], HALO_BYTES);
        tc::tma_load_4d(sm.halo[buf], &tin, &sm.halo_full[buf], 0, tx * TX - 1, ty * TR - 1, f);
      }
    }
  } else if (warp == 1) {
    {                                                    // ---------------- MMA issuer
      constexpr uint32_t idesc = tc::idesc_f16(128, N);   // (whole warp, elected lane issues)
      tc::mbar_wait(&sm.w_full, 0);
      if (lane == 0) CT_AT(1);
      const uint64_t b0 = tc::sdesc(tc::smem_u32(sm.w), N * 16, 128);
      int i = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int buf = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        tc::mbar_wait(&sm.halo_full[buf], ph);
        if (lane == 0 && i < 16) CT_AT(4 + 5 * i);
        tc::mbar_wait(&sm.tmem_empty[buf], ph ^ 1);
        tc::fence_after();
        // Base descriptors once per tile; each MMA adds a compile-time offset to the
        // 16-byte-unit address field (never carries: smem < 256 KB).
        const uint64_t a0 = tc::sdesc_sw128(tc::smem_u32(sm.halo[buf]), 0);
#pragma unroll
        for (int r = 0; r < TR; ++r) {
          const uint32_t d = tbase + (uint32_t)(buf * TR * N + r * N);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int dy = tap / 3, dx = tap % 3;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const uint32_t row = (uint32_t)((r + dy) * HX + dx);      // first pixel row
              tc::mma_f16_warp(d, a0 + (row * 8 + ks * 2), b0 + (uint64_t)((tap * 8 + 2 * ks) * N),
                               idesc, (tap | ks) != 0);
            }
          }
        }
        tc::mma_commit_warp(&sm.halo_empty[buf]);
        tc::mma_commit_warp(&sm.tmem_full[buf]);
        if (lane == 0 && i < 16) CT_AT(5 + 5 * i);
      }
    }
  } else {                                               // ---------------- epilogue
    const int q = warp & 3;              // TMEM lanes 32q..32q+31 (fixed by warp id % 4)
    const int rh = (warp - 2) >> 2;      // warps 2-5 rows 0,2,..; warps 6-9 rows 1,3,..
    const size_t plane = (size_t)a.H * a.W;
    float bias[N];
#pragma unroll
    for (int c = 0; c < N; ++c) bias[c] = __ldg(a.bias + c);
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int buf = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      const int tx = t % tiles_x, rest = t / tiles_x;
      const int ty = rest % tiles_y, f = rest / tiles_y;
      tc::mbar_wait(&sm.tmem_full[buf], ph);
      tc::fence_after();
      if (warp == 2 && lane == 0 && i < 16) CT_AT(6 + 5 * i);
#pragma unroll
      for (int k = 0; k < TR / 2; ++k) {
        const int r = rh + 2 * k;
        const int y = ty * TR + r;
        uint32_t v[N];
        const uint32_t taddr = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * TR * N + r * N);
#pragma unroll
        for (int j = 0; j < N / 16; ++j) tc::tmem_ld16(taddr + 16 * j, v + 16 * j);
        tc::tmem_wait_ld();
        // fp16 + LeakyReLU in registers, then two 16-pixel rounds through the warp's
        // staging buffer (16-B chunk c of pixel p at p*128 + ((c ^ (p & 7)) << 4): the
        // row-per-lane writes and the lane-per-chunk reads are both conflict-free)
        uint32_t pk[N / 2];
#pragma unroll
        for (int c = 0; c < N; c += 2) {
          float u0 = __uint_as_float(v[c]) + bias[c];
          float u1 = __uint_as_float(v[c + 1]) + bias[c + 1];
          u0 = u0 >= 0.f ? u0 : 0.2f * u0;
          u1 = u1 >= 0.f ? u1 : 0.2f * u1;
          pk[c / 2] = pack_half2(u0, u1);
        }
        uint8_t* st = sm.stage[warp - 2];
        const bool row_ok = y < a.H;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int p = lane - 16 * half;                  // pixel slot of this lane
          if (p >= 0 && p < 16) {
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8)
              *reinterpret_cast<uint4*>(st + p * 128 + ((c8 ^ (p & 7)) << 4)) =
                  make_uint4(pk[4 * c8], pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
          }
          __syncwarp();
          const int x0w = tx * TX + 32 * q + 16 * half;    // first pixel of this round
#pragma unroll
          for (int it = 0; it < 4; ++it) {                 // 4 pixels x 8 chunks per pass
            const int pp = 4 * it + (lane >> 3), c8 = lane & 7;
            const int xx = x0w + pp;
            if (row_ok && xx < a.W) {
              const uint4 val = *reinterpret_cast<const uint4*>(st + pp * 128 + ((c8 ^ (pp & 7)) << 4));
              reinterpret_cast<uint4*>(a.out16 + ((size_t)f * plane + (size_t)y * a.W + xx) * 64)[c8] = val;
            }
          }
          __syncwarp();
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.tmem_empty[buf]);
      if (warp == 2 && lane == 0 && i < 16) CT_AT(7 + 5 * i);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) CT_AT(2);
  if (warp == 1) tc::tmem_dealloc<COLS>(tbase);
}

// ---------------------------------------------------------------------------------------
// decode.2 as a tap-expanded GEMM (3 output channels): instead of 9 taps x 4 K-steps of a
// 128 x 16 MMA per output row (the A operand, 4 KB, re-read from smem 36 times), every halo
// row is multiplied ONCE by the 27 (tap, co) filter columns:
//     E[p][3*tap + co] = sum_ci d0[p][ci] * W2[co][ci][tap]       (M=128 pixels, N=32, K=64)
// and the 3x3 neighbourhood is summed in the epilogue:
//     out[y][x][co] = b[co] + sum_{dy,dx} E_{y+dy-1}[x+dx-1][3*(3dy+dx) + co]
// (E = 0 off-image because TMA zero-fills d0 there = the conv's zero padding).  Per output
// row and channel the three dx columns collapse to A = sum_dy E[.][dx=0], B = .., C = ..,
// so out(lane) = A(lane-1) + B(lane) + C(lane+1): two warp shuffles plus a boundary value
// through smem.  Tile: TR_TE output rows x 126 output pixels (the 128 MMA rows are pixels
// x0-1 .. x0+126).  Warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (two per TMEM lane quarter,
// each owning TR_TE/2 output rows; one named barrier per tile for the quarter edges).
constexpr int TR_TE = 4;
constexpr int TW_TE = 126;
constexpr int EPI_TE = 8;                     // epilogue warps
constexpr int ROWS_W = TR_TE / 2;             // output rows per epilogue warp
constexpr int THREADS_TE = 64 + 32 * EPI_TE;

struct __align__(1024) TeSmem {
  static constexpr int HALO_BYTES = (TR_TE + 2) * HX * 128;
  static constexpr int HALO_STRIDE = (HALO_BYTES + 1023) & ~1023;
  uint8_t halo[2][HALO_STRIDE];
  uint8_t w[32 * 128];                        // [u 32][ci 64] fp16, K-major 128B-swizzled
  float edge[2][TR_TE][4][2][3];              // per buffer, row, quarter: (A lane 31, C lane 0)
  uint64_t halo_full[2], halo_empty[2], tmem_full[2], tmem_empty[2], w_full;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(THREADS_TE, 1)
dec2_te_kernel(const __grid_constant__ CUtensorMap tin, ConvTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TeSmem& sm = *reinterpret_cast<TeSmem*>(smem_raw);
  constexpr uint32_t COLS = 512;              // 2 buffers x (TR_TE+2) rows x 32 columns
  constexpr int HALO_BYTES = TeSmem::HALO_BYTES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_x = (a.W + TW_TE - 1) / TW_TE, tiles_y = (a.H + TR_TE - 1) / TR_TE;
  const int n_tiles = a.frames * tiles_y * tiles_x;

  if (threadIdx.x == 0) CT_AT(0);
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&sm.halo_full[b], 1);
      tc::mbar_init(&sm.halo_empty[b], 1);
      tc::mbar_init(&sm.tmem_full[b], 1);
      tc::mbar_init(&sm.tmem_empty[b], EPI_TE);
    }
    tc::mbar_init(&sm.w_full, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tin);
    tc::mbar_arrive_expect_tx(&sm.w_full, 32 * 128);
    tc::bulk_load(sm.w, a.w, 32 * 128, &sm.w_full);
  }
  pdl_wait();                    // predecessor complete: its outputs and its TMEM are free
  if (warp == 1) tc::tmem_alloc<COLS>(&sm.tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {                                     // ---------------- TMA producer
      int i = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int buf = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        const int tx = t % tiles_x, rest = t / tiles_x;
        const int ty = rest % tiles_y, f = rest / tiles_y;
        tc::mbar_wait(&sm.halo_empty[buf], ph ^ 1);
        if (i < 16) CT_AT(3 + 5 * i);
        tc::mbar_arrive_expect_tx(&sm.halo_full[buf], HALO_BYTES);
        tc::tma_load_4d(sm.halo[buf], &tin, &sm.halo_full[buf], 0, tx * TW_TE - 1, ty * TR_TE - 1, f);
      }
    }
  } else if (warp == 1) {                                // ---------------- MMA issuer
    constexpr uint32_t idesc = tc::idesc_f16(128, 32);
    tc::mbar_wait(&sm.w_full, 0);
    if (lane == 0) CT_AT(1);
    const uint64_t b0 = tc::sdesc_sw128(tc::smem_u32(sm.w), 0);
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int buf = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      tc::mbar_wait(&sm.halo_full[buf], ph);
      if (lane == 0 && i < 16) CT_AT(4 + 5 * i);
      tc::mbar_wait(&sm.tmem_empty[buf], ph ^ 1);
      tc::fence_after();
      const uint64_t a0 = tc::sdesc_sw128(tc::smem_u32(sm.halo[buf]), 0);
#pragma unroll
      for (int hr = 0; hr < TR_TE + 2; ++hr) {
        const uint32_t d = tbase + (uint32_t)(buf * (TR_TE + 2) * 32 + hr * 32);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc::mma_f16_warp(d, a0 + (uint64_t)(hr * HX * 8 + ks * 2), b0 + (uint64_t)(ks * 2), idesc,
                           ks != 0);
      }
      tc::mma_commit_warp(&sm.halo_empty[buf]);
      tc::mma_commit_warp(&sm.tmem_full[buf]);
      if (lane == 0 && i < 16) CT_AT(5 + 5 * i);
    }
  } else {                                               // ---------------- epilogue
    const int q = warp & 3;                              // lanes 32q.. = pixels x0-1+32q..
    const int rh = (warp - 2) >> 2;                      // output rows ROWS_W*rh ..
    const int l = 32 * q + lane;
    const size_t plane = (size_t)a.H * a.W;
    float bias[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) bias[c] = __ldg(a.bias + c);
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int buf = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      const int tx = t % tiles_x, rest = t / tiles_x;
      const int ty = rest % tiles_y, f = rest / tiles_y;
      const int x = tx * TW_TE - 1 + l;                  // this lane's pixel
      const bool out_lane = l >= 1 && l <= TW_TE && x < a.W;
      // alpha / frame of this lane's output pixels, fetched while the MMAs run
      float al[ROWS_W], fr[ROWS_W][3];
      uint8_t fr8[ROWS_W][3];
#pragma unroll
      for (int k = 0; k < ROWS_W; ++k) {
        const int y = ty * TR_TE + ROWS_W * rh + k;
        const bool ok = out_lane && y < a.H;
        const size_t pix = (size_t)(ok ? y : 0) * a.W + (ok ? x : 0);
        al[k] = ok && a.alpha ? __ldg(a.alpha + (size_t)f * plane + pix) : 1.f;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          fr[k][ch] = ok && a.out_f32 ? __ldg(a.rgb_f32 + ((size_t)f * 3 + ch) * plane + pix) : 0.f;
          fr8[k][ch] = ok && a.out_u8 ? __ldg(a.rgb_u8 + ((size_t)f * plane + pix) * 3 + ch) : 0;
        }
      }
      tc::mbar_wait(&sm.tmem_full[buf], ph);
      tc::fence_after();
      if (warp == 2 && lane == 0 && i < 16) CT_AT(6 + 5 * i);
      // E rows ROWS_W*rh .. +ROWS_W+1 for this lane: column 3*tap + co, tap = 3*dy + dx
      float e[ROWS_W + 2][27];
#pragma unroll
      for (int hr = 0; hr < ROWS_W + 2; ++hr) {
        uint32_t v[32];
        const uint32_t taddr = tbase + ((uint32_t)(32 * q) << 16) +
                               (uint32_t)(buf * (TR_TE + 2) * 32 + (ROWS_W * rh + hr) * 32);
        tc::tmem_ld16(taddr, v);
        tc::tmem_ld16(taddr + 16, v + 16);
        tc::tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 27; ++u) e[hr][u] = __uint_as_float(v[u]);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.tmem_empty[buf]);   // TMEM free for tile i+2
      // per output row and channel: A (dx=0), B (dx=1), C (dx=2) summed over dy
      float A[ROWS_W][3], B[ROWS_W][3], Cc[ROWS_W][3];
#pragma unroll
      for (int k = 0; k < ROWS_W; ++k)
#pragma unroll
        for (int co = 0; co < 3; ++co) {
          A[k][co] = e[k][co] + e[k + 1][9 + co] + e[k + 2][18 + co];
          B[k][co] = e[k][3 + co] + e[k + 1][12 + co] + e[k + 2][21 + co];
          Cc[k][co] = e[k][6 + co] + e[k + 1][15 + co] + e[k + 2][24 + co];
        }
      // lane 31's A and lane 0's C cross to the neighbouring quarter (one barrier per tile;
      // the edge slots are double-buffered by tile parity)
#pragma unroll
      for (int k = 0; k < ROWS_W; ++k) {
        float* ed = &sm.edge[buf][ROWS_W * rh + k][q][0][0];
        if (lane == 31) { ed[0] = A[k][0]; ed[1] = A[k][1]; ed[2] = A[k][2]; }
        if (lane == 0) { ed[3] = Cc[k][0]; ed[4] = Cc[k][1]; ed[5] = Cc[k][2]; }
      }
      asm volatile("bar.sync 1, %0;\n" :: "r"(32 * EPI_TE) : "memory");
      bool bad = false;
#pragma unroll
      for (int k = 0; k < ROWS_W; ++k) {
        const int r = ROWS_W * rh + k;
        float o[3];
#pragma unroll
        for (int co = 0; co < 3; ++co) {
          float left = __shfl_up_sync(0xffffffffu, A[k][co], 1);
          float right = __shfl_down_sync(0xffffffffu, Cc[k][co], 1);
          if (lane == 0) left = q > 0 ? sm.edge[buf][r][q - 1][0][co] : 0.f;
          if (lane == 31) right = q < 3 ? sm.edge[buf][r][q + 1][1][co] : 0.f;
          o[co] = left + B[k][co] + right;
        }
        const int y = ty * TR_TE + r;
        if (!out_lane || y >= a.H) continue;
        const size_t pix = (size_t)y * a.W + x;
        const float alr = al[k];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float raw = o[ch] + bias[ch];
          const float out01 = (tanhf(raw) + 1.0f) * 0.5f;
          bad |= !isfinite(out01);
          const size_t pl = ((size_t)f * 3 + ch) * plane + pix;
          if (a.fill) a.fill[pl] = out01;
          if (a.out_f32)
            a.out_f32[pl] = __fadd_rn(__fmul_rn(alr, out01), __fmul_rn(__fsub_rn(1.0f, alr), fr[k][ch]));
          if (a.out_u8) {
            const uint8_t fill8 = (uint8_t)fminf(fmaxf(rintf(__fmul_rn(out01, 255.0f)), 0.f), 255.f);
            const uint8_t src8 = fr8[k][ch];
            uint8_t ov;
            if (alr == 0.f) ov = src8;
            else if (alr == 1.f) ov = fill8;
            else ov = (uint8_t)fminf(fmaxf(rintf(__fadd_rn(__fmul_rn(alr, (float)fill8),
                                                            __fmul_rn(__fsub_rn(1.0f, alr), (float)src8))), 0.f), 255.f);
            a.out_u8[((size_t)f * plane + pix) * 3 + ch] = ov;
          }
        }
      }
      if (bad) atomicOr(a.flags + f, 1);
      if (warp == 2 && lane == 0 && i < 16) CT_AT(7 + 5 * i);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) CT_AT(2);
  if (warp == 1) tc::tmem_dealloc<COLS>(tbase);
}

template <int N, int TR>
void launch(const CUtensorMap& tin, const ConvTcArgs& a, cudaStream_t s) {
  static int sms = 0;
  const int smem = (int)sizeof(ConvSmem<N, TR>);
  if (!sms) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(conv3x3_tc_kernel<N, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  const int tiles = a.frames * ((a.H + TR - 1) / TR) * ((a.W + TX - 1) / TX);
  const int grid = tiles < sms ? tiles : sms;
  launch_pdl(conv3x3_tc_kernel<N, TR>, dim3(grid), dim3(THREADS), smem, s, tin, a);
#ifdef DR_TRACE
  conv_trace_snapshot(s, grid);
#endif
}

}  // namespace

size_t conv_tc_weight_bytes(int n) { return (size_t)9 * 8 * n * 16; }

int conv_tc_rows(int n) { return n == 64 ? 2 : 4; }   // decode.0 tiles: 2 output rows

int dec2_te_rows() { return TR_TE; }

void launch_dec2_te(const CUtensorMap& tin, const ConvTcArgs& a, cudaStream_t s) {
  static int sms = 0;
  const int smem = (int)sizeof(TeSmem);
  if (!sms) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(dec2_te_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  const int tiles = a.frames * ((a.H + TR_TE - 1) / TR_TE) * ((a.W + TW_TE - 1) / TW_TE);
  const int grid = tiles < sms ? tiles : sms;
  launch_pdl(dec2_te_kernel, dim3(grid), dim3(THREADS_TE), smem, s, tin, a);
#ifdef DR_TRACE
  conv_trace_snapshot(s, grid);
#endif
}

void launch_conv3x3_tc(int n, const CUtensorMap& tin, const ConvTcArgs& a, cudaStream_t s) {
  (void)n;                                     // decode.0 only (decode.2: launch_dec2_te)
  launch<64, 2>(tin, a, s);
}

}  // namespace dr

#ifdef DR_TRACE
#include <vector>
namespace dr {
namespace {
std::vector<std::vector<unsigned long long>>& conv_trace_store() {
  static std::vector<std::vector<unsigned long long>> v;
  return v;
}
}  // namespace
void conv_trace_snapshot(cudaStream_t s, int n_cta) {
  if (conv_trace_store().size() >= 16) return;
  cudaStreamSynchronize(s);
  std::vector<unsigned long long> h((size_t)std::min(n_cta, 256) * CT_SLOTS);
  cudaMemcpyFromSymbol(h.data(), g_conv_trace, h.size() * sizeof(unsigned long long));
  conv_trace_store().push_back(std::move(h));
}
}  // namespace dr
extern "C" int dr_debug_conv_trace(int idx, unsigned long long* host, int n) {
  auto& v = dr::conv_trace_store();
  if (idx < 0 || idx >= (int)v.size()) return -1;
  const int k = std::min(n, (int)v[idx].size());
  for (int i = 0; i < k; ++i) host[i] = v[idx][i];
  return k;
}
#endif
