// 3x3 convolutions of the decoder on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
//   decode.0  Conv2d(64, 64, 3, pad 1) + LeakyReLU(0.2)          dstt.py:241-242
//   decode.2  Conv2d(64, 3, 3, pad 1), (tanh+1)/2, u8 conversion, non-finite guard and
//             the alpha composite                               dstt.py:243, :267, :322-325;
//                                                               base.py:87-88
//             -- as a tap-expanded GEMM fused into decode.0's epilogue: per pixel
//             E[3*tap + co] = sum_ci d0[ci] * W2[co][ci][tap] (a 128x32x64 MMA with the
//             fp16 d0 row as a TMEM A operand), stored as fp16 planes; dec2_gather_kernel
//             sums the 3x3 neighbourhood and runs the tail.  The 64-channel d0 raster is
//             never written.
//
// Implicit GEMM, M = 128 pixels of one output row, N = 64 output channels, K = 9 taps x 64
// input channels.  A persistent CTA owns the whole
// fp16 weight image in smem (one bulk copy) and walks TR-row x 128-pixel tiles:
//   warp 0      TMA: the (TR+2) x 130-pixel x 64-channel input halo of the next tile, one
//               box, 128B-swizzled K-major rows (128 B = one pixel); off-image rows and
//               columns are zero-filled by TMA = the conv's zero padding
//   warp 1      one thread issues TR x 9 x 4 tcgen05.mma (128 x N x 16) per tile into a
//               double-buffered TMEM accumulator; tap (dy,dx) is just a descriptor offset
//   warps 2-9   epilogue (two warps per TMEM lane quarter, alternate rows): tcgen05.ld
//               (lane = pixel), bias (registers) + LeakyReLU, fp16; fused: into TMEM as the
//               A operand of E, E planes stored one tile later
// Double-buffered halo and TMEM let TMA, MMA and the epilogue overlap; 2-row tiles (74 KB
// of weights + 2 x 65 KB halo).
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

template <int N, int TR, bool FUSE>
struct __align__(1024) ConvSmem {
  static constexpr int HALO_BYTES = (TR + 2) * HX * 128;    // [row][px][64 ch] fp16
  static constexpr int HALO_STRIDE = (HALO_BYTES + 1023) & ~1023;   // keep 1024 alignment
  uint8_t halo[2][HALO_STRIDE];
  uint8_t w[9 * 8 * N * 16];                 // [tap][k-chunk][co][8 ci] fp16
  uint8_t w2[FUSE ? 32 * 128 : 16];          // fused: decode.2 tap-expanded weights (SW128)
  // raster store staging: per epilogue warp 16 pixels x 128 B (transpose for full-line
  // coalesced stores: 8 lanes write one pixel's 128 B, one instruction = 4 whole lines)
  uint8_t stage[FUSE ? 1 : 8][FUSE ? 16 : 16 * 128];
  uint64_t halo_full[2], halo_empty[2], tmem_full[2], tmem_empty[2], w_full;
  uint64_t a2_full[2], e_full[2];            // fused: A2 (fp16 d0 in TMEM) ready / E ready
  uint32_t tmem_base;
};

template <int N, int TR>
constexpr uint32_t tmem_cols_d() {
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

// FUSE (decode.0 -> decode.2): after the D0 epilogue (bias, LeakyReLU, fp16) writes its
// row back into the first 32 TMEM columns of the same D0 row, the MMA warp multiplies that
// A operand (TMEM, 128 px x 64 ci) by w2 (smem, 32 x 64) into E (TMEM columns 256 + ..):
// E[p][3*tap + co] = sum_ci d0[p][ci] * W2[co][ci][tap]; the epilogue stores its 27
// columns as fp16 planes.  The 64-channel d0 raster is never written.
template <int N, int TR, bool FUSE>
__global__ void __launch_bounds__(THREADS, 1)
conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tin, ConvTcArgs a) {
  using Smem = ConvSmem<N, TR, FUSE>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr uint32_t COLS = FUSE ? 512 : tmem_cols_d<N, TR>();
  constexpr uint32_t ACOL = 2 * TR * N;       // fused: A2 columns (2 buffers x TR x 32)
  constexpr uint32_t ECOL = ACOL + 2 * TR * 32;   // fused: E columns (2 buffers x TR x 32)
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
      tc::mbar_init(&sm.a2_full[b], 8);
      tc::mbar_init(&sm.e_full[b], 1);
    }
    tc::mbar_init(&sm.w_full, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tin);
    tc::mbar_arrive_expect_tx(&sm.w_full, WBYTES + (FUSE ? 32 * 128 : 0));
    for (uint32_t off = 0; off < WBYTES; off += 16384) {   // constant: before the wait
      const uint32_t n = WBYTES - off < 16384 ? WBYTES - off : 16384;
      tc::bulk_load(sm.w + off, reinterpret_cast<const uint8_t*>(a.w) + off, n, &sm.w_full);
    }
    if constexpr (FUSE) tc::bulk_load(sm.w2, a.w2, 32 * 128, &sm.w_full);
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
      // fused: E(j) = A2(j) [TMEM, fp16 d0 rows] x w2^T once the epilogue wrote A2(j)
      auto e_mma = [&](int j) {
        const int bj = j & 1;
        tc::mbar_wait(&sm.a2_full[bj], (uint32_t)(j >> 1) & 1u);
        tc::fence_after();
        constexpr uint32_t idesc2 = tc::idesc_f16(128, 32);
        const uint64_t bw2 = tc::sdesc_sw128(tc::smem_u32(sm.w2), 0);
#pragma unroll
        for (int r = 0; r < TR; ++r)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc::mma_ts_f16_warp(tbase + ECOL + (uint32_t)(bj * TR * 32 + r * 32),
                                tbase + ACOL + (uint32_t)(bj * TR * 32 + r * 32 + 8 * ks),
                                bw2 + (uint64_t)(2 * ks), idesc2, ks != 0);
        tc::mma_commit_warp(&sm.e_full[bj]);
      };
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
        if constexpr (FUSE) if (i > 0) e_mma(i - 1);      // behind D0(i) in the pipe
      }
      if constexpr (FUSE) if (i > 0) e_mma(i - 1);
    }
  } else {                                               // ---------------- epilogue
    const int q = warp & 3;              // TMEM lanes 32q..32q+31 (fixed by warp id % 4)
    const int rh = (warp - 2) >> 2;      // warps 2-5 rows 0,2,..; warps 6-9 rows 1,3,..
    const size_t plane = (size_t)a.H * a.W;
    float bias[N];
#pragma unroll
    for (int c = 0; c < N; ++c) bias[c] = __ldg(a.bias + c);
    // fused: store the 27 E columns of tile j (tile index t_j) as fp16 planes
    auto e_phase = [&](int j, int t_j) {
      const int bj = j & 1;
      tc::mbar_wait(&sm.e_full[bj], (uint32_t)(j >> 1) & 1u);
      tc::fence_after();
      const int txj = t_j % tiles_x, restj = t_j / tiles_x;
      const int tyj = restj % tiles_y, fj = restj / tiles_y;
#pragma unroll
      for (int k = 0; k < TR / 2; ++k) {
        const int r = rh + 2 * k;
        const int y = tyj * TR + r, x = txj * TX + 32 * q + lane;
        uint32_t ev[32];
        const uint32_t eaddr = tbase + ((uint32_t)(32 * q) << 16) + ECOL + (uint32_t)(bj * TR * 32 + r * 32);
        tc::tmem_ld16(eaddr, ev);
        tc::tmem_ld16(eaddr + 16, ev + 16);
        tc::tmem_wait_ld();
        if (y < a.H && x < a.W) {
          __half* ep = a.e_planes + ((size_t)fj * 27 * plane) + (size_t)y * a.W + x;
#pragma unroll
          for (int u = 0; u < 27; ++u) ep[(size_t)u * plane] = __float2half_rn(__uint_as_float(ev[u]));
        }
      }
    };
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
        if constexpr (FUSE) {
          // fp16 LeakyReLU(d0) into this row's A2 columns = the A operand of E
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            float u0 = __uint_as_float(v[c]) + bias[c];
            float u1 = __uint_as_float(v[c + 1]) + bias[c + 1];
            u0 = u0 >= 0.f ? u0 : 0.2f * u0;
            u1 = u1 >= 0.f ? u1 : 0.2f * u1;
            pk[c / 2] = pack_half2(u0, u1);
          }
          tc::tmem_st32(tbase + ((uint32_t)(32 * q) << 16) + ACOL + (uint32_t)(buf * TR * 32 + r * 32), pk);
          tc::tmem_wait_st();
        } else {
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
      }
      if constexpr (FUSE) {
        // D0(i) is consumed (A2 has its own columns): free it for MMA1(i+2) at once, hand
        // A2(i) to the MMA warp, then store E of the PREVIOUS tile (its MMA2 ran behind
        // MMA1(i), so it is ready by now)
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&sm.a2_full[buf]);
          tc::mbar_arrive(&sm.tmem_empty[buf]);
        }
        if (i > 0) e_phase(i - 1, t - (int)gridDim.x);
      }
      if constexpr (!FUSE) {
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sm.tmem_empty[buf]);
      }
      if (warp == 2 && lane == 0 && i < 16) CT_AT(7 + 5 * i);
    }
    if constexpr (FUSE) if (i > 0) e_phase(i - 1, (int)blockIdx.x + (i - 1) * (int)gridDim.x);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) CT_AT(2);
  if (warp == 1) tc::tmem_dealloc<COLS>(tbase);
}

// ---------------------------------------------------------------------------------------
// The CTA that finishes last publishes the flags words (every CTA's atomicOr happens before
// its counter increment; the last one acquires them all) when a mirror is requested.
DR_DEV void mirror_flags(const ConvTcArgs& a) {
  if (!a.flags_mirror && !a.mirror_after_spans) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    if (atomicAdd(a.done, 1u) == total - 1) {
      __threadfence();
      int* fm = a.flags_mirror;
      if (a.mirror_after_spans) {
        const int4 sp = a.spans[a.H - 1];
        const size_t n = (size_t)sp.z + 3 * (size_t)(sp.y - sp.x);
        fm = reinterpret_cast<int*>(a.packed + ((n + 3) & ~(size_t)3));
      }
      for (int i = 0; i < a.frames; ++i) fm[i] = atomicOr(a.flags + i, 0);
      *a.done = 0;
    }
  }
}

DR_DEV void gather_pixel(const ConvTcArgs& a, const float (&bias)[3], int x, int y, int f) {
  const size_t plane = (size_t)a.H * a.W;
  const __half* ep = a.e_planes + (size_t)f * 27 * plane;
  float o[3] = {bias[0], bias[1], bias[2]};
#pragma unroll
  for (int dy = 0; dy < 3; ++dy) {
    const int yy = y + dy - 1;
    if (yy < 0 || yy >= a.H) continue;
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
      const int xx = x + dx - 1;
      if (xx < 0 || xx >= a.W) continue;
      const size_t pix = (size_t)yy * a.W + xx;
#pragma unroll
      for (int co = 0; co < 3; ++co)
        o[co] += __half2float(ep[(size_t)(3 * (3 * dy + dx) + co) * plane + pix]);
    }
  }
  const size_t pix = (size_t)y * a.W + x;
  const float alr = a.alpha ? __ldg(a.alpha + (size_t)f * plane + pix) : 1.f;
  int4 sp = make_int4(0, 0, 0, 0);
  if (a.packed) sp = __ldg(a.spans + y);
  const bool in_span = a.packed && x >= sp.x && x < sp.y;
  bool bad = false;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const float out01 = tanh01(o[ch]);
    bad |= !isfinite(out01);
    const size_t pl = ((size_t)f * 3 + ch) * plane + pix;
    if (a.fill) a.fill[pl] = out01;
    if (a.out_f32)
      a.out_f32[pl] = __fadd_rn(__fmul_rn(alr, out01), __fmul_rn(__fsub_rn(1.0f, alr), __ldg(a.rgb_f32 + pl)));
    if (a.out_u8 || in_span) {
      const uint8_t fill8 = (uint8_t)fminf(fmaxf(rintf(__fmul_rn(out01, 255.0f)), 0.f), 255.f);
      const uint8_t src8 = __ldg(a.rgb_u8 + ((size_t)f * plane + pix) * 3 + ch);
      uint8_t ov;
      if (alr == 0.f) ov = src8;
      else if (alr == 1.f) ov = fill8;
      else ov = (uint8_t)fminf(fmaxf(rintf(__fadd_rn(__fmul_rn(alr, (float)fill8),
                                                      __fmul_rn(__fsub_rn(1.0f, alr), (float)src8))), 0.f), 255.f);
      if (a.out_u8) a.out_u8[((size_t)f * plane + pix) * 3 + ch] = ov;
      if (in_span) a.packed[sp.z + 3 * (x - sp.x) + ch] = ov;
    }
  }
  if (bad) {
    atomicOr(a.flags + f, 1);
    __threadfence();                 // performed before this CTA counts itself done
  }
}

// decode.2 gather + tail over the fused decode.0's E planes: one thread per output pixel,
// out[co] = b[co] + sum_{dy,dx} E[3*(3dy+dx)+co][y+dy-1][x+dx-1] (0 off-image = the conv's
// zero padding), then (tanh + 1) / 2, non-finite guard and the alpha composite.  Each E
// value feeds exactly one output pixel, so the 27 reads per pixel are coalesced plane rows
// with no reuse to stage.
__global__ void __launch_bounds__(256) dec2_gather_kernel(ConvTcArgs a) {
  const int x = blockIdx.x * 256 + threadIdx.x, y = blockIdx.y, f = blockIdx.z;
  pdl_trigger();
  float bias[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) bias[c] = __ldg(a.bias + c);
  pdl_wait();
  if (x < a.W) gather_pixel(a, bias, x, y, f);
  mirror_flags(a);
}

// PX consecutive pixels per thread (W % PX == 0): each (dy, dx, co) E plane row segment is
// one 2*PX-byte load; the x - 1 / x + PX neighbours come from the adjacent lanes (shuffles)
// or, at warp edges, one 2-byte load.  Same summation order and tail as gather_pixel.
template <int PX> struct VecOf;
template <> struct VecOf<2> { using T = uint32_t; };
template <> struct VecOf<4> { using T = uint2; };
template <> struct VecOf<8> { using T = uint4; };
template <int PX>
DR_DEV void unpack_vec(const typename VecOf<PX>::T& v, float* e) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < PX / 2; ++i) {
    const float2 p2 = unpack_half2(w[i]);
    e[2 * i] = p2.x;
    e[2 * i + 1] = p2.y;
  }
}

template <int PX, int TPB>
__global__ void __launch_bounds__(TPB) dec2_gather_vec_kernel(ConvTcArgs a) {
  using V = typename VecOf<PX>::T;
  const int lane = threadIdx.x & 31;
  const int x0 = PX * (blockIdx.x * TPB + threadIdx.x), y = blockIdx.y, f = blockIdx.z;
  pdl_trigger();
  float bias[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) bias[c] = __ldg(a.bias + c);
  pdl_wait();
  const bool act = x0 < a.W;
  const size_t plane = (size_t)a.H * a.W;
  const __half* ep = a.e_planes + (size_t)f * 27 * plane;
  // the composite's inputs first: their loads fly with the 27 plane loads below
  const size_t pix0 = (size_t)y * a.W + x0;
  float alr[PX], rgbf[3][PX];
  uint8_t src[3 * PX];
  if (act) {
#pragma unroll
    for (int i = 0; i < PX; ++i) alr[i] = a.alpha ? __ldg(a.alpha + (size_t)f * plane + pix0 + i) : 1.f;
    if (a.out_f32) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch)
#pragma unroll
        for (int i = 0; i < PX; ++i) rgbf[ch][i] = __ldg(a.rgb_f32 + ((size_t)f * 3 + ch) * plane + pix0 + i);
    }
    if (a.out_u8 || a.packed) {                   // 3*PX bytes, 2*PX-byte aligned
      const uint16_t* s8 = reinterpret_cast<const uint16_t*>(a.rgb_u8 + ((size_t)f * plane + pix0) * 3);
#pragma unroll
      for (int k = 0; k < 3 * PX / 2; ++k) *reinterpret_cast<uint16_t*>(src + 2 * k) = __ldg(s8 + k);
    }
  }
  float o[3][PX];
#pragma unroll
  for (int co = 0; co < 3; ++co)
#pragma unroll
    for (int i = 0; i < PX; ++i) o[co][i] = bias[co];
#pragma unroll
  for (int dy = 0; dy < 3; ++dy) {
    const int yy = y + dy - 1;
    const bool rowok = yy >= 0 && yy < a.H;          // uniform over the CTA
    if (!rowok) continue;
#pragma unroll
    for (int co = 0; co < 3; ++co) {
      float e[3][PX];
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const __half* pl = ep + (size_t)(3 * (3 * dy + dx) + co) * plane + (size_t)yy * a.W;
        V v;
        if (act) v = __ldg(reinterpret_cast<const V*>(pl + x0));
        else memset(&v, 0, sizeof(v));
        unpack_vec<PX>(v, e[dx]);
      }
      // dx = 0 needs E at x - 1 (x = x0 .. x0 + PX - 1); dx = 2 at x + 1
      float left = __shfl_up_sync(0xffffffffu, e[0][PX - 1], 1);
      float right = __shfl_down_sync(0xffffffffu, e[2][0], 1);
      if (lane == 0) {
        const __half* pl = ep + (size_t)(3 * (3 * dy + 0) + co) * plane + (size_t)yy * a.W;
        left = (act && x0 > 0) ? __half2float(pl[x0 - 1]) : 0.f;
      }
      if (lane == 31 || x0 + PX >= a.W) {
        const __half* pl = ep + (size_t)(3 * (3 * dy + 2) + co) * plane + (size_t)yy * a.W;
        right = (act && x0 + PX < a.W) ? __half2float(pl[x0 + PX]) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        const float l = i == 0 ? left : e[0][i - 1];
        const float r = i == PX - 1 ? right : e[2][i + 1];
        o[co][i] += l;
        o[co][i] += e[1][i];
        o[co][i] += r;
      }
    }
  }
  if (act) {
    int4 sp = make_int4(0, 0, 0, 0);
    if (a.packed) sp = __ldg(a.spans + y);
    uint8_t dst[3 * PX];
    bool bad = false;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float out01[PX];
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        out01[i] = tanh01(o[ch][i]);
        bad |= !isfinite(out01[i]);
      }
      const size_t pl = ((size_t)f * 3 + ch) * plane + pix0;
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        if (a.fill) a.fill[pl + i] = out01[i];
        if (a.out_f32)
          a.out_f32[pl + i] = __fadd_rn(__fmul_rn(alr[i], out01[i]),
                                        __fmul_rn(__fsub_rn(1.0f, alr[i]), rgbf[ch][i]));
      }
      if (a.out_u8 || a.packed) {
#pragma unroll
        for (int i = 0; i < PX; ++i) {
          const uint8_t fill8 = (uint8_t)fminf(fmaxf(rintf(__fmul_rn(out01[i], 255.0f)), 0.f), 255.f);
          const uint8_t src8 = src[3 * i + ch];
          uint8_t ov;
          if (alr[i] == 0.f) ov = src8;
          else if (alr[i] == 1.f) ov = fill8;
          else ov = (uint8_t)fminf(fmaxf(rintf(__fadd_rn(__fmul_rn(alr[i], (float)fill8),
                                                          __fmul_rn(__fsub_rn(1.0f, alr[i]), (float)src8))), 0.f), 255.f);
          dst[3 * i + ch] = ov;
        }
      }
    }
    if (a.out_u8) {
      uint16_t* d8 = reinterpret_cast<uint16_t*>(a.out_u8 + ((size_t)f * plane + pix0) * 3);
#pragma unroll
      for (int k = 0; k < 3 * PX / 2; ++k) d8[k] = *reinterpret_cast<const uint16_t*>(dst + 2 * k);
    }
    if (a.packed) {
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        const int x = x0 + i;
        if (x >= sp.x && x < sp.y)
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) a.packed[sp.z + 3 * (x - sp.x) + ch] = dst[3 * i + ch];
      }
    }
    if (bad) {
      atomicOr(a.flags + f, 1);
      __threadfence();               // performed before this CTA counts itself done
    }
  }
  mirror_flags(a);
}


template <int N, int TR, bool FUSE>
void launch(const CUtensorMap& tin, const ConvTcArgs& a, cudaStream_t s) {
  static unsigned long long init = 0;
  const int smem = (int)sizeof(ConvSmem<N, TR, FUSE>);
  once_per_device(init, [&] {
    cudaFuncSetAttribute(conv3x3_tc_kernel<N, TR, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  const int sms = device_sms();
  const int tiles = a.frames * ((a.H + TR - 1) / TR) * ((a.W + TX - 1) / TX);
  const int grid = tiles < sms ? tiles : sms;
  launch_pdl(conv3x3_tc_kernel<N, TR, FUSE>, dim3(grid), dim3(THREADS), smem, s, tin, a);
#ifdef DR_TRACE
  conv_trace_snapshot(s, grid);
#endif
}

}  // namespace

size_t conv_tc_weight_bytes(int n) { return (size_t)9 * 8 * n * 16; }

int conv_tc_rows(int n) { return n == 64 ? 2 : 4; }   // decode.0 tiles: 2 output rows

void launch_dec2_gather(const ConvTcArgs& a, cudaStream_t s) {
  constexpr int PX = 4, TPB = 128;               // 4 pixels per thread, vector loads / stores
  if (a.W % PX == 0) {
    dim3 grid((a.W / PX + TPB - 1) / TPB, a.H, a.frames);
    launch_pdl(dec2_gather_vec_kernel<PX, TPB>, grid, dim3(TPB), 0, s, a);
    return;
  }
  dim3 grid((a.W + 255) / 256, a.H, a.frames);
  launch_pdl(dec2_gather_kernel, grid, dim3(256), 0, s, a);
}

void launch_conv3x3_tc(int n, const CUtensorMap& tin, const ConvTcArgs& a, cudaStream_t s) {
  (void)n;                                     // decode.0 only (decode.2: E planes + gather)
  if (a.e_planes) launch<64, 2, true>(tin, a, s);
  else launch<64, 2, false>(tin, a, s);
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
