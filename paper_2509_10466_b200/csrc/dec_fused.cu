// The decoder tail on the 5th-gen tensor cores: Vec2Patch o decode.0 -> LeakyReLU ->
// decode.2 -> (tanh + 1) / 2 -> alpha composite, without a 64-channel raster.
// Reference: Vec2Patch dstt.py:198-221 (ConvTranspose2d(64, 64, k=10, s=8), crop 1),
// decode dstt.py:240-244 (Conv3x3 64->64, LeakyReLU(0.2), Conv3x3 64->3), output :267,
// composite SURVEY A16 (base.py:87-88).
//
// Algebra.  Both convolutions before the LeakyReLU are linear, so decode.0's pre-activation
// is a stride-8 transposed convolution of the tokens with a 12 x 12 kernel
//   K[u][v] = sum_{dy,dx} Wc[dy][dx] Wv[u+dy+1][v+dx+1],   u, v in [-2, 9],
// plus the combined bias bc + sum Wc bv -- exact wherever decode.0's 3x3 window stays
// inside the image.  Pixel (8ty+py, 8tx+px) takes tokens ty-1 (py <= 1), ty, ty+1
// (py >= 6) and likewise in x: 144 taps over the 64 phases (py, px), 2.25 tokens x 64
// channels per pixel instead of Vec2Patch + decode.0's 100 + 576 -- 4.8 GFLOP per 512^2
// frame instead of 22.7.  On the image border decode.0 reads zero padding where the
// combined form reads the cropped canvas ring: there the decode.0 taps that read the ring
// are subtracted (per edge a 12-tap kernel over the edge's token row / column, corners add
// back the doubly removed tap; tables built at dr_create, the algebra checked in float64).
//
// Kernels (one frame batch):
//   dec_fused   one CTA per tile of 16 x 8 tokens = 128 x 64 pixels (and 1 of `groups`
//               parts of its 64 phases).  Per phase:
//                 MMA warp   D = sum over the phase's 1/2/4 taps of A x Wcomb[tap]^T
//                            (M = 128 token positions, N = 64, K = 64); A = the TMA-loaded
//                            halo'd token tile (18 x 10 tokens, 128B-swizzled rows, row
//                            stride 10 -> descriptor SBO 1280), the tap's token shift is a
//                            row offset; tap images stream through a smem ring
//                 epilogue 1 (8 warps) D + bias -> LeakyReLU -> fp16 into TMEM (A2); image
//                            border pixels also store their pre-activation for dec_border
//                 E warp     E = A2 x W2te^T (TMEM A operand, N = 32: 27 = 9 taps x 3
//                            channels of decode.2 per pixel)
//                 epilogue 2 (4 warps) scatters E into the tile's fp32 output accumulator
//                            in shared memory (+1 pixel ring), phase after phase (fixed
//                            order: deterministic); image-border sources are skipped
//               Four D, A2 and E buffers in TMEM let the phases overlap.  Then every pixel
//               whose 3x3 window stays inside the tile and off the image border is finished
//               (bias, tanh, composite, u8, non-finite flag); the others and the ring go to
//               per-tile partial planes.
//   dec_border  one warp per image-border pixel: its correct pre-activation (the stored
//               combined one minus the ring taps), LeakyReLU, and its 27 decode.2 taps E
//   dec_fixup   the remaining pixels: partial planes of every tile whose 1-pixel-expanded
//               area holds the pixel (a fixed order), plus the border sources' E, then the
//               tail; the last CTA mirrors the flags (host path)
#include <cuda.h>
#include <math.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "kernels.h"
#include "tc.cuh"

namespace dr {

namespace {

constexpr int TY = 16, TX = 8;                   // token cells per tile (M = 128)
constexpr int TPY = 8 * TY, TPX = 8 * TX;        // 128 x 64 pixels
constexpr int HTY = TY + 2, HTX = TX + 2;        // halo'd token tile
constexpr int SLOT_BYTES = 2 * 256 * 16;         // one K step of an offset block: 8 KB
constexpr int BLK_BYTES = 4 * SLOT_BYTES;        // one offset block (4 K steps): 32 KB
constexpr int NBLK = 2;                          // weight ring (offset blocks)
constexpr int NBUF = 2;                          // quad buffers in TMEM (256 columns each)
constexpr int ACC_RS = 72, ACC_ROWS = TPY + 2;   // accumulator row stride / rows (+ring)
constexpr int ACC_C0 = 4;                        // column of tile pixel 0 (ring at 3 and 68)
#ifndef DR_DEC_FINISH_RUNS
#define DR_DEC_FINISH_RUNS 2
#endif
constexpr int NWARP = 15;
constexpr int THREADS = 32 * NWARP;
constexpr int W_LOAD = 0, W_MMA = 1, W_EPI1 = 2, W_EPI2 = 10, W_EMMA = 14;
constexpr uint32_t TM_COLS = 512;

struct __align__(1024) DecSmem {
  uint8_t tok[HTY * HTX * 128];                  // 23040 B, SW128 rows (one token per row)
  alignas(1024) uint8_t w2[32 * 128];            // SW128 [32][64] fp16
  alignas(1024) uint8_t w[NBLK][BLK_BYTES];
  float acc[3][ACC_ROWS][ACC_RS];                // [co][qy + 1][swizzled qx + ACC_C0]
  alignas(16) float bias[64];
  float b2[4];
  uint64_t tok_full, w_full[NBLK], w_empty[NBLK];
  uint64_t d_full[NBUF], d_empty[NBUF], a2_full[NBUF][4], e_full[NBUF][4];
  uint32_t tmem_base;
};
static_assert(sizeof(DecSmem) + 1024 <= 227 * 1024, "fused decoder shared memory");

// The i-th phase quad of cluster rank `grp` of `G`: whole quad rows, 16 / G quads each.
// (Anti-diagonal classes (gy + gx) % G balance the offset blocks better, 9 / 8 / 9 / 8 vs
// 12 / 6 / 6 / 12 at G = 4, but lose epilogue 2's row carry: measured slower.)
DR_DEV int quad_at(int grp, int G, int i) { return grp * (16 / G) + i; }
// global offset block of this CTA's kk-th weight block (the prologue's first blocks)
DR_DEV int block_at(int grp, int G, int kk) { return dec_quad_first(quad_at(grp, G, 0)) + kk; }

// token-tile row offset of the A operand for token offset (du, dv)
DR_DEV int tok_off(int du, int dv) { return (1 + du) * HTX + (1 + dv); }

// Seam partial sums of a tile (the pixels dec_fixup finishes): its accumulator on the band
// of tile rows -1..1 and ye-2..ye (full width -1..xe) and columns -1..1, xe-2..xe of the
// rows between (ye x xe = the tile's extent in the image); [3 channels][DEC_BAND] fp32 per
// tile, contiguous, so dec_fixup's reads are compact.
constexpr int DEC_BAND = 6 * (TPX + 2) + 6 * (TPY - 4);
DR_DEV int band_idx(int yl, int xl, int ye, int xe) {
  const int w2 = xe + 2;
  if (yl <= 1) return (yl + 1) * w2 + xl + 1;
  if (yl >= ye - 2) return (yl - ye + 5) * w2 + xl + 1;
  return 6 * w2 + (yl - 2) * 6 + (xl <= 1 ? xl + 1 : xl - xe + 5);
}

// K-major SWIZZLE_128B descriptor with an explicit stride between 8-row groups
DR_DEV uint64_t sdesc_sw128_sbo(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}

// accumulator column of tile pixel column qx (-1..64) at c = qx + ACC_C0 in row r = qy + 1:
// 8-column blocks XOR-swizzled by the token row within 4 and the 32-pixel half, so the 32
// lanes of an epilogue-2 warp (4 token rows x 8 token columns, same phase) hit 32 banks.
// A run of 4 pixels from a multiple of 4 stays one 16-byte group (acc_vec4).
DR_DEV int acc_swz(int r, int c) { return ((r >> 3) & 3) | (((c >> 5) & 1) << 2); }
DR_DEV int acc_col(int r, int c) { return c ^ acc_swz(r, c); }

// border-correction table layout (floats): edges [4][12][64 ci][64 co], edge bias [4][64],
// corners [4][64 ci][64 co], corner bias [4][64]; edges 0 top, 1 bottom, 2 left, 3 right;
// corners 0 TL, 1 TR, 2 BL, 3 BR
constexpr size_t DK_EDGE = 0, DK_EB = (size_t)4 * 12 * 4096, DK_CORNER = DK_EB + 256,
                 DK_CB = DK_CORNER + (size_t)4 * 4096, DK_TOTAL = DK_CB + 256;

DR_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
DR_DEV uint32_t map_rank(uint32_t local_saddr, int rank) {
  uint32_t remote;
  asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local_saddr), "r"(rank));
  return remote;
}
// (not volatile: read only after a cluster barrier, so the loads may be scheduled freely)
DR_DEV float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(addr));
  return v;
}
DR_DEV float4 ld_dsmem_f32x4(uint32_t addr) {
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

DR_DEV bool on_border(int y, int x, int H, int W) { return y == 0 || x == 0 || y == H - 1 || x == W - 1; }
// index of an image-border pixel: top row, bottom row, left column, right column
DR_DEV int border_index(int y, int x, int H, int W) {
  if (y == 0) return x;
  if (y == H - 1) return W + x;
  if (x == 0) return 2 * W + (y - 1);
  return 2 * W + (H - 2) + (y - 1);
}

#ifdef DR_TRACE
// Diagnostic build only: per CTA, cycles spent in each wait (scripts/dec_trace.py).  Slots:
// 0 start / 12 main loop end / 13 exit (globaltimer ns); cycles: 2 MMA w_full, 3 MMA
// d_empty, 4 E-warp a2_full, 5 E-warp e_empty, 6 epi1 d_full, 8 epi1 a2_empty, 9 epi2
// e_full, 10 epi2 phase barrier; 14 SM id
__device__ unsigned long long g_dec_trace[4096 * 16];
// per-phase timeline of CTA 0 (clock64): [0] D MMAs committed, [1] epilogue 1 done (set 0/1),
// [2] E MMAs committed, [3] epilogue 2 done; [4][0] kernel start; [5] D MMAs begin
__device__ long long g_dec_tl[6][64];
#define DT_TL(k, i) do { if (DT_CTA == 0 && (i) < 64) g_dec_tl[k][i] = clock64(); } while (0)
#define DT_CTA (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z))
#define DT_SET(slot, v) do { if (DT_CTA < 4096) g_dec_trace[DT_CTA * 16 + (slot)] = (v); } while (0)
#define DT_WAIT(slot, stmt) do { const long long t0_ = clock64(); stmt; \
    if (lane == 0 && DT_CTA < 4096) atomicAdd(&g_dec_trace[DT_CTA * 16 + (slot)], (unsigned long long)(clock64() - t0_)); } while (0)
DR_DEV unsigned long long dt_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define DT_SET(slot, v) do {} while (0)
#define DT_WAIT(slot, stmt) stmt
#define DT_TL(k, i) do {} while (0)
#endif

}  // namespace

// Tail of one output pixel: o = decode.2 output before tanh (bias included); alr / src are
// the pixel's alpha and input (preloaded by the caller).
DR_DEV void dec_emit(const ConvTcArgs& a, int f, int y, int x, const float (&o)[3], float alr,
                     const float (&srcf)[3], const uint8_t (&src8)[3]) {
  const size_t plane = (size_t)a.H * a.W;
  const size_t pix = (size_t)y * a.W + x;
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
    if (a.out_f32) a.out_f32[pl] = __fadd_rn(__fmul_rn(alr, out01), __fmul_rn(__fsub_rn(1.0f, alr), srcf[ch]));
    if (a.out_u8 || in_span) {
      const uint8_t fill8 = (uint8_t)fminf(fmaxf(rintf(__fmul_rn(out01, 255.0f)), 0.f), 255.f);
      uint8_t ov;
      if (alr == 0.f) ov = src8[ch];
      else if (alr == 1.f) ov = fill8;
      else ov = (uint8_t)fminf(fmaxf(rintf(__fadd_rn(__fmul_rn(alr, (float)fill8),
                                                      __fmul_rn(__fsub_rn(1.0f, alr), (float)src8[ch]))), 0.f), 255.f);
      if (a.out_u8) a.out_u8[((size_t)f * plane + pix) * 3 + ch] = ov;
      if (in_span) a.packed[sp.z + 3 * (x - sp.x) + ch] = ov;
    }
  }
  if (bad) atomicOr(a.flags + f, 1);
}

// inputs of one output pixel for dec_emit
DR_DEV void dec_inputs(const ConvTcArgs& a, int f, int y, int x, float* alr, float (&srcf)[3],
                       uint8_t (&src8)[3]) {
  const size_t plane = (size_t)a.H * a.W;
  const size_t pix = (size_t)y * a.W + x;
  *alr = a.alpha ? __ldg(a.alpha + (size_t)f * plane + pix) : 1.f;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    srcf[ch] = a.out_f32 ? __ldg(a.rgb_f32 + ((size_t)f * 3 + ch) * plane + pix) : 0.f;
    src8[ch] = a.rgb_u8 ? __ldg(a.rgb_u8 + ((size_t)f * plane + pix) * 3 + ch) : 0;
  }
}

namespace {

__global__ void __launch_bounds__(THREADS, 1)
dec_fused_kernel(const __grid_constant__ CUtensorMap tokmap, const __grid_constant__ DecArgs a) {
  extern __shared__ uint8_t smem_raw[];
  DecSmem& sm = *reinterpret_cast<DecSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.groups;
  const int tile_x = blockIdx.x, tile_y = blockIdx.y / G, grp = blockIdx.y - tile_y * G;
  const int f = blockIdx.z;
  const int ty0 = tile_y * TY, tx0 = tile_x * TX;          // first token cell
  const int y0 = 8 * ty0, x0 = 8 * tx0;                    // first pixel
  const int nq4 = 16 / G;                                   // this CTA's phase quads
  int nblk = 0;                                              // ... and their offset blocks
  for (int i = 0; i < nq4; ++i) {
    const int g = quad_at(grp, G, i);
    nblk += dec_quad_noff(g >> 2) * dec_quad_noff(g & 3);
  }
  const int H = a.H, W = a.W;
  const int NB = 2 * W + 2 * (H - 2);

  pdl_trigger();
#ifdef DR_TRACE
  if (threadIdx.x < 16) DT_SET(threadIdx.x, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    DT_SET(0, dt_ns());
    DT_TL(4, 0);
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    DT_SET(14, smid);
  }
#endif
  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.tok_full, 1);
    for (int i = 0; i < NBLK; ++i) {
      tc::mbar_init(&sm.w_full[i], 1);
      tc::mbar_init(&sm.w_empty[i], 1);
    }
    for (int i = 0; i < NBUF; ++i) {
      tc::mbar_init(&sm.d_full[i], 1);
      tc::mbar_init(&sm.d_empty[i], 4);
      for (int p = 0; p < 4; ++p) {
        tc::mbar_init(&sm.a2_full[i][p], 8);
        tc::mbar_init(&sm.e_full[i][p], 1);
      }
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tokmap);
    // constant weights: the first taps and decode.2's image before waiting on the
    // predecessor grid
    tc::mbar_arrive_expect_tx(&sm.tok_full, (uint32_t)(HTY * HTX * 128 + 32 * 128));
    tc::bulk_load(sm.w2, a.w2, 32 * 128, &sm.tok_full);
    for (int k = 0; k < NBLK && k < nblk; ++k) {
      tc::mbar_arrive_expect_tx(&sm.w_full[k], BLK_BYTES);
      tc::bulk_load(sm.w[k], reinterpret_cast<const uint8_t*>(a.wcomb) + (size_t)block_at(grp, G, k) * BLK_BYTES,
                    BLK_BYTES, &sm.w_full[k]);
    }
  }
  // zero the accumulator (the ring included), biases to smem
  {
    float4* z = reinterpret_cast<float4*>(&sm.acc[0][0][0]);
    for (int i = threadIdx.x; i < 3 * ACC_ROWS * ACC_RS / 4; i += THREADS) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x < 64) sm.bias[threadIdx.x] = __ldg(a.bcomb + threadIdx.x);
    if (threadIdx.x < 3) sm.b2[threadIdx.x] = __ldg(a.b2 + threadIdx.x);
  }
  pdl_wait();                    // predecessor complete: tokens written, its TMEM free
  if (threadIdx.x == 0) tc::tma_load_4d(sm.tok, &tokmap, &sm.tok_full, 0, tx0, ty0, f);
  if (warp == W_MMA) tc::tmem_alloc<TM_COLS>(&sm.tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = sm.tmem_base;

  // TMEM: quad buffer b = columns [256 b, 256 b + 256); phase p of the quad owns columns
  // 256 b + 64 p .. +63: D (fp32, pre-filled with the combined bias), then in place its
  // LeakyReLU'd fp16 A2 (first 32 columns) and decode.2's E (last 32)
  auto qcol = [&](int b, int p) { return tbase + (uint32_t)(256 * b + 64 * p); };
  if (warp == W_LOAD) {
    if (lane == 0) {                                       // ------------------- loads
      int k = 0;                                           // this CTA's offset blocks in order
      for (int i = 0; i < nq4; ++i) {
        const int g = quad_at(grp, G, i), gb = dec_quad_first(g);
        const int n = dec_quad_noff(g >> 2) * dec_quad_noff(g & 3);
        for (int bo = 0; bo < n; ++bo, ++k) {
          if (k < NBLK) continue;                          // issued in the prologue
          const int sl = k % NBLK;
          tc::mbar_wait(&sm.w_empty[sl], (uint32_t)(k / NBLK - 1) & 1u);
          tc::mbar_arrive_expect_tx(&sm.w_full[sl], BLK_BYTES);
          tc::bulk_load(sm.w[sl], reinterpret_cast<const uint8_t*>(a.wcomb) + (size_t)(gb + bo) * BLK_BYTES,
                        BLK_BYTES, &sm.w_full[sl]);
        }
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------- D(quad) += tokens(offset) x Wcomb(quad, offset)
    constexpr uint32_t idesc = tc::idesc_f16(128, 256);
    tc::mbar_wait(&sm.tok_full, 0);
    tc::fence_after();
    const uint64_t a0 = sdesc_sw128_sbo(tc::smem_u32(sm.tok), HTX * 128);
    const uint64_t b0 = tc::sdesc(tc::smem_u32(sm.w[0]), 256 * 16, 128);
    int k = 0;                                             // offset block
    for (int i = 0; i < nq4; ++i) {
      const int g = quad_at(grp, G, i), gy = g >> 2, gx = g & 3, b = i & 1;
      DT_WAIT(3, tc::mbar_wait(&sm.d_empty[b], (uint32_t)(i >> 1) & 1u));   // E of quad i-2 read
      tc::fence_after();
      if (lane == 0) DT_TL(5, i);
      for (int ia = 0; ia < dec_quad_noff(gy); ++ia)
        for (int ib = 0; ib < dec_quad_noff(gx); ++ib, ++k) {
          const uint32_t first = ia == 0 && ib == 0;        // first block: overwrite D
          const int off = tok_off(dec_quad_off(gy, ia), dec_quad_off(gx, ib));
          const int sl = k % NBLK;
          DT_WAIT(2, tc::mbar_wait(&sm.w_full[sl], (uint32_t)(k / NBLK) & 1u));
          tc::fence_after();
          const uint64_t bb = b0 + (uint64_t)(sl * (BLK_BYTES / 16));
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc::mma_f16_warp(qcol(b, 0), a0 + (uint64_t)(off * 8 + ks * 2),
                             bb + (uint64_t)(ks * (SLOT_BYTES / 16)), idesc, (first && ks == 0) ? 0u : 1u);
          tc::mma_commit_warp(&sm.w_empty[sl]);
        }
      tc::mma_commit_warp(&sm.d_full[b]);
      if (lane == 0) DT_TL(0, i);
    }
  } else if (warp == W_EMMA) {
    // --------------------------------------------------------------- E = A2 x W2te
    constexpr uint32_t idesc2 = tc::idesc_f16(128, 32);
    tc::mbar_wait(&sm.tok_full, 0);                        // w2 landed with the tokens
    const uint64_t bw2 = tc::sdesc_sw128(tc::smem_u32(sm.w2), 0);
    for (int i = 0; i < nq4; ++i) {
      const int b = i & 1;
      for (int p = 0; p < 4; ++p) {
        DT_WAIT(4, tc::mbar_wait(&sm.a2_full[b][p], (uint32_t)(i >> 1) & 1u));
        tc::fence_after();
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc::mma_ts_f16_warp(qcol(b, p) + 32, qcol(b, p) + 8 * ks, bw2 + (uint64_t)(2 * ks), idesc2,
                              ks != 0);
        tc::mma_commit_warp(&sm.e_full[b][p]);
      }
      if (lane == 0) DT_TL(2, i);
    }
  } else if (warp < W_EPI2) {
    // --------------------------------------------------------------- epilogue 1
    // two sets of 4 warps (one per TMEM lane quarter); set s takes channels 32 s .. 32 s + 31
    // of every phase, in phase order (phase p's A2 is complete after 8 arrivals): D (bias
    // included) -> LeakyReLU -> fp16 A2 in place.  The next phase's D is loaded from TMEM
    // while this one is converted.
    const int q = warp & 3, set = (warp - W_EPI1) >> 2;
    const int row = 32 * q + lane;                        // token position in the tile
    const int tyl = row >> 3, txl = row & 7;
    const uint32_t lrow = ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * set);
    const __half2 slope = __float2half2_rn(0.2f);
    for (int i = 0; i < nq4; ++i) {
      const int g = quad_at(grp, G, i), b = i & 1;
      DT_WAIT(6, tc::mbar_wait(&sm.d_full[b], (uint32_t)(i >> 1) & 1u));
      tc::fence_after();
      uint32_t v[2][32];
      DR_TMEM_LD16(qcol(b, 0) + lrow, v[0]);
      DR_TMEM_LD16(qcol(b, 0) + lrow + 16, (v[0] + 16));
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int py = 2 * (g >> 2) + (p >> 1), px = 2 * (g & 3) + (p & 1);
        const int y = y0 + 8 * tyl + py, x = x0 + 8 * txl + px;
        tc::tmem_wait_ld();
        // both sets of this lane quarter hold their D(p) before either overwrites the
        // columns with A2 (set 1's A2 lands in set 0's channel columns 16 .. 31)
        asm volatile("bar.sync %0, 64;\n" :: "r"(3 + q) : "memory");
        if (p < 3) {
          DR_TMEM_LD16(qcol(b, p + 1) + lrow, v[(p + 1) & 1]);
          DR_TMEM_LD16(qcol(b, p + 1) + lrow + 16, (v[(p + 1) & 1] + 16));
        }
        uint32_t* vp = v[p & 1];
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {                  // combined bias: 128-bit broadcasts
          const float4 bb = reinterpret_cast<const float4*>(sm.bias)[8 * set + c4];
          vp[4 * c4] = __float_as_uint(__uint_as_float(vp[4 * c4]) + bb.x);
          vp[4 * c4 + 1] = __float_as_uint(__uint_as_float(vp[4 * c4 + 1]) + bb.y);
          vp[4 * c4 + 2] = __float_as_uint(__uint_as_float(vp[4 * c4 + 2]) + bb.z);
          vp[4 * c4 + 3] = __float_as_uint(__uint_as_float(vp[4 * c4 + 3]) + bb.w);
        }
        if (y < H && x < W && on_border(y, x, H, W)) {
          // image border: the combined pre-activation is redone by dec_border
          float4* bdst = reinterpret_cast<float4*>(a.bd0 + ((size_t)f * NB + border_index(y, x, H, W)) * 64 + 32 * set);
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            bdst[c4] = make_float4(__uint_as_float(vp[4 * c4]), __uint_as_float(vp[4 * c4 + 1]),
                                   __uint_as_float(vp[4 * c4 + 2]), __uint_as_float(vp[4 * c4 + 3]));
        }
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {                    // LeakyReLU(0.2) on fp16 pairs
          const uint32_t h = pack_half2(__uint_as_float(vp[2 * c]), __uint_as_float(vp[2 * c + 1]));
          const __half2 hv = *reinterpret_cast<const __half2*>(&h);
          const __half2 r = __hmax2(hv, __hmul2(hv, slope));
          pk[c] = *reinterpret_cast<const uint32_t*>(&r);
        }
        // A2 columns of channels 32 set .. : 16 fp16 pairs at column 64 p + 16 set
        DR_TMEM_ST16(qcol(b, p) + (lrow - (uint32_t)(32 * set)) + (uint32_t)(16 * set), pk);
        tc::tmem_wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sm.a2_full[b][p]);
      }
      if (lane == 0 && q == 0) DT_TL(1, i);
    }
  } else {
    // --------------------------------------------------------------- epilogue 2
    // one warp per lane quarter scatters all 27 E values of its pixels.  Within a quad no
    // two lanes hit the same accumulator (a phase's sources are 8 pixels apart and the
    // quad's phases differ by at most one pixel), so only program order per lane and one
    // barrier per quad (the wrap from px / py 6, 7 to 0, 1 of the next cell) order the
    // read-modify-writes.  The quad's TMEM buffer is released as soon as its last E is in
    // registers.
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const int tyl = row >> 3, txl = row & 7;
    const uint32_t lrow = (uint32_t)(32 * q) << 16;
    auto release = [&](int b) {                           // buffer b free for D
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.d_empty[b]);
    };
    for (int b = 0; b < NBUF; ++b) release(b);
    // The quad's 4 phases x 9 taps land on the 4 x 4 pixel block at (2 gy - 1, 2 gx - 1)
    // of the lane's cell: summed in registers.  Along a quad row (gx = 0..3; a CTA's quads
    // are whole rows) the next block shares two columns, which stay in registers: per quad
    // one read-modify-write per pixel of the two columns left behind (all four at gx = 3).
    float blk[3][4][4];
    for (int i = 0; i < nq4; ++i) {
      const int g = quad_at(grp, G, i), b = i & 1, gy = g >> 2, gx = g & 3;
      const bool carry = gx > 0;                          // previous quad: same row, gx - 1
#pragma unroll
      for (int co = 0; co < 3; ++co)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          blk[co][u][0] = carry ? blk[co][u][2] : 0.f;
          blk[co][u][1] = carry ? blk[co][u][3] : 0.f;
          blk[co][u][2] = blk[co][u][3] = 0.f;
        }
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int dy = p >> 1, dx = p & 1;
        uint32_t ev[1][32];
        DT_WAIT(9, tc::mbar_wait(&sm.e_full[b][p], (uint32_t)(i >> 1) & 1u));
        tc::fence_after();
        DR_TMEM_LD16(qcol(b, p) + lrow + 32, ev[0]);
        DR_TMEM_LD16(qcol(b, p) + lrow + 48, (ev[0] + 16));
        tc::tmem_wait_ld();
        if (p == 3 && i + 2 < nq4) release(b);
        const int y = y0 + 8 * tyl + 2 * gy + dy, x = x0 + 8 * txl + 2 * gx + dx;   // source
        if (y < H && x < W && !on_border(y, x, H, W)) {
#pragma unroll
          for (int ky = 0; ky < 3; ++ky)
#pragma unroll
            for (int kx = 0; kx < 3; ++kx)
#pragma unroll
              for (int co = 0; co < 3; ++co)
                blk[co][dy - ky + 2][dx - kx + 2] += __uint_as_float(ev[0][3 * (3 * ky + kx) + co]);
        }
      }
      {
        const int r0 = 8 * tyl + 2 * gy, c0 = 8 * txl + 2 * gx - 1 + ACC_C0;   // block origin
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (v >= 2 && gx != 3) continue;                // (carried to gx + 1)
            const int r = r0 + u, cc = acc_col(r, c0 + v);
#pragma unroll
            for (int co = 0; co < 3; ++co) sm.acc[co][r][cc] += blk[co][u][v];
          }
      }
      __syncwarp();
      DT_WAIT(10, asm volatile("bar.sync 2, 128;\n" ::: "memory"));   // quad order
      if (lane == 0 && warp == W_EPI2) DT_TL(3, i);
    }
  }

  // ------------------------------------------------------------------- finish the tile
  // With G > 1 the G CTAs of a tile form a cluster: after a cluster barrier each finishes
  // 1/G of the tile's rows, summing the G accumulators (distributed shared memory, rank
  // order: deterministic); a second barrier keeps every accumulator alive until all reads
  // are done.
  tc::fence_before();
  __syncthreads();
#ifdef DR_TRACE
  if (threadIdx.x == 0) DT_SET(12, dt_ns());
#endif
  if (warp == W_MMA) tc::tmem_dealloc<TM_COLS>(tbase);
  if (G > 1) cluster_sync_all();
  const int ye = min(TPY, H - y0), xe = min(TPX, W - x0);
  const int rows_per = TPY / G, rbeg = grp * rows_per, rend = min(ye, rbeg + rows_per);
  const bool nb_up = y0 > 0, nb_dn = y0 + TPY < H, nb_l = x0 > 0, nb_r = x0 + TPX < W;
  const size_t plane = (size_t)H * W;
  const int ntx = (W + TPX - 1) / TPX, nty = (H + TPY - 1) / TPY;
  float* band = a.part + ((size_t)(f * nty + tile_y) * ntx + tile_x) * 3 * DEC_BAND;
  // accumulator value summed over the cluster's ranks (in rank order)
  uint32_t acc_rank[4] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (G > 1 && q < G) acc_rank[q] = map_rank(tc::smem_u32(&sm.acc[0][0][0]), q);
  auto accv = [&](int co, int r, int c) -> float {
    if (G == 1) return sm.acc[co][r][c];
    const uint32_t off = (uint32_t)(((co * ACC_ROWS + r) * ACC_RS + c) * 4);
    float p[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) p[q] = q < G ? ld_dsmem_f32(acc_rank[q] + off) : 0.f;
    float v = p[0];
#pragma unroll
    for (int q = 1; q < 4; ++q) if (q < G) v += p[q];
    return v;
  };
  // the 4 pixels xl .. xl+3 (xl % 4 == 0) of row r, channel co: one 16-byte group (every
  // rank's, summed in rank order), un-permuted
  auto acc_run = [&](int co, int r, int xl, float (&o)[4]) {
    const int c = xl + ACC_C0, g = acc_swz(r, c), base = c ^ (g & 4);
    float4 v;
    if (G == 1) {
      v = *reinterpret_cast<const float4*>(&sm.acc[co][r][base]);
    } else {
      const uint32_t off = (uint32_t)(((co * ACC_ROWS + r) * ACC_RS + base) * 4);
      v = ld_dsmem_f32x4(acc_rank[0] + off);
#pragma unroll
      for (int q = 1; q < 4; ++q)
        if (q < G) {
          const float4 w = ld_dsmem_f32x4(acc_rank[q] + off);
          v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
        }
    }
    const float e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = e4[e ^ (g & 3)];
  };
  // pixel of the tile (+ ring) that dec_fixup finishes: next to another tile or within one
  // pixel of the image border
  auto is_fix = [&](int yl, int xl, int y, int x) {
    return (yl == 0 && nb_up) || (yl == TPY - 1 && nb_dn) || (xl == 0 && nb_l) ||
           (xl == TPX - 1 && nb_r) || y <= 1 || x <= 1 || y >= H - 2 || x >= W - 2;
  };
  // interior pixels in runs of 4 along x (vector loads / stores), two runs per thread per
  // pass with the inputs loaded up front; runs holding a dec_fixup pixel go pixel by pixel
  const int nq = xe >> 2;                                  // runs per row (xe % 8 == 0)
  // Runs without any dec_fixup pixel form a rectangle [ra, rb) x [ca, cb) of the block
  // (fixup rows / columns only occur at its edges); they come first so that warps do not
  // diverge between the vector path and the pixel-by-pixel one.
  const int ra = min(rend, max(rbeg, y0 == 0 ? 2 : (nb_up ? 1 : 0)));
  const int rb = max(ra, min(rend, nb_dn ? TPY - 1 : H - 2 - y0));
  const int ca = (nb_l || x0 == 0) ? 1 : 0, cb = max(ca, (nb_r || x0 + xe >= W) ? nq - 1 : nq);
  const int n_clean = (rb - ra) * (cb - ca);
  const int n_top = (ra - rbeg) * nq, n_mid = (rb - ra) * (ca + nq - cb);
  const int nrun = max(0, rend - rbeg) * nq;
  auto run_at = [&](int id, int* yl, int* xl) {
    if (id < n_clean) {
      *yl = ra + id / (cb - ca);
      *xl = 4 * (ca + id % (cb - ca));
      return;
    }
    id -= n_clean;
    if (id < n_top) { *yl = rbeg + id / nq; *xl = 4 * (id % nq); return; }
    id -= n_top;
    if (id < n_mid) {
      const int w = ca + nq - cb, c = id % w;
      *yl = ra + id / w;
      *xl = 4 * (c < ca ? c : cb + (c - ca));
      return;
    }
    id -= n_mid;
    *yl = rb + id / nq;
    *xl = 4 * (id % nq);
  };
  const ConvTcArgs& t = a.tail;
  constexpr int NJ = DR_DEC_FINISH_RUNS;                  // runs in flight per thread
  for (int idx = threadIdx.x; idx < nrun; idx += NJ * THREADS) {
    int yy[NJ], xx[NJ];
    bool act[NJ], fast[NJ], need[NJ];
    float4 al[NJ], rf[NJ][3];
    uint32_t r8[NJ][3];
    // inputs of all runs first (vector loads), then the tails
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int id = idx + j * THREADS;
      act[j] = id < nrun;
      int yl = 0, xl = 0;
      if (act[j]) run_at(id, &yl, &xl);
      yy[j] = y0 + yl;
      xx[j] = x0 + xl;
      const bool f0 = is_fix(yl, xl, yy[j], xx[j]), f3 = is_fix(yl, xl + 3, yy[j], xx[j] + 3);
      // is_fix is monotone inside a run except at its ends: only x = tile / image edges
      need[j] = act[j] && !(f0 && f3 && is_fix(yl, xl + 1, yy[j], xx[j] + 1) && is_fix(yl, xl + 2, yy[j], xx[j] + 2));
      fast[j] = act[j] && !f0 && !f3 && !t.packed;
      if (need[j]) {
        const size_t pix = (size_t)yy[j] * W + xx[j];
        al[j] = t.alpha ? __ldg(reinterpret_cast<const float4*>(t.alpha + (size_t)f * plane + pix))
                        : make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          if (t.out_f32) rf[j][ch] = __ldg(reinterpret_cast<const float4*>(t.rgb_f32 + ((size_t)f * 3 + ch) * plane + pix));
          if (t.rgb_u8) r8[j][ch] = __ldg(reinterpret_cast<const uint32_t*>(t.rgb_u8 + ((size_t)f * plane + pix) * 3) + ch);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if (!act[j]) continue;
      const int r = yy[j] - y0 + 1;
      if (!fast[j]) {
        // pixel by pixel: partial sums for dec_fixup's pixels, the tail (preloaded inputs)
        const float alv[4] = {al[j].x, al[j].y, al[j].z, al[j].w};
        uint8_t src[12];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) *reinterpret_cast<uint32_t*>(src + 4 * ch) = r8[j][ch];
        float run[3][4];
#pragma unroll
        for (int co = 0; co < 3; ++co) acc_run(co, r, xx[j] - x0, run[co]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int x = xx[j] + e;
          float o[3] = {run[0][e], run[1][e], run[2][e]};
          if (is_fix(yy[j] - y0, x - x0, yy[j], x)) {
            const int bi = band_idx(yy[j] - y0, x - x0, ye, xe);
#pragma unroll
            for (int co = 0; co < 3; ++co) band[co * DEC_BAND + bi] = o[co];
          } else {
#pragma unroll
            for (int co = 0; co < 3; ++co) o[co] += sm.b2[co];
            const float rfe[4][3] = {{rf[j][0].x, rf[j][1].x, rf[j][2].x}, {rf[j][0].y, rf[j][1].y, rf[j][2].y},
                                     {rf[j][0].z, rf[j][1].z, rf[j][2].z}, {rf[j][0].w, rf[j][1].w, rf[j][2].w}};
            const float srcf[3] = {rfe[e][0], rfe[e][1], rfe[e][2]};
            const uint8_t src8[3] = {src[3 * e], src[3 * e + 1], src[3 * e + 2]};
            dec_emit(t, f, yy[j], x, o, alv[e], srcf, src8);
          }
        }
        continue;
      }
      // 4 pixels: tanh tail, composite, vector stores
      const float alv[4] = {al[j].x, al[j].y, al[j].z, al[j].w};
      float out01[3][4];
      bool bad = false;
#pragma unroll
      for (int co = 0; co < 3; ++co) {
        float run[4];
        acc_run(co, r, xx[j] - x0, run);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          out01[co][e] = tanh01(run[e] + sm.b2[co]);
          bad |= !isfinite(out01[co][e]);
        }
      }
      const size_t pix = (size_t)yy[j] * W + xx[j];
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const size_t pl = ((size_t)f * 3 + ch) * plane + pix;
        if (t.fill) *reinterpret_cast<float4*>(t.fill + pl) = make_float4(out01[ch][0], out01[ch][1], out01[ch][2], out01[ch][3]);
        if (t.out_f32) {
          const float src[4] = {rf[j][ch].x, rf[j][ch].y, rf[j][ch].z, rf[j][ch].w};
          float o4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            o4[e] = __fadd_rn(__fmul_rn(alv[e], out01[ch][e]), __fmul_rn(__fsub_rn(1.0f, alv[e]), src[e]));
          *reinterpret_cast<float4*>(t.out_f32 + pl) = make_float4(o4[0], o4[1], o4[2], o4[3]);
        }
      }
      if (t.out_u8) {
        uint8_t src[12], dst[12];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) *reinterpret_cast<uint32_t*>(src + 4 * ch) = r8[j][ch];
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const uint8_t fill8 = (uint8_t)fminf(fmaxf(rintf(__fmul_rn(out01[ch][e], 255.0f)), 0.f), 255.f);
            const uint8_t s8 = src[3 * e + ch];
            const float alr = alv[e];
            uint8_t ov;
            if (alr == 0.f) ov = s8;
            else if (alr == 1.f) ov = fill8;
            else ov = (uint8_t)fminf(fmaxf(rintf(__fadd_rn(__fmul_rn(alr, (float)fill8),
                                                            __fmul_rn(__fsub_rn(1.0f, alr), (float)s8))), 0.f), 255.f);
            dst[3 * e + ch] = ov;
          }
        uint32_t* d8 = reinterpret_cast<uint32_t*>(t.out_u8 + ((size_t)f * plane + pix) * 3);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) d8[ch] = *reinterpret_cast<const uint32_t*>(dst + 4 * ch);
      }
      if (bad) atomicOr(t.flags + f, 1);
    }
  }
#ifdef DR_TRACE
  __syncthreads();
  if (threadIdx.x == 0) DT_SET(11, dt_ns());
#endif
  // the outer ring (contributions to the neighbouring tiles' pixels): the top ring row with
  // the first row block, the bottom one with the last, the side columns with each block
  for (int idx = threadIdx.x; idx < 2 * (TPX + 2) + 2 * rows_per; idx += THREADS) {
    int yl, xl;
    if (idx < TPX + 2) {
      if (grp != 0) continue;
      yl = -1; xl = idx - 1;
    } else if (idx < 2 * (TPX + 2)) {
      if (grp != G - 1) continue;
      yl = TPY; xl = idx - (TPX + 2) - 1;
    } else if (idx < 2 * (TPX + 2) + rows_per) {
      yl = rbeg + idx - 2 * (TPX + 2); xl = -1;
    } else {
      yl = rbeg + idx - 2 * (TPX + 2) - rows_per; xl = TPX;
    }
    const int y = y0 + yl, x = x0 + xl;
    if (y < 0 || x < 0 || y >= H || x >= W) continue;
    const int r = yl + 1, cc = acc_col(r, xl + ACC_C0), bi = band_idx(yl, xl, ye, xe);
#pragma unroll
    for (int co = 0; co < 3; ++co) band[co * DEC_BAND + bi] = accv(co, r, cc);
  }
  if (G > 1) cluster_sync_all();                           // the ranks' reads are done
#ifdef DR_TRACE
  __syncthreads();
  if (threadIdx.x == 0) DT_SET(13, dt_ns());
#endif
}

// Image-border pixels: pre-activation = the combined one (stored by dec_fused) minus the
// decode.0 taps reading the canvas ring, LeakyReLU, fp16, then decode.2's 27 taps.  One CTA
// per (frame, edge, phase r = position mod 8) for the edge's pixels at positions r + 8k
// (corners excluded; one CTA per corner below): they share the 1-2 correction
// matrices dK[edge][v] (v = r, and r + 8 for r <= 1 / r - 8 for r >= 6), staged in shared
// memory with the edge's token row; per 64 pixels a [64 px x 64 ci] x [64 ci x 64 co]
// product per tap, LeakyReLU, fp16 rounding, then the 27 decode.2 taps.
struct BorderSmem {
  float k[2][64][64];                            // [tap][ci][co]
  float tok[66][68];                             // tokens k0-1 .. k0+64 of the edge line
  float d0[64][68];                              // rows 16-byte aligned (float4 reads)
  float w2[27][68];                              // 16-byte rows; a quarter warp's 8 u hit 32 banks
  float eb[64];
};

__global__ void __launch_bounds__(256) dec_border_kernel(const __grid_constant__ DecArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  BorderSmem& sm = *reinterpret_cast<BorderSmem*>(smem_raw);
  pdl_trigger();
  const int H = a.H, W = a.W, NB = 2 * W + 2 * (H - 2);
  const int tid = threadIdx.x;
  const int sp = a.border_split;                        // CTAs per (frame, edge, phase)
  const int nmain = a.frames * 32 * sp;
  if ((int)blockIdx.x >= nmain) {
    // one CTA per image corner: thread (co, q) sums a quarter (16 ci) of every correction
    // gemv of the pixel (its two edges' taps, minus the corner table), reduced in smem
    const int c = (int)blockIdx.x - nmain, f = c >> 2, k = c & 3;
    const int y = (k & 2) ? H - 1 : 0, x = (k & 1) ? W - 1 : 0;
    const int co = tid & 63, q = tid >> 6;
    const int PC = a.Cc + 2, PR = a.R + 2;
    pdl_wait();
    const __half* tokf = a.tok16 + (size_t)f * PR * PC * 64;
    auto part16 = [&](const float* kmat, int ty, int tx) {  // sum over ci in [16q, 16q+16)
      const __half* tp = tokf + ((size_t)(ty + 1) * PC + (tx + 1)) * 64 + 16 * q;
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) acc = fmaf(__half2float(tp[i]), __ldg(kmat + (size_t)(16 * q + i) * 64 + co), acc);
      return acc;
    };
    float corr = 0.f;
#pragma unroll
    for (int ed = 0; ed < 4; ++ed) {
      const bool on = ed == 0 ? y == 0 : (ed == 1 ? y == H - 1 : (ed == 2 ? x == 0 : x == W - 1));
      if (!on) continue;
      if (q == 0) corr += __ldg(a.dk + DK_EB + ed * 64 + co);
      const bool along_x = ed < 2;
      const int pos = along_x ? x : y;
      const int line = ed == 0 ? 0 : (ed == 1 ? a.R - 1 : (ed == 2 ? 0 : a.Cc - 1));
      const int nlim = along_x ? a.Cc : a.R;
      for (int t = pos / 8 - 1; t <= pos / 8 + 1; ++t) {
        const int v = pos - 8 * t;
        if (v < -2 || v > 9 || t < 0 || t >= nlim) continue;
        corr += part16(a.dk + DK_EDGE + (size_t)(ed * 12 + v + 2) * 4096, along_x ? line : t, along_x ? t : line);
      }
    }
    {   // the doubly removed corner tap
      const bool top = (k & 2) == 0, left = (k & 1) == 0;
      const int c4 = (top ? 0 : 2) + (left ? 0 : 1);
      corr -= part16(a.dk + DK_CORNER + (size_t)c4 * 4096, top ? 0 : a.R - 1, left ? 0 : a.Cc - 1);
      if (q == 0) corr -= __ldg(a.dk + DK_CB + c4 * 64 + co);
    }
    float* red = &sm.d0[0][0];                           // [4][64] partials, then d0
    red[q * 64 + co] = corr;
    __syncthreads();
    const int bi = border_index(y, x, H, W);
    if (tid < 64) {
      const float cs = (red[co] + red[64 + co]) + (red[128 + co] + red[192 + co]);
      float d = a.bd0[((size_t)f * NB + bi) * 64 + co] - cs;
      d = d >= 0.f ? d : 0.2f * d;
      sm.w2[0][co] = __half2float(__float2half_rn(d));    // decode.0's output is fp16
    }
    __syncthreads();
    if (tid < 27) {
      float e = 0.f;
      for (int cc = 0; cc < 64; ++cc) e = fmaf(__ldg(a.w2f + tid * 64 + cc), sm.w2[0][cc], e);
      a.be[((size_t)f * NB + bi) * 27 + tid] = e;
    }
    return;
  }
  const int bq = blockIdx.x / sp, part = blockIdx.x - bq * sp;
  const int f = bq / 32, ed = (bq >> 3) & 3, r = bq & 7;
  const bool along_x = ed < 2;
  const int len = along_x ? W : H;
  const int line = ed == 0 ? 0 : (ed == 1 ? a.R - 1 : (ed == 2 ? 0 : a.Cc - 1));
  const int nlim = along_x ? a.Cc : a.R;
  const int nt = (r <= 1 || r >= 6) ? 2 : 1, dt1 = r <= 1 ? -1 : 1;   // tap 1: token k + dt1
  // constants first (before the predecessor grid completes)
  for (int t = 0; t < nt; ++t) {
    const int v = t == 0 ? r : r - 8 * dt1;
    const float4* src = reinterpret_cast<const float4*>(a.dk + DK_EDGE + (size_t)(ed * 12 + v + 2) * 4096);
    float4* dst = reinterpret_cast<float4*>(&sm.k[t][0][0]);
    for (int i = tid; i < 1024; i += 256) dst[i] = __ldg(src + i);
  }
  for (int i = tid; i < 27 * 64; i += 256) sm.w2[i >> 6][i & 63] = __ldg(a.w2f + i);
  if (tid < 64) sm.eb[tid] = __ldg(a.dk + DK_EB + ed * 64 + tid);
  // this CTA's share of the edge pixels r + 8k, k in [k_lo, k_hi]
  const int k_first = r == 0 ? 1 : 0, k_last = (len - 2 - r) >= 0 ? (len - 2 - r) / 8 : -1;
  const int nk = k_last - k_first + 1, per = (nk + sp - 1) / sp;
  const int k_lo = k_first + part * per, k_hi = min(k_last, k_lo + per - 1);
  const int PC = a.Cc + 2, PR = a.R + 2;
  pdl_wait();
  const __half* tokf = a.tok16 + (size_t)f * PR * PC * 64;
  for (int kb = k_lo; kb <= k_hi; kb += 64) {
    const int cnt = min(64, k_hi - kb + 1);              // pixels of this pass
    __syncthreads();
    for (int i = tid; i < 66 * 32; i += 256) {          // tokens kb-1 .. kb+64, half2 pairs
      const int j = i >> 5, c2 = i & 31, t = kb - 1 + j;
      float2 v = make_float2(0.f, 0.f);
      if (t >= 0 && t < nlim) {
        const int ty = along_x ? line : t, tx = along_x ? t : line;
        v = __half22float2(reinterpret_cast<const __half2*>(tokf + ((size_t)(ty + 1) * PC + (tx + 1)) * 64)[c2]);
      }
      sm.tok[j][2 * c2] = v.x;
      sm.tok[j][2 * c2 + 1] = v.y;
    }
    __syncthreads();
    // thread (channel quad cq, pg) takes channels 4cq .. 4cq+3 of the pixels j = pg + 16i:
    // 4 of them per pass, 1 when the pass has <= 16 (small batches).  Every broadcast
    // token float4 feeds 16 FMAs, the weights come as float4 quads.
    const int cq = tid & 15, pg16 = tid >> 4;
    auto corr_pass = [&](auto ni_tag) {
      constexpr int NI = decltype(ni_tag)::value;
      float4 acc[NI], pre[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        acc[i] = *reinterpret_cast<const float4*>(&sm.eb[4 * cq]);
        // the pixels' stored pre-activations, loaded before the products
        const int k = kb + pg16 + 16 * i, pos = r + 8 * k;
        const int y = along_x ? (ed == 0 ? 0 : H - 1) : pos, x = along_x ? pos : (ed == 2 ? 0 : W - 1);
        pre[i] = k <= k_hi ? __ldg(reinterpret_cast<const float4*>(
                                 a.bd0 + ((size_t)f * NB + border_index(y, x, H, W)) * 64 + 4 * cq))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      auto fma4 = [](float4 t, float4 w0, float4 w1, float4 w2, float4 w3, float4 c) {
        c.x = fmaf(t.x, w0.x, fmaf(t.y, w1.x, fmaf(t.z, w2.x, fmaf(t.w, w3.x, c.x))));
        c.y = fmaf(t.x, w0.y, fmaf(t.y, w1.y, fmaf(t.z, w2.y, fmaf(t.w, w3.y, c.y))));
        c.z = fmaf(t.x, w0.z, fmaf(t.y, w1.z, fmaf(t.z, w2.z, fmaf(t.w, w3.z, c.z))));
        c.w = fmaf(t.x, w0.w, fmaf(t.y, w1.w, fmaf(t.z, w2.w, fmaf(t.w, w3.w, c.w))));
        return c;
      };
      for (int t = 0; t < nt; ++t) {
        const int o = 1 + (t == 0 ? 0 : dt1);            // token row of pixel j: j + o
#pragma unroll 2
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 w0 = *reinterpret_cast<const float4*>(&sm.k[t][4 * c4][4 * cq]);
          const float4 w1 = *reinterpret_cast<const float4*>(&sm.k[t][4 * c4 + 1][4 * cq]);
          const float4 w2 = *reinterpret_cast<const float4*>(&sm.k[t][4 * c4 + 2][4 * cq]);
          const float4 w3 = *reinterpret_cast<const float4*>(&sm.k[t][4 * c4 + 3][4 * cq]);
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            const float4 tv = *reinterpret_cast<const float4*>(&sm.tok[pg16 + 16 * i + o][4 * c4]);
            acc[i] = fma4(tv, w0, w1, w2, w3, acc[i]);
          }
        }
      }
      auto tail = [](float p, float q) {
        float d = p - q;
        d = d >= 0.f ? d : 0.2f * d;
        return __half2float(__float2half_rn(d));          // decode.0's output is fp16
      };
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int j = pg16 + 16 * i, k = kb + j;
        float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k <= k_hi)
          d = make_float4(tail(pre[i].x, acc[i].x), tail(pre[i].y, acc[i].y),
                          tail(pre[i].z, acc[i].z), tail(pre[i].w, acc[i].w));
        *reinterpret_cast<float4*>(&sm.d0[j][4 * cq]) = d;
      }
    };
    if (cnt <= 16) corr_pass(std::integral_constant<int, 1>{});
    else corr_pass(std::integral_constant<int, 4>{});
    __syncthreads();
    for (int i = tid; i < cnt * 27; i += 256) {
      const int j = i / 27, u = i - 27 * j, k = kb + j, pos = r + 8 * k;
      if (k > k_hi) continue;
      float e0 = 0.f, e1 = 0.f;                          // two chains, 128-bit operand loads
#pragma unroll 4
      for (int c = 0; c < 64; c += 8) {
        const float4 wa = *reinterpret_cast<const float4*>(&sm.w2[u][c]);
        const float4 da = *reinterpret_cast<const float4*>(&sm.d0[j][c]);
        const float4 wb = *reinterpret_cast<const float4*>(&sm.w2[u][c + 4]);
        const float4 db = *reinterpret_cast<const float4*>(&sm.d0[j][c + 4]);
        e0 = fmaf(wa.x, da.x, fmaf(wa.y, da.y, fmaf(wa.z, da.z, fmaf(wa.w, da.w, e0))));
        e1 = fmaf(wb.x, db.x, fmaf(wb.y, db.y, fmaf(wb.z, db.z, fmaf(wb.w, db.w, e1))));
      }
      const float e = e0 + e1;
      const int y = along_x ? (ed == 0 ? 0 : H - 1) : pos, x = along_x ? pos : (ed == 2 ? 0 : W - 1);
      a.be[((size_t)f * NB + border_index(y, x, H, W)) * 27 + u] = e;
    }
  }
}

// The pixels dec_fused left: the sum of the band partials of every tile whose 1-pixel-
// expanded area holds the pixel (<= 4 tiles, a fixed order), plus the image-border
// sources' E, then the tail.  The last CTA mirrors the flags (host path).
__global__ void __launch_bounds__(256) dec_fixup_kernel(const __grid_constant__ DecArgs a) {
  pdl_trigger();
  const int f = blockIdx.y;
  const int H = a.H, W = a.W, NB = 2 * W + 2 * (H - 2);
  const int nr = a.n_fix_rows, nc = a.n_fix_cols;
  const long n_runs = (long)nr * (W / 4);                // fix rows, in runs of 4
  const long n_items = n_runs + (long)(H - nr) * nc;
  float b2[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) b2[c] = __ldg(a.b2 + c);
  pdl_wait();
  const int ntx = (W + TPX - 1) / TPX, nty = (H + TPY - 1) / TPY;
  const ConvTcArgs& tl = a.tail;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n_items; i += (long)gridDim.x * blockDim.x) {
    int y, x, n;
    if (i < n_runs) {                                   // 4 pixels of a finished row
      const int r = (int)(i / (W / 4));
      y = a.fix_rows[r];
      x = 4 * (int)(i - (long)r * (W / 4));
      n = 4;
    } else {                                            // a fix column of another row
      const long j = i - n_runs;
      int yy = (int)(j / nc);
      x = a.fix_cols[(int)(j - (long)yy * nc)];
      for (int k = 0; k < nr; ++k)                      // the yy-th row not in fix_rows
        if (yy >= a.fix_rows[k]) ++yy;
      y = yy;
      n = 1;
    }
    const int ty_a = max(0, y - 1) / TPY, ty_b = min(H - 1, y + 1) / TPY;
    const int tx_a = max(0, x - 1) / TPX, tx_b = min(W - 1, x + n) / TPX;
    float o[4][3];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int co = 0; co < 3; ++co) o[e][co] = b2[co];
    // tile (ty, tx) holds pixel (y, x') iff y - y0 in [-1, ye] and x' - x0 in [-1, xe]
    for (int ty = ty_a; ty <= ty_b; ++ty) {
      const int yl = y - TPY * ty, ye = min(TPY, H - TPY * ty);
      if (yl < -1 || yl > ye) continue;
      for (int tx = tx_a; tx <= tx_b; ++tx) {
        const int xe = min(TPX, W - TPX * tx);
        const float* bp = a.part + ((size_t)(f * nty + ty) * ntx + tx) * 3 * DEC_BAND;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int xl = x + e - TPX * tx;
          if (e >= n || xl < -1 || xl > xe) continue;
          const int bi = band_idx(yl, xl, ye, xe);
#pragma unroll
          for (int co = 0; co < 3; ++co) o[e][co] += __ldg(bp + co * DEC_BAND + bi);
        }
      }
    }
    for (int e = 0; e < n; ++e) {
      const int xe = x + e;
      float oo[3] = {o[e][0], o[e][1], o[e][2]};
      if (y <= 1 || xe <= 1 || y >= H - 2 || xe >= W - 2) {
        // image-border sources p = (y + ky - 1, xe + kx - 1), tap (ky, kx): all nine loads
        // issued before the sums (fixed tap order)
        float ev9[9][3];
#pragma unroll
        for (int t9 = 0; t9 < 9; ++t9) {
          const int ky = t9 / 3, kx = t9 % 3, py = y + ky - 1, px = xe + kx - 1;
          const bool src = py >= 0 && px >= 0 && py < H && px < W && on_border(py, px, H, W);
          const float* ev = a.be + ((size_t)f * NB + (src ? border_index(py, px, H, W) : 0)) * 27 + 3 * t9;
#pragma unroll
          for (int co = 0; co < 3; ++co) ev9[t9][co] = src ? __ldg(ev + co) : 0.f;
        }
#pragma unroll
        for (int t9 = 0; t9 < 9; ++t9)
#pragma unroll
          for (int co = 0; co < 3; ++co) oo[co] += ev9[t9][co];
      }
      float alr, srcf[3];
      uint8_t src8[3];
      dec_inputs(tl, f, y, xe, &alr, srcf, src8);
      dec_emit(tl, f, y, xe, oo, alr, srcf, src8);
    }
  }
  // flags mirror (host path): the last CTA to finish publishes the frames' flags
  const ConvTcArgs& t = a.tail;
  if (t.flags_mirror || t.mirror_after_spans) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned total = gridDim.x * gridDim.y * gridDim.z;
      if (atomicAdd(t.done, 1u) == total - 1) {
        __threadfence();
        int* fm = t.flags_mirror;
        if (t.mirror_after_spans) {
          const int4 sp = t.spans[t.H - 1];
          const size_t n = (size_t)sp.z + 3 * (size_t)(sp.y - sp.x);
          fm = reinterpret_cast<int*>(t.packed + ((n + 3) & ~(size_t)3));
        }
        for (int k = 0; k < t.frames; ++k) fm[k] = atomicOr(t.flags + k, 0);
        *t.done = 0;
      }
    }
  }
}

}  // namespace

size_t dec_border_table_floats() { return DK_TOTAL; }
size_t dec_part_floats(int frames, int H, int W) {
  return (size_t)frames * ((H + TPY - 1) / TPY) * ((W + TPX - 1) / TPX) * 3 * DEC_BAND;
}
int dec_border_pixels(int H, int W) { return 2 * W + 2 * (H - 2); }

// Phase groups per tile: enough CTAs for about one wave at small batch (4 at one 512^2
// frame: 32 tiles).
int dec_groups(int frames, int H, int W, int sms) {
  const int tiles = frames * ((H + TPY - 1) / TPY) * ((W + TPX - 1) / TPX);
  if (tiles >= sms) return 1;
  if (2 * tiles >= sms) return 2;
  return 4;
}

void dec_fix_lines(DecArgs& a) {
  std::vector<int> rows = {0, 1, a.H - 2, a.H - 1}, cols = {0, 1, a.W - 2, a.W - 1};
  for (int k = TPY; k < a.H; k += TPY) { rows.push_back(k - 1); rows.push_back(k); }
  for (int k = TPX; k < a.W; k += TPX) { cols.push_back(k - 1); cols.push_back(k); }
  auto finish = [](std::vector<int>& v, int n, short* out, int* cnt) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    v.erase(std::remove_if(v.begin(), v.end(), [n](int e) { return e < 0 || e >= n; }), v.end());
    *cnt = (int)std::min<size_t>(v.size(), DEC_MAX_FIX);
    for (int i = 0; i < *cnt; ++i) out[i] = (short)v[i];
  };
  finish(rows, a.H, a.fix_rows, &a.n_fix_rows);
  finish(cols, a.W, a.fix_cols, &a.n_fix_cols);
}

#ifdef DR_TRACE
std::vector<std::vector<unsigned long long>>& dec_trace_store() {
  static std::vector<std::vector<unsigned long long>> v;
  return v;
}
#endif

void launch_dec_fused(const CUtensorMap& tok4d, const DecArgs& a, cudaStream_t s) {
  static unsigned long long init = 0;
  const int smem = (int)sizeof(DecSmem) + 1024;
  once_per_device(init, [&] {
    cudaFuncSetAttribute(dec_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  const dim3 grid((a.W + TPX - 1) / TPX, ((a.H + TPY - 1) / TPY) * a.groups, a.frames);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;         // the G phase groups of a tile
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = a.groups;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, dec_fused_kernel, tok4d, a);
#ifdef DR_TRACE
  if (dec_trace_store().size() < 4) {
    cudaStreamSynchronize(s);
    const int n = std::min(4096, (int)(grid.x * grid.y * grid.z));
    std::vector<unsigned long long> h((size_t)n * 16);
    cudaMemcpyFromSymbol(h.data(), g_dec_trace, h.size() * sizeof(unsigned long long));
    dec_trace_store().push_back(std::move(h));
    std::vector<unsigned long long> tl(6 * 64);
    cudaMemcpyFromSymbol(tl.data(), g_dec_tl, tl.size() * sizeof(long long));
    dec_trace_store().push_back(std::move(tl));
  }
#endif
}

void launch_dec_border(const DecArgs& a, cudaStream_t s) {
  static unsigned long long init = 0;
  const int smem = (int)sizeof(BorderSmem);
  once_per_device(init, [&] {
    cudaFuncSetAttribute(dec_border_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  // frames x 4 edges x 8 phases (x split: about two CTAs per SM at small batches), then one
  // CTA per corner
  DecArgs b = a;
  b.border_split = std::min(4, std::max(1, (device_sms() + a.frames * 32 - 1) / (a.frames * 32)));
  const int blocks = a.frames * 32 * b.border_split + 4 * a.frames;
  launch_pdl(dec_border_kernel, dim3(blocks), dim3(256), smem, s, b);
}

void launch_dec_fixup(const DecArgs& a, cudaStream_t s) {
  const long n_items = (long)a.n_fix_rows * (a.W / 4) + (long)(a.H - a.n_fix_rows) * a.n_fix_cols;
  const int blocks = (int)std::max<long>(1, std::min<long>((n_items + 255) / 256, 1024));
  launch_pdl(dec_fixup_kernel, dim3(blocks, a.frames), dim3(256), 0, s, a);
}

}  // namespace dr

#ifdef DR_TRACE
extern "C" int dr_debug_dec_trace(int idx, unsigned long long* host, int n) {
  auto& v = dr::dec_trace_store();
  if (idx < 0 || idx >= (int)v.size()) return -1;
  const int k = std::min(n, (int)v[idx].size());
  for (int i = 0; i < k; ++i) host[i] = v[idx][i];
  return k;
}
#endif
