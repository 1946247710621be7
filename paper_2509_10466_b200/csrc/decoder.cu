// Token grid -> raster -> RGB fill -> alpha composite.
//
//  vec2patch  ConvTranspose2d(64,64,k=10,s=8) + crop 1 (dstt.py:198-221) as an
//             output-stationary phase GEMM: canvas pixel (8i+py, 8j+px) sums token (i,j)
//             through kernel tap (py,px), plus (i-1,j) through (py+8,px) when py<2, etc.
//             (1, 2 or 4 taps per pixel; 100 taps x 64 x 64 MACs per token in total)
//  decode0    Conv3x3(64->64, pad 1) + LeakyReLU(0.2) (dstt.py:241-242), implicit GEMM
//             M = pixels, K = 9 taps x 64, N = 64, over a swizzled smem halo tile
//  decode2    Conv3x3(64->3, pad 1) (:243), (tanh+1)/2 (:267), non-finite guard
//             (:322-323), u8 conversion (:324-325) and the alpha composite (base.py:87-88
//             generalised to a feathered alpha), all fused in one tail
// Rasters are NHWC fp16 (128 B per pixel) so every implicit-GEMM A row is one cache line.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

// ------------------------------------------------------------------ vec2patch
constexpr int V2P_WARPS = 4;

DR_DEV void load_tok_a(uint32_t a[4][4], const __half* __restrict__ tok, int i, int j0,
                       int R, int Cc, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool iv = i >= 0 && i < R;
  const int ja = j0 + g, jb = j0 + g + 8;
  const bool va = iv && ja >= 0 && ja < Cc, vb = iv && jb >= 0 && jb < Cc;
  const uint32_t* ra = reinterpret_cast<const uint32_t*>(tok + (size_t)(i * Cc + ja) * C);
  const uint32_t* rb = reinterpret_cast<const uint32_t*>(tok + (size_t)(i * Cc + jb) * C);
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) {
    a[kt][0] = va ? __ldg(ra + kt * 8 + t) : 0u;
    a[kt][1] = vb ? __ldg(rb + kt * 8 + t) : 0u;
    a[kt][2] = va ? __ldg(ra + kt * 8 + 4 + t) : 0u;
    a[kt][3] = vb ? __ldg(rb + kt * 8 + 4 + t) : 0u;
  }
}

DR_DEV void mma_tap(float (*acc)[4], const uint32_t (*a)[4], const uint2* __restrict__ w,
                    int tap, int lane) {
  const uint2* wt = w + (size_t)tap * 32 * 32;     // 32 fragments per tap
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const uint2 b = ld_frag(wt, nt * 4 + kt, lane);
      mma16816(acc[nt], a[kt], b.x, b.y);
    }
}

__global__ void __launch_bounds__(V2P_WARPS * 32) v2p_kernel(DecodeArgs a) {
  __shared__ __align__(16) uint32_t stage[V2P_WARPS][16][32];   // 16 px x 64 ch fp16
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nJ = (a.Cc + 1 + 15) / 16;
  const long gw = (long)blockIdx.x * V2P_WARPS + warp;
  const long total = (long)a.frames * (a.R + 1) * nJ;
  if (gw >= total) return;
  const int jc = (int)(gw % nJ);
  const long r2 = gw / nJ;
  const int i = (int)(r2 % (a.R + 1));
  const int f = (int)(r2 / (a.R + 1));
  const int j0 = jc * 16;
  const __half* tok = a.tok16 + (size_t)f * a.R * a.Cc * C;
  uint32_t t0[4][4], tu[4][4], tl[4][4], tul[4][4];
  load_tok_a(t0, tok, i, j0, a.R, a.Cc, lane);
  load_tok_a(tu, tok, i - 1, j0, a.R, a.Cc, lane);
  load_tok_a(tl, tok, i, j0 - 1, a.R, a.Cc, lane);
  load_tok_a(tul, tok, i - 1, j0 - 1, a.R, a.Cc, lane);
  uint32_t* st = &stage[warp][0][0];
#pragma unroll 1
  for (int py = 0; py < 8; ++py) {
    const int y = 8 * i + py - 1;
    if (y < 0 || y >= a.H) continue;
#pragma unroll 1
    for (int px = 0; px < 8; ++px) {
      float acc[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float b0 = __ldg(a.bv2p + nt * 8 + 2 * t), b1 = __ldg(a.bv2p + nt * 8 + 2 * t + 1);
        acc[nt][0] = b0; acc[nt][1] = b1; acc[nt][2] = b0; acc[nt][3] = b1;
      }
      mma_tap(acc, t0, a.wv2p, py * 10 + px, lane);
      if (py < 2) mma_tap(acc, tu, a.wv2p, (py + 8) * 10 + px, lane);
      if (px < 2) mma_tap(acc, tl, a.wv2p, py * 10 + px + 8, lane);
      if (py < 2 && px < 2) mma_tap(acc, tul, a.wv2p, (py + 8) * 10 + px + 8, lane);
      // stage 16 pixels x 64 channels; 16-byte chunk swizzle (chunk ^ (row & 7))
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int chunk = nt, word = t;            // channel pair (nt*8 + 2t) -> word t of chunk nt
        st[g * 32 + ((chunk ^ (g & 7)) * 4) + word] = pack_half2(acc[nt][0], acc[nt][1]);
        st[(g + 8) * 32 + ((chunk ^ ((g + 8) & 7)) * 4) + word] = pack_half2(acc[nt][2], acc[nt][3]);
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int row = it * 4 + (lane >> 3), chunk = lane & 7;
        const int x = 8 * (j0 + row) + px - 1;
        if (x >= 0 && x < a.W) {
          const uint4 v = *reinterpret_cast<const uint4*>(st + row * 32 + ((chunk ^ (row & 7)) * 4));
          *reinterpret_cast<uint4*>(a.raster + (((size_t)f * a.H + y) * a.W + x) * C + chunk * 8) = v;
        }
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ 3x3 convolutions
constexpr int CT_H = 8, CT_W = 32;                 // output tile
constexpr int HALO_H = CT_H + 2, HALO_W = CT_W + 2;
constexpr int HALO_BYTES = HALO_H * HALO_W * 128;

// Load the (CT_H+2) x (CT_W+2) x 64-channel fp16 halo into smem with zero padding.
// Pixel p, 16-byte chunk c is stored at p*128 + ((c ^ (p & 7)) * 16).
DR_DEV void load_halo(uint8_t* smem, const __half* __restrict__ src, int f, int y0, int x0,
                      int H, int W) {
  for (int e = threadIdx.x; e < HALO_H * HALO_W * 8; e += blockDim.x) {
    const int p = e >> 3, c = e & 7;
    const int hy = p / HALO_W, hx = p - hy * HALO_W;
    const int y = y0 + hy - 1, x = x0 + hx - 1;
    const bool v = y >= 0 && y < H && x >= 0 && x < W;
    const __half* g = v ? src + (((size_t)f * H + y) * W + x) * C + c * 8 : src;
    cp_async16_zfill(smem + p * 128 + ((c ^ (p & 7)) * 16), g, v);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
}

// A fragments (16 px x 16 ch) for k-tile kt of the pixel run starting at halo pixel p0.
DR_DEV void halo_a(uint32_t a[4], const uint8_t* smem, int p0, int kt, int lane) {
  const int mi = lane >> 3;
  const int p = p0 + (lane & 7) + (mi & 1) * 8;
  const int c = 2 * kt + (mi >> 1);
  ldmatrix_x4(a, smem + p * 128 + ((c ^ (p & 7)) * 16));
}

__global__ void __launch_bounds__(256) decode0_kernel(DecodeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int x0 = blockIdx.x * CT_W, y0 = blockIdx.y * CT_H, f = blockIdx.z;
  load_halo(smem, a.raster, f, y0, x0, a.H, a.W);
  float acc[2][8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const float b0 = __ldg(a.bd0 + nt * 8 + 2 * t), b1 = __ldg(a.bd0 + nt * 8 + 2 * t + 1);
#pragma unroll
    for (int m = 0; m < 2; ++m) { acc[m][nt][0] = b0; acc[m][nt][1] = b1; acc[m][nt][2] = b0; acc[m][nt][3] = b1; }
  }
#pragma unroll 1
  for (int tap = 0; tap < 9; ++tap) {
    const int dy = tap / 3, dx = tap - dy * 3;
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      uint32_t a0[4], a1[4];
      halo_a(a0, smem, (warp + dy) * HALO_W + dx, kt, lane);
      halo_a(a1, smem, (warp + dy) * HALO_W + dx + 16, kt, lane);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const uint2 b = ld_frag(a.wd0, (tap * 8 + nt) * 4 + kt, lane);
        mma16816(acc[0][nt], a0, b.x, b.y);
        mma16816(acc[1][nt], a1, b.x, b.y);
      }
    }
  }
  __syncthreads();                                   // halo no longer needed: reuse for staging
  uint32_t* st = reinterpret_cast<uint32_t*>(smem);  // [CT_H][CT_W][32 words], swizzled
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) { const float u = acc[m][nt][e]; v[e] = u >= 0.f ? u : 0.2f * u; }
      const int pa = warp * CT_W + m * 16 + g, pb = pa + 8;
      st[pa * 32 + ((nt ^ (pa & 7)) * 4) + t] = pack_half2(v[0], v[1]);
      st[pb * 32 + ((nt ^ (pb & 7)) * 4) + t] = pack_half2(v[2], v[3]);
    }
  __syncthreads();
  for (int e = threadIdx.x; e < CT_H * CT_W * 8; e += blockDim.x) {
    const int p = e >> 3, c = e & 7;
    const int y = y0 + p / CT_W, x = x0 + (p % CT_W);
    if (y < a.H && x < a.W) {
      const uint4 v = *reinterpret_cast<const uint4*>(st + p * 32 + ((c ^ (p & 7)) * 4));
      *reinterpret_cast<uint4*>(a.d0 + (((size_t)f * a.H + y) * a.W + x) * C + c * 8) = v;
    }
  }
}

__global__ void __launch_bounds__(256) decode2_kernel(DecodeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int x0 = blockIdx.x * CT_W, y0 = blockIdx.y * CT_H, f = blockIdx.z;
  load_halo(smem, a.d0, f, y0, x0, a.H, a.W);
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll 1
  for (int tap = 0; tap < 9; ++tap) {
    const int dy = tap / 3, dx = tap - dy * 3;
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      uint32_t a0[4], a1[4];
      halo_a(a0, smem, (warp + dy) * HALO_W + dx, kt, lane);
      halo_a(a1, smem, (warp + dy) * HALO_W + dx + 16, kt, lane);
      const uint2 b = ld_frag(a.wd2, tap * 4 + kt, lane);
      mma16816(acc[0], a0, b.x, b.y);
      mma16816(acc[1], a1, b.x, b.y);
    }
  }
  if (t >= 2) return;                                // channels 2t, 2t+1: only 0..2 are real
  const int y = y0 + warp;
  if (y >= a.H) return;
  const size_t plane = (size_t)a.H * a.W;
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int x = x0 + m * 16 + g + half * 8;
      if (x >= a.W) continue;
      const size_t pix = (size_t)y * a.W + x;
      const float al = a.alpha ? a.alpha[(size_t)f * plane + pix] : 1.f;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ch = 2 * t + e;
        if (ch >= 3) continue;
        const float raw = acc[m][half * 2 + e] + __ldg(a.bd2 + ch);
        const float out01 = (tanhf(raw) + 1.0f) * 0.5f;
        if (!isfinite(out01)) atomicOr(a.flags + f, 1);
        if (a.fill) a.fill[((size_t)f * 3 + ch) * plane + pix] = out01;
        if (a.out_f32) {
          const float fr = a.rgb_f32[((size_t)f * 3 + ch) * plane + pix];
          a.out_f32[((size_t)f * 3 + ch) * plane + pix] =
              __fadd_rn(__fmul_rn(al, out01), __fmul_rn(__fsub_rn(1.0f, al), fr));
        }
        if (a.out_u8) {
          const float s = fminf(fmaxf(rintf(__fmul_rn(out01, 255.0f)), 0.f), 255.f);
          const uint8_t fill8 = (uint8_t)s;
          const uint8_t src8 = a.rgb_u8[((size_t)f * plane + pix) * 3 + ch];
          uint8_t o;
          if (al == 0.f) o = src8;
          else if (al == 1.f) o = fill8;
          else {
            const float mix = __fadd_rn(__fmul_rn(al, (float)fill8),
                                        __fmul_rn(__fsub_rn(1.0f, al), (float)src8));
            o = (uint8_t)fminf(fmaxf(rintf(mix), 0.f), 255.f);
          }
          a.out_u8[((size_t)f * plane + pix) * 3 + ch] = o;
        }
      }
    }
}

}  // namespace

void launch_vec2patch(const DecodeArgs& a, cudaStream_t s) {
  const int nJ = (a.Cc + 1 + 15) / 16;
  const long warps = (long)a.frames * (a.R + 1) * nJ;
  v2p_kernel<<<(unsigned)((warps + V2P_WARPS - 1) / V2P_WARPS), V2P_WARPS * 32, 0, s>>>(a);
}

void launch_decode0(const DecodeArgs& a, cudaStream_t s) {
  static bool attr = false;
  const int smem = HALO_BYTES > CT_H * CT_W * 128 ? HALO_BYTES : CT_H * CT_W * 128;
  if (!attr) {
    cudaFuncSetAttribute(decode0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(decode2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((a.W + CT_W - 1) / CT_W, (a.H + CT_H - 1) / CT_H, a.frames);
  decode0_kernel<<<grid, 256, smem, s>>>(a);
}

void launch_decode2(const DecodeArgs& a, cudaStream_t s) {
  const int smem = HALO_BYTES;
  dim3 grid((a.W + CT_W - 1) / CT_W, (a.H + CT_H - 1) / CT_H, a.frames);
  decode2_kernel<<<grid, 256, smem, s>>>(a);
}

}  // namespace dr
