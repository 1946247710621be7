// Mask stage: privacy mask m0 -> dilated m1 -> feathered alpha, token validity, and the
// packed fp16 network input.  HBM-bound integer/byte work; no tensor cores.
//
//  pack_bits   m0 u8 rows -> 32-pixel bit words (warp ballot, coalesced byte reads)
//  dilate      m1 = m0 (+) L1-ball(r) == r-fold 3x3-cross dilation (masks.py:17, :193;
//              SURVEY A2): OR over rows dy of the row dilated horizontally by r-|dy|,
//              on bit words (shift/or), bit-exact by construction; off-frame = 0
//  token_pack  token valid = any pixel of the patch outside m1; network
//              input cat[rgb zeroed in m1, m1] as fp16 in conv-weight (c,ky,kx) order
//              (dstt.py:253, :314-316; u8 -> f32 is an IEEE divide by 255); redaction
//              check of the u8 API (base.py:76-79) -> flags bit 1
//  feather     alpha = max(m1, G_sigma(m1)) with scipy.ndimage.gaussian_filter semantics
//              (mode 'nearest', truncate 4): vertical then horizontal pass, each in
//              float64 in scipy's symmetric-filter summation order, rounded to float32
//              between passes, so alpha is bit-identical to scipy
#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

__global__ void pack_bits_kernel(const uint8_t* __restrict__ m0, uint32_t* __restrict__ bits,
                                 int frames, int H, int W, int Ww) {
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long total = (long)frames * H * Ww;
  if (warp >= total) return;
  const int w = (int)(warp % Ww);
  const long row = warp / Ww;                       // frame * H + y
  const int x = w * 32 + lane;
  const bool set = x < W && m0[row * W + x] != 0;
  const uint32_t word = __ballot_sync(0xffffffffu, set);
  if (lane == 0) bits[row * Ww + w] = word;
}

__global__ void dilate_kernel(const uint32_t* __restrict__ b0, uint32_t* __restrict__ b1,
                              uint8_t* __restrict__ m1, float* __restrict__ alpha, int frames,
                              int H, int W, int Ww, int r) {
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)frames * H * Ww;
  if (idx >= total) return;
  const int w = (int)(idx % Ww);
  const long row = idx / Ww;
  const int y = (int)(row % H);
  const long f = row / H;
  const uint32_t* fb = b0 + f * (long)H * Ww;
  uint32_t acc = 0;
  for (int dy = -r; dy <= r; ++dy) {
    const int yy = y + dy;
    if (yy < 0 || yy >= H) continue;
    const int k = r - (dy < 0 ? -dy : dy);
    const uint32_t cur = fb[(long)yy * Ww + w];
    const uint32_t lf = w > 0 ? fb[(long)yy * Ww + w - 1] : 0u;
    const uint32_t rt = w + 1 < Ww ? fb[(long)yy * Ww + w + 1] : 0u;
    uint32_t hd = cur;
    for (int s = 1; s <= k; ++s)
      hd |= (cur << s) | (lf >> (32 - s)) | (cur >> s) | (rt << (32 - s));
    acc |= hd;
  }
  const int valid_bits = W - w * 32;
  if (valid_bits < 32) acc &= (1u << valid_bits) - 1u;
  b1[idx] = acc;
  const long px = row * W + (long)w * 32;
  if (m1) {
    for (int i = 0; i < 32 && i < valid_bits; ++i) m1[px + i] = (acc >> i) & 1u;
  }
  if (alpha) {
    for (int i = 0; i < 32 && i < valid_bits; ++i) alpha[px + i] = (float)((acc >> i) & 1u);
  }
}

// One warp per token.  P = patch size (8: 4 ch x 8 rows lanes, 4: 4 ch x 4 rows).
template <int P>
__global__ void token_pack_kernel(MaskArgs a) {
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int R = a.H / P, Cc = a.W / P, T = R * Cc;
  if (warp >= (long)a.frames * T) return;
  const int f = (int)(warp / T), tok = (int)(warp - (long)f * T);
  const int i = tok / Cc, j = tok - i * Cc;
  const int Ww = (a.W + 31) / 32;
  constexpr int ROWS = P;                 // lanes: c = lane / ROWS, ky = lane % ROWS
  const bool active = lane < 4 * ROWS;
  const int c = lane / ROWS, ky = lane % ROWS;
  const int y = i * P + ky, x0 = j * P;
  uint32_t mbits = 0, m0bits = 0;
  if (active) {
    const long wrow = ((long)f * a.H + y) * Ww + (x0 >> 5);
    mbits = (a.bits1[wrow] >> (x0 & 31)) & ((1u << P) - 1u);
    m0bits = (a.bits0[wrow] >> (x0 & 31)) & ((1u << P) - 1u);
  }
  const bool any_unmasked = __any_sync(0xffffffffu, active && mbits != ((1u << P) - 1u));
  if (lane == 0) a.token_valid[warp] = any_unmasked ? 1 : 0;
  if (a.xin == nullptr) return;
  float v[P];
  bool dirty = false;
  if (!active) {
#pragma unroll
    for (int kx = 0; kx < P; ++kx) v[kx] = 0.f;
  } else if (c == 3) {
#pragma unroll
    for (int kx = 0; kx < P; ++kx) v[kx] = (float)((mbits >> kx) & 1u);
  } else if (a.rgb_f32) {
    const float* src = a.rgb_f32 + (((long)f * 3 + c) * a.H + y) * a.W + x0;
#pragma unroll
    for (int kx = 0; kx < P; kx += 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(src + kx));
      v[kx] = q.x; v[kx + 1] = q.y; v[kx + 2] = q.z; v[kx + 3] = q.w;
    }
#pragma unroll
    for (int kx = 0; kx < P; ++kx) if ((mbits >> kx) & 1u) v[kx] = 0.f;
  } else {
    const uint8_t* src = a.rgb_u8 + (((long)f * a.H + y) * a.W + x0) * 3 + c;
#pragma unroll
    for (int kx = 0; kx < P; ++kx) {
      const uint8_t u = __ldg(src + 3 * kx);
      dirty |= ((m0bits >> kx) & 1u) && u != 0;
      v[kx] = ((mbits >> kx) & 1u) ? 0.f : __fdiv_rn((float)u, 255.0f);
    }
  }
  const bool any_dirty = __any_sync(0xffffffffu, dirty);
  if (a.flags && any_dirty && lane == 0) atomicOr(a.flags + f, 2);
  if (!active) return;
  __half* dst = a.xin + ((long)f * T + tok) * (4 * P * P) + c * P * P + ky * P;
  uint32_t packed[P / 2];
#pragma unroll
  for (int kx = 0; kx < P; kx += 2) packed[kx / 2] = pack_half2(v[kx], v[kx + 1]);
  if constexpr (P == 8) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  } else {
    *reinterpret_cast<uint2*>(dst) = make_uint2(packed[0], packed[1]);
  }
}

// Fused separable feather on a TILE_H x TILE_W tile; vertical pass into smem (float32),
// horizontal pass out.  The summation order replicates scipy's NI_Correlate1D for
// symmetric weights: out = x[0]*w[0]; for jj=-R..-1: out += (x[jj] + x[-jj]) * w[jj].
constexpr int FT_H = 16, FT_W = 64, FT_MAXR = 32;

__global__ void __launch_bounds__(256) feather_kernel(MaskArgs a) {
  __shared__ float vs[FT_H][FT_W + 2 * FT_MAXR];
  __shared__ double wsm[2 * FT_MAXR + 1];
  const int R = a.feather_radius;
  const int Ww = (a.W + 31) / 32;
  const int x0 = blockIdx.x * FT_W, y0 = blockIdx.y * FT_H, f = blockIdx.z;
  for (int i = threadIdx.x; i < 2 * R + 1; i += blockDim.x) wsm[i] = a.feather_w[i];
  __syncthreads();
  const uint32_t* fb = a.bits1 + (long)f * a.H * Ww;
  const double* wc = wsm + R;                       // centre tap
  const int span = FT_W + 2 * R;
  for (int e = threadIdx.x; e < FT_H * span; e += blockDim.x) {
    const int ty = e / span, tx = e - ty * span;
    const int y = y0 + ty;
    int x = x0 + tx - R;
    x = x < 0 ? 0 : (x >= a.W ? a.W - 1 : x);     // 'nearest' in x (input to pass 2)
    if (y >= a.H) { vs[ty][tx] = 0.f; continue; }
    auto bit = [&](int yy) -> double {
      yy = yy < 0 ? 0 : (yy >= a.H ? a.H - 1 : yy);
      return (double)((fb[(long)yy * Ww + (x >> 5)] >> (x & 31)) & 1u);
    };
    double acc = __dmul_rn(bit(y), wc[0]);
    for (int jj = -R; jj < 0; ++jj)
      acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(bit(y + jj), bit(y - jj)), wc[jj]));
    vs[ty][tx] = (float)acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < FT_H * FT_W; e += blockDim.x) {
    const int ty = e / FT_W, tx = e - ty * FT_W;
    const int y = y0 + ty, x = x0 + tx;
    if (y >= a.H || x >= a.W) continue;
    // pass-2 input at column x+d: smem column tx + R + d, clamped to the frame
    auto g = [&](int d) -> double {
      int xx = x + d;
      xx = xx < 0 ? 0 : (xx >= a.W ? a.W - 1 : xx);
      return (double)vs[ty][xx - x0 + R];
    };
    double acc = __dmul_rn(g(0), wc[0]);
    for (int jj = -R; jj < 0; ++jj)
      acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(g(jj), g(-jj)), wc[jj]));
    const float m = (float)((fb[(long)y * Ww + (x >> 5)] >> (x & 31)) & 1u);
    a.alpha[((long)f * a.H + y) * a.W + x] = fmaxf(m, (float)acc);
  }
}

}  // namespace

void launch_mask_stage(const MaskArgs& a, cudaStream_t s) {
  const int Ww = (a.W + 31) / 32;
  const long words = (long)a.frames * a.H * Ww;
  pack_bits_kernel<<<(unsigned)((words + 7) / 8), 256, 0, s>>>(a.m0, a.bits0, a.frames, a.H, a.W, Ww);
  dilate_kernel<<<(unsigned)((words + 127) / 128), 128, 0, s>>>(
      a.bits0, a.bits1, a.m1, a.feather_radius == 0 ? a.alpha : nullptr, a.frames, a.H, a.W,
      Ww, a.radius);
  if (a.token_valid) {
    const long toks = (long)a.frames * (a.H / a.patch) * (a.W / a.patch);
    if (a.patch == 8)
      token_pack_kernel<8><<<(unsigned)((toks + 7) / 8), 256, 0, s>>>(a);
    else if (a.patch == 4)
      token_pack_kernel<4><<<(unsigned)((toks + 7) / 8), 256, 0, s>>>(a);
  }
  if (a.feather_radius > 0 && a.alpha) {
    dim3 grid((a.W + FT_W - 1) / FT_W, (a.H + FT_H - 1) / FT_H, a.frames);
    feather_kernel<<<grid, 256, 0, s>>>(a);
  }
}

}  // namespace dr
