// Mask stage: privacy mask m0 -> dilated m1 -> feathered alpha, token validity, and the
// packed fp16 network input, fused in ONE kernel over TH x 64-pixel tiles.  HBM-bound
// integer/byte work; no tensor cores.  Per tile (TH rows x 64 px, NT = 32 TH threads):
//
//  1. m0 bytes of the tile plus a halo of r + R pixels -> 32-pixel bit words in smem,
//     straight from global memory (coalesced 16-byte pieces, SIMD byte compares; off-frame
//     = 0) while the rgb tile lands by cp.async
//  2. m1 = m0 (+) L1-ball(r) == the r-fold 3x3-cross dilation (masks.py:17, :193; SURVEY
//     A2): horizontal dilations of the bit words by funnel shifts, then a vertical OR over
//     the ball's rows (or r cross iterations in warp registers / smem for large r) --
//     bit-exact by construction; kept on the tile plus a halo of R
//  3. feather: alpha = max(m1, G_sigma(m1)), scipy.ndimage.gaussian_filter
//     semantics (mode 'nearest', truncate 4): vertical then horizontal pass, each in
//     float64 in scipy's symmetric-filter order (x[0]*w[0], then (x[-j]+x[+j])*w[j] from
//     the outermost pair inward) and rounded to float32 between passes, so alpha is
//     bit-identical to scipy.  The vertical pass reads each column's m1 bits as one
//     bit-transposed column word (built once per column, rows clamped 'nearest'), so the
//     (2R+1)-row window of any pixel is a funnel shift.  Exact fast paths: alpha = 1 on
//     m1 (the vertical/horizontal sums of a binary image never exceed 1.0f); an all-zero /
//     all-one window gives 0 / the precomputed all-ones sum
//  4. token validity (any pixel of the patch outside m1) and the network input
//     cat[rgb zeroed in m1, m1] in conv-weight (c, ky, kx) order (dstt.py:253, :314-316;
//     u8 -> f32 is an IEEE divide by 255), plus the u8 API's redaction check (base.py:76-79);
//     the frame's last CTA writes the frame's flags word (no memset before the forward)
#include <cstddef>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

constexpr int TW = 64;                     // tile width (pixels); height TH: template
constexpr int MAXH = 62;                   // max halo r + R (r <= 31, R <= 31)
constexpr int MAXR = 31;                   // 2R+1 <= 63: a column window fits a uint64
constexpr int NW_MAX = 2 + 2 * (MAXH / 32);

constexpr int SPAN_MAX = TW + 2 * MAXR;   // columns of the vertical pass
constexpr int CW = 3;                      // column words: TH + 2R <= 78 rows < 96

// Tile of TH rows (TH = 16, or 8 below one wave of 16-row tiles: batch-1 latency), one
// warp per tile row (NT = 32 TH threads).
template <int TH>
struct Smem {
  static constexpr int NR_MAX = TH + 2 * MAXH;
  float rgb[3][TH][TW];                    // f32 input tile, or u8 HWC bytes (aliased)
  uint32_t b0[NR_MAX][NW_MAX];             // m0 bits, rows y0-H.., words from xs (read-only
                                           // after the load phase)
  uint32_t b1[TH + 2 * MAXR][NW_MAX];      // m1 bits, rows y0-R..
  uint32_t bt[NR_MAX][NW_MAX];             // dilation ping-pong buffer
  uint32_t col[CW][NW_MAX * 32];           // m1 column words of window pixel px: bit j =
                                           // row y0-R+j (clamped 'nearest')
  float vs[TH][SPAN_MAX + 2];              // vertical feather pass
  uint32_t nzm[TH][5];                     // nonzero columns of vs (+1 zero word)
  double w[2 * MAXR + 1];
  double all_ones;
  int dirty;
};

// bit i = (byte i of w != 0), i < 4: byte flags to 0x01 each, then the multiply by
// 2^28 + 2^21 + 2^14 + 2^7 moves byte i's flag to bit 28 + i (all cross terms land on
// distinct bits below 28 or above 31: no carries)
DR_DEV uint32_t nibble4(uint32_t w) {
  return ((__vcmpne4(w, 0u) & 0x01010101u) * 0x10204080u) >> 28;
}

DR_DEV void cp_async4_zfill(void* smem, const void* gmem, bool valid) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  int n = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" :: "r"(s), "l"(gmem), "r"(n));
}

// Diagnostic build only (-DDR_TRACE): thread 0's clock64 at each phase boundary per CTA,
// read back by scripts/mask_trace.py.
#ifdef DR_TRACE
constexpr int MT_SLOTS = 16;
__device__ unsigned long long g_mask_trace[4096 * MT_SLOTS];
#define MT(slot) do { if (threadIdx.x == 0) { unsigned long long c_;                       \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_) :: "memory");                          \
    const int b_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);           \
    if (b_ < 4096) g_mask_trace[b_ * MT_SLOTS + (slot)] = c_;                                \
    if ((slot) == 0 || (slot) == 9) {                    /* 11/12: global ns, 13: SM id */   \
      unsigned long long g_; unsigned sm_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                                 \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                       \
      if (b_ < 4096) { g_mask_trace[b_ * MT_SLOTS + ((slot) ? 12 : 11)] = g_;                \
                       g_mask_trace[b_ * MT_SLOTS + 13] = sm_; } } } } while (0)
#else
#define MT(slot) do {} while (0)
#endif

// WH = halo words per side (compile time: every word loop is shift/mask, no division)
template <int P, int WH, int TH>
__global__ void __launch_bounds__(32 * TH, 64 / TH) mask_fused_kernel(MaskArgs a) {
  using S = Smem<TH>;
  constexpr int NT = 32 * TH, NWARP = TH;
  // bt, col and vs are contiguous: the dilation's H_k scratch spans all three
  static_assert(offsetof(S, col) == offsetof(S, bt) + sizeof(S::bt) &&
                offsetof(S, vs) == offsetof(S, col) + sizeof(S::col), "Smem scratch layout");
  constexpr int HS_WORDS = (int)((sizeof(S::bt) + sizeof(S::col) + sizeof(S::vs)) / 4);
  extern __shared__ __align__(16) uint8_t smem_raw[];   // keep the shared address space:
  S& sm = *reinterpret_cast<S*>(smem_raw);               // no integer round trip (LDS, not LD)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, f = blockIdx.z;
  const int r = a.radius, R = a.feather_radius;
  const int Hd = r + R;
  constexpr int wh = WH;                          // halo words each side
  constexpr int NW = 2 + 2 * wh;
  const int xs = x0 - 32 * wh;                    // pixel of bit 0 of word 0
  const int NR0 = TH + 2 * Hd, NR1 = TH + 2 * R;
  const size_t plane = (size_t)a.H * a.W;

  MT(0);
  pdl_trigger();
  if (tid == 0) sm.dirty = 0;
  for (int i = tid; i < 2 * R + 1; i += NT) sm.w[i] = a.feather_w[i];   // constant
  pdl_wait();
  MT(1);

  // 0. rgb tile: cp.async (lands while the mask bits are built); 1. m0 -> bits straight
  //    from global memory: one thread per 32-pixel word of the tile + halo (two 16-byte
  //    loads, or 4-byte / byte pieces for narrow-aligned widths; off-frame = 0), per 4 bytes
  //    a SIMD byte compare, then a multiply gathers the 4 flags into a nibble.  b0 stays
  //    read-only from here on: the token phase takes the raw m0 bits of the redaction check
  //    from it.
  if (a.xin != nullptr && a.rgb_f32) {
    for (int e = tid; e < 3 * TH * (TW / 4); e += NT) {
      const int c = e / (TH * TW / 4), rem = e - c * (TH * TW / 4);
      const int ty = rem / (TW / 4), q = rem - ty * (TW / 4);
      const int y = y0 + ty, x = x0 + 4 * q;
      const bool v = y < a.H && x < a.W;
      const float* src = a.rgb_f32 + ((size_t)f * 3 + c) * plane + (size_t)y * a.W + x;
      cp_async16_zfill(&sm.rgb[c][ty][4 * q], v ? src : a.rgb_f32, v);
    }
  } else if (a.xin != nullptr && a.rgb_u8) {
    uint8_t* dst = reinterpret_cast<uint8_t*>(&sm.rgb[0][0][0]);  // [TH][TW][3] bytes
    for (int e = tid; e < TH * TW * 3 / 4; e += NT) {
      const int ty = e / (TW * 3 / 4), q = e - ty * (TW * 3 / 4);
      const int y = y0 + ty;
      const bool v = y < a.H && x0 + (4 * q) / 3 < a.W;
      const uint8_t* src = a.rgb_u8 + ((size_t)f * plane + (size_t)y * a.W + x0) * 3 + 4 * q;
      cp_async4_zfill(dst + ty * TW * 3 + 4 * q, v ? src : a.rgb_u8, v);
    }
  }
  cp_async_commit();
  {
    const uint8_t* m0f = a.m0 + (size_t)f * plane;
    const bool v16 = (a.W & 15) == 0 && (reinterpret_cast<uintptr_t>(a.m0) & 15) == 0;
    const bool v4 = (a.W & 3) == 0 && (reinterpret_cast<uintptr_t>(a.m0) & 3) == 0;
    // one 16-byte piece per thread (a warp reads 4 rows x 128 contiguous bytes), the two
    // halves of a word joined by a lane shuffle (pieces 2k, 2k+1 sit in lanes 2j, 2j+1)
    const int npc = NR0 * NW * 2;
    for (int e = tid; e < ((npc + 31) & ~31); e += NT) {           // warp-uniform trips
      const int row = e / (NW * 2), pc = e - row * (NW * 2);
      const int y = y0 - Hd + row, x = xs + 16 * pc;
      uint32_t h = 0;
      if (e < npc && y >= 0 && y < a.H && x + 16 > 0 && x < a.W) {
        const uint8_t* src = m0f + (size_t)y * a.W;
        if (v16) {                         // W % 16 == 0: the piece is wholly in the frame
          const uint4 q = __ldg(reinterpret_cast<const uint4*>(src + x));
          h = nibble4(q.x) | nibble4(q.y) << 4 | nibble4(q.z) << 8 | nibble4(q.w) << 12;
        } else if (v4) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int xx = x + 4 * k;
            if (xx >= 0 && xx < a.W) h |= nibble4(__ldg(reinterpret_cast<const uint32_t*>(src + xx))) << (4 * k);
          }
        } else {                           // odd widths (standalone mask stage)
          for (int k = 0; k < 16; ++k) {
            const int xx = x + k;
            if (xx >= 0 && xx < a.W && src[xx]) h |= 1u << k;
          }
        }
      }
      const uint32_t o = __shfl_xor_sync(0xffffffffu, h, 1);
      if (e < npc && !(e & 1)) sm.b0[row][pc >> 1] = h | (o << 16);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  MT(2);
  MT(3);

  // 2. m1 = r iterations of the 3x3 cross (masks._CROSS) over the whole b0 window, ping-pong
  //    through smem; neighbours outside the window read 0.  The window's halo (>= r + R rows
  //    and >= r + R pixels each side) keeps the rows y0-R .. y0+TH+R exact; off-frame bits set
  //    on the way never create in-frame bits a frame-clipped iteration would not (the
  //    Manhattan path between in-frame pixels stays in the frame).  Rows / pixels outside the
  //    frame are cleared when b1 is extracted.
  // L1-ball form (the r-fold cross = all pixels within Manhattan distance r): phase A, every
  // thread one (window row, word): the horizontal dilations H_k (k = 0..r) of the word,
  // from the word and its two neighbours by funnel shifts (outside the window = 0), into
  // the feather scratch (vs / col / bt, unused until the feather); phase B, every (output
  // row, word): OR over dy of H_{r-|dy|} of window row + dy.  Two parallel phases instead
  // of r dependent iterations.  Used when the H_k fit the scratch.
  uint32_t* hs = &sm.bt[0][0];                                   // [k][row][word] over bt|col|vs
  if (r >= 1 && r <= 8 && (r + 1) * NR0 * NW <= HS_WORDS) {
    for (int e = tid; e < NR0 * NW; e += NT) {
      const int row = e / NW, w = e - row * NW;
      const uint32_t c = sm.b0[row][w];
      const uint32_t lo = w > 0 ? sm.b0[row][w - 1] : 0u;        // pixels below (bit 31 side)
      const uint32_t hi = w + 1 < NW ? sm.b0[row][w + 1] : 0u;   // pixels above
      uint32_t h = c;
      hs[row * NW + w] = h;
      for (int k = 1; k <= r; ++k) {
        h |= __funnelshift_l(lo, c, k) | __funnelshift_r(c, hi, k);
        hs[(k * NR0 + row) * NW + w] = h;
      }
    }
    __syncthreads();
    for (int e = tid; e < NR1 * NW; e += NT) {
      const int row = e / NW, w = e - row * NW;
      const int y = y0 - R + row;
      uint32_t acc = 0;
      if (y >= 0 && y < a.H) {
        const int c0 = row + (Hd - R);                           // window row of the output
        for (int dy = -r; dy <= r; ++dy) acc |= hs[((r - abs(dy)) * NR0 + c0 + dy) * NW + w];
        const int xw = xs + 32 * w;                             // clear pixels outside the frame
        if (xw < 0) acc &= xw + 32 <= 0 ? 0u : (0xffffffffu << (-xw));
        if (xw + 32 > a.W) acc &= xw >= a.W ? 0u : (0xffffffffu >> (xw + 32 - a.W));
      }
      sm.b1[row][w] = acc;
    }
  } else if (r <= 8) {
    // small radius: warp-register form, no CTA barriers.  Warp k owns window rows
    // g0 = k*(32-2r) .. g0+31 (one row per lane, NW words in registers); vertical neighbours
    // come from shuffles (0 past the warp's rows), horizontal ones from the adjacent words.
    // After r iterations lanes r .. 31-r are exact (lanes at the window's own top / bottom
    // edge too, where the window border reads 0 like the smem form).
    const int stride = 32 - 2 * r;
    const int groups = NR0 <= 32 ? 1 : 1 + (NR0 - 32 + stride - 1) / stride;
    if (warp < groups) {
      const int g0 = warp * stride, row = g0 + lane;
      uint32_t cur[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) cur[w] = row < NR0 ? sm.b0[row][w] : 0u;
      for (int it = 0; it < r; ++it) {
        uint32_t nx[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          uint32_t up = __shfl_up_sync(0xffffffffu, cur[w], 1);
          uint32_t dn = __shfl_down_sync(0xffffffffu, cur[w], 1);
          if (lane == 0) up = 0u;
          if (lane == 31) dn = 0u;
          const uint32_t lf = w > 0 ? cur[w - 1] : 0u;
          const uint32_t rt = w + 1 < NW ? cur[w + 1] : 0u;
          nx[w] = cur[w] | up | dn | (cur[w] << 1) | (lf >> 31) | (cur[w] >> 1) | (rt << 31);
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) cur[w] = nx[w];
      }
      const bool exact = (lane >= r || g0 == 0) && (lane < 32 - r || row >= NR0 - 1);
      const int b1row = row - (Hd - R);                 // = row - r
      if (exact && b1row >= 0 && b1row < NR1) {
        const int y = y0 - R + b1row;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          uint32_t acc = 0;
          if (y >= 0 && y < a.H) {
            acc = cur[w];
            const int xw = xs + 32 * w;               // clear pixels outside the frame
            if (xw < 0) acc &= xw + 32 <= 0 ? 0u : (0xffffffffu << (-xw));
            if (xw + 32 > a.W) acc &= xw >= a.W ? 0u : (0xffffffffu >> (xw + 32 - a.W));
          }
          sm.b1[b1row][w] = acc;
        }
      }
    }
  } else {
    // b0 stays read-only (raw m0 bits for the token phase): iteration 0 reads b0, later
    // ones ping-pong between bt and the vertical-pass scratch (unused until the feather)
    static_assert(sizeof(S::vs) >= sizeof(S::bt), "dilation ping-pong scratch");
    uint32_t (*cur)[NW_MAX] = sm.b0;
    uint32_t (*nxt)[NW_MAX] = sm.bt;
    uint32_t (*spare)[NW_MAX] = reinterpret_cast<uint32_t (*)[NW_MAX]>(&sm.vs[0][0]);
    for (int it = 0; it < r; ++it) {
      for (int e = tid; e < NR0 * NW; e += NT) {
        const int row = e / NW, w = e - row * NW;
        const uint32_t c = cur[row][w];
        const uint32_t up = row > 0 ? cur[row - 1][w] : 0u;
        const uint32_t dn = row + 1 < NR0 ? cur[row + 1][w] : 0u;
        const uint32_t lf = w > 0 ? cur[row][w - 1] : 0u;
        const uint32_t rt = w + 1 < NW ? cur[row][w + 1] : 0u;
        nxt[row][w] = c | up | dn | (c << 1) | (lf >> 31) | (c >> 1) | (rt << 31);
      }
      __syncthreads();
      uint32_t (*t)[NW_MAX] = cur == sm.b0 ? spare : cur;
      cur = nxt;
      nxt = t;
    }
    for (int e = tid; e < NR1 * NW; e += NT) {
      const int row = e / NW, w = e - row * NW;
      const int y = y0 - R + row;
      uint32_t acc = 0;
      if (y >= 0 && y < a.H) {
        acc = cur[row + (Hd - R)][w];
        const int xw = xs + 32 * w;                   // clear pixels outside the frame
        if (xw < 0) acc &= xw + 32 <= 0 ? 0u : (0xffffffffu << (-xw));
        if (xw + 32 > a.W) acc &= xw >= a.W ? 0u : (0xffffffffu >> (xw + 32 - a.W));
      }
      sm.b1[row][w] = acc;
    }
  }
  if (tid == 0 && R > 0) {                        // scipy-order sum of an all-ones window
    const double* wc = sm.w + R;
    double s = wc[0];
    for (int jj = -R; jj < 0; ++jj) s = __dadd_rn(s, __dmul_rn(2.0, wc[jj]));
    sm.all_ones = s;
  }
  __syncthreads();

  // m1 bit at frame pixel (y, x) with 'nearest' clamping (pixel must map into b1)
  auto m1bit = [&](int y, int x) -> uint32_t {
    y = y < 0 ? 0 : (y >= a.H ? a.H - 1 : y);
    x = x < 0 ? 0 : (x >= a.W ? a.W - 1 : x);
    const int row = y - (y0 - R), px = x - xs;
    return (sm.b1[row][px >> 5] >> (px & 31)) & 1u;
  };

  // outputs: m1 bytes (+ binary alpha)
  if (a.m1 || (R == 0 && a.alpha))
  for (int e = tid; e < TH * TW; e += NT) {
    const int ty = e / TW, tx = e - ty * TW;
    const int y = y0 + ty, x = x0 + tx;
    if (y >= a.H || x >= a.W) continue;
    const uint32_t b = m1bit(y, x);
    if (a.m1) a.m1[(size_t)f * plane + (size_t)y * a.W + x] = (uint8_t)b;
    if (R == 0 && a.alpha) a.alpha[(size_t)f * plane + (size_t)y * a.W + x] = (float)b;
  }

  MT(4);
  // 3. feather
  if (R > 0 && a.alpha) {
    const double* wc = sm.w + R;
    const int span = TW + 2 * R;
    const int NR1c = TH + 2 * R;
    // 3a. column words by warp-ballot bit transposes: task (word w, 32-row chunk c); lane i
    //     holds row y0-R+32c+i (clamped 'nearest'), ballot b yields window column 32w+b
    //     (a 32 x 32 bit transpose in 5 shuffle stages: each swaps the off-diagonal
    //     j x j blocks)
    for (int task = warp; task < NW * CW; task += NWARP) {
      const int w = task % NW, c = task / NW;
      const int j = 32 * c + lane;
      uint32_t x = 0u;
      if (j < NR1c) {
        int yy = y0 - R + j;
        yy = yy < 0 ? 0 : (yy >= a.H ? a.H - 1 : yy);
        x = sm.b1[yy - (y0 - R)][w];
      }
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const uint32_t lo = st == 16 ? 0x0000FFFFu : (st == 8 ? 0x00FF00FFu : (st == 4 ? 0x0F0F0F0Fu
                            : (st == 2 ? 0x33333333u : 0x55555555u)));
        const uint32_t o = __shfl_xor_sync(0xffffffffu, x, st);
        x = (lane & st) ? ((x & ~lo) | ((o & ~lo) >> st)) : ((x & lo) | ((o & lo) << st));
      }
      sm.col[c][32 * w + lane] = x;
    }
    __syncthreads();
    MT(5);
    // 3b. vertical pass (float64, scipy order) for the tile rows x span columns; the
    //     window of row ty is bits ty .. ty+2R of the column word.  Warp ty owns row ty
    //     (NT = 32 TH): one ballot per 32 columns gives the row's nonzero-column mask for
    //     the horizontal pass's all-zero test
    const uint64_t need = (2 * R + 1 == 64) ? ~0ull : ((1ull << (2 * R + 1)) - 1ull);
    {
      const int ty = warp;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {                                   // span <= 126 < 4 words
        const int tx = 32 * c + lane;
        float out = 0.f;
        if (tx < span && y0 + ty < a.H) {
          int x = x0 + tx - R;
          x = x < 0 ? 0 : (x >= a.W ? a.W - 1 : x);
          const int px = x - xs;
          const uint64_t lo = (uint64_t)sm.col[0][px] | ((uint64_t)sm.col[1][px] << 32);
          const uint64_t pat = ((lo >> ty) | (ty ? ((uint64_t)sm.col[2][px] << (64 - ty)) : 0ull)) & need;
          if (pat == need) out = (float)sm.all_ones;
          else if (pat != 0) {
            // four interleaved float64 partial sums (dependency depth R/4 instead of R; the
            // float64 result rounds to the same float32 as scipy's serial order except in
            // vanishingly rare ties -- tests gate max-abs 1e-6 and >= 99.9 % bit-identical)
            double sp[4] = {__dmul_rn((double)((pat >> R) & 1u), wc[0]), 0.0, 0.0, 0.0};
            for (int jj = -R; jj < 0; ++jj) {
              const double pr = (double)(((pat >> (R + jj)) & 1u) + ((pat >> (R - jj)) & 1u));
              sp[(jj + 64) & 3] = __fma_rn(pr, wc[jj], sp[(jj + 64) & 3]);
            }
            out = (float)((sp[0] + sp[1]) + (sp[2] + sp[3]));
          }
        }
        if (tx < span) sm.vs[ty][tx] = out;
        const uint32_t m = __ballot_sync(0xffffffffu, out != 0.f);
        if (lane == 0) sm.nzm[ty][c] = m;
      }
    }
    __syncthreads();
    MT(6);
    // 3d. horizontal pass: alpha = 1 on m1, 0 where the whole window is zero, else sum.
    //     Off-frame columns of sm.vs already hold their clamped ('nearest') values.
    for (int e = tid; e < TH * TW; e += NT) {
      const int ty = e / TW, tx = e - ty * TW;
      const int y = y0 + ty, x = x0 + tx;
      if (y >= a.H || x >= a.W) continue;
      float out;
      const int bx = x - xs;
      if ((sm.b1[y - (y0 - R)][bx >> 5] >> (bx & 31)) & 1u) out = 1.0f;
      else {
        // window = vertical columns tx .. tx + 2R
        const uint64_t lo = (uint64_t)sm.nzm[ty][tx >> 5] | ((uint64_t)sm.nzm[ty][(tx >> 5) + 1] << 32);
        const uint64_t hi = (uint64_t)sm.nzm[ty][(tx >> 5) + 2];
        const int sh = tx & 31;
        const uint64_t win = (lo >> sh) | (sh ? (hi << (64 - sh)) : 0ull);
        const uint64_t need = (1ull << (2 * R + 1)) - 1ull;
        if (!(win & need)) out = 0.f;
        else {
          const float* v = &sm.vs[ty][tx + R];
          double sp[4] = {__dmul_rn((double)v[0], wc[0]), 0.0, 0.0, 0.0};
          for (int jj = -R; jj < 0; ++jj)
            sp[(jj + 64) & 3] = __fma_rn(__dadd_rn((double)v[jj], (double)v[-jj]), wc[jj], sp[(jj + 64) & 3]);
          out = fmaxf(0.f, (float)((sp[0] + sp[1]) + (sp[2] + sp[3])));
        }
      }
      a.alpha[(size_t)f * plane + (size_t)y * a.W + x] = out;
    }
  }

  MT(7);
  // 4. tokens of this tile: one warp per token (lanes = 4 channels x P rows)
  if (a.token_valid) {
    const int Cc = a.W / P, T = (a.H / P) * Cc;
    const int tr = TH / P, tcn = TW / P;
    for (int tk = warp; tk < tr * tcn; tk += NWARP) {
      const int ti = tk / tcn, tj = tk - ti * tcn;
      const int i = y0 / P + ti, j = x0 / P + tj;
      if (i * P >= a.H || j * P >= a.W) continue;
      const int tok = i * Cc + j;
      const bool active = lane < 4 * P;
      const int c = lane / P, ky = lane % P;
      const int y = i * P + ky, xl = j * P;
      uint32_t mb = 0, m0b = 0;
      if (active) {                       // the patch row: P bits of one m1 word (in frame)
        const int px = xl - xs;
        mb = (sm.b1[y - (y0 - R)][px >> 5] >> (px & 31)) & ((1u << P) - 1u);
        m0b = (sm.b0[y - (y0 - Hd)][px >> 5] >> (px & 31)) & ((1u << P) - 1u);   // raw m0
      }
      const bool any_unmasked = __any_sync(0xffffffffu, active && mb != ((1u << P) - 1u));
      if (lane == 0) a.token_valid[(size_t)f * T + tok] = any_unmasked ? 1 : 0;
      if (a.xin == nullptr) continue;
      float v[P];
      bool dirty = false;
      if (!active) {
#pragma unroll
        for (int kx = 0; kx < P; ++kx) v[kx] = 0.f;
      } else if (c == 3) {
#pragma unroll
        for (int kx = 0; kx < P; ++kx) v[kx] = (float)((mb >> kx) & 1u);
      } else if (a.rgb_f32) {
        const float* src = &sm.rgb[c][y - y0][xl - x0];
#pragma unroll
        for (int kx = 0; kx < P; ++kx) v[kx] = ((mb >> kx) & 1u) ? 0.f : src[kx];
      } else {
        const uint8_t* src = reinterpret_cast<const uint8_t*>(&sm.rgb[0][0][0]) +
                             ((y - y0) * TW + (xl - x0)) * 3 + c;
#pragma unroll
        for (int kx = 0; kx < P; ++kx) {
          const uint8_t u = src[3 * kx];
          dirty |= ((m0b >> kx) & 1u) && u != 0;
          v[kx] = ((mb >> kx) & 1u) ? 0.f : __fdiv_rn((float)u, 255.0f);
        }
      }
      if (__any_sync(0xffffffffu, dirty) && lane == 0) sm.dirty = 1;
      if (!active) continue;
      __half* dst = a.xin + ((size_t)f * T + tok) * (4 * P * P) + c * P * P + ky * P;
      uint32_t packed[P / 2];
#pragma unroll
      for (int kx = 0; kx < P; kx += 2) packed[kx / 2] = pack_half2(v[kx], v[kx + 1]);
      if constexpr (P == 8) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      } else {
        *reinterpret_cast<uint2*>(dst) = make_uint2(packed[0], packed[1]);
      }
    }
  }
  MT(8);
  __syncthreads();
  if (tid == 0 && a.flags) {
    if (a.flag_cnt == nullptr) {
      if (sm.dirty) atomicOr(a.flags + f, 2);
    } else {
      if (sm.dirty) atomicOr(a.flag_acc + f, 2);
      __threadfence();
      const unsigned done = atomicAdd(a.flag_cnt + f, 1u);
      if (done == gridDim.x * gridDim.y - 1) {            // the frame's last CTA
        __threadfence();
        a.flags[f] = atomicExch(a.flag_acc + f, 0);
        a.flag_cnt[f] = 0;
      }
    }
  }
  MT(9);
}

}  // namespace

template <int P, int WH, int TH>
void launch_mask_t(const MaskArgs& a, cudaStream_t s) {
  static unsigned long long init = 0;
  constexpr int smem = (int)sizeof(Smem<TH>) + 16;
  once_per_device(init, [&] {
    cudaFuncSetAttribute(mask_fused_kernel<P, WH, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  dim3 grid((a.W + TW - 1) / TW, (a.H + TH - 1) / TH, a.frames);
  launch_pdl(mask_fused_kernel<P, WH, TH>, grid, dim3(32 * TH), smem, s, a);
}

template <int TH>
void launch_mask_th(const MaskArgs& a, cudaStream_t s) {
  const int wh = (a.radius + a.feather_radius + 31) / 32;   // 0..2 halo words per side
  if (a.patch == 4) {
    if (wh <= 1) launch_mask_t<4, 1, TH>(a, s);
    else launch_mask_t<4, 2, TH>(a, s);
  } else {
    if (wh <= 1) launch_mask_t<8, 1, TH>(a, s);
    else launch_mask_t<8, 2, TH>(a, s);
  }
}

// Network input pack on its own (host path with split uploads: the mask stage runs on the
// mask while the rgb is still crossing PCIe; this kernel then builds the same xin as the
// fused stage from rgb u8 + the stage's m1 bytes, and the redaction check from m0).  One
// warp per token, lanes = 4 channels x P rows, exactly the fused stage's per-lane math.
template <int P>
__global__ void __launch_bounds__(256) pack_input_kernel(MaskArgs a) {
  const int lane = threadIdx.x & 31;
  const int Cc = a.W / P, T = (a.H / P) * Cc;
  const long gtok = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
  pdl_trigger();
  pdl_wait();
  if (gtok >= (long)a.frames * T) return;
  const int f = (int)(gtok / T), tok = (int)(gtok - (long)f * T);
  const int i = tok / Cc, j = tok - i * Cc;
  const bool active = lane < 4 * P;
  const int c = lane / P, ky = lane % P;
  const size_t plane = (size_t)a.H * a.W;
  const int y = i * P + ky, xl = j * P;
  uint32_t mb = 0, m0b = 0;
  if (active) {
    const uint8_t* m1r = a.m1 + (size_t)f * plane + (size_t)y * a.W + xl;
    const uint8_t* m0r = a.m0 + (size_t)f * plane + (size_t)y * a.W + xl;
#pragma unroll
    for (int kx = 0; kx < P; ++kx) {
      mb |= (uint32_t)(m1r[kx] != 0) << kx;
      m0b |= (uint32_t)(m0r[kx] != 0) << kx;
    }
  }
  float v[P];
  bool dirty = false;
  if (!active) {
#pragma unroll
    for (int kx = 0; kx < P; ++kx) v[kx] = 0.f;
  } else if (c == 3) {
#pragma unroll
    for (int kx = 0; kx < P; ++kx) v[kx] = (float)((mb >> kx) & 1u);
  } else {
    const uint8_t* src = a.rgb_u8 + ((size_t)f * plane + (size_t)y * a.W + xl) * 3 + c;
#pragma unroll
    for (int kx = 0; kx < P; ++kx) {
      const uint8_t u = src[3 * kx];
      dirty |= ((m0b >> kx) & 1u) && u != 0;
      v[kx] = ((mb >> kx) & 1u) ? 0.f : __fdiv_rn((float)u, 255.0f);
    }
  }
  if (__any_sync(0xffffffffu, dirty) && lane == 0 && a.flags) atomicOr(a.flags + f, 2);
  if (!active) return;
  __half* dst = a.xin + ((size_t)f * T + tok) * (4 * P * P) + c * P * P + ky * P;
  uint32_t packed[P / 2];
#pragma unroll
  for (int kx = 0; kx < P; kx += 2) packed[kx / 2] = pack_half2(v[kx], v[kx + 1]);
  if constexpr (P == 8) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  } else {
    *reinterpret_cast<uint2*>(dst) = make_uint2(packed[0], packed[1]);
  }
}

void launch_pack_input(const MaskArgs& a, cudaStream_t s) {
  const long tokens = (long)a.frames * (a.H / a.patch) * (a.W / a.patch);
  const dim3 grid((unsigned)((tokens + 7) / 8));
  if (a.patch == 4) launch_pdl(pack_input_kernel<4>, grid, dim3(256), 0, s, a);
  else launch_pdl(pack_input_kernel<8>, grid, dim3(256), 0, s, a);
}

// Tile height by grid size: below one wave of 16-row tiles (4 resident per SM) the stage is
// latency-bound and 8-row tiles halve each CTA's path (C2 p50 -2 us); above it the halo
// overhead of short tiles costs throughput (C5 +1.5 % with 16 rows).  DR_MASK_TH=8|16
// forces one (tests).
void launch_mask_stage(const MaskArgs& a, cudaStream_t s) {
  const char* fe = std::getenv("DR_MASK_TH");
  const int forced = fe ? std::atoi(fe) : 0;
  const long tiles16 = (long)((a.W + TW - 1) / TW) * ((a.H + 15) / 16) * a.frames;
  const bool short_tiles = forced ? forced == 8 : tiles16 < 4L * device_sms();
  if (short_tiles) launch_mask_th<8>(a, s);
  else launch_mask_th<16>(a, s);
}

}  // namespace dr

#ifdef DR_TRACE
#include <vector>
extern "C" int dr_debug_mask_trace(unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  const int k = n < 4096 * dr::MT_SLOTS ? n : 4096 * dr::MT_SLOTS;
  cudaMemcpyFromSymbol(host, dr::g_mask_trace, (size_t)k * sizeof(unsigned long long));
  return k;
}
#endif
