// Internal kernel interfaces of libdrb200 (not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dr {

constexpr int C = 64;        // channels (token width)
constexpr int HEADS = 4;
constexpr int DH = 16;       // head dim
constexpr int FF = 128;      // FFN hidden

// Weights of one transformer block for the tcgen05 token chains (token_tc.cu): one image,
// K-major 128B-swizzled fp16 [Wqkv 192][Wo 64][W1 128][W2 2 K-atoms x 64] rows of 128 B,
// then the block's fp32 LayerNorm affine and biases (token_tc_block_image_bytes()).
struct BlockW {
  const uint8_t* img;
};

struct TokenArgs {
  int n_tok;              // tokens in this launch (frames * T)
  int tile_rows;          // tcgen05 path: tokens per CTA (32/64/128; 0 = pick by n_tok)
  int T;                  // tokens per frame
  // mode EMBED
  const __half* xin;      // [n_tok][kin] fp16 patch-major network input
  int kin;
  const uint8_t* we_img;  // tcgen05 image of We (4 K-atoms x 64 rows x 128 B), then be
  // mode POST (out-proj + residual + LN2 + FFN + residual)
  const __half* attn;     // [n_tok][64] fp16 attention output (heads concatenated)
  const float* resid_in;  // [n_tok][64] fp32 residual stream (also SLOTKV input)
  BlockW cur;
  // outputs
  float* resid_out;       // [n_tok][64] fp32 (may alias resid_in)
  int has_next;
  BlockW next;            // LN1 + QKV of the following block
  __half* q; __half* k; __half* v;   // [frames][HEADS][T][DH]
  __half* tok16;          // fp16 copy when there is no next block, on the zero-padded
                          // [frames][(R+2)(Cc+2)][64] grid that Vec2Patch reads
  int R, Cc;              // token grid
  // last block only: K/V of the new memory slot for every temporal block (slot K/V cache)
  int n_kv;
  // SLOTKV only: skip the entry pdl_wait (the slot input is not produced by the previous
  // kernel) and wait at exit, so the projection overlaps the predecessor (the mask stage)
  int late_wait;
  BlockW kv_w[4];
  __half* kv_k[4];
  __half* kv_v[4];
};
constexpr int MAX_TEMPORAL = 4;

enum TokenMode { TOK_EMBED = 0, TOK_POST = 1, TOK_SLOTKV = 2 };

// tcgen05 + TMEM.  128-token tiles take their inputs by TMA when the maps are given
// (2-D, 128B-swizzled, box 128 rows: m_in = xin [n][256] fp16 (EMBED) / attn [n][64] fp16
// (POST), box 64 halves; m_res = residual [n][64] fp32, box 32 floats), else by cp.async.
void launch_token_tc(int mode, const TokenArgs& a, cudaStream_t s,
                     const CUtensorMap* m_in = nullptr, const CUtensorMap* m_res = nullptr);
size_t token_tc_block_image_bytes();   // per block: weights + 704 fp32 params
size_t token_tc_embed_image_bytes();   // We + be
int token_tc_tile_rows(int n_tok, int sms);   // tokens per CTA the token kernels use

// ---------------------------------------------------------------- attention
struct AttnArgs {
  // queries: [frames][HEADS][T][DH]; q-range of this launch is a band per group
  const __half* q;
  // key segments (up to 3): cur frame K/V, slot0 K/V, slot1 K/V, each [fr][HEADS][T][DH]
  const __half* k[3]; const __half* v[3];
  int seg_frame_stride[3];   // 1 if per-frame, 0 if the segment is shared (broadcast slot)
  int n_seg;
  int T;                     // tokens per frame
  int groups;                // row bands (1 for spatial)
  int band;                  // tokens per band (T / groups)
  int frames;
  __half* out;               // [frames][T][64]
  // mask-aware (null = off): key validity of the current frame's tokens [frames][T]
  const uint8_t* key_valid;
  int mask_mode;             // 0 off, 1 spatial (fallback if none valid), 2 temporal raw,
                             // 3 temporal collapsed (mask iff frame has no valid token)
  // key split: CTAs (one cluster) per query tile, 1..4; 0 = chosen by attention_ksplit
  int ksplit;
  // all-zero memory slots (temporal blocks): LN1(0) = beta, so every key of such a slot is
  // the same k0 = Wk beta + bk with value v0 = Wv beta + bv.  Their `const_mult` (band per
  // zero slot) identical keys enter the softmax as one key of that multiplicity:
  // const_kv = [k0 (64) | v0 (64)] fp32 (fp16-rounded values), 0 = none.
  const float* const_kv;
  int const_mult;
};
void launch_attention(const AttnArgs& a, cudaStream_t s);
int attention_ksplit(const AttnArgs& a);

// ---------------------------------------------------------------- mask stage
struct MaskArgs {
  int frames, H, W, patch;
  int radius;                // dilation radius (3x3-cross iterations)
  int feather_radius;        // 0 = binary alpha
  const double* feather_w;   // [2*feather_radius+1] device
  const uint8_t* m0;         // [frames][H][W] nonzero = private
  const float* rgb_f32;      // [frames][3][H][W] or null
  const uint8_t* rgb_u8;     // [frames][H][W][3] or null
  uint32_t* bits0;           // [frames][H][Wwords] scratch
  uint32_t* bits1;           // [frames][H][Wwords] scratch (m1)
  uint8_t* m1;               // [frames][H][W] out (optional)
  float* alpha;              // [frames][H][W] out
  float* gtmp;               // [frames][H][W] scratch (vertical pass)
  uint8_t* token_valid;      // [frames][T] out
  __half* xin;               // [frames][T][4*p*p] out (optional)
  int* flags;                // [frames] out: bit1 = input not redacted inside m0
  // with flag_acc / flag_cnt (engine-owned, [frames] each, zero between stages) the stage
  // WRITES flags[f] (no memset before the forward): CTAs OR their redaction bit into
  // flag_acc[f] and count themselves in flag_cnt[f]; the frame's last CTA moves flag_acc[f]
  // into flags[f] and resets both words.  Without them it ORs into a zeroed flags word.
  int* flag_acc;
  unsigned* flag_cnt;
};
void launch_mask_stage(const MaskArgs& a, cudaStream_t s);
// xin + redaction check alone, from u8 rgb, m0 and the stage's m1 bytes
void launch_pack_input(const MaskArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- decoder
// tcgen05 3x3 convolution (conv_tc.cu).  Input = TMA tensor map over an NHWC fp16
// raster [frames][H][W][64] (box 64 ch x 130 px x 4 rows, 128B swizzle).  Weights: fp16
// image [tap 9][k-chunk 8][co N][8 ci], N = 64 (decode.0) or 16 (decode.2, 3 real).
struct ConvTcArgs {
  int frames, H, W;
  const void* w;             // weight image, conv_tc_weight_bytes(N)
  const float* bias;         // [N real]
  __half* out16;             // decode.0: [frames][H][W][64]
  // decode.2 tail: alpha [frames][H][W]; rgb/out f32 [frames][3][H][W] (float API) or
  // u8 [frames][H][W][3] (u8 API); fill = raw network output; flags bit0 = non-finite
  const float* alpha;
  const float* rgb_f32;
  const uint8_t* rgb_u8;
  float* fill;
  float* out_f32;
  uint8_t* out_u8;
  int* flags;
  // fused decode.0 -> decode.2 (tap-expanded): decode.0's epilogue multiplies its fp16
  // LeakyReLU output by w2 (K-major 128B-swizzled [32 u][64 ci], u = 3*(3*ky+kx)+co) on
  // the tensor cores and stores E as fp16 planes [frames][27][H][W] instead of the 64-ch
  // raster; launch_dec2_gather then sums the 3x3 neighbourhood and runs the tail
  __half* e_planes;
  const void* w2;
  // decode.2 gather (optional): the last CTA to finish copies flags[0..frames) here;
  // `done` is a zeroed counter the last CTA re-arms
  int* flags_mirror;
  unsigned* done;
  // host path: with spans set, the mirror lives after the packed bytes, at
  // align4(spans[H-1].z + 3 * (spans[H-1].y - spans[H-1].x)) (fixed kernel arguments, so
  // the host path's launch sequence can be replayed from a CUDA graph)
  int mirror_after_spans;
  // decode.2 gather (optional, one frame): also write the u8 composite of the pixels in
  // row y's span [spans[y].x, spans[y].y) to packed + spans[y].z + 3 * (x - x0)
  const int4* spans;
  uint8_t* packed;
};
}  // namespace dr
#include <cuda.h>
namespace dr {
size_t conv_tc_weight_bytes(int n);
int conv_tc_rows(int n);   // output rows per tile; the input TMA box is rows + 2 tall

// tcgen05 Vec2Patch (v2p_tc.cu).  Tokens: fp16 [frames][(R+2)(Cc+2)][64], zero-padded grid
// (token (i,j) at padded (i+1, j+1)), TMA box 64 ch x 128 positions, 128B swizzle.
// Weights: [tap a*10+b][k-chunk 8][co 64][8 ci] fp16.
struct V2pArgs {
  int frames, H, W, R, Cc;
  const void* w;
  const float* bias;
  __half* raster;            // [frames][H][W][64]
};
size_t v2p_tc_weight_bytes();
void launch_v2p_tc(const CUtensorMap& tok, const V2pArgs& a, cudaStream_t s);
void launch_conv3x3_tc(int n, const CUtensorMap& tin, const ConvTcArgs& a, cudaStream_t s);
// decode.2 gather + tail over the E planes the fused decode.0 wrote (conv_tc.cu)
void launch_dec2_gather(const ConvTcArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- fused decoder
// (dec_fused.cu) Vec2Patch o decode.0 as one stride-8 transposed convolution with a 12x12
// kernel, LeakyReLU, decode.2's tap-expanded GEMM and the 3x3 gather in shared memory,
// tanh and the composite -- per tile of 16 x 8 tokens (128 x 64 px), no 64-channel raster.
// The combined form is exact off the image border; border pixels (decode.0 reads zero
// padding there, the combined form the cropped canvas ring) are redone by dec_border from
// the tile pass's pre-activations, and every pixel next to another tile (or within one
// pixel of the image border) is finished by dec_fixup from per-tile partial sums; with
// `groups` > 1 the 64 phases of a tile are split over a cluster of that many CTAs, whose
// accumulators are summed through distributed shared memory.
constexpr int DEC_MAX_FIX = 128;
// Phase quads of the fused decoder: quad g = (gy, gx) of a 4 x 4 grid holds the phases
// py in {2gy, 2gy+1}, px in {2gx, 2gx+1}, which read the same token offsets: du in {0},
// plus -1 (tap u = py + 8) for gy = 0 and +1 (u = py - 8) for gy = 3; likewise dv.  One
// MMA with N = 256 (4 phases x 64 channels) per offset and K step.
__host__ __device__ inline int dec_quad_noff(int gq) { return (gq == 0 || gq == 3) ? 2 : 1; }
__host__ __device__ inline int dec_quad_off(int gq, int i) { return i == 0 ? 0 : (gq == 0 ? -1 : 1); }
__host__ __device__ inline int dec_quad_first(int g) {     // offset blocks before quad g
  int n = 0;
  for (int k = 0; k < g; ++k) n += dec_quad_noff(k >> 2) * dec_quad_noff(k & 3);
  return n;
}
struct DecArgs {
  int frames, H, W, R, Cc;
  int groups;                // parts per tile (cluster size): 1, 2 or 4; each takes 16 / groups quads
  int border_split;          // dec_border CTAs per (frame, edge, phase) (set by its launcher)
  // 36 offset blocks in quad order, offsets du-major: [k-chunk 8][4 phases x 64 co][8 ci]
  // fp16 (phase p = 2 (py & 1) + (px & 1) of the quad)
  const void* wcomb;
  const float* bcomb;        // [64] combined bias
  const void* w2;            // decode.2 tap-expanded weights, K-major SW128 [32 u][64 ci]
  const float* w2f;          // decode.2 weights fp32 [27 u][64 ci] (u = 3*(3*ky+kx)+co)
  const float* b2;           // [3]
  const float* dk;           // border-correction tables (engine.cu, dec_border_table_floats)
  const __half* tok16;       // padded token grid [frames][R+2][Cc+2][64]
  float* part;               // seam partial sums [frames][tile][3][band] (dec_part_floats)
  float* bd0;                // border pixels' combined pre-activation [frames][NB][64]
  float* be;                 // border pixels' decode.2 taps E [frames][NB][27]
  // rows / columns dec_fixup finishes (seams and the 2-pixel image border band), sorted
  int n_fix_rows, n_fix_cols;
  short fix_rows[DEC_MAX_FIX], fix_cols[DEC_MAX_FIX];
  ConvTcArgs tail;           // composite / output / flags fields (alpha .. packed)
};
size_t dec_border_table_floats();
size_t dec_part_floats(int frames, int H, int W);
int dec_groups(int frames, int H, int W, int sms);
int dec_border_pixels(int H, int W);                 // 2W + 2(H-2)
void dec_fix_lines(DecArgs& a);                      // fills n_fix_rows/cols, fix_rows/cols
void launch_dec_fused(const CUtensorMap& tok4d, const DecArgs& a, cudaStream_t s);
void launch_dec_border(const DecArgs& a, cudaStream_t s);
void launch_dec_fixup(const DecArgs& a, cudaStream_t s);   // fix pixels + flags mirror

// ---------------------------------------------------------------- frame byte kernels
// (frame_ops.cu): display composite / upscale2x, merge + redact, point-cloud pack.
struct DisplayArgs {
  int height, width, channels;     // source raster; channels 1 or 3 (HWC u8)
  const uint8_t* original;         // captured frame
  const uint8_t* inpainted;        // engine output (or null: plain upscale)
  const uint8_t* mask;             // [H][W] privacy mask (or null)
  int engine_failed;               // 1: zero inside the upscaled mask
  uint8_t* out;                    // [2H][2W][channels]
};
void launch_display(const DisplayArgs& a, cudaStream_t s);

struct MergeRedactArgs {
  int n_masks, height, width;
  const uint8_t* masks;            // [n][H][W]
  const uint8_t* private_flags;    // [n] device
  const uint8_t* rgb_in;           // [H][W][3] or null
  uint8_t* merged;                 // [H][W] or null
  uint8_t* rgb_out;                // [H][W][3] or null
};
void launch_merge_redact(const MergeRedactArgs& a, cudaStream_t s);

struct PointCloudArgs {
  int height, width;
  const float* depth;              // [H][W]
  const uint8_t* rgb;              // [H][W][3]
  double inv_fx, inv_fy, cx, cy;
  int* row_counts;                 // [H] scratch
  float* xyz;                      // [<= H*W][3]
  uint8_t* colors;                 // [<= H*W][3]
  int* count;                      // [1]
};
void launch_pointcloud(const PointCloudArgs& a, cudaStream_t s);

}  // namespace dr
