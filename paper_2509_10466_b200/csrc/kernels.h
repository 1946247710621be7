// Internal kernel interfaces of libdrb200 (not part of the C-ABI).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dr {

constexpr int C = 64;        // channels (token width)
constexpr int HEADS = 4;
constexpr int DH = 16;       // head dim
constexpr int FF = 128;      // FFN hidden

// Fragment-packed fp16 weights of one transformer block (see pack.cpp).
struct BlockW {
  const float* ln1_w; const float* ln1_b;
  const uint2* wqkv; const float* bqkv;   // N=192 (q|k|v), K=64 : [24][4][32]
  const uint2* wo;   const float* bo;     // N=64,  K=64  : [8][4][32]
  const float* ln2_w; const float* ln2_b;
  const uint2* w1;   const float* b1;     // N=128, K=64  : [16][4][32]
  const uint2* w2;   const float* b2;     // N=64,  K=128 : [8][8][32]
};

struct TokenArgs {
  int n_tok;              // tokens in this launch (frames * T)
  int T;                  // tokens per frame
  // mode EMBED
  const __half* xin;      // [n_tok][kin] fp16 patch-major network input
  const uint2* we; const float* be; int kin;
  // mode POST (out-proj + residual + LN2 + FFN + residual)
  const __half* attn;     // [n_tok][64] fp16 attention output (heads concatenated)
  const float* resid_in;  // [n_tok][64] fp32 residual stream (also SLOTKV input)
  BlockW cur;
  // outputs
  float* resid_out;       // [n_tok][64] fp32 (may alias resid_in)
  int has_next;
  BlockW next;            // LN1 + QKV of the following block
  __half* q; __half* k; __half* v;   // [frames][HEADS][T][DH]
  __half* tok16;          // [n_tok][64] fp16 copy when there is no next block
};

enum TokenMode { TOK_EMBED = 0, TOK_POST = 1, TOK_SLOTKV = 2 };

void launch_token(int mode, const TokenArgs& a, cudaStream_t s);

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
};
void launch_attention(const AttnArgs& a, cudaStream_t s);

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
};
void launch_mask_stage(const MaskArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- decoder
struct DecodeArgs {
  int frames, H, W, R, Cc;   // image and token grid
  const __half* tok16;       // [frames][T][64]
  const uint2* wv2p; const float* bv2p;   // [100][8][4][32] frags
  const uint2* wd0; const float* bd0;     // [9][8][4][32]
  const uint2* wd2; const float* bd2;     // [9][1][4][32] (N padded 3->8)
  __half* raster;            // [frames][H][W][64]
  __half* d0;                // [frames][H][W][64]
  // tail
  const float* alpha;        // [frames][H][W]
  const float* rgb_f32;      // [frames][3][H][W] (float API) or null
  const uint8_t* rgb_u8;     // [frames][H][W][3] (u8 API) or null
  float* fill;               // [frames][3][H][W] raw network output (optional)
  float* out_f32;            // [frames][3][H][W] composite (float API)
  uint8_t* out_u8;           // [frames][H][W][3] composite (u8 API)
  int* flags;                // bit0 = non-finite network output
};
void launch_vec2patch(const DecodeArgs& a, cudaStream_t s);
void launch_decode0(const DecodeArgs& a, cudaStream_t s);
void launch_decode2(const DecodeArgs& a, cudaStream_t s);

}  // namespace dr
