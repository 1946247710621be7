// Token-wise fused GEMM chains of the DSTT blocks (reference dstt.py:102-150, :185-195).
//
// One warp owns 16 tokens and keeps them in registers for the whole chain; every GEMM is
// m16n8k16 HMMA with fp16 operands and fp32 accumulators; LayerNorm statistics, GELU,
// biases and the residual stream stay fp32.  The chains:
//   TOK_EMBED : x = patch_embed(xin)                                  (dstt.py:246-254)
//   TOK_POST  : x = r + attn*Wo^T + bo ; x += W2 gelu(W1 LN2(x) + b1) + b2   (:146-149)
//   then, if a next block exists: y = LN1'(x); [q|k|v] = y*Wqkv'^T + b  (:141-142, :106-117)
//   TOK_SLOTKV: k,v = LN1(slot)*Wk,v^T + b for a memory slot          (:188-190)
// Activations move through HBM only as the fp32 residual stream, fp16 q/k/v and the fp16
// attention output: 256 + 384 + 128 B per token per block.
#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

constexpr int WARPS = 2;   // 32 tokens per CTA: 128 CTAs at one 512^2 frame

struct Frag16x64 {         // 16 tokens x 64 channels, C-fragment layout (fp32)
  float v[8][4];
};

DR_DEV void load_rows_f32(Frag16x64& x, const float* __restrict__ src, int n0, int n_tok,
                          int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool v0 = n0 + g < n_tok, v1 = n0 + g + 8 < n_tok;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    float2 a = v0 ? __ldg(reinterpret_cast<const float2*>(src + (size_t)(n0 + g) * C + nt * 8 + 2 * t))
                  : make_float2(0.f, 0.f);
    float2 b = v1 ? __ldg(reinterpret_cast<const float2*>(src + (size_t)(n0 + g + 8) * C + nt * 8 + 2 * t))
                  : make_float2(0.f, 0.f);
    x.v[nt][0] = a.x; x.v[nt][1] = a.y; x.v[nt][2] = b.x; x.v[nt][3] = b.y;
  }
}

DR_DEV void store_rows_f32(const Frag16x64& x, float* dst, int n0, int n_tok, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool v0 = n0 + g < n_tok, v1 = n0 + g + 8 < n_tok;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    if (v0) *reinterpret_cast<float2*>(dst + (size_t)(n0 + g) * C + nt * 8 + 2 * t) =
        make_float2(x.v[nt][0], x.v[nt][1]);
    if (v1) *reinterpret_cast<float2*>(dst + (size_t)(n0 + g + 8) * C + nt * 8 + 2 * t) =
        make_float2(x.v[nt][2], x.v[nt][3]);
  }
}

// fp16 tokens onto the zero-padded (R+2) x (Cc+2) grid of Vec2Patch.
DR_DEV size_t padded_pos(int n, int T, int R, int Cc) {
  const int f = n / T, t = n - f * T;
  const int i = t / Cc, j = t - i * Cc;
  return ((size_t)f * (R + 2) + i + 1) * (Cc + 2) + j + 1;
}

DR_DEV void store_rows_padded_f16(const Frag16x64& x, __half* dst, int n0, int n_tok, int T,
                                  int R, int Cc, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool v0 = n0 + g < n_tok, v1 = n0 + g + 8 < n_tok;
  __half* r0 = dst + (v0 ? padded_pos(n0 + g, T, R, Cc) : 0) * C;
  __half* r1 = dst + (v1 ? padded_pos(n0 + g + 8, T, R, Cc) : 0) * C;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    if (v0) *reinterpret_cast<uint32_t*>(r0 + nt * 8 + 2 * t) = pack_half2(x.v[nt][0], x.v[nt][1]);
    if (v1) *reinterpret_cast<uint32_t*>(r1 + nt * 8 + 2 * t) = pack_half2(x.v[nt][2], x.v[nt][3]);
  }
}

// A fragments (4 k-tiles of 16) of a 16 x 64 fp16 row-major tile in global memory.
DR_DEV void load_a_f16(uint32_t a[4][4], const __half* __restrict__ src, int ld, int n0,
                       int n_tok, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool v0 = n0 + g < n_tok, v1 = n0 + g + 8 < n_tok;
  const uint32_t* r0 = reinterpret_cast<const uint32_t*>(src + (size_t)(n0 + g) * ld);
  const uint32_t* r1 = reinterpret_cast<const uint32_t*>(src + (size_t)(n0 + g + 8) * ld);
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) {
    a[kt][0] = v0 ? __ldg(r0 + kt * 8 + t) : 0u;
    a[kt][1] = v1 ? __ldg(r1 + kt * 8 + t) : 0u;
    a[kt][2] = v0 ? __ldg(r0 + kt * 8 + 4 + t) : 0u;
    a[kt][3] = v1 ? __ldg(r1 + kt * 8 + 4 + t) : 0u;
  }
}

// LayerNorm over the 64 channels of each row (eps 1e-5, biased variance), emitted
// directly as fp16 A fragments for the next GEMM.
DR_DEV void layer_norm_to_a(const Frag16x64& x, const float* __restrict__ w,
                            const float* __restrict__ b, uint32_t a[4][4], int lane) {
  const int t = lane & 3;
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) { s0 += x.v[nt][0] + x.v[nt][1]; s1 += x.v[nt][2] + x.v[nt][3]; }
  const float mu0 = quad_sum(s0) * (1.f / 64.f), mu1 = quad_sum(s1) * (1.f / 64.f);
  float q0 = 0.f, q1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    float d;
    d = x.v[nt][0] - mu0; q0 += d * d;
    d = x.v[nt][1] - mu0; q0 += d * d;
    d = x.v[nt][2] - mu1; q1 += d * d;
    d = x.v[nt][3] - mu1; q1 += d * d;
  }
  const float r0 = rsqrtf(quad_sum(q0) * (1.f / 64.f) + 1e-5f);
  const float r1 = rsqrtf(quad_sum(q1) * (1.f / 64.f) + 1e-5f);
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int nt = 2 * kt + h;
      const int col = nt * 8 + 2 * t;
      const float w0 = __ldg(w + col), w1 = __ldg(w + col + 1);
      const float b0 = __ldg(b + col), b1 = __ldg(b + col + 1);
      a[kt][2 * h + 0] = pack_half2((x.v[nt][0] - mu0) * r0 * w0 + b0, (x.v[nt][1] - mu0) * r0 * w1 + b1);
      a[kt][2 * h + 1] = pack_half2((x.v[nt][2] - mu1) * r1 * w0 + b0, (x.v[nt][3] - mu1) * r1 * w1 + b1);
    }
  }
}

// acc[nt] (+)= A(16 x 16*KT) * W^T for n-tiles [nt0, nt0+NT) of a packed weight with KT
// k-tiles.
template <int NT, int KT>
DR_DEV void gemm_acc(float (*acc)[4], const uint32_t (*a)[4], const uint2* __restrict__ w,
                     int nt0, int lane) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const uint2 b = ld_frag(w, (nt0 + nt) * KT + kt, lane);
      mma16816(acc[nt], a[kt], b.x, b.y);
    }
  }
}

DR_DEV void init_bias(float (*acc)[4], int nt_count, const float* __restrict__ bias,
                      int col0, int lane) {
  const int t = lane & 3;
  for (int nt = 0; nt < nt_count; ++nt) {
    const float b0 = __ldg(bias + col0 + nt * 8 + 2 * t), b1 = __ldg(bias + col0 + nt * 8 + 2 * t + 1);
    acc[nt][0] = b0; acc[nt][1] = b1; acc[nt][2] = b0; acc[nt][3] = b1;
  }
}

// LN1 + q/k/v projection of one block, written head-major [frame][head][T][16].
DR_DEV void qkv_out(const Frag16x64& x, const BlockW& w, __half* q, __half* k, __half* v,
                    int n0, int n_tok, int T, int first_pair, int lane) {
  uint32_t a[4][4];
  layer_norm_to_a(x, w.ln1_w, w.ln1_b, a, lane);
  const int g = lane >> 2, t = lane & 3;
  const int na = n0 + g, nb = n0 + g + 8;
  const int fa = na / T, ta = na - fa * T, fb = nb / T, tb = nb - fb * T;
#pragma unroll 1
  for (int p = first_pair; p < 12; ++p) {   // 12 head-sized (16-col) output groups
    float acc[2][4];
    init_bias(acc, 2, w.bqkv, p * 16, lane);
    gemm_acc<2, 4>(acc, a, w.wqkv, 2 * p, lane);
    const int which = p >> 2, h = p & 3;
    __half* dst = which == 0 ? q : (which == 1 ? k : v);
    if (na < n_tok) {
      uint32_t* r = reinterpret_cast<uint32_t*>(dst + ((size_t)(fa * HEADS + h) * T + ta) * DH);
      r[t] = pack_half2(acc[0][0], acc[0][1]);
      r[4 + t] = pack_half2(acc[1][0], acc[1][1]);
    }
    if (nb < n_tok) {
      uint32_t* r = reinterpret_cast<uint32_t*>(dst + ((size_t)(fb * HEADS + h) * T + tb) * DH);
      r[t] = pack_half2(acc[0][2], acc[0][3]);
      r[4 + t] = pack_half2(acc[1][2], acc[1][3]);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32) token_kernel(TokenArgs a) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n0 = (blockIdx.x * WARPS + warp) * 16;
  if (n0 >= a.n_tok) return;
  Frag16x64 x;

  if constexpr (MODE == TOK_SLOTKV) {
    load_rows_f32(x, a.resid_in, n0, a.n_tok, lane);
    qkv_out(x, a.next, a.q, a.k, a.v, n0, a.n_tok, a.T, 4, lane);
    return;
  } else if constexpr (MODE == TOK_EMBED) {
    init_bias(x.v, 8, a.be, 0, lane);
    const int g = lane >> 2, t = lane & 3;
    const bool v0 = n0 + g < a.n_tok, v1 = n0 + g + 8 < a.n_tok;
    const uint32_t* r0 = reinterpret_cast<const uint32_t*>(a.xin + (size_t)(n0 + g) * a.kin);
    const uint32_t* r1 = reinterpret_cast<const uint32_t*>(a.xin + (size_t)(n0 + g + 8) * a.kin);
    const int KT = a.kin / 16;
#pragma unroll 2
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t af[4];
      af[0] = v0 ? __ldg(r0 + kt * 8 + t) : 0u;
      af[1] = v1 ? __ldg(r1 + kt * 8 + t) : 0u;
      af[2] = v0 ? __ldg(r0 + kt * 8 + 4 + t) : 0u;
      af[3] = v1 ? __ldg(r1 + kt * 8 + 4 + t) : 0u;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const uint2 b = ld_frag(a.we, nt * KT + kt, lane);
        mma16816(x.v[nt], af, b.x, b.y);
      }
    }
  } else {  // TOK_POST
    load_rows_f32(x, a.resid_in, n0, a.n_tok, lane);
    {
      uint32_t ao[4][4];
      load_a_f16(ao, a.attn, C, n0, a.n_tok, lane);
      float acc[8][4];
      init_bias(acc, 8, a.cur.bo, 0, lane);
      gemm_acc<8, 4>(acc, ao, a.cur.wo, 0, lane);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) x.v[nt][i] += acc[nt][i];
    }
    uint32_t ya[4][4];
    layer_norm_to_a(x, a.cur.ln2_w, a.cur.ln2_b, ya, lane);
    float out2[8][4];
    init_bias(out2, 8, a.cur.b2, 0, lane);
#pragma unroll
    for (int half = 0; half < 2; ++half) {     // hidden 128 = 2 x 64
      float hacc[8][4];
      init_bias(hacc, 8, a.cur.b1, half * 64, lane);
      gemm_acc<8, 4>(hacc, ya, a.cur.w1, half * 8, lane);
      uint32_t ha[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ha[j][0] = pack_half2(gelu_erf(hacc[2 * j][0]), gelu_erf(hacc[2 * j][1]));
        ha[j][1] = pack_half2(gelu_erf(hacc[2 * j][2]), gelu_erf(hacc[2 * j][3]));
        ha[j][2] = pack_half2(gelu_erf(hacc[2 * j + 1][0]), gelu_erf(hacc[2 * j + 1][1]));
        ha[j][3] = pack_half2(gelu_erf(hacc[2 * j + 1][2]), gelu_erf(hacc[2 * j + 1][3]));
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint2 b = ld_frag(a.cur.w2, nt * 8 + half * 4 + j, lane);
          mma16816(out2[nt], ha[j], b.x, b.y);
        }
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) x.v[nt][i] += out2[nt][i];
  }

  store_rows_f32(x, a.resid_out, n0, a.n_tok, lane);
  if (a.has_next) {
    qkv_out(x, a.next, a.q, a.k, a.v, n0, a.n_tok, a.T, 0, lane);
  } else if (a.tok16) {
    store_rows_padded_f16(x, a.tok16, n0, a.n_tok, a.T, a.R, a.Cc, lane);
  }
}

}  // namespace

void launch_token(int mode, const TokenArgs& a, cudaStream_t s) {
  const int tiles = (a.n_tok + 15) / 16;
  dim3 grid((tiles + WARPS - 1) / WARPS), block(WARPS * 32);
  switch (mode) {
    case TOK_EMBED: token_kernel<TOK_EMBED><<<grid, block, 0, s>>>(a); break;
    case TOK_POST: token_kernel<TOK_POST><<<grid, block, 0, s>>>(a); break;
    default: token_kernel<TOK_SLOTKV><<<grid, block, 0, s>>>(a); break;
  }
}

}  // namespace dr
