// Token-wise fused GEMM chains of the DSTT blocks (reference dstt.py:102-150, :185-195).
//
// A CTA of 4 warps owns 16 tokens; the N dimension of every GEMM is split across the
// warps (warp w owns output columns [16w,16w+16) of the 64-wide GEMMs, [32w,32w+32) of
// FFN1, 3 of the 12 head-sized q|k|v groups), so a 512^2 frame (4096 tokens) keeps ~7
// warps per SM busy instead of ~2.  LayerNorm row statistics and the fp16 A operands
// (LN output, GELU output) are exchanged through shared memory.  All GEMMs are m16n8k16
// HMMA with fp16 operands and fp32 accumulators; LN, GELU (exact erf), biases and the
// residual stream stay fp32.  Chains:
//   TOK_EMBED : x = patch_embed(xin)                                    (dstt.py:246-254)
//   TOK_POST  : x = r + attn*Wo^T + bo ; x += W2 gelu(W1 LN2(x) + b1) + b2   (:146-149)
//   then, if a next block exists: y = LN1'(x); [q|k|v] = y*Wqkv'^T + b  (:141-142, :106-117)
//   TOK_SLOTKV: k,v = LN1(slot)*Wk,v^T + b for a memory slot            (:188-190)
// HBM traffic per token per block: fp32 residual in/out (512 B), fp16 attention output
// (128 B) and q/k/v (384 B).
#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

constexpr int WARPS = 4;
constexpr int LDY = 72;    // smem row stride (halves) of the 16 x 64 LN output
constexpr int LDH = 136;   // smem row stride (halves) of the 16 x 128 GELU output

struct Smem {
  __half y[16][LDY];
  __half h[16][LDH];
  float stat[WARPS][16];
};

// Slice of 16 tokens x 16 channels (2 n-tiles) in C-fragment layout.
struct Slice {
  float v[2][4];
};

DR_DEV void init_bias(float (*acc)[4], int nt_count, const float* __restrict__ bias,
                      int col0, int lane) {
  const int t = lane & 3;
  for (int nt = 0; nt < nt_count; ++nt) {
    const float b0 = __ldg(bias + col0 + nt * 8 + 2 * t), b1 = __ldg(bias + col0 + nt * 8 + 2 * t + 1);
    acc[nt][0] = b0; acc[nt][1] = b1; acc[nt][2] = b0; acc[nt][3] = b1;
  }
}

DR_DEV void load_slice_f32(Slice& x, const float* __restrict__ src, int n0, int n_tok,
                           int col0, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool v0 = n0 + g < n_tok, v1 = n0 + g + 8 < n_tok;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int c = col0 + nt * 8 + 2 * t;
    const float2 a = v0 ? __ldg(reinterpret_cast<const float2*>(src + (size_t)(n0 + g) * C + c)) : make_float2(0.f, 0.f);
    const float2 b = v1 ? __ldg(reinterpret_cast<const float2*>(src + (size_t)(n0 + g + 8) * C + c)) : make_float2(0.f, 0.f);
    x.v[nt][0] = a.x; x.v[nt][1] = a.y; x.v[nt][2] = b.x; x.v[nt][3] = b.y;
  }
}

DR_DEV void store_slice_f32(const Slice& x, float* dst, int n0, int n_tok, int col0, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool v0 = n0 + g < n_tok, v1 = n0 + g + 8 < n_tok;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int c = col0 + nt * 8 + 2 * t;
    if (v0) *reinterpret_cast<float2*>(dst + (size_t)(n0 + g) * C + c) = make_float2(x.v[nt][0], x.v[nt][1]);
    if (v1) *reinterpret_cast<float2*>(dst + (size_t)(n0 + g + 8) * C + c) = make_float2(x.v[nt][2], x.v[nt][3]);
  }
}

// fp16 tokens onto the zero-padded (R+2) x (Cc+2) grid that Vec2Patch reads.
DR_DEV size_t padded_pos(int n, int T, int R, int Cc) {
  const int f = n / T, t = n - f * T;
  const int i = t / Cc, j = t - i * Cc;
  return ((size_t)f * (R + 2) + i + 1) * (Cc + 2) + j + 1;
}

DR_DEV void store_slice_padded_f16(const Slice& x, __half* dst, int n0, int n_tok, int T, int R,
                                   int Cc, int col0, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool v0 = n0 + g < n_tok, v1 = n0 + g + 8 < n_tok;
  __half* r0 = dst + (v0 ? padded_pos(n0 + g, T, R, Cc) : 0) * C;
  __half* r1 = dst + (v1 ? padded_pos(n0 + g + 8, T, R, Cc) : 0) * C;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int c = col0 + nt * 8 + 2 * t;
    if (v0) *reinterpret_cast<uint32_t*>(r0 + c) = pack_half2(x.v[nt][0], x.v[nt][1]);
    if (v1) *reinterpret_cast<uint32_t*>(r1 + c) = pack_half2(x.v[nt][2], x.v[nt][3]);
  }
}

// LayerNorm (eps 1e-5, biased variance) of the 16 rows whose 64 channels are spread over
// the 4 warps; writes this warp's 16 normalised columns (fp16) into sm.y.  Two CTA
// barriers (row sums, then centred sums of squares).  Ends with sm.y complete.
DR_DEV void layer_norm_to_smem(const Slice& x, const float* __restrict__ w,
                               const float* __restrict__ b, Smem& sm, int col0, int warp,
                               int lane) {
  const int g = lane >> 2, t = lane & 3;
  float s0 = x.v[0][0] + x.v[0][1] + x.v[1][0] + x.v[1][1];
  float s1 = x.v[0][2] + x.v[0][3] + x.v[1][2] + x.v[1][3];
  s0 = quad_sum(s0);
  s1 = quad_sum(s1);
  if (t == 0) { sm.stat[warp][g] = s0; sm.stat[warp][g + 8] = s1; }
  __syncthreads();
  const float mu0 = (sm.stat[0][g] + sm.stat[1][g] + sm.stat[2][g] + sm.stat[3][g]) * (1.f / 64.f);
  const float mu1 = (sm.stat[0][g + 8] + sm.stat[1][g + 8] + sm.stat[2][g + 8] + sm.stat[3][g + 8]) * (1.f / 64.f);
  float q0 = 0.f, q1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    float d;
    d = x.v[nt][0] - mu0; q0 += d * d;
    d = x.v[nt][1] - mu0; q0 += d * d;
    d = x.v[nt][2] - mu1; q1 += d * d;
    d = x.v[nt][3] - mu1; q1 += d * d;
  }
  q0 = quad_sum(q0);
  q1 = quad_sum(q1);
  __syncthreads();                                     // everyone has read the row sums
  if (t == 0) { sm.stat[warp][g] = q0; sm.stat[warp][g + 8] = q1; }
  __syncthreads();
  const float r0 = rsqrtf((sm.stat[0][g] + sm.stat[1][g] + sm.stat[2][g] + sm.stat[3][g]) * (1.f / 64.f) + 1e-5f);
  const float r1 = rsqrtf((sm.stat[0][g + 8] + sm.stat[1][g + 8] + sm.stat[2][g + 8] + sm.stat[3][g + 8]) * (1.f / 64.f) + 1e-5f);
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int c = col0 + nt * 8 + 2 * t;
    const float w0 = __ldg(w + c), w1 = __ldg(w + c + 1), b0 = __ldg(b + c), b1 = __ldg(b + c + 1);
    *reinterpret_cast<uint32_t*>(&sm.y[g][c]) =
        pack_half2((x.v[nt][0] - mu0) * r0 * w0 + b0, (x.v[nt][1] - mu0) * r0 * w1 + b1);
    *reinterpret_cast<uint32_t*>(&sm.y[g + 8][c]) =
        pack_half2((x.v[nt][2] - mu1) * r1 * w0 + b0, (x.v[nt][3] - mu1) * r1 * w1 + b1);
  }
  __syncthreads();
}

// A fragments of a 16 x (16*KT) fp16 tile in smem (row stride ld halves).
template <int KT>
DR_DEV void smem_a(uint32_t (*a)[4], const __half* base, int ld, int lane) {
  const int m = lane >> 3;
  const int row = (lane & 7) + (m & 1) * 8;
#pragma unroll
  for (int kt = 0; kt < KT; ++kt) ldmatrix_x4(a[kt], base + row * ld + kt * 16 + (m >> 1) * 8);
}

// acc[nt] += A * W^T over n-tiles [nt0, nt0+NT) of a packed weight with KT k-tiles.
template <int NT, int KT>
DR_DEV void gemm(float (*acc)[4], const uint32_t (*a)[4], const uint2* __restrict__ w, int nt0,
                 int lane) {
  uint2 b[NT][KT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) b[nt][kt] = ld_frag(w, (nt0 + nt) * KT + kt, lane);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) mma16816(acc[nt], a[kt], b[nt][kt].x, b[nt][kt].y);
}

// LN1 + q/k/v projection groups [p0, p0+np) (16 columns = one head of q, k or v each),
// written head-major [frame][head][T][16].
DR_DEV void qkv_groups(const Slice& x, const BlockW& w, __half* q, __half* k, __half* v,
                       int n0, int n_tok, int T, int p0, int np, Smem& sm, int col0, int warp,
                       int lane) {
  layer_norm_to_smem(x, w.ln1_w, w.ln1_b, sm, col0, warp, lane);
  uint32_t a[4][4];
  smem_a<4>(a, &sm.y[0][0], LDY, lane);
  const int g = lane >> 2, t = lane & 3;
  const int na = n0 + g, nb = n0 + g + 8;
  const int fa = na / T, ta = na - fa * T, fb = nb / T, tb = nb - fb * T;
  for (int p = p0; p < p0 + np; ++p) {
    float acc[2][4];
    init_bias(acc, 2, w.bqkv, p * 16, lane);
    gemm<2, 4>(acc, a, w.wqkv, 2 * p, lane);
    const int which = p >> 2, h = p & 3;
    __half* dst = which == 0 ? q : (which == 1 ? k : v);
    // q, k, v rows are stored with the UMMA 32-byte swizzle (16-byte chunk c of token t at
    // c ^ ((t >> 2) & 1)): the attention kernel's bulk copies land as SWIZZLE_32B operands.
    const int sa = ((ta >> 2) & 1) * 4, sb = ((tb >> 2) & 1) * 4;
    if (na < n_tok) {
      uint32_t* r = reinterpret_cast<uint32_t*>(dst + ((size_t)(fa * HEADS + h) * T + ta) * DH);
      r[sa + t] = pack_half2(acc[0][0], acc[0][1]);
      r[(4 ^ sa) + t] = pack_half2(acc[1][0], acc[1][1]);
    }
    if (nb < n_tok) {
      uint32_t* r = reinterpret_cast<uint32_t*>(dst + ((size_t)(fb * HEADS + h) * T + tb) * DH);
      r[sb + t] = pack_half2(acc[0][2], acc[0][3]);
      r[(4 ^ sb) + t] = pack_half2(acc[1][2], acc[1][3]);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32) token_kernel(TokenArgs a) {
  __shared__ __align__(16) Smem sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n0 = blockIdx.x * 16;
  const int col0 = 16 * warp;                          // this warp's 16 of the 64 channels
  Slice x;
  pdl_trigger();
  pdl_wait();

  if constexpr (MODE == TOK_SLOTKV) {
    load_slice_f32(x, a.resid_in, n0, a.n_tok, col0, lane);
    qkv_groups(x, a.next, a.q, a.k, a.v, n0, a.n_tok, a.T, 4 + 2 * warp, 2, sm, col0, warp, lane);
    return;
  } else if constexpr (MODE == TOK_EMBED) {
    init_bias(x.v, 2, a.be, col0, lane);
    const int g = lane >> 2, t = lane & 3;
    const bool v0 = n0 + g < a.n_tok, v1 = n0 + g + 8 < a.n_tok;
    const uint32_t* r0 = reinterpret_cast<const uint32_t*>(a.xin + (size_t)(n0 + g) * a.kin);
    const uint32_t* r1 = reinterpret_cast<const uint32_t*>(a.xin + (size_t)(n0 + g + 8) * a.kin);
    const int KT = a.kin / 16;
#pragma unroll 4
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t af[4];
      af[0] = v0 ? __ldg(r0 + kt * 8 + t) : 0u;
      af[1] = v1 ? __ldg(r1 + kt * 8 + t) : 0u;
      af[2] = v0 ? __ldg(r0 + kt * 8 + 4 + t) : 0u;
      af[3] = v1 ? __ldg(r1 + kt * 8 + 4 + t) : 0u;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const uint2 b = ld_frag(a.we, (2 * warp + nt) * KT + kt, lane);
        mma16816(x.v[nt], af, b.x, b.y);
      }
    }
  } else {  // TOK_POST
    load_slice_f32(x, a.resid_in, n0, a.n_tok, col0, lane);
    {
      uint32_t ao[4][4];
      const int g = lane >> 2, t = lane & 3;
      const bool v0 = n0 + g < a.n_tok, v1 = n0 + g + 8 < a.n_tok;
      const uint32_t* r0 = reinterpret_cast<const uint32_t*>(a.attn + (size_t)(n0 + g) * C);
      const uint32_t* r1 = reinterpret_cast<const uint32_t*>(a.attn + (size_t)(n0 + g + 8) * C);
#pragma unroll
      for (int kt = 0; kt < 4; ++kt) {
        ao[kt][0] = v0 ? __ldg(r0 + kt * 8 + t) : 0u;
        ao[kt][1] = v1 ? __ldg(r1 + kt * 8 + t) : 0u;
        ao[kt][2] = v0 ? __ldg(r0 + kt * 8 + 4 + t) : 0u;
        ao[kt][3] = v1 ? __ldg(r1 + kt * 8 + 4 + t) : 0u;
      }
      float acc[2][4];
      init_bias(acc, 2, a.cur.bo, col0, lane);
      gemm<2, 4>(acc, ao, a.cur.wo, 2 * warp, lane);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) x.v[nt][i] += acc[nt][i];
    }
    layer_norm_to_smem(x, a.cur.ln2_w, a.cur.ln2_b, sm, col0, warp, lane);
    {
      uint32_t ya[4][4];
      smem_a<4>(ya, &sm.y[0][0], LDY, lane);
      float hacc[4][4];                                // FFN1 columns [32w, 32w+32)
      init_bias(hacc, 4, a.cur.b1, 32 * warp, lane);
      gemm<4, 4>(hacc, ya, a.cur.w1, 4 * warp, lane);
      const int g = lane >> 2, t = lane & 3;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = 32 * warp + nt * 8 + 2 * t;
        *reinterpret_cast<uint32_t*>(&sm.h[g][c]) = pack_half2(gelu_erf(hacc[nt][0]), gelu_erf(hacc[nt][1]));
        *reinterpret_cast<uint32_t*>(&sm.h[g + 8][c]) = pack_half2(gelu_erf(hacc[nt][2]), gelu_erf(hacc[nt][3]));
      }
    }
    __syncthreads();
    {
      uint32_t ha[8][4];
      smem_a<8>(ha, &sm.h[0][0], LDH, lane);
      float acc[2][4];
      init_bias(acc, 2, a.cur.b2, col0, lane);
      gemm<2, 8>(acc, ha, a.cur.w2, 2 * warp, lane);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) x.v[nt][i] += acc[nt][i];
    }
  }

  store_slice_f32(x, a.resid_out, n0, a.n_tok, col0, lane);
  if (a.has_next) {
    __syncthreads();                                   // sm.y / sm.h reads are done
    qkv_groups(x, a.next, a.q, a.k, a.v, n0, a.n_tok, a.T, 3 * warp, 3, sm, col0, warp, lane);
  } else {
    if (a.tok16) store_slice_padded_f16(x, a.tok16, n0, a.n_tok, a.T, a.R, a.Cc, col0, lane);
    // K/V of the new memory slot for every temporal block: the next frames read them
    // from the slot K/V cache instead of re-projecting the slot (dstt.py:188-190).
    for (int i = 0; i < a.n_kv; ++i) {
      __syncthreads();                                 // sm.y / sm.h reads are done
      qkv_groups(x, a.kv_w[i], nullptr, a.kv_k[i], a.kv_v[i], n0, a.n_tok, a.T, 4 + 2 * warp, 2,
                 sm, col0, warp, lane);
    }
  }
}

}  // namespace

void launch_token(int mode, const TokenArgs& a, cudaStream_t s) {
  dim3 grid((a.n_tok + 15) / 16), block(WARPS * 32);
  switch (mode) {
    case TOK_EMBED: launch_pdl(token_kernel<TOK_EMBED>, grid, block, 0, s, a); break;
    case TOK_POST: launch_pdl(token_kernel<TOK_POST>, grid, block, 0, s, a); break;
    default: launch_pdl(token_kernel<TOK_SLOTKV>, grid, block, 0, s, a); break;
  }
}

}  // namespace dr
