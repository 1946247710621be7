// Fused single-pass attention for the DSTT blocks, head_dim 16.
//
// Reference: scaled_dot_product (dstt.py:89-99) inside MultiHeadAttention (:111-120);
// spatial blocks attend over the whole frame (:146-150), temporal blocks attend a row
// band of queries to cat[band(cur), band(slot0), band(slot1)] (:166-191).  The reference
// materialises the T x T weights; here scores live only in registers: online softmax in
// the log2 domain (one FFMA + one MUFU ex2 per score), P packed to fp16 in registers and
// fed straight back into the P*V HMMA.  With dh=16 the kernel is bound by MUFU ex2
// (16/clk/SM) and by issue, not by the tensor pipe (64 MMA flops per score), so the
// design goal is latency hiding: a CTA = 4 query tiles x 2 key halves = 8 warps that
// share the cp.async-staged K/V blocks; the two halves' (max, sum, O) are merged through
// smem at the end.  Accumulator chains are split (two O / l partials) for ILP.
//
// Mask-aware mode (NEW): keys of fully-masked tokens of the current frame get
// -inf; memory-slot keys are always valid; a spatial block whose frame has no valid key
// falls back to unmasked attention.  The MAT validity update is resolved on the host
// into a per-block mask_mode (see engine.cu).
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

constexpr int QT = 4;                 // query tiles of 16 per CTA
constexpr int KS = 2;                 // key splits per CTA
constexpr int WARPS = QT * KS;
constexpr int KB = 64;                // keys per block
constexpr int STAGES = 3;

struct __align__(128) Smem {
  __half k[STAGES][KS][KB][DH];
  __half v[STAGES][KS][KB][DH];
  float bias[STAGES][KS][KB];
  float ml[QT][32][4];                // key-half 1 partials: m0, m1, l0, l1 per lane
  float o[QT][32][8];
};

// Swizzled 16-byte chunk position inside a 32-byte key row (conflict-free ldmatrix).
DR_DEV int swz(int key, int chunk) { return chunk ^ ((key >> 2) & 1); }

template <bool MASKED>
__global__ void __launch_bounds__(WARPS * 32) attn_kernel(AttnArgs a) {
  __shared__ Smem sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qt = warp & (QT - 1), kh = warp / QT;
  const int g = lane >> 2, t = lane & 3;
  const int h = blockIdx.y;
  const int frame = blockIdx.z / a.groups, grp = blockIdx.z - frame * a.groups;
  const int band0 = grp * a.band;
  const int n_keys = a.n_seg * a.band;
  const int n_kb = (n_keys + KB - 1) / KB;
  const int nkb_h = (n_kb + 1) / 2;            // blocks per key half

  int any_valid = 1;
  if constexpr (MASKED) {
    if (a.mask_mode == 1 || a.mask_mode == 3) {
      const uint8_t* kv = a.key_valid + (size_t)frame * a.T;
      int mine = 0;
      for (int i = tid; i < a.T; i += WARPS * 32) mine |= kv[i];
      any_valid = __syncthreads_or(mine);
    }
  }

  auto load_stage = [&](int kb, int st) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int idx = tid + c * WARPS * 32;            // 0..511
      const int half = idx >> 8, rem = idx & 255;
      const int which = rem >> 7, key = (rem & 127) >> 1, chunk = rem & 1;
      const int blk = half * nkb_h + kb;
      const int kk = blk * KB + key;
      const bool valid = kb < nkb_h && blk < n_kb && kk < n_keys;
      const int seg = valid ? kk / a.band : 0;
      const int tok = band0 + (valid ? kk - seg * a.band : 0);
      const int stride = seg == 0 ? a.seg_frame_stride[0]
                       : (seg == 1 ? a.seg_frame_stride[1] : a.seg_frame_stride[2]);
      const int fr = stride ? frame : 0;
      const __half* kb_ = seg == 0 ? a.k[0] : (seg == 1 ? a.k[1] : a.k[2]);
      const __half* vb_ = seg == 0 ? a.v[0] : (seg == 1 ? a.v[1] : a.v[2]);
      const __half* src = (which ? vb_ : kb_) + ((size_t)(fr * HEADS + h) * a.T + tok) * DH + chunk * 8;
      __half* dst = which ? &sm.v[st][half][key][swz(key, chunk) * 8]
                          : &sm.k[st][half][key][swz(key, chunk) * 8];
      cp_async16_zfill(dst, src, valid);
    }
    if (tid < KS * KB) {                               // key bias: 0 valid, -inf masked
      const int half = tid / KB, key = tid - half * KB;
      const int blk = half * nkb_h + kb;
      const int kk = blk * KB + key;
      float bias = -INFINITY;
      if (kb < nkb_h && blk < n_kb && kk < n_keys) {
        bool ok = true;
        if constexpr (MASKED) {
          const int seg = kk / a.band;
          if (seg == 0 && a.mask_mode != 0) {
            const bool kv = a.key_valid[(size_t)frame * a.T + band0 + kk] != 0;
            if (a.mask_mode == 1) ok = kv || !any_valid;
            else if (a.mask_mode == 2) ok = kv;
            else ok = any_valid;
          }
        }
        bias = ok ? 0.f : -INFINITY;
      }
      sm.bias[st][half][key] = bias;
    }
  };

  // Query fragment (16 queries x 16 dims) straight from global.
  const int q0 = blockIdx.x * (QT * 16) + qt * 16;
  const bool qv0 = q0 + g < a.band, qv1 = q0 + g + 8 < a.band;
  uint32_t qa[4];
  {
    const __half* qb = a.q + ((size_t)(frame * HEADS + h) * a.T + band0 + q0) * DH;
    const uint32_t* r0 = reinterpret_cast<const uint32_t*>(qb + g * DH);
    const uint32_t* r1 = reinterpret_cast<const uint32_t*>(qb + (g + 8) * DH);
    qa[0] = qv0 ? __ldg(r0 + t) : 0u;
    qa[1] = qv1 ? __ldg(r1 + t) : 0u;
    qa[2] = qv0 ? __ldg(r0 + 4 + t) : 0u;
    qa[3] = qv1 ? __ldg(r1 + 4 + t) : 0u;
  }

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkb_h) load_stage(s, s);
    cp_async_commit();
  }

  const float sl2 = 0.25f * 1.4426950408889634f;   // 1/sqrt(16) * log2(e)
  float m0 = -INFINITY, m1 = -INFINITY;
  float l0a = 0.f, l0b = 0.f, l1a = 0.f, l1b = 0.f;
  float oe[2][4] = {}, oo[2][4] = {};               // even / odd key sub-tile partials

  for (int kb = 0; kb < nkb_h; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kb + STAGES - 1;
      if (nk < nkb_h) load_stage(nk, nk % STAGES);
      cp_async_commit();
    }
    const int st = kb % STAGES;

    float s[8][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t kf[4];
      const int key = 16 * j + (lane & 7) + ((lane >> 4) & 1) * 8;
      const int chunk = (lane >> 3) & 1;
      ldmatrix_x4(kf, &sm.k[st][kh][key][swz(key, chunk) * 8]);
#pragma unroll
      for (int e = 0; e < 4; ++e) { s[2 * j][e] = 0.f; s[2 * j + 1][e] = 0.f; }
      mma16816(s[2 * j], qa, kf[0], kf[1]);
      mma16816(s[2 * j + 1], qa, kf[2], kf[3]);
    }
    // key bias: always in mask-aware mode, else only on a partial / empty last block
    if (MASKED || (kh * nkb_h + kb + 1) * KB > n_keys) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float2 b = *reinterpret_cast<const float2*>(&sm.bias[st][kh][nt * 8 + 2 * t]);
        s[nt][0] += b.x; s[nt][1] += b.y; s[nt][2] += b.x; s[nt][3] += b.y;
      }
    }
    float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
    float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
    float mx0b = fmaxf(fmaxf(s[2][0], s[2][1]), fmaxf(s[3][0], s[3][1]));
    float mx1b = fmaxf(fmaxf(s[2][2], s[2][3]), fmaxf(s[3][2], s[3][3]));
#pragma unroll
    for (int nt = 4; nt < 8; nt += 2) {
      mx0 = fmaxf(mx0, fmaxf(fmaxf(s[nt][0], s[nt][1]), fmaxf(s[nt + 1][0], s[nt + 1][1])));
      mx1 = fmaxf(mx1, fmaxf(fmaxf(s[nt][2], s[nt][3]), fmaxf(s[nt + 1][2], s[nt + 1][3])));
    }
    mx0 = quad_max(fmaxf(mx0, mx0b)) * sl2;
    mx1 = quad_max(fmaxf(mx1, mx1b)) * sl2;
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float base0 = mn0 == -INFINITY ? 0.f : mn0;
    const float base1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = ex2(m0 - base0), c1 = ex2(m1 - base1);
    m0 = mn0; m1 = mn1;
    uint32_t pa[4][4];
    float ps0a = 0.f, ps0b = 0.f, ps1a = 0.f, ps1b = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = ex2(fmaf(s[nt][0], sl2, -base0));
      const float p1 = ex2(fmaf(s[nt][1], sl2, -base0));
      const float p2 = ex2(fmaf(s[nt][2], sl2, -base1));
      const float p3 = ex2(fmaf(s[nt][3], sl2, -base1));
      if (nt & 1) { ps0b += p0 + p1; ps1b += p2 + p3; }
      else { ps0a += p0 + p1; ps1a += p2 + p3; }
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_half2(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_half2(p2, p3);
    }
    l0a = l0a * c0 + ps0a; l0b = l0b * c0 + ps0b;
    l1a = l1a * c1 + ps1a; l1b = l1b * c1 + ps1b;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      oe[nt][0] *= c0; oe[nt][1] *= c0; oe[nt][2] *= c1; oe[nt][3] *= c1;
      oo[nt][0] *= c0; oo[nt][1] *= c0; oo[nt][2] *= c1; oo[nt][3] *= c1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t vf[4];
      const int mi = lane >> 3;
      const int key = 16 * j + (lane & 7) + (mi & 1) * 8;
      const int chunk = mi >> 1;
      ldmatrix_x4_trans(vf, &sm.v[st][kh][key][swz(key, chunk) * 8]);
      float (*o)[4] = (j & 1) ? oo : oe;
      mma16816(o[0], pa[j], vf[0], vf[1]);
      mma16816(o[1], pa[j], vf[2], vf[3]);
    }
  }
  cp_async_wait<0>();

  float l0 = quad_sum(l0a + l0b), l1 = quad_sum(l1a + l1b);
  float o[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[nt][e] = oe[nt][e] + oo[nt][e];

  // merge the two key halves (log2-domain running max / sum / O)
  if (kh == 1) {
    float* ml = sm.ml[qt][lane];
    ml[0] = m0; ml[1] = m1; ml[2] = l0; ml[3] = l1;
    float* po = sm.o[qt][lane];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) po[nt * 4 + e] = o[nt][e];
  }
  __syncthreads();
  if (kh == 1) return;
  {
    const float* ml = sm.ml[qt][lane];
    const float* po = sm.o[qt][lane];
    const float M0 = fmaxf(m0, ml[0]), M1 = fmaxf(m1, ml[1]);
    const float b0 = M0 == -INFINITY ? 0.f : M0, b1 = M1 == -INFINITY ? 0.f : M1;
    const float a0 = ex2(m0 - b0), a1 = ex2(m1 - b1);
    const float d0 = ex2(ml[0] - b0), d1 = ex2(ml[1] - b1);
    l0 = l0 * a0 + ml[2] * d0;
    l1 = l1 * a1 + ml[3] * d1;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      o[nt][0] = o[nt][0] * a0 + po[nt * 4 + 0] * d0;
      o[nt][1] = o[nt][1] * a0 + po[nt * 4 + 1] * d0;
      o[nt][2] = o[nt][2] * a1 + po[nt * 4 + 2] * d1;
      o[nt][3] = o[nt][3] * a1 + po[nt * 4 + 3] * d1;
    }
  }
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  __half* ob = a.out + ((size_t)frame * a.T + band0 + q0) * C + h * DH;
  if (qv0) {
    uint32_t* r = reinterpret_cast<uint32_t*>(ob + (size_t)g * C);
    r[t] = pack_half2(o[0][0] * inv0, o[0][1] * inv0);
    r[4 + t] = pack_half2(o[1][0] * inv0, o[1][1] * inv0);
  }
  if (qv1) {
    uint32_t* r = reinterpret_cast<uint32_t*>(ob + (size_t)(g + 8) * C);
    r[t] = pack_half2(o[0][2] * inv1, o[0][3] * inv1);
    r[4 + t] = pack_half2(o[1][2] * inv1, o[1][3] * inv1);
  }
}

}  // namespace

void launch_attention(const AttnArgs& a, cudaStream_t s) {
  dim3 grid((a.band + QT * 16 - 1) / (QT * 16), HEADS, a.frames * a.groups);
  if (a.mask_mode != 0 && a.key_valid)
    attn_kernel<true><<<grid, WARPS * 32, 0, s>>>(a);
  else
    attn_kernel<false><<<grid, WARPS * 32, 0, s>>>(a);
}

}  // namespace dr
