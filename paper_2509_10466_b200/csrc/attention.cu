// Fused single-pass attention for the DSTT blocks, head_dim 16.
//
// Reference: scaled_dot_product (dstt.py:89-99) inside MultiHeadAttention (:111-120);
// spatial blocks attend over the whole frame (:146-150), temporal blocks attend a row
// band of queries to cat[band(cur), band(slot0), band(slot1)] (:166-191).  The reference
// materialises the T x T weights; here scores live only in registers: online softmax in
// the log2 domain (one FFMA + one MUFU ex2 per score), P packed to fp16 in registers and
// fed straight back into the P*V HMMA.  With dh=16 the kernel is MUFU-bound (SURVEY
// §0.7): 16 ex2/clk/SM against 64 HMMA flops per score.
//
// Mask-aware mode (NEW): keys of fully-masked tokens of the current frame get
// -inf; memory-slot keys are always valid; a spatial block whose frame has no valid key
// falls back to unmasked attention.  The MAT validity update is resolved on the host
// into a per-block mask_mode (see engine.cpp).
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

constexpr int WARPS = 4;     // 64 queries per CTA
constexpr int KB = 64;       // keys per pipeline stage
constexpr int STAGES = 3;

struct __align__(128) Smem {
  __half k[STAGES][KB][DH];
  __half v[STAGES][KB][DH];
  float bias[STAGES][KB];
};

// Swizzled 16-byte chunk position inside a 32-byte key row (conflict-free ldmatrix).
DR_DEV int swz(int key, int chunk) { return chunk ^ ((key >> 2) & 1); }

template <bool MASKED>
__global__ void __launch_bounds__(WARPS * 32) attn_kernel(AttnArgs a) {
  __shared__ Smem sm;
  __shared__ int any_valid_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int h = blockIdx.y;
  const int frame = blockIdx.z / a.groups, grp = blockIdx.z - frame * a.groups;
  const int band0 = grp * a.band;
  const int n_keys = a.n_seg * a.band;
  const int n_kb = (n_keys + KB - 1) / KB;

  int any_valid = 1;
  if constexpr (MASKED) {
    if (a.mask_mode == 1 || a.mask_mode == 3) {
      const uint8_t* kv = a.key_valid + (size_t)frame * a.T;
      int mine = 0;
      for (int i = tid; i < a.T; i += WARPS * 32) mine |= kv[i];
      any_valid = __syncthreads_or(mine);
    }
  }
  (void)any_valid_s;

  auto load_stage = [&](int kb, int st) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int idx = tid + c * WARPS * 32;            // 0..255
      const int which = idx >> 7, key = (idx & 127) >> 1, chunk = idx & 1;
      const int kk = kb * KB + key;
      const bool valid = kk < n_keys;
      const int seg = valid ? kk / a.band : 0;
      const int tok = band0 + (valid ? kk - seg * a.band : 0);
      const int stride = seg == 0 ? a.seg_frame_stride[0]
                       : (seg == 1 ? a.seg_frame_stride[1] : a.seg_frame_stride[2]);
      const int fr = stride ? frame : 0;
      const __half* kb_ = seg == 0 ? a.k[0] : (seg == 1 ? a.k[1] : a.k[2]);
      const __half* vb_ = seg == 0 ? a.v[0] : (seg == 1 ? a.v[1] : a.v[2]);
      const __half* base = which ? vb_ : kb_;
      const __half* src = base + ((size_t)(fr * HEADS + h) * a.T + tok) * DH + chunk * 8;
      __half* dst = which ? &sm.v[st][key][swz(key, chunk) * 8] : &sm.k[st][key][swz(key, chunk) * 8];
      cp_async16_zfill(dst, src, valid);
    }
    if constexpr (MASKED) {
      if (tid < KB) {
        const int kk = kb * KB + tid;
        float bias = -INFINITY;
        if (kk < n_keys) {
          const int seg = kk / a.band;
          bool ok = true;
          if (seg == 0 && a.mask_mode != 0) {
            const int tok = band0 + kk;
            const bool kv = a.key_valid[(size_t)frame * a.T + tok] != 0;
            if (a.mask_mode == 1) ok = kv || !any_valid;
            else if (a.mask_mode == 2) ok = kv;
            else ok = any_valid;
          }
          bias = ok ? 0.f : -INFINITY;
        }
        sm.bias[st][tid] = bias;
      }
    }
  };

  // Query fragment (16 queries x 16 dims) straight from global.
  const int q0 = blockIdx.x * (WARPS * 16) + warp * 16;
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
    if (s < n_kb) load_stage(s, s);
    cp_async_commit();
  }

  const float sl2 = 0.25f * 1.4426950408889634f;   // 1/sqrt(16) * log2(e)
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  const bool partial_last = (n_keys % KB) != 0;

  for (int kb = 0; kb < n_kb; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kb + STAGES - 1;
      if (nk < n_kb) load_stage(nk, nk % STAGES);
      cp_async_commit();
    }
    const int st = kb % STAGES;

    float s[8][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t kf[4];
      const int key = 16 * j + (lane & 7) + ((lane >> 4) & 1) * 8;
      const int chunk = (lane >> 3) & 1;
      ldmatrix_x4(kf, &sm.k[st][key][swz(key, chunk) * 8]);
#pragma unroll
      for (int e = 0; e < 4; ++e) { s[2 * j][e] = 0.f; s[2 * j + 1][e] = 0.f; }
      mma16816(s[2 * j], qa, kf[0], kf[1]);
      mma16816(s[2 * j + 1], qa, kf[2], kf[3]);
    }
    if constexpr (MASKED) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float b0 = sm.bias[st][nt * 8 + 2 * t], b1 = sm.bias[st][nt * 8 + 2 * t + 1];
        s[nt][0] += b0; s[nt][1] += b1; s[nt][2] += b0; s[nt][3] += b1;
      }
    } else {
      if (partial_last && kb == n_kb - 1) {
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const int col = kb * KB + nt * 8 + 2 * t;
          if (col >= n_keys) { s[nt][0] = -INFINITY; s[nt][2] = -INFINITY; }
          if (col + 1 >= n_keys) { s[nt][1] = -INFINITY; s[nt][3] = -INFINITY; }
        }
      }
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
    mx0 = quad_max(mx0) * sl2;
    mx1 = quad_max(mx1) * sl2;
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float base0 = mn0 == -INFINITY ? 0.f : mn0;
    const float base1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = ex2(m0 - base0), c1 = ex2(m1 - base1);
    m0 = mn0; m1 = mn1;
    float ps0 = 0.f, ps1 = 0.f;
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = ex2(fmaf(s[nt][0], sl2, -base0));
      const float p1 = ex2(fmaf(s[nt][1], sl2, -base0));
      const float p2 = ex2(fmaf(s[nt][2], sl2, -base1));
      const float p3 = ex2(fmaf(s[nt][3], sl2, -base1));
      ps0 += p0 + p1; ps1 += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_half2(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_half2(p2, p3);
    }
    l0 = l0 * c0 + ps0;
    l1 = l1 * c1 + ps1;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) { o[nt][0] *= c0; o[nt][1] *= c0; o[nt][2] *= c1; o[nt][3] *= c1; }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t vf[4];
      const int mi = lane >> 3;
      const int key = 16 * j + (lane & 7) + (mi & 1) * 8;
      const int chunk = mi >> 1;
      ldmatrix_x4_trans(vf, &sm.v[st][key][swz(key, chunk) * 8]);
      mma16816(o[0], pa[j], vf[0], vf[1]);
      mma16816(o[1], pa[j], vf[2], vf[3]);
    }
  }
  cp_async_wait<0>();

  l0 = quad_sum(l0);
  l1 = quad_sum(l1);
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
  dim3 grid((a.band + WARPS * 16 - 1) / (WARPS * 16), HEADS, a.frames * a.groups);
  if (a.mask_mode != 0 && a.key_valid)
    attn_kernel<true><<<grid, WARPS * 32, 0, s>>>(a);
  else
    attn_kernel<false><<<grid, WARPS * 32, 0, s>>>(a);
}

}  // namespace dr
