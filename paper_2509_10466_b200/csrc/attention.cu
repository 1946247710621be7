// Fused single-pass attention for the DSTT blocks, head_dim 16.
//
// Reference: scaled_dot_product (dstt.py:89-99) inside MultiHeadAttention (:111-120);
// spatial blocks attend over the whole frame (:146-150), temporal blocks attend a row
// band of queries to cat[band(cur), band(slot0), band(slot1)] (:166-191).  The reference
// materialises the T x T weights; here scores live only in registers: online softmax in
// the log2 domain (one FFMA + one MUFU ex2 per score), P packed to fp16 in registers and
// fed straight back into the P*V HMMA.
//
// With dh = 16 the floor is MUFU ex2 (measured 16/clk/SM on B200, profiles/r01/
// pipe_microbench_b200.txt), so everything else per score must stay small:
//  * a dedicated producer warp streams 128-key K/V blocks with cp.async.bulk into a
//    3-stage ring (full/empty mbarriers, no CTA-wide barrier per block); the QKV producer
//    (token_kernels.cu) already stored K/V with the 16-byte chunk swizzle that makes
//    ldmatrix conflict-free, so no per-key index math runs on the math warps;
//  * row sums come out of the P*V HMMA through a constant ones column (no FADD chain);
//  * the running max is rescaled lazily (only when a row max grows by > 2^8, exact
//    because numerator and denominator share the stale max);
//  * the key-tail masking exists only in a separate instantiation for the last, partial
//    block, so the steady-state block body carries no per-score selects;
//  * 8 math warps = 4 query tiles x 2 key halves share the smem ring; the two halves'
//    (max, sum, O) are merged through smem at the end.
//
// Mask-aware mode (NEW): keys of fully-masked tokens of the current frame get
// -inf; memory-slot keys are always valid; a spatial block whose frame has no valid key
// falls back to unmasked attention.  The MAT validity update is resolved on the host
// into a per-block mask_mode (see engine.cu).
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace dr {

namespace {

constexpr int QT = 4;                 // query tiles of 16 per CTA
constexpr int KS = 2;                 // key splits per CTA
constexpr int MATH_WARPS = QT * KS;
constexpr int THREADS = (MATH_WARPS + 1) * 32;   // + producer warp
constexpr int KB = 128;               // keys per block
constexpr int STAGES = 3;
constexpr float RESCALE_SLACK = 8.f;  // log2 units: p <= 2^8 between rescales

struct __align__(128) Smem {
  __half k[STAGES][KS][KB][DH];
  __half v[STAGES][KS][KB][DH];
  float bias[STAGES][KS][KB];         // mask-aware mode only
  float ml[QT][32][4];                // key-half 1 partials: m0, m1, l0, l1 per lane
  float o[QT][32][8];
  uint64_t full[STAGES], empty[STAGES];
};

// Swizzled 16-byte chunk position inside a 32-byte key row (conflict-free ldmatrix).
DR_DEV int swz(int key, int chunk) { return chunk ^ ((key >> 2) & 1); }

DR_DEV float max3(float a, float b, float c) { return fmaxf(a, fmaxf(b, c)); }

struct SoftmaxState {
  float m0, m1;
  float oe[3][4], oo[3][4];           // [dims 0-7, dims 8-15, row sum] for even/odd j
};

// 64 keys for one warp (16 queries): S = Q K^T, online softmax, O += P V.
template <bool MASKED, bool PARTIAL>
DR_DEV void attend_64(SoftmaxState& st, const uint32_t* qa, const __half (*ks)[DH],
                      const __half (*vs)[DH], const float* bias, int n_valid, int lane) {
  const int t = lane & 3;
  const float sl2 = 0.25f * 1.4426950408889634f;   // 1/sqrt(16) * log2(e)
  float s[8][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t kf[4];
    const int key = 16 * j + (lane & 7) + ((lane >> 4) & 1) * 8;
    const int chunk = (lane >> 3) & 1;
    ldmatrix_x4(kf, &ks[key][swz(key, chunk) * 8]);
#pragma unroll
    for (int e = 0; e < 4; ++e) { s[2 * j][e] = 0.f; s[2 * j + 1][e] = 0.f; }
    mma16816(s[2 * j], qa, kf[0], kf[1]);
    mma16816(s[2 * j + 1], qa, kf[2], kf[3]);
  }
  if constexpr (MASKED) {
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float2 b = *reinterpret_cast<const float2*>(&bias[nt * 8 + 2 * t]);
      s[nt][0] += b.x; s[nt][1] += b.y; s[nt][2] += b.x; s[nt][3] += b.y;
    }
  }
  if constexpr (PARTIAL) {
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int col = nt * 8 + 2 * t;
      if (col >= n_valid) { s[nt][0] = -INFINITY; s[nt][2] = -INFINITY; }
      if (col + 1 >= n_valid) { s[nt][1] = -INFINITY; s[nt][3] = -INFINITY; }
    }
  }
  float mx0 = max3(s[0][0], s[0][1], s[1][0]), mx1 = max3(s[0][2], s[0][3], s[1][2]);
  float nx0 = max3(s[1][1], s[2][0], s[2][1]), nx1 = max3(s[1][3], s[2][2], s[2][3]);
#pragma unroll
  for (int nt = 3; nt < 7; nt += 2) {
    mx0 = max3(mx0, s[nt][0], s[nt][1]);
    mx1 = max3(mx1, s[nt][2], s[nt][3]);
    nx0 = max3(nx0, s[nt + 1][0], s[nt + 1][1]);
    nx1 = max3(nx1, s[nt + 1][2], s[nt + 1][3]);
  }
  mx0 = max3(mx0, nx0, fmaxf(s[7][0], s[7][1]));
  mx1 = max3(mx1, nx1, fmaxf(s[7][2], s[7][3]));
  mx0 = quad_max(mx0) * sl2;
  mx1 = quad_max(mx1) * sl2;
  if (__builtin_expect(__any_sync(0xffffffffu, mx0 > st.m0 + RESCALE_SLACK ||
                                               mx1 > st.m1 + RESCALE_SLACK), 0)) {
    const float mn0 = fmaxf(st.m0, mx0), mn1 = fmaxf(st.m1, mx1);
    const float c0 = ex2(st.m0 - (mn0 == -INFINITY ? 0.f : mn0));
    const float c1 = ex2(st.m1 - (mn1 == -INFINITY ? 0.f : mn1));
    st.m0 = mn0; st.m1 = mn1;
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      st.oe[nt][0] *= c0; st.oe[nt][1] *= c0; st.oe[nt][2] *= c1; st.oe[nt][3] *= c1;
      st.oo[nt][0] *= c0; st.oo[nt][1] *= c0; st.oo[nt][2] *= c1; st.oo[nt][3] *= c1;
    }
  }
  const float base0 = st.m0 == -INFINITY ? 0.f : st.m0;
  const float base1 = st.m1 == -INFINITY ? 0.f : st.m1;
  const uint32_t ones = (lane >> 2) == 0 ? 0x3C003C00u : 0u;   // B column 0 = 1 -> row sum
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    // (Offloading a quarter of these to ex2_poly on the FMA pipe measured slower at batch
    //  1: the kernel is issue/latency-bound there, not MUFU-bound.)
    auto e2 = [](float x) { return ex2(x); };
    uint32_t pa[4];
    pa[0] = pack_half2(e2(fmaf(s[2 * j][0], sl2, -base0)), e2(fmaf(s[2 * j][1], sl2, -base0)));
    pa[1] = pack_half2(e2(fmaf(s[2 * j][2], sl2, -base1)), e2(fmaf(s[2 * j][3], sl2, -base1)));
    pa[2] = pack_half2(e2(fmaf(s[2 * j + 1][0], sl2, -base0)), e2(fmaf(s[2 * j + 1][1], sl2, -base0)));
    pa[3] = pack_half2(e2(fmaf(s[2 * j + 1][2], sl2, -base1)), e2(fmaf(s[2 * j + 1][3], sl2, -base1)));
    uint32_t vf[4];
    const int mi = lane >> 3;
    const int key = 16 * j + (lane & 7) + (mi & 1) * 8;
    const int chunk = mi >> 1;
    ldmatrix_x4_trans(vf, &vs[key][swz(key, chunk) * 8]);
    float (*o)[4] = (j & 1) ? st.oo : st.oe;
    mma16816(o[0], pa, vf[0], vf[1]);
    mma16816(o[1], pa, vf[2], vf[3]);
    mma16816(o[2], pa, ones, ones);
  }
}

template <bool MASKED>
__global__ void __launch_bounds__(THREADS, 2) attn_kernel(AttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];  // direct cast keeps LDS addressing
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int h = blockIdx.y;
  const int frame = blockIdx.z / a.groups, grp = blockIdx.z - frame * a.groups;
  const int band0 = grp * a.band;
  const int n_keys = a.n_seg * a.band;
  const int n_kb = (n_keys + KB - 1) / KB;
  const int nkb_h = (n_kb + 1) / 2;            // blocks per key half

  pdl_trigger();
  // zero the K/V ring once: tails of partial blocks must hold finite values
  {
    uint4* z = reinterpret_cast<uint4*>(&sm.k[0][0][0][0]);
    constexpr int n16 = (int)(2 * sizeof(sm.k) / 16);
    for (int i = tid; i < n16; i += THREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&sm.full[s], 1);
      tc::mbar_init(&sm.empty[s], MATH_WARPS);
    }
    tc::fence_barrier_init();
  }
  pdl_wait();                                     // q / k / v / key_valid of the predecessor
  int any_valid = 1;
  if constexpr (MASKED) {
    if (a.mask_mode == 1 || a.mask_mode == 3) {
      const uint8_t* kv = a.key_valid + (size_t)frame * a.T;
      int mine = 0;
      for (int i = tid; i < a.T; i += THREADS) mine |= kv[i];
      any_valid = __syncthreads_or(mine);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();

  if (warp == MATH_WARPS) {
    // ------------------------------------------------------------ producer warp
    for (int kb = 0; kb < nkb_h; ++kb) {
      const int st = kb % STAGES;
      if (kb >= STAGES) tc::mbar_wait(&sm.empty[st], (uint32_t)(kb / STAGES - 1) & 1u);
      if constexpr (MASKED) {                    // key bias: 0 valid, -inf masked
        for (int e = lane; e < KS * KB; e += 32) {
          const int half = e / KB, key = e - half * KB;
          const int blk = half * nkb_h + kb;
          const int kk = blk * KB + key;
          float bias = -INFINITY;
          if (blk < n_kb && kk < n_keys) {
            bool ok = true;
            if (kk < a.band && a.mask_mode != 0) {        // current-frame keys only
              const bool kv = a.key_valid[(size_t)frame * a.T + band0 + kk] != 0;
              if (a.mask_mode == 1) ok = kv || !any_valid;
              else if (a.mask_mode == 2) ok = kv;
              else ok = any_valid;
            }
            bias = ok ? 0.f : -INFINITY;
          }
          sm.bias[st][half][key] = bias;
        }
        __syncwarp();
      }
      if (lane == 0) {
        uint32_t bytes = 0;
        for (int half = 0; half < KS; ++half) {
          const int blk = half * nkb_h + kb;
          if (blk >= n_kb) continue;
          bytes += 2u * (uint32_t)(min(blk * KB + KB, n_keys) - blk * KB) * (DH * 2);
        }
        tc::mbar_arrive_expect_tx(&sm.full[st], bytes);   // release: bias visible
        for (int half = 0; half < KS; ++half) {
          const int blk = half * nkb_h + kb;
          if (blk >= n_kb) continue;
          const int kk0 = blk * KB, kk1 = min(kk0 + KB, n_keys);
          int kk = kk0;
          while (kk < kk1) {                     // split at segment boundaries (<= 3)
            const int seg = kk >= a.band ? (kk >= 2 * a.band ? 2 : 1) : 0;
            const int end = min(kk1, (seg + 1) * a.band);
            const int stride = seg == 0 ? a.seg_frame_stride[0]
                             : (seg == 1 ? a.seg_frame_stride[1] : a.seg_frame_stride[2]);
            const int fr = stride ? frame : 0;
            const size_t off = ((size_t)(fr * HEADS + h) * a.T + band0 + kk - seg * a.band) * DH;
            const __half* ksrc = (seg == 0 ? a.k[0] : (seg == 1 ? a.k[1] : a.k[2])) + off;
            const __half* vsrc = (seg == 0 ? a.v[0] : (seg == 1 ? a.v[1] : a.v[2])) + off;
            const uint32_t n = (uint32_t)(end - kk) * DH * 2;
            tc::bulk_load(&sm.k[st][half][kk - kk0][0], ksrc, n, &sm.full[st]);
            tc::bulk_load(&sm.v[st][half][kk - kk0][0], vsrc, n, &sm.full[st]);
            kk = end;
          }
        }
      }
    }
    __syncthreads();                              // matches the math warps' merge barrier
    return;
  }

  // -------------------------------------------------------------- math warps
  const int qt = warp & (QT - 1), kh = warp / QT;
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
  SoftmaxState ss;
  ss.m0 = -INFINITY;
  ss.m1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 3; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) { ss.oe[nt][e] = 0.f; ss.oo[nt][e] = 0.f; }

  for (int kb = 0; kb < nkb_h; ++kb) {
    const int st = kb % STAGES;
    tc::mbar_wait(&sm.full[st], (uint32_t)(kb / STAGES) & 1u);
    const int blk = kh * nkb_h + kb;
    if (blk < n_kb) {                                          // warp-uniform
      const int n_valid = min(KB, n_keys - blk * KB);
#pragma unroll 1
      for (int sub = 0; sub < KB / 64; ++sub) {
        const int nv = n_valid - 64 * sub;
        if (nv <= 0) break;
        const __half (*ks)[DH] = sm.k[st][kh] + 64 * sub;
        const __half (*vs)[DH] = sm.v[st][kh] + 64 * sub;
        const float* bs = sm.bias[st][kh] + 64 * sub;
        if (nv >= 64)
          attend_64<MASKED, false>(ss, qa, ks, vs, bs, 64, lane);
        else
          attend_64<MASKED, true>(ss, qa, ks, vs, bs, nv, lane);
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&sm.empty[st]);
  }

  float o[3][4];
#pragma unroll
  for (int nt = 0; nt < 3; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[nt][e] = ss.oe[nt][e] + ss.oo[nt][e];
  float l0 = __shfl_sync(0xffffffffu, o[2][0], lane & ~3);   // row sums live in column 0
  float l1 = __shfl_sync(0xffffffffu, o[2][2], lane & ~3);
  float m0 = ss.m0, m1 = ss.m1;

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
  static bool init = false;
  const int smem = (int)sizeof(Smem);
  if (!init) {
    cudaFuncSetAttribute(attn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  dim3 grid((a.band + QT * 16 - 1) / (QT * 16), HEADS, a.frames * a.groups);
  if (a.mask_mode != 0 && a.key_valid)
    launch_pdl(attn_kernel<true>, grid, dim3(THREADS), smem, s, a);
  else
    launch_pdl(attn_kernel<false>, grid, dim3(THREADS), smem, s, a);
}

}  // namespace dr
