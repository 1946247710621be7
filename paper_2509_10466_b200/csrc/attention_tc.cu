// Fused attention on the 5th-gen tensor cores (tcgen05 + TMEM), head_dim 16.
//
// Reference: scaled_dot_product (dstt.py:89-99) inside MultiHeadAttention (:111-120);
// spatial blocks attend over the whole frame (:146-150), temporal blocks attend a row band
// of queries to cat[band(cur), band(slot0), band(slot1)] (:166-191).
//
// With head_dim 16 the kernel is bound by the softmax exponentials (64 MMA flops per exp),
// and the softmax warps are latency-bound unless each SM sub-partition runs several of them
// (scripts/softmax_microbench2.cu: 2 warps per sub-partition reach ~11 scores/clk/SM, 4
// reach ~15-17).  So one CTA = QT query tiles of 128 rows (QT = 4: 512 queries) x one head x
// one of `ksplit` key parts, and all QT tiles share one K/V stream:
//   warps 0 .. 4QT-1  softmax: tile w/4, TMEM lane quarter w%4 (thread = query row); per
//                     64-key block ONE TMEM load of the 64 scores (S released at once, so
//                     S(j+1) is computed under softmax(j)), block max first (3-input max),
//                     then p = 2^(s*scale - base) (FFMA2, ex2 on MUFU, 1 pair in POLY_EVERY
//                     by a polynomial on the FMA pipe), fp16 pairs stored to P in TMEM
//   warp 4QT          producer: cp.async.bulk of Q tiles and of the 64-key K / V blocks
//                     into a 4-stage ring (mask-aware mode: the key bias row too)
//   warp 4QT+1        MMA issuer, per block and tile: S = Q K^T (M=128 N=64 K=16) and
//                     O += P [V | 1] (4 x M=128 N=32 K=16, A = P from TMEM, B = V MN-major
//                     plus a constant ones block: column 16 of O accumulates the row sum)
// TMEM: 128 columns per tile (S fp32 64 | P fp16 pairs 32 | O 32), 512 for QT = 4.
// The running base is the block max, raised lazily (only when a block max exceeds it by
// > 2^8, exact since numerator and denominator share it): the max is taken before the
// exponentials, so a raise rescales this warp's O rows in TMEM and never redoes a sweep.
// Key parts of a tile form a thread-block cluster; ranks 1.. ship (m, l, o) rows to rank
// 0 through distributed shared memory.  The QKV producer (token_tc.cu) stores q/k/v rows
// with the 16-byte chunk swizzle of the UMMA 32-byte swizzle mode, so bulk copies land as
// valid SWIZZLE_32B operands.
//
// Mask-aware mode (NEW): keys of fully-masked tokens of the current frame get
// -inf; memory-slot keys are always valid; a spatial block whose frame has no valid key
// falls back to unmasked attention (per-block mode resolved on the host, engine.cu).
#include <math.h>

#include <cmath>

#include <algorithm>
#include <cstdlib>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace dr {

namespace {

constexpr int QROWS = 128;
constexpr int KB = 64;                        // keys per block
constexpr int STAGES = 4;
constexpr int MAX_KSPLIT = 4;                 // key parts per query tile (cluster size)
// per tile: S fp32 64 columns | P fp16 pairs 32 | O 32 (16 + row sum)
constexpr uint32_t TM_S = 0, TM_P = 64, TM_O = 96, TM_TILE = 128;
constexpr float RESCALE_SLACK = 8.f;          // log2 units: p <= 2^8 between rescales
#ifndef DR_POLY_EVERY
#define DR_POLY_EVERY 3
#endif
constexpr int POLY_EVERY = DR_POLY_EVERY;     // 1 pair in POLY_EVERY via ex2_poly2 (0 = none)
constexpr int ROW_BYTES = DH * 2;             // 32 B per token row

template <int QT>
constexpr int attn_threads() { return 32 * (4 * QT + 2); }
// resident CTAs per SM: TMEM (QT x 128 columns of 512) and registers
template <int QT>
constexpr int attn_ctas_per_sm() { return 4 / QT; }
template <int QT>
constexpr uint32_t attn_tmem_cols() { return QT * TM_TILE; }

template <int QT, int KSPLIT>
struct __align__(1024) Smem {
  __half q[QT][QROWS][DH];                    // 4 KB per tile, SW32 K-major A operands
  __half k[STAGES][KB][DH];                   // SW32 K-major B operand of S
  __half v[STAGES][2][KB][DH];                // [0] V block, [1] constant ones block
  float bias[STAGES][KB];                     // mask-aware mode only
  uint64_t q_full, kv_full[STAGES], kv_empty[STAGES], o_done;
  uint64_t s_full[QT], s_free[QT], p_full[QT], pv_done[QT];
  // rank 0: (m, l, o[16]) rows of ranks 1.. (bulk-copied in); ranks 1..: staging in [0]
  float mrg[KSPLIT > 1 ? KSPLIT - 1 : 1][QT * QROWS][20];
  uint64_t mrg_full;                          // rank 0: complete_tx of the ranks' bulk copies
  uint32_t tmem_base;
};

// SWIZZLE_32B shared-memory descriptors (layout type 6), version 1.
DR_DEV uint64_t sdesc_sw32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (6ull << 61);
}

// A operand in TMEM (P), B in smem.
DR_DEV void mma_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
      :: "r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}

#define DR_TMEM_LD32(taddr, r)                                                               \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"   \
               "%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29," \
               "%30,%31}, [%32];\n"                                                          \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),     \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),   \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),            \
                 "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),            \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]),            \
                 "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
               : "r"(taddr))
#define DR_TMEM_ST32(taddr, r)                                                               \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,"   \
               "%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,"    \
               "%28,%29,%30,%31,%32};\n"                                                     \
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),         \
                  "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),         \
                  "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),    \
                  "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),    \
                  "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),    \
                  "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory")
DR_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

DR_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
DR_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n"
               ::: "memory");
}
DR_DEV uint32_t map_cluster(uint32_t local_saddr, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local_saddr), "r"(cta));
  return remote;
}
DR_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = tc::smem_u32(bar);
  const long long t0 = clock64();
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    if (clock64() - t0 > (1ll << 32)) __trap();        // protocol bug: fail loudly
  }
}

DR_DEV int seg_of(int kk, int band) { return kk >= band ? (kk >= 2 * band ? 2 : 1) : 0; }


// Diagnostic build only (-DDR_TRACE, build.py --trace): global-timer stamps per CTA taken by
// softmax warp 0, read back by scripts/attn_trace.py.  Slots: 0 entry, 1 TMEM allocated,
// 2 S(0) in registers, 3 softmax loop done, 4 merge done, 5 exit, 6 SM id, 7 key blocks,
// 8 O in registers, 9 DSMEM stores issued, 10 key part.
#ifdef DR_TRACE
constexpr int TRACE_CTAS = 8192;
__device__ unsigned long long g_trace[TRACE_CTAS * 16];
DR_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DR_TRACE_AT(slot, value)                                                             \
  do {                                                                                       \
    const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);        \
    if (warp == 0 && lane == 0 && cta_ < TRACE_CTAS) g_trace[cta_ * 16 + (slot)] = (value);   \
  } while (0)
#define DR_TRACE_T(slot) DR_TRACE_AT(slot, gtimer())
#else
#define DR_TRACE_AT(slot, value) do {} while (0)
#define DR_TRACE_T(slot) do {} while (0)
#endif

DR_DEV void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" :: "r"(id), "r"(n) : "memory");
}

DR_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <bool MASKED, int KSPLIT, int QT>
__global__ void __cluster_dims__(KSPLIT, 1, 1)
__launch_bounds__(attn_threads<QT>(), attn_ctas_per_sm<QT>()) attn_tc_kernel(AttnArgs a) {
  using SmemT = Smem<QT, KSPLIT>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SmemT& sm = *reinterpret_cast<SmemT*>(smem_raw);
  constexpr int NSOFT = 4 * QT;                           // softmax warps
  constexpr int THREADS = attn_threads<QT>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qgroup = blockIdx.x / KSPLIT, h = blockIdx.y;
  const int crank = KSPLIT > 1 ? (int)cluster_rank() : 0;  // key part
  const int frame = blockIdx.z / a.groups, grp = blockIdx.z - frame * a.groups;
  const int band0 = grp * a.band;
  const int q0 = qgroup * QT * QROWS;                     // first query (within the band)
  const int n_keys = a.n_seg * a.band;
  const int n_kb = (n_keys + KB - 1) / KB;
  const int nkb_h = (n_kb + KSPLIT - 1) / KSPLIT;
  const int kb0 = crank * nkb_h;
  const int nb = max(0, min(n_kb, kb0 + nkb_h) - kb0);   // this CTA's key blocks

  DR_TRACE_T(0);
  pdl_trigger();
  // constant smem: zero Q / K / V rings (finite stale tails), ones blocks for row sums
  {
    uint4* z = reinterpret_cast<uint4*>(&sm.q[0][0][0]);
    const int n16 = (int)((sizeof(sm.q) + sizeof(sm.k) + sizeof(sm.v)) / 16);
    for (int i = threadIdx.x; i < n16; i += THREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < STAGES * KB; i += THREADS) {
    const int st = i / KB, key = i - st * KB;
    // element (dim 0, key) of the ones block: chunk 0 sits at chunk (key >> 2) & 1
    sm.v[st][1][key][((key >> 2) & 1) * 8] = __float2half(1.0f);
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.q_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&sm.kv_full[s], 1);
      tc::mbar_init(&sm.kv_empty[s], 1);
    }
    for (int t = 0; t < QT; ++t) {
      tc::mbar_init(&sm.s_full[t], 1);
      tc::mbar_init(&sm.s_free[t], 4);
      tc::mbar_init(&sm.p_full[t], 4);
      tc::mbar_init(&sm.pv_done[t], 1);
    }
    tc::mbar_init(&sm.o_done, 1);
    if (KSPLIT > 1) {
      tc::mbar_init(&sm.mrg_full, 1);
      if (crank == 0)   // armed before the cluster barrier, i.e. before any copy can land
        tc::mbar_arrive_expect_tx(&sm.mrg_full, (uint32_t)((KSPLIT - 1) * QT * QROWS * 80));
    }
    tc::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  // cluster-wide: all ranks' barriers are initialised before any remote arrive (the only
  // cluster barrier; it runs before pdl_wait, overlapping the predecessor kernel)
  if (KSPLIT > 1) cluster_sync();
  pdl_wait();
  // TMEM is allocated only after the predecessor grid completed (PDL early trigger: a CTA
  // never holds TMEM while waiting on another grid, so allocations cannot deadlock)
  if (warp == NSOFT + 1) tc::tmem_alloc<attn_tmem_cols<QT>()>(&sm.tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = sm.tmem_base;
  DR_TRACE_T(1);
#ifdef DR_TRACE
  {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    DR_TRACE_AT(6, smid);
    DR_TRACE_AT(7, nb);
    DR_TRACE_AT(10, crank);
  }
#endif

  int any_valid = 1;
  if constexpr (MASKED) {
    if (a.mask_mode == 1 || a.mask_mode == 3) {
      const uint8_t* kv = a.key_valid + (size_t)frame * a.T;
      int mine = 0;
      for (int i = threadIdx.x; i < a.T; i += THREADS) mine |= kv[i];
      any_valid = __syncthreads_or(mine);
    }
  }

  if (warp == NSOFT) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      const int nq = max(0, min(QT * QROWS, a.band - q0));
      tc::mbar_arrive_expect_tx(&sm.q_full, (uint32_t)nq * ROW_BYTES);
      if (nq > 0)
        tc::bulk_load(&sm.q[0][0][0], a.q + ((size_t)(frame * HEADS + h) * a.T + band0 + q0) * DH,
                      (uint32_t)nq * ROW_BYTES, &sm.q_full);
    }
    for (int j = 0; j < nb; ++j) {
      const int st = j % STAGES;
      if (j >= STAGES) tc::mbar_wait(&sm.kv_empty[st], (uint32_t)(j / STAGES - 1) & 1u);
      const int kk0 = (kb0 + j) * KB, kk1 = min(kk0 + KB, n_keys);
      if constexpr (MASKED) {
        for (int key = lane; key < KB; key += 32) {
          const int kk = kk0 + key;
          float bias = -INFINITY;
          if (kk < kk1) {
            bool ok = true;
            if (kk < a.band && a.mask_mode != 0) {          // current-frame keys only
              const bool kv = a.key_valid[(size_t)frame * a.T + band0 + kk] != 0;
              if (a.mask_mode == 1) ok = kv || !any_valid;
              else if (a.mask_mode == 2) ok = kv;
              else ok = any_valid;
            }
            bias = ok ? 0.f : -INFINITY;
          }
          sm.bias[st][key] = bias;
        }
        __syncwarp();
      }
      if (lane == 0) {
        tc::mbar_arrive_expect_tx(&sm.kv_full[st], 2u * (uint32_t)(kk1 - kk0) * ROW_BYTES);
        int kk = kk0;
        while (kk < kk1) {                                  // split at segment boundaries
          const int seg = seg_of(kk, a.band);
          const int end = min(kk1, (seg + 1) * a.band);
          const int stride = seg == 0 ? a.seg_frame_stride[0]
                           : (seg == 1 ? a.seg_frame_stride[1] : a.seg_frame_stride[2]);
          const size_t off = ((size_t)((stride ? frame : 0) * HEADS + h) * a.T + band0 + kk - seg * a.band) * DH;
          const __half* ks = (seg == 0 ? a.k[0] : (seg == 1 ? a.k[1] : a.k[2])) + off;
          const __half* vs = (seg == 0 ? a.v[0] : (seg == 1 ? a.v[1] : a.v[2])) + off;
          const uint32_t n = (uint32_t)(end - kk) * ROW_BYTES;
          tc::bulk_load(&sm.k[st][kk - kk0][0], ks, n, &sm.kv_full[st]);
          tc::bulk_load(&sm.v[st][0][kk - kk0][0], vs, n, &sm.kv_full[st]);
          kk = end;
        }
      }
    }
  } else if (warp == NSOFT + 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = tc::idesc_f16(128, KB);                   // K-major B
    constexpr uint32_t idesc_pv = tc::idesc_f16(128, 32) | (1u << 16);     // MN-major B
    // Per block j: S_t(j+1) for every tile t once softmax_t released S_t(j) (s_free), then
    // O_t += P_t(j) [V_j | 1] once P_t(j) is written (p_full).  Softmax_t(j+1) waits
    // pv_done_t(j) before it overwrites P_t or rescales O_t.  tcgen05 ops complete in issue
    // order, so S_t(j) ready implies P_t(j-2) V complete: pv_done_t is then in phase j-1 or
    // later, never two phases behind (no parity aliasing).
    tc::mbar_wait(&sm.q_full, 0);
    auto s_mma = [&](int jj) {
      const int st = jj % STAGES;
      tc::mbar_wait(&sm.kv_full[st], (uint32_t)(jj / STAGES) & 1u);
      tc::fence_after();
      const uint64_t kd = sdesc_sw32(tc::smem_u32(&sm.k[st][0][0]), 16, 256);
#pragma unroll
      for (int t = 0; t < QT; ++t) {
        if (jj > 0) {
          tc::mbar_wait(&sm.s_free[t], (uint32_t)(jj - 1) & 1u);
          tc::fence_after();
        }
        const uint64_t qd = sdesc_sw32(tc::smem_u32(&sm.q[t][0][0]), 16, 256);
        tc::mma_f16_warp(tbase + t * TM_TILE + TM_S, qd, kd, idesc_s, 0);
        tc::mma_commit_warp(&sm.s_full[t]);
      }
    };
    if (nb > 0) s_mma(0);
    for (int j = 0; j < nb; ++j) {
      const int st = j % STAGES;
      if (j + 1 < nb) s_mma(j + 1);
      const uint64_t vd = sdesc_sw32(tc::smem_u32(&sm.v[st][0][0][0]), KB * ROW_BYTES, 256);
#pragma unroll
      for (int t = 0; t < QT; ++t) {
        tc::mbar_wait(&sm.p_full[t], (uint32_t)j & 1u);
        tc::fence_after();
        const uint32_t pcol = tbase + t * TM_TILE + TM_P;
#pragma unroll
        for (int kk = 0; kk < KB / 16; ++kk)
          mma_ts_warp(tbase + t * TM_TILE + TM_O, pcol + 8 * kk,
                      vd + (uint64_t)(kk * 16 * ROW_BYTES / 16), idesc_pv, (j | kk) != 0);
        tc::mma_commit_warp(&sm.pv_done[t]);
      }
      tc::mma_commit_warp(&sm.kv_empty[st]);
    }
    // the final O reads have their own single-phase barrier
    if (nb > 0) tc::mma_commit_warp(&sm.o_done);
  } else {
    // ---------------------------------------------------------------- softmax warps
    const int t = warp >> 2;                           // query tile
    const int q = warp & 3;                            // TMEM lanes 32q.. (warp id % 4)
    const int row = t * QROWS + 32 * q + lane;         // query row within the CTA
    const uint32_t lane_base = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(t * TM_TILE);
    const float sl2 = 0.25f * 1.4426950408889634f;     // 1/sqrt(16) * log2(e)
    const uint64_t sl2_2 = f2_pack(sl2, sl2);
    float m = -INFINITY;                               // running base (scaled, log2)
    // Each 64-key block is taken in two 32-column halves (32 score registers live, so 4
    // tiles x 4 warps fit the register file): per half, the max first, then the base (a
    // raise rescales O, and in the second half also the first half's stored P), then the
    // exponentials.
    auto scale_tmem16 = [&](uint32_t col, float f, bool half2) {
      uint32_t v[16];
      tc::tmem_ld16(col, v);
      tc::tmem_wait_ld();
      if (half2) {
        const __half2 f2 = __float2half2_rn(f);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          __half2 x = *reinterpret_cast<__half2*>(&v[c]);
          x = __hmul2(x, f2);
          v[c] = *reinterpret_cast<uint32_t*>(&x);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = __float_as_uint(__uint_as_float(v[c]) * f);
      }
      DR_TMEM_ST16(col, v);
    };
    for (int j = 0; j < nb; ++j) {
      const int st = j % STAGES;
      const int n_valid = min(KB, n_keys - (kb0 + j) * KB);
      tc::mbar_wait(&sm.s_full[t], (uint32_t)j & 1u);
      tc::fence_after();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t r[32];
        DR_TMEM_LD32(lane_base + TM_S + 32 * hh, r);
        tc::tmem_wait_ld();
        if (hh == 1) {
          // S(j) is in registers: hand the S columns back to the MMA warp for S(j+1)
          tc::fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&sm.s_free[t]);
          if (j == 0) DR_TRACE_T(2);
        }
        if (MASKED || n_valid < KB) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            float v = __uint_as_float(r[c]);
            if constexpr (MASKED) v += sm.bias[st][32 * hh + c];
            else v = 32 * hh + c < n_valid ? v : -INFINITY;
            r[c] = __float_as_uint(v);
          }
        }
        float mx[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          mx[i] = fmax3(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]), -INFINITY);
#pragma unroll
        for (int c = 8; c < 32; c += 2)
          mx[(c >> 1) & 3] = fmax3(mx[(c >> 1) & 3], __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
        const float hmax = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3])) * sl2;
        const bool need = hmax > m + RESCALE_SLACK;
        if (__any_sync(0xffffffffu, need)) {
          const float mn = need ? hmax : m;
          const float cfac = (need && m != -INFINITY) ? ex2(m - mn) : (need ? 0.f : 1.f);
          if (j > 0) {
            // O holds the blocks before j once P(j-1) V has landed
            tc::mbar_wait(&sm.pv_done[t], (uint32_t)(j - 1) & 1u);
            tc::fence_after();
            scale_tmem16(lane_base + TM_O, cfac, false);
            scale_tmem16(lane_base + TM_O + 16, cfac, false);
          }
          if (hh == 1) {
            tmem_wait_st();                            // the first half's P stores
            scale_tmem16(lane_base + TM_P, cfac, true);
          }
          m = mn;
        }
        const float base = m == -INFINITY ? 0.f : m;
        const uint64_t nbase2 = f2_pack(-base, -base);
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(r[2 * c]), __uint_as_float(r[2 * c + 1])),
                                     sl2_2, nbase2);
          if (POLY_EVERY > 0 && c % POLY_EVERY == POLY_EVERY - 1) {
            const float2 e = f2_unpack(ex2_poly2(x2));
            pk[c] = pack_half2(e.x, e.y);
          } else {
            const float2 xv = f2_unpack(x2);
            pk[c] = pack_half2(ex2(xv.x), ex2(xv.y));
          }
        }
        // P(j-1) V must have read the P columns before they are overwritten
        if (hh == 0 && j > 0) {
          tc::mbar_wait(&sm.pv_done[t], (uint32_t)(j - 1) & 1u);
          tc::fence_after();
        }
        DR_TMEM_ST16(lane_base + TM_P + 16 * hh, pk);
      }
      tmem_wait_st();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.p_full[t]);
    }
    DR_TRACE_T(3);
    float o[16], l = 0.f;
    if (nb > 0) {
      tc::mbar_wait(&sm.o_done, 0);                   // committed once, after the last P*V
      tc::fence_after();
      uint32_t orr[32];
      DR_TMEM_LD32(lane_base + TM_O, orr);
      tc::tmem_wait_ld();
#pragma unroll
      for (int d = 0; d < 16; ++d) o[d] = __uint_as_float(orr[d]);
      l = __uint_as_float(orr[16]);
    } else {
#pragma unroll
      for (int d = 0; d < 16; ++d) o[d] = 0.f;
    }
    DR_TRACE_T(8);
    // ---- merge the key parts: ranks 1.. stage their (m, l, o) rows in their own shared
    // memory, then one bulk copy (TMA engine, shared::cta -> shared::cluster) moves the
    // whole block into rank 0's mrg buffer with complete_tx on rank 0's mrg_full; rank 0
    // combines.  A final cluster barrier keeps every rank's shared memory alive until
    // rank 0 is done.
    if constexpr (KSPLIT > 1) {
      if (crank != 0) {
        float4* st4 = reinterpret_cast<float4*>(&sm.mrg[0][row][0]);
        st4[0] = make_float4(m, l, 0.f, 0.f);
#pragma unroll
        for (int d = 0; d < 16; d += 4) st4[1 + d / 4] = make_float4(o[d], o[d + 1], o[d + 2], o[d + 3]);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        named_bar_sync(1, 32 * NSOFT);                  // all staged rows written
        if (warp == 0 && lane == 0) {
          const uint32_t dst = map_cluster(tc::smem_u32(&sm.mrg[crank - 1][0][0]), 0);
          const uint32_t bar = map_cluster(tc::smem_u32(&sm.mrg_full), 0);
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes"
              " [%0], [%1], %2, [%3];\n"
              :: "r"(dst), "r"(tc::smem_u32(&sm.mrg[0][0][0])), "r"((uint32_t)(QT * QROWS * 80)),
                 "r"(bar) : "memory");
        }
        DR_TRACE_T(9);
      } else {
        DR_TRACE_T(9);
        mbar_wait_cluster(&sm.mrg_full, 0);
        float M = m;
#pragma unroll
        for (int r1 = 0; r1 < KSPLIT - 1; ++r1) M = fmaxf(M, sm.mrg[r1][row][0]);
        const float b = M == -INFINITY ? 0.f : M;
        const float a0 = ex2(m - b);
        m = b;                                          // o, l are relative to b now
        l *= a0;
#pragma unroll
        for (int d = 0; d < 16; ++d) o[d] *= a0;
#pragma unroll
        for (int r1 = 0; r1 < KSPLIT - 1; ++r1) {
          const float4* mr = reinterpret_cast<const float4*>(&sm.mrg[r1][row][0]);
          const float4 ml = mr[0];
          const float a1 = ex2(ml.x - b);
          l += ml.y * a1;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 o1 = mr[1 + q4];
            o[4 * q4] += o1.x * a1;
            o[4 * q4 + 1] += o1.y * a1;
            o[4 * q4 + 2] += o1.z * a1;
            o[4 * q4 + 3] += o1.w * a1;
          }
        }
      }
    }
    DR_TRACE_T(4);
    if (crank == 0 && q0 + row < a.band) {
      if (a.const_mult > 0) {
        // the zero slots' keys: one key k0 of multiplicity const_mult, value v0.  q row in
        // the SW32 layout: logical 16-byte chunk c at chunk c ^ ((row >> 2) & 1).
        const __half* qr = &sm.q[t][32 * q + lane][0];
        const int sw = (lane >> 2) & 1;
        const float* k0 = a.const_kv + h * DH;
        float dot = 0.f;
#pragma unroll
        for (int d = 0; d < DH; ++d) dot = fmaf(__half2float(qr[(((d >> 3) ^ sw) << 3) | (d & 7)]), __ldg(k0 + d), dot);
        const float s0 = dot * sl2;
        const float ob = m == -INFINITY ? 0.f : m;    // base of o and l
        const float nb2 = fmaxf(ob, s0);
        const float f = ex2(ob - nb2), w0 = (float)a.const_mult * ex2(s0 - nb2);
        const float* v0 = a.const_kv + C + h * DH;
        l = l * f + w0;
#pragma unroll
        for (int d = 0; d < DH; ++d) o[d] = fmaf(o[d], f, w0 * __ldg(v0 + d));
      }
      const float inv = l > 0.f ? 1.f / l : 0.f;
      uint32_t outp[8];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        outp[2 * q4] = pack_half2(o[4 * q4] * inv, o[4 * q4 + 1] * inv);
        outp[2 * q4 + 1] = pack_half2(o[4 * q4 + 2] * inv, o[4 * q4 + 3] * inv);
      }
      uint4* dst = reinterpret_cast<uint4*>(a.out + ((size_t)frame * a.T + band0 + q0 + row) * C + h * DH);
      dst[0] = make_uint4(outp[0], outp[1], outp[2], outp[3]);
      dst[1] = make_uint4(outp[4], outp[5], outp[6], outp[7]);
    }
  }
  tc::fence_before();
  __syncthreads();
  DR_TRACE_T(5);
  if (warp == NSOFT + 1) tc::tmem_dealloc<attn_tmem_cols<QT>()>(tbase);
  if (KSPLIT > 1) cluster_sync();                      // rank 0 has consumed the copies
}
}  // namespace


namespace {
int sm_count() { return device_sms(); }
int tiles_per_band(const AttnArgs& a) { return (a.band + QROWS - 1) / QROWS; }
int cta_groups(const AttnArgs& a, int qt) {
  return (tiles_per_band(a) + qt - 1) / qt * HEADS * a.frames * a.groups;
}

template <bool M, int K, int QT>
void launch_one(const AttnArgs& a, cudaStream_t s) {
  static unsigned long long init = 0;
  constexpr int smem = (int)sizeof(Smem<QT, K>);
  static_assert(smem + 1024 <= 227 * 1024 / attn_ctas_per_sm<QT>(), "attention smem caps residency");
  static_assert(attn_ctas_per_sm<QT>() * attn_tmem_cols<QT>() <= 512, "TMEM over-subscribed");
  once_per_device(init, [&] {
    cudaFuncSetAttribute(attn_tc_kernel<M, K, QT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  const dim3 grid(K * ((tiles_per_band(a) + QT - 1) / QT), HEADS, a.frames * a.groups);
  launch_pdl(attn_tc_kernel<M, K, QT>, grid, dim3(attn_threads<QT>()), smem, s, a);
}
template <bool M, int QT>
void launch_qt(const AttnArgs& a, int k, cudaStream_t s) {
  if constexpr (QT == 1) {                 // 4 CTAs per SM: a 4-way merge buffer does not fit
    if (k == 2) launch_one<M, 2, QT>(a, s);
    else launch_one<M, 1, QT>(a, s);
  } else {
    if (k == 4) launch_one<M, 4, QT>(a, s);
    else if (k == 2) launch_one<M, 2, QT>(a, s);
    else launch_one<M, 1, QT>(a, s);
  }
}

// Modelled makespan (us) of a launch with QT query tiles per CTA and k key parts.
// Measured on B200 (scripts/attn_trace.py): a 4-tile CTA alone on an SM takes 1.19 us per
// 64-key block and ~3.5 us fixed (prologue, first S, O read); a k > 1 merge ~1.5 us.  The
// SM's softmax throughput at c resident tiles relative to 4 (softmax_microbench2): 0.44,
// 0.69, 0.91, 1.  Clusters of 4 fit 142 SMs (GPC packing), of 1-2 all.
double attn_cost(const AttnArgs& a, int qt, int k) {
  static const double eff[5] = {0.0, 0.44, 0.69, 0.91, 1.0};
  const int res = 4 / qt;
  const int sms = k == 4 ? sm_count() * 142 / 148 : sm_count();
  const long n_cta = (long)cta_groups(a, qt) * k;
  const int n_kb = (a.n_seg * a.band + KB - 1) / KB;
  const double blocks = (n_kb + k - 1) / k;
  const long per_sm = (n_cta + sms - 1) / sms;
  // In a single wave, two co-resident CTAs overlap each other's fixed phases (measured at
  // C2: 2 tiles x 4 key parts, 256 CTAs, 5303 frames/s vs 4 x 4, 128 CTAs, 5155)
  const bool one_wave = per_sm <= res;
  auto wave = [&](long c) {                // c CTAs resident on one SM
    const int tiles = (int)std::min<long>(4, c * qt);
    const double fixed = (3.5 + (k > 1 ? 1.5 : 0.0)) / (one_wave ? std::sqrt((double)std::min<long>(c, 2)) : 1.0);
    return fixed + blocks * 1.19 * (tiles / 4.0) / eff[tiles];
  };
  const long full = per_sm / res, rem = per_sm % res;
  return full * wave(res) + (rem ? wave(rem) : 0.0);
}

void attention_plan(const AttnArgs& a, int* qt_out, int* k_out) {
  static const int forced_k = [] {
    const char* e = std::getenv("DR_ATTN_KSPLIT");            // tests / diagnostics
    return e ? std::atoi(e) : 0;
  }();
  static const int forced_qt = [] {
    const char* e = std::getenv("DR_ATTN_QT");
    return e ? std::atoi(e) : 0;
  }();
  const int tpb = tiles_per_band(a);
  int best_qt = 1, best_k = 1;
  double best = 1e30;
  for (int qt = 4; qt >= 1; qt /= 2) {
    if (qt > 1 && tpb < qt) continue;                         // idle tiles
    if (forced_qt && qt != forced_qt) continue;
    for (int k = 1; k <= (qt == 1 ? 2 : MAX_KSPLIT); k *= 2) {
      if (forced_k && k != forced_k) continue;
      const double c = attn_cost(a, qt, k);
      if (c < best * 0.98) { best = c; best_qt = qt; best_k = k; }
    }
  }
  *qt_out = best_qt;
  *k_out = best_k;
}
}  // namespace

int attention_ksplit(const AttnArgs& a) {
  int qt, k;
  attention_plan(a, &qt, &k);
  return k;
}

#ifdef DR_TRACE
void trace_snapshot(cudaStream_t s, int n_cta);
#endif

void launch_attention(const AttnArgs& a_in, cudaStream_t s) {
  AttnArgs a = a_in;
  int qt, k;
  attention_plan(a, &qt, &k);
  const bool masked = a.mask_mode != 0 && a.key_valid;
  if (qt == 4) {
    if (masked) launch_qt<true, 4>(a, k, s); else launch_qt<false, 4>(a, k, s);
  } else if (qt == 2) {
    if (masked) launch_qt<true, 2>(a, k, s); else launch_qt<false, 2>(a, k, s);
  } else {
    if (masked) launch_qt<true, 1>(a, k, s); else launch_qt<false, 1>(a, k, s);
  }
#ifdef DR_TRACE
  trace_snapshot(s, k * ((tiles_per_band(a) + qt - 1) / qt) * HEADS * a.frames * a.groups);
#endif
}

}  // namespace dr

#ifdef DR_TRACE
// Diagnostic build only: launch_attention() snapshots g_trace after each of the first 16
// launches (synchronising the stream); this returns launch `idx`'s per-CTA stamps.
#include <vector>
namespace dr {
std::vector<std::vector<unsigned long long>>& trace_store() {
  static std::vector<std::vector<unsigned long long>> v;
  return v;
}
void trace_snapshot(cudaStream_t s, int n_cta) {
  if (trace_store().size() >= 16) return;
  cudaStreamSynchronize(s);
  std::vector<unsigned long long> h((size_t)std::min(n_cta, TRACE_CTAS) * 16);
  cudaMemcpyFromSymbol(h.data(), g_trace, h.size() * sizeof(unsigned long long));
  trace_store().push_back(std::move(h));
}
}  // namespace dr
extern "C" int dr_debug_attn_trace(int idx, unsigned long long* host, int n) {
  auto& v = dr::trace_store();
  if (idx < 0 || idx >= (int)v.size()) return -1;
  const int k = std::min(n, (int)v[idx].size());
  for (int i = 0; i < k; ++i) host[i] = v[idx][i];
  return k;
}
#endif

// Occupancy diagnostics of the attention kernel (QT = 4, no split): out[0] CTAs per SM,
// out[1] registers per thread, out[2] static smem, out[3] dynamic smem, out[4] last error.
extern "C" int dr_debug_attn_occupancy(int* out) {
  const int smem = (int)sizeof(dr::Smem<4, 1>);
  auto* kern = dr::attn_tc_kernel<false, 1, 4>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kern);
  int n = -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, dr::attn_threads<4>(), smem);
  out[0] = n; out[1] = fa.numRegs; out[2] = (int)fa.sharedSizeBytes; out[3] = smem;
  out[4] = (int)cudaGetLastError();
  return 0;
}
