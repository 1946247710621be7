// Fused attention on the 5th-gen tensor cores (tcgen05 + TMEM), head_dim 16.
//
// Reference: scaled_dot_product (dstt.py:89-99) inside MultiHeadAttention (:111-120);
// spatial blocks attend over the whole frame (:146-150), temporal blocks attend a row band
// of queries to cat[band(cur), band(slot0), band(slot1)] (:166-191).
//
// One CTA = 128 queries x one head x one of `ksplit` key parts (1 or 2, per launch); the
// parts of a tile form a thread-block cluster and merge through distributed shared memory
// into rank 0.  Per 64-key block:
//   MMA warp      S = Q K^T         tcgen05.mma M=128 N=64 K=16, smem x smem -> TMEM
//                 O += P [V | 1]    4 x tcgen05.mma M=128 N=32 K=16, A = P from TMEM, B = V
//                                   (MN-major) plus a constant ones block at the LBO offset,
//                                   so column 16 of O accumulates the softmax row sum
//   4 softmax warps (thread = query row = TMEM lane): ONE tcgen05.ld sweep of its 64
//                 scores, released at once so that S(j+1) is computed under softmax(j):
//                 one FFMA + one ex2 per score (log2 domain; a quarter of them on the FMA
//                 pipe) against the running base, row max tracked on the side, fp16 pack,
//                 tcgen05.st P; no shuffles, no per-key index math on the math warps
//   producer warp cp.async.bulk of the 64-key K and V blocks into a 4-stage ring
// The QKV producer (token_tc.cu) stores q/k/v rows with the 16-byte chunk swizzle of
// the UMMA 32-byte swizzle mode, so bulk copies land as valid SWIZZLE_32B operands.
// The running max is rescaled lazily (only when a row max grows by > 2^8; exact because
// numerator and denominator share the stale max); a rescale reads, scales and writes the
// warp's O rows in TMEM between P*V MMAs.
//
// Mask-aware mode (NEW): keys of fully-masked tokens of the current frame get
// -inf; memory-slot keys are always valid; a spatial block whose frame has no valid key
// falls back to unmasked attention (per-block mode resolved on the host, engine.cu).
#include <math.h>

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
constexpr int THREADS = 192;                  // warp 0 loads, warp 1 MMA, warps 2-5 softmax
// Two CTAs per SM (168 registers per thread).  A third CTA needs <= 96 registers (the
// register file is split per SM sub-partition and a 6-warp CTA puts two warps on two of
// them); measured, the 96-register softmax is ~40% slower per block, which three-way
// interleaving does not recover (0.42 vs 0.37 us per 128x64 block per SM).  The keys of a
// query tile are split over `ksplit` CTAs (chosen per launch, attention_ksplit): 2 at
// batch 1 (256 CTAs for 148 SMs), 1 at large batch (no merge at all).
constexpr int CTAS_PER_SM = 2;
constexpr int MAX_KSPLIT = 2;                 // larger clusters pack poorly into GPCs
// TMEM, 128 columns (up to four CTAs per SM): S fp32 64 cols (single: the softmax warps
// release it as soon as S(j) is in registers, so S(j+1) is computed under softmax(j)),
// P fp16 pairs 32 cols, O 32 cols (16 + row sum)
constexpr uint32_t TM_S = 0, TM_P = 64, TM_O = 96, TM_COLS = 128;
constexpr float RESCALE_SLACK = 8.f;          // log2 units: p <= 2^8 between rescales
#ifndef DR_POLY_EVERY
#define DR_POLY_EVERY 3
#endif
#ifndef DR_ATTN_F32X2
#define DR_ATTN_F32X2 1                        // packed fp32 pairs (FFMA2) in the softmax
#endif
constexpr int POLY_EVERY = DR_POLY_EVERY;     // 1 pair in POLY_EVERY via ex2_poly (0 = none)
constexpr int ROW_BYTES = DH * 2;             // 32 B per token row

struct __align__(1024) Smem {
  __half q[QROWS][DH];                        // 4 KB, SW32 K-major A operand
  __half k[STAGES][KB][DH];                   // SW32 K-major B operand of S
  __half v[STAGES][2][KB][DH];                // [0] V block, [1] constant ones block (+4 KB)
  float bias[STAGES][KB];                     // mask-aware mode only
  uint64_t q_full, kv_full[STAGES], kv_empty[STAGES], s_full, s_free, p_full, pv_done, o_done;
  float mrg[MAX_KSPLIT - 1][QROWS][20];       // rank 0: m, l, o[16] of ranks 1.. (+pad)
  uint64_t mrg_full;                          // rank 0: remote arrivals of the other ranks' rows
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
#define DR_TMEM_ST16(taddr, r)                                                               \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,"   \
               "%10,%11,%12,%13,%14,%15,%16};\n"                                             \
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),         \
                  "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),         \
                  "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory")
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
DR_DEV void st_cluster_v4(uint32_t remote, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};\n"
               :: "r"(remote), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
// arrive on an mbarrier in another CTA of the cluster, releasing this thread's prior
// shared::cluster stores to whoever acquires the phase
DR_DEV void mbar_arrive_remote(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n"
               :: "r"(remote_bar) : "memory");
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
// softmax warp 2, read back by scripts/attn_trace.py.  Slots: 0 entry, 1 after pdl_wait,
// 2 S(0) in registers, 3 softmax loop done, 4 merge done, 5 exit, 6 SM id, 7 blocks,
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
    if (warp == 2 && lane == 0 && cta_ < TRACE_CTAS) g_trace[cta_ * 16 + (slot)] = (value);   \
  } while (0)
#define DR_TRACE_T(slot) DR_TRACE_AT(slot, gtimer())
// cycle accumulators (clock64): 11 softmax wait on S, 12 softmax wait on the S TMEM load,
// 13 softmax loop total, 14 rescale passes, 15 MMA warp wait on P (warp 1)
#define DR_CYC(var) long long var = clock64()
#define DR_ACC(acc, since) acc += clock64() - (since)
#define DR_TRACE_W1(slot, value)                                                             \
  do {                                                                                       \
    const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);        \
    if (warp == 1 && lane == 0 && cta_ < TRACE_CTAS) g_trace[cta_ * 16 + (slot)] = (value);   \
  } while (0)
#else
#define DR_CYC(var) do {} while (0)
#define DR_ACC(acc, since) do {} while (0)
#define DR_TRACE_W1(slot, value) do {} while (0)
#define DR_TRACE_AT(slot, value) do {} while (0)
#define DR_TRACE_T(slot) do {} while (0)
#endif

template <bool MASKED, int KSPLIT>
__global__ void __cluster_dims__(KSPLIT, 1, 1) __launch_bounds__(THREADS, CTAS_PER_SM)
attn_tc_kernel(AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int ksplit = KSPLIT;
  const int qtile = blockIdx.x / ksplit, h = blockIdx.y;
  const int crank = (int)cluster_rank();                  // key part
  const int frame = blockIdx.z / a.groups, grp = blockIdx.z - frame * a.groups;
  const int band0 = grp * a.band;
  const int q0 = qtile * QROWS;
  const int n_keys = a.n_seg * a.band;
  const int n_kb = (n_keys + KB - 1) / KB;
  const int nkb_h = (n_kb + ksplit - 1) / ksplit;
  const int kb0 = crank * nkb_h;
  const int nb = max(0, min(n_kb, kb0 + nkb_h) - kb0);   // this CTA's blocks

  DR_TRACE_T(0);
  pdl_trigger();
  // constant smem: zero Q / K / V rings (finite stale tails), ones blocks for row sums
  {
    uint4* z = reinterpret_cast<uint4*>(&sm.q[0][0]);
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
    tc::mbar_init(&sm.s_full, 1);
    tc::mbar_init(&sm.s_free, 4);
    tc::mbar_init(&sm.p_full, 4);
    tc::mbar_init(&sm.pv_done, 1);
    tc::mbar_init(&sm.o_done, 1);
    if (ksplit > 1) tc::mbar_init(&sm.mrg_full, (ksplit - 1) * QROWS);
    tc::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  // cluster-wide: all ranks' barriers are initialised before any remote arrive (the only
  // cluster barrier; it runs before pdl_wait, overlapping the predecessor kernel)
  if (ksplit > 1) cluster_sync();
  pdl_wait();
  // TMEM is allocated only after the predecessor grid completed (PDL early trigger: a CTA
  // never holds TMEM while waiting on another grid, so allocations cannot deadlock)
  if (warp == 1) tc::tmem_alloc<TM_COLS>(&sm.tmem_base);
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

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      const int nq = max(0, min(QROWS, a.band - q0));
      tc::mbar_arrive_expect_tx(&sm.q_full, (uint32_t)nq * ROW_BYTES);
      if (nq > 0)
        tc::bulk_load(&sm.q[0][0], a.q + ((size_t)(frame * HEADS + h) * a.T + band0 + q0) * DH,
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
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = tc::idesc_f16(128, KB);                   // K-major B
    constexpr uint32_t idesc_pv = tc::idesc_f16(128, 32) | (1u << 16);     // MN-major B
    // Issue order: S(0), then per block j: [s_free(j): S(j) is in the softmax registers]
    // S(j+1) -> s_full; [p_full(j): P(j) written] O += P(j) V_j -> kv_empty, pv_done.
    // Softmax(j+1) waits pv_done(j) before it overwrites P or rescales O.  tcgen05 ops
    // complete in issue order, so S(j) ready implies P(j-2)V complete: pv_done is then in
    // phase j-1 or later, never two phases behind (no parity aliasing).
    const uint64_t qd = sdesc_sw32(tc::smem_u32(&sm.q[0][0]), 16, 256);
    tc::mbar_wait(&sm.q_full, 0);
    auto s_mma = [&](int jj) {
      const int st = jj % STAGES;
      tc::mbar_wait(&sm.kv_full[st], (uint32_t)(jj / STAGES) & 1u);
      tc::fence_after();
      const uint64_t kd = sdesc_sw32(tc::smem_u32(&sm.k[st][0][0]), 16, 256);
      tc::mma_f16_warp(tbase + TM_S, qd, kd, idesc_s, 0);
      tc::mma_commit_warp(&sm.s_full);
    };
    if (nb > 0) s_mma(0);
#ifdef DR_TRACE
    long long cyc_p = 0;
#endif
    for (int j = 0; j < nb; ++j) {
      const int st = j % STAGES;
      if (j + 1 < nb) {
        tc::mbar_wait(&sm.s_free, (uint32_t)j & 1u);
        tc::fence_after();
        s_mma(j + 1);
      }
#ifdef DR_TRACE
      DR_CYC(t_p);
#endif
      tc::mbar_wait(&sm.p_full, (uint32_t)j & 1u);
#ifdef DR_TRACE
      DR_ACC(cyc_p, t_p);
#endif
      tc::fence_after();
      const uint64_t vd = sdesc_sw32(tc::smem_u32(&sm.v[st][0][0][0]), KB * ROW_BYTES, 256);
      const uint32_t pcol = tbase + TM_P;
#pragma unroll
      for (int kk = 0; kk < KB / 16; ++kk)
        mma_ts_warp(tbase + TM_O, pcol + 8 * kk, vd + (uint64_t)(kk * 16 * ROW_BYTES / 16),
                    idesc_pv, (j | kk) != 0);
      tc::mma_commit_warp(&sm.kv_empty[st]);
      tc::mma_commit_warp(&sm.pv_done);
    }
    // the final O read has its own single-phase barrier
    if (nb > 0) tc::mma_commit_warp(&sm.o_done);
#ifdef DR_TRACE
    DR_TRACE_W1(15, (unsigned long long)cyc_p);
#endif
  } else {
    // ---------------------------------------------------------------- softmax warps
    const int q = warp & 3;                            // TMEM lanes 32q.. (warp id % 4)
    const int row = 32 * q + lane;
    const uint32_t lane_base = tbase + ((uint32_t)(32 * q) << 16);
    const float sl2 = 0.25f * 1.4426950408889634f;     // 1/sqrt(16) * log2(e)
    float m = -INFINITY;
    uint32_t r[KB];                                    // this row's scores of S(j)
    // wait for S(jj) and start the TMEM loads; the registers are scoreboarded, the consumer
    // waits on first use
#ifdef DR_TRACE
    long long cyc_s = 0, cyc_ld = 0, n_resc = 0;
    const long long cyc_loop0 = clock64();
#endif
    auto load_s = [&](int jj) {
#ifdef DR_TRACE
      DR_CYC(t_s);
#endif
      tc::mbar_wait(&sm.s_full, (uint32_t)jj & 1u);
#ifdef DR_TRACE
      DR_ACC(cyc_s, t_s);
#endif
      tc::fence_after();
      const uint32_t s_col = lane_base + TM_S;
#pragma unroll
      for (int ch = 0; ch < KB / 32; ++ch) DR_TMEM_LD32(s_col + 32 * ch, (r + 32 * ch));
    };
    if (nb > 0) load_s(0);
    for (int j = 0; j < nb; ++j) {
      const int st = j % STAGES;
      const int n_valid = min(KB, n_keys - (kb0 + j) * KB);
      const uint32_t p_col = lane_base + TM_P;
#ifdef DR_TRACE
      DR_CYC(t_ld);
#endif
      tc::tmem_wait_ld();
#ifdef DR_TRACE
      DR_ACC(cyc_ld, t_ld);
#endif
      // S(j) is in registers: hand the S columns back to the MMA warp for S(j+1)
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.s_free);
      if (j == 0) DR_TRACE_T(2);
      // key bias / tail mask for score column c of this block
      auto adjust = [&](float v, int c) -> float {
        if constexpr (MASKED) return v + sm.bias[st][c];
        return c < n_valid ? v : -INFINITY;
      };
      const bool full = MASKED ? false : n_valid == KB;
      // One pass over S (each score is read from TMEM once): p = 2^(s*scale - base) as fp16
      // pairs into P buffer b while tracking the block's row max; returns the scaled max.
      // (FULL is compile-time so the tail/bias masking is never if-converted into the
      // common full-block sweep)
      auto sweep = [&](float base, auto track, auto full_tag) -> float {
        constexpr bool FULL = decltype(full_tag)::value;
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#if DR_ATTN_F32X2
        const uint64_t sl2_2 = f2_pack(sl2, sl2), nbase2 = f2_pack(-base, -base);
#endif
#pragma unroll
        for (int ch = 0; ch < KB / 32; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int k0 = 32 * ch + 2 * c;
            float s0 = __uint_as_float(r[k0]), s1 = __uint_as_float(r[k0 + 1]);
            if constexpr (!FULL) {
              s0 = adjust(s0, k0);
              s1 = adjust(s1, k0 + 1);
            }
            if constexpr (decltype(track)::value) mx[c & 3] = fmaxf(mx[c & 3], fmaxf(s0, s1));
            // x = s * scale - base for both scores in one packed FFMA2
#if DR_ATTN_F32X2
            const float2 xv = f2_unpack(f2_fma(f2_pack(s0, s1), sl2_2, nbase2));
#else
            const float2 xv = make_float2(fmaf(s0, sl2, -base), fmaf(s1, sl2, -base));
#endif
            // FULL sweeps evaluate POLY_SHARE of the exponentials on the FMA pipe (MUFU
            // offload; the polynomial's 7.5e-5 relative error is below P's fp16 rounding)
            if (FULL && POLY_EVERY > 0 && c % POLY_EVERY == POLY_EVERY - 1) {
#if DR_ATTN_F32X2
              const float2 e = f2_unpack(ex2_poly2(f2_pack(xv.x, xv.y)));
              pk[c] = pack_half2(e.x, e.y);
#else
              pk[c] = pack_half2(ex2_poly(xv.x), ex2_poly(xv.y));
#endif
            } else {
              pk[c] = pack_half2(ex2(xv.x), ex2(xv.y));
            }
          }
          // P(j-1)*V must have read the P columns (first chunk only; a redo sweep finds
          // the phase already complete: P(j)*V is not issued before this warp arrives)
          if (ch == 0 && j > 0) {
            tc::mbar_wait(&sm.pv_done, (uint32_t)(j - 1) & 1u);
            tc::fence_after();
          }
          DR_TMEM_ST16(p_col + 16 * ch, pk);
        }
        return fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2;
      };
      const float base0 = m == -INFINITY ? 0.f : m;
      const float rmax = full ? sweep(base0, std::true_type{}, std::true_type{})
                              : sweep(base0, std::true_type{}, std::false_type{});
      // The running base m may lag the true max by RESCALE_SLACK (p <= 2^8, exact since
      // numerator and denominator share it); past that, rescale O and redo the sweep (rare
      // after the first block).  S(j) is still intact in registers.
      const bool need = rmax > m + RESCALE_SLACK;
      if (__any_sync(0xffffffffu, need)) {
#ifdef DR_TRACE
        ++n_resc;
#endif
        const float mn = need ? rmax : m;
        if (j > 0) {                                   // rescale this warp's O rows
          // P(j-1)*V has landed in O (waited in the sweep above)
          const float cfac = (need && m != -INFINITY) ? ex2(m - mn) : (need ? 0.f : 1.f);
#pragma unroll 1
          for (int h16 = 0; h16 < 2; ++h16) {          // 16 columns at a time (registers)
            uint32_t o[16];
            tc::tmem_ld16(lane_base + TM_O + 16 * h16, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 16; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * cfac);
            DR_TMEM_ST16(lane_base + TM_O + 16 * h16, o);
          }
        }
        m = mn;
        tmem_wait_st();                                // P stores of the optimistic sweep
        sweep(m == -INFINITY ? 0.f : m, std::false_type{}, std::false_type{});  // any block
      }
      // prefetch S(j+1) (normally complete already: issued when S(j) was released) so its
      // TMEM load latency overlaps the completion of the P(j) stores and the hand-off
      if (j + 1 < nb) load_s(j + 1);
      tmem_wait_st();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.p_full);
    }
    DR_TRACE_T(3);
#ifdef DR_TRACE
    DR_TRACE_AT(11, (unsigned long long)cyc_s);
    DR_TRACE_AT(12, (unsigned long long)cyc_ld);
    DR_TRACE_AT(13, (unsigned long long)(clock64() - cyc_loop0));
    DR_TRACE_AT(14, (unsigned long long)n_resc);
#endif
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
    DR_TRACE_AT(10, crank);
    // ---- merge the key parts: ranks 1.. ship their (m, l, o) row into rank 0's shared
    // memory (5 vector DSMEM stores) and arrive on rank 0's mrg_full with release
    // semantics; rank 0 acquires it.  No end-of-kernel cluster barrier: the other ranks may
    // retire at once, rank 0 (the only CTA whose shared memory is accessed remotely)
    // outlives the stores it waits on.
    if (crank != 0) {
      const uint32_t dst = map_cluster(tc::smem_u32(&sm.mrg[crank - 1][row][0]), 0);
      st_cluster_v4(dst, m, l, 0.f, 0.f);
#pragma unroll
      for (int d = 0; d < 16; d += 4) st_cluster_v4(dst + 16 + 4 * d, o[d], o[d + 1], o[d + 2], o[d + 3]);
      mbar_arrive_remote(map_cluster(tc::smem_u32(&sm.mrg_full), 0));
      DR_TRACE_T(9);
    } else if (ksplit > 1) {
      DR_TRACE_T(9);
      mbar_wait_cluster(&sm.mrg_full, 0);
      float M = m;
#pragma unroll
      for (int r1 = 0; r1 < ksplit - 1; ++r1) M = fmaxf(M, sm.mrg[r1][row][0]);
      const float b = M == -INFINITY ? 0.f : M;
      const float a0 = ex2(m - b);
      l *= a0;
#pragma unroll
      for (int d = 0; d < 16; ++d) o[d] *= a0;
#pragma unroll
      for (int r1 = 0; r1 < ksplit - 1; ++r1) {
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
    DR_TRACE_T(4);
    if (crank == 0 && q0 + row < a.band) {
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
  if (warp == 1) tc::tmem_dealloc<TM_COLS>(tbase);
}

}  // namespace

#ifdef DR_TRACE
void trace_snapshot(cudaStream_t s, int n_cta);
#endif

namespace {
int sm_count() { return device_sms(); }
int q_tiles(const AttnArgs& a) { return (a.band + QROWS - 1) / QROWS * HEADS * a.frames * a.groups; }
}  // namespace

// Key split of a launch: the k in 1..MAX_KSPLIT minimising the modelled makespan -- full
// waves of CTAS_PER_SM CTAs per SM, then a tail wave at the concurrency it reaches -- of CTAs
// of ceil(blocks / k) key blocks (+1 block-equivalent of merge for k > 1), with the measured
// per-block time per CTA at 1 / 2 resident CTAs (see CTAS_PER_SM).
int attention_ksplit(const AttnArgs& a) {
  const int sms = sm_count(), tiles = q_tiles(a);
  const int n_kb = (a.n_seg * a.band + KB - 1) / KB;
  const double t_conc[CTAS_PER_SM + 1] = {0.0, 0.575, 0.74};   // us per block per CTA
  static const int forced = [] {
    const char* e = std::getenv("DR_ATTN_KSPLIT");            // tests / diagnostics
    return e ? std::atoi(e) : 0;
  }();
  if (forced >= 1 && forced <= MAX_KSPLIT) return forced;
  int best = 1;
  double best_cost = 1e30;
  for (int k = 1; k <= MAX_KSPLIT; ++k) {
    const long n_cta = (long)tiles * k;
    const long slots = (long)sms * CTAS_PER_SM;
    const double blocks = (n_kb + k - 1) / k + (k > 1 ? 1 : 0);
    const long full = n_cta / slots, rem = n_cta - full * slots;
    const int conc_tail = (int)std::min<long>(CTAS_PER_SM, (rem + sms - 1) / sms);
    const double cost = blocks * (full * t_conc[CTAS_PER_SM] + (rem ? t_conc[conc_tail] : 0.0));
    if (cost < best_cost * 0.98) { best_cost = cost; best = k; }
  }
  return best;
}

void launch_attention(const AttnArgs& a_in, cudaStream_t s) {
  static unsigned long long init = 0;
  // Residency is capped by registers (168 per thread, two CTAs); TMEM (128 columns per CTA)
  // holds four, so tcgen05.alloc never waits; shared memory must not be the cap.
  static_assert(sizeof(Smem) + 1024 <= 227 * 1024 / CTAS_PER_SM, "attention smem caps residency");
  static_assert(CTAS_PER_SM * TM_COLS <= 512, "TMEM over-subscribed");
  const int smem = (int)sizeof(Smem);
  once_per_device(init, [&] {
    cudaFuncSetAttribute(attn_tc_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_tc_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_tc_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_tc_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  AttnArgs a = a_in;
  const int k = (a.ksplit >= 1 && a.ksplit <= MAX_KSPLIT) ? a.ksplit : attention_ksplit(a);
  const dim3 grid(k * ((a.band + QROWS - 1) / QROWS), HEADS, a.frames * a.groups);
  const bool masked = a.mask_mode != 0 && a.key_valid;
  if (k == 2)
    launch_pdl(masked ? attn_tc_kernel<true, 2> : attn_tc_kernel<false, 2>, grid, dim3(THREADS), smem, s, a);
  else
    launch_pdl(masked ? attn_tc_kernel<true, 1> : attn_tc_kernel<false, 1>, grid, dim3(THREADS), smem, s, a);
#ifdef DR_TRACE
  trace_snapshot(s, (int)(grid.x * grid.y * grid.z));
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

// Occupancy diagnostics of the attention kernel: out[0] CTAs per SM, out[1] registers per
// thread, out[2] static smem, out[3] dynamic smem, out[4] last CUDA error.
extern "C" int dr_debug_attn_occupancy(int* out) {
  const int smem = (int)sizeof(dr::Smem);
  cudaFuncSetAttribute(dr::attn_tc_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, dr::attn_tc_kernel<false, 2>);
  int n = -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dr::attn_tc_kernel<false, 2>, dr::THREADS, smem);
  out[0] = n; out[1] = fa.numRegs; out[2] = (int)fa.sharedSizeBytes; out[3] = smem;
  out[4] = (int)cudaGetLastError();
  return 0;
}
