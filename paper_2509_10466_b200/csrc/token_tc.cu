// Token-wise GEMM chains of the DSTT blocks on the 5th-gen tensor cores (tcgen05 + TMEM),
// reference dstt.py:102-150 (MultiHeadAttention projections, _FeedForward, pre-norm
// residual blocks), :185-195 (temporal block), :246-254 (patch embed).
//
// Every GEMM is D[128 x N] (TMEM, fp32) = A[128 x K] (smem, fp16, K-major 128B-swizzled)
// x W^T (smem, fp16, pre-swizzled K-major image bulk-copied once with the block's fp32
// biases / LayerNorm affine), issued by one elected lane of warp 0.  The chain between
// GEMMs never leaves the SM:
//   TOK_EMBED : x = xin We^T + be                                         (dstt.py:246-254)
//   TOK_POST  : x = r + attn Wo^T + bo ; x += W2 gelu(W1 LN2(x) + b1) + b2  (:146-149)
//   then, next block:  [q|k|v] = LN1'(x) Wqkv'^T + b                      (:141-142, :106-117)
//   last block:        tok16 = fp16(x) on the padded Vec2Patch grid, and for every
//                      temporal block j: [k|v]_j = LN1_j(x) Wkv_j^T + b    (:188-190, slot K/V)
//   TOK_SLOTKV: [k|v] = LN1(slot) Wkv^T + b for a memory slot             (:188-190)
//
// Thread layout: 32 warps; warp w reads TMEM lane quarter w % 4 (token row 32*(w%4) + lane,
// the tcgen05.ld restriction) and column group w / 4 (8 of the 64 channels, 16 of the 128
// FFN columns, 24 of the 192 q|k|v columns), so the fp32 epilogues (bias, residual,
// LayerNorm, GELU) run 8 threads per token row.  A CTA owns `tile_rows` = 128, 64 or 32
// tokens (MMA M is always 128; rows past the tile are never read): at batch 1 a 512^2 frame
// (4096 tokens) runs as 128 CTAs of 32 tokens, the idle lane quarters exit after the
// prologue and the active warps synchronise on a named barrier.  The path is latency-bound
// at batch 1 (a chain of 4 dependent GEMMs per tile) and tensor/L2-bound at batch 64.
// TMEM: 256 columns (D1 @0 N=64, D2 @64 N=128, D3 @0 N=64, D4 @64 N=192).
#include <cuda.h>

#include <type_traits>

#include "kernels.h"
#include "tc.cuh"

#define DR_DEV_HOST_INLINE __host__ __device__ __forceinline__

namespace dr {

namespace {

constexpr int M = 128;
constexpr int CG = 8;                        // column groups per token row
constexpr int THREADS = 32 * 4 * CG;         // 1024
constexpr int ATOM_A = M * 128;              // one 128-row x 64-half swizzled K-atom (16 KB)
constexpr int TM_COLS = 256;
constexpr int PRM_BYTES = 704 * 4;           // fp32 params of one block (Prm)

// Smem offsets (bytes, from a 1024-aligned base).  `big` holds the 128 x 256 xin tile
// (EMBED) or the 128 x 128 GELU output (POST).
constexpr int OFF_A = 0;
constexpr int OFF_BIG = ATOM_A;

// cp.async staging of a 128-token tile's inputs, chunk-major so that a warp's 32 rows are
// contiguous: attn [8 chunks][128 rows][16 B], residual [8 chunk pairs][128 rows][32 B]
constexpr int STAGE_ATTN = 8 * 128 * 16, STAGE_BYTES = STAGE_ATTN + 8 * 128 * 32;

struct Ctl {
  float red[2][CG][M];                       // LayerNorm partial sums per column group
  uint64_t w_bar, mma_bar, in_bar;
  uint32_t tmem_base;
};

struct Prm {                                 // float offsets inside a params block
  static constexpr int ln1_w = 0, ln1_b = 64, bqkv = 128, bo = 320, ln2_w = 384, ln2_b = 448,
                       b1 = 512, b2 = 640;
};

// Weight image of one block (bytes): [Wqkv 192 rows][Wo 64][W1 128][W2 2 atoms x 64]
// [fp32 params, PRM_BYTES].
constexpr int IMG_QKV = 0, IMG_O = 192 * 128, IMG_1 = IMG_O + 64 * 128, IMG_2 = IMG_1 + 128 * 128;
constexpr int IMG_PRM = IMG_2 + 2 * 64 * 128;
constexpr int IMG_BYTES = IMG_PRM + PRM_BYTES;
constexpr int IMG_KV = IMG_QKV + 64 * 128;   // k|v rows of Wqkv (128 rows)
constexpr int WE_BYTES = 4 * 64 * 128;       // embed image: We, then be (64 fp32)

DR_DEV uint32_t sw128(int row, int chunk) {  // byte offset of 16-B chunk in a K-atom
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// D[tmem col] (+)= A (atoms of 128 rows) x B (atoms of N rows)^T over `atoms` x 64 K.
DR_DEV void gemm_issue(uint32_t d, uint32_t a_addr, uint32_t b_addr, int n, int atoms,
                       uint64_t* bar) {
  const uint32_t idesc = tc::idesc_f16(M, n);
  const uint64_t ad = tc::sdesc_sw128(a_addr, 0), bd = tc::sdesc_sw128(b_addr, 0);
  for (int kb = 0; kb < atoms; ++kb)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      tc::mma_f16_warp(d, ad + (uint64_t)(kb * (ATOM_A >> 4) + 2 * ks),
                       bd + (uint64_t)(kb * (n * 128 >> 4) + 2 * ks), idesc, (kb | ks) != 0);
  tc::mma_commit_warp(bar);
}

struct Thr {
  int warp, row, cg, n;                      // token row in tile, column group, token index
  int f, tk;                                 // frame, token within frame
  int nact;                                  // threads of the active warps (CG x tile rows)
  uint32_t lane_base;                        // TMEM lane field of this warp's quarter
  bool valid;
};

// Barrier over the active warps only (named barrier 1); the idle lane quarters of a small
// tile exit after the prologue.
DR_DEV void sync_act(const Thr& t) { asm volatile("bar.sync 1, %0;\n" :: "r"(t.nact) : "memory"); }

// Generic-proxy smem writes -> visible to the tensor core; TMEM reads ordered before the
// next MMA; then one barrier.
#define publish(t) do { publish_(t); TT(); } while (0)
DR_DEV void publish_(const Thr& t) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc::fence_before();
  sync_act(t);
  tc::fence_after();
}

#define wait_mma(c, p) do { wait_mma_(c, p); TT(); } while (0)
DR_DEV void wait_mma_(Ctl& ctl, uint32_t& phase) {
  tc::mbar_wait(&ctl.mma_bar, phase);
  phase ^= 1u;
  tc::fence_after();
}

template <int N>
DR_DEV void tmem_row(uint32_t tbase, const Thr& t, int col, float (&v)[N]) {
  static_assert(N == 8 || N == 16, "");
  uint32_t r[N];
  if constexpr (N == 16) tc::tmem_ld16(tbase + t.lane_base + (uint32_t)col, r);
  else tc::tmem_ld8(tbase + t.lane_base + (uint32_t)col, r);
  tc::tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = __uint_as_float(r[i]);
}

DR_DEV uint4 pack8(const float* v, const float* bias) {
  return make_uint4(pack_half2(v[0] + bias[0], v[1] + bias[1]), pack_half2(v[2] + bias[2], v[3] + bias[3]),
                    pack_half2(v[4] + bias[4], v[5] + bias[5]), pack_half2(v[6] + bias[6], v[7] + bias[7]));
}

// Row LayerNorm (eps 1e-5, biased variance) over 64 channels split in CG groups of 8, with
// one CTA barrier: every group publishes its mean and sum of squared deviations, which
// combine exactly (Chan et al.: M2 = sum M2_g + 8 sum (m_g - mu)^2).  Writes this thread's
// 8 normalised values (one fp16 chunk) into the A atom.  (ctl.red is rewritten only after
// a later publish barrier, so one barrier per LayerNorm suffices.)
DR_DEV void layer_norm_to_a(const float (&x)[8], const float* w, const float* b, uint8_t* sa,
                            Ctl& ctl, const Thr& t) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  const float mg = s * 0.125f;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float d = x[i] - mg;
    q += d * d;
  }
  ctl.red[0][t.cg][t.row] = mg;
  ctl.red[1][t.cg][t.row] = q;
  sync_act(t);
  float m[CG], mu = 0.f;
#pragma unroll
  for (int g = 0; g < CG; ++g) {
    m[g] = ctl.red[0][g][t.row];
    mu += m[g];
  }
  mu *= 1.f / CG;
  float var = 0.f, dm = 0.f;
#pragma unroll
  for (int g = 0; g < CG; ++g) {
    var += ctl.red[1][g][t.row];
    const float e = m[g] - mu;
    dm += e * e;
  }
  var = fmaf(8.f, dm, var);
  const float rs = rsqrtf(var * (1.f / 64.f) + 1e-5f);
  const int c = 8 * t.cg;
  float y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = (x[i] - mu) * rs * w[c + i];
  *reinterpret_cast<uint4*>(sa + sw128(t.row, t.cg)) = pack8(y, b + c);
}

// One 8-column chunk (half a head of q, k or v) + bias -> fp16 head-major
// [frame][head][T][16] with the UMMA 32-byte swizzle the attention kernel's bulk copies
// expect (chunk c of token t at c ^ ((t >> 2) & 1)).
DR_DEV void store_chunk(const float (&v)[8], const float* bias, __half* dst, int T, const Thr& t,
                        int h, int c) {
  if (!t.valid) return;
  uint4* r = reinterpret_cast<uint4*>(dst + ((size_t)(t.f * HEADS + h) * T + t.tk) * DH);
  r[c ^ ((t.tk >> 2) & 1)] = pack8(v, bias);
}

// Small tiles (rows < 128) leave lane quarters idle; the FFN1 GELU, the one heavy
// elementwise phase, is spread over all 1024 threads of the CTA: the active warps dump the
// raw FFN1 accumulator to smem (fp32 [rows][128]) and every thread evaluates rows/8
// contiguous columns (bias + GELU -> fp16 into the 128B-swizzled H operand).  Named
// barriers 2 and 3 span the whole CTA (the idle warps join only for this phase).
DR_DEV void gelu_spread(const float* gscr, const float* b1, uint8_t* big, int rows) {
  const int n = rows >> 3;                                 // 4 (32 rows) or 8 (64 rows)
  const int e0 = threadIdx.x * n;
  const int row = e0 >> 7, col = e0 & 127;
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < n) v[i] = gelu_erf(gscr[e0 + i] + b1[col + i]);
  uint8_t* dst = big + (col >> 6) * ATOM_A + sw128(row, (col & 63) >> 3) + ((col & 7) << 1);
  if (n == 8) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]),
                                                pack_half2(v[4], v[5]), pack_half2(v[6], v[7]));
  } else {
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]));
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc::fence_before();
  asm volatile("bar.sync 3, %0;\n" :: "r"(THREADS) : "memory");
  tc::fence_after();
}

// Smem layout after the activation tiles: weight images (1024-aligned), then the fp32
// params blocks (current block, then next block or one per slot-K/V block).
struct WLayout {
  int w_bytes;      // weight images
  int n_nx;         // params blocks after the current one
  DR_DEV_HOST_INLINE int total() const { return w_bytes + (1 + n_nx) * PRM_BYTES; }
};
template <int MODE>
DR_DEV_HOST_INLINE WLayout wlayout(const TokenArgs& a) {
  WLayout l;
  if (MODE == TOK_EMBED) { l.w_bytes = WE_BYTES + 192 * 128; l.n_nx = 1; }
  else if (MODE == TOK_POST) {
    l.w_bytes = (IMG_PRM - IMG_O) + (a.has_next ? 192 * 128 : a.n_kv * 128 * 128);
    l.n_nx = a.has_next ? 1 : a.n_kv;
  } else { l.w_bytes = 128 * 128; l.n_nx = 1; }
  return l;
}

// Diagnostic build only (-DDR_TRACE): thread 0's clock64 at each phase boundary, per CTA
// (scripts/token_trace.py).  Stamps are sequential: entry, prologue, pdl_wait, then one per
// publish / MMA wait, and exit.
#ifdef DR_TRACE
constexpr int TT_SLOTS = 32;
__device__ unsigned long long g_tok_trace[1024 * TT_SLOTS];
#define TT() do { if (threadIdx.x == 0 && blockIdx.x < 1024 && tt_i < TT_SLOTS) {            \
    unsigned long long c_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_) :: "memory");   \
    g_tok_trace[blockIdx.x * TT_SLOTS + tt_i++] = c_; } } while (0)
#else
#define TT() do {} while (0)
#endif

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) token_tc_kernel(
    const __grid_constant__ TokenArgs a, const __grid_constant__ CUtensorMap m_in,
    const __grid_constant__ CUtensorMap m_res, int tma) {
#ifdef DR_TRACE
  int tt_i = 0;
#endif
  TT();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  const int lane = threadIdx.x & 31;
  Thr t;
  t.warp = threadIdx.x >> 5;
  t.row = 32 * (t.warp & 3) + lane;
  t.cg = t.warp >> 2;
  t.lane_base = (uint32_t)(32 * (t.warp & 3)) << 16;
  const int rows = a.tile_rows;                           // 32, 64 or 128 tokens per CTA
  t.nact = CG * rows;
  // 128-token tiles: persistent, the CTA walks tiles blockIdx.x, + gridDim.x, ... with the
  // block weights loaded once (smaller tiles: one tile per CTA, gridDim = tiles)
  const int n_tiles = (a.n_tok + rows - 1) / rows;
  auto set_tile = [&](int tile) {
    t.n = tile * rows + t.row;
    t.valid = t.row < rows && t.n < a.n_tok;
    t.f = t.n / a.T;
    t.tk = t.n - t.f * a.T;
  };
  set_tile(blockIdx.x);
  uint8_t* sa = sm + OFF_A;
  uint8_t* big = sm + OFF_BIG;
  constexpr int big_bytes = MODE == TOK_EMBED ? 4 * ATOM_A : (MODE == TOK_POST ? 2 * ATOM_A : 0);
  uint8_t* sw = big + big_bytes;                          // weight images
  const WLayout L = wlayout<MODE>(a);
  // params: EMBED keeps `be` (64 floats) in the current-params slot
  const float* prm = reinterpret_cast<const float*>(sw + L.w_bytes);
  auto prm_nx = [&](int j) { return prm + (1 + j) * (PRM_BYTES / 4); };
  Ctl& ctl = *reinterpret_cast<Ctl*>(sw + L.total());
  float* gscr = reinterpret_cast<float*>(sw + L.total() + ((sizeof(Ctl) + 15) & ~15));

  pdl_trigger();
  if (threadIdx.x == 0) {
    tc::mbar_init(&ctl.w_bar, 1);
    tc::mbar_init(&ctl.mma_bar, 1);
    tc::mbar_init(&ctl.in_bar, 1);
    tc::fence_barrier_init();
    if (tma) {
      tc::tma_prefetch(&m_in);
      if (MODE != TOK_EMBED) tc::tma_prefetch(&m_res);
    }
  }
  __syncthreads();
  if (t.row >= rows) {                                     // idle lane quarter (small tiles)
    if constexpr (MODE == TOK_POST) {                      // ... joins only the GELU phase
      tc::mbar_wait(&ctl.w_bar, 0);                        // FFN1 bias is in smem
      asm volatile("bar.sync 2, %0;\n" :: "r"(THREADS) : "memory");
      gelu_spread(gscr, prm + Prm::b1, big, rows);
    }
    return;
  }
  TT();

  if (threadIdx.x == 0) {                                  // constant weights: before pdl_wait
    uint8_t* pc = sw + L.w_bytes;
    if constexpr (MODE == TOK_EMBED) {
      tc::mbar_arrive_expect_tx(&ctl.w_bar, (uint32_t)(L.w_bytes + 256 + PRM_BYTES));
      tc::bulk_load(sw, a.we_img, WE_BYTES, &ctl.w_bar);
      tc::bulk_load(sw + WE_BYTES, a.next.img + IMG_QKV, 192 * 128, &ctl.w_bar);
      tc::bulk_load(pc, a.we_img + WE_BYTES, 256, &ctl.w_bar);
      tc::bulk_load(pc + PRM_BYTES, a.next.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
    } else if constexpr (MODE == TOK_POST) {
      tc::mbar_arrive_expect_tx(&ctl.w_bar, (uint32_t)L.total());
      tc::bulk_load(sw, a.cur.img + IMG_O, IMG_PRM - IMG_O, &ctl.w_bar);
      tc::bulk_load(pc, a.cur.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
      uint8_t* d = sw + (IMG_PRM - IMG_O);
      if (a.has_next) {
        tc::bulk_load(d, a.next.img + IMG_QKV, 192 * 128, &ctl.w_bar);
        tc::bulk_load(pc + PRM_BYTES, a.next.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
      } else {
        for (int j = 0; j < a.n_kv; ++j) {
          tc::bulk_load(d + j * 128 * 128, a.kv_w[j].img + IMG_KV, 128 * 128, &ctl.w_bar);
          tc::bulk_load(pc + (1 + j) * PRM_BYTES, a.kv_w[j].img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
        }
      }
    } else {
      tc::mbar_arrive_expect_tx(&ctl.w_bar, (uint32_t)(L.w_bytes + PRM_BYTES));
      tc::bulk_load(sw, a.next.img + IMG_KV, 128 * 128, &ctl.w_bar);
      tc::bulk_load(pc + PRM_BYTES, a.next.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
    }
  }
  // SLOTKV with late_wait reads only the caller-provided slot: it runs alongside its
  // predecessor and waits for it at exit instead (after releasing TMEM)
  if (!(MODE == TOK_SLOTKV && a.late_wait)) pdl_wait();
  // TMEM only after the predecessor grid completed (PDL early trigger: no CTA holds TMEM
  // while it waits on another grid, so allocations cannot deadlock)
  if (t.warp == 0) tc::tmem_alloc<TM_COLS>(&ctl.tmem_base);
  tc::fence_before();
  sync_act(t);
  tc::fence_after();
  const uint32_t tbase = ctl.tmem_base;
  TT();

  uint32_t phase = 0;
  float x[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // residual: 8 of 64 channels
  const int c0 = 8 * t.cg;
  // Inputs of tile `tile` for this thread, started with cp.async (no registers held):
  // EMBED straight into the swizzled xin operand (free once the embed GEMM has read it),
  // POST / SLOTKV into the staging area (the residual, POST also the attention row chunk).
  uint8_t* stage = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gscr) + 1023) & ~uintptr_t(1023));
  const bool staged = rows == 128 && !tma;
  // TMA path (128-token tiles, maps given): thread 0 loads a tile's rows as 128B-swizzled
  // boxes -- EMBED into the xin operand, POST the attention rows (= the out-proj A operand)
  // and the residual's two 32-float boxes into the staging area; completion on in_bar
  auto tma_fetch = [&](int tile) {
    const int r0 = tile * rows;
    if constexpr (MODE == TOK_EMBED) {
      tc::mbar_arrive_expect_tx(&ctl.in_bar, 4u * ATOM_A);
#pragma unroll
      for (int j = 0; j < 4; ++j) tc::tma_load_2d(big + j * ATOM_A, &m_in, &ctl.in_bar, 64 * j, r0);
    } else {
      tc::mbar_arrive_expect_tx(&ctl.in_bar, (MODE == TOK_POST ? 3u : 2u) * ATOM_A);
      if constexpr (MODE == TOK_POST) tc::tma_load_2d(stage, &m_in, &ctl.in_bar, 0, r0);
#pragma unroll
      for (int j = 0; j < 2; ++j) tc::tma_load_2d(stage + (1 + j) * ATOM_A, &m_res, &ctl.in_bar, 32 * j, r0);
    }
  };
  auto prefetch = [&](int tile) {
    const int n = tile * rows + t.row;
    const bool v = t.row < rows && n < a.n_tok;
    const int nn = v ? n : 0;
    if constexpr (MODE == TOK_EMBED) {
      const uint4* src = reinterpret_cast<const uint4*>(a.xin + (size_t)nn * a.kin) + 4 * t.cg;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ch = 4 * t.cg + c;
        cp_async16_zfill(big + (ch >> 3) * ATOM_A + sw128(t.row, ch & 7), src + c, v);
      }
    } else {
      const float4* src = reinterpret_cast<const float4*>(a.resid_in + (size_t)nn * C + c0);
      uint8_t* dr = stage + STAGE_ATTN + (t.cg * 128 + t.row) * 32;
      cp_async16_zfill(dr, src, v);
      cp_async16_zfill(dr + 16, src + 1, v);
      if constexpr (MODE == TOK_POST)
        cp_async16_zfill(stage + (t.cg * 128 + t.row) * 16,
                         reinterpret_cast<const uint4*>(a.attn + (size_t)nn * C) + t.cg, v);
    }
    cp_async_commit();
  };
  if (staged) prefetch(blockIdx.x);
  if (tma && threadIdx.x == 0) tma_fetch(blockIdx.x);
  uint32_t in_phase = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
  set_tile(tile);
  const int next_tile = tile + gridDim.x;
  if (tma) {
    tc::mbar_wait(&ctl.in_bar, in_phase);
    in_phase ^= 1u;
  }
  auto store_resid = [&]() {
    if (!t.valid) return;
    float4* dst = reinterpret_cast<float4*>(a.resid_out + (size_t)t.n * C + c0);
    dst[0] = make_float4(x[0], x[1], x[2], x[3]);
    dst[1] = make_float4(x[4], x[5], x[6], x[7]);
  };
  auto add_d64 = [&](int col, const float* bias) {        // x += D[:, col + c0 .. +8] + bias
    float v[8];
    tmem_row<8>(tbase, t, col + c0, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] += v[i] + bias[c0 + i];
  };

  // ------------------------------------------------------------ stage 0: first GEMM input
  if constexpr (MODE == TOK_EMBED) {
    // xin row: 256 halves = 4 K-atoms of 8 chunks; this thread copies chunks 4cg..4cg+3
    if (staged) {
      cp_async_wait<0>();
    } else if (!tma) {
      const uint4* src = reinterpret_cast<const uint4*>(a.xin + (size_t)t.n * a.kin) + 4 * t.cg;
      uint4 r[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) r[c] = t.valid ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ch = 4 * t.cg + c;
        *reinterpret_cast<uint4*>(big + (ch >> 3) * ATOM_A + sw128(t.row, ch & 7)) = r[c];
      }
    }
    publish(t);
    tc::mbar_wait(&ctl.w_bar, 0);
    tc::fence_after();
    if (t.warp == 0) gemm_issue(tbase, tc::smem_u32(big), tc::smem_u32(sw), 64, 4, &ctl.mma_bar);
    wait_mma(ctl, phase);
    if (staged && next_tile < n_tiles) prefetch(next_tile);   // xin operand read: refill
    if (tma && threadIdx.x == 0 && next_tile < n_tiles) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      tma_fetch(next_tile);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 0.f;
    add_d64(0, prm);
    store_resid();
  } else {
    float4 f0, f1;
    if (tma) {
      const uint8_t* bx = stage + (1 + (t.cg >> 2)) * ATOM_A + t.row * 128;
      const int c = 2 * (t.cg & 3), sw = t.row & 7;
      f0 = *reinterpret_cast<const float4*>(bx + ((c ^ sw) << 4));
      f1 = *reinterpret_cast<const float4*>(bx + (((c + 1) ^ sw) << 4));
    } else if (staged) {
      cp_async_wait<0>();
      TT();
      const float4* st = reinterpret_cast<const float4*>(stage + STAGE_ATTN + (t.cg * 128 + t.row) * 32);
      f0 = st[0];
      f1 = st[1];
      if (MODE == TOK_SLOTKV && next_tile < n_tiles) prefetch(next_tile);
    } else {
      const float4* src = reinterpret_cast<const float4*>(a.resid_in + (size_t)t.n * C + c0);
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      f0 = t.valid ? __ldg(src) : z;
      f1 = t.valid ? __ldg(src + 1) : z;
    }
    x[0] = f0.x; x[1] = f0.y; x[2] = f0.z; x[3] = f0.w;
    x[4] = f1.x; x[5] = f1.y; x[6] = f1.z; x[7] = f1.w;
  }

  if constexpr (MODE == TOK_POST) {
    // ---------------------------------------------------------- out-proj + residual
    if (!tma) {
      uint4 r0;
      if (staged) {
        r0 = *reinterpret_cast<const uint4*>(stage + (t.cg * 128 + t.row) * 16);
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(a.attn + (size_t)t.n * C) + t.cg;
        r0 = t.valid ? __ldg(src) : make_uint4(0, 0, 0, 0);
      }
      *reinterpret_cast<uint4*>(sa + sw128(t.row, t.cg)) = r0;
    }
    if (staged && next_tile < n_tiles) prefetch(next_tile);   // staging consumed: refill
    publish(t);
    tc::mbar_wait(&ctl.w_bar, 0);
    tc::fence_after();
    const uint32_t wo = tc::smem_u32(sw), w1 = wo + (IMG_1 - IMG_O), w2 = wo + (IMG_2 - IMG_O);
    if (t.warp == 0) gemm_issue(tbase, tc::smem_u32(tma ? stage : sa), wo, 64, 1, &ctl.mma_bar);
    wait_mma(ctl, phase);
    if (tma && threadIdx.x == 0 && next_tile < n_tiles) {   // attn operand + residual read
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      tma_fetch(next_tile);
    }
    add_d64(0, prm + Prm::bo);
    TT();
    // ---------------------------------------------------------- LN2 -> FFN1 -> GELU
    layer_norm_to_a(x, prm + Prm::ln2_w, prm + Prm::ln2_b, sa, ctl, t);
    TT();
    publish(t);
    if (t.warp == 0) gemm_issue(tbase + 64, tc::smem_u32(sa), w1, 128, 1, &ctl.mma_bar);
    wait_mma(ctl, phase);
    if (rows == 128) {
      const int col = 16 * t.cg;                           // FFN columns [16cg, 16cg+16)
      float v[16];
      tmem_row<16>(tbase, t, 64 + col, v);
      const float* b1 = prm + Prm::b1 + col;
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = gelu_erf(v[i] + b1[i]);
      const float zero[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint8_t* atom = big + (col >> 6) * ATOM_A;
      const int ch = (col & 63) >> 3;
      *reinterpret_cast<uint4*>(atom + sw128(t.row, ch)) = pack8(v, zero);
      *reinterpret_cast<uint4*>(atom + sw128(t.row, ch + 1)) = pack8(v + 8, zero);
      publish(t);
    } else {
      const int col = 16 * t.cg;
      float v[16];
      tmem_row<16>(tbase, t, 64 + col, v);
      TT();
      float4* g4 = reinterpret_cast<float4*>(gscr + t.row * 128 + col);
#pragma unroll
      for (int i = 0; i < 4; ++i) g4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      tc::fence_before();                                  // D2 reads done before D3 MMAs
      asm volatile("bar.sync 2, %0;\n" :: "r"(THREADS) : "memory");
      TT();
      gelu_spread(gscr, prm + Prm::b1, big, rows);
      TT();
    }
    // ---------------------------------------------------------- FFN2 + residual
    if (t.warp == 0) gemm_issue(tbase, tc::smem_u32(big), w2, 64, 2, &ctl.mma_bar);
    wait_mma(ctl, phase);
    add_d64(0, prm + Prm::b2);
    store_resid();
    TT();
  }

  // ------------------------------------------------------------ LN1' + projections
  const uint32_t wnext = tc::smem_u32(sw) + (MODE == TOK_EMBED ? WE_BYTES
                                            : (MODE == TOK_POST ? IMG_PRM - IMG_O : 0));
  if constexpr (MODE == TOK_SLOTKV) {
    tc::mbar_wait(&ctl.w_bar, 0);
    tc::fence_after();
  }
  const bool qkv = MODE == TOK_EMBED || (MODE == TOK_POST && a.has_next);
  if (qkv) {
    const float* pn = prm_nx(0);
    layer_norm_to_a(x, pn + Prm::ln1_w, pn + Prm::ln1_b, sa, ctl, t);
    TT();
    publish(t);
    if (t.warp == 0) gemm_issue(tbase + 64, tc::smem_u32(sa), wnext, 192, 1, &ctl.mma_bar);
    wait_mma(ctl, phase);
#pragma unroll
    for (int i = 0; i < 3; ++i) {                          // 8-column chunks u = 3cg + i of 24
      const int u = 3 * t.cg + i, p = u >> 1, which = p >> 2, h = p & 3;
      float v[8];
      tmem_row<8>(tbase, t, 64 + 8 * u, v);
      __half* dst = which == 0 ? a.q : (which == 1 ? a.k : a.v);
      store_chunk(v, pn + Prm::bqkv + 8 * u, dst, a.T, t, h, u & 1);
    }
    TT();
  } else {
    // k|v only: SLOTKV (one block) or the last block's slot K/V for every temporal block
    const int n_kv = MODE == TOK_SLOTKV ? 1 : a.n_kv;
    if constexpr (MODE == TOK_POST) {
      if (a.tok16 && t.valid) {                            // fp16 tokens for Vec2Patch
        const int i = t.tk / a.Cc, j = t.tk - i * a.Cc;
        const size_t pos = ((size_t)t.f * (a.R + 2) + i + 1) * (a.Cc + 2) + j + 1;
        const float zero[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        *reinterpret_cast<uint4*>(a.tok16 + pos * C + c0) = pack8(x, zero);
      }
    }
    for (int j = 0; j < n_kv; ++j) {
      const float* pn = prm_nx(j);
      __half* kd = MODE == TOK_SLOTKV ? a.k : a.kv_k[j];
      __half* vd = MODE == TOK_SLOTKV ? a.v : a.kv_v[j];
      layer_norm_to_a(x, pn + Prm::ln1_w, pn + Prm::ln1_b, sa, ctl, t);
      publish(t);
      if (t.warp == 0)
        gemm_issue(tbase + 64, tc::smem_u32(sa), wnext + j * 128 * 128, 128, 1, &ctl.mma_bar);
      wait_mma(ctl, phase);
#pragma unroll
      for (int i = 0; i < 2; ++i) {                        // chunks u = 2cg + i of 16 (k|v)
        const int u = 2 * t.cg + i, p = 4 + (u >> 1), h = p & 3;
        float v[8];
        tmem_row<8>(tbase, t, 64 + 8 * u, v);
        store_chunk(v, pn + Prm::bqkv + 64 + 8 * u, p < 8 ? kd : vd, a.T, t, h, u & 1);
      }
    }
  }
  }  // tiles
  tc::fence_before();
  sync_act(t);
  TT();
  if (t.warp == 0) tc::tmem_dealloc<TM_COLS>(tbase);
  if (MODE == TOK_SLOTKV && a.late_wait) pdl_wait();
}

// generic-proxy A/H writes visible to the tensor core, TMEM reads ordered before the next
// MMA, one CTA barrier
DR_DEV void publish_all() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}

// ---------------------------------------------------------------------------------------
// Small tiles, quarter-spread (default): the tile's rows are placed RQ = ROWS/4 per TMEM
// lane quarter (A row 32q + j), so every quarter -- every SM sub-partition -- owns rows,
// and the 16x256b TMEM load shape (thread t: lanes t/4 and t/4 + 8, columns 2(t%4), +1 of
// each 8-column group; measured, scripts/tmem_layout_probe.cu) hands a warp its quarter's
// rows 4 threads per row.  Epilogues run straight from TMEM on the quarter's warps (row
// statistics: two xor shuffles), with no accumulator round trip through shared memory.
// 16 warps: quarter q = w % 4, column slice w / 4 (64 columns each).
constexpr int QWARPS = 16;

#define DR_TMEM_LD_16x256b_X8(taddr, r)                                                     \
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"  \
               "%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29," \
               "%30,%31}, [%32];\n"                                                         \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),    \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),  \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),           \
                 "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),           \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]),           \
                 "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])            \
               : "r"(taddr))

// 64 accumulator columns of this warp's quarter: v[h][2k + e] = row (t/4 + 8h), column
// col0 + 8k + 2(t%4) + e
template <int NH>
DR_DEV void q_load64(uint32_t tbase, int quarter, int col0, float (&v)[NH][16]) {
  uint32_t r[32];
  DR_TMEM_LD_16x256b_X8(tbase + ((uint32_t)(32 * quarter) << 16) + (uint32_t)col0, r);
  tc::tmem_wait_ld();
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      v[h][2 * k] = __uint_as_float(r[4 * k + 2 * h]);
      v[h][2 * k + 1] = __uint_as_float(r[4 * k + 2 * h + 1]);
    }
}

#define DR_TMEM_LD_16x256b_X4(taddr, r)                                                     \
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"  \
               "%11,%12,%13,%14,%15}, [%16];\n"                                               \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),    \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),  \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                         \
               : "r"(taddr))
// 32 accumulator columns: v[h][2k + e] = row (t/4 + 8h), column col0 + 8k + 2(t%4) + e
template <int NH>
DR_DEV void q_load32(uint32_t tbase, int quarter, int col0, float (&v)[NH][8]) {
  uint32_t r[16];
  DR_TMEM_LD_16x256b_X4(tbase + ((uint32_t)(32 * quarter) << 16) + (uint32_t)col0, r);
  tc::tmem_wait_ld();
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      v[h][2 * k] = __uint_as_float(r[4 * k + 2 * h]);
      v[h][2 * k + 1] = __uint_as_float(r[4 * k + 2 * h + 1]);
    }
}

DR_DEV float quad4_sum(float v) {                // the 4 threads of a row (t%4)
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

// LayerNorm of one row held as 16 values per thread (4 threads per row) -> fp16 into the
// A atom at row arow, chunks k, bytes 4*(t%4)
DR_DEV void q_ln_to_a(const float (&x)[16], const float* w, const float* b, uint8_t* sa,
                      int arow, int cl) {
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) sum += x[i];
  const float mu = quad4_sum(sum) * (1.f / 64.f);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float d = x[i] - mu;
    q += d * d;
  }
  const float rs = rsqrtf(quad4_sum(q) * (1.f / 64.f) + 1e-5f);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = 8 * k + cl;
    const float y0 = (x[2 * k] - mu) * rs * w[c] + b[c];
    const float y1 = (x[2 * k + 1] - mu) * rs * w[c + 1] + b[c + 1];
    *reinterpret_cast<uint32_t*>(sa + sw128(arow, k) + 2 * cl) = pack_half2(y0, y1);
  }
}

template <int MODE, int RQ>
__global__ void __launch_bounds__(32 * QWARPS, 1) token_q_kernel(TokenArgs a) {
#ifdef DR_TRACE
  int tt_i = 0;
#endif
  TT();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  constexpr int ROWS = 4 * RQ, NH = RQ / 8;      // rows per tile, rows per thread (1 or 2)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, slice = warp >> 2;
  const int cl = 2 * (lane & 3);                  // this thread's column pair in each group
  uint8_t* sa = sm + OFF_A;
  uint8_t* big = sm + OFF_BIG;
  constexpr int big_bytes = MODE == TOK_EMBED ? 4 * ATOM_A : (MODE == TOK_POST ? 2 * ATOM_A : 0);
  uint8_t* sw = big + big_bytes;
  const WLayout L = wlayout<MODE>(a);
  const float* prm = reinterpret_cast<const float*>(sw + L.w_bytes);
  auto prm_nx = [&](int j) { return prm + (1 + j) * (PRM_BYTES / 4); };
  Ctl& ctl = *reinterpret_cast<Ctl*>(sw + L.total());

  // this thread's rows (in its quarter): j = lane/4 + 8h -> token n, frame f, token tk
  int nq[NH], fq[NH], tkq[NH];
  bool vq[NH];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = (lane >> 2) + 8 * h;
    nq[h] = blockIdx.x * ROWS + quarter * RQ + j;
    vq[h] = nq[h] < a.n_tok;
    fq[h] = nq[h] / a.T;
    tkq[h] = nq[h] - fq[h] * a.T;
  }
  auto arow = [&](int h) { return 32 * quarter + (lane >> 2) + 8 * h; };

  pdl_trigger();
  if (threadIdx.x == 0) {
    tc::mbar_init(&ctl.w_bar, 1);
    tc::mbar_init(&ctl.mma_bar, 1);
    tc::fence_barrier_init();
    uint8_t* pc = sw + L.w_bytes;                          // constant weights: before pdl_wait
    if constexpr (MODE == TOK_EMBED) {
      tc::mbar_arrive_expect_tx(&ctl.w_bar, (uint32_t)(L.w_bytes + 256 + PRM_BYTES));
      tc::bulk_load(sw, a.we_img, WE_BYTES, &ctl.w_bar);
      tc::bulk_load(sw + WE_BYTES, a.next.img + IMG_QKV, 192 * 128, &ctl.w_bar);
      tc::bulk_load(pc, a.we_img + WE_BYTES, 256, &ctl.w_bar);
      tc::bulk_load(pc + PRM_BYTES, a.next.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
    } else if constexpr (MODE == TOK_POST) {
      tc::mbar_arrive_expect_tx(&ctl.w_bar, (uint32_t)L.total());
      tc::bulk_load(sw, a.cur.img + IMG_O, IMG_PRM - IMG_O, &ctl.w_bar);
      tc::bulk_load(pc, a.cur.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
      uint8_t* d = sw + (IMG_PRM - IMG_O);
      if (a.has_next) {
        tc::bulk_load(d, a.next.img + IMG_QKV, 192 * 128, &ctl.w_bar);
        tc::bulk_load(pc + PRM_BYTES, a.next.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
      } else {
        for (int j = 0; j < a.n_kv; ++j) {
          tc::bulk_load(d + j * 128 * 128, a.kv_w[j].img + IMG_KV, 128 * 128, &ctl.w_bar);
          tc::bulk_load(pc + (1 + j) * PRM_BYTES, a.kv_w[j].img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
        }
      }
    } else {
      tc::mbar_arrive_expect_tx(&ctl.w_bar, (uint32_t)(L.w_bytes + PRM_BYTES));
      tc::bulk_load(sw, a.next.img + IMG_KV, 128 * 128, &ctl.w_bar);
      tc::bulk_load(pc + PRM_BYTES, a.next.img + IMG_PRM, PRM_BYTES, &ctl.w_bar);
    }
  }
  __syncthreads();                              // barriers initialised before any wait
  TT();
  // SLOTKV with late_wait reads only the caller-provided slot: it runs alongside its
  // predecessor and waits for it at exit instead (after releasing TMEM)
  if (!(MODE == TOK_SLOTKV && a.late_wait)) pdl_wait();
  // TMEM only after the predecessor grid completed (see token_tc_kernel)
  if (warp == 0) tc::tmem_alloc<TM_COLS>(&ctl.tmem_base);
  TT();

  uint32_t phase = 0;
  auto mma_wait = [&](bool consumer) {          // consumers wait; everybody flips the phase
    if (consumer) {
      tc::mbar_wait(&ctl.mma_bar, phase);
      tc::fence_after();
    }
    phase ^= 1u;
  };

  // residual stream: warps 0-3 (slice 0) own it, 16 values per row and thread (loaded
  // first: these register loads fly while the GEMM input below is staged)
  float x[NH][16];
  const bool xw = slice == 0;
  if constexpr (MODE != TOK_EMBED) {
    if (xw) {
#pragma unroll
      for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 v = vq[h] ? __ldg(reinterpret_cast<const float2*>(a.resid_in + (size_t)nq[h] * C + 8 * k + cl))
                                 : make_float2(0.f, 0.f);
          x[h][2 * k] = v.x;
          x[h][2 * k + 1] = v.y;
        }
    }
  }
  // ------------------------------------------------------------ first GEMM input
  // A rows of token row r of the tile: 32 * (r / RQ) + r % RQ
  if constexpr (MODE == TOK_EMBED) {
    for (int e = threadIdx.x; e < ROWS * 32; e += 32 * QWARPS) {   // 16-byte chunks of xin
      const int r = e >> 5, ch = e & 31;
      const int n = blockIdx.x * ROWS + r;
      const uint4 v = n < a.n_tok ? __ldg(reinterpret_cast<const uint4*>(a.xin + (size_t)n * a.kin) + ch)
                                  : make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(big + (ch >> 3) * ATOM_A + sw128(32 * (r / RQ) + r % RQ, ch & 7)) = v;
    }
  } else if constexpr (MODE == TOK_POST) {
    for (int e = threadIdx.x; e < ROWS * 8; e += 32 * QWARPS) {    // 16-byte chunks of attn
      const int r = e >> 3, ch = e & 7;
      const int n = blockIdx.x * ROWS + r;
      const uint4 v = n < a.n_tok ? __ldg(reinterpret_cast<const uint4*>(a.attn + (size_t)n * C) + ch)
                                  : make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(sa + sw128(32 * (r / RQ) + r % RQ, ch)) = v;
    }
  }
  tc::mbar_wait(&ctl.w_bar, 0);                 // weights and params in smem
  publish_all();
  TT();
  const uint32_t tbase = ctl.tmem_base;
  auto store_resid = [&]() {
#pragma unroll
    for (int h = 0; h < NH; ++h)
      if (vq[h])
#pragma unroll
        for (int k = 0; k < 8; ++k)
          *reinterpret_cast<float2*>(a.resid_out + (size_t)nq[h] * C + 8 * k + cl) =
              make_float2(x[h][2 * k], x[h][2 * k + 1]);
  };
  auto add_acc = [&](const float* bias) {       // x += D[:, 0..63] + bias (slice-0 warps)
    float d[NH][16];
    q_load64<NH>(tbase, quarter, 0, d);
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        x[h][2 * k] += d[h][2 * k] + bias[8 * k + cl];
        x[h][2 * k + 1] += d[h][2 * k + 1] + bias[8 * k + cl + 1];
      }
  };

  if constexpr (MODE == TOK_EMBED) {
    if (warp == 0) gemm_issue(tbase, tc::smem_u32(big), tc::smem_u32(sw), 64, 4, &ctl.mma_bar);
    mma_wait(xw);
    if (xw) {
#pragma unroll
      for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[h][i] = 0.f;
      add_acc(prm);
      store_resid();
    }
    TT();
  }
  if constexpr (MODE == TOK_POST) {
    const uint32_t wo = tc::smem_u32(sw), w1 = wo + (IMG_1 - IMG_O), w2 = wo + (IMG_2 - IMG_O);
    // ---------------------------------------------------------- out-proj + residual, LN2
    if (warp == 0) gemm_issue(tbase, tc::smem_u32(sa), wo, 64, 1, &ctl.mma_bar);
    mma_wait(xw);
    if (xw) {
      add_acc(prm + Prm::bo);
#pragma unroll
      for (int h = 0; h < NH; ++h) q_ln_to_a(x[h], prm + Prm::ln2_w, prm + Prm::ln2_b, sa, arow(h), cl);
    }
    publish_all();
    TT();
    // ---------------------------------------------------------- FFN1 + GELU (4 slices of 32)
    if (warp == 0) gemm_issue(tbase + 64, tc::smem_u32(sa), w1, 128, 1, &ctl.mma_bar);
    mma_wait(true);
    {
      float d[NH][8];
      q_load32<NH>(tbase, quarter, 64 + 32 * slice, d);
      const float* b1 = prm + Prm::b1 + 32 * slice;
      uint8_t* atom = big + (slice >> 1) * ATOM_A;
#pragma unroll
      for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = 8 * k + cl;
          const uint32_t hv = pack_half2(gelu_erf(d[h][2 * k] + b1[c]), gelu_erf(d[h][2 * k + 1] + b1[c + 1]));
          *reinterpret_cast<uint32_t*>(atom + sw128(arow(h), 4 * (slice & 1) + k) + 2 * cl) = hv;
        }
    }
    publish_all();
    TT();
    // ---------------------------------------------------------- FFN2 + residual
    if (warp == 0) gemm_issue(tbase, tc::smem_u32(big), w2, 64, 2, &ctl.mma_bar);
    mma_wait(xw);
    if (xw) {
      add_acc(prm + Prm::b2);
      store_resid();
    }
    TT();
  }

  // ------------------------------------------------------------ LN1' + projections
  const uint32_t wnext = tc::smem_u32(sw) + (MODE == TOK_EMBED ? WE_BYTES
                                            : (MODE == TOK_POST ? IMG_PRM - IMG_O : 0));
  const bool qkv = MODE == TOK_EMBED || (MODE == TOK_POST && a.has_next);
  if (qkv) {
    const float* pn = prm_nx(0);
    if (xw) {
#pragma unroll
      for (int h = 0; h < NH; ++h) q_ln_to_a(x[h], pn + Prm::ln1_w, pn + Prm::ln1_b, sa, arow(h), cl);
    }
    publish_all();
    TT();
    if (warp == 0) gemm_issue(tbase + 64, tc::smem_u32(sa), wnext, 192, 1, &ctl.mma_bar);
    mma_wait(slice < 3);
    if (slice < 3) {                            // 64 of the 192 q|k|v columns per slice
      float d[NH][16];
      q_load64<NH>(tbase, quarter, 64 + 64 * slice, d);
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        if (!vq[h]) continue;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int u = 8 * slice + k, p = u >> 1, which = p >> 2, hd = p & 3, c = u & 1;
          __half* dst = which == 0 ? a.q : (which == 1 ? a.k : a.v);
          const float* bias = pn + Prm::bqkv + 8 * u + cl;
          uint8_t* row = reinterpret_cast<uint8_t*>(dst + ((size_t)(fq[h] * HEADS + hd) * a.T + tkq[h]) * DH);
          *reinterpret_cast<uint32_t*>(row + 16 * (c ^ ((tkq[h] >> 2) & 1)) + 2 * cl) =
              pack_half2(d[h][2 * k] + bias[0], d[h][2 * k + 1] + bias[1]);
        }
      }
    }
  } else {
    // k|v only: SLOTKV (one block) or the last block's slot K/V for every temporal block
    const int n_kv = MODE == TOK_SLOTKV ? 1 : a.n_kv;
    if constexpr (MODE == TOK_POST) {
      if (a.tok16 && xw) {                      // fp16 tokens for Vec2Patch
#pragma unroll
        for (int h = 0; h < NH; ++h)
          if (vq[h]) {
            const int ti = tkq[h] / a.Cc, tj = tkq[h] - ti * a.Cc;
            const size_t pos = ((size_t)fq[h] * (a.R + 2) + ti + 1) * (a.Cc + 2) + tj + 1;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<uint32_t*>(a.tok16 + pos * C + 8 * k + cl) = pack_half2(x[h][2 * k], x[h][2 * k + 1]);
          }
      }
    }
    for (int j = 0; j < n_kv; ++j) {
      const float* pn = prm_nx(j);
      __half* kd = MODE == TOK_SLOTKV ? a.k : a.kv_k[j];
      __half* vd = MODE == TOK_SLOTKV ? a.v : a.kv_v[j];
      if (xw) {
#pragma unroll
        for (int h = 0; h < NH; ++h) q_ln_to_a(x[h], pn + Prm::ln1_w, pn + Prm::ln1_b, sa, arow(h), cl);
      }
      publish_all();
      if (warp == 0)
        gemm_issue(tbase + 64, tc::smem_u32(sa), wnext + j * 128 * 128, 128, 1, &ctl.mma_bar);
      mma_wait(slice < 2);
      if (slice < 2) {                          // k (slice 0) | v (slice 1), 64 columns each
        float d[NH][16];
        q_load64<NH>(tbase, quarter, 64 + 64 * slice, d);
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          if (!vq[h]) continue;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int u = 8 * slice + k, p = 4 + (u >> 1), hd = p & 3, c = u & 1;
            const float* bias = pn + Prm::bqkv + 64 + 8 * u + cl;
            uint8_t* row = reinterpret_cast<uint8_t*>((p < 8 ? kd : vd) + ((size_t)(fq[h] * HEADS + hd) * a.T + tkq[h]) * DH);
            *reinterpret_cast<uint32_t*>(row + 16 * (c ^ ((tkq[h] >> 2) & 1)) + 2 * cl) =
                pack_half2(d[h][2 * k] + bias[0], d[h][2 * k + 1] + bias[1]);
          }
        }
      }
      // the next block's LN rewrites A only after this MMA completed (consumers waited)
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
    }
  }
  tc::fence_before();
  __syncthreads();
  TT();
  if (warp == 0) tc::tmem_dealloc<TM_COLS>(tbase);
  if (MODE == TOK_SLOTKV && a.late_wait) pdl_wait();
}

template <int MODE>
int smem_bytes(const TokenArgs& a) {
  constexpr int big = MODE == TOK_EMBED ? 4 * ATOM_A : (MODE == TOK_POST ? 2 * ATOM_A : 0);
  // small tiles: the fp32 accumulator dump (rows x (192 + 4)); large: none
  // 128-token tiles: the next tile's attn / residual rows staged by cp.async (token_tc_kernel)
  const int scratch = a.tile_rows < 128 ? a.tile_rows * 196 * 4 : (MODE == TOK_EMBED ? 0 : STAGE_BYTES + 1024);
  return ATOM_A + big + wlayout<MODE>(a).total() + (((int)sizeof(Ctl) + 15) & ~15) + scratch + 1024;
}

}  // namespace

size_t token_tc_block_image_bytes() { return IMG_BYTES; }
size_t token_tc_embed_image_bytes() { return WE_BYTES + 256; }

// Tokens per CTA: the largest of 128 / 64 / 32 that still gives >= one CTA per SM.
int token_tc_tile_rows(int n_tok, int sms) {
  for (int r = 128; r > 32; r >>= 1)
    if ((n_tok + r - 1) / r >= sms) return r;
  return 32;
}

#ifdef DR_TRACE
void tok_trace_snapshot(cudaStream_t s, int n_cta, int mode);
#endif

void launch_token_tc(int mode, const TokenArgs& a_in, cudaStream_t s, const CUtensorMap* m_in,
                     const CUtensorMap* m_res) {
  static unsigned long long init = 0;
  once_per_device(init, [] {
    const int mx = 227 * 1024;
    cudaFuncSetAttribute(token_tc_kernel<TOK_EMBED>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_tc_kernel<TOK_POST>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_tc_kernel<TOK_SLOTKV>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_q_kernel<TOK_EMBED, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_q_kernel<TOK_POST, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_q_kernel<TOK_SLOTKV, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_q_kernel<TOK_EMBED, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_q_kernel<TOK_POST, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(token_q_kernel<TOK_SLOTKV, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  });
  const int sms = device_sms();
  TokenArgs a = a_in;
  if (a.tile_rows != 32 && a.tile_rows != 64 && a.tile_rows != 128)
    a.tile_rows = token_tc_tile_rows(a.n_tok, sms);
  dim3 grid((a.n_tok + a.tile_rows - 1) / a.tile_rows), block(THREADS);
  const dim3 grid_tc(a.tile_rows == 128 ? std::min<unsigned>(grid.x, (unsigned)sms) : grid.x);
  if (a.tile_rows < 128 && a.kin == (mode == TOK_EMBED ? 256 : a.kin)) {
    const int smem = mode == TOK_EMBED ? smem_bytes<TOK_EMBED>(a)
                   : (mode == TOK_POST ? smem_bytes<TOK_POST>(a) : smem_bytes<TOK_SLOTKV>(a));
    const dim3 qb(32 * QWARPS);
    if (a.tile_rows == 32) {
      if (mode == TOK_EMBED) launch_pdl(token_q_kernel<TOK_EMBED, 8>, grid, qb, smem, s, a);
      else if (mode == TOK_POST) launch_pdl(token_q_kernel<TOK_POST, 8>, grid, qb, smem, s, a);
      else launch_pdl(token_q_kernel<TOK_SLOTKV, 8>, grid, qb, smem, s, a);
    } else {
      if (mode == TOK_EMBED) launch_pdl(token_q_kernel<TOK_EMBED, 16>, grid, qb, smem, s, a);
      else if (mode == TOK_POST) launch_pdl(token_q_kernel<TOK_POST, 16>, grid, qb, smem, s, a);
      else launch_pdl(token_q_kernel<TOK_SLOTKV, 16>, grid, qb, smem, s, a);
    }
#ifdef DR_TRACE
    tok_trace_snapshot(s, (int)grid.x, mode);
#endif
    return;
  }
  // TMA inputs: 128-token tiles with the maps this mode needs
  const int tma = a.tile_rows == 128 && m_in && (mode == TOK_EMBED || m_res) && mode != TOK_SLOTKV;
  CUtensorMap zin{}, zres{};
  const CUtensorMap& mi = tma ? *m_in : zin;
  const CUtensorMap& mr = (tma && m_res) ? *m_res : zres;
  switch (mode) {
    case TOK_EMBED:
      launch_pdl(token_tc_kernel<TOK_EMBED>, grid_tc, block, smem_bytes<TOK_EMBED>(a), s, a, mi, mr, tma);
      break;
    case TOK_POST:
      launch_pdl(token_tc_kernel<TOK_POST>, grid_tc, block, smem_bytes<TOK_POST>(a), s, a, mi, mr, tma);
      break;
    default:
      launch_pdl(token_tc_kernel<TOK_SLOTKV>, grid_tc, block, smem_bytes<TOK_SLOTKV>(a), s, a, mi, mr, tma);
      break;
  }
#ifdef DR_TRACE
  tok_trace_snapshot(s, (int)grid.x, mode);
#endif
}

}  // namespace dr

#ifdef DR_TRACE
#include <vector>
namespace dr {
namespace {
std::vector<std::vector<unsigned long long>>& tok_trace_store() {
  static std::vector<std::vector<unsigned long long>> v;
  return v;
}
}  // namespace
void tok_trace_snapshot(cudaStream_t s, int n_cta, int mode) {
  if (tok_trace_store().size() >= 16) return;
  cudaStreamSynchronize(s);
  std::vector<unsigned long long> h((size_t)std::min(n_cta, 1024) * TT_SLOTS + 1);
  cudaMemcpyFromSymbol(h.data(), g_tok_trace, (h.size() - 1) * sizeof(unsigned long long));
  h.back() = (unsigned long long)mode;
  cudaMemsetAsync(nullptr, 0, 0, s);
  tok_trace_store().push_back(std::move(h));
}
}  // namespace dr
extern "C" int dr_debug_tok_trace(int idx, unsigned long long* host, int n) {
  auto& v = dr::tok_trace_store();
  if (idx < 0 || idx >= (int)v.size()) return -1;
  const int k = std::min(n, (int)v[idx].size());
  for (int i = 0; i < k; ++i) host[i] = v[idx][i];
  return k;
}
#endif
