// C-ABI of libdrb200.so: engine lifetime, weight repack, workspace, and the per-frame
// launch sequence (mask stage -> slot K/V -> embed -> S/T blocks -> decoder tail).
// See include/dr_b200.h for the contract and the reference interfaces replaced.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <immintrin.h>

#include "../../include/dr_b200.h"
#include "kernels.h"

using namespace dr;

namespace {

thread_local std::string g_err;

// memcpy with non-temporal (streaming) stores for buffers a DMA engine reads next: lines
// left dirty in the CPU caches make the H2D snoop them (measured on the B200 box, 1 MB:
// 34.9 us after memcpy vs 25.3 us after streaming stores, scripts/pcie_microbench.cu).
void memcpy_nt(uint8_t* dst, const uint8_t* src, size_t n) {
  size_t head = (16 - ((uintptr_t)dst & 15)) & 15;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head; src += head; n -= head;
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

// Evict lines from the CPU caches: a DMA write into lines the CPU holds is slowed by the
// snoops (768 KB D2H: 30.4 us into just-read lines, 19.9 us after clflushopt,
// scripts/pcie_microbench.cu).  Run on the pinned D2H staging buffer after the copy-out,
// off the caller's critical path (WorkPool::run_async).
__attribute__((target("clflushopt"))) void evict_lines(const uint8_t* p, size_t n) {
  const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)63, a1 = (uintptr_t)p + n;
  for (uintptr_t a = a0; a < a1; a += 64) _mm_clflushopt(reinterpret_cast<void*>(a));
  _mm_sfence();
}

// Host staging work (pageable <-> pinned copies, span scatter, cache eviction) split over a
// small pool of worker threads: one core moves ~20 GB/s, so a 512^2 frame's ~1.8 MB of
// staging would otherwise cost ~100 us per call.  The workers spin for ~2 ms after each job
// (a frame loop calls again well within that) and then sleep, so back-to-back calls pay no
// thread wake-up latency.  A job is fn(part, parts); run() has the caller take part 0 and
// waits, run_async() leaves every part to the workers and returns (the next job waits).
class WorkPool {
 public:
  using Fn = std::function<void(int, int)>;
  static WorkPool& get() {
    static WorkPool pool;
    return pool;
  }
  int parts() const { return (int)workers_.size() + 1; }
  void run(Fn fn) {
    if (workers_.empty()) {
      fn(0, 1);
      return;
    }
    std::lock_guard<std::mutex> job(job_mu_);            // one job at a time (engines on
    post(std::move(fn), 1);                              // several host threads)
    fn_(0, parts());
    while (pending_.load(std::memory_order_acquire) != 0) {
    }
  }
  void run_async(Fn fn) {
    if (workers_.empty()) {
      fn(0, 1);
      return;
    }
    std::lock_guard<std::mutex> job(job_mu_);
    post(std::move(fn), 0);
  }
  // wait for an asynchronous job (run_async) to finish, e.g. before freeing its buffer
  void drain() {
    std::lock_guard<std::mutex> job(job_mu_);
    while (pending_.load(std::memory_order_acquire) != 0) {
    }
  }
  ~WorkPool() {
    while (pending_.load(std::memory_order_acquire) != 0) {
    }
    stop_.store(true);
    gen_.fetch_add(1);
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  WorkPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    unsigned cap = 11;                          // DR_POOL_THREADS: worker count override
    if (const char* e = std::getenv("DR_POOL_THREADS")) cap = (unsigned)std::max(0, std::atoi(e));
    const int n = (int)std::min(cap, hw > 1 ? hw - 1 : 0u);
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
  }
  // publish a job once the previous (possibly asynchronous) one has drained; worker w
  // (1..n) takes part w - 1 + first of parts n + first
  void post(Fn fn, int first) {
    while (pending_.load(std::memory_order_acquire) != 0) {
    }
    std::lock_guard<std::mutex> lk(mu_);
    fn_ = std::move(fn);
    first_ = first;
    pending_.store((int)workers_.size(), std::memory_order_relaxed);
    gen_.fetch_add(1, std::memory_order_release);
    cv_.notify_all();
  }
  void loop(int w) {
    uint64_t seen = 0;
    while (true) {
      // spin ~2 ms for the next job, then block on the condition variable
      auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(2)) {
      }
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load()) return;
      fn_(w - 1 + first_, (int)workers_.size() + first_);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex job_mu_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  std::atomic<bool> stop_{false};
  Fn fn_;
  int first_ = 1;
};

// [part * n / parts, (part + 1) * n / parts) rounded to 64-byte boundaries
inline void part_range(size_t n, int part, int parts, size_t* b, size_t* e) {
  const size_t chunk = ((n + parts - 1) / parts + 63) & ~(size_t)63;
  *b = std::min(n, (size_t)part * chunk);
  *e = std::min(n, *b + chunk);
}

// Copy modes: plain; CP_NT streaming stores (the destination is a pinned buffer a DMA
// reads next).
enum CopyMode { CP_PLAIN = 0, CP_NT = 1 };

// Copy split over the pool (small copies inline).
void par_memcpy(void* dst, const void* src, size_t n, int mode = CP_PLAIN) {
  uint8_t* d = static_cast<uint8_t*>(dst);
  const uint8_t* s = static_cast<const uint8_t*>(src);
  auto one = [mode](uint8_t* dd, const uint8_t* ss, size_t nn) {
    if (mode == CP_NT) memcpy_nt(dd, ss, nn);
    else std::memcpy(dd, ss, nn);
  };
  if (n < 192 * 1024) {
    one(d, s, n);
    return;
  }
  WorkPool::get().run([&](int part, int parts) {
    size_t b, e;
    part_range(n, part, parts, &b, &e);
    if (e > b) one(d + b, s + b, e - b);
  });
}

// out[y] = op over v[y - r .. y + r] (clipped to [0, n)), op = min or max, in O(n):
// van Herk / Gil-Werman prefix and suffix runs over blocks of 2r + 1 on an array padded
// with the identity.
template <bool MAX>
void window_reduce(const int* v, int n, int r, int identity, int* out, std::vector<int>& buf) {
  const int k = 2 * r + 1, m = n + 2 * r;
  const int mb = (m + k - 1) / k * k;
  buf.assign(3 * (size_t)mb, identity);
  int* a = buf.data();
  int* g = a + mb;
  int* h = g + mb;
  auto op = [](int x, int y) { return MAX ? std::max(x, y) : std::min(x, y); };
  for (int i = 0; i < n; ++i) a[i + r] = v[i];
  for (int b = 0; b < mb; b += k) {
    g[b] = a[b];
    for (int i = b + 1; i < b + k; ++i) g[i] = op(g[i - 1], a[i]);
    h[b + k - 1] = a[b + k - 1];
    for (int i = b + k - 2; i >= b; --i) h[i] = op(h[i + 1], a[i]);
  }
  for (int y = 0; y < n; ++y) out[y] = op(h[y], g[y + 2 * r]);   // padded window [y, y + 2r]
}

// first / last nonzero byte of a row (-1, -1 if none), 16 bytes at a time
void row_extent(const uint8_t* row, int w, int* first, int* last) {
  int x = 0, f = -1;
  for (; x + 16 <= w && f < 0; x += 16) {
    const int nz = ~_mm_movemask_epi8(_mm_cmpeq_epi8(
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(row + x)), _mm_setzero_si128())) & 0xFFFF;
    if (nz) f = x + __builtin_ctz(nz);
  }
  for (; x < w && f < 0; ++x)
    if (row[x]) f = x;
  *first = f;
  if (f < 0) {
    *last = -1;
    return;
  }
  int l = f, e = w;
  for (; e - 16 >= f; e -= 16) {
    const int nz = ~_mm_movemask_epi8(_mm_cmpeq_epi8(
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(row + e - 16)), _mm_setzero_si128())) & 0xFFFF;
    if (nz) {
      l = e - 16 + 31 - __builtin_clz(nz);
      *last = l;
      return;
    }
  }
  for (int xx = e - 1; xx > f; --xx)
    if (row[xx]) {
      l = xx;
      break;
    }
  *last = l;
}

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(DR_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
  } while (0)

// tcgen05 operand image of W (N x K row-major): K-atoms of 64 halves; atom kb = N rows of
// 128 B, 16-byte chunk c of row n stored at chunk c ^ (n & 7) (the UMMA / TMA 128-byte
// swizzle on a 1024-byte aligned base).
void pack_sw128(const float* W, int N, int K, std::vector<uint8_t>& out) {
  const size_t base = out.size();
  out.resize(base + (size_t)N * K * 2);
  for (int kb = 0; kb < K / 64; ++kb)
    for (int n = 0; n < N; ++n)
      for (int c = 0; c < 8; ++c)
        for (int j = 0; j < 8; ++j) {
          const __half h = __float2half_rn(W[(size_t)n * K + kb * 64 + c * 8 + j]);
          const size_t off = base + ((size_t)kb * N + n) * 128 + ((c ^ (n & 7)) * 16) + j * 2;
          std::memcpy(&out[off], &h, 2);
        }
}

void append_f32(const float* v, int64_t n, std::vector<uint8_t>& out) {
  const size_t o = out.size();
  out.resize(o + (size_t)n * 4);
  std::memcpy(&out[o], v, (size_t)n * 4);
}

struct Blk {
  size_t img;                                               // tcgen05 image byte offset
  bool temporal;
  size_t zkv = 0;            // temporal: fparams offset of the zero slot's [k0 | v0]
};

inline float round_half(float x) { return __half2float(__float2half_rn(x)); }

// scipy.ndimage._filters._gaussian_kernel1d (order 0) in float64, radius int(4 sigma + 0.5)
std::vector<double> feather_taps(double sigma) {
  const int r = sigma > 0 ? (int)(4.0 * sigma + 0.5) : 0;
  std::vector<double> fw(2 * r + 1, 1.0);
  if (r == 0) return fw;
  double sum = 0;
  for (int i = -r; i <= r; ++i) {
    fw[i + r] = std::exp(-0.5 / (sigma * sigma) * (double)i * (double)i);
    sum += fw[i + r];
  }
  for (double& x : fw) x /= sum;
  return fw;
}

// TMA view of an NHWC fp16 raster [frames][H][W][64]: box = 8 channels x 130 px x 4 rows
// (one K-chunk plane of the conv halo; coordinates may be negative / past the edge, the
// out-of-bounds elements are zero-filled = the conv's zero padding).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && fn)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return encode;
}

int make_nhwc_map(CUtensorMap* map, void* base, int frames, int H, int W, int box_rows,
                  int box_px = 130) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (!encode) return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)frames};
  const cuuint64_t strides[3] = {128, (cuuint64_t)W * 128, (cuuint64_t)H * W * 128};
  const cuuint32_t box[4] = {64, (cuuint32_t)box_px, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return DR_OK;
}

// tcgen05 conv weight image, K-major no-swizzle core matrices: [tap][k-chunk][co][8 ci]
// fp16, from a PyTorch Conv2d weight [co_real][c][3][3]; rows co >= co_real are zero.
void pack_conv_tc(const float* w, int c, int co_real, int co_pad, std::vector<uint16_t>& out) {
  for (int tap = 0; tap < 9; ++tap)
    for (int ch = 0; ch < c / 8; ++ch)
      for (int co = 0; co < co_pad; ++co)
        for (int j = 0; j < 8; ++j) {
          const float v = co < co_real ? w[((size_t)co * c + ch * 8 + j) * 9 + tap] : 0.f;
          const __half h = __float2half_rn(v);
          uint16_t u;
          std::memcpy(&u, &h, 2);
          out.push_back(u);
        }
}

}  // namespace

struct dr_engine {
  dr_config cfg{};
  int device = 0;
  int H = 0, W = 0, R = 0, Cc = 0, T = 0, nb = 0, n_temporal = 0, feather_r = 0;
  std::vector<Blk> blk;
  size_t bv2p = 0, bd0 = 0, bd2 = 0;
  float* fparams = nullptr;          // decoder biases (Vec2Patch, decode.0, decode.2)
  uint8_t* timg = nullptr;           // tcgen05 token-GEMM images: We + be, then per block
  double* feather_w = nullptr;
  uint8_t* wtc = nullptr;            // tcgen05 conv weight images: decode.0 then decode.2
  // Decoder: the fused tile pass (dec_fused.cu: 144 taps of the combined 12x12 Vec2Patch o
  // decode.0 kernel, combined bias, border-correction tables) for batches that fill the
  // GPU with tiles, else Vec2Patch -> decode.0 (+ decode.2's E planes) -> decode.2 gather,
  // whose finer grids suit one frame.  DR_DEC_FUSED=1 / 0 forces one (tests, A/B).
  int dec_force = -1;
  // auto: fused from 96 tiles of 128 x 64 px (512^2: batch >= 3; 1024^2: every frame --
  // measured at batch 1: 512^2 unfused ahead by ~4 us, 1024^2 fused ahead by 47 us)
  static constexpr int kFusedMinTiles = 96;
  int frame_tiles() const { return ((H + 127) / 128) * ((W + 63) / 64); }
  int unfused_max_frames() const { return (kFusedMinTiles - 1) / frame_tiles(); }
  bool use_fused(int frames) const {
    return dec_force >= 0 ? dec_force != 0 : frames > unfused_max_frames();
  }
  uint8_t* wcomb = nullptr;
  float* bcomb = nullptr;
  float* dk = nullptr;
  float* part = nullptr;             // dec_fused partial sums (workspace)
  int unf_frames = 0;                // frames the unfused decoder's buffers hold
  float* bord_d0 = nullptr;          // border pixels' combined pre-activation (workspace)
  float* bord_e = nullptr;           // border pixels' decode.2 taps (workspace)
  float* w2f = nullptr;              // decode.2 weights fp32 [27][64]
  CUtensorMap map_tok4{};
  size_t wtc_v2p = 0;                // byte offset of the Vec2Patch image
  size_t te_d2 = 0;                  // decode.2 tap-expanded image (in timg)
  CUtensorMap map_raster{}, map_tok{};
  // 128-token tile inputs of the token chains (2-D, rows of the workspace buffers)
  CUtensorMap map_xin{}, map_attn{}, map_res[2]{};
  bool tok_maps = false;
  // workspace
  int cap = 0;
  void* ws = nullptr;
  uint32_t *bits0 = nullptr, *bits1 = nullptr;
  uint8_t *m1 = nullptr, *tv = nullptr;
  float *alpha = nullptr, *resid[2] = {nullptr, nullptr};
  __half *xin = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *attn = nullptr,
         *tok16 = nullptr, *raster = nullptr, *eplanes = nullptr, *slotkv = nullptr;
  int* flags = nullptr;
  int* flag_acc = nullptr;           // mask stage's per-frame redaction OR + CTA count
  unsigned* flag_cnt = nullptr;      // (self-resetting, zeroed at allocation)
  // host-buffer path (dr_inpaint_u8_host): device frame buffers + 3-slot ring
  uint8_t *h_rgb = nullptr, *h_m0 = nullptr, *h_out = nullptr;   // device
  float* ring[3] = {nullptr, nullptr, nullptr};
  int mem0 = 0, mem1 = 0;                                        // ring index of slots
  bool ring_own[3] = {false, false, false};                      // written by dr_forward
  bool ring_zero[3] = {true, true, true};                        // still the zero slot
  int last_launches = 0;                                         // kernels of the last call
  size_t last_d2h = 0;                                           // host path: D2H bytes
  int stop_after = -1;               // DR_STOP_AFTER=k (diagnostics): launch only k kernels
  uint8_t* pin = nullptr;                                        // pinned staging
  int* flags_mirror = nullptr;       // host path: decode.2's last CTA copies flags here
  cudaEvent_t rgb_ready = nullptr;   // host path: rgb upload done (split uploads), else null
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t rgb_event = nullptr;
  const int4* pack_spans = nullptr;  // host path: per-row [x0, x1, byte offset] (device)
  uint8_t* pack_out = nullptr;       // host path: span-packed composite (device)
  std::vector<int> span_first, span_last;   // host path scratch: masked extent per row
  std::vector<int> span_wmin, span_wmax, span_buf;
  unsigned* d_done = nullptr;        // decode.2 finished-CTA counter (flags mirror)
  // host path CUDA graphs: dr_forward's launch sequence depends only on a few ring / slot
  // K/V cache decisions, so each distinct signature is captured once and replayed
  bool dry = false;                  // dr_forward: host-side decisions only, no launches
  bool capturing = false;            // dr_forward under host-path graph capture
  std::vector<intptr_t> sig;         // dr_forward: what its launches depended on
  struct HostGraph { std::vector<intptr_t> key; cudaGraphExec_t exec; };
  std::vector<HostGraph> hgraphs;
  int host_graph = 1;                // DR_HOST_GRAPH=0: direct launches
  cudaStream_t cap_stream = nullptr; // capture stream (the caller's may be the legacy one)
  cudaEvent_t fork_ev = nullptr;
  // memory-slot K/V projections on a side branch next to the mask stage (DR_SLOTKV_SIDE=0:
  // in line); off while profiling or truncating, where stages must stay serial
  int slotkv_side = 1;
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_fork = nullptr, side_join = nullptr;
  void clear_graphs() {
    for (auto& g : hgraphs) cudaGraphExecDestroy(g.exec);
    hgraphs.clear();
  }
  // optional per-stage CUDA events (dr_profile): ev[0] before the first stage
  static constexpr int kMaxEv = 64;
  int profiling = 0, n_ev = 0;
  cudaEvent_t ev[kMaxEv] = {};
  int ev_kind[kMaxEv] = {};

  void mark(int kind, cudaStream_t s) {
    if (!profiling || n_ev >= kMaxEv) return;
    if (!ev[n_ev]) cudaEventCreate(&ev[n_ev]);
    ev_kind[n_ev] = kind;
    // under stream capture the record becomes an event node of the graph, so a replay
    // re-records every stage boundary (in-graph stage times)
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev[n_ev++], s, cudaEventRecordExternal);
    else cudaEventRecord(ev[n_ev++], s);
  }

  BlockW block_w(int i) const {
    BlockW w;
    w.img = timg + blk[i].img;
    return w;
  }

  size_t frame_px() const { return (size_t)H * W; }
  int sm_count() {
    if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return sms;
  }
  int sms = 0;

  // DR_TOK_ROWS=32|64|128 (tests): force the token kernels' tile size, e.g. the 128-row
  // throughput kernel (and its last-block slot K/V fill) on a batch-1 frame
  int tok_rows = 0;
  int tile_rows(int n_tok) { return tok_rows ? tok_rows : token_tc_tile_rows(n_tok, sm_count()); }
  void launch_tok(int mode, const TokenArgs& a_in, cudaStream_t s) const {
    TokenArgs a = a_in;
    if (tok_rows) a.tile_rows = tok_rows;
    const CUtensorMap* mi = nullptr;
    const CUtensorMap* mr = nullptr;
    if (tok_maps && mode == TOK_EMBED && a.xin == xin) mi = &map_xin;
    if (tok_maps && mode == TOK_POST && a.attn == attn) {
      mi = &map_attn;
      mr = a.resid_in == resid[0] ? &map_res[0] : (a.resid_in == resid[1] ? &map_res[1] : nullptr);
    }
    launch_token_tc(mode, a, s, mi, mr);
  }

  // Slot K/V cache: KV_ENTRIES entries (3 per memory stream: slot0, slot1, new slot),
  // each n_temporal x {K, V} images of [cap][HEADS][T][DH] fp16, keyed by the slot
  // tensor's device pointer, LRU replacement.
  static constexpr int KV_ENTRIES = 6;
  struct KvEntry {
    const float* ptr;
    int frames;
    bool batched;
    uint64_t used;
  };
  KvEntry kvc[KV_ENTRIES] = {};
  uint64_t kv_tick = 0;

  __half* kv_ptr(int entry, int ti, int which) const {         // which: 0 K, 1 V
    return slotkv + ((size_t)(entry * MAX_TEMPORAL + ti) * 2 + which) * ((size_t)cap * T * C);
  }
  void kv_set(int i, const float* p, int frames, bool batched) {
    kvc[i] = {p, frames, batched, ++kv_tick};
  }
  int kv_find(const float* p, int frames, int batched) {
    for (int i = 0; i < KV_ENTRIES; ++i)  // one frame: [1][T][C] and [T][C] are the same
      if (kvc[i].ptr == p && kvc[i].frames == frames &&
          (frames == 1 || kvc[i].batched == (batched != 0))) {
        kvc[i].used = ++kv_tick;
        return i;
      }
    return -1;
  }
  // An entry for pointer p that is not `x0` / `x1`: the one already keyed by p, else LRU.
  int kv_pick(int x0, int x1, const float* p) const {
    for (int i = 0; i < KV_ENTRIES; ++i)
      if (i != x0 && i != x1 && kvc[i].ptr == p) return i;
    int best = -1;
    for (int i = 0; i < KV_ENTRIES; ++i)
      if (i != x0 && i != x1 && (best < 0 || kvc[i].used < kvc[best].used)) best = i;
    return best;
  }

  void free_ws() {
    clear_graphs();
    if (ws) cudaFree(ws);
    ws = nullptr;
    cap = 0;
    for (auto& k : kvc) k = {nullptr, 0, false, 0};
  }

  int ensure(int frames) {
    if (frames <= cap) return DR_OK;
    free_ws();
    const int Ww = (W + 31) / 32;
    const size_t px = frame_px() * frames, tok = (size_t)T * frames;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
    const size_t o_b0 = take((size_t)frames * H * Ww * 4), o_b1 = take((size_t)frames * H * Ww * 4);
    const size_t o_m1 = take(px), o_tv = take(tok), o_alpha = take(px * 4);
    const size_t o_r0 = take(tok * C * 4), o_r1 = take(tok * C * 4);
    const size_t o_xin = take(tok * 4 * cfg.patch * cfg.patch * 2);
    const size_t o_q = take(tok * C * 2), o_k = take(tok * C * 2), o_v = take(tok * C * 2);
    const size_t npad = (size_t)frames * (R + 2) * (Cc + 2);
    const size_t o_at = take(tok * C * 2), o_t16 = take(npad * C * 2);
    // unfused decoder buffers for the batches it runs (<= unf frames), fused ones likewise
    const int unf = use_fused(1) ? 0 : (dec_force == 0 ? frames : std::min(frames, unfused_max_frames()));
    const bool fus = use_fused(frames);
    const size_t upx = frame_px() * unf;
    const size_t o_ras = take(upx * C * 2), o_ep = take(upx * 27 * 2);
    const size_t o_part = take(fus ? dec_part_floats(frames, H, W) * 4 : 0);
    const size_t nbp = (size_t)frames * dec_border_pixels(H, W);
    const size_t o_bd0 = take(fus ? nbp * 64 * 4 : 0), o_be = take(fus ? nbp * 27 * 4 : 0);
    const size_t o_skv = take((size_t)KV_ENTRIES * MAX_TEMPORAL * 2 * tok * C * 2);
    const size_t o_fl = take((size_t)frames * 4), o_fla = take((size_t)frames * 8);
    CUDA_TRY(cudaMalloc(&ws, off));
    uint8_t* b = static_cast<uint8_t*>(ws);
    bits0 = (uint32_t*)(b + o_b0); bits1 = (uint32_t*)(b + o_b1);
    m1 = b + o_m1; tv = b + o_tv; alpha = (float*)(b + o_alpha);
    resid[0] = (float*)(b + o_r0); resid[1] = (float*)(b + o_r1);
    xin = (__half*)(b + o_xin);
    q = (__half*)(b + o_q); k = (__half*)(b + o_k); v = (__half*)(b + o_v);
    attn = (__half*)(b + o_at); tok16 = (__half*)(b + o_t16);
    raster = (__half*)(b + o_ras); eplanes = (__half*)(b + o_ep);
    slotkv = (__half*)(b + o_skv); flags = (int*)(b + o_fl);
    flag_acc = (int*)(b + o_fla); flag_cnt = (unsigned*)(b + o_fla + (size_t)frames * 4);
    CUDA_TRY(cudaMemset(flag_acc, 0, (size_t)frames * 8));
    part = fus ? (float*)(b + o_part) : nullptr;
    bord_d0 = fus ? (float*)(b + o_bd0) : nullptr;
    bord_e = fus ? (float*)(b + o_be) : nullptr;
    unf_frames = unf;
    cap = frames;
    CUDA_TRY(cudaMemset(tok16, 0, npad * C * 2));    // the grid padding stays zero
    if (fus) {
      const int rc = make_token_map4(&map_tok4, tok16, frames, R + 2, Cc + 2);
      if (rc) return rc;
    }
    {   // token-chain inputs: 128-row boxes, 128B-swizzled
      const cuuint64_t n = (cuuint64_t)frames * T;
      int rc = make_rows_map(&map_xin, xin, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4 * cfg.patch * cfg.patch, n, 64);
      if (!rc) rc = make_rows_map(&map_attn, attn, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, C, n, 64);
      if (!rc) rc = make_rows_map(&map_res[0], resid[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, C, n, 32);
      if (!rc) rc = make_rows_map(&map_res[1], resid[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, C, n, 32);
      if (rc) return rc;
      tok_maps = true;
    }
    if (unf > 0) {
      int rc = make_nhwc_map(&map_raster, raster, unf, H, W, conv_tc_rows(64) + 2);
      if (rc) return rc;
      rc = make_token_map(&map_tok, tok16, unf, (R + 2) * (Cc + 2));
      if (rc) return rc;
    }
    return DR_OK;
  }

  // 2-D TMA view of a row-major [n][width] buffer: box = `box` elements (128 B) x 128 rows,
  // 128B swizzle (the UMMA K-major layout)
  int make_rows_map(CUtensorMap* map, void* base, CUtensorMapDataType dt, int width,
                    cuuint64_t n, int box) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode) return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int esz = dt == CU_TENSOR_MAP_DATA_TYPE_FLOAT32 ? 4 : 2;
    const cuuint64_t dims[2] = {(cuuint64_t)width, n};
    const cuuint64_t strides[1] = {(cuuint64_t)width * esz};
    const cuuint32_t bx[2] = {(cuuint32_t)box, 128};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, dt, 2, base, dims, strides, bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled (token rows) failed: " + std::to_string((int)r));
    return DR_OK;
  }

  // 4-D TMA view of the padded token grid [frames][rows][cols][64] for the fused decoder:
  // box = 64 ch x 10 columns x 18 rows (a 16 x 8 token tile with its 1-token halo)
  int make_token_map4(CUtensorMap* map, void* base, int frames, int rows, int cols) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode) return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[4] = {64, (cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)frames};
    const cuuint64_t strides[3] = {128, (cuuint64_t)cols * 128, (cuuint64_t)rows * cols * 128};
    const cuuint32_t box[4] = {64, 10, 18, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled (token tile) failed: " + std::to_string((int)r));
    return DR_OK;
  }


  // TMA view of the padded fp16 token grid [frames][np][64]: box 64 ch x 128 positions.
  int make_token_map(CUtensorMap* map, void* base, int frames, int np) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode) return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {64, (cuuint64_t)np, (cuuint64_t)frames};
    const cuuint64_t strides[2] = {128, (cuuint64_t)np * 128};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(DR_ERR_CUDA, "cuTensorMapEncodeTiled (tokens) failed: " + std::to_string((int)r));
    return DR_OK;
  }
};

namespace {

int check_cfg(const dr_config* c) {
  if (!c) return fail(DR_ERR_CONFIG, "null config");
  if (c->width <= 0 || c->height <= 0 || c->patch <= 0)
    return fail(DR_ERR_CONFIG, "width, height and patch must be positive");
  if (c->width % c->patch || c->height % c->patch)
    return fail(DR_ERR_CONFIG, "width and height must be divisible by patch size");
  if (c->heads <= 0 || c->channels % c->heads)
    return fail(DR_ERR_CONFIG, "channels must be divisible by head count");
  if (c->kernel < c->patch) return fail(DR_ERR_CONFIG, "reconstruction kernel must be >= patch size");
  if (c->temporal_groups <= 0 || (c->height / c->patch) % c->temporal_groups)
    return fail(DR_ERR_CONFIG, "token rows must split evenly into temporal groups");
  if (c->n_blocks <= 0 || c->n_blocks > 16)
    return fail(DR_ERR_CONFIG, "block sequence must hold 1..16 blocks");
  for (int i = 0; i < c->n_blocks; ++i)
    if (c->blocks[i] != 'S' && c->blocks[i] != 'T')
      return fail(DR_ERR_CONFIG, "block sequence must be a nonempty mix of 'S'/'T'");
  if (c->mask_dilate < 0 || c->mask_dilate > 31)
    return fail(DR_ERR_CONFIG, "mask_dilate must be in [0, 31]");
  if (!(c->mask_feather_sigma >= 0.f) || (int)(4.0 * c->mask_feather_sigma + 0.5) > 31)
    return fail(DR_ERR_CONFIG, "mask_feather_sigma must be in [0, 7.8] (feather radius <= 31)");
  // Shapes the sm_100a kernels are specialised for (the reference default network).
  if (c->channels != C || c->heads != HEADS || c->patch != 8 || c->kernel != 10)
    return fail(DR_ERR_CONFIG,
                "B200 kernels support channels=64, heads=4, patch=8, kernel=10 (got channels=" +
                    std::to_string(c->channels) + ", heads=" + std::to_string(c->heads) +
                    ", patch=" + std::to_string(c->patch) + ", kernel=" +
                    std::to_string(c->kernel) + ")");
  // attention K/V rows are swizzled in 8-token groups: every band must start on one
  if (((c->height / c->patch) / c->temporal_groups * (c->width / c->patch)) % 8 != 0)
    return fail(DR_ERR_CONFIG, "B200 kernels need a multiple of 8 tokens per temporal band");
  return DR_OK;
}

}  // namespace

extern "C" {

const char* dr_last_error(void) { return g_err.c_str(); }

int32_t dr_version(void) { return 1; }

int dr_create(const dr_config* cfg, const float* const* weights, const int64_t* numels,
              int32_t n_tensors, int32_t device, dr_engine** out) {
  if (!out) return fail(DR_ERR_CONFIG, "null output pointer");
  *out = nullptr;
  int rc = check_cfg(cfg);
  if (rc) return rc;
  const int nb = cfg->n_blocks;
  const int expect = 2 + 16 * nb + 6;
  if (n_tensors != expect)
    return fail(DR_ERR_CONFIG, "weights file has " + std::to_string(n_tensors) +
                                   " tensors, model needs " + std::to_string(expect));
  const int c = cfg->channels, p = cfg->patch, kk = cfg->kernel;
  std::vector<int64_t> want = {(int64_t)c * 4 * p * p, c};
  for (int i = 0; i < nb; ++i) {
    const int64_t blockn[16] = {c, c, c * c, c, c * c, c, c * c, c, c * c, c, c, c,
                                2 * c * c, 2 * c, 2 * c * c, c};
    want.insert(want.end(), blockn, blockn + 16);
  }
  const int64_t tail[6] = {(int64_t)c * c * kk * kk, c, (int64_t)c * c * 9, c, 3 * c * 9, 3};
  want.insert(want.end(), tail, tail + 6);
  for (int i = 0; i < expect; ++i) {
    if (!weights[i]) return fail(DR_ERR_CONFIG, "null weight tensor " + std::to_string(i));
    if (numels[i] != want[i])
      return fail(DR_ERR_CONFIG, "tensor " + std::to_string(i) + ": " + std::to_string(numels[i]) +
                                     " elements, model needs " + std::to_string(want[i]));
  }
  CUDA_TRY(cudaSetDevice(device));

  dr_engine* e = new dr_engine();
  e->cfg = *cfg;
  e->device = device;
  e->H = cfg->height; e->W = cfg->width;
  e->R = e->H / p; e->Cc = e->W / p; e->T = e->R * e->Cc;
  e->nb = nb;

  std::vector<float> fp;
  std::vector<uint8_t> ti;
  // embed Conv2d(4, C, p, p): W[co][ci*p*p + ky*p + kx] is already the flatten order.
  pack_sw128(weights[0], c, 4 * p * p, ti);                    // We: 64 x 256
  append_f32(weights[1], numels[1], ti);                       // be
  auto addf = [&](int idx) { size_t o = fp.size(); fp.insert(fp.end(), weights[idx], weights[idx] + numels[idx]); return o; };

  for (int i = 0; i < nb; ++i) {
    const int base = 2 + 16 * i;
    Blk b;
    b.temporal = cfg->blocks[i] == 'T';
    std::vector<float> wqkv(weights[base + 2], weights[base + 2] + numels[base + 2]);
    wqkv.insert(wqkv.end(), weights[base + 4], weights[base + 4] + numels[base + 4]);
    wqkv.insert(wqkv.end(), weights[base + 6], weights[base + 6] + numels[base + 6]);
    b.img = ti.size();
    pack_sw128(wqkv.data(), 3 * c, c, ti);
    pack_sw128(weights[base + 8], c, c, ti);
    pack_sw128(weights[base + 12], 2 * c, c, ti);
    pack_sw128(weights[base + 14], c, 2 * c, ti);
    {   // fp32 params: ln1_w ln1_b bq bk bv bo ln2_w ln2_b b1 b2 (token_tc.cu Prm)
      const int order[10] = {0, 1, 3, 5, 7, 9, 10, 11, 13, 15};
      for (int oi : order) append_f32(weights[base + oi], numels[base + oi], ti);
    }
    if (ti.size() - b.img != token_tc_block_image_bytes()) {
      dr_destroy(e);
      return fail(DR_ERR_CONFIG, "internal: token image size mismatch");
    }
    if (b.temporal) {
      // K / V of an all-zero memory slot: LN1(0) = beta (dstt.py:186-190), so every slot
      // token projects to k0 = Wk beta + bk, v0 = Wv beta + bv (fp16 operands, as the
      // slot K/V kernel computes them, rounded to fp16 like its stores)
      b.zkv = fp.size();
      const float* beta = weights[base + 1];
      for (int which = 0; which < 2; ++which) {
        const float* w = weights[base + 4 + 2 * which];
        const float* bias = weights[base + 5 + 2 * which];
        for (int co = 0; co < c; ++co) {
          double acc = 0.0;
          for (int j = 0; j < c; ++j) acc += (double)round_half(beta[j]) * round_half(w[(size_t)co * c + j]);
          fp.push_back(round_half((float)(acc + bias[co])));
        }
      }
      e->n_temporal++;
    }
    if (e->n_temporal > MAX_TEMPORAL) {
      dr_destroy(e);
      return fail(DR_ERR_CONFIG, "B200 engine supports at most 4 temporal blocks");
    }
    e->blk.push_back(b);
  }
  const int tb = 2 + 16 * nb;
  {   // decode.2 tap-expanded weights: row u = 3*(3*ky + kx) + co, K = ci (27 rows of 32)
    std::vector<float> te(32 * (size_t)c, 0.f);
    const float* w2 = weights[tb + 4];                          // [3][c][3][3]
    for (int co = 0; co < 3; ++co)
      for (int ci = 0; ci < c; ++ci)
        for (int tap = 0; tap < 9; ++tap) te[(size_t)(3 * tap + co) * c + ci] = w2[((size_t)co * c + ci) * 9 + tap];
    while (ti.size() % 1024) ti.push_back(0);
    e->te_d2 = ti.size();
    pack_sw128(te.data(), 32, c, ti);
  }
  e->bv2p = addf(tb + 1);
  e->bd0 = addf(tb + 3);
  e->bd2 = addf(tb + 5);
  // tcgen05 weight images, K-major no-swizzle core matrices [tap][k-chunk][co][8 ci] fp16:
  // decode.0 (N=64), then Vec2Patch (100 taps a*10+b, B[n=co][k=ci]
  // = ConvTranspose2d weight[ci][co][a][b]).
  std::vector<uint16_t> tcimg;
  pack_conv_tc(weights[tb + 2], c, c, 64, tcimg);
  e->wtc_v2p = tcimg.size() * 2;
  {
    const float* wt = weights[tb];
    for (int a = 0; a < kk; ++a)
      for (int bb = 0; bb < kk; ++bb)
        for (int ch = 0; ch < c / 8; ++ch)
          for (int co = 0; co < c; ++co)
            for (int j = 0; j < 8; ++j) {
              const int ci = ch * 8 + j;
              const __half h = __float2half_rn(wt[(((size_t)ci * c + co) * kk + a) * kk + bb]);
              uint16_t u;
              std::memcpy(&u, &h, 2);
              tcimg.push_back(u);
            }
  }

  // Fused decoder (dec_fused.cu): Vec2Patch o decode.0 as one transposed convolution,
  // Wcomb[co][ci][u][v] = sum_{dy,dx,c'} Wc[co][c'][dy][dx] Wv[ci][c'][u+dy][v+dx], u, v in
  // [-2, 9], 144 tap images [(u+2)*12 + (v+2)][k-chunk][co][8 ci] fp16; bcomb = bc + sum
  // Wc bv; and the border-correction tables (float64 accumulation).
  if (const char* df = std::getenv("DR_DEC_FUSED")) e->dec_force = std::atoi(df) != 0 ? 1 : 0;
  std::vector<uint16_t> combimg((size_t)144 * 64 * 64);
  std::vector<float> bcomb(64);
  std::vector<float> dkt(dec_border_table_floats(), 0.f);
  {
    const float* wv = weights[tb];                       // [ci][c'][10][10]
    const float* wc = weights[tb + 2];                   // [co][c'][3][3]
    const float* bv = weights[tb + 1];
    const float* bc = weights[tb + 3];
    auto WC = [&](int co, int cp, int ky, int kx) { return (double)wc[((size_t)co * 64 + cp) * 9 + ky * 3 + kx]; };
    auto WV = [&](int ci, int cp, int a, int b) { return (double)wv[(((size_t)ci * 64 + cp) * 10 + a) * 10 + b]; };
    WorkPool::get().run([&](int part, int parts) {
      std::vector<double> acc((size_t)64 * 64);
      for (int tap = part; tap < 144; tap += parts) {
        const int u = tap / 12 - 2, v = tap % 12 - 2;
        std::fill(acc.begin(), acc.end(), 0.0);
        for (int dy = 0; dy < 3; ++dy)
          for (int dx = 0; dx < 3; ++dx) {
            const int ay = u + dy, ax = v + dx;
            if (ay < 0 || ay >= 10 || ax < 0 || ax >= 10) continue;
            for (int co = 0; co < 64; ++co)
              for (int cp = 0; cp < 64; ++cp) {
                const double wcv = WC(co, cp, dy, dx);
                for (int ci = 0; ci < 64; ++ci) acc[(size_t)co * 64 + ci] += wcv * WV(ci, cp, ay, ax);
              }
          }
        uint16_t* dst = combimg.data() + (size_t)tap * 64 * 64;    // [k-chunk][co][8 ci]
        for (int ch = 0; ch < 8; ++ch)
          for (int co = 0; co < 64; ++co)
            for (int j = 0; j < 8; ++j) {
              const __half hv = __float2half_rn((float)acc[(size_t)co * 64 + ch * 8 + j]);
              std::memcpy(dst + ((size_t)ch * 64 + co) * 8 + j, &hv, 2);
            }
      }
    });
    // regroup the tap images into the kernel's stream order: per phase quad and token
    // offset one [k-chunk 8][4 phases x 64 co][8 ci] block (kernels.h dec_quad_*)
    {
      std::vector<uint16_t> grp(combimg.size());
      size_t blk = 0;
      for (int g = 0; g < 16; ++g) {
        const int gy = g >> 2, gx = g & 3;
        for (int ia = 0; ia < dec_quad_noff(gy); ++ia)
          for (int ib = 0; ib < dec_quad_noff(gx); ++ib, ++blk) {
            const int du = dec_quad_off(gy, ia), dv = dec_quad_off(gx, ib);
            uint16_t* dst = grp.data() + blk * 256 * 64;
            for (int q = 0; q < 4; ++q) {
              const int py = 2 * gy + (q >> 1), px = 2 * gx + (q & 1);
              const int tap = (py - 8 * du + 2) * 12 + (px - 8 * dv + 2);
              const uint16_t* src = combimg.data() + (size_t)tap * 64 * 64;
              for (int ch = 0; ch < 8; ++ch)
                std::memcpy(dst + ((size_t)ch * 256 + q * 64) * 8, src + (size_t)ch * 64 * 8, 64 * 8 * 2);
            }
          }
      }
      combimg.swap(grp);
    }
    for (int co = 0; co < 64; ++co) {
      double b = bc[co];
      for (int cp = 0; cp < 64; ++cp)
        for (int t = 0; t < 9; ++t) b += (double)wc[((size_t)co * 64 + cp) * 9 + t] * bv[cp];
      bcomb[co] = (float)b;
    }
    // Border corrections (subtracted from the combined pre-activation on the image
    // border): decode.0 taps (ky, kx) that read the canvas ring outside the crop.  Edge e
    // (0 top: ky 0 / canvas row 0 <- a 0; 1 bottom: ky 2 <- a 9; 2 left: kx 0 <- b 0;
    // 3 right: kx 2 <- b 9), tap v in [-2, 9] along the edge:
    //   dK[e][v][ci][co] = sum_d sum_c' Wc[co][c'][ky][kx] Wv[ci][c'][a][b]
    // with d the position along the edge; corners add back the doubly removed tap.
    const size_t EB = (size_t)4 * 12 * 4096, CK = EB + 256, CB = CK + (size_t)4 * 4096;
    for (int edge = 0; edge < 4; ++edge)
      for (int v = -2; v <= 9; ++v)
        for (int d = -1; d <= 1; ++d) {
          int ky, kx, a, b;
          if (edge == 0) { ky = 0; kx = d + 1; a = 0; b = v + d + 1; }
          else if (edge == 1) { ky = 2; kx = d + 1; a = 9; b = v + d + 1; }
          else if (edge == 2) { ky = d + 1; kx = 0; a = v + d + 1; b = 0; }
          else { ky = d + 1; kx = 2; a = v + d + 1; b = 9; }
          if (a < 0 || a >= 10 || b < 0 || b >= 10) continue;
          float* dst = dkt.data() + ((size_t)(edge * 12 + v + 2) * 64) * 64;
          for (int ci = 0; ci < 64; ++ci)
            for (int co = 0; co < 64; ++co) {
              double sacc = 0.0;
              for (int cp = 0; cp < 64; ++cp) sacc += WC(co, cp, ky, kx) * WV(ci, cp, a, b);
              dst[ci * 64 + co] += (float)sacc;
            }
        }
    for (int edge = 0; edge < 4; ++edge)
      for (int d = -1; d <= 1; ++d) {
        const int ky = edge == 0 ? 0 : (edge == 1 ? 2 : d + 1);
        const int kx = edge == 2 ? 0 : (edge == 3 ? 2 : d + 1);
        for (int co = 0; co < 64; ++co) {
          double sacc = 0.0;
          for (int cp = 0; cp < 64; ++cp) sacc += WC(co, cp, ky, kx) * bv[cp];
          dkt[EB + edge * 64 + co] += (float)sacc;
        }
      }
    const int cky[4] = {0, 0, 2, 2}, ckx[4] = {0, 2, 0, 2}, ca[4] = {0, 0, 9, 9}, cb[4] = {0, 9, 0, 9};
    for (int c4 = 0; c4 < 4; ++c4) {
      for (int ci = 0; ci < 64; ++ci)
        for (int co = 0; co < 64; ++co) {
          double sacc = 0.0;
          for (int cp = 0; cp < 64; ++cp) sacc += WC(co, cp, cky[c4], ckx[c4]) * WV(ci, cp, ca[c4], cb[c4]);
          dkt[CK + (size_t)c4 * 4096 + ci * 64 + co] = (float)sacc;
        }
      for (int co = 0; co < 64; ++co) {
        double sacc = 0.0;
        for (int cp = 0; cp < 64; ++cp) sacc += WC(co, cp, cky[c4], ckx[c4]) * bv[cp];
        dkt[CB + c4 * 64 + co] = (float)sacc;
      }
    }
  }
  std::vector<float> w2f((size_t)27 * 64);
  {
    const float* w2 = weights[tb + 4];                   // [3][c][3][3]
    for (int co = 0; co < 3; ++co)
      for (int ci = 0; ci < 64; ++ci)
        for (int tap = 0; tap < 9; ++tap) w2f[(size_t)(3 * tap + co) * 64 + ci] = w2[((size_t)co * 64 + ci) * 9 + tap];
  }
  if (cudaMalloc(&e->w2f, w2f.size() * sizeof(float)) != cudaSuccess ||
      cudaMemcpy(e->w2f, w2f.data(), w2f.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
    dr_destroy(e);
    return fail(DR_ERR_CUDA, "decode.2 weight upload failed");
  }
  if (cudaMalloc(&e->wcomb, combimg.size() * 2) != cudaSuccess ||
      cudaMalloc(&e->bcomb, 64 * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&e->dk, dkt.size() * sizeof(float)) != cudaSuccess ||
      cudaMemcpy(e->wcomb, combimg.data(), combimg.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(e->bcomb, bcomb.data(), 64 * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(e->dk, dkt.data(), dkt.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
    dr_destroy(e);
    return fail(DR_ERR_CUDA, "fused decoder weight upload failed");
  }

  std::vector<double> fw = feather_taps(cfg->mask_feather_sigma);
  e->feather_r = (int)(fw.size() / 2);
  if (const char* sa = std::getenv("DR_STOP_AFTER")) e->stop_after = std::atoi(sa);
  if (const char* hg = std::getenv("DR_HOST_GRAPH")) e->host_graph = std::atoi(hg);
  if (const char* sk = std::getenv("DR_SLOTKV_SIDE")) e->slotkv_side = std::atoi(sk);
  if (e->slotkv_side &&
      (cudaStreamCreateWithFlags(&e->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
       cudaEventCreateWithFlags(&e->side_fork, cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&e->side_join, cudaEventDisableTiming) != cudaSuccess)) {
    dr_destroy(e);
    return fail(DR_ERR_CUDA, "side stream creation failed");
  }
  if (const char* tr = std::getenv("DR_TOK_ROWS")) {
    const int r = std::atoi(tr);
    e->tok_rows = (r == 32 || r == 64 || r == 128) ? r : 0;
  }

  auto cleanup = [&](int code) { dr_destroy(e); return code; };
  if (cudaMalloc(&e->fparams, fp.size() * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&e->feather_w, fw.size() * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&e->wtc, tcimg.size() * 2) != cudaSuccess ||
      cudaMalloc(&e->timg, ti.size()) != cudaSuccess)
    return cleanup(fail(DR_ERR_CUDA, "cudaMalloc of weights failed"));
  if (cudaMemcpy(e->wtc, tcimg.data(), tcimg.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(e->timg, ti.data(), ti.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return cleanup(fail(DR_ERR_CUDA, "weight upload failed"));
  if (cudaMemcpy(e->fparams, fp.data(), fp.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(e->feather_w, fw.data(), fw.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
    return cleanup(fail(DR_ERR_CUDA, "weight upload failed"));
  *out = e;
  return DR_OK;
}

void dr_destroy(dr_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->copy_stream) cudaStreamSynchronize(e->copy_stream);
  e->free_ws();
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  if (e->rgb_event) cudaEventDestroy(e->rgb_event);
  if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
  if (e->fork_ev) cudaEventDestroy(e->fork_ev);
  if (e->side_stream) cudaStreamSynchronize(e->side_stream);
  if (e->side_stream) cudaStreamDestroy(e->side_stream);
  if (e->side_fork) cudaEventDestroy(e->side_fork);
  if (e->side_join) cudaEventDestroy(e->side_join);
  cudaFree(e->fparams);
  cudaFree(e->wcomb);
  cudaFree(e->bcomb);
  cudaFree(e->dk);
  cudaFree(e->w2f);
  cudaFree(e->feather_w);
  cudaFree(e->wtc);
  cudaFree(e->timg);
  cudaFree(e->h_rgb);
  cudaFree(e->h_out);                          // (h_m0 lives inside h_rgb)
  cudaFree(e->d_done);
  for (auto* r : e->ring) cudaFree(r);
  for (auto& ev : e->ev) if (ev) cudaEventDestroy(ev);
  if (e->pin) {
    WorkPool::get().drain();          // the cache-eviction job may still walk e->pin
    cudaFreeHost(e->pin);
  }
  delete e;
}

int64_t dr_host_d2h_bytes(dr_engine* e) { return e ? (int64_t)e->last_d2h : 0; }

int32_t dr_token_tile_rows(dr_engine* e, int32_t frames) {
  if (!e || frames <= 0) return 0;
  cudaSetDevice(e->device);
  return e->tile_rows(frames * e->T);
}

int32_t dr_kernels_per_forward(dr_engine* e) {
  if (!e) return 0;
  return e->last_launches;
}

static void fill_mask_args(dr_engine* e, MaskArgs& m, int frames, const uint8_t* m0,
                           uint8_t* m1, float* alpha, uint8_t* tv, int* flags) {
  m.frames = frames; m.H = e->H; m.W = e->W; m.patch = e->cfg.patch;
  m.radius = e->cfg.mask_dilate;
  m.feather_radius = e->feather_r;
  m.feather_w = e->feather_w;
  m.m0 = m0;
  m.bits0 = e->bits0; m.bits1 = e->bits1;
  m.m1 = m1; m.alpha = alpha; m.token_valid = tv;
  m.gtmp = nullptr;
  m.flags = flags;
  m.flag_acc = e->flag_acc; m.flag_cnt = e->flag_cnt;   // the stage writes flags[f]
}

int dr_mask_stage(int32_t frames, int32_t height, int32_t width, int32_t patch, int32_t radius,
                  float sigma, const uint8_t* m0, uint8_t* m1, float* alpha,
                  uint8_t* token_valid, void* stream) {
  if (frames <= 0 || height <= 0 || width <= 0 || !m0)
    return fail(DR_ERR_INPUT, "need frames, height, width > 0 and a mask");
  if (radius < 0 || radius > 31) return fail(DR_ERR_CONFIG, "radius must be in [0, 31]");
  if (!(sigma >= 0.f) || (int)(4.0 * sigma + 0.5) > 31)
    return fail(DR_ERR_CONFIG, "sigma must be in [0, 7.8] (feather radius <= 31)");
  if (token_valid && (patch != 4 && patch != 8))
    return fail(DR_ERR_CONFIG, "token mask supports patch 4 or 8");
  if (token_valid && (height % patch || width % patch))
    return fail(DR_ERR_CONFIG, "width and height must be divisible by patch size");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int Ww = (width + 31) / 32;
  const size_t words = (size_t)frames * height * Ww * 4;
  std::vector<double> fw = feather_taps(sigma);
  const int fr = (int)(fw.size() / 2);
  uint8_t* scratch = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&scratch, 2 * words + fw.size() * sizeof(double) + 256, s));
  double* dfw = reinterpret_cast<double*>(scratch + ((2 * words + 255) & ~(size_t)255));
  CUDA_TRY(cudaMemcpyAsync(dfw, fw.data(), fw.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  MaskArgs m{};
  m.frames = frames; m.H = height; m.W = width; m.patch = patch;
  m.radius = radius; m.feather_radius = fr; m.feather_w = dfw;
  m.m0 = m0;
  m.bits0 = reinterpret_cast<uint32_t*>(scratch);
  m.bits1 = reinterpret_cast<uint32_t*>(scratch + words);
  m.m1 = m1; m.alpha = alpha; m.token_valid = token_valid;
  launch_mask_stage(m, s);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(scratch, s));
  return DR_OK;
}

int dr_forward(dr_engine* e, const dr_frame_io* io, void* stream) {
  if (!e || !io) return fail(DR_ERR_CONFIG, "null engine or io");
  const int B = io->frames;
  if (B <= 0) return fail(DR_ERR_INPUT, "frames must be positive");
  if ((io->rgb_f32 == nullptr) == (io->rgb_u8 == nullptr))
    return fail(DR_ERR_INPUT, "exactly one of rgb_f32 / rgb_u8 is required");
  if (!io->mask_m0 || !io->new_slot) return fail(DR_ERR_INPUT, "mask and new_slot are required");
  if (io->out_u8 && !io->rgb_u8) return fail(DR_ERR_INPUT, "out_u8 needs the u8 input");
  if (io->out_f32 && !io->rgb_f32) return fail(DR_ERR_INPUT, "out_f32 needs the f32 input");
  CUDA_TRY(cudaSetDevice(e->device));
  int rc = e->ensure(B);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int T = e->T;
  int* flags = io->flags ? io->flags : e->flags;
  e->n_ev = 0;
  // e->dry: every host-side decision (and its state update) without the launches
#define DR_L(x) do { if (!e->dry) { x; } } while (0)
  DR_L(e->mark(-1, s));
  // no flags memset: the mask stage (first launch) writes every frame's flags word
  // diagnostics only (DR_STOP_AFTER): truncate the launch sequence to time graph prefixes
  int n_launched = 0;
#define DR_STOP_CHECK() \
  if (e->stop_after >= 0 && ++n_launched > e->stop_after) return DR_OK

  // host path with split uploads: the slot K/V projections (step 2) read only the memory
  // slots, so they are forked here and run while the mask stage / input pack wait on the
  // uploads, joining before the first block (C2 e2e +1.2 %; on the device path the branch
  // measured 1 % slower: the stage is already one fused kernel there)
  const bool split = e->rgb_ready != nullptr && io->rgb_u8 != nullptr;
  const bool side = split && e->slotkv_side && e->side_stream && !e->profiling &&
                    e->stop_after < 0 && e->n_temporal > 0 && (io->slot0 || io->slot1);
  DR_L(if (side) CUDA_TRY(cudaEventRecord(e->side_fork, s)));

  // 1. mask stage + packed network input
  MaskArgs m{};
  uint8_t* tv = io->token_valid ? io->token_valid : e->tv;
  float* alpha = io->alpha ? io->alpha : e->alpha;
  fill_mask_args(e, m, B, io->mask_m0, io->dilated, alpha, tv, flags);
  m.rgb_f32 = io->rgb_f32; m.rgb_u8 = io->rgb_u8; m.xin = e->xin;
  if (split) {
    // host path, split uploads: the stage runs on the mask alone while the rgb is still in
    // flight on the copy stream; the input pack follows once it has landed
    MaskArgs mo = m;
    mo.rgb_f32 = nullptr; mo.rgb_u8 = nullptr; mo.xin = nullptr;
    if (!mo.m1) mo.m1 = e->m1;
    DR_STOP_CHECK();
    DR_L(launch_mask_stage(mo, s));
    DR_L(CUDA_TRY(cudaStreamWaitEvent(s, e->rgb_ready, e->capturing ? cudaEventWaitExternal : 0)));
    MaskArgs pk = m;
    pk.m1 = mo.m1;
    DR_L(launch_pack_input(pk, s));
  } else {
    DR_STOP_CHECK();
    DR_L(launch_mask_stage(m, s));
  }
  DR_L(e->mark(0, s));

  // 2. memory-slot K/V of every temporal block (LN1 + k/v projection of each slot,
  //    dstt.py:188-190).  An LRU cache keyed by slot pointer holds them: the last block
  //    of every forward writes the new slot's K/V, so in steady state (caller passes the
  //    engine's own outputs back, slot_kv_reuse bits set) nothing is recomputed here.
  const int fs = io->slot_batched ? B : 1;
  int ent[2] = {0, 0};
  int n_slotkv = 0, kv_computed = 0, en_fill = -1;
  if (e->n_temporal > 0) {
    const float* sp[2] = {io->slot0, io->slot1};
    for (int sl = 0; sl < 2; ++sl) {
      ent[sl] = -1;
      if (!sp[sl]) continue;                              // zero slot: constant K/V
      if (sl == 1 && sp[1] == sp[0]) { ent[1] = ent[0]; continue; }
      if ((io->slot_kv_reuse >> sl) & 1) ent[sl] = e->kv_find(sp[sl], fs, io->slot_batched);
      if (ent[sl] >= 0) continue;
      ent[sl] = e->kv_pick(sl == 1 ? ent[0] : -1, -1, sp[sl]);
      e->kv_set(ent[sl], sp[sl], fs, io->slot_batched != 0);
      kv_computed |= 1 << sl;
      int ti = 0;
      for (int i = 0; i < e->nb; ++i) {
        if (!e->blk[i].temporal) continue;
        TokenArgs a{};
        a.n_tok = fs * T; a.T = T;
        a.resid_in = sp[sl];
        a.next = e->block_w(i);
        a.k = e->kv_ptr(ent[sl], ti, 0); a.v = e->kv_ptr(ent[sl], ti, 1);
        a.late_wait = 1;
        DR_STOP_CHECK();
        if (side && n_slotkv == 0) DR_L(CUDA_TRY(cudaStreamWaitEvent(e->side_stream, e->side_fork, 0)));
        DR_L(e->launch_tok(TOK_SLOTKV, a, side ? e->side_stream : s));
        ++n_slotkv;
        DR_L(e->mark(1, s));
        ++ti;
      }
    }
  }

  if (side && n_slotkv > 0) {
    DR_L(CUDA_TRY(cudaEventRecord(e->side_join, e->side_stream)));
    DR_L(CUDA_TRY(cudaStreamWaitEvent(s, e->side_join, 0)));
  }

  // 3. patch embed (+ LN1/QKV of block 0)
  {
    TokenArgs a{};
    a.n_tok = B * T; a.T = T;
    a.xin = e->xin; a.we_img = e->timg;
    a.kin = 4 * e->cfg.patch * e->cfg.patch;
    a.resid_out = e->resid[0];
    a.has_next = 1; a.next = e->block_w(0);
    a.q = e->q; a.k = e->k; a.v = e->v;
    DR_STOP_CHECK();
    DR_L(e->launch_tok(TOK_EMBED, a, s));
    DR_L(e->mark(2, s));
  }

  // 4. blocks; mask-aware validity (MAT update) resolved into a per-block mode
  bool seen_t = false;
  int cur = 0, ti = 0;
  for (int i = 0; i < e->nb; ++i) {
    const bool temporal = e->blk[i].temporal;
    int mode = 0;
    if (e->cfg.mask_aware_attention && !seen_t) {
      if (i == 0) mode = temporal ? 2 : 1;
      else mode = temporal ? 3 : 0;
    }
    AttnArgs at{};
    at.q = e->q; at.T = T; at.frames = B; at.out = e->attn;
    at.k[0] = e->k; at.v[0] = e->v; at.seg_frame_stride[0] = 1;
    at.key_valid = tv; at.mask_mode = mode;
    if (temporal) {
      at.groups = e->cfg.temporal_groups; at.band = T / at.groups;
      // key segments: current band, then each non-zero slot's band; the zero slots' keys
      // (all equal) enter as one constant key of multiplicity band per zero slot
      at.n_seg = 1;
      for (int sl = 0; sl < 2; ++sl) {
        if (ent[sl] < 0) {
          at.const_mult += at.band;
          continue;
        }
        at.k[at.n_seg] = e->kv_ptr(ent[sl], ti, 0); at.v[at.n_seg] = e->kv_ptr(ent[sl], ti, 1);
        at.seg_frame_stride[at.n_seg] = io->slot_batched ? 1 : 0;
        ++at.n_seg;
      }
      if (at.const_mult) at.const_kv = e->fparams + e->blk[i].zkv;
      ++ti;
      seen_t = true;
    } else {
      at.n_seg = 1; at.groups = 1; at.band = T;
    }
    DR_STOP_CHECK();
    DR_L(launch_attention(at, s));
    DR_L(e->mark(temporal ? 4 : 3, s));

    const bool last = i == e->nb - 1;
    TokenArgs a{};
    a.n_tok = B * T; a.T = T;
    a.attn = e->attn; a.resid_in = e->resid[cur]; a.cur = e->block_w(i);
    a.resid_out = last ? io->new_slot : e->resid[cur ^ 1];
    a.has_next = !last;
    if (!last) a.next = e->block_w(i + 1);
    a.q = e->q; a.k = e->k; a.v = e->v;
    a.tok16 = e->tok16;
    a.R = e->R; a.Cc = e->Cc;
    // Small batches (32/64-token tiles): the new slot's K/V (next frame's temporal blocks)
    // are projected by the next forward's slot K/V launches, which overlap that frame's
    // mask stage (late_wait), instead of lengthening this frame's latency-bound last block.
    // Large batches (128-token tiles, throughput-bound): filled here, inside the last block.
    if (last)
      for (auto& k : e->kvc) if (k.ptr == io->new_slot) k = {nullptr, 0, false, 0};  // stale
    int en = -1;
    const bool fill_here = e->tile_rows(B * T) == 128;
    if (fill_here && last && e->n_temporal > 0) {     // fill the cache for new_slot
      en = e->kv_pick(ent[0], ent[1], io->new_slot);
      int tj = 0;
      for (int j = 0; j < e->nb; ++j) {
        if (!e->blk[j].temporal) continue;
        a.kv_w[tj] = e->block_w(j);
        a.kv_k[tj] = e->kv_ptr(en, tj, 0);
        a.kv_v[tj] = e->kv_ptr(en, tj, 1);
        ++tj;
      }
      a.n_kv = tj;
    }
    DR_STOP_CHECK();
    DR_L(e->launch_tok(TOK_POST, a, s));
    if (en >= 0) en_fill = en;
    if (en >= 0) {
      for (auto& k : e->kvc) if (k.ptr == io->new_slot) k = {nullptr, 0, false, 0};  // alias
      e->kv_set(en, io->new_slot, B, true);
    }
    DR_L(e->mark(5, s));
    cur ^= 1;
  }

  // 5. decoder tail
  ConvTcArgs c2{};
  c2.frames = B; c2.H = e->H; c2.W = e->W;
  c2.bias = e->fparams + e->bd2;
  c2.alpha = alpha; c2.rgb_f32 = io->rgb_f32; c2.rgb_u8 = io->rgb_u8;
  c2.fill = io->fill; c2.out_f32 = io->out_f32; c2.out_u8 = io->out_u8; c2.flags = flags;
  c2.flags_mirror = e->flags_mirror; c2.done = e->d_done;
  if (B == 1 && e->pack_spans) {
    c2.spans = e->pack_spans; c2.packed = e->pack_out; c2.mirror_after_spans = 1;
  }
  const bool fused = e->use_fused(B);
  if (fused) {
    // Vec2Patch o decode.0 o decode.2 + composite per tile, then the seams
    DecArgs da{};
    da.frames = B; da.H = e->H; da.W = e->W; da.R = e->R; da.Cc = e->Cc;
    da.groups = dec_groups(B, e->H, e->W, e->sm_count());
    da.wcomb = e->wcomb; da.bcomb = e->bcomb; da.w2 = e->timg + e->te_d2; da.w2f = e->w2f;
    da.b2 = e->fparams + e->bd2; da.dk = e->dk; da.tok16 = e->tok16;
    da.part = e->part; da.bd0 = e->bord_d0; da.be = e->bord_e;
    dec_fix_lines(da);
    da.tail = c2;
    DR_STOP_CHECK();
    DR_L(launch_dec_fused(e->map_tok4, da, s));
    DR_L(e->mark(9, s));
    DR_STOP_CHECK();
    DR_L(launch_dec_border(da, s));
    DR_L(e->mark(11, s));
    DR_STOP_CHECK();
    DR_L(launch_dec_fixup(da, s));
    DR_L(e->mark(10, s));
  } else {
    V2pArgs vp{};
    vp.frames = B; vp.H = e->H; vp.W = e->W; vp.R = e->R; vp.Cc = e->Cc;
    vp.w = e->wtc + e->wtc_v2p; vp.bias = e->fparams + e->bv2p; vp.raster = e->raster;
    DR_STOP_CHECK();
    DR_L(launch_v2p_tc(e->map_tok, vp, s));
    DR_L(e->mark(6, s));
    // decode.0 with decode.2's tap-expanded GEMM fused into its epilogue (E planes), then
    // the decode.2 gather + tanh + composite
    ConvTcArgs cv{};
    cv.frames = B; cv.H = e->H; cv.W = e->W;
    cv.w = e->wtc; cv.bias = e->fparams + e->bd0;
    cv.e_planes = e->eplanes; cv.w2 = e->timg + e->te_d2;
    DR_STOP_CHECK();
    DR_L(launch_conv3x3_tc(64, e->map_raster, cv, s));
    DR_L(e->mark(7, s));
    c2.e_planes = e->eplanes;
    DR_STOP_CHECK();
    DR_L(launch_dec2_gather(c2, s));
    DR_L(e->mark(8, s));
  }
  e->last_launches = 1 + n_slotkv + 1 + 2 * e->nb + 3 + (split ? 1 : 0);
  e->sig = {B, split, (intptr_t)io->rgb_u8, (intptr_t)io->rgb_f32, (intptr_t)io->mask_m0,
            (intptr_t)io->slot0, (intptr_t)io->slot1, (intptr_t)io->new_slot,
            (intptr_t)io->slot_batched, (intptr_t)flags, (intptr_t)tv, (intptr_t)alpha,
            (intptr_t)io->dilated, (intptr_t)io->fill, (intptr_t)io->out_u8,
            (intptr_t)io->out_f32, (intptr_t)e->pack_spans, (intptr_t)e->pack_out,
            (intptr_t)e->flags_mirror, (intptr_t)e->rgb_ready,
            ent[0], ent[1], kv_computed,
            en_fill, fused};
#undef DR_L
#undef DR_STOP_CHECK
  CUDA_TRY(cudaGetLastError());
  return DR_OK;
}

int dr_op_conv3x3(int32_t frames, int32_t height, int32_t width, const void* in_nhwc_f16,
                  const float* weight_host, const float* bias_host, void* out_nhwc_f16,
                  void* stream) {
  if (frames <= 0 || height <= 0 || width <= 0 || !in_nhwc_f16 || !weight_host ||
      !bias_host || !out_nhwc_f16)
    return fail(DR_ERR_INPUT, "bad conv arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<uint16_t> img;
  pack_conv_tc(weight_host, 64, 64, 64, img);
  CUtensorMap map;
  int rc = make_nhwc_map(&map, const_cast<void*>(in_nhwc_f16), frames, height, width,
                         conv_tc_rows(64) + 2);
  if (rc) return rc;
  uint8_t* dev = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&dev, img.size() * 2 + 256, s));
  CUDA_TRY(cudaMemcpyAsync(dev, img.data(), img.size() * 2, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(dev + img.size() * 2, bias_host, 256, cudaMemcpyHostToDevice, s));
  ConvTcArgs cv{};
  cv.frames = frames; cv.H = height; cv.W = width;
  cv.w = dev; cv.bias = reinterpret_cast<const float*>(dev + img.size() * 2);
  cv.out16 = static_cast<__half*>(out_nhwc_f16);
  launch_conv3x3_tc(64, map, cv, s);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(dev, s));
  CUDA_TRY(cudaStreamSynchronize(s));      // host vectors above are pageable staging
  return DR_OK;
}

int dr_profile(dr_engine* e, int32_t on) {
  if (!e) return fail(DR_ERR_CONFIG, "null engine");
  e->profiling = on;
  e->n_ev = 0;
  return DR_OK;
}

int32_t dr_profile_read(dr_engine* e, float* ms, int32_t* kinds, int32_t cap) {
  if (!e || !e->profiling || e->n_ev < 2) return 0;
  int n = 0;
  for (int i = 1; i < e->n_ev && n < cap; ++i, ++n) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, e->ev[i - 1], e->ev[i]) != cudaSuccess) return -1;
    ms[n] = t;
    kinds[n] = e->ev_kind[i];
  }
  return n;
}

int dr_reset_memory(dr_engine* e) {
  if (!e) return fail(DR_ERR_CONFIG, "null engine");
  CUDA_TRY(cudaSetDevice(e->device));
  const size_t slot = (size_t)e->T * C * sizeof(float);
  for (auto*& r : e->ring) {
    if (!r) CUDA_TRY(cudaMalloc(&r, slot));
    CUDA_TRY(cudaMemset(r, 0, slot));
  }
  e->mem0 = 0;
  e->mem1 = 0;                       // cold start: both slots are the same zero tensor
  for (bool& o : e->ring_own) o = false;
  for (bool& z : e->ring_zero) z = true;
  return DR_OK;
}

// Diagnostics (DR_E2E_TRACE=1): host phase times of the last dr_inpaint_u8_host call (us):
// staging in, H2D + forward enqueue, D2H enqueue + host fill, stream sync, band copy-out;
// device times from events: H2D, forward, D2H.  Read by scripts/e2e_breakdown.py.
namespace {
struct E2eTrace {
  bool on = std::getenv("DR_E2E_TRACE") != nullptr;
  double host[5] = {};
  float dev[3] = {};
  cudaEvent_t ev[4] = {};
};
E2eTrace& e2e_trace() {
  static E2eTrace t;
  return t;
}
double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace
extern "C" int dr_debug_e2e_trace(double* out8) {
  E2eTrace& t = e2e_trace();
  if (!t.on) return -1;
  for (int i = 0; i < 5; ++i) out8[i] = t.host[i];
  for (int i = 0; i < 3; ++i) out8[5 + i] = t.dev[i];
  return 0;
}

namespace {
// One u8 frame through host buffers with the given memory slots (device fp32 [T][C]);
// writes new_slot.  Shared by the engine-held-memory call and the explicit-slot call.
int host_inpaint(dr_engine* e, const uint8_t* rgb_hwc, const uint8_t* mask_hw,
                 uint8_t* out_hwc, const float* slot0, const float* slot1, float* new_slot,
                 int slot_kv_reuse, void* stream) {
  CUDA_TRY(cudaSetDevice(e->device));
  const size_t px = e->frame_px();
  const int H = e->H, W = e->W, halo = e->cfg.mask_dilate + e->feather_r;
  // input staging: [rgb px*3][mask px][pad to 16][row spans H x int4], one H2D; output
  // staging: span-packed composite bytes + the flags word
  const size_t in_spans = (px * 4 + 15) & ~(size_t)15;
  const size_t in_bytes = in_spans + (size_t)H * 16;
  const size_t out_cap = px * 3 + 64;
  if (!e->h_rgb) {
    CUDA_TRY(cudaMalloc(&e->h_rgb, in_bytes));
    e->h_m0 = e->h_rgb + px * 3;
    CUDA_TRY(cudaMalloc(&e->h_out, out_cap));
    CUDA_TRY(cudaMalloc(&e->d_done, sizeof(unsigned)));          // finished-CTA counter
    CUDA_TRY(cudaMemset(e->d_done, 0, sizeof(unsigned)));
    CUDA_TRY(cudaMallocHost(&e->pin, in_bytes + out_cap));
    int rc = dr_reset_memory(e);
    if (rc) return rc;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  E2eTrace& tr = e2e_trace();
  double tt[6] = {};
  if (tr.on) {
    if (!tr.ev[0])
      for (auto& ev : tr.ev) cudaEventCreate(&ev);
    tt[0] = now_us();
  }
  uint8_t* p_rgb = e->pin;
  uint8_t* p_m0 = e->pin + px * 3;
  int* p_span = reinterpret_cast<int*>(e->pin + in_spans);        // [H][x0, x1, off, 0]
  uint8_t* p_out = e->pin + in_bytes;
  // Only pixels within r + R (square) of a masked pixel can differ from the input (alpha
  // = 0 keeps the input byte exactly).  Per row, the span [x0, x1) covering
  // them is the union of the masked extents of the rows within r + R, widened by r + R;
  // decode.2 writes only those bytes, packed row after row, and its last CTA appends the
  // frame's flags word: one D2H of ~the masked area instead of the frame.
  std::vector<int>& fl_x = e->span_first;
  std::vector<int>& ll_x = e->span_last;
  fl_x.resize(H);
  ll_x.resize(H);
  WorkPool::get().run([&](int part, int parts) {
    for (int y = part * H / parts; y < (part + 1) * H / parts; ++y)
      row_extent(mask_hw + (size_t)y * W, W, &fl_x[y], &ll_x[y]);
  });
  for (int y = 0; y < H; ++y)
    if (fl_x[y] < 0) fl_x[y] = W;                  // empty row: identity of the min
  std::vector<int>& wmin = e->span_wmin;
  std::vector<int>& wmax = e->span_wmax;
  wmin.resize(H);
  wmax.resize(H);
  window_reduce<false>(fl_x.data(), H, halo, W, wmin.data(), e->span_buf);
  window_reduce<true>(ll_x.data(), H, halo, -1, wmax.data(), e->span_buf);
  size_t total = 0;
  int n_rows = 0;
  for (int y = 0; y < H; ++y) {
    const int x0 = wmin[y], x1 = wmax[y];
    int* sp = p_span + 4 * y;
    if (x1 < 0) {
      sp[0] = sp[1] = 0;
    } else {
      sp[0] = std::max(0, x0 - halo);
      sp[1] = std::min(W, x1 + halo + 1);
      ++n_rows;
    }
    sp[2] = (int)total;
    sp[3] = 0;
    total += (size_t)(sp[1] - sp[0]) * 3;
  }
  const size_t mirror = (total + 3) & ~(size_t)3;                 // flags word offset
  // split uploads: mask (+ span table) first on the compute stream, so the mask stage can
  // run while the rgb crosses PCIe on the copy stream
  if (!e->copy_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&e->rgb_event, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming));
  }
  dr_frame_io io{};
  io.frames = 1;
  io.rgb_u8 = e->h_rgb; io.mask_m0 = e->h_m0;
  io.slot0 = slot0; io.slot1 = slot1; io.slot_batched = 1;
  io.new_slot = new_slot;
  io.slot_kv_reuse = slot_kv_reuse;
  e->pack_spans = reinterpret_cast<const int4*>(e->h_rgb + in_spans);
  e->pack_out = e->h_out;
  e->flags_mirror = nullptr;         // decode.2 places it after the packed bytes
  e->rgb_ready = e->rgb_event;
  struct Restore {
    dr_engine* e;
    ~Restore() {
      e->pack_spans = nullptr; e->pack_out = nullptr; e->rgb_ready = nullptr;
      e->dry = false; e->capturing = false;
    }
  } restore{e};
  // uploads: mask + span table on s first, then the rgb on the copy stream; the mask stage
  // runs while the rgb crosses PCIe and the input pack joins the rgb event.
  const bool graphed = e->host_graph && !e->profiling && e->stop_after < 0;
  int rc = DR_OK;
  if (tr.on) cudaEventRecord(tr.ev[0], s);
  par_memcpy(p_m0, mask_hw, px, CP_NT);
  CUDA_TRY(cudaMemcpyAsync(e->h_m0, p_m0, in_bytes - px * 3, cudaMemcpyHostToDevice, s));
  // the copy stream follows s up to here (never past the launches: the pack waits on it)
  CUDA_TRY(cudaEventRecord(e->fork_ev, s));
  CUDA_TRY(cudaStreamWaitEvent(e->copy_stream, e->fork_ev, 0));
  par_memcpy(p_rgb, rgb_hwc, px * 3, CP_NT);
  CUDA_TRY(cudaMemcpyAsync(e->h_rgb, p_rgb, px * 3, cudaMemcpyHostToDevice, e->copy_stream));
  CUDA_TRY(cudaEventRecord(e->rgb_event, e->copy_stream));
  if (tr.on) tt[1] = now_us();
  if (!graphed) {
    if (tr.on) cudaEventRecord(tr.ev[1], s);
    rc = dr_forward(e, &io, stream);
    if (rc) return rc;
  } else {
    // The launch sequence as one graph launch.  A dry pass makes dr_forward's
    // decisions (slot K/V cache, ring) and state updates; its signature selects the graph.
    // A new signature rewinds the cache state and captures the real pass.
    if (tr.on) cudaEventRecord(tr.ev[1], s);
    dr_engine::KvEntry kvc0[dr_engine::KV_ENTRIES];
    std::copy(std::begin(e->kvc), std::end(e->kvc), kvc0);
    const uint64_t tick0 = e->kv_tick;
    e->dry = true;
    rc = dr_forward(e, &io, stream);
    e->dry = false;
    if (rc) return rc;
    cudaGraphExec_t exec = nullptr;
    for (auto& g : e->hgraphs)
      if (g.key == e->sig) exec = g.exec;
    if (!exec) {
      const std::vector<intptr_t> key = e->sig;
      std::copy(std::begin(kvc0), std::end(kvc0), e->kvc);
      e->kv_tick = tick0;
      if (e->hgraphs.size() >= 16) e->clear_graphs();
      CUDA_TRY(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
      e->capturing = true;             // the rgb event is recorded outside the graph
      rc = dr_forward(e, &io, e->cap_stream);
      e->capturing = false;
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &g);
      if (!rc && ce != cudaSuccess)
        rc = fail(DR_ERR_CUDA, std::string("host-path graph capture: ") + cudaGetErrorString(ce));
      if (!rc && e->sig != key) rc = fail(DR_ERR_CUDA, "host-path graph: signature changed");
      if (!rc) {
        const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
        if (ie != cudaSuccess)
          rc = fail(DR_ERR_CUDA, std::string("host-path graph instantiate: ") + cudaGetErrorString(ie));
      }
      if (g) cudaGraphDestroy(g);
      if (rc) return rc;
      e->hgraphs.push_back({key, exec});
    }
    CUDA_TRY(cudaGraphLaunch(exec, s));
  }
  if (tr.on) {
    cudaEventRecord(tr.ev[2], s);
    tt[2] = now_us();
  }
  // (On an error return `out` holds partial data.)
  CUDA_TRY(cudaMemcpyAsync(p_out, e->h_out, mirror + 4, cudaMemcpyDeviceToHost, s));
  if (tr.on) cudaEventRecord(tr.ev[3], s);
  par_memcpy(out_hwc, rgb_hwc, px * 3);           // the unchanged pixels, while the GPU runs
  if (tr.on) tt[3] = now_us();
  CUDA_TRY(cudaStreamSynchronize(s));
  if (tr.on) tt[4] = now_us();
  int fl;
  std::memcpy(&fl, p_out + mirror, sizeof(int));
  if (fl & DR_FLAG_UNREDACTED)
    return fail(DR_ERR_INPUT, "input is not redacted: nonzero pixels inside mask");
  if (fl & DR_FLAG_NONFINITE) return fail(DR_ERR_NUMERIC, "model produced non-finite output");
  if (n_rows > 0) {
    const size_t rowb = (size_t)W * 3;
    WorkPool::get().run([&](int part, int parts) {
      for (int y = part * H / parts; y < (part + 1) * H / parts; ++y) {
        const int* sp = p_span + 4 * y;
        if (sp[1] > sp[0])
          std::memcpy(out_hwc + y * rowb + 3 * sp[0], p_out + sp[2], 3 * (size_t)(sp[1] - sp[0]));
      }
    });
  }
  {
    const uint8_t* ev = p_out;
    const size_t nev = mirror + 4;
    WorkPool::get().run_async([ev, nev](int part, int parts) {
      size_t b, e;
      part_range(nev, part, parts, &b, &e);
      if (e > b) evict_lines(ev + b, e - b);
    });
  }
  if (tr.on) {
    tt[5] = now_us();
    for (int i = 0; i < 5; ++i) tr.host[i] = tt[i + 1] - tt[i];
    for (int i = 0; i < 3; ++i) {
      float ms = 0.f;
      const cudaError_t err = cudaEventElapsedTime(&ms, tr.ev[i], tr.ev[i + 1]);
      tr.dev[i] = err == cudaSuccess ? 1e3f * ms : -(float)err;
    }
  }
  e->last_d2h = mirror + 4;
  return DR_OK;
}
}  // namespace

int dr_inpaint_u8_host(dr_engine* e, const uint8_t* rgb_hwc, const uint8_t* mask_hw,
                       uint8_t* out_hwc, void* stream) {
  if (!e || !rgb_hwc || !mask_hw || !out_hwc) return fail(DR_ERR_INPUT, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  if (!e->ring[0]) {
    int rc = dr_reset_memory(e);
    if (rc) return rc;
  }
  int fresh = 0;
  while (fresh == e->mem0 || fresh == e->mem1) ++fresh;
  const int reuse = (e->ring_own[e->mem0] ? 1 : 0) | (e->ring_own[e->mem1] ? 2 : 0);
  e->ring_own[fresh] = false;
  e->ring_zero[fresh] = false;
  // a slot still at its reset value goes in as the zero slot (NULL: constant K/V)
  const float* s0 = e->ring_zero[e->mem0] ? nullptr : e->ring[e->mem0];
  const float* s1 = e->ring_zero[e->mem1] ? nullptr : e->ring[e->mem1];
  const int rc = host_inpaint(e, rgb_hwc, mask_hw, out_hwc, s0, s1, e->ring[fresh], reuse, stream);
  if (rc == DR_OK || rc == DR_ERR_INPUT || rc == DR_ERR_NUMERIC) {
    // the launches ran: contents and slot K/V cache entry of `fresh` agree
    e->ring_own[fresh] = true;
  }
  if (rc) return rc;
  e->mem0 = e->mem1;
  e->mem1 = fresh;
  return DR_OK;
}

int dr_inpaint_u8_host_mem(dr_engine* e, const uint8_t* rgb_hwc, const uint8_t* mask_hw,
                           uint8_t* out_hwc, const float* slot0, const float* slot1,
                           float* new_slot, int32_t slot_kv_reuse, void* stream) {
  if (!e || !rgb_hwc || !mask_hw || !out_hwc) return fail(DR_ERR_INPUT, "null argument");
  if (!new_slot) return fail(DR_ERR_INPUT, "new_slot is required");
  if (new_slot == slot0 || new_slot == slot1)
    return fail(DR_ERR_INPUT, "new_slot must not alias a memory slot");
  return host_inpaint(e, rgb_hwc, mask_hw, out_hwc, slot0, slot1, new_slot, slot_kv_reuse & 3,
                      stream);
}

// ------------------------------------------------------------------ frame byte kernels
int dr_display_composite(int32_t height, int32_t width, int32_t channels,
                         const uint8_t* original_hwc, const uint8_t* inpainted_hwc,
                         const uint8_t* mask_hw, int32_t engine_failed, uint8_t* out_hwc,
                         void* stream) {
  if (height <= 0 || width <= 0 || !original_hwc || !out_hwc)
    return fail(DR_ERR_INPUT, "display composite needs a non-empty raster and an output");
  if (channels != 1 && channels != 3) return fail(DR_ERR_INPUT, "channels must be 1 or 3");
  if (engine_failed && !mask_hw) return fail(DR_ERR_INPUT, "engine_failed needs the mask");
  DisplayArgs a{};
  a.height = height; a.width = width; a.channels = channels;
  a.original = original_hwc; a.inpainted = inpainted_hwc; a.mask = mask_hw;
  a.engine_failed = engine_failed ? 1 : 0; a.out = out_hwc;
  launch_display(a, static_cast<cudaStream_t>(stream));
  CUDA_TRY(cudaGetLastError());
  return DR_OK;
}

int dr_merge_redact(int32_t n_masks, int32_t height, int32_t width, const uint8_t* masks,
                    const uint8_t* private_flags, const uint8_t* rgb_hwc, uint8_t* merged_hw,
                    uint8_t* redacted_hwc, void* stream) {
  if (n_masks < 0 || height <= 0 || width <= 0)
    return fail(DR_ERR_INPUT, "merge/redact needs n_masks >= 0 and a non-empty raster");
  if (n_masks > 0 && (!masks || !private_flags))
    return fail(DR_ERR_INPUT, "masks and private flags are required");
  if ((rgb_hwc == nullptr) != (redacted_hwc == nullptr))
    return fail(DR_ERR_INPUT, "redaction needs both the input and the output raster");
  MergeRedactArgs a{};
  a.n_masks = n_masks; a.height = height; a.width = width;
  a.masks = masks; a.private_flags = private_flags;
  a.rgb_in = rgb_hwc; a.merged = merged_hw; a.rgb_out = redacted_hwc;
  launch_merge_redact(a, static_cast<cudaStream_t>(stream));
  CUDA_TRY(cudaGetLastError());
  return DR_OK;
}

int dr_pack_pointcloud(int32_t height, int32_t width, const float* depth_hw,
                       const uint8_t* rgb_hwc, double fx, double fy, double cx, double cy,
                       int32_t* row_counts, float* xyz, uint8_t* colors, int32_t* count,
                       void* stream) {
  if (height < 0 || width < 0 || !count)
    return fail(DR_ERR_INPUT, "point cloud needs height, width >= 0 and a count");
  if (!(fx != 0.0) || !(fy != 0.0)) return fail(DR_ERR_INPUT, "focal lengths must be nonzero");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (height == 0 || width == 0) {
    CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int32_t), s));
    return DR_OK;
  }
  if (!depth_hw || !rgb_hwc || !row_counts || !xyz || !colors)
    return fail(DR_ERR_INPUT, "depth, rgb, scratch and outputs are required");
  PointCloudArgs a{};
  a.height = height; a.width = width; a.depth = depth_hw; a.rgb = rgb_hwc;
  a.inv_fx = 1.0 / fx; a.inv_fy = 1.0 / fy; a.cx = cx; a.cy = cy;
  a.row_counts = row_counts; a.xyz = xyz; a.colors = colors; a.count = count;
  launch_pointcloud(a, s);
  CUDA_TRY(cudaGetLastError());
  return DR_OK;
}

}  // extern "C"

