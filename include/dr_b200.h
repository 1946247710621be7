/*
 * dr_b200.h -- C-ABI of libdrb200.so, the B200 (sm_100a) masked-inpainting hot path of
 * arXiv 2509.10466 (reference package `dimreal`, /root/reference/pkg).
 *
 * Plain C types only: device pointers, sizes, a cudaStream_t passed as void*.  Every
 * device-pointer entry point is stream-ordered and never synchronises the host; results
 * and the per-frame status flags are valid once the stream reaches the end of the call.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/dimreal):
 *   dr_create          DsttEngine.__init__ + load_weights     inpaint/dstt.py:292-299, :331-342
 *   dr_forward         DsttModel.forward + the engine composite
 *                                                             inpaint/dstt.py:256-268,
 *                                                             inpaint/base.py:52-89
 *   dr_inpaint_u8_host InpaintEngine.inpaint / DsttEngine._fill on host u8 buffers
 *                                                             inpaint/base.py:52-89,
 *                                                             inpaint/dstt.py:313-326
 *   dr_mask_stage      new: dilate (masks._CROSS, masks.py:17/:193), feather, token mask
 *   dr_display_composite  upscale2x + _composite_upscaled      pipeline.py:120-131, :203-222,
 *                                                             _kernels.py:13-46
 *   dr_merge_redact    merge_private_masks + redact            masks.py:128-154
 *   dr_pack_pointcloud transplant_pointcloud / pack_pointcloud pipeline.py:147-157,
 *                                                             _kernels.py:49-93
 *   dr_last_error      exception message of the failing call
 * Error codes map onto the reference exceptions (errors.py:4-33):
 *   DR_ERR_CONFIG -> ConfigError, DR_ERR_INPUT -> InputError,
 *   DR_ERR_NUMERIC -> EngineNumericError, DR_ERR_CUDA -> RuntimeError.
 */
#ifndef DR_B200_H
#define DR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DR_OK 0
#define DR_ERR_CONFIG 1
#define DR_ERR_INPUT 2
#define DR_ERR_NUMERIC 3
#define DR_ERR_CUDA 4

/* per-frame status bits written to dr_frame_io.flags */
#define DR_FLAG_NONFINITE 1    /* network output not finite  -> EngineNumericError */
#define DR_FLAG_UNREDACTED 2   /* u8 input nonzero inside m0 -> InputError         */

/* DsttConfig (inpaint/dstt.py:35-86) plus the mask-stage fields. */
typedef struct dr_config {
  int32_t width, height, patch, channels, kernel, heads, temporal_groups;
  int32_t n_blocks;
  char blocks[16];               /* 'S' / 'T', n_blocks of them */
  int32_t mask_dilate;           /* r: 3x3-cross dilation iterations (0 = off)       */
  float mask_feather_sigma;      /* Gaussian feather sigma (0 = binary alpha)        */
  int32_t mask_aware_attention;  /* 1 = exclude fully masked tokens as keys (MAT)    */
} dr_config;

typedef struct dr_engine dr_engine;

typedef struct dr_frame_io {
  int32_t frames;                /* B                                                */
  const float* rgb_f32;          /* [B][3][H][W] in [0,1], or NULL                   */
  const uint8_t* rgb_u8;         /* [B][H][W][3], or NULL (exactly one rgb input)    */
  const uint8_t* mask_m0;        /* [B][H][W], nonzero = private                     */
  const float* slot0;            /* memory, oldest first: [B][T][C] or [T][C], or    */
  const float* slot1;            /* NULL = the all-zero slot (InpaintMemory.zero)    */
  int32_t slot_batched;          /* 1: slots are [B][T][C]; 0: one [T][C] for all    */
  float* new_slot;               /* [B][T][C] out: post-block tokens (required)      */
  float* out_f32;                /* [B][3][H][W] composite (float API), or NULL      */
  uint8_t* out_u8;               /* [B][H][W][3] composite (u8 API), or NULL         */
  float* fill;                   /* [B][3][H][W] raw network output, or NULL         */
  uint8_t* dilated;              /* [B][H][W] m1, or NULL                            */
  float* alpha;                  /* [B][H][W] feathered alpha, or NULL               */
  uint8_t* token_valid;          /* [B][T] token validity, or NULL                   */
  int32_t* flags;                /* [B] DR_FLAG_* bits, or NULL (engine-internal)    */
  /* Slot K/V cache (bit0: slot0, bit1: slot1).  Set a bit only when that slot is the
   * unmodified new_slot output of an earlier dr_forward of this engine: its per-temporal-
   * block K/V, produced by that call, are then reused instead of re-projected.  0 always
   * computes them (correct for any slot contents). */
  int32_t slot_kv_reuse;
} dr_frame_io;

/* A NULL slot is the cold memory slot (all zeros, InpaintMemory.from_zero_slot, memory.py:32-34).  Its tokens are
 * identical, so its keys are one constant per temporal block: no slot K/V projection is
 * launched, and attention takes its `band` equal keys as one key of that multiplicity --
 * the same softmax, without the 2 x band redundant scores per query. */

/* Build an engine on `device` from the 72 DRWT tensors in state_dict order (host fp32
 * pointers, element counts checked against cfg).  Weights are repacked once into
 * fragment-major fp16 images; they are immutable afterwards. */
int dr_create(const dr_config* cfg, const float* const* weights, const int64_t* numels,
              int32_t n_tensors, int32_t device, dr_engine** out);

void dr_destroy(dr_engine* e);

/* Thread-local message of the last failing call on this thread. */
const char* dr_last_error(void);

int32_t dr_version(void);

/* Full path on device buffers: mask stage -> forward -> composite.  Stream-ordered. */
int dr_forward(dr_engine* e, const dr_frame_io* io, void* stream);

/* The mask stage alone, no engine needed: m0 [B][H][W] -> m1 (u8), alpha (f32) and token
 * validity [B][(H/patch)*(W/patch)] (patch 4 or 8).  Any output may be NULL.  Scratch is
 * stream-ordered (cudaMallocAsync).  radius <= 31, sigma <= 7.8. */
int dr_mask_stage(int32_t frames, int32_t height, int32_t width, int32_t patch, int32_t radius,
                  float sigma, const uint8_t* m0, uint8_t* m1, float* alpha,
                  uint8_t* token_valid, void* stream);

/* One u8 frame through host buffers, like InpaintEngine.inpaint: copies rgb/mask in,
 * runs the path with the engine-held 2-slot memory (FIFO advanced once per call), copies
 * the composite out and synchronises.  Rows that cannot change are filled from the input
 * on the host while the GPU runs (see dr_host_d2h_bytes).  On an error return the
 * contents of out_hwc are unspecified.  Returns DR_ERR_INPUT if the frame is not
 * redacted inside the mask, DR_ERR_NUMERIC on a non-finite network output. */
int dr_inpaint_u8_host(dr_engine* e, const uint8_t* rgb_hwc, const uint8_t* mask_hw,
                       uint8_t* out_hwc, void* stream);

/* dr_inpaint_u8_host with the memory passed explicitly, the reference signature
 * InpaintEngine.inpaint(rgb, mask, memory) (base.py:52-89, called by
 * LocalEngineClient.inpaint_frame, service.py:198-204): slot0 / slot1 are the memory's
 * two device fp32 [T][C] slots (oldest first; NULL = zero slot), new_slot receives the post-block tokens
 * (the caller pushes it: memory.py:40-45).  Bit i of slot_kv_reuse may be set only if
 * slot i is unchanged since this engine wrote it as a new_slot (its cached K/V are
 * reused).  Same staging, graphs and errors as dr_inpaint_u8_host. */
int dr_inpaint_u8_host_mem(dr_engine* e, const uint8_t* rgb_hwc, const uint8_t* mask_hw,
                           uint8_t* out_hwc, const float* slot0, const float* slot1,
                           float* new_slot, int32_t slot_kv_reuse, void* stream);

/* Device->host bytes the last dr_inpaint_u8_host copied: only pixels within mask_dilate +
 * feather radius (square) of a masked pixel can differ from the input (the composite keeps
 * the input byte where alpha = 0), so only each row's span covering them is read back,
 * packed (+ 4 flag bytes). */
int64_t dr_host_d2h_bytes(dr_engine* e);

/* Reset the engine-held memory of dr_inpaint_u8_host to two zero slots. */
int dr_reset_memory(dr_engine* e);

/* Number of kernels one dr_forward launches for `frames` frames (for accounting). */
int32_t dr_kernels_per_forward(dr_engine* e);

/* Tokens per CTA the token-chain kernels use for `frames` frames: 128 selects the
 * throughput kernel (whose last block also fills the new slot's K/V cache), 32 / 64 the
 * latency kernel (DR_TOK_ROWS at dr_create forces one). */
int32_t dr_token_tile_rows(dr_engine* e, int32_t frames);

/* Op-level entry for parity tests of the tcgen05 implicit-GEMM convolution
 * (decode.0 form, dstt.py:241-242): out = LeakyReLU_0.2(conv3x3(in) + bias), NHWC fp16
 * rasters [frames][H][W][64], weight [64][64][3][3] fp32 host, bias [64] fp32 host. */
int dr_op_conv3x3(int32_t frames, int32_t height, int32_t width, const void* in_nhwc_f16,
                  const float* weight_host, const float* bias_host, void* out_nhwc_f16,
                  void* stream);

/* Per-stage CUDA events on the launch stream (off by default).  After the stream has
 * passed a dr_forward, dr_profile_read fills ms[i] / kinds[i] for each stage and returns
 * the count (-1 on an event error).  Kinds: 0 mask stage, 1 slot K/V, 2 embed,
 * 3 spatial attention, 4 temporal attention, 5 out-proj+FFN+QKV, 6 vec2patch,
 * 7 decode.0, 8 decode.2+composite. */
int dr_profile(dr_engine* e, int32_t on);
int32_t dr_profile_read(dr_engine* e, float* ms, int32_t* kinds, int32_t cap);

/* ---------------------------------------------------------------------------------------
 * Frame byte kernels either side of the network (all device pointers, stream-ordered).
 * ------------------------------------------------------------------------------------- */

/* Display path of Pipeline.step (pipeline.py:307-314) in one pass: out (2H x 2W x C) =
 * upscale2x(original) (pipeline.py:120-131, _kernels.py:13-46), and inside the
 * nearest-upscaled mask either upscale2x(inpainted) (_composite_upscaled,
 * pipeline.py:203-222) or 0 when engine_failed (fail-closed, pipeline.py:309-311).
 * mask / inpainted may be NULL (plain upscale2x, pipeline.upscale2x).  C = 1 or 3. */
int dr_display_composite(int32_t height, int32_t width, int32_t channels,
                         const uint8_t* original_hwc, const uint8_t* inpainted_hwc,
                         const uint8_t* mask_hw, int32_t engine_failed, uint8_t* out_hwc,
                         void* stream);

/* merge_private_masks + redact (masks.py:128-154): merged = OR of masks[k] over the k
 * with private_flags[k] != 0 (device u8 [n]); redacted = rgb with the merged pixels
 * zeroed.  merged / (rgb, redacted) may be NULL. */
int dr_merge_redact(int32_t n_masks, int32_t height, int32_t width, const uint8_t* masks,
                    const uint8_t* private_flags, const uint8_t* rgb_hwc, uint8_t* merged_hw,
                    uint8_t* redacted_hwc, void* stream);

/* pack_pointcloud / transplant_pointcloud (_kernels.py:49-93, pipeline.py:147-157):
 * back-project every depth > 0 pixel in row-major order; xyz [count][3] f32, colors
 * [count][3] u8 (capacity H*W), *count (device int) = number of points.  row_counts is
 * device scratch of H ints.  Bit-identical to the numba kernel (float64 arithmetic,
 * float32 store). */
int dr_pack_pointcloud(int32_t height, int32_t width, const float* depth_hw,
                       const uint8_t* rgb_hwc, double fx, double fy, double cx, double cy,
                       int32_t* row_counts, float* xyz, uint8_t* colors, int32_t* count,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DR_B200_H */
