// Per-frame byte kernels on either side of the inpainting network, all
// HBM-bound integer/byte work (no tensor cores):
//
//  * display composite: Pipeline.step's post stage (reference pipeline.py:307-314) fused
//    into one pass -- upscale2x of the captured frame (pipeline.py:120-131, numba kernel
//    _kernels.py:13-46: out[2y+ky, 2x+kx] = (9a + 3a_y2 + 3a_x2 + a_y2x2 + 8) >> 4 with the
//    clamped neighbour toward the sample point), and inside the nearest-upscaled privacy
//    mask either upscale2x of the inpainted raster (_composite_upscaled, pipeline.py:
//    203-222; the crop's clamping equals frame clamping for every masked pixel because the
//    crop pads the bbox by 2) or 0 when the engine failed (fail-closed, :309-311).  With no
//    mask it is the plain upscale2x (1 or 3 channels).
//    CTA = 16 x 64 source pixels: the (16+2) x (64+2) halo of both rasters is staged in
//    smem by coalesced byte loads; each thread emits 4 source pixels = two output rows of
//    8C bytes (8-byte stores when the row pitch allows).
//  * merge + redact: merge_private_masks (masks.py:128-142: OR of the PRIVATE tracks'
//    masks) fused with redact (masks.py:145-154: zero rgb inside the union).
//  * point-cloud transplant: pack_pointcloud (_kernels.py:49-93, pipeline.py:147-157):
//    stream compaction of depth > 0 pixels in row-major order, xyz = ((x - cx) * inv_fx *
//    d, (y - cy) * inv_fy * d, d) evaluated in float64 and rounded to float32 exactly like
//    the numba kernel (x - cx promotes to float64, d float32 -> float64).  Two kernels:
//    per-row valid counts (one CTA per row, float4 loads), then one CTA per row = exclusive
//    offset of its row (block reduction over the counts before it) + a ballot/popc block
//    scan, compacted in smem and written with coalesced stores.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace dr {

namespace {

constexpr int DTH = 16, DTW = 64;            // display tile (source pixels)

template <int CH>
__global__ void __launch_bounds__(256) display_kernel(DisplayArgs a) {
  __shared__ uint8_t so[DTH + 2][(DTW + 2) * CH];
  __shared__ uint8_t si[DTH + 2][(DTW + 2) * CH];
  __shared__ uint8_t sm[DTH][DTW];
  __shared__ int any_mask;
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * DTW, y0 = blockIdx.y * DTH;
  const int H = a.height, W = a.width;
  if (tid == 0) any_mask = 0;
  __syncthreads();
  // mask tile (source resolution) + whether this tile needs the inpainted raster
  int mine = 0;
  for (int e = tid; e < DTH * DTW; e += 256) {
    const int ty = e / DTW, tx = e - ty * DTW;
    const int y = y0 + ty, x = x0 + tx;
    const uint8_t m = (a.mask && y < H && x < W) ? (a.mask[(size_t)y * W + x] != 0) : 0;
    sm[ty][tx] = m;
    mine |= m;
  }
  if (mine) any_mask = 1;
  // halo rows y0-1 .. y0+DTH, columns x0-1 .. x0+DTW, clamped (nearest) at the frame edge;
  // one warp per halo row, lanes over the row's bytes (coalesced)
  const int rowb = (DTW + 2) * CH;
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < DTH + 2; r += 8) {
    const int y = min(max(y0 - 1 + r, 0), H - 1);
    const uint8_t* src = a.original + (size_t)y * W * CH;
    for (int cb = lane; cb < rowb; cb += 32) {
      const int xs = cb / CH, c = cb - xs * CH;
      so[r][cb] = src[(size_t)min(max(x0 - 1 + xs, 0), W - 1) * CH + c];
    }
  }
  __syncthreads();
  const bool need_inp = any_mask && !a.engine_failed && a.inpainted;
  if (need_inp) {
    for (int r = warp; r < DTH + 2; r += 8) {
      const int y = min(max(y0 - 1 + r, 0), H - 1);
      const uint8_t* src = a.inpainted + (size_t)y * W * CH;
      for (int cb = lane; cb < rowb; cb += 32) {
        const int xs = cb / CH, c = cb - xs * CH;
        si[r][cb] = src[(size_t)min(max(x0 - 1 + xs, 0), W - 1) * CH + c];
      }
    }
    __syncthreads();
  }
  // thread -> source row ty, 4 source pixels tx0 .. tx0+3
  const int ty = tid >> 4, tx0 = (tid & 15) * 4;
  const int y = y0 + ty;
  if (y >= H || x0 + tx0 >= W) return;
  const int npx = min(4, W - (x0 + tx0));
  uint8_t out[2][8 * CH];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const bool m = sm[ty][tx0 + p] != 0;
    const uint8_t (*src)[(DTW + 2) * CH] = (m && need_inp) ? si : so;
    const int xs = tx0 + p + 1;                          // halo column of the pixel
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      int nb[3][3];                                      // 3x3 neighbourhood (halo coords)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) nb[dy][dx] = src[ty + dy][(xs - 1 + dx) * CH + c];
#pragma unroll
      for (int ky = 0; ky < 2; ++ky)
#pragma unroll
        for (int kx = 0; kx < 2; ++kx) {
          int v = (9 * nb[1][1] + 3 * nb[2 * ky][1] + 3 * nb[1][2 * kx] + nb[2 * ky][2 * kx] + 8) >> 4;
          if (m && a.engine_failed) v = 0;
          out[ky][(2 * p + kx) * CH + c] = (uint8_t)v;
        }
    }
  }
  const size_t pitch = (size_t)2 * W * CH;
#pragma unroll
  for (int ky = 0; ky < 2; ++ky) {
    uint8_t* dst = a.out + (size_t)(2 * y + ky) * pitch + (size_t)2 * (x0 + tx0) * CH;
    if (npx == 4 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        uint2 v;
        memcpy(&v, &out[ky][8 * q], 8);
        reinterpret_cast<uint2*>(dst)[q] = v;
      }
    } else {
      for (int b = 0; b < 2 * npx * CH; ++b) dst[b] = out[ky][b];
    }
  }
}

__global__ void __launch_bounds__(256) merge_redact_kernel(MergeRedactArgs a) {
  const size_t n = (size_t)a.height * a.width;
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) {
    uint8_t m = 0;
    for (int k = 0; k < a.n_masks; ++k)
      if (a.private_flags[k]) m |= (uint8_t)(a.masks[(size_t)k * n + i] != 0);
    if (a.merged) a.merged[i] = m;
    if (a.rgb_out) {
#pragma unroll
      for (int c = 0; c < 3; ++c) a.rgb_out[3 * i + c] = m ? (uint8_t)0 : a.rgb_in[3 * i + c];
    }
  }
}

// one CTA per row: number of depth > 0 pixels
__global__ void __launch_bounds__(128) pc_count_kernel(PointCloudArgs a) {
  __shared__ int red[4];
  const int y = blockIdx.x, tid = threadIdx.x;
  const float* row = a.depth + (size_t)y * a.width;
  int n = 0;
  if ((a.width & 3) == 0 && (reinterpret_cast<uintptr_t>(a.depth) & 15) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (int i = tid; i < a.width / 4; i += 128) {
      const float4 v = __ldg(r4 + i);
      n += (v.x > 0.f) + (v.y > 0.f) + (v.z > 0.f) + (v.w > 0.f);
    }
  } else {
    for (int x = tid; x < a.width; x += 128) n += row[x] > 0.f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((tid & 31) == 0) red[tid >> 5] = n;
  __syncthreads();
  if (tid == 0) a.row_counts[y] = red[0] + red[1] + red[2] + red[3];
}

// one CTA per row: offset = sum of the counts of the rows above; the row is compacted in
// chunks of 1024 pixels (4 per thread, ballot + popc block scan) into smem, then written
// out with coalesced 4-byte (xyz) and byte (colors) stores.
constexpr int PC_CHUNK = 1024;
__global__ void __launch_bounds__(256) pc_pack_kernel(PointCloudArgs a) {
  __shared__ int red[8];
  __shared__ int wsum[8][4];
  __shared__ float sxyz[PC_CHUNK * 3];
  __shared__ uint8_t scol[PC_CHUNK * 3];
  const int y = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int s = 0;
  for (int i = tid; i < y; i += 256) s += __ldg(a.row_counts + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  const float* row = a.depth + (size_t)y * a.width;
  const uint8_t* rgb = a.rgb + (size_t)y * a.width * 3;
  const double yy = ((double)y - a.cy) * a.inv_fy;
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) base += red[w];
  if (y == a.height - 1 && tid == 0) *a.count = base + a.row_counts[y];
  for (int x0 = 0; x0 < a.width; x0 += PC_CHUNK) {
    // pixel x0 + 256 j + tid, j = 0..3: coalesced loads, order = (j, warp, lane)
    float d[4];
    uint32_t bal[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int x = x0 + 256 * j + tid;
      d[j] = x < a.width ? __ldg(row + x) : 0.f;
      bal[j] = __ballot_sync(0xffffffffu, d[j] > 0.f);
      if (lane == 0) wsum[warp][j] = __popc(bal[j]);
    }
    __syncthreads();
    int chunk = 0, pre[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        if (w == warp) pre[j] = chunk;
        chunk += wsum[w][j];
      }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (d[j] > 0.f) {
        const int x = x0 + 256 * j + tid;
        const int k = pre[j] + __popc(bal[j] & ((1u << lane) - 1u));
        const double dd = (double)d[j];
        sxyz[3 * k + 0] = (float)(((double)x - a.cx) * a.inv_fx * dd);
        sxyz[3 * k + 1] = (float)(yy * dd);
        sxyz[3 * k + 2] = d[j];
        scol[3 * k + 0] = rgb[3 * x]; scol[3 * k + 1] = rgb[3 * x + 1]; scol[3 * k + 2] = rgb[3 * x + 2];
      }
    }
    __syncthreads();
    float* gx = a.xyz + 3 * (size_t)base;
    uint8_t* gc = a.colors + 3 * (size_t)base;
    for (int i = tid; i < 3 * chunk; i += 256) {
      gx[i] = sxyz[i];
      gc[i] = scol[i];
    }
    base += chunk;
    __syncthreads();
  }
}

}  // namespace

void launch_display(const DisplayArgs& a, cudaStream_t s) {
  dim3 grid((a.width + DTW - 1) / DTW, (a.height + DTH - 1) / DTH);
  if (a.channels == 1) display_kernel<1><<<grid, 256, 0, s>>>(a);
  else display_kernel<3><<<grid, 256, 0, s>>>(a);
}

void launch_merge_redact(const MergeRedactArgs& a, cudaStream_t s) {
  const size_t n = (size_t)a.height * a.width;
  const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  merge_redact_kernel<<<blocks, 256, 0, s>>>(a);
}

void launch_pointcloud(const PointCloudArgs& a, cudaStream_t s) {
  pc_count_kernel<<<a.height, 128, 0, s>>>(a);
  pc_pack_kernel<<<a.height, 256, 0, s>>>(a);
}

}  // namespace dr
