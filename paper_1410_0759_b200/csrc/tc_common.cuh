// Shared host/device helpers of the tensor-core convolution kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace dnnp {
namespace tc {

// fp32 -> (hi, lo) bf16 pair, a ~= hi + lo with 16 mantissa bits
__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// Stream-ordered scratch memory.  Every op takes its scratch from a
// grow-only arena kept per (device, stream): nested Workspaces of one op
// bump-allocate from it and release in LIFO order; consecutive ops reuse the
// same bytes (the stream orders them).  When an op needs more than the arena
// holds it falls back to cudaMallocAsync for that call and the arena is
// regrown (stream-ordered) to the op's high-water mark when the outermost
// Workspace closes, so steady-state calls allocate nothing.  The arena lock
// is held from the first Workspace of an op to its last (host-side calls on
// one stream are serialized; the reference serializes on the GIL).
struct ArenaState;
struct Workspace {
  void* p = nullptr;
  cudaStream_t st;
  explicit Workspace(cudaStream_t s);
  ~Workspace();
  cudaError_t alloc(size_t bytes);
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;

 private:
  ArenaState* a_;
  size_t saved_off_ = 0;
  bool fallback_ = false;
  size_t fb_bytes_ = 0;
};

void pool_keep_memory();     // creates this device's library pool (lib_pool)
cudaMemPool_t lib_pool();    // the library's stream-ordered pool on the current device

// main-kernel timing hooks (no-ops unless dnnp_kernel_timing(1)); tags:
// 1 conv TMA, 2 wgrad TMA, 3 conv cp.async, 4 wgrad cp.async
void ktime_begin(cudaStream_t st, int tag);
void ktime_end(cudaStream_t st);

// Row-major 2-D bf16 matrix [rows][cols] (row pitch `pitch_elems`) as a TMA
// tiled tensor map with a {box_cols, box_rows} box and the given swizzle.
cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                         uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows,
                         CUtensorMapSwizzle swizzle);

// 3-D bf16 tiled tensor map (dims innermost first, byte strides of dims 1, 2;
// strides need not be monotonic, e.g. {channel, pixel, channel block}).
cudaError_t make_tmap_3d(CUtensorMap* map, const void* base, const uint64_t dims[3],
                         const uint64_t strides_bytes[2], const uint32_t box[3],
                         CUtensorMapSwizzle swizzle);

// 4-D im2col tensor map over a packed [N][H][W][C] bf16 plane: `ppc` output
// pixels per load, `cpp` channels per pixel, bounding box corners (W, H) in
// [-128, 127], traversal strides <= 8.  Verified on B200 by
// tools/probe_im2col.cu: a load at (c, w, h, n) with offsets (ow, oh) reads
// input pixel (start + (ow, oh)) for each of the ppc positions obtained by
// walking w over [lower_w, W + upper_w) with stride_w, then h, then n.
struct Im2colGeom {
  int64_t N, H, W, C;
  int lower_w, lower_h, upper_w, upper_h;
  int stride_w, stride_h;
  int cpp, ppc;
};
cudaError_t make_tmap_im2col(CUtensorMap* map, const void* base, const Im2colGeom& g,
                             CUtensorMapSwizzle swizzle);

// Space-to-depth packing for strided convolutions with few channels:
// x'[n][h'][w'][(rh*v + rw)*C + c] = x[n][c][h'*u + rh - pad_h][w'*v + rw - pad_w]
// (zero outside the image), channels padded to Cp.
cudaError_t pack_act_s2d(const View4& v, const float* x, int u, int vv, int pad_h, int pad_w,
                         int H2, int W2, int Cp, __nv_bfloat16* hi, __nv_bfloat16* lo,
                         cudaStream_t st);

// Horizontal tap folding for stride-(u, v) convolutions with few channels
// (paper Table-2 layer1: C = 3, 11 x 11): the S horizontal taps become
// channels, x'[n][h][q][j*C + c] = x[n][c][h][q*v + j - pad_w] (zero outside),
// so the convolution runs as R x 1 over S*C channels with no horizontal
// stride or padding (a reduction S*C padded once, not C padded S times).
cudaError_t pack_act_fold(const View4& v, const float* x, int S, int vv, int pad_w, int Q, int Cp,
                          __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t st);
// whether folding applies (and pays) for a problem; s2d takes precedence
bool fold_taps(int64_t C, int64_t S, int64_t u, int64_t v, bool s2d);

// Packed-operand reuse inside one fused call (thread local): the fused
// backward entry packs dy once and registers it; backward-data and
// backward-filter then take the registered planes instead of repacking.
void packed_set(const float* src, const View4& v, int Cp, const __nv_bfloat16* hi,
                const __nv_bfloat16* lo);
bool packed_get(const float* src, const View4& v, int Cp, const __nv_bfloat16** hi,
                const __nv_bfloat16** lo);
void packed_clear();

// Strided fp32 4-D view -> channel-innermost bf16 hi/lo planes
// [n][h][w][Cp] (Cp = channels padded to a multiple of 8, zero filled).
cudaError_t pack_act(const View4& v, const float* x, int Cp, __nv_bfloat16* hi, __nv_bfloat16* lo,
                     cudaStream_t st);

}  // namespace tc
}  // namespace dnnp
