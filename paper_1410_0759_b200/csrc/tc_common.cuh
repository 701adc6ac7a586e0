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

// fp32 -> (big, small) tf32 pair in fp32 containers (the 3xTF32 split):
// big = tf32(v) rounded to nearest (low 13 mantissa bits zero), small =
// tf32(v - big), the residual is exact in fp32; a ~= big + small with 22
// mantissa bits, the MMA ignores the zeroed low bits.
__device__ __forceinline__ void split_tf32(float v, float& big, float& small) {
  uint32_t b, s;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(v));
  const float r = v - __uint_as_float(b);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(s) : "f"(r));
  big = __uint_as_float(b);
  small = __uint_as_float(s);
}

// One packed element (element offset o of both planes), ES as below.
template <int ES>
__device__ __forceinline__ void store_split1(void* hi, void* lo, int64_t o, float v) {
  if constexpr (ES == 2) {
    __nv_bfloat16 h, l;
    split_bf16(v, h, l);
    static_cast<__nv_bfloat16*>(hi)[o] = h;
    static_cast<__nv_bfloat16*>(lo)[o] = l;
  } else {
    float h, l;
    split_tf32(v, h, l);
    static_cast<float*>(hi)[o] = h;
    static_cast<float*>(lo)[o] = l;
  }
}

// Eight consecutive packed elements (element offset o of both planes):
// ES = 2 -> BF16 hi / lo (one 16-byte store per plane), ES = 4 -> TF32
// big / small in fp32 containers (two 16-byte stores per plane).
template <int ES>
__device__ __forceinline__ void store_split8(void* hi, void* lo, int64_t o, const float (&v)[8]) {
  if constexpr (ES == 2) {
    __align__(16) __nv_bfloat16 vh[8], vl[8];
#pragma unroll
    for (int k = 0; k < 8; k++) split_bf16(v[k], vh[k], vl[k]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(hi) + o) = *reinterpret_cast<const uint4*>(vh);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(lo) + o) = *reinterpret_cast<const uint4*>(vl);
  } else {
    __align__(16) float vh[8], vl[8];
#pragma unroll
    for (int k = 0; k < 8; k++) split_tf32(v[k], vh[k], vl[k]);
    uint4* h4 = reinterpret_cast<uint4*>(static_cast<float*>(hi) + o);
    uint4* l4 = reinterpret_cast<uint4*>(static_cast<float*>(lo) + o);
    h4[0] = reinterpret_cast<const uint4*>(vh)[0];
    h4[1] = reinterpret_cast<const uint4*>(vh)[1];
    l4[0] = reinterpret_cast<const uint4*>(vl)[0];
    l4[1] = reinterpret_cast<const uint4*>(vl)[1];
  }
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

// Programmatic dependent launch for the kernel chain of one call (operand
// pack -> filter pack -> GEMM): appends the programmatic-serialization
// attribute unless DNNP_NO_PDL; the dependent kernel calls pdl_wait() before
// reading its producers' output.
inline void add_pdl_attr(cudaLaunchAttribute* attrs, unsigned* n) {
  if (::dnnp::tune_env("DNNP_NO_PDL")) return;
  attrs[*n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[*n].val.programmaticStreamSerializationAllowed = 1;
  ++*n;
}

void pool_keep_memory();     // creates this device's library pool (lib_pool)
cudaMemPool_t lib_pool();    // the library's stream-ordered pool on the current device

// main-kernel timing hooks (no-ops unless dnnp_kernel_timing(1)); tags:
// 1 conv TMA, 2 wgrad TMA, 3 conv cp.async, 4 wgrad cp.async
void ktime_begin(cudaStream_t st, int tag);
void ktime_end(cudaStream_t st);

// Row-major 2-D matrix [rows][cols] (row pitch `pitch_elems`) of bf16 (es =
// 2) or fp32 / tf32 (es = 4) as a TMA tiled tensor map with a {box_cols,
// box_rows} box and the given swizzle.
cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                         uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows,
                         CUtensorMapSwizzle swizzle, int es = 2);

// 3-D bf16 tiled tensor map (dims innermost first, byte strides of dims 1, 2;
// strides need not be monotonic, e.g. {channel, pixel, channel block}).
cudaError_t make_tmap_3d(CUtensorMap* map, const void* base, const uint64_t dims[3],
                         const uint64_t strides_bytes[2], const uint32_t box[3],
                         CUtensorMapSwizzle swizzle, int es = 2);

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
                             CUtensorMapSwizzle swizzle, int es = 2);

// Space-to-depth packing for strided convolutions with few channels:
// x'[n][h'][w'][(rh*v + rw)*C + c] = x[n][c][h'*u + rh - pad_h][w'*v + rw - pad_w]
// (zero outside the image), channels padded to Cp.
cudaError_t pack_act_s2d(const View4& v, const float* x, int u, int vv, int pad_h, int pad_w,
                         int H2, int W2, int Cp, void* hi, void* lo, cudaStream_t st,
                         int es = 2);

// Horizontal tap folding for stride-(u, v) convolutions with few channels
// (paper Table-2 layer1: C = 3, 11 x 11): the S horizontal taps become
// channels, x'[n][h][q][j*C + c] = x[n][c][h][q*v + j - pad_w] (zero outside),
// so the convolution runs as R x 1 over S*C channels with no horizontal
// stride or padding (a reduction S*C padded once, not C padded S times).
cudaError_t pack_act_fold(const View4& v, const float* x, int S, int vv, int pad_w, int Q, int Cp,
                          void* hi, void* lo, cudaStream_t st, int es = 2);
// whether folding applies (and pays) for a problem; s2d takes precedence
bool fold_taps(int64_t C, int64_t S, int64_t u, int64_t v, bool s2d);

// Packed-operand reuse inside one fused call (thread local): the fused
// backward entry packs dy once and registers it; backward-data and
// backward-filter then take the registered planes instead of repacking.
void packed_set(const float* src, const View4& v, int Cp, const void* hi, const void* lo,
                int es = 2);
bool packed_get(const float* src, const View4& v, int Cp, const void** hi, const void** lo,
                int es = 2);
void packed_clear();

// Strided fp32 4-D view -> channel-innermost split planes [n][h][w][Cp]
// (Cp = channels padded to a multiple of 8, zero filled): BF16 hi / lo (es =
// 2) or TF32 big / small in fp32 containers (es = 4).
// The next pack launch on this thread triggers its dependents at its start
// (the caller launches the independent filter pack programmatically next).
void pack_trigger_early(bool on);
// pack_act onto a zero-bordered grid (Hp, Wp), the tensor at (top, left)
cudaError_t pack_act_border(const View4& v, const float* x, int Cp, int top, int left, int Hp,
                            int Wp, void* hi, void* lo, cudaStream_t st, int es = 2);
cudaError_t pack_act(const View4& v, const float* x, int Cp, void* hi, void* lo, cudaStream_t st,
                     int es = 2);

}  // namespace tc
}  // namespace dnnp
