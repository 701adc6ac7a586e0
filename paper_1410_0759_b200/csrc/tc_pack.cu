// Operand packing for the tensor-core convolution: strided fp32 activations
// -> channel-innermost BF16 hi/lo planes, staged through shared memory so
// that both the (pixel-contiguous) reads and the (channel-contiguous)
// 16-byte writes are coalesced.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <string>
#include <unordered_map>
#include <mutex>
#include <atomic>
#include <vector>

#include "tc_common.cuh"

namespace dnnp {
namespace tc {

namespace {

constexpr int kPix = 32;   // pixels per tile
constexpr int kCh = 64;    // channels per slab

// Strided fp32 -> channel-innermost bf16 hi/lo planes through a 64 x 32
// shared tile: reads are one channel x 32 consecutive pixels per warp
// instruction (128 B for NCHW), writes are 4 pixels x 8 channel groups per
// warp instruction (contiguous 16-byte chunks).  Grid-stride over
// (pixel tile, channel slab) jobs.  S2D: the packed pixel grid is the
// space-to-depth grid (H2 x W2 super-pixels, channel c' = (rh*u2 + rw)*C + c
// reading x[c][h2*u + rh - pad_h][w2*v + rw - pad_w], zero outside).
// Early programmatic trigger of the operand packs: set by a caller whose
// next kernel (the filter pack) does not read the pack's output and itself
// waits for it before completing -- the two packs then run concurrently.
thread_local bool t_pack_early = false;
inline int early_flag() { return t_pack_early ? 1 : 0; }

struct S2dGeom {
  int u, v, pad_h, pad_w;
};

template <bool S2D, int ES>
__global__ void __launch_bounds__(256) pack_act_kernel(View4 v, const float* __restrict__ x, int Cp,
                                                       void* __restrict__ hi,
                                                       void* __restrict__ lo, int64_t npix,
                                                       MagicDiv dHW, MagicDiv dW, S2dGeom sg) {
  __shared__ float tile[kCh][kPix + 1];
  const int lp = threadIdx.x & 31, lc = threadIdx.x >> 5;  // read role: pixel, channel phase
  const int wp = threadIdx.x >> 3, wg = threadIdx.x & 7;   // write role: pixel, channel group
  // 32-bit job arithmetic (the host guarantees jobs < 2^31): a 64-bit
  // division per job cost as much as the 8 elements it moves
  const uint32_t ntiles = uint32_t((npix + kPix - 1) / kPix);
  const uint32_t nslabs = uint32_t((Cp + kCh - 1) / kCh);
  const int Cs = S2D ? sg.u * sg.v * int(v.c) : int(v.c);  // real channels of the packed grid
  for (uint32_t job = blockIdx.x; job < ntiles * nslabs; job += gridDim.x) {
    const uint32_t pt = nslabs == 1 ? job : job / nslabs;
    const int slab = int(job - pt * nslabs);
    const int c_lo = slab * kCh, nch = min(kCh, Cp - c_lo);
    const int64_t pix = int64_t(pt) * kPix + lp;
    if (pix < npix) {
      uint32_t n, rem, h, w;
      mdivmod(uint32_t(pix), dHW, n, rem);
      mdivmod(rem, dW, h, w);
      if (!S2D) {
        const float* src = x + int64_t(n) * v.sn + int64_t(h) * v.sh + int64_t(w) * v.sw +
                           int64_t(c_lo) * v.sc;
        const int cvalid = Cs - c_lo < nch ? Cs - c_lo : nch;
#pragma unroll
        for (int i = 0; i < kCh / 8; i++) {
          const int c = lc + 8 * i;
          tile[c][lp] = c < cvalid ? __ldg(src + int64_t(c) * v.sc) : 0.0f;
        }
      } else {
        const float* src = x + int64_t(n) * v.sn;
        const int hb = int(h) * sg.u - sg.pad_h, wb = int(w) * sg.v - sg.pad_w;
#pragma unroll
        for (int i = 0; i < kCh / 8; i++) {
          const int cp = c_lo + lc + 8 * i;
          float val = 0.0f;
          if (cp < Cs) {
            const int q = cp / int(v.c), c = cp - q * int(v.c);
            const int hh = hb + q / sg.v, ww = wb + q % sg.v;
            if (unsigned(hh) < unsigned(v.h) && unsigned(ww) < unsigned(v.w))
              val = __ldg(src + int64_t(c) * v.sc + int64_t(hh) * v.sh + int64_t(ww) * v.sw);
          }
          tile[lc + 8 * i][lp] = val;
        }
      }
    }
    __syncthreads();
    const int64_t opix = int64_t(pt) * kPix + wp;
    if (opix < npix && wg * 8 < nch) {
      float v8[8];
#pragma unroll
      for (int k = 0; k < 8; k++) v8[k] = tile[wg * 8 + k][wp];
      const int64_t o = opix * Cp + c_lo + wg * 8;
      store_split8<ES>(hi, lo, o, v8);
    }
    __syncthreads();
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

// Same transpose with 64-pixel jobs: each thread loads 16 values (two
// 32-pixel halves x 8 channel phases) before the barrier, twice the bytes in
// flight per synchronisation of the 32-pixel version.
// Border: the packed grid is (Hp, Wp) with the tensor at (top, left) and
// zeros around it (Hp = 0: the tensor's own grid); the halo kernel's input.
struct Border {
  int top, left, Hp, Wp;
};

template <int PIXJ, int ES>
__global__ void __launch_bounds__(256, 8) pack_act_wide_kernel(View4 v, const float* __restrict__ x,
                                                            int Cp, void* __restrict__ hi,
                                                            void* __restrict__ lo,
                                                            uint32_t npix, MagicDiv dHW,
                                                            MagicDiv dW, Border bd = Border{0, 0, 0, 0}, int early = 0) {
  if (early) pdl_trigger();  // the next kernel does not read this one: let it launch now
  __shared__ float tile[kCh][PIXJ + 1];
  constexpr int HALVES = PIXJ / 32;
  const int lp = threadIdx.x & 31, lc = threadIdx.x >> 5;  // read role: pixel, channel phase
  const int wp = threadIdx.x >> 3, wg = threadIdx.x & 7;   // write role: pixel, channel group
  const uint32_t ntiles = (npix + PIXJ - 1) / PIXJ;
  const uint32_t nslabs = uint32_t((Cp + kCh - 1) / kCh);
  const int C = int(v.c);
  for (uint32_t job = blockIdx.x; job < ntiles * nslabs; job += gridDim.x) {
    const uint32_t pt = nslabs == 1 ? job : job / nslabs;
    const int slab = int(job - pt * nslabs);
    const int c_lo = slab * kCh, nch = min(kCh, Cp - c_lo);
    const int cvalid = C - c_lo < nch ? C - c_lo : nch;
    float val[HALVES][kCh / 8];
#pragma unroll
    for (int hf = 0; hf < HALVES; hf++) {
      const uint32_t pix = pt * PIXJ + hf * 32 + lp;
      const float* src = nullptr;
      if (pix < npix) {
        uint32_t n, rem, h, w;
        mdivmod(pix, dHW, n, rem);
        mdivmod(rem, dW, h, w);
        const int hh = int(h) - bd.top, ww = int(w) - bd.left;
        if (!bd.Hp || (unsigned(hh) < unsigned(v.h) && unsigned(ww) < unsigned(v.w)))
          src = x + int64_t(n) * v.sn + int64_t(hh) * v.sh + int64_t(ww) * v.sw + int64_t(c_lo) * v.sc;
      }
#pragma unroll
      for (int i = 0; i < kCh / 8; i++) {
        const int c = lc + 8 * i;
        val[hf][i] = (src && c < cvalid) ? __ldg(src + int64_t(c) * v.sc) : 0.0f;
      }
    }
#pragma unroll
    for (int hf = 0; hf < HALVES; hf++)
#pragma unroll
      for (int i = 0; i < kCh / 8; i++) tile[lc + 8 * i][hf * 32 + lp] = val[hf][i];
    __syncthreads();
#pragma unroll
    for (int hf = 0; hf < PIXJ / 32; hf++) {
      const int px = hf * 32 + wp;
      const uint32_t opix = pt * PIXJ + px;
      if (opix < npix && wg * 8 < nch) {
        float v8[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v8[k] = tile[wg * 8 + k][px];
        const int64_t o = int64_t(opix) * Cp + c_lo + wg * 8;
        store_split8<ES>(hi, lo, o, v8);
      }
    }
    __syncthreads();
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

// Cp <= 16: one thread per pixel reads its C values (pixel-contiguous across
// the warp for NCHW) and writes Cp/8 16-byte chunks (contiguous across the warp).
template <int ES>
__global__ void __launch_bounds__(256) pack_act_small_kernel(View4 v, const float* __restrict__ x,
                                                             int Cp, void* __restrict__ hi,
                                                             void* __restrict__ lo,
                                                             int64_t npix, MagicDiv dHW, MagicDiv dW, int early = 0) {
  if (early) pdl_trigger();  // the next kernel does not read this one: let it launch now
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t pix = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pix < npix; pix += stride) {
    uint32_t n, rem, h, w;
    mdivmod(uint32_t(pix), dHW, n, rem);
    mdivmod(rem, dW, h, w);
    const float* src = x + int64_t(n) * v.sn + int64_t(h) * v.sh + int64_t(w) * v.sw;
    for (int g = 0; g < Cp / 8; g++) {
      float v8[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int c = g * 8 + k;
        v8[k] = c < v.c ? __ldg(src + int64_t(c) * v.sc) : 0.0f;
      }
      const int64_t o = pix * Cp + g * 8;
      store_split8<ES>(hi, lo, o, v8);
    }
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

// Space-to-depth: one thread per super-pixel (n, h', w'); walks its Cp
// channels (rh, rw, c) with running counters and writes 16-byte chunks
// (contiguous across the warp).
template <int ES>
__global__ void __launch_bounds__(256) pack_act_s2d_kernel(View4 v, const float* __restrict__ x,
                                                           int u, int vv, int pad_h, int pad_w,
                                                           int H2, int W2, int Cp,
                                                           void* __restrict__ hi,
                                                           void* __restrict__ lo,
                                                           int64_t npix, MagicDiv dHW, MagicDiv dW, int early = 0) {
  if (early) pdl_trigger();  // the next kernel does not read this one: let it launch now
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int C = int(v.c), Cs = u * vv * C;
  for (int64_t pix = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pix < npix; pix += stride) {
    uint32_t n, rem, h2, w2;
    mdivmod(uint32_t(pix), dHW, n, rem);
    mdivmod(rem, dW, h2, w2);
    const int hb = int(h2) * u - pad_h, wb = int(w2) * vv - pad_w;
    const float* src = x + int64_t(n) * v.sn;
    int c = 0, rw = 0, rh = 0;
    for (int g = 0; g < Cp / 8; g++) {
      float v8[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        float val = 0.0f;
        if (g * 8 + k < Cs) {
          const int h = hb + rh, w = wb + rw;
          if (unsigned(h) < unsigned(v.h) && unsigned(w) < unsigned(v.w))
            val = __ldg(src + int64_t(c) * v.sc + int64_t(h) * v.sh + int64_t(w) * v.sw);
          if (++c == C) {
            c = 0;
            if (++rw == vv) {
              rw = 0;
              ++rh;
            }
          }
        }
        v8[k] = val;
      }
      const int64_t o = pix * Cp + g * 8;
      store_split8<ES>(hi, lo, o, v8);
    }
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

// Space-to-depth, one block per output row (n, h'): the u input rows of
// every channel are read coalesced along w into shared memory as
// [w'][(rh*v + rw)*C + c], then the contiguous W' x Cp output row is written
// with 16-byte stores.
template <int ES>
__global__ void __launch_bounds__(256) pack_act_s2d_row_kernel(View4 v, const float* __restrict__ x,
                                                               int u, int vv, int pad_h, int pad_w,
                                                               int H2, int W2, int Cp,
                                                               void* __restrict__ hi,
                                                               void* __restrict__ lo) {
  extern __shared__ float srow[];
  const int Cps = Cp + 1;  // odd pitch: fewer bank conflicts on the scatter
  const int C = int(v.c);
  const int WV = W2 * vv;  // input columns covered by the row
  for (int row = blockIdx.x; row < int(v.n) * H2; row += gridDim.x) {
    const int n = row / H2, h2 = row - n * H2;
    const float* src = x + int64_t(n) * v.sn;
    const int items = C * u * WV;
    for (int t = threadIdx.x; t < items; t += blockDim.x) {
      const int wc = t % WV, q = t / WV;
      const int rh = q % u, c = q / u;
      const int h = h2 * u + rh - pad_h, w = wc - pad_w;
      float val = 0.0f;
      if (unsigned(h) < unsigned(v.h) && unsigned(w) < unsigned(v.w))
        val = __ldg(src + int64_t(c) * v.sc + int64_t(h) * v.sh + int64_t(w) * v.sw);
      const int w2 = wc / vv, rw = wc - w2 * vv;
      srow[w2 * Cps + (rh * vv + rw) * C + c] = val;
    }
    // zero the channel padding
    const int Cs = u * vv * C;
    for (int t = threadIdx.x; t < W2 * (Cp - Cs); t += blockDim.x) {
      const int w2 = t / (Cp - Cs), cc = Cs + t % (Cp - Cs);
      srow[w2 * Cps + cc] = 0.0f;
    }
    __syncthreads();
    const int groups = Cp / 8;
    const int64_t obase = int64_t(row) * W2 * Cp;
    for (int t = threadIdx.x; t < W2 * groups; t += blockDim.x) {
      const int w2 = t / groups, g = t - w2 * groups;
      float v8[8];
#pragma unroll
      for (int k = 0; k < 8; k++) v8[k] = srow[w2 * Cps + g * 8 + k];
      const int64_t o = obase + int64_t(w2) * Cp + g * 8;
      store_split8<ES>(hi, lo, o, v8);
    }
    __syncthreads();
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

// Space-to-depth fast path for dense NCHW rows (sw == 1, sh == W, W % 4 == 0):
// one block per output row (n, h'): the C x u input rows are read with
// 16-byte loads into shared memory (zero margins for the padding), then the
// W' x Cp output row -- contiguous in the packed plane -- is written with
// 16-byte stores.
template <int ES>
__global__ void __launch_bounds__(256) pack_act_s2d_dense_kernel(View4 v, const float* __restrict__ x,
                                                                 int u, int vv, int pad_h, int pad_w,
                                                                 int H2, int W2, int Cp,
                                                                 void* __restrict__ hi,
                                                                 void* __restrict__ lo) {
  extern __shared__ float srow[];  // [C*u][SW], SW = W2*v rounded up to 4
  const int C = int(v.c), W = int(v.w);
  const int SW = (W2 * vv + 3) & ~3;
  const int nrow = C * u;
  const int row = blockIdx.x;
  const int n = row / H2, h2 = row - n * H2;
  // zero the whole staging row block, then drop the in-range input in
  for (int t = threadIdx.x; t < nrow * SW; t += blockDim.x) srow[t] = 0.0f;
  __syncthreads();
  const int W4 = W >> 2;
  for (int t = threadIdx.x; t < nrow * W4; t += blockDim.x) {
    const int q = t / W4, w4 = t - q * W4;
    const int c = q / u, rh = q - c * u;
    const int h = h2 * u + rh - pad_h;
    if (unsigned(h) >= unsigned(v.h)) continue;
    const float4 val = __ldg(reinterpret_cast<const float4*>(x + int64_t(n) * v.sn + int64_t(c) * v.sc +
                                                              int64_t(h) * v.sh) + w4);
    const int wp = w4 * 4 + pad_w;  // staging column of input column 4*w4
    float* d = srow + q * SW;
    if (wp + 0 < SW) d[wp + 0] = val.x;
    if (wp + 1 < SW) d[wp + 1] = val.y;
    if (wp + 2 < SW) d[wp + 2] = val.z;
    if (wp + 3 < SW) d[wp + 3] = val.w;
  }
  __syncthreads();
  const int groups = Cp / 8, Cs = u * vv * C;
  const int64_t obase = int64_t(row) * W2 * Cp;
  for (int t = threadIdx.x; t < W2 * groups; t += blockDim.x) {
    const int w2 = t / groups, g = t - w2 * groups;
    float v8[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int cp = g * 8 + k;
      float val = 0.0f;
      if (cp < Cs) {
        const int qq = cp / C, c = cp - qq * C;  // qq = rh * v + rw
        const int rh = qq / vv, rw = qq - rh * vv;
        val = srow[(c * u + rh) * SW + w2 * vv + rw];
      }
      v8[k] = val;
    }
    const int64_t o = obase + int64_t(w2) * Cp + g * 8;
    store_split8<ES>(hi, lo, o, v8);
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

// Space-to-depth for dense NCHW input with even v and pad_w (AlexNet conv1:
// 4 x 4 phases, pad 2): one block = 64 consecutive super-pixels of one
// super-row (n, h') x all (rh, c); warp (rh, c) reads, per super-pixel, the v
// input columns [w'v - pad_w, w'v - pad_w + v) of row h'u + rh - pad_h as
// v/2 float2 loads (the warp covers 32 v consecutive floats: coalesced, an
// input byte is read once), stages them in shared memory as [pixel][Cs],
// then each thread splits and writes 16-byte hi / lo chunks of the
// contiguous 64 x Cp output block.  (32 super-pixels per block: 3.4 TB/s,
// latency-bound; measured per call under ncu.)
template <int V, int ES>
__global__ void __launch_bounds__(512) pack_act_s2d_quad_kernel(View4 v, const float* __restrict__ x,
                                                                int u, int pad_h, int pad_w, int H2,
                                                                int W2, int Cp, int nwb,
                                                                void* __restrict__ hi,
                                                                void* __restrict__ lo, int early = 0) {
  if (early) pdl_trigger();  // the next kernel does not read this one: let it launch now
  constexpr int PIX = 64;           // super-pixels per block (two per lane): ~2x the bytes in flight
  extern __shared__ float stile[];  // [PIX][Cp + 1]
  const int C = int(v.c), Cs = u * V * C, pitch = Cp + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t job = blockIdx.x;
  const uint32_t row = job / uint32_t(nwb), wb = job - row * uint32_t(nwb);
  const int n = int(row / uint32_t(H2)), h2 = int(row - uint32_t(n) * uint32_t(H2));
  for (int q = warp; q < u * C; q += nwarps) {  // q = rh * C + c
    const int rh = q / C, c = q - rh * C;
    const int h = h2 * u + rh - pad_h;
    const float* src = x + int64_t(n) * v.sn + int64_t(c) * v.sc + int64_t(h) * v.sh;
    const bool hok = unsigned(h) < unsigned(v.h);
    float2 val[2][V / 2];
#pragma unroll
    for (int s2 = 0; s2 < 2; s2++) {
      const int w2 = int(wb) * PIX + s2 * 32 + lane;
      const int w0 = w2 * V - pad_w;
#pragma unroll
      for (int k = 0; k < V / 2; k++) {
        const int w = w0 + 2 * k;  // pairs are all-in or all-out (even pad, even W)
        val[s2][k] = (w2 < W2 && hok && unsigned(w) < unsigned(v.w))
                         ? __ldg(reinterpret_cast<const float2*>(src + w))
                         : make_float2(0.0f, 0.0f);
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < 2; s2++) {
#pragma unroll
      for (int k = 0; k < V / 2; k++) {
        float* d = stile + (s2 * 32 + lane) * pitch + (rh * V + 2 * k) * C + c;
        d[0] = val[s2][k].x;
        d[C] = val[s2][k].y;
      }
    }
  }
  for (int t = threadIdx.x; t < PIX * (Cp - Cs); t += blockDim.x) {
    const int pi = t / (Cp - Cs), cc = Cs + t % (Cp - Cs);
    stile[pi * pitch + cc] = 0.0f;
  }
  __syncthreads();
  const int groups = Cp / 8;
  const int64_t obase = (int64_t(row) * W2 + int64_t(wb) * PIX) * Cp;
  for (int t = threadIdx.x; t < PIX * groups; t += blockDim.x) {
    const int pi = t / groups, g = t - pi * groups;
    if (int(wb) * PIX + pi >= W2) continue;
    float v8[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v8[k] = stile[pi * pitch + g * 8 + k];
    const int64_t o = obase + int64_t(pi) * Cp + g * 8;
    store_split8<ES>(hi, lo, o, v8);
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

// Tap folding: one thread per output pixel (n, h, q), walking its Cp folded
// channels (j, c) with running counters; loads are pixel-consecutive across
// the warp (w = q v + j - pad_w), writes 16-byte hi / lo chunks.
template <int ES>
__global__ void __launch_bounds__(256) pack_act_fold_kernel(View4 v, const float* __restrict__ x,
                                                            int S, int vv, int pad_w, int Q,
                                                            int Cp, void* __restrict__ hi,
                                                            void* __restrict__ lo,
                                                            uint32_t npix, MagicDiv dHQ,
                                                            MagicDiv dQ, int early = 0) {
  if (early) pdl_trigger();  // the next kernel does not read this one: let it launch now
  const int C = int(v.c), Cs = S * C;
  for (uint32_t pix = blockIdx.x * blockDim.x + threadIdx.x; pix < npix;
       pix += gridDim.x * blockDim.x) {
    uint32_t n, rem, h, q;
    mdivmod(pix, dHQ, n, rem);
    mdivmod(rem, dQ, h, q);
    const float* src = x + int64_t(n) * v.sn + int64_t(h) * v.sh;
    const int wb = int(q) * vv - pad_w;
    int c = 0, j = 0;
    for (int g = 0; g < Cp / 8; g++) {
      float v8[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        float val = 0.0f;
        if (g * 8 + k < Cs) {
          const int w = wb + j;
          if (unsigned(w) < unsigned(v.w)) val = __ldg(src + int64_t(c) * v.sc + int64_t(w) * v.sw);
          if (++c == C) {
            c = 0;
            ++j;
          }
        }
        v8[k] = val;
      }
      const int64_t o = int64_t(pix) * Cp + g * 8;
      store_split8<ES>(hi, lo, o, v8);
    }
  }
  pdl_trigger();  // this CTA is done: the call's next kernel may launch
}

}  // namespace

template <int ES>
static cudaError_t pack_act_s2d_t(const View4& v, const float* x, int u, int vv, int pad_h, int pad_w,
                         int H2, int W2, int Cp, void* hi, void* lo,
                         cudaStream_t st) {
  const int64_t npix = v.n * H2 * W2;
  if (npix >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
  {
    // float2 quads: dense rows, even v / pad_w / W / strides, 8-byte base
    const int nwb = int(ceil_div(W2, 64));
    const size_t sm = size_t(64) * (Cp + 1) * sizeof(float);
    const bool quad = (vv == 2 || vv == 4 || vv == 8) && v.sw == 1 && pad_w % 2 == 0 &&
                      v.w % 2 == 0 && v.sh % 2 == 0 && v.sc % 2 == 0 && v.sn % 2 == 0 &&
                      (reinterpret_cast<uintptr_t>(x) & 7) == 0 && sm <= 48 * 1024 &&
                      v.n * H2 * nwb < (int64_t(1) << 31) && !::dnnp::tune_env("DNNP_S2D_NO_QUAD");
    if (quad) {
      const unsigned grid = unsigned(v.n * H2 * nwb);
      const int threads = int(std::min<int64_t>(512, std::max<int64_t>(128, v.c * u * 32)));
      cudaError_t e;
      if (vv == 2)
        pack_act_s2d_quad_kernel<2, ES><<<grid, threads, sm, st>>>(v, x, u, pad_h, pad_w, H2, W2, Cp,
                                                               nwb, hi, lo, early_flag());
      else if (vv == 4)
        pack_act_s2d_quad_kernel<4, ES><<<grid, threads, sm, st>>>(v, x, u, pad_h, pad_w, H2, W2, Cp,
                                                               nwb, hi, lo, early_flag());
      else
        pack_act_s2d_quad_kernel<8, ES><<<grid, threads, sm, st>>>(v, x, u, pad_h, pad_w, H2, W2, Cp,
                                                               nwb, hi, lo, early_flag());
      e = cudaGetLastError();
      note_launch();
      return e;
    }
  }
  {
    const int SW = (W2 * vv + 3) & ~3;
    const size_t sm = size_t(v.c) * u * SW * sizeof(float);
    const bool dense = v.sw == 1 && v.sh == v.w && v.w % 4 == 0 && v.h * v.w <= v.sc &&
                       (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (v.sn % 4) == 0 &&
                       (v.sc % 4) == 0 && sm <= 48 * 1024 && W2 * vv >= v.w + pad_w &&
                       ::dnnp::tune_env("DNNP_S2D_DENSE") != nullptr;
    if (dense && v.n * H2 < (int64_t(1) << 31)) {
      pack_act_s2d_dense_kernel<ES><<<unsigned(v.n * H2), 256, sm, st>>>(v, x, u, vv, pad_h, pad_w, H2,
                                                                     W2, Cp, hi, lo);
      note_launch();
      return cudaGetLastError();
    }
  }
  if (::dnnp::tune_env("DNNP_S2D_TILE")) {
    const int64_t jobs = ceil_div(npix, kPix) * ceil_div(Cp, kCh);
    if (jobs >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    const unsigned grid = unsigned(std::min<int64_t>(jobs, int64_t(kNumSMs) * 32));
    pack_act_kernel<true, ES><<<grid, 256, 0, st>>>(v, x, Cp, hi, lo, npix,
                                                make_magic(uint32_t(H2 * W2)), make_magic(uint32_t(W2)),
                                                S2dGeom{u, vv, pad_h, pad_w});
    note_launch();
    return cudaGetLastError();
  }
  const size_t row_smem = size_t(W2) * (Cp + 1) * sizeof(float);
  if (::dnnp::tune_env("DNNP_S2D_ROWS") && row_smem <= 48 * 1024 && v.n * H2 < (int64_t(1) << 31)) {
    const unsigned grid = unsigned(std::min<int64_t>(v.n * H2, int64_t(kNumSMs) * 8));
    pack_act_s2d_row_kernel<ES><<<grid, 256, row_smem, st>>>(v, x, u, vv, pad_h, pad_w, H2, W2, Cp, hi,
                                                         lo);
    note_launch();
    return cudaGetLastError();
  }
  pack_act_s2d_kernel<ES><<<grid_for(npix, 256, 8), 256, 0, st>>>(
      v, x, u, vv, pad_h, pad_w, H2, W2, Cp, hi, lo, npix, make_magic(uint32_t(H2 * W2)),
      make_magic(uint32_t(W2)), early_flag());
  note_launch();
  return cudaGetLastError();
}

cudaError_t pack_act_s2d(const View4& v, const float* x, int u, int vv, int pad_h, int pad_w,
                         int H2, int W2, int Cp, void* hi, void* lo,
                         cudaStream_t st, int es) {
  return es == 4 ? pack_act_s2d_t<4>(v, x, u, vv, pad_h, pad_w, H2, W2, Cp, hi, lo, st) : pack_act_s2d_t<2>(v, x, u, vv, pad_h, pad_w, H2, W2, Cp, hi, lo, st);
}

struct ArenaState {
  std::recursive_mutex mu;
  void* base = nullptr;
  size_t cap = 0, off = 0, high = 0;
  size_t fb = 0;  // outstanding fallback bytes (allocated outside the arena)
  int depth = 0;
};

static std::mutex g_arena_map_mu;
static std::map<std::pair<int, cudaStream_t>, ArenaState*> g_arenas;

static ArenaState* arena_for(cudaStream_t st) {
  std::mutex& map_mu = g_arena_map_mu;
  auto& arenas = g_arenas;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(map_mu);
  ArenaState*& a = arenas[{dev, st}];
  if (!a) {
    pool_keep_memory();
    a = new ArenaState;  // lives for the process
  }
  return a;
}

// caller-supplied workspace override (thread local, LIFO like the arena)
struct UserWs {
  char* base = nullptr;
  size_t cap = 0, off = 0, high = 0;
  bool active = false;
  bool dry = false;  // workspace query: carve-outs from a fake base, nothing runs
};
static thread_local UserWs g_uws;

// Fake, 1024-aligned device address the dry run hands out: only ever
// encoded into tensor maps and kernel parameters of a captured (never
// launched) graph, never dereferenced.
static char* const kDryBase = reinterpret_cast<char*>(uintptr_t(1) << 44);

void dry_run_begin() {
  g_uws = UserWs{};
  g_uws.base = kDryBase;
  g_uws.cap = ~size_t(0) >> 2;
  g_uws.active = true;
  g_uws.dry = true;
}

bool dry_run() { return g_uws.active && g_uws.dry; }

void user_workspace_begin(void* base, size_t bytes) {
  g_uws.base = static_cast<char*>(base);
  g_uws.cap = bytes;
  g_uws.off = g_uws.high = 0;
  g_uws.active = true;
}

void user_workspace_end(size_t* need) {
  if (need) *need = g_uws.high;
  g_uws = UserWs{};
}

Workspace::Workspace(cudaStream_t s) : st(s), a_(arena_for(s)) {
  a_->mu.lock();
  a_->depth++;
  saved_off_ = g_uws.active ? g_uws.off : a_->off;
}

cudaError_t Workspace::alloc(size_t bytes) {
  bytes = (bytes + 1023) & ~size_t(1023);
  if (g_uws.active) {
    // 1024-byte aligned carve-outs of the caller's buffer
    const uintptr_t b = (reinterpret_cast<uintptr_t>(g_uws.base) + 1023) & ~uintptr_t(1023);
    const size_t skew = b - reinterpret_cast<uintptr_t>(g_uws.base);
    g_uws.high = std::max(g_uws.high, skew + g_uws.off + bytes);
    if (skew + g_uws.off + bytes > g_uws.cap) return cudaErrorMemoryAllocation;
    p = reinterpret_cast<char*>(b) + g_uws.off;
    g_uws.off += bytes;
    return cudaSuccess;
  }
  // the high-water mark counts fallback bytes too, so a call's footprint is
  // right even before the arena has grown to it
  a_->high = std::max(a_->high, a_->off + a_->fb + bytes);
  if (a_->base && a_->off + bytes <= a_->cap) {
    p = static_cast<char*>(a_->base) + a_->off;
    a_->off += bytes;
    return cudaSuccess;
  }
  fallback_ = true;
  fb_bytes_ = bytes;
  a_->fb += bytes;
  return cudaMallocFromPoolAsync(&p, bytes, lib_pool(), st);
}

Workspace::~Workspace() {
  if (g_uws.active) {
    g_uws.off = saved_off_;
    --a_->depth;
    a_->mu.unlock();
    return;
  }
  if (fallback_ && p) cudaFreeAsync(p, st);
  if (fallback_) a_->fb -= fb_bytes_;
  a_->off = saved_off_;
  if (--a_->depth == 0 && a_->high > a_->cap) {
    if (a_->base) cudaFreeAsync(a_->base, st);
    const size_t ncap = a_->high + a_->high / 4;
    if (cudaMallocFromPoolAsync(&a_->base, ncap, lib_pool(), st) == cudaSuccess) {
      a_->cap = ncap;
    } else {
      cudaGetLastError();
      a_->base = nullptr;
      a_->cap = 0;
    }
  }
  a_->mu.unlock();
}

void scratch_measure_begin(cudaStream_t st) {
  ArenaState* a = arena_for(st);
  std::lock_guard<std::recursive_mutex> g(a->mu);
  a->high = a->off;
}

size_t scratch_measure_end(cudaStream_t st) {
  ArenaState* a = arena_for(st);
  std::lock_guard<std::recursive_mutex> g(a->mu);
  return a->high - a->off;
}

// ---- main-kernel timing (bench roofline) ----------------------------------
struct KTime {
  int tag;
  cudaEvent_t a, b;
};
static std::mutex g_kt_mu;
static std::vector<KTime> g_kt;
static std::atomic<int> g_kt_on{0};

// Events come from a pool (created once, reused after every reset); inside
// a CUDA-graph capture they are recorded as external event nodes, so a
// replayed graph timestamps its kernels like an eager run.
static std::vector<cudaEvent_t> g_kt_pool;
static size_t g_kt_next = 0;

static cudaEvent_t kt_event() {
  if (g_kt_next == g_kt_pool.size()) {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    g_kt_pool.push_back(e);
  }
  return g_kt_pool[g_kt_next++];
}

static void kt_record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else
    cudaEventRecord(e, st);
}

static int g_kt_sel = -1;     // time only the launch with this ordinal (-1: all)
static int g_kt_count = 0;    // main-kernel launches since the last reset
static bool g_kt_open = false;

void ktime_begin(cudaStream_t st, int tag) {
  if (!g_kt_on.load()) return;
  std::lock_guard<std::mutex> g(g_kt_mu);
  const int ord = g_kt_count++;
  g_kt_open = g_kt_sel < 0 || ord == g_kt_sel;
  if (!g_kt_open) return;
  KTime k{tag, kt_event(), kt_event()};
  kt_record(k.a, st);
  g_kt.push_back(k);
}

void ktime_end(cudaStream_t st) {
  if (!g_kt_on.load()) return;
  std::lock_guard<std::mutex> g(g_kt_mu);
  if (g_kt_open && !g_kt.empty()) kt_record(g_kt.back().b, st);
  g_kt_open = false;
}

struct ScratchScope {
  cudaStream_t st;
  std::vector<Workspace*> ws;  // nested, closed in reverse order
};

ScratchScope* scratch_open(cudaStream_t st) { return new ScratchScope{st, {}}; }

cudaError_t scratch_alloc(ScratchScope* s, size_t bytes, void** p) {
  Workspace* w = new Workspace(s->st);
  s->ws.push_back(w);
  const cudaError_t e = w->alloc(bytes);
  *p = w->p;
  return e;
}

void scratch_close(ScratchScope* s) {
  if (!s) return;
  for (auto it = s->ws.rbegin(); it != s->ws.rend(); ++it) delete *it;
  delete s;
}

// The library's own stream-ordered pool per device (the process' default
// pool is left alone, so torch's caching allocator and the host application
// see their memory returned): freed scratch above kPoolKeep bytes goes back
// to the device at the next synchronisation; the grow-only arenas are live
// allocations of this pool and are not affected.
constexpr uint64_t kPoolKeep = uint64_t(256) << 20;

cudaMemPool_t lib_pool() {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPool_t pool = nullptr;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
    uint64_t thr = kPoolKeep;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  } else {
    cudaGetLastError();
    cudaDeviceGetDefaultMemPool(&pool, dev);  // untouched attributes
  }
  pools[dev] = pool;
  return pool;
}

void pool_keep_memory() { (void)lib_pool(); }

// Encoded tensor maps are cached by their full argument list (base address
// included): a repeated call on the same buffers -- every step of a training
// loop, the arena's planes at the same offsets -- skips the driver encode
// (~1 us each, four per convolution).  FIFO eviction past kTmapCache entries.
constexpr size_t kTmapCache = 512;
struct TmapCache {
  std::mutex mu;
  std::unordered_map<std::string, CUtensorMap> map;
  std::deque<std::string> order;
};
static TmapCache& tmap_cache() {
  static TmapCache* c = new TmapCache;  // lives for the process
  return *c;
}
template <class Key, class F>
static cudaError_t cached_tmap(CUtensorMap* out, const Key& k, F&& encode) {
  std::string key(reinterpret_cast<const char*>(&k), sizeof(Key));
  TmapCache& c = tmap_cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.map.find(key);
    if (it != c.map.end()) {
      *out = it->second;
      return cudaSuccess;
    }
  }
  const cudaError_t e = encode(out);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> g(c.mu);
    if (c.map.size() >= kTmapCache) {
      c.map.erase(c.order.front());
      c.order.pop_front();
    }
    if (c.map.emplace(key, *out).second) c.order.push_back(key);
  }
  return e;
}

static CUtensorMapDataType tmap_dtype(int es) {
  return es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
}

static cudaError_t encode_tmap_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                                  uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows,
                                  CUtensorMapSwizzle swizzle, int es);

cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                         uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows,
                         CUtensorMapSwizzle swizzle, int es) {
  struct K {
    int kind;
    int es;
    const void* base;
    uint64_t cols, rows, pitch;
    uint32_t bc, br;
    int sw;
  } k;
  memset(&k, 0, sizeof k);
  k.kind = 2; k.es = es; k.base = base; k.cols = cols; k.rows = rows; k.pitch = pitch_elems;
  k.bc = box_cols; k.br = box_rows; k.sw = int(swizzle);
  return cached_tmap(map, k, [&](CUtensorMap* m) {
    return encode_tmap_2d(m, base, cols, rows, pitch_elems, box_cols, box_rows, swizzle, es);
  });
}

static cudaError_t encode_tmap_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                                  uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows,
                                  CUtensorMapSwizzle swizzle, int es) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
    fn = reinterpret_cast<Fn>(p);
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {pitch_elems * cuuint64_t(es)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, tmap_dtype(es), 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static cudaError_t encode_tmap_3d(CUtensorMap* map, const void* base, const uint64_t dims[3],
                                  const uint64_t strides_bytes[2], const uint32_t box[3],
                                  CUtensorMapSwizzle swizzle, int es);

cudaError_t make_tmap_3d(CUtensorMap* map, const void* base, const uint64_t dims[3],
                         const uint64_t strides_bytes[2], const uint32_t box[3],
                         CUtensorMapSwizzle swizzle, int es) {
  struct K {
    int kind;
    int es;
    const void* base;
    uint64_t d[3], s[2];
    uint32_t b[3];
    int sw;
  } k;
  memset(&k, 0, sizeof k);
  k.kind = 3; k.es = es; k.base = base;
  for (int i = 0; i < 3; i++) k.d[i] = dims[i], k.b[i] = box[i];
  k.s[0] = strides_bytes[0]; k.s[1] = strides_bytes[1];
  k.sw = int(swizzle);
  return cached_tmap(map, k, [&](CUtensorMap* m) {
    return encode_tmap_3d(m, base, dims, strides_bytes, box, swizzle, es);
  });
}

static cudaError_t encode_tmap_3d(CUtensorMap* map, const void* base, const uint64_t dims[3],
                                  const uint64_t strides_bytes[2], const uint32_t box[3],
                                  CUtensorMapSwizzle swizzle, int es) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
    fn = reinterpret_cast<Fn>(p);
  }
  const cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  const cuuint64_t st[2] = {strides_bytes[0], strides_bytes[1]};
  const cuuint32_t b[3] = {box[0], box[1], box[2]};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, tmap_dtype(es), 3, const_cast<void*>(base), d, st, b, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static cudaError_t encode_tmap_im2col(CUtensorMap* map, const void* base, const Im2colGeom& g,
                                      CUtensorMapSwizzle swizzle, int es);

cudaError_t make_tmap_im2col(CUtensorMap* map, const void* base, const Im2colGeom& g,
                             CUtensorMapSwizzle swizzle, int es) {
  struct K {
    int kind;
    int es;
    const void* base;
    Im2colGeom g;
    int sw;
  } k;
  memset(&k, 0, sizeof k);
  k.kind = 4; k.es = es; k.base = base; k.g = g; k.sw = int(swizzle);
  return cached_tmap(map, k, [&](CUtensorMap* m) {
    return encode_tmap_im2col(m, base, g, swizzle, es);
  });
}

static cudaError_t encode_tmap_im2col(CUtensorMap* map, const void* base, const Im2colGeom& g,
                                      CUtensorMapSwizzle swizzle, int es) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                          const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
    fn = reinterpret_cast<Fn>(p);
  }
  const cuuint64_t dims[4] = {cuuint64_t(g.C), cuuint64_t(g.W), cuuint64_t(g.H), cuuint64_t(g.N)};
  const cuuint64_t eb = cuuint64_t(es);
  const cuuint64_t strides[3] = {cuuint64_t(g.C) * eb, cuuint64_t(g.C) * eb * g.W,
                                 cuuint64_t(g.C) * eb * g.W * g.H};
  const int lower[2] = {g.lower_w, g.lower_h};  // W first (innermost spatial dim)
  const int upper[2] = {g.upper_w, g.upper_h};
  const cuuint32_t estr[4] = {1, cuuint32_t(g.stride_w), cuuint32_t(g.stride_h), 1};
  CUresult r = fn(map, tmap_dtype(es), 4, const_cast<void*>(base), dims, strides,
                  lower, upper, cuuint32_t(g.cpp), cuuint32_t(g.ppc), estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

struct PackedRef {
  const float* src = nullptr;
  View4 v{};
  int Cp = 0;
  int es = 2;
  const void* hi = nullptr;
  const void* lo = nullptr;
};
static thread_local PackedRef g_packed;

void packed_set(const float* src, const View4& v, int Cp, const void* hi, const void* lo, int es) {
  g_packed = PackedRef{src, v, Cp, es, hi, lo};
}

bool packed_get(const float* src, const View4& v, int Cp, const void** hi, const void** lo,
                int es) {
  const PackedRef& r = g_packed;
  if (!r.src || r.src != src || r.Cp != Cp || r.es != es || r.v.n != v.n || r.v.c != v.c ||
      r.v.h != v.h || r.v.w != v.w || r.v.sn != v.sn || r.v.sc != v.sc || r.v.sh != v.sh ||
      r.v.sw != v.sw)
    return false;
  *hi = r.hi;
  *lo = r.lo;
  return true;
}

void packed_clear() { g_packed = PackedRef{}; }

cudaError_t shared_dy_pack(ScratchScope* sc, const View4& v, const float* dy, int Cp,
                           cudaStream_t st) {
  const size_t elems = size_t(v.n) * v.h * v.w * Cp;
  void* buf = nullptr;
  cudaError_t e = scratch_alloc(sc, elems * 4, &buf);
  if (e != cudaSuccess) return e;
  auto* hi = static_cast<__nv_bfloat16*>(buf);  // BF16x3 planes (the default math)
  auto* lo = hi + elems;
  if ((e = pack_act(v, dy, Cp, hi, lo, st)) != cudaSuccess) return e;
  packed_set(dy, v, Cp, hi, lo, 2);
  return cudaSuccess;
}

void shared_dy_clear() { packed_clear(); }

bool fold_taps(int64_t C, int64_t S, int64_t u, int64_t v, bool s2d) {
  if (s2d || ::dnnp::tune_env("DNNP_TC_NO_FOLD") || S < 2 || S * C > 64 || v > 8) return false;
  // reduction per vertical tap: folded S*C padded once vs C padded S times
  const int64_t folded = ceil_div(S * C, 16) * 16, plain = S * ceil_div(C, 16) * 16;
  return folded * 4 <= plain * 3;
}

template <int ES>
static cudaError_t pack_act_fold_t(const View4& v, const float* x, int S, int vv, int pad_w, int Q, int Cp,
                          void* hi, void* lo, cudaStream_t st) {
  const int64_t npix = v.n * v.h * Q;
  if (npix >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
  pack_act_fold_kernel<ES><<<grid_for(npix, 256, 8), 256, 0, st>>>(
      v, x, S, vv, pad_w, Q, Cp, hi, lo, uint32_t(npix), make_magic(uint32_t(v.h * Q)),
      make_magic(uint32_t(Q)), early_flag());
  note_launch();
  return cudaGetLastError();
}

cudaError_t pack_act_fold(const View4& v, const float* x, int S, int vv, int pad_w, int Q, int Cp,
                          void* hi, void* lo, cudaStream_t st, int es) {
  return es == 4 ? pack_act_fold_t<4>(v, x, S, vv, pad_w, Q, Cp, hi, lo, st) : pack_act_fold_t<2>(v, x, S, vv, pad_w, Q, Cp, hi, lo, st);
}

template <int ES>
static cudaError_t pack_act_t(const View4& v, const float* x, int Cp, void* hi, void* lo,
                     cudaStream_t st) {
  const int64_t npix = v.n * v.h * v.w;
  if (npix >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
  if (Cp <= 16) {
    pack_act_small_kernel<ES><<<grid_for(npix, 256, 8), 256, 0, st>>>(
        v, x, Cp, hi, lo, npix, make_magic(uint32_t(v.h * v.w)), make_magic(uint32_t(v.w)), early_flag());
    note_launch();
    return cudaGetLastError();
  }
  const int pj = ::dnnp::tune_env("DNNP_PACK_PIX") ? atoi(::dnnp::tune_env("DNNP_PACK_PIX")) : 64;
  if (pj == 64 || pj == 128) {
    const int64_t jobs = ceil_div(npix, int64_t(pj)) * ceil_div(Cp, kCh);
    if (jobs >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    const unsigned grid = unsigned(std::min<int64_t>(jobs, int64_t(kNumSMs) * 16));
    if (pj == 64)
      pack_act_wide_kernel<64, ES><<<grid, 256, 0, st>>>(v, x, Cp, hi, lo, uint32_t(npix),
                                                     make_magic(uint32_t(v.h * v.w)),
                                                     make_magic(uint32_t(v.w)), Border{0, 0, 0, 0},
                                                     early_flag());
    else
      pack_act_wide_kernel<128, ES><<<grid, 256, 0, st>>>(v, x, Cp, hi, lo, uint32_t(npix),
                                                      make_magic(uint32_t(v.h * v.w)),
                                                      make_magic(uint32_t(v.w)), Border{0, 0, 0, 0},
                                                      early_flag());
    note_launch();
    return cudaGetLastError();
  }
  const int64_t jobs = ceil_div(npix, kPix) * ceil_div(Cp, kCh);
  if (jobs >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  const unsigned grid = unsigned(std::min<int64_t>(jobs, int64_t(kNumSMs) * 32));
  pack_act_kernel<false, ES><<<grid, 256, 0, st>>>(v, x, Cp, hi, lo, npix,
                                               make_magic(uint32_t(v.h * v.w)),
                                               make_magic(uint32_t(v.w)), S2dGeom{1, 1, 0, 0});
  note_launch();
  return cudaGetLastError();
}

template <int ES>
static cudaError_t pack_act_border_t(const View4& v, const float* x, int Cp, int top, int left,
                                     int Hp, int Wp, void* hi, void* lo, cudaStream_t st) {
  const int64_t npix = v.n * Hp * Wp;
  const int64_t jobs = ceil_div(npix, int64_t(64)) * ceil_div(Cp, kCh);
  if (npix >= (int64_t(1) << 32) || jobs >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  const unsigned grid = unsigned(std::min<int64_t>(jobs, int64_t(kNumSMs) * 16));
  pack_act_wide_kernel<64, ES><<<grid, 256, 0, st>>>(v, x, Cp, hi, lo, uint32_t(npix),
                                                     make_magic(uint32_t(Hp * Wp)),
                                                     make_magic(uint32_t(Wp)),
                                                     Border{top, left, Hp, Wp}, early_flag());
  note_launch();
  return cudaGetLastError();
}

cudaError_t pack_act_border(const View4& v, const float* x, int Cp, int top, int left, int Hp,
                            int Wp, void* hi, void* lo, cudaStream_t st, int es) {
  return es == 4 ? pack_act_border_t<4>(v, x, Cp, top, left, Hp, Wp, hi, lo, st)
                 : pack_act_border_t<2>(v, x, Cp, top, left, Hp, Wp, hi, lo, st);
}

void pack_trigger_early(bool on) { t_pack_early = on && !::dnnp::tune_env("DNNP_PACK_LATE"); }

cudaError_t pack_act(const View4& v, const float* x, int Cp, void* hi, void* lo,
                     cudaStream_t st, int es) {
  return es == 4 ? pack_act_t<4>(v, x, Cp, hi, lo, st) : pack_act_t<2>(v, x, Cp, hi, lo, st);
}

}  // namespace tc
}  // namespace dnnp

// additive C entry: the largest scratch footprint (bytes) any operation
// took from the per-stream arenas since the last reset -- the device
// counterpart of the reference's scratch allocation log (scratch.py,
// test_scratch.py): implicit kernels need the packed operands only, the
// explicit engine also the lowered data matrix.
extern "C" int64_t dnnp_scratch_high_water(int reset) {
  using namespace dnnp::tc;
  std::vector<ArenaState*> all;
  {
    // copy under the map lock, then lock arenas one at a time (an op holding
    // its arena may be waiting for the map lock in a nested Workspace)
    std::lock_guard<std::mutex> g(g_arena_map_mu);
    for (auto& kv : g_arenas) all.push_back(kv.second);
  }
  size_t high = 0;
  for (ArenaState* a : all) {
    std::lock_guard<std::recursive_mutex> ga(a->mu);
    high = std::max(high, a->high);
    if (reset) a->high = a->off;
  }
  return int64_t(high);
}

// additive C entries: time every main GEMM kernel (CUDA events around the
// launch on the caller's stream) so a benchmark can report per-kernel
// durations measured inside its own timed region
extern "C" int dnnp_kernel_timing(int enable) {
  using namespace dnnp::tc;
  std::lock_guard<std::mutex> g(g_kt_mu);
  g_kt.clear();  // the events return to the pool
  g_kt_next = 0;
  g_kt_count = 0;
  g_kt_open = false;
  // enable: 1 = every main GEMM launch; k >= 2 = only the launch with
  // ordinal k - 2 (0-based, since this reset) -- two event nodes instead of
  // two per kernel when a replayed graph times its dominant kernel
  g_kt_sel = enable >= 2 ? enable - 2 : -1;
  g_kt_on.store(enable ? 1 : 0);
  return 0;
}

// fills up to max (duration ms, kernel tag) pairs in launch order and
// returns how many kernels were timed; synchronizes on the recorded events
extern "C" int dnnp_kernel_times(float* ms, int* tags, int max) {
  using namespace dnnp::tc;
  std::lock_guard<std::mutex> g(g_kt_mu);
  int n = 0;
  for (auto& k : g_kt) {
    if (n < max) {
      float t = -1.0f;
      if (cudaEventSynchronize(k.b) == cudaSuccess) cudaEventElapsedTime(&t, k.a, k.b);
      if (ms) ms[n] = t;
      if (tags) tags[n] = k.tag;
    }
    n++;
  }
  return n;
}
