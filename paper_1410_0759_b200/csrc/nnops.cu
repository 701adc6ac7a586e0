// Bandwidth-bound primitives on strided 4-D views: activation, softmax,
// pooling (forward + backward), transform, add_broadcast and the conv bias
// gradient.  Reference semantics: pkg/src/dnnp/nnops.py, tensor.py:241-271,
// conv.py:754-760.
//
// Element-wise ops run either over the raw span (all operands share one dense
// layout: 128-bit vectorised grid-stride loop) or over rows of the innermost
// output dimension (any strides: one warp per row, lanes along the row).
// Roundings follow numpy's evaluation order with explicit _rn intrinsics so
// that e.g. activation backward, transform and pooling backward are bit-exact.
#include <atomic>
#include <type_traits>
#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "tc_common.cuh"

namespace dnnp {

static std::atomic<long long> g_launches{0};
void note_launch(int count) {
  if (!tc::dry_run()) g_launches += count;  // a workspace query launches nothing
}

MagicDiv make_magic(uint32_t d) {
  // reference intdiv.py:74-101 (Hacker's Delight unsigned magic numbers)
  MagicDiv m{d, 1, 0, 0};
  if (d <= 1) return m;
  const unsigned __int128 word = (unsigned __int128)1 << 32;
  const unsigned __int128 nc = (word / d) * d - 1;
  unsigned __int128 mul = 0;
  int p = 32;
  for (; p <= 64; p++) {
    unsigned __int128 two_p = (unsigned __int128)1 << p;
    unsigned __int128 rem = (two_p - 1) % d;
    if (two_p > nc * (d - 1 - rem)) {
      mul = (two_p + d - 1 - rem) / d;
      break;
    }
  }
  m.shift = uint32_t(p - 32);
  if (mul < word) {
    m.mul = uint32_t(mul);
    m.add = 0;
  } else {
    m.mul = uint32_t(mul - word);
    m.add = 1;
  }
  return m;
}

// ------------------------------------------------------------ iteration

// An element-wise launch over up to three operands sharing extents; dims are
// permuted so the output's finest-stride dim is innermost.
struct EwGeom {
  int64_t ext[4];
  int64_t st[3][4];
  int64_t rows;   // ext[0]*ext[1]*ext[2]
  MagicDiv d2, d1;  // row decode: r -> (i0, i1, i2)
  int use_magic;
  int64_t chunks;   // pieces of length kEwChunk per row (long merged rows)
  int vec;          // innermost stride 1 for every operand and 16-byte aligned rows
};
constexpr int64_t kEwChunk = 2048;

static EwGeom make_ew(const View4* views[3], int nops, int out_index) {
  const View4& o = *views[out_index];
  int64_t oe[4] = {o.n, o.c, o.h, o.w};
  int64_t os[4] = {o.sn, o.sc, o.sh, o.sw};
  int perm[4] = {0, 1, 2, 3};
  // stable sort by |stride| descending, extent-1 dims pushed outward
  for (int i = 0; i < 4; i++)
    for (int j = i + 1; j < 4; j++) {
      auto key = [&](int d) { return oe[d] == 1 ? INT64_MAX : (os[d] < 0 ? -os[d] : os[d]); };
      if (key(perm[j]) > key(perm[i])) std::swap(perm[i], perm[j]);
    }
  EwGeom g;
  for (int k = 0; k < 4; k++) g.ext[k] = oe[perm[k]];
  for (int op = 0; op < 3; op++) {
    if (op >= nops) {
      for (int k = 0; k < 4; k++) g.st[op][k] = 0;
      continue;
    }
    const View4& v = *views[op];
    int64_t s[4] = {v.sn, v.sc, v.sh, v.sw};
    int64_t e[4] = {v.n, v.c, v.h, v.w};
    for (int k = 0; k < 4; k++) g.st[op][k] = e[perm[k]] == 1 ? 0 : s[perm[k]];
  }
  // merge adjacent dims that are contiguous for every operand (a channel
  // slice of an NCHW parent becomes one long row per image)
  for (int k = 2; k >= 0; k--) {
    if (g.ext[k] == 1) continue;
    bool ok = true;
    for (int op = 0; op < nops; op++)
      if (g.st[op][k] != g.st[op][k + 1] * g.ext[k + 1]) ok = false;
    if (!ok) continue;
    // fold dim k into k+1, shift the outer dims in (extent-1 dim at the top)
    g.ext[k + 1] *= g.ext[k];
    for (int j = k; j > 0; j--) {
      g.ext[j] = g.ext[j - 1];
      for (int op = 0; op < 3; op++) g.st[op][j] = g.st[op][j - 1];
    }
    g.ext[0] = 1;
    for (int op = 0; op < 3; op++) g.st[op][0] = 0;
    k++;  // re-examine position k (now the next outer dim) against the merged one
  }
  g.rows = g.ext[0] * g.ext[1] * g.ext[2];
  g.chunks = (g.ext[3] + kEwChunk - 1) / kEwChunk;
  g.vec = 1;
  for (int op = 0; op < nops; op++)
    if (g.st[op][3] != 1 || g.st[op][0] % 4 || g.st[op][1] % 4 || g.st[op][2] % 4) g.vec = 0;
  g.use_magic = g.rows < (int64_t(1) << 32);
  g.d2 = make_magic(uint32_t(g.ext[2]));
  g.d1 = make_magic(uint32_t(g.ext[1]));
  return g;
}

// shared dense layout: identical strides and span == size
static bool same_dense(const View4* views[3], int nops) {
  const View4& a = *views[0];
  for (int i = 1; i < nops; i++) {
    const View4& b = *views[i];
    if (a.sn != b.sn || a.sc != b.sc || a.sh != b.sh || a.sw != b.sw) return false;
  }
  int64_t e[4] = {a.n, a.c, a.h, a.w}, s[4] = {a.sn, a.sc, a.sh, a.sw};
  int64_t maxo = 0;
  for (int k = 0; k < 4; k++) maxo += (e[k] - 1) * (s[k] > 0 ? s[k] : 0);
  for (int k = 0; k < 4; k++)
    if (s[k] < 0) return false;
  return maxo + 1 == a.size();
}

// Strided rows: work item = (row, chunk of kEwChunk innermost elements), one
// warp per item; when every operand's rows are contiguous and 16-byte aligned
// (g.vec and aligned bases, checked on the host) lanes move 16-byte vectors.
template <typename Op, typename T>
__global__ void __launch_bounds__(256) ew_rows_kernel(EwGeom g, const T* __restrict__ a,
                                                      const T* __restrict__ b, T* out, Op op) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t items = g.rows * g.chunks;
  for (int64_t it = warp; it < items; it += nwarps) {
    const int64_t r = it / g.chunks, ch = it - r * g.chunks;
    int64_t i0, i1, i2;
    if (g.use_magic) {
      uint32_t q, rem;
      mdivmod(uint32_t(r), g.d2, q, rem);
      i2 = rem;
      uint32_t q2, rem2;
      mdivmod(q, g.d1, q2, rem2);
      i1 = rem2;
      i0 = q2;
    } else {
      i2 = r % g.ext[2];
      int64_t t = r / g.ext[2];
      i1 = t % g.ext[1];
      i0 = t / g.ext[1];
    }
    int64_t base[3];
#pragma unroll
    for (int k = 0; k < 3; k++) base[k] = i0 * g.st[k][0] + i1 * g.st[k][1] + i2 * g.st[k][2];
    const int64_t j0 = ch * kEwChunk, j1 = min(g.ext[3], j0 + kEwChunk);
    if (g.vec) {
      constexpr int V = 16 / sizeof(T);
      using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
      // batches of 4 vectors per lane, all loaded before any store
      constexpr int NV = int(kEwChunk / (32 * V)), U = 4;
      const int64_t jend = j1 - (j1 - j0) % V;
      for (int u0 = 0; u0 < NV; u0 += U) {
        Vec va[U], vb[U], vo[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int64_t j = j0 + (int64_t(u0 + u) * 32 + lane) * V;
          if (j < jend) {
            if (a) va[u] = *reinterpret_cast<const Vec*>(a + base[0] + j);
            if (b) vb[u] = *reinterpret_cast<const Vec*>(b + base[1] + j);
            if (Op::kReadsOut) vo[u] = *reinterpret_cast<const Vec*>(out + base[2] + j);
          }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int64_t j = j0 + (int64_t(u0 + u) * 32 + lane) * V;
          if (j < jend) {
            const T* pa = reinterpret_cast<const T*>(&va[u]);
            const T* pb = reinterpret_cast<const T*>(&vb[u]);
            T* po = reinterpret_cast<T*>(&vo[u]);
#pragma unroll
            for (int k = 0; k < V; k++)
              po[k] = op(a ? pa[k] : T(0), b ? pb[k] : T(0), Op::kReadsOut ? po[k] : T(0));
            *reinterpret_cast<Vec*>(out + base[2] + j) = vo[u];
          }
        }
      }
      const int64_t tail = j1 - (j1 - j0) % V;  // ragged end of the chunk
      for (int64_t j = tail + lane; j < j1; j += 32) {
        T* po = out + base[2] + j;
        *po = op(a ? a[base[0] + j] : T(0), b ? b[base[1] + j] : T(0), Op::kReadsOut ? *po : T(0));
      }
    } else {
      for (int64_t j = j0 + lane; j < j1; j += 32) {
        T va = a ? a[base[0] + j * g.st[0][3]] : T(0);
        T vb = b ? b[base[1] + j * g.st[1][3]] : T(0);
        T* po = out + base[2] + j * g.st[2][3];
        *po = op(va, vb, Op::kReadsOut ? *po : T(0));
      }
    }
  }
}

// Dense elementwise: every lane moves U 16-byte vectors per iteration,
// all loads issued before any store (out may alias an input element-wise, so
// the batching is explicit rather than left to __restrict__).
template <typename Op, typename T>
__global__ void __launch_bounds__(256) ew_dense_kernel(int64_t n, const T* __restrict__ a,
                                                       const T* __restrict__ b, T* out, Op op,
                                                       int vec) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  if (vec) {
    constexpr int V = 16 / sizeof(T);
    constexpr int U = 4;
    using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    const int64_t nv = n / V;
    int64_t i = tid;
    for (; i + (U - 1) * nth < nv; i += U * nth) {
      Vec va[U], vb[U], vo[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (a) va[u] = reinterpret_cast<const Vec*>(a)[i + u * nth];
        if (b) vb[u] = reinterpret_cast<const Vec*>(b)[i + u * nth];
        if (Op::kReadsOut) vo[u] = reinterpret_cast<const Vec*>(out)[i + u * nth];
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const T* pa = reinterpret_cast<const T*>(&va[u]);
        const T* pb = reinterpret_cast<const T*>(&vb[u]);
        T* po = reinterpret_cast<T*>(&vo[u]);
#pragma unroll
        for (int k = 0; k < V; k++)
          po[k] = op(a ? pa[k] : T(0), b ? pb[k] : T(0), Op::kReadsOut ? po[k] : T(0));
      }
#pragma unroll
      for (int u = 0; u < U; u++) reinterpret_cast<Vec*>(out)[i + u * nth] = vo[u];
    }
    for (; i < nv; i += nth) {
      Vec va, vb, vo;
      if (a) va = reinterpret_cast<const Vec*>(a)[i];
      if (b) vb = reinterpret_cast<const Vec*>(b)[i];
      if (Op::kReadsOut) vo = reinterpret_cast<const Vec*>(out)[i];
      const T* pa = reinterpret_cast<const T*>(&va);
      const T* pb = reinterpret_cast<const T*>(&vb);
      T* po = reinterpret_cast<T*>(&vo);
#pragma unroll
      for (int k = 0; k < V; k++)
        po[k] = op(a ? pa[k] : T(0), b ? pb[k] : T(0), Op::kReadsOut ? po[k] : T(0));
      reinterpret_cast<Vec*>(out)[i] = vo;
    }
    for (int64_t j = nv * V + tid; j < n; j += nth)
      out[j] = op(a ? a[j] : T(0), b ? b[j] : T(0), Op::kReadsOut ? out[j] : T(0));
  } else {
    for (int64_t i = tid; i < n; i += nth)
      out[i] = op(a ? a[i] : T(0), b ? b[i] : T(0), Op::kReadsOut ? out[i] : T(0));
  }
}

template <typename Op, typename T>
static cudaError_t run_ew(const View4& va, const T* a, const View4* vb, const T* b,
                          const View4& vo, T* out, Op op, cudaStream_t st) {
  const View4* views[3] = {&va, vb ? vb : &va, &vo};
  const View4* dense_views[3] = {&va, vb ? vb : &vo, &vo};
  const int64_t n = vo.size();
  if (n == 0) return cudaSuccess;
  if (same_dense(dense_views, 3)) {
    bool aligned = (reinterpret_cast<uintptr_t>(a) % 16 == 0) &&
                   (!b || reinterpret_cast<uintptr_t>(b) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    const int V = 16 / sizeof(T);
    unsigned grid = grid_for(aligned ? ceil_div(n, V) : n, 256, 8);
    ew_dense_kernel<Op, T><<<grid, 256, 0, st>>>(n, a, b, out, op, aligned ? 1 : 0);
  } else {
    EwGeom g = make_ew(views, vb ? 3 : 3, 2);
    if (!vb)
      for (int k = 0; k < 4; k++) g.st[1][k] = 0;
    if ((reinterpret_cast<uintptr_t>(a) | (b ? reinterpret_cast<uintptr_t>(b) : 0) |
         reinterpret_cast<uintptr_t>(out)) % 16)
      g.vec = 0;
    unsigned grid = grid_for(g.rows * g.chunks * 32, 256, 16);
    ew_rows_kernel<Op, T><<<grid, 256, 0, st>>>(g, a, b, out, op);
  }
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------- activation

// reference nnops.py:54-70: stable sigmoid, relu = np.maximum(x, 0) (NaN
// propagates, -0 -> +0), tanh.
template <int KIND>
struct ActFwd {
  static constexpr bool kReadsOut = false;
  template <typename T>
  __device__ T operator()(T x, T, T) const {
    if (KIND == 1) return (x > T(0) || x != x) ? x : T(0);
    if (KIND == 2) return tanh(x);
    T e = exp(-fabs(x));
    return x >= T(0) ? T(1) / dadd<T>(T(1), e) : e / dadd<T>(T(1), e);
  }
};
// reference nnops.py:73-88, evaluated in numpy's order:
//   sigmoid (dy*y)*(1-y); relu dy*(y>0); tanh dy*(1-y*y)
template <int KIND>
struct ActBwd {
  static constexpr bool kReadsOut = false;
  template <typename T>
  __device__ T operator()(T y, T dy, T) const {
    if (KIND == 1) return dmul<T>(dy, y > T(0) ? T(1) : T(0));
    if (KIND == 2) return dmul<T>(dy, dsub<T>(T(1), dmul<T>(y, y)));
    return dmul<T>(dmul<T>(dy, y), dsub<T>(T(1), y));
  }
};

template <typename T>
static cudaError_t act_fwd_t(int kind, const View4& xv, const T* x, const View4& yv, T* y,
                             cudaStream_t st) {
  switch (kind) {
    case 0: return run_ew(xv, x, nullptr, (const T*)nullptr, yv, y, ActFwd<0>{}, st);
    case 1: return run_ew(xv, x, nullptr, (const T*)nullptr, yv, y, ActFwd<1>{}, st);
    default: return run_ew(xv, x, nullptr, (const T*)nullptr, yv, y, ActFwd<2>{}, st);
  }
}
template <typename T>
static cudaError_t act_bwd_t(int kind, const View4& yv, const T* y, const View4& dyv, const T* dy,
                             const View4& dxv, T* dx, cudaStream_t st) {
  switch (kind) {
    case 0: return run_ew(yv, y, &dyv, dy, dxv, dx, ActBwd<0>{}, st);
    case 1: return run_ew(yv, y, &dyv, dy, dxv, dx, ActBwd<1>{}, st);
    default: return run_ew(yv, y, &dyv, dy, dxv, dx, ActBwd<2>{}, st);
  }
}

cudaError_t activation_forward(int kind, Dtype dt, const View4& xv, const void* x,
                               const View4& yv, void* y, cudaStream_t st) {
  return dt == F32 ? act_fwd_t(kind, xv, (const float*)x, yv, (float*)y, st)
                   : act_fwd_t(kind, xv, (const double*)x, yv, (double*)y, st);
}
cudaError_t activation_backward(int kind, Dtype dt, const View4& yv, const void* y,
                                const View4& dyv, const void* dy, const View4& dxv, void* dx,
                                cudaStream_t st) {
  return dt == F32 ? act_bwd_t(kind, yv, (const float*)y, dyv, (const float*)dy, dxv,
                               (float*)dx, st)
                   : act_bwd_t(kind, yv, (const double*)y, dyv, (const double*)dy, dxv,
                               (double*)dx, st);
}

// -------------------------------------------------- transform / broadcast

// dst := alpha*src (+ beta*dst): numpy `d *= beta; d += alpha * s`
// (reference tensor.py:241-251), each product/sum rounded separately.
template <bool BETA>
struct Axpby {
  static constexpr bool kReadsOut = BETA;
  double alpha, beta;
  template <typename T>
  __device__ T operator()(T s, T, T d) const {
    T as = dmul<T>(s, T(alpha));
    return BETA ? dadd<T>(dmul<T>(d, T(beta)), as) : as;
  }
};

cudaError_t transform(Dtype dt, const View4& sv, const void* s, const View4& dv, void* d,
                      double alpha, double beta, cudaStream_t st) {
  if (dt == F32) {
    if (beta == 0.0)
      return run_ew(sv, (const float*)s, nullptr, (const float*)nullptr, dv, (float*)d,
                    Axpby<false>{alpha, beta}, st);
    return run_ew(sv, (const float*)s, nullptr, (const float*)nullptr, dv, (float*)d,
                  Axpby<true>{alpha, beta}, st);
  }
  if (beta == 0.0)
    return run_ew(sv, (const double*)s, nullptr, (const double*)nullptr, dv, (double*)d,
                  Axpby<false>{alpha, beta}, st);
  return run_ew(sv, (const double*)s, nullptr, (const double*)nullptr, dv, (double*)d,
                Axpby<true>{alpha, beta}, st);
}

cudaError_t add_broadcast(Dtype dt, const View4& bv, const void* b, const View4& ov, void* o,
                          double alpha, double beta, cudaStream_t st) {
  // broadcast dims of the bias carry stride 0 and the output's extent
  View4 bb = bv;
  if (bb.n == 1) { bb.n = ov.n; bb.sn = 0; }
  if (bb.c == 1) { bb.c = ov.c; bb.sc = 0; }
  if (bb.h == 1) { bb.h = ov.h; bb.sh = 0; }
  if (bb.w == 1) { bb.w = ov.w; bb.sw = 0; }
  const View4* views[3] = {&bb, &bb, &ov};
  EwGeom g = make_ew(views, 3, 2);
  // make_ew zeroes strides of extent-1 dims using the op's own extents; the
  // broadcast view already has stride 0 there.
  for (int k = 0; k < 4; k++) g.st[1][k] = 0;
  unsigned grid = grid_for(g.rows * 32, 256, 16);
  if (dt == F32) {
    if (beta == 0.0)
      ew_rows_kernel<Axpby<false>, float><<<grid, 256, 0, st>>>(
          g, (const float*)b, nullptr, (float*)o, Axpby<false>{alpha, beta});
    else
      ew_rows_kernel<Axpby<true>, float><<<grid, 256, 0, st>>>(
          g, (const float*)b, nullptr, (float*)o, Axpby<true>{alpha, beta});
  } else {
    if (beta == 0.0)
      ew_rows_kernel<Axpby<false>, double><<<grid, 256, 0, st>>>(
          g, (const double*)b, nullptr, (double*)o, Axpby<false>{alpha, beta});
    else
      ew_rows_kernel<Axpby<true>, double><<<grid, 256, 0, st>>>(
          g, (const double*)b, nullptr, (double*)o, Axpby<true>{alpha, beta});
  }
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- softmax
//
// per_image: one group = the (c, h, w) box of one image; per_spatial: one
// group = the c fibre at one (n, h, w) (reference nnops.py:91-117).

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Group element g (0 <= g < C*H*W) of image n -> offset.
struct ImgGeom {
  View4 v;
  MagicDiv dHW, dW;
};
__device__ __forceinline__ int64_t img_off(const ImgGeom& ig, int64_t n, uint32_t g) {
  uint32_t c, rem, h, w;
  mdivmod(g, ig.dHW, c, rem);
  mdivmod(rem, ig.dW, h, w);
  return n * ig.v.sn + c * ig.v.sc + h * ig.v.sh + w * ig.v.sw;
}

// Block reduction helpers (256 threads).
template <typename T>
__device__ T block_reduce_max(T v, T* sh) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  T r = sh[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); i++) r = fmax(r, sh[i]);
  __syncthreads();
  return r;
}
template <typename T>
__device__ T block_reduce_sum(T v, T* sh) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  T r = T(0);
  for (int i = 0; i < (int)(blockDim.x >> 5); i++) r += sh[i];
  __syncthreads();
  return r;
}

// Phase 1 of per-image softmax: each block reduces a chunk of a group to
// (max, sum exp(x - max)) [forward] or sum(y*dy) [backward].
template <typename T, bool BWD>
__global__ void __launch_bounds__(256) softmax_img_partial(ImgGeom ga, const T* a, ImgGeom gb,
                                                          const T* b, int64_t G, int chunks,
                                                          T* part) {
  __shared__ T sh[32];
  const int64_t n = blockIdx.y;
  const int64_t per = (G + chunks - 1) / chunks;
  const int64_t g0 = blockIdx.x * per, g1 = min(G, g0 + per);
  if (!BWD) {
    T m = T(-INFINITY);
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) m = fmax(m, a[img_off(ga, n, g)]);
    m = block_reduce_max(m, sh);
    T s = T(0);
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) s += exp(a[img_off(ga, n, g)] - m);
    s = block_reduce_sum(s, sh);
    if (threadIdx.x == 0) {
      part[(n * chunks + blockIdx.x) * 2] = m;
      part[(n * chunks + blockIdx.x) * 2 + 1] = s;
    }
  } else {
    T s = T(0);
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x)
      s += a[img_off(ga, n, g)] * b[img_off(gb, n, g)];
    s = block_reduce_sum(s, sh);
    if (threadIdx.x == 0) part[n * chunks + blockIdx.x] = s;
  }
}

// Phase 2: combine the partials of the group and write the chunk.
template <typename T, bool BWD>
__global__ void __launch_bounds__(256) softmax_img_apply(ImgGeom ga, const T* a, ImgGeom gb,
                                                        const T* b, ImgGeom go, T* o, int64_t G,
                                                        int chunks, const T* part) {
  const int64_t n = blockIdx.y;
  const int64_t per = (G + chunks - 1) / chunks;
  const int64_t g0 = blockIdx.x * per, g1 = min(G, g0 + per);
  if (!BWD) {
    T M = T(-INFINITY);
    for (int i = 0; i < chunks; i++) M = fmax(M, part[(n * chunks + i) * 2]);
    T S = T(0);
    for (int i = 0; i < chunks; i++) {
      T mi = part[(n * chunks + i) * 2];
      S += part[(n * chunks + i) * 2 + 1] * exp(mi - M);
    }
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x)
      o[img_off(go, n, g)] = exp(a[img_off(ga, n, g)] - M) / S;
  } else {
    T D = T(0);
    for (int i = 0; i < chunks; i++) D += part[n * chunks + i];
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) {
      T yv = a[img_off(ga, n, g)];
      o[img_off(go, n, g)] = dmul<T>(yv, dsub<T>(b[img_off(gb, n, g)], D));
    }
  }
}

// Small groups (G <= 32 * PER, e.g. 1000 classes): one warp per image, the
// whole group held in registers -- one read and one write per element and a
// single launch instead of partial + apply.  Same operations as the two
// kernels above (fmax / exp / divide; dsub / dmul for the backward).
template <typename T, bool BWD, int PER, bool CONTIG>
__global__ void __launch_bounds__(256) softmax_img_warp(ImgGeom ga, const T* a, ImgGeom gb,
                                                       const T* b, ImgGeom go, T* o, int64_t G,
                                                       int64_t nimg) {
  const int lane = threadIdx.x & 31;
  const int64_t n = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n >= nimg) return;
  // CONTIG: every operand's image is one dense run (offset n * sn + g): no
  // index decode per element (the decode cost more than the bytes moved)
  auto off = [&](const ImgGeom& ig, uint32_t g) -> int64_t {
    return CONTIG ? n * ig.v.sn + g : img_off(ig, n, g);
  };
  T va[PER], vb[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const int64_t g = lane + 32 * k;
    if (g < G) {
      va[k] = __ldg(a + off(ga, uint32_t(g)));
      if (BWD) vb[k] = __ldg(b + off(gb, uint32_t(g)));
    }
  }
  if (!BWD) {
    T m = T(-INFINITY);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (lane + 32 * k < G) m = fmax(m, va[k]);
    m = warp_max(m);
    T sum = T(0);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (lane + 32 * k < G) {
        va[k] = exp(va[k] - m);
        sum += va[k];
      }
    sum = warp_sum(sum);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (lane + 32 * k < G) o[off(go, uint32_t(lane + 32 * k))] = va[k] / sum;
  } else {
    T d = T(0);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (lane + 32 * k < G) d += va[k] * vb[k];
    d = warp_sum(d);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (lane + 32 * k < G)
        o[off(go, uint32_t(lane + 32 * k))] = dmul<T>(va[k], dsub<T>(vb[k], d));
  }
}

// Per-image softmax, one 128-thread block per image (groups of 129..1024
// elements): each thread holds PER <= 8 elements in registers, so every
// element is read once and written once; two-level (warp shuffle, then
// shared memory) reductions.  Four warps per image instead of one keep ~4x
// the bytes in flight per SM (the warp-per-image form was latency-bound:
// 1024 images = 7 warps per SM).
template <typename T, bool BWD, int PER, bool CONTIG>
__global__ void __launch_bounds__(128) softmax_img_block(ImgGeom ga, const T* a, ImgGeom gb,
                                                        const T* b, ImgGeom go, T* o, int64_t G) {
  __shared__ T red[4];
  const int64_t n = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  auto off = [&](const ImgGeom& ig, uint32_t g) -> int64_t {
    return CONTIG ? n * ig.v.sn + g : img_off(ig, n, g);
  };
  T va[PER], vb[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const int64_t g = t + 128 * k;
    if (g < G) {
      va[k] = __ldg(a + off(ga, uint32_t(g)));
      if (BWD) vb[k] = __ldg(b + off(gb, uint32_t(g)));
    }
  }
  if (!BWD) {
    T m = T(-INFINITY);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (t + 128 * k < G) m = fmax(m, va[k]);
    m = warp_max(m);
    if (lane == 0) red[wid] = m;
    __syncthreads();
    m = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
    __syncthreads();
    T sum = T(0);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (t + 128 * k < G) {
        va[k] = exp(va[k] - m);
        sum += va[k];
      }
    sum = warp_sum(sum);
    if (lane == 0) red[wid] = sum;
    __syncthreads();
    sum = (red[0] + red[1]) + (red[2] + red[3]);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (t + 128 * k < G) o[off(go, uint32_t(t + 128 * k))] = va[k] / sum;
  } else {
    T d = T(0);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (t + 128 * k < G) d += va[k] * vb[k];
    d = warp_sum(d);
    if (lane == 0) red[wid] = d;
    __syncthreads();
    d = (red[0] + red[1]) + (red[2] + red[3]);
#pragma unroll
    for (int k = 0; k < PER; k++)
      if (t + 128 * k < G) o[off(go, uint32_t(t + 128 * k))] = dmul<T>(va[k], dsub<T>(vb[k], d));
  }
}

// per_spatial: one thread per (n, h, w) position, loop over channels.
struct PosGeom {
  View4 v;
  MagicDiv dHW, dW;
};
__device__ __forceinline__ int64_t pos_base(const PosGeom& pg, uint32_t pos) {
  uint32_t n, rem, h, w;
  mdivmod(pos, pg.dHW, n, rem);
  mdivmod(rem, pg.dW, h, w);
  return n * pg.v.sn + h * pg.v.sh + w * pg.v.sw;
}

template <typename T, bool BWD>
__global__ void __launch_bounds__(256) softmax_spatial(PosGeom ga, const T* a, PosGeom gb,
                                                      const T* b, PosGeom go, T* o, int64_t npos,
                                                      int64_t C) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t pos = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pos < npos; pos += stride) {
    const int64_t ba = pos_base(ga, pos), bo = pos_base(go, pos);
    if (!BWD) {
      T m = T(-INFINITY);
      for (int64_t c = 0; c < C; c++) m = fmax(m, a[ba + c * ga.v.sc]);
      T s = T(0);
      for (int64_t c = 0; c < C; c++) s += exp(a[ba + c * ga.v.sc] - m);
      for (int64_t c = 0; c < C; c++) o[bo + c * go.v.sc] = exp(a[ba + c * ga.v.sc] - m) / s;
    } else {
      const int64_t bb = pos_base(gb, pos);
      T d = T(0);
      for (int64_t c = 0; c < C; c++) d += a[ba + c * ga.v.sc] * b[bb + c * gb.v.sc];
      for (int64_t c = 0; c < C; c++)
        o[bo + c * go.v.sc] = dmul<T>(a[ba + c * ga.v.sc], dsub<T>(b[bb + c * gb.v.sc], d));
    }
  }
}

// per_spatial with C <= CMAX channels: the position's channels are read
// once into registers (max, exponentials, sum and output from them; the
// loop form read the input three times)
template <typename T, bool BWD, int CMAX>
__global__ void __launch_bounds__(256) softmax_spatial_reg(PosGeom ga, const T* a, PosGeom gb,
                                                          const T* b, PosGeom go, T* o,
                                                          int64_t npos, int C) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t pos = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pos < npos; pos += stride) {
    const int64_t ba = pos_base(ga, uint32_t(pos)), bo = pos_base(go, uint32_t(pos));
    T va[CMAX], vb[CMAX];
    const int64_t bb = BWD ? pos_base(gb, uint32_t(pos)) : 0;
#pragma unroll
    for (int c = 0; c < CMAX; c++)
      if (c < C) {
        va[c] = __ldg(a + ba + c * ga.v.sc);
        if (BWD) vb[c] = __ldg(b + bb + c * gb.v.sc);
      }
    if (!BWD) {
      T m = T(-INFINITY);
#pragma unroll
      for (int c = 0; c < CMAX; c++)
        if (c < C) m = fmax(m, va[c]);
      T sum = T(0);
#pragma unroll
      for (int c = 0; c < CMAX; c++)
        if (c < C) {
          va[c] = exp(va[c] - m);
          sum += va[c];
        }
#pragma unroll
      for (int c = 0; c < CMAX; c++)
        if (c < C) o[bo + c * go.v.sc] = va[c] / sum;
    } else {
      T d = T(0);
#pragma unroll
      for (int c = 0; c < CMAX; c++)
        if (c < C) d += va[c] * vb[c];
#pragma unroll
      for (int c = 0; c < CMAX; c++)
        if (c < C) o[bo + c * go.v.sc] = dmul<T>(va[c], dsub<T>(vb[c], d));
    }
  }
}

// one image's (c, h, w) elements form a single dense run
static bool img_dense(const View4& v) {
  return (v.w == 1 || v.sw == 1) && (v.h == 1 || v.sh == v.w * (v.w == 1 ? 1 : v.sw)) &&
         (v.c == 1 || v.sc == v.h * v.w);
}

static ImgGeom img_geom(const View4& v) {
  return ImgGeom{v, make_magic(uint32_t(v.h * v.w)), make_magic(uint32_t(v.w))};
}
static PosGeom pos_geom(const View4& v) {
  return PosGeom{v, make_magic(uint32_t(v.h * v.w)), make_magic(uint32_t(v.w))};
}

template <typename T, bool BWD>
static cudaError_t softmax_t(int mode, const View4& av, const T* a, const View4* bv, const T* b,
                             const View4& ov, T* o, cudaStream_t st) {
  if (av.c * av.h * av.w >= (int64_t(1) << 32) || av.n * av.h * av.w >= (int64_t(1) << 32))
    return cudaErrorInvalidValue;
  if (mode == 0 && av.c * av.h * av.w <= 1024 && !::dnnp::tune_env("DNNP_SOFTMAX_NO_WARP")) {
    const int64_t G = av.c * av.h * av.w;
    const unsigned grid = unsigned(ceil_div(av.n, 8));
    ImgGeom ga = img_geom(av), gb = img_geom(bv ? *bv : av), go = img_geom(ov);
    const bool contig = img_dense(av) && img_dense(ov) && (!bv || img_dense(*bv));
    auto go_per = [&](auto perc) {
      if (contig)
        softmax_img_warp<T, BWD, decltype(perc)::value, true><<<grid, 256, 0, st>>>(
            ga, a, gb, b, go, o, G, av.n);
      else
        softmax_img_warp<T, BWD, decltype(perc)::value, false><<<grid, 256, 0, st>>>(
            ga, a, gb, b, go, o, G, av.n);
    };
    auto go_blk = [&](auto perc) {
      constexpr int PER = decltype(perc)::value;
      const unsigned nb = unsigned(av.n);
      if (contig)
        softmax_img_block<T, BWD, PER, true><<<nb, 128, 0, st>>>(ga, a, gb, b, go, o, G);
      else
        softmax_img_block<T, BWD, PER, false><<<nb, 128, 0, st>>>(ga, a, gb, b, go, o, G);
    };
    if (G <= 128) go_per(std::integral_constant<int, 4>());
    else if (av.n >= (int64_t(1) << 31) || ::dnnp::tune_env("DNNP_SOFTMAX_WARP_ONLY")) {
      if (G <= 256) go_per(std::integral_constant<int, 8>());
      else if (G <= 512) go_per(std::integral_constant<int, 16>());
      else go_per(std::integral_constant<int, 32>());
    } else if (G <= 256) go_blk(std::integral_constant<int, 2>());
    else if (G <= 512) go_blk(std::integral_constant<int, 4>());
    else go_blk(std::integral_constant<int, 8>());
    note_launch();
    return cudaGetLastError();
  }
  if (mode == 0) {
    const int64_t G = av.c * av.h * av.w;
    // enough blocks to fill the GPU, at least ~2K elements per block
    int64_t chunks = ceil_div(int64_t(kNumSMs) * 4, av.n);
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, ceil_div(G, 2048)));
    chunks = std::min<int64_t>(chunks, 65535);
    tc::Workspace ws(st);
    cudaError_t e = ws.alloc(sizeof(T) * 2 * av.n * chunks);
    if (e != cudaSuccess) return e;
    T* part = static_cast<T*>(ws.p);
    dim3 grid(unsigned(chunks), unsigned(av.n));
    ImgGeom ga = img_geom(av), gb = img_geom(bv ? *bv : av), go = img_geom(ov);
    softmax_img_partial<T, BWD><<<grid, 256, 0, st>>>(ga, a, gb, b, G, int(chunks), part);
    softmax_img_apply<T, BWD><<<grid, 256, 0, st>>>(ga, a, gb, b, go, o, G, int(chunks), part);
    note_launch(2);
    return cudaGetLastError();
  }
  const int64_t npos = av.n * av.h * av.w;
  if (av.c <= 32 && !::dnnp::tune_env("DNNP_SOFTMAX_NO_REG")) {
    const unsigned grid = grid_for(npos, 256, 8);
    if (av.c <= 8)
      softmax_spatial_reg<T, BWD, 8><<<grid, 256, 0, st>>>(pos_geom(av), a, pos_geom(bv ? *bv : av),
                                                           b, pos_geom(ov), o, npos, int(av.c));
    else
      softmax_spatial_reg<T, BWD, 32><<<grid, 256, 0, st>>>(pos_geom(av), a, pos_geom(bv ? *bv : av),
                                                            b, pos_geom(ov), o, npos, int(av.c));
    note_launch();
    return cudaGetLastError();
  }
  softmax_spatial<T, BWD><<<grid_for(npos, 256, 8), 256, 0, st>>>(
      pos_geom(av), a, pos_geom(bv ? *bv : av), b, pos_geom(ov), o, npos, av.c);
  note_launch();
  return cudaGetLastError();
}

cudaError_t softmax_forward(int mode, Dtype dt, const View4& xv, const void* x, const View4& yv,
                            void* y, cudaStream_t st) {
  return dt == F32 ? softmax_t<float, false>(mode, xv, (const float*)x, nullptr, nullptr, yv,
                                             (float*)y, st)
                   : softmax_t<double, false>(mode, xv, (const double*)x, nullptr, nullptr, yv,
                                              (double*)y, st);
}
cudaError_t softmax_backward(int mode, Dtype dt, const View4& yv, const void* y,
                             const View4& dyv, const void* dy, const View4& dxv, void* dx,
                             cudaStream_t st) {
  return dt == F32 ? softmax_t<float, true>(mode, yv, (const float*)y, &dyv, (const float*)dy,
                                            dxv, (float*)dx, st)
                   : softmax_t<double, true>(mode, yv, (const double*)y, &dyv,
                                             (const double*)dy, dxv, (double*)dx, st);
}

// ---------------------------------------------------------------- pooling

struct PoolGeom {
  View4 x, y;  // y: pooled output (or dy)
  int64_t N, C, H, W, P, Q;
  int64_t wh, ww, sh, sw, ph, pw;
  MagicDiv dQ, dP, dC, dW, dH, dSH, dSW;
};

// Forward: one thread per pooled element; window clipped to the image
// (reference nnops.py:150-200).  Max takes the first maximum in (h, w) scan
// order with numpy argmax NaN semantics (the first NaN wins); argmax is the
// LOGICAL NCHW index.  Average divides by the in-image count.  32-bit index
// arithmetic (extents < 2^31 checked on the host), 64-bit only for offsets.
template <typename T, int KW>
__global__ void __launch_bounds__(256) pool_fwd_kernel(PoolGeom g, const T* __restrict__ x,
                                                       T* __restrict__ y, int64_t* argmax,
                                                       int kind, int64_t total) {
  const int H = int(g.H), W = int(g.W), C = int(g.C);
  const int wh = int(g.wh), ww = int(g.ww);
  const int64_t xsh = g.x.sh, xsw = g.x.sw;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < uint32_t(total); i += stride) {
    uint32_t t, q, p, c, n;
    mdivmod(i, g.dQ, t, q);
    mdivmod(t, g.dP, t, p);
    mdivmod(t, g.dC, n, c);
    const int hs0 = int(p) * int(g.sh) - int(g.ph), ws0 = int(q) * int(g.sw) - int(g.pw);
    const int hs = max(0, hs0), he = min(H, hs0 + wh);
    const int ws = max(0, ws0), we = min(W, ws0 + ww);
    const T* xb = x + int64_t(n) * g.x.sn + int64_t(c) * g.x.sc;
    T out;
    if (KW > 0 && hs0 >= 0 && ws0 >= 0 && hs0 + KW <= H && ws0 + KW <= W) {
      // interior window of the specialised size: KW*KW independent loads,
      // branch-free first-max / first-NaN selection (or the scan-order sum)
      T v[KW > 0 ? KW * KW : 1];
#pragma unroll
      for (int a = 0; a < KW; a++)
#pragma unroll
        for (int b = 0; b < KW; b++) v[a * KW + b] = __ldg(xb + (hs0 + a) * xsh + (ws0 + b) * xsw);
      if (kind == 0) {
        T best = v[0];
        int bk = 0;
#pragma unroll
        for (int k = 1; k < KW * KW; k++) {
          const bool take = v[k] > best || (v[k] != v[k] && best == best);
          best = take ? v[k] : best;
          bk = take ? k : bk;
        }
        out = best;
        if (argmax)
          argmax[i] = ((int64_t(n) * C + c) * H + hs0 + bk / (KW > 0 ? KW : 1)) * W + ws0 + bk % (KW > 0 ? KW : 1);
      } else {
        T sacc = T(0);
#pragma unroll
        for (int k = 0; k < KW * KW; k++) sacc = dadd<T>(sacc, v[k]);
        out = sacc / T(KW > 0 ? KW * KW : 1);
      }
    } else if (kind == 0) {
      T best = xb[hs * xsh + ws * xsw];
      int bh = hs, bw = ws;
      bool nan = best != best;
      for (int h = hs; h < he && !nan; h++) {
        const T* xr = xb + h * xsh;
        for (int w = ws; w < we; w++) {
          const T v = xr[w * xsw];
          if (v != v || v > best) {
            best = v;
            bh = h;
            bw = w;
            if (v != v) {
              nan = true;  // the first NaN wins
              break;
            }
          }
        }
      }
      out = best;
      if (argmax) argmax[i] = ((int64_t(n) * C + c) * H + bh) * W + bw;
    } else {
      T s = T(0);
      for (int h = hs; h < he; h++)
        for (int w = ws; w < we; w++) s = dadd<T>(s, xb[h * xsh + w * xsw]);
      out = s / T((he - hs) * (we - ws));
    }
    y[int64_t(n) * g.y.sn + int64_t(c) * g.y.sc + int64_t(p) * g.y.sh + int64_t(q) * g.y.sw] = out;
  }
}

// Backward as a gather over the windows covering each input element, in
// ascending (p, q) order starting from 0: this is exactly the summation
// order of the reference's zero-fill + np.add.at / per-window += loops
// (nnops.py:218-246), so max and average backward are bit-exact.  CL walks
// the elements channel-fastest (n, h, w, c) for channels-innermost views, so
// dy reads and dx writes coalesce there.
template <typename T, bool CL = false>
__global__ void __launch_bounds__(256) pool_bwd_kernel(PoolGeom g, const T* __restrict__ dy,
                                                       T* __restrict__ dx,
                                                       const int64_t* __restrict__ argmax,
                                                       int kind, int64_t total) {
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q);
  const int wh = int(g.wh), ww = int(g.ww), sh = int(g.sh), sw = int(g.sw);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < uint32_t(total); i += stride) {
    uint32_t t, w, h, c, n;
    if (CL) {
      mdivmod(i, g.dC, t, c);
      mdivmod(t, g.dW, t, w);
      mdivmod(t, g.dH, n, h);
    } else {
      mdivmod(i, g.dW, t, w);
      mdivmod(t, g.dH, t, h);
      mdivmod(t, g.dC, n, c);
    }
    // p covers h iff p*sh - ph <= h < p*sh - ph + wh
    const int hp = int(h) + int(g.ph), wp = int(w) + int(g.pw);
    const int p0 = hp - wh + 1 > 0 ? int(mdiv(uint32_t(hp - wh + sh), g.dSH)) : 0;
    const int p1 = min(P - 1, int(mdiv(uint32_t(hp), g.dSH)));
    const int q0 = wp - ww + 1 > 0 ? int(mdiv(uint32_t(wp - ww + sw), g.dSW)) : 0;
    const int q1 = min(Q - 1, int(mdiv(uint32_t(wp), g.dSW)));
    const uint32_t plane = n * uint32_t(g.C) + c;
    const int64_t me = (int64_t(plane) * H + h) * W + w;
    const T* dyb = dy + int64_t(n) * g.y.sn + int64_t(c) * g.y.sc;
    const int64_t* amb = argmax ? argmax + int64_t(plane) * P * Q : nullptr;
    T acc = T(0);
    for (int p = p0; p <= p1; p++)
      for (int q = q0; q <= q1; q++) {
        const T d = dyb[p * g.y.sh + q * g.y.sw];
        if (kind == 0) {
          if (amb[p * Q + q] == me) acc = dadd<T>(acc, d);
        } else {
          const int hs0 = p * sh - int(g.ph), ws0 = q * sw - int(g.pw);
          const int cnt = (min(H, hs0 + wh) - max(0, hs0)) * (min(W, ws0 + ww) - max(0, ws0));
          acc = dadd<T>(acc, d / T(cnt));
        }
      }
    dx[int64_t(n) * g.x.sn + int64_t(c) * g.x.sc + int64_t(h) * g.x.sh + int64_t(w) * g.x.sw] = acc;
  }
}

// Flags argmax entries that do not point inside their own window (only
// possible for caller-made argmax buffers); those take the serial path.
__global__ void pool_argmax_check(PoolGeom g, const int64_t* __restrict__ argmax, int64_t total,
                                  int* bad) {
  const uint32_t stride = gridDim.x * blockDim.x;
  const int64_t HW = g.H * g.W;
  bool any = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < uint32_t(total); i += stride) {
    uint32_t t, q, p;
    mdivmod(i, g.dQ, t, q);
    mdivmod(t, g.dP, t, p);  // t = plane
    const int64_t hw = argmax[i] - int64_t(t) * HW;
    bool ok = hw >= 0 && hw < HW;
    if (ok) {
      uint32_t h, w;
      mdivmod(uint32_t(hw), g.dW, h, w);
      const int hs0 = int(p) * int(g.sh) - int(g.ph), ws0 = int(q) * int(g.sw) - int(g.pw);
      ok = int(h) >= hs0 && int(h) < hs0 + int(g.wh) && int(w) >= ws0 && int(w) < ws0 + int(g.ww);
    }
    any |= !ok;
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *bad = 1;
}

// Plane-tiled forms (one block per (n, c) plane, the plane staged in shared
// memory with coalesced loads; same window semantics and summation order as
// the per-element kernels above).
// Contiguous plane <-> shared memory with 16-byte global accesses: scalar
// head up to the first 16-byte boundary, vectors, scalar tail (planes of odd
// size start at any 4-byte offset).  Every vector is issued before any
// shared-memory store, so a thread keeps all its loads in flight.
template <typename T>
__device__ __forceinline__ void plane_to_smem(T* xs, const T* __restrict__ xb, int n) {
  constexpr int V = 16 / sizeof(T);
  const int mis = int((reinterpret_cast<uintptr_t>(xb) / sizeof(T)) % V);
  const int head = min(n, (V - mis) % V);
  const int nv = (n - head) / V;
  const int B = blockDim.x;
  if (int(threadIdx.x) < head) xs[threadIdx.x] = xb[threadIdx.x];
  const uint4* src = reinterpret_cast<const uint4*>(xb + head);
  int j = threadIdx.x;
  for (; j + 3 * B < nv; j += 4 * B) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) v[k] = __ldg(src + j + k * B);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const T* e = reinterpret_cast<const T*>(&v[k]);
#pragma unroll
      for (int l = 0; l < V; l++) xs[head + (j + k * B) * V + l] = e[l];
    }
  }
  for (; j < nv; j += B) {
    const uint4 v = __ldg(src + j);
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int l = 0; l < V; l++) xs[head + j * V + l] = e[l];
  }
  for (int i = head + nv * V + threadIdx.x; i < n; i += B) xs[i] = xb[i];
}

template <typename T>
__device__ __forceinline__ void smem_to_plane(T* __restrict__ xb, const T* xs, int n) {
  constexpr int V = 16 / sizeof(T);
  const int mis = int((reinterpret_cast<uintptr_t>(xb) / sizeof(T)) % V);
  const int head = min(n, (V - mis) % V);
  const int nv = (n - head) / V;
  const int B = blockDim.x;
  if (int(threadIdx.x) < head) xb[threadIdx.x] = xs[threadIdx.x];
  uint4* dst = reinterpret_cast<uint4*>(xb + head);
  for (int j = threadIdx.x; j < nv; j += B) {
    uint4 v;
    T* e = reinterpret_cast<T*>(&v);
#pragma unroll
    for (int l = 0; l < V; l++) e[l] = xs[head + j * V + l];
    dst[j] = v;
  }
  for (int i = head + nv * V + threadIdx.x; i < n; i += B) xb[i] = xs[i];
}

// Max over a KW x KW window in (h, w) scan order, branch-free: a later value
// replaces the best when greater, or when it is NaN and the best is not, so
// the first maximum and the first NaN win (reference nnops.py:180-197).
template <typename T, int KW>
__device__ __forceinline__ void window_max(const T* xs, int W, int base, T& best, int& bi) {
  best = xs[base];
  bi = base;
#pragma unroll
  for (int a = 0; a < KW; a++)
#pragma unroll
    for (int b = 0; b < KW; b++) {
      if (a == 0 && b == 0) continue;
      const int idx = base + a * W + b;
      const T v = xs[idx];
      const bool take = v > best || (v != v && best == best);
      best = take ? v : best;
      bi = take ? idx : bi;
    }
}

// Pipelined plane forward (dense NCHW planes): a persistent block streams
// its planes through two shared-memory buffers with cp.async, the next
// plane's bytes in flight while the current one is reduced (the one-plane-
// per-block kernel waited a full memory latency per plane).  Element i of
// a plane sits at buf + mis + i, mis = the plane's 16-byte misalignment in
// elements, so the body moves as aligned 16-byte copies.
__device__ __forceinline__ void cpa4(void* dst, const void* src) {
  const uint32_t d = uint32_t(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa8(void* dst, const void* src) {
  const uint32_t d = uint32_t(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  const uint32_t d = uint32_t(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T>
__device__ __forceinline__ int plane_async(T* buf, const T* __restrict__ xb, int n) {
  constexpr int V = 16 / sizeof(T);
  const int mis = int((reinterpret_cast<uintptr_t>(xb) / sizeof(T)) % V);
  const int head = min(n, (V - mis) % V);
  const int nv = (n - head) / V;
  T* xs = buf + mis;
  if (int(threadIdx.x) < head) {
    if (sizeof(T) == 4) cpa4(xs + threadIdx.x, xb + threadIdx.x);
    else cpa8(xs + threadIdx.x, xb + threadIdx.x);
  }
  for (int j = threadIdx.x; j < nv; j += blockDim.x) cpa16(xs + head + j * V, xb + head + j * V);
  for (int i = head + nv * V + threadIdx.x; i < n; i += blockDim.x) {
    if (sizeof(T) == 4) cpa4(xs + i, xb + i);
    else cpa8(xs + i, xb + i);
  }
  return mis;
}

template <typename T, int KW>
__global__ void __launch_bounds__(256) pool_fwd_pipe_kernel(PoolGeom g, const T* __restrict__ x,
                                                            T* __restrict__ y, int64_t* argmax,
                                                            int kind, int pitch) {
  extern __shared__ __align__(16) uint8_t psm[];
  T* bufs = reinterpret_cast<T*>(psm);  // [2][pitch], pitch >= H*W + 16 / sizeof(T)
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int wh = int(g.wh), ww = int(g.ww);
  const int planes = int(g.N) * C, HW = H * W;
  auto base_of = [&](int pl) {
    uint32_t nu, cu;
    mdivmod(uint32_t(pl), g.dC, nu, cu);
    return x + int64_t(nu) * g.x.sn + int64_t(cu) * g.x.sc;
  };
  int pl = blockIdx.x, it = 0;
  int mis_cur = 0, mis_next = 0;
  if (pl < planes) mis_cur = plane_async(bufs, base_of(pl), HW);
  cpa_commit();
  for (; pl < planes; pl += gridDim.x, it++) {
    const int nxt = pl + gridDim.x;
    if (nxt < planes) mis_next = plane_async(bufs + ((it + 1) & 1) * pitch, base_of(nxt), HW);
    cpa_commit();
    cpa_wait<1>();
    __syncthreads();
    const T* xs = bufs + (it & 1) * pitch + mis_cur;
    uint32_t nu, cu;
    mdivmod(uint32_t(pl), g.dC, nu, cu);
    T* yb = y + int64_t(nu) * g.y.sn + int64_t(cu) * g.y.sc;
    for (int o = threadIdx.x; o < P * Q; o += blockDim.x) {
      uint32_t pu, qu;
      mdivmod(uint32_t(o), g.dQ, pu, qu);
      const int p = int(pu), q = int(qu);
      const int hs0 = p * int(g.sh) - int(g.ph), ws0 = q * int(g.sw) - int(g.pw);
      T out;
      if (KW > 0 && hs0 >= 0 && ws0 >= 0 && hs0 + KW <= H && ws0 + KW <= W) {
        const int b0 = hs0 * W + ws0;
        if (kind == 0) {
          int bi;
          window_max<T, KW>(xs, W, b0, out, bi);
          if (argmax) argmax[int64_t(pl) * P * Q + o] = int64_t(pl) * HW + bi;
        } else {
          T sacc = T(0);
#pragma unroll
          for (int a = 0; a < KW; a++)
#pragma unroll
            for (int b = 0; b < KW; b++) sacc = dadd<T>(sacc, xs[b0 + a * W + b]);
          out = sacc / T(KW > 0 ? KW * KW : 1);
        }
      } else {
        const int hs = max(0, hs0), he = min(H, hs0 + wh);
        const int ws = max(0, ws0), we = min(W, ws0 + ww);
        if (kind == 0) {
          T best = xs[hs * W + ws];
          int bi = hs * W + ws;
          for (int h = hs; h < he; h++)
            for (int w = ws; w < we; w++) {
              const T v = xs[h * W + w];
              const bool take = v > best || (v != v && best == best);
              best = take ? v : best;
              bi = take ? h * W + w : bi;
            }
          out = best;
          if (argmax) argmax[int64_t(pl) * P * Q + o] = int64_t(pl) * HW + bi;
        } else {
          T sacc = T(0);
          for (int h = hs; h < he; h++)
            for (int w = ws; w < we; w++) sacc = dadd<T>(sacc, xs[h * W + w]);
          out = sacc / T((he - hs) * (we - ws));
        }
      }
      yb[p * g.y.sh + q * g.y.sw] = out;
    }
    mis_cur = mis_next;
    __syncthreads();  // the buffer is refilled two planes later
  }
  cpa_wait<0>();
}

// Channels-innermost forward (NHWC-like views, x.sc == y.sc == 1): a block
// = one output row segment (n, p, 32 q) x 32 channels; lane = channel, so
// every window load and y store is a contiguous 32-channel run; the argmax
// (logical NCHW index, stored in the dense [N][C][P][Q] buffer) goes
// through a shared-memory transpose so its stores are q-contiguous.
template <typename T, int KIND>
__global__ void __launch_bounds__(256) pool_fwd_cl_kernel(PoolGeom g, const T* __restrict__ x,
                                                          T* __restrict__ y, int64_t* argmax,
                                                          int nqb, int ncb) {
  constexpr int kind = KIND;
  __shared__ int64_t am[32][33];
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int wh = int(g.wh), ww = int(g.ww);
  uint32_t b = blockIdx.x;
  const int cb = int(b % uint32_t(ncb));
  b /= uint32_t(ncb);
  const int qb = int(b % uint32_t(nqb));
  b /= uint32_t(nqb);
  const int p = int(b % uint32_t(P)), n = int(b / uint32_t(P));
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 x 4 consecutive q
  const int c = cb * 32 + lane;
  const bool cok = c < C;
  const T* xb = x + int64_t(n) * g.x.sn + int64_t(cok ? c : 0) * g.x.sc;
  const int hs0 = p * int(g.sh) - int(g.ph);
  const int hs = max(0, hs0), he = min(H, hs0 + wh);
  // 3 x 3 / stride 2 (AlexNet pool): a thread takes 4 consecutive outputs
  // whose windows overlap, issuing the 3 x 9 loads together (27 instead of
  // 36), when the four windows are interior
  if (KIND != 0 && wh == 3 && ww == 3 && g.sh == 2 && g.sw == 2 && hs0 >= 0 && hs0 + 3 <= H) {
    const int q0 = qb * 32 + ty * 4;
    const int ws0 = q0 * 2 - int(g.pw);
    if (cok && q0 + 3 < Q && ws0 >= 0 && ws0 + 9 <= W) {
      T v[3][9];
#pragma unroll
      for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 9; b++)
          v[a][b] = xb[int64_t(hs0 + a) * g.x.sh + int64_t(ws0 + b) * g.x.sw];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        T out;
        int64_t bi = 0;
        if (kind == 0) {
          T best = v[0][2 * k];
          int bk = 0;
#pragma unroll
          for (int a = 0; a < 3; a++)
#pragma unroll
            for (int b = 0; b < 3; b++) {
              if (a == 0 && b == 0) continue;
              const T u = v[a][2 * k + b];
              const bool take = u > best || (u != u && best == best);
              best = take ? u : best;
              bk = take ? a * 3 + b : bk;
            }
          out = best;
          bi = ((int64_t(n) * C + c) * H + hs0 + bk / 3) * W + ws0 + 2 * k + bk % 3;
        } else {
          T sacc = T(0);
#pragma unroll
          for (int a = 0; a < 3; a++)
#pragma unroll
            for (int b = 0; b < 3; b++) sacc = dadd<T>(sacc, v[a][2 * k + b]);
          out = sacc / T(9);
        }
        y[int64_t(n) * g.y.sn + int64_t(c) * g.y.sc + int64_t(p) * g.y.sh +
          int64_t(q0 + k) * g.y.sw] = out;
        am[lane][ty * 4 + k] = bi;
      }
      goto done;
    }
  }
  // generic path: average pooling keeps the fast path's 4 consecutive
  // outputs per thread; max pooling interleaves the warps over q (measured
  // faster for it: neighbouring windows are read at the same time)
  for (int k = 0; k < 4; k++) {
    const int qi = kind != 0 ? ty * 4 + k : ty + 8 * k;
    const int q = qb * 32 + qi;
    if (q >= Q) break;
    const int ws0 = q * int(g.sw) - int(g.pw);
    const int ws = max(0, ws0), we = min(W, ws0 + ww);
    T out = T(0);
    int64_t bi = 0;
    if (cok) {
      if (kind == 0 && wh == 3 && ww == 3) {
        // 3 x 3: all nine (predicated) loads issued before the first compare
        // (113 -> 87 us on the section-8(d) NHWC shape)
        T v[9];
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
          for (int b = 0; b < 3; b++) {
            const int h = hs0 + a, w = ws0 + b;
            const bool ok = h >= 0 && h < H && w >= 0 && w < W;
            v[a * 3 + b] = ok ? xb[int64_t(h) * g.x.sh + int64_t(w) * g.x.sw] : T(0);
          }
        // first valid element seeds the scan (the reference's window order)
        T best = T(0);
        int bk = -1;
#pragma unroll
        for (int k9 = 0; k9 < 9; k9++) {
          const int h = hs0 + k9 / 3, w = ws0 + k9 % 3;
          const bool ok = h >= 0 && h < H && w >= 0 && w < W;
          const T u = v[k9];
          const bool take = ok && (bk < 0 || u > best || (u != u && best == best));
          best = take ? u : best;
          bk = take ? k9 : bk;
        }
        out = best;
        bi = ((int64_t(n) * C + c) * H + hs0 + bk / 3) * W + ws0 + bk % 3;
      } else if (kind == 0) {
        T best = xb[int64_t(hs) * g.x.sh + int64_t(ws) * g.x.sw];
        int bh = hs, bw = ws;
        for (int h = hs; h < he; h++)
          for (int w = ws; w < we; w++) {
            const T v = xb[int64_t(h) * g.x.sh + int64_t(w) * g.x.sw];
            const bool take = v > best || (v != v && best == best);
            best = take ? v : best;
            bh = take ? h : bh;
            bw = take ? w : bw;
          }
        out = best;
        bi = ((int64_t(n) * C + c) * H + bh) * W + bw;
      } else {
        T sacc = T(0);
        for (int h = hs; h < he; h++)
          for (int w = ws; w < we; w++) sacc = dadd<T>(sacc, xb[int64_t(h) * g.x.sh + int64_t(w) * g.x.sw]);
        out = sacc / T((he - hs) * (we - ws));
      }
      y[int64_t(n) * g.y.sn + int64_t(c) * g.y.sc + int64_t(p) * g.y.sh + int64_t(q) * g.y.sw] = out;
    }
    am[lane][qi] = bi;
  }
done:
  if (kind != 0 || !argmax) return;
  __syncthreads();
  // argmax rows: channel cb*32 + r, q-contiguous
  for (int r = ty; r < 32; r += 8) {
    const int cc = cb * 32 + r, q = qb * 32 + lane;
    if (cc < C && q < Q) argmax[((int64_t(n) * C + cc) * P + p) * Q + q] = am[r][lane];
  }
}

template <typename T, int KW>
__global__ void __launch_bounds__(256) pool_fwd_plane_kernel(PoolGeom g, const T* __restrict__ x,
                                                             T* __restrict__ y, int64_t* argmax,
                                                             int kind) {
  extern __shared__ __align__(16) uint8_t psm[];
  T* xs = reinterpret_cast<T*>(psm);
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int wh = int(g.wh), ww = int(g.ww);
  const int planes = int(g.N) * C;
  for (int pl = blockIdx.x; pl < planes; pl += gridDim.x) {
    uint32_t nu, cu;
    mdivmod(uint32_t(pl), g.dC, nu, cu);
    const int n = int(nu), c = int(cu);
    const T* xb = x + int64_t(n) * g.x.sn + int64_t(c) * g.x.sc;
    if (g.x.sw == 1 && g.x.sh == W) {
      plane_to_smem(xs, xb, H * W);  // contiguous plane: 16-byte loads
    } else {
      for (int i = threadIdx.x; i < H * W; i += blockDim.x) {
        uint32_t h, w;
        mdivmod(uint32_t(i), g.dW, h, w);
        xs[i] = xb[int(h) * g.x.sh + int(w) * g.x.sw];
      }
    }
    __syncthreads();
    T* yb = y + int64_t(n) * g.y.sn + int64_t(c) * g.y.sc;
    for (int o = threadIdx.x; o < P * Q; o += blockDim.x) {
      uint32_t pu, qu;
      mdivmod(uint32_t(o), g.dQ, pu, qu);
      const int p = int(pu), q = int(qu);
      const int hs0 = p * int(g.sh) - int(g.ph), ws0 = q * int(g.sw) - int(g.pw);
      const int hs = max(0, hs0), he = min(H, hs0 + wh);
      const int ws = max(0, ws0), we = min(W, ws0 + ww);
      T out;
      if (KW > 0 && hs0 >= 0 && ws0 >= 0 && hs0 + KW <= H && ws0 + KW <= W) {
        // interior window of the specialised size: unrolled, branch-free
        const int base = hs0 * W + ws0;
        if (kind == 0) {
          int bi;
          window_max<T, KW>(xs, W, base, out, bi);
          if (argmax) argmax[int64_t(pl) * P * Q + o] = int64_t(pl) * H * W + bi;
        } else {
          T sacc = T(0);
#pragma unroll
          for (int a = 0; a < KW; a++)
#pragma unroll
            for (int b = 0; b < KW; b++) sacc = dadd<T>(sacc, xs[base + a * W + b]);
          out = sacc / T(KW > 0 ? KW * KW : 1);
        }
      } else if (kind == 0) {
        T best = xs[hs * W + ws];
        int bi = hs * W + ws;
        bool nan = best != best;
        for (int h = hs; h < he && !nan; h++)
          for (int w = ws; w < we; w++) {
            const T v = xs[h * W + w];
            if (v != v || v > best) {
              best = v;
              bi = h * W + w;
              if (v != v) {
                nan = true;  // the first NaN wins
                break;
              }
            }
          }
        out = best;
        if (argmax) argmax[int64_t(pl) * P * Q + o] = int64_t(pl) * H * W + bi;
      } else {
        T sacc = T(0);
        for (int h = hs; h < he; h++)
          for (int w = ws; w < we; w++) sacc = dadd<T>(sacc, xs[h * W + w]);
        out = sacc / T((he - hs) * (we - ws));
      }
      yb[p * g.y.sh + q * g.y.sw] = out;
    }
    __syncthreads();
  }
}

// Backward: the plane's dy (and argmax) staged in shared memory; argmax
// entries are validated on the way in (an entry outside its own window sets
// *bad and the serial reference-order scatter redoes the whole op).
template <typename T, int KIND, int MAXK>
__global__ void __launch_bounds__(256) pool_bwd_plane_kernel(PoolGeom g, const T* __restrict__ dy,
                                                             T* __restrict__ dx,
                                                             const int64_t* __restrict__ argmax,
                                                             int* bad) {
  extern __shared__ __align__(16) uint8_t psm[];
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int wh = int(g.wh), ww = int(g.ww), sh = int(g.sh), sw = int(g.sw);
  const int ph = int(g.ph), pw = int(g.pw);
  const int PQ = P * Q, HW = H * W;
  // covering-window ranges per input row / column, shared by every plane:
  // rowtab[h] = (p0, p1), coltab[w] = (q0, q1)
  int2* rowtab = reinterpret_cast<int2*>(psm);
  int2* coltab = rowtab + H;
  uint8_t* body = psm + ((size_t(H + W) * 8 + 15) & ~size_t(15));
  int* as = reinterpret_cast<int*>(body);  // max: plane-local argmax (h * W + w) or -1
  T* ds = reinterpret_cast<T*>(body + ((size_t(PQ) * 4 + 15) & ~size_t(15)));  // dy (avg: dy / count)
  T* xs = ds + PQ;                        // max: the dx plane being assembled
  for (int i = threadIdx.x; i < H + W; i += blockDim.x) {
    const bool row = i < H;
    const int e = row ? i : i - H;
    const int k = row ? wh : ww, s = row ? sh : sw, n = row ? P : Q;
    const int ep = e + (row ? ph : pw);
    const MagicDiv dv = row ? g.dSH : g.dSW;
    const int lo = ep - k + 1 > 0 ? int(mdiv(uint32_t(ep - k + s), dv)) : 0;
    const int hi = min(n - 1, int(mdiv(uint32_t(ep), dv)));
    rowtab[i] = make_int2(lo, hi);
  }
  const int planes = int(g.N) * C;
  for (int pl = blockIdx.x; pl < planes; pl += gridDim.x) {
    uint32_t nu, cu;
    mdivmod(uint32_t(pl), g.dC, nu, cu);
    const T* dyb = dy + int64_t(nu) * g.y.sn + int64_t(cu) * g.y.sc;
    bool badl = false;
    const int64_t abase = int64_t(pl) * HW;
    // staged in batches of LB per thread: all LB loads are issued before any
    // is consumed, so one block keeps LB round trips in flight, not one
    constexpr int LB = 4;
    for (int i0 = threadIdx.x; i0 < PQ; i0 += LB * blockDim.x) {
      T dv[LB];
      int64_t av[LB];
#pragma unroll
      for (int u = 0; u < LB; u++) {
        const int i = i0 + u * int(blockDim.x);
        if (i < PQ) {
          uint32_t pu, qu;
          mdivmod(uint32_t(i), g.dQ, pu, qu);
          dv[u] = dyb[int(pu) * g.y.sh + int(qu) * g.y.sw];
          if (KIND == 0) av[u] = argmax[int64_t(pl) * PQ + i];
        }
      }
#pragma unroll
      for (int u = 0; u < LB; u++) {
      const int i = i0 + u * int(blockDim.x);
      if (i >= PQ) break;
      uint32_t pu, qu;
      mdivmod(uint32_t(i), g.dQ, pu, qu);
      const int p = int(pu), q = int(qu);
      const T d = dv[u];
      const int hs0 = p * sh - ph, ws0 = q * sw - pw;
      if (KIND == 0) {
        ds[i] = d;
        const int64_t hw = av[u] - abase;
        int loc = -1;
        if (hw >= 0 && hw < int64_t(HW)) {
          uint32_t h, w;
          mdivmod(uint32_t(hw), g.dW, h, w);
          if (int(h) >= hs0 && int(h) < hs0 + wh && int(w) >= ws0 && int(w) < ws0 + ww) loc = int(hw);
        }
        badl |= loc < 0;
        as[i] = loc;
      } else {
        const int cnt = (min(H, hs0 + wh) - max(0, hs0)) * (min(W, ws0 + ww) - max(0, ws0));
        ds[i] = d / T(cnt);  // the reference adds dy / count per window (nnops.py:237-246)
      }
      }
    }
    if (KIND == 0) {
      if (badl) *bad = 1;
      for (int i = threadIdx.x; i < HW; i += blockDim.x) xs[i] = T(0);
    }
    __syncthreads();
    T* dxb = dx + int64_t(nu) * g.x.sn + int64_t(cu) * g.x.sc;
    if (KIND == 0) {
      // window-driven: the first window (ascending (p, q)) whose argmax is
      // element t sums every covering window targeting t, in order
      for (int o = threadIdx.x; o < PQ; o += blockDim.x) {
        const int t = as[o];
        if (t < 0) continue;
        uint32_t hu, wu;
        mdivmod(uint32_t(t), g.dW, hu, wu);
        const int2 pr = rowtab[hu], qr = coltab[wu];
        const int p0 = pr.x, p1 = pr.y, q0 = qr.x, q1 = qr.y;
        bool first = true;
        T acc = T(0);
        for (int p = p0; p <= p1; p++)
          for (int q = q0; q <= q1; q++) {
            const int oo = p * Q + q;
            if (as[oo] == t) {
              if (oo < o) first = false;
              acc = dadd<T>(acc, ds[oo]);
            }
          }
        if (first) xs[t] = acc;
      }
      __syncthreads();
      if (g.x.sw == 1 && g.x.sh == W) {
        smem_to_plane(dxb, xs, HW);
      } else {
        for (int i = threadIdx.x; i < HW; i += blockDim.x) {
          uint32_t hu, wu;
          mdivmod(uint32_t(i), g.dW, hu, wu);
          dxb[int(hu) * g.x.sh + int(wu) * g.x.sw] = xs[i];
        }
      }
    } else {
      for (int i = threadIdx.x; i < HW; i += blockDim.x) {
        uint32_t hu, wu;
        mdivmod(uint32_t(i), g.dW, hu, wu);
        const int2 pr = rowtab[hu], qr = coltab[wu];
        const int p0 = pr.x, p1 = pr.y, q0 = qr.x, q1 = qr.y;
        T acc = T(0);
        if (MAXK > 0) {
#pragma unroll
          for (int dp = 0; dp < MAXK; dp++)
#pragma unroll
            for (int dq = 0; dq < MAXK; dq++)
              if (p0 + dp <= p1 && q0 + dq <= q1) acc = dadd<T>(acc, ds[(p0 + dp) * Q + q0 + dq]);
        } else {
          for (int p = p0; p <= p1; p++)
            for (int q = q0; q <= q1; q++) acc = dadd<T>(acc, ds[p * Q + q]);
        }
        dxb[int(hu) * g.x.sh + int(wu) * g.x.sw] = acc;
      }
    }
    __syncthreads();
  }
}

// Channels-innermost backward: one (n, h) row of dx per block iteration.
// The dy rows of the windows covering h (at most RM of them) are staged in
// shared memory channel-fastest (avg: dy / count; max: dy plus the
// plane-local argmax, validated -- an entry outside its window sets *bad and
// the serial scatter redoes the op), then every (w, c) of the row sums its
// covering windows in ascending (p, q) order from 0: the reference order
// (nnops.py:218-246), so the result is bit-exact.  dy reads and dx writes
// coalesce along c.
// V channels per thread (one 16-byte vector when V > 1: needs C, every
// non-channel stride and both base pointers in units of V).
template <typename T, int V>
struct alignas(V * sizeof(T)) ChanVec {
  T v[V];
};

template <typename T, int KIND, int V>
__global__ void __launch_bounds__(256) pool_bwd_cl_kernel(PoolGeom g, const T* __restrict__ dy,
                                                          T* __restrict__ dx,
                                                          const int64_t* __restrict__ argmax,
                                                          int* bad, int RM, MagicDiv dQCV,
                                                          MagicDiv dCV) {
  using VT = ChanVec<T, V>;
  extern __shared__ __align__(16) uint8_t psm[];
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int wh = int(g.wh), ww = int(g.ww), sh = int(g.sh), sw = int(g.sw);
  const int ph = int(g.ph), pw = int(g.pw);
  const int CV = C / V, QCV = Q * CV;
  int2* coltab = reinterpret_cast<int2*>(psm);
  VT* ds = reinterpret_cast<VT*>(psm + ((size_t(W) * 8 + 15) & ~size_t(15)));
  int* as = reinterpret_cast<int*>(ds + size_t(RM) * QCV);  // max: per channel, V per vector
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    const int wp = w + pw;
    const int lo = wp - ww + 1 > 0 ? int(mdiv(uint32_t(wp - ww + sw), g.dSW)) : 0;
    coltab[w] = make_int2(lo, min(Q - 1, int(mdiv(uint32_t(wp), g.dSW))));
  }
  const int rows = int(g.N) * H;
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    uint32_t nu, hu;
    mdivmod(uint32_t(row), g.dH, nu, hu);
    const int n = int(nu), h = int(hu);
    const int hp = h + ph;
    const int p0 = hp - wh + 1 > 0 ? int(mdiv(uint32_t(hp - wh + sh), g.dSH)) : 0;
    const int p1 = min(P - 1, int(mdiv(uint32_t(hp), g.dSH)));
    const int nr = max(0, p1 - p0 + 1);
    const T* dyn = dy + int64_t(n) * g.y.sn;
    bool badl = false;
    for (int i = threadIdx.x; i < nr * QCV; i += blockDim.x) {
      uint32_t r, rem, q, cv;
      mdivmod(uint32_t(i), dQCV, r, rem);
      mdivmod(rem, dCV, q, cv);
      const int p = p0 + int(r);
      VT d = *reinterpret_cast<const VT*>(dyn + int64_t(cv) * V + p * g.y.sh + int(q) * g.y.sw);
      const int hs0 = p * sh - ph, ws0 = int(q) * sw - pw;
      if (KIND == 0) {
        ds[i] = d;
#pragma unroll
        for (int j = 0; j < V; j++) {
          const int64_t plane = int64_t(n) * C + int64_t(cv) * V + j;
          const int64_t hw = argmax[(plane * P + p) * Q + q] - plane * H * W;
          int loc = -1;
          if (hw >= 0 && hw < int64_t(H) * W) {
            uint32_t ah, aw;
            mdivmod(uint32_t(hw), g.dW, ah, aw);
            if (int(ah) >= hs0 && int(ah) < hs0 + wh && int(aw) >= ws0 && int(aw) < ws0 + ww)
              loc = int(hw);
          }
          badl |= loc < 0;
          as[i * V + j] = loc;
        }
      } else {
        const int cnt = (min(H, hs0 + wh) - max(0, hs0)) * (min(W, ws0 + ww) - max(0, ws0));
#pragma unroll
        for (int j = 0; j < V; j++) d.v[j] = d.v[j] / T(cnt);
        ds[i] = d;
      }
    }
    if (KIND == 0 && badl) *bad = 1;
    __syncthreads();
    T* dxr = dx + int64_t(n) * g.x.sn + int64_t(h) * g.x.sh;
    for (int e = threadIdx.x; e < W * CV; e += blockDim.x) {
      uint32_t wu, cv;
      mdivmod(uint32_t(e), dCV, wu, cv);
      const int2 qr = coltab[wu];
      const int me = h * W + int(wu);
      VT acc;
#pragma unroll
      for (int j = 0; j < V; j++) acc.v[j] = T(0);
      for (int r = 0; r < nr; r++)
        for (int q = qr.x; q <= qr.y; q++) {
          const int idx = r * QCV + q * CV + int(cv);
          const VT d = ds[idx];
#pragma unroll
          for (int j = 0; j < V; j++) {
            if (KIND == 0) {
              if (as[idx * V + j] == me) acc.v[j] = dadd<T>(acc.v[j], d.v[j]);
            } else {
              acc.v[j] = dadd<T>(acc.v[j], d.v[j]);
            }
          }
        }
      *reinterpret_cast<VT*>(dxr + int64_t(cv) * V + int64_t(wu) * g.x.sw) = acc;
    }
    __syncthreads();
  }
}

// Serial reference-order scatter (np.add.at in flat (n,c,p,q) order).
template <typename T>
__global__ void pool_bwd_serial(PoolGeom g, const T* dy, T* dx, const int64_t* argmax,
                                int64_t total, const int* bad) {
  if (!*bad || threadIdx.x != 0 || blockIdx.x != 0) return;
  // reset dx (the gather pass wrote it) then scatter in order
  for (int64_t i = 0; i < g.N * g.C * g.H * g.W; i++) {
    int64_t w = i % g.W, h = (i / g.W) % g.H, c = (i / (g.W * g.H)) % g.C, n = i / (g.W * g.H * g.C);
    dx[voff(g.x, n, c, h, w)] = T(0);
  }
  const int64_t limit = g.N * g.C * g.H * g.W;
  for (int64_t i = 0; i < total; i++) {
    int64_t a = argmax[i];
    if (a < 0 || a >= limit) continue;
    int64_t w = a % g.W, h = (a / g.W) % g.H, c = (a / (g.W * g.H)) % g.C, n = a / (g.W * g.H * g.C);
    const int64_t q = i % g.Q, p = (i / g.Q) % g.P, pc = (i / (g.Q * g.P)) % g.C,
                  pn = i / (g.Q * g.P * g.C);
    T* t = dx + voff(g.x, n, c, h, w);
    *t = dadd<T>(*t, dy[voff(g.y, pn, pc, p, q)]);
  }
}

// ---------------------------------------------------------------------------
// 3 x 3 / stride 2 / no padding pooling on planes with unit-stride rows (the
// AlexNet / OverFeat pooling layer; SURVEY 8(d) "B" shape 55 -> 27).  One
// warp per (plane, 32 output columns); lane q owns output column q and walks
// the output rows.  Forward is separable: the 3-wide row reduction of input
// row h (first max / first NaN in w order, with its column) is computed once
// and shared by the two output rows whose windows contain it (h = 2p + 2 is
// the last row of window p and the first of p + 1); the 3-row combination
// in h order keeps the reference's row-major first-max / first-NaN pick
// (nnops.py:180-197).  ~20 instructions per output instead of a window scan
// out of shared memory; every input byte is read from DRAM once.
template <typename T>
struct RowBest {
  T v;
  int w;
};

// a later candidate wins when greater, or when it is NaN and the best is not
template <typename T>
__device__ __forceinline__ void take_best(RowBest<T>& b, T v, int w) {
  const bool take = v > b.v || (v != v && b.v == b.v);
  b.v = take ? v : b.v;
  b.w = take ? w : b.w;
}

// Warps: (plane, 32-column block, chunk of kPoolRows output rows); chunks
// keep the per-warp loop short, so the grid runs as several full waves
// (one warp per plane was ~1.15 waves of 27-row loops: the tail doubled
// the time) and more loads are in flight per SM.
constexpr int kPoolRows = 7;

// One chunk of RP output rows of one lane: the 2 RP + 1 input rows x 3
// columns are loaded up front (one memory latency per warp), row-reduced,
// then combined in h order.  Offsets are 32-bit inside one image (the host
// checks the image span), rows / columns step by the view's strides, so the
// same code serves unit-stride rows (lane = output column) and
// channels-innermost views (lane = channel).  RP is a compile-time count:
// full chunks carry no per-row predicates.
// EX = false (max): plain '>' comparisons -- the same first-maximum result
// whenever the chunk holds no NaN; returns whether it saw one (the caller
// then redoes the chunk with EX = true: the first NaN wins, numpy argmax).
template <typename T, int KIND, int RP, bool EX = true>
__device__ __forceinline__ bool pool3s2_fwd_chunk(const T* __restrict__ xi, int xo, int xsh, int xsw,
                                                  T* __restrict__ yi, int yo, int ysh,
                                                  int64_t* __restrict__ ab, int64_t abase, int aq,
                                                  int W, int p0, int w0) {
  constexpr int NR = 2 * RP + 1;
  T v[NR][3];
  bool nan = false;
#pragma unroll
  for (int r = 0; r < NR; r++) {
    const int o = xo + (2 * p0 + r) * xsh;
    v[r][0] = __ldg(xi + o);
    v[r][1] = __ldg(xi + o + xsw);
    v[r][2] = __ldg(xi + o + 2 * xsw);
    if (!EX && KIND == 0) nan |= (v[r][0] != v[r][0]) | (v[r][1] != v[r][1]) | (v[r][2] != v[r][2]);
  }
  if (!EX && KIND == 0 && nan) return true;
  T bv[NR];
  int bw[NR];
#pragma unroll
  for (int r = 0; r < NR; r++) {
    if (KIND == 0) {
      // a later value wins when greater, or when it is NaN and the best is not
      T b = v[r][0];
      int w = 0;
      bool t = v[r][1] > b || (EX && v[r][1] != v[r][1] && b == b);
      b = t ? v[r][1] : b;
      w = t ? 1 : w;
      t = v[r][2] > b || (EX && v[r][2] != v[r][2] && b == b);
      bv[r] = t ? v[r][2] : b;
      bw[r] = t ? 2 : w;
    } else {
      bv[r] = dadd<T>(dadd<T>(v[r][0], v[r][1]), v[r][2]);
    }
  }
#pragma unroll
  for (int i = 0; i < RP; i++) {
    const int p = p0 + i;
    if (KIND == 0) {
      T b = bv[2 * i];
      int code = bw[2 * i];  // 3 * (row in window) + column
      bool t = bv[2 * i + 1] > b || (EX && bv[2 * i + 1] != bv[2 * i + 1] && b == b);
      b = t ? bv[2 * i + 1] : b;
      code = t ? 3 + bw[2 * i + 1] : code;
      t = bv[2 * i + 2] > b || (EX && bv[2 * i + 2] != bv[2 * i + 2] && b == b);
      b = t ? bv[2 * i + 2] : b;
      code = t ? 6 + bw[2 * i + 2] : code;
      yi[yo + p * ysh] = b;
      if (ab) {
        const int rr = code >= 6 ? 2 : (code >= 3 ? 1 : 0);
        ab[int64_t(p) * aq] = abase + int64_t(2 * p + rr) * W + (w0 + code - 3 * rr);
      }
    } else {
      yi[yo + p * ysh] = dadd<T>(dadd<T>(bv[2 * i], bv[2 * i + 1]), bv[2 * i + 2]) / T(9);
    }
  }
  return false;
}

// Warps: (image or plane, 32 lanes, chunk of kPoolRows output rows).
// CL = 0: lane = output column q of one (n, c) plane; CL = 1: lane =
// channel c of one output column q (channels-innermost views).
template <typename T, int KIND, int CL>
__global__ void __launch_bounds__(128) pool3s2_fwd_kernel(PoolGeom g, const T* __restrict__ x,
                                                          T* __restrict__ y,
                                                          int64_t* __restrict__ argmax, int nlb,
                                                          int nrc) {
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  // CL = 0: warps over (n, c, q block, row chunk); CL = 1: (n, q, c block, row chunk)
  const int outer = CL ? int(g.N) * Q : int(g.N) * C;
  if (gw >= outer * nlb * nrc) return;
  const int rc = gw % nrc, t = gw / nrc;
  const int o = t / nlb, lb = t - o * nlb;
  int n, c, q;
  if (CL) {
    n = o / Q;
    q = o - n * Q;
    c = lb * 32 + lane;
    if (c >= C) return;
  } else {
    n = o / C;
    c = o - n * C;
    q = lb * 32 + lane;
    if (q >= Q) return;
  }
  const int p0 = rc * kPoolRows, rows = min(P - p0, kPoolRows);
  const int w0 = 2 * q;
  const T* xi = x + int64_t(n) * g.x.sn;
  T* yi = y + int64_t(n) * g.y.sn;
  const int xo = int(c * g.x.sc + w0 * g.x.sw), yo = int(c * g.y.sc + q * g.y.sw);
  const int xsh = int(g.x.sh), xsw = int(g.x.sw), ysh = int(g.y.sh);
  const int pl = n * C + c;
  int64_t* ab = argmax ? argmax + int64_t(pl) * P * Q + q : nullptr;
  const int64_t abase = int64_t(pl) * H * W;
#define DNNP_POOL_CHUNK(RP)                                                                   \
  if (pool3s2_fwd_chunk<T, KIND, RP, KIND != 0>(xi, xo, xsh, xsw, yi, yo, ysh, ab, abase, Q, W, p0, w0)) \
    pool3s2_fwd_chunk<T, KIND, RP, true>(xi, xo, xsh, xsw, yi, yo, ysh, ab, abase, Q, W, p0, w0)
  switch (rows) {
    case 7: DNNP_POOL_CHUNK(7); break;
    case 6: DNNP_POOL_CHUNK(6); break;
    case 5: DNNP_POOL_CHUNK(5); break;
    case 4: DNNP_POOL_CHUNK(4); break;
    case 3: DNNP_POOL_CHUNK(3); break;
    case 2: DNNP_POOL_CHUNK(2); break;
    default: DNNP_POOL_CHUNK(1); break;
  }
#undef DNNP_POOL_CHUNK
}

// Backward of the same geometry, gather form in the reference's summation
// order: input (h, w) receives, in ascending (p, q), dy[p][q] of every
// covering window whose argmax is (h, w) (max) or dy / 9 (average), starting
// from 0 (nnops.py:203-246, np.add.at in flat (n, c, p, q) order).  Lane l
// owns window q = 32 jb + l and input columns 2q, 2q + 1; column 2q + 2 is
// the next lane's 2(q + 1), whose share of window q arrives by shuffle and
// is added before that lane's own window (ascending q).  Each window's
// argmax is decoded once into its (row, col) inside the window and the nine
// per-position contributions are selects (adding +0.0 leaves a sum that
// starts at +0.0 unchanged, so the result is bit-identical to the scatter).
// Rows 2p, 2p + 1 complete after window row p; row 2p + 2 carries into p + 1;
// a row chunk [p0, p1) starts by re-deriving window row p0 - 1's share of
// input row 2p0.  Max: an argmax outside its window sets *bad (the serial
// scatter redoes the op).
template <typename T, int KIND>
__global__ void __launch_bounds__(128) pool3s2_bwd_kernel(PoolGeom g, const T* __restrict__ dy,
                                                          T* __restrict__ dx,
                                                          const int64_t* __restrict__ argmax,
                                                          int* bad, int nqb, int nrc) {
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int planes = int(g.N) * C;
  if (gw >= planes * nqb * nrc) return;  // warp-uniform
  const int rc = gw % nrc, tt = gw / nrc;
  const int pl = tt / nqb, jb = tt - pl * nqb;
  const int q = jb * 32 + lane;           // this lane's window column
  const int w0 = 2 * q;
  const int p0 = rc * kPoolRows, p1 = min(P, p0 + kPoolRows);
  const bool own = q < Q;                 // lane has a window
  const bool live = w0 < W;               // lane owns input columns
  const bool has1 = w0 + 1 < W;
  const bool edge = lane == 0 && q > 0 && q - 1 < Q;  // window q - 1 is in the previous warp
  const int n = pl / C, c = pl - n * C;
  const T* dyb = dy + int64_t(n) * g.y.sn + int64_t(c) * g.y.sc;
  T* dxb = dx + int64_t(n) * g.x.sn + int64_t(c) * g.x.sc + int64_t(w0) * g.x.sw;
  const int64_t* ab = argmax ? argmax + int64_t(pl) * P * Q : nullptr;
  const int64_t abase = int64_t(pl) * H * W;
  // window (p, qq): its dy (avg: / 9) and the argmax position inside the
  // window, pos = 3 row + col in [0, 9), or -1 when outside (max)
  auto fetch = [&](int p, int qq, T& d, int& pos) {
    d = __ldg(dyb + int64_t(p) * g.y.sh + int64_t(qq) * g.y.sw);
    pos = -1;
    if (KIND == 0) {
      const int64_t rel = __ldg(ab + int64_t(p) * Q + qq) - abase -
                          (int64_t(2 * p) * W + 2 * qq);
      if (rel >= 0 && rel < 3 * int64_t(W)) {
        uint32_t r, cc;
        mdivmod(uint32_t(rel), g.dW, r, cc);
        if (cc <= 2) pos = int(r) * 3 + int(cc);
      }
    } else {
      d = d / T(9);
    }
  };
  constexpr int NW = kPoolRows + 1;  // window rows p0 - 1 .. p1 - 1
  T dv[NW], de[NW];
  int pv[NW], pe[NW];
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const int p = p0 - 1 + i;
    dv[i] = de[i] = T(0);
    pv[i] = pe[i] = -1;
    if (p >= 0 && p < p1) {
      if (own) fetch(p, q, dv[i], pv[i]);
      if (edge) fetch(p, q - 1, de[i], pe[i]);
    }
  }
  // the share of window (., q) at window row r, window column cc
  auto sel = [&](T d, int pos, bool has, int r, int cc) -> T {
    return has && (KIND != 0 || pos == 3 * r + cc) ? d : T(0);
  };
  bool badl = false;
  T e0 = T(0), e1 = T(0);  // pending row 2p (columns 2q, 2q + 1)
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const int p = p0 - 1 + i;
    if (p >= p1) break;
    if (p < p0 && p < 0) continue;
    // column-2 shares of window q - 1, rows 0..2 (shuffle; lane 0 decodes it)
    T prev[3];
#pragma unroll
    for (int r = 0; r < 3; r++) {
      const T mine = sel(dv[i], pv[i], own, r, 2);
      const T up = __shfl_up_sync(0xffffffffu, mine, 1);
      prev[r] = lane == 0 ? sel(de[i], pe[i], edge, r, 2) : up;
    }
    if (p < p0) {  // window row p0 - 1: only its last row (2 p0) is this chunk's
      e0 = dadd<T>(dadd<T>(T(0), prev[2]), sel(dv[i], pv[i], own, 2, 0));
      e1 = dadd<T>(T(0), sel(dv[i], pv[i], own, 2, 1));
      continue;
    }
    if (KIND == 0 && own && pv[i] < 0) badl = true;
    const int h0 = 2 * p;
    // row h0: pending (window row p - 1), then (p, q - 1), then (p, q)
    const T o0 = dadd<T>(dadd<T>(e0, prev[0]), sel(dv[i], pv[i], own, 0, 0));
    const T o1 = dadd<T>(e1, sel(dv[i], pv[i], own, 0, 1));
    const T m0 = dadd<T>(dadd<T>(T(0), prev[1]), sel(dv[i], pv[i], own, 1, 0));
    const T m1 = dadd<T>(T(0), sel(dv[i], pv[i], own, 1, 1));
    e0 = dadd<T>(dadd<T>(T(0), prev[2]), sel(dv[i], pv[i], own, 2, 0));
    e1 = dadd<T>(T(0), sel(dv[i], pv[i], own, 2, 1));
    if (live) {
      T* r0p = dxb + int64_t(h0) * g.x.sh;
      r0p[0] = o0;
      if (has1) r0p[g.x.sw] = o1;
      r0p += g.x.sh;
      r0p[0] = m0;
      if (has1) r0p[g.x.sw] = m1;
    }
  }
  if (p1 == P && live) {
    // the last pending row and any rows past the last window (zero)
    for (int h = 2 * P; h < H; h++) {
      const T v0 = h == 2 * P ? e0 : T(0), v1 = h == 2 * P ? e1 : T(0);
      dxb[int64_t(h) * g.x.sh] = v0;
      if (has1) dxb[int64_t(h) * g.x.sh + g.x.sw] = v1;
    }
  }
  if (KIND == 0 && badl) atomicExch(bad, 1);
}

// Lean 3 x 3 / 2 backward (unit-stride dx rows): every window sends its dy
// (max: to one element, avg: dy / 9 to all nine) and a dx element sums the
// <= 4 windows that reach it in window row-major order, as the reference's
// scatter does (bit-exact).  Lane = window column q (and dx columns 2q,
// 2q + 1), loop = window rows p: per row one window fetch, two shuffles for
// the left neighbour (p, q - 1), the row-(p - 1) windows carried in
// registers; outputs the 2 x 2 block (2p + a, 2q + b).
template <typename T, int KIND>
__global__ void __launch_bounds__(128, sizeof(T) == 4 ? 12 : 8) pool3s2_bwd_lean_kernel(PoolGeom g, const T* __restrict__ dy,
                                                               T* __restrict__ dx,
                                                               const int64_t* __restrict__ argmax,
                                                               int* bad, int nqb, int nrc, int rows,
                                                               int vec) {
  const int H = int(g.H), W = int(g.W), P = int(g.P), Q = int(g.Q), C = int(g.C);
  const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int planes = int(g.N) * C;
  if (gw >= planes * nqb * nrc) return;  // warp-uniform
  const int rc = gw % nrc, tt = gw / nrc;
  const int pl = tt / nqb, jb = tt - pl * nqb;
  const int q = jb * 32 + lane;
  const int p0 = rc * rows, p1 = min(P, p0 + rows);
  const int n = pl / C, c = pl - n * C;
  const T* dyb = dy + int64_t(n) * g.y.sn + int64_t(c) * g.y.sc;
  T* dxb = dx + int64_t(n) * g.x.sn + int64_t(c) * g.x.sc;
  const int64_t* ab = KIND == 0 ? argmax + int64_t(pl) * P * Q : nullptr;
  const int64_t abase = int64_t(pl) * H * W;
  const bool edge = lane == 0 && q > 0 && q - 1 < Q;  // window q - 1 lives in the previous warp
  bool badl = false;
  // window (p, qq): value and code = 3 r + cc of its target (max; -1: none),
  // 9 = every position (avg)
  auto fetch = [&](int p, int qq, T& v, int& code) {
    v = T(0);
    code = -1;
    if (p < 0 || p >= P || qq < 0 || qq >= Q) return;
    v = __ldg(dyb + int64_t(p) * g.y.sh + int64_t(qq) * g.y.sw);
    if (KIND == 0) {
      const int64_t rel = __ldg(ab + int64_t(p) * Q + qq) - abase - (int64_t(2 * p) * W + 2 * qq);
      if (rel >= 0 && rel < 3 * int64_t(W)) {
        const int rl = int(rel);
        const int r = rl >= 2 * W ? 2 : (rl >= W ? 1 : 0);
        const int cc = rl - r * W;
        if (cc <= 2) code = 3 * r + cc;
      }
      if (code < 0) badl = true;
    } else {
      v = v / T(9);
      code = 9;
    }
  };
  // contribution of a window with (v, code) to block element (a, b) when it
  // would reach it at window position (r, cc)
  auto hit = [](T v, int code, int r, int cc) -> T {
    return (KIND != 0 ? code == 9 : code == 3 * r + cc) ? v : T(0);
  };
  T vU, vUL;  // windows (p - 1, q) and (p - 1, q - 1)
  int cU, cUL;
  fetch(p0 - 1, q, vU, cU);
  {
    T lv = __shfl_up_sync(0xffffffffu, vU, 1);
    int lc = __shfl_up_sync(0xffffffffu, cU, 1);
    if (edge) fetch(p0 - 1, q - 1, lv, lc);
    vUL = lane == 0 && !edge ? T(0) : lv;
    cUL = lane == 0 && !edge ? -1 : lc;
  }
  const int w0 = 2 * q;
  const bool live = w0 < W, has1 = w0 + 1 < W;
  for (int p = p0; p < p1; p++) {
    T v;
    int cd;
    fetch(p, q, v, cd);
    T vL = __shfl_up_sync(0xffffffffu, v, 1);
    int cL = __shfl_up_sync(0xffffffffu, cd, 1);
    if (edge) fetch(p, q - 1, vL, cL);
    if (lane == 0 && !edge) {
      vL = T(0);
      cL = -1;
    }
    // window order: (p-1, q-1), (p-1, q), (p, q-1), (p, q)
    const T o00 = dadd<T>(dadd<T>(dadd<T>(dadd<T>(T(0), hit(vUL, cUL, 2, 2)), hit(vU, cU, 2, 0)),
                                 hit(vL, cL, 0, 2)), hit(v, cd, 0, 0));
    const T o01 = dadd<T>(dadd<T>(T(0), hit(vU, cU, 2, 1)), hit(v, cd, 0, 1));
    const T o10 = dadd<T>(dadd<T>(T(0), hit(vL, cL, 1, 2)), hit(v, cd, 1, 0));
    const T o11 = dadd<T>(T(0), hit(v, cd, 1, 1));
    if (live) {
      T* r0p = dxb + int64_t(2 * p) * g.x.sh + w0;
      if (vec && has1) {
        using T2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;
        T2 a, b;
        a.x = o00; a.y = o01;
        b.x = o10; b.y = o11;
        *reinterpret_cast<T2*>(r0p) = a;
        *reinterpret_cast<T2*>(r0p + g.x.sh) = b;
      } else {
        r0p[0] = o00;
        if (has1) r0p[1] = o01;
        r0p[g.x.sh] = o10;
        if (has1) r0p[g.x.sh + 1] = o11;
      }
    }
    vUL = vL;
    cUL = cL;
    vU = v;
    cU = cd;
  }
  if (p1 == P && live) {
    // row 2P: the row-(P - 1) windows' last rows; rows past it: zero
    for (int h = 2 * P; h < H; h++) {
      T o0 = T(0), o1 = T(0);
      if (h == 2 * P) {
        o0 = dadd<T>(dadd<T>(T(0), hit(vUL, cUL, 2, 2)), hit(vU, cU, 2, 0));
        o1 = dadd<T>(T(0), hit(vU, cU, 2, 1));
      }
      dxb[int64_t(h) * g.x.sh + w0] = o0;
      if (has1) dxb[int64_t(h) * g.x.sh + w0 + 1] = o1;
    }
  }
  if (KIND == 0 && badl) atomicExch(bad, 1);
}

// whether the 3 x 3 / 2 plane kernels take this problem
// the geometry of the 3 x 3 / 2 kernels (no padding, every window inside)
static bool pool3s2_geom(const PoolProblem& pp, const View4& xv, const View4& yv) {
  auto span = [](const View4& v) {  // largest element offset inside one image
    return (v.c - 1) * v.sc + (v.h - 1) * v.sh + (v.w - 1) * v.sw;
  };
  return pp.wh == 3 && pp.ww == 3 && pp.sh == 2 && pp.sw == 2 && pp.ph == 0 && pp.pw == 0 &&
         xv.h >= 3 && xv.w >= 3 && pp.P == (xv.h - 3) / 2 + 1 && pp.Q == (xv.w - 3) / 2 + 1 &&
         span(xv) < (int64_t(1) << 31) && span(yv) < (int64_t(1) << 31) &&
         xv.n * xv.c * xv.h * xv.w < (int64_t(1) << 40) &&
         xv.n * xv.c * ceil_div(xv.w, 64) * ceil_div(xv.h, 14) < (int64_t(1) << 26) &&
         xv.n * pp.Q * ceil_div(xv.c, 32) * ceil_div(xv.h, 14) < (int64_t(1) << 26) &&
         !::dnnp::tune_env("DNNP_POOL_NO_3S2");
}
// forward: any strides (lanes along w for unit-stride rows, else along c)
static bool pool3s2_ok(const PoolProblem& pp, const View4& xv, const View4& yv) {
  return pool3s2_geom(pp, xv, yv);
}
// backward: unit-stride rows (lanes along w, shuffles between windows)
static bool pool3s2_bwd_ok(const PoolProblem& pp, const View4& xv, const View4& yv) {
  return pool3s2_geom(pp, xv, yv) && xv.sw == 1 && yv.sw == 1;
}

// Plane kernels: one (n, c) plane per block iteration, staged in shared
// memory.  Small blocks and an uncapped grid keep many planes per SM in
// flight, so one block's load phase overlaps another's compute phase.
static int pool_threads() {
  static int t = [] {
    const char* e = ::dnnp::tune_env("DNNP_POOL_THREADS");
    const int v = e ? atoi(e) : 128;
    return (v == 64 || v == 128 || v == 256) ? v : 128;
  }();
  return t;
}
static int64_t pool_grid_cap() {
  static int64_t c = [] {
    const char* e = ::dnnp::tune_env("DNNP_POOL_GRID");
    return e ? int64_t(atoll(e)) : (int64_t(1) << 30);
  }();
  return c;
}

static PoolGeom pool_geom(const PoolProblem& pp, const View4& xv, const View4& yv) {
  PoolGeom g;
  g.x = xv;
  g.y = yv;
  g.N = xv.n; g.C = xv.c; g.H = xv.h; g.W = xv.w; g.P = pp.P; g.Q = pp.Q;
  g.wh = pp.wh; g.ww = pp.ww; g.sh = pp.sh; g.sw = pp.sw; g.ph = pp.ph; g.pw = pp.pw;
  g.dQ = make_magic(uint32_t(pp.Q));
  g.dP = make_magic(uint32_t(pp.P));
  g.dC = make_magic(uint32_t(xv.c));
  g.dW = make_magic(uint32_t(xv.w));
  g.dH = make_magic(uint32_t(xv.h));
  g.dSH = make_magic(uint32_t(pp.sh));
  g.dSW = make_magic(uint32_t(pp.sw));
  return g;
}

cudaError_t pool_forward(const PoolProblem& pp, Dtype dt, const View4& xv, const void* x,
                         const View4& yv, void* y, int64_t* argmax, cudaStream_t st) {
  const int64_t total = yv.size();
  if (total >= (int64_t(1) << 32) || xv.size() >= (int64_t(1) << 32))
    return cudaErrorInvalidValue;
  PoolGeom g = pool_geom(pp, xv, yv);
  const size_t eb = dt == F32 ? 4 : 8;
  const size_t psm = size_t(xv.h) * xv.w * eb;
  if (pool3s2_ok(pp, xv, yv)) {
    // lanes along the unit-stride dimension: output columns (rows with sw
    // == 1) or channels (channels-innermost views)
    const bool cl = xv.sw != 1;
    const int nlb = int(ceil_div(cl ? xv.c : pp.Q, 32)), nrc = int(ceil_div(pp.P, kPoolRows));
    const unsigned blocks = unsigned(ceil_div(xv.n * (cl ? pp.Q : xv.c) * nlb * nrc, 4));
    auto go = [&](auto tag, auto kind, auto clc) {
      using TT = decltype(tag);
      pool3s2_fwd_kernel<TT, decltype(kind)::value, decltype(clc)::value><<<blocks, 128, 0, st>>>(
          g, (const TT*)x, (TT*)y, argmax, nlb, nrc);
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    if (dt == F32) {
      if (pp.kind == 0) { if (cl) go(float(), I0(), I1()); else go(float(), I0(), I0()); }
      else { if (cl) go(float(), I1(), I1()); else go(float(), I1(), I0()); }
    } else {
      if (pp.kind == 0) { if (cl) go(double(), I0(), I1()); else go(double(), I0(), I0()); }
      else { if (cl) go(double(), I1(), I1()); else go(double(), I1(), I0()); }
    }
    note_launch();
    return cudaGetLastError();
  }
  if (xv.sc == 1 && yv.sc == 1 && xv.c >= 16 && !::dnnp::tune_env("DNNP_POOL_NO_CL")) {
    // channels innermost: channel-vectorised rows instead of planes
    const int nqb = int(ceil_div(pp.Q, 32)), ncb = int(ceil_div(xv.c, 32));
    const int64_t blocks = xv.n * pp.P * nqb * ncb;
    if (blocks < (int64_t(1) << 31)) {
      auto go = [&](auto tag, auto kc) {
        using TT = decltype(tag);
        pool_fwd_cl_kernel<TT, decltype(kc)::value><<<unsigned(blocks), 256, 0, st>>>(
            g, (const TT*)x, (TT*)y, argmax, nqb, ncb);
      };
      using I0 = std::integral_constant<int, 0>;
      using I1 = std::integral_constant<int, 1>;
      if (dt == F32) {
        if (pp.kind == 0) go(float(), I0()); else go(float(), I1());
      } else {
        if (pp.kind == 0) go(double(), I0()); else go(double(), I1());
      }
      note_launch();
      return cudaGetLastError();
    }
  }
  const bool dense_planes = xv.sw == 1 && xv.sh == xv.w;
  const int pitch = int(((xv.h * xv.w + 16 / eb) * eb + 15) / 16 * 16 / eb);
  const size_t ppipe = size_t(2) * pitch * eb;
  // the cp.async pipeline pays for fp64 planes (max-pool 50 -> 61% of HBM);
  // fp32 stays on the one-plane-per-block kernel (issue-bound either way,
  // and faster on channel-slice views)
  if (dt == F64 && dense_planes && ppipe <= 96 * 1024 && xv.n * xv.c < (int64_t(1) << 31) &&
      !::dnnp::tune_env("DNNP_POOL_NO_PIPE") && !::dnnp::tune_env("DNNP_POOL_DIRECT")) {
    const int kw = (pp.wh == pp.ww && (pp.wh == 2 || pp.wh == 3)) ? int(pp.wh) : 0;
    const int per_sm = std::max(1, int(std::min<size_t>(4, (200 * 1024) / ppipe)));
    const unsigned pg = unsigned(std::min<int64_t>(xv.n * xv.c, int64_t(kNumSMs) * per_sm));
    auto go = [&](auto tag, auto kwc) {
      using TT = decltype(tag);
      auto kfn = pool_fwd_pipe_kernel<TT, decltype(kwc)::value>;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ppipe));
      kfn<<<pg, 256, ppipe, st>>>(g, (const TT*)x, (TT*)y, argmax, pp.kind, pitch);
    };
    using K0 = std::integral_constant<int, 0>;
    using K2 = std::integral_constant<int, 2>;
    using K3 = std::integral_constant<int, 3>;
    if (dt == F32) {
      if (kw == 3) go(float(), K3()); else if (kw == 2) go(float(), K2()); else go(float(), K0());
    } else {
      if (kw == 3) go(double(), K3()); else if (kw == 2) go(double(), K2()); else go(double(), K0());
    }
    note_launch();
    return cudaGetLastError();
  }
  if (psm <= 48 * 1024 && xv.n * xv.c < (int64_t(1) << 31) && !::dnnp::tune_env("DNNP_POOL_DIRECT")) {
    const int thr = pool_threads();
    const unsigned pg = unsigned(std::min<int64_t>(xv.n * xv.c, pool_grid_cap()));
    const int kw = (pp.wh == pp.ww && (pp.wh == 2 || pp.wh == 3)) ? int(pp.wh) : 0;
    auto go = [&](auto tag, auto kwc) {
      using TT = decltype(tag);
      pool_fwd_plane_kernel<TT, decltype(kwc)::value><<<pg, thr, psm, st>>>(
          g, (const TT*)x, (TT*)y, argmax, pp.kind);
    };
    using K0 = std::integral_constant<int, 0>;
    using K2 = std::integral_constant<int, 2>;
    using K3 = std::integral_constant<int, 3>;
    if (dt == F32) {
      if (kw == 3) go(float(), K3()); else if (kw == 2) go(float(), K2()); else go(float(), K0());
    } else {
      if (kw == 3) go(double(), K3()); else if (kw == 2) go(double(), K2()); else go(double(), K0());
    }
    note_launch();
    return cudaGetLastError();
  }
  unsigned grid = grid_for(total, 256, 8);
  const int kwd = (pp.wh == pp.ww && (pp.wh == 2 || pp.wh == 3)) ? int(pp.wh) : 0;
  auto god = [&](auto tag, auto kwc) {
    using TT = decltype(tag);
    pool_fwd_kernel<TT, decltype(kwc)::value><<<grid, 256, 0, st>>>(g, (const TT*)x, (TT*)y,
                                                                     argmax, pp.kind, total);
  };
  {
    using K0 = std::integral_constant<int, 0>;
    using K2 = std::integral_constant<int, 2>;
    using K3 = std::integral_constant<int, 3>;
    if (dt == F32) {
      if (kwd == 3) god(float(), K3()); else if (kwd == 2) god(float(), K2()); else god(float(), K0());
    } else {
      if (kwd == 3) god(double(), K3()); else if (kwd == 2) god(double(), K2()); else god(double(), K0());
    }
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t pool_backward(const PoolProblem& pp, Dtype dt, const View4& dyv, const void* dy,
                          const View4& dxv, void* dx, const int64_t* argmax, cudaStream_t st) {
  const int64_t total = dxv.size(), ptotal = dyv.size();
  if (total >= (int64_t(1) << 32) || ptotal >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
  PoolGeom g = pool_geom(pp, dxv, dyv);
  const size_t eb = dt == F32 ? 4 : 8;
  const size_t psm = ((size_t(dxv.h + dxv.w) * 8 + 15) & ~size_t(15)) +
                     ((size_t(dyv.h) * dyv.w * 4 + 15) & ~size_t(15)) + size_t(dyv.h) * dyv.w * eb +
                     (pp.kind == 0 ? size_t(dxv.h) * dxv.w * eb : 0);
  if (pool3s2_bwd_ok(pp, dxv, dyv)) {
    int* bad = nullptr;
    tc::Workspace ws(st);
    if (pp.kind == 0) {
      cudaError_t e = ws.alloc(sizeof(int));
      if (e != cudaSuccess) return e;
      bad = static_cast<int*>(ws.p);
      cudaMemsetAsync(bad, 0, sizeof(int), st);
    }
    // lanes = window columns plus the input columns past the last window
    const int nqb = int(ceil_div(ceil_div(dxv.w, 2), 32)), nrc = int(ceil_div(pp.P, kPoolRows));
    const unsigned blocks = unsigned(ceil_div(dxv.n * dxv.c * nqb * nrc, 4));
    if (!::dnnp::tune_env("DNNP_POOL_NO_LEAN")) {
      const int vec = (dxv.sh % 2 == 0 && dxv.sc % 2 == 0 && dxv.sn % 2 == 0 &&
                       reinterpret_cast<uintptr_t>(dx) % (2 * eb) == 0) ? 1 : 0;
      const int rows = ::dnnp::tune_env("DNNP_POOL_ROWS") ? std::max(1, atoi(::dnnp::tune_env("DNNP_POOL_ROWS")))
                                                          : kPoolRows;
      const int nrl = int(ceil_div(pp.P, rows));
      const unsigned lblocks = unsigned(ceil_div(dxv.n * dxv.c * nqb * nrl, 4));
      if (dt == F32) {
        if (pp.kind == 0)
          pool3s2_bwd_lean_kernel<float, 0><<<lblocks, 128, 0, st>>>(g, (const float*)dy, (float*)dx, argmax, bad, nqb, nrl, rows, vec);
        else
          pool3s2_bwd_lean_kernel<float, 1><<<lblocks, 128, 0, st>>>(g, (const float*)dy, (float*)dx, argmax, bad, nqb, nrl, rows, vec);
      } else {
        if (pp.kind == 0)
          pool3s2_bwd_lean_kernel<double, 0><<<lblocks, 128, 0, st>>>(g, (const double*)dy, (double*)dx, argmax, bad, nqb, nrl, rows, vec);
        else
          pool3s2_bwd_lean_kernel<double, 1><<<lblocks, 128, 0, st>>>(g, (const double*)dy, (double*)dx, argmax, bad, nqb, nrl, rows, vec);
      }
    } else if (dt == F32) {
      if (pp.kind == 0)
        pool3s2_bwd_kernel<float, 0><<<blocks, 128, 0, st>>>(g, (const float*)dy, (float*)dx, argmax, bad, nqb, nrc);
      else
        pool3s2_bwd_kernel<float, 1><<<blocks, 128, 0, st>>>(g, (const float*)dy, (float*)dx, argmax, bad, nqb, nrc);
    } else {
      if (pp.kind == 0)
        pool3s2_bwd_kernel<double, 0><<<blocks, 128, 0, st>>>(g, (const double*)dy, (double*)dx, argmax, bad, nqb, nrc);
      else
        pool3s2_bwd_kernel<double, 1><<<blocks, 128, 0, st>>>(g, (const double*)dy, (double*)dx, argmax, bad, nqb, nrc);
    }
    note_launch();
    if (pp.kind == 0) {
      if (dt == F32)
        pool_bwd_serial<float><<<1, 32, 0, st>>>(g, (const float*)dy, (float*)dx, argmax, ptotal, bad);
      else
        pool_bwd_serial<double><<<1, 32, 0, st>>>(g, (const double*)dy, (double*)dx, argmax, ptotal, bad);
      note_launch();
    }
    return cudaGetLastError();
  }
  // channels innermost: the element-wise gather in (n, h, w, c) order (the
  // plane kernel would read and write every plane at stride C)
  const bool cl = dxv.sc == 1 && dyv.sc == 1 && dxv.c >= 16 && !::dnnp::tune_env("DNNP_POOL_NO_CL");
  const int rm = int(ceil_div(pp.wh, pp.sh));
  const size_t clsm = ((size_t(dxv.w) * 8 + 15) & ~size_t(15)) +
                      size_t(rm) * dyv.w * dyv.c * (eb + (pp.kind == 0 ? 4 : 0));
  if (cl && clsm <= 48 * 1024 && dxv.n * dxv.h < (int64_t(1) << 31)) {
    tc::Workspace ws(st);
    cudaError_t e = ws.alloc(sizeof(int));
    if (e != cudaSuccess) return e;
    int* bad = static_cast<int*>(ws.p);
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    const unsigned grid = unsigned(std::min<int64_t>(dxv.n * dxv.h, int64_t(1) << 30));
    // 16-byte channel vectors when every non-channel stride, C and both
    // base pointers allow it
    const int vv = int(16 / eb);
    const bool vec = !::dnnp::tune_env("DNNP_POOL_NO_VEC") && dxv.c % vv == 0 &&
                     dxv.sn % vv == 0 && dxv.sh % vv == 0 && dxv.sw % vv == 0 &&
                     dyv.sn % vv == 0 && dyv.sh % vv == 0 && dyv.sw % vv == 0 &&
                     (uintptr_t(dx) % 16) == 0 && (uintptr_t(dy) % 16) == 0;
    const int cvn = vec ? int(dxv.c) / vv : int(dxv.c);
    const MagicDiv dqcv = make_magic(uint32_t(dyv.w * cvn)), dcv = make_magic(uint32_t(cvn));
    auto launch = [&](auto tag, auto kindc) {
      using TT = decltype(tag);
      constexpr int VV = int(16 / sizeof(TT));
      if (vec)
        pool_bwd_cl_kernel<TT, decltype(kindc)::value, VV><<<grid, 256, clsm, st>>>(
            g, (const TT*)dy, (TT*)dx, argmax, bad, rm, dqcv, dcv);
      else
        pool_bwd_cl_kernel<TT, decltype(kindc)::value, 1><<<grid, 256, clsm, st>>>(
            g, (const TT*)dy, (TT*)dx, argmax, bad, rm, dqcv, dcv);
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    if (dt == F32) {
      if (pp.kind == 0) launch(float(), I0()); else launch(float(), I1());
    } else {
      if (pp.kind == 0) launch(double(), I0()); else launch(double(), I1());
    }
    note_launch();
    if (pp.kind == 0) {
      if (dt == F32)
        pool_bwd_serial<float><<<1, 32, 0, st>>>(g, (const float*)dy, (float*)dx, argmax,
                                                 ptotal, bad);
      else
        pool_bwd_serial<double><<<1, 32, 0, st>>>(g, (const double*)dy, (double*)dx, argmax,
                                                  ptotal, bad);
      note_launch();
    }
    return cudaGetLastError();
  }
  if (!cl && psm <= 48 * 1024 && dxv.n * dxv.c < (int64_t(1) << 31) &&
      !::dnnp::tune_env("DNNP_POOL_BWD_DIRECT") && dxv.h * dxv.w < (int64_t(1) << 31)) {
    tc::Workspace ws(st);
    cudaError_t e = ws.alloc(sizeof(int));
    if (e != cudaSuccess) return e;
    int* bad = static_cast<int*>(ws.p);
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    const unsigned pg = unsigned(std::min<int64_t>(dxv.n * dxv.c, pool_grid_cap()));
    const int thr = pool_threads();
    // windows covering one element per dim: ceil(window / stride)
    const int64_t kmax = std::max(ceil_div(pp.wh, pp.sh), ceil_div(pp.ww, pp.sw));
    const int mk = kmax <= 2 ? 2 : (kmax <= 4 ? 4 : 0);
    auto launch = [&](auto tag, auto kindc, auto mkc) {
      using TT = decltype(tag);
      pool_bwd_plane_kernel<TT, decltype(kindc)::value, decltype(mkc)::value>
          <<<pg, thr, psm, st>>>(g, (const TT*)dy, (TT*)dx, argmax, bad);
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I4 = std::integral_constant<int, 4>;
    if (dt == F32) {
      if (pp.kind == 0) {
        if (mk == 2) launch(float(), I0(), I2()); else if (mk == 4) launch(float(), I0(), I4()); else launch(float(), I0(), I0());
      } else {
        if (mk == 2) launch(float(), I1(), I2()); else if (mk == 4) launch(float(), I1(), I4()); else launch(float(), I1(), I0());
      }
    } else {
      if (pp.kind == 0) {
        if (mk == 2) launch(double(), I0(), I2()); else if (mk == 4) launch(double(), I0(), I4()); else launch(double(), I0(), I0());
      } else {
        if (mk == 2) launch(double(), I1(), I2()); else if (mk == 4) launch(double(), I1(), I4()); else launch(double(), I1(), I0());
      }
    }
    note_launch();
    if (pp.kind == 0) {
      if (dt == F32)
        pool_bwd_serial<float><<<1, 32, 0, st>>>(g, (const float*)dy, (float*)dx, argmax,
                                                 ptotal, bad);
      else
        pool_bwd_serial<double><<<1, 32, 0, st>>>(g, (const double*)dy, (double*)dx, argmax,
                                                  ptotal, bad);
      note_launch();
    }
    return cudaGetLastError();
  }
  unsigned grid = grid_for(total, 256, 8);
  if (cl) {
    if (dt == F32)
      pool_bwd_kernel<float, true><<<grid, 256, 0, st>>>(g, (const float*)dy, (float*)dx,
                                                         argmax, pp.kind, total);
    else
      pool_bwd_kernel<double, true><<<grid, 256, 0, st>>>(g, (const double*)dy, (double*)dx,
                                                          argmax, pp.kind, total);
  } else if (dt == F32) {
    pool_bwd_kernel<float><<<grid, 256, 0, st>>>(g, (const float*)dy, (float*)dx, argmax,
                                                 pp.kind, total);
  } else {
    pool_bwd_kernel<double><<<grid, 256, 0, st>>>(g, (const double*)dy, (double*)dx, argmax,
                                                  pp.kind, total);
  }
  note_launch();
  if (pp.kind == 0) {
    tc::Workspace ws(st);
    cudaError_t e = ws.alloc(sizeof(int));
    if (e != cudaSuccess) return e;
    int* bad = static_cast<int*>(ws.p);
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    pool_argmax_check<<<grid_for(ptotal, 256, 4), 256, 0, st>>>(g, argmax, ptotal, bad);
    if (dt == F32)
      pool_bwd_serial<float><<<1, 32, 0, st>>>(g, (const float*)dy, (float*)dx, argmax, ptotal,
                                               bad);
    else
      pool_bwd_serial<double><<<1, 32, 0, st>>>(g, (const double*)dy, (double*)dx, argmax,
                                                ptotal, bad);
    note_launch(2);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------- conv bias gradient
//
// db[k] = sum_{n,p,q} dy[n,k,p,q] (reference conv.py:754-760).  Two
// deterministic phases: K x S blocks reduce contiguous slices of the
// (n, p, q) range, then one thread per k adds the S partials in order.
template <typename T>
__global__ void __launch_bounds__(256) bias_partial(View4 v, const T* __restrict__ dy, int S,
                                                    MagicDiv dPQ, MagicDiv dQ, T* part) {
  __shared__ T sh[32];
  const int64_t k = blockIdx.y;
  const int64_t L = v.n * v.h * v.w;
  const int64_t per = (L + S - 1) / S;
  const int64_t j0 = blockIdx.x * per, j1 = min(L, j0 + per);
  T s = T(0);
  for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    uint32_t n, rem, p, q;
    mdivmod(uint32_t(j), dPQ, n, rem);
    mdivmod(rem, dQ, p, q);
    s += dy[n * v.sn + k * v.sc + p * v.sh + q * v.sw];
  }
  s = block_reduce_sum(s, sh);
  if (threadIdx.x == 0) part[k * S + blockIdx.x] = s;
}
template <typename T, typename TO>
__global__ void bias_final(const T* part, int S, int64_t K, View4 ov, TO* db) {
  int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  T s = T(0);
  for (int i = 0; i < S; i++) s += part[k * S + i];
  db[k * ov.sc] = TO(s);
}

template <typename T>
static cudaError_t bias_t(const View4& v, const T* dy, const View4& ov, Dtype dbt, void* db,
                          cudaStream_t st) {
  const int64_t L = v.n * v.h * v.w;
  if (L >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
  int64_t S = std::max<int64_t>(1, ceil_div(int64_t(kNumSMs) * 8, v.c));
  S = std::min<int64_t>(S, std::max<int64_t>(1, ceil_div(L, 1024)));
  tc::Workspace ws(st);
  cudaError_t e = ws.alloc(sizeof(T) * v.c * S);
  if (e != cudaSuccess) return e;
  T* part = static_cast<T*>(ws.p);
  bias_partial<T><<<dim3(unsigned(S), unsigned(v.c)), 256, 0, st>>>(
      v, dy, int(S), make_magic(uint32_t(v.h * v.w)), make_magic(uint32_t(v.w)), part);
  unsigned g = unsigned(ceil_div(v.c, 128));
  if (dbt == F32)
    bias_final<T, float><<<g, 128, 0, st>>>(part, int(S), v.c, ov, (float*)db);
  else
    bias_final<T, double><<<g, 128, 0, st>>>(part, int(S), v.c, ov, (double*)db);
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t conv_backward_bias(const View4& dyv, Dtype dt, const void* dy, const View4& dbv,
                               Dtype dbt, void* db, cudaStream_t st) {
  return dt == F32 ? bias_t(dyv, (const float*)dy, dbv, dbt, db, st)
                   : bias_t(dyv, (const double*)dy, dbv, dbt, db, st);
}

}  // namespace dnnp

extern "C" int64_t dnnp_kernel_launch_count(void) { return dnnp::g_launches.load(); }
