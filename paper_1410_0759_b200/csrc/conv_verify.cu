// Device loop nests for verification (the GPU CLI's --verify; SURVEY 8(f)
// rank 1).  The reference harness checks every engine against an
// independent path, its direct engine (pkg/src/dnnp/bench.py:196-203); the
// device counterpart here is the definition of each pass written as a plain
// loop nest (the reference's tests/oracles.py shape), fp64 accumulation in a
// fixed order, one thread per output element.  It shares nothing with the
// implicit-GEMM kernels -- no packing, no magic division, no tensor cores,
// no tiling -- so an error in those shows up against it.  Not a product
// path: it is only reachable through dnnp_convolution_verify_reference.
#include <cstdint>

#include "common.cuh"

namespace dnnp {
namespace {

// input coordinate of tap r at output p (reference conv.py:182-192 access)
__device__ __forceinline__ int64_t tap_in(int64_t p, int64_t stride, int64_t R, int64_t r,
                                          int64_t pad, bool flip) {
  return p * stride + (flip ? R - 1 - r : r) - pad;
}

template <typename T>
__global__ void verify_fwd(ConvProblem pr, const T* x, const T* f, double* y) {
  const int64_t total = pr.N * pr.K * pr.P * pr.Q;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = i % pr.Q, p = (i / pr.Q) % pr.P, k = (i / (pr.Q * pr.P)) % pr.K,
                  n = i / (pr.Q * pr.P * pr.K);
    double acc = 0.0;
    for (int64_t c = 0; c < pr.C; c++)
      for (int64_t r = 0; r < pr.R; r++) {
        const int64_t h = tap_in(p, pr.u, pr.R, r, pr.pad_h, pr.flip);
        if (h < 0 || h >= pr.H) continue;
        for (int64_t s = 0; s < pr.S; s++) {
          const int64_t w = tap_in(q, pr.v, pr.S, s, pr.pad_w, pr.flip);
          if (w < 0 || w >= pr.W) continue;
          acc = fma(double(f[((k * pr.C + c) * pr.R + r) * pr.S + s]),
                    double(x[voff(pr.x, n, c, h, w)]), acc);
        }
      }
    y[i] = acc;  // dense NCHW
  }
}

template <typename T>
__global__ void verify_bwd_data(ConvProblem pr, const T* dy, const T* f, double* dx) {
  const int64_t total = pr.N * pr.C * pr.H * pr.W;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = i % pr.W, h = (i / pr.W) % pr.H, c = (i / (pr.W * pr.H)) % pr.C,
                  n = i / (pr.W * pr.H * pr.C);
    double acc = 0.0;
    for (int64_t k = 0; k < pr.K; k++)
      for (int64_t r = 0; r < pr.R; r++) {
        // outputs p whose tap r reads row h: p * u = h + pad - tap
        const int64_t ph = h + pr.pad_h - (pr.flip ? pr.R - 1 - r : r);
        if (ph < 0 || ph % pr.u) continue;
        const int64_t p = ph / pr.u;
        if (p >= pr.P) continue;
        for (int64_t s = 0; s < pr.S; s++) {
          const int64_t qw = w + pr.pad_w - (pr.flip ? pr.S - 1 - s : s);
          if (qw < 0 || qw % pr.v) continue;
          const int64_t q = qw / pr.v;
          if (q >= pr.Q) continue;
          acc = fma(double(f[((k * pr.C + c) * pr.R + r) * pr.S + s]),
                    double(dy[voff(pr.y, n, k, p, q)]), acc);
        }
      }
    dx[i] = acc;
  }
}

template <typename T>
__global__ void verify_bwd_filter(ConvProblem pr, const T* dy, const T* x, double* df) {
  const int64_t total = pr.K * pr.C * pr.R * pr.S;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = i % pr.S, r = (i / pr.S) % pr.R, c = (i / (pr.S * pr.R)) % pr.C,
                  k = i / (pr.S * pr.R * pr.C);
    double acc = 0.0;
    for (int64_t n = 0; n < pr.N; n++)
      for (int64_t p = 0; p < pr.P; p++) {
        const int64_t h = tap_in(p, pr.u, pr.R, r, pr.pad_h, pr.flip);
        if (h < 0 || h >= pr.H) continue;
        for (int64_t q = 0; q < pr.Q; q++) {
          const int64_t w = tap_in(q, pr.v, pr.S, s, pr.pad_w, pr.flip);
          if (w < 0 || w >= pr.W) continue;
          acc = fma(double(dy[voff(pr.y, n, k, p, q)]), double(x[voff(pr.x, n, c, h, w)]), acc);
        }
      }
    df[i] = acc;
  }
}

template <typename T>
cudaError_t launch(int pass, const ConvProblem& pr, const void* a, const void* b, double* out,
                   cudaStream_t st) {
  const int64_t total = pass == 0   ? pr.N * pr.K * pr.P * pr.Q
                        : pass == 1 ? pr.N * pr.C * pr.H * pr.W
                                    : pr.K * pr.C * pr.R * pr.S;
  const unsigned grid = grid_for(total, 128, 64);
  const T* ta = static_cast<const T*>(a);
  const T* tb = static_cast<const T*>(b);
  if (pass == 0) verify_fwd<T><<<grid, 128, 0, st>>>(pr, ta, tb, out);
  else if (pass == 1) verify_bwd_data<T><<<grid, 128, 0, st>>>(pr, ta, tb, out);
  else verify_bwd_filter<T><<<grid, 128, 0, st>>>(pr, ta, tb, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

// pass 0: out[N][K][P][Q] = conv(x = a, f = b); pass 1: out[N][C][H][W] =
// bwd_data(dy = a, f = b); pass 2: out[K][C][R][S] = bwd_filter(dy = a, x = b).
// Output dense and fp64, whatever the input type.
cudaError_t conv_verify_reference(int pass, const ConvProblem& pr, Dtype dt, const void* a,
                                  const void* b, double* out, cudaStream_t st) {
  return dt == F64 ? launch<double>(pass, pr, a, b, out, st)
                   : launch<float>(pass, pr, a, b, out, st);
}

}  // namespace dnnp
