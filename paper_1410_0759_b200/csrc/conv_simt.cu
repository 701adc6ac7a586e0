// SIMT implicit-GEMM convolution (forward, backward-data, backward-filter)
// for fp64 (production path) and fp32 (DNNP_MATH_SIMT_FP32 / ineligible
// shapes).  The lowered data matrix is never materialised: every tile of it
// is gathered straight from the strided input with magic-number index
// decode, as in the reference's virtual provider (conv.py:235-356) driven by
// the tiled engine (gemm.py:140-181).
//
// GEMM orientation (M rows are output pixels so the epilogue writes
// contiguous runs of q):
//   forward      C[NPQ x K]   = im2col(x)[NPQ x CRS] . F[K x CRS]^T
//   backward-data C[NHW x C]  = gather(dy)[NHW x KRS] . F^T      (gather form,
//                 no scatter/atomics: every dx element is owned by one thread)
//   backward-filter C[K x CRS] = dy[K x NPQ] . im2col(x)[NPQ x CRS], split-K
//                 over NPQ with a fixed-order reduction (deterministic).
#include <algorithm>

#include <type_traits>

#include "common.cuh"
#include "tc_common.cuh"

namespace dnnp {

enum Pass { FWD = 0, DGRAD = 1, WGRAD = 2 };

struct SimtArgs {
  ConvProblem p;
  const void* a_src;  // FWD: x, DGRAD: dy, WGRAD: dy
  const void* b_src;  // FWD: f, DGRAD: f,  WGRAD: x
  void* out;          // FWD: y, DGRAD: dx, WGRAD: df or split workspace
  int64_t M, Ncol, Kred;
  int64_t k_per_split;
  double alpha, beta;
  int accumulate;
  int splits;
  // decoders
  MagicDiv dRS, dS, dPQ, dQ, dHW, dW, dU, dV;
  // backward-data stride phases: blockIdx.z = phase (ph, pw); rows (n, i, j)
  // of the phase grid Hph x Wph (h = i*u + ph), reduction (k, jr, js) over
  // the gather offsets r' = t0(ph) + u*jr only (the other u-1 of every u taps
  // never reach a pixel of this phase)
  int Hph, Wph, nRp, nSp;
  MagicDiv dHWph, dWph, dRSph, dSph;
};

template <typename T>
struct SimtCfg;
template <>
struct SimtCfg<float> {
  static constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;
};
template <>
struct SimtCfg<double> {
  static constexpr int BM = 64, BN = 64, BK = 8, TM = 4, TN = 4;
};
// fp64 backward-data: 16-deep k-steps halve the barriers per FMA of the
// phase-gathered reduction (AlexNet conv2-5 bwd-data 5.2-8.5 -> 6.4-9.6 TF/s;
// the same change costs forward / backward-filter, tools/bench_f64.py)
struct SimtCfgDgrad64 {
  static constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
};
// Narrow GEMM outputs (N <= 16 columns, e.g. table2 layer1 bwd-data: C = 3):
// a 64-wide tile wastes >= 75% of its FMAs, so rows take the width.
template <typename T>
struct SimtNarrow;
template <>
struct SimtNarrow<float> {
  static constexpr int BM = 128, BN = 16, BK = 16, TM = 8, TN = 2;
};
template <>
struct SimtNarrow<double> {
  static constexpr int BM = 128, BN = 16, BK = 16, TM = 4, TN = 2;
};

// A(m, k) element of the pass' left operand.
template <typename T, int PASS>
struct RowCtx {
  int64_t base;     // pass-specific row base offset
  int32_t hb, wb;   // FWD: p*u - pad_h, q*v - pad_w; DGRAD: h + pad_h, w + pad_w
  uint32_t n;
  bool valid;
};

template <typename T, int PASS>
__device__ __forceinline__ RowCtx<T, PASS> row_ctx(const SimtArgs& a, int64_t m) {
  RowCtx<T, PASS> rc;
  rc.valid = m < a.M;
  const ConvProblem& p = a.p;
  if (!rc.valid) {
    rc.base = 0; rc.hb = rc.wb = 0; rc.n = 0;
    return rc;
  }
  if (PASS == FWD) {
    uint32_t n, rem, pp, qq;
    mdivmod(uint32_t(m), a.dPQ, n, rem);
    mdivmod(rem, a.dQ, pp, qq);
    rc.n = n;
    rc.base = int64_t(n) * p.x.sn;
    rc.hb = int32_t(pp * p.u - p.pad_h);
    rc.wb = int32_t(qq * p.v - p.pad_w);
  } else if (PASS == DGRAD) {
    uint32_t n, rem, i, j;
    mdivmod(uint32_t(m), a.dHWph, n, rem);
    mdivmod(rem, a.dWph, i, j);
    const int u = int(p.u), v = int(p.v);
    const int ph = int(blockIdx.z) / v, pw = int(blockIdx.z) - (int(blockIdx.z) / v) * v;
    const int h = int(i) * u + ph, w = int(j) * v + pw;
    rc.valid = h < p.H && w < p.W;
    rc.n = n;
    rc.base = int64_t(n) * p.y.sn;
    rc.hb = int32_t(h + p.pad_h);
    rc.wb = int32_t(w + p.pad_w);
  } else {  // WGRAD: row = output channel k of dy
    rc.n = 0;
    rc.base = m * p.y.sc;
    rc.hb = rc.wb = 0;
  }
  return rc;
}

template <typename T, int PASS>
__device__ __forceinline__ T load_a(const SimtArgs& a, const RowCtx<T, PASS>& rc, int64_t k,
                                    int t0h, int t0w) {
  const ConvProblem& p = a.p;
  if (!rc.valid || k >= a.Kred) return T(0);
  const T* src = static_cast<const T*>(a.a_src);
  if (PASS == FWD) {
    uint32_t c, rs, r, s;
    mdivmod(uint32_t(k), a.dRS, c, rs);
    mdivmod(rs, a.dS, r, s);
    const int32_t hr = p.flip ? int32_t(p.R - 1 - r) : int32_t(r);
    const int32_t wr = p.flip ? int32_t(p.S - 1 - s) : int32_t(s);
    const int32_t h = rc.hb + hr, w = rc.wb + wr;
    if (uint32_t(h) >= uint32_t(p.H) || uint32_t(w) >= uint32_t(p.W)) return T(0);
    return src[rc.base + int64_t(c) * p.x.sc + int64_t(h) * p.x.sh + int64_t(w) * p.x.sw];
  } else if (PASS == DGRAD) {
    uint32_t kk, rs, jr, js;
    mdivmod(uint32_t(k), a.dRSph, kk, rs);
    mdivmod(rs, a.dSph, jr, js);
    const int32_t ro = t0h + int32_t(p.u) * int32_t(jr);  // gather offset
    const int32_t so = t0w + int32_t(p.v) * int32_t(js);
    if (ro >= p.R || so >= p.S) return T(0);
    const int32_t th = rc.hb - ro, tw = rc.wb - so;  // = p*u, q*v exactly
    if (th < 0 || tw < 0) return T(0);
    const uint32_t pp = mdiv(uint32_t(th), a.dU), qq = mdiv(uint32_t(tw), a.dV);
    if (pp >= uint32_t(p.P) || qq >= uint32_t(p.Q)) return T(0);
    return src[rc.base + int64_t(kk) * p.y.sc + int64_t(pp) * p.y.sh + int64_t(qq) * p.y.sw];
  } else {
    uint32_t n, rem, pp, qq;
    mdivmod(uint32_t(k), a.dPQ, n, rem);
    mdivmod(rem, a.dQ, pp, qq);
    return src[rc.base + int64_t(n) * p.y.sn + int64_t(pp) * p.y.sh + int64_t(qq) * p.y.sw];
  }
}

// B(col, k) element of the right operand (stored as [col][k]).
template <typename T, int PASS>
__device__ __forceinline__ T load_b(const SimtArgs& a, int64_t col, int64_t k, int t0h, int t0w) {
  const ConvProblem& p = a.p;
  if (col >= a.Ncol || k >= a.Kred) return T(0);
  const T* src = static_cast<const T*>(a.b_src);
  if (PASS == FWD) {
    return src[col * a.Kred + k];  // f[kout][crs]
  } else if (PASS == DGRAD) {
    uint32_t kk, rs, jr, js;
    mdivmod(uint32_t(k), a.dRSph, kk, rs);
    mdivmod(rs, a.dSph, jr, js);
    const int32_t ro = t0h + int32_t(p.u) * int32_t(jr);
    const int32_t so = t0w + int32_t(p.v) * int32_t(js);
    if (ro >= p.R || so >= p.S) return T(0);
    const int32_t r = p.flip ? int32_t(p.R - 1 - ro) : ro, s = p.flip ? int32_t(p.S - 1 - so) : so;
    return src[((int64_t(kk) * p.C + col) * p.R + r) * p.S + s];  // f[kout][c][r][s]
  } else {
    uint32_t c, rs, r, s, n, rem, pp, qq;
    mdivmod(uint32_t(col), a.dRS, c, rs);
    mdivmod(rs, a.dS, r, s);
    mdivmod(uint32_t(k), a.dPQ, n, rem);
    mdivmod(rem, a.dQ, pp, qq);
    const int32_t hr = p.flip ? int32_t(p.R - 1 - r) : int32_t(r);
    const int32_t wr = p.flip ? int32_t(p.S - 1 - s) : int32_t(s);
    const int32_t h = int32_t(pp * p.u - p.pad_h) + hr;
    const int32_t w = int32_t(qq * p.v - p.pad_w) + wr;
    if (uint32_t(h) >= uint32_t(p.H) || uint32_t(w) >= uint32_t(p.W)) return T(0);
    return src[int64_t(n) * p.x.sn + int64_t(c) * p.x.sc + int64_t(h) * p.x.sh +
               int64_t(w) * p.x.sw];
  }
}

template <typename T, int PASS, class CFG>
__global__ void __launch_bounds__((CFG::BM / CFG::TM) * (CFG::BN / CFG::TN))
    conv_simt_kernel(SimtArgs a) {
  constexpr int BM = CFG::BM, BN = CFG::BN, BK = CFG::BK;
  constexpr int TM = CFG::TM, TN = CFG::TN;
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int LA = BM * BK / NT, LB = BN * BK / NT;
  static_assert(NT % BM == 0 || PASS == WGRAD, "row-fast A mapping");
  __shared__ T As[2][BK][BM + 4];
  __shared__ T Bs[2][BK][BN + 4];

  const int tid = threadIdx.x;
  const int64_t m0 = int64_t(blockIdx.x) * BM, n0 = int64_t(blockIdx.y) * BN;
  const int64_t kbeg = (PASS == WGRAD ? int64_t(blockIdx.z) : 0) * a.k_per_split;
  const int64_t kend = min(a.Kred, kbeg + a.k_per_split);

  // A mapping: FWD/DGRAD rows fastest (coalesced along q / w); WGRAD k fastest.
  int a_mi[LA], a_ki[LA];
  RowCtx<T, PASS> rc[LA];
#pragma unroll
  for (int j = 0; j < LA; j++) {
    int e = tid + j * NT;
    if (PASS == WGRAD) {
      a_ki[j] = e % BK;
      a_mi[j] = e / BK;
    } else {
      a_mi[j] = e % BM;
      a_ki[j] = e / BM;
    }
    rc[j] = row_ctx<T, PASS>(a, m0 + a_mi[j]);
  }
  int b_ni[LB], b_ki[LB];
#pragma unroll
  for (int j = 0; j < LB; j++) {
    int e = tid + j * NT;
    b_ki[j] = e % BK;
    b_ni[j] = e / BK;
  }

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) acc[i][j] = T(0);

  int t0h = 0, t0w = 0;
  if (PASS == DGRAD) {
    const int v = int(a.p.v);
    t0h = (int(blockIdx.z) / v + int(a.p.pad_h)) % int(a.p.u);
    t0w = (int(blockIdx.z) - (int(blockIdx.z) / v) * v + int(a.p.pad_w)) % v;
  }
  T ra[LA], rb[LB];
  auto gload = [&](int64_t k0) {
#pragma unroll
    for (int j = 0; j < LA; j++) {
      int64_t k = k0 + a_ki[j];
      ra[j] = k < kend ? load_a<T, PASS>(a, rc[j], k, t0h, t0w) : T(0);
    }
#pragma unroll
    for (int j = 0; j < LB; j++) {
      int64_t k = k0 + b_ki[j];
      rb[j] = k < kend ? load_b<T, PASS>(a, n0 + b_ni[j], k, t0h, t0w) : T(0);
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int j = 0; j < LA; j++) As[buf][a_ki[j]][a_mi[j]] = ra[j];
#pragma unroll
    for (int j = 0; j < LB; j++) Bs[buf][b_ki[j]][b_ni[j]] = rb[j];
  };

  const int tr = tid / (BN / TN), tc = tid % (BN / TN);
  int buf = 0;
  if (kbeg < kend) {
    gload(kbeg);
    sstore(0);
    __syncthreads();
    for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
      const bool more = k0 + BK < kend;
      if (more) gload(k0 + BK);
#pragma unroll
      for (int kk = 0; kk < BK; kk++) {
        T av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; i++) av[i] = As[buf][kk][tr + i * (BM / TM)];
#pragma unroll
        for (int j = 0; j < TN; j++) bv[j] = Bs[buf][kk][tc + j * (BN / TN)];
#pragma unroll
        for (int i = 0; i < TM; i++)
#pragma unroll
          for (int j = 0; j < TN; j++) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
      if (more) {
        sstore(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }

  // epilogue
  const ConvProblem& p = a.p;
  T* out = static_cast<T*>(a.out);
#pragma unroll
  for (int i = 0; i < TM; i++) {
    const int64_t m = m0 + tr + i * (BM / TM);
    if (m >= a.M) continue;
    int64_t rowoff;
    if (PASS == FWD) {
      uint32_t n, rem, pp, qq;
      mdivmod(uint32_t(m), a.dPQ, n, rem);
      mdivmod(rem, a.dQ, pp, qq);
      rowoff = int64_t(n) * p.y.sn + int64_t(pp) * p.y.sh + int64_t(qq) * p.y.sw;
    } else if (PASS == DGRAD) {
      uint32_t n, rem, ii, jj;
      mdivmod(uint32_t(m), a.dHWph, n, rem);
      mdivmod(rem, a.dWph, ii, jj);
      const int h = int(ii) * int(p.u) + int(blockIdx.z) / int(p.v);
      const int w = int(jj) * int(p.v) + int(blockIdx.z) % int(p.v);
      if (h >= p.H || w >= p.W) continue;
      rowoff = int64_t(n) * p.x.sn + int64_t(h) * p.x.sh + int64_t(w) * p.x.sw;
    } else {
      rowoff = m * a.Ncol + int64_t(blockIdx.z) * a.M * a.Ncol * (a.splits > 1 ? 1 : 0);
    }
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int64_t col = n0 + tc + j * (BN / TN);
      if (col >= a.Ncol) continue;
      const T v = acc[i][j];
      if (PASS == FWD) {
        T* dst = out + rowoff + col * p.y.sc;
        T r = dmul<T>(v, T(a.alpha));
        if (a.beta != 0.0) r = dadd<T>(dmul<T>(*dst, T(a.beta)), r);
        *dst = r;
      } else if (PASS == DGRAD) {
        T* dst = out + rowoff + col * p.x.sc;
        *dst = a.accumulate ? dadd<T>(*dst, v) : v;
      } else {
        T* dst = out + rowoff + col;
        *dst = (a.splits == 1 && a.accumulate) ? dadd<T>(*dst, v) : v;
      }
    }
  }
}

// df[i] (+)= sum_z ws[z][i] in ascending z (deterministic split-K reduction)
template <typename T>
__global__ void splitk_reduce(const T* __restrict__ ws, int splits, int64_t count, T* df,
                              int accumulate) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    T s = ws[i];
    for (int z = 1; z < splits; z++) s = dadd<T>(s, ws[int64_t(z) * count + i]);
    df[i] = accumulate ? dadd<T>(df[i], s) : s;
  }
}

static void fill_divs(SimtArgs& a) {
  const ConvProblem& p = a.p;
  a.dRS = make_magic(uint32_t(p.R * p.S));
  a.dS = make_magic(uint32_t(p.S));
  a.dPQ = make_magic(uint32_t(p.P * p.Q));
  a.dQ = make_magic(uint32_t(p.Q));
  a.dHW = make_magic(uint32_t(p.H * p.W));
  a.dW = make_magic(uint32_t(p.W));
  a.dU = make_magic(uint32_t(p.u));
  a.dV = make_magic(uint32_t(p.v));
  a.dHWph = make_magic(uint32_t(a.Hph * a.Wph > 0 ? a.Hph * a.Wph : 1));
  a.dWph = make_magic(uint32_t(a.Wph > 0 ? a.Wph : 1));
  a.dRSph = make_magic(uint32_t(a.nRp * a.nSp > 0 ? a.nRp * a.nSp : 1));
  a.dSph = make_magic(uint32_t(a.nSp > 0 ? a.nSp : 1));
}

template <typename T, int PASS, class CFG = SimtCfg<T>>
static cudaError_t launch_simt_cfg(SimtArgs& a, cudaStream_t st) {
  constexpr int BM = CFG::BM, BN = CFG::BN, BK = CFG::BK;
  constexpr int NT = (BM / CFG::TM) * (BN / CFG::TN);
  fill_divs(a);
  const int64_t gm = ceil_div(a.M, BM), gn = ceil_div(a.Ncol, BN);
  a.splits = 1;
  a.k_per_split = a.Kred;
  T* ws = nullptr;
  tc::Workspace wsa(st);
  void* final_out = a.out;
  if (PASS == WGRAD) {
    int64_t tiles = gm * gn;
    int64_t want = ceil_div(int64_t(kNumSMs) * 3, tiles);
    int64_t maxs = std::max<int64_t>(1, a.Kred / (BK * 16));
    int64_t s = std::max<int64_t>(1, std::min<int64_t>({want, maxs, 256}));
    if (s > 1) {
      a.k_per_split = ceil_div(ceil_div(a.Kred, s), BK) * BK;
      s = ceil_div(a.Kred, a.k_per_split);
    }
    a.splits = int(s);
    if (a.splits > 1) {
      cudaError_t e = wsa.alloc(sizeof(T) * a.splits * a.M * a.Ncol);
      if (e != cudaSuccess) return e;
      ws = static_cast<T*>(wsa.p);
      a.out = ws;
    }
  }
  dim3 grid(unsigned(gm), unsigned(gn),
            unsigned(PASS == DGRAD ? a.p.u * a.p.v : a.splits));
  if (gn > 65535) return cudaErrorInvalidConfiguration;
  conv_simt_kernel<T, PASS, CFG><<<grid, NT, 0, st>>>(a);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (ws) {
    const int64_t count = a.M * a.Ncol;
    splitk_reduce<T><<<grid_for(count, 256, 8), 256, 0, st>>>(ws, a.splits, count,
                                                              static_cast<T*>(final_out),
                                                              a.accumulate);
    note_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  return e;
}

template <typename T, int PASS>
static cudaError_t launch_simt(SimtArgs& a, cudaStream_t st) {
  if (PASS != WGRAD && a.Ncol <= 16 && a.M >= 4096 && !::dnnp::tune_env("DNNP_SIMT_NO_NARROW"))
    return launch_simt_cfg<T, PASS, SimtNarrow<T>>(a, st);
  if constexpr (PASS == DGRAD && std::is_same<T, double>::value)
    return launch_simt_cfg<T, PASS, SimtCfgDgrad64>(a, st);
  return launch_simt_cfg<T, PASS, SimtCfg<T>>(a, st);
}

template <typename T>
static cudaError_t simt_forward(const ConvProblem& p, const void* x, const void* f, void* y,
                                double alpha, double beta, cudaStream_t st) {
  SimtArgs a{};
  a.p = p;
  a.a_src = x;
  a.b_src = f;
  a.out = y;
  a.M = p.N * p.P * p.Q;
  a.Ncol = p.K;
  a.Kred = p.C * p.R * p.S;
  a.alpha = alpha;
  a.beta = beta;
  return launch_simt<T, FWD>(a, st);
}
template <typename T>
static cudaError_t simt_bwd_data(const ConvProblem& p, const void* dy, const void* f, void* dx,
                                 bool acc, cudaStream_t st) {
  SimtArgs a{};
  a.p = p;
  a.a_src = dy;
  a.b_src = f;
  a.out = dx;
  a.Hph = int(ceil_div(p.H, p.u));
  a.Wph = int(ceil_div(p.W, p.v));
  a.nRp = int(ceil_div(p.R, p.u));
  a.nSp = int(ceil_div(p.S, p.v));
  a.M = p.N * a.Hph * a.Wph;
  a.Ncol = p.C;
  a.Kred = p.K * a.nRp * a.nSp;
  a.accumulate = acc;
  return launch_simt<T, DGRAD>(a, st);
}
template <typename T>
static cudaError_t simt_bwd_filter(const ConvProblem& p, const void* dy, const void* x, void* df,
                                  bool acc, cudaStream_t st) {
  SimtArgs a{};
  a.p = p;
  a.a_src = dy;
  a.b_src = x;
  a.out = df;
  a.M = p.K;
  a.Ncol = p.C * p.R * p.S;
  a.Kred = p.N * p.P * p.Q;
  a.accumulate = acc;
  return launch_simt<T, WGRAD>(a, st);
}

// ---- tensor-core path (conv_tc.cu, wgrad_tc.cu) -----------------------------
// es: the fp32 split, 2 = BF16x3 (kind::f16), 4 = 3xTF32 (kind::tf32)
cudaError_t tc_forward(const ConvProblem& p, const float* x, const float* f, float* y,
                       double alpha, double beta, cudaStream_t st, int es);
cudaError_t tc_backward_data(const ConvProblem& p, const float* dy, const float* f, float* dx,
                             bool acc, cudaStream_t st, int es);
cudaError_t tc_backward_filter(const ConvProblem& p, const float* dy, const float* x, float* df,
                               bool acc, cudaStream_t st, int es);
cudaError_t tc_forward_fused(const ConvProblem& p, const float* x, const float* f, float* y,
                             double alpha, double beta, const ConvEpilogue& ep, cudaStream_t st,
                             int es);
cudaError_t tc_backward_data_fused(const ConvProblem& p, const float* dy, const float* f,
                                   float* dx, bool acc, const ConvEpilogue& ep, cudaStream_t st,
                                   int es);

// math (dnnp_math_mode): 0 default (BF16x3 tensor cores when eligible), 1
// SIMT fp32, 2 force BF16x3 tensor cores, 3 3xTF32 tensor cores (geometries
// outside the TMA im2col kernels run the SIMT fp32 kernels instead)
static bool use_tc(const ConvProblem& p, Dtype dt, int math, int pass, cudaError_t* err) {
  *err = cudaSuccess;
  if (dt != F32 || math == 1) return false;
  bool ok = tc_eligible(p, pass);
  if (!ok && math == 2) *err = cudaErrorNotSupported;
  return ok;
}

static int split_es(int math) { return math == 3 ? 4 : 2; }

// A 3xTF32 call the TMA kernels cannot take (NotSupported before any
// output write) continues on the SIMT fp32 kernels.
static bool tf32_fallback(int math, cudaError_t e) {
  if (math != 3 || e != cudaErrorNotSupported) return false;
  cudaGetLastError();
  return true;
}

// Explicit lowering (engine EXPLICIT, forward): D[n][(c,r,s)][p][q] =
// x[n][c][access(p, r)][access(q, s)] (0 outside), the reference's
// lower_explicit data matrix (conv.py:494-525) stored as an NCHW tensor of
// C*R*S channels, then the 1x1 convolution of D with the filter viewed as
// K x CRS.  The lowered matrix is the auxiliary memory the implicit kernels
// avoid (the paper's point); kept as the negative control.
template <typename T>
__global__ void __launch_bounds__(256) lower_kernel(const ConvProblem p, const T* __restrict__ x,
                                                    T* __restrict__ d, uint32_t total, MagicDiv dQ,
                                                    MagicDiv dP, MagicDiv dCRS, MagicDiv dS,
                                                    MagicDiv dR) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t t, q, pp, cp, n, rs, s, c, r;
    mdivmod(i, dQ, t, q);
    mdivmod(t, dP, t, pp);
    mdivmod(t, dCRS, n, cp);
    mdivmod(cp, dS, rs, s);
    mdivmod(rs, dR, c, r);
    const int64_t h = int64_t(pp) * p.u + (p.flip ? p.R - 1 - r : r) - p.pad_h;
    const int64_t w = int64_t(q) * p.v + (p.flip ? p.S - 1 - s : s) - p.pad_w;
    T v = T(0);
    if (h >= 0 && h < p.H && w >= 0 && w < p.W)
      v = x[int64_t(n) * p.x.sn + int64_t(c) * p.x.sc + h * p.x.sh + w * p.x.sw];
    d[i] = v;
  }
}

static cudaError_t explicit_forward(const ConvProblem& p, Dtype dt, const void* x, const void* f,
                                    void* y, double alpha, double beta, int math,
                                    cudaStream_t st) {
  const int64_t crs = p.C * p.R * p.S, total = p.N * crs * p.P * p.Q;
  const size_t es = dt == F64 ? 8 : 4;
  if (total * int64_t(es) > (int64_t(4) << 30) || total >= (int64_t(1) << 32))
    return cudaErrorMemoryAllocation;  // AllocTooLarge (reference conv.py:31)
  tc::ScratchScope* sc = tc::scratch_open(st);
  void* d = nullptr;
  cudaError_t e = tc::scratch_alloc(sc, size_t(total) * es, &d);
  if (e == cudaSuccess) {
    const unsigned grid = unsigned(std::min<int64_t>((total + 255) / 256, int64_t(148) * 16));
    const MagicDiv dQ = make_magic(uint32_t(p.Q)), dP = make_magic(uint32_t(p.P)),
                   dCRS = make_magic(uint32_t(crs)), dS = make_magic(uint32_t(p.S)),
                   dR = make_magic(uint32_t(p.R));
    if (dt == F32)
      lower_kernel<float><<<grid, 256, 0, st>>>(p, (const float*)x, (float*)d, uint32_t(total), dQ,
                                                dP, dCRS, dS, dR);
    else
      lower_kernel<double><<<grid, 256, 0, st>>>(p, (const double*)x, (double*)d, uint32_t(total),
                                                 dQ, dP, dCRS, dS, dR);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    ConvProblem q = p;  // 1x1 convolution of D (C*R*S channels) with the K x CRS filter
    q.C = crs;
    q.H = p.P;
    q.W = p.Q;
    q.R = q.S = 1;
    q.u = q.v = 1;
    q.pad_h = q.pad_w = 0;
    q.flip = false;
    q.engine = 2;
    q.x = View4{p.N, crs, p.P, p.Q, crs * p.P * p.Q, p.P * p.Q, p.Q, 1};
    e = conv_forward(q, dt, d, f, y, alpha, beta, math, st);
  }
  tc::scratch_close(sc);
  return e;
}

cudaError_t conv_forward(const ConvProblem& p, Dtype dt, const void* x, const void* f, void* y,
                         double alpha, double beta, int math, cudaStream_t st) {
  cudaError_t e;
  if (p.engine == 1) return explicit_forward(p, dt, x, f, y, alpha, beta, math, st);
  if (use_tc(p, dt, math, FWD, &e)) {
    e = tc_forward(p, (const float*)x, (const float*)f, (float*)y, alpha, beta, st, split_es(math));
    if (!tf32_fallback(math, e)) return e;
    e = cudaSuccess;
  }
  if (e != cudaSuccess) return e;
  return dt == F32 ? simt_forward<float>(p, x, f, y, alpha, beta, st)
                   : simt_forward<double>(p, x, f, y, alpha, beta, st);
}

cudaError_t conv_backward_data(const ConvProblem& p, Dtype dt, const void* dy, const void* f,
                               void* dx, bool accumulate, int math, cudaStream_t st) {
  cudaError_t e;
  if (use_tc(p, dt, math, DGRAD, &e)) {
    e = tc_backward_data(p, (const float*)dy, (const float*)f, (float*)dx, accumulate, st,
                         split_es(math));
    if (!tf32_fallback(math, e)) return e;
    e = cudaSuccess;
  }
  if (e != cudaSuccess) return e;
  return dt == F32 ? simt_bwd_data<float>(p, dy, f, dx, accumulate, st)
                   : simt_bwd_data<double>(p, dy, f, dx, accumulate, st);
}

cudaError_t conv_backward_filter(const ConvProblem& p, Dtype dt, const void* dy, const void* x,
                                 void* df, bool accumulate, int math, cudaStream_t st) {
  cudaError_t e;
  if (use_tc(p, dt, math, WGRAD, &e)) {
    e = tc_backward_filter(p, (const float*)dy, (const float*)x, (float*)df, accumulate, st,
                           split_es(math));
    if (!tf32_fallback(math, e)) return e;
    e = cudaSuccess;
  }
  if (e != cudaSuccess) return e;
  return dt == F32 ? simt_bwd_filter<float>(p, dy, x, df, accumulate, st)
                   : simt_bwd_filter<double>(p, dy, x, df, accumulate, st);
}

cudaError_t conv_backward_both(const ConvProblem& p, Dtype dt, const void* dy, const void* f,
                               const void* x, void* dx, void* df, bool accumulate, int math,
                               cudaStream_t st) {
  cudaError_t e;
  const bool tcd = use_tc(p, dt, math, DGRAD, &e);
  if (e != cudaSuccess) return e;
  const bool tcw = use_tc(p, dt, math, WGRAD, &e);
  if (e != cudaSuccess) return e;
  // one dy pack serves both GEMMs when their packed widths agree (K % 64 == 0)
  if (tcd && tcw && math != 3 && p.K % 64 == 0 && !::dnnp::tune_env("DNNP_NO_SHARED_DY")) {
    tc::ScratchScope* sc = tc::scratch_open(st);
    e = tc::shared_dy_pack(sc, p.y, static_cast<const float*>(dy), int(p.K), st);
    if (e == cudaSuccess) e = conv_backward_data(p, dt, dy, f, dx, accumulate, math, st);
    if (e == cudaSuccess) e = conv_backward_filter(p, dt, dy, x, df, accumulate, math, st);
    tc::shared_dy_clear();
    tc::scratch_close(sc);
    return e;
  }
  e = conv_backward_data(p, dt, dy, f, dx, accumulate, math, st);
  if (e == cudaSuccess) e = conv_backward_filter(p, dt, dy, x, df, accumulate, math, st);
  return e;
}

static bool same_strides(const View4& a, const View4& b) {
  return a.sn == b.sn && a.sc == b.sc && a.sh == b.sh && a.sw == b.sw;
}

// Fused forward: in the tensor-core epilogue when the path allows, else the
// same result as conv -> add_broadcast -> activation (all device kernels).
cudaError_t conv_forward_fused(const ConvProblem& p, Dtype dt, const void* x, const void* f,
                               void* y, double alpha, double beta, int math,
                               const ConvEpilogue& ep, cudaStream_t st) {
  cudaError_t e;
  if (use_tc(p, dt, math, FWD, &e)) {
    e = tc_forward_fused(p, (const float*)x, (const float*)f, (float*)y, alpha, beta, ep, st,
                         split_es(math));
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
  } else if (e != cudaSuccess) {
    return e;
  }
  if ((e = conv_forward(p, dt, x, f, y, alpha, beta, math, st)) != cudaSuccess) return e;
  if (ep.bias && (e = add_broadcast(dt, ep.biasv, ep.bias, p.y, y, 1.0, 1.0, st)) != cudaSuccess)
    return e;
  if (ep.act >= 0) return activation_forward(ep.act, dt, p.y, y, p.y, y, st);
  return cudaSuccess;
}

// Fused backward-data: gated in the epilogue when g shares dx's strides,
// else conv_bwd_data into scratch -> activation_backward -> (+)= dx.
cudaError_t conv_backward_data_fused(const ConvProblem& p, Dtype dt, const void* dy,
                                     const void* f, void* dx, bool accumulate, int math,
                                     const ConvEpilogue& ep, cudaStream_t st) {
  cudaError_t e;
  if (use_tc(p, dt, math, DGRAD, &e)) {
    if (same_strides(ep.gatev, p.x)) {
      e = tc_backward_data_fused(p, (const float*)dy, (const float*)f, (float*)dx, accumulate,
                                 ep, st, split_es(math));
      if (e != cudaErrorNotSupported) return e;
      cudaGetLastError();
    }
  } else if (e != cudaSuccess) {
    return e;
  }
  if (!accumulate) {
    if ((e = conv_backward_data(p, dt, dy, f, dx, false, math, st)) != cudaSuccess) return e;
    return activation_backward(ep.gate, dt, ep.gatev, ep.gatep, p.x, dx, p.x, dx, st);
  }
  const size_t es = dt == F64 ? 8 : 4;
  tc::ScratchScope* sc = tc::scratch_open(st);
  void* tmp = nullptr;
  e = tc::scratch_alloc(sc, size_t(p.x.size()) * es, &tmp);
  if (e == cudaSuccess) {
    ConvProblem q = p;  // dense NCHW scratch for the un-gated gradient
    q.x.sw = 1;
    q.x.sh = q.x.w;
    q.x.sc = q.x.h * q.x.w;
    q.x.sn = q.x.c * q.x.sc;
    e = conv_backward_data(q, dt, dy, f, tmp, false, math, st);
    if (e == cudaSuccess) e = activation_backward(ep.gate, dt, ep.gatev, ep.gatep, q.x, tmp, q.x, tmp, st);
    if (e == cudaSuccess) e = transform(dt, q.x, tmp, p.x, dx, 1.0, 1.0, st);
  }
  tc::scratch_close(sc);
  return e;
}

}  // namespace dnnp
