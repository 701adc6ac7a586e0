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
// fp64 GEMMs with at least a wave of 128 x 128 tiles: 8 x 8 outputs per
// thread (one broadcast A load + one B load per 8 DFMAs per operand; the 4 x 4
// tile above is shared-memory- and issue-bound at ~35% of the DFMA pipe)
struct SimtCfgBig64 {
  static constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;
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

// Outputs of at most 4 columns (AlexNet conv1 bwd-data: C = 3): one row per
// thread and the whole width in registers, so 3/4 of the FMAs are useful
// instead of 3/16 (fp64 conv1 bwd-data N=16 2.75 -> see tools/bench_f64.py).
struct SimtTiny {
  static constexpr int BM = 64, BN = 4, BK = 16, TM = 1, TN = 4;
};

// Row (output-pixel) context of an A operand row.  FWD / DGRAD: A(m, k) =
// src[base + koff(k)] when 0 <= hb + dr(k) < lim_h and 0 <= wb + dw(k) <
// lim_w, so the per-element work is two adds, two compares and a load; the
// k decode (dr, dw, koff) is done once per k-step by one lane (KDec below).
//   FWD:   hb, wb = p*u - pad_h, q*v - pad_w; base = x(n, hb, wb); dr = r
//   DGRAD: hb, wb = i + (ph + pad_h) / u, j + (pw + pad_w) / v (the dy row
//          of tap 0 of the phase); base = dy(n, hb, wb); dr = -jr, so that
//          hb + dr = (h + pad_h - r) / u exactly for the phase's taps r
template <typename T, int PASS>
struct RowCtx {
  int64_t base;     // pass-specific row base offset
  int32_t hb, wb;
  bool valid;
};

template <typename T, int PASS>
__device__ __forceinline__ RowCtx<T, PASS> row_ctx(const SimtArgs& a, int64_t m) {
  RowCtx<T, PASS> rc;
  rc.valid = m < a.M;
  const ConvProblem& p = a.p;
  if (!rc.valid) {
    rc.base = 0; rc.hb = rc.wb = 0;
    return rc;
  }
  if (PASS == FWD) {
    uint32_t n, rem, pp, qq;
    mdivmod(uint32_t(m), a.dPQ, n, rem);
    mdivmod(rem, a.dQ, pp, qq);
    rc.hb = int32_t(pp * p.u - p.pad_h);
    rc.wb = int32_t(qq * p.v - p.pad_w);
    rc.base = int64_t(n) * p.x.sn + int64_t(rc.hb) * p.x.sh + int64_t(rc.wb) * p.x.sw;
  } else if (PASS == DGRAD) {
    uint32_t n, rem, i, j;
    mdivmod(uint32_t(m), a.dHWph, n, rem);
    mdivmod(rem, a.dWph, i, j);
    const int u = int(p.u), v = int(p.v);
    const int ph = int(blockIdx.z) / v, pw = int(blockIdx.z) - (int(blockIdx.z) / v) * v;
    rc.valid = int(i) * u + ph < p.H && int(j) * v + pw < p.W;
    rc.hb = int32_t(i) + (ph + int(p.pad_h)) / u;
    rc.wb = int32_t(j) + (pw + int(p.pad_w)) / v;
    rc.base = int64_t(n) * p.y.sn + int64_t(rc.hb) * p.y.sh + int64_t(rc.wb) * p.y.sw;
  } else {  // WGRAD: row = output channel k of dy
    rc.base = m * p.y.sc;
    rc.hb = rc.wb = 0;
  }
  return rc;
}

// Per-k decode of the FWD / DGRAD reduction index, computed by lane k - k0
// of each warp and broadcast with shuffles (every thread used to redo the two
// magic divisions per element: 3-4x the FMA count of a thin tile).  An
// out-of-range k (past kend, or a tap outside the phase) gets dr = kNoTap,
// which fails the row bound check, and boff = -1.
constexpr int32_t kNoTap = -(1 << 30);
struct KDec {
  int64_t aoff;  // A: channel / tap offset from the row base
  int64_t boff;  // DGRAD B: f[kk][0][r][s] offset (add col * R * S)
  int32_t dr, dw;
};

template <typename T, int PASS>
__device__ __forceinline__ KDec k_decode(const SimtArgs& a, int64_t k, int64_t kend, int t0h,
                                         int t0w) {
  KDec d;
  d.aoff = 0;
  d.boff = -1;
  d.dr = kNoTap;
  d.dw = 0;
  if (k >= kend) return d;
  const ConvProblem& p = a.p;
  if (PASS == FWD) {
    uint32_t c, rs, r, s;
    mdivmod(uint32_t(k), a.dRS, c, rs);
    mdivmod(rs, a.dS, r, s);
    d.dr = p.flip ? int32_t(p.R - 1 - r) : int32_t(r);
    d.dw = p.flip ? int32_t(p.S - 1 - s) : int32_t(s);
    d.aoff = int64_t(c) * p.x.sc + int64_t(d.dr) * p.x.sh + int64_t(d.dw) * p.x.sw;
  } else {
    uint32_t kk, rs, jr, js;
    mdivmod(uint32_t(k), a.dRSph, kk, rs);
    mdivmod(rs, a.dSph, jr, js);
    const int32_t ro = t0h + int32_t(p.u) * int32_t(jr);  // filter tap of this phase
    const int32_t so = t0w + int32_t(p.v) * int32_t(js);
    if (ro >= p.R || so >= p.S) return d;
    d.dr = -int32_t(jr);
    d.dw = -int32_t(js);
    d.aoff = int64_t(kk) * p.y.sc - int64_t(jr) * p.y.sh - int64_t(js) * p.y.sw;
    const int32_t r = p.flip ? int32_t(p.R - 1 - ro) : ro, s = p.flip ? int32_t(p.S - 1 - so) : so;
    d.boff = (int64_t(kk) * p.C * p.R + r) * p.S + s;  // f[kout][c][r][s]
  }
  return d;
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
  const T* asrc = static_cast<const T*>(a.a_src);
  const T* bsrc = static_cast<const T*>(a.b_src);
  const uint32_t lim_h = uint32_t(PASS == FWD ? a.p.H : a.p.P);
  const uint32_t lim_w = uint32_t(PASS == FWD ? a.p.W : a.p.Q);
  const int64_t fcol = int64_t(a.p.R) * a.p.S;
  // WGRAD B columns (c, r, s) of this thread: x offset and tap; hr = kNoTap
  // for columns past Ncol
  int64_t wq_off[PASS == WGRAD ? LB : 1];
  int32_t wq_hr[PASS == WGRAD ? LB : 1], wq_wr[PASS == WGRAD ? LB : 1];
  if constexpr (PASS == WGRAD) {
    static_assert(NT % BK == 0, "one reduction pixel per thread and k-step");
    const ConvProblem& p = a.p;
#pragma unroll
    for (int j = 0; j < LB; j++) {
      const int64_t col = n0 + b_ni[j];
      wq_off[j] = 0;
      wq_hr[j] = kNoTap;
      wq_wr[j] = 0;
      if (col < a.Ncol) {
        uint32_t c, rs, r, s;
        mdivmod(uint32_t(col), a.dRS, c, rs);
        mdivmod(rs, a.dS, r, s);
        wq_hr[j] = p.flip ? int32_t(p.R - 1 - r) : int32_t(r);
        wq_wr[j] = p.flip ? int32_t(p.S - 1 - s) : int32_t(s);
        wq_off[j] = int64_t(c) * p.x.sc + int64_t(wq_hr[j]) * p.x.sh + int64_t(wq_wr[j]) * p.x.sw;
      }
    }
  }
  auto gload = [&](int64_t k0) {
    if constexpr (PASS == WGRAD) {
      // every load of this thread is at reduction pixel k0 + tid % BK: one
      // decode per k-step; the column (c, r, s) decode is hoisted (wq_*)
      const int64_t k = k0 + tid % BK;
      int64_t aoff = 0, boff = 0;
      int32_t hk = kNoTap, wk = 0;
      if (k < kend) {
        const ConvProblem& p = a.p;
        uint32_t n, rem, pp, qq;
        mdivmod(uint32_t(k), a.dPQ, n, rem);
        mdivmod(rem, a.dQ, pp, qq);
        aoff = int64_t(n) * p.y.sn + int64_t(pp) * p.y.sh + int64_t(qq) * p.y.sw;
        hk = int32_t(pp * p.u - p.pad_h);
        wk = int32_t(qq * p.v - p.pad_w);
        boff = int64_t(n) * p.x.sn + int64_t(hk) * p.x.sh + int64_t(wk) * p.x.sw;
      }
#pragma unroll
      for (int j = 0; j < LA; j++) ra[j] = rc[j].valid && k < kend ? asrc[rc[j].base + aoff] : T(0);
#pragma unroll
      for (int j = 0; j < LB; j++) {
        const bool ok = uint32_t(hk + wq_hr[j]) < uint32_t(a.p.H) &&
                        uint32_t(wk + wq_wr[j]) < uint32_t(a.p.W);
        rb[j] = ok ? bsrc[boff + wq_off[j]] : T(0);
      }
    } else {
      static_assert(BK <= 32 && NT % 32 == 0, "one k per lane");
      const int lane = tid & 31;
      const KDec d = k_decode<T, PASS>(a, lane < BK ? k0 + lane : kend, kend, t0h, t0w);
#pragma unroll
      for (int j = 0; j < LA; j++) {
        const int64_t ao = __shfl_sync(0xffffffffu, d.aoff, a_ki[j]);
        const int32_t dr = __shfl_sync(0xffffffffu, d.dr, a_ki[j]);
        const int32_t dw = __shfl_sync(0xffffffffu, d.dw, a_ki[j]);
        const bool ok = rc[j].valid && uint32_t(rc[j].hb + dr) < lim_h &&
                        uint32_t(rc[j].wb + dw) < lim_w;
        ra[j] = ok ? asrc[rc[j].base + ao] : T(0);
      }
#pragma unroll
      for (int j = 0; j < LB; j++) {
        const int64_t col = n0 + b_ni[j];
        if (PASS == FWD) {
          const int64_t k = k0 + b_ki[j];
          rb[j] = k < kend && col < a.Ncol ? bsrc[col * a.Kred + k] : T(0);  // f[kout][crs]
        } else {
          const int64_t bo = __shfl_sync(0xffffffffu, d.boff, b_ki[j]);
          rb[j] = bo >= 0 && col < a.Ncol ? bsrc[bo + col * fcol] : T(0);
        }
      }
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

// ---- backward-data for thin outputs (C <= 4) -------------------------------
// AlexNet conv1 / Table-2 layer1 backward-data produce C = 3 channels from a
// long reduction (K x taps): as a GEMM every gathered dy element feeds only 3
// FMAs.  Direct convolution instead: a CTA owns a 32 x 32 tile of one stride
// phase's pixels, stages the dy halo of one dy channel at a time in shared
// memory (cp.async, double-buffered, zero-filled outside the image) plus that
// channel's phase taps, and every thread slides a register window along its
// row: (8 + nSp - 1) loads and nSp * C broadcast filter loads per 8 * nSp * C
// FMAs.  Lane = tile row, warp = 8-column group, odd row pitch: the window
// loads are bank-conflict free.
namespace thin {
constexpr int TH = 32, TM = 8, WARPS = 4, TW = WARPS * TM, NT = 32 * WARPS;

__device__ __forceinline__ void cp_async_el(void* dst, const void* src, int bytes, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                 "r"(ok ? 8 : 0));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
                 "r"(ok ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

struct Args {
  ConvProblem p;
  const void* dy;
  const void* f;
  void* dx;
  int accumulate;
  int nRp, tiles_w;
};

template <typename T, int CM, int NSP>
__global__ void __launch_bounds__(NT) dgrad_thin_kernel(const Args a) {
  extern __shared__ __align__(16) unsigned char thin_smem[];
  const ConvProblem& p = a.p;
  const int u = int(p.u), v = int(p.v), nRp = a.nRp;
  const int RH = TH + nRp - 1;
  constexpr int RWP = (TW + NSP - 1) | 1;  // odd pitch: lanes (rows) spread over the banks
  const int halo = RH * RWP;
  const int ftaps = nRp * NSP * CM;
  T* ys = reinterpret_cast<T*>(thin_smem);  // [2][RH][RWP]
  T* fs = ys + 2 * halo;                    // [2][nRp][NSP][CM]

  const int phase = blockIdx.z, ph = phase / v, pw = phase - (phase / v) * v;
  const int t0h = (ph + int(p.pad_h)) % u, t0w = (pw + int(p.pad_w)) % v;
  const int bh = (ph + int(p.pad_h)) / u, bw = (pw + int(p.pad_w)) / v;
  const int nRv = (int(p.R) - t0h + u - 1) / u;  // phase taps that exist
  const int nSv = (int(p.S) - t0w + v - 1) / v;
  const int n = blockIdx.y;
  const int ti = int(blockIdx.x) / a.tiles_w, tj = int(blockIdx.x) - ti * a.tiles_w;
  const int i0 = ti * TH, j0 = tj * TW;
  const int pr0 = i0 + bh - (nRp - 1), pc0 = j0 + bw - (NSP - 1);  // dy origin of the halo
  const T* dy = static_cast<const T*>(a.dy) + int64_t(n) * p.y.sn;
  const T* f = static_cast<const T*>(a.f);
  const int tid = threadIdx.x;

  auto stage = [&](int kk, int b) {
    const T* src = dy + int64_t(kk) * p.y.sc;
    T* dst = ys + b * halo;
    for (int e = tid; e < RH * RWP; e += NT) {
      const int lr = e / RWP, lc = e - lr * RWP;
      const int pp = pr0 + lr, qq = pc0 + lc;
      const bool ok = lc < TW + NSP - 1 && unsigned(pp) < unsigned(p.P) && unsigned(qq) < unsigned(p.Q);
      cp_async_el(dst + e, ok ? src + int64_t(pp) * p.y.sh + int64_t(qq) * p.y.sw : src,
                  int(sizeof(T)), ok);
    }
    T* fd = fs + b * ftaps;
    for (int e = tid; e < ftaps; e += NT) {
      const int c = e % CM, t = e / CM, js = t % NSP, jr = t / NSP;
      const int r = t0h + u * jr, s = t0w + v * js;
      const bool ok = c < p.C && jr < nRv && js < nSv;
      const int rr = p.flip ? int(p.R) - 1 - r : r, ss = p.flip ? int(p.S) - 1 - s : s;
      cp_async_el(fd + e, ok ? f + ((int64_t(kk) * p.C + c) * p.R + rr) * p.S + ss : f,
                  int(sizeof(T)), ok);
    }
    cp_async_commit();
  };

  const int li = tid & 31, lj0 = (tid >> 5) * TM;
  T acc[TM][CM];
#pragma unroll
  for (int m = 0; m < TM; m++)
#pragma unroll
    for (int c = 0; c < CM; c++) acc[m][c] = T(0);

  stage(0, 0);
  for (int kk = 0; kk < int(p.K); kk++) {
    const int b = kk & 1;
    cp_async_wait0();
    __syncthreads();  // buffer b landed for everyone; buffer b^1 is free
    if (kk + 1 < int(p.K)) stage(kk + 1, b ^ 1);
    const T* yb = ys + b * halo;
    const T* fb = fs + b * ftaps;
    for (int jr = 0; jr < nRv; jr++) {
      const T* row = yb + (li + nRp - 1 - jr) * RWP + lj0;
      T win[TM + NSP - 1];
#pragma unroll
      for (int w = 0; w < TM + NSP - 1; w++) win[w] = row[w];
      const T* fr = fb + jr * NSP * CM;
#pragma unroll
      for (int js = 0; js < NSP; js++) {
        if (js < nSv) {
          T fv[CM];
#pragma unroll
          for (int c = 0; c < CM; c++) fv[c] = fr[js * CM + c];
#pragma unroll
          for (int m = 0; m < TM; m++)
#pragma unroll
            for (int c = 0; c < CM; c++) acc[m][c] = fma(win[m + NSP - 1 - js], fv[c], acc[m][c]);
        }
      }
    }
  }

  const int i = i0 + li, h = i * u + ph;
  if (h >= p.H) return;
  T* dx = static_cast<T*>(a.dx) + int64_t(n) * p.x.sn + int64_t(h) * p.x.sh;
#pragma unroll
  for (int m = 0; m < TM; m++) {
    const int w = (j0 + lj0 + m) * v + pw;
    if (w >= p.W) break;
#pragma unroll
    for (int c = 0; c < CM; c++) {
      if (c < p.C) {
        T* dst = dx + int64_t(c) * p.x.sc + int64_t(w) * p.x.sw;
        *dst = a.accumulate ? dadd<T>(*dst, acc[m][c]) : acc[m][c];
      }
    }
  }
}

template <typename T, int CM, int NSP>
static cudaError_t launch_cm_nsp(const Args& a, dim3 grid, cudaStream_t st) {
  const int RH = TH + a.nRp - 1;
  constexpr int RWP = (TW + NSP - 1) | 1;
  const size_t smem = sizeof(T) * (2 * size_t(RH) * RWP + 2 * size_t(a.nRp) * NSP * CM);
  auto k = dgrad_thin_kernel<T, CM, NSP>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  k<<<grid, NT, smem, st>>>(a);
  note_launch();
  return cudaGetLastError();
}

template <typename T, int CM>
static cudaError_t launch_cm(const Args& a, int nsp, dim3 grid, cudaStream_t st) {
  if (nsp <= 3) return launch_cm_nsp<T, CM, 3>(a, grid, st);
  if (nsp <= 5) return launch_cm_nsp<T, CM, 5>(a, grid, st);
  if (nsp <= 7) return launch_cm_nsp<T, CM, 7>(a, grid, st);
  if (nsp <= 11) return launch_cm_nsp<T, CM, 11>(a, grid, st);
  return launch_cm_nsp<T, CM, 16>(a, grid, st);
}

// C <= 4, phase taps per row <= 16 and a halo that fits shared memory
bool applies(const ConvProblem& p) {
  if (p.C > 4 || p.K < 1 || ::dnnp::tune_env("DNNP_SIMT_NO_THIN")) return false;
  const int64_t nRp = ceil_div(p.R, p.u), nSp = ceil_div(p.S, p.v);
  if (nSp > 16 || nRp > 64) return false;
  const int64_t Hph = ceil_div(p.H, p.u), Wph = ceil_div(p.W, p.v);
  return p.N * Hph * Wph >= 4096 && p.N <= 65535 && p.u * p.v <= 65535;
}

template <typename T>
cudaError_t launch(const ConvProblem& p, const void* dy, const void* f, void* dx, bool acc,
                   cudaStream_t st) {
  Args a{};
  a.p = p;
  a.dy = dy;
  a.f = f;
  a.dx = dx;
  a.accumulate = acc;
  a.nRp = int(ceil_div(p.R, p.u));
  const int64_t Hph = ceil_div(p.H, p.u), Wph = ceil_div(p.W, p.v);
  a.tiles_w = int(ceil_div(Wph, TW));
  const dim3 grid(unsigned(ceil_div(Hph, TH) * a.tiles_w), unsigned(p.N), unsigned(p.u * p.v));
  const int nsp = int(ceil_div(p.S, p.v));
  switch (p.C) {
    case 1: return launch_cm<T, 1>(a, nsp, grid, st);
    case 2: return launch_cm<T, 2>(a, nsp, grid, st);
    case 3: return launch_cm<T, 3>(a, nsp, grid, st);
    default: return launch_cm<T, 4>(a, nsp, grid, st);
  }
}
}  // namespace thin

template <typename T, int PASS>
static cudaError_t launch_simt(SimtArgs& a, cudaStream_t st) {
  if (PASS != WGRAD && a.Ncol <= 4 && a.M >= 4096 && !::dnnp::tune_env("DNNP_SIMT_NO_TINY"))
    return launch_simt_cfg<T, PASS, SimtTiny>(a, st);
  if (PASS != WGRAD && a.Ncol <= 16 && a.M >= 4096 && !::dnnp::tune_env("DNNP_SIMT_NO_NARROW"))
    return launch_simt_cfg<T, PASS, SimtNarrow<T>>(a, st);
  if constexpr (std::is_same<T, double>::value) {
    // FWD / DGRAD: a full wave of tiles and <= 1/8 of the columns padding
    // (AlexNet N=128: conv3-5 fwd +12-17%, conv4/5 bwd-data +7-13%; 64 / 192
    // output columns lose 25-35%); WGRAD: split-K fills the machine, any
    // M >= 128 (conv2-5 bwd-filter +10-40%; tools/bench_f64.py)
    const int64_t ncp = ceil_div(a.Ncol, 128) * 128;
    const int64_t big_tiles = ceil_div(a.M, 128) * (ncp / 128) *
                              (PASS == DGRAD ? a.p.u * a.p.v : 1);
    const bool big = PASS == WGRAD ? a.M >= 128
                                   : big_tiles >= kNumSMs && (ncp - a.Ncol) * 8 <= ncp;
    if ((big || ::dnnp::tune_env("DNNP_SIMT_BIG")) && !::dnnp::tune_env("DNNP_SIMT_NO_BIG"))
      return launch_simt_cfg<T, PASS, SimtCfgBig64>(a, st);
    if constexpr (PASS == DGRAD) return launch_simt_cfg<T, PASS, SimtCfgDgrad64>(a, st);
  }
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
  if (thin::applies(p)) return thin::launch<T>(p, dy, f, dx, acc, st);
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
