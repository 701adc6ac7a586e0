// tcgen05 implicit-GEMM convolution for fp32 via the BF16x3 split.
//
// Each fp32 operand value a is carried as a_hi = bf16(a), a_lo = bf16(a - a_hi)
// (16 of its 24 mantissa bits); the product uses three 5th-gen tensor-core
// MMAs per k-step into one FP32 TMEM accumulator:
//     D += A_lo.B_hi + A_hi.B_lo + A_hi.B_hi         (A_lo.B_lo ~ 2^-16 dropped)
// which keeps fp32-class accuracy (normalised error ~1e-6, north_star bar
// 1e-4) at 2/3 of the TF32 tensor rate.
//
// Data path (the lowered im2col matrix is never materialised, paper Sec. 3):
//   1. pack kernels: input -> channel-innermost bf16 hi/lo planes (any input
//      strides; channels padded to a multiple of 8 = one 16-byte chunk);
//      filter -> [Ncol][K_red] bf16 hi/lo in the kernel's reduction order;
//      a chunk table decoding every 16-byte reduction chunk into its
//      (dh, dw, channel) im2col offset.
//   2. conv_tc_kernel: 128 x BN output tile per CTA.  Warps 0-3 gather the
//      A tile (one output pixel per thread; 16-byte cp.async with zero-fill
//      outside the image) and copy the B tile into 128B-swizzled K-major
//      shared memory; warp 4 allocates TMEM and one lane issues the
//      tcgen05.mma stream; an mbarrier ring (full/empty) pipelines STAGES
//      k-blocks of 64; warps 0-3 then drain TMEM (tcgen05.ld) and apply the
//      alpha/beta epilogue straight into the caller's strided output.
//
// Forward:        M = N*P*Q pixels,  Ncol = K,  red = R*S*Cp   (Cp = C padded)
// Backward-data:  M = N*H*W pixels,  Ncol = C,  red = R*S*Kp   (unit stride:
//   dx = conv of dy padded by R-1-pad with the rotated, transposed filter).
#include <algorithm>
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace dnnp {

namespace {

constexpr int kBM = 128;        // tile rows (UMMA M)
constexpr int kBK = 64;         // bf16 elements per k-block = one 128 B swizzle row
constexpr int kProducers = 128; // warps 0-3
constexpr int kThreads = 160;   // + warp 4 (TMEM alloc + MMA issue)

struct TcParams {
  int64_t M;             // GEMM rows = output pixels
  int Ncol;              // valid output channels
  int OH, OW;            // output pixel grid of one image
  int IH, IW, Cp;        // packed input [N][IH][IW][Cp]
  int u, v, pad_h, pad_w;
  int KC;                // valid 16-byte reduction chunks
  int nkb;               // k-blocks
  int Ktot;              // nkb * 64 (row pitch of the packed filter)
  const uint32_t* ctab;  // chunk -> (dh << 24) | (dw << 16) | c0
  const __nv_bfloat16* a_hi;
  const __nv_bfloat16* a_lo;
  const __nv_bfloat16* b_hi;
  const __nv_bfloat16* b_lo;
  float* out;
  int64_t o_sn, o_sc, o_sh, o_sw;
  float alpha, beta;
  MagicDiv dOHW, dOW;
};

template <int BN>
struct TcCfg {
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int LAG = STAGES >= 4 ? 2 : 1;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ TcParams P) {
  using Cfg = TcCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = int64_t(blockIdx.x) * kBM;
  const int n0 = blockIdx.y * BN;

  if (warp == 4) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; s++) {
        ptx::mbar_init(&full[s], kProducers);
        ptx::mbar_init(&empty[s], 1);
      }
      ptx::mbar_init(tmem_full, 1);
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;
  const uint32_t smem0 = ptx::smem_u32(smem);

  if (warp < 4) {
    // ------------------------------------------------------------ producer
    const int t = threadIdx.x;
    const int64_t m = m0 + t;
    const bool row_ok = m < P.M;
    uint32_t img = 0, oh = 0, ow = 0;
    if (row_ok) {
      uint32_t rem;
      mdivmod(uint32_t(m), P.dOHW, img, rem);
      mdivmod(rem, P.dOW, oh, ow);
    }
    const int ih0 = int(oh) * P.u - P.pad_h, iw0 = int(ow) * P.v - P.pad_w;
    const int64_t pix0 = int64_t(img) * P.IH * P.IW;
    const uint32_t a_row = uint32_t((t >> 3) * 1024 + (t & 7) * 128);
    const int sw = t & 7;
    for (int kb = 0; kb < P.nkb; kb++) {
      const int s = kb % STAGES;
      if (kb >= STAGES) ptx::mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      const uint32_t sa_hi = smem0 + s * Cfg::STAGE_BYTES;
      const uint32_t sa_lo = sa_hi + Cfg::A_BYTES;
      const uint32_t sb_hi = sa_lo + Cfg::A_BYTES;
      const uint32_t sb_lo = sb_hi + Cfg::B_BYTES;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int ch = kb * 8 + j;
        bool ok = row_ok && ch < P.KC;
        int64_t src = 0;
        if (ok) {
          const uint32_t e = __ldg(P.ctab + ch);
          const int ih = ih0 + int(e >> 24), iw = iw0 + int((e >> 16) & 255);
          ok = unsigned(ih) < unsigned(P.IH) && unsigned(iw) < unsigned(P.IW);
          src = (pix0 + int64_t(ih) * P.IW + iw) * P.Cp + (e & 0xFFFF);
        }
        const uint32_t dst = a_row + uint32_t((j ^ sw) << 4);
        ptx::cp_async16(sa_hi + dst, P.a_hi + (ok ? src : 0), ok ? 16u : 0u);
        ptx::cp_async16(sa_lo + dst, P.a_lo + (ok ? src : 0), ok ? 16u : 0u);
      }
#pragma unroll
      for (int i = 0; i < BN / 16; i++) {
        const int q = t + i * kProducers;  // 16-byte chunk of the B tile
        const int row = q >> 3, j = q & 7;
        const int64_t src = int64_t(n0 + row) * P.Ktot + kb * kBK + j * 8;
        const uint32_t dst = uint32_t((row >> 3) * 1024 + (row & 7) * 128 + ((j ^ (row & 7)) << 4));
        ptx::cp_async16(sb_hi + dst, P.b_hi + src, 16u);
        ptx::cp_async16(sb_lo + dst, P.b_lo + src, 16u);
      }
      ptx::cp_async_commit();
      if (kb >= Cfg::LAG) {
        ptx::cp_async_wait<Cfg::LAG>();
        ptx::fence_proxy_async();
        ptx::mbar_arrive(&full[(kb - Cfg::LAG) % STAGES]);
      }
    }
    ptx::cp_async_wait<0>();
    ptx::fence_proxy_async();
    for (int kb = std::max(0, P.nkb - Cfg::LAG); kb < P.nkb; kb++)
      ptx::mbar_arrive(&full[kb % STAGES]);

    // ------------------------------------------------------------ epilogue
    ptx::mbar_wait(tmem_full, 0);
    ptx::tc_fence_after();
    const int64_t ooff = int64_t(img) * P.o_sn + int64_t(oh) * P.o_sh + int64_t(ow) * P.o_sw;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      ptx::tmem_ld32(tmem_d + (uint32_t(warp * 32) << 16) + uint32_t(c0), r);
      ptx::tmem_ld_wait();
      if (row_ok) {
#pragma unroll
        for (int i = 0; i < 32; i++) {
          const int col = n0 + c0 + i;
          if (col < P.Ncol) {
            float* dst = P.out + ooff + int64_t(col) * P.o_sc;
            float val = __fmul_rn(__uint_as_float(r[i]), P.alpha);
            if (P.beta != 0.0f) val = __fadd_rn(__fmul_rn(*dst, P.beta), val);
            *dst = val;
          }
        }
      }
    }
    ptx::tc_fence_before();
  } else if (lane == 0) {
    // --------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = ptx::idesc_bf16(kBM, BN, 0, 0);
    uint32_t acc = 0;
    for (int kb = 0; kb < P.nkb; kb++) {
      const int s = kb % STAGES;
      ptx::mbar_wait(&full[s], (kb / STAGES) & 1);
      ptx::tc_fence_after();
      const uint32_t sa_hi = smem0 + s * Cfg::STAGE_BYTES;
      const uint32_t sa_lo = sa_hi + Cfg::A_BYTES;
      const uint32_t sb_hi = sa_lo + Cfg::A_BYTES;
      const uint32_t sb_lo = sb_hi + Cfg::B_BYTES;
      const uint64_t dah = ptx::desc_kmajor_sw128(sa_hi), dal = ptx::desc_kmajor_sw128(sa_lo);
      const uint64_t dbh = ptx::desc_kmajor_sw128(sb_hi), dbl = ptx::desc_kmajor_sw128(sb_lo);
#pragma unroll
      for (int kk = 0; kk < kBK / 16; kk++) {
        const uint64_t o = uint64_t(kk * 2);  // 32 bytes along K, in 16-byte units
        ptx::mma_bf16(tmem_d, dal + o, dbh + o, idesc, acc);
        acc = 1;
        ptx::mma_bf16(tmem_d, dah + o, dbl + o, idesc, 1);
        ptx::mma_bf16(tmem_d, dah + o, dbh + o, idesc, 1);
      }
      ptx::mma_commit(&empty[s]);
    }
    ptx::mma_commit(tmem_full);
  }
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_d);
  }
}

// --------------------------------------------------------------- packing

__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// x[n, c, h, w] (any strides) -> hi/lo[n][h][w][Cp], zero channels >= C.
__global__ void __launch_bounds__(256) pack_act_kernel(View4 v, const float* __restrict__ x, int Cp,
                                                       __nv_bfloat16* __restrict__ hi,
                                                       __nv_bfloat16* __restrict__ lo,
                                                       int64_t npix, MagicDiv dHW, MagicDiv dW) {
  const int groups = Cp / 8;
  const int64_t total = npix * groups;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t pix = i % npix;
    const int g = int(i / npix);
    uint32_t n, rem, h, w;
    mdivmod(uint32_t(pix), dHW, n, rem);
    mdivmod(rem, dW, h, w);
    const float* src = x + int64_t(n) * v.sn + int64_t(h) * v.sh + int64_t(w) * v.sw;
    __align__(16) __nv_bfloat16 vh[8], vl[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int c = g * 8 + k;
      const float val = c < v.c ? src[int64_t(c) * v.sc] : 0.0f;
      split_bf16(val, vh[k], vl[k]);
    }
    const int64_t o = pix * Cp + g * 8;
    *reinterpret_cast<uint4*>(hi + o) = *reinterpret_cast<const uint4*>(vh);
    *reinterpret_cast<uint4*>(lo + o) = *reinterpret_cast<const uint4*>(vl);
  }
}

// Packed B operand [Np][Ktot] in the reduction order chunk = (dh*S + dw)*Cg + g,
// element = chunk*8 + i, with channel cin = g*8 + i of the packed input.
//   forward:  row = output channel k; value f[k][cin][r][s], r = flip ? R-1-dh : dh
//   bwd-data: row = dx channel c;     value f[cin][c][r][s], r = flip ? dh : R-1-dh
// Also writes the chunk table for the producer.
__global__ void __launch_bounds__(256) pack_filter_kernel(const float* __restrict__ f, int K, int C,
                                                          int R, int S, int flip, int dgrad,
                                                          int Np, int Ktot, int Cgrp, int KC,
                                                          __nv_bfloat16* __restrict__ hi,
                                                          __nv_bfloat16* __restrict__ lo,
                                                          uint32_t* __restrict__ ctab) {
  const int64_t total = int64_t(Np) * Ktot;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int row = int(idx / Ktot), k = int(idx % Ktot);
    const int ch = k >> 3, i = k & 7;
    float val = 0.0f;
    if (ch < KC) {
      const int tap = ch / Cgrp, g = ch % Cgrp;
      const int dh = tap / S, dw = tap % S;
      const int cin = g * 8 + i;
      if (row == 0 && i == 0) ctab[ch] = (uint32_t(dh) << 24) | (uint32_t(dw) << 16) | uint32_t(g * 8);
      if (!dgrad) {
        const int r = flip ? R - 1 - dh : dh, s = flip ? S - 1 - dw : dw;
        if (row < K && cin < C) val = f[((int64_t(row) * C + cin) * R + r) * S + s];
      } else {
        const int r = flip ? dh : R - 1 - dh, s = flip ? dw : S - 1 - dw;
        if (row < C && cin < K) val = f[((int64_t(cin) * C + row) * R + r) * S + s];
      }
    }
    __nv_bfloat16 h, l;
    split_bf16(val, h, l);
    hi[idx] = h;
    lo[idx] = l;
  }
}

// ------------------------------------------------------------- launching

struct Workspace {
  void* p = nullptr;
  cudaStream_t st;
  explicit Workspace(cudaStream_t s) : st(s) {}
  ~Workspace() {
    if (p) cudaFreeAsync(p, st);
  }
};

void pool_keep_memory() {
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

template <int BN>
cudaError_t launch_gemm(const TcParams& prm, int64_t mtiles, int ntiles, cudaStream_t st) {
  using Cfg = TcCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid{unsigned(mtiles), unsigned(ntiles), 1u};
  conv_tc_kernel<BN><<<grid, kThreads, Cfg::SMEM, st>>>(prm);
  note_launch();
  return cudaGetLastError();
}

// Pick the N tile: tile time ~ BN + fixed overhead; waves on 148 SMs.
int pick_bn(int64_t M, int ncol) {
  static const int cands[] = {32, 64, 128, 192, 256};
  const int64_t mt = ceil_div(M, kBM);
  int best = 256;
  double best_cost = 1e30;
  for (int bn : cands) {
    if (bn > 32 && bn / 2 >= ncol && bn != 192) continue;  // no point in >2x padding
    const int64_t tiles = mt * ceil_div(ncol, bn);
    const int64_t waves = ceil_div(tiles, kNumSMs);
    const double cost = double(waves) * (bn + 48) + double(ceil_div(ncol, bn)) * 4;
    if (cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

// Shared driver: pack input + filter, run the GEMM into the strided output.
cudaError_t run_tc(bool dgrad, const ConvProblem& p, const float* in, const View4& inv,
                   const float* f, float* out, const View4& outv, float alpha, float beta,
                   cudaStream_t st) {
  pool_keep_memory();
  // geometry of the implicit GEMM
  const int Cin = int(dgrad ? p.K : p.C);          // packed input channels
  const int Ncol = int(dgrad ? p.C : p.K);         // output channels
  const int IH = int(dgrad ? p.P : p.H), IW = int(dgrad ? p.Q : p.W);
  const int OH = int(dgrad ? p.H : p.P), OW = int(dgrad ? p.W : p.Q);
  const int Cp = int(ceil_div(Cin, 8) * 8), Cgrp = Cp / 8;
  const int KC = int(p.R * p.S) * Cgrp;
  const int nkb = int(ceil_div(KC, 8));
  const int Ktot = nkb * kBK;
  const int64_t N = p.N;
  const int64_t M = N * OH * OW;
  const int bn = pick_bn(M, Ncol);
  const int Np = int(ceil_div(Ncol, bn) * bn);

  const size_t act_elems = size_t(N) * IH * IW * Cp;
  const size_t flt_elems = size_t(Np) * Ktot;
  const size_t bytes = (2 * act_elems + 2 * flt_elems) * 2 + size_t(KC) * 4 + 256;
  Workspace ws(st);
  cudaError_t e = cudaMallocAsync(&ws.p, bytes, st);
  if (e != cudaSuccess) return e;
  auto* a_hi = static_cast<__nv_bfloat16*>(ws.p);
  auto* a_lo = a_hi + act_elems;
  auto* b_hi = a_lo + act_elems;
  auto* b_lo = b_hi + flt_elems;
  auto* ctab = reinterpret_cast<uint32_t*>(b_lo + flt_elems);

  const int64_t npix = N * IH * IW;
  pack_act_kernel<<<grid_for(npix * Cgrp, 256, 16), 256, 0, st>>>(
      inv, in, Cp, a_hi, a_lo, npix, make_magic(uint32_t(IH * IW)), make_magic(uint32_t(IW)));
  pack_filter_kernel<<<grid_for(int64_t(Np) * Ktot, 256, 16), 256, 0, st>>>(
      f, int(p.K), int(p.C), int(p.R), int(p.S), p.flip ? 1 : 0, dgrad ? 1 : 0, Np, Ktot, Cgrp,
      KC, b_hi, b_lo, ctab);
  note_launch(2);

  TcParams prm{};
  prm.M = M;
  prm.Ncol = Ncol;
  prm.OH = OH;
  prm.OW = OW;
  prm.IH = IH;
  prm.IW = IW;
  prm.Cp = Cp;
  if (!dgrad) {
    prm.u = int(p.u);
    prm.v = int(p.v);
    prm.pad_h = int(p.pad_h);
    prm.pad_w = int(p.pad_w);
  } else {  // unit stride: dy gathered with padding R-1-pad
    prm.u = 1;
    prm.v = 1;
    prm.pad_h = int(p.R - 1 - p.pad_h);
    prm.pad_w = int(p.S - 1 - p.pad_w);
  }
  prm.KC = KC;
  prm.nkb = nkb;
  prm.Ktot = Ktot;
  prm.ctab = ctab;
  prm.a_hi = a_hi;
  prm.a_lo = a_lo;
  prm.b_hi = b_hi;
  prm.b_lo = b_lo;
  prm.out = out;
  prm.o_sn = outv.sn;
  prm.o_sc = outv.sc;
  prm.o_sh = outv.sh;
  prm.o_sw = outv.sw;
  prm.alpha = alpha;
  prm.beta = beta;
  prm.dOHW = make_magic(uint32_t(OH * OW));
  prm.dOW = make_magic(uint32_t(OW));
  const int64_t mt = ceil_div(M, kBM);
  const int nt = Np / bn;
  switch (bn) {
    case 32: e = launch_gemm<32>(prm, mt, nt, st); break;
    case 64: e = launch_gemm<64>(prm, mt, nt, st); break;
    case 128: e = launch_gemm<128>(prm, mt, nt, st); break;
    case 192: e = launch_gemm<192>(prm, mt, nt, st); break;
    default: e = launch_gemm<256>(prm, mt, nt, st); break;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace

// FWD / DGRAD eligibility of the tensor-core path.
bool tc_eligible(const ConvProblem& p, int pass) {
  if (p.R > 255 || p.S > 255) return false;
  const int64_t lim = int64_t(1) << 31;
  if (pass == 0) {
    if (p.N * p.P * p.Q >= lim || ceil_div(p.C, 8) * 8 * p.R * p.S >= (1 << 24)) return false;
    return p.C <= 65535 && p.K <= 65535;
  }
  if (pass == 1) {
    if (p.u != 1 || p.v != 1) return false;
    if (p.N * p.H * p.W >= lim || ceil_div(p.K, 8) * 8 * p.R * p.S >= (1 << 24)) return false;
    return p.C <= 65535 && p.K <= 65535;
  }
  return false;
}

cudaError_t tc_forward(const ConvProblem& p, const float* x, const float* f, float* y,
                       double alpha, double beta, cudaStream_t st) {
  return run_tc(false, p, x, p.x, f, y, p.y, float(alpha), float(beta), st);
}

cudaError_t tc_backward_data(const ConvProblem& p, const float* dy, const float* f, float* dx,
                             bool acc, cudaStream_t st) {
  return run_tc(true, p, dy, p.y, f, dx, p.x, 1.0f, acc ? 1.0f : 0.0f, st);
}

cudaError_t tc_backward_filter(const ConvProblem&, const float*, const float*, float*, bool,
                               cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace dnnp
