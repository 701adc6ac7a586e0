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

__device__ __forceinline__ int64_t ceil_div_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

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
            const float accv = P.nkb > 0 ? __uint_as_float(r[i]) : 0.0f;
            float val = __fmul_rn(accv, P.alpha);
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

// ------------------------------------------------------ backward-filter
//
// dW[k][(dh, dw, c)] = sum over output pixels g of dy[g][k] * x[g shifted by
// (dh, dw)][c].  GEMM rows = output channels k (A = packed dy, MN-major: the
// 128 k of one pixel are contiguous), columns = the forward reduction order
// (B = im2col of packed x, MN-major: 8 channels of one tap per 16-byte
// chunk, gathered per pixel), reduction = pixels, split over gridDim.z.
// Partial tiles go to ws[z][row][col]; wgrad_reduce sums them in z order.
struct WgParams {
  int64_t NPQ;          // pixels
  int64_t pix_per_split;
  int P, Q, H, W;
  int u, v, pad_h, pad_w;
  int Kp, Cp;           // channel pitches of packed dy / packed x
  int KC;               // valid chunks (columns / 8)
  int ncol_p;           // padded column count (ws row pitch)
  int mrows_p;          // padded row count
  const uint32_t* ctab;
  const __nv_bfloat16* dy_hi;
  const __nv_bfloat16* dy_lo;
  const __nv_bfloat16* x_hi;
  const __nv_bfloat16* x_lo;
  float* ws;
  MagicDiv dPQ, dQ;
};

template <int BN>
struct WgCfg {
  static constexpr int A_BYTES = 128 * 128;   // 128 channels x 64 pixels, bf16
  static constexpr int B_BYTES = BN * 128;    // BN columns x 64 pixels
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int LAG = STAGES >= 4 ? 2 : 1;
  static constexpr int TMEM_COLS = BN <= 64 ? 64 : (BN <= 128 ? 128 : 256);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t LBO = 8 * 1024;   // 64-wide MN blocks
  static constexpr uint32_t SBO = 1024;       // 8-pixel K groups
};

// MN-major SW128 offset of (mn, kp) inside an operand tile of one k-block
__device__ __forceinline__ uint32_t mn_off(int mn_chunk, int kp) {
  const int blk = mn_chunk >> 3, jj = mn_chunk & 7;
  return uint32_t(blk * 8192 + (kp >> 3) * 1024 + (kp & 7) * 128 + ((jj ^ (kp & 7)) << 4));
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) wgrad_tc_kernel(const __grid_constant__ WgParams P) {
  using Cfg = WgCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.y * BN;
  const int64_t pbeg = int64_t(blockIdx.z) * P.pix_per_split;
  const int64_t pend = min(P.NPQ, pbeg + P.pix_per_split);
  const int nkb = int(ceil_div_dev(pend - pbeg, 64));

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
    const int t = threadIdx.x;
    const int kp = t & 63, half = t >> 6;
    for (int kb = 0; kb < nkb; kb++) {
      const int s = kb % STAGES;
      if (kb >= STAGES) ptx::mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      const uint32_t sa_hi = smem0 + s * Cfg::STAGE_BYTES;
      const uint32_t sa_lo = sa_hi + Cfg::A_BYTES;
      const uint32_t sb_hi = sa_lo + Cfg::A_BYTES;
      const uint32_t sb_lo = sb_hi + Cfg::B_BYTES;
      const int64_t g = pbeg + int64_t(kb) * 64 + kp;
      const bool pix_ok = g < pend;
      uint32_t n = 0, pp = 0, qq = 0;
      if (pix_ok) {
        uint32_t rem;
        mdivmod(uint32_t(g), P.dPQ, n, rem);
        mdivmod(rem, P.dQ, pp, qq);
      }
      // A: 8 of the 16 channel chunks of this pixel
#pragma unroll
      for (int jj = 0; jj < 8; jj++) {
        const int j = half * 8 + jj;
        const int c0 = m0 + j * 8;
        const bool ok = pix_ok && c0 < P.Kp;
        const int64_t src = ok ? g * P.Kp + c0 : 0;
        const uint32_t dst = mn_off(j, kp);
        ptx::cp_async16(sa_hi + dst, P.dy_hi + src, ok ? 16u : 0u);
        ptx::cp_async16(sa_lo + dst, P.dy_lo + src, ok ? 16u : 0u);
      }
      // B: half of the BN/8 column chunks, gathered through the chunk table
      const int ih0 = int(pp) * P.u - P.pad_h, iw0 = int(qq) * P.v - P.pad_w;
      const int64_t pix0 = int64_t(n) * P.H * P.W;
#pragma unroll
      for (int jj = 0; jj < BN / 16; jj++) {
        const int j = half * (BN / 16) + jj;
        const int ch = n0 / 8 + j;
        bool ok = pix_ok && ch < P.KC;
        int64_t src = 0;
        if (ok) {
          const uint32_t e = __ldg(P.ctab + ch);
          const int ih = ih0 + int(e >> 24), iw = iw0 + int((e >> 16) & 255);
          ok = unsigned(ih) < unsigned(P.H) && unsigned(iw) < unsigned(P.W);
          src = (pix0 + int64_t(ih) * P.W + iw) * P.Cp + (e & 0xFFFF);
        }
        const uint32_t dst = mn_off(j, kp);
        ptx::cp_async16(sb_hi + dst, P.x_hi + (ok ? src : 0), ok ? 16u : 0u);
        ptx::cp_async16(sb_lo + dst, P.x_lo + (ok ? src : 0), ok ? 16u : 0u);
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
    for (int kb = max(0, nkb - Cfg::LAG); kb < nkb; kb++) ptx::mbar_arrive(&full[kb % STAGES]);

    // epilogue: row = output channel m0 + t, partial sums to ws[z][row][col]
    ptx::mbar_wait(tmem_full, 0);
    ptx::tc_fence_after();
    float* dst = P.ws + (int64_t(blockIdx.z) * P.mrows_p + m0 + t) * P.ncol_p + n0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      ptx::tmem_ld32(tmem_d + (uint32_t(warp * 32) << 16) + uint32_t(c0), r);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 v4 = nkb > 0 ? make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                          __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(dst + c0 + i) = v4;
      }
    }
    ptx::tc_fence_before();
  } else if (lane == 0) {
    constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 1, 1);
    uint32_t acc = 0;
    for (int kb = 0; kb < nkb; kb++) {
      const int s = kb % STAGES;
      ptx::mbar_wait(&full[s], (kb / STAGES) & 1);
      ptx::tc_fence_after();
      const uint32_t sa_hi = smem0 + s * Cfg::STAGE_BYTES;
      const uint32_t sa_lo = sa_hi + Cfg::A_BYTES;
      const uint32_t sb_hi = sa_lo + Cfg::A_BYTES;
      const uint32_t sb_lo = sb_hi + Cfg::B_BYTES;
      const uint64_t dah = ptx::desc_mnmajor_sw128(sa_hi, Cfg::LBO, Cfg::SBO);
      const uint64_t dal = ptx::desc_mnmajor_sw128(sa_lo, Cfg::LBO, Cfg::SBO);
      const uint64_t dbh = ptx::desc_mnmajor_sw128(sb_hi, Cfg::LBO, Cfg::SBO);
      const uint64_t dbl = ptx::desc_mnmajor_sw128(sb_lo, Cfg::LBO, Cfg::SBO);
#pragma unroll
      for (int kk = 0; kk < 4; kk++) {
        const uint64_t o = uint64_t(kk * 2 * Cfg::SBO) >> 4;  // 16 pixels = 2 K groups
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

// dW[k][c][r][s] (+)= sum_z ws[z][k][col] with col = chunk*8 + i decoded by
// the forward chunk table; fixed z order => deterministic.
__global__ void __launch_bounds__(256) wgrad_reduce(const float* __restrict__ ws, int splits,
                                                    int mrows_p, int ncol_p, int K, int C, int R,
                                                    int S, int flip, int KC,
                                                    const uint32_t* __restrict__ ctab,
                                                    float* __restrict__ df, int accumulate) {
  const int64_t total = int64_t(K) * KC * 8;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t plane = int64_t(mrows_p) * ncol_p;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int k = int(idx / (int64_t(KC) * 8)), col = int(idx % (int64_t(KC) * 8));
    const uint32_t e = ctab[col >> 3];
    const int cin = int(e & 0xFFFF) + (col & 7);
    if (cin >= C) continue;
    const int dh = int(e >> 24), dw = int((e >> 16) & 255);
    const int r = flip ? R - 1 - dh : dh, s = flip ? S - 1 - dw : dw;
    const float* src = ws + int64_t(k) * ncol_p + col;
    float acc = src[0];
    for (int z = 1; z < splits; z++) acc = __fadd_rn(acc, src[z * plane]);
    float* d = df + ((int64_t(k) * C + cin) * R + r) * S + s;
    *d = accumulate ? __fadd_rn(*d, acc) : acc;
  }
}

// Chunk table of the forward reduction order (tap = dh*S + dw, then channel group).
__global__ void fwd_ctab_kernel(int S, int Cgrp, int KC, uint32_t* ctab) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= KC) return;
  const int tap = ch / Cgrp, g = ch % Cgrp;
  ctab[ch] = (uint32_t(tap / S) << 24) | (uint32_t(tap % S) << 16) | uint32_t(g * 8);
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

// Packed B operand [Np][Ktot] in the reduction order chunk = (dh*nS + dw)*Cg + g,
// element = chunk*8 + i, with channel cin = g*8 + i of the packed input.
//   forward:  row = output channel k; value f[k][cin][r][s], r = flip ? R-1-dh : dh
//   bwd-data: row = dx channel c;     value f[cin][c][r][s] where the
//             mode-adjusted tap is r' = t0h + u*(nR-1-dh) (one stride phase)
//             and r = flip ? R-1-r' : r'.
// Also writes the chunk table for the producer.
struct TapMap {
  int nR, nS;        // taps of this GEMM along h / w
  int t0h, t0w;      // first mode-adjusted tap of the phase (bwd-data)
  int su, sv;        // tap step (= conv stride, bwd-data)
};

__global__ void __launch_bounds__(256) pack_filter_kernel(const float* __restrict__ f, int K, int C,
                                                          int R, int S, int flip, int dgrad,
                                                          TapMap tm, int Np, int Ktot, int Cgrp,
                                                          int KC, __nv_bfloat16* __restrict__ hi,
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
      const int dh = tap / tm.nS, dw = tap % tm.nS;
      const int cin = g * 8 + i;
      if (row == 0 && i == 0) ctab[ch] = (uint32_t(dh) << 24) | (uint32_t(dw) << 16) | uint32_t(g * 8);
      if (!dgrad) {
        const int r = flip ? R - 1 - dh : dh, s = flip ? S - 1 - dw : dw;
        if (row < K && cin < C) val = f[((int64_t(row) * C + cin) * R + r) * S + s];
      } else {
        const int rp = tm.t0h + tm.su * (tm.nR - 1 - dh), sp = tm.t0w + tm.sv * (tm.nS - 1 - dw);
        const int r = flip ? R - 1 - rp : rp, s = flip ? S - 1 - sp : sp;
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

// One implicit GEMM over a packed input: output pixel grid (OH, OW) written
// through `out` with strides (o_sn, o_sc, o_sh, o_sw), gather
// ih = oh*u - pad_h + dh over dh < tm.nR (and likewise for w).
struct SubGemm {
  int OH, OW, u, v, pad_h, pad_w;
  TapMap tm;
  float* out;
  int64_t o_sn, o_sc, o_sh, o_sw;
};

cudaError_t run_sub(bool dgrad, const ConvProblem& p, const SubGemm& g, const __nv_bfloat16* a_hi,
                    const __nv_bfloat16* a_lo, int IH, int IW, int Cp, int Ncol, const float* f,
                    float alpha, float beta, cudaStream_t st) {
  const int Cgrp = Cp / 8;
  const int KC = g.tm.nR * g.tm.nS * Cgrp;
  const int nkb = int(ceil_div(KC, 8));
  const int Ktot = std::max(1, nkb) * kBK;
  const int64_t M = p.N * g.OH * g.OW;
  const int bn = pick_bn(M, Ncol);
  const int Np = int(ceil_div(Ncol, bn) * bn);
  const size_t flt_elems = size_t(Np) * Ktot;
  Workspace ws(st);
  cudaError_t e = cudaMallocAsync(&ws.p, flt_elems * 4 + size_t(std::max(KC, 1)) * 4 + 256, st);
  if (e != cudaSuccess) return e;
  auto* b_hi = static_cast<__nv_bfloat16*>(ws.p);
  auto* b_lo = b_hi + flt_elems;
  auto* ctab = reinterpret_cast<uint32_t*>(b_lo + flt_elems);
  pack_filter_kernel<<<grid_for(int64_t(Np) * Ktot, 256, 16), 256, 0, st>>>(
      f, int(p.K), int(p.C), int(p.R), int(p.S), p.flip ? 1 : 0, dgrad ? 1 : 0, g.tm, Np, Ktot,
      Cgrp, KC, b_hi, b_lo, ctab);
  note_launch();

  TcParams prm{};
  prm.M = M;
  prm.Ncol = Ncol;
  prm.OH = g.OH;
  prm.OW = g.OW;
  prm.IH = IH;
  prm.IW = IW;
  prm.Cp = Cp;
  prm.u = g.u;
  prm.v = g.v;
  prm.pad_h = g.pad_h;
  prm.pad_w = g.pad_w;
  prm.KC = KC;
  prm.nkb = nkb;
  prm.Ktot = Ktot;
  prm.ctab = ctab;
  prm.a_hi = a_hi;
  prm.a_lo = a_lo;
  prm.b_hi = b_hi;
  prm.b_lo = b_lo;
  prm.out = g.out;
  prm.o_sn = g.o_sn;
  prm.o_sc = g.o_sc;
  prm.o_sh = g.o_sh;
  prm.o_sw = g.o_sw;
  prm.alpha = alpha;
  prm.beta = beta;
  prm.dOHW = make_magic(uint32_t(g.OH * g.OW));
  prm.dOW = make_magic(uint32_t(g.OW));
  const int64_t mt = ceil_div(M, kBM);
  const int nt = Np / bn;
  switch (bn) {
    case 32: e = launch_gemm<32>(prm, mt, nt, st); break;
    case 64: e = launch_gemm<64>(prm, mt, nt, st); break;
    case 128: e = launch_gemm<128>(prm, mt, nt, st); break;
    case 192: e = launch_gemm<192>(prm, mt, nt, st); break;
    default: e = launch_gemm<256>(prm, mt, nt, st); break;
  }
  return e;
}

// Shared driver: pack the input once, then one GEMM (forward) or one GEMM
// per stride phase (backward-data) into the strided output.
cudaError_t run_tc(bool dgrad, const ConvProblem& p, const float* in, const View4& inv,
                   const float* f, float* out, const View4& outv, float alpha, float beta,
                   cudaStream_t st) {
  pool_keep_memory();
  const int Cin = int(dgrad ? p.K : p.C);   // packed input channels
  const int Ncol = int(dgrad ? p.C : p.K);  // output channels
  const int IH = int(dgrad ? p.P : p.H), IW = int(dgrad ? p.Q : p.W);
  const int Cp = int(ceil_div(Cin, 8) * 8), Cgrp = Cp / 8;
  const int64_t N = p.N;
  const size_t act_elems = size_t(N) * IH * IW * Cp;
  Workspace ws(st);
  cudaError_t e = cudaMallocAsync(&ws.p, act_elems * 4 + 256, st);
  if (e != cudaSuccess) return e;
  auto* a_hi = static_cast<__nv_bfloat16*>(ws.p);
  auto* a_lo = a_hi + act_elems;
  const int64_t npix = N * IH * IW;
  pack_act_kernel<<<grid_for(npix * Cgrp, 256, 16), 256, 0, st>>>(
      inv, in, Cp, a_hi, a_lo, npix, make_magic(uint32_t(IH * IW)), make_magic(uint32_t(IW)));
  note_launch();

  if (!dgrad) {
    SubGemm g{int(p.P), int(p.Q), int(p.u), int(p.v), int(p.pad_h), int(p.pad_w),
              TapMap{int(p.R), int(p.S), 0, 0, 1, 1}, out, outv.sn, outv.sc, outv.sh, outv.sw};
    return run_sub(false, p, g, a_hi, a_lo, IH, IW, Cp, Ncol, f, alpha, beta, st);
  }
  // backward-data: dx rows h = ph + u*i take taps r' = t0 + u*j, t0 = (ph + pad) mod u,
  // reading dy row p = i + (ph + pad - t0)/u - j  (gather form, no atomics)
  for (int ph = 0; ph < int(p.u) && ph < int(p.H); ph++) {
    for (int pw = 0; pw < int(p.v) && pw < int(p.W); pw++) {
      SubGemm g{};
      const int t0h = int((ph + p.pad_h) % p.u), t0w = int((pw + p.pad_w) % p.v);
      g.tm.nR = t0h < p.R ? int(ceil_div(p.R - t0h, p.u)) : 0;
      g.tm.nS = t0w < p.S ? int(ceil_div(p.S - t0w, p.v)) : 0;
      g.tm.t0h = t0h;
      g.tm.t0w = t0w;
      g.tm.su = int(p.u);
      g.tm.sv = int(p.v);
      g.OH = int(ceil_div(p.H - ph, p.u));
      g.OW = int(ceil_div(p.W - pw, p.v));
      g.u = g.v = 1;
      g.pad_h = g.tm.nR - 1 - int((ph + p.pad_h - t0h) / p.u);
      g.pad_w = g.tm.nS - 1 - int((pw + p.pad_w - t0w) / p.v);
      g.out = out + ph * outv.sh + pw * outv.sw;
      g.o_sn = outv.sn;
      g.o_sc = outv.sc;
      g.o_sh = outv.sh * p.u;
      g.o_sw = outv.sw * p.v;
      e = run_sub(true, p, g, a_hi, a_lo, IH, IW, Cp, Ncol, f, alpha, beta, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
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
    if (p.u > 64 || p.v > 64) return false;
    if (p.N * p.H * p.W >= lim || ceil_div(p.K, 8) * 8 * p.R * p.S >= (1 << 24)) return false;
    return p.C <= 65535 && p.K <= 65535;
  }
  if (pass == 2) {
    if (p.N * p.P * p.Q >= lim || p.N * p.H * p.W >= lim) return false;
    return p.C <= 65535 && p.K <= 65535 && ceil_div(p.C, 8) * 8 * p.R * p.S < (1 << 24);
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

template <int BN>
cudaError_t launch_wgrad(const WgParams& prm, int mt, int nt, int splits, cudaStream_t st) {
  using Cfg = WgCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(wgrad_tc_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid{unsigned(mt), unsigned(nt), unsigned(splits)};
  wgrad_tc_kernel<BN><<<grid, kThreads, Cfg::SMEM, st>>>(prm);
  note_launch();
  return cudaGetLastError();
}

cudaError_t tc_backward_filter(const ConvProblem& p, const float* dy, const float* x, float* df,
                               bool acc, cudaStream_t st) {
  pool_keep_memory();
  const int Kp = int(ceil_div(p.K, 8) * 8), Cp = int(ceil_div(p.C, 8) * 8), Cgrp = Cp / 8;
  const int KC = int(p.R * p.S) * Cgrp;
  const int64_t NPQ = p.N * p.P * p.Q, NHW = p.N * p.H * p.W;
  const int ncol = KC * 8;
  const int bn = ncol <= 64 ? 64 : (ncol <= 128 ? 128 : 256);
  const int nt = int(ceil_div(ncol, bn)), mt = int(ceil_div(p.K, 128));
  const int ncol_p = nt * bn, mrows_p = mt * 128;
  const int64_t kblocks = ceil_div(NPQ, 64);
  int64_t splits = ceil_div(int64_t(kNumSMs) * 2, int64_t(mt) * nt);
  splits = std::max<int64_t>(1, std::min<int64_t>({splits, kblocks / 4 > 0 ? kblocks / 4 : 1, 64}));
  const int64_t pps = ceil_div(kblocks, splits) * 64;
  splits = ceil_div(NPQ, pps);

  const size_t dy_elems = size_t(NPQ) * Kp, x_elems = size_t(NHW) * Cp;
  const size_t ws_floats = size_t(splits) * mrows_p * ncol_p;
  Workspace ws(st);
  cudaError_t e = cudaMallocAsync(&ws.p, (dy_elems + x_elems) * 4 + ws_floats * 4 + size_t(KC) * 4 + 512, st);
  if (e != cudaSuccess) return e;
  auto* dy_hi = static_cast<__nv_bfloat16*>(ws.p);
  auto* dy_lo = dy_hi + dy_elems;
  auto* x_hi = dy_lo + dy_elems;
  auto* x_lo = x_hi + x_elems;
  float* part = reinterpret_cast<float*>(x_lo + x_elems);
  auto* ctab = reinterpret_cast<uint32_t*>(part + ws_floats);

  pack_act_kernel<<<grid_for(NPQ * (Kp / 8), 256, 16), 256, 0, st>>>(
      p.y, dy, Kp, dy_hi, dy_lo, NPQ, make_magic(uint32_t(p.P * p.Q)), make_magic(uint32_t(p.Q)));
  pack_act_kernel<<<grid_for(NHW * Cgrp, 256, 16), 256, 0, st>>>(
      p.x, x, Cp, x_hi, x_lo, NHW, make_magic(uint32_t(p.H * p.W)), make_magic(uint32_t(p.W)));
  fwd_ctab_kernel<<<unsigned(ceil_div(KC, 256)), 256, 0, st>>>(int(p.S), Cgrp, KC, ctab);
  note_launch(3);

  WgParams prm{};
  prm.NPQ = NPQ;
  prm.pix_per_split = pps;
  prm.P = int(p.P); prm.Q = int(p.Q); prm.H = int(p.H); prm.W = int(p.W);
  prm.u = int(p.u); prm.v = int(p.v); prm.pad_h = int(p.pad_h); prm.pad_w = int(p.pad_w);
  prm.Kp = Kp;
  prm.Cp = Cp;
  prm.KC = KC;
  prm.ncol_p = ncol_p;
  prm.mrows_p = mrows_p;
  prm.ctab = ctab;
  prm.dy_hi = dy_hi; prm.dy_lo = dy_lo; prm.x_hi = x_hi; prm.x_lo = x_lo;
  prm.ws = part;
  prm.dPQ = make_magic(uint32_t(p.P * p.Q));
  prm.dQ = make_magic(uint32_t(p.Q));
  switch (bn) {
    case 64: e = launch_wgrad<64>(prm, mt, nt, int(splits), st); break;
    case 128: e = launch_wgrad<128>(prm, mt, nt, int(splits), st); break;
    default: e = launch_wgrad<256>(prm, mt, nt, int(splits), st); break;
  }
  if (e != cudaSuccess) return e;
  wgrad_reduce<<<grid_for(int64_t(p.K) * ncol, 256, 16), 256, 0, st>>>(
      part, int(splits), mrows_p, ncol_p, int(p.K), int(p.C), int(p.R), int(p.S), p.flip ? 1 : 0,
      KC, ctab, df, acc ? 1 : 0);
  note_launch();
  return cudaGetLastError();
}

}  // namespace dnnp
