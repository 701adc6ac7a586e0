// tcgen05 backward-filter convolution, fp32 via the BF16x3 split.
//
// dW[k][(dh, dw, c)] = sum over output pixels g of dy[g][k] * x[g + (dh,dw)][c]
// (reference conv.py:710-717: gemm(dy_map [K x NPQ], lowered^T [NPQ x CRS])).
// GEMM rows = output channels k, columns = the forward reduction order
// (tap, channel), reduction = pixels, split over gridDim.z (split-K).
//   A = packed dy [pixel][Kp]: MN-major (the k of one pixel are contiguous)
//   B = im2col of packed x: MN-major, 8 channels of one tap per 16-byte
//       chunk gathered per pixel through the chunk table (zero-fill outside)
// Stages hold 32 pixels in 128B-swizzled MN-major tiles.  Every split writes
// its partial tile to a workspace; wgrad_reduce sums the splits in fixed order
// and scatters into the KCRS filter (deterministic; accumulate adds last).
#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"
#include "tc_ptx.cuh"

namespace dnnp {
namespace tc {
namespace {

constexpr int kProdWarps = 8;  // gather/TMA producers; warps 0-3 also run the epilogue
constexpr int kThreads = (kProdWarps + 1) * 32;  // + MMA warp
constexpr int kPx = 32;        // pixels (reduction rows) per stage

struct WgParams {
  CUtensorMap tm_dyhi;   // packed dy [NPQ][Kp], box {64 channels, 32 pixels}, 128B swizzle
  CUtensorMap tm_dylo;
  int64_t NPQ;
  int64_t pix_per_split;
  int P, Q, H, W;
  int u, v, pad_h, pad_w;
  int Kp, Cp;
  int KC;
  int ncol_p, mrows_p;
  const uint32_t* ctab;
  const __nv_bfloat16* dy_hi;
  const __nv_bfloat16* dy_lo;
  const __nv_bfloat16* x_hi;
  const __nv_bfloat16* x_lo;
  float* ws;
  MagicDiv dPQ, dQ;
};

template <int BN>
struct WCfg {
  static constexpr uint32_t LBO = (kPx / 8) * 1024;  // stride of 64-wide MN blocks
  static constexpr uint32_t SBO = 1024;              // stride of 8-pixel K groups
  static constexpr int A_BYTES = 2 * LBO;            // 128 channels
  static constexpr int B_BYTES = (BN / 64) * LBO;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES =
      (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = BN <= 64 ? 64 : (BN <= 128 ? 128 : 256);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN>
__device__ __forceinline__ uint32_t mn_off(int mn_chunk, int kp) {
  const int blk = mn_chunk >> 3, jj = mn_chunk & 7;
  return uint32_t(blk * WCfg<BN>::LBO + (kp >> 3) * 1024 + (kp & 7) * 128 + ((jj ^ (kp & 7)) << 4));
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) wgrad_tc_kernel(const __grid_constant__ WgParams P) {
  using C = WCfg<BN>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.y * BN;
  const int64_t pbeg = int64_t(blockIdx.z) * P.pix_per_split;
  const int64_t pend = min(P.NPQ, pbeg + P.pix_per_split);
  const int nkb = pend > pbeg ? int((pend - pbeg + kPx - 1) / kPx) : 0;

  if (warp == kProdWarps) {
    if (lane == 0) {
      for (int s = 0; s < S; s++) {
        ptx::mbar_init(&full[s], kProdWarps * 32 + 1);  // gather arrivals + expect_tx (TMA dy)
        ptx::mbar_init(&empty[s], 1);
      }
      ptx::mbar_init(tmem_full, 1);
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;
  const uint32_t smem0 = ptx::smem_u32(smem);
  pdl_wait();  // programmatic launch behind the packs: read nothing they write before this

  if (warp < kProdWarps) {
    // A (dy, dense per pixel) arrives by TMA; B (im2col of x) is gathered with
    // one lane per 16-byte column chunk so that a warp reads one pixel's
    // contiguous channel runs.  Pixel decodes are done once per warp (one lane
    // per pixel) and broadcast; each lane keeps its chunk's constant offset.
    const int t = threadIdx.x;
    constexpr int NCH = BN / 8;                  // column chunks per pixel
    constexpr int LP = NCH < 32 ? NCH : 32;      // lanes per pixel
    constexpr int PPI = 32 / LP;                 // pixels per warp instruction
    constexpr int PPW = kPx / kProdWarps;        // pixels per warp per stage
    constexpr int ITER = PPW / PPI;
    constexpr int NQ = (NCH + 31) / 32;
    const int jl = lane % LP, sub = lane / LP;
    const int nbox = min(2, (P.Kp - m0 + 63) / 64);
    const uint32_t a_bytes = uint32_t(nbox) * C::LBO;  // per plane
    if (t == 0) {
      ptx::tma_prefetch(&P.tm_dyhi);
      ptx::tma_prefetch(&P.tm_dylo);
    }
    int cdh[NQ], cdw[NQ];
    int64_t coff[NQ];
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      const int ch = n0 / 8 + jl + q * 32;
      const uint32_t e = ch < P.KC ? __ldg(P.ctab + ch) : 0u;
      cdh[q] = ch < P.KC ? int(e >> 24) : (1 << 20);  // out of range => masked
      cdw[q] = int((e >> 16) & 255);
      coff[q] = (int64_t(cdh[q] & 0xFF) * P.W + cdw[q]) * P.Cp + (e & 0xFFFF);
    }
    for (int kb = 0; kb < nkb; kb++) {
      const int s = kb % S;
      if (kb >= S) ptx::mbar_wait(&empty[s], ((kb / S) - 1) & 1);
      const uint32_t sa_hi = smem0 + s * C::STAGE_BYTES;
      const uint32_t sa_lo = sa_hi + C::A_BYTES;
      const uint32_t sb_hi = sa_lo + C::A_BYTES;
      const uint32_t sb_lo = sb_hi + C::B_BYTES;
      const int64_t gk = pbeg + int64_t(kb) * kPx;
      if (t == 0) {
        ptx::mbar_arrive_expect_tx(&full[s], 2 * a_bytes);
        for (int b = 0; b < nbox; b++) {
          ptx::tma_load_2d(sa_hi + b * C::LBO, &P.tm_dyhi, m0 + 64 * b, int(gk), &full[s]);
          ptx::tma_load_2d(sa_lo + b * C::LBO, &P.tm_dylo, m0 + 64 * b, int(gk), &full[s]);
        }
      }
      // lane l < PPW decodes pixel warp*PPW + l of this stage
      int my_ih0 = -(1 << 20), my_iw0 = 0;
      int64_t my_base = 0;
      if (lane < PPW) {
        const int64_t g = gk + warp * PPW + lane;
        if (g < pend) {
          uint32_t n, rem, pp, qq;
          mdivmod(uint32_t(g), P.dPQ, n, rem);
          mdivmod(rem, P.dQ, pp, qq);
          my_ih0 = int(pp) * P.u - P.pad_h;
          my_iw0 = int(qq) * P.v - P.pad_w;
          my_base = ((int64_t(n) * P.H + my_ih0) * P.W + my_iw0) * P.Cp;
        }
      }
#pragma unroll
      for (int ii = 0; ii < ITER; ii++) {
        const int pl = ii * PPI + sub;  // pixel within this warp's set
        const int ih0 = __shfl_sync(0xffffffffu, my_ih0, pl);
        const int iw0 = __shfl_sync(0xffffffffu, my_iw0, pl);
        const int64_t base = __shfl_sync(0xffffffffu, my_base, pl);
        const int kp = warp * PPW + pl;
#pragma unroll
        for (int q = 0; q < NQ; q++) {
          const int ih = ih0 + cdh[q], iw = iw0 + cdw[q];
          const bool ok = unsigned(ih) < unsigned(P.H) && unsigned(iw) < unsigned(P.W);
          const int64_t src = ok ? base + coff[q] : 0;
          const uint32_t dst = mn_off<BN>(jl + q * 32, kp);
          ptx::cp_async16(sb_hi + dst, P.x_hi + src, ok ? 16u : 0u);
          ptx::cp_async16(sb_lo + dst, P.x_lo + src, ok ? 16u : 0u);
        }
      }
      ptx::cp_async_mbar_arrive(&full[s]);
    }
    ptx::cp_async_wait<0>();

    // epilogue (warps 0-3 = TMEM lane quadrants): row = output channel m0 + t
    if (warp < 4) {
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
        const float4 v4 =
            nkb > 0 ? make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                  __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(dst + c0 + i) = v4;
      }
    }
    ptx::tc_fence_before();
    }
  } else {
    // whole MMA warp runs the loop; one elected lane issues (uniform registers)
    constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 1, 1);
    uint32_t acc = 0;
    for (int kb = 0; kb < nkb; kb += 2) {
      const int npair = nkb - kb >= 2 ? 2 : 1;
      ptx::mbar_wait(&full[kb % S], (kb / S) & 1);
      if (npair == 2) ptx::mbar_wait(&full[(kb + 1) % S], ((kb + 1) / S) & 1);
      ptx::fence_proxy_async();  // producers' cp.async writes -> async proxy
      ptx::tc_fence_after();
      for (int q = 0; q < npair; q++) {
        const int s = (kb + q) % S;
        const uint32_t sa_hi = smem0 + s * C::STAGE_BYTES;
        const uint64_t dah = ptx::desc_mnmajor_sw128(sa_hi, C::LBO, C::SBO);
        const uint64_t dal = ptx::desc_mnmajor_sw128(sa_hi + C::A_BYTES, C::LBO, C::SBO);
        const uint64_t dbh = ptx::desc_mnmajor_sw128(sa_hi + 2 * C::A_BYTES, C::LBO, C::SBO);
        const uint64_t dbl =
            ptx::desc_mnmajor_sw128(sa_hi + 2 * C::A_BYTES + C::B_BYTES, C::LBO, C::SBO);
#pragma unroll
        for (int kk = 0; kk < kPx / 16; kk++) {
          const uint64_t o = uint64_t(kk * 2 * C::SBO) >> 4;  // 16 pixels = 2 K groups
          ptx::mma_bf16_elect(tmem_d, dal + o, dbh + o, idesc, acc);
          acc = 1;
          ptx::mma_bf16_elect(tmem_d, dah + o, dbl + o, idesc, 1);
          ptx::mma_bf16_elect(tmem_d, dah + o, dbh + o, idesc, 1);
        }
        ptx::mma_commit_elect(&empty[s]);
      }
    }
    ptx::mma_commit_elect(tmem_full);
  }
  __syncthreads();
  if (warp == kProdWarps) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::TMEM_COLS>(tmem_d);
  }
}

// dW[k][c][r][s] (+)= sum_z ws[z][k][col], col = chunk*8 + i decoded by the
// forward chunk table; fixed z order => deterministic.
__global__ void __launch_bounds__(256) wgrad_reduce(const float* __restrict__ ws, int splits,
                                                    int mrows_p, int ncol_p, int K, int Cc, int R,
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
    if (cin >= Cc) continue;
    const int dh = int(e >> 24), dw = int((e >> 16) & 255);
    const int r = flip ? R - 1 - dh : dh, s = flip ? S - 1 - dw : dw;
    const float* src = ws + int64_t(k) * ncol_p + col;
    float acc = src[0];
    for (int z = 1; z < splits; z++) acc = __fadd_rn(acc, src[z * plane]);
    float* d = df + ((int64_t(k) * Cc + cin) * R + r) * S + s;
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

template <int BN>
cudaError_t launch_wgrad(const WgParams& prm, int mt, int nt, int splits, cudaStream_t st) {
  using CC = WCfg<BN>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(wgrad_tc_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const dim3 grid{unsigned(mt), unsigned(nt), unsigned(splits)};
  ktime_begin(st, 4);
  wgrad_tc_kernel<BN><<<grid, kThreads, CC::SMEM, st>>>(prm);
  ktime_end(st);
  note_launch();
  return cudaGetLastError();
}

}  // namespace
// ===========================================================================
// TMA im2col backward-filter.
//
// GEMM: D[col][k] = sum over output pixels g of x_im2col[g][col] * dy[g][k],
// rows = the forward reduction columns col = tap * Cpf + c (x operand, A),
// columns = output channels k (dy operand, B), reduction = pixels.  Both
// operands are MN-major 128B-swizzled tiles of 64-wide blocks x PX (32 or 64) pixels:
//   x  block = one im2col TMA load (PX pixels x 64 channels of one tap,
//              zero fill at the border / past the last image),
//   dy blocks = ONE 3-D tiled TMA load per plane over the view
//              {64 channels, pixels, channel block} (block-major in smem).
// TMA costs ~190-270 cycles per instruction whatever the box size
// (profiles/r01/tma_rate_probe_v2_depth.txt), so stages are 64 pixels deep
// and dy needs one instruction per plane.  NC = 2 runs the tile on a CTA
// pair (M = 256 rows, each CTA loads half of the BN dy channels).
// Split-K over pixels (multiples of PX: only the last stage of the last
// split runs past NPQ, where both loads zero-fill); each split writes an fp32
// partial tile, wgrad_reduce_tma sums splits in fixed order and scatters into
// KCRS (deterministic).
// ===========================================================================
namespace {

constexpr int kWgThreads = 8 * 32;  // warps 0-2 TMA, 3 MMA + TMEM, 4-7 epilogue

struct WgTmaParams {
  CUtensorMap tm_xhi;   // im2col maps of the packed x planes, 64 channels x PX pixels
  CUtensorMap tm_xlo;
  CUtensorMap tm_dyhi;  // packed dy as {64, NPQ, Kp/64}, box {64, PX, BN/NC/64}
  CUtensorMap tm_dylo;
  int64_t pix_per_split, NPQ;
  int lower_h, lower_w, u, v;  // window origin of output pixel (p, q): lower + o * stride
  int nCB, tapW, taps, Cext;   // x column blocks per tap, taps per window row, taps, OOB channel
  int mrows_p, ncol_p;         // workspace tile pitch
  float* ws;
  MagicDiv dPQ, dQ;
  unsigned long long* trace;
};

// Longest reduction (pixels) accumulated in one TMEM accumulator.  The
// tensor-core fp32 accumulation truncates, so its error grows linearly with
// the chain (measured: 2.8e-5 of max|dW| at 8k pixels, 4.7e-5 at 16k,
// 3.7e-4 at 222k); longer reductions are split and the splits summed in IEEE
// fp32 by the reduce kernel, which keeps every wgrad at the north_star 1e-4
// bar whatever N*P*Q is.  16k costs nothing on AlexNet (8k cost conv1/conv2
// ~10%, tools/wg_chain.py).
static int64_t max_chain(int px) {
  int64_t c = 16384;
  if (const char* e = ::dnnp::tune_env("DNNP_WG_CHAIN")) c = std::max<int64_t>(atoll(e), px);
  return c / px * px;
}

// ES: bytes per packed element (2 = BF16x3, 4 = 3xTF32).  An x block is one
// 128-byte-row MN block: XW = 128 / ES channels (64 bf16, 32 tf32) x PX
// pixels; BW: width (channels) of one dy MN block: 64 bf16 (128-byte
// swizzle) or 32 (bf16: 64-byte swizzle, lets a CTA pair split BN = 64 or
// 192 into halves; tf32: the 128-byte rows of the 128B_ATOM_32B swizzle,
// the only MN-major tf32 layout, tools/probe_tf32.cu).
template <int BN, int NC, int PX, int BW = 64, int ES = 2>
struct WgCfg {
  static constexpr int XW = 128 / ES;          // channels of one x MN block
  static constexpr int XB = 128 / XW;          // x blocks per 128 columns
  static constexpr int KSTEP = 32 / ES;        // pixels per MMA k-step
  static constexpr int BLK = PX * 128;         // one x MN block
  static constexpr int BBLK = PX * BW * ES;    // one BW-wide MN block of dy
  static constexpr int B_BLKS = BN / NC / BW;  // dy blocks loaded by each CTA
  static_assert(B_BLKS * BW * NC == BN, "dy blocks must tile the CTA's columns");
  static_assert(ES == 2 || BW * ES == 128, "tf32 dy blocks are 128-byte rows");
  static constexpr int A_BYTES = XB * BLK;     // 128 x-columns
  static constexpr int B_BYTES = B_BLKS * BBLK;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES =
      (225 * 1024 - 2048) / STAGE_BYTES > 8 ? 8 : (225 * 1024 - 2048) / STAGE_BYTES;
  // two accumulators, even / odd k-blocks: each fp32 TMEM chain is half the
  // split's pixels (tcgen05 accumulation truncates: error grows with chain
  // length); the epilogue adds them in IEEE fp32
  static constexpr int TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, int NC, int PX, int BW, int ES>
__global__ void __launch_bounds__(kWgThreads, 1) wgrad_tma_kernel(const __grid_constant__ WgTmaParams P) {
  using C = WgCfg<BN, NC, PX, BW, ES>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = NC == 2 ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int m0 = (blockIdx.x / NC) * (128 * NC) + int(rank) * 128;  // this CTA's x columns
  const int n0 = blockIdx.y * BN;
  const int64_t pbeg = int64_t(blockIdx.z) * P.pix_per_split;
  const int64_t pend = min(P.NPQ, pbeg + P.pix_per_split);
  const int nkb = pend > pbeg ? int((pend - pbeg + PX - 1) / PX) : 0;
  constexpr int kMmaW = 3;  // warps 0-2 TMA producers, 3 MMA, 4-7 epilogue

  if (warp == kMmaW) {
    if (lane == 0) {
      for (int s = 0; s < S; s++) {
        ptx::mbar_init(&full[s], NC);
        ptx::mbar_init(&empty[s], 1);
      }
      ptx::mbar_init(tmem_full, 1);
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc_g<C::TMEM_COLS, NC>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (NC == 2) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;
  const uint32_t smem0 = ptx::smem_u32(smem);
  pdl_wait();  // programmatic launch behind the packs: read nothing they write before this

  if (warp < 3) {
    // three producers (one TMA instruction costs its thread ~110-130 cycles):
    // warp 0 x hi (and arms the stage), warp 1 x lo, warp 2 dy hi + lo
    const int pw = warp;
    if (lane == 0) {
      if (pw == 0) ptx::tma_prefetch(&P.tm_xhi);
      if (pw == 1) ptx::tma_prefetch(&P.tm_xlo);
      if (pw == 2) {
        ptx::tma_prefetch(&P.tm_dyhi);
        ptx::tma_prefetch(&P.tm_dylo);
      }
      const CUtensorMap* tmx = pw == 0 ? &P.tm_xhi : &P.tm_xlo;
      const int dyblk0 = (n0 + int(rank) * (BN / NC)) / BW;  // this CTA's first dy channel block
      for (int kb = 0; kb < nkb; kb++) {
        const int s = kb % S;
        const bool tr = P.trace && pw == 0 && blockIdx.x == 0 && blockIdx.y == 0 &&
                        blockIdx.z == 0 && kb < 1024;
        if (tr) P.trace[kb * 4 + 0] = clock64();
        if (kb >= S) ptx::mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        if (tr) P.trace[kb * 4 + 1] = clock64();
        if (pw == 0) {
          if (leader) ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES * NC);
          else ptx::mbar_arrive_cluster(&full[s], 0);
        }
        const uint32_t bar = NC == 2 ? ptx::leader_addr(&full[s]) : ptx::smem_u32(&full[s]);
        const int64_t g = pbeg + int64_t(kb) * PX;
        const uint32_t base = smem0 + s * C::STAGE_BYTES;
        if (pw < 2) {
          uint32_t img, rem, pp, qq;
          mdivmod(uint32_t(g), P.dPQ, img, rem);
          mdivmod(rem, P.dQ, pp, qq);
          const int h0 = P.lower_h + int(pp) * P.u, w0 = P.lower_w + int(qq) * P.v;
          const uint32_t xb = base + (pw == 1 ? C::A_BYTES : 0);
#pragma unroll
          for (int j = 0; j < C::XB; j++) {
            const int blk = m0 / C::XW + j;
            const int tap = blk / P.nCB, cb = blk - tap * P.nCB;
            const bool real = tap < P.taps;
            const int c = real ? cb * C::XW : P.Cext;
            const uint16_t dh = uint16_t(real ? tap / P.tapW : 0), dw = uint16_t(real ? tap % P.tapW : 0);
            if constexpr (NC == 2)
              ptx::tma_load_im2col_pair(xb + j * C::BLK, tmx, c, w0, h0, int(img), dw, dh, bar);
            else
              ptx::tma_load_im2col(xb + j * C::BLK, tmx, c, w0, h0, int(img), dw, dh, &full[s]);
          }
        } else {
          const uint32_t db = base + 2 * C::A_BYTES;
          if constexpr (NC == 2) {
            ptx::tma_load_3d_pair(db, &P.tm_dyhi, 0, int(g), dyblk0, bar);
            ptx::tma_load_3d_pair(db + C::B_BYTES, &P.tm_dylo, 0, int(g), dyblk0, bar);
          } else {
            ptx::tma_load_3d(db, &P.tm_dyhi, 0, int(g), dyblk0, &full[s]);
            ptx::tma_load_3d(db + C::B_BYTES, &P.tm_dylo, 0, int(g), dyblk0, &full[s]);
          }
        }
      }
    }
  } else if (warp == kMmaW) {
    if (leader) {
      constexpr uint32_t idesc = ES == 4 ? ptx::idesc_tf32(128 * NC, BN, 1, 1)
                                         : ptx::idesc_bf16(128 * NC, BN, 1, 1);
      uint32_t accv[2] = {0, 0};
      for (int kb = 0; kb < nkb; kb++) {
        const int s = kb % S;
        const uint32_t dacc = tmem_d + uint32_t((kb & 1) * BN);
        uint32_t acc = accv[kb & 1];
        ptx::mbar_wait_spin(&full[s], (kb / S) & 1);
        ptx::tc_fence_after();
        if (P.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && kb < 1024 && lane == 0)
          P.trace[kb * 4 + 2] = clock64();
        const uint32_t sa = smem0 + s * C::STAGE_BYTES;
        const uint32_t sb = sa + 2 * C::A_BYTES;
        uint64_t dah, dal, dbh, dbl;
        if constexpr (ES == 4) {
          dah = ptx::desc_mnmajor_b32(sa, C::BLK);
          dal = ptx::desc_mnmajor_b32(sa + C::A_BYTES, C::BLK);
          dbh = ptx::desc_mnmajor_b32(sb, C::BBLK);
          dbl = ptx::desc_mnmajor_b32(sb + C::B_BYTES, C::BBLK);
        } else {
          dah = ptx::desc_mnmajor_sw128(sa, C::BLK, 1024);
          dal = ptx::desc_mnmajor_sw128(sa + C::A_BYTES, C::BLK, 1024);
          dbh = BW == 64 ? ptx::desc_mnmajor_sw128(sb, C::BBLK, 1024)
                         : ptx::desc_mnmajor_sw64(sb, C::BBLK, 512);
          dbl = BW == 64 ? ptx::desc_mnmajor_sw128(sb + C::B_BYTES, C::BBLK, 1024)
                         : ptx::desc_mnmajor_sw64(sb + C::B_BYTES, C::BBLK, 512);
        }
#pragma unroll
        for (int kk = 0; kk < PX / C::KSTEP; kk++) {
          // one k-step = KSTEP pixels: KSTEP rows of 128 B (x), of BW * ES B (dy)
          const uint64_t o = uint64_t(kk * C::KSTEP * 128) >> 4;
          const uint64_t ob = uint64_t(kk * C::KSTEP * BW * ES) >> 4;
          ptx::mma_split_elect<NC, ES>(dacc, dal + o, dbh + ob, idesc, acc);
          ptx::mma_split_elect<NC, ES>(dacc, dah + o, dbl + ob, idesc, 1);
          ptx::mma_split_elect<NC, ES>(dacc, dah + o, dbh + ob, idesc, 1);
          acc = 1;
        }
        accv[kb & 1] = 1;
        if constexpr (NC == 2) ptx::mma_commit_pair_elect(&empty[s]);
        else ptx::mma_commit_elect(&empty[s]);
      }
      if constexpr (NC == 2) ptx::mma_commit_pair_elect(tmem_full);
      else ptx::mma_commit_elect(tmem_full);
    }
  } else {
    const int ew = warp & 3;
    const int r = ew * 32 + lane;
    ptx::mbar_wait(tmem_full, 0);
    ptx::tc_fence_after();
    float* dst = P.ws + (int64_t(blockIdx.z) * P.mrows_p + m0 + r) * P.ncol_p + n0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
      ptx::tmem_ld32(tmem_d + (uint32_t(ew * 32) << 16) + uint32_t(c0), v);
      if (nkb > 1) {  // the odd k-blocks' accumulator
        uint32_t w[32];
        ptx::tmem_ld32(tmem_d + (uint32_t(ew * 32) << 16) + uint32_t(BN + c0), w);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i++)
          v[i] = __float_as_uint(__fadd_rn(__uint_as_float(v[i]), __uint_as_float(w[i])));
      }
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 v4 =
            nkb > 0 ? make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                  __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(dst + c0 + i) = v4;
      }
    }
  }
  ptx::tc_fence_before();
  if constexpr (NC == 2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == kMmaW) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_g<C::TMEM_COLS, NC>(tmem_d);
  }
}

// df[k][c][r][s] (+)= sum_z ws[z][col][k].  One thread per workspace
// element (col, k), k fastest, so the split reads are coalesced; the x column
// col = tap * Cpf + cg decodes to the filter element it holds: tap = (dh', dw'),
// cg = ((rh * sv) + rw) * C + c, gather offset r' = dh' * su + rh (zero-padding
// columns and offsets >= R hold no filter element), r = R-1-r' in CONVOLUTION mode.
struct WgReduceGeom {
  int K, C, R, S, flip;
  int su, sv, S2, Cpf;  // space-to-depth factors, taps per window row, columns per tap
  int ncolx;            // taps * Cpf
  int splits, mrows_p, ncol_p;
};

__global__ void __launch_bounds__(256) wgrad_reduce_tma(WgReduceGeom g, const float* __restrict__ ws,
                                                        float* __restrict__ df, int accumulate) {
  const int total = g.ncolx * g.K;
  const int stride = gridDim.x * blockDim.x;
  const int64_t plane = int64_t(g.mrows_p) * g.ncol_p;
  const int Cg = g.su * g.sv * g.C;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int k = idx % g.K, col = idx / g.K;
    const int tap = col / g.Cpf, cg = col - tap * g.Cpf;
    if (cg >= Cg) continue;
    const int ph = cg / g.C, c = cg - ph * g.C;
    const int ro = (tap / g.S2) * g.su + ph / g.sv, so = (tap % g.S2) * g.sv + ph % g.sv;
    if (ro >= g.R || so >= g.S) continue;
    const int r = g.flip ? g.R - 1 - ro : ro, s = g.flip ? g.S - 1 - so : so;
    const float* src = ws + int64_t(col) * g.ncol_p + k;
    // loads issued 8 ahead, sums kept in split order (deterministic)
    float acc = __ldcg(src);
    int z = 1;
    for (; z + 8 <= g.splits; z += 8) {
      float t[8];
#pragma unroll
      for (int q = 0; q < 8; q++) t[q] = __ldcg(src + (z + q) * plane);
#pragma unroll
      for (int q = 0; q < 8; q++) acc = __fadd_rn(acc, t[q]);
    }
    for (; z < g.splits; z++) acc = __fadd_rn(acc, __ldcg(src + z * plane));
    float* d = df + ((int64_t(k) * g.C + c) * g.R + r) * g.S + s;
    *d = accumulate ? __fadd_rn(*d, acc) : acc;
  }
}

#include "wgrad_halo.cuh"

template <int BN, int NC, int PX, int BW = 64, int ES = 2>
cudaError_t launch_wgrad_tma(const WgTmaParams& prm, dim3 grid, cudaStream_t st) {
  using CC = WgCfg<BN, NC, PX, BW, ES>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(wgrad_tma_kernel<BN, NC, PX, BW, ES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kWgThreads);
  cfg.dynamicSmemBytes = CC::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  unsigned nattr = 1;
  add_pdl_attr(attr, &nattr);
  cfg.attrs = attr;
  cfg.numAttrs = nattr;
  ktime_begin(st, 2);
  cudaError_t e = cudaLaunchKernelEx(&cfg, wgrad_tma_kernel<BN, NC, PX, BW, ES>, prm);
  ktime_end(st);
  note_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

// Halo form of the space-to-depth backward-filter (wgrad_halo.cuh):
// cudaErrorNotSupported when it does not apply.
cudaError_t wgrad_halo(const ConvProblem& p, const float* dy, const float* x, float* df, bool acc,
                       cudaStream_t st, int es) {
  if (es != 2 || ::dnnp::tune_env("DNNP_TC_NO_HALO")) return cudaErrorNotSupported;
  if (!(p.u > 1 || p.v > 1) || p.u > 8 || p.v > 8 || p.C * p.u * p.v > 64 || p.K > 64)
    return cudaErrorNotSupported;
  const int su = int(p.u), sv = int(p.v);
  const int R2 = int(ceil_div(p.R, su)), S2 = int(ceil_div(p.S, sv));
  const int IH = int(p.P) - 1 + R2, IW = int(p.Q) - 1 + S2;
  // leader taps: rows 0, 2, ..; the peer computes each one row down
  std::vector<int> lt;
  for (int th = 0; th < R2; th += 2)
    for (int tw = 0; tw < S2; tw++) lt.push_back(th * S2 + tw);
  const int ng = int(ceil_div(int64_t(lt.size()), 2));
  if (ng > kWhMaxG) return cudaErrorNotSupported;
  WgHaloParams prm{};
  int shmax = 0;
  for (int g = 0; g < ng; g++) {
    for (int b = 0; b < 2; b++) {
      const size_t i = std::min(lt.size() - 1, size_t(2 * g + b));
      const int t = lt[i], th = t / S2, tw = t % S2;
      prm.sh[g][b] = th * IW + tw;
      shmax = std::max(shmax, prm.sh[g][b]);
      const bool dup = size_t(2 * g + b) >= lt.size();
      prm.tap[0][g][b] = dup ? -1 : t;
      prm.tap[1][g][b] = (dup || th + 1 >= R2) ? -1 : (th + 1) * S2 + tw;
    }
  }
  const int RH = kWhChunk + shmax;
  if (RH > 256) return cudaErrorNotSupported;
  const int64_t npix = p.N * int64_t(IH) * IW;
  const int64_t chunks = ceil_div(npix, int64_t(kWhChunk));
  const int64_t Pp = chunks * kWhChunk;
  const int ncl = int(std::min<int64_t>(chunks, kNumSMs / 2));
  // accumulation chain per cluster <= max_chain pixels (fp32 TMEM truncation)
  if (ceil_div(chunks, int64_t(ncl)) * kWhChunk > max_chain(kWhChunk) || Pp >= (int64_t(1) << 31))
    return cudaErrorNotSupported;
  const int Cpf = 64, taps = R2 * S2, ncolx = taps * Cpf;
  const size_t x_elems = size_t(npix) * 64, dy_elems = size_t(64) * Pp;
  const size_t ws_floats = size_t(ncl) * ncolx * 64;
  Workspace wsp(st);
  cudaError_t e = wsp.alloc((x_elems + dy_elems) * 4 + ws_floats * 4 + 1024);
  if (e != cudaSuccess) return e;
  char* base = static_cast<char*>(wsp.p);
  void* x_hi = base;
  void* x_lo = base + x_elems * 2;
  auto* d_hi = reinterpret_cast<__nv_bfloat16*>(base + x_elems * 4);
  auto* d_lo = d_hi + dy_elems;
  float* part = reinterpret_cast<float*>(base + ((x_elems * 4 + dy_elems * 4 + 255) & ~size_t(255)));
  if ((e = pack_act_s2d(p.x, x, su, sv, int(p.pad_h), int(p.pad_w), IH, IW, 64, x_hi, x_lo, st, es)) !=
      cudaSuccess)
    return e;
  {
    const dim3 grid(unsigned(ceil_div(Pp, int64_t(512))), unsigned(ceil_div(p.K, int64_t(8))));
    pack_dy_grid_kernel<<<grid, 256, 0, st>>>(p.y, dy, IH, IW, int(p.K), npix, Pp, d_hi, d_lo);
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if ((e = make_tmap_2d(&prm.tm_xhi, x_hi, 64, uint64_t(npix), 64, 64, uint32_t(RH),
                        CU_TENSOR_MAP_SWIZZLE_128B, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_xlo, x_lo, 64, uint64_t(npix), 64, 64, uint32_t(RH),
                        CU_TENSOR_MAP_SWIZZLE_128B, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_dhi, d_hi, uint64_t(Pp), uint64_t(p.K), uint64_t(Pp), 64, 64,
                        CU_TENSOR_MAP_SWIZZLE_128B, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_dlo, d_lo, uint64_t(Pp), uint64_t(p.K), uint64_t(Pp), 64, 64,
                        CU_TENSOR_MAP_SWIZZLE_128B, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_dq, d_hi, uint64_t(Pp), uint64_t(p.K), uint64_t(Pp), 64, 32,
                        CU_TENSOR_MAP_SWIZZLE_128B, 2)) != cudaSuccess)
    return e;
  prm.chunks = int(chunks);
  prm.RH = RH;
  prm.off1 = IW;
  prm.ng = ng;
  prm.Cpf = Cpf;
  prm.ncolx = ncolx;
  prm.arr_bytes = uint32_t(ceil_div(int64_t(RH) * 128, 1024) * 1024);
  prm.ws = part;
  const size_t smem = size_t(2) * (2 * prm.arr_bytes + 2 * 64 * 128 + 2 * 32 * 128) + 2048;
  {
    static int attr_dev = -1;
    static size_t attr_smem = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev || smem > attr_smem) {
      e = cudaFuncSetAttribute(wgrad_halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      attr_dev = dev;
      attr_smem = smem;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(ncl * 2));
  cfg.blockDim = dim3(kWhThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  unsigned nattr = 1;
  add_pdl_attr(attr, &nattr);
  cfg.attrs = attr;
  cfg.numAttrs = nattr;
  ktime_begin(st, 2);
  e = cudaLaunchKernelEx(&cfg, wgrad_halo_kernel, prm);
  ktime_end(st);
  note_launch();
  if (e != cudaSuccess) return e;
  WgReduceGeom rg{};
  rg.K = int(p.K);
  rg.C = int(p.C);
  rg.R = int(p.R);
  rg.S = int(p.S);
  rg.flip = p.flip ? 1 : 0;
  rg.su = su;
  rg.sv = sv;
  rg.S2 = S2;
  rg.Cpf = Cpf;
  rg.ncolx = ncolx;
  rg.splits = ncl;
  rg.mrows_p = ncolx;
  rg.ncol_p = 64;
  wgrad_reduce_tma<<<grid_for(int64_t(ncolx) * p.K, 256, 16), 256, 0, st>>>(rg, part, df, acc ? 1 : 0);
  note_launch();
  return cudaGetLastError();
}

// TMA path of backward-filter; returns cudaErrorNotSupported when the
// geometry does not fit the im2col tensor map (caller falls back).
cudaError_t wgrad_tma(const ConvProblem& p, const float* dy, const float* x, float* df, bool acc,
                      cudaStream_t st, int es) {
  if (::dnnp::tune_env("DNNP_TC_NO_TMA")) return cudaErrorNotSupported;
  {
    const cudaError_t he = wgrad_halo(p, dy, x, df, acc, st, es);
    if (he != cudaErrorNotSupported) return he;
  }
  const bool s2d = !::dnnp::tune_env("DNNP_TC_NO_S2D") && (p.u > 1 || p.v > 1) && p.u <= 8 && p.v <= 8 &&
                   p.C * p.u * p.v <= 64;
  // horizontal tap folding (stride-1-style few-channel layers): the S taps
  // as channels, the reduce maps folded channel j*C + c back to s = j
  const bool fold = fold_taps(p.C, p.S, p.u, p.v, s2d) && p.Q * p.v + p.S <= (int64_t(1) << 20);
  const int su = s2d ? int(p.u) : 1, sv = s2d ? int(p.v) : (fold ? int(p.S) : 1);
  const int R2 = int(ceil_div(p.R, su)), S2 = fold ? 1 : int(ceil_div(p.S, sv));
  const int Cg = su * sv * int(p.C);                 // GEMM channels per tap
  const int Cp = int(ceil_div(Cg, 16) * 16);         // packed x channels
  const int xw = 128 / es;                           // channels of one x block (128-byte rows)
  const int nCB = int(ceil_div(Cp, xw)), Cpf = nCB * xw;
  const int taps = R2 * S2;
  const int ncolx = taps * Cpf;                      // x-operand extent (padded)
  const int IH = s2d ? int(p.P) - 1 + R2 : int(p.H);
  const int IW = s2d ? int(p.Q) - 1 + S2 : (fold ? int(p.Q) : int(p.W));
  const int gu = s2d ? 1 : int(p.u), gv = (s2d || fold) ? 1 : int(p.v);
  const int gph = s2d ? 0 : int(p.pad_h), gpw = (s2d || fold) ? 0 : int(p.pad_w);
  if (gu > 8 || gv > 8 || R2 > 128 || S2 > 128) return cudaErrorNotSupported;
  const int lower_h = -gph, lower_w = -gpw;
  const int upper_h = (int(p.P) - 1) * gu + 1 - gph - IH;
  const int upper_w = (int(p.Q) - 1) * gv + 1 - gpw - IW;
  for (int c : {lower_h, lower_w, upper_h, upper_w})
    if (c < -128 || c > 127) return cudaErrorNotSupported;
  const int64_t NPQ = p.N * p.P * p.Q;
  if (NPQ >= (int64_t(1) << 31) || p.N * IH * IW >= (int64_t(1) << 31)) return cudaErrorNotSupported;

  // tile: 128*nc x-columns by bn output channels; pairs when both halves of
  // the dy columns are whole 64-channel blocks
  const int Kp64 = int(ceil_div(p.K, 64) * 64);
  int bn = Kp64 <= 256 ? Kp64 : (Kp64 % 256 == 0 ? 256 : (Kp64 % 192 == 0 ? 192 : 128));
  if (const char* e = ::dnnp::tune_env("DNNP_TC_BN")) {
    const int v = atoi(e);  // only the instantiated column tiles
    if (v == 64 || v == 128 || v == 192 || v == 256) bn = v;
  }
  // CTA pairs split the dy columns in halves: 64-channel blocks (128-byte
  // swizzle) when bn / 2 is a multiple of 64, else 32-channel blocks (64-byte
  // swizzle) for bn = 192 (conv2 122.9 vs 137.2 us, conv3 67.6 vs 73.9 us);
  // bn = 64 keeps single CTAs (conv1: the 256-row pair tiles pad 576 x-columns
  // to 768, 178 vs 147 us; DNNP_WG_BW32_64 forces the pair)
  int nc = (bn % 128 == 0 || (bn == 192 && !::dnnp::tune_env("DNNP_WG_NO_BW32")) ||
            (bn == 64 && ::dnnp::tune_env("DNNP_WG_BW32_64")))
               ? 2
               : 1;
  if (const char* e = ::dnnp::tune_env("DNNP_TC_NC")) {
    const int v = atoi(e);
    if (v == 1 || v == 2) nc = v;
  }
  if (nc == 2 && bn % 64) nc = 1;
  if (nc == 2 && bn % 128 && bn != 64 && bn != 192) nc = 1;
  const bool bw32 = es == 4 || (nc == 2 && bn % 128 != 0);
  const int dbw = bw32 ? 32 : 64;  // dy block width of the tensor map (tf32: 128-byte rows)
  const int mrows = int(ceil_div(ncolx, 128 * nc) * 128 * nc);
  const int ncols = int(ceil_div(Kp64, bn) * bn);
  const int mt = mrows / (128 * nc), nt = ncols / bn;
  // pixels per stage: 64 (measured faster than 32 even where only two
  // 64-deep stages fit, e.g. conv2 BN=192: 202 vs 266 us)
  // 128 pixels per stage when each CTA holds <= 64 dy channels (conv1:
  // 146 -> 126 us): the TMA engine spends ~200-280 cycles per box whatever
  // its size up to 16 KB, so bigger boxes move more bytes per box; the
  // 96 KB stages still double-buffer.  Wider dy tiles would leave one stage.
  // (3xTF32: the same stage bytes, so half the pixels)
  int px = (bn / nc <= 64 ? 128 : 64) * 2 / es;
  if (const char* e = ::dnnp::tune_env("DNNP_WG_PX"); e && es == 2) {
    const int v = atoi(e);
    px = v == 32 ? 32 : (v == 128 ? 128 : 64);
  }
  const int64_t kblocks = ceil_div(NPQ, px);
  int64_t splits = std::max<int64_t>(1, int64_t(kNumSMs) / (int64_t(mt) * nt * nc));
  splits = std::min<int64_t>({splits, std::max<int64_t>(1, kblocks / 4), 256});
  const int64_t pps = std::min(ceil_div(kblocks, splits) * px, max_chain(px));
  splits = ceil_div(NPQ, pps);

  const size_t dy_elems = size_t(NPQ) * Kp64, x_elems = size_t(p.N) * IH * IW * Cp;
  const size_t ws_floats = size_t(splits) * mrows * ncols;
  Workspace wsp(st);
  cudaError_t e = wsp.alloc((dy_elems + x_elems) * 2 * es + ws_floats * 4 + 512);
  if (e != cudaSuccess) return e;
  char* base = static_cast<char*>(wsp.p);
  void* dy_hi = base;
  void* dy_lo = base + dy_elems * es;
  void* x_hi = base + 2 * dy_elems * es;
  void* x_lo = base + (2 * dy_elems + x_elems) * es;
  float* part = reinterpret_cast<float*>(base + 2 * (dy_elems + x_elems) * es);
  {
    const void *ph = nullptr, *pl = nullptr;
    if (packed_get(dy, p.y, Kp64, &ph, &pl, es)) {  // packed once by the fused backward entry
      dy_hi = const_cast<void*>(ph);
      dy_lo = const_cast<void*>(pl);
    } else if ((e = pack_act(p.y, dy, Kp64, dy_hi, dy_lo, st, es)) != cudaSuccess) {
      return e;
    }
  }
  if (fold)
    e = pack_act_fold(p.x, x, int(p.S), int(p.v), int(p.pad_w), IW, Cp, x_hi, x_lo, st, es);
  else if (s2d)
    e = pack_act_s2d(p.x, x, su, sv, int(p.pad_h), int(p.pad_w), IH, IW, Cp, x_hi, x_lo, st, es);
  else
    e = pack_act(p.x, x, Cp, x_hi, x_lo, st, es);
  if (e != cudaSuccess) return e;

  WgTmaParams prm{};
  Im2colGeom ig{};
  ig.N = p.N;
  ig.H = IH;
  ig.W = IW;
  ig.C = Cp;
  ig.lower_h = lower_h;
  ig.lower_w = lower_w;
  ig.upper_h = upper_h;
  ig.upper_w = upper_w;
  ig.stride_h = gu;
  ig.stride_w = gv;
  ig.cpp = xw;
  ig.ppc = px;
  // MN-major operands: 128-byte swizzle (bf16), the 32-byte-atom 128-byte
  // swizzle for tf32 (descriptor layout SWIZZLE_128B_BASE32B)
  const CUtensorMapSwizzle xsw =
      es == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  if ((e = make_tmap_im2col(&prm.tm_xhi, x_hi, ig, xsw, es)) != cudaSuccess) return e;
  if ((e = make_tmap_im2col(&prm.tm_xlo, x_lo, ig, xsw, es)) != cudaSuccess) return e;
  {
    const uint64_t dims[3] = {uint64_t(dbw), uint64_t(NPQ), uint64_t(Kp64 / dbw)};
    const uint64_t strides[2] = {uint64_t(Kp64) * es, uint64_t(dbw) * es};
    const uint32_t box[3] = {uint32_t(dbw), uint32_t(px), uint32_t(bn / nc / dbw)};
    const CUtensorMapSwizzle dsw = es == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                   : bw32  ? CU_TENSOR_MAP_SWIZZLE_64B
                                           : CU_TENSOR_MAP_SWIZZLE_128B;
    if ((e = make_tmap_3d(&prm.tm_dyhi, dy_hi, dims, strides, box, dsw, es)) != cudaSuccess)
      return e;
    if ((e = make_tmap_3d(&prm.tm_dylo, dy_lo, dims, strides, box, dsw, es)) != cudaSuccess)
      return e;
  }
  prm.pix_per_split = pps;
  prm.NPQ = NPQ;
  prm.lower_h = lower_h;
  prm.lower_w = lower_w;
  prm.u = gu;
  prm.v = gv;
  prm.nCB = nCB;
  prm.tapW = S2;
  prm.taps = taps;
  prm.Cext = Cp;
  prm.mrows_p = mrows;
  prm.ncol_p = ncols;
  prm.ws = part;
  prm.dPQ = make_magic(uint32_t(p.P * p.Q));
  prm.dQ = make_magic(uint32_t(p.Q));
  static unsigned long long* tbuf = nullptr;
  const bool want_trace = ::dnnp::diag_env("DNNP_TC_TRACE") != nullptr;
  if (want_trace && !tbuf) cudaMalloc(&tbuf, 8192 * sizeof(unsigned long long));
  if (want_trace) cudaMemsetAsync(tbuf, 0, 8192 * sizeof(unsigned long long), st);
  prm.trace = want_trace ? tbuf : nullptr;
  const dim3 grid{unsigned(mt * nc), unsigned(nt), unsigned(splits)};
  auto go = [&](auto pxc) {
    constexpr int PX = decltype(pxc)::value;
    if (nc == 2 && bw32) {
      switch (bn) {
        case 64: return launch_wgrad_tma<64, 2, PX, 32>(prm, grid, st);
        default: return launch_wgrad_tma<192, 2, PX, 32>(prm, grid, st);
      }
    }
    if (nc == 2) {
      switch (bn) {
        case 128: return launch_wgrad_tma<128, 2, PX>(prm, grid, st);
        default: return launch_wgrad_tma<256, 2, PX>(prm, grid, st);
      }
    }
    switch (bn) {
      case 64: return launch_wgrad_tma<64, 1, PX>(prm, grid, st);
      case 128: return launch_wgrad_tma<128, 1, PX>(prm, grid, st);
      case 192: return launch_wgrad_tma<192, 1, PX>(prm, grid, st);
      default: return launch_wgrad_tma<256, 1, PX>(prm, grid, st);
    }
  };
  // 3xTF32: 32-channel dy blocks, 64 pixels per stage for <= 64 dy channels
  // per CTA, else 32 (the bf16 stage bytes)
  auto go_tf32 = [&]() -> cudaError_t {
    if (nc == 2) {
      switch (bn) {
        case 64: return launch_wgrad_tma<64, 2, 64, 32, 4>(prm, grid, st);
        case 128: return launch_wgrad_tma<128, 2, 64, 32, 4>(prm, grid, st);
        case 192: return launch_wgrad_tma<192, 2, 32, 32, 4>(prm, grid, st);
        default: return launch_wgrad_tma<256, 2, 32, 32, 4>(prm, grid, st);
      }
    }
    switch (bn) {
      case 64: return launch_wgrad_tma<64, 1, 64, 32, 4>(prm, grid, st);
      case 128: return launch_wgrad_tma<128, 1, 32, 32, 4>(prm, grid, st);
      case 192: return launch_wgrad_tma<192, 1, 32, 32, 4>(prm, grid, st);
      default: return launch_wgrad_tma<256, 1, 32, 32, 4>(prm, grid, st);
    }
  };
  if (es == 4)
    e = go_tf32();
  else
    e = px == 32    ? go(std::integral_constant<int, 32>())
        : px == 128 ? go(std::integral_constant<int, 128>())
                    : go(std::integral_constant<int, 64>());
  if (e != cudaSuccess) return e;
  if (want_trace) {
    static unsigned long long h[8192];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, tbuf, sizeof h, cudaMemcpyDeviceToHost);
    fprintf(stderr, "WGTRACE mt=%d nt=%d bn=%d nc=%d splits=%lld\n", mt, nt, bn, nc,
            (long long)splits);
    const unsigned long long t0 = h[0];
    for (int i = 0; i < 1024 && h[i * 4]; i++)
      fprintf(stderr, "st %4d P[%8lld %8lld] M[%8lld]\n", i, (long long)(h[i * 4] - t0),
              (long long)(h[i * 4 + 1] - t0), (long long)(h[i * 4 + 2] - t0));
  }
  WgReduceGeom rg{};
  rg.K = int(p.K);
  rg.C = int(p.C);
  rg.R = int(p.R);
  rg.S = int(p.S);
  rg.flip = p.flip ? 1 : 0;
  rg.su = su;
  rg.sv = sv;
  rg.S2 = S2;
  rg.Cpf = Cpf;
  rg.ncolx = ncolx;
  rg.splits = int(splits);
  rg.mrows_p = mrows;
  rg.ncol_p = ncols;
  wgrad_reduce_tma<<<grid_for(int64_t(ncolx) * p.K, 256, 16), 256, 0, st>>>(rg, part, df,
                                                                            acc ? 1 : 0);
  note_launch();
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t tc_backward_filter(const ConvProblem& p, const float* dy, const float* x, float* df,
                               bool acc, cudaStream_t st, int es) {
  using namespace tc;
  pool_keep_memory();
  {
    const cudaError_t te = wgrad_tma(p, dy, x, df, acc, st, es);
    if (te != cudaErrorNotSupported) return te;
  }
  if (es == 4) return cudaErrorNotSupported;  // 3xTF32: the caller runs SIMT fp32
  const int Kp = int(ceil_div(p.K, 8) * 8), Cp = int(ceil_div(p.C, 8) * 8), Cgrp = Cp / 8;
  const int KC = int(p.R * p.S) * Cgrp;
  const int64_t NPQ = p.N * p.P * p.Q, NHW = p.N * p.H * p.W;
  const int ncol = KC * 8;
  const int bn = ncol <= 64 ? 64 : (ncol <= 128 ? 128 : 256);
  const int nt = int(ceil_div(ncol, bn)), mt = int(ceil_div(p.K, 128));
  const int ncol_p = nt * bn, mrows_p = mt * 128;
  const int64_t kblocks = ceil_div(NPQ, kPx);
  int64_t splits = ceil_div(int64_t(kNumSMs) * 2, int64_t(mt) * nt);
  splits = std::max<int64_t>(1, std::min<int64_t>({splits, std::max<int64_t>(1, kblocks / 8), 128}));
  const int64_t pps = std::min(ceil_div(kblocks, splits) * kPx, max_chain(kPx));
  splits = ceil_div(NPQ, pps);

  const size_t dy_elems = size_t(NPQ) * Kp, x_elems = size_t(NHW) * Cp;
  const size_t ws_floats = size_t(splits) * mrows_p * ncol_p;
  Workspace ws(st);
  cudaError_t e = ws.alloc((dy_elems + x_elems) * 4 + ws_floats * 4 + size_t(KC) * 4 + 512);
  if (e != cudaSuccess) return e;
  auto* dy_hi = static_cast<__nv_bfloat16*>(ws.p);
  auto* dy_lo = dy_hi + dy_elems;
  auto* x_hi = dy_lo + dy_elems;
  auto* x_lo = x_hi + x_elems;
  float* part = reinterpret_cast<float*>(x_lo + x_elems);
  auto* ctab = reinterpret_cast<uint32_t*>(part + ws_floats);

  if ((e = pack_act(p.y, dy, Kp, dy_hi, dy_lo, st)) != cudaSuccess) return e;
  if ((e = pack_act(p.x, x, Cp, x_hi, x_lo, st)) != cudaSuccess) return e;
  fwd_ctab_kernel<<<unsigned(ceil_div(KC, 256)), 256, 0, st>>>(int(p.S), Cgrp, KC, ctab);
  note_launch();

  WgParams prm{};
  prm.NPQ = NPQ;
  prm.pix_per_split = pps;
  prm.P = int(p.P);
  prm.Q = int(p.Q);
  prm.H = int(p.H);
  prm.W = int(p.W);
  prm.u = int(p.u);
  prm.v = int(p.v);
  prm.pad_h = int(p.pad_h);
  prm.pad_w = int(p.pad_w);
  prm.Kp = Kp;
  prm.Cp = Cp;
  prm.KC = KC;
  prm.ncol_p = ncol_p;
  prm.mrows_p = mrows_p;
  prm.ctab = ctab;
  if ((e = make_tmap_2d(&prm.tm_dyhi, dy_hi, uint64_t(Kp), uint64_t(NPQ), uint64_t(Kp), 64, kPx,
                       CU_TENSOR_MAP_SWIZZLE_128B)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_dylo, dy_lo, uint64_t(Kp), uint64_t(NPQ), uint64_t(Kp), 64, kPx,
                       CU_TENSOR_MAP_SWIZZLE_128B)) != cudaSuccess)
    return e;
  prm.dy_hi = dy_hi;
  prm.dy_lo = dy_lo;
  prm.x_hi = x_hi;
  prm.x_lo = x_lo;
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
