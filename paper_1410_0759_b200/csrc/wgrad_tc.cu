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
  wgrad_tc_kernel<BN><<<grid, kThreads, CC::SMEM, st>>>(prm);
  note_launch();
  return cudaGetLastError();
}

}  // namespace
}  // namespace tc

cudaError_t tc_backward_filter(const ConvProblem& p, const float* dy, const float* x, float* df,
                               bool acc, cudaStream_t st) {
  using namespace tc;
  pool_keep_memory();
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
  const int64_t pps = ceil_div(kblocks, splits) * kPx;
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
