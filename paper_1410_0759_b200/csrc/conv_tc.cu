// tcgen05 implicit-GEMM convolution, fp32 via the BF16x3 split: forward and
// backward-data.
//
// Each fp32 operand value a is carried as a_hi = bf16(a), a_lo = bf16(a - a_hi)
// (16 of its 24 mantissa bits); every k-step issues three 5th-gen tensor-core
// MMAs into one FP32 TMEM accumulator:
//     D += A_lo.B_hi + A_hi.B_lo + A_hi.B_hi         (A_lo.B_lo ~ 2^-16 dropped)
// keeping fp32-class accuracy (normalised error ~4e-6 measured; bar 1e-4) at
// 2/3 of the TF32 tensor rate.
//
// The lowered im2col matrix is never materialised (paper Sec. 3): packing
// kernels produce channel-innermost BF16 hi/lo planes of the input (x for
// forward, dy for backward-data) and of the filter in the kernel's reduction
// order; the GEMM kernel gathers its A tile on the fly with 16-byte cp.async
// (zero-fill outside the image) through a chunk table decoding every 8-channel
// reduction chunk into its (dh, dw, c0) im2col offset.
//
// Kernel: persistent, warp specialised, one CTA per SM, 128 x BN tiles.
//   warps 0-7  producers: A gather (4 lanes per output pixel row, 16-byte
//              cp.async) + B tile by TMA into 64B-swizzled K-major stages
//              of 32 reduction elements
//   warp  8    TMEM allocation; lane 0 issues the tcgen05.mma stream
//   warps 9-12 epilogue: tcgen05.ld from a double-buffered TMEM accumulator,
//              alpha/beta blend straight into the caller's strided output,
//              overlapping the next tile's main loop
// mbarrier rings: full/empty per stage (producers <-> MMA), tfull/tempty per
// accumulator buffer (MMA <-> epilogue).
//
// Forward:        rows = N*P*Q output pixels, columns = K, red = R*S*Cp.
// Backward-data:  "super-pixel" form.  dx pixel (ph + u*i, pw + v*j) only
//   receives taps r' = t0(ph) + u*jr, which read dy row i + base(ph) - jr; the
//   union over phases of those offsets is a small window.  One stride-1 GEMM
//   over super-pixels (n, i, j) with columns (ph, pw, c) and reduction
//   (window tap, k) computes every phase at once (gather form, no atomics,
//   deterministic); for u = v = 1 it is the plain transposed convolution.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"
#include "tc_ptx.cuh"

namespace dnnp {
namespace tc {
namespace {

constexpr int kBM = 128;         // tile rows (UMMA M)
constexpr int kBK = 32;          // reduction elements per stage (64 B swizzle rows)
constexpr int kProdWarps = 8;    // A-gather producers (thread 0 also issues the B TMA)
constexpr int kMmaWarp = kProdWarps;
constexpr int kTmaWarp = kProdWarps + 1;
constexpr int kThreads = (kProdWarps + 2 + 4) * 32;  // + MMA warp + TMA warp + 4 epilogue warps
constexpr int kCtabSmem = 4096;  // chunk-table entries staged in shared memory

struct TcParams {
  CUtensorMap tm_bhi;            // packed filter planes [Np][Ktot], box {32, BN}, 64B swizzle
  CUtensorMap tm_blo;
  int64_t M;                     // GEMM rows
  int Ncol;                      // valid columns
  int OH, OW;                    // GEMM row grid of one image
  int IH, IW, Cp;                // packed input [N][IH][IW][Cp]
  int u, v, pad_h, pad_w;        // gather: ih = oh*u - pad_h + dh
  int KC, nkb, Ktot;             // 16 B reduction chunks, k-blocks, packed filter pitch
  int kb_lo;                     // first k-block of this launch (reduction segment [kb_lo, nkb))
  int nt, tiles;                 // column tiles, total tiles
  const uint32_t* ctab;          // chunk -> (dh << 24) | (dw << 16) | c0
  const __nv_bfloat16* a_hi;
  const __nv_bfloat16* a_lo;
  const __nv_bfloat16* b_hi;
  const __nv_bfloat16* b_lo;
  float* out;
  int64_t o_sn, o_sc, o_sh, o_sw;
  int out_mode;                  // 0: column = channel; 1: super-pixel column table
  int o_u, o_v, o_H, o_W;        // super-pixel: h = oh*o_u + ph < o_H
  const uint32_t* coltab;        // column -> (ph << 24) | (pw << 16) | c
  float alpha, beta;
  int products;                  // 3 (BF16x3); 1 only for bottleneck experiments
  int plain;                     // alpha == 1, beta == 0, nkb > 0: epilogue stores acc as is
  int skip;                      // experiments: 1 = skip A gather, 2 = skip B TMA
  unsigned long long* trace;     // debug: per-stage clock64 stamps of CTA 0 (or null)
  MagicDiv dOHW, dOW;
};

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = kBM * kBK * 2;  // 8 KB per plane
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES =
      (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS =
      2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512));
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + kCtabSmem * 4;
};

// byte offset of 16-byte chunk j of row r in a K-major 64B-swizzled tile
__device__ __forceinline__ uint32_t sw64(int r, int j) {
  return uint32_t((r >> 3) * 512 + (r & 7) * 64 + ((j ^ ((r >> 1) & 3)) << 4));
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ TcParams P) {
  using C = Cfg<BN>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* ctab_s = reinterpret_cast<uint32_t*>(smem + S * C::STAGE_BYTES + 256);
  const bool ctab_in_smem = P.KC <= kCtabSmem;
  if (ctab_in_smem)
    for (int i = threadIdx.x; i < P.KC; i += blockDim.x) ctab_s[i] = __ldg(P.ctab + i);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int s = 0; s < S; s++) {
        ptx::mbar_init(&full[s], kProdWarps * 32 + 1);  // gather arrivals + expect_tx (TMA B)
        ptx::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; b++) {
        ptx::mbar_init(&tfull[b], 1);
        ptx::mbar_init(&tempty[b], 128);
      }
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t smem0 = ptx::smem_u32(smem);
  if (P.trace && threadIdx.x == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    P.trace[3000 + blockIdx.x * 4 + 0] = gt;
    P.trace[3000 + blockIdx.x * 4 + 1] = clock64();
  }

  if (warp < kProdWarps) {
    // =================================================== producers
    // A: lane quad (t & 3) = 16-byte chunk of the 64-byte k-block row, rows
    // (t >> 2) + RSTEP*i: 4 lanes read one pixel's contiguous 64 bytes.
    // B: one elected thread streams the filter tile with TMA.
    const int t = threadIdx.x;
    constexpr int RSTEP = kProdWarps * 8;   // rows covered per i-step
    constexpr int RPT = kBM / RSTEP;        // rows per thread
    const int j = t & 3, rb = t >> 2;
    int it = 0;
    for (int tile = blockIdx.x; tile < P.tiles; tile += gridDim.x) {
      const int64_t mbase = int64_t(tile / P.nt) * kBM;
      int ih0[RPT], iw0[RPT];
      int64_t pix0[RPT];
      bool rok[RPT];
#pragma unroll
      for (int i = 0; i < RPT; i++) {
        const int64_t m = mbase + rb + RSTEP * i;
        rok[i] = m < P.M;
        uint32_t img = 0, oh = 0, ow = 0;
        if (rok[i]) {
          uint32_t rem;
          mdivmod(uint32_t(m), P.dOHW, img, rem);
          mdivmod(rem, P.dOW, oh, ow);
        }
        ih0[i] = int(oh) * P.u - P.pad_h;
        iw0[i] = int(ow) * P.v - P.pad_w;
        pix0[i] = int64_t(img) * P.IH * P.IW;
      }
      for (int kb = P.kb_lo; kb < P.nkb; kb++, it++) {
        const int s = it % S;
        const bool tr = P.trace && blockIdx.x == 0 && t == 0 && it < 256;
        if (tr) P.trace[it * 8 + 0] = clock64();
        if (it >= S) ptx::mbar_wait(&empty[s], ((it / S) - 1) & 1);
        if (tr) P.trace[it * 8 + 1] = clock64();
        const uint32_t sa_hi = smem0 + s * C::STAGE_BYTES;
        const uint32_t sa_lo = sa_hi + C::A_BYTES;
        const uint32_t sb_hi = sa_lo + C::A_BYTES;
        const uint32_t sb_lo = sb_hi + C::B_BYTES;
        const int ch = kb * 4 + j;
        const bool ch_ok = ch < P.KC;
        const uint32_t e = ch_ok ? (ctab_in_smem ? ctab_s[ch] : __ldg(P.ctab + ch)) : 0u;
        const int dh = int(e >> 24), dw = int((e >> 16) & 255), c0 = int(e & 0xFFFF);
#pragma unroll
        for (int i = 0; i < RPT && !(P.skip & 1); i++) {
          const int ih = ih0[i] + dh, iw = iw0[i] + dw;
          const bool ok = ch_ok && rok[i] && unsigned(ih) < unsigned(P.IH) &&
                          unsigned(iw) < unsigned(P.IW);
          const int64_t src = ok ? (pix0[i] + int64_t(ih) * P.IW + iw) * P.Cp + c0 : 0;
          const uint32_t dst = sw64(rb + RSTEP * i, j);
          ptx::cp_async16(sa_hi + dst, P.a_hi + src, ok ? 16u : 0u);
          ptx::cp_async16(sa_lo + dst, P.a_lo + src, ok ? 16u : 0u);
        }
        ptx::cp_async_mbar_arrive(&full[s]);
        if (tr) P.trace[it * 8 + 2] = clock64();
      }
    }
    ptx::cp_async_wait<0>();
  } else if (warp == kMmaWarp) {
    // =================================================== MMA issuer
    // The whole warp runs the loop (warp-uniform descriptors stay in uniform
    // registers); one elected lane issues each tcgen05.mma / commit.
    {
      constexpr uint32_t idesc = ptx::idesc_bf16(kBM, BN, 0, 0);
      int it = 0, lt = 0;
      for (int tile = blockIdx.x; tile < P.tiles; tile += gridDim.x, lt++) {
        const int buf = lt & 1;
        ptx::mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t dacc = tmem_base + uint32_t(buf * BN);
        uint32_t acc = 0;
        // two stages per iteration: one barrier-wait/fence/loop overhead per 12 MMAs
        for (int kb = P.kb_lo; kb < P.nkb; kb += 2) {
          const int npair = P.nkb - kb >= 2 ? 2 : 1;
          const bool tr = P.trace && blockIdx.x == 0 && lane == 0 && it < 256;
          if (tr) P.trace[it * 8 + 3] = clock64();
          ptx::mbar_wait(&full[it % S], (it / S) & 1);
          if (npair == 2) ptx::mbar_wait(&full[(it + 1) % S], ((it + 1) / S) & 1);
          if (tr) P.trace[it * 8 + 4] = clock64();
          ptx::fence_proxy_async();  // producers' cp.async writes -> async proxy
          ptx::tc_fence_after();
          if (tr) P.trace[it * 8 + 6] = clock64();
          for (int q = 0; q < npair; q++, it++) {
            const int s = it % S;
            const uint32_t sa_hi = smem0 + s * C::STAGE_BYTES;
            const uint64_t dah = ptx::desc_kmajor_sw64(sa_hi);
            const uint64_t dal = ptx::desc_kmajor_sw64(sa_hi + C::A_BYTES);
            const uint64_t dbh = ptx::desc_kmajor_sw64(sa_hi + 2 * C::A_BYTES);
            const uint64_t dbl = ptx::desc_kmajor_sw64(sa_hi + 2 * C::A_BYTES + C::B_BYTES);
#pragma unroll
            for (int kk = 0; kk < kBK / 16; kk++) {
              const uint64_t o = uint64_t(kk * 2);  // +32 bytes along K
              if (P.products == 3) {
                ptx::mma_bf16_elect(dacc, dal + o, dbh + o, idesc, acc);
                acc = 1;
                ptx::mma_bf16_elect(dacc, dah + o, dbl + o, idesc, 1);
              }
              ptx::mma_bf16_elect(dacc, dah + o, dbh + o, idesc, acc);
              acc = 1;
            }
            ptx::mma_commit_elect(&empty[s]);
          }
          if (tr) P.trace[(it - npair) * 8 + 5] = clock64();
        }
        ptx::mma_commit_elect(&tfull[buf]);
      }
    }
  } else if (warp == kTmaWarp) {
    // =================================================== B tile by TMA
    if (lane == 0) {
      ptx::tma_prefetch(&P.tm_bhi);
      ptx::tma_prefetch(&P.tm_blo);
      int it = 0;
      for (int tile = blockIdx.x; tile < P.tiles; tile += gridDim.x) {
        const int n0 = (tile % P.nt) * BN;
        for (int kb = P.kb_lo; kb < P.nkb; kb++, it++) {
          const int s = it % S;
          if (it >= S) ptx::mbar_wait(&empty[s], ((it / S) - 1) & 1);
          const uint32_t sb_hi = smem0 + s * C::STAGE_BYTES + 2 * C::A_BYTES;
          if (P.skip & 2) {
            ptx::mbar_arrive(&full[s]);
          } else {
            ptx::mbar_arrive_expect_tx(&full[s], 2 * C::B_BYTES);
            ptx::tma_load_2d(sb_hi, &P.tm_bhi, kb * kBK, n0, &full[s]);
            ptx::tma_load_2d(sb_hi + C::B_BYTES, &P.tm_blo, kb * kBK, n0, &full[s]);
          }
        }
      }
    }
  } else {
    // =================================================== epilogue
    const int ew = warp & 3;  // TMEM lane quadrant of this warp
    const int r = ew * 32 + lane;
    int lt = 0;
    for (int tile = blockIdx.x; tile < P.tiles; tile += gridDim.x, lt++) {
      const int buf = lt & 1;
      const int64_t m = int64_t(tile / P.nt) * kBM + r;
      const int n0 = (tile % P.nt) * BN;
      const bool row_ok = m < P.M;
      uint32_t img = 0, oh = 0, ow = 0;
      if (row_ok) {
        uint32_t rem;
        mdivmod(uint32_t(m), P.dOHW, img, rem);
        mdivmod(rem, P.dOW, oh, ow);
      }
      const bool etr = P.trace && blockIdx.x == 0 && threadIdx.x == kThreads - 128 && lt < 16;
      if (etr) P.trace[2048 + lt * 4 + 0] = clock64();
      ptx::mbar_wait(&tfull[buf], (lt >> 1) & 1);
      if (etr) P.trace[2048 + lt * 4 + 1] = clock64();
      ptx::tc_fence_after();
      const int64_t rowoff =
          P.out_mode == 0 ? int64_t(img) * P.o_sn + int64_t(oh) * P.o_sh + int64_t(ow) * P.o_sw
                          : int64_t(img) * P.o_sn;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        ptx::tmem_ld32(tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(buf * BN + c0), v);
        ptx::tmem_ld_wait();
        if (!row_ok) continue;
        const int cbase = n0 + c0;
        if (P.out_mode == 0 && P.plain && cbase + 32 <= P.Ncol) {
          // y = acc: one store per element through a running column pointer
          float* dst = P.out + rowoff + int64_t(cbase) * P.o_sc;
          const int64_t sc = P.o_sc;
#pragma unroll
          for (int i = 0; i < 32; i++) {
            *dst = __uint_as_float(v[i]);
            dst += sc;
          }
        } else if (P.out_mode == 0) {
          float* rowp = P.out + rowoff + int64_t(cbase) * P.o_sc;
#pragma unroll
          for (int i = 0; i < 32; i++) {
            if (cbase + i < P.Ncol) {
              float* dst = rowp + int64_t(i) * P.o_sc;
              const float accv = P.nkb > P.kb_lo ? __uint_as_float(v[i]) : 0.0f;
              float val = __fmul_rn(accv, P.alpha);
              if (P.beta != 0.0f) val = __fadd_rn(__fmul_rn(*dst, P.beta), val);
              *dst = val;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; i++) {
            const int col = cbase + i;
            if (col < P.Ncol) {
              const uint32_t e = __ldg(P.coltab + col);
              const int h = int(oh) * P.o_u + int(e >> 24);
              const int w = int(ow) * P.o_v + int((e >> 16) & 255);
              if (h < P.o_H && w < P.o_W) {
                float* dst = P.out + rowoff + int64_t(e & 0xFFFF) * P.o_sc + int64_t(h) * P.o_sh +
                             int64_t(w) * P.o_sw;
                const float accv = P.nkb > P.kb_lo ? __uint_as_float(v[i]) : 0.0f;
                float val = __fmul_rn(accv, P.alpha);
                if (P.beta != 0.0f) val = __fadd_rn(__fmul_rn(*dst, P.beta), val);
                *dst = val;
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      if (etr) P.trace[2048 + lt * 4 + 2] = clock64();
      ptx::mbar_arrive(&tempty[buf]);
    }
  }
  __syncthreads();
  if (P.trace && threadIdx.x == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    P.trace[3000 + blockIdx.x * 4 + 2] = gt;
    P.trace[3000 + blockIdx.x * 4 + 3] = clock64();
  }
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

#include "conv_tma.cuh"
#include "conv_halo.cuh"

// ---------------------------------------------------------- filter packing

// Geometry of the reduction / column orders of one GEMM.
//  forward:  column = output channel k; chunk = (dh*S + dw)*Cgrp + g over the
//            R x S taps; gather offset (dh, dw).
//  bwd-data: column = (ph*v + pw)*C + c; chunk = (dh*WinW + dw)*Kg + g over
//            the super-pixel window; dh corresponds to phase tap
//            jr = base(ph) - dh - lo_h when 0 <= jr < nR(ph), gather offset
//            r' = t0(ph) + u*jr; zero otherwise.
//  space-to-depth (su * sv > 1): the GEMM problem is the stride-1
//            convolution over x'[n][h'][w'][(rh*sv + rw)*C0 + c]; GEMM channel
//            cg decodes to (rh, rw, c) and a GEMM gather offset t to the
//            original offset t*su + rh (zero when >= R0).
// The filter value for gather offset r' is f[..][R0-1-r'] in CONVOLUTION
// mode and f[..][r'] in CROSS_CORRELATION mode (reference conv.py:182-192).
struct PackGeom {
  int K, C, R, S, flip, dgrad;
  int u, v, pad_h, pad_w;  // bwd-data phases
  int winH, winW, lo_h, lo_w;
  int Ncol, Np, Ktot, Cgrp, KC;
  int su, sv, C0, R0, S0;  // space-to-depth factors and the original C, R, S
  // column blocking (TMA path, small GEMM N): GEMM row j covers bw adjacent
  // output columns, GEMM column = e * Ncol0 + n; the blocked taps along w
  // (tapW) map to the unblocked tap dw = dwb - e * vstep (valid in [0, Sg)).
  int tapH, tapW, bw, Ncol0, vstep, Sg;
  // bdir = 1: the block runs down the output rows instead: blocked tap row
  // dhb maps to dh = dhb - e * ustep (valid in [0, Rg)); bdir = 2: a 2-D
  // block of bh rows x bw columns, e = eh * bw + ew
  int bdir, ustep, Rg, bh;
};

__device__ __forceinline__ float fetch_filter(const PackGeom& g, const float* __restrict__ f,
                                              int k, int cg, int tr, int ts) {
  int c = cg, rh = 0, rw = 0;
  if (g.su * g.sv > 1) {
    const int ph = cg / g.C0;
    c = cg - ph * g.C0;
    rw = ph % g.sv;
    rh = ph / g.sv;
  }
  int r = tr * g.su + rh, s = ts * g.sv + rw;
  if (k >= g.K || c >= g.C0 || r >= g.R0 || s >= g.S0) return 0.0f;
  if (g.flip) {
    r = g.R0 - 1 - r;
    s = g.S0 - 1 - s;
  }
  return f[((int64_t(k) * g.C0 + c) * g.R0 + r) * g.S0 + s];
}

__device__ __forceinline__ int phase_tap(int ph, int dh, int lo, int u, int pad, int R) {
  const int t0 = (ph + pad) % u;
  const int nR = t0 < R ? (R - t0 + u - 1) / u : 0;
  const int base = (ph + pad - t0) / u;
  const int jr = base - dh - lo;
  if (jr < 0 || jr >= nR) return -1;
  return t0 + u * jr;  // gather offset r'
}

// Filter packing, one block per (GEMM column row, tap): the tap's gather
// offsets (and the bwd-data phase taps) are resolved once per block, threads
// walk the tap's Cpf reduction channels (coalesced 2-byte stores).  Block
// x == taps zero-fills the K padding tail.
template <int ES>
__global__ void __launch_bounds__(128) pack_filter_tap_kernel(PackGeom g, const float* __restrict__ f,
                                                              void* __restrict__ hi,
                                                              void* __restrict__ lo,
                                                              uint32_t* __restrict__ ctab,
                                                              uint32_t* __restrict__ coltab, int taps) {
  const int row = blockIdx.y, tap = blockIdx.x;
  const int Cpf = g.Cgrp * 8;
  const int64_t rbase = int64_t(row) * g.Ktot;
  if (tap == taps) {  // padding tail of the reduction
    for (int k = taps * Cpf + threadIdx.x; k < g.Ktot; k += blockDim.x)
      store_split1<ES>(hi, lo, rbase + k, 0.0f);
    return;
  }
  const int dhb = tap / g.tapW, dwb = tap - (tap / g.tapW) * g.tapW;
  const int e = row / g.Ncol0, r0 = row - e * g.Ncol0;  // column block, unblocked column
  const int eh = g.bdir == 2 ? e / g.bw : (g.bdir ? e : 0);
  const int ew = g.bdir == 2 ? e - eh * g.bw : (g.bdir ? 0 : e);
  const int dw = dwb - ew * g.vstep;
  const int dh = dhb - eh * g.ustep;
  const bool tap_ok = row < g.Ncol && dw >= 0 && dw < g.Sg && dh >= 0 && dh < g.Rg;
  int c_col = 0, rp = -1, sp = -1, ph = 0, pw = 0;
  if (g.dgrad && row < g.Ncol) {
    const int phase = r0 / g.C;
    c_col = r0 - phase * g.C;
    ph = phase / g.v;
    pw = phase - ph * g.v;
    rp = phase_tap(ph, dh, g.lo_h, g.u, g.pad_h, g.R);
    sp = tap_ok ? phase_tap(pw, dw, g.lo_w, g.v, g.pad_w, g.S) : -1;
  }
  if (tap == 0 && threadIdx.x == 0 && row < g.Ncol && (g.dgrad || g.bw > 1)) {
    uint32_t oh_, ow_, oc_;
    if (!g.dgrad) {
      oh_ = uint32_t(eh), ow_ = uint32_t(ew), oc_ = uint32_t(r0);
    } else if (g.su * g.sv > 1) {  // space-to-depth column (rh, rw, c)
      const int q = r0 / g.C0;
      oh_ = uint32_t(q / g.sv), ow_ = uint32_t(e * g.sv + q % g.sv), oc_ = uint32_t(r0 - q * g.C0);
    } else {
      oh_ = uint32_t(eh * g.u + ph), ow_ = uint32_t(ew * g.v + pw), oc_ = uint32_t(c_col);
    }
    coltab[row] = (oh_ << 24) | (ow_ << 16) | oc_;
  }
  if (row == 0)
    for (int grp = threadIdx.x; grp < g.Cgrp; grp += blockDim.x)
      ctab[tap * g.Cgrp + grp] = (uint32_t(dhb) << 24) | (uint32_t(dwb) << 16) | uint32_t(grp * 8);
  for (int cin = threadIdx.x; cin < Cpf; cin += blockDim.x) {
    float val = 0.0f;
    if (!g.dgrad) {
      if (tap_ok && r0 < g.K && cin < g.C) val = fetch_filter(g, f, r0, cin, dh, dw);
    } else if (row < g.Ncol && cin < g.K && rp >= 0 && sp >= 0) {
      val = fetch_filter(g, f, cin, c_col, rp, sp);
    }
    store_split1<ES>(hi, lo, rbase + tap * Cpf + cin, val);
  }
}

// Filter packing, one thread per 8 consecutive packed elements (one GEMM
// column row, one tap, 8 reduction channels): a grid-stride loop over the
// whole [Np][Ktot] operand, one 16-byte store per plane (bf16) and 8 gathered
// filter loads.  The same element map as the per-(tap, row) kernel, which
// spawned (taps + 1) x Np tiny blocks (4-11 us per AlexNet layer, launch
// and scheduling bound for ~1 M elements); the column (bwd-data / blocked)
// and chunk tables are filled by the same grid.
template <int ES>
__global__ void __launch_bounds__(256) pack_filter_vec_kernel(PackGeom g, const float* __restrict__ f,
                                                              void* __restrict__ hi,
                                                              void* __restrict__ lo,
                                                              uint32_t* __restrict__ ctab,
                                                              uint32_t* __restrict__ coltab, int taps,
                                                              MagicDiv dK8, MagicDiv dC8) {
  const int Cpf = g.Cgrp * 8;
  const uint32_t k8n = uint32_t(g.Ktot / 8);
  const uint32_t total8 = uint32_t(g.Np) * k8n;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (uint32_t i = tid; i < total8; i += stride) {
    uint32_t row32, k8;
    mdivmod(i, dK8, row32, k8);
    const int row = int(row32), kcol = int(k8) * 8;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = 0.0f;
    if (kcol < taps * Cpf && row < g.Ncol) {
      uint32_t tapu, c8;
      mdivmod(k8, dC8, tapu, c8);
      const int tap = int(tapu), cin0 = int(c8) * 8;
      const int dhb = tap / g.tapW, dwb = tap - dhb * g.tapW;
      const int e = row / g.Ncol0, r0 = row - e * g.Ncol0;
      const int eh = g.bdir == 2 ? e / g.bw : (g.bdir ? e : 0);
      const int ew = g.bdir == 2 ? e - eh * g.bw : (g.bdir ? 0 : e);
      const int dw = dwb - ew * g.vstep, dh = dhb - eh * g.ustep;
      const bool tap_ok = dw >= 0 && dw < g.Sg && dh >= 0 && dh < g.Rg;
      if (!g.dgrad) {
        if (tap_ok && r0 < g.K) {
#pragma unroll
          for (int j = 0; j < 8; j++)
            if (cin0 + j < g.C) v[j] = fetch_filter(g, f, r0, cin0 + j, dh, dw);
        }
      } else {
        const int phase = r0 / g.C, c_col = r0 - phase * g.C;
        const int ph = phase / g.v, pw = phase - ph * g.v;
        const int rp = phase_tap(ph, dh, g.lo_h, g.u, g.pad_h, g.R);
        const int sp = tap_ok ? phase_tap(pw, dw, g.lo_w, g.v, g.pad_w, g.S) : -1;
        if (rp >= 0 && sp >= 0) {
#pragma unroll
          for (int j = 0; j < 8; j++)
            if (cin0 + j < g.K) v[j] = fetch_filter(g, f, cin0 + j, c_col, rp, sp);
        }
      }
    }
    store_split8<ES>(hi, lo, int64_t(row) * g.Ktot + kcol, v);
  }
  // chunk table (cp.async gather; row 0 of the per-tap kernel)
  for (uint32_t i = tid; i < uint32_t(taps * g.Cgrp); i += stride) {
    const int tap = int(i) / g.Cgrp, grp = int(i) - tap * g.Cgrp;
    ctab[i] = (uint32_t(tap / g.tapW) << 24) | (uint32_t(tap % g.tapW) << 16) | uint32_t(grp * 8);
  }
  // column table (bwd-data phases / blocked columns)
  if (g.dgrad || g.bw > 1) {
    for (uint32_t i = tid; i < uint32_t(g.Ncol); i += stride) {
      const int row = int(i);
      const int e = row / g.Ncol0, r0 = row - e * g.Ncol0;
      const int eh = g.bdir == 2 ? e / g.bw : (g.bdir ? e : 0);
      const int ew = g.bdir == 2 ? e - eh * g.bw : (g.bdir ? 0 : e);
      uint32_t oh_, ow_, oc_;
      if (!g.dgrad) {
        oh_ = uint32_t(eh), ow_ = uint32_t(ew), oc_ = uint32_t(r0);
      } else if (g.su * g.sv > 1) {  // space-to-depth column (rh, rw, c)
        const int q = r0 / g.C0;
        oh_ = uint32_t(q / g.sv), ow_ = uint32_t(e * g.sv + q % g.sv), oc_ = uint32_t(r0 - q * g.C0);
      } else {
        const int phase = r0 / g.C, c_col = r0 - phase * g.C;
        const int ph = phase / g.v, pw = phase - ph * g.v;
        oh_ = uint32_t(eh * g.u + ph), ow_ = uint32_t(ew * g.v + pw), oc_ = uint32_t(c_col);
      }
      coltab[row] = (oh_ << 24) | (ow_ << 16) | oc_;
    }
  }
  // launched programmatically beside the operand pack (which it does not
  // read; the pack triggers at its start): complete only once that pack has,
  // so the GEMM's single wait covers both producers -- and trigger the GEMM
  // only then, so its persistent CTAs do not take SMs the pack still needs
  pdl_wait();
  pdl_trigger();
}

// Forward filter packing, one block per GEMM column row (all taps): the
// row's filter f[k][:][:][:] (contiguous C*R*S floats) is staged in shared
// memory with coalesced loads, then each warp writes whole taps of the packed
// row (lanes along the channels).  Coalesced, but only Np blocks: measured
// slower than the per-(tap, row) kernel (8.3 vs ~5 us per AlexNet layer), so
// it is opt-in (DNNP_PACK_ROWS).
template <int ES>
__global__ void __launch_bounds__(256) pack_filter_row_kernel(PackGeom g, const float* __restrict__ f,
                                                              void* __restrict__ hi,
                                                              void* __restrict__ lo,
                                                              uint32_t* __restrict__ ctab,
                                                              uint32_t* __restrict__ coltab, int taps) {
  extern __shared__ float sf[];
  const int row = blockIdx.x;
  const int Cpf = g.Cgrp * 8;
  const int64_t rbase = int64_t(row) * g.Ktot;
  const int e = row / g.Ncol0, r0 = row - e * g.Ncol0;
  const int nf = g.C0 * g.R0 * g.S0;
  const bool live = row < g.Ncol && r0 < g.K;
  if (live) {
    const float* src = f + int64_t(r0) * nf;
    for (int i = threadIdx.x; i < nf; i += blockDim.x) sf[i] = __ldg(src + i);
  }
  if (threadIdx.x == 0 && row < g.Ncol && g.bw > 1) {
    const uint32_t eh = g.bdir ? uint32_t(e) : 0u, ew = g.bdir ? 0u : uint32_t(e);
    coltab[row] = (eh << 24) | (ew << 16) | uint32_t(r0);
  }
  if (row == 0)
    for (int i = threadIdx.x; i < taps * g.Cgrp; i += blockDim.x) {
      const int tap = i / g.Cgrp, grp = i - tap * g.Cgrp;
      ctab[i] = (uint32_t(tap / g.tapW) << 24) | (uint32_t(tap % g.tapW) << 16) | uint32_t(grp * 8);
    }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int tap = warp; tap < taps; tap += nw) {
    const int dhb = tap / g.tapW, dwb = tap - dhb * g.tapW;
    const int dw = g.bdir ? dwb : dwb - e * g.vstep;
    const int dh = g.bdir ? dhb - e * g.ustep : dhb;
    const bool tap_ok = live && dw >= 0 && dw < g.Sg && dh >= 0 && dh < g.Rg;
    for (int cin = lane; cin < Cpf; cin += 32) {
      float val = 0.0f;
      if (tap_ok && cin < g.C) {
        // fetch_filter's map, reading the staged row
        int c = cin, rh = 0, rw = 0;
        if (g.su * g.sv > 1) {
          const int ph = cin / g.C0;
          c = cin - ph * g.C0;
          rw = ph % g.sv;
          rh = ph / g.sv;
        }
        int r = dh * g.su + rh, s2 = dw * g.sv + rw;
        if (c < g.C0 && r < g.R0 && s2 < g.S0) {
          if (g.flip) {
            r = g.R0 - 1 - r;
            s2 = g.S0 - 1 - s2;
          }
          val = sf[(c * g.R0 + r) * g.S0 + s2];
        }
      }
      store_split1<ES>(hi, lo, rbase + tap * Cpf + cin, val);
    }
  }
  for (int k = taps * Cpf + threadIdx.x; k < g.Ktot; k += blockDim.x)
    store_split1<ES>(hi, lo, rbase + k, 0.0f);
}

// Scatter form of the filter packing: one thread per filter element (read
// coalesced) computes its single position in the packed GEMM operand; the
// padding is zeroed by a memset first.  Inverse of the tap kernel's map:
// gather offset r' -> (space-to-depth tap r'/su, phase r'%su); for the
// super-pixel bwd-data form t0 = r' % u, jr = r' / u, phase ph = (t0 - pad)
// mod u and window tap dh = base(ph) - jr - lo.
template <int ES>
__global__ void __launch_bounds__(256) pack_filter_scatter_kernel(PackGeom g, const float* __restrict__ f,
                                                                  void* __restrict__ hi,
                                                                  void* __restrict__ lo) {
  const int total = g.K * g.C0 * g.R0 * g.S0;
  const int Cpf = g.Cgrp * 8;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int s = idx % g.S0;
    int t = idx / g.S0;
    const int r = t % g.R0;
    t /= g.R0;
    const int c0 = t % g.C0, k = t / g.C0;
    const int ro = g.flip ? g.R0 - 1 - r : r, so = g.flip ? g.S0 - 1 - s : s;
    const int rt = ro / g.su, st = so / g.sv;
    const int cg = ((ro % g.su) * g.sv + so % g.sv) * g.C0 + c0;
    int64_t o;
    if (!g.dgrad) {
      o = int64_t(k) * g.Ktot + (rt * g.S + st) * Cpf + cg;
    } else {
      const int t0h = rt % g.u, jrh = rt / g.u;
      const int ph = ((t0h - g.pad_h) % g.u + g.u) % g.u;
      const int dh = (ph + g.pad_h - t0h) / g.u - jrh - g.lo_h;
      const int t0w = st % g.v, jrw = st / g.v;
      const int pw = ((t0w - g.pad_w) % g.v + g.v) % g.v;
      const int dw = (pw + g.pad_w - t0w) / g.v - jrw - g.lo_w;
      const int row = (ph * g.v + pw) * g.C + cg;
      o = int64_t(row) * g.Ktot + (dh * g.winW + dw) * Cpf + k;
    }
    store_split1<ES>(hi, lo, o, __ldg(f + idx));
  }
}

// chunk table (cp.async kernel) and bwd-data column table
__global__ void pack_tables_kernel(PackGeom g, uint32_t* __restrict__ ctab, uint32_t* __restrict__ coltab,
                                   int want_ctab) {
  const int nS = g.dgrad ? g.winW : g.S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max(g.KC, g.Ncol); i += gridDim.x * blockDim.x) {
    if (want_ctab && i < g.KC) {
      const int tap = i / g.Cgrp, grp = i % g.Cgrp;
      ctab[i] = (uint32_t(tap / nS) << 24) | (uint32_t(tap % nS) << 16) | uint32_t(grp * 8);
    }
    if (g.dgrad && i < g.Ncol) {
      uint32_t e;
      if (g.su * g.sv > 1) {
        const int q = i / g.C0, c = i - q * g.C0;
        e = (uint32_t(q / g.sv) << 24) | (uint32_t(q % g.sv) << 16) | uint32_t(c);
      } else {
        const int c = i % g.C, phase = i / g.C;
        e = (uint32_t(phase / g.v) << 24) | (uint32_t(phase % g.v) << 16) | uint32_t(c);
      }
      coltab[i] = e;
    }
  }
}

// ------------------------------------------------------------- launching

template <int BN>
cudaError_t launch_gemm(const TcParams& prm, cudaStream_t st) {
  using CC = Cfg<BN>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const unsigned grid = unsigned(std::min<int64_t>(prm.tiles, kNumSMs));
  ktime_begin(st, 3);
  conv_tc_kernel<BN><<<grid, kThreads, CC::SMEM, st>>>(prm);
  ktime_end(st);
  note_launch();
  return cudaGetLastError();
}

template <int BN, int CB, int NC, int ES>
cudaError_t launch_tma(const TmaParams& prm, cudaStream_t st) {
  using CC = TCfg<BN, CB, NC, ES>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(conv_tma_kernel<BN, CB, NC, ES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM);
    if (e != cudaSuccess) return e;
    if (NC == 2) {
      e = cudaFuncSetAttribute(conv_tma_kernel<BN, CB, NC, ES>,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
      (void)e;
    }
    attr_dev = dev;
  }
  const int clusters =
      prm.clusters > 0 ? prm.clusters : int(std::min<int64_t>(prm.tiles, kNumSMs / NC));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(clusters * NC));
  cfg.blockDim = dim3(kTmaThreads);
  cfg.dynamicSmemBytes = CC::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  unsigned nattr = 1;
  add_pdl_attr(attr, &nattr);  // prologue overlaps the packs; pdl_wait() before any operand read
  cfg.attrs = attr;
  cfg.numAttrs = nattr;
  if (::dnnp::diag_env("DNNP_TC_DIAG")) {
    int ncl = -1;
    cudaError_t qe = cudaOccupancyMaxActiveClusters(&ncl, conv_tma_kernel<BN, CB, NC, ES>, &cfg);
    fprintf(stderr, "DIAG conv_tma<%d,%d,%d,%d> smem=%d grid=%d maxActiveClusters=%d (%s)\n", BN, CB, NC, ES,
            CC::SMEM, clusters * NC, ncl, cudaGetErrorString(qe));
  }
  ktime_begin(st, 1);
  cudaError_t e = cudaLaunchKernelEx(&cfg, conv_tma_kernel<BN, CB, NC, ES>, prm);
  ktime_end(st);
  note_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int CB, int NC, int ES>
cudaError_t launch_tma_bn(int bn, const TmaParams& prm, cudaStream_t st) {
  switch (bn) {
    case 64: return launch_tma<64, CB, NC, ES>(prm, st);
    case 128: return launch_tma<128, CB, NC, ES>(prm, st);
    case 192: return launch_tma<192, CB, NC, ES>(prm, st);
    default: return launch_tma<256, CB, NC, ES>(prm, st);
  }
}

// Tile shape for the TMA kernel: NC CTAs x 128 rows by bn columns.  Per SM
// and 64-deep stage: the MMAs take 6*bn cycles; the SM ingests the A tile
// (128 rows x 128 B x hi/lo = 32 KB) plus its share of B (bn/NC rows x
// 256 B) at ~57 B/clk when every SM streams (profiles/r01/tma_burst_probe.txt);
// the single producer issues (64/cb) * 4 TMA instructions at ~120 cycles.
// Persistent clusters run ceil(tiles / clusters) waves of such tiles.
void pick_tile_tma(int64_t M, int ncol, int cb, int* bn_out, int* nc_out) {
  static const int cands[] = {64, 128, 192, 256};
  double best = 1e30;
  *bn_out = 256;
  *nc_out = 1;
  const int max_nc = ::dnnp::tune_env("DNNP_TC_NO_PAIRS") ? 1 : 2;
  for (int nc = 1; nc <= max_nc; nc++) {
    for (int bn : cands) {
      if (bn >= 2 * ncol && bn > 64) continue;
      const int64_t tiles = ceil_div(M, 128 * nc) * ceil_div(ncol, bn);
      const double waves = std::ceil(double(tiles) / (kNumSMs / nc));
      const double bytes = 32768.0 + 256.0 * bn / nc;
      const double issue = 4.0 * (64 / cb) * 120.0;
      const double step = std::max({6.0 * bn, bytes / 57.0, issue}) + (nc == 2 ? 150.0 : 100.0);
      const double cost = waves * step;
      if (cost < best - 1e-9) {
        best = cost;
        *bn_out = bn;
        *nc_out = nc;
      }
    }
  }
}

// Column tile of the cp.async kernel: persistent CTAs stream tiles, so the
// cost model is the number of tile waves times the per-tile column work.
int pick_bn(int64_t M, int ncol) {
  static const int cands[] = {32, 64, 128, 192, 256};
  const int64_t mt = ceil_div(M, kBM);
  int best = 256;
  double best_cost = 1e30;
  for (int bn : cands) {
    if (bn >= 2 * ncol && bn > 32) continue;
    const int64_t tiles = mt * ceil_div(ncol, bn);
    const double waves = double(tiles) / kNumSMs;
    const double cost = std::max(1.0, std::ceil(waves * 4.0) / 4.0) * (bn + 24.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

struct Gemm {
  int OH, OW, u, v, pad_h, pad_w;  // gather: ih = oh*u - pad_h + dh over the packed input
  PackGeom pg;
  int out_mode, o_u, o_v, o_H, o_W, o_ph, o_pw;
  int tma;                         // 1: TMA im2col kernel, 0: cp.async gather kernel
};

// TMA bounding box of one spatial dim: lower = -pad, upper such that the
// traversal visits exactly `out` window origins with the given stride.
inline void tma_corners(int in, int out, int stride, int pad, int* lower, int* upper) {
  *lower = -pad;
  *upper = (out - 1) * stride + 1 - pad - in;
}

bool tma_geometry_ok(const Gemm& g, int IH, int IW, int taps_h, int taps_w, int64_t M) {
  if (g.u < 1 || g.v < 1 || g.u > 8 || g.v > 8) return false;
  if (taps_h > 128 || taps_w > 128 || M >= (int64_t(1) << 31)) return false;
  int lh, uh, lw, uw;
  tma_corners(IH, g.OH, g.u, g.pad_h, &lh, &uh);
  tma_corners(IW, g.OW, g.v, g.pad_w, &lw, &uw);
  for (int c : {lh, uh, lw, uw})
    if (c < -128 || c > 127) return false;
  return true;
}

// TMA channel block per im2col load: the widest of 64/32/16 whose padding of
// Cp stays <= 1/3 (wider rows = fewer TMA pixel requests; the TMA engine
// handles ~1 im2col pixel row per 2.5 cycles whatever its width).
// 3xTF32 (es = 4): 32-channel blocks only (128-byte rows; the instantiated
// tf32 kernels), Cp padded up to them by out-of-bounds zero fill.
int pick_cb(int Cp, int es = 2) {
  if (es == 4) return 32;
  for (int cb : {64, 32, 16})
    if (ceil_div(Cp, cb) * cb * 3 <= int64_t(Cp) * 4) return cb;
  return 16;
}

// Reduction segments.  tcgen05's fp32 accumulation truncates, so the error
// of one TMEM accumulator grows linearly with its reduction length (measured
// ~4e-5 of max|y| at 10k products); reductions longer than kMaxChain run as
// several launches over k-block ranges, chained through the output with
// IEEE fp32 adds in the epilogue (beta = 1 after the first), which keeps
// every shape at the north_star 1e-4 bar.
int reduction_segments(int nkb, int depth) {
  int64_t chain = 8192;
  if (const char* e = ::dnnp::tune_env("DNNP_TC_CHAIN")) chain = std::max<int64_t>(atoll(e), depth);
  const int per = int(std::max<int64_t>(1, chain / depth));
  return std::max(1, (nkb + per - 1) / per);
}

// es: bytes per packed element of the planes a_hi / a_lo (2 = BF16x3, 4 =
// 3xTF32; the tf32 split runs on the TMA kernel only).
cudaError_t run_gemm(const ConvProblem& p, Gemm g, const void* a_hi, const void* a_lo, int IH,
                     int IW, int Cp, const float* f, float* out, const View4& ov, float alpha,
                     float beta, const EpiOp& epi, cudaStream_t st, int es) {
  const bool fused = epi.act >= 0 || epi.gate >= 0 || epi.bias != nullptr;
  if (fused && !g.tma) return cudaErrorNotSupported;  // caller runs the unfused sequence
  if (es == 4 && !g.tma) return cudaErrorNotSupported;  // caller runs SIMT fp32
  PackGeom& pg = g.pg;
  const int CB = g.tma ? pick_cb(Cp, es) : 8;
  const int Cpf = int(ceil_div(Cp, CB) * CB);  // filter columns per tap (channel blocks padded)
  pg.Cgrp = Cpf / 8;
  const int taps = pg.tapH * pg.tapW;
  pg.KC = taps * pg.Cgrp;
  const int depth = g.tma ? 128 / es : kBK;  // one stage = 128 bytes of reduction per row
  const int nkb = int(ceil_div(int64_t(pg.KC) * 8, depth));
  pg.Ktot = std::max(1, nkb) * depth;
  const int64_t M = p.N * g.OH * g.OW;
  int bn = pick_bn(M, pg.Ncol), nc = 1;
  if (g.tma) pick_tile_tma(M, pg.Ncol, CB, &bn, &nc);
  if (g.tma) {
    // A/B overrides, accepted only for the instantiated tile shapes
    if (const char* e = ::dnnp::tune_env("DNNP_TC_NC")) {
      const int v = atoi(e);
      if (v == 1 || v == 2) nc = v;
    }
    if (const char* e = ::dnnp::tune_env("DNNP_TC_BN")) {
      const int v = atoi(e);
      if (v == 64 || v == 128 || v == 192 || v == 256) bn = v;
    }
  }
  pg.Np = int(ceil_div(pg.Ncol, bn) * bn);
  const size_t flt = size_t(pg.Np) * pg.Ktot;
  Workspace ws(st);
  cudaError_t e = ws.alloc(flt * 2 * es + size_t(pg.KC + pg.Np + 2) * 4 + 256);
  if (e != cudaSuccess) return e;
  void* b_hi = ws.p;
  void* b_lo = static_cast<char*>(ws.p) + flt * es;
  auto* ctab = reinterpret_cast<uint32_t*>(static_cast<char*>(b_lo) + flt * es);
  auto* coltab = ctab + pg.KC + 1;
  const size_t frow = size_t(pg.C0) * pg.R0 * pg.S0 * sizeof(float);
  // (row-staged variant: opt-in, measured slower -- Np blocks are too few)
  if (!pg.dgrad && frow <= 48 * 1024 && ::dnnp::tune_env("DNNP_PACK_ROWS")) {
    if (es == 4)
      pack_filter_row_kernel<4><<<unsigned(pg.Np), 256, frow, st>>>(pg, f, b_hi, b_lo, ctab, coltab,
                                                                    taps);
    else
      pack_filter_row_kernel<2><<<unsigned(pg.Np), 256, frow, st>>>(pg, f, b_hi, b_lo, ctab, coltab,
                                                                    taps);
  } else if (::dnnp::tune_env("DNNP_PACK_TAP")) {
    // per-(tap, row) blocks (the round-1 kernel; A/B only)
    const dim3 fgrid(unsigned(taps + 1), unsigned(pg.Np));
    if (es == 4)
      pack_filter_tap_kernel<4><<<fgrid, 128, 0, st>>>(pg, f, b_hi, b_lo, ctab, coltab, taps);
    else
      pack_filter_tap_kernel<2><<<fgrid, 128, 0, st>>>(pg, f, b_hi, b_lo, ctab, coltab, taps);
  } else if (!::dnnp::tune_env("DNNP_PACK_SCATTER") || pg.bw > 1) {
    const int64_t total8 = int64_t(pg.Np) * (pg.Ktot / 8);
    if (total8 >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
    const unsigned fgrid = grid_for(std::max<int64_t>(total8, pg.KC), 256, 8);
    const MagicDiv dK8 = make_magic(uint32_t(pg.Ktot / 8)), dC8 = make_magic(uint32_t(pg.Cgrp));
    cudaLaunchConfig_t fc{};
    fc.gridDim = dim3(fgrid);
    fc.blockDim = dim3(256);
    fc.stream = st;
    cudaLaunchAttribute fa[1];
    unsigned nfa = 0;
    add_pdl_attr(fa, &nfa);
    fc.attrs = fa;
    fc.numAttrs = nfa;
    e = es == 4 ? cudaLaunchKernelEx(&fc, pack_filter_vec_kernel<4>, pg, f, b_hi, b_lo, ctab, coltab,
                                     taps, dK8, dC8)
                : cudaLaunchKernelEx(&fc, pack_filter_vec_kernel<2>, pg, f, b_hi, b_lo, ctab, coltab,
                                     taps, dK8, dC8);
    if (e != cudaSuccess) return e;
  } else {
    if (!tc::dry_run() && (e = cudaMemsetAsync(b_hi, 0, flt * 2 * es, st)) != cudaSuccess)
      return e;  // hi and lo planes
    const int64_t nf = int64_t(pg.K) * pg.C0 * pg.R0 * pg.S0;
    if (es == 4)
      pack_filter_scatter_kernel<4><<<grid_for(nf, 256, 8), 256, 0, st>>>(pg, f, b_hi, b_lo);
    else
      pack_filter_scatter_kernel<2><<<grid_for(nf, 256, 8), 256, 0, st>>>(pg, f, b_hi, b_lo);
    note_launch();
    pack_tables_kernel<<<grid_for(std::max(pg.KC, pg.Ncol), 256, 2), 256, 0, st>>>(pg, ctab, coltab,
                                                                                  g.tma ? 0 : 1);
    note_launch();
  }
  note_launch();
  const int64_t tiles = ceil_div(M, kBM * nc) * (pg.Np / bn);
  if (tiles >= (int64_t(1) << 31)) return cudaErrorInvalidValue;

  if (g.tma) {
    // ------------------------------------------------ TMA im2col kernel
    TmaParams prm{};
    Im2colGeom ig{};
    ig.N = p.N;
    ig.H = IH;
    ig.W = IW;
    ig.C = Cp;
    tma_corners(IH, g.OH, g.u, g.pad_h, &ig.lower_h, &ig.upper_h);
    tma_corners(IW, g.OW, g.v, g.pad_w, &ig.lower_w, &ig.upper_w);
    ig.stride_h = g.u;
    ig.stride_w = g.v;
    ig.cpp = CB;
    ig.ppc = kBM;
    const int rb = CB * es;  // sub-tile row bytes = swizzle span
    const CUtensorMapSwizzle sw = rb == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                             : CU_TENSOR_MAP_SWIZZLE_32B;
    if ((e = make_tmap_im2col(&prm.tm_ahi, a_hi, ig, sw, es)) != cudaSuccess) return e;
    if ((e = make_tmap_im2col(&prm.tm_alo, a_lo, ig, sw, es)) != cudaSuccess) return e;
    if ((e = make_tmap_2d(&prm.tm_bhi, b_hi, uint64_t(pg.Ktot), uint64_t(pg.Np), uint64_t(pg.Ktot),
                          uint32_t(CB), uint32_t(bn / nc), sw, es)) != cudaSuccess)
      return e;
    if ((e = make_tmap_2d(&prm.tm_blo, b_lo, uint64_t(pg.Ktot), uint64_t(pg.Np), uint64_t(pg.Ktot),
                          uint32_t(CB), uint32_t(bn / nc), sw, es)) != cudaSuccess)
      return e;
    prm.M = M;
    prm.Ncol = pg.Ncol;
    prm.lower_h = ig.lower_h;
    prm.lower_w = ig.lower_w;
    prm.u = g.u;
    prm.v = g.v;
    prm.nCB = Cpf / CB;
    prm.tapW = pg.tapW;
    prm.KCH = taps * prm.nCB;
    prm.nkb = nkb;
    prm.Cext = Cp;
    prm.nt = pg.Np / bn;
    prm.tiles = int(tiles);
    prm.out = out;
    prm.o_sn = ov.sn;
    prm.o_sc = ov.sc;
    prm.o_sh = ov.sh;
    prm.o_sw = ov.sw;
    prm.out_mode = g.out_mode;
    {
      const int64_t span = std::abs(ov.sc) * (ov.c + 1) + std::abs(ov.sh) * (g.o_u + 1) +
                           std::abs(ov.sw) * (g.o_v + 1);
      prm.off32 = span < (int64_t(1) << 31) ? 1 : 0;
    }
    prm.o_u = g.o_u;
    prm.o_v = g.o_v;
    prm.o_H = g.o_H;
    prm.o_W = g.o_W;
    prm.o_ph = g.o_ph;
    prm.o_pw = g.o_pw;
    prm.coltab = coltab;
    prm.alpha = alpha;
    prm.beta = beta;
    prm.plain = (alpha == 1.0f && beta == 0.0f && !fused) ? 1 : 0;
    prm.epi = epi;
    prm.dOHW = make_magic(uint32_t(g.OH * g.OW));
    prm.dOW = make_magic(uint32_t(g.OW));
    prm.skip = ::dnnp::diag_env("DNNP_TC_SKIP") ? atoi(::dnnp::diag_env("DNNP_TC_SKIP")) : 0;
    prm.prefetch = ::dnnp::diag_env("DNNP_TC_PREFETCH") ? atoi(::dnnp::diag_env("DNNP_TC_PREFETCH")) : 0;
    int nseg = reduction_segments(nkb, depth);
    // a gated sum spread over segments cannot also add the caller's dx
    if (epi.gate >= 0 && nseg > 1 && beta != 0.0f) return cudaErrorNotSupported;
    // stream-K over the last, partial wave of tiles
    Workspace skw(st);
    {
      int G = int(std::min<int64_t>(tiles, kNumSMs / nc));
      const int T = int(tiles);
      int W = T / G, R = T % G;
      // stream-K over a partial last wave: default when the reduction is long
      // enough (>= 32 k-blocks) to amortise the partial-tile fixup (measured:
      // conv3 bwd-data 88 -> 74 us, conv2 bwd-data 150 -> 144 us; neutral or
      // worse for short reductions, conv1 fwd 115 -> 121 us, tools/env_ab.py)
      const bool sk_want = ::dnnp::tune_env("DNNP_TC_SK") ? true : nkb >= 32;
      bool use_sk = nseg == 1 && sk_want && !::dnnp::tune_env("DNNP_TC_NO_SK") && W >= 1 && R > 0 &&
                    double(R) / G < 0.85 && int64_t(R) * nkb < (int64_t(1) << 30);
      // Split-K for grids under half a wave (small minibatches, SURVEY
      // configs[2]): every tile is cut along the reduction into pieces of
      // >= 4 k-blocks spread over up to all SMs; each piece's chain stays
      // under the accumulation cap, the finisher adds pieces in IEEE fp32.
      {
        const int Gmax = kNumSMs / nc, per_cap = std::max(1, 8192 / depth);
        if (!use_sk && !::dnnp::tune_env("DNNP_TC_NO_SPLIT") && T * 2 <= Gmax && nkb >= 8 &&
            int64_t(T) * nkb < (int64_t(1) << 30)) {
          int Gs = int(std::min<int64_t>(Gmax, int64_t(T) * (nkb / 4)));
          const int64_t U = int64_t(T) * nkb;
          if (ceil_div(U, int64_t(Gs)) > per_cap) Gs = int(std::min<int64_t>(Gmax, ceil_div(U, int64_t(per_cap))));
          if (Gs > T && ceil_div(U, int64_t(Gs)) <= per_cap) {
            G = Gs;
            W = 0;
            R = T;
            use_sk = true;
            nseg = 1;
          }
        }
      }
      prm.clusters = G;
      if (use_sk) {
        const int U = R * nkb, G2 = std::min(G, U);
        int maxp = 1;
        for (int tl = 0; tl < R; tl++) {
          const int first = sk_owner(tl * nkb, U, G2), last = sk_owner(tl * nkb + nkb - 1, U, G2);
          maxp = std::max(maxp, last - first + 1);
        }
        const size_t part_bytes = size_t(R) * nc * maxp * kBM * bn * sizeof(float);
        const size_t cnt_bytes = size_t(R) * nc * sizeof(int);
        if ((e = skw.alloc(part_bytes + cnt_bytes)) != cudaSuccess) return e;
        prm.skws = static_cast<float*>(skw.p);
        prm.skcnt = reinterpret_cast<int*>(static_cast<char*>(skw.p) + part_bytes);
        if (!tc::dry_run() && (e = cudaMemsetAsync(prm.skcnt, 0, cnt_bytes, st)) != cudaSuccess)
          return e;
        prm.sk = 1;
        prm.W = W;
        prm.U = U;
        prm.maxp = maxp;
      }
    }
    static unsigned long long* tbuf = nullptr;
    const bool want_trace = ::dnnp::diag_env("DNNP_TC_TRACE") != nullptr;
    if (want_trace && !tbuf) cudaMalloc(&tbuf, 8192 * sizeof(unsigned long long));
    if (want_trace) cudaMemsetAsync(tbuf, 0, 8192 * sizeof(unsigned long long), st);
    prm.trace = want_trace ? tbuf : nullptr;
    prm.nseg = nseg;
    prm.kb_lo = 0;
    {
      if (es == 4)  // 3xTF32: 32 tf32 channels = 128-byte rows
        e = nc == 2 ? launch_tma_bn<32, 2, 4>(bn, prm, st) : launch_tma_bn<32, 1, 4>(bn, prm, st);
      else if (nc == 2)
        e = CB == 64   ? launch_tma_bn<64, 2, 2>(bn, prm, st)
            : CB == 32 ? launch_tma_bn<32, 2, 2>(bn, prm, st)
                       : launch_tma_bn<16, 2, 2>(bn, prm, st);
      else
        e = CB == 64   ? launch_tma_bn<64, 1, 2>(bn, prm, st)
            : CB == 32 ? launch_tma_bn<32, 1, 2>(bn, prm, st)
                       : launch_tma_bn<16, 1, 2>(bn, prm, st);
    }
    if (want_trace) {
      static unsigned long long h[8192];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, tbuf, sizeof h, cudaMemcpyDeviceToHost);
      fprintf(stderr, "TMATRACE M=%lld ncol=%d bn=%d cb=%d nc=%d nkb=%d tiles=%d\n", (long long)M,
              pg.Ncol, bn, CB, nc, nkb, prm.tiles);
      const unsigned long long t0 = h[0];
      for (int i = 0; i < 1024 && h[i * 4]; i++)
        fprintf(stderr, "st %4d P[%8lld %8lld] M[%8lld %8lld]\n", i, (long long)(h[i * 4] - t0),
                (long long)(h[i * 4 + 1] - t0), (long long)(h[i * 4 + 2] - t0),
                (long long)(h[i * 4 + 3] - t0));
      for (int i = 0; i < 64 && h[4096 + i * 4]; i++)
        fprintf(stderr, "ep %2d [%8lld %8lld %8lld]\n", i, (long long)(h[4096 + i * 4] - t0),
                (long long)(h[4096 + i * 4 + 1] - t0), (long long)(h[4096 + i * 4 + 2] - t0));
    }
    return e;
  }

  // -------------------------------------------------- cp.async gather kernel
  TcParams prm{};
  prm.M = M;
  prm.Ncol = pg.Ncol;
  prm.OH = g.OH;
  prm.OW = g.OW;
  prm.IH = IH;
  prm.IW = IW;
  prm.Cp = Cp;
  prm.u = g.u;
  prm.v = g.v;
  prm.pad_h = g.pad_h;
  prm.pad_w = g.pad_w;
  prm.KC = pg.KC;
  prm.nkb = nkb;
  prm.Ktot = pg.Ktot;
  prm.nt = pg.Np / bn;
  prm.tiles = int(tiles);
  e = make_tmap_2d(&prm.tm_bhi, b_hi, uint64_t(pg.Ktot), uint64_t(pg.Np), uint64_t(pg.Ktot), kBK,
                   uint32_t(bn), CU_TENSOR_MAP_SWIZZLE_64B);
  if (e != cudaSuccess) return e;
  e = make_tmap_2d(&prm.tm_blo, b_lo, uint64_t(pg.Ktot), uint64_t(pg.Np), uint64_t(pg.Ktot), kBK,
                   uint32_t(bn), CU_TENSOR_MAP_SWIZZLE_64B);
  if (e != cudaSuccess) return e;
  prm.ctab = ctab;
  prm.a_hi = static_cast<const __nv_bfloat16*>(a_hi);
  prm.a_lo = static_cast<const __nv_bfloat16*>(a_lo);
  prm.b_hi = static_cast<const __nv_bfloat16*>(b_hi);
  prm.b_lo = static_cast<const __nv_bfloat16*>(b_lo);
  prm.out = out;
  prm.o_sn = ov.sn;
  prm.o_sc = ov.sc;
  prm.o_sh = ov.sh;
  prm.o_sw = ov.sw;
  prm.out_mode = g.out_mode;
  prm.o_u = g.o_u;
  prm.o_v = g.o_v;
  prm.o_H = g.o_H;
  prm.o_W = g.o_W;
  prm.coltab = coltab;
  prm.alpha = alpha;
  prm.beta = beta;
  prm.plain = (alpha == 1.0f && beta == 0.0f && nkb > 0) ? 1 : 0;
  static unsigned long long* trace_buf = nullptr;
  const bool want_trace = ::dnnp::diag_env("DNNP_TC_TRACE") != nullptr;
  if (want_trace && !trace_buf) cudaMalloc(&trace_buf, 8192 * sizeof(unsigned long long));
  if (want_trace) cudaMemsetAsync(trace_buf, 0, 8192 * sizeof(unsigned long long), st);
  prm.trace = want_trace ? trace_buf : nullptr;
  prm.skip = ::dnnp::diag_env("DNNP_TC_SKIP") ? atoi(::dnnp::diag_env("DNNP_TC_SKIP")) : 0;
  prm.products = ::dnnp::diag_env("DNNP_TC_PRODUCTS") ? atoi(::dnnp::diag_env("DNNP_TC_PRODUCTS")) : 3;
  prm.dOHW = make_magic(uint32_t(g.OH * g.OW));
  prm.dOW = make_magic(uint32_t(g.OW));
  const int nseg = reduction_segments(nkb, kBK);
  for (int sg = 0; sg < nseg && e == cudaSuccess; sg++) {
    prm.kb_lo = int(int64_t(nkb) * sg / nseg);
    prm.nkb = int(int64_t(nkb) * (sg + 1) / nseg);
    if (sg > 0) {
      prm.beta = 1.0f;
      prm.plain = 0;
    }
    switch (bn) {
      case 32: e = launch_gemm<32>(prm, st); break;
      case 64: e = launch_gemm<64>(prm, st); break;
      case 128: e = launch_gemm<128>(prm, st); break;
      case 192: e = launch_gemm<192>(prm, st); break;
      default: e = launch_gemm<256>(prm, st); break;
    }
  }
  if (want_trace) {
    static unsigned long long h[8192];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost);
    fprintf(stderr, "TRACE M=%lld ncol=%d bn=%d nkb=%d tiles=%d\n", (long long)M, pg.Ncol, bn, nkb,
            prm.tiles);
    const unsigned long long t0 = h[0];
    for (int i = 0; i < 256 && i < nkb * 3; i++)
      fprintf(stderr, "st %3d P[%7lld %7lld %7lld] M[%7lld %7lld fence %7lld kk0 %7lld commit %7lld]\n", i,
              (long long)(h[i * 8] - t0), (long long)(h[i * 8 + 1] - t0), (long long)(h[i * 8 + 2] - t0),
              (long long)(h[i * 8 + 3] - t0), (long long)(h[i * 8 + 4] - t0), (long long)(h[i * 8 + 6] - t0),
              (long long)(h[i * 8 + 7] - t0), (long long)(h[i * 8 + 5] - t0));
  }
  return e;
}

// ------------------------------------------------------------ halo kernel
template <int BN, int CB>
cudaError_t launch_halo(const HaloParams& prm, size_t smem, cudaStream_t st) {
  auto kern = conv_halo_kernel<BN, CB, 2>;
  // the attribute is per device; re-set only when the device or a larger size is asked for
  static int attr_dev = -1;
  static size_t attr_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaSuccess;
  if (attr_dev != dev || smem > attr_smem) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr_dev = dev;
    attr_smem = smem;
  }
  const int clusters = int(std::min<int64_t>(prm.tiles, kNumSMs / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(clusters * 2));
  cfg.blockDim = dim3(kHaloThreads);
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
  ktime_begin(st, 1);
  e = cudaLaunchKernelEx(&cfg, kern, prm);
  ktime_end(st);
  note_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Halo form of an unblocked stride-1 TMA geometry g (space-to-depth forward
// or backward-data): returns cudaErrorNotSupported when it does not apply
// (the caller then runs the im2col kernel).  Forward reads the packed input
// as produced (its grid already covers every tap: IH = OH + tapH - 1);
// backward-data packs dy with a zero border of (-lo_h, -lo_w).
cudaError_t run_halo(bool dgrad, const ConvProblem& p, const Gemm& g, const float* in,
                     const View4& inv, int IH, int IW, int Cp, const float* f, float* out,
                     const View4& ov, float alpha, float beta, const EpiOp& epi, cudaStream_t st,
                     int es) {
  const bool fused = epi.act >= 0 || epi.gate >= 0 || epi.bias != nullptr;
  const bool force = ::dnnp::tune_env("DNNP_TC_HALO") != nullptr;
  if (es != 2 || fused || !g.tma || g.u != 1 || g.v != 1 || ::dnnp::tune_env("DNNP_TC_NO_HALO") != nullptr)
    return cudaErrorNotSupported;
  PackGeom pg = g.pg;
  if (pg.Ncol > kHaloMaxCols || pg.bw != 1 || pg.bdir != 0 || Cp % 16 != 0) return cudaErrorNotSupported;
  const int tapH = pg.tapH, tapW = pg.tapW;
  const int top = g.pad_h, left = g.pad_w;  // zero border of the packed grid
  if (top < 0 || left < 0 || (!dgrad && (top || left))) return cudaErrorNotSupported;
  const int IHp = g.OH + tapH - 1, IWp = g.OW + tapW - 1;
  if (!dgrad && (IHp > IH || IWp > IW)) return cudaErrorNotSupported;
  const int IHg = dgrad ? IHp : IH, IWg = dgrad ? IWp : IW;  // packed grid
  const int RH = kBM + (tapH - 1) * IWg + (tapW - 1);
  if (RH > 256) return cudaErrorNotSupported;
  if (!force && double(g.OH) * g.OW < 0.8 * double(IHg) * IWg) return cudaErrorNotSupported;
  const int64_t Mflat = p.N * int64_t(IHg) * IWg;
  if (Mflat + 2 * kBM >= (int64_t(1) << 31)) return cudaErrorNotSupported;
  const int CB = Cp % 64 == 0 ? 64 : Cp % 32 == 0 ? 32 : 16;
  const int BN = pg.Ncol <= 48 ? 48 : 64;
  const int nCB = Cp / CB, taps = tapH * tapW, RB = CB * 2;
  const uint32_t arr = uint32_t(ceil_div(int64_t(RH) * RB, 1024) * 1024);
  const uint32_t b_bytes = uint32_t(taps * nCB * (BN + BN / 2) * RB);  // P + Q sub-tiles
  const uint32_t stage = uint32_t(nCB) * 2u * arr;
  const size_t budget = 227 * 1024 - 1024 /* alignment */ - 1024 /* barriers, column table */;
  if (b_bytes + 2 * size_t(stage) > budget) return cudaErrorNotSupported;
  const int stages = int(std::min<size_t>(4, (budget - b_bytes) / stage));
  const size_t smem = size_t(b_bytes) + size_t(stages) * stage + 2048;

  // filter planes [BN][Ktot] in the (tap, channel) order of the halo MMAs
  pg.Cgrp = Cp / 8;
  pg.KC = taps * pg.Cgrp;
  const int depth = 64;
  const int nkb = int(ceil_div(int64_t(pg.KC) * 8, depth));
  pg.Ktot = std::max(1, nkb) * depth;
  pg.Np = BN;
  const size_t flt = size_t(pg.Np) * pg.Ktot;
  const size_t act = size_t(Mflat) * Cp;
  Workspace ws(st);
  cudaError_t e = ws.alloc(flt * 4 + size_t(pg.KC + pg.Np + 2) * 4 + act * 4 + 512);
  if (e != cudaSuccess) return e;
  char* base = static_cast<char*>(ws.p);
  void* b_hi = base;
  void* b_lo = base + flt * 2;
  auto* ctab = reinterpret_cast<uint32_t*>(base + flt * 4);
  auto* coltab = ctab + pg.KC + 1;
  char* abase = base + ((flt * 4 + size_t(pg.KC + pg.Np + 2) * 4 + 255) & ~size_t(255));
  void* a_hi = abase;
  void* a_lo = abase + act * 2;
  pack_trigger_early(true);  // the filter pack next is independent of this pack (see run_tc)
  if (!dgrad)
    e = pack_act_s2d(inv, in, int(p.u), int(p.v), int(p.pad_h), int(p.pad_w), IH, IW, Cp, a_hi, a_lo,
                     st, es);
  else
    e = pack_act_border(inv, in, Cp, top, left, IHg, IWg, a_hi, a_lo, st, es);
  pack_trigger_early(false);
  if (e != cudaSuccess) return e;
  {
    const int64_t total8 = int64_t(pg.Np) * (pg.Ktot / 8);
    const unsigned fgrid = grid_for(std::max<int64_t>(total8, pg.KC), 256, 8);
    const MagicDiv dK8 = make_magic(uint32_t(pg.Ktot / 8)), dC8 = make_magic(uint32_t(pg.Cgrp));
    cudaLaunchConfig_t fc{};
    fc.gridDim = dim3(fgrid);
    fc.blockDim = dim3(256);
    fc.stream = st;
    cudaLaunchAttribute fa[1];
    unsigned nfa = 0;
    add_pdl_attr(fa, &nfa);
    fc.attrs = fa;
    fc.numAttrs = nfa;
    e = cudaLaunchKernelEx(&fc, pack_filter_vec_kernel<2>, pg, f, b_hi, b_lo, ctab, coltab, taps, dK8,
                           dC8);
    note_launch();
    if (e != cudaSuccess) return e;
  }
  HaloParams prm{};
  const CUtensorMapSwizzle sw = RB == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : RB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                           : CU_TENSOR_MAP_SWIZZLE_32B;
  if ((e = make_tmap_2d(&prm.tm_ahi, a_hi, uint64_t(Cp), uint64_t(Mflat), uint64_t(Cp), uint32_t(CB),
                        uint32_t(RH), sw, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_alo, a_lo, uint64_t(Cp), uint64_t(Mflat), uint64_t(Cp), uint32_t(CB),
                        uint32_t(RH), sw, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_bhi, b_hi, uint64_t(pg.Ktot), uint64_t(pg.Np), uint64_t(pg.Ktot),
                        uint32_t(CB), uint32_t(BN), sw, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_blo, b_lo, uint64_t(pg.Ktot), uint64_t(pg.Np), uint64_t(pg.Ktot),
                        uint32_t(CB), uint32_t(BN), sw, 2)) != cudaSuccess)
    return e;
  if ((e = make_tmap_2d(&prm.tm_bq, b_hi, uint64_t(pg.Ktot), uint64_t(pg.Np), uint64_t(pg.Ktot),
                        uint32_t(CB), uint32_t(BN / 2), sw, 2)) != cudaSuccess)
    return e;
  prm.Mflat = Mflat;
  prm.IWp = IWg;
  prm.tapH = tapH;
  prm.tapW = tapW;
  prm.nCB = nCB;
  prm.RH = RH;
  prm.OHv = g.OH;
  prm.OWv = g.OW;
  prm.Ncol = pg.Ncol;
  prm.tiles = int(ceil_div(Mflat, int64_t(2 * kBM)));
  prm.stages = stages;
  prm.arr_bytes = arr;
  prm.b_bytes = b_bytes;
  prm.dImg = make_magic(uint32_t(IHg * IWg));
  prm.dW = make_magic(uint32_t(IWg));
  prm.out = out;
  prm.o_sn = ov.sn;
  prm.o_sc = ov.sc;
  prm.o_sh = ov.sh;
  prm.o_sw = ov.sw;
  prm.out_mode = g.out_mode;
  prm.o_u = g.o_u;
  prm.o_v = g.o_v;
  prm.o_H = g.o_H;
  prm.o_W = g.o_W;
  prm.o_ph = g.o_ph;
  prm.o_pw = g.o_pw;
  prm.coltab = coltab;
  prm.alpha = alpha;
  prm.beta = beta;
  prm.plain = alpha == 1.0f && beta == 0.0f;
  {
    // coalesced super-pixel stores (conv1 backward-data geometry)
    const uintptr_t a = reinterpret_cast<uintptr_t>(out);
    prm.fast = (dgrad && g.out_mode == 1 && prm.plain && BN == 48 && pg.Ncol == 48 && p.C == 3 &&
                g.o_u == 4 && g.o_v == 4 && g.o_pw == 2 && ov.sw == 1 && a % 16 == 0 && ov.sn % 4 == 0 &&
                ov.sc % 4 == 0 && ov.sh % 4 == 0 && p.N < 65536 && !::dnnp::tune_env("DNNP_HALO_NO_FAST"))
                   ? 3
                   : 0;
  }
  // experiments (-DDNNP_DIAG builds): 1 = no loads after the first stages, 2 = no stores, 4 = no MMAs
  prm.dbg = ::dnnp::diag_env("DNNP_HALO_DBG") ? atoi(::dnnp::diag_env("DNNP_HALO_DBG")) : 0;
  if (BN == 48)
    return CB == 64 ? launch_halo<48, 64>(prm, smem, st)
           : CB == 32 ? launch_halo<48, 32>(prm, smem, st) : launch_halo<48, 16>(prm, smem, st);
  return CB == 64 ? launch_halo<64, 64>(prm, smem, st)
         : CB == 32 ? launch_halo<64, 32>(prm, smem, st) : launch_halo<64, 16>(prm, smem, st);
}

// super-pixel window of one spatial dim: offsets base(ph) - jr over all phases
void phase_window(int u, int pad, int R, int* lo, int* win) {
  int mn = 1 << 30, mx = -(1 << 30);
  for (int ph = 0; ph < u; ph++) {
    const int t0 = (ph + pad) % u;
    const int nR = t0 < R ? (R - t0 + u - 1) / u : 0;
    const int base = (ph + pad - t0) / u;
    for (int jr = 0; jr < nR; jr++) {
      mn = std::min(mn, base - jr);
      mx = std::max(mx, base - jr);
    }
  }
  if (mn > mx) mn = mx = 0;
  *lo = mn;
  *win = mx - mn + 1;
}

bool env_off(const char* name) { return ::dnnp::tune_env(name) != nullptr; }

cudaError_t run_tc(bool dgrad, const ConvProblem& p, const float* in, const View4& inv,
                   const float* f, float* out, const View4& outv, float alpha, float beta,
                   const EpiOp& epi, cudaStream_t st, int es) {
  pool_keep_memory();
  Gemm g{};
  PackGeom& pg = g.pg;
  pg.K = int(p.K);
  pg.C = int(p.C);
  pg.R = int(p.R);
  pg.S = int(p.S);
  pg.flip = p.flip ? 1 : 0;
  pg.dgrad = dgrad ? 1 : 0;
  pg.u = pg.v = 1;
  pg.su = pg.sv = 1;
  pg.C0 = int(p.C);
  pg.R0 = int(p.R);
  pg.S0 = int(p.S);
  const bool tma_on = !env_off("DNNP_TC_NO_TMA");
  // Space-to-depth for strided convolutions with few input channels (AlexNet
  // conv1: C=3, 11x11, stride 4): the u x v phases of the input become
  // channels, the problem becomes a stride-1 conv with ceil(R/u) x ceil(S/v)
  // taps over u*v*C channels, so the MMA reduction is not 62% zero padding.
  const bool s2d = tma_on && !env_off("DNNP_TC_NO_S2D") && (p.u > 1 || p.v > 1) && p.u <= 8 &&
                   p.v <= 8 && p.C * p.u * p.v <= 64;
  int IH, IW, Cp;
  int64_t Nimg = p.N;
  bool fold = !dgrad && tma_on && fold_taps(p.C, p.S, p.u, p.v, s2d);
  if (fold) {
    // horizontal taps folded into channels: R x 1 over S*C channels (kept
    // only when the im2col map accepts the geometry)
    Gemm gf = g;
    PackGeom& pf = gf.pg;
    pf.su = 1;
    pf.sv = int(p.S);
    pf.C = int(p.S * p.C);
    pf.S = 1;
    gf.tma = 1;
    gf.OH = int(p.P);
    gf.OW = int(p.Q);
    gf.u = int(p.u);
    gf.v = 1;
    gf.pad_h = int(p.pad_h);
    gf.pad_w = 0;
    pf.Ncol = int(p.K);
    gf.out_mode = 0;
    if (tma_geometry_ok(gf, int(p.H), int(p.Q), pf.R, 1, Nimg * gf.OH * gf.OW)) {
      g = gf;
      IH = int(p.H);
      IW = int(p.Q);
      Cp = int(ceil_div(pg.C, 16) * 16);
    } else {
      fold = false;
    }
  }
  if (fold) {
  } else if (s2d) {
    const int u = int(p.u), v = int(p.v);
    const int R2 = int(ceil_div(p.R, u)), S2 = int(ceil_div(p.S, v));
    int H2 = int(p.P) - 1 + R2, W2 = int(p.Q) - 1 + S2;
    if (dgrad) {
      H2 = std::max<int>(H2, int(ceil_div(p.H + p.pad_h, u)));
      W2 = std::max<int>(W2, int(ceil_div(p.W + p.pad_w, v)));
    }
    pg.su = u;
    pg.sv = v;
    pg.C = u * v * int(p.C);
    pg.R = R2;
    pg.S = S2;
    g.tma = 1;
    if (!dgrad) {
      IH = H2;
      IW = W2;
      Cp = int(ceil_div(pg.C, 16) * 16);
      g.OH = int(p.P);
      g.OW = int(p.Q);
      g.u = g.v = 1;
      g.pad_h = g.pad_w = 0;
      pg.Ncol = int(p.K);
      g.out_mode = 0;
    } else {
      IH = int(p.P);
      IW = int(p.Q);
      Cp = int(ceil_div(p.K, 16) * 16);
      pg.pad_h = pg.pad_w = 0;
      phase_window(1, 0, R2, &pg.lo_h, &pg.winH);
      phase_window(1, 0, S2, &pg.lo_w, &pg.winW);
      g.OH = H2;
      g.OW = W2;
      g.u = g.v = 1;
      g.pad_h = -pg.lo_h;
      g.pad_w = -pg.lo_w;
      pg.Ncol = pg.C;
      g.out_mode = 1;
      g.o_u = u;
      g.o_v = v;
      g.o_H = int(p.H);
      g.o_W = int(p.W);
      g.o_ph = int(p.pad_h);
      g.o_pw = int(p.pad_w);
    }
    if (!tma_geometry_ok(g, IH, IW, dgrad ? pg.winH : pg.R, dgrad ? pg.winW : pg.S,
                         Nimg * g.OH * g.OW))
      return cudaErrorNotSupported;
  } else {
    IH = int(dgrad ? p.P : p.H);
    IW = int(dgrad ? p.Q : p.W);
    if (!dgrad) {
      g.OH = int(p.P);
      g.OW = int(p.Q);
      g.u = int(p.u);
      g.v = int(p.v);
      g.pad_h = int(p.pad_h);
      g.pad_w = int(p.pad_w);
      pg.Ncol = int(p.K);
      g.out_mode = 0;
    } else {
      pg.u = int(p.u);
      pg.v = int(p.v);
      pg.pad_h = int(p.pad_h);
      pg.pad_w = int(p.pad_w);
      phase_window(pg.u, pg.pad_h, pg.R, &pg.lo_h, &pg.winH);
      phase_window(pg.v, pg.pad_w, pg.S, &pg.lo_w, &pg.winW);
      g.OH = int(ceil_div(p.H, p.u));
      g.OW = int(ceil_div(p.W, p.v));
      g.u = g.v = 1;
      g.pad_h = -pg.lo_h;
      g.pad_w = -pg.lo_w;
      pg.Ncol = int(p.u * p.v * p.C);
      g.out_mode = (p.u == 1 && p.v == 1) ? 0 : 1;  // unit stride: column = channel
      g.o_u = int(p.u);
      g.o_v = int(p.v);
      g.o_H = int(p.H);
      g.o_W = int(p.W);
    }
    g.tma = tma_on && tma_geometry_ok(g, IH, IW, dgrad ? pg.winH : pg.R, dgrad ? pg.winW : pg.S,
                                      Nimg * g.OH * g.OW);
    const int Cin = int(dgrad ? p.K : p.C);
    Cp = int(ceil_div(Cin, g.tma ? 16 : 8) * (g.tma ? 16 : 8));
  }
  pg.tapH = dgrad ? pg.winH : pg.R;
  pg.tapW = dgrad ? pg.winW : pg.S;
  pg.Sg = pg.tapW;
  pg.Rg = pg.tapH;
  pg.bdir = 0;
  pg.bh = 1;
  pg.ustep = dgrad ? 1 : g.u;
  pg.bw = 1;
  pg.Ncol0 = pg.Ncol;
  pg.vstep = dgrad ? 1 : g.v;
  if (s2d) {
    // AlexNet conv1: halo tiles instead of one im2col box per tap
    const cudaError_t he = run_halo(dgrad, p, g, in, inv, IH, IW, Cp, f, out, outv, alpha, beta, epi,
                                    st, es);
    if (he != cudaErrorNotSupported) return he;
  }
  // Column blocking for small GEMM N (conv2 bwd-data C=64): one GEMM row computes bw = 2
  // adjacent output columns, doubling N; the A operand (im2col, the bulk of
  // the TMA traffic) shrinks to (S + v) / (2 S) of its bytes.
  // (measured: helps the unit-stride bwd-data of conv2, 233 -> 204 us; not the
  // space-to-depth conv1 passes, whose epilogue then dominates)
  // unit-stride bwd-data: rows of 2 outputs (coalesced epilogue; conv2
  // 144 -> 142 us), except very narrow outputs, which block up to 8 columns
  const bool dgrad_rows = dgrad && !s2d && g.out_mode == 0 && pg.Ncol > 16 &&
                          !env_off("DNNP_TC_DGRAD_COLS");
  const bool blockable =
      g.tma && !fold && !dgrad_rows && pg.Ncol <= 64 && !env_off("DNNP_TC_NO_BLOCK") &&
      (env_off("DNNP_TC_BLOCK_S2D") ? (!dgrad ? g.out_mode == 0 : (s2d || g.out_mode == 0))
                                    : (!s2d && g.out_mode == 0 && (env_off("DNNP_TC_BLOCK") || dgrad)));
  if (blockable) {
    // blocking factor: 2, or up to 8 (the im2col traversal stride limit) for
    // very narrow unit-stride bwd-data outputs (table2 layer1: C = 3), by the
    // useful fraction of the MMA work: (bw N / padded) * S / (S + bw - 1)
    int bw = 2;
    if (dgrad && !s2d && g.out_mode == 0 && !env_off("DNNP_TC_BW2")) {
      double best = -1.0;
      for (int b : {2, 4, 8}) {
        const int n = b * pg.Ncol;
        if (n > 256) break;
        const double pad = double(ceil_div(n, 64) * 64);
        const double sc = (n / pad) * double(pg.Sg) / double(pg.Sg + (b - 1) * pg.vstep);
        if (sc > best + 1e-9) {
          best = sc;
          bw = b;
        }
      }
    }
    Gemm gb = g;
    PackGeom& pb = gb.pg;
    pb.bw = bw;
    pb.Ncol = bw * pg.Ncol;
    pb.tapW = pg.tapW + (bw - 1) * pg.vstep;
    gb.OW = int(ceil_div(g.OW, bw));
    gb.v = g.v * bw;
    if (!dgrad) {
      gb.out_mode = 1;
      gb.o_u = 1;
      gb.o_v = bw;
      gb.o_H = g.OH;
      gb.o_W = g.OW;
      gb.o_ph = gb.o_pw = 0;
    } else if (s2d) {
      gb.o_v = g.o_v * bw;
    } else {
      gb.out_mode = 1;
      gb.o_u = 1;
      gb.o_v = bw;
      gb.o_H = int(p.H);
      gb.o_W = int(p.W);
      gb.o_ph = gb.o_pw = 0;
    }
    // very narrow unit-stride bwd-data (bw > 2): also 2 rows -> a 2 x bw
    // block (N = 2 bw C; table2 layer1, C = 3)
    if (dgrad && !s2d && bw > 2 && 2 * pb.Ncol <= 128 && !env_off("DNNP_TC_NO_2D")) {
      Gemm g2 = gb;
      PackGeom& p2 = g2.pg;
      p2.bdir = 2;
      p2.bh = 2;
      p2.Ncol = 2 * pb.Ncol;
      p2.tapH = pg.tapH + pg.ustep;
      g2.OH = int(ceil_div(g.OH, 2));
      g2.u = g.u * 2;
      g2.o_u = 2;
      if (tma_geometry_ok(g2, IH, IW, p2.tapH, p2.tapW, Nimg * g2.OH * g2.OW)) gb = g2;
    }
    if (tma_geometry_ok(gb, IH, IW, gb.pg.tapH, gb.pg.tapW, Nimg * gb.OH * gb.OW)) g = gb;
  } else if ((!dgrad || dgrad_rows) && g.tma && !fold && g.out_mode == 0 && pg.Ncol <= 64 &&
             !env_off("DNNP_TC_NO_VBLOCK")) {
    // Row blocking for narrow forward GEMMs (conv1: K = 64): one GEMM row
    // computes 2 vertically adjacent outputs, doubling N while the A bytes
    // per output drop to (R + u) / 2R; unlike column blocking the epilogue
    // stores stay contiguous (lanes = consecutive output columns).
    int bh = 2;
    if (const char* e = ::dnnp::tune_env("DNNP_TC_VBH")) bh = std::max(2, std::min(8, atoi(e)));
    Gemm gb = g;
    PackGeom& pb = gb.pg;
    pb.bdir = 1;
    pb.bw = bh;
    pb.Ncol = bh * pg.Ncol;
    pb.tapH = pg.tapH + (bh - 1) * pg.ustep;
    gb.OH = int(ceil_div(g.OH, bh));
    gb.u = g.u * bh;
    gb.out_mode = 1;
    gb.o_u = bh;
    gb.o_v = 1;
    gb.o_H = dgrad ? int(p.H) : g.OH;
    gb.o_W = dgrad ? int(p.W) : g.OW;
    gb.o_ph = gb.o_pw = 0;
    if (gb.u <= 8 && tma_geometry_ok(gb, IH, IW, pb.tapH, pb.tapW, Nimg * gb.OH * gb.OW)) g = gb;
  }
  if (es == 4 && !g.tma) return cudaErrorNotSupported;  // 3xTF32 runs on the TMA kernel only
  const size_t act = size_t(p.N) * IH * IW * Cp;
  Workspace ws(st);
  {
    // dy already packed by the fused backward entry (same view, width and split)
    const void *ph = nullptr, *pl = nullptr;
    if (dgrad && !fold && packed_get(in, inv, Cp, &ph, &pl, es))
      return run_gemm(p, g, ph, pl, IH, IW, Cp, f, out, outv, alpha, beta, epi, st, es);
  }
  cudaError_t e = ws.alloc(act * 2 * es + 256);
  if (e != cudaSuccess) return e;
  void* a_hi = ws.p;
  void* a_lo = static_cast<char*>(ws.p) + act * es;
  // the filter pack launched next (programmatic) is independent of this
  // pack: both run at once; the filter pack's last wait orders the GEMM
  pack_trigger_early(g.tma);
  if (fold)
    e = pack_act_fold(inv, in, int(p.S), int(p.v), int(p.pad_w), IW, Cp, a_hi, a_lo, st, es);
  else if (s2d && !dgrad)
    e = pack_act_s2d(inv, in, int(p.u), int(p.v), int(p.pad_h), int(p.pad_w), IH, IW, Cp, a_hi,
                     a_lo, st, es);
  else
    e = pack_act(inv, in, Cp, a_hi, a_lo, st, es);
  pack_trigger_early(false);
  if (e != cudaSuccess) return e;
  return run_gemm(p, g, a_hi, a_lo, IH, IW, Cp, f, out, outv, alpha, beta, epi, st, es);
}

}  // namespace
}  // namespace tc

// FWD / DGRAD / WGRAD eligibility of the tensor-core path.
bool tc_eligible(const ConvProblem& p, int pass) {
  if (p.R > 255 || p.S > 255 || p.C > 65535 || p.K > 65535) return false;
  const int64_t lim = int64_t(1) << 31;
  if (pass == 0) return p.N * p.P * p.Q < lim && ceil_div(p.C, 8) * 8 * p.R * p.S < (1 << 24);
  if (pass == 1) {
    if (p.u > 16 || p.v > 16 || p.u * p.v * p.C > 65535) return false;
    return p.N * p.H * p.W < lim &&
           ceil_div(p.K, 8) * 8 * (p.R + p.u) * (p.S + p.v) < (1 << 24);
  }
  if (pass == 2)
    return p.N * p.P * p.Q < lim && p.N * p.H * p.W < lim &&
           ceil_div(p.C, 8) * 8 * p.R * p.S < (1 << 24);
  return false;
}

static tc::EpiOp no_epi() { return tc::EpiOp{-1, -1, nullptr, 0, nullptr}; }

cudaError_t tc_forward(const ConvProblem& p, const float* x, const float* f, float* y,
                       double alpha, double beta, cudaStream_t st, int es) {
  return tc::run_tc(false, p, x, p.x, f, y, p.y, float(alpha), float(beta), no_epi(), st, es);
}

cudaError_t tc_backward_data(const ConvProblem& p, const float* dy, const float* f, float* dx,
                             bool acc, cudaStream_t st, int es) {
  return tc::run_tc(true, p, dy, p.y, f, dx, p.x, 1.0f, acc ? 1.0f : 0.0f, no_epi(), st, es);
}

// Fused forms; cudaErrorNotSupported (before any write to the output) when
// the geometry takes a kernel without the fused epilogue.
cudaError_t tc_forward_fused(const ConvProblem& p, const float* x, const float* f, float* y,
                             double alpha, double beta, const ConvEpilogue& ep, cudaStream_t st,
                             int es) {
  tc::EpiOp e = no_epi();
  e.act = ep.act;
  e.bias = static_cast<const float*>(ep.bias);
  e.bias_sc = ep.bias_stride;
  return tc::run_tc(false, p, x, p.x, f, y, p.y, float(alpha), float(beta), e, st, es);
}

cudaError_t tc_backward_data_fused(const ConvProblem& p, const float* dy, const float* f,
                                   float* dx, bool acc, const ConvEpilogue& ep, cudaStream_t st,
                                   int es) {
  tc::EpiOp e = no_epi();
  e.gate = ep.gate;
  e.gatep = static_cast<const float*>(ep.gatep);
  return tc::run_tc(true, p, dy, p.y, f, dx, p.x, 1.0f, acc ? 1.0f : 0.0f, e, st, es);
}

}  // namespace dnnp
