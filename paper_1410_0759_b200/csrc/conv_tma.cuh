// tcgen05 implicit-GEMM convolution with the A operand gathered by TMA in
// im2col mode (forward and backward-data; included by conv_tc.cu).
//
// The packed input planes [N][IH][IW][Cp] (BF16 hi / lo) are described by
// two im2col tensor maps: one load = 128 consecutive output pixels (walking
// W -> H -> N inside the bounding box, zero fill at the image border) x CB
// channels of one filter tap, written 32B/64B-swizzled straight into the
// K-major A stage.  No producer warps: one thread streams A and B (the
// packed filter, tiled TMA) for every stage, so the gather costs no issue
// slots and no per-row address arithmetic (the cp.async kernel in conv_tc.cu
// spent ~500 cycles per stage there, more than the MMAs of the stage).
//
// Warps: 0 = TMA producer (one elected lane), 1 = TMEM allocation + MMA issue
// (warp-collective loop, elected issue), 2-5 = epilogue (TMEM lane quadrant
// warp % 4), double-buffered accumulator so the epilogue of tile i overlaps
// the main loop of tile i + 1.
#pragma once

constexpr int kTmaThreads = 6 * 32;

struct TmaParams {
  CUtensorMap tm_ahi;  // im2col maps of the packed input planes
  CUtensorMap tm_alo;
  CUtensorMap tm_bhi;  // packed filter [Np][Ktot], box {CB, BN}
  CUtensorMap tm_blo;
  int64_t M;           // GEMM rows = N * OH * OW
  int Ncol;            // valid GEMM columns
  int lower_h, lower_w, u, v;  // window origin of output pixel (oh, ow): lower + o * stride
  int nCB, tapW, KCH, nkb;     // channel blocks per tap, taps per window row, chunks, k-blocks
  int Cext;                    // channel extent of the A maps (OOB coordinate for padding chunks)
  int nt, tiles;
  float* out;
  int64_t o_sn, o_sc, o_sh, o_sw;
  int out_mode;                // 0: column = channel; 1: column table (ph, pw, c)
  int o_u, o_v, o_H, o_W, o_ph, o_pw;  // mode 1: h = oh * o_u + ph - o_ph
  const uint32_t* coltab;
  float alpha, beta;
  int plain;                   // alpha == 1, beta == 0: store the accumulator as is
  MagicDiv dOHW, dOW;
};

template <int BN, int CB>
struct TCfg {
  static constexpr int SUB = kBK / CB;       // chunks (sub-tiles) per stage
  static constexpr int A_SUB = kBM * CB * 2; // bytes of one A sub-tile (one plane)
  static constexpr int B_SUB = BN * CB * 2;
  static constexpr int A_BYTES = SUB * A_SUB;
  static constexpr int B_BYTES = SUB * B_SUB;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES =
      (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS =
      2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512));
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int CB>
__device__ __forceinline__ uint64_t tma_kdesc(uint32_t addr) {
  if constexpr (CB == 32) return ptx::desc_kmajor_sw64(addr);
  else return ptx::desc_kmajor_sw32(addr);
}

template <int BN, int CB>
__global__ void __launch_bounds__(kTmaThreads, 1) conv_tma_kernel(const __grid_constant__ TmaParams P) {
  using C = TCfg<BN, CB>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < S; s++) {
        ptx::mbar_init(&full[s], 1);   // producer's arrive.expect_tx; TMA completes the tx
        ptx::mbar_init(&empty[s], 1);  // MMA commit
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

  if (warp == 0) {
    // ================================================ TMA producer
    if (lane == 0) {
      ptx::tma_prefetch(&P.tm_ahi);
      ptx::tma_prefetch(&P.tm_alo);
      ptx::tma_prefetch(&P.tm_bhi);
      ptx::tma_prefetch(&P.tm_blo);
      int it = 0;
      for (int tile = blockIdx.x; tile < P.tiles; tile += gridDim.x) {
        const uint32_t m0 = uint32_t(tile / P.nt) * kBM;
        const int n0 = (tile % P.nt) * BN;
        uint32_t img, rem, oh, ow;
        mdivmod(m0, P.dOHW, img, rem);
        mdivmod(rem, P.dOW, oh, ow);
        const int h0 = P.lower_h + int(oh) * P.u, w0 = P.lower_w + int(ow) * P.v;
        int kc = 0, cb = 0, dh = 0, dw = 0;
        for (int kb = 0; kb < P.nkb; kb++, it++) {
          const int s = it % S;
          if (it >= S) ptx::mbar_wait(&empty[s], ((it / S) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          const uint32_t base = smem0 + s * C::STAGE_BYTES;
#pragma unroll
          for (int j = 0; j < C::SUB; j++, kc++) {
            const bool real = kc < P.KCH;
            const int c = real ? cb * CB : P.Cext;  // padding chunk: all-OOB box -> zeros
            const uint16_t ow16 = uint16_t(real ? dw : 0), oh16 = uint16_t(real ? dh : 0);
            ptx::tma_load_im2col(base + j * C::A_SUB, &P.tm_ahi, c, w0, h0, int(img), ow16, oh16,
                                 &full[s]);
            ptx::tma_load_im2col(base + C::A_BYTES + j * C::A_SUB, &P.tm_alo, c, w0, h0, int(img),
                                 ow16, oh16, &full[s]);
            ptx::tma_load_2d(base + 2 * C::A_BYTES + j * C::B_SUB, &P.tm_bhi, kc * CB, n0,
                             &full[s]);
            ptx::tma_load_2d(base + 2 * C::A_BYTES + C::B_BYTES + j * C::B_SUB, &P.tm_blo,
                             kc * CB, n0, &full[s]);
            if (++cb == P.nCB) {
              cb = 0;
              if (++dw == P.tapW) {
                dw = 0;
                ++dh;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================ MMA issuer
    constexpr uint32_t idesc = ptx::idesc_bf16(kBM, BN, 0, 0);
    int it = 0, lt = 0;
    for (int tile = blockIdx.x; tile < P.tiles; tile += gridDim.x, lt++) {
      const int buf = lt & 1;
      ptx::mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t dacc = tmem_base + uint32_t(buf * BN);
      uint32_t acc = 0;
      for (int kb = 0; kb < P.nkb; kb += 2) {
        const int npair = P.nkb - kb >= 2 ? 2 : 1;
        ptx::mbar_wait_spin(&full[it % S], (it / S) & 1);
        if (npair == 2) ptx::mbar_wait_spin(&full[(it + 1) % S], ((it + 1) / S) & 1);
        ptx::tc_fence_after();
        for (int q = 0; q < npair; q++, it++) {
          const int s = it % S;
          const uint32_t base = smem0 + s * C::STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; kk++) {
            // one 16-deep k-step: CB=32 -> +32 B inside the 64 B row; CB=16 -> next sub-tile
            const uint32_t ao = CB == 32 ? uint32_t(kk * 32) : uint32_t(kk * C::A_SUB);
            const uint32_t bo = CB == 32 ? uint32_t(kk * 32) : uint32_t(kk * C::B_SUB);
            const uint64_t dah = tma_kdesc<CB>(base + ao);
            const uint64_t dal = tma_kdesc<CB>(base + C::A_BYTES + ao);
            const uint64_t dbh = tma_kdesc<CB>(base + 2 * C::A_BYTES + bo);
            const uint64_t dbl = tma_kdesc<CB>(base + 2 * C::A_BYTES + C::B_BYTES + bo);
            ptx::mma_bf16_elect(dacc, dal, dbh, idesc, acc);
            ptx::mma_bf16_elect(dacc, dah, dbl, idesc, 1);
            ptx::mma_bf16_elect(dacc, dah, dbh, idesc, 1);
            acc = 1;
          }
          ptx::mma_commit_elect(&empty[s]);
        }
      }
      ptx::mma_commit_elect(&tfull[buf]);
    }
  } else {
    // ================================================ epilogue
    const int ew = warp & 3;  // TMEM lane quadrant accessible to this warp
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
      ptx::mbar_wait(&tfull[buf], (lt >> 1) & 1);
      ptx::tc_fence_after();
      const int64_t rowoff =
          P.out_mode == 0 ? int64_t(img) * P.o_sn + int64_t(oh) * P.o_sh + int64_t(ow) * P.o_sw
                          : int64_t(img) * P.o_sn;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        const int cbase = n0 + c0;
        if (cbase >= P.Ncol) break;  // warp-uniform: padded columns are never loaded
        uint32_t v[32];
        ptx::tmem_ld32(tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(buf * BN + c0), v);
        ptx::tmem_ld_wait();
        if (!row_ok) continue;
        if (P.out_mode == 0 && P.plain && cbase + 32 <= P.Ncol) {
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
              float val = __fmul_rn(__uint_as_float(v[i]), P.alpha);
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
              const int h = int(oh) * P.o_u + int(e >> 24) - P.o_ph;
              const int w = int(ow) * P.o_v + int((e >> 16) & 255) - P.o_pw;
              if (unsigned(h) < unsigned(P.o_H) && unsigned(w) < unsigned(P.o_W)) {
                float* dst = P.out + rowoff + int64_t(e & 0xFFFF) * P.o_sc + int64_t(h) * P.o_sh +
                             int64_t(w) * P.o_sw;
                float val = __fmul_rn(__uint_as_float(v[i]), P.alpha);
                if (P.beta != 0.0f) val = __fadd_rn(__fmul_rn(*dst, P.beta), val);
                *dst = val;
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[buf]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}
