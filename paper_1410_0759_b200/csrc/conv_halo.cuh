// tcgen05 convolution over a HALO tile (forward and backward-data of
// stride-1 problems over a zero-bordered packed input; included by
// conv_tc.cu).  Used for the space-to-depth forms of AlexNet conv1 (forward:
// 3 x 3 taps over 48 channels; backward-data: 3 x 3 window over 64 dy
// channels), whose im2col kernel streams one TMA box per tap and is bound by
// the SM's L2 ingest (every x element re-read once per tap).
//
// The packed input [N][IHp][IWp][Cp] is read as a flat matrix of pixel rows;
// an output position is computed on the same flat grid (m = n*IHp*IWp +
// oh*IWp + ow, the few positions with oh >= OH or ow >= OW are discarded), so
// filter tap (th, tw) of output row m reads input row m + th*IWp + tw: a
// constant shift.  A CTA loads ONE halo of 128 + (tapH-1)*IWp + (tapW-1)
// consecutive rows per channel block (a single 2-D TMA box), and the A
// operand of every tap is the 128-row window starting at that shift --
// addressed by the UMMA descriptor start address alone (a K-major swizzled
// operand may start at any row: the swizzle is a function of the absolute
// shared-memory address; tools/probe_halo.cu, every row offset, SW128 / 64 /
// 32).  The filter (<= 64 columns) stays resident in shared memory for the
// whole persistent kernel.  Per tile the SM ingests the halo once instead of
// taps x 128 rows.
//
// Warps: 0 = TMA producer (one elected lane), 1 .. kHaloIssuers = MMA issue
// (leader CTA of the pair; warp 1 also allocates TMEM), then 8 epilogue warps
// (TMEM lane quadrant warp % 4, two 32-column halves), which copy their
// accumulator chunk to registers and free the TMEM buffer before storing.  A 64-column tile's MMA (M = 256, N <= 64,
// K = 16) runs ~32 cycles, about what one warp needs to build and issue it,
// so consecutive tiles go to different issuer warps, each with its own TMEM
// accumulator; the tensor pipe interleaves their MMAs.  Halo stages are
// ring-buffered.
#pragma once

constexpr int kHaloIssuers = 2;
constexpr int kHaloEpi0 = 1 + kHaloIssuers;  // first epilogue warp
constexpr int kHaloThreads = (kHaloEpi0 + 8) * 32;
constexpr int kHaloMaxCols = 64;

struct HaloParams {
  CUtensorMap tm_ahi;   // packed input planes as [rows][Cp], box {CB, RH}
  CUtensorMap tm_alo;
  CUtensorMap tm_bhi;   // packed filter planes [Np][Ktot], box {CB, BN}
  CUtensorMap tm_blo;
  CUtensorMap tm_bq;    // hi plane, box {CB, BN / 2}
  int64_t Mflat;        // N * IHp * IWp
  int IWp, tapH, tapW, nCB, RH;
  int OHv, OWv;         // valid output extent of one image's flat grid
  int Ncol;
  int tiles;            // ceil(Mflat / (128 * NC))
  int stages;
  uint32_t arr_bytes;   // one (channel block, plane) halo array, 1024-aligned
  uint32_t b_bytes;     // resident filter (both planes, every tap and block)
  MagicDiv dImg, dW;    // IHp * IWp, IWp
  float* out;
  int64_t o_sn, o_sc, o_sh, o_sw;
  int out_mode;         // 0: column = channel; 1: column table (ph, pw, c)
  int o_u, o_v, o_H, o_W, o_ph, o_pw;
  const uint32_t* coltab;
  float alpha, beta;
  int plain;
  int fast;  // 3: super-pixel dx rows of a stride-4, pad-2, 3-channel backward-data (see epilogue)
  int dbg;  // experiments only (DNNP_HALO_DBG, -DDNNP_DIAG builds)
};

template <int BN, int CB, int NC>
__global__ void __launch_bounds__(kHaloThreads, 1) conv_halo_kernel(const __grid_constant__ HaloParams P) {
  constexpr int RB = CB * 2;     // bytes of one operand row (= swizzle span)
  constexpr int KPS = RB / 32;   // 16-deep k-steps per row
  // Resident filter, per (tap, channel block) kc: a P sub-tile of BN rows
  // (leader: W_hi, peer: W_lo) and a Q sub-tile of BN/2 rows (W_hi rows
  // [rank * BN/2, +BN/2)).  Per 16-deep k-step the BF16x3 split is two MMAs:
  //   A_hi x [W_hi | W_lo]  (N = 2 BN: hi.hi -> cols [0, BN), hi.lo -> [BN, 2 BN))
  //   A_lo x W_hi           (N = BN, accumulated onto cols [0, BN))
  // and the epilogue adds the two column halves -- 11 KB of operand reads
  // per SM and k-step instead of 15 KB for three MMAs (with N <= 64 the
  // MMAs are bound by shared-memory operand reads, not by the tensor pipe).
  static_assert(NC == 2, "the split across the pair needs both CTAs");
  constexpr uint32_t P_SUB = BN * RB, Q_SUB = (BN / 2) * RB, KC_BYTES = P_SUB + Q_SUB;
  constexpr int NI = kHaloIssuers;
  constexpr int ACC = 2 * BN;  // accumulator columns per buffer
  constexpr int TMEM_COLS = NI * ACC <= 128 ? 128 : (NI * ACC <= 256 ? 256 : 512);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int S = P.stages;
  const uint32_t stage_bytes = uint32_t(P.nCB) * 2u * P.arr_bytes;
  uint8_t* bar_base = smem + P.b_bytes + uint32_t(S) * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_base);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + NI;
  uint64_t* bfull = tempty + NI;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  long long* col_off = reinterpret_cast<long long*>(bar_base + 256);
  int* col_hw = reinterpret_cast<int*>(col_off + kHaloMaxCols);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = NC == 2 ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int cid = int(blockIdx.x) / NC, ncl = int(gridDim.x) / NC;
  const int taps = P.tapH * P.tapW;

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < S; s++) {
        ptx::mbar_init(&full[s], NC);
        ptx::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < NI; b++) {
        ptx::mbar_init(&tfull[b], 1);
        ptx::mbar_init(&tempty[b], 8 * NC);  // one arrival per epilogue warp of each CTA
      }
      ptx::mbar_init(bfull, NC);
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc_g<TMEM_COLS, NC>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (NC == 2) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t smem0 = ptx::smem_u32(smem);
  const uint32_t sb0 = smem0;                // resident filter: sub-tile (kc, plane)
  const uint32_t sa0 = smem0 + P.b_bytes;    // halo stages: (stage, cb, plane)
  pdl_wait();  // the packs (launched before) must be visible from here on

  if (warp == 0) {
    // ================================================ TMA producer
    if (lane == 0) {
      ptx::tma_prefetch(&P.tm_ahi);
      ptx::tma_prefetch(&P.tm_alo);
      ptx::tma_prefetch(&P.tm_bhi);
      ptx::tma_prefetch(&P.tm_blo);
      ptx::tma_prefetch(&P.tm_bq);
      // resident filter: every (tap, channel block) sub-tile of this CTA's rows
      if (leader) ptx::mbar_arrive_expect_tx(bfull, P.b_bytes * NC);
      else ptx::mbar_arrive_cluster(bfull, 0);
      {
        const uint32_t bar = NC == 2 ? ptx::leader_addr(bfull) : ptx::smem_u32(bfull);
        const int kcs = taps * P.nCB;
        for (int kc = 0; kc < kcs; kc++) {
          const uint32_t d = sb0 + uint32_t(kc) * KC_BYTES;
          ptx::tma_load_2d_pair(d, leader ? &P.tm_bhi : &P.tm_blo, kc * CB, 0, bar);
          ptx::tma_load_2d_pair(d + P_SUB, &P.tm_bq, kc * CB, int(rank) * (BN / 2), bar);
        }
      }
      const uint32_t tx = uint32_t(P.nCB) * 2u * uint32_t(P.RH) * RB;
      int it = 0;
      for (int tile = cid; tile < P.tiles; tile += ncl, it++) {
        const int s = it % S;
        if (it >= S) ptx::mbar_wait(&empty[s], ((it / S) - 1) & 1);
        const bool noload = (P.dbg & 1) && it >= S;
        if (leader) ptx::mbar_arrive_expect_tx(&full[s], noload ? 0u : tx * NC);
        else ptx::mbar_arrive_cluster(&full[s], 0);
        if (noload) continue;
        const uint32_t bar = NC == 2 ? ptx::leader_addr(&full[s]) : ptx::smem_u32(&full[s]);
        const int row0 = tile * (kBM * NC) + int(rank) * kBM;
        for (int cb = 0; cb < P.nCB; cb++) {
          const uint32_t d = sa0 + uint32_t(s) * stage_bytes + uint32_t(cb) * 2u * P.arr_bytes;
          if constexpr (NC == 2) {
            ptx::tma_load_2d_pair(d, &P.tm_ahi, cb * CB, row0, bar);
            ptx::tma_load_2d_pair(d + P.arr_bytes, &P.tm_alo, cb * CB, row0, bar);
          } else {
            ptx::tma_load_2d(d, &P.tm_ahi, cb * CB, row0, &full[s]);
            ptx::tma_load_2d(d + P.arr_bytes, &P.tm_alo, cb * CB, row0, &full[s]);
          }
        }
      }
    }
  } else if (warp <= NI) {
    // ================================================ MMA issuers (leader CTA)
    // issuer mi takes the tiles it = mi, mi + NI, ... into TMEM buffer mi.
    // Descriptors: one per operand base, then start-address increments
    // (the 14-bit address field cannot carry: shared memory < 256 KB).
    const int mi = warp - 1;
    if (leader) {
      constexpr uint32_t idesc2 = ptx::idesc_bf16(kBM * NC, 2 * BN, 0, 0);
      constexpr uint32_t idesc1 = ptx::idesc_bf16(kBM * NC, BN, 0, 0);
      ptx::mbar_wait(bfull, 0);
      ptx::tc_fence_after();
      const uint64_t dB0 = tma_kdesc<RB>(sb0), dA0 = tma_kdesc<RB>(sa0);
      const uint32_t arr16 = P.arr_bytes >> 4;
      const uint32_t dacc = tmem_base + uint32_t(mi * ACC);
      int it = mi, use = 0;
      for (int tile = cid + mi * ncl; tile < P.tiles; tile += NI * ncl, it += NI, use++) {
        ptx::mbar_wait(&tempty[mi], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const int s = it % S;
        ptx::mbar_wait_spin(&full[s], (it / S) & 1);
        ptx::tc_fence_after();
        const uint64_t dAs = dA0 + ((uint32_t(s) * stage_bytes) >> 4);
        uint32_t acc = 0;
        int kc = 0;
        for (int th = 0; th < P.tapH; th++) {
          for (int tw = 0; tw < P.tapW; tw++) {
            // this tap's A window: the halo shifted by th rows of IWp pixels + tw
            const uint64_t dAt = dAs + ((uint32_t(th * P.IWp + tw) * RB) >> 4);
            for (int cb = 0; cb < P.nCB; cb++, kc++) {
              const uint64_t ah = dAt + uint32_t(cb) * 2u * arr16;
              const uint64_t bp = dB0 + ((uint32_t(kc) * KC_BYTES) >> 4);
#pragma unroll
              for (int kk = 0; kk < KPS; kk++) {
                const uint64_t dah = ah + 2u * kk, dal = dah + arr16;
                const uint64_t dbp = bp + 2u * kk, dbq = dbp + (P_SUB >> 4);
                if (!(P.dbg & 4)) {
                  ptx::mma_split_elect<NC, 2>(dacc, dah, dbp, idesc2, acc);  // hi.hi | hi.lo
                  ptx::mma_split_elect<NC, 2>(dacc, dal, dbq, idesc1, 1);    // + lo.hi
                }
                acc = 1;
              }
            }
          }
        }
        if constexpr (NC == 2) {
          ptx::mma_commit_pair_elect(&empty[s]);
          ptx::mma_commit_pair_elect(&tfull[mi]);
        } else {
          ptx::mma_commit_elect(&empty[s]);
          ptx::mma_commit_elect(&tfull[mi]);
        }
      }
    }
  } else {
    // ================================================ epilogue
    const int ew = warp & 3;                         // TMEM lane quadrant of this warp
    const int es = (warp - kHaloEpi0) >> 2;
    // this warp's columns: 32 per warp set; fast path: one half of the
    // (ph, pw, c) super-pixel columns each (ph 0-1 / 2-3, 24 columns)
    const int c0 = P.fast ? 24 * es : 32 * es;
    const int r = ew * 32 + lane;                    // tile row
    const int et = threadIdx.x - kHaloEpi0 * 32;     // 0..255
    if (P.out_mode == 1) {
      for (int c = et; c < P.Ncol; c += 256) {
        const uint32_t e = __ldg(P.coltab + c);
        const int ph = int(e >> 24), pw = int((e >> 16) & 255);
        col_off[c] = int64_t(e & 0xFFFF) * P.o_sc + int64_t(ph) * P.o_sh + int64_t(pw) * P.o_sw;
        col_hw[c] = (ph << 16) | pw;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    const int nv = min(32, P.Ncol - c0);
    int it = 0;
    for (int tile = cid; tile < P.tiles; tile += ncl, it++) {
      const int buf = it % NI;
      const int64_t m = int64_t(tile) * (kBM * NC) + int64_t(rank) * kBM + r;
      uint32_t img = 0, oh = 0, ow = 0;
      bool ok = m < P.Mflat && nv > 0;
      if (ok) {
        uint32_t rem;
        mdivmod(uint32_t(m), P.dImg, img, rem);
        mdivmod(rem, P.dW, oh, ow);
        ok = int(oh) < P.OHv && int(ow) < P.OWv;
      }
      ptx::mbar_wait(&tfull[buf], (it / NI) & 1);
      ptx::tc_fence_after();
      uint32_t v[32];
      if (c0 < BN) {
        uint32_t w[32];
        const uint32_t ta = tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(buf * ACC + c0);
        ptx::tmem_ld32(ta, v);
        ptx::tmem_ld32(ta + BN, w);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = __float_as_uint(__fadd_rn(__uint_as_float(v[i]), __uint_as_float(w[i])));
      }
      // the accumulator is in registers: hand the buffer back to the MMA
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (NC == 1) ptx::mbar_arrive(&tempty[buf]);
        else ptx::mbar_arrive_cluster(&tempty[buf], 0);
      }
      if (P.fast == 3 && !(P.dbg & 2)) {
        // dx rows of super-pixels (u = v = 4, pad 2, C = 3, plain store):
        // super-pixel j covers w = 4j - 2 .. 4j + 1, so the aligned float4 at
        // w = 4j is (pw 2, 3 of j | pw 0, 1 of j + 1): one shuffle pair per
        // row segment and contiguous 512-byte warp stores instead of 12
        // scattered 4-byte stores per lane.
        const int hb = int(oh) * 4 - P.o_ph, wj = int(ow) * 4;
        const uint32_t key = ok ? img * 65536u + oh : 0xFFFFFFFFu;
        const uint32_t nkey = __shfl_down_sync(0xFFFFFFFFu, key, 1);
        const int nw = __shfl_down_sync(0xFFFFFFFFu, int(ow), 1);
        const bool cnext = lane < 31 && ok && nkey == key && nw == int(ow) + 1 && wj + 3 < P.o_W;
        const bool cprev = __shfl_up_sync(0xFFFFFFFFu, cnext, 1) && lane > 0;
#pragma unroll
        for (int php = 0; php < 2; php++) {
          const int h = hb + 2 * es + php;
          const bool hok = ok && unsigned(h) < unsigned(P.o_H);
#pragma unroll
          for (int c = 0; c < 3; c++) {
            const float x0 = __uint_as_float(v[(php * 4 + 0) * 3 + c]);
            const float x1 = __uint_as_float(v[(php * 4 + 1) * 3 + c]);
            const float x2 = __uint_as_float(v[(php * 4 + 2) * 3 + c]);
            const float x3 = __uint_as_float(v[(php * 4 + 3) * 3 + c]);
            const float n0 = __shfl_down_sync(0xFFFFFFFFu, x0, 1);
            const float n1 = __shfl_down_sync(0xFFFFFFFFu, x1, 1);
            if (!hok) continue;
            float* d = P.out + int64_t(img) * P.o_sn + int64_t(c) * P.o_sc + int64_t(h) * P.o_sh + wj;
            if (cnext) {
              *reinterpret_cast<float4*>(d) = make_float4(x2, x3, n0, n1);
            } else {
              if (wj < P.o_W) d[0] = x2;
              if (wj + 1 < P.o_W) d[1] = x3;
            }
            if (!cprev) {
              if (wj >= 2 && wj - 2 < P.o_W) d[-2] = x0;
              if (wj >= 1 && wj - 1 < P.o_W) d[-1] = x1;
            }
          }
        }
        continue;
      }
      if (!ok || (P.dbg & 2)) continue;
      if (P.out_mode == 0) {
        float* dst = P.out + int64_t(img) * P.o_sn + int64_t(oh) * P.o_sh + int64_t(ow) * P.o_sw +
                     int64_t(c0) * P.o_sc;
        if (P.plain) {
#pragma unroll
          for (int i = 0; i < 32; i++)
            if (i < nv) dst[int64_t(i) * P.o_sc] = __uint_as_float(v[i]);
        } else {
          store_cols(dst, P.o_sc, nv, v, P.beta != 0.0f, nullptr, 0, OpAxpby{P.alpha, P.beta});
        }
      } else {
        // column table: (ph, pw, c) of super-pixel (oh, ow)
        const int hb = int(oh) * P.o_u - P.o_ph, wb = int(ow) * P.o_v - P.o_pw;
        float* rb = P.out + int64_t(img) * P.o_sn + int64_t(hb) * P.o_sh + int64_t(wb) * P.o_sw;
#pragma unroll
        for (int i = 0; i < 32; i++) {
          if (i < nv) {
            const int hw = col_hw[c0 + i];
            if (unsigned(hb + (hw >> 16)) < unsigned(P.o_H) &&
                unsigned(wb + (hw & 0xFFFF)) < unsigned(P.o_W)) {
              float* d = rb + col_off[c0 + i];
              const float a = __uint_as_float(v[i]);
              *d = P.plain ? a
                           : (P.beta != 0.0f ? __fadd_rn(__fmul_rn(*d, P.beta), __fmul_rn(a, P.alpha))
                                             : __fmul_rn(a, P.alpha));
            }
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  if constexpr (NC == 2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_g<TMEM_COLS, NC>(tmem_base);
  }
}
