// tcgen05 backward-filter over a HALO of packed pixels (space-to-depth
// backward-filter of AlexNet conv1: 3 x 3 taps over 48 channels, 64 dy
// channels; included by wgrad_tc.cu).
//
// dW[(tap, c)][k] = sum_p x[p + shift(tap)][c] * dy[p][k] over the output
// pixels p, laid out on the packed input's flat grid (p = n*IH*IW + oh*IW +
// ow; dy is packed onto the same grid with zeros at the IW - Q, IH - P
// positions that are not output pixels, so they add nothing).  A cluster of
// two CTAs (tcgen05 cta_group::2, M = 256) owns a contiguous range of
// 128-pixel chunks (split-K; partial sums to the workspace, summed in split
// order by wgrad_reduce_tma).  Per chunk each CTA loads ONE halo of x rows
// (one 2-D TMA box per plane) and the chunk's dy; the A operand (x, MN-major:
// 64 channels per 128-byte pixel row, reduction = pixels) of a tap starts at
// the tap's pixel shift, and an M = 128 tile holds TWO taps -- the second
// 64-wide M block at LBO = (shift difference) x 128 bytes.  Any start row and
// LBO are legal (tools/probe_halo_mn.cu).  The descriptor is the pair's, so
// the peer CTA loads its halo one tap row (IW pixels) later: its two M blocks
// are the leader's taps one row down.  Taps: leader rows 0 and 2, peer rows 1
// (and 3, which does not exist: discarded) -> 3 pair-MMAs cover 9 taps.
//
// BF16x3 as two MMAs per 16-pixel k-step and tap pair:
//   A_hi x [dy_hi | dy_lo]   N = 128 (leader holds dy_hi, peer dy_lo)
//   A_lo x dy_hi             N = 64  (each CTA holds 32 rows of dy_hi)
// three accumulators of 128 columns in TMEM (384 of 512); the epilogue adds
// the column halves and writes the chunk range's partial [tap][c][k].
#pragma once

constexpr int kWhThreads = 6 * 32;  // TMA, MMA, 4 epilogue warps
constexpr int kWhChunk = 128;       // pixels per stage
constexpr int kWhMaxG = 3;          // tap-pair MMAs (accumulators of 128 columns)

struct WgHaloParams {
  CUtensorMap tm_xhi;   // packed x [rows][64], box {64, RH}
  CUtensorMap tm_xlo;
  CUtensorMap tm_dhi;   // dy [64 k][Pp pixels] (pixels contiguous), box {64, 64}
  CUtensorMap tm_dlo;
  CUtensorMap tm_dq;    // dy hi, box {64 pixels, 32 k}
  int chunks;           // Pp / 128
  int RH;               // halo rows
  int off1;             // peer halo offset (pixels) = IW
  int ng;               // tap-pair MMAs
  int sh[kWhMaxG][2];   // leader's pixel shifts of the two M blocks of pair g
  int tap[2][kWhMaxG][2];  // [rank][g][block]: tap index, -1 = discarded rows
  int Cpf;              // workspace columns per tap
  int ncolx;            // workspace rows per split = taps * Cpf
  uint32_t arr_bytes;   // one x halo plane, 1024-aligned
  float* ws;            // partials [cluster][ncolx][64]
};

__global__ void __launch_bounds__(kWhThreads, 1) wgrad_halo_kernel(const __grid_constant__ WgHaloParams P) {
  constexpr uint32_t P_SUB = 64 * 128;  // one 64-pixel block of 64 dy rows (K-major, 128B rows)
  constexpr uint32_t Q_SUB = 32 * 128;  // one 64-pixel block of 32 dy rows
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t stage_bytes = 2 * P.arr_bytes + 2 * P_SUB + 2 * Q_SUB;
  constexpr int S = 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = int(blockIdx.x) / 2, ncl = int(gridDim.x) / 2;
  const int c_lo = int(int64_t(P.chunks) * cid / ncl), c_hi = int(int64_t(P.chunks) * (cid + 1) / ncl);

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < S; s++) {
        ptx::mbar_init(&full[s], 2);
        ptx::mbar_init(&empty[s], 1);
      }
      ptx::mbar_init(done, 1);
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc_g<512, 2>(tmem_slot);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t smem0 = ptx::smem_u32(smem);
  pdl_wait();

  if (warp == 0) {
    // ================================================ TMA producer
    if (lane == 0) {
      ptx::tma_prefetch(&P.tm_xhi);
      ptx::tma_prefetch(&P.tm_xlo);
      ptx::tma_prefetch(&P.tm_dhi);
      ptx::tma_prefetch(&P.tm_dlo);
      ptx::tma_prefetch(&P.tm_dq);
      const uint32_t tx = stage_bytes - 2 * P.arr_bytes + 2u * uint32_t(P.RH) * 128u;
      int it = 0;
      for (int ch = c_lo; ch < c_hi; ch++, it++) {
        const int s = it % S;
        if (it >= S) ptx::mbar_wait(&empty[s], ((it / S) - 1) & 1);
        if (leader) ptx::mbar_arrive_expect_tx(&full[s], tx * 2);
        else ptx::mbar_arrive_cluster(&full[s], 0);
        const uint32_t bar = ptx::leader_addr(&full[s]);
        const uint32_t st0 = smem0 + uint32_t(s) * stage_bytes;
        const int p0 = ch * kWhChunk;
        const int xr = p0 + int(rank) * P.off1;
        ptx::tma_load_2d_pair(st0, &P.tm_xhi, 0, xr, bar);
        ptx::tma_load_2d_pair(st0 + P.arr_bytes, &P.tm_xlo, 0, xr, bar);
        const uint32_t dp = st0 + 2 * P.arr_bytes, dq = dp + 2 * P_SUB;
        for (int j = 0; j < 2; j++) {
          ptx::tma_load_2d_pair(dp + j * P_SUB, leader ? &P.tm_dhi : &P.tm_dlo, p0 + 64 * j, 0, bar);
          ptx::tma_load_2d_pair(dq + j * Q_SUB, &P.tm_dq, p0 + 64 * j, 32 * int(rank), bar);
        }
      }
    }
  } else if (warp == 1) {
    // ================================================ MMA issuer (leader CTA)
    if (leader) {
      // A MN-major (x: channels contiguous), B K-major (dy: pixels contiguous)
      constexpr uint32_t idesc2 = ptx::idesc_bf16(256, 128, 1, 0);
      constexpr uint32_t idesc1 = ptx::idesc_bf16(256, 64, 1, 0);
      // descriptors: built once, then start-address increments (16 pixel
      // rows = 2048 B per k-step for x; 32 B per k-step inside a dy row)
      uint64_t dxh[kWhMaxG];
      for (int g = 0; g < kWhMaxG; g++)
        dxh[g] = ptx::desc_mnmajor_sw128(smem0 + uint32_t(P.sh[g][0]) * 128u,
                                         uint32_t(P.sh[g][1] - P.sh[g][0]) * 128u, 1024);
      const uint64_t dP0 = ptx::desc_kmajor_sw128(smem0 + 2 * P.arr_bytes);
      const uint32_t arr16 = P.arr_bytes >> 4, stage16 = stage_bytes >> 4;
      uint32_t acc = 0;
      int it = 0;
      for (int ch = c_lo; ch < c_hi; ch++, it++) {
        const int s = it % S;
        ptx::mbar_wait_spin(&full[s], (it / S) & 1);
        ptx::tc_fence_after();
        const uint32_t so = uint32_t(s) * stage16;
#pragma unroll
        for (int kk = 0; kk < kWhChunk / 16; kk++) {
          const uint64_t dbp = dP0 + so + uint32_t(kk >> 2) * (P_SUB >> 4) + uint32_t(kk & 3) * 2u;
          const uint64_t dbq = dP0 + so + 2 * (P_SUB >> 4) + uint32_t(kk >> 2) * (Q_SUB >> 4) +
                               uint32_t(kk & 3) * 2u;
#pragma unroll
          for (int g = 0; g < kWhMaxG; g++) {
            if (g < P.ng) {
              const uint64_t dah = dxh[g] + so + uint32_t(kk) * 128u;
              const uint64_t dal = dah + arr16;
              const uint32_t dacc = tmem_base + uint32_t(g * 128);
              ptx::mma_split_elect<2, 2>(dacc, dah, dbp, idesc2, acc);  // hi.hi | hi.lo
              ptx::mma_split_elect<2, 2>(dacc, dal, dbq, idesc1, 1);    // + lo.hi
            }
          }
          acc = 1;
        }
        ptx::mma_commit_pair_elect(&empty[s]);
      }
      ptx::mma_commit_pair_elect(done);
    }
  } else {
    // ================================================ epilogue: partial sums
    const int ew = warp & 3;
    const int r = ew * 32 + lane;  // accumulator row: M block r / 64, channel r % 64
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    const bool any = c_hi > c_lo;
    for (int g = 0; g < P.ng; g++) {
      uint32_t v[64];
      const uint32_t ta = tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(g * 128);
      {
        uint32_t a[32], b[32];
        ptx::tmem_ld32(ta, a);
        ptx::tmem_ld32(ta + 64, b);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = __float_as_uint(__fadd_rn(__uint_as_float(a[i]), __uint_as_float(b[i])));
        ptx::tmem_ld32(ta + 32, a);
        ptx::tmem_ld32(ta + 96, b);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i++)
          v[32 + i] = __float_as_uint(__fadd_rn(__uint_as_float(a[i]), __uint_as_float(b[i])));
      }
      const int tp = P.tap[rank][g][r >> 6];
      if (tp < 0) continue;
      float4* dst = reinterpret_cast<float4*>(P.ws + (int64_t(cid) * P.ncolx + tp * P.Cpf + (r & 63)) * 64);
#pragma unroll
      for (int q = 0; q < 16; q++) {
        float4 o;
        o.x = any ? __uint_as_float(v[4 * q + 0]) : 0.0f;
        o.y = any ? __uint_as_float(v[4 * q + 1]) : 0.0f;
        o.z = any ? __uint_as_float(v[4 * q + 2]) : 0.0f;
        o.w = any ? __uint_as_float(v[4 * q + 3]) : 0.0f;
        dst[q] = o;
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_g<512, 2>(tmem_base);
  }
}

// dy [N][K][P][Q] (any strides) -> planes [K][Pp] over the packed input's
// flat pixel grid p = n*IH*IW + oh*IW + ow (zero where oh >= P, ow >= Q or
// p >= N*IH*IW), BF16 hi / lo.  A block covers 512 consecutive grid pixels x
// 8 k (two pixels per thread: 4-byte stores of both planes, coalesced loads
// along ow).
__global__ void __launch_bounds__(256) pack_dy_grid_kernel(View4 v, const float* __restrict__ dy,
                                                           int IH, int IW, int K, int64_t npix,
                                                           int64_t Pp, __nv_bfloat16* __restrict__ hi,
                                                           __nv_bfloat16* __restrict__ lo) {
  const int64_t p = (int64_t(blockIdx.x) * 256 + threadIdx.x) * 2;
  if (p >= Pp) return;
  int64_t off[2];
  bool in[2];
#pragma unroll
  for (int e = 0; e < 2; e++) {
    const int64_t pe = p + e;
    const int64_t n = pe / (int64_t(IH) * IW);
    const int rem = int(pe - n * IH * IW), oh = rem / IW, ow = rem - oh * IW;
    in[e] = pe < npix && oh < v.h && ow < v.w;
    off[e] = in[e] ? n * v.sn + int64_t(oh) * v.sh + int64_t(ow) * v.sw : 0;
  }
  const int k0 = blockIdx.y * 8, k1 = min(K, k0 + 8);
  for (int k = k0; k < k1; k++) {
    const float a = in[0] ? __ldg(dy + off[0] + int64_t(k) * v.sc) : 0.0f;
    const float b = in[1] ? __ldg(dy + off[1] + int64_t(k) * v.sc) : 0.0f;
    const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    const float2 hf = __bfloat1622float2(h2);
    *reinterpret_cast<__nv_bfloat162*>(hi + int64_t(k) * Pp + p) = h2;
    *reinterpret_cast<__nv_bfloat162*>(lo + int64_t(k) * Pp + p) = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  }
  pdl_trigger();
}
