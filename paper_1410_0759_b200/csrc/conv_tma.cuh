// tcgen05 implicit-GEMM convolution with the A operand gathered by TMA in
// im2col mode (forward and backward-data; included by conv_tc.cu).
//
// The packed input planes [N][IH][IW][Cp] (BF16 hi / lo) are described by
// two im2col tensor maps: one load = 128 consecutive output pixels (walking
// W -> H -> N inside the bounding box, zero fill at the image border) x CB
// channels of one filter tap, written 32B/64B/128B-swizzled straight into the
// K-major A stage.  One thread streams A and B (the packed filter, tiled TMA)
// for every stage: no per-row address arithmetic, no producer warps.
//
// NC = 2 runs the tile on a CTA pair (cluster of 2 on one TPC,
// tcgen05.mma.cta_group::2, M = 256): each CTA gathers its own 128 pixel
// rows and HALF of the BN filter rows, so the bytes each SM ingests per
// stage drop from 32 KB + 256*BN to 32 KB + 128*BN -- every SM streaming at
// once gets ~57 B/clk (profiles/r01/tma_burst_probe.txt), below what a
// 128 x BN BF16x3 tile consumes for BN < 256.
//
// Schedule: persistent clusters walk whole tiles for the full waves; when the
// last wave would be partial ("stream-K"), its tiles are cut along the
// reduction into equal contiguous unit ranges, one per cluster.  A tile cut
// into pieces accumulates each piece in TMEM, the epilogue writes it as an
// fp32 partial and bumps the tile's counter; the last piece to arrive sums
// all partials in piece order (deterministic) and writes the output.
//
// Warps: 0 = TMA producer (one elected lane, both CTAs), 1 = TMEM allocation
// + MMA issue (leader CTA only; warp-collective loop, elected issue), 2-5 =
// epilogue (TMEM lane quadrant warp % 4), double-buffered accumulator so the
// epilogue of one work item overlaps the main loop of the next.
#pragma once

constexpr int kTmaThreads = 10 * 32;  // TMA warp, MMA warp, 8 epilogue warps
constexpr int kColCache = 512;        // mode-1 column table cached in shared memory
constexpr int kTK = 64;  // reduction depth of one BF16 stage (4 k-steps of 16)

// Fused epilogue operations (additive C entries
// dnnp_convolution_bias_activation_forward / _backward_data_activation).
// Forward: y = act(alpha*conv + beta*y + bias[k]).  Backward-data: dx =
// act'(g) * conv (+ beta*dx), g = the activation output that fed the conv,
// read at the same offset as dx (the host requires identical strides).
// Activation formulas: reference nnops.py:54-88 (same as nnops.cu ActFwd/ActBwd).
struct EpiOp {
  int act;              // forward activation of the sum: -1 none, 0 sigmoid, 1 relu, 2 tanh
  int gate;             // backward-data: -1 none, else the activation kind of g
  const float* bias;    // per output channel (stride bias_sc), or null
  int64_t bias_sc;
  const float* gatep;   // g, same strides as the output
  __device__ __forceinline__ bool any() const { return act >= 0 || gate >= 0 || bias != nullptr; }
};

__device__ __forceinline__ float epi_act_fwd(int kind, float x) {
  if (kind == 1) return (x > 0.0f || x != x) ? x : 0.0f;
  if (kind == 2) return tanhf(x);
  const float e = expf(-fabsf(x));
  return x >= 0.0f ? 1.0f / __fadd_rn(1.0f, e) : e / __fadd_rn(1.0f, e);
}

__device__ __forceinline__ float epi_act_bwd(int kind, float y, float dy) {
  if (kind == 1) return __fmul_rn(dy, y > 0.0f ? 1.0f : 0.0f);
  if (kind == 2) return __fmul_rn(dy, __fsub_rn(1.0f, __fmul_rn(y, y)));
  return __fmul_rn(__fmul_rn(dy, y), __fsub_rn(1.0f, y));
}

// Per-element output operations, one functor per (op, activation) so that the
// 32-column store loops are branch-free (a runtime switch per element made
// the epilogue instruction-latency bound: 5x the plain store time).
// acc = accumulator, old = stored value (read only when needed), aux = the
// gate value g (backward-data) or bias[k] (forward).
struct OpAxpby {  // alpha * acc + beta * old (also the non-final reduction segments)
  float alpha, beta;
  __device__ __forceinline__ float operator()(float acc, float old, float) const {
    const float v = __fmul_rn(acc, alpha);
    return beta != 0.0f ? __fadd_rn(__fmul_rn(old, beta), v) : v;
  }
};
template <int ACT>
struct OpBiasAct {  // act(alpha * acc + beta * old + bias)
  float alpha, beta;
  bool bias;
  __device__ __forceinline__ float operator()(float acc, float old, float aux) const {
    float v = __fmul_rn(acc, alpha);
    if (beta != 0.0f) v = __fadd_rn(__fmul_rn(old, beta), v);
    if (bias) v = __fadd_rn(v, aux);
    return ACT < 0 ? v : epi_act_fwd(ACT, v);
  }
};
template <int KIND, bool SEGD>
struct OpGate {  // act'(g) * acc (+ beta * old); segmented: act'(g) * (old + acc)
  float beta;
  __device__ __forceinline__ float operator()(float acc, float old, float g) const {
    if (SEGD) return epi_act_bwd(KIND, g, __fadd_rn(old, acc));
    const float v = epi_act_bwd(KIND, g, acc);
    return beta != 0.0f ? __fadd_rn(__fmul_rn(old, beta), v) : v;
  }
};

// 32 channel columns of one row at rowp (stride sc), nv of them valid; all
// loads of a half are issued before its stores
template <class Op>
__device__ __forceinline__ void store_cols(float* rowp, int64_t sc, int nv, const uint32_t* v,
                                           bool rd_old, const float* auxp, int64_t aux_sc,
                                           const Op& op) {
#pragma unroll
  for (int h = 0; h < 32; h += 16) {
    // unconditional loads (invalid columns read column 0): predicated or
    // branched loads let the compiler pair each load with its use
    float old[16], aux[16];
    if (rd_old) {
#pragma unroll
      for (int j = 0; j < 16; j++) old[j] = rowp[h + j < nv ? int64_t(h + j) * sc : 0];
    } else {
#pragma unroll
      for (int j = 0; j < 16; j++) old[j] = 0.0f;
    }
    if (auxp) {
#pragma unroll
      for (int j = 0; j < 16; j++) aux[j] = __ldg(auxp + (h + j < nv ? int64_t(h + j) * aux_sc : 0));
    } else {
#pragma unroll
      for (int j = 0; j < 16; j++) aux[j] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < 16; j++)
      if (h + j < nv) rowp[int64_t(h + j) * sc] = op(__uint_as_float(v[h + j]), old[j], aux[j]);
  }
}

// scattered columns: element offsets off[] (relative to out) with valid mask;
// aux from auxp + off (gate) or bias + ch * bsc
template <class Op>
__device__ __forceinline__ void store_scatter(float* out, const int64_t* off, uint32_t okm,
                                              const int* ch, const float* v, bool rd_old,
                                              const float* gatep, const float* biasp, int64_t bsc,
                                              const Op& op) {
  // unconditional loads (invalid elements have off = 0, ch = 0)
  float old[16], aux[16];
#pragma unroll
  for (int j = 0; j < 16; j++) old[j] = rd_old ? out[off[j]] : 0.0f;
  if (gatep) {
#pragma unroll
    for (int j = 0; j < 16; j++) aux[j] = __ldg(gatep + off[j]);
  } else if (biasp) {
#pragma unroll
    for (int j = 0; j < 16; j++) aux[j] = __ldg(biasp + ch[j] * bsc);
  } else {
#pragma unroll
    for (int j = 0; j < 16; j++) aux[j] = 0.0f;
  }
#pragma unroll
  for (int j = 0; j < 16; j++)
    if ((okm >> j) & 1u) out[off[j]] = op(v[j], old[j], aux[j]);
}

// Calls f(op) with the functor for this element class (one switch per chunk).
template <class F>
__device__ __forceinline__ void with_op(const EpiOp& E, bool fuse, bool segd, float alpha,
                                        float beta, F&& f) {
  if (!fuse) {
    f(OpAxpby{alpha, beta});
  } else if (E.gate >= 0) {
    switch (E.gate * 2 + (segd ? 1 : 0)) {
      case 0: f(OpGate<0, false>{beta}); break;
      case 1: f(OpGate<0, true>{beta}); break;
      case 2: f(OpGate<1, false>{beta}); break;
      case 3: f(OpGate<1, true>{beta}); break;
      case 4: f(OpGate<2, false>{beta}); break;
      default: f(OpGate<2, true>{beta}); break;
    }
  } else {
    const bool b = E.bias != nullptr;
    switch (E.act) {
      case 0: f(OpBiasAct<0>{alpha, beta, b}); break;
      case 1: f(OpBiasAct<1>{alpha, beta, b}); break;
      case 2: f(OpBiasAct<2>{alpha, beta, b}); break;
      default: f(OpBiasAct<-1>{alpha, beta, b}); break;
    }
  }
}

struct TmaParams {
  CUtensorMap tm_ahi;  // im2col maps of the packed input planes
  CUtensorMap tm_alo;
  CUtensorMap tm_bhi;  // packed filter [Np][Ktot], box {CB, BN / NC}
  CUtensorMap tm_blo;
  int64_t M;           // GEMM rows = N * OH * OW
  int Ncol;            // valid GEMM columns
  int lower_h, lower_w, u, v;  // window origin of output pixel (oh, ow): lower + o * stride
  int nCB, tapW, KCH, nkb;     // channel blocks per tap, taps per window row, chunks, k-blocks
  int kb_lo;                   // first k-block of this launch (reduction segment [kb_lo, nkb))
  int nseg;                    // reduction segments per tile (consecutive work items of one
                               // cluster; segment s > 0 adds alpha*acc to the stored output)
  int Cext;                    // channel extent of the A maps (OOB coordinate for padding chunks)
  int nt, tiles;               // column tiles, tiles (of NC * 128 rows)
  // stream-K: full waves W (tiles cid + i*G), then units [cid*U/G, (cid+1)*U/G)
  // of the last R = tiles - W*G tiles; U = R * nkb.  sk = 0: plain persistent.
  int sk, W, U, maxp;
  int clusters;                // launched clusters (0: min(tiles, SMs / NC))
  float* skws;                 // partials [R][NC][maxp][128][BN]
  int* skcnt;                  // arrival counters [R][NC], zero on entry, reset by the finisher
  float* out;
  int64_t o_sn, o_sc, o_sh, o_sw;
  int out_mode;                // 0: column = channel; 1: column table (ph, pw, c)
  int off32;                   // mode 1: every column offset fits in int32
  int o_u, o_v, o_H, o_W, o_ph, o_pw;  // mode 1: h = oh * o_u + ph - o_ph
  const uint32_t* coltab;
  float alpha, beta;
  int plain;                   // alpha == 1, beta == 0: store the accumulator as is
  EpiOp epi;                   // fused bias / activation / activation-backward (plain == 0)
  MagicDiv dOHW, dOW;
  int skip;                    // experiments: 1 = no A loads, 2 = no loads, 4 = no MMAs
  int prefetch;                // L2 prefetch of the next tile's im2col window
  unsigned long long* trace;   // debug: CTA-0 clock64 stamps (or null)
};

// ES: bytes per packed element, 2 = BF16x3 (kind::f16), 4 = 3xTF32
// (kind::tf32, fp32 containers).  A stage always holds 128 bytes of
// reduction per row (kTK bf16 or kTK / 2 tf32 channels) in four 32-byte
// k-steps, so both splits share the stage geometry and the MMA schedule.
template <int ES>
constexpr int stage_depth() { return 128 / ES; }

template <int BN, int CB, int NC, int ES>
struct TCfg {
  static constexpr int BNL = BN / NC;        // filter rows loaded by each CTA
  static constexpr int SUB = stage_depth<ES>() / CB;  // chunks (sub-tiles) per stage
  static constexpr int RB = CB * ES;         // bytes of one sub-tile row (swizzle span)
  static constexpr int A_SUB = kBM * RB;     // bytes of one A sub-tile (one plane)
  static constexpr int B_SUB = BNL * RB;
  static constexpr int A_BYTES = SUB * A_SUB;
  static constexpr int B_BYTES = SUB * B_SUB;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // per CTA
  static constexpr int COLTAB_BYTES = kColCache * 16;  // int64 + int32 offset, packed (ph, pw)
  static constexpr int STAGES = (225 * 1024 - 2048 - COLTAB_BYTES) / STAGE_BYTES > 8
                                    ? 8
                                    : (225 * 1024 - 2048 - COLTAB_BYTES) / STAGE_BYTES;
  // DUAL (BN <= 128, room in TMEM): even / odd k-blocks of a work item
  // accumulate into two accumulators the epilogue adds in IEEE fp32 (each
  // truncating tcgen05 chain is half as long); ACC columns per buffer
  static constexpr bool DUAL = BN <= 128;
  static constexpr int ACC = DUAL ? 2 * BN : BN;
  static constexpr int TMEM_COLS =
      2 * ACC <= 64 ? 64 : (2 * ACC <= 128 ? 128 : (2 * ACC <= 256 ? 256 : 512));
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + COLTAB_BYTES;
};

template <int RB>  // row bytes of the K-major sub-tile
__device__ __forceinline__ uint64_t tma_kdesc(uint32_t addr) {
  if constexpr (RB == 128) return ptx::desc_kmajor_sw128(addr);
  else if constexpr (RB == 64) return ptx::desc_kmajor_sw64(addr);
  else return ptx::desc_kmajor_sw32(addr);
}

// Owner cluster of stream-K unit x: the largest j with floor(j*U/G) <= x
// (G <= U, so every cluster owns at least one unit).
__host__ __device__ __forceinline__ int sk_owner(int x, int U, int G) {
  int j = int((int64_t(x) * G) / U);
  while (j + 1 < G && int((int64_t(j + 1) * U) / G) <= x) j++;
  while (j > 0 && int((int64_t(j) * U) / G) > x) j--;
  return j;
}

// The sequence of work items of one cluster: (tile, k-block range, piece of
// the tile, pieces of the tile); every role of the cluster walks it alike.
struct WorkIter {
  int cid, G, nkb, kb_lo, tiles, sk, W, U, G2, nseg;
  int i, u, uend;
  int seg;  // reduction segment of the last item (0 unless P.nseg > 1)
  __device__ void init(const TmaParams& P, int cid_, int G_) {
    cid = cid_;
    G = G_;
    nkb = P.nkb;
    kb_lo = P.kb_lo;
    nseg = P.nseg;
    seg = 0;
    tiles = P.tiles;
    sk = P.sk;
    W = P.W;
    U = P.U;
    i = 0;
    // the last-wave units are spread over G2 = min(G, U) clusters so that
    // every participating cluster owns >= 1 unit (consecutive piece numbers)
    G2 = min(G, U);
    u = (sk && cid < G2) ? int((int64_t(cid) * U) / G2) : 0;
    uend = (sk && cid < G2) ? int((int64_t(cid + 1) * U) / G2) : 0;
  }
  __device__ bool next(int& tile, int& kb0, int& kb1, int& piece, int& np) {
    if (nseg > 1) {
      const int t = i / nseg;
      seg = i - t * nseg;
      tile = cid + t * G;
      if (tile >= tiles) return false;
      i++;
      const int span = nkb - kb_lo;
      kb0 = kb_lo + int(int64_t(span) * seg / nseg);
      kb1 = kb_lo + int(int64_t(span) * (seg + 1) / nseg);
      piece = 0;
      np = 1;
      return true;
    }
    if (!sk) {
      tile = cid + i * G;
      if (tile >= tiles) return false;
      i++;
      kb0 = kb_lo;
      kb1 = nkb;
      piece = 0;
      np = 1;
      return true;
    }
    if (i < W) {
      tile = cid + i * G;
      i++;
      kb0 = 0;
      kb1 = nkb;
      piece = 0;
      np = 1;
      return true;
    }
    if (u >= uend) return false;
    const int tl = u / nkb;
    tile = W * G + tl;
    kb0 = u - tl * nkb;
    kb1 = min(nkb, kb0 + (uend - u));
    const int first = sk_owner(tl * nkb, U, G2), last = sk_owner(tl * nkb + nkb - 1, U, G2);
    piece = cid - first;
    np = last - first + 1;
    u += kb1 - kb0;
    return true;
  }
};

template <int BN, int CB, int NC, int ES>
__global__ void __launch_bounds__(kTmaThreads, 1) conv_tma_kernel(const __grid_constant__ TmaParams P) {
  using C = TCfg<BN, CB, NC, ES>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* sk_flag = reinterpret_cast<int*>(tmem_slot + 1);
  long long* col_off = reinterpret_cast<long long*>(smem + S * C::STAGE_BYTES + 256);
  int* col_hw = reinterpret_cast<int*>(col_off + kColCache);
  int* col_off32 = col_hw + kColCache;  // when P.off32: the offsets as int32 (16-byte reads)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = NC == 2 ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int cid = int(blockIdx.x) / NC, ncl = int(gridDim.x) / NC;  // cluster id / count

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < S; s++) {
        ptx::mbar_init(&full[s], NC);  // each CTA's producer arrives (leader adds expect_tx)
        ptx::mbar_init(&empty[s], 1);  // MMA commit (multicast to both CTAs)
      }
      for (int b = 0; b < 2; b++) {
        ptx::mbar_init(&tfull[b], 1);
        ptx::mbar_init(&tempty[b], 8 * NC);  // one arrival per epilogue warp of each CTA
      }
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc_g<C::TMEM_COLS, NC>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (NC == 2) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t smem0 = ptx::smem_u32(smem);
  // launched programmatically behind the operand / filter packs: everything
  // above (barriers, TMEM) overlapped their tail; nothing below may run
  // before their writes are visible
  pdl_wait();
  WorkIter wi;
  wi.init(P, cid, ncl);
  int tile, kb0, kb1, piece, np;

  if (warp == 0) {
    // ================================================ TMA producer
    if (lane == 0) {
      ptx::tma_prefetch(&P.tm_ahi);
      ptx::tma_prefetch(&P.tm_alo);
      ptx::tma_prefetch(&P.tm_bhi);
      ptx::tma_prefetch(&P.tm_blo);
      int it = 0;
      while (wi.next(tile, kb0, kb1, piece, np)) {
        const uint32_t m0 = uint32_t(tile / P.nt) * (kBM * NC) + rank * kBM;
        const int n0 = (tile % P.nt) * BN + int(rank) * C::BNL;
        uint32_t img, rem, oh, ow;
        mdivmod(m0, P.dOHW, img, rem);
        mdivmod(rem, P.dOW, oh, ow);
        const int h0 = P.lower_h + int(oh) * P.u, w0 = P.lower_w + int(ow) * P.v;
        if (P.prefetch && np == 1 && tile + ncl < P.tiles) {
          // warm L2 with the next tile's window (first and last tap, every
          // channel block): its first loads otherwise pay DRAM latency
          const uint32_t m1 = uint32_t((tile + ncl) / P.nt) * (kBM * NC) + rank * kBM;
          uint32_t img1, rem1, oh1, ow1;
          mdivmod(m1, P.dOHW, img1, rem1);
          mdivmod(rem1, P.dOW, oh1, ow1);
          const int h1 = P.lower_h + int(oh1) * P.u, w1 = P.lower_w + int(ow1) * P.v;
          const int taps = (P.KCH + P.nCB - 1) / P.nCB;
          const int lt = taps - 1;
          for (int cbp = 0; cbp < P.nCB; cbp++) {
            ptx::tma_prefetch_im2col(&P.tm_ahi, cbp * CB, w1, h1, int(img1), 0, 0);
            ptx::tma_prefetch_im2col(&P.tm_alo, cbp * CB, w1, h1, int(img1), 0, 0);
            ptx::tma_prefetch_im2col(&P.tm_ahi, cbp * CB, w1, h1, int(img1), uint16_t(lt % P.tapW),
                                     uint16_t(lt / P.tapW));
            ptx::tma_prefetch_im2col(&P.tm_alo, cbp * CB, w1, h1, int(img1), uint16_t(lt % P.tapW),
                                     uint16_t(lt / P.tapW));
          }
        }
        int kc = kb0 * C::SUB;
        int tapi = kc / P.nCB, cb = kc - tapi * P.nCB;
        int dh = tapi / P.tapW, dw = tapi - dh * P.tapW;
        for (int kb = kb0; kb < kb1; kb++, it++) {
          const int s = it % S;
          const bool tr = P.trace && blockIdx.x == 0 && it < 1024;
          if (tr) P.trace[it * 4 + 0] = clock64();
          if (it >= S) ptx::mbar_wait(&empty[s], ((it / S) - 1) & 1);
          if (tr) P.trace[it * 4 + 1] = clock64();
          const uint32_t tx = (P.skip & 2) ? 0u : (P.skip & 1) ? 2 * C::B_BYTES : C::STAGE_BYTES;
          if (leader) ptx::mbar_arrive_expect_tx(&full[s], tx * NC);
          else ptx::mbar_arrive_cluster(&full[s], 0);
          if (P.skip & 2) {
            kc += C::SUB;
            continue;
          }
          const uint32_t bar = NC == 2 ? ptx::leader_addr(&full[s]) : ptx::smem_u32(&full[s]);
          const uint32_t base = smem0 + s * C::STAGE_BYTES;
#pragma unroll
          for (int j = 0; j < C::SUB; j++, kc++) {
            const bool real = kc < P.KCH;
            const int c = real ? cb * CB : P.Cext;  // padding chunk: all-OOB box -> zeros
            const uint16_t ow16 = uint16_t(real ? dw : 0), oh16 = uint16_t(real ? dh : 0);
            const uint32_t da = base + j * C::A_SUB;
            const uint32_t db = base + 2 * C::A_BYTES + j * C::B_SUB;
            if constexpr (NC == 2) {
              if (!(P.skip & 1)) {
                ptx::tma_load_im2col_pair(da, &P.tm_ahi, c, w0, h0, int(img), ow16, oh16, bar);
                ptx::tma_load_im2col_pair(da + C::A_BYTES, &P.tm_alo, c, w0, h0, int(img), ow16,
                                          oh16, bar);
              }
              ptx::tma_load_2d_pair(db, &P.tm_bhi, kc * CB, n0, bar);
              ptx::tma_load_2d_pair(db + C::B_BYTES, &P.tm_blo, kc * CB, n0, bar);
            } else {
              if (!(P.skip & 1)) {
                ptx::tma_load_im2col(da, &P.tm_ahi, c, w0, h0, int(img), ow16, oh16, &full[s]);
                ptx::tma_load_im2col(da + C::A_BYTES, &P.tm_alo, c, w0, h0, int(img), ow16, oh16,
                                     &full[s]);
              }
              ptx::tma_load_2d(db, &P.tm_bhi, kc * CB, n0, &full[s]);
              ptx::tma_load_2d(db + C::B_BYTES, &P.tm_blo, kc * CB, n0, &full[s]);
            }
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
    // ================================================ MMA issuer (leader CTA)
    if (leader) {
      constexpr uint32_t idesc = ES == 4 ? ptx::idesc_tf32(kBM * NC, BN, 0, 0)
                                         : ptx::idesc_bf16(kBM * NC, BN, 0, 0);
      int it = 0, lt = 0;
      while (wi.next(tile, kb0, kb1, piece, np)) {
        const int buf = lt & 1;
        ptx::mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t dacc0 = tmem_base + uint32_t(buf * C::ACC);
        uint32_t accv[2] = {0, 0};
        for (int kb = kb0; kb < kb1; kb++, it++) {
          const int s = it % S;
          const int half = C::DUAL ? ((kb - kb0) & 1) : 0;
          const uint32_t dacc = dacc0 + uint32_t(half * BN);
          uint32_t acc = accv[half];
          ptx::mbar_wait_spin(&full[s], (it / S) & 1);
          ptx::tc_fence_after();
          if (P.trace && blockIdx.x == 0 && it < 1024 && lane == 0) P.trace[it * 4 + 2] = clock64();
          const uint32_t base = smem0 + s * C::STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4 && !(P.skip & 4); kk++) {
            // 32-byte k-step kk (16 bf16 / 8 tf32 deep): sub-tile kk / (RB/32),
            // +32 B per step inside its rows
            constexpr int KPS = C::RB / 32;  // k-steps per sub-tile row
            const int sub = kk / KPS, ko = (kk % KPS) * 32;
            const uint32_t ao = uint32_t(sub * C::A_SUB + ko);
            const uint32_t bo = uint32_t(sub * C::B_SUB + ko);
            const uint64_t dah = tma_kdesc<C::RB>(base + ao);
            const uint64_t dal = tma_kdesc<C::RB>(base + C::A_BYTES + ao);
            const uint64_t dbh = tma_kdesc<C::RB>(base + 2 * C::A_BYTES + bo);
            const uint64_t dbl = tma_kdesc<C::RB>(base + 2 * C::A_BYTES + C::B_BYTES + bo);
            // lo.hi + hi.lo + hi.hi into one fp32 accumulator (lo.lo dropped)
            ptx::mma_split_elect<NC, ES>(dacc, dal, dbh, idesc, acc);
            ptx::mma_split_elect<NC, ES>(dacc, dah, dbl, idesc, 1);
            ptx::mma_split_elect<NC, ES>(dacc, dah, dbh, idesc, 1);
            acc = 1;
          }
          accv[half] = 1;
          if constexpr (NC == 2) ptx::mma_commit_pair_elect(&empty[s]);
          else ptx::mma_commit_elect(&empty[s]);
          if (P.trace && blockIdx.x == 0 && it < 1024 && lane == 0) P.trace[it * 4 + 3] = clock64();
        }
        if constexpr (NC == 2) ptx::mma_commit_pair_elect(&tfull[buf]);
        else ptx::mma_commit_elect(&tfull[buf]);
        lt++;
      }
    }
  } else {
    // ================================================ epilogue
    // 8 warps: quadrant ew = warp % 4 holds TMEM lanes (rows) 32*ew.., the
    // two warp sets split the 32-column chunks between them
    const int ew = warp & 3, es = (warp - 2) >> 2;
    // 32 accumulator columns of the work item (DUAL: both halves added)
    auto ld_acc = [&](int buf, int c0, bool two, uint32_t (&v)[32]) {
      const uint32_t ta = tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(buf * C::ACC + c0);
      ptx::tmem_ld32(ta, v);
      if (C::DUAL && two) {
        uint32_t w[32];
        ptx::tmem_ld32(ta + BN, w);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i++)
          v[i] = __float_as_uint(__fadd_rn(__uint_as_float(v[i]), __uint_as_float(w[i])));
      } else {
        ptx::tmem_ld_wait();
      }
    };
    const int r = ew * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..255 over the eight epilogue warps
    const bool ctab_smem = P.out_mode == 1 && P.Ncol <= kColCache;
    if (ctab_smem) {
      // column -> (offset of (c, ph, pw) from the row base, (ph, pw)) in shared memory
      for (int c = et; c < P.Ncol; c += 256) {
        const uint32_t e = __ldg(P.coltab + c);
        const int ph = int(e >> 24), pw = int((e >> 16) & 255);
        col_off[c] = int64_t(e & 0xFFFF) * P.o_sc + int64_t(ph) * P.o_sh + int64_t(pw) * P.o_sw;
        col_off32[c] = int(col_off[c]);
        col_hw[c] = (ph << 16) | pw;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    int lt = 0;
    while (wi.next(tile, kb0, kb1, piece, np)) {
      const int buf = lt & 1;
      const int64_t m = int64_t(tile / P.nt) * (kBM * NC) + int64_t(rank) * kBM + r;
      const int n0 = (tile % P.nt) * BN;
      const bool row_ok = m < P.M;
      uint32_t img = 0, oh = 0, ow = 0;
      if (row_ok) {
        uint32_t rem;
        mdivmod(uint32_t(m), P.dOHW, img, rem);
        mdivmod(rem, P.dOW, oh, ow);
      }
      const bool etr = P.trace && blockIdx.x == 0 && r == 0 && es == 0 && lt < 64;
      if (etr) P.trace[4096 + lt * 4 + 0] = clock64();
      ptx::mbar_wait(&tfull[buf], (lt >> 1) & 1);
      if (etr) P.trace[4096 + lt * 4 + 1] = clock64();
      ptx::tc_fence_after();
      bool finisher = true;
      float* part = nullptr;
      if (np > 1) {
        // partial piece: park the raw accumulator, count arrivals; the last
        // piece of the tile reduces all pieces in order
        const int slot = (tile - P.W * ncl) * NC + int(rank);
        part = P.skws + (int64_t(slot) * P.maxp) * (kBM * BN);
        // column-major [col][row] so each warp store / load is 128 contiguous bytes
        float* mine = part + int64_t(piece) * (kBM * BN) + r;
#pragma unroll 1
        for (int c0 = 32 * es; c0 < BN; c0 += 64) {
          uint32_t v[32];
          ld_acc(buf, c0, kb1 - kb0 > 1, v);
#pragma unroll
          for (int i = 0; i < 32; i++) __stcg(mine + (c0 + i) * kBM, __uint_as_float(v[i]));
        }
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (et == 0) {
          const int prev = atomicAdd(P.skcnt + slot, 1);
          const bool last = prev == np - 1;
          if (last) P.skcnt[slot] = 0;  // ready for the next launch
          *sk_flag = last ? 1 : 0;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        finisher = *sk_flag != 0;
        if (finisher) __threadfence();
      }
      if (finisher) {
        // segments after the first add to what the first stored
        const float beta = wi.seg ? 1.0f : P.beta;
        const bool plain = P.plain && wi.seg == 0;
        const bool last = wi.seg == P.nseg - 1 || P.nseg <= 1;
        const bool segd = P.nseg > 1;
        // mode 0: row base at the output pixel; mode 1: at (oh*o_u - o_ph, ow*o_v - o_pw)
        const int hb = int(oh) * P.o_u - P.o_ph, wb = int(ow) * P.o_v - P.o_pw;
        const int64_t rowoff =
            P.out_mode == 0 ? int64_t(img) * P.o_sn + int64_t(oh) * P.o_sh + int64_t(ow) * P.o_sw
                            : int64_t(img) * P.o_sn + int64_t(hb) * P.o_sh + int64_t(wb) * P.o_sw;
#pragma unroll 1
        for (int c0 = 32 * es; c0 < BN; c0 += 64) {
          const int cbase = n0 + c0;
          if (cbase >= P.Ncol) break;  // warp-uniform: padded columns are never loaded
          uint32_t v[32];
          if (np == 1) {
            ld_acc(buf, c0, kb1 - kb0 > 1, v);
          } else {
            const float* src = part + int64_t(c0) * kBM + r;
#pragma unroll
            for (int i = 0; i < 32; i++) v[i] = __float_as_uint(__ldcg(src + i * kBM));
            for (int q = 1; q < np; q++) {
              const float* sq = src + int64_t(q) * (kBM * BN);
#pragma unroll
              for (int i = 0; i < 32; i++)
                v[i] = __float_as_uint(__fadd_rn(__uint_as_float(v[i]), __ldcg(sq + i * kBM)));
            }
          }
          if (!row_ok) continue;
          if (P.out_mode == 0 && plain && cbase + 32 <= P.Ncol) {
            float* dst = P.out + rowoff + int64_t(cbase) * P.o_sc;
            const int64_t sc = P.o_sc;
#pragma unroll
            for (int i = 0; i < 32; i++) {
              *dst = __uint_as_float(v[i]);
              dst += sc;
            }
          } else if (P.out_mode == 0) {
            float* rowp = P.out + rowoff + int64_t(cbase) * P.o_sc;
            const int nv = min(32, P.Ncol - cbase);
            const bool fuse = last && P.epi.any();
            const bool gate = fuse && P.epi.gate >= 0;
            const float* auxp = gate ? P.epi.gatep + rowoff + int64_t(cbase) * P.o_sc
                                : (fuse && P.epi.bias) ? P.epi.bias + int64_t(cbase) * P.epi.bias_sc
                                                       : nullptr;
            const int64_t aux_sc = gate ? P.o_sc : P.epi.bias_sc;
            with_op(P.epi, fuse, segd, P.alpha, beta, [&](const auto& op) {
              store_cols(rowp, P.o_sc, nv, v, beta != 0.0f, auxp, aux_sc, op);
            });
          } else if (plain && ctab_smem && P.off32 && cbase + 32 <= P.Ncol &&
                     hb >= 0 && hb + P.o_u <= P.o_H && wb >= 0 && wb + P.o_v <= P.o_W) {
            // interior row (every (ph, pw) of the row's super-pixel in range):
            // offsets four at a time, no per-element bounds checks
            float* rb = P.out + rowoff;
            const int4* co = reinterpret_cast<const int4*>(col_off32 + cbase);
#pragma unroll
            for (int q = 0; q < 8; q++) {
              const int4 o = co[q];
              rb[o.x] = __uint_as_float(v[4 * q + 0]);
              rb[o.y] = __uint_as_float(v[4 * q + 1]);
              rb[o.z] = __uint_as_float(v[4 * q + 2]);
              rb[o.w] = __uint_as_float(v[4 * q + 3]);
            }
          } else if (plain && ctab_smem) {
#pragma unroll
            for (int i = 0; i < 32; i++) {
              const int col = cbase + i;
              if (col < P.Ncol) {
                const int hw = col_hw[col];
                if (unsigned(hb + (hw >> 16)) < unsigned(P.o_H) &&
                    unsigned(wb + (hw & 0xFFFF)) < unsigned(P.o_W))
                  P.out[rowoff + col_off[col]] = __uint_as_float(v[i]);
              }
            }
          } else {
            // scattered columns (super-pixel / space-to-depth / blocked):
            // offsets from the column table, loads of a half before its stores
            const bool fuse = last && P.epi.any();
            const bool gate = fuse && P.epi.gate >= 0, bias = fuse && P.epi.bias != nullptr;
#pragma unroll
            for (int h = 0; h < 32; h += 16) {
              int64_t off[16];
              int ch[16];
              float acc[16];
              uint32_t okm = 0;
#pragma unroll
              for (int j = 0; j < 16; j++) {
                const int col = cbase + h + j;
                off[j] = 0;
                ch[j] = 0;
                acc[j] = __uint_as_float(v[h + j]);
                if (col < P.Ncol) {
                  int ph, pw;
                  int64_t o;
                  if (ctab_smem) {
                    const int hw = col_hw[col];
                    ph = hw >> 16;
                    pw = hw & 0xFFFF;
                    o = col_off[col];
                    if (bias) ch[j] = int(__ldg(P.coltab + col) & 0xFFFF);
                  } else {
                    const uint32_t e = __ldg(P.coltab + col);
                    ph = int(e >> 24);
                    pw = int((e >> 16) & 255);
                    ch[j] = int(e & 0xFFFF);
                    o = int64_t(ch[j]) * P.o_sc + int64_t(ph) * P.o_sh + int64_t(pw) * P.o_sw;
                  }
                  if (unsigned(hb + ph) < unsigned(P.o_H) && unsigned(wb + pw) < unsigned(P.o_W)) {
                    okm |= 1u << j;
                    off[j] = rowoff + o;
                  }
                }
              }
              if (plain) {
#pragma unroll
                for (int j = 0; j < 16; j++)
                  if ((okm >> j) & 1u) P.out[off[j]] = acc[j];
              } else {
                with_op(P.epi, fuse, segd, P.alpha, beta, [&](const auto& op) {
                  store_scatter(P.out, off, okm, ch, acc, beta != 0.0f,
                                gate ? P.epi.gatep : nullptr, bias ? P.epi.bias : nullptr,
                                P.epi.bias_sc, op);
                });
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (etr) P.trace[4096 + lt * 4 + 2] = clock64();
      if (lane == 0) {
        if (NC == 1) ptx::mbar_arrive(&tempty[buf]);
        else ptx::mbar_arrive_cluster(&tempty[buf], 0);
      }
      lt++;
    }
  }
  ptx::tc_fence_before();
  if constexpr (NC == 2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_g<C::TMEM_COLS, NC>(tmem_base);
  }
}
