// Probe: MN-major SW128 tcgen05 operands over a halo.  A backward-filter
// GEMM over a halo of packed pixels X[k][c] (pixel k, 64 channels c
// contiguous, one 128-byte row per pixel, loaded by one 2-D TMA box) needs
// A(m, k) = X[off + k + (m / 64) * delta][m % 64]: the reduction (pixel) index
// starts at an arbitrary row `off` and the two 64-wide M blocks of an M=128
// tile are the same halo at two pixel shifts, i.e. LBO = delta * 128 bytes
// (not a multiple of the 1024-byte swizzle atom).  B(n, k) = Y[k][n] (dy,
// MN-major, aligned).  D = A . B^T, M=128, N=64, K=16 per MMA, 4 MMAs (K=64);
// small-integer inputs, exact check.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_halo_mn probe_halo_mn.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 64, K = 64, RH = 256;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__device__ uint64_t mkdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}

__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      int off, int delta, float* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;              // RH rows x 128 B
  uint8_t* sb = sm + RH * 128;   // K rows x 128 B
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                 "r"(uint32_t((RH + K) * 128)));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sa)), "l"(&ta), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sb)), "l"(&tb), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    // kind::f16, BF16 x BF16 -> F32, A and B MN-major
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    for (int kk = 0; kk < K / 16; kk++) {
      // 16 K-rows per MMA = 2 groups of 8 rows (SBO = 1024 B)
      const uint64_t da = mkdesc(su32(sa) + uint32_t(off + 16 * kk) * 128, uint32_t(delta) * 128, 1024);
      const uint64_t db = mkdesc(su32(sb) + uint32_t(16 * kk) * 128, 8192, 1024);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(kk) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}" ::"r"(su32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 32; i++) out[row * N + c0 + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                           CUtensorMapFloatOOBfill);
static EncFn enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<EncFn>(p);
}

static bool map2d(CUtensorMap* m, void* base, uint64_t rows, uint32_t box_rows) {
  const cuuint64_t dims[2] = {64, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main() {
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<float> X(RH * 64), Y(K * 64);
  srand(5);
  for (auto& v : X) v = float(rand() % 7 - 3);
  for (auto& v : Y) v = float(rand() % 7 - 3);
  std::vector<__nv_bfloat16> Xb(X.size()), Yb(Y.size());
  for (size_t i = 0; i < X.size(); i++) Xb[i] = __float2bfloat16(X[i]);
  for (size_t i = 0; i < Y.size(); i++) Yb[i] = __float2bfloat16(Y[i]);
  __nv_bfloat16 *dX, *dY;
  float* dO;
  cudaMalloc(&dX, Xb.size() * 2);
  cudaMalloc(&dY, Yb.size() * 2);
  cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dX, Xb.data(), Xb.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Yb.data(), Yb.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  if (!map2d(&ta, dX, RH, RH) || !map2d(&tb, dY, K, K)) {
    printf("encode failed\n");
    return 1;
  }
  const int cases[][2] = {{0, 64}, {0, 8}, {0, 1}, {3, 1}, {5, 2}, {1, 57}, {7, 58}, {2, 114},
                          {6, 3}, {9, 13}, {0, 0}, {4, 100}};
  for (const auto& c : cases) {
    const int off = c[0], delta = c[1];
    cudaMemset(dO, 0, M * N * 4);
    probe<<<1, 128, 64 * 1024>>>(ta, tb, off, delta, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("off %d delta %d CUDA_ERROR %s\n", off, delta, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> O(M * N);
    cudaMemcpy(O.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; m++)
      for (int n = 0; n < N; n++) {
        double r = 0;
        for (int k = 0; k < K; k++) r += double(X[(off + k + (m / 64) * delta) * 64 + m % 64]) * Y[k * 64 + n];
        if (std::abs(O[m * N + n] - r) > 0) bad++;
      }
    printf("off %2d delta %3d: %s (%d bad)\n", off, delta, bad ? "BAD" : "ok", bad);
  }
  return 0;
}
