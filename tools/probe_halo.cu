// Probe: can a K-major swizzled tcgen05 operand start at an arbitrary ROW of a
// TMA-loaded tile (not a multiple of the 8-row swizzle atom)?  That is what a
// halo'd convolution needs: one TMA load of (128 + halo) consecutive packed
// pixel rows, then every filter tap's A operand = the 128-row window starting
// at the tap's flat offset, addressed by the descriptor start address.
//
// A tile: RH rows x W bf16 (W = 64 / 32 / 16 -> SW128 / SW64 / SW32), loaded
// by one 2-D TMA box {W, RH}.  For off = 0..15 and three descriptor
// base-offset policies, D = A[off : off + 128] . B^T (M=128, N=64, K=W) is
// compared exactly with the host product (small-integer inputs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_halo probe_halo.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 64, RH = 144;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__device__ uint64_t mkdesc(uint32_t addr, uint32_t sbo, uint32_t layout, uint32_t base_off) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(base_off & 7) << 49;
  d |= uint64_t(layout) << 61;
  return d;
}

struct Cfg {
  int W;             // bf16 per row (64 / 32 / 16)
  uint32_t layout;   // 2 = SW128, 4 = SW64, 6 = SW32
  int off;           // start row of the A window
  int policy;        // base offset: 0 = 0, 1 = (addr >> 7) & 7, 2 = off & 7
};

__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      Cfg cfg, float* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int rowb = cfg.W * 2;
  uint8_t* sa = sm;                                          // RH rows
  uint8_t* sb = sm + ((RH * rowb + 1023) & ~1023);           // N rows
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
                 "r"(uint32_t((RH + N) * rowb)));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sa)), "l"(&ta), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sb)), "l"(&tb), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) |
                           (uint32_t(M >> 4) << 24);
    const uint32_t sbo = 8 * rowb;
    for (int kk = 0; kk < cfg.W / 16; kk++) {
      const uint32_t aaddr = su32(sa) + uint32_t(cfg.off * rowb) + kk * 32;
      const uint32_t bo = cfg.policy == 0 ? 0 : cfg.policy == 1 ? (aaddr >> 7) & 7 : uint32_t(cfg.off & 7);
      const uint64_t da = mkdesc(aaddr, sbo, cfg.layout, bo);
      const uint64_t db = mkdesc(su32(sb) + kk * 32, sbo, cfg.layout, 0);
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

static bool map2d(CUtensorMap* m, void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo,
                  CUtensorMapSwizzle sw) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * 2};
  const cuuint32_t box[2] = {bi, bo};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("  encode failed: %d\n", int(r));
  return r == CUDA_SUCCESS;
}

int main() {
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  struct Sw {
    int W;
    uint32_t layout;
    CUtensorMapSwizzle sw;
    const char* name;
  } sws[] = {{64, 2, CU_TENSOR_MAP_SWIZZLE_128B, "SW128"},
             {32, 4, CU_TENSOR_MAP_SWIZZLE_64B, "SW64"},
             {16, 6, CU_TENSOR_MAP_SWIZZLE_32B, "SW32"}};
  float* dO;
  cudaMalloc(&dO, M * N * 4);
  for (const Sw& s : sws) {
    const int W = s.W;
    std::vector<float> A(RH * W), B(N * W);
    srand(11 + W);
    for (auto& v : A) v = float(rand() % 7 - 3);
    for (auto& v : B) v = float(rand() % 7 - 3);
    std::vector<__nv_bfloat16> Ab(A.size()), Bb(B.size());
    for (size_t i = 0; i < A.size(); i++) Ab[i] = __float2bfloat16(A[i]);
    for (size_t i = 0; i < B.size(); i++) Bb[i] = __float2bfloat16(B[i]);
    __nv_bfloat16 *dA, *dB;
    cudaMalloc(&dA, Ab.size() * 2);
    cudaMalloc(&dB, Bb.size() * 2);
    cudaMemcpy(dA, Ab.data(), Ab.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bb.data(), Bb.size() * 2, cudaMemcpyHostToDevice);
    CUtensorMap ta, tb;
    if (!map2d(&ta, dA, W, RH, W, RH, s.sw) || !map2d(&tb, dB, W, N, W, N, s.sw)) return 1;
    for (int policy = 0; policy < 3; policy++) {
      printf("%-6s policy %d:", s.name, policy);
      for (int off = 0; off < 16; off++) {
        cudaMemset(dO, 0, M * N * 4);
        probe<<<1, 128, 64 * 1024>>>(ta, tb, Cfg{W, s.layout, off, policy}, dO);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf(" CUDA_ERROR %s\n", cudaGetErrorString(e));
          return 1;
        }
        std::vector<float> O(M * N);
        cudaMemcpy(O.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < M; m++)
          for (int n = 0; n < N; n++) {
            double r = 0;
            for (int k = 0; k < W; k++) r += double(A[(off + m) * W + k]) * B[n * W + k];
            if (std::abs(O[m * N + n] - r) > 0) bad++;
          }
        printf(" %d:%s", off, bad ? "BAD" : "ok");
      }
      printf("\n");
    }
    cudaFree(dA);
    cudaFree(dB);
  }
  return 0;
}
