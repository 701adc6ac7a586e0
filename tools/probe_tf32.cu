// Probe: tcgen05.mma.kind::tf32 operand layouts on sm_100a.
//   K-major SW128 (32 fp32 per 128-byte row, k-step = +32 B), and
//   MN-major with the 128B_ATOM_32B TMA swizzle / SWIZZLE_128B_BASE32B
//   descriptor (layout type 1), k-step = 8 rows, for a range of SBO / LBO.
// D[m][n] = sum_k A(m,k) B(n,k), M=128, N=64, K=32, one CTA; inputs are small
// integers (exact in tf32), so the check is exact.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_tf32 probe_tf32.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 64, K = 32;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__device__ uint64_t mkdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout) << 61;
  return d;
}

struct Cfg {
  int mn_major;          // 0: K-major operands, 1: MN-major operands
  uint32_t layout;       // descriptor layout type
  uint32_t a_lbo, a_sbo, b_lbo, b_sbo;
  uint32_t kstep_bytes;  // start-address advance per 8-deep k-step
};

__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      Cfg cfg, float* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;                 // 16 KB
  uint8_t* sb = sm + M * K * 4;     // 8 KB
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
                 "r"(uint32_t((M + N) * K * 4)));
    if (!cfg.mn_major) {
      // A global [M][K] (k contiguous): box {32 k, 128 m}; B [N][K]: box {32, 64}
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sa)), "l"(&ta), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sb)), "l"(&tb), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
    } else {
      // A global [K][M] (m contiguous): per 32-wide m block, box {32 m, 32 k}
      for (int j = 0; j < M / 32; j++)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(sa + j * cfg.a_lbo)), "l"(&ta), "r"(j * 32), "r"(0), "r"(su32(&bar)) : "memory");
      for (int j = 0; j < N / 32; j++)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(sb + j * cfg.b_lbo)), "l"(&tb), "r"(j * 32), "r"(0), "r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(cfg.mn_major) << 15) |
                           (uint32_t(cfg.mn_major) << 16) | (uint32_t(N >> 3) << 17) |
                           (uint32_t(M >> 4) << 24);
    for (int kk = 0; kk < K / 8; kk++) {
      const uint64_t da = mkdesc(su32(sa) + kk * cfg.kstep_bytes, cfg.a_lbo, cfg.a_sbo, cfg.layout);
      const uint64_t db = mkdesc(su32(sb) + kk * cfg.kstep_bytes, cfg.b_lbo, cfg.b_sbo, cfg.layout);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
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
  const cuuint64_t strides[1] = {inner * 4};
  const cuuint32_t box[2] = {bi, bo};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("  encode failed: %d\n", int(r));
  return r == CUDA_SUCCESS;
}

int main() {
  std::vector<float> A(M * K), B(N * K);  // logical A(m,k), B(n,k)
  srand(7);
  for (auto& v : A) v = float(rand() % 7 - 3);
  for (auto& v : B) v = float(rand() % 7 - 3);
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; m++)
    for (int n = 0; n < N; n++)
      for (int k = 0; k < K; k++) ref[m * N + n] += double(A[m * K + k]) * B[n * K + k];
  // K-major copies [M][K], MN-major copies [K][M]
  std::vector<float> Ak(A), Bk(B), Am(K * M), Bm(K * N);
  for (int m = 0; m < M; m++)
    for (int k = 0; k < K; k++) Am[k * M + m] = A[m * K + k];
  for (int n = 0; n < N; n++)
    for (int k = 0; k < K; k++) Bm[k * N + n] = B[n * K + k];
  float *dAk, *dBk, *dAm, *dBm, *dO;
  cudaMalloc(&dAk, Ak.size() * 4);
  cudaMalloc(&dBk, Bk.size() * 4);
  cudaMalloc(&dAm, Am.size() * 4);
  cudaMalloc(&dBm, Bm.size() * 4);
  cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dAk, Ak.data(), Ak.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dBk, Bk.data(), Bk.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dAm, Am.data(), Am.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dBm, Bm.data(), Bm.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);

  struct Case {
    const char* name;
    Cfg cfg;
    CUtensorMapSwizzle sw;
  };
  std::vector<Case> cases = {
      {"kmajor_sw128", {0, 2, 16, 1024, 16, 1024, 32}, CU_TENSOR_MAP_SWIZZLE_128B},
      {"mn_b32_sbo512", {1, 1, 4096, 512, 4096, 512, 1024}, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B},
      {"mn_b32_sbo1024", {1, 1, 4096, 1024, 4096, 1024, 1024}, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B},
      {"mn_b32_sbo512_swap", {1, 1, 512, 4096, 512, 4096, 1024}, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B},
      {"mn_sw128_sbo1024", {1, 2, 4096, 1024, 4096, 1024, 1024}, CU_TENSOR_MAP_SWIZZLE_128B},
  };
  for (auto& c : cases) {
    CUtensorMap ta, tb;
    bool ok;
    if (!c.cfg.mn_major)
      ok = map2d(&ta, dAk, K, M, 32, M, c.sw) && map2d(&tb, dBk, K, N, 32, N, c.sw);
    else
      ok = map2d(&ta, dAm, M, K, 32, 32, c.sw) && map2d(&tb, dBm, N, K, 32, 32, c.sw);
    if (!ok) {
      printf("%-22s ENCODE_FAIL\n", c.name);
      continue;
    }
    cudaMemset(dO, 0, M * N * 4);
    probe<<<1, 128, 64 * 1024>>>(ta, tb, c.cfg, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%-22s CUDA_ERROR %s\n", c.name, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> O(M * N);
    cudaMemcpy(O.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxd = 0;
    for (int i = 0; i < M * N; i++) {
      const double d = std::abs(O[i] - ref[i]);
      if (d > 0) bad++;
      if (d > maxd) maxd = d;
    }
    printf("%-22s %s  bad=%d/%d maxdiff=%g  O[0]=%g ref[0]=%g O[1]=%g ref[1]=%g\n", c.name,
           bad ? "FAIL" : "PASS", bad, M * N, maxd, O[0], ref[0], O[1], ref[1]);
  }
  return 0;
}
