// Probe: TMA multicast across CTA pairs in a 4-CTA cluster (two tcgen05
// cta_group::2 pairs: {0,1}, {2,3}).  Question for sharing the filter tile
// of the im2col kernel between two pairs: when CTA r issues
//   cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global
//       .mbarrier::complete_tx::bytes.multicast::cluster [dst], [map, {x, y}], [bar], mask
// with bar = the LEADER copy of a barrier (peer bit cleared), does every
// destination CTA's data land at dst and is the transaction counted on the
// leader barrier of EACH destination's pair?
//
// Setup: every CTA loads a different 16-row slice of a 64 x 64 bf16 matrix and
// multicasts it to {itself, the same-rank CTA of the other pair} (mask
// (1 << r) | (1 << (r ^ 2))), so each CTA receives two slices (its own and
// the other pair's same-rank CTA's) = 2 x 2 KB; each pair leader expects the
// bytes landing in both CTAs of its pair (4 slices = 8 KB).  Leaders wait
// with a clock bound (a hang would mean the bytes go elsewhere); then every
// CTA checks its two slices.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_mcast probe_mcast.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__global__ void __cluster_dims__(4, 1, 1) probe(const __grid_constant__ CUtensorMap tm, int* result) {
  __shared__ __align__(1024) uint8_t buf[2][16 * 128];  // slice from pair A's / pair B's CTA
  __shared__ uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const bool leader = (rank & 1) == 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    // the leader of each pair expects the bytes that land in both of its CTAs
    if (leader)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                   "r"(4u * 16u * 128u));
    // slot 0 holds pair A's slices ({0,1}), slot 1 pair B's: same offsets in all CTAs
    const uint32_t dst = su32(&buf[rank >> 1][0]);
    const uint32_t bar_leader = su32(&bar) & 0xFEFFFFFFu;
    const uint16_t mask = uint16_t((1u << rank) | (1u << (rank ^ 2u)));
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(int(rank) * 16), "r"(bar_leader), "h"(mask)
        : "memory");
  }
  int ok = 1;
  if (leader && threadIdx.x == 0) {
    const long long t0 = clock64();
    uint32_t done = 0;
    while (!done && clock64() - t0 < 2000000000LL) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(su32(&bar)));
    }
    if (!done) ok = 0;  // timed out
    result[8 + rank] = done ? 1 : -1;
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  // check: slot j holds rows of the slice loaded by CTA (2 j + (rank & 1))
  if (threadIdx.x == 0) {
    int bad = 0;
    for (int j = 0; j < 2; j++) {
      const int src = 2 * j + int(rank & 1);
      for (int row = 0; row < 16; row++)
        for (int c = 0; c < 64; c++) {
          // 128B swizzle: chunk (c / 8) of row at chunk ^ (row & 7)
          const int chunk = (c >> 3) ^ (row & 7);
          const __nv_bfloat16 v =
              reinterpret_cast<const __nv_bfloat16*>(&buf[j][row * 128 + chunk * 16])[c & 7];
          const float want = __bfloat162float(__float2bfloat16(float((src * 16 + row) * 64 + c) / 64.0f));
          if (__bfloat162float(v) != want) bad++;
        }
    }
    result[rank] = ok ? bad : -1;
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                           CUtensorMapFloatOOBfill);

int main() {
  std::vector<__nv_bfloat16> h(64 * 64);
  for (int i = 0; i < 64 * 64; i++) h[i] = __float2bfloat16(float(i) / 64.0f);
  __nv_bfloat16* d;
  int* r;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&r, 64 * sizeof(int));
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(r, 0, 64 * sizeof(int));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {64, 64};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {64, 16};
  const cuuint32_t es[2] = {1, 1};
  if (reinterpret_cast<EncFn>(p)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  probe<<<4, 32>>>(tm, r);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  std::vector<int> hr(64);
  cudaMemcpy(hr.data(), r, 64 * sizeof(int), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 4; i++)
    printf("CTA %d: %s (bad elements %d)%s\n", i, hr[i] == 0 ? "ok" : "FAIL", hr[i],
           (i & 1) == 0 ? (hr[8 + i] == 1 ? ", leader barrier completed" : ", leader barrier TIMED OUT") : "");
  return 0;
}
