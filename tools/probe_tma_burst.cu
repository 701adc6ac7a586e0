// Probe: is TMA throughput limited by the issuing thread or by the TMA unit?
// Issue B loads back-to-back (distinct smem slots, one mbarrier, expect_tx of
// the total) from 1, 2 or 4 issuing warps, then wait; report cycles per load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tma_burst probe_tma_burst.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void burst(const __grid_constant__ CUtensorMap tm, int nloads, int box_bytes, int issuers,
                      int rounds, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long total = 0;
  for (int rd = 0; rd < rounds; rd++) {
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                   "r"(nloads * box_bytes));
    __syncthreads();
    if (lane == 0 && warp < issuers) {
      for (int i = warp; i < nloads; i += issuers) {
        const uint32_t dst = su32(buf + i * box_bytes);
        const int idx = (blockIdx.x * 977 + rd * 4099 + i * 131) % (16 * 4096 - 256);
        if (MODE == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(idx), "r"(su32(&bar))
              : "memory");
        } else {
          const int w = idx % 64, h = (idx / 64) % 64, n = idx / 4096;
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&bar)), "r"(0), "r"(w - 1), "r"(h - 1),
              "r"(n), "h"(uint16_t(i % 3)), "h"(uint16_t(1))
              : "memory");
        }
      }
    }
    if (threadIdx.x == 0) {
      asm volatile(
          "{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
              su32(&bar)),
          "r"(rd & 1)
          : "memory");
      total += clock64() - t0;
    }
  }
  if (threadIdx.x == 0) out[blockIdx.x] = total / rounds;
}

typedef CUresult (*EncTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
typedef CUresult (*EncIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int N = 16, H = 64, W = 64, C = 64;
  void* d = nullptr;
  cudaMalloc(&d, size_t(N) * H * W * C * 2);
  cudaMemset(d, 0, size_t(N) * H * W * C * 2);
  long long* dout;
  cudaMalloc(&dout, 256 * sizeof(long long));
  void *p1, *p2;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p1, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p2, cudaEnableDefault, &q);
  EncTiled enc_t = (EncTiled)p1;
  EncIm2col enc_i = (EncIm2col)p2;
  cudaFuncSetAttribute(burst<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(burst<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int mode = 0; mode < 2; mode++) {
    for (int rows : {32, 64, 128}) {
      CUtensorMap tm;
      if (mode == 0) {
        const cuuint64_t dims[2] = {64, (cuuint64_t)N * H * W};
        const cuuint64_t strides[1] = {128};
        const cuuint32_t box[2] = {64, (cuuint32_t)rows};
        const cuuint32_t es[2] = {1, 1};
        enc_t(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        const cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
        const cuuint64_t strides[3] = {128, 128ull * W, 128ull * W * H};
        const int lower[2] = {-1, -1}, upper[2] = {-1, -1};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        enc_i(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, strides, lower, upper, 64, rows, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      const int bb = rows * 128;
      const int nloads = (200 * 1024) / bb > 48 ? 48 : (200 * 1024) / bb;
      for (int issuers : {1, 2, 4}) {
        for (int ctas : {1, 148}) {
          if (mode == 0) burst<0><<<ctas, 128, nloads * bb + 1024>>>(tm, nloads, bb, issuers, 20, dout);
          else burst<1><<<ctas, 128, nloads * bb + 1024>>>(tm, nloads, bb, issuers, 20, dout);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          std::vector<long long> h(ctas);
          cudaMemcpy(h.data(), dout, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
          double avg = 0;
          for (auto v : h) avg += double(v) / ctas;
          printf("%s rows=%3d (%5d B) loads=%2d issuers=%d ctas=%3d: burst %7.0f cyc, %6.1f cyc/load, %6.1f B/clk\n",
                 mode ? "im2col" : "tiled ", rows, bb, nloads, issuers, ctas, avg, avg / nloads,
                 double(nloads) * bb / avg);
        }
      }
    }
  }
  return 0;
}
