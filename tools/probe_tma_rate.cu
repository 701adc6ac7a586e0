// Probe: TMA load throughput per SM for the box shapes the conv kernels use.
// One CTA per SM (grid = nctas), one thread streams `iters` loads of one box
// shape into a ring of 4 smem slots (mbarrier per slot, waits before reuse),
// reports cycles per load and the aggregate bytes/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tma_rate probe_tma_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int MODE, int SLOTS>  // 0 tiled 2d, 1 im2col 4d
__global__ void rate_kernel(const __grid_constant__ CUtensorMap tm, int iters, int box_bytes,
                            int c_extent_blocks, int npix_total, int ppc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[SLOTS];
  long long tissue = 0;
  if (threadIdx.x != 0) return;
  for (int i = 0; i < SLOTS; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const int s = it % SLOTS;
    if (it >= SLOTS) {
      const uint32_t par = ((it / SLOTS) - 1) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
              su32(&bar[s])),
          "r"(par)
          : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])),
                 "r"(box_bytes));
    const uint32_t dst = su32(buf + s * box_bytes);
    // walk the tensor so that loads hit different (L2-resident) lines
    const int idx = (blockIdx.x * 7919 + it * 131) % npix_total;
    const long long ti = clock64();
    if (MODE == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(idx), "r"(su32(&bar[s]))
          : "memory");
    } else {
      // pixel idx of a 64 x 64 image grid (W = 64, H = 64): w, h, n
      const int w = idx % 64, h = (idx / 64) % 64, n = idx / 4096;
      const uint16_t ow = uint16_t(it % 3), oh = uint16_t((it / 3) % 3);
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&bar[s])), "r"(0), "r"(w - 1), "r"(h - 1),
          "r"(n), "h"(ow), "h"(oh)
          : "memory");
    }
    tissue += clock64() - ti;
  }
  for (int s = 0; s < SLOTS; s++) {
    const int last = iters - SLOTS + s;
    const uint32_t par = (last / SLOTS) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
            su32(&bar[last % SLOTS])),
        "r"(par)
        : "memory");
  }
  out[blockIdx.x] = clock64() - t0;
  out[256 + blockIdx.x] = tissue;
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
  const int N = 16, H = 64, W = 64, C = 64;  // 16 x 64 x 64 x 64 bf16 = 8 MB (L2 resident)
  void* d = nullptr;
  cudaMalloc(&d, size_t(N) * H * W * C * 2);
  cudaMemset(d, 0, size_t(N) * H * W * C * 2);
  long long* dout;
  cudaMalloc(&dout, 512 * sizeof(long long));
  void* p1 = nullptr;
  void* p2 = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p1, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p2, cudaEnableDefault, &q);
  EncTiled enc_t = (EncTiled)p1;
  EncIm2col enc_i = (EncIm2col)p2;
  const int npix = N * H * W;
  const int iters = 2000;
  auto run = [&](auto kern, const CUtensorMap& tm, int slots, int box_bytes, int rows, const char* name, int ch) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int nctas : {1, 148}) {
      kern<<<nctas, 32, slots * box_bytes + 1024>>>(tm, iters, box_bytes, 1, npix, rows, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("kernel error %s\n", cudaGetErrorString(e)); exit(1); }
      std::vector<long long> h(512);
      cudaMemcpy(h.data(), dout, 512 * sizeof(long long), cudaMemcpyDeviceToHost);
      double avg = 0, iss = 0;
      for (int i = 0; i < nctas; i++) { avg += double(h[i]) / nctas; iss += double(h[256 + i]) / nctas; }
      printf("%s rows=%3d ch=%2d (%5d B) slots=%2d ctas=%3d: %7.1f cyc/load (issue %6.1f)  %6.1f B/clk/SM\n",
             name, rows, ch, box_bytes, slots, nctas, avg / iters, iss / iters, double(box_bytes) * iters / avg);
    }
  };
  for (int mode = 0; mode < 2; mode++) {
    for (int rows : {32, 128}) {
      const int ch = 64;
      CUtensorMap tm;
      const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
      CUresult r;
      if (mode == 0) {
        const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)npix};
        const cuuint64_t strides[1] = {(cuuint64_t)C * 2};
        const cuuint32_t box[2] = {(cuuint32_t)ch, (cuuint32_t)rows};
        const cuuint32_t es[2] = {1, 1};
        r = enc_t(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
        const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * W, (cuuint64_t)C * 2 * W * H};
        const int lower[2] = {-1, -1}, upper[2] = {-1, -1};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        r = enc_i(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, strides, lower, upper, ch, rows, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (r != CUDA_SUCCESS) { printf("encode failed\n"); continue; }
      const int bb = rows * ch * 2;
      const char* nm = mode ? "im2col" : "tiled ";
      if (mode == 0) {
        run(rate_kernel<0, 2>, tm, 2, bb, rows, nm, ch);
        run(rate_kernel<0, 4>, tm, 4, bb, rows, nm, ch);
        run(rate_kernel<0, 8>, tm, 8, bb, rows, nm, ch);
        if (bb * 16 <= 190 * 1024) run(rate_kernel<0, 16>, tm, 16, bb, rows, nm, ch);
        if (bb * 32 <= 190 * 1024) run(rate_kernel<0, 32>, tm, 32, bb, rows, nm, ch);
      } else {
        run(rate_kernel<1, 2>, tm, 2, bb, rows, nm, ch);
        run(rate_kernel<1, 4>, tm, 4, bb, rows, nm, ch);
        run(rate_kernel<1, 8>, tm, 8, bb, rows, nm, ch);
        if (bb * 16 <= 190 * 1024) run(rate_kernel<1, 16>, tm, 16, bb, rows, nm, ch);
        if (bb * 32 <= 190 * 1024) run(rate_kernel<1, 32>, tm, 32, bb, rows, nm, ch);
      }
    }
  }
  return 0;
}
