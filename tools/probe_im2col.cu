// Probe: semantics of TMA im2col loads (cuTensorMapEncodeIm2col +
// cp.async.bulk.tensor.4d.im2col) on sm_100a.  Loads one box per case and
// prints the decoded (n, h, w, c) of every smem row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_im2col probe_im2col.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void load_kernel(const __grid_constant__ CUtensorMap tm, int c, int w, int h, int n,
                            int ow, int oh, uint16_t* out, int bytes) {
  __shared__ alignas(1024) uint16_t buf[16384];
  __shared__ alignas(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t sd = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes));
    uint16_t o_w = (uint16_t)ow, o_h = (uint16_t)oh;
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(sd),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(sb), "r"(c), "r"(w), "r"(h), "r"(n), "h"(o_w),
        "h"(o_h)
        : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            sb)
        : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                          const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int N = 2, H = 7, W = 9, C = 64;
  uint16_t* hx = new uint16_t[N * H * W * C];
  for (int n = 0; n < N; n++)
    for (int h = 0; h < H; h++)
      for (int w = 0; w < W; w++)
        for (int c = 0; c < C; c++)
          hx[((n * H + h) * W + w) * C + c] = uint16_t(0x8000 | (n << 14) | (h << 10) | (w << 6) | c);
  uint16_t *dx, *dout;
  cudaMalloc(&dx, N * H * W * C * 2);
  cudaMalloc(&dout, 65536);
  cudaMemcpy(dx, hx, N * H * W * C * 2, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  struct Case {
    const char* name;
    int lw, lh, uw, uh, su, sv, cpp, ppc;
    int c, w, h, n, ow, oh;
  } cases[] = {
      {"pad1 R3 s1 start(-1,-1) off(0,0)", -1, -1, -1, -1, 1, 1, 8, 24, 0, -1, -1, 0, 0, 0},
      {"pad1 R3 s1 start(-1,-1) off(2,1)", -1, -1, -1, -1, 1, 1, 8, 24, 0, -1, -1, 0, 2, 1},
      {"pad1 R3 s1 start(3,5) n0 wrap to n1", -1, -1, -1, -1, 1, 1, 8, 24, 8, 3, 5, 0, 1, 1},
      {"pad2 R5 s2 start(-2,-2) off(0,0)", -2, -2, -2, -2, 2, 2, 8, 16, 0, -2, -2, 0, 0, 0},
      {"pad0 R3 s1 upper+1 (window extends)", 0, 0, 1, 1, 1, 1, 8, 24, 0, 0, 0, 0, 0, 0},
  };
  for (auto& cs : cases) {
    CUtensorMap tm;
    const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    const int lower[2] = {cs.lw, cs.lh};
    const int upper[2] = {cs.uw, cs.uh};
    const cuuint32_t es[4] = {1, (cuuint32_t)cs.sv, (cuuint32_t)cs.su, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, dx, dims, strides, lower, upper, cs.cpp,
                     cs.ppc, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("== %s (encode %d)\n", cs.name, (int)r);
    if (r != CUDA_SUCCESS) continue;
    const int bytes = cs.cpp * cs.ppc * 2;
    cudaMemset(dout, 0xFF, 65536);
    load_kernel<<<1, 128>>>(tm, cs.c, cs.w, cs.h, cs.n, cs.ow, cs.oh, dout, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("  kernel error %s\n", cudaGetErrorString(e));
      return 1;
    }
    uint16_t hb[16384];
    cudaMemcpy(hb, dout, bytes, cudaMemcpyDeviceToHost);
    for (int row = 0; row < cs.ppc; row++) {
      uint16_t v = hb[row * cs.cpp];
      uint16_t v1 = hb[row * cs.cpp + cs.cpp - 1];
      if (v == 0)
        printf("  row %2d: zero (last %04x)\n", row, v1);
      else
        printf("  row %2d: n%d h%d w%d c%d..c%d\n", row, (v >> 14) & 1, (v >> 10) & 15,
               (v >> 6) & 15, v & 63, v1 & 63);
    }
  }
  return 0;
}
