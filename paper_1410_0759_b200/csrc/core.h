// Internal interface between the C-ABI host core (api.cpp) and the CUDA
// kernel launchers (*.cu).  Plain structs, no torch types.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dnnp {

enum Dtype : int { F32 = 0, F64 = 1 };

// A 4-D strided view: extents and element strides (reference tensor.py:104-139).
struct View4 {
  int64_t n, c, h, w;
  int64_t sn, sc, sh, sw;
  int64_t size() const { return n * c * h * w; }
};

// Exact unsigned magic division for 32-bit numerators
// (reference intdiv.py:74-101, Hacker's Delight 2nd ed. ch. 10).
struct MagicDiv {
  uint32_t d;     // divisor
  uint32_t mul;   // multiplier (low 32 bits when add == 1)
  uint32_t shift;
  uint32_t add;   // 1 -> 33-bit multiplier, add-corrected form
};
MagicDiv make_magic(uint32_t d);

// One convolution problem, shared by forward / backward-data / backward-filter.
// x is the convolution input (or dx), y the output (or dy); the filter is
// always dense KCRS (reference conv.py:72-97).
struct ConvProblem {
  int64_t N, C, H, W, K, R, S, P, Q;
  int64_t u, v, pad_h, pad_w;
  bool flip;  // CONVOLUTION mode: tap r reads h = p*u + (R-1-r) - pad (conv.py:182-192)
  View4 x, y;
  // dnnp_engine: 1 = EXPLICIT materialises the lowered data matrix (forward;
  // the memory negative control, reference conv.py:494-535); DIRECT and
  // IMPLICIT (and every backward pass) run the implicit-GEMM kernels
  int engine = 2;
};

namespace tc {
// create the library's own stream-ordered memory pool on this device (bounded release threshold)
void pool_keep_memory();
// Scratch scope for host code (api.cpp): allocations come from the
// per-stream arena (tc_common.cuh Workspace) and are released when the scope
// closes; the arena stays locked for the scope's lifetime.
struct ScratchScope;
ScratchScope* scratch_open(cudaStream_t st);
cudaError_t scratch_alloc(ScratchScope* s, size_t bytes, void** p);
void scratch_close(ScratchScope* s);
// Caller-supplied workspace (the paper's minimal-workspace contract, additive
// *_ex entries): while active on this thread, every scratch allocation is
// carved from [base, base + bytes) instead of the library's arena, and an
// allocation past the end fails with cudaErrorMemoryAllocation.
void user_workspace_begin(void* base, size_t bytes);
// ends the override; *need = the bytes the call asked for in total
void user_workspace_end(size_t* need);
// Workspace query without executing the pass: scratch is carved from a fake
// base (high-water measured by user_workspace_end), the caller runs the pass
// on a capturing stream so no kernel executes, and the few memsets of the
// pass are skipped while dry_run() is true.
void dry_run_begin();
bool dry_run();
// Fused backward: pack dy once into scratch from scope sc and register it
// for the backward-data / backward-filter calls that follow on this thread;
// shared_dy_clear() ends the registration.
cudaError_t shared_dy_pack(ScratchScope* sc, const View4& v, const float* dy, int Cp,
                           cudaStream_t st);
void shared_dy_clear();
// scratch footprint measurement of one call on stream st
void scratch_measure_begin(cudaStream_t st);
size_t scratch_measure_end(cudaStream_t st);
}  // namespace tc

// Tuning switches (DNNP_* environment variables that force one kernel
// variant for tests and A/B measurements; every default is chosen from the
// problem shape).  The environment is read once and cached; the additive
// dnnp_reload_tuning() re-reads it.  None of these changes what is computed
// (only which correct kernel variant computes it): the diagnostic switches
// that do (skipped loads / MMAs, single-product MMA, traces) exist only in
// builds with -DDNNP_DIAG.
const char* tune_env(const char* name);  // cached getenv
void tune_reload();
// Diagnostic switches (DNNP_TC_SKIP / _PRODUCTS / _TRACE / _DIAG / _PREFETCH):
// compiled out of release builds, where they always read as unset.
inline const char* diag_env(const char* name) {
#ifdef DNNP_DIAG
  return tune_env(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Launch bookkeeping: every kernel this library launches bumps a counter
// so benches/tests can prove native kernels ran.
void note_launch(int count = 1);

// ---- convolution (conv_simt.cu, conv_tc.cu) -------------------------------
// y := alpha*conv(x,f) + beta*y      (beta == 0: y never read)
cudaError_t conv_forward(const ConvProblem& p, Dtype dt, const void* x, const void* f,
                         void* y, double alpha, double beta, int math, cudaStream_t st);
// dx := conv_bwd_data(dy, f) (+ dx if accumulate)
cudaError_t conv_backward_data(const ConvProblem& p, Dtype dt, const void* dy, const void* f,
                               void* dx, bool accumulate, int math, cudaStream_t st);
// Fused epilogues (additive).  Forward: y := act(alpha*conv
// + beta*y + bias[k]) (act -1: none; bias null: none).  Backward-data: dx :=
// act'(g) * conv_bwd_data(dy) (+ dx if accumulate), g the activation output
// that fed the convolution, viewed by gatev.
struct ConvEpilogue {
  int act = -1;
  const void* bias = nullptr;
  int64_t bias_stride = 0;  // element stride of the bias over k
  View4 biasv{};
  int gate = -1;
  const void* gatep = nullptr;
  View4 gatev{};
};
cudaError_t conv_forward_fused(const ConvProblem& p, Dtype dt, const void* x, const void* f,
                               void* y, double alpha, double beta, int math,
                               const ConvEpilogue& ep, cudaStream_t st);
cudaError_t conv_backward_data_fused(const ConvProblem& p, Dtype dt, const void* dy,
                                     const void* f, void* dx, bool accumulate, int math,
                                     const ConvEpilogue& ep, cudaStream_t st);
// Fused backward (additive): dx and df from one dy; on the tensor-core path
// dy is packed once for both GEMMs.  Same results as the two calls.
cudaError_t conv_backward_both(const ConvProblem& p, Dtype dt, const void* dy, const void* f,
                               const void* x, void* dx, void* df, bool accumulate, int math,
                               cudaStream_t st);
// df := conv_bwd_filter(dy, x) (+ df if accumulate)
cudaError_t conv_backward_filter(const ConvProblem& p, Dtype dt, const void* dy, const void* x,
                                 void* df, bool accumulate, int math, cudaStream_t st);
// db[k] = sum_{n,p,q} dy[n,k,p,q]  (dy dtype dt, db dtype dbt)
cudaError_t conv_backward_bias(const View4& dy, Dtype dt, const void* dyp, const View4& db,
                               Dtype dbt, void* dbp, cudaStream_t st);
// Verification loop nests (conv_verify.cu): pass 0 out = conv(a = x, b = f),
// 1 out = bwd_data(a = dy, b = f), 2 out = bwd_filter(a = dy, b = x); dense
// fp64 output, fp64 accumulation, one thread per output element.
cudaError_t conv_verify_reference(int pass, const ConvProblem& p, Dtype dt, const void* a,
                                  const void* b, double* out, cudaStream_t st);
// whether the tcgen05 path would be used for a forward problem (tests/bench)
bool tc_eligible(const ConvProblem& p, int pass);

// ---- NCCL, loaded at run time (nccl_dist.cpp) ------------------------------
namespace nccl {
bool available(const char** why);
const char* error_string(int r);
int unique_id(void* out128);                                     // ncclResult_t
int comm_init(void** comm, const void* id128, int nranks, int rank);
int comm_destroy(void* comm);
int allreduce_sum(const void* send, void* recv, size_t count, bool f64, void* comm,
                  cudaStream_t st);
}  // namespace nccl

// ---- elementwise / reductions (nnops.cu) -----------------------------------
cudaError_t activation_forward(int kind, Dtype dt, const View4& xv, const void* x,
                               const View4& yv, void* y, cudaStream_t st);
cudaError_t activation_backward(int kind, Dtype dt, const View4& yv, const void* y,
                                const View4& dyv, const void* dy, const View4& dxv, void* dx,
                                cudaStream_t st);
cudaError_t softmax_forward(int mode, Dtype dt, const View4& xv, const void* x,
                            const View4& yv, void* y, cudaStream_t st);
cudaError_t softmax_backward(int mode, Dtype dt, const View4& yv, const void* y,
                             const View4& dyv, const void* dy, const View4& dxv, void* dx,
                             cudaStream_t st);

struct PoolProblem {
  int kind;  // 0 max, 1 average
  int64_t wh, ww, sh, sw, ph, pw;
  int64_t P, Q;
};
cudaError_t pool_forward(const PoolProblem& pp, Dtype dt, const View4& xv, const void* x,
                         const View4& yv, void* y, int64_t* argmax, cudaStream_t st);
cudaError_t pool_backward(const PoolProblem& pp, Dtype dt, const View4& dyv, const void* dy,
                          const View4& dxv, void* dx, const int64_t* argmax,
                          cudaStream_t st);

// ---- tensor utilities (nnops.cu) -------------------------------------------
cudaError_t transform(Dtype dt, const View4& sv, const void* s, const View4& dv, void* d,
                      double alpha, double beta, cudaStream_t st);
cudaError_t add_broadcast(Dtype dt, const View4& bv, const void* b, const View4& ov, void* o,
                          double alpha, double beta, cudaStream_t st);

}  // namespace dnnp
