// C-ABI host core of libdnnp.so.
//
// Replaces the reference's C shim + embedded CPython bridge
// (pkg/capi/src/dnnp_capi.c and pkg/capi/bridge/dnnp_capi_bridge.py) with a
// native implementation: live-object registry, descriptor setters/getters,
// the span guard, the exact stride-aliasing check (tensor.py:44-101), view
// bounds (tensor.py:191-197), the shape/element-type checks of conv.py and
// nnops.py, the exception -> status map (dnnp_capi_bridge.py:30-46), and
// host/device buffer staging.  Compute goes straight to CUDA kernels.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <deque>
#include <map>
#include <mutex>
#include <new>
#include <type_traits>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/dnnp.h"
#include "core.h"

using dnnp::View4;

// --------------------------------------------------------------- tuning

namespace dnnp {
namespace {
std::mutex g_tune_mu;
std::map<std::string, const char*> g_tune;  // name -> cached value (nullptr: unset)
std::deque<std::string> g_tune_vals;        // grows only: returned pointers stay valid
}  // namespace

const char* tune_env(const char* name) {
  std::lock_guard<std::mutex> g(g_tune_mu);
  auto it = g_tune.find(name);
  if (it != g_tune.end()) return it->second;
  const char* v = getenv(name);
  const char* keep = nullptr;
  if (v) {
    g_tune_vals.emplace_back(v);
    keep = g_tune_vals.back().c_str();
  }
  g_tune.emplace(name, keep);
  return keep;
}

void tune_reload() {
  std::lock_guard<std::mutex> g(g_tune_mu);
  g_tune.clear();
}
}  // namespace dnnp

// --------------------------------------------------------------- objects

struct dnnp_context {
  int64_t threads = 1;
  cudaStream_t stream = nullptr;
  int math = DNNP_MATH_DEFAULT;
  void* comm = nullptr;     // ncclComm_t for the batch-sharded backward-filter
  bool owns_comm = false;   // created by dnnp_nccl_comm_create (destroyed with the handle)
};

struct dnnp_tensor_desc_t {
  bool configured = false;
  dnnp_elem_type elem = DNNP_F32;
  int64_t n = 0, c = 0, h = 0, w = 0;
  int64_t sn = 0, sc = 0, sh = 0, sw = 0;
  int inj = -1;  // cached aliasing verdict: -1 unknown, 0 injective, 1 aliasing
};

struct dnnp_filter_desc_t {
  bool configured = false;
  dnnp_elem_type elem = DNNP_F32;
  int64_t k = 0, c = 0, r = 0, s = 0;
};

struct dnnp_conv_desc_t {
  bool configured = false;
  int64_t u = 1, v = 1, pad_h = 0, pad_w = 0;
  dnnp_conv_mode mode = DNNP_CONVOLUTION;
  int accumulate = 0;
};

struct dnnp_pooling_desc_t {
  bool configured = false;
  dnnp_pool_kind kind = DNNP_POOL_MAX;
  int64_t wh = 0, ww = 0, sh = 0, sw = 0, ph = 0, pw = 0;
};

namespace {

// Descriptors bigger than this many elements are rejected outright
// (reference dnnp_capi.c:25-27).
constexpr int64_t kMaxSpanElems = int64_t(1) << 40;
// Offsets of boxes up to this size are checked exhaustively (tensor.py:28).
constexpr int64_t kExhaustiveLimit = int64_t(1) << 22;

enum Kind { KIND_HANDLE = 1, KIND_TENSOR, KIND_FILTER, KIND_CONV, KIND_POOL };

// Live-object registry (reference dnnp_capi.c:69-132): stale or double
// destroyed pointers are detected instead of dereferenced.
std::mutex g_reg_lock;
std::unordered_set<const void*> g_reg[KIND_POOL + 1];
bool g_created_once = false;  // dnnp_conv_output_shape needs a prior create

bool reg_add(const void* p, int kind) {
  std::lock_guard<std::mutex> g(g_reg_lock);
  return g_reg[kind].insert(p).second;
}
bool reg_has(const void* p, int kind) {
  if (!p) return false;
  std::lock_guard<std::mutex> g(g_reg_lock);
  return g_reg[kind].count(p) != 0;
}
bool reg_remove(const void* p, int kind) {
  if (!p) return false;
  std::lock_guard<std::mutex> g(g_reg_lock);
  return g_reg[kind].erase(p) != 0;
}

thread_local std::string t_last_error;

dnnp_status fail(dnnp_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return st;
}

inline size_t elem_size(dnnp_elem_type t) { return t == DNNP_F64 ? 8 : 4; }

// ------------------------------------------------------- stride algebra

// reference dnnp_capi.c:211-230
bool span_ok(const dnnp_tensor_desc_t* d) {
  const int64_t ext[4] = {d->n, d->c, d->h, d->w};
  const int64_t str[4] = {d->sn, d->sc, d->sh, d->sw};
  __int128 hi = 0, lo = 0;
  for (int i = 0; i < 4; i++) {
    __int128 t = (__int128)(ext[i] - 1) * (__int128)str[i];
    if (t > 0) hi += t; else lo += t;
  }
  return hi < (__int128)kMaxSpanElems && lo > -(__int128)kMaxSpanElems;
}

// Sufficient disjointness test: sorted by |stride|, every stride exceeds the
// span of the finer dimensions (reference tensor.py:44-56).
bool sorted_spans_disjoint(const int64_t* ext, const int64_t* str) {
  std::vector<std::pair<int64_t, int64_t>> dims;
  for (int i = 0; i < 4; i++)
    if (ext[i] > 1) dims.push_back({str[i] < 0 ? -str[i] : str[i], ext[i]});
  std::sort(dims.begin(), dims.end());
  __int128 span = 0;
  for (auto& d : dims) {
    if ((__int128)d.first <= span) return false;
    span += (__int128)(d.second - 1) * d.first;
  }
  return true;
}

// Exhaustive: materialise all offsets and look for a duplicate (tensor.py:59-63).
bool aliases_exhaustive(const int64_t* ext, const int64_t* str) {
  std::vector<int64_t> offs(1, 0);
  for (int i = 0; i < 4; i++) {
    std::vector<int64_t> next;
    next.reserve(offs.size() * ext[i]);
    for (int64_t o : offs)
      for (int64_t j = 0; j < ext[i]; j++) next.push_back(o + j * str[i]);
    offs.swap(next);
  }
  std::sort(offs.begin(), offs.end());
  return std::adjacent_find(offs.begin(), offs.end()) != offs.end();
}

// Delta sweep: aliasing iff a nonzero delta vector (|delta_i| < extent_i)
// maps to offset 0.  Solve for the largest-extent dimension and sweep the
// delta box of the others (tensor.py:66-81).
bool aliases_delta(const int64_t* ext, const int64_t* str) {
  std::vector<std::pair<int64_t, int64_t>> dims;
  for (int i = 0; i < 4; i++)
    if (ext[i] > 1) dims.push_back({ext[i], str[i]});
  size_t solve = 0;
  for (size_t i = 1; i < dims.size(); i++)
    if (dims[i].first > dims[solve].first) solve = i;
  const int64_t e_t = dims[solve].first, s_t = dims[solve].second;
  std::vector<int64_t> total(1, 0);
  for (size_t i = 0; i < dims.size(); i++) {
    if (i == solve) continue;
    std::vector<int64_t> next;
    next.reserve(total.size() * (2 * dims[i].first - 1));
    for (int64_t t : total)
      for (int64_t dlt = -(dims[i].first - 1); dlt <= dims[i].first - 1; dlt++)
        next.push_back(t + dlt * dims[i].second);
    total.swap(next);
  }
  for (int64_t t : total) {
    if (t == 0) continue;  // the trivial all-zero delta
    // numpy semantics: floor modulo / floor division
    int64_t q = t / s_t, r = t % s_t;
    if (r != 0 && ((r < 0) != (s_t < 0))) { q -= 1; r += s_t; }
    if (r == 0 && (q < 0 ? -q : q) <= e_t - 1) return true;
  }
  return false;
}

// true iff the strided map is one-to-one (reference tensor.py:84-101)
bool injective(const int64_t* ext, const int64_t* str) {
  for (int i = 0; i < 4; i++)
    if (ext[i] > 1 && str[i] == 0) return false;
  if (sorted_spans_disjoint(ext, str)) return true;
  int64_t box = 1;
  for (int i = 0; i < 4; i++) box *= ext[i];
  return box <= kExhaustiveLimit ? !aliases_exhaustive(ext, str) : !aliases_delta(ext, str);
}

int64_t min_offset(const dnnp_tensor_desc_t* d) {
  const int64_t ext[4] = {d->n, d->c, d->h, d->w}, str[4] = {d->sn, d->sc, d->sh, d->sw};
  int64_t m = 0;
  for (int i = 0; i < 4; i++) m += std::min<int64_t>(0, (ext[i] - 1) * str[i]);
  return m;
}
int64_t max_offset(const dnnp_tensor_desc_t* d) {
  const int64_t ext[4] = {d->n, d->c, d->h, d->w}, str[4] = {d->sn, d->sc, d->sh, d->sw};
  int64_t m = 0;
  for (int i = 0; i < 4; i++) m += std::max<int64_t>(0, (ext[i] - 1) * str[i]);
  return m;
}

View4 view_of(const dnnp_tensor_desc_t* d) {
  return View4{d->n, d->c, d->h, d->w, d->sn, d->sc, d->sh, d->sw};
}

// reference dnnp_capi.c:232-241
bool tensor_usable(dnnp_tensor_desc d, const void* buf) {
  return reg_has(d, KIND_TENSOR) && d->configured && buf && span_ok(d);
}
bool filter_usable(dnnp_filter_desc d, const void* buf) {
  return reg_has(d, KIND_FILTER) && d->configured && buf;
}

// Binding a descriptor to a buffer, as the bridge's _tensor() does
// (dnnp_capi_bridge.py:60-66 -> make_desc -> check_injective, then
// TensorView bounds): aliasing -> BAD_PARAM, negative reach -> SHAPE_MISMATCH.
dnnp_status bind_view(dnnp_tensor_desc d, const char* what) {
  if (d->inj < 0) {
    const int64_t ext[4] = {d->n, d->c, d->h, d->w}, str[4] = {d->sn, d->sc, d->sh, d->sw};
    d->inj = injective(ext, str) ? 0 : 1;
  }
  if (d->inj) return fail(DNNP_STATUS_BAD_PARAM, "%s: strides alias", what);
  if (min_offset(d) < 0)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "%s: descriptor maps below the buffer start", what);
  return DNNP_STATUS_OK;
}

// Output extent of a strided zero-padded window (reference conv.py:165-179):
// ceil((H - R + 1 + 2 pad) / u); <= 0 numerators are EmptyOutput.
bool output_extent(int64_t in, int64_t filt, int64_t stride, int64_t pad, int64_t* out) {
  if (in < 1 || filt < 1 || stride < 1 || pad < 0) return false;
  int64_t numer = in - filt + 1 + 2 * pad;
  if (numer < 1) return false;
  *out = (numer + stride - 1) / stride;
  return true;
}

// ------------------------------------------------------------ device glue

dnnp_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DNNP_STATUS_OK;
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation)
    return fail(DNNP_STATUS_ALLOC_FAILED, "%s: %s", what, cudaGetErrorString(e));
  return fail(DNNP_STATUS_NOT_SUPPORTED, "%s: %s", what, cudaGetErrorString(e));
}

dnnp_status need_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(DNNP_STATUS_NOT_SUPPORTED,
                "no CUDA device: dnnp computes on the GPU only (no CPU fallback)");
  }
  return DNNP_STATUS_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// One caller buffer as seen by a kernel.  Host buffers are staged through a
// stream-ordered device allocation covering [0, span) elements; device
// buffers are used in place.
struct Staged {
  const void* user = nullptr;
  void* dev = nullptr;
  size_t bytes = 0;
  bool host = false;
  bool out = false;
};

class Stager {
 public:
  explicit Stager(cudaStream_t st) : st_(st) {}
  ~Stager() { dnnp::tc::scratch_close(scratch_); }
  // copy_in: the kernel (or the gaps of a strided view) needs the caller's
  // current contents.
  dnnp_status add(const void* user, size_t bytes, bool out, bool copy_in, void** dev) {
    Staged b;
    b.user = user;
    b.bytes = bytes;
    b.out = out;
    b.host = !is_device_ptr(user);
    if (!b.host) {
      b.dev = const_cast<void*>(user);
    } else {
      // staging buffers come from the per-stream scratch arena (no
      // allocation in steady state); released when the call returns
      if (!scratch_) scratch_ = dnnp::tc::scratch_open(st_);
      cudaError_t e = dnnp::tc::scratch_alloc(scratch_, std::max<size_t>(bytes, 16), &b.dev);
      if (e != cudaSuccess) return cuda_status(e, "staging allocation");
      if (copy_in) {
        e = cudaMemcpyAsync(b.dev, user, bytes, cudaMemcpyHostToDevice, st_);
        if (e != cudaSuccess) return cuda_status(e, "host->device copy");
      }
      any_host_ = true;
    }
    bufs_.push_back(b);
    *dev = b.dev;
    return DNNP_STATUS_OK;
  }
  // A device staging buffer from this call's scratch scope (no copy).
  dnnp_status scratch(size_t bytes, void** dev) {
    if (!scratch_) scratch_ = dnnp::tc::scratch_open(st_);
    cudaError_t e = dnnp::tc::scratch_alloc(scratch_, std::max<size_t>(bytes, 16), dev);
    if (e != cudaSuccess) return cuda_status(e, "staging allocation");
    any_host_ = true;
    return DNNP_STATUS_OK;
  }
  // Copy staged outputs back and wait when any host buffer took part.
  dnnp_status finish(cudaError_t launch) {
    if (launch != cudaSuccess) {
      if (any_host_) cudaStreamSynchronize(st_);
      return cuda_status(launch, "kernel launch");
    }
    for (auto& b : bufs_) {
      if (b.host && b.out) {
        cudaError_t e = cudaMemcpyAsync(const_cast<void*>(b.user), b.dev, b.bytes,
                                        cudaMemcpyDeviceToHost, st_);
        if (e != cudaSuccess) return cuda_status(e, "device->host copy");
      }
    }
    if (any_host_) {
      cudaError_t e = cudaStreamSynchronize(st_);
      if (e != cudaSuccess) return cuda_status(e, "stream synchronize");
    }
    return DNNP_STATUS_OK;
  }

 private:
  cudaStream_t st_;
  std::vector<Staged> bufs_;
  bool any_host_ = false;
  dnnp::tc::ScratchScope* scratch_ = nullptr;
};

size_t span_bytes(dnnp_tensor_desc d) { return size_t(max_offset(d) + 1) * elem_size(d->elem); }
// A view with no gaps inside its span: writing the span writes only the view.
bool dense_view(dnnp_tensor_desc d) { return max_offset(d) + 1 == d->n * d->c * d->h * d->w; }

// ------------------------------------------- caller-supplied workspace
// The *_ex entries run the plain entry with this thread's workspace set: the
// compute's scratch is carved from the caller's device buffer (host operands
// are still staged through the library's own arena), and the chunked host
// pipeline is not used.
struct ExWorkspace {
  void* p = nullptr;
  size_t bytes = 0;
  bool on = false;
};
static thread_local ExWorkspace g_exws;

template <class F>
static cudaError_t with_workspace(F&& compute, size_t* need) {
  if (!g_exws.on) return compute();
  dnnp::tc::user_workspace_begin(g_exws.p, g_exws.bytes);
  cudaError_t e = compute();
  dnnp::tc::user_workspace_end(need);
  return e;
}

static dnnp_status ws_status(cudaError_t e, size_t need, const char* what) {
  if (e == cudaErrorMemoryAllocation && g_exws.on && need > g_exws.bytes)
    return fail(DNNP_STATUS_ALLOC_FAILED, "%s: workspace of %zu bytes too small (needs %zu)", what,
                g_exws.bytes, need);
  return DNNP_STATUS_OK;
}

// ------------------------------------------- pipelined host staging
// Batch-separable convolutions with HOST buffers: the N images go through in
// chunks; chunk i's inputs copy host->device on a copy-in stream while chunk
// i-1 computes on the handle's stream and chunk i-2's outputs copy back on a
// copy-out stream, so both PCIe directions and the GPU work overlap (the
// call stays synchronous, as the reference's).  A buffer qualifies when the
// image stride covers its per-image footprint (chunk byte ranges disjoint).
struct ChunkBuf {
  const void* user;
  dnnp_tensor_desc d;
  bool out, copy_in;
  void* dev = nullptr;
};

static void copy_streams(cudaStream_t* in, cudaStream_t* out) {
  static std::mutex mu;
  static std::map<int, std::pair<cudaStream_t, cudaStream_t>> m;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto& c = m[dev];
  if (!c.first) {
    cudaStreamCreateWithFlags(&c.first, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&c.second, cudaStreamNonBlocking);
  }
  *in = c.first;
  *out = c.second;
}

static int64_t image_bytes(dnnp_tensor_desc d) {  // footprint of one image
  return (max_offset(d) - (d->n - 1) * d->sn + 1) * int64_t(elem_size(d->elem));
}

static bool pipeline_ok(const std::vector<ChunkBuf>& bufs, int64_t N) {
  static const bool off = getenv("DNNP_NO_PIPELINE") != nullptr;
  if (off || N < 2 || g_exws.on) return false;
  size_t total = 0;
  for (const auto& b : bufs) {
    const dnnp_tensor_desc d = b.d;
    if (d->n != N || is_device_ptr(b.user) || d->sn < 0 || d->sc < 0 || d->sh < 0 || d->sw < 0)
      return false;
    if (d->sn * int64_t(elem_size(d->elem)) < image_bytes(d)) return false;
    total += span_bytes(d);
  }
  return total >= (size_t(16) << 20);
}

// compute(n0, nb, devs): launch the work of images [n0, n0 + nb) on st.
template <class F>
static dnnp_status run_pipelined(cudaStream_t st, Stager& sg, std::vector<ChunkBuf>& bufs,
                                 int64_t N, F&& compute) {
  dnnp_status rs;
  size_t total = 0;
  for (auto& b : bufs) {
    if ((rs = sg.scratch(span_bytes(b.d), &b.dev))) return rs;
    total += span_bytes(b.d);
  }
  // ~16 MB chunks (2..16 of them; more, smaller chunks measured slower:
  // every chunk repeats the packing and GEMM launches, tools/e2e_probe.py)
  static const int64_t shift = getenv("DNNP_PIPE_SHIFT") ? atoll(getenv("DNNP_PIPE_SHIFT")) : 24;
  static const int64_t minc = getenv("DNNP_PIPE_MIN") ? atoll(getenv("DNNP_PIPE_MIN")) : 2;
  const int64_t chunks =
      std::max<int64_t>(std::min<int64_t>(minc, N), std::min<int64_t>({16, N, int64_t(total >> shift)}));
  const int64_t nb = (N + chunks - 1) / chunks;
  cudaStream_t ci, co;
  copy_streams(&ci, &co);
  std::vector<cudaEvent_t> evs;
  auto mk = [&]() {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    evs.push_back(e);
    return e;
  };
  cudaError_t e = cudaSuccess;
  // the staging memory may still be read by earlier work on st
  cudaEvent_t e0 = mk();
  cudaEventRecord(e0, st);
  cudaStreamWaitEvent(ci, e0, 0);
  cudaStreamWaitEvent(co, e0, 0);
  for (int64_t n0 = 0; n0 < N && e == cudaSuccess; n0 += nb) {
    const int64_t cnt = std::min(nb, N - n0);
    auto range = [&](const ChunkBuf& b, size_t* off, size_t* len) {
      const int64_t es = int64_t(elem_size(b.d->elem));
      *off = size_t(n0 * b.d->sn * es);
      *len = size_t((cnt - 1) * b.d->sn * es + image_bytes(b.d));
    };
    for (const auto& b : bufs) {
      if (b.out && !b.copy_in) continue;
      size_t off, len;
      range(b, &off, &len);
      e = cudaMemcpyAsync(static_cast<char*>(b.dev) + off, static_cast<const char*>(b.user) + off,
                          len, cudaMemcpyHostToDevice, ci);
      if (e != cudaSuccess) break;
    }
    cudaEvent_t ein = mk();
    cudaEventRecord(ein, ci);
    cudaStreamWaitEvent(st, ein, 0);
    if (e == cudaSuccess) e = compute(n0, cnt);
    cudaEvent_t edone = mk();
    cudaEventRecord(edone, st);
    cudaStreamWaitEvent(co, edone, 0);
    for (const auto& b : bufs) {
      if (!b.out || e != cudaSuccess) continue;
      size_t off, len;
      range(b, &off, &len);
      e = cudaMemcpyAsync(static_cast<char*>(const_cast<void*>(b.user)) + off,
                          static_cast<char*>(b.dev) + off, len, cudaMemcpyDeviceToHost, co);
    }
  }
  cudaEvent_t eend = mk();
  cudaEventRecord(eend, co);
  cudaStreamWaitEvent(st, eend, 0);
  rs = sg.finish(e);  // remaining (non-batched) outputs, then synchronise st
  for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
  return rs;
}

static View4 shift_images(View4 v, int64_t nb) {
  v.n = nb;
  return v;
}

double read_scalar(const void* p, dnnp_elem_type t) {
  return t == DNNP_F64 ? *static_cast<const double*>(p)
                       : double(*static_cast<const float*>(p));
}

bool same_extents(dnnp_tensor_desc a, dnnp_tensor_desc b) {
  return a->n == b->n && a->c == b->c && a->h == b->h && a->w == b->w;
}

bool engine_valid(dnnp_engine e) {
  return e == DNNP_ENGINE_DIRECT || e == DNNP_ENGINE_EXPLICIT || e == DNNP_ENGINE_IMPLICIT;
}

// _check_triplet + conv_out_shape (reference conv.py:195-232)
dnnp_status conv_shape(dnnp_tensor_desc x, dnnp_filter_desc f, dnnp_conv_desc cd,
                       int64_t* P, int64_t* Q) {
  if (x->elem != f->elem)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "element types of input and filter differ");
  if (x->c != f->c)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "input channels %lld vs filter channels %lld",
                (long long)x->c, (long long)f->c);
  if (!output_extent(x->h, f->r, cd->u, cd->pad_h, P) ||
      !output_extent(x->w, f->s, cd->v, cd->pad_w, Q))
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "convolution produces no output");
  return DNNP_STATUS_OK;
}

// _check_out (reference conv.py:226-232)
dnnp_status check_out(dnnp_tensor_desc o, int64_t n, int64_t k, int64_t p, int64_t q,
                      dnnp_elem_type t, const char* what) {
  if (o->n != n || o->c != k || o->h != p || o->w != q)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "%s extents (%lld,%lld,%lld,%lld), expected "
                "(%lld,%lld,%lld,%lld)", what, (long long)o->n, (long long)o->c,
                (long long)o->h, (long long)o->w, (long long)n, (long long)k, (long long)p,
                (long long)q);
  if (o->elem != t) return fail(DNNP_STATUS_SHAPE_MISMATCH, "%s element type mismatch", what);
  return DNNP_STATUS_OK;
}

dnnp::ConvProblem make_problem(dnnp_tensor_desc x, dnnp_filter_desc f, dnnp_conv_desc cd,
                               dnnp_tensor_desc y, int64_t P, int64_t Q) {
  dnnp::ConvProblem p;
  p.N = x->n; p.C = x->c; p.H = x->h; p.W = x->w;
  p.K = f->k; p.R = f->r; p.S = f->s; p.P = P; p.Q = Q;
  p.u = cd->u; p.v = cd->v; p.pad_h = cd->pad_h; p.pad_w = cd->pad_w;
  p.flip = cd->mode == DNNP_CONVOLUTION;
  p.x = view_of(x);
  p.y = view_of(y);
  return p;
}

// 32-bit index decode limit of the lowered matrix (reference conv.py:254-255
// guards 2^31; the device decode here is exact below 2^32).
dnnp_status check_decode_range(const dnnp::ConvProblem& p) {
  const int64_t lim = int64_t(1) << 32;
  if (p.C * p.R * p.S >= lim || p.N * p.P * p.Q >= lim || p.N * p.H * p.W >= lim ||
      p.K * p.R * p.S >= lim)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "lowered index space exceeds 32-bit decode range");
  return DNNP_STATUS_OK;
}

// The explicit engine materialises the C R S x N P Q lowered matrix (data
// matrix forward / backward-filter, gradient matrix backward-data) and
// refuses it above the reference's limit: AllocTooLarge -> ALLOC_FAILED
// (conv.py:31, 507-511 lower_explicit, 615-618 backward-data, 701
// backward-filter via lower_explicit).
constexpr int64_t kLoweredLimit = int64_t(4) << 30;
dnnp_status explicit_guard(const dnnp::ConvProblem& pr, dnnp_engine engine, dnnp_elem_type elem,
                           const char* what) {
  if (engine != DNNP_ENGINE_EXPLICIT) return DNNP_STATUS_OK;
  const __int128 need = (__int128)pr.C * pr.R * pr.S * pr.N * pr.P * pr.Q * elem_size(elem);
  if (need > kLoweredLimit)
    return fail(DNNP_STATUS_ALLOC_FAILED, "explicit engine (%s): lowered matrix needs %lld bytes, limit %lld",
                what, (long long)need, (long long)kLoweredLimit);
  return DNNP_STATUS_OK;
}

}  // namespace

// =================================================================== ABI

extern "C" {

int64_t dnnp_version(void) { return DNNP_VERSION; }

void dnnp_reload_tuning(void) { dnnp::tune_reload(); }

dnnp_status dnnp_magic_divider(uint32_t divisor, uint32_t* multiplier, uint32_t* shift,
                               int* add_indicator) {
  if (!multiplier || !shift || !add_indicator)
    return fail(DNNP_STATUS_BAD_PARAM, "magic_divider: NULL out-pointer");
  if (divisor < 1) return fail(DNNP_STATUS_BAD_PARAM, "magic_divider: divisor must be >= 1");
  const dnnp::MagicDiv m = dnnp::make_magic(divisor);
  *multiplier = m.mul;
  *shift = m.shift;
  *add_indicator = int(m.add);
  return DNNP_STATUS_OK;
}

const char* dnnp_status_string(dnnp_status status) {
  switch (status) {
    case DNNP_STATUS_OK: return "ok";
    case DNNP_STATUS_BAD_PARAM: return "bad_param";
    case DNNP_STATUS_SHAPE_MISMATCH: return "shape_mismatch";
    case DNNP_STATUS_ALLOC_FAILED: return "alloc_failed";
    case DNNP_STATUS_NOT_SUPPORTED: return "not_supported";
    default: return "unknown";
  }
}

const char* dnnp_last_error(void) { return t_last_error.c_str(); }

// ---------------------------------------------------------------- handle

dnnp_status dnnp_create(dnnp_handle* handle) {
  if (!handle) return fail(DNNP_STATUS_BAD_PARAM, "handle out-pointer is NULL");
  *handle = nullptr;
  auto* ctx = new (std::nothrow) dnnp_context();
  if (!ctx) return fail(DNNP_STATUS_ALLOC_FAILED, "out of host memory");
  reg_add(ctx, KIND_HANDLE);
  {
    std::lock_guard<std::mutex> g(g_reg_lock);
    g_created_once = true;
  }
  *handle = ctx;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_destroy(dnnp_handle handle) {
  if (!reg_remove(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "not a live handle");
  if (handle->owns_comm) dnnp::nccl::comm_destroy(handle->comm);
  delete handle;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_set_threads(dnnp_handle handle, int64_t threads) {
  if (!reg_has(handle, KIND_HANDLE) || threads < 1)
    return fail(DNNP_STATUS_BAD_PARAM, "bad handle or threads < 1");
  handle->threads = threads;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_get_threads(dnnp_handle handle, int64_t* threads) {
  if (!reg_has(handle, KIND_HANDLE) || !threads) return fail(DNNP_STATUS_BAD_PARAM, "bad args");
  *threads = handle->threads;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_set_stream(dnnp_handle handle, void* stream) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  handle->stream = static_cast<cudaStream_t>(stream);
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_get_stream(dnnp_handle handle, void** stream) {
  if (!reg_has(handle, KIND_HANDLE) || !stream) return fail(DNNP_STATUS_BAD_PARAM, "bad args");
  *stream = handle->stream;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_synchronize(dnnp_handle handle) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  dnnp_status st = need_device();
  if (st) return st;
  return cuda_status(cudaStreamSynchronize(handle->stream), "synchronize");
}

dnnp_status dnnp_set_math(dnnp_handle handle, int math) {
  if (!reg_has(handle, KIND_HANDLE) || math < DNNP_MATH_DEFAULT || math > DNNP_MATH_TC_TF32X3)
    return fail(DNNP_STATUS_BAD_PARAM, "bad handle or math mode");
  handle->math = math;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_get_math(dnnp_handle handle, int* math) {
  if (!reg_has(handle, KIND_HANDLE) || !math) return fail(DNNP_STATUS_BAD_PARAM, "bad args");
  *math = handle->math;
  return DNNP_STATUS_OK;
}

// ----------------------------------------------------------- descriptors

#define DNNP_CREATE_DESTROY(name, htype, kind)                                   \
  dnnp_status dnnp_##name##_create(htype* desc) {                                \
    if (!desc) return fail(DNNP_STATUS_BAD_PARAM, #name ": NULL out-pointer");  \
    *desc = nullptr;                                                            \
    using obj_t = std::remove_pointer<htype>::type;                              \
    auto* d = new (std::nothrow) obj_t();                                       \
    if (!d) return fail(DNNP_STATUS_ALLOC_FAILED, "out of host memory");        \
    reg_add(d, kind);                                                           \
    *desc = d;                                                                  \
    return DNNP_STATUS_OK;                                                      \
  }                                                                             \
  dnnp_status dnnp_##name##_destroy(htype desc) {                                \
    if (!reg_remove(desc, kind)) return fail(DNNP_STATUS_BAD_PARAM, #name ": not live"); \
    delete desc;                                                                \
    return DNNP_STATUS_OK;                                                      \
  }

DNNP_CREATE_DESTROY(tensor_desc, dnnp_tensor_desc, KIND_TENSOR)
DNNP_CREATE_DESTROY(filter_desc, dnnp_filter_desc, KIND_FILTER)
DNNP_CREATE_DESTROY(conv_desc, dnnp_conv_desc, KIND_CONV)
DNNP_CREATE_DESTROY(pooling_desc, dnnp_pooling_desc, KIND_POOL)

static bool elem_valid(dnnp_elem_type t) { return t == DNNP_F32 || t == DNNP_F64; }

dnnp_status dnnp_tensor_desc_set_ex(dnnp_tensor_desc d, dnnp_elem_type type, int64_t n,
                                    int64_t c, int64_t h, int64_t w, int64_t sn, int64_t sc,
                                    int64_t sh, int64_t sw) {
  if (!reg_has(d, KIND_TENSOR) || !elem_valid(type))
    return fail(DNNP_STATUS_BAD_PARAM, "tensor_desc_set: bad descriptor or element type");
  if (n < 1 || c < 1 || h < 1 || w < 1)
    return fail(DNNP_STATUS_BAD_PARAM, "tensor_desc_set: extents must be >= 1");
  d->elem = type;
  d->n = n; d->c = c; d->h = h; d->w = w;
  d->sn = sn; d->sc = sc; d->sh = sh; d->sw = sw;
  d->inj = -1;
  if (!span_ok(d)) {
    d->configured = false;
    return fail(DNNP_STATUS_BAD_PARAM, "tensor_desc_set: span exceeds 2^40 elements");
  }
  d->configured = true;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_tensor_desc_set(dnnp_tensor_desc d, dnnp_elem_type type, int64_t n, int64_t c,
                                 int64_t h, int64_t w) {
  if (n < 1 || c < 1 || h < 1 || w < 1)
    return fail(DNNP_STATUS_BAD_PARAM, "tensor_desc_set: extents must be >= 1");
  return dnnp_tensor_desc_set_ex(d, type, n, c, h, w, c * h * w, h * w, w, 1);
}

dnnp_status dnnp_tensor_desc_get(dnnp_tensor_desc d, dnnp_elem_type* type, int64_t* n,
                                 int64_t* c, int64_t* h, int64_t* w, int64_t* sn, int64_t* sc,
                                 int64_t* sh, int64_t* sw) {
  if (!reg_has(d, KIND_TENSOR) || !d->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "tensor_desc_get: not configured");
  if (!type || !n || !c || !h || !w || !sn || !sc || !sh || !sw)
    return fail(DNNP_STATUS_BAD_PARAM, "tensor_desc_get: NULL out-pointer");
  *type = d->elem;
  *n = d->n; *c = d->c; *h = d->h; *w = d->w;
  *sn = d->sn; *sc = d->sc; *sh = d->sh; *sw = d->sw;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_check_strides(const int64_t extents[4], const int64_t strides[4]) {
  if (!extents || !strides) return fail(DNNP_STATUS_BAD_PARAM, "NULL arrays");
  for (int i = 0; i < 4; i++)
    if (extents[i] < 1) return fail(DNNP_STATUS_BAD_PARAM, "extents must be >= 1");
  if (!injective(extents, strides)) return fail(DNNP_STATUS_BAD_PARAM, "strides alias");
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_filter_desc_set(dnnp_filter_desc d, dnnp_elem_type type, int64_t k, int64_t c,
                                 int64_t r, int64_t s) {
  if (!reg_has(d, KIND_FILTER) || !elem_valid(type))
    return fail(DNNP_STATUS_BAD_PARAM, "filter_desc_set: bad descriptor or element type");
  if (k < 1 || c < 1 || r < 1 || s < 1)
    return fail(DNNP_STATUS_BAD_PARAM, "filter_desc_set: extents must be >= 1");
  if ((__int128)k * c * r * s >= (__int128)kMaxSpanElems)
    return fail(DNNP_STATUS_BAD_PARAM, "filter_desc_set: too large");
  d->elem = type;
  d->k = k; d->c = c; d->r = r; d->s = s;
  d->configured = true;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_filter_desc_get(dnnp_filter_desc d, dnnp_elem_type* type, int64_t* k,
                                 int64_t* c, int64_t* r, int64_t* s) {
  if (!reg_has(d, KIND_FILTER) || !d->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "filter_desc_get: not configured");
  if (!type || !k || !c || !r || !s) return fail(DNNP_STATUS_BAD_PARAM, "NULL out-pointer");
  *type = d->elem;
  *k = d->k; *c = d->c; *r = d->r; *s = d->s;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_conv_desc_set(dnnp_conv_desc d, int64_t u, int64_t v, int64_t pad_h,
                               int64_t pad_w, dnnp_conv_mode mode, int accumulate) {
  if (!reg_has(d, KIND_CONV)) return fail(DNNP_STATUS_BAD_PARAM, "conv_desc_set: not live");
  if (u < 1 || v < 1 || pad_h < 0 || pad_w < 0)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_desc_set: stride < 1 or pad < 0");
  if (mode != DNNP_CONVOLUTION && mode != DNNP_CROSS_CORRELATION)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_desc_set: bad mode");
  d->u = u; d->v = v; d->pad_h = pad_h; d->pad_w = pad_w;
  d->mode = mode;
  d->accumulate = accumulate ? 1 : 0;
  d->configured = true;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_conv_desc_get(dnnp_conv_desc d, int64_t* u, int64_t* v, int64_t* pad_h,
                               int64_t* pad_w, dnnp_conv_mode* mode, int* accumulate) {
  if (!reg_has(d, KIND_CONV) || !d->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_desc_get: not configured");
  if (!u || !v || !pad_h || !pad_w || !mode || !accumulate)
    return fail(DNNP_STATUS_BAD_PARAM, "NULL out-pointer");
  *u = d->u; *v = d->v; *pad_h = d->pad_h; *pad_w = d->pad_w;
  *mode = d->mode;
  *accumulate = d->accumulate;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_pooling_desc_set(dnnp_pooling_desc d, dnnp_pool_kind kind, int64_t wh,
                                  int64_t ww, int64_t sh, int64_t sw, int64_t ph, int64_t pw) {
  if (!reg_has(d, KIND_POOL)) return fail(DNNP_STATUS_BAD_PARAM, "pooling_desc_set: not live");
  if (kind != DNNP_POOL_MAX && kind != DNNP_POOL_AVERAGE)
    return fail(DNNP_STATUS_BAD_PARAM, "pooling_desc_set: bad kind");
  if (wh < 1 || ww < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0)
    return fail(DNNP_STATUS_BAD_PARAM, "pooling_desc_set: bad window/stride/pad");
  d->kind = kind;
  d->wh = wh; d->ww = ww; d->sh = sh; d->sw = sw; d->ph = ph; d->pw = pw;
  d->configured = true;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_pooling_desc_get(dnnp_pooling_desc d, dnnp_pool_kind* kind, int64_t* wh,
                                  int64_t* ww, int64_t* sh, int64_t* sw, int64_t* ph,
                                  int64_t* pw) {
  if (!reg_has(d, KIND_POOL) || !d->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "pooling_desc_get: not configured");
  if (!kind || !wh || !ww || !sh || !sw || !ph || !pw)
    return fail(DNNP_STATUS_BAD_PARAM, "NULL out-pointer");
  *kind = d->kind;
  *wh = d->wh; *ww = d->ww; *sh = d->sh; *sw = d->sw; *ph = d->ph; *pw = d->pw;
  return DNNP_STATUS_OK;
}

// reference dnnp_capi.c:523-559 + dnnp_capi_bridge.py:189-198
dnnp_status dnnp_conv_output_shape(dnnp_tensor_desc x, dnnp_filter_desc f, dnnp_conv_desc conv,
                                   int64_t* n, int64_t* k, int64_t* p, int64_t* q) {
  {
    std::lock_guard<std::mutex> g(g_reg_lock);
    if (!g_created_once)
      return fail(DNNP_STATUS_BAD_PARAM, "conv_output_shape before the first dnnp_create");
  }
  if (!reg_has(x, KIND_TENSOR) || !x->configured || !reg_has(f, KIND_FILTER) ||
      !f->configured || !reg_has(conv, KIND_CONV) || !conv->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_output_shape: descriptor not configured");
  {
    const int64_t ext[4] = {x->n, x->c, x->h, x->w}, str[4] = {x->sn, x->sc, x->sh, x->sw};
    if (!injective(ext, str)) return fail(DNNP_STATUS_BAD_PARAM, "input strides alias");
  }
  int64_t P, Q;
  // conv_out_shape only checks channels and extents (not element types)
  if (x->c != f->c)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "input channels vs filter channels");
  if (!output_extent(x->h, f->r, conv->u, conv->pad_h, &P) ||
      !output_extent(x->w, f->s, conv->v, conv->pad_w, &Q))
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "convolution produces no output");
  if (n) *n = x->n;
  if (k) *k = f->k;
  if (p) *p = P;
  if (q) *q = Q;
  return DNNP_STATUS_OK;
}

// ------------------------------------------------------ convolution (hot)

dnnp_status dnnp_convolution_forward(dnnp_handle handle, const void* alpha, dnnp_tensor_desc xd,
                                     const void* x, dnnp_filter_desc fd, const void* f,
                                     dnnp_conv_desc cd, dnnp_engine engine, const void* beta,
                                     dnnp_tensor_desc yd, void* y) {
  if (!reg_has(handle, KIND_HANDLE) || !alpha || !beta)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_forward: bad handle or scalar pointer");
  if (!tensor_usable(xd, x) || !filter_usable(fd, f) || !tensor_usable(yd, y))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_forward: unusable descriptor or NULL buffer");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_forward: conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "conv_forward: bad engine");
  dnnp_status st;
  if ((st = bind_view(xd, "x")) || (st = bind_view(yd, "y"))) return st;
  double a = read_scalar(alpha, yd->elem), b = read_scalar(beta, yd->elem);
  int64_t P, Q;
  if ((st = conv_shape(xd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(yd, xd->n, fd->k, P, Q, xd->elem, "output"))) return st;
  if (cd->accumulate) b = 1.0;  // reference conv.py:573-574
  dnnp::ConvProblem pr = make_problem(xd, fd, cd, yd, P, Q);
  pr.engine = int(engine);
  if ((st = check_decode_range(pr))) return st;
  if ((st = explicit_guard(pr, engine, xd->elem, "forward"))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *dx, *df, *dy;
  size_t fbytes = size_t(fd->k * fd->c * fd->r * fd->s) * elem_size(fd->elem);
  {
    std::vector<ChunkBuf> cb = {{x, xd, false, true}, {y, yd, true, b != 0.0 || !dense_view(yd)}};
    if (pr.engine != DNNP_ENGINE_EXPLICIT && pipeline_ok(cb, xd->n)) {
      if ((st = sg.add(f, fbytes, false, true, &df))) return st;
      const size_t es = elem_size(xd->elem);
      return run_pipelined(handle->stream, sg, cb, xd->n, [&](int64_t n0, int64_t nb) {
        dnnp::ConvProblem q = pr;
        q.N = nb;
        q.x = shift_images(pr.x, nb);
        q.y = shift_images(pr.y, nb);
        return dnnp::conv_forward(q, dnnp::Dtype(xd->elem),
                                  static_cast<char*>(cb[0].dev) + n0 * xd->sn * es, df,
                                  static_cast<char*>(cb[1].dev) + n0 * yd->sn * es, a, b,
                                  handle->math, handle->stream);
      });
    }
  }
  if ((st = sg.add(x, span_bytes(xd), false, true, &dx))) return st;
  if ((st = sg.add(f, fbytes, false, true, &df))) return st;
  if ((st = sg.add(y, span_bytes(yd), true, b != 0.0 || !dense_view(yd), &dy))) return st;
  size_t need = 0;
  cudaError_t e = with_workspace([&] {
    return dnnp::conv_forward(pr, dnnp::Dtype(xd->elem), dx, df, dy, a, b, handle->math,
                              handle->stream);
  }, &need);
  if ((st = ws_status(e, need, "convolution_forward_ex"))) {
    sg.finish(cudaSuccess);
    return st;
  }
  return sg.finish(e);
}

dnnp_status dnnp_convolution_backward_data(dnnp_handle handle, dnnp_filter_desc fd,
                                           const void* f, dnnp_tensor_desc dyd, const void* dy,
                                           dnnp_conv_desc cd, dnnp_engine engine,
                                           dnnp_tensor_desc dxd, void* dx) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (!filter_usable(fd, f) || !tensor_usable(dyd, dy) || !tensor_usable(dxd, dx))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_backward_data: unusable descriptor or buffer");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "bad engine");
  dnnp_status st;
  if ((st = bind_view(dyd, "dy")) || (st = bind_view(dxd, "dx"))) return st;
  int64_t P, Q;
  if ((st = conv_shape(dxd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(dyd, dxd->n, fd->k, P, Q, dxd->elem, "output gradient"))) return st;
  dnnp::ConvProblem pr = make_problem(dxd, fd, cd, dyd, P, Q);
  if ((st = check_decode_range(pr))) return st;
  if ((st = explicit_guard(pr, engine, dxd->elem, "backward_data"))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *ddy, *dff, *ddx;
  size_t fbytes = size_t(fd->k * fd->c * fd->r * fd->s) * elem_size(fd->elem);
  if ((st = sg.add(f, fbytes, false, true, &dff))) return st;
  {
    std::vector<ChunkBuf> cb = {{dy, dyd, false, true},
                                {dx, dxd, true, cd->accumulate || !dense_view(dxd)}};
    if (pipeline_ok(cb, dxd->n)) {
      const size_t es = elem_size(dxd->elem);
      return run_pipelined(handle->stream, sg, cb, dxd->n, [&](int64_t n0, int64_t nb) {
        dnnp::ConvProblem q = pr;
        q.N = nb;
        q.x = shift_images(pr.x, nb);
        q.y = shift_images(pr.y, nb);
        return dnnp::conv_backward_data(q, dnnp::Dtype(dxd->elem),
                                        static_cast<char*>(cb[0].dev) + n0 * dyd->sn * es, dff,
                                        static_cast<char*>(cb[1].dev) + n0 * dxd->sn * es,
                                        cd->accumulate != 0, handle->math, handle->stream);
      });
    }
  }
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &ddy))) return st;
  if ((st = sg.add(dx, span_bytes(dxd), true, cd->accumulate || !dense_view(dxd), &ddx)))
    return st;
  size_t need = 0;
  cudaError_t e = with_workspace([&] {
    return dnnp::conv_backward_data(pr, dnnp::Dtype(dxd->elem), ddy, dff, ddx,
                                    cd->accumulate != 0, handle->math, handle->stream);
  }, &need);
  if ((st = ws_status(e, need, "convolution_backward_data_ex"))) {
    sg.finish(cudaSuccess);
    return st;
  }
  return sg.finish(e);
}

dnnp_status dnnp_convolution_backward_filter(dnnp_handle handle, dnnp_tensor_desc xd,
                                             const void* x, dnnp_tensor_desc dyd, const void* dy,
                                             dnnp_conv_desc cd, dnnp_engine engine,
                                             dnnp_filter_desc fd, void* df) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (!tensor_usable(xd, x) || !tensor_usable(dyd, dy) || !filter_usable(fd, df))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_backward_filter: unusable descriptor or buffer");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "bad engine");
  dnnp_status st;
  if ((st = bind_view(dyd, "dy")) || (st = bind_view(xd, "x"))) return st;
  int64_t P, Q;
  if ((st = conv_shape(xd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(dyd, xd->n, fd->k, P, Q, xd->elem, "output gradient"))) return st;
  dnnp::ConvProblem pr = make_problem(xd, fd, cd, dyd, P, Q);
  if ((st = check_decode_range(pr))) return st;
  if ((st = explicit_guard(pr, engine, xd->elem, "backward_filter"))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *dxx, *ddy, *ddf;
  size_t fbytes = size_t(fd->k * fd->c * fd->r * fd->s) * elem_size(fd->elem);
  {
    std::vector<ChunkBuf> cb = {{x, xd, false, true}, {dy, dyd, false, true}};
    if (pipeline_ok(cb, xd->n)) {
      if ((st = sg.add(df, fbytes, true, cd->accumulate != 0, &ddf))) return st;
      const size_t es = elem_size(xd->elem);
      // later chunks add to the first chunks' partial dW (IEEE fp32 / fp64)
      return run_pipelined(handle->stream, sg, cb, xd->n, [&](int64_t n0, int64_t nb) {
        dnnp::ConvProblem q = pr;
        q.N = nb;
        q.x = shift_images(pr.x, nb);
        q.y = shift_images(pr.y, nb);
        return dnnp::conv_backward_filter(q, dnnp::Dtype(xd->elem),
                                          static_cast<char*>(cb[1].dev) + n0 * dyd->sn * es,
                                          static_cast<char*>(cb[0].dev) + n0 * xd->sn * es, ddf,
                                          cd->accumulate != 0 || n0 > 0, handle->math,
                                          handle->stream);
      });
    }
  }
  if ((st = sg.add(x, span_bytes(xd), false, true, &dxx))) return st;
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &ddy))) return st;
  if ((st = sg.add(df, fbytes, true, cd->accumulate != 0, &ddf))) return st;
  size_t need = 0;
  cudaError_t e = with_workspace([&] {
    return dnnp::conv_backward_filter(pr, dnnp::Dtype(xd->elem), ddy, dxx, ddf,
                                      cd->accumulate != 0, handle->math, handle->stream);
  }, &need);
  if ((st = ws_status(e, need, "convolution_backward_filter_ex"))) {
    sg.finish(cudaSuccess);
    return st;
  }
  return sg.finish(e);
}

// reference dnnp_capi_bridge.py:116-124 + conv.py:754-760
dnnp_status dnnp_convolution_backward_bias(dnnp_handle handle, dnnp_tensor_desc dyd,
                                           const void* dy, dnnp_tensor_desc dbd, void* db) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (!tensor_usable(dyd, dy) || !tensor_usable(dbd, db))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_backward_bias: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(dbd, "db")) || (st = bind_view(dyd, "dy"))) return st;
  if (dbd->n != 1 || dbd->c != dyd->c || dbd->h != 1 || dbd->w != 1)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "bias gradient must be (1, %lld, 1, 1)",
                (long long)dyd->c);
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *ddy, *ddb;
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &ddy))) return st;
  if ((st = sg.add(db, span_bytes(dbd), true, !dense_view(dbd), &ddb))) return st;
  cudaError_t e = dnnp::conv_backward_bias(view_of(dyd), dnnp::Dtype(dyd->elem), ddy,
                                           view_of(dbd), dnnp::Dtype(dbd->elem), ddb,
                                           handle->stream);
  return sg.finish(e);
}

// ------------------------------------------------ fused backward (additive)

// dx and dw of one layer in one call (a training step's backward): the same
// checks as dnnp_convolution_backward_data / _backward_filter; on the
// tensor-core path dy is packed once for both GEMMs.
dnnp_status dnnp_convolution_backward(dnnp_handle handle, dnnp_filter_desc fd, const void* f,
                                      dnnp_tensor_desc dyd, const void* dy, dnnp_tensor_desc xd,
                                      const void* x, dnnp_conv_desc cd, dnnp_engine engine,
                                      dnnp_tensor_desc dxd, void* dx, dnnp_filter_desc dfd,
                                      void* df) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (!filter_usable(fd, f) || !tensor_usable(dyd, dy) || !tensor_usable(xd, x) ||
      !tensor_usable(dxd, dx) || !filter_usable(dfd, df))
    return fail(DNNP_STATUS_BAD_PARAM, "convolution_backward: unusable descriptor or buffer");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "bad engine");
  dnnp_status st;
  if ((st = bind_view(dyd, "dy")) || (st = bind_view(dxd, "dx")) || (st = bind_view(xd, "x")))
    return st;
  if (xd->n != dxd->n || xd->c != dxd->c || xd->h != dxd->h || xd->w != dxd->w ||
      xd->elem != dxd->elem)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "convolution_backward: x and dx differ in shape");
  if (fd->k != dfd->k || fd->c != dfd->c || fd->r != dfd->r || fd->s != dfd->s ||
      fd->elem != dfd->elem)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "convolution_backward: w and dw differ in shape");
  int64_t P, Q;
  if ((st = conv_shape(xd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(dyd, xd->n, fd->k, P, Q, xd->elem, "output gradient"))) return st;
  dnnp::ConvProblem pr = make_problem(xd, fd, cd, dyd, P, Q);
  if ((st = check_decode_range(pr))) return st;
  if ((st = explicit_guard(pr, engine, xd->elem, "backward"))) return st;
  if ((st = need_device())) return st;
  // dx must use dx's strides (same as x's here when the views agree)
  dnnp::ConvProblem prd = pr;
  prd.x = view_of(dxd);
  if (prd.x.sn != pr.x.sn || prd.x.sc != pr.x.sc || prd.x.sh != pr.x.sh || prd.x.sw != pr.x.sw) {
    // different x / dx layouts: the two plain calls
    if ((st = dnnp_convolution_backward_data(handle, fd, f, dyd, dy, cd, engine, dxd, dx))) return st;
    return dnnp_convolution_backward_filter(handle, xd, x, dyd, dy, cd, engine, dfd, df);
  }
  Stager sg(handle->stream);
  void *dff, *ddy, *dxx, *ddx, *ddf;
  size_t fbytes = size_t(fd->k * fd->c * fd->r * fd->s) * elem_size(fd->elem);
  if ((st = sg.add(f, fbytes, false, true, &dff))) return st;
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &ddy))) return st;
  if ((st = sg.add(x, span_bytes(xd), false, true, &dxx))) return st;
  if ((st = sg.add(dx, span_bytes(dxd), true, cd->accumulate || !dense_view(dxd), &ddx))) return st;
  if ((st = sg.add(df, fbytes, true, cd->accumulate != 0, &ddf))) return st;
  cudaError_t e = dnnp::conv_backward_both(pr, dnnp::Dtype(xd->elem), ddy, dff, dxx, ddx, ddf,
                                           cd->accumulate != 0, handle->math, handle->stream);
  return sg.finish(e);
}

// ------------------------------------------------ workspace (additive)

dnnp_status dnnp_convolution_forward_ex(dnnp_handle handle, const void* alpha,
                                        dnnp_tensor_desc xd, const void* x, dnnp_filter_desc fd,
                                        const void* f, dnnp_conv_desc cd, dnnp_engine engine,
                                        const void* beta, dnnp_tensor_desc yd, void* y,
                                        void* workspace, size_t workspace_bytes) {
  if (workspace_bytes && !workspace)
    return fail(DNNP_STATUS_BAD_PARAM, "convolution_forward_ex: NULL workspace");
  g_exws = ExWorkspace{workspace, workspace_bytes, true};
  const dnnp_status st = dnnp_convolution_forward(handle, alpha, xd, x, fd, f, cd, engine, beta, yd, y);
  g_exws = ExWorkspace{};
  return st;
}

dnnp_status dnnp_convolution_backward_data_ex(dnnp_handle handle, dnnp_filter_desc fd,
                                              const void* f, dnnp_tensor_desc dyd, const void* dy,
                                              dnnp_conv_desc cd, dnnp_engine engine,
                                              dnnp_tensor_desc dxd, void* dx, void* workspace,
                                              size_t workspace_bytes) {
  if (workspace_bytes && !workspace)
    return fail(DNNP_STATUS_BAD_PARAM, "convolution_backward_data_ex: NULL workspace");
  g_exws = ExWorkspace{workspace, workspace_bytes, true};
  const dnnp_status st = dnnp_convolution_backward_data(handle, fd, f, dyd, dy, cd, engine, dxd, dx);
  g_exws = ExWorkspace{};
  return st;
}

dnnp_status dnnp_convolution_backward_filter_ex(dnnp_handle handle, dnnp_tensor_desc xd,
                                                const void* x, dnnp_tensor_desc dyd,
                                                const void* dy, dnnp_conv_desc cd,
                                                dnnp_engine engine, dnnp_filter_desc fd, void* df,
                                                void* workspace, size_t workspace_bytes) {
  if (workspace_bytes && !workspace)
    return fail(DNNP_STATUS_BAD_PARAM, "convolution_backward_filter_ex: NULL workspace");
  g_exws = ExWorkspace{workspace, workspace_bytes, true};
  const dnnp_status st =
      dnnp_convolution_backward_filter(handle, xd, x, dyd, dy, cd, engine, fd, df);
  g_exws = ExWorkspace{};
  return st;
}

// Exact device workspace of one pass, without executing it: the pass is
// planned exactly as a real call would plan it (same tile choice, same
// scratch carve-outs), on fake device addresses, with its launches captured
// into a CUDA graph that is discarded unlaunched.  The returned size includes
// 1023 bytes of slack for the 1024-byte alignment the *_ex carve-out applies
// to the caller's base pointer (0 stays 0: nothing is carved).
dnnp_status dnnp_get_convolution_workspace_size(dnnp_handle handle, int pass,
                                                dnnp_tensor_desc xd, dnnp_filter_desc fd,
                                                dnnp_conv_desc cd, dnnp_tensor_desc yd,
                                                dnnp_engine engine, size_t* bytes) {
  if (!reg_has(handle, KIND_HANDLE) || !bytes || pass < 0 || pass > 2)
    return fail(DNNP_STATUS_BAD_PARAM, "get_convolution_workspace_size: bad arguments");
  if (!reg_has(xd, KIND_TENSOR) || !xd->configured || !reg_has(yd, KIND_TENSOR) ||
      !yd->configured || !reg_has(fd, KIND_FILTER) || !fd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "get_convolution_workspace_size: descriptor not configured");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "bad engine");
  dnnp_status st;
  if ((st = bind_view(xd, "x")) || (st = bind_view(yd, "y"))) return st;
  int64_t P, Q;
  if ((st = conv_shape(xd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(yd, xd->n, fd->k, P, Q, xd->elem, "output"))) return st;
  dnnp::ConvProblem pr = make_problem(xd, fd, cd, yd, P, Q);
  pr.engine = pass == 0 ? int(engine) : 2;
  if ((st = check_decode_range(pr))) return st;
  if ((st = explicit_guard(pr, engine, xd->elem, "workspace query"))) return st;
  if ((st = need_device())) return st;
  // one capture stream per device for queries (capture is thread-local)
  static std::mutex qmu;
  static std::map<int, cudaStream_t> qstreams;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t s = nullptr;
  {
    std::lock_guard<std::mutex> g(qmu);
    cudaStream_t& q = qstreams[dev];
    if (!q && cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking) != cudaSuccess) q = nullptr;
    s = q;
  }
  if (!s) return cuda_status(cudaErrorNotSupported, "get_convolution_workspace_size");
  // fake, aligned operand addresses: the captured launches never run
  void* const fx = reinterpret_cast<void*>(uintptr_t(1) << 42);
  void* const fy = reinterpret_cast<void*>(uintptr_t(2) << 42);
  void* const ff = reinterpret_cast<void*>(uintptr_t(3) << 42);
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  size_t need = 0;
  if (e == cudaSuccess) {
    dnnp::tc::dry_run_begin();
    const dnnp::Dtype dt = dnnp::Dtype(xd->elem);
    if (pass == 0)
      e = dnnp::conv_forward(pr, dt, fx, ff, fy, 1.0, 0.0, handle->math, s);
    else if (pass == 1)
      e = dnnp::conv_backward_data(pr, dt, fy, ff, fx, false, handle->math, s);
    else
      e = dnnp::conv_backward_filter(pr, dt, fy, fx, ff, false, handle->math, s);
    dnnp::tc::user_workspace_end(&need);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (graph) cudaGraphDestroy(graph);
    if (e == cudaSuccess) e = ce;
  }
  cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "get_convolution_workspace_size");
  *bytes = need ? need + 1023 : 0;
  return DNNP_STATUS_OK;
}

// Verification reference (additive; the GPU CLI's --verify): the pass as a
// plain fp64 loop nest on the device, independent of the implicit-GEMM
// kernels.  Device buffers only; out is a dense fp64 buffer of the pass's
// output extents (y: N K P Q, dx: N C H W, df: K C R S).
dnnp_status dnnp_convolution_verify_reference(dnnp_handle handle, int pass, dnnp_tensor_desc xd,
                                              dnnp_filter_desc fd, dnnp_conv_desc cd,
                                              dnnp_tensor_desc yd, const void* a, const void* b,
                                              double* out) {
  if (!reg_has(handle, KIND_HANDLE) || pass < 0 || pass > 2 || !a || !b || !out)
    return fail(DNNP_STATUS_BAD_PARAM, "convolution_verify_reference: bad arguments");
  if (!reg_has(xd, KIND_TENSOR) || !xd->configured || !reg_has(yd, KIND_TENSOR) ||
      !yd->configured || !reg_has(fd, KIND_FILTER) || !fd->configured ||
      !reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "convolution_verify_reference: descriptor not configured");
  dnnp_status st;
  if ((st = bind_view(xd, "x")) || (st = bind_view(yd, "y"))) return st;
  int64_t P, Q;
  if ((st = conv_shape(xd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(yd, xd->n, fd->k, P, Q, xd->elem, "output"))) return st;
  if ((st = need_device())) return st;
  const dnnp::ConvProblem pr = make_problem(xd, fd, cd, yd, P, Q);
  const cudaError_t e = dnnp::conv_verify_reference(pass, pr, dnnp::Dtype(xd->elem), a, b, out,
                                                    handle->stream);
  return cuda_status(e, "convolution_verify_reference");
}

// ------------------------------------------------ NCCL (additive)

static dnnp_status nccl_status(int r, const char* what) {
  if (r == 0) return DNNP_STATUS_OK;
  return fail(DNNP_STATUS_NOT_SUPPORTED, "%s: NCCL error %d (%s)", what, r,
              dnnp::nccl::error_string(r));
}

dnnp_status dnnp_nccl_unique_id(void* id, size_t bytes) {
  if (!id || bytes < 128) return fail(DNNP_STATUS_BAD_PARAM, "nccl_unique_id: need 128 bytes");
  const char* why = nullptr;
  if (!dnnp::nccl::available(&why)) return fail(DNNP_STATUS_NOT_SUPPORTED, "%s", why);
  return nccl_status(dnnp::nccl::unique_id(id), "ncclGetUniqueId");
}

dnnp_status dnnp_nccl_comm_create(dnnp_handle handle, const void* id, int nranks, int rank) {
  if (!reg_has(handle, KIND_HANDLE) || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(DNNP_STATUS_BAD_PARAM, "nccl_comm_create: bad arguments");
  const char* why = nullptr;
  if (!dnnp::nccl::available(&why)) return fail(DNNP_STATUS_NOT_SUPPORTED, "%s", why);
  dnnp_status st;
  if ((st = need_device())) return st;
  void* comm = nullptr;
  if ((st = nccl_status(dnnp::nccl::comm_init(&comm, id, nranks, rank), "ncclCommInitRank")))
    return st;
  if (handle->owns_comm) dnnp::nccl::comm_destroy(handle->comm);
  handle->comm = comm;
  handle->owns_comm = true;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_set_nccl_comm(dnnp_handle handle, void* comm) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (handle->owns_comm) dnnp::nccl::comm_destroy(handle->comm);
  handle->comm = comm;
  handle->owns_comm = false;
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_allreduce_sum(dnnp_handle handle, void* buf, int64_t count, dnnp_elem_type type) {
  if (!reg_has(handle, KIND_HANDLE) || !buf || count < 0 || !elem_valid(type))
    return fail(DNNP_STATUS_BAD_PARAM, "allreduce_sum: bad arguments");
  if (!handle->comm) return fail(DNNP_STATUS_BAD_PARAM, "allreduce_sum: no communicator on the handle");
  if (!is_device_ptr(buf)) return fail(DNNP_STATUS_BAD_PARAM, "allreduce_sum: device buffer required");
  return nccl_status(dnnp::nccl::allreduce_sum(buf, buf, size_t(count), type == DNNP_F64,
                                               handle->comm, handle->stream),
                     "ncclAllReduce");
}

// Backward-filter of a batch shard followed by ONE allreduce(sum) of dW over
// the handle's communicator: each rank passes its own N/G
// images of x and dy; df receives the gradient of the whole minibatch.
// Accumulate adds the reduced gradient to the prior df AFTER the reduction
// (reducing df itself would sum G copies of it).  Device buffers only.
dnnp_status dnnp_convolution_backward_filter_allreduce(dnnp_handle handle, dnnp_tensor_desc xd,
                                                       const void* x, dnnp_tensor_desc dyd,
                                                       const void* dy, dnnp_conv_desc cd,
                                                       dnnp_engine engine, dnnp_filter_desc fd,
                                                       void* df) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (!handle->comm)
    return fail(DNNP_STATUS_BAD_PARAM, "backward_filter_allreduce: no communicator on the handle");
  if (!tensor_usable(xd, x) || !tensor_usable(dyd, dy) || !filter_usable(fd, df))
    return fail(DNNP_STATUS_BAD_PARAM, "backward_filter_allreduce: unusable descriptor or buffer");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "bad engine");
  dnnp_status st;
  if ((st = bind_view(dyd, "dy")) || (st = bind_view(xd, "x"))) return st;
  int64_t P, Q;
  if ((st = conv_shape(xd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(dyd, xd->n, fd->k, P, Q, xd->elem, "output gradient"))) return st;
  dnnp::ConvProblem pr = make_problem(xd, fd, cd, dyd, P, Q);
  if ((st = check_decode_range(pr))) return st;
  if ((st = explicit_guard(pr, engine, xd->elem, "backward_filter_allreduce"))) return st;
  if ((st = need_device())) return st;
  if (!is_device_ptr(x) || !is_device_ptr(dy) || !is_device_ptr(df))
    return fail(DNNP_STATUS_BAD_PARAM, "backward_filter_allreduce: device buffers required");
  const size_t count = size_t(fd->k * fd->c * fd->r * fd->s);
  const bool f64 = fd->elem == DNNP_F64;
  const dnnp::Dtype dt = dnnp::Dtype(xd->elem);
  if (!cd->accumulate) {
    cudaError_t e = dnnp::conv_backward_filter(pr, dt, dy, x, df, false, handle->math, handle->stream);
    if (e != cudaSuccess) return cuda_status(e, "backward_filter_allreduce");
    return nccl_status(dnnp::nccl::allreduce_sum(df, df, count, f64, handle->comm, handle->stream),
                       "ncclAllReduce");
  }
  // accumulate: partial into scratch (non-accumulating), reduce it, then df += sum
  dnnp::tc::ScratchScope* sc = dnnp::tc::scratch_open(handle->stream);
  void* part = nullptr;
  cudaError_t e = dnnp::tc::scratch_alloc(sc, count * elem_size(fd->elem), &part);
  if (e == cudaSuccess)
    e = dnnp::conv_backward_filter(pr, dt, dy, x, part, false, handle->math, handle->stream);
  if (e != cudaSuccess) {
    dnnp::tc::scratch_close(sc);
    return cuda_status(e, "backward_filter_allreduce");
  }
  st = nccl_status(dnnp::nccl::allreduce_sum(part, part, count, f64, handle->comm, handle->stream),
                   "ncclAllReduce");
  if (!st) {
    const View4 v{1, int64_t(count), 1, 1, int64_t(count), 1, 1, 1};
    st = cuda_status(dnnp::transform(dt, v, part, v, df, 1.0, 1.0, handle->stream),
                     "backward_filter_allreduce accumulate");
  }
  dnnp::tc::scratch_close(sc);
  return st;
}

// ------------------------------------------------ fused epilogues (additive)

static bool act_valid(dnnp_activation_kind k);
static dnnp_status check_like(dnnp_tensor_desc a, dnnp_tensor_desc b, const char* what);

dnnp_status dnnp_convolution_bias_activation_forward(
    dnnp_handle handle, const void* alpha, dnnp_tensor_desc xd, const void* x, dnnp_filter_desc fd,
    const void* f, dnnp_conv_desc cd, dnnp_engine engine, const void* beta, dnnp_tensor_desc bd,
    const void* bias, int activation, dnnp_tensor_desc yd, void* y) {
  if (!reg_has(handle, KIND_HANDLE) || !alpha || !beta)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_bias_act: bad handle or scalar pointer");
  if (activation != DNNP_ACTIVATION_NONE && !act_valid(dnnp_activation_kind(activation)))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_bias_act: bad activation kind");
  if (!tensor_usable(xd, x) || !filter_usable(fd, f) || !tensor_usable(yd, y))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_bias_act: unusable descriptor or NULL buffer");
  if ((bd == nullptr) != (bias == nullptr) || (bd && !tensor_usable(bd, bias)))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_bias_act: bias descriptor and buffer must pair");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv_bias_act: conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "conv_bias_act: bad engine");
  dnnp_status st;
  if ((st = bind_view(xd, "x")) || (st = bind_view(yd, "y"))) return st;
  if (bd && (st = bind_view(bd, "bias"))) return st;
  double a = read_scalar(alpha, yd->elem), b = read_scalar(beta, yd->elem);
  int64_t P, Q;
  if ((st = conv_shape(xd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(yd, xd->n, fd->k, P, Q, xd->elem, "output"))) return st;
  if (bd && (bd->n != 1 || bd->c != fd->k || bd->h != 1 || bd->w != 1 || bd->elem != yd->elem))
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "bias must be (1, %lld, 1, 1) of y's type",
                (long long)fd->k);
  if (cd->accumulate) b = 1.0;  // reference conv.py:573-574
  dnnp::ConvProblem pr = make_problem(xd, fd, cd, yd, P, Q);
  if ((st = check_decode_range(pr))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *dx, *df, *dy, *db = nullptr;
  size_t fbytes = size_t(fd->k * fd->c * fd->r * fd->s) * elem_size(fd->elem);
  if ((st = sg.add(x, span_bytes(xd), false, true, &dx))) return st;
  if ((st = sg.add(f, fbytes, false, true, &df))) return st;
  if (bd && (st = sg.add(bias, span_bytes(bd), false, true, &db))) return st;
  if ((st = sg.add(y, span_bytes(yd), true, b != 0.0 || !dense_view(yd), &dy))) return st;
  dnnp::ConvEpilogue ep;
  ep.act = activation;
  if (bd) {
    ep.bias = db;
    ep.biasv = view_of(bd);
    ep.bias_stride = ep.biasv.sc;
  }
  cudaError_t e = dnnp::conv_forward_fused(pr, dnnp::Dtype(xd->elem), dx, df, dy, a, b,
                                           handle->math, ep, handle->stream);
  return sg.finish(e);
}

dnnp_status dnnp_convolution_backward_data_activation(
    dnnp_handle handle, dnnp_filter_desc fd, const void* f, dnnp_tensor_desc dyd, const void* dy,
    dnnp_conv_desc cd, dnnp_engine engine, dnnp_activation_kind activation, dnnp_tensor_desc gd,
    const void* g, dnnp_tensor_desc dxd, void* dx) {
  if (!reg_has(handle, KIND_HANDLE) || !act_valid(activation))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_bwd_data_act: bad handle or activation kind");
  if (!filter_usable(fd, f) || !tensor_usable(dyd, dy) || !tensor_usable(dxd, dx) ||
      !tensor_usable(gd, g))
    return fail(DNNP_STATUS_BAD_PARAM, "conv_bwd_data_act: unusable descriptor or buffer");
  if (!reg_has(cd, KIND_CONV) || !cd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "conv descriptor not configured");
  if (!engine_valid(engine)) return fail(DNNP_STATUS_BAD_PARAM, "bad engine");
  dnnp_status st;
  if ((st = bind_view(dyd, "dy")) || (st = bind_view(dxd, "dx")) || (st = bind_view(gd, "y")))
    return st;
  int64_t P, Q;
  if ((st = conv_shape(dxd, fd, cd, &P, &Q))) return st;
  if ((st = check_out(dyd, dxd->n, fd->k, P, Q, dxd->elem, "output gradient"))) return st;
  if ((st = check_like(gd, dxd, "conv_bwd_data_act"))) return st;
  dnnp::ConvProblem pr = make_problem(dxd, fd, cd, dyd, P, Q);
  if ((st = check_decode_range(pr))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *ddy, *dff, *ddx, *dg;
  size_t fbytes = size_t(fd->k * fd->c * fd->r * fd->s) * elem_size(fd->elem);
  if ((st = sg.add(f, fbytes, false, true, &dff))) return st;
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &ddy))) return st;
  if ((st = sg.add(g, span_bytes(gd), false, true, &dg))) return st;
  if ((st = sg.add(dx, span_bytes(dxd), true, cd->accumulate || !dense_view(dxd), &ddx)))
    return st;
  dnnp::ConvEpilogue ep;
  ep.gate = activation;
  ep.gatep = dg;
  ep.gatev = view_of(gd);
  cudaError_t e = dnnp::conv_backward_data_fused(pr, dnnp::Dtype(dxd->elem), ddy, dff, ddx,
                                                 cd->accumulate != 0, handle->math, ep,
                                                 handle->stream);
  return sg.finish(e);
}

// ------------------------------------------------ activation / softmax

static bool act_valid(dnnp_activation_kind k) {
  return k == DNNP_ACTIVATION_SIGMOID || k == DNNP_ACTIVATION_RELU || k == DNNP_ACTIVATION_TANH;
}
static bool softmax_valid(dnnp_softmax_mode m) {
  return m == DNNP_SOFTMAX_PER_IMAGE || m == DNNP_SOFTMAX_PER_SPATIAL;
}
// _check_like (reference nnops.py:45-51)
static dnnp_status check_like(dnnp_tensor_desc a, dnnp_tensor_desc b, const char* what) {
  if (!same_extents(a, b)) return fail(DNNP_STATUS_SHAPE_MISMATCH, "%s: extents differ", what);
  if (a->elem != b->elem) return fail(DNNP_STATUS_SHAPE_MISMATCH, "%s: element types differ", what);
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_activation_forward(dnnp_handle handle, dnnp_activation_kind kind,
                                    dnnp_tensor_desc xd, const void* x, dnnp_tensor_desc yd,
                                    void* y) {
  if (!reg_has(handle, KIND_HANDLE) || !act_valid(kind))
    return fail(DNNP_STATUS_BAD_PARAM, "bad handle or activation kind");
  if (!tensor_usable(xd, x) || !tensor_usable(yd, y))
    return fail(DNNP_STATUS_BAD_PARAM, "activation: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(xd, "x")) || (st = bind_view(yd, "y"))) return st;
  if ((st = check_like(xd, yd, "activation"))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *dxp, *dyp;
  if ((st = sg.add(x, span_bytes(xd), false, true, &dxp))) return st;
  if ((st = sg.add(y, span_bytes(yd), true, !dense_view(yd), &dyp))) return st;
  return sg.finish(dnnp::activation_forward(kind, dnnp::Dtype(xd->elem), view_of(xd), dxp,
                                            view_of(yd), dyp, handle->stream));
}

dnnp_status dnnp_activation_backward(dnnp_handle handle, dnnp_activation_kind kind,
                                     dnnp_tensor_desc yd, const void* y, dnnp_tensor_desc dyd,
                                     const void* dy, dnnp_tensor_desc dxd, void* dx) {
  if (!reg_has(handle, KIND_HANDLE) || !act_valid(kind))
    return fail(DNNP_STATUS_BAD_PARAM, "bad handle or activation kind");
  if (!tensor_usable(yd, y) || !tensor_usable(dyd, dy) || !tensor_usable(dxd, dx))
    return fail(DNNP_STATUS_BAD_PARAM, "activation backward: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(yd, "y")) || (st = bind_view(dyd, "dy")) || (st = bind_view(dxd, "dx")))
    return st;
  if ((st = check_like(yd, dyd, "activation backward")) ||
      (st = check_like(yd, dxd, "activation backward")))
    return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *a, *b, *c;
  if ((st = sg.add(y, span_bytes(yd), false, true, &a))) return st;
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &b))) return st;
  if ((st = sg.add(dx, span_bytes(dxd), true, !dense_view(dxd), &c))) return st;
  return sg.finish(dnnp::activation_backward(kind, dnnp::Dtype(yd->elem), view_of(yd), a,
                                             view_of(dyd), b, view_of(dxd), c, handle->stream));
}

dnnp_status dnnp_softmax_forward(dnnp_handle handle, dnnp_softmax_mode mode, dnnp_tensor_desc xd,
                                 const void* x, dnnp_tensor_desc yd, void* y) {
  if (!reg_has(handle, KIND_HANDLE) || !softmax_valid(mode))
    return fail(DNNP_STATUS_BAD_PARAM, "bad handle or softmax mode");
  if (!tensor_usable(xd, x) || !tensor_usable(yd, y))
    return fail(DNNP_STATUS_BAD_PARAM, "softmax: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(xd, "x")) || (st = bind_view(yd, "y"))) return st;
  if ((st = check_like(xd, yd, "softmax"))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *a, *b;
  if ((st = sg.add(x, span_bytes(xd), false, true, &a))) return st;
  if ((st = sg.add(y, span_bytes(yd), true, !dense_view(yd), &b))) return st;
  return sg.finish(dnnp::softmax_forward(mode, dnnp::Dtype(xd->elem), view_of(xd), a,
                                         view_of(yd), b, handle->stream));
}

dnnp_status dnnp_softmax_backward(dnnp_handle handle, dnnp_softmax_mode mode,
                                  dnnp_tensor_desc yd, const void* y, dnnp_tensor_desc dyd,
                                  const void* dy, dnnp_tensor_desc dxd, void* dx) {
  if (!reg_has(handle, KIND_HANDLE) || !softmax_valid(mode))
    return fail(DNNP_STATUS_BAD_PARAM, "bad handle or softmax mode");
  if (!tensor_usable(yd, y) || !tensor_usable(dyd, dy) || !tensor_usable(dxd, dx))
    return fail(DNNP_STATUS_BAD_PARAM, "softmax backward: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(yd, "y")) || (st = bind_view(dyd, "dy")) || (st = bind_view(dxd, "dx")))
    return st;
  if ((st = check_like(yd, dyd, "softmax backward")) ||
      (st = check_like(yd, dxd, "softmax backward")))
    return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *a, *b, *c;
  if ((st = sg.add(y, span_bytes(yd), false, true, &a))) return st;
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &b))) return st;
  if ((st = sg.add(dx, span_bytes(dxd), true, !dense_view(dxd), &c))) return st;
  return sg.finish(dnnp::softmax_backward(mode, dnnp::Dtype(yd->elem), view_of(yd), a,
                                          view_of(dyd), b, view_of(dxd), c, handle->stream));
}

// ------------------------------------------------------------------ pooling

// pool_out_shape + the EmptyWindow scan of pool_forward (nnops.py:142-200):
// a window lying entirely in the padding is an error.
static dnnp_status pool_shape(dnnp_pooling_desc pd, dnnp_tensor_desc xd, dnnp::PoolProblem* pp) {
  int64_t P, Q;
  if (!output_extent(xd->h, pd->wh, pd->sh, pd->ph, &P) ||
      !output_extent(xd->w, pd->ww, pd->sw, pd->pw, &Q))
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "pooling produces no output");
  pp->kind = pd->kind == DNNP_POOL_MAX ? 0 : 1;
  pp->wh = pd->wh; pp->ww = pd->ww; pp->sh = pd->sh; pp->sw = pd->sw;
  pp->ph = pd->ph; pp->pw = pd->pw; pp->P = P; pp->Q = Q;
  return DNNP_STATUS_OK;
}
static dnnp_status pool_windows_nonempty(const dnnp::PoolProblem& pp, int64_t H, int64_t W) {
  for (int64_t p = 0; p < pp.P; p++) {
    int64_t hs = p * pp.sh - pp.ph;
    if (std::max<int64_t>(0, hs) >= std::min<int64_t>(H, hs + pp.wh))
      return fail(DNNP_STATUS_SHAPE_MISMATCH, "pooling window row %lld lies in padding",
                  (long long)p);
  }
  for (int64_t q = 0; q < pp.Q; q++) {
    int64_t ws = q * pp.sw - pp.pw;
    if (std::max<int64_t>(0, ws) >= std::min<int64_t>(W, ws + pp.ww))
      return fail(DNNP_STATUS_SHAPE_MISMATCH, "pooling window col %lld lies in padding",
                  (long long)q);
  }
  return DNNP_STATUS_OK;
}

dnnp_status dnnp_pooling_forward(dnnp_handle handle, dnnp_pooling_desc pd, dnnp_tensor_desc xd,
                                 const void* x, dnnp_tensor_desc yd, void* y, int64_t* argmax) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (!reg_has(pd, KIND_POOL) || !pd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "pooling descriptor not configured");
  if (!tensor_usable(xd, x) || !tensor_usable(yd, y))
    return fail(DNNP_STATUS_BAD_PARAM, "pooling: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(xd, "x")) || (st = bind_view(yd, "y"))) return st;
  dnnp::PoolProblem pp;
  if ((st = pool_shape(pd, xd, &pp))) return st;
  if (yd->n != xd->n || yd->c != xd->c || yd->h != pp.P || yd->w != pp.Q || yd->elem != xd->elem)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "pooled output must be (%lld,%lld,%lld,%lld)",
                (long long)xd->n, (long long)xd->c, (long long)pp.P, (long long)pp.Q);
  if ((st = pool_windows_nonempty(pp, xd->h, xd->w))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *a, *b, *am = nullptr;
  if ((st = sg.add(x, span_bytes(xd), false, true, &a))) return st;
  if ((st = sg.add(y, span_bytes(yd), true, !dense_view(yd), &b))) return st;
  if (argmax && pp.kind == 0) {
    size_t abytes = size_t(yd->n * yd->c * yd->h * yd->w) * 8;
    if ((st = sg.add(argmax, abytes, true, false, &am))) return st;
  }
  return sg.finish(dnnp::pool_forward(pp, dnnp::Dtype(xd->elem), view_of(xd), a, view_of(yd), b,
                                      static_cast<int64_t*>(am), handle->stream));
}

dnnp_status dnnp_pooling_backward(dnnp_handle handle, dnnp_pooling_desc pd, dnnp_tensor_desc yd,
                                  const void* y, dnnp_tensor_desc dyd, const void* dy,
                                  dnnp_tensor_desc xd, const void* x, dnnp_tensor_desc dxd,
                                  void* dx, const int64_t* argmax) {
  if (!reg_has(handle, KIND_HANDLE)) return fail(DNNP_STATUS_BAD_PARAM, "bad handle");
  if (!reg_has(pd, KIND_POOL) || !pd->configured)
    return fail(DNNP_STATUS_BAD_PARAM, "pooling descriptor not configured");
  if (!tensor_usable(yd, y) || !tensor_usable(dyd, dy) || !tensor_usable(xd, x) ||
      !tensor_usable(dxd, dx))
    return fail(DNNP_STATUS_BAD_PARAM, "pooling backward: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(yd, "y")) || (st = bind_view(dyd, "dy")) || (st = bind_view(xd, "x")) ||
      (st = bind_view(dxd, "dx")))
    return st;
  dnnp::PoolProblem pp;
  if ((st = pool_shape(pd, xd, &pp))) return st;
  if ((st = check_like(xd, dxd, "pool backward"))) return st;
  for (dnnp_tensor_desc t : {yd, dyd})
    if (t->n != xd->n || t->c != xd->c || t->h != pp.P || t->w != pp.Q || t->elem != xd->elem)
      return fail(DNNP_STATUS_SHAPE_MISMATCH, "pooled gradient shape mismatch");
  if (pp.kind == 0 && !argmax)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "max pooling backward needs the forward argmax");
  if (pp.kind == 1 && (st = pool_windows_nonempty(pp, xd->h, xd->w))) return st;
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *b, *d, *am = nullptr;
  if ((st = sg.add(dy, span_bytes(dyd), false, true, &b))) return st;
  if ((st = sg.add(dx, span_bytes(dxd), true, !dense_view(dxd), &d))) return st;
  if (pp.kind == 0) {
    size_t abytes = size_t(yd->n * yd->c * yd->h * yd->w) * 8;
    if ((st = sg.add(argmax, abytes, false, true, &am))) return st;
  }
  return sg.finish(dnnp::pool_backward(pp, dnnp::Dtype(xd->elem), view_of(dyd), b, view_of(dxd),
                                       d, static_cast<const int64_t*>(am), handle->stream));
}

// --------------------------------------------------------- tensor utilities

// reference tensor.py:241-251 (np.may_share_memory on the two buffers)
dnnp_status dnnp_transform(dnnp_handle handle, const void* alpha, dnnp_tensor_desc sd,
                           const void* src, const void* beta, dnnp_tensor_desc dd, void* dst) {
  if (!reg_has(handle, KIND_HANDLE) || !alpha || !beta)
    return fail(DNNP_STATUS_BAD_PARAM, "transform: bad handle or scalar pointer");
  if (!tensor_usable(sd, src) || !tensor_usable(dd, dst))
    return fail(DNNP_STATUS_BAD_PARAM, "transform: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(sd, "src")) || (st = bind_view(dd, "dst"))) return st;
  double a = read_scalar(alpha, dd->elem), b = read_scalar(beta, dd->elem);
  if ((st = check_like(sd, dd, "transform"))) return st;
  {
    auto s0 = reinterpret_cast<uintptr_t>(src), s1 = s0 + span_bytes(sd);
    auto d0 = reinterpret_cast<uintptr_t>(dst), d1 = d0 + span_bytes(dd);
    if (s0 < d1 && d0 < s1)
      return fail(DNNP_STATUS_SHAPE_MISMATCH, "transform requires disjoint buffers");
  }
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *a_, *b_;
  if ((st = sg.add(src, span_bytes(sd), false, true, &a_))) return st;
  if ((st = sg.add(dst, span_bytes(dd), true, b != 0.0 || !dense_view(dd), &b_))) return st;
  return sg.finish(dnnp::transform(dnnp::Dtype(dd->elem), view_of(sd), a_, view_of(dd), b_, a, b,
                                   handle->stream));
}

// reference tensor.py:254-271
dnnp_status dnnp_add_broadcast(dnnp_handle handle, const void* alpha, dnnp_tensor_desc bd,
                               const void* bias, const void* beta, dnnp_tensor_desc od,
                               void* out) {
  if (!reg_has(handle, KIND_HANDLE) || !alpha || !beta)
    return fail(DNNP_STATUS_BAD_PARAM, "add_broadcast: bad handle or scalar pointer");
  if (!tensor_usable(bd, bias) || !tensor_usable(od, out))
    return fail(DNNP_STATUS_BAD_PARAM, "add_broadcast: unusable descriptor or buffer");
  dnnp_status st;
  if ((st = bind_view(bd, "bias")) || (st = bind_view(od, "out"))) return st;
  double a = read_scalar(alpha, od->elem), b = read_scalar(beta, od->elem);
  if (bd->elem != od->elem)
    return fail(DNNP_STATUS_SHAPE_MISMATCH, "add_broadcast: element types differ");
  const int64_t be[4] = {bd->n, bd->c, bd->h, bd->w}, oe[4] = {od->n, od->c, od->h, od->w};
  for (int i = 0; i < 4; i++)
    if (be[i] != 1 && be[i] != oe[i])
      return fail(DNNP_STATUS_SHAPE_MISMATCH, "bias does not broadcast onto the output");
  if ((st = need_device())) return st;
  Stager sg(handle->stream);
  void *a_, *b_;
  if ((st = sg.add(bias, span_bytes(bd), false, true, &a_))) return st;
  if ((st = sg.add(out, span_bytes(od), true, b != 0.0 || !dense_view(od), &b_))) return st;
  return sg.finish(dnnp::add_broadcast(dnnp::Dtype(od->elem), view_of(bd), a_, view_of(od), b_,
                                       a, b, handle->stream));
}

}  // extern "C"
