"""ctypes binding of libdnnp.so (the C ABI declared in include/dnnp.h).

The shared library is built in-tree by __graft_entry__.build() (or
`make -C paper_1410_0759_b200/csrc`).  There is no Python or CPU compute
fallback: if the library is missing, importing a compute entry raises.
"""
import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DNNP_LIB_PATH") or os.path.join(_HERE, "libdnnp.so")  # override: A/B builds

OK, BAD_PARAM, SHAPE_MISMATCH, ALLOC_FAILED, NOT_SUPPORTED = 0, 1, 2, 3, 4
F32, F64 = 0, 1

_lib = None
_lock = threading.Lock()

c_i64 = ctypes.c_int64
c_i64p = ctypes.POINTER(ctypes.c_int64)
vp = ctypes.c_void_p

# name -> argtypes (all return dnnp_status as int unless listed in _RESTYPES)
_SIGS = {
    "dnnp_version": [],
    "dnnp_status_string": [ctypes.c_int],
    "dnnp_last_error": [],
    "dnnp_kernel_launch_count": [],
    "dnnp_reload_tuning": [],
    "dnnp_magic_divider": [ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32),
                           ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int)],
    "dnnp_kernel_timing": [ctypes.c_int],
    "dnnp_scratch_high_water": [ctypes.c_int],
    "dnnp_kernel_times": [ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int), ctypes.c_int],
    "dnnp_create": [ctypes.POINTER(vp)],
    "dnnp_destroy": [vp],
    "dnnp_set_threads": [vp, c_i64],
    "dnnp_get_threads": [vp, c_i64p],
    "dnnp_set_stream": [vp, vp],
    "dnnp_get_stream": [vp, ctypes.POINTER(vp)],
    "dnnp_synchronize": [vp],
    "dnnp_set_math": [vp, ctypes.c_int],
    "dnnp_get_math": [vp, ctypes.POINTER(ctypes.c_int)],
    "dnnp_tensor_desc_create": [ctypes.POINTER(vp)],
    "dnnp_tensor_desc_destroy": [vp],
    "dnnp_tensor_desc_set": [vp, ctypes.c_int, c_i64, c_i64, c_i64, c_i64],
    "dnnp_tensor_desc_set_ex": [vp, ctypes.c_int] + [c_i64] * 8,
    "dnnp_tensor_desc_get": [vp, ctypes.POINTER(ctypes.c_int)] + [c_i64p] * 8,
    "dnnp_check_strides": [c_i64p, c_i64p],
    "dnnp_filter_desc_create": [ctypes.POINTER(vp)],
    "dnnp_filter_desc_destroy": [vp],
    "dnnp_filter_desc_set": [vp, ctypes.c_int, c_i64, c_i64, c_i64, c_i64],
    "dnnp_filter_desc_get": [vp, ctypes.POINTER(ctypes.c_int)] + [c_i64p] * 4,
    "dnnp_conv_desc_create": [ctypes.POINTER(vp)],
    "dnnp_conv_desc_destroy": [vp],
    "dnnp_conv_desc_set": [vp, c_i64, c_i64, c_i64, c_i64, ctypes.c_int, ctypes.c_int],
    "dnnp_conv_desc_get": [vp, c_i64p, c_i64p, c_i64p, c_i64p, ctypes.POINTER(ctypes.c_int),
                           ctypes.POINTER(ctypes.c_int)],
    "dnnp_pooling_desc_create": [ctypes.POINTER(vp)],
    "dnnp_pooling_desc_destroy": [vp],
    "dnnp_pooling_desc_set": [vp, ctypes.c_int] + [c_i64] * 6,
    "dnnp_pooling_desc_get": [vp, ctypes.POINTER(ctypes.c_int)] + [c_i64p] * 6,
    "dnnp_conv_output_shape": [vp, vp, vp, c_i64p, c_i64p, c_i64p, c_i64p],
    "dnnp_convolution_forward": [vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp],
    "dnnp_convolution_backward_data": [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp],
    "dnnp_convolution_backward": [vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp, vp],
    "dnnp_get_convolution_workspace_size": [vp, ctypes.c_int, vp, vp, vp, vp, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_size_t)],
    "dnnp_convolution_forward_ex": [vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp, vp,
                                    ctypes.c_size_t],
    "dnnp_convolution_backward_data_ex": [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp,
                                          ctypes.c_size_t],
    "dnnp_convolution_backward_filter_ex": [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp,
                                            ctypes.c_size_t],
    "dnnp_convolution_bias_activation_forward": [vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp,
                                                 vp, vp, ctypes.c_int, vp, vp],
    "dnnp_convolution_backward_data_activation": [vp, vp, vp, vp, vp, vp, ctypes.c_int,
                                                  ctypes.c_int, vp, vp, vp, vp],
    "dnnp_convolution_backward_filter": [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp],
    "dnnp_convolution_backward_bias": [vp, vp, vp, vp, vp],
    "dnnp_convolution_verify_reference": [vp, ctypes.c_int, vp, vp, vp, vp, vp, vp, vp],
    "dnnp_nccl_unique_id": [vp, ctypes.c_size_t],
    "dnnp_nccl_comm_create": [vp, vp, ctypes.c_int, ctypes.c_int],
    "dnnp_set_nccl_comm": [vp, vp],
    "dnnp_allreduce_sum": [vp, vp, c_i64, ctypes.c_int],
    "dnnp_convolution_backward_filter_allreduce": [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp],
    "dnnp_activation_forward": [vp, ctypes.c_int, vp, vp, vp, vp],
    "dnnp_activation_backward": [vp, ctypes.c_int, vp, vp, vp, vp, vp, vp],
    "dnnp_softmax_forward": [vp, ctypes.c_int, vp, vp, vp, vp],
    "dnnp_softmax_backward": [vp, ctypes.c_int, vp, vp, vp, vp, vp, vp],
    "dnnp_pooling_forward": [vp, vp, vp, vp, vp, vp, vp],
    "dnnp_pooling_backward": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
    "dnnp_transform": [vp, vp, vp, vp, vp, vp, vp],
    "dnnp_add_broadcast": [vp, vp, vp, vp, vp, vp, vp],
}
_RESTYPES = {
    "dnnp_reload_tuning": None,
    "dnnp_version": c_i64,
    "dnnp_status_string": ctypes.c_char_p,
    "dnnp_last_error": ctypes.c_char_p,
    "dnnp_kernel_launch_count": c_i64,
    "dnnp_scratch_high_water": c_i64,
}
SYMBOLS = tuple(_SIGS)


def lib():
    """The loaded libdnnp.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = L
    return _lib


def last_error():
    msg = lib().dnnp_last_error()
    return msg.decode() if msg else ""


def check(status, what=""):
    if status != OK:
        cls = errors.STATUS_ERRORS.get(status, errors.DnnpError)
        raise cls(f"{what}: {last_error()}" if what else last_error())


_handles = threading.local()


def handle():
    """Per-thread dnnp handle (handles are cheap; streams are per call)."""
    h = getattr(_handles, "h", None)
    if h is None:
        h = vp()
        check(lib().dnnp_create(ctypes.byref(h)), "dnnp_create")
        _handles.h = h
    return h


def set_stream(stream_ptr):
    """Bind this thread's handle to a cudaStream_t (skipped when unchanged)."""
    if getattr(_handles, "stream", -1) == stream_ptr:
        return
    check(lib().dnnp_set_stream(handle(), vp(stream_ptr)), "dnnp_set_stream")
    _handles.stream = stream_ptr


def set_math(mode):
    check(lib().dnnp_set_math(handle(), int(mode)), "dnnp_set_math")


def get_math():
    v = ctypes.c_int()
    check(lib().dnnp_get_math(handle(), ctypes.byref(v)), "dnnp_get_math")
    return v.value


def reload_tuning():
    """Re-read the DNNP_* kernel-variant switches (cached by the library)."""
    lib().dnnp_reload_tuning()


def magic_divider(d):
    """(multiplier, shift, add_indicator) of the kernels' index-decode divider."""
    m, s, a = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_int()
    check(lib().dnnp_magic_divider(int(d), ctypes.byref(m), ctypes.byref(s), ctypes.byref(a)),
          "dnnp_magic_divider")
    return int(m.value), int(s.value), bool(a.value)


def kernel_launch_count():
    return int(lib().dnnp_kernel_launch_count())


def kernel_timing(enable=True, only=None):
    """Start (clearing) or stop CUDA-event timing of the main GEMM kernels;
    only=i times just the i-th main launch after this call."""
    if not enable:
        lib().dnnp_kernel_timing(0)
    else:
        lib().dnnp_kernel_timing(1 if only is None else 2 + int(only))


def scratch_high_water(reset=False):
    """Largest scratch footprint (bytes) of any operation since the last reset."""
    return int(lib().dnnp_scratch_high_water(1 if reset else 0))


def kernel_times():
    """[(ms, tag), ...] of the main GEMM kernels timed since kernel_timing(True)."""
    n = int(lib().dnnp_kernel_times(None, None, 0))
    ms = (ctypes.c_float * max(n, 1))()
    tags = (ctypes.c_int * max(n, 1))()
    lib().dnnp_kernel_times(ms, tags, n)
    return [(float(ms[i]), int(tags[i])) for i in range(n)]


class TensorDescHandle:
    """RAII wrapper of a C tensor descriptor."""

    def __init__(self, elem, extents, strides):
        L = lib()
        self.h = vp()
        check(L.dnnp_tensor_desc_create(ctypes.byref(self.h)), "tensor_desc_create")
        st = L.dnnp_tensor_desc_set_ex(self.h, elem, *[int(e) for e in extents],
                                       *[int(s) for s in strides])
        if st != OK:
            L.dnnp_tensor_desc_destroy(self.h)
            self.h = None
            check(st, "tensor_desc_set_ex")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dnnp_tensor_desc_destroy(self.h)


class FilterDescHandle:
    def __init__(self, elem, k, c, r, s):
        L = lib()
        self.h = vp()
        check(L.dnnp_filter_desc_create(ctypes.byref(self.h)), "filter_desc_create")
        st = L.dnnp_filter_desc_set(self.h, elem, k, c, r, s)
        if st != OK:
            L.dnnp_filter_desc_destroy(self.h)
            self.h = None
            check(st, "filter_desc_set")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dnnp_filter_desc_destroy(self.h)


class ConvDescHandle:
    def __init__(self, u, v, ph, pw, mode, accumulate):
        L = lib()
        self.h = vp()
        check(L.dnnp_conv_desc_create(ctypes.byref(self.h)), "conv_desc_create")
        st = L.dnnp_conv_desc_set(self.h, u, v, ph, pw, mode, int(bool(accumulate)))
        if st != OK:
            L.dnnp_conv_desc_destroy(self.h)
            self.h = None
            check(st, "conv_desc_set")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dnnp_conv_desc_destroy(self.h)


class PoolDescHandle:
    def __init__(self, kind, wh, ww, sh, sw, ph, pw):
        L = lib()
        self.h = vp()
        check(L.dnnp_pooling_desc_create(ctypes.byref(self.h)), "pooling_desc_create")
        st = L.dnnp_pooling_desc_set(self.h, kind, wh, ww, sh, sw, ph, pw)
        if st != OK:
            L.dnnp_pooling_desc_destroy(self.h)
            self.h = None
            check(st, "pooling_desc_set")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dnnp_pooling_desc_destroy(self.h)
