"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/dnnp.h declares, and keeps the reference's status contract
(pkg/capi/src/dnnp_capi.c + dnnp_capi_bridge.py) for descriptors and
argument validation.  Compute entries on a GPU-less host fail loudly with
NOT_SUPPORTED (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, has_cuda

from paper_1410_0759_b200 import _lib

HEADER = os.path.join(ROOT, "include", "dnnp.h")
LIB = os.path.join(ROOT, "paper_1410_0759_b200", "libdnnp.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dnnp_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 36
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (dnnp_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    L = _lib.lib()
    for s in syms:
        assert hasattr(L, s)
    assert set(_lib.SYMBOLS) <= set(syms)


def test_reference_symbol_set_is_covered():
    # the 36 functions of the reference header (dnnp.h:74-226)
    ref36 = """version status_string create destroy set_threads get_threads
    tensor_desc_create tensor_desc_destroy tensor_desc_set tensor_desc_set_ex tensor_desc_get
    filter_desc_create filter_desc_destroy filter_desc_set filter_desc_get
    conv_desc_create conv_desc_destroy conv_desc_set conv_desc_get
    pooling_desc_create pooling_desc_destroy pooling_desc_set pooling_desc_get
    conv_output_shape convolution_forward convolution_backward_data
    convolution_backward_filter convolution_backward_bias activation_forward
    activation_backward softmax_forward softmax_backward pooling_forward pooling_backward
    transform add_broadcast""".split()
    assert len(ref36) == 36
    syms = set(declared_symbols())
    assert {"dnnp_" + s for s in ref36} <= syms


def _build_conformance(tmp_path):
    exe = tmp_path / "conformance"
    subprocess.run(["gcc", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), "-o", str(exe),
                    os.path.join(ROOT, "tests", "capi", "conformance.c"),
                    "-L" + os.path.dirname(LIB), "-ldnnp",
                    "-Wl,-rpath," + os.path.dirname(LIB), "-lpthread", "-lm"], check=True)
    return exe


def test_capi_conformance_status_contract(tmp_path):
    exe = _build_conformance(tmp_path)
    r = subprocess.run([str(exe), "--status-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "0 failed" in r.stdout


REF_TEST = "/root/reference/pkg/capi/tests/test_capi.c"


@pytest.mark.skipif(not os.path.exists(REF_TEST), reason="reference tree not mounted")
def test_reference_capi_test_links_unchanged(tmp_path):
    """The reference's own C test program compiles unchanged against
    include/dnnp.h + libdnnp.so; without a GPU every status check passes and
    only the compute checks report NOT_SUPPORTED."""
    exe = tmp_path / "test_capi"
    subprocess.run(["gcc", "-O2", "-I" + os.path.join(ROOT, "include"), "-o", str(exe), REF_TEST,
                    "-L" + os.path.dirname(LIB), "-ldnnp", "-Wl,-rpath," + os.path.dirname(LIB),
                    "-lpthread", "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    fails = [ln for ln in r.stdout.splitlines() if "FAIL" in ln]
    if has_cuda():
        assert r.returncode == 0, fails
    else:
        compute = ("convolution", "engine", "agree", "transform", "round trip", "pooling",
                   "concurrent")
        assert all(any(k in ln for k in compute) for ln in fails), fails
        assert "44 passed" in r.stdout


def test_check_strides_native():
    L = _lib.lib()

    def chk(ext, st):
        e = (ctypes.c_int64 * 4)(*ext)
        s = (ctypes.c_int64 * 4)(*st)
        return L.dnnp_check_strides(e, s)

    assert chk([2, 3, 4, 5], [60, 20, 5, 1]) == 0
    assert chk([2, 3, 4, 5], [60, 1, 15, 3]) == 0       # NHWC
    assert chk([1, 2, 2, 2], [8, 0, 2, 1]) == 1         # zero stride
    assert chk([2, 2, 2, 2], [4, 2, 2, 1]) == 1         # overlap
    assert chk([1, 3, 4, 4], [0, 20, 5, 1]) == 0        # padded rows
    # brute-force agreement on random small stride sets (test_tensor.py style)
    rng = np.random.default_rng(5)
    for _ in range(200):
        ext = [int(v) for v in rng.integers(1, 4, 4)]
        st = [int(v) for v in rng.integers(-6, 7, 4)]
        offs = np.zeros(1, dtype=np.int64)
        for e, s in zip(ext, st):
            offs = (offs[:, None] + np.arange(e) * s).ravel()
        alias = np.unique(offs).size != offs.size
        assert chk(ext, st) == (1 if alias else 0), (ext, st)


def test_large_box_delta_path():
    L = _lib.lib()
    # box > 2^22 takes the delta sweep (tensor.py:66-81)
    e = (ctypes.c_int64 * 4)(64, 64, 64, 64)
    ok = (ctypes.c_int64 * 4)(64 ** 3, 64 ** 2, 64, 1)
    bad = (ctypes.c_int64 * 4)(64 ** 3, 64 ** 2, 64, 2)
    assert L.dnnp_check_strides(e, ok) == 0
    assert L.dnnp_check_strides(e, bad) == 1


@pytest.mark.skipif(has_cuda(), reason="checks the GPU-less behaviour")
def test_compute_without_gpu_fails_loudly():
    import paper_1410_0759_b200 as dp
    x = dp.TensorView.from_array(np.ones((1, 1, 2, 2)))
    y = dp.empty_view(x.desc)
    with pytest.raises(dp.NotSupported, match="no CUDA device"):
        dp.activation_forward("relu", x, y)
