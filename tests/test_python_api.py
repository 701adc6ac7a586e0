"""Host-side behaviour of the Python mirror (names, argument meaning and
error classes of pkg/src/dnnp), no GPU needed."""
import numpy as np
import pytest

import paper_1410_0759_b200 as dp


def test_public_names_match_reference():
    # pkg/src/dnnp/__init__.py:8-70 (scratch/gemm internals excluded: CPU engine details)
    names = """ConvDesc ConvMode Engine FilterDesc FilterView access conv_backward_bias
    conv_backward_data conv_backward_filter conv_forward conv_out_shape make_filter_desc
    output_extent pad_preset AliasingStrides AllocTooLarge ConfigInvalid DimMismatch DnnpError
    EmptyOutput EmptyWindow IncompatibleBroadcast MissingArgmax OverlappingBuffers ParseError
    ShapeMismatch VerifyFailed ZeroDivisor ZeroExtent MagicDivider div_mod make_divider
    ActivationKind PoolKind PoolingDesc SoftmaxMode activation_backward activation_forward
    pool_backward pool_forward pool_out_shape softmax_backward softmax_forward TensorDesc
    TensorView add_broadcast empty_view make_desc transform zeros_view""".split()
    missing = [n for n in names if not hasattr(dp, n)]
    assert not missing, missing


def test_make_desc_layouts_and_errors():
    d = dp.make_desc(2, 3, 4, 5)
    assert d.strides == (60, 20, 5, 1)
    assert dp.make_desc(2, 3, 4, 5, layout="nhwc").strides == (60, 1, 15, 3)
    with pytest.raises(dp.ZeroExtent):
        dp.make_desc(0, 1, 1, 1)
    with pytest.raises(dp.AliasingStrides):
        dp.make_desc(1, 2, 2, 2, layout="custom", strides=(8, 0, 2, 1))
    with pytest.raises(dp.ShapeMismatch):
        dp.make_desc(1, 1, 1, 1, layout="custom")
    with pytest.raises(dp.ShapeMismatch):
        dp.make_desc(1, 1, 1, 1, layout="weird")


def test_view_bounds():
    d = dp.make_desc(1, 1, 2, 2)
    with pytest.raises(dp.ShapeMismatch):
        dp.TensorView(d, np.zeros(3))
    with pytest.raises(dp.ShapeMismatch):
        dp.TensorView(d, np.zeros(4, dtype=np.float64))
    neg = dp.make_desc(1, 1, 2, 2, layout="custom", strides=(4, 4, -2, 1))
    with pytest.raises(dp.ShapeMismatch):
        dp.TensorView(neg, np.zeros(8, dtype=np.float32))
    v = dp.TensorView(d, np.arange(4.0, dtype=np.float32))
    assert v.array[0, 0, 1, 1] == 3.0


def test_conv_params():
    # test_conv_params.py:13-20 and the Eq.2 accessing function
    assert dp.output_extent(128, 11, 1, 0) == 118
    assert dp.output_extent(5, 3, 2, 1) == 3
    with pytest.raises(dp.EmptyOutput):
        dp.output_extent(2, 5, 1, 0)
    assert dp.access(0, 1, 3, 0, 0) == 2
    assert dp.access(0, 1, 3, 0, 0, "cross_correlation") == 0
    assert dp.pad_preset("same", 3, 5) == (1, 2)
    x = dp.make_desc(2, 3, 7, 7)
    f = dp.make_filter_desc(4, 3, 3, 3)
    assert dp.conv_out_shape(x, f, dp.ConvDesc(2, 2, 1, 1)) == (2, 4, 4, 4)
    with pytest.raises(dp.ShapeMismatch):
        dp.conv_out_shape(x, dp.make_filter_desc(4, 2, 3, 3), dp.ConvDesc())
    with pytest.raises(dp.ShapeMismatch):
        dp.ConvDesc(0, 1)


def test_magic_divider_mirror():
    md = dp.make_divider(7)
    assert (md.multiplier, md.shift, md.add_indicator) == (0x24924925, 3, True)
    ns = np.arange(1 << 18, dtype=np.uint32)
    for d in (1, 2, 3, 7, 56, 3136, 13924):
        assert np.array_equal(dp.make_divider(d).div(ns), ns // d)
    with pytest.raises(dp.ZeroDivisor):
        dp.make_divider(0)


def test_pool_desc_validation():
    with pytest.raises(dp.ShapeMismatch):
        dp.PoolingDesc("max", 0, 1)
    pd = dp.PoolingDesc("max", 3, 3, 2, 2)
    assert dp.pool_out_shape(pd, dp.make_desc(1, 1, 55, 55)) == (1, 1, 27, 27)


def test_errors_raised_before_compute():
    x = dp.TensorView.from_array(np.ones((1, 1, 4, 4)))
    y = dp.TensorView.from_array(np.ones((1, 1, 4, 3)))
    with pytest.raises(dp.ShapeMismatch):
        dp.activation_forward("relu", x, y)
    with pytest.raises(dp.OverlappingBuffers):
        dp.transform(x, x)
    pd = dp.PoolingDesc("max", 2, 2, 2, 2)
    yy = dp.TensorView.from_array(np.ones((1, 1, 2, 2)))
    with pytest.raises(dp.MissingArgmax):
        dp.pool_backward(pd, yy, yy, x, dp.TensorView.from_array(np.ones((1, 1, 4, 4))))
    with pytest.raises(dp.IncompatibleBroadcast):
        dp.add_broadcast(dp.TensorView.from_array(np.ones((1, 2, 1, 1))), x)
