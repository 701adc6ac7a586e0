"""Seeded random convolution geometries through every tensor-core path the
host heuristics can pick (space-to-depth, tap folding, column blocking up to
8, CTA pairs, stream-K, small-grid split-K, reduction segments, scattered
epilogues) against the C oracle, fwd / bwd-data / bwd-filter, both modes,
NCHW / NHWC, with and without accumulate.  Bar: north_star fp32 1e-4
normalised."""
import numpy as np
import pytest

from test_gpu_tc_paths import check, env, run_case

pytestmark = pytest.mark.gpu


def shapes(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        n = int(rng.integers(1, 4))
        c = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 24, 48, 64, 96]))
        k = int(rng.choice([1, 3, 8, 16, 24, 40, 64, 96, 128, 200]))
        r = int(rng.integers(1, 8))
        s = int(rng.integers(1, 12))
        u = int(rng.choice([1, 1, 1, 2, 3, 4]))
        v = int(rng.choice([1, 1, 1, 2, 3, 4]))
        ph = int(rng.integers(0, r))
        pw = int(rng.integers(0, s))
        h = int(rng.integers(max(1, r - 2 * ph), 30))
        w = int(rng.integers(max(1, s - 2 * pw), 30))
        if h + 2 * ph < r or w + 2 * pw < s:
            continue
        out.append((n, c, h, w, k, r, s, u, v, ph, pw))
    return out


FUZZ = shapes(2014, 24)


@pytest.mark.parametrize("shape", FUZZ, ids=[f"f{i}" for i in range(len(FUZZ))])
def test_fuzz_geometry(shape):
    i = FUZZ.index(shape)
    mode = "convolution" if i % 2 == 0 else "cross_correlation"
    lay = "nhwc" if i % 3 == 0 else "nchw"
    check(run_case(shape, mode=mode, layout_in=lay, accumulate=(i % 4 == 1), seed=100 + i))


def test_fuzz_forced_paths():
    """The same geometries with the opt-in / alternative schedules forced."""
    for kv in ({"DNNP_TC_SK": 1}, {"DNNP_TC_NO_SPLIT": 1}, {"DNNP_TC_CHAIN": 256, "DNNP_WG_CHAIN": 128},
               {"DNNP_TC_NO_FOLD": 1, "DNNP_TC_BW2": 1}, {"DNNP_TC_NC": 1}):
        with env(**kv):
            for j, shape in enumerate(FUZZ[:8]):
                check(run_case(shape, seed=200 + j))
