"""GPU bench CLI (paper_1410_0759_b200/bench_cli.py): suite parsing, FLOP
accounting, CSV/JSON schema and exit codes on CPU; timing + verification on
the GPU.  Mirrors the reference harness tests (pkg/tests/test_bench.py:31-240)."""
import io
import json
from dataclasses import replace

import pytest

from paper_1410_0759_b200 import ConfigInvalid, ParseError, VerifyFailed
from paper_1410_0759_b200 import bench_cli as bc

TINY_SUITE = """
# two small layers
tiny1 2 2 6 6 3 3 3 1 1 0 0
tiny2 2 3 5 5 2 2 2 1 1 1 1   # trailing comment
"""


def test_flops_table2_layer5():
    # 2 * 128 * 384 * 128 * 3 * 3 * 11 * 11
    assert bc.flop_count(bc.Layer("layer5", 128, 128, 13, 13, 384, 3, 3)) == 13_702_791_168


def test_flops_unit_and_linear_in_batch():
    assert bc.flop_count(bc.Layer("one", 1, 1, 1, 1, 1, 1, 1)) == 2
    base = bc.Layer("l", 4, 3, 9, 9, 5, 3, 3, 2, 2, 1, 1)
    assert bc.flop_count(replace(base, n=12)) == 3 * bc.flop_count(base)


def test_parse_suite():
    layers = bc.parse_suite(TINY_SUITE)
    assert [l.name for l in layers] == ["tiny1", "tiny2"]
    assert layers[1].pad_w == 1 and layers[0].u == 1


@pytest.mark.parametrize("text", ["oops 1 2 3\n", "l 1 2 3 4 5 6 x 1 1 0 0\n", "# nothing\n\n"])
def test_parse_errors(text):
    with pytest.raises(ParseError):
        bc.parse_suite(text)


@pytest.mark.parametrize("name,count", [("table2", 5), ("alexnet.suite", 5), ("overfeat_vgg", None)])
def test_bundled_suites(name, count):
    layers = bc.load_suite(name)
    if count is not None:
        assert len(layers) == count
    for l in layers:
        bc._validate(l)
        assert bc.flop_count(l) > 0


def test_missing_suite():
    with pytest.raises(ParseError):
        bc.load_suite("/nonexistent/x.suite")


def test_invalid_layer():
    with pytest.raises(ConfigInvalid):
        bc._validate(bc.Layer("bad", 1, 1, 3, 3, 1, 5, 5))


def _rows():
    return [bc.Row("layer1", "implicit", "f32", 128, 10, 0.5, 20.0, 12.5, None),
            bc.Row("layer1/bwd_data", "implicit", "f32", 128, 10, 0.25, 40.0, None, 1e-6),
            bc.Row("suite_mean", "implicit", "f32", None, None, None, 30.0, None, None)]


def test_csv_roundtrip_and_header():
    buf = io.StringIO()
    bc.emit_csv(_rows(), buf)
    assert buf.getvalue().splitlines()[0] == ",".join(bc.COLUMNS)
    assert bc.read_csv(io.StringIO(buf.getvalue())) == _rows()


def test_json_roundtrip_matches_csv():
    buf = io.StringIO()
    bc.emit_json(_rows(), buf)
    assert bc.read_json(io.StringIO(buf.getvalue())) == _rows()
    assert list(json.loads(buf.getvalue())[0]) == list(bc.COLUMNS)


def test_table_renders_percent():
    t = bc.table(_rows())
    assert "12%" in t or "13%" in t
    assert "suite_mean" in t


def test_exit_codes_without_gpu(tmp_path):
    assert bc.main(["bogus"]) == 1
    assert bc.main(["run", "--suite", str(tmp_path / "none.suite")]) == 1
    suite = tmp_path / "t.suite"
    suite.write_text(TINY_SUITE)
    assert bc.main(["sweep", "--suite", str(suite), "--layer", "nope"]) == 1
    assert bc.main(["run", "--suite", str(suite), "--passes", "sideways"]) == 1
    assert bc.main(["run", "--suite", str(suite), "--format", "xml"]) == 1
    assert bc.main(["run", "--suite", str(suite), "--engines", "winograd"]) == 1


@pytest.mark.gpu
def test_gpu_run_verify_all_passes(tmp_path, capsys):
    suite = tmp_path / "t.suite"
    suite.write_text(TINY_SUITE + "strided 3 5 17 15 7 5 3 2 3 2 1\n")
    out = tmp_path / "r.csv"
    rc = bc.main(["run", "--suite", str(suite), "--passes", "fwd,bwd_data,bwd_filter",
                  "--verify", "--batch", "4", "--repeats", "2", "--peak", "1000",
                  "--format", "csv,json", "--out", str(out), "--quiet"])
    assert rc == 0
    rows = bc.read_csv(open(tmp_path / "r.csv"))
    assert rows == bc.read_json(open(tmp_path / "r.json"))
    per_layer = [r for r in rows if not r.layer.startswith("suite_")]
    assert len(per_layer) == 9
    assert all(r.max_abs_err is not None and r.max_abs_err <= 1e-4 for r in per_layer)
    assert all(r.seconds > 0 and r.gflops > 0 and r.peak_pct is not None for r in per_layer)
    names = {r.layer for r in rows}
    assert {"suite_mean", "suite_weighted", "suite_weighted/bwd_filter"} <= names
    w = next(r for r in rows if r.layer == "suite_weighted")
    fw = [r for r in per_layer if "/" not in r.layer]
    assert w.flops == sum(r.flops for r in fw)


@pytest.mark.gpu
def test_gpu_verify_failure_exit_two(tmp_path, monkeypatch):
    suite = tmp_path / "t.suite"
    suite.write_text(TINY_SUITE)
    monkeypatch.setitem(bc.ABS_TOL, "f32", -1.0)
    with pytest.raises(VerifyFailed) as ei:
        bc.run_suite(bc.parse_suite(TINY_SUITE), verify=True, batch=2, repeats=1,
                     passes=("fwd",))
    assert len(ei.value.results) == 4
    assert bc.main(["run", "--suite", str(suite), "--verify", "--batch", "2", "--repeats", "1",
                    "--out", str(tmp_path / "o.csv"), "--quiet"]) == 2
    assert (tmp_path / "o.csv").exists()


@pytest.mark.gpu
def test_gpu_sweep(tmp_path):
    suite = tmp_path / "t.suite"
    suite.write_text(TINY_SUITE)
    rows = bc.sweep(bc.parse_suite(TINY_SUITE)[0], [1, 2, 4], repeats=2,
                    passes=("fwd", "bwd_filter"))
    assert len(rows) == 6
    assert max(r.ratio_pct for r in rows) == pytest.approx(100.0)
    assert bc.main(["sweep", "--suite", str(suite), "--layer", "tiny2", "--batches", "1,2",
                    "--out", str(tmp_path / "s.csv"), "--quiet"]) == 0
    assert open(tmp_path / "s.csv").readline().strip() == ",".join(bc.SWEEP_COLUMNS)
