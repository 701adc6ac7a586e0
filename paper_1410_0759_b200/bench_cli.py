"""GPU benchmark CLI in the reference harness's vocabulary (SURVEY.md 8(f)
rank 1; reference pkg/src/dnnp/bench.py:38-51 suite format and FLOP
accounting, :101-129 flop_count, :284-319 CSV/JSON schema, :478-493 exit
codes).

    python -m paper_1410_0759_b200.bench_cli run [--suite S] [--dtype f32|f64]
        [--batch N] [--repeats R] [--passes fwd,bwd_data,bwd_filter]
        [--engines implicit,...] [--verify] [--peak GFLOPS]
        [--format csv|json|csv,json] [--out FILE] [--quiet]
    python -m paper_1410_0759_b200.bench_cli sweep --layer L [--batches 1,2,...]

Same suite files (name N C H W K R S u v pad_h pad_w, '#' comments), same
flops (2 N K C R S P Q per pass), same CSV columns (layer, engine, dtype,
batch, flops, seconds, gflops, peak_pct, max_abs_err) and the reference's
summary rows (suite_mean, suite_weighted).  GPU additions: backward passes
(rows are named "<layer>" for forward, "<layer>/bwd_data", "<layer>/bwd_filter"
so the schema is unchanged), seconds are the median of CUDA-event timings of
device-resident calls.  All three engine labels run the same implicit-GEMM
kernels (north_star: no multi-backend dispatch).  --verify compares each pass
with an independent device loop nest in fp64 (dnnp_convolution_verify_reference,
csrc/conv_verify.cu: the counterpart of the reference's direct-engine check,
bench.py:196-203; tests pin it to the C oracle) at the reference's
tolerances (1e-4 f32, 1e-10 f64), applied to max|err| / max(1, max|ref|):
an absolute bound for unit-scale outputs, the north_star normalised bound for
the long reductions (dW sums N*P*Q products) whose magnitude grows with the
layer.  Exit status: 0 ok, 2 verification failure, 1 usage / configuration
error.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import statistics
import sys
from dataclasses import asdict, dataclass, replace  # noqa: F401 (replace re-exported)

COLUMNS = ("layer", "engine", "dtype", "batch", "flops", "seconds", "gflops", "peak_pct",
           "max_abs_err")
SWEEP_COLUMNS = ("layer", "engine", "dtype", "batch", "flops", "seconds", "gflops", "ratio_pct")
PASSES = ("fwd", "bwd_data", "bwd_filter")
ABS_TOL = {"f32": 1e-4, "f64": 1e-10}
SUITE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "suites")


from .errors import ConfigInvalid, DnnpError, ParseError, VerifyFailed


@dataclass(frozen=True)
class Layer:
    name: str
    n: int
    c: int
    h: int
    w: int
    k: int
    r: int
    s: int
    u: int = 1
    v: int = 1
    pad_h: int = 0
    pad_w: int = 0

    def out_hw(self):
        from . import conv
        p = conv.output_extent(self.h, self.r, self.u, self.pad_h)
        q = conv.output_extent(self.w, self.s, self.v, self.pad_w)
        return p, q

    def flops(self):
        p, q = self.out_hw()
        return 2 * self.n * self.k * self.c * self.r * self.s * p * q


def flop_count(layer):
    """2 N K C R S P Q: one multiply-add is two flops; the same count for each
    backward pass (reference bench.py:126-129)."""
    return layer.flops()


def peak_percent(gflops, peak_gflops):
    return 100.0 * gflops / peak_gflops


@dataclass
class Row:
    layer: str
    engine: str
    dtype: str
    batch: int | None
    flops: int | None
    seconds: float | None
    gflops: float | None
    peak_pct: float | None
    max_abs_err: float | None


@dataclass
class SweepRow:
    layer: str
    engine: str
    dtype: str
    batch: int
    flops: int
    seconds: float
    gflops: float
    ratio_pct: float


def parse_suite(text):
    """Layers of a suite text; '#' starts a comment, blank lines are skipped."""
    out = []
    for no, line in enumerate(text.splitlines(), 1):
        body = line.split("#", 1)[0].split()
        if not body:
            continue
        if len(body) != 12:
            raise ParseError(f"line {no}: expected 'name N C H W K R S u v pad_h pad_w', "
                           f"got {len(body)} fields")
        try:
            vals = [int(t) for t in body[1:]]
        except ValueError as e:
            raise ParseError(f"line {no}: {e}") from None
        out.append(Layer(body[0], *vals))
    if not out:
        raise ParseError("suite contains no layers")
    return out


def load_suite(spec):
    """A suite by path, else by bundled name (with or without .suite)."""
    if os.path.isfile(spec):
        with open(spec) as fh:
            return parse_suite(fh.read())
    name = spec if spec.endswith(".suite") else spec + ".suite"
    path = os.path.join(SUITE_DIR, name)
    if os.path.isfile(path):
        with open(path) as fh:
            return parse_suite(fh.read())
    raise ParseError(f"no such suite file: {spec}")


def _validate(layer):
    try:
        p, q = layer.out_hw()
    except DnnpError as e:
        raise ConfigInvalid(f"layer {layer.name}: {e}") from None
    if min(layer.n, layer.c, layer.h, layer.w, layer.k, layer.r, layer.s, p, q) < 1:
        raise ConfigInvalid(f"layer {layer.name}: non-positive extent")


class _Problem:
    """Device tensors of one layer (seeded uniform(-0.5, 0.5), the reference
    generator default_rng([seed, index]))."""

    def __init__(self, layer, dtype, seed, index, like=None):
        import numpy as np
        import torch

        from . import conv, tensor
        self.layer = layer
        p, q = layer.out_hw()
        npdt = np.float32 if dtype == "f32" else np.float64
        if like is None:
            rng = np.random.default_rng([seed, index])
            x = rng.uniform(-0.5, 0.5, layer.n * layer.c * layer.h * layer.w).astype(npdt)
            f = rng.uniform(-0.5, 0.5, layer.k * layer.c * layer.r * layer.s).astype(npdt)
            dy = rng.uniform(-0.5, 0.5, layer.n * layer.k * p * q).astype(npdt)
        else:
            x, f, dy = (like.host[k].astype(npdt) for k in ("x", "f", "dy"))
        self.host = {"x": x, "f": f, "dy": dy}
        dev = torch.device("cuda")
        mk = tensor.make_desc
        self.cd = conv.ConvDesc(layer.u, layer.v, layer.pad_h, layer.pad_w)
        self.x = tensor.TensorView(mk(layer.n, layer.c, layer.h, layer.w, elem_type=dtype),
                                   torch.from_numpy(x).to(dev))
        self.f = conv.FilterView(conv.make_filter_desc(layer.k, layer.c, layer.r, layer.s,
                                                       elem_type=dtype),
                                 torch.from_numpy(f).to(dev))
        self.dy = tensor.TensorView(mk(layer.n, layer.k, p, q, elem_type=dtype),
                                    torch.from_numpy(dy).to(dev))
        self.y = tensor.empty_view(mk(layer.n, layer.k, p, q, elem_type=dtype), device=dev)
        self.dx = tensor.empty_view(mk(layer.n, layer.c, layer.h, layer.w, elem_type=dtype),
                                    device=dev)
        self.df = conv.FilterView(conv.make_filter_desc(layer.k, layer.c, layer.r, layer.s,
                                                        elem_type=dtype),
                                  torch.empty(layer.k * layer.c * layer.r * layer.s,
                                              dtype=self.x.buf.dtype, device=dev))

    def op(self, pas, engine):
        from . import conv
        if pas == "fwd":
            return lambda: conv.conv_forward(self.x, self.f, self.cd, engine, self.y)
        if pas == "bwd_data":
            return lambda: conv.conv_backward_data(self.dy, self.f, self.cd, engine, self.dx)
        return lambda: conv.conv_backward_filter(self.dy, self.x, self.cd, engine, self.df)

    def result(self, pas):
        return {"fwd": self.y.buf, "bwd_data": self.dx.buf, "bwd_filter": self.df.buf}[pas]


def _time(op, repeats):
    import torch
    op()  # warm-up
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        op()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    return statistics.median(times)


def _reference(layer, prob, pas):
    """The same pass as a plain fp64 loop nest on the device (libdnnp's
    dnnp_convolution_verify_reference: no packing, no tensor cores, fixed
    summation order) on the same inputs -- the counterpart of the reference
    harness's check against its direct engine (bench.py:196-203)."""
    import torch

    from . import _lib
    p, q = layer.out_hw()
    n_out = {"fwd": layer.n * layer.k * p * q, "bwd_data": layer.n * layer.c * layer.h * layer.w,
             "bwd_filter": layer.k * layer.c * layer.r * layer.s}[pas]
    out = torch.empty(n_out, dtype=torch.float64, device="cuda")
    code = PASSES.index(pas)
    a = prob.x if pas == "fwd" else prob.dy
    b = prob.f if pas != "bwd_filter" else prob.x
    _lib.check(_lib.lib().dnnp_convolution_verify_reference(
        _lib.handle(), code, prob.x.desc.c_desc(), prob.f.desc.c_desc(), prob.cd.c_desc(),
        prob.y.desc.c_desc(), a.ptr, b.ptr, out.data_ptr()), "convolution_verify_reference")
    torch.cuda.synchronize()
    return out


def run_suite(layers, engines=("implicit",), dtype="f32", batch=None, repeats=5,
              passes=PASSES, verify=False, peak=None, seed=2014, progress=None):
    """Rows of every layer x pass x engine plus per (engine, pass) summary rows;
    raises VerifyFailed (carrying the rows) when a pass strays beyond the
    per-dtype absolute tolerance."""
    rows, failures = [], []
    groups = {}
    if verify and batch is None:
        batch = 16  # the reference's verify batch (bench.py:50)
    for index, base in enumerate(layers):
        layer = replace(base, n=batch) if batch else base
        _validate(layer)
        prob = _Problem(layer, dtype, seed, index)
        fl = layer.flops()
        for pas in passes:
            label = layer.name if pas == "fwd" else f"{layer.name}/{pas}"
            ref = _reference(layer, prob, pas) if verify else None
            for eng in engines:
                if progress:
                    progress(f"{label} [{eng}/{dtype}]")
                sec = _time(prob.op(pas, eng), repeats)
                gf = fl / sec / 1e9
                err = None
                if verify:
                    err = float((prob.result(pas).double() - ref).abs().max())
                    scale = max(1.0, float(ref.abs().max()))
                    if err > ABS_TOL[dtype] * scale:
                        failures.append(f"{label}/{eng}: {err:.3e} (max|ref| {scale:.3g})")
                row = Row(label, eng, dtype, layer.n, fl, sec, gf,
                          100.0 * gf / peak if peak else None, err)
                rows.append(row)
                groups.setdefault((eng, pas), []).append(row)
    for (eng, pas), grp in groups.items():
        suffix = "" if pas == "fwd" else f"/{pas}"
        mean = sum(r.gflops for r in grp) / len(grp)
        tf, ts = sum(r.flops for r in grp), sum(r.seconds for r in grp)
        rows.append(Row("suite_mean" + suffix, eng, dtype, batch, None, None, mean,
                        100.0 * mean / peak if peak else None, None))
        rows.append(Row("suite_weighted" + suffix, eng, dtype, batch, tf, ts, tf / ts / 1e9,
                        100.0 * (tf / ts / 1e9) / peak if peak else None, None))
    if failures:
        raise VerifyFailed("; ".join(failures), rows)
    return rows


def sweep(layer, batches, engine="implicit", dtype="f32", repeats=5, passes=("fwd",), seed=2014,
          progress=None):
    pts = []
    for b in batches:
        lay = replace(layer, n=int(b))
        _validate(lay)
        prob = _Problem(lay, dtype, seed, int(b))
        for pas in passes:
            if progress:
                progress(f"{lay.name} batch={b} {pas}")
            sec = _time(prob.op(pas, engine), repeats)
            name = lay.name if pas == "fwd" else f"{lay.name}/{pas}"
            pts.append((name, int(b), lay.flops(), sec, lay.flops() / sec / 1e9))
    best = max(p[4] for p in pts)
    return [SweepRow(n, engine, dtype, b, fl, s, g, 100.0 * g / best) for n, b, fl, s, g in pts]


def _csv(rows, columns, fh):
    w = csv.writer(fh)
    w.writerow(columns)
    for r in rows:
        vals = []
        for c in columns:
            v = getattr(r, c)
            vals.append("" if v is None else (repr(v) if isinstance(v, float) else v))
        w.writerow(vals)


def emit_csv(rows, fh):
    _csv(rows, COLUMNS, fh)


def read_csv(fh):
    rows = list(csv.reader(fh))
    if not rows or tuple(rows[0]) != COLUMNS:
        raise ParseError("bad CSV header")
    conv = {"batch": int, "flops": int, "seconds": float, "gflops": float, "peak_pct": float,
            "max_abs_err": float}
    out = []
    for rec in rows[1:]:
        d = dict(zip(COLUMNS, rec))
        out.append(Row(**{k: (conv[k](v) if v else None) if k in conv else v
                          for k, v in d.items()}))
    return out


def emit_json(rows, fh):
    json.dump([asdict(r) for r in rows], fh, indent=2)
    fh.write("\n")


def read_json(fh):
    return [Row(**d) for d in json.load(fh)]


def table(rows):
    out = [f"{'layer':<24}{'engine':<10}{'dtype':<6}{'batch':>6}{'gflops':>12}{'peak':>7}"
           f"{'max_err':>11}"]
    for r in rows:
        out.append(f"{r.layer:<24}{r.engine:<10}{r.dtype:<6}"
                   f"{('-' if r.batch is None else r.batch):>6}"
                   f"{('-' if r.gflops is None else f'{r.gflops:.1f}'):>12}"
                   f"{('-' if r.peak_pct is None else f'{r.peak_pct:.0f}%'):>7}"
                   f"{('-' if r.max_abs_err is None else f'{r.max_abs_err:.2e}'):>11}")
    return "\n".join(out)


def _formats(spec):
    fm = [f.strip().lower() for f in spec.split(",") if f.strip()]
    bad = [f for f in fm if f not in ("csv", "json")]
    if bad:
        raise ConfigInvalid(f"unknown output format {bad[0]!r}")
    return fm or ["csv"]


def _emit(rows, formats, out, columns):
    for fmt in formats:
        def write(fh):
            if fmt == "json":
                emit_json(rows, fh)
            else:
                _csv(rows, columns, fh)
        if out:
            path = out if len(formats) == 1 else os.path.splitext(out)[0] + "." + fmt
            with open(path, "w", newline="") as fh:
                write(fh)
        else:
            buf = io.StringIO()
            write(buf)
            sys.stdout.write(buf.getvalue())


def build_parser():
    ap = argparse.ArgumentParser(prog="dnnp-gpu-bench",
                                 description="Time and verify the B200 convolution kernels.")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--suite", default="table2.suite")
        p.add_argument("--dtype", default="f32", choices=("f32", "f64"))
        p.add_argument("--batch", type=int, default=None)
        p.add_argument("--repeats", type=int, default=5)
        p.add_argument("--seed", type=int, default=2014)
        p.add_argument("--passes", default="fwd", help="comma list of fwd,bwd_data,bwd_filter")
        p.add_argument("--format", default="csv")
        p.add_argument("--out", default=None)
        p.add_argument("--quiet", action="store_true")

    run = sub.add_parser("run")
    common(run)
    run.add_argument("--engines", default="implicit")
    run.add_argument("--verify", action="store_true")
    run.add_argument("--peak", type=float, default=None, help="peak GFLOPS for peak_pct")
    sw = sub.add_parser("sweep")
    common(sw)
    sw.add_argument("--layer", required=True)
    sw.add_argument("--engine", default="implicit")
    sw.add_argument("--batches", default="1,2,4,8,16,32,64,128,256")
    return ap


def _passes(spec):
    ps = [p.strip() for p in spec.split(",") if p.strip()]
    for p in ps:
        if p not in PASSES:
            raise ConfigInvalid(f"unknown pass {p!r}")
    return ps


def main(argv=None):
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code in (0, None) else 1
    progress = None if args.quiet else (lambda m: print(f"  running {m}", file=sys.stderr,
                                                        flush=True))
    try:
        layers = load_suite(args.suite)
        formats = _formats(args.format)
        passes = _passes(args.passes)
        if args.command == "run":
            engines = [e.strip() for e in args.engines.split(",") if e.strip()]
            for e in engines:
                if e not in ("direct", "explicit", "implicit"):
                    raise ConfigInvalid(f"unknown engine {e!r}")
            try:
                rows = run_suite(layers, engines, args.dtype, args.batch, args.repeats, passes,
                                 args.verify, args.peak, args.seed, progress)
                failed = False
            except VerifyFailed as e:
                print(f"VERIFY FAILED: {e}", file=sys.stderr)
                rows, failed = e.results, True
            _emit(rows, formats, args.out, COLUMNS)
            print(table(rows))
            return 2 if failed else 0
        by_name = {l.name: l for l in layers}
        if args.layer not in by_name:
            raise ConfigInvalid(f"layer {args.layer!r} not in suite ({', '.join(by_name)})")
        batches = [int(b) for b in args.batches.split(",") if b.strip()]
        if not batches:
            raise ConfigInvalid("empty batch list")
        rows = sweep(by_name[args.layer], batches, args.engine, args.dtype, args.repeats, passes,
                     args.seed, progress)
        _emit(rows, formats, args.out, SWEEP_COLUMNS)
        for r in rows:
            print(f"{r.layer:<24}{r.engine:<10}{r.dtype:<6}{r.batch:>6}{r.gflops:>12.1f}"
                  f"{r.ratio_pct:>6.0f}%")
        return 0
    except DnnpError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    raise SystemExit(main())
