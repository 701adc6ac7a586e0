#!/usr/bin/env python3
"""Benchmark: AlexNet conv1-5 forward / backward-data / backward-filter, fp32,
N=128 per GPU (BASELINE.json configs[1]; weak scaling to N=1024 on 8 GPUs =
configs[3], with the dW NCCL allreduce).

One step = fwd + bwd-data + bwd-filter of all five layers over one batch of
synthetic inputs (uniform(-0.5, 0.5) from default_rng([2014, layer]) as the
reference bench, pkg/src/dnnp/bench.py:151-157), inputs resident in HBM.
Metric = algorithmic conv TFLOP/s, F = 2*N*K*C*R*S*P*Q per pass
(bench.py:126-129).  L2 is flushed (256 MiB write) between timed steps,
outside the per-step CUDA-event windows.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# torchvision / "one weird trick" AlexNet convs: name, C, H(=W), K, R(=S), stride, pad
ALEXNET = [
    ("conv1", 3, 224, 64, 11, 4, 2),
    ("conv2", 64, 27, 192, 5, 1, 2),
    ("conv3", 192, 13, 384, 3, 1, 1),
    ("conv4", 384, 13, 256, 3, 1, 1),
    ("conv5", 256, 13, 256, 3, 1, 1),
]
PASSES = ("fwd", "bwd_data", "bwd_filter")
# ONE metric string for both arms (the driver pairs the lines by it); the %
# of tensor peak is reported in roofline.frac / pct_tf32_peak, not here
METRIC = "conv TFLOP/s fwd/bwd-data/bwd-filter (AlexNet conv1-5)"
N_PER_GPU = 128
REF_SAMPLE_N = 8      # --impl reference: images per timed step (bounded CPU sample)
CPU_SAMPLE_N = 128    # cpu_baseline leg: the full N=128 workload once (~10-20 s)
REF_BASE_N = 16       # cpu_baseline leg: real reference (direct engine) images per step


def out_extent(h, r, u, pad):
    return -(-(h - r + 1 + 2 * pad) // u)


def layer_flops(n, c, h, k, r, u, pad):
    p = out_extent(h, r, u, pad)
    return 2 * n * k * c * r * r * p * p


def sustained_tf32_peak():
    """TF32-equivalent sustained peak: 1/2 of the measured back-to-back bf16
    GEMM rate (MEASURED_PEAKS.json bf16_tflops_sustained)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)["bf16_tflops_sustained"] / 2.0
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        return m["hbm_gbs"], m["bf16_tflops"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region:
    the sampler (20 ms period) is started and has produced its first sample
    before the region begins; samples are time-stamped by a reader thread and
    only those taken inside the region (plus one period after it) count."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 20

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.stamped = []
        self.lines = []

    def _reader(self):
        for ln in self.proc.stdout:
            self.stamped.append((time.perf_counter(), ln))

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._reader, daemon=True)
            self.thread.start()
            t0 = time.perf_counter()
            while not self.stamped and time.perf_counter() - t0 < 5.0:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        self.t_begin = time.perf_counter()
        return self

    def __exit__(self, *a):
        self.t_end = time.perf_counter()
        if self.proc is not None:
            # at least one sample after the region (the region may be shorter than a period)
            deadline = time.perf_counter() + 1.0
            while time.perf_counter() < deadline and not any(t > self.t_end for t, _ in self.stamped):
                time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            lim = self.t_end + self.PERIOD_MS / 1e3
            inside = [ln for t, ln in self.stamped if self.t_begin <= t <= lim and ln.strip()]
            if not inside:  # a region shorter than one period: the nearest samples
                inside = [ln for t, ln in self.stamped if t >= self.t_begin][:1]
            self.lines = inside

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(n, device, torch):
    """Per-layer x, f, dy (synthetic, reference bench generator) on device."""
    layers = []
    for idx, (name, c, h, k, r, u, pad) in enumerate(ALEXNET):
        p = out_extent(h, r, u, pad)
        g = np.random.default_rng([2014, idx])
        x = torch.from_numpy(g.uniform(-0.5, 0.5, n * c * h * h).astype(np.float32))
        f = torch.from_numpy(g.uniform(-0.5, 0.5, k * c * r * r).astype(np.float32))
        dy = torch.from_numpy(g.uniform(-0.5, 0.5, n * k * p * p).astype(np.float32))
        layers.append(dict(name=name, n=n, c=c, h=h, k=k, r=r, u=u, pad=pad, p=p,
                           x=x.to(device), f=f.to(device), dy=dy.to(device),
                           flops=layer_flops(n, c, h, k, r, u, pad)))
    return layers


def build_views(dp, layers, torch, device):
    for L in layers:
        n, c, h, k, r, p = L["n"], L["c"], L["h"], L["k"], L["r"], L["p"]
        L["cd"] = dp.ConvDesc(L["u"], L["u"], L["pad"], L["pad"], "convolution")
        L["xv"] = dp.TensorView(dp.make_desc(n, c, h, h), L["x"])
        L["fv"] = dp.FilterView(dp.make_filter_desc(k, c, r, r), L["f"])
        L["yv"] = dp.empty_view(dp.make_desc(n, k, p, p), device=device)
        L["dyv"] = dp.TensorView(dp.make_desc(n, k, p, p), L["dy"])
        L["dxv"] = dp.empty_view(dp.make_desc(n, c, h, h), device=device)
        L["df"] = torch.empty(k * c * r * r, device=device)
        L["dfv"] = dp.FilterView(dp.make_filter_desc(k, c, r, r), L["df"])


def run_step_fused(dp, layers, torch):
    """The same step through the framework's fused backward entry (dx and dW
    of a layer in one call, dy packed once) -- informational, not the
    headline (which keeps the reference API's three calls per layer)."""
    for L in layers:
        dp.conv_forward(L["xv"], L["fv"], L["cd"], "implicit", L["yv"])
        dp.conv_backward(L["dyv"], L["fv"], L["xv"], L["cd"], "implicit", L["dxv"], L["dfv"])


def run_step(dp, layers, torch, events=None, allreduce=None):
    for li, L in enumerate(layers):
        ops = (
            lambda: dp.conv_forward(L["xv"], L["fv"], L["cd"], "implicit", L["yv"]),
            lambda: dp.conv_backward_data(L["dyv"], L["fv"], L["cd"], "implicit", L["dxv"]),
            lambda: dp.conv_backward_filter(L["dyv"], L["xv"], L["cd"], "implicit", L["dfv"]),
        )
        for pi, op in enumerate(ops):
            if events is not None:
                events[(li, pi)][0].record()
            op()
            if events is not None:
                events[(li, pi)][1].record()
        if allreduce is not None:
            allreduce(L["df"])
    if allreduce is not None and hasattr(allreduce, "__self__"):
        allreduce.__self__.wait()  # the step ends when every dW is reduced


def cpu_baseline(threads, sample_n=2, gpu_out=None):
    """The C oracle (restatement of the reference implicit engine) on host
    cores, on a bounded sample of the same workload (N=sample_n per layer).
    gpu_out: {layer: (y, dx, df)} host copies of the GPU results for the same
    inputs (sample_n must then be the GPU batch): returns the normalised
    errors max|gpu - oracle| / max|oracle| per layer and pass as the third
    value (the parity check of the benchmarked configuration itself)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    total_flops = 0
    dt = 0.0
    errs = {}
    for idx, (name, c, h, k, r, u, pad) in enumerate(ALEXNET):
        n = sample_n
        p = out_extent(h, r, u, pad)
        g = np.random.default_rng([2014, idx])
        x = g.uniform(-0.5, 0.5, n * c * h * h).astype(np.float32)
        f = g.uniform(-0.5, 0.5, k * c * r * r).astype(np.float32)
        dy = g.uniform(-0.5, 0.5, n * k * p * p).astype(np.float32)
        xg = [n, c, h, h, c * h * h, h * h, h, 1]
        yg = [n, k, p, p, k * p * p, p * p, p, 1]
        cg = [u, u, pad, pad, 0, 0]
        y = np.zeros(n * k * p * p, np.float32)
        dx = np.zeros(n * c * h * h, np.float32)
        df = np.zeros(k * c * r * r, np.float32)
        t0 = time.perf_counter()  # inputs generated outside the timed region
        orc.conv_forward(xg, x, [k, c, r, r], f, cg, yg, y, threads=threads)
        orc.conv_backward_data([k, c, r, r], f, yg, dy, cg, xg, dx)
        orc.conv_backward_filter(xg, x, yg, dy, cg, [k, c, r, r], df, threads=threads)
        dt += time.perf_counter() - t0
        total_flops += 3 * layer_flops(n, c, h, k, r, u, pad)
        if gpu_out is not None and name in gpu_out:
            for pas, got, ref in zip(PASSES, gpu_out[name], (y, dx, df)):
                errs[f"{name}.{pas}"] = float(np.abs(got.astype(np.float64) - ref).max()
                                             / max(float(np.abs(ref).max()), 1e-30))
    return total_flops / dt / 1e12, dt, errs


REF_LAYERS_SRC = os.path.join(ROOT, "baseline", "_ref")


def ref_worker(engine, n, steps, warmup, threads):
    """One arm of the real reference (baseline/_ref, the unmodified numpy
    package through its public API: conv_forward / conv_backward_data /
    conv_backward_filter, pkg/src/dnnp/conv.py:565-751) on AlexNet conv1-5
    at N=n; prints per-step seconds as JSON.  Run in a subprocess so that
    OPENBLAS_NUM_THREADS is fixed before numpy loads."""
    sys.path.insert(0, REF_LAYERS_SRC)
    from dnnp.conv import (ConvDesc, FilterView, conv_backward_data, conv_backward_filter,
                           conv_forward)
    from dnnp.tensor import TensorView, empty_view, make_desc
    layers = []
    for idx, (name, c, h, k, r, u, pad) in enumerate(ALEXNET):
        p = out_extent(h, r, u, pad)
        g = np.random.default_rng([2014, idx])  # reference bench.py:151-157
        x = g.uniform(-0.5, 0.5, (n, c, h, h)).astype(np.float32)
        f = g.uniform(-0.5, 0.5, (k, c, r, r)).astype(np.float32)
        dy = g.uniform(-0.5, 0.5, (n, k, p, p)).astype(np.float32)
        layers.append((ConvDesc(u, u, pad, pad), TensorView.from_array(x),
                       FilterView.from_array(f), TensorView.from_array(dy),
                       empty_view(make_desc(n, k, p, p)), empty_view(make_desc(n, c, h, h)),
                       FilterView.from_array(np.zeros_like(f))))

    def step():
        for cd, xv, fv, dyv, yv, dxv, dfv in layers:
            conv_forward(xv, fv, cd, engine, yv, threads=threads)
            conv_backward_data(dyv, fv, cd, engine, dxv, threads=threads)
            conv_backward_filter(dyv, xv, cd, engine, dfv, threads=threads)
    for _ in range(warmup):
        step()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"engine": engine, "n": n, "seconds": ts}))


def run_reference_arm(engine, n, steps, warmup):
    """Spawn ref_worker: implicit = the paper's algorithm with the
    reference's own tile threads (--threads nproc, OPENBLAS_NUM_THREADS=1);
    direct = the strongest reference CPU path (BLAS threads = nproc; the
    direct engine ignores --threads, conv.py:575-576).  Returns
    (TFLOP/s median, seconds per step median) or None if unavailable."""
    if not os.path.isdir(os.path.join(REF_LAYERS_SRC, "dnnp")):
        return None
    nproc = os.cpu_count() or 1
    env = dict(os.environ)
    env["OPENBLAS_NUM_THREADS"] = "1" if engine == "implicit" else str(nproc)
    env["OMP_NUM_THREADS"] = env["OPENBLAS_NUM_THREADS"]
    threads = nproc if engine == "implicit" else 1
    cmd = [sys.executable, os.path.abspath(__file__), "--ref-worker", engine, "--batch", str(n),
           "--steps", str(steps), "--warmup", str(warmup), "--ref-threads", str(threads)]
    try:
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
        rec = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None
    sec = float(np.median(rec["seconds"]))
    flops = 3 * sum(layer_flops(n, c, h, k, r, u, pad) for _, c, h, k, r, u, pad in ALEXNET)
    return flops / sec / 1e12, sec


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def main_reference(args):
    """--impl reference: the REAL reference (baseline/_ref, unmodified numpy
    package) on the host cores, same metric/config, a bounded sample per
    step: its direct engine (the strongest reference CPU path, BLAS over all
    cores) is the line's value; the implicit engine (the paper's algorithm)
    is reported beside it.  Falls back to the C oracle port only when
    baseline/_ref is missing."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    nproc = os.cpu_count() or 1
    sample_n = args.ref_n
    direct = run_reference_arm("direct", sample_n, args.steps, min(args.warmup, 1))
    implicit = run_reference_arm("implicit", REF_SAMPLE_N, 1, 0) if direct else None
    if direct is not None:
        value, sec = direct
        kind = "reference"
        sample = (f"AlexNet conv1-5 fwd+bwd_data+bwd_filter fp32 at N={sample_n} per step "
                  "(config N=128 scaled: flops linear in N); unmodified reference package "
                  "(baseline/_ref) direct engine, OpenBLAS over all cores")
    else:
        vals = [cpu_baseline(nproc, sample_n=REF_SAMPLE_N)[:2] for _ in range(args.steps)]
        value = float(np.median([v for v, _ in vals]))
        sec = float(np.median([d for _, d in vals]))
        kind = "port"
        sample = (f"AlexNet conv1-5 at N={REF_SAMPLE_N}: C oracle restating the reference "
                  "implicit engine (baseline/_ref missing)")
    cb = {"value": value, "unit": "TFLOP/s", "cores": nproc, "kind": kind, "sample": sample,
          "cpu_model": cpu_model()}
    if implicit is not None:
        cb["engines"] = {"direct": round(direct[0], 5), "implicit": round(implicit[0], 5),
                         "implicit_sample_n": REF_SAMPLE_N}
    print(json.dumps({
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "alexnet_conv1-5_fwd_bwdd_bwdf_N128_fp32_nchw",
                   "sample_n": sample_n},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--math", type=int, default=0,
                    help="0 default (BF16x3), 1 SIMT fp32, 2 force BF16x3, 3 3xTF32")
    ap.add_argument("--eager", action="store_true",
                    help="submit every step eagerly (no CUDA-graph replay at N=1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--no-bw", action="store_true", help="skip the bandwidth-primitive table")
    ap.add_argument("--no-sweep", action="store_true", help="skip the small-batch sweep")
    ap.add_argument("--batch", type=int, default=N_PER_GPU)
    ap.add_argument("--ref-n", type=int, default=16,
                    help="--impl reference: images per timed CPU step")
    ap.add_argument("--ref-worker", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--ref-threads", type=int, default=1, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ref_worker:
        return ref_worker(args.ref_worker, args.batch, args.steps, args.warmup, args.ref_threads)
    if args.impl == "reference":
        return main_reference(args)
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist
    import paper_1410_0759_b200 as dp

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        # NCCL INFO lines (transport / ring setup) in the log: evidence of the
        # ranks' communicator for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=device)
    dp.set_math(args.math)

    layers = make_inputs(args.batch, device, torch)
    build_views(dp, layers, torch, device)
    # dW allreduces on a communication stream, overlapped with the following
    # layers' work; the step waits for them at its end (inside the timing)
    overlap = None
    allreduce = None
    comm_note = None
    if ws > 1:
        # the library's own NCCL communicator (libdnnp loads libnccl; torch
        # only broadcasts the 128-byte unique id and runs the barriers)
        try:
            from paper_1410_0759_b200.dist import NativeOverlappedAllreduce
            overlap = NativeOverlappedAllreduce.from_torch()
            comm_note = "libdnnp NCCL communicator (dnnp_nccl_comm_create), comm stream"
        except Exception as e:
            from paper_1410_0759_b200.dist import OverlappedAllreduce
            overlap = OverlappedAllreduce()
            comm_note = f"torch.distributed NCCL (native comm failed: {type(e).__name__})"
        allreduce = overlap.submit
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    for _ in range(args.warmup):
        run_step(dp, layers, torch, allreduce=allreduce)
    torch.cuda.synchronize()

    nl = len(layers)
    nops = nl * 3

    # per-op breakdown and the dominant kernel: an instrumented eager pass
    # (per-op events + CUDA events around every main GEMM kernel)
    op_ms = {(li, pi): [] for li in range(nl) for pi in range(3)}
    pre_kern = {}
    for _ in range(2):
        evs = {(li, pi): (torch.cuda.Event(enable_timing=True),
                          torch.cuda.Event(enable_timing=True))
               for li in range(nl) for pi in range(3)}
        flush.fill_(1.0)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        dp.kernel_timing(True)
        run_step(dp, layers, torch, events=evs, allreduce=allreduce)
        torch.cuda.synchronize()
        kt = dp.kernel_times()
        dp.kernel_timing(False)
        for key, (a, b) in evs.items():
            op_ms[key].append(a.elapsed_time(b))
        if len(kt) == nops:  # one main kernel per op, ops in step order
            for i, (ms, _tag) in enumerate(kt):
                pre_kern.setdefault(i, []).append(ms)
    if pre_kern:
        dom_idx = max(range(nops), key=lambda i: float(np.sum(pre_kern.get(i, [0.0]))))
    else:
        dom_idx = max(op_ms, key=lambda k: float(np.sum(op_ms[k])))
        dom_idx = dom_idx[0] * 3 + dom_idx[1]

    # The timed steps.  One-GPU runs capture the step (15 library calls,
    # ~50 kernels) once into a CUDA graph and replay it: the same kernels on
    # the same data, without per-launch host latency between them.  The
    # dominant kernel is bracketed by CUDA events recorded as external event
    # nodes of the graph (two nodes: timing every kernel this way costs ~8%
    # of the step), so each replay times it inside the timed region.
    # Multi-GPU runs capture the step too when the dW reductions go through
    # the library's own NCCL communicator (the same submission as N=1);
    # --eager forces eager everywhere.
    graph, graph_note = None, "eager"
    launches_per_step = None
    native_comm = comm_note is not None and comm_note.startswith("libdnnp")
    if (ws == 1 or native_comm) and not args.eager:
        try:
            dp.kernel_timing(True, only=dom_idx)
            l0 = dp.kernel_launch_count()
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    run_step(dp, layers, torch, allreduce=allreduce)
            launches_per_step = dp.kernel_launch_count() - l0
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            graph, graph_note = g, "cuda_graph"
        except Exception as e:  # fall back to eager submission
            dp.kernel_timing(False)
            graph, graph_note = None, f"eager (graph capture failed: {type(e).__name__})"
            torch.cuda.synchronize()

    step_ms = []
    kern_ms = {}
    launches0 = dp.kernel_launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush, outside the timed window
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            if graph is None:
                dp.kernel_timing(True, only=dom_idx)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            if graph is not None:
                graph.replay()
            else:
                run_step(dp, layers, torch, allreduce=allreduce)
            s1.record()
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            kt = dp.kernel_times()
            if len(kt) == 1:
                kern_ms.setdefault(dom_idx, []).append(kt[0][0])
    dp.kernel_timing(False)
    if graph is not None:
        launches = launches_per_step * args.steps
    else:
        launches = dp.kernel_launch_count() - launches0
    # the other ops' kernel times: from the instrumented eager pass
    for i, v in pre_kern.items():
        kern_ms.setdefault(i, v)

    # sustained: the same graph replayed back to back for >= 3 s (no flush,
    # no host sync between steps), clocks sampled meanwhile -- the rate a
    # training loop sees once the GPU settles at its power-limited clock
    sustained = None
    if graph is not None and not args.no_sustained:
        try:
            nrep = max(1, int(3000.0 / max(float(np.median(step_ms)), 0.05)))
            if ws > 1:
                # every rank must replay the same number of graphs: each one
                # holds the dW allreduces (a mismatch would hang the group)
                t = torch.tensor([nrep], device=device, dtype=torch.int64)
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                nrep = int(t.item())
                dist.barrier()
            torch.cuda.synchronize()
            with ClockSampler(local) as clk_s:
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record()
                for _ in range(nrep):
                    graph.replay()
                a1.record()
                torch.cuda.synchronize()
            sec = a0.elapsed_time(a1) / 1e3
            sflops = 3 * sum(L["flops"] for L in layers)
            sustained = {"seconds": round(sec, 3), "steps": nrep,
                         "ms_per_step": round(sec * 1e3 / nrep, 4),
                         "tflops": round(sflops * nrep / sec / 1e12, 2),
                         "clocks": clk_s.summary(),
                         "tf32_sustained_peak": sustained_tf32_peak(),
                         "note": "graph replays back to back, L2 not flushed, inputs resident"}
        except Exception as e:
            print(f"sustained run failed: {type(e).__name__}: {e}", file=sys.stderr)

    # the fp32 split sweep: the same step (same calls, same data) in the
    # 3xTF32 mode, replayed as a graph (N=1 only): step time, throughput and
    # the fraction of each split's own tensor ceiling (BF16x3: bf16 / 3,
    # 3xTF32: tf32 / 3 = bf16 / 6)
    tf32_ms = None
    if graph is not None and args.math == 0:
        try:
            dp.set_math(3)
            run_step(dp, layers, torch)
            torch.cuda.synchronize()
            cap3 = torch.cuda.Stream()
            cap3.wait_stream(torch.cuda.current_stream())
            g3 = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap3):
                with torch.cuda.graph(g3, stream=cap3):
                    run_step(dp, layers, torch)
            torch.cuda.synchronize()
            ts = []
            for _ in range(max(3, args.steps)):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
                g3.replay()
                t1.record()
                torch.cuda.synchronize()
                ts.append(t0.elapsed_time(t1))
            tf32_ms = float(np.median(ts))
            del g3
        except Exception as e:  # report, never fail the headline
            print(f"tf32x3 sweep failed: {type(e).__name__}: {e}", file=sys.stderr)
            tf32_ms = None
        finally:
            dp.set_math(args.math)
            run_step(dp, layers, torch)  # leave the BF16x3 results in the buffers
            torch.cuda.synchronize()

    # the framework path: fused backward entry, replayed as a graph (N=1 only)
    fused_ms = None
    if graph is not None and hasattr(dp, "conv_backward"):
        try:
            run_step_fused(dp, layers, torch)
            torch.cuda.synchronize()
            cap2 = torch.cuda.Stream()
            cap2.wait_stream(torch.cuda.current_stream())
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap2):
                with torch.cuda.graph(g2, stream=cap2):
                    run_step_fused(dp, layers, torch)
            torch.cuda.synchronize()
            ts = []
            for _ in range(max(3, args.steps)):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record()
                g2.replay()
                f1.record()
                torch.cuda.synchronize()
                ts.append(f0.elapsed_time(f1))
            fused_ms = float(np.median(ts))
            del g2
        except Exception:
            fused_ms = None

    # eager submission of the same step, uninstrumented (for reference)
    eager_ms = []
    for _ in range(3):
        flush.fill_(1.0)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        run_step(dp, layers, torch, allreduce=allreduce)
        a1.record()
        torch.cuda.synchronize()
        eager_ms.append(a0.elapsed_time(a1))
    # host copies of the last step's results (parity check in the cpu leg)
    gpu_out = {}
    if ws == 1 and not args.no_cpu:
        for L in layers:
            gpu_out[L["name"]] = (L["yv"].buf.cpu().numpy(), L["dxv"].buf.cpu().numpy(),
                                  L["df"].cpu().numpy())
    if os.environ.get("DNNP_BENCH_DEBUG"):
        for (li, pi), v in op_ms.items():
            print(f"{layers[li]['name']}.{PASSES[pi]}: " + " ".join(f"{x:.3f}" for x in v),
                  file=sys.stderr)
    total_ms = float(np.sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    step_flops = 3 * sum(L["flops"] for L in layers)
    value = step_flops * ws * args.steps / (total_ms / 1e3) / 1e12

    hbm, bf16, peak_src = peaks()
    tf32_peak = bf16 / 2.0
    per = {}
    dominant, dom_ms = (dom_idx // 3, dom_idx % 3), float("inf")
    for (li, pi), v in op_ms.items():
        L = layers[li]
        avg = float(np.mean(v))
        tf = L["flops"] / (avg / 1e3) / 1e12
        ent = {"ms": round(avg, 4), "tflops": round(tf, 2),
               "pct_tf32_peak": round(100 * tf / tf32_peak, 1)}
        kv = kern_ms.get(li * 3 + pi)
        if kv:
            kavg = float(np.mean(kv))
            ent["kernel_ms"] = round(kavg, 4)
            ent["kernel_tflops"] = round(L["flops"] / (kavg / 1e3) / 1e12, 2)
        per[f"{L['name']}.{PASSES[pi]}"] = ent

    dl, dpi = dominant
    kv = kern_ms.get(dl * 3 + dpi)
    dom_avg = float(np.mean(kv)) if kv else float(np.mean(op_ms[dominant]))
    achieved = layers[dl]["flops"] / (dom_avg / 1e3) / 1e12
    traffic = None
    ingest = None
    tpath = os.path.join(ROOT, "profiles", "dominant_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            key = f"{layers[dl]['name']}.{PASSES[dpi]}"
            traffic = tj.get(key)
            ib = tj.get("ingest", {}).get(key)
            if ib:
                # L2 -> SM operand ingest (ncu bytes per launch over the live
                # kernel time) against ~57 B/clk/SM x 148 SMs at the max clock
                # (profiles/r01/tma_burst_probe.txt): the bound of narrow-N GEMMs
                ceil_tbs = 57.0 * 148 * 1.965e9 / 1e12
                ach = ib / (dom_avg / 1e3) / 1e12
                ingest = {"bytes_per_launch": ib, "achieved_TBps": round(ach, 2),
                          "ceiling_TBps": round(ceil_tbs, 2), "frac": round(ach / ceil_tbs, 3)}
        except Exception:
            traffic = None

    # the dominant op's DRAM traffic with its operand packs (ncu over the
    # op's kernels, profiles/r02/op_traffic.json) against its algorithmic
    # x + f + y bytes: the pack pre-pass's share of the traffic
    op_traffic = None
    opath = os.path.join(ROOT, "profiles", "r02", "op_traffic.json")
    if os.path.exists(opath):
        try:
            op_traffic = json.load(open(opath))["ops"].get(f"{layers[dl]['name']}.{PASSES[dpi]}")
        except Exception:
            op_traffic = None

    # ---- e2e: same step through the C ABI with pinned HOST buffers --------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(dp, layers, torch, device, ws, args, step_flops)

    line = {
        "metric": METRIC,
        "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic uniform(-0.5,0.5), default_rng([2014, layer]) as reference bench",
        "config": {"workload": "alexnet_conv1-5_fwd_bwdd_bwdf_N128_fp32_nchw",
                   "batch_per_gpu": args.batch, "global_batch": args.batch * ws,
                   "layers": "torchvision AlexNet conv1-5 (64/192/384/256/256)",
                   "parallelism": f"batch-shard dp{ws}" + (" + dW allreduce" if ws > 1 else ""),
                   "comm": comm_note,
                   "l2": "flushed (256 MiB write) between timed steps",
                   "submission": graph_note,
                   "eager_ms_per_step": round(float(np.median(eager_ms)), 4),
                   "fused_backward_ms_per_step": (round(fused_ms, 4) if fused_ms else None),
                   "math": ["default(tcgen05 BF16x3 when eligible)", "simt_fp32",
                            "tcgen05_bf16x3", "tcgen05_3xtf32"][args.math]},
        "pct_tf32_peak": round(100 * value / ws / tf32_peak, 2),
        "per_layer": per,
        "per_layer_note": ("ms / tflops: per-op CUDA events of an instrumented eager pass; "
                           "kernel_ms: the dominant kernel's from the timed steps, the others' "
                           "from the instrumented pass"),
        "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": tf32_peak,
                     "unit": "TFLOP/s", "frac": round(achieved / tf32_peak, 4),
                     "traffic": traffic,
                     "kernel": f"{layers[dl]['name']}.{PASSES[dpi]}",
                     "kernel_ms": round(dom_avg, 4),
                     "timing": ("CUDA events around the main GEMM kernel inside the timed steps"
                                + (" (external event nodes of the replayed graph)"
                                   if graph is not None else "")
                                if kv else "CUDA events around the whole op"),
                     "peak_basis": f"TF32 dense = 1/2 of bf16 {bf16} TF/s, {peak_src}",
                     "bf16x3_ceiling": round(bf16 / 3.0, 1),
                     "frac_of_bf16x3_ceiling": round(achieved / (bf16 / 3.0), 4),
                     "work_per_launch_flops": layers[dl]["flops"],
                     "l2_to_sm_ingest": ingest,
                     "op_traffic": op_traffic},
        "sustained": sustained,
        "math_sweep": math_sweep(step_flops, total_ms / args.steps, tf32_ms, bf16),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if rank == 0 and ws == 1 and not args.no_sweep:
        try:
            line["small_batch_sweep"] = small_batch_sweep(dp, torch)
        except Exception as e:
            print(f"small-batch sweep failed: {type(e).__name__}: {e}", file=sys.stderr)
    if rank == 0 and ws == 1 and not args.no_bw:
        try:
            line["bandwidth_ops"] = bandwidth_ops(dp, torch, hbm)
        except Exception as e:
            print(f"bandwidth ops failed: {type(e).__name__}: {e}", file=sys.stderr)
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        # parity of the benchmarked step itself: the C oracle on the same
        # N=128 inputs, compared with the GPU results of the last step
        v, dt, perr = cpu_baseline(threads, sample_n=CPU_SAMPLE_N,
                                   gpu_out=gpu_out if args.batch == CPU_SAMPLE_N else None)
        if perr:
            line["parity"] = {"vs": "C oracle (oracle/, pinned to reference golden vectors)",
                              "metric": "max|gpu - oracle| / max|oracle| per layer and pass",
                              "tolerance": 1e-4, "max": max(perr.values()),
                              "pass": max(perr.values()) <= 1e-4,
                              "errors": {k: float(f"{e:.3g}") for k, e in perr.items()}}
        direct = run_reference_arm("direct", REF_BASE_N, 2, 1)
        implicit = run_reference_arm("implicit", REF_SAMPLE_N, 1, 0) if direct else None
        cb = {"unit": "TFLOP/s", "cores": threads, "cpu_model": cpu_model(),
              "c_oracle_port": {"value": round(v, 5), "sample": (
                  f"N={CPU_SAMPLE_N} ({dt:.1f} s): C restatement of the reference implicit "
                  f"engine, fwd/bwd-filter tiles over {threads} threads, bwd-data serial "
                  "(as conv.py:668-670)")}}
        if direct is not None:
            cb.update({"value": round(direct[0], 5), "kind": "reference",
                       "sample": (f"AlexNet conv1-5 fwd+bwd_data+bwd_filter fp32 at "
                                  f"N={REF_BASE_N} per step (flops linear in N): unmodified "
                                  "reference package (baseline/_ref), direct engine, OpenBLAS "
                                  f"over {threads} cores"),
                       "engines": {"direct": round(direct[0], 5),
                                   "implicit": round(implicit[0], 5) if implicit else None,
                                   "implicit_sample_n": REF_SAMPLE_N}})
        else:
            cb.update({"value": round(v, 5), "kind": "port",
                       "sample": cb["c_oracle_port"]["sample"]})
        line["cpu_baseline"] = cb
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))


def math_sweep(step_flops, bf16x3_ms, tf32x3_ms, bf16_peak):
    """Both fp32 splits of the same step against their own tensor ceilings:
    BF16x3 issues 3 bf16 MMAs per product (ceiling bf16 / 3), 3xTF32 issues 3
    tf32 MMAs at half the bf16 rate (ceiling bf16 / 6)."""
    out = {}
    for name, ms, ceil in (("bf16x3", bf16x3_ms, bf16_peak / 3.0),
                           ("tf32x3", tf32x3_ms, bf16_peak / 6.0)):
        if ms is None:
            out[name] = None
            continue
        tf = step_flops / (ms / 1e3) / 1e12
        out[name] = {"ms_per_step": round(ms, 4), "tflops": round(tf, 2),
                     "ceiling_tflops": round(ceil, 1), "frac_of_ceiling": round(tf / ceil, 4)}
    out["note"] = ("same AlexNet conv1-5 step (graph replay, L2 flushed); algorithmic flops; "
                   "the split's extra MMAs are not counted")
    return out


def bandwidth_ops(dp, torch, hbm_peak):
    """BASELINE configs[4] / SURVEY 8(d) "B": the bandwidth-bound primitives
    at their shapes (activation and 3x3/2 pooling on 128x64x55x55, softmax
    per-image 1024x1000x1x1 and per-spatial 16x21x64x64), fp32, on dense
    NCHW, NHWC and a channel slice [16:48) of a 64-channel parent.  Each op
    is timed alone: a 1 GiB write plus a 256 MiB read flush L2 (empty and
    clean) before it, CUDA events around its launch on the library's stream
    (the launch is queued behind the flush, so host dispatch is outside the
    window), median of 5.  Algorithmic bytes per SURVEY 8(d)."""
    wflush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
    rflush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def view(n, c, h, w, layout):
        if layout == "slice":
            buf = torch.rand(n * 64 * h * w, device="cuda") - 0.5
            d = dp.make_desc(n, 32, h, w, layout="custom", strides=[64 * h * w, h * w, w, 1])
            return dp.TensorView(d, buf[16 * h * w:])
        d = dp.make_desc(n, c, h, w, layout=layout)
        return dp.TensorView(d, torch.rand(d.max_offset() + 1, device="cuda") - 0.5)

    def timed(op):
        op()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            wflush.fill_(1.0)
            rflush.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    out = {}
    for lay in ("nchw", "nhwc", "slice"):
        c = 32 if lay == "slice" else 64
        x, y, dy, dx = (view(128, c, 55, 55, lay) for _ in range(4))
        E = 128 * c * 55 * 55
        ops = [("act_fwd_relu", 8 * E, lambda: dp.activation_forward("relu", x, y)),
               ("act_bwd_relu", 12 * E, lambda: dp.activation_backward("relu", y, dy, dx))]
        for kind in ("max", "average"):
            pd = dp.PoolingDesc(kind, 3, 3, 2, 2, 0, 0)
            py, pdy = view(128, c, 27, 27, lay), view(128, c, 27, 27, lay)
            am = (torch.empty((128, c, 27, 27), dtype=torch.int64, device="cuda")
                  if kind == "max" else None)
            Ep = 128 * c * 27 * 27
            byt = 4 * E + (12 if kind == "max" else 4) * Ep
            dp.pool_forward(pd, x, py, am)
            ops.append((f"pool_fwd_{kind}", byt, lambda pd=pd, py=py, am=am:
                        dp.pool_forward(pd, x, py, am)))
            ops.append((f"pool_bwd_{kind}", byt, lambda pd=pd, py=py, pdy=pdy, am=am:
                        dp.pool_backward(pd, py, pdy, x, dx, am)))
        for mode, (n, cc, h, w) in (("per_image", (1024, 1000, 1, 1)),
                                    ("per_spatial", (16, 21, 64, 64))):
            if lay == "slice":
                cc = 32
            a, b, d2 = view(n, cc, h, w, lay), view(n, cc, h, w, lay), view(n, cc, h, w, lay)
            En = n * cc * h * w
            ops.append((f"softmax_fwd_{mode}", 8 * En, lambda a=a, b=b, mode=mode:
                        dp.softmax_forward(mode, a, b)))
            ops.append((f"softmax_bwd_{mode}", 12 * En, lambda a=a, b=b, d2=d2, mode=mode:
                        dp.softmax_backward(mode, a, b, d2)))
        for name, byt, op in ops:
            ms = timed(op)
            gbs = byt / (ms / 1e3) / 1e9
            out[f"{name}.{lay}"] = {"bytes": int(byt), "us": round(ms * 1e3, 2),
                                    "GBps": round(gbs, 1), "frac_hbm": round(gbs / hbm_peak, 3)}
    del wflush, rflush
    return {"hbm_peak_GBps": hbm_peak, "dtype": "f32", "ops": out,
            "method": "L2 flushed clean (1 GiB write + 256 MiB read) before each op; CUDA "
                      "events around the op; median of 5; algorithmic bytes (SURVEY 8(d))"}


SWEEP_LAYERS = [  # OverFeat-fast conv2 / conv3 (suites/overfeat_vgg.suite): C, H, K, R, pad
    ("of_conv2", 96, 24, 256, 5, 2),
    ("of_conv3", 256, 12, 512, 3, 1),
]
SWEEP_BATCHES = (1, 2, 4, 8, 16, 32, 64, 128, 256)


def small_batch_sweep(dp, torch):
    """BASELINE configs[2]: forward throughput across minibatch sizes
    (reference bench.py:260-281 batch_sweep; rate relative to the best in the
    sweep).  Two per-call times: `device` = 20 calls replayed as one CUDA
    graph (the GPU's own time, no host dispatch), `eager` = 20 back-to-back
    calls through the Python API without synchronisation (max of host
    submission and GPU time, what an eager framework loop sees)."""
    out = {}
    for name, c, h, k, r, pad in SWEEP_LAYERS:
        rows = []
        for n in SWEEP_BATCHES:
            p = out_extent(h, r, 1, pad)
            g = np.random.default_rng([2014, n])
            x = torch.from_numpy(g.uniform(-0.5, 0.5, n * c * h * h).astype(np.float32)).cuda()
            f = torch.from_numpy(g.uniform(-0.5, 0.5, k * c * r * r).astype(np.float32)).cuda()
            xv = dp.TensorView(dp.make_desc(n, c, h, h), x)
            fv = dp.FilterView(dp.make_filter_desc(k, c, r, r), f)
            yv = dp.empty_view(dp.make_desc(n, k, p, p), device="cuda")
            cd = dp.ConvDesc(1, 1, pad, pad)
            op = lambda: dp.conv_forward(xv, fv, cd, "implicit", yv)  # noqa: E731
            for _ in range(3):
                op()
            torch.cuda.synchronize()
            reps = 20
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(gr, stream=s):
                    for _ in range(reps):
                        op()
            torch.cuda.synchronize()
            gr.replay()  # the first launch of a graph uploads it: not timed
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            dev_us = e0.elapsed_time(e1) * 1e3 / (3 * reps)
            del gr
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                op()
            e1.record()
            torch.cuda.synchronize()
            eager_us = e0.elapsed_time(e1) * 1e3 / reps
            fl = layer_flops(n, c, h, k, r, 1, pad)
            rows.append({"n": n, "device_us": round(dev_us, 2), "eager_us": round(eager_us, 2),
                         "device_tflops": round(fl / dev_us / 1e6, 2),
                         "eager_tflops": round(fl / eager_us / 1e6, 2)})
        best = max(rr["device_tflops"] for rr in rows)
        best_e = max(rr["eager_tflops"] for rr in rows)
        for rr in rows:
            rr["device_pct_of_best"] = round(100 * rr["device_tflops"] / best, 1)
            rr["eager_pct_of_best"] = round(100 * rr["eager_tflops"] / best_e, 1)
        out[name] = rows
    return {"layers": out, "pass": "forward", "dtype": "f32",
            "note": "rate relative to the best batch of the sweep (reference batch_sweep)"}


def run_e2e(dp, layers, torch, device, ws, args, step_flops):
    """Same step through the public API with pinned host buffers: every step
    copies its inputs host->device and results device->host (C-ABI staging)."""
    host = []
    h2d = d2h = 0
    for L in layers:
        n, c, h, k, r, p = L["n"], L["c"], L["h"], L["k"], L["r"], L["p"]
        hx = L["x"].cpu().pin_memory()
        hf = L["f"].cpu().pin_memory()
        hdy = L["dy"].cpu().pin_memory()
        hy = torch.empty(n * k * p * p, pin_memory=True)
        hdx = torch.empty(n * c * h * h, pin_memory=True)
        hdf = torch.empty(k * c * r * r, pin_memory=True)
        host.append(dict(
            cd=L["cd"], x=dp.TensorView(dp.make_desc(n, c, h, h), hx.numpy()),
            f=dp.FilterView(dp.make_filter_desc(k, c, r, r), hf.numpy()),
            dy=dp.TensorView(dp.make_desc(n, k, p, p), hdy.numpy()),
            y=dp.TensorView(dp.make_desc(n, k, p, p), hy.numpy()),
            dx=dp.TensorView(dp.make_desc(n, c, h, h), hdx.numpy()),
            df=dp.FilterView(dp.make_filter_desc(k, c, r, r), hdf.numpy()), keep=(hx, hf, hdy, hy, hdx, hdf)))
        fb = k * c * r * r * 4
        xb, yb = n * c * h * h * 4, n * k * p * p * 4
        h2d += (xb + fb) + (yb + fb) + (xb + yb)   # fwd, bwd-data, bwd-filter inputs
        d2h += yb + xb + fb
    def step():
        for H in host:
            dp.conv_forward(H["x"], H["f"], H["cd"], "implicit", H["y"])
            dp.conv_backward_data(H["dy"], H["f"], H["cd"], "implicit", H["dx"])
            dp.conv_backward_filter(H["dy"], H["x"], H["cd"], "implicit", H["df"])
    step()
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    ms = []
    for _ in range(steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    if os.environ.get("DNNP_BENCH_DEBUG"):
        print("e2e step ms:", " ".join(f"{m:.2f}" for m in ms), file=sys.stderr)
    tot = float(np.sum(ms))
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([tot], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    val = step_flops * ws * steps / (tot / 1e3) / 1e12
    return {"value": round(val, 3), "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "path": "C ABI with pinned host buffers (staged H2D/D2H inside every call)"}


if __name__ == "__main__":
    main()
