"""Benchmark of the texpr compiled-graph hot path on B200.

Headline (BASELINE.json metric, configs[1]): the fused elementwise expression
sigmoid(a*b+c)**2 - d over 2^28 fp32 elements per GPU, HBM GB/s
(20 B/element algorithmic traffic).  One step = one call of the compiled
function over device-resident inputs (5.4 GB per step > L2, so no flush is
needed).  ``e2e`` is the same metric through the public call with pinned host
inputs (H2D inside the timed region) and the result read back to the host.

Extra sections in the same JSON line: the MLP training step (config 4, and
the data-parallel config 5 when N > 1), the logistic-regression step
(config 1) and the CAReduce kernels (config 3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EW_N = 1 << 28
EW_BYTES_PER_ELEM = 20
MLP_FLOP_PER_SAMPLE = 113.75e6  # 931.87 GFLOP / 8192 samples
TF32_NOMINAL = 1130.0           # dense TF32 TFLOP/s, B200 nominal (B200_PROFILING.md); no measured TF32 peak exists


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"], "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "src": "fallback"}


class Clocks:
    """Sample SM clocks and throttle reasons during the timed region (NVML)."""

    def __init__(self, index=0):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _loop(self):
        nv = self.nv
        names = {getattr(nv, k, None): k for k in ("nvmlClocksThrottleReasonHwSlowdown",
                                                     "nvmlClocksThrottleReasonHwThermalSlowdown",
                                                     "nvmlClocksThrottleReasonSwThermalSlowdown",
                                                     "nvmlClocksThrottleReasonSwPowerCap")}
        label = {"nvmlClocksThrottleReasonHwSlowdown": "hw_slowdown",
                 "nvmlClocksThrottleReasonHwThermalSlowdown": "hw_thermal_slowdown",
                 "nvmlClocksThrottleReasonSwThermalSlowdown": "sw_thermal_slowdown",
                 "nvmlClocksThrottleReasonSwPowerCap": "sw_power_cap"}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, k in names.items():
                    if bit is not None and r & bit:
                        self.reasons.add(label[k])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- helpers

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def barrier_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def time_device_block(fn_launch, lib, stream, steps):
    """Mean ms per step of `steps` back-to-back calls bracketed by one event
    pair (a training loop: host enqueue overlaps the device work)."""
    a, b = lib.event_create(), lib.event_create()
    lib.stream_sync(stream)
    lib.event_record(a, stream)
    for _ in range(steps):
        fn_launch()
    lib.event_record(b, stream)
    lib.stream_sync(stream)
    return lib.elapsed_ms(a, b) / steps


def time_device(fn_launch, lib, stream, steps):
    """Per-step CUDA-event durations (ms) on the launching stream."""
    evs = [(lib.event_create(), lib.event_create()) for _ in range(steps)]
    lib.stream_sync(stream)
    for a, b in evs:
        lib.event_record(a, stream)
        fn_launch()
        lib.event_record(b, stream)
    lib.stream_sync(stream)
    return [lib.elapsed_ms(a, b) for a, b in evs]


# ---------------------------------------------------------------- workloads

def bench_ew(T, C, steps, warmup, lib_holder):
    import torch
    g = C.build_ew(T)
    f = T.compile(g["inputs"], g["outputs"])
    gen = torch.Generator(device="cuda").manual_seed(0)
    ins = [torch.randn(EW_N, device="cuda", dtype=torch.float32, generator=gen) for _ in range(4)]
    for _ in range(warmup):
        f.call_device(*ins)
    lib = lib_holder()
    stream = f._stream
    ms = time_device(lambda: f.call_device(*ins), lib, stream, steps)
    # correctness spot check against the oracle formula on a sample
    out = f.call_device(*ins, sync=True)
    idx = torch.randint(0, EW_N, (4096,), device="cuda", generator=gen)
    from oracle import texpr_numpy as O
    want = O.eval_composite_plain(f.order[0].op.program, [x[idx].cpu().numpy() for x in ins])[0]
    np.testing.assert_allclose(out[idx].cpu().numpy(), want, rtol=1e-5, atol=1e-6)
    return f, ins, ms


def bench_ew_e2e(f, steps=5):
    import torch
    host = [torch.randn(EW_N, dtype=torch.float32).pin_memory() for _ in range(4)]
    f(*host)  # warm: builds the chunk pipeline (slot plans, captured graphs)
    f(*host)
    t0 = time.perf_counter()
    for _ in range(steps):
        out = f(*host)
    dt = (time.perf_counter() - t0) / steps
    assert out.shape == (EW_N,)
    del host
    # the reference's own call convention: pageable NumPy arrays in, NumPy out
    rng = np.random.default_rng(2)
    arrs = [rng.standard_normal(EW_N, dtype=np.float32) for _ in range(4)]
    f(*arrs)
    t0 = time.perf_counter()
    for _ in range(max(2, steps // 2)):
        out = f(*arrs)
    dt_np = (time.perf_counter() - t0) / max(2, steps // 2)
    return dt, 4 * EW_N * 4, EW_N * 4, dt_np


def link_bandwidth(nbytes=1 << 30, reps=3):
    """Pinned host<->device copy rates on this box (the e2e path's link bound):
    H2D alone, D2H alone, and both directions at once."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    th = timed(lambda: d.copy_(h, non_blocking=True))
    td = timed(lambda: h2.copy_(d2, non_blocking=True))
    tb = timed(both)
    return {"h2d_gbs": round(nbytes / th / 1e9, 1), "d2h_gbs": round(nbytes / td / 1e9, 1),
            "duplex_gbs_each": round(nbytes / tb / 1e9, 1)}


def cpu_ew_baseline(T, C, budget_s=12.0, n=1 << 24):
    from oracle import configs as Cc
    from oracle import texpr_numpy as O
    g = Cc.build_ew(T)
    cpu = Cc.CpuFunction(T, g["inputs"], g["outputs"])
    prog = cpu.fg.toposort()[0].op.program
    ins = C.inputs_ew(n, seed=1)
    times = []
    t_start = time.perf_counter()
    while len(times) < 3 or (time.perf_counter() - t_start < budget_s and len(times) < 10):
        t0 = time.perf_counter()
        O.eval_composite(prog, ins)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": round(EW_BYTES_PER_ELEM * n / med / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{n} elements x {len(times)} reps of the reference's chunked Composite evaluation "
                      "(oracle/texpr_numpy.eval_composite_chunked, NumPy single-threaded ufuncs), kernel-only"}


def attach_cpu_path(line, T, C, args):
    """The reference's CPU path beside every config (rank 0, N=1 only): the
    real reference from baseline/_ref when installed (tools/ref_bench.py),
    else the oracle port for config 2 only."""
    tab = None
    if not args.no_cpu_table:
        from tools import ref_bench
        try:
            tab = ref_bench.table(reps=5)
        except Exception as e:  # pragma: no cover
            tab = {"error": repr(e)[:300]}
    if not tab or "error" in tab or "error" in tab.get("config2_ew_2p28", {"error": 1}):
        line["cpu_baseline"] = cpu_ew_baseline(T, C)
        if tab:
            line["cpu_path"] = tab
        return
    host = tab["host"]
    c2 = tab["config2_ew_2p28"]
    line["cpu_baseline"] = {"value": c2["kernel"], "unit": "GB/s", "cores": 1, "kind": "reference",
                            "sample": "full 2^28-element workload, texpr from baseline/_ref through its public API, "
                                      "1 warm-up + median of 5 calls; kernel-only = sum of Profile.node_time "
                                      "(NumPy elementwise is single-threaded)",
                            "e2e_value": c2["e2e"], "host_cores": host["cpu_count"], "cpu_model": host["cpu_model"]}
    line["cpu_path"] = tab
    ex = line.get("extra", {})
    pairs = (("mlp_b8192_1gpu", "config4_mlp_b8192"), ("mlp_b8192_1gpu_3xtf32", "config4_mlp_b8192"),
             ("mlp_b8192_1gpu_simt", "config4_mlp_b8192"), ("mlp_dp_global65536", "config5_mlp_global65536"),
             ("mlp_dp_global65536_3xtf32", "config5_mlp_global65536"), ("conv3x3_n32c64h56", "conv3x3_n32c64h56"),
             ("logreg_n600", "config1_logreg_n600"))
    for ours, ref in pairs:
        if isinstance(ex.get(ours), dict) and "e2e" in tab.get(ref, {}):
            r = tab[ref]
            ex[ours]["cpu_baseline"] = {"unit": r["unit"], "e2e": r["e2e"], "kernel": r["kernel"], "kind": "reference",
                                        "cores": host["cpu_count"], "blas": host["blas"]}
    if isinstance(ex.get("lstm_ptb_words_per_s"), dict) and "small" in tab.get("lstm_ptb", {}):
        r = tab["lstm_ptb"]
        ex["lstm_ptb_words_per_s"]["cpu_baseline"] = {
            "unit": "words/s", "kind": "reference", "cores": host["cpu_count"],
            **{m: {"e2e": r[m]["e2e"], "kernel": r[m]["kernel"]} for m in ("small", "medium") if m in r}}
    if isinstance(ex.get("careduce_16384sq_GBs"), dict) and "sum_axis0" in tab.get("config3_careduce_16384sq", {}):
        r = tab["config3_careduce_16384sq"]
        ex["careduce_cpu_baseline"] = {k: {"e2e": v["e2e"], "kernel": v["kernel"]} for k, v in r.items()
                                       if isinstance(v, dict)}
        ex["careduce_cpu_baseline"]["unit"] = "GB/s"
        ex["careduce_cpu_baseline"]["note"] = "the reference's argmax is ArgmaxOnehot (one-hot of the input's shape)"


def bench_mlp(T, C, B, steps, warmup, lib_holder, dp=None, n_global=None, gemm_mode="auto"):
    import torch
    g = C.build_mlp(T, B=B, n_global=n_global)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"], data_parallel=dp, gemm_mode=gemm_mode)
    x, y = C.inputs_mlp(B=B, seed=1 + (dp.rank if dp else 0))
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(warmup):
        f.call_device(xd, yd)
    lib = lib_holder()
    ms = time_device(lambda: f.call_device(xd, yd), lib, f._stream, steps)
    cost = float(f.call_device(xd, yd, sync=True)[0].item())
    return f, ms, cost


def kernel_launches(f):
    """Launch closures of the function's (single) step plan: one per kernel
    or library call the captured graph replays."""
    plan = next(iter(f._plans.values()))
    return len(plan.launches)


def tf32_peak_cublas(n=8192, iters=20):
    """cuBLAS TF32 GEMM throughput on this box (the TF32 roofline reference;
    MEASURED_PEAKS.json only has bf16)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(iters):
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    torch.backends.cuda.matmul.allow_tf32 = False
    return 2 * n ** 3 / (best * 1e-3) / 1e12


def bench_logreg(T, C, steps, warmup, lib_holder):
    import torch
    g = C.build_logreg(T)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    x, y = C.inputs_logreg()
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(warmup):
        f.call_device(xd, yd)
    lib = lib_holder()
    ms = [time_device_block(lambda: f.call_device(xd, yd), lib, f._stream, steps * 10) for _ in range(5)]
    t0 = time.perf_counter()
    for _ in range(steps):
        f(x, y)
    e2e = (time.perf_counter() - t0) / steps
    return ms, e2e, kernel_launches(f)


def bench_lstm(T, lib_holder, steps=10):
    """PTB-shaped LSTM language-model training steps through scan (PAPER.md
    section 5.3 shapes: batch 20, small 200x20 steps, medium 600x40 steps,
    vocabulary 10000, per-step softmax-xent, BPTT, SGD on every weight)."""
    import torch
    from tools.lstm_bench import CONFIGS, build
    lib = lib_holder()
    out = {}
    for name, (H, L) in CONFIGS.items():
        step, host = build(T, H, L)
        dev = [torch.from_numpy(v).cuda() for v in host]
        for _ in range(3):
            step.call_device(*dev)
        ms = time_device_block(lambda: step.call_device(*dev), lib, step._stream, steps)
        out[name] = {"hidden": H, "steps": L, "batch": 20, "ms_per_batch": round(ms, 3),
                     "words_per_s": round(20 * L / (ms * 1e-3), 1)}
        del step, dev
    return out


def bench_conv(T, lib_holder, steps=10):
    """Convolution layer training step (tools/ref_bench.conv_graph: 3x3, pad 1,
    N=32 C=K=64 56x56, forward + grad_w + grad_x + SGD) at TF32 and 3xTF32."""
    import torch
    from tools import ref_bench as R
    x, f0 = R.conv_inputs()
    xd = torch.from_numpy(x).cuda()
    lib = lib_holder()
    out = {"shape": dict(R.CONV), "flop_per_step": R.CONV_FLOP}
    for mode in ("auto", "3xtf32"):
        ins, outs, ups = R.conv_graph(T, f0)
        f = T.compile(ins, outs, updates=ups, gemm_mode=mode)
        for _ in range(3):
            f.call_device(xd)
        ms = time_device_block(lambda: f.call_device(xd), lib, f._stream, steps)
        out["tf32" if mode == "auto" else mode] = {"ms_per_step": round(ms, 3),
                                                   "tflops": round(R.CONV_FLOP / (ms * 1e-3) / 1e12, 1)}
        del f
    return out


def bench_reduce(T, C, steps, lib_holder):
    import torch
    n = 16384
    X = torch.randn(n, n, device="cuda", dtype=torch.float32, generator=torch.Generator(device="cuda").manual_seed(0))
    v = T.matrix("X", dtype="float32")
    res = {}
    lib = lib_holder()
    for kind, build in (("sum", T.sum), ("max", T.max), ("argmax", T.argmax)):
        for ax, tag in (((0,), "axis0"), ((1,), "axis1"), (None, "all")):
            f = T.compile([v], build(v, axis=ax))
            f.call_device(X)
            ms = time_device(lambda: f.call_device(X), lib, f._stream, steps)
            med = statistics.median(ms)
            res[f"{kind}_{tag}"] = round(n * n * 4 / (med * 1e-3) / 1e9, 1)
    return res


# ---------------------------------------------------------------- main

def run_reference(args):
    """--impl reference: the reference's own CPU path on the same workload and
    metric.  The unmodified reference package from baseline/_ref, called
    through its public API (texpr.compile + f(*host arrays)) on the full 2^28
    config-2 workload: ``value`` is kernel-only (the sum of its
    Profile.node_time, runtime.py:113-160), ``e2e`` the whole call including
    its input/output copies (runtime.py:163-171, :412-417).  Without
    baseline/_ref: the oracle port on a bounded 2^24 sample."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from tools import ref_bench
    tx = ref_bench.load_reference()
    if tx is not None:
        run_reference_texpr(args, tx, ws)
        return
    import paper_1605_02688_b200 as T
    from oracle import configs as C
    from oracle import texpr_numpy as O
    n = 1 << 24
    g = C.build_ew(T)
    cpu = C.CpuFunction(T, g["inputs"], g["outputs"])
    prog = cpu.fg.toposort()[0].op.program
    ins = C.inputs_ew(n, seed=1)
    for _ in range(args.warmup):
        O.eval_composite(prog, ins)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.eval_composite(prog, ins)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    v = EW_BYTES_PER_ELEM * n * args.steps / total / 1e9
    line = {"metric": "fused-elemwise HBM GB/s", "value": round(v, 3), "unit": "GB/s", "impl": "reference",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
            "higher_is_better": True, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config2: sigmoid(a*b+c)**2-d fp32", "elements_per_step": n,
                       "sample": "bounded 2^24-element sample of the 2^28 workload"},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": 1, "kind": "port",
                             "sample": f"{n} elements per step, reference chunked Composite algorithm"},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def self_launch(args) -> int:
    """``--gpus N`` without a launcher: re-exec through torch.distributed.run
    (one process per GPU over NCCL, rendezvous on 127.0.0.1).  Fails loudly
    when fewer than N GPUs are visible (the reference arm runs on rank 0 only
    and needs no GPU)."""
    import socket
    import subprocess
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
            return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_reference_texpr(args, tx, ws):
    from tools import ref_bench
    n = EW_N
    a, bb, c, d = (tx.vector(k, dtype="float32") for k in "abcd")
    f = tx.compile([a, bb, c, d], tx.sigmoid(a * bb + c) ** 2 - d, preset="fast_run")
    ins = [np.random.default_rng(i).standard_normal(n, dtype=np.float32) for i in range(4)]
    for _ in range(args.warmup):
        f(*ins)
    e2e, kern = [], []
    for _ in range(args.steps):
        k0 = sum(f.profile.node_time.values())
        t0 = time.perf_counter()
        f(*ins)
        e2e.append(time.perf_counter() - t0)
        kern.append(sum(f.profile.node_time.values()) - k0)
    host = ref_bench.host_info()
    v = EW_BYTES_PER_ELEM * n * args.steps / sum(kern) / 1e9
    ve = EW_BYTES_PER_ELEM * n * args.steps / sum(e2e) / 1e9
    line = {"metric": "fused-elemwise HBM GB/s", "value": round(v, 3), "unit": "GB/s", "impl": "reference",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * sum(kern) / args.steps, 3), "higher_is_better": True, "dtype": "f32",
            "data": "synthetic (NumPy default_rng, host)",
            "config": {"workload": "config2: sigmoid(a*b+c)**2-d, 2^28 fp32 elements (full size)",
                       "elements_per_step": n, "preset": "fast_run (one composite[5])"},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": 1, "kind": "reference",
                             "sample": f"full 2^28-element workload per step, texpr from baseline/_ref, "
                                       f"kernel-only = sum of Profile.node_time",
                             "host_cores": host["cpu_count"], "cpu_model": host["cpu_model"]},
            "e2e": {"value": round(ve, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "ms_per_step": round(1e3 * sum(e2e) / args.steps, 1),
                    "path": "texpr CompiledFunction.__call__ with NumPy inputs (includes its input/output copies)"}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-extra", action="store_true")
    ap.add_argument("--no-cpu-table", action="store_true",
                    help="skip the reference CPU-path table (headline cpu_baseline falls back to the port sample)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1605_02688_b200 as T
    from oracle import configs as C
    from paper_1605_02688_b200 import native
    pk = peaks()

    def lib_holder():
        return native.device_library(local)

    barrier(ws)
    with Clocks(local) as clk:
        f, ins, ms = bench_ew(T, C, args.steps, args.warmup, lib_holder)
    barrier(ws)
    step_ms = barrier_max(sum(ms) / len(ms), ws)
    kern_ms = statistics.mean(ms)
    bytes_step = EW_BYTES_PER_ELEM * EW_N
    value = ws * bytes_step / (step_ms * 1e-3) / 1e9
    achieved = bytes_step / (kern_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("ew_fused", None)
    line = {
        "metric": "fused-elemwise HBM GB/s", "value": round(value, 1), "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (torch.randn on device, seed 0)",
        "config": {"workload": "config2: sigmoid(a*b+c)**2-d, 2^28 fp32 elements per GPU (replicas)",
                   "elements_per_gpu": EW_N, "bytes_per_step_per_gpu": bytes_step,
                   "l2": "inputs 4.3 GB + output 1.1 GB per step > 126 MB L2 (no flush needed)",
                   "parallelism": f"replicas x{ws}"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
                     "peak_source": ("of measured: MEASURED_PEAKS.json hbm_gbs (copy)" if pk["src"] == "measured"
                                     else "of fallback: B200_PROFILING.md 6.65 TB/s (MEASURED_PEAKS.json absent)"),
                     "kernel": "tx_ew_flat (NVRTC composite[5])"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0:
        try:
            dt, hb, db, dt_np = bench_ew_e2e(f)
            line["e2e"] = {"value": round(bytes_step / dt / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": hb,
                           "d2h_bytes_per_step": db, "ms_per_step": round(dt * 1e3, 2),
                           "path": "CompiledFunction.__call__ with pinned host torch tensors -> numpy result "
                                   "(chunk-pipelined H2D / kernel / D2H, stream.py)",
                           "numpy_pageable": {"value": round(bytes_step / dt_np / 1e9, 2), "unit": "GB/s",
                                              "ms_per_step": round(dt_np * 1e3, 2),
                                              "path": "CompiledFunction.__call__ with pageable NumPy inputs"}}
            try:
                lk = link_bandwidth()
                bound_s = max(hb / (lk["h2d_gbs"] * 1e9), db / (lk["d2h_gbs"] * 1e9))
                lk["e2e_bound_gbs"] = round(bytes_step / bound_s / 1e9, 2)
                lk["e2e_frac_of_link_bound"] = round((bytes_step / dt / 1e9) / lk["e2e_bound_gbs"], 3)
                line["e2e"]["link"] = lk
            except Exception as e:  # pragma: no cover
                line["e2e"]["link"] = {"error": repr(e)[:200]}
        except Exception as e:  # pragma: no cover
            line["e2e"] = {"error": repr(e)}
    del f, ins
    torch.cuda.empty_cache()
    if not args.skip_extra:
        extra = {}
        try:
            extra["tf32_cublas_tflops_8192cubed"] = round(tf32_peak_cublas(), 1)
        except Exception as e:
            extra["tf32_cublas_tflops_8192cubed"] = repr(e)[:200]
        try:
            fm, ms_m, cost = bench_mlp(T, C, 8192, max(5, args.steps // 2), 3, lib_holder)
            med = statistics.median(ms_m)
            extra["mlp_b8192_1gpu"] = {"samples_per_s": round(8192 / (med * 1e-3), 1), "ms_per_step": round(med, 3),
                                       "tflops": round(MLP_FLOP_PER_SAMPLE * 8192 / (med * 1e-3) / 1e12, 1),
                                       "frac_of_tf32_nominal_1130": round(MLP_FLOP_PER_SAMPLE * 8192 / (med * 1e-3) / 1e12 / TF32_NOMINAL, 3),
                                       "frac_of_tf32_cublas_measured": (round(MLP_FLOP_PER_SAMPLE * 8192 / (med * 1e-3) / 1e12
                                                                              / extra["tf32_cublas_tflops_8192cubed"], 3)
                                                                        if isinstance(extra.get("tf32_cublas_tflops_8192cubed"), float) else None),
                                       "precision": "tf32 tensor-core GEMMs (fp32 accumulate)",
                                       "cost_after": cost,
                                       "graph_nodes": len([1 for n in fm.order if not getattr(n.op, 'view_capable', False)]),
                                       "launches_per_step": kernel_launches(fm)}
            del fm
        except Exception as e:
            extra["mlp_b8192_1gpu"] = {"error": repr(e)[:300]}
        torch.cuda.empty_cache()
        # the same step at the reference's arithmetic precision (fp32 sgemm):
        # 3xTF32 tensor-core GEMMs, and the CUDA-core fp32 FMA GEMMs
        for mode, label in (("3xtf32", "3xtf32 tensor-core GEMMs (big/small TF32 split, promoted fp32 "
                                        "accumulation; sgemm-class error)"),
                            ("simt", "fp32 CUDA-core FMA GEMMs (exact fp32 products)")):
            try:
                fm, ms_m, cost = bench_mlp(T, C, 8192, 5, 3, lib_holder, gemm_mode=mode)
                med = statistics.median(ms_m)
                extra[f"mlp_b8192_1gpu_{mode}"] = {
                    "samples_per_s": round(8192 / (med * 1e-3), 1), "ms_per_step": round(med, 3),
                    "tflops": round(MLP_FLOP_PER_SAMPLE * 8192 / (med * 1e-3) / 1e12, 1), "precision": label,
                    "cost_after": cost, "launches_per_step": kernel_launches(fm)}
                del fm
            except Exception as e:
                extra[f"mlp_b8192_1gpu_{mode}"] = {"error": repr(e)[:300]}
            torch.cuda.empty_cache()
        from paper_1605_02688_b200.dp import DataParallel
        for mode, key, label in (("auto", "mlp_dp_global65536", "tf32 tensor-core GEMMs (fp32 accumulate)"),
                                 ("3xtf32", "mlp_dp_global65536_3xtf32", "3xtf32 tensor-core GEMMs (sgemm-class)")):
            try:
                G = 65536
                dp = DataParallel(world_size=ws, rank=rank)
                fd, ms_d, cost_d = bench_mlp(T, C, G // ws, max(5, args.steps // 2) if mode == "auto" else 5, 3,
                                             lib_holder, dp=dp, n_global=G, gemm_mode=mode)
                med = barrier_max(statistics.median(ms_d), ws)
                extra[key] = {
                    "samples_per_s": round(G / (med * 1e-3), 1), "ms_per_step": round(med, 3), "n_gpus": ws,
                    "per_gpu_batch": G // ws, "scaling": "strong (fixed global batch)", "precision": label,
                    "tflops_total": round(MLP_FLOP_PER_SAMPLE * G / (med * 1e-3) / 1e12, 1),
                    "allreduce_buckets": len(fd._plans[next(iter(fd._plans))].buckets) if fd._plans else None,
                    "allreduce_bytes_per_step": 20037642 * 4 + 4, "cost_after": cost_d}
                del fd
            except Exception as e:
                extra[key] = {"error": repr(e)[:300]}
            torch.cuda.empty_cache()
        torch.cuda.empty_cache()
        try:
            ms_l, e2e_l, nl = bench_logreg(T, C, 20, 5, lib_holder)
            med = statistics.median(ms_l)
            extra["logreg_n600"] = {"samples_per_s": round(600 / (med * 1e-3), 1), "us_per_step": round(med * 1e3, 2),
                                    "e2e_us_per_step": round(e2e_l * 1e6, 1), "launches_per_step": nl}
        except Exception as e:
            extra["logreg_n600"] = {"error": repr(e)[:300]}
        try:
            extra["conv3x3_n32c64h56"] = bench_conv(T, lib_holder)
        except Exception as e:
            extra["conv3x3_n32c64h56"] = {"error": repr(e)[:300]}
        try:
            extra["lstm_ptb_words_per_s"] = bench_lstm(T, lib_holder)
        except Exception as e:
            extra["lstm_ptb_words_per_s"] = {"error": repr(e)[:300]}
        try:
            extra["careduce_16384sq_GBs"] = bench_reduce(T, C, 10, lib_holder)
            extra["careduce_frac_of_hbm_peak"] = {k: round(v / pk["hbm_gbs"], 3)
                                                  for k, v in extra["careduce_16384sq_GBs"].items()}
        except Exception as e:
            extra["careduce_16384sq_GBs"] = {"error": repr(e)[:300]}
        line["extra"] = extra
    if rank == 0 and ws == 1:
        attach_cpu_path(line, T, C, args)
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
