#!/usr/bin/env python3
"""bench.py -- FlashSVD rank-aware streaming encoder on B200.

Workload (BASELINE.json configs[1]): 12-layer BERT-Base low-rank encoder,
batch 32 per GPU, seq 512, d=768, 12 heads, FFN 3072, per-head rank 32,
out-proj / FFN rank 384, bf16, random-init factors (synthetic data).  A step
is one full 12-layer forward of every micro-batch a rank owns through
fsvd_model_fwd (the C-ABI device API), plus -- with N > 1 -- the NCCL gather
of the outputs to rank 0 (the path's only exchange).

Multi-GPU: `--gpus N` with no torchrun environment re-launches this script
as N ranks (`python -m torch.distributed.run --nproc-per-node N`), one
process per GPU.  The global batch (`--global-batch`, default 32 x N: weak
scaling; BASELINE configs[4] is `--global-batch 2048`) is split
contiguously by `shard.shard_range`; each rank runs its shard in micro-batches
of `--batch` sequences.

Prints ONE JSON line on rank 0.  `--impl reference` times the reference CPU
implementation (oracle/_ref, the unmodified reference library compiled from
its sources) on the host cores instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import datetime
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/sec & peak activation MiB, BERT-Base rank-aware encoder, seq 512"
UNIT = "tokens/s"
D, DF, H, G, R, PR, FR, LAYERS = 768, 3072, 12, 12, 32, 384, 384, 12
BATCH, SEQ = 32, 512
MODE_NAMES = {2: "flash_v1", 3: "flash_v2", 0: "dense", 1: "naive_lowrank"}
WEIGHT_SEED = 1234  # identical model on every rank and in the reference arm


def algorithmic_flops_per_token_layer(d=D, df=DF, g=G, r=R, pr=PR, fr=FR, m=SEQ):
    """F = 2d(3Gr) + 6r d + 4 M d + 4 d pr + 2 fr (2d + 2df)."""
    return 2 * d * 3 * g * r + 6 * r * d + 4 * m * d + 4 * d * pr + 2 * fr * (2 * d + 2 * df)


def ffn_flops_per_token(d=D, df=DF, fr=FR):
    return 2 * fr * (2 * d + 2 * df)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_block(args, ws):
    """The `config` object both arms print (the workload the metric is quoted on)."""
    gb = global_batch(args, ws)
    return {"workload": f"BERT-Base low-rank encoder, {args.layers} layers, global batch {gb} "
                        f"({args.batch}/GPU micro-batches), seq {args.seq}, d={D}, H={H}, d_ff={DF}, "
                        f"r={R}, pr=fr={PR}, {MODE_NAMES[args.mode]}",
            "batch_per_gpu": args.batch, "global_batch": gb, "seq_len": args.seq,
            "layers": args.layers, "mode": MODE_NAMES[args.mode],
            "parallelism": f"batch-shard x{ws}" + (" + NCCL output gather to rank 0" if ws > 1 else ""),
            "l2": "flushed (256 MiB write) between timed steps"}


def global_batch(args, ws):
    return args.global_batch if args.global_batch else args.batch * ws


# --------------------------------------------------------------------------- launcher
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(n):
    """One process per GPU: re-exec this script under torch.distributed.run
    with the same arguments; rank 0's JSON line reaches our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Clocks:
    """nvidia-smi sampler (every 10 ms, host-timestamped).  Started before the
    warm-up and waited on until it has produced a sample, so it is running
    when the timed region opens; stop() keeps the samples stamped inside
    [mark(), stop()] -- the timed region -- and falls back to the samples
    under load when the region was shorter than the sampling period."""

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self.t0 = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-i", str(gpu_index), "-lms", "10"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def wait_ready(self, timeout=10.0):
        """Block until the sampler has written its first line."""
        end = time.time() + timeout
        while self.p is not None and time.time() < end:
            try:
                if os.path.getsize(self.f.name) > 0:
                    return
            except OSError:
                pass
            time.sleep(0.01)

    def mark(self):
        self.t0 = time.time()

    def stop(self):
        if self.p is None:
            return None
        t1 = time.time()
        time.sleep(0.03)  # the sample in flight when the region closed
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]),
                             {n for n, v in zip(names, parts[5:9]) if v.lower().startswith("active")}))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return None
        mx = max(r[2] for r in rows)
        inside = [r for r in rows if self.t0 is not None and self.t0 <= r[0] <= t1 + 0.005]
        window = "timed region"
        if not inside:  # region shorter than the sampling period: samples under load
            inside = [r for r in rows if r[1] > 0.5 * mx] or rows
            window = "under load around the timed region"
        reasons = set().union(*(r[3] for r in inside))
        return {"sm_mhz": statistics.median(r[1] for r in inside), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(inside), "window": window}


# This pool's MEASURED_PEAKS.json as recorded in SURVEY.md (line 6) when the
# driver-written file is not present in the snapshot.
SURVEY_PEAKS = {"hbm_gbs": 6531.6, "bf16_tflops": 1628.9, "bf16_tflops_sustained": 1400.1}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return dict(SURVEY_PEAKS), "measured (MEASURED_PEAKS.json values recorded in SURVEY.md)"


def load_ncu_traffic(prefix):
    """DRAM bytes (read + write) per launch of the kernel whose name starts with
    `prefix`, from the newest committed `ncu --set full` summary in profiles/."""
    import glob
    import re

    def order(path):  # (round, version): r01_ncu_summary.json < r01_ncu_summary_v4.json
        m = re.search(r"r(\d+)_ncu_summary(?:_v(\d+))?\.json$", path)
        return (int(m.group(1)), int(m.group(2) or 0)) if m else (-1, -1)

    paths = glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary*.json"))
    for path in sorted(paths, key=order, reverse=True):
        try:
            with open(path) as f:
                s = json.load(f)
        except Exception:
            continue
        for name, k in s.get("kernels", {}).items():
            if name.startswith(prefix) and "dram_bytes_read" in k:
                return {"bytes": int(k["dram_bytes_read"] + k.get("dram_bytes_write", 0)),
                        "read": int(k["dram_bytes_read"]), "write": int(k.get("dram_bytes_write", 0)),
                        "source": os.path.relpath(path, ROOT), "kernel": name}
    return None


# --------------------------------------------------------------------------- reference arm
class ReferenceSample:
    """The reference CPU implementation (oracle/_ref: the unmodified reference
    library; the C restatement when it was not built) on a bounded sample of
    the bench workload: one sample = ONE layer of the same 12-layer model
    (layers taken in turn, so every layer is exercised) on `batch` sequences
    of length 512, through the reference's run_model (encoder.cpp:262-293)
    with every host thread.  Every layer has the same shape, so a 12-layer
    forward costs 12 samples: tokens/s = batch * 512 / (12 * sample time)."""

    def __init__(self, mode, batch, layers=LAYERS, seq=SEQ):
        import numpy as np
        import oracle
        from paper_2508_01506_b200 import abi
        from paper_2508_01506_b200.model import random_layer
        if not oracle.Reference.available():
            try:
                oracle.build(ref=True)
            except Exception:
                pass
        if oracle.Reference.available():
            self.chk, self.kind = oracle.Reference(), "reference"
        else:
            self.chk, self.kind = oracle.Restatement(), "port"
        self.cores = os.cpu_count() or 1
        os.environ["FLASHSVD_THREADS"] = str(self.cores)
        rng = np.random.default_rng(WEIGHT_SEED)
        self.layers = [random_layer(D, DF, H, G, R, PR, FR, rng) for _ in range(layers)]
        self.x = np.random.default_rng(7).standard_normal((batch, seq, D)).astype(np.float32)
        self.plan = abi.TilePlan(16, 16, 32, 1 << 20)
        self.mode, self.batch, self.seq, self.n = mode, batch, seq, 0

    def run(self):
        """One sample; returns its wall time in seconds."""
        layer = self.layers[self.n % len(self.layers)]
        self.n += 1
        t0 = time.perf_counter()
        self.chk.run_model(self.x, [layer], self.mode, self.plan)
        return time.perf_counter() - t0

    def tokens_per_s(self, t_sample):
        return self.batch * self.seq / (len(self.layers) * t_sample)

    def describe(self, n_samples):
        return (f"{n_samples} samples; one sample = 1 of the {len(self.layers)} layers (in turn) on "
                f"{self.batch} x {self.seq} tokens through the reference run_model "
                f"{MODE_NAMES[self.mode]} with {self.cores} threads; tokens/s of the "
                f"{len(self.layers)}-layer forward = {self.batch}*{self.seq} / "
                f"({len(self.layers)} * sample time)")


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    ref = ReferenceSample(args.mode, args.ref_batch, args.layers, args.seq)
    for _ in range(args.warmup):
        ref.run()
    times = [ref.run() for _ in range(args.steps)]
    t = sum(times) / len(times)
    tok_s = ref.tokens_per_s(t)
    cpu = {"value": tok_s, "unit": UNIT, "cores": ref.cores if ref.kind == "reference" else 1,
           "kind": ref.kind, "sample": ref.describe(args.steps)}
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (random-init SVD factors, N(0,1) activations)",
        "config": config_block(args, ws),
        "step": f"one step = one sample (see cpu_baseline.sample); ms_per_step is the measured "
                f"sample time, value extrapolates it to the {args.layers}-layer forward",
        "cpu_baseline": cpu,
        "e2e": {"value": tok_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_sample(args, steps=8, warmup=1):
    """The reference arm itself (`--impl reference`, same model, same sample)
    for `steps` samples, run on rank 0 at N=1 in a fresh process: inside the
    GPU process the reference's large per-call host allocations run measurably
    slower, and the two CPU numbers must agree."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE")}
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--steps", str(steps),
           "--warmup", str(warmup), "--mode", str(args.mode), "--ref-batch", str(args.ref_batch),
           "--layers", str(args.layers), "--seq", str(args.seq), "--batch", str(args.batch)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode != 0 or not lines:
        raise RuntimeError(f"reference arm failed: rc={r.returncode} {r.stderr[-300:]}")
    return json.loads(lines[-1])["cpu_baseline"]


# --------------------------------------------------------------------------- CPU self-test
def run_cpu_selftest(args):
    """The N>1 launcher / shard / gather / max-over-ranks path on CPU (gloo).
    The per-rank "forward" is a stand-in torch op (the sm_100a kernels need a
    B200); rank 0 checks that the gathered global batch equals the op applied
    to the unsharded batch and prints the bench line with `selftest: true`."""
    import torch
    import torch.distributed as dist
    from paper_2508_01506_b200.shard import gather_outputs, shard_range
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    gb = global_batch(args, ws)
    a, b = shard_range(gb, ws, rank)
    xg = torch.randn((gb, args.seq, 8), generator=torch.Generator().manual_seed(3))

    def fwd(t):
        return torch.tanh(t * 1.5 + 0.25)

    times = []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        outs = [fwd(xg[s:min(s + args.batch, b)]) for s in range(a, b, args.batch)]
        local = torch.cat(outs) if outs else xg[a:a]
        full = gather_outputs(local, ws, rank, gb)
        times.append(time.perf_counter() - t0)
    ms = torch.tensor([1e3 * sum(times[args.warmup:]) / args.steps])
    if ws > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        assert torch.equal(full, fwd(xg)), "gathered output differs from the unsharded op"
        print(json.dumps({"metric": METRIC, "value": gb * args.seq / (float(ms) * 1e-3), "unit": UNIT,
                          "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": float(ms), "selftest": True,
                          "shards": [list(shard_range(gb, ws, r)) for r in range(ws)],
                          "config": config_block(args, ws)}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2508_01506_b200 import abi
    from paper_2508_01506_b200.model import layer_descs, random_layer
    from paper_2508_01506_b200.shard import shard_range

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # --dist-path runs the N > 1 code (gather, pipelined e2e) on a 1-rank NCCL
    # group: the multi-rank path exercised on a single GPU
    multi = ws > 1 or args.dist_path
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    elif multi:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0,
                                world_size=1, device_id=dev)
    L = abi.lib()
    if not L.fsvd_device_available():
        raise RuntimeError("no usable sm_100 device: " + L.fsvd_last_error().decode())
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    B, M = args.batch, args.seq
    T = B * M
    mode = args.mode
    gb = global_batch(args, ws)
    s0, s1 = shard_range(gb, ws, rank)
    micro = [(s, min(s + B, s1)) for s in range(s0, s1, B)]  # this rank's micro-batches
    n_micro_max = math.ceil(max(b - a for a, b in (shard_range(gb, ws, r) for r in range(ws))) / B)
    shard_pad = n_micro_max * B  # the gather moves equal-size (padded) shards

    rng = np.random.default_rng(WEIGHT_SEED)  # identical weights on every rank
    layers = [random_layer(D, DF, H, G, R, PR, FR, rng) for _ in range(args.layers)]
    descs = layer_descs(layers)
    packs = []
    for i in range(args.layers):
        p = C.c_void_p()
        abi.check(L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
        packs.append(p)
    parr = (C.c_void_p * len(packs))(*[p.value for p in packs])
    assert L.fsvd_layer_pack_uses_tensor_cores(packs[0]) == 1
    wsb = C.c_size_t()
    abi.check(L.fsvd_workspace_bytes_ln(parr, len(packs), B, M, mode, 0, C.byref(wsb)))
    torch.cuda.synchronize(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    base_alloc = torch.cuda.memory_allocated(dev)
    work = torch.empty(wsb.value, dtype=torch.uint8, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(100 + rank)
    # this rank's shard, resident in HBM: [shard_pad, M, D] (padding rows are
    # never computed; they keep the gather's shards equal-sized)
    # The forward runs in place (fsvd_model_fwd with out == x), the dataflow of
    # the serving call fsvd_model_fwd_stream: one [B, M, d] activation buffer
    # per micro-batch; the pristine input stays on the host for the checks.
    x = torch.empty((shard_pad, M, D), device=dev, dtype=torch.bfloat16).normal_(generator=gen)
    out = x
    act_bytes = torch.cuda.max_memory_allocated(dev) - base_alloc  # workspace + shard buffer
    x0_host = x.cpu()
    gbufs = [torch.empty_like(out) for _ in range(ws)] if (multi and rank == 0) else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def fwd(i, xin=None, xout=None):
        a, b = micro[i]
        xin = x[a - s0:b - s0] if xin is None else xin
        xout = out[a - s0:b - s0] if xout is None else xout
        abi.check(L.fsvd_model_fwd(parr, len(packs), mode, 0, b - a, M, C.c_void_p(xin.data_ptr()),
                                   C.c_void_p(xout.data_ptr()), C.c_void_p(work.data_ptr()),
                                   wsb.value, sp))

    # N > 1: the output gather to rank 0 (NCCL over NVLink) is part of every
    # step, issued asynchronously right after the step's forward so that it
    # overlaps the next step's forward; consecutive steps alternate between
    # two batch buffers (and two gather destinations on rank 0), and a buffer
    # is reused only after its gather has completed
    bufs = [x, torch.empty_like(x)] if multi else [x]
    gdst = [gbufs, [torch.empty_like(out) for _ in range(ws)]] if (multi and rank == 0) else [None, None]
    pending = [None, None]
    step_no = [0]

    def step():
        k = step_no[0] % len(bufs)
        step_no[0] += 1
        if pending[k] is not None:
            pending[k].wait()
            pending[k] = None
        for i in range(len(micro)):
            a, b = micro[i]
            fwd(i, bufs[k][a - s0:b - s0], bufs[k][a - s0:b - s0])
        if multi:
            pending[k] = dist.gather(bufs[k], gdst[k], dst=0, async_op=True)

    def drain():
        for k in range(2):
            if pending[k] is not None:
                pending[k].wait()
                pending[k] = None

    clocks = Clocks(local)  # sampling from the warm-up on
    for _ in range(args.warmup):
        step()
    drain()
    torch.cuda.synchronize(dev)
    assert torch.isfinite(out[:s1 - s0].float()).all().item(), "non-finite output"
    clocks.wait_ready()

    # ---------------- timed region (device-resident inputs) ----------------
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clocks.mark()
    if multi:
        dist.barrier()
    torch.cuda.synchronize(dev)
    n0 = L.fsvd_kernel_launch_count()
    for i in range(args.steps):
        flush.zero_()  # L2 flush between steps (outside the events)
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    # the last steps' gathers complete inside the timed total
    ed0, ed1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ed0.record(stream)
    drain()
    ed1.record(stream)
    torch.cuda.synchronize(dev)
    launches = L.fsvd_kernel_launch_count() - n0
    if multi:
        dist.barrier()
    clk = clocks.stop()
    # the reference result for the e2e checks: one forward of the pristine input
    x.copy_(x0_host.to(dev))
    for i in range(len(micro)):
        fwd(i)
    torch.cuda.synchronize(dev)
    x_in = x0_host.to(dev)  # device copy of the pristine input (after the memory measurement)
    ms = (sum(a.elapsed_time(b) for a, b in evs) + ed0.elapsed_time(ed1)) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if multi:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = gb * M / (ms_max * 1e-3)

    gather_ms = None
    if multi:  # the gather alone, for the breakdown
        dist.barrier()
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(5):
            dist.gather(out, gbufs, dst=0)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gt = torch.tensor([g0.elapsed_time(g1) / 5], device=dev)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gather_ms = float(gt.item())
        if rank == 0:  # rank r's shard arrived intact
            for r in range(ws):
                a, b = shard_range(gb, ws, r)
                assert torch.isfinite(gbufs[r][:b - a].float()).all().item()
            assert torch.equal(gbufs[0], out)

    # ---------------- e2e: pinned host input -> model -> host output ----------------
    e2e = e2e_single(args, L, parr, packs, x_in, out, stream, dev) if not multi else \
        e2e_multi(args, L, parr, packs, x_in, out, work, wsb.value, stream, dev, ws, rank, gb, micro,
                  s0, shard_pad)

    # ---------------- e2e through the reference-signature drop-in ----------------
    if rank == 0 and not multi and not args.no_dropin_e2e:
        e2e["dropin"] = e2e_dropin(args, L, layers, x_in, out)

    # ---------------- dominant-kernel roofline (FFN) ----------------
    peaks, peak_src = load_peaks()
    roof = roofline(args, L, packs, work, wsb, stream, dev, peaks, peak_src, ms_max, gb, ws) \
        if rank == 0 else None

    # ---------------- peak activation memory ----------------
    mem = memory_block(args, L, parr, packs, act_bytes, ws, rank, gbufs) if rank == 0 else {}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(args)
        except Exception as e:  # report, do not fail the bench
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "weak" if not args.global_batch else "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init SVD factors, N(0,1) activations)",
            "config": config_block(args, ws),
            "e2e": e2e,
            "gpu_launches": int(launches // max(args.steps, 1)) * args.steps,
            "launches_per_step": int(launches // max(args.steps, 1)),
            "roofline": roof,
            "peak_activation_mib": mem,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        if args.dist_path and ws == 1:
            line["dist_path"] = "N > 1 code path on a 1-rank NCCL group"
        if gather_ms is not None:
            line["gather_ms"] = round(gather_ms, 3)
            line["gather_bytes_per_step"] = (ws - 1) * shard_pad * M * D * 2
        print(json.dumps(line), flush=True)
    for p in packs:
        L.fsvd_layer_pack_destroy(p)
    if multi:
        dist.destroy_process_group()
    return 0


def e2e_single(args, L, parr, packs, x, out, stream, dev):
    """fsvd_model_fwd_stream (the library's serving call): every step copies
    its batch in from pinned host memory and its result back out; copies of
    neighbouring steps overlap the forward on the library's internal streams."""
    import torch
    from paper_2508_01506_b200 import abi
    B, M = args.batch, args.seq
    T = B * M
    sp = C.c_void_p(stream.cuda_stream)
    n = max(4, args.steps)
    xh = torch.empty((B, M, D), dtype=torch.bfloat16, pin_memory=True)
    xh.copy_(x[:B].cpu())
    ohs = [torch.empty_like(xh, pin_memory=True) for _ in range(2)]
    xa = (C.c_void_p * n)(*([xh.data_ptr()] * n))
    oa = (C.c_void_p * n)(*[ohs[i & 1].data_ptr() for i in range(n)])
    sws = C.c_size_t()
    abi.check(L.fsvd_stream_workspace_bytes(parr, len(packs), B, M, args.mode, C.byref(sws)))
    swork = torch.empty(sws.value, dtype=torch.uint8, device=dev)

    def run(k):
        abi.check(L.fsvd_model_fwd_stream(parr, len(packs), args.mode, 0, B, M, k, xa, oa,
                                          C.c_void_p(swork.data_ptr()), sws.value, sp))
    run(2)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(n)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    assert torch.equal(ohs[(n - 1) & 1], out[:B].cpu()), "e2e output differs from device run"
    ms = e0.elapsed_time(e1) / n
    return {"value": round(T / (ms * 1e-3), 1), "unit": UNIT,
            "h2d_bytes_per_step": T * D * 2, "d2h_bytes_per_step": T * D * 2,
            "ms_per_step": round(ms, 4),
            "api": "fsvd_model_fwd_stream (C-ABI): per step, pinned-host bf16 batch in, "
                   "12-layer forward, result out; copies overlap neighbouring steps"}


def e2e_dropin(args, L, layers, x, out):
    """fsvd_run_model -- the C-ABI behind flashsvd::b200::run_model, the
    reference's run_model signature (encoder.hpp:90-92): fp32 host tensors in
    and out, synchronous, every layer passed as fp32 factor arrays on every
    call (the reference bench's loop, commands.cpp:289-307).  The first call
    builds and caches the device packs; the timed calls hash the factors,
    find the cached packs and run H2D -> 12 layers -> D2H."""
    import numpy as np
    import torch
    from paper_2508_01506_b200 import abi
    from paper_2508_01506_b200.model import layer_descs
    B, M = args.batch, args.seq
    xh = np.ascontiguousarray(x[:B].float().cpu().numpy())
    oh = np.zeros_like(xh)
    descs = layer_descs(layers)
    plan = abi.TilePlan(16, 16, 32, 1 << 20)

    def call():
        abi.check(L.fsvd_run_model(abi.fptr(xh), B, M, D, descs, len(layers), args.mode, plan, 0,
                                   b"layer", abi.BF16, None, abi.fptr(oh)))
    t0 = time.perf_counter()
    call()
    first = time.perf_counter() - t0
    n = 5
    t0 = time.perf_counter()
    for _ in range(n):
        call()
    ms = (time.perf_counter() - t0) / n * 1e3
    ref = out[:B].float().cpu().numpy()
    diff = float(np.abs(oh - ref).max())
    assert diff <= 0.05 * float(np.abs(ref).max()), f"drop-in output differs: {diff}"
    return {"value": round(B * M / (ms * 1e-3), 1), "unit": UNIT, "ms_per_step": round(ms, 3),
            "first_call_ms": round(first * 1e3, 1), "h2d_bytes_per_step": B * M * D * 4,
            "d2h_bytes_per_step": B * M * D * 4,
            "api": "fsvd_run_model (flashsvd::b200::run_model): fp32 host tensors, factors "
                   "passed per call, device packs found in the content-hashed pack cache; "
                   "host wall clock per synchronous call"}


def e2e_multi(args, L, parr, packs, x, out, work, wsb, stream, dev, ws, rank, gb, micro, s0,
              shard_pad):
    """N > 1 serving loop: per step every rank copies its shard in from pinned
    host memory, runs the 12-layer forward (fsvd_model_fwd), the outputs are
    gathered to rank 0 over NCCL, and rank 0 copies the global batch back to
    pinned host memory.  Two slots: step i's H2D, forward, gather and D2H
    overlap steps i-1 / i+1 on separate streams."""
    import torch
    import torch.distributed as dist
    from paper_2508_01506_b200 import abi
    M = args.seq
    sp = C.c_void_p(stream.cuda_stream)
    n = max(4, args.steps)
    xh = torch.empty_like(x, device="cpu").pin_memory()
    xh.copy_(x.cpu())
    xd = [torch.empty_like(x) for _ in range(2)]
    od = [torch.empty_like(x) for _ in range(2)]
    gbuf = [[torch.empty_like(x) for _ in range(ws)] for _ in range(2)] if rank == 0 else None
    oh = [[torch.empty_like(xh).pin_memory() for _ in range(ws)] for _ in range(2)] if rank == 0 else None
    s_in, s_comm, s_out = (torch.cuda.Stream(dev) for _ in range(3))
    ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "fwd", "gat", "out")}

    def fwd_all(xin, xout):
        for a, b in micro:
            abi.check(L.fsvd_model_fwd(parr, len(packs), args.mode, 0, b - a, M,
                                       C.c_void_p(xin[a - s0].data_ptr()),
                                       C.c_void_p(xout[a - s0].data_ptr()),
                                       C.c_void_p(work.data_ptr()), wsb, sp))

    def loop(k_steps):
        for i in range(k_steps):
            k = i & 1
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(ev["fwd"][k])  # xd[k] free once forward i-2 is done
                xd[k].copy_(xh, non_blocking=True)
                ev["in"][k].record(s_in)
            stream.wait_event(ev["in"][k])
            if i >= 2:
                stream.wait_event(ev["gat"][k])  # od[k] free once gather i-2 is done
            fwd_all(xd[k], od[k])
            ev["fwd"][k].record(stream)
            with torch.cuda.stream(s_comm):
                s_comm.wait_event(ev["fwd"][k])
                if rank == 0 and i >= 2:
                    s_comm.wait_event(ev["out"][k])  # gbuf[k] free once D2H i-2 is done
                dist.gather(od[k], gbuf[k] if rank == 0 else None, dst=0)
                ev["gat"][k].record(s_comm)
            if rank == 0:
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev["gat"][k])
                    for r in range(ws):
                        oh[k][r].copy_(gbuf[k][r], non_blocking=True)
                    ev["out"][k].record(s_out)
        stream.wait_stream(s_in)
        stream.wait_stream(s_comm)
        stream.wait_stream(s_out)

    loop(2)
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    loop(n)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = torch.tensor([e0.elapsed_time(e1) / n], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        assert torch.equal(oh[(n - 1) & 1][0], out.cpu()), "e2e rank-0 shard differs from device run"
    ms = float(ms.item())
    return {"value": round(gb * M / (ms * 1e-3), 1), "unit": UNIT,
            "h2d_bytes_per_step": gb * M * D * 2, "d2h_bytes_per_step": ws * shard_pad * M * D * 2,
            "ms_per_step": round(ms, 4),
            "api": "per rank: pinned-host shard -> fsvd_model_fwd (C-ABI) -> NCCL gather to rank 0 "
                   "-> rank 0 copies the global batch to pinned host; steps pipelined over 2 slots"}


def roofline(args, L, packs, work, wsb, stream, dev, peaks, peak_src, ms_max, gb, ws):
    import torch
    from paper_2508_01506_b200 import abi
    B, M, mode = args.batch, args.seq, args.mode
    T = B * M
    sp = C.c_void_p(stream.cuda_stream)
    ffn_variant = 2 if mode == abi.MODE_FLASH_V2 else 1
    resid = torch.randn((B, M, D), device=dev, dtype=torch.float32).to(torch.bfloat16)
    ffn_out = torch.empty_like(resid)
    # the sublayer entry points run the unfused schedules, whose transients
    # exceed the compact layer workspace: a scratch of their own (allocated
    # after the peak-memory measurement)
    work = torch.empty(max(wsb.value, T * (3 * H + 2 * G) * R * 2 * 2, T * 2 * FR * 2 * 2),
                       dtype=torch.uint8, device=dev)
    ffn_ws = C.c_size_t(work.numel())
    reps = 20
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sub = {}
    fbw = C.c_size_t()
    abi.check(L.fsvd_ffn_block_workspace_bytes(packs[0], ffn_variant, B, M, C.byref(fbw)))
    fwork = torch.empty(fbw.value, dtype=torch.uint8, device=dev)
    for name, fn in (
            ("ffn_block_fwd", lambda: L.fsvd_ffn_block_fwd(
                packs[0], ffn_variant, B, M, C.c_void_p(resid.data_ptr()),
                C.c_void_p(ffn_out.data_ptr()), C.c_void_p(fwork.data_ptr()), fbw.value, sp)),
            ("ffn_fwd", lambda: L.fsvd_ffn_fwd(
                packs[0], ffn_variant, B, M, C.c_void_p(resid.data_ptr()),
                C.c_void_p(ffn_out.data_ptr()), C.c_void_p(work.data_ptr()), ffn_ws, sp)),
            ("attention_fwd", lambda: L.fsvd_attention_fwd(
                packs[0], B, M, C.c_void_p(resid.data_ptr()), C.c_void_p(ffn_out.data_ptr()),
                C.c_void_p(work.data_ptr()), ffn_ws, sp)),
            ("outproj_fwd", lambda: L.fsvd_outproj_fwd(
                packs[0], B, M, C.c_void_p(resid.data_ptr()), C.c_void_p(ffn_out.data_ptr()),
                C.c_void_p(work.data_ptr()), ffn_ws, sp)),
            ("layer_fwd", lambda: L.fsvd_layer_fwd(
                packs[0], mode, 0, B, M, C.c_void_p(resid.data_ptr()),
                C.c_void_p(ffn_out.data_ptr()), C.c_void_p(work.data_ptr()), ffn_ws, sp))):
        for _ in range(3):
            abi.check(fn())
        torch.cuda.synchronize(dev)
        k0.record(stream)
        for _ in range(reps):
            abi.check(fn())
        k1.record(stream)
        torch.cuda.synchronize(dev)
        sub[name] = round(k0.elapsed_time(k1) / reps, 4)
    # the dominant kernel as it runs in the step: K4 with the residual + LN2
    # epilogue (fsvd_ffn_block_fwd launches exactly that kernel)
    k_ms = sub["ffn_block_fwd"]
    flops = T * ffn_flops_per_token()
    achieved = flops / (k_ms * 1e-3) / 1e12
    peak = peaks.get("bf16_tflops", SURVEY_PEAKS["bf16_tflops"])
    pair = os.environ.get("FSVD_FFN_PAIR", "1") != "0"
    kname = (("k_ffn2 (CTA pair)" if pair else "k_ffn") + " with the residual + LN2 epilogue"
             if ffn_variant == 2 else "k_ffn_stream+k_gemm_ln")
    tr = load_ncu_traffic("k_ffn2<" if pair and ffn_variant == 2 else "k_ffn<")
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": tr["bytes"] if tr else None,
            "kernel": kname, "kernel_ms": round(k_ms, 4),
            "algorithmic_flop_per_launch": flops,
            "algorithmic_bytes_per_launch": T * D * 2 * 3,
            "sublayer_ms": sub, "traffic_source": tr,
            "peak_source": f"{peak_src}: burst bf16 (kernel timed alone)",
            "model_frac_of_sustained": round(
                gb * M * args.layers * algorithmic_flops_per_token_layer() / (ms_max * 1e-3) / 1e12
                / (ws * peaks.get("bf16_tflops_sustained", SURVEY_PEAKS["bf16_tflops_sustained"])),
                4)}


def memory_block(args, L, parr, packs, act_bytes, ws, rank, gbufs):
    """Peak activation memory of one rank (identical on every rank), against
    (a) our own planner's dense-reconstruction schedules and (b) a
    dense-reconstruction GPU baseline measured now, in this run: the same
    encoder in plain PyTorch with the weights rebuilt from the factors per call
    (tools/torch_baseline.py, allocations above weights and input)."""
    from paper_2508_01506_b200 import abi
    B, M = args.batch, args.seq
    T = B * M
    es = 2
    mem = {}

    def ws_for(m):
        b = C.c_size_t()
        abi.check(L.fsvd_workspace_bytes_ln(parr, len(packs), B, M, m, 0, C.byref(b)))
        return b.value
    # Activations of one micro-batch, every schedule counted the same way: the
    # [T, d] batch buffer the forward runs in (in place, as the serving call
    # does: input in, output out of the same buffer) plus what the schedule
    # holds beside it.  The dense-reconstruction baseline keeps the residual
    # copy and one [T, d] intermediate next to its largest transient (dense
    # Q|K|V or the [T, d_ff] hidden).
    io = T * D * es
    mem["accounting"] = ("in place: one [T, d] batch buffer + schedule workspace; "
                         "baselines: + residual copy + [T, d] intermediate + largest transient")
    mem["flash_v1_mib"] = round((ws_for(abi.MODE_FLASH_V1) + io) / 2**20, 1)
    mem["flash_v2_mib"] = round((ws_for(abi.MODE_FLASH_V2) + io) / 2**20, 1)
    dense_tr = max(3 * D, DF) * T * es
    naive_tr = max(3 * G * 32 + 3 * D, PR, 2 * FR + DF) * T * es
    mem["dense_baseline_mib"] = round((2 * T * D * es + dense_tr + io) / 2**20, 1)
    mem["naive_lowrank_baseline_mib"] = round((2 * T * D * es + naive_tr + io) / 2**20, 1)
    sel = mem["flash_v2_mib"] if args.mode == abi.MODE_FLASH_V2 else mem["flash_v1_mib"]
    mem["reduction_vs_dense"] = round(1 - sel / mem["dense_baseline_mib"], 4)
    mem["reduction_vs_naive_lowrank"] = round(1 - sel / mem["naive_lowrank_baseline_mib"], 4)
    # out of place (separate input and output buffers), both sides
    mem["out_of_place"] = {
        "flash_mib": round(sel + io / 2**20, 1),
        "dense_baseline_mib": round(mem["dense_baseline_mib"] + io / 2**20, 1),
        "reduction_vs_dense": round(1 - (sel + io / 2**20) / (mem["dense_baseline_mib"] + io / 2**20), 4)}
    ours_above = ws_for(args.mode) / 2**20  # workspace (the forward runs in the input buffer)
    mem["above_weights_and_input_mib"] = round(ours_above, 1)
    mem["measured_torch_allocator_mib"] = round(act_bytes / 2**20, 1)
    if gbufs is not None:
        mem["rank0_gather_buffers_mib"] = round(sum(g.numel() * g.element_size() for g in gbufs) / 2**20, 1)
    if not args.no_torch_baseline and (B, M) == (BATCH, SEQ):
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import torch_baseline
            ref_mib = torch_baseline.peak_activation_mib("naive_lowrank", args.layers)
            mem["torch_dense_reconstruction_measured_mib"] = round(ref_mib, 1)
            mem["reduction_vs_torch_dense_reconstruction"] = round(1 - ours_above / ref_mib, 4)
            mem["torch_baseline_source"] = ("measured in this run: tools/torch_baseline.py "
                                            "peak_activation_mib('naive_lowrank'), B=32, M=512, "
                                            f"{args.layers} layers, torch.cuda.max_memory_allocated "
                                            "above weights and input")
        except Exception as e:
            mem["torch_baseline_error"] = str(e)[:200]
    mem["meter_transient_mib"] = {
        "flash": round(4 * 3 * G * B * M * R / 2**20, 1),
        "naive_lowrank": round(4 * max(3 * B * M * D, B * M * DF) / 2**20, 1),
        "dense": round(4 * (3 * B * M * D + B * H * M * M) / 2**20, 1)}
    return mem


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", type=int, default=3, help="2 = flash_v1, 3 = flash_v2")
    ap.add_argument("--batch", type=int, default=BATCH, help="micro-batch (sequences per forward)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="total sequences per step over all ranks (0: batch x N, weak scaling)")
    ap.add_argument("--seq", type=int, default=SEQ)
    ap.add_argument("--layers", type=int, default=LAYERS)
    ap.add_argument("--ref-batch", type=int, default=16,
                    help="sequences per reference sample (16: the reference's best tokens/s on 16 host cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-torch-baseline", action="store_true")
    ap.add_argument("--no-dropin-e2e", action="store_true")
    ap.add_argument("--cpu-selftest", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--dist-path", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return relaunch(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    if args.cpu_selftest:
        return run_cpu_selftest(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
