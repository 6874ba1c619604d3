#!/usr/bin/env python
"""Benchmark: target words/sec of the synchronous data-parallel training step
(BASELINE.json metric), Transformer-base by default.

  python bench.py [--gpus N --steps K --warmup W] [--config base|tiny|big|shallow|deep]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
  python bench.py --impl reference      # the reference's own CPU step (oracle/_ref)

`--gpus N` without a torchrun environment launches the N ranks itself
(torch.distributed.run, 127.0.0.1); under torchrun WORLD_SIZE must equal N.

One "step" is one synchronous update (train.cpp:221-272): every rank builds
the loss of one token-budget batch, runs forward/backward, the gradients are
all-reduced (NCCL) and Adam+EMA is applied.  Batches come from the
reference's own batching of the SURVEY 8(d) synthetic corpus, so the units
are the reference's target words (incl. </s>).

value   = sum of target words of all ranks' timed updates / max-over-ranks
          device time (CUDA events on the compute stream, no host syncs
          inside the timed region; token ids/masks uploaded per step).
e2e     = same through the public training-loop call (update_pipelined: the
          loss of every update read back to the host, one update late), wall
          clock, H2D/D2H bytes counted.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# load every kernel image when the context is created (before timing), not
# at a variant's first launch inside a timed step (lazy loading stalls a
# fresh box for tens of milliseconds on a cold file cache)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.environ.get("MTK_PKG_ROOT") or ROOT)

METRIC = "target words/sec, Transformer-base training step at 1/2/4/8 B200"


def _pure(name):
    """paper_1804_00344_b200/<name>.py loaded by path: pure Python, so the
    reference arm never imports the package (and never maps its .so files)."""
    import importlib.util
    path = os.path.join(os.environ.get("MTK_PKG_ROOT") or ROOT, "paper_1804_00344_b200",
                        name + ".py")
    spec = importlib.util.spec_from_file_location(f"_mtk_pure_{name}", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
DATA = "synthetic: SURVEY.md 8(d) splitmix64 corpus, lengths 16..32+</s>, ids uniform in [2,V)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="base")
    p.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--dropout", type=float, default=None,
                   help="override the config's dropout (SURVEY 8(d): 0 for parity, 0.1 for "
                        "throughput); TF32 mode draws device (Philox) masks")
    return p.parse_args()


def dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as td
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        td.init_process_group("gloo", rank=rank, world_size=world)
    return rank, world, local


def all_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as td
    t = torch.tensor([x], dtype=torch.float64)
    td.all_reduce(t, op=td.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as td
        td.barrier()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md).  The
    sampler starts before the warm-up (nvidia-smi's own start-up stalls the
    driver for a moment -- not inside the timed steps); only samples that
    arrive between mark() and stop() are kept (the last earlier one if the
    timed region is shorter than the 200 ms sampling period)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []  # (arrival time, line)
        self.t0 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark(self):
        self.t0 = time.monotonic()

    def stop(self, t_end=None):
        """t_end: end of the timed region (monotonic); called after later work
        so the sample straddling the end has arrived and the GPU never idles
        between the timed and the e2e legs (an idle gap lets the clocks drop)."""
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = t_end if t_end is not None else time.monotonic()
        if t_end is None:
            time.sleep(0.25)  # let the sample straddling the end arrive
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = self.t0 if self.t0 is not None else 0.0
        inside = [ln for t, ln in self.lines if t0 <= t <= t1 + 0.25]
        if not inside:
            before = [ln for t, ln in self.lines if t < t0]
            inside = before[-1:]
        for ln in inside:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return j["hbm_gbs"], j.get("bf16_tflops_sustained", j["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def traffic_per_call(config, cls, calls_per_step):
    """dram__bytes_read.sum + dram__bytes_write.sum of the class per C-ABI call,
    from the committed ncu capture of one update (tools/traffic.py)."""
    for tag in ("r02c", "r02b", "r01"):
        path = os.path.join(ROOT, "profiles", f"{tag}_traffic_{config}.json")
        if os.path.exists(path):
            break
    try:
        with open(path) as f:
            j = json.load(f)["classes"][cls]
        return round(j["dram_bytes"] / max(calls_per_step, 1)), os.path.relpath(path, ROOT)
    except Exception:
        return None, None


# ------------------------------------------------------------ CPU reference

def cpu_reference(cfg_text, vocab, threads=None, steps=2):
    """The UNMODIFIED reference trainSync (oracle/_ref, train.cpp:200-300) on a
    bounded sample of the workload: `threads` workers, each one single-sentence
    batch (token budget 66 slots) per update.  Runs 1 update (warm-up: replica
    set-up, first-touch) and then 1 + `steps` updates from the same batches;
    the rate is (words of the extra `steps` updates) / (time difference).
    Returns (words/s, words, seconds, threads)."""
    from oracle import refbind as R
    synth = _pure("synth")
    threads = threads or os.cpu_count() or 1
    n = threads * (steps + 1) * 2 + 16
    src, tgt = synth.corpus(n, vocab)
    ex = R.Examples(src, tgt)
    budget = 66
    bl = R.make_batches(ex, budget, 1)
    words = [float(b["tgt_mask"].sum()) for b in bl]
    w1 = sum(words[:threads])
    wk = sum(words[: threads * (steps + 1)])
    model = R.RefModel(cfg_text, 1)
    t0 = time.perf_counter()
    model.train(ex, workers=threads, budget=budget, seed=1, epochs=1, max_updates=1)
    t1 = time.perf_counter()
    model.train(ex, workers=threads, budget=budget, seed=1, epochs=1, max_updates=steps + 1)
    t2 = time.perf_counter()
    dt = (t2 - t1) - (t1 - t0)
    if dt <= 0:  # timing noise on a tiny sample: fall back to the full second run
        dt, wk, w1 = t2 - t1, wk, 0.0
    return (wk - w1) / dt, wk - w1, dt, threads


# ------------------------------------------------------------ B200 arm

def run_b200(a):
    rank, world, local = dist()
    from paper_1804_00344_b200 import (CONFIGS, TOKEN_BUDGET, algorithmic_flops, config_text,
                                       mtk as M)
    import torch
    if torch.cuda.device_count() < world:
        sys.exit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} GPU(s) visible")
    M.select_device(local)
    M.set_precision(a.precision)
    if world > 1:
        import torch
        import torch.distributed as td
        buf = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = torch.tensor(list(M.nccl_unique_id()), dtype=torch.uint8)
        td.broadcast(buf, 0)
        M.set_distributed(rank, world, bytes(buf.tolist()))
    nccl_ranks = M.comm_ranks()
    if nccl_ranks != world:
        sys.exit(f"bench.py: NCCL communicator has {nccl_ranks} ranks, expected {world}")
    spec = dict(CONFIGS[a.config])
    if a.dropout is not None:
        spec["dropout"] = a.dropout
    cfg = config_text(**spec)
    budget = TOKEN_BUDGET[a.config]
    vocab = spec["vocab"]

    model = M.Model(cfg)
    g = M.ExpressionGraph(1)
    model.register_params(g)
    g.clear()
    adam = M.Adam(M.adam_defaults_for(cfg))
    avg = M.AveragedParameters(0.9999)
    opts = M.TrainOptions()
    opts.workers = world
    opts.token_budget = budget
    opts.seed = 1
    stepper = M.SyncStepper(model, g, adam, avg, opts)

    prof_steps, e2e_steps = 2, max(3, min(a.steps, 20))
    updates = a.warmup + a.steps + e2e_steps + prof_steps
    per_batch = max(1, budget // 70)
    n_pairs = int(updates * world * per_batch * 1.15) + 64
    ex = M.synth_examples(n_pairs, vocab)
    batches = M.make_batches(ex, budget, 1, True)  # epoch 0 (train.cpp:183-190)
    while len(batches) < updates * world:
        n_pairs = int(n_pairs * 1.3)
        ex = M.synth_examples(n_pairs, vocab)
        batches = M.make_batches(ex, budget, 1, True)

    def group(u):
        return batches[u * world:(u + 1) * world]

    clocks = Clocks(local)
    clocks.start()
    u = 0
    for _ in range(a.warmup):
        stepper.update(group(u), u, True)
        u += 1
    # size the device workspaces for the largest update of the measured
    # region (untimed, parameters restored by replaying nothing: the extra
    # warm-up update is part of warm-up): no allocation inside timed steps
    n_meas = a.steps + e2e_steps
    big = max(range(u, u + n_meas), key=lambda k: sum(b.padded_slots() for b in group(k)))
    # (through the pipelined call, so its pinned loss slots and events exist
    # before the e2e leg: their first-use allocation costs 5-30 ms)
    stepper.update_pipelined(group(big), u)
    stepper.flush_pipelined()

    # ---- value: device-timed, inputs uploaded per step, no host sync inside
    barrier(world)
    M.sync()
    gc.disable()  # no collector pauses inside the timed / e2e loops
    clocks.mark()
    l0 = M.launch_count()
    e0 = M.event_record()
    marks = [e0]
    words = 0.0
    u_timed = u  # the e2e leg replays these batches (same workload mix)
    th0 = time.perf_counter()
    th0_mono = time.monotonic()
    for _ in range(a.steps):
        grp = group(u)
        words += sum(b.target_tokens() for b in grp)
        stepper.update(grp, u, False)
        marks.append(M.event_record())  # per-step device time (diagnostics)
        u += 1
    host_ms = (time.perf_counter() - th0) * 1e3 / a.steps
    if os.environ.get("MTK_TRACE_BLOCK"):
        print(f"[bench] timed region host {th0_mono:.6f} .. {time.monotonic():.6f}",
              file=sys.stderr)
    e1 = marks[-1]
    step_list = [M.event_elapsed_ms_keep(marks[i], marks[i + 1]) for i in range(a.steps)]
    for m in marks[1:-1]:
        M.event_destroy(m)
    ms = M.event_elapsed_ms(e0, e1)
    launches = M.launch_count() - l0
    t_timed_end = time.monotonic()
    ms_max = all_max(ms, world)
    value = words / (ms_max / 1e3)

    # ---- e2e: public training-loop call (SyncStepper.update_pipelined: host
    # batches uploaded every step, every step's loss read back to the host one
    # update later, as a training loop logs it), wall clock
    barrier(world)
    M.sync()
    h0, d0 = M.h2d_bytes(), M.d2h_bytes()
    t0 = time.perf_counter()
    ewords = 0.0
    losses = []
    for k in range(e2e_steps):
        grp = group(u_timed + k % a.steps)  # the timed region's batches, in order
        ewords += sum(b.target_tokens() for b in grp)
        r = stepper.update_pipelined(grp, u)
        if os.environ.get("MTK_E2E_TRACE"):
            print(f"[e2e] step {k} t={time.perf_counter() - t0:.4f}", file=sys.stderr)
        if k > 0:
            losses.append(r.loss)
        u += 1
    losses.append(stepper.flush_pipelined().loss)
    M.sync()
    et = all_max(time.perf_counter() - t0, world)
    h2d = (M.h2d_bytes() - h0) / e2e_steps
    d2h = (M.d2h_bytes() - d0) / e2e_steps
    gc.enable()
    clk = clocks.stop(t_timed_end)

    # ---- per-kernel-class device time (events around each C-ABI call)
    M.sync()
    # The GPU sleeps while the host queues the profiled steps, so the
    # per-class event timings below measure device time, not host gaps.
    M.gpu_sleep(int(max(200.0, 3 * host_ms * prof_steps) * 1e3))
    M.prof_enable(True)
    pe0 = M.event_record()
    prof_batches = []
    for _ in range(prof_steps):
        grp = group(u)
        prof_batches += grp[rank * (len(grp) // world):(rank + 1) * (len(grp) // world)] if world > 1 else grp
        stepper.update(grp, u, True)
        u += 1
    pe1 = M.event_record()
    step_ms = M.event_elapsed_ms(pe0, pe1) / prof_steps
    rep = M.prof_report()
    M.prof_enable(False)
    classes = {}
    for line in rep.strip().splitlines():
        name, n, tms, work = line.split()
        classes[name] = dict(launches=int(n) / prof_steps, ms=float(tms) / prof_steps,
                             work=float(work) / prof_steps)
    # Events around every call break programmatic dependent launch, so the
    # bracketed times carry a per-launch overhead: the classes sum to more
    # than the unperturbed step.  Model it as a constant per launch, o =
    # (sum - step) / launches, and report corrected times (raw kept).
    tot_ms = sum(c["ms"] for c in classes.values())
    tot_l = sum(c["launches"] for c in classes.values())
    over = max(0.0, (tot_ms - ms_max / a.steps) / tot_l) if tot_l else 0.0
    for c in classes.values():
        c["ms_corr"] = max(c["ms"] - over * c["launches"], 0.05 * c["ms"])
    hbm, tflops, src = peaks()
    # SURVEY 8(d) algorithmic FLOPs of the profiled batches over REAL tokens
    flops = {"gemm": 0.0, "attention": 0.0, "total": 0.0}
    for b in prof_batches:
        f = algorithmic_flops(a.config, b.src_mask().sum(axis=1), b.tgt_mask().sum(axis=1))
        for k in flops:
            flops[k] += f[k] / prof_steps
    tensor_classes = {"gemm_tc", "gemm_fp32", "attention", "rnn_scan", "rnn_scan_bwd"}
    # the persistent scans report executed FLOPs over the padded b x T grid:
    # scale them to real tokens (the 8(d) basis) by the batches' fill ratio
    real = sum(float(b.src_mask().sum() + b.tgt_mask().sum()) for b in prof_batches)
    padded = sum(float(b.src_mask().size + b.tgt_mask().size) for b in prof_batches)
    fill = real / padded if padded else 1.0

    scan_flops = sum(v["work"] for k, v in classes.items() if k.startswith("rnn_scan")) * fill

    def class_flops(k):
        if k.startswith("rnn_scan"):
            return classes[k]["work"] * fill
        if k == "attention":
            return flops["attention"]
        if scan_flops:  # RNN: the GEMMs do what the scans (incl. their attention) do not
            return max(flops["total"] - scan_flops, 0.0)
        return flops["gemm"]
    dom = max(classes, key=lambda k: classes[k]["ms_corr"]) if classes else None
    roof = None
    if dom:
        c = classes[dom]
        tensor = dom in tensor_classes or dom.startswith("gemm")
        if tensor:
            alg = class_flops(dom)
        else:
            alg = c["work"]
        per_launch_work = alg / max(c["launches"], 1)
        per_launch_s = c["ms_corr"] / max(c["launches"], 1) / 1e3
        achieved = per_launch_work / per_launch_s / (1e12 if tensor else 1e9)
        peak = tflops if tensor else hbm
        traffic, tsrc = traffic_per_call(a.config, dom, c["launches"])
        roof = {"bound": "tensor" if tensor else "hbm", "kernel": dom,
                "achieved": round(achieved, 2), "peak": peak,
                "unit": "TFLOP/s" if tensor else "GB/s", "frac": round(achieved / peak, 4),
                "frac_tf32_peak": round(achieved / (peak / 2), 4) if tensor else None,
                "traffic": traffic, "traffic_source": tsrc,
                "algorithmic_per_launch": per_launch_work,
                "algorithmic_basis": ("recurrent/attention products executed in the scan "
                                      "(rnn_persist.cu scan_flops) x real/padded token fill "
                                      f"{fill:.3f}" if dom.startswith("rnn_scan") else
                                      "SURVEY 8(d) FLOPs over real (unpadded) tokens of the profiled batches")
                                     if tensor else "algorithmic bytes per call (DESIGN.md 5)",
                "launches_per_step": c["launches"],
                "ms_per_step": round(c["ms_corr"], 3), "ms_per_step_raw": round(c["ms"], 3),
                "peak_source": f"{src} (bf16 dense, sustained); frac_tf32_peak uses half of it",
                "share_of_step": round(c["ms_corr"] / (ms_max / a.steps), 4),
                "note": "GEMMs run tcgen05 kind::tf32 on fp32 storage"}
    breakdown = {}
    for k, v in classes.items():
        tensor = k in tensor_classes or k.startswith("gemm")
        entry = {"ms_per_step": round(v["ms_corr"], 3), "ms_per_step_raw": round(v["ms"], 3),
                 "share": round(v["ms_corr"] / (ms_max / a.steps), 4),
                 "launches_per_step": v["launches"]}
        if tensor and k != "gemm_fp32":
            alg = class_flops(k)
            entry["tflops"] = round(alg / (v["ms_corr"] / 1e3) / 1e12, 2)
            entry["frac_bf16_peak"] = round(alg / (v["ms_corr"] / 1e3) / 1e12 / tflops, 4)
        elif v["work"] > 0:
            entry["gbs"] = round(v["work"] / (v["ms_corr"] / 1e3) / 1e9, 1)
            entry["frac_hbm_peak"] = round(v["work"] / (v["ms_corr"] / 1e3) / 1e9 / hbm, 4)
        breakdown[k] = entry
    # Unperturbed per-class device time: CUPTI kernel records (torch.profiler)
    # of prof_steps plain updates -- no events between kernels, so PDL and
    # the launch overlap stay as in the timed region.
    cupti = None
    try:
        import torch.profiler as tp
        M.sync()
        with tp.profile(activities=[tp.ProfilerActivity.CUDA]) as prof:
            for k in range(prof_steps):  # the timed region's batches again
                stepper.update(group(u_timed + k), u, True)
                u += 1
            M.sync()
        def klass(n):
            for key, cls in (("gemm_tf32_tc", "gemm_tc"), ("splitk_reduce", "gemm_tc"),
                             ("gemm_fp32", "gemm_fp32"), ("attn_", "attention"),
                             ("ln_", "layernorm"), ("colred", "layernorm"), ("xent", "xent"),
                             ("loss_sum", "xent"), ("adam", "adam_ema"), ("finite", "adam_ema"),
                             ("rnn_scan_fwd", "rnn_scan"), ("rnn_scan_bwd", "rnn_scan_bwd"),
                             ("rnn_key_grad", "rnn_scan_bwd"), ("transpose_jobs", "rnn_scan"),
                             ("copy_jobs", "rnn_scan_bwd"), ("embed", "embed"),
                             ("scatter", "embed"), ("gather", "embed"), ("dropout", "dropout"),
                             ("gru_", "gru"), ("bahdanau", "bahdanau"), ("lstm", "lstm")):
                if key in n:
                    return cls
            return "other"
        # With programmatic dependent launch a kernel starts while its
        # predecessor drains and waits in griddepcontrol.wait, so raw kernel
        # durations overlap.  Attribute each instant of the device timeline to
        # the kernel that finishes it: exclusive = end - max(start, previous end).
        kev = []
        for e in prof.events():
            dt = str(getattr(e, "device_type", ""))
            if "CUDA" not in dt:
                continue
            tr = e.time_range
            kev.append((tr.start, tr.end, e.name))
        kev.sort()
        agg = {}
        prev_end = None
        for st_, en_, name in kev:
            excl = en_ - (st_ if prev_end is None else max(st_, prev_end))
            prev_end = en_ if prev_end is None else max(prev_end, en_)
            c = agg.setdefault(klass(name), {"ms": 0.0, "launches": 0})
            c["ms"] += max(excl, 0.0) / 1e3 / prof_steps
            c["launches"] += 1 / prof_steps
        tot = sum(v["ms"] for v in agg.values())
        cupti = {k: {"ms_per_step": round(v["ms"], 3), "launches_per_step": v["launches"],
                     "share_of_kernel_time": round(v["ms"] / tot, 4) if tot else None}
                 for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["ms"])}
        if roof and roof["kernel"] in agg:  # the dominant class from the unperturbed capture
            c = agg[roof["kernel"]]
            per_launch_s = c["ms"] / max(c["launches"], 1) / 1e3
            ach = roof["algorithmic_per_launch"] * roof["launches_per_step"] / max(c["launches"], 1) \
                / per_launch_s / (1e12 if roof["bound"] == "tensor" else 1e9)
            roof["achieved_cupti"] = round(ach, 2)
            roof["frac_cupti"] = round(ach / roof["peak"], 4)
            roof["ms_per_step_cupti"] = round(c["ms"], 3)
    except Exception as e:  # reported, not fatal
        cupti = {"error": str(e)[:200]}

    # whole-job algorithmic FLOPs of the timed updates (all ranks' batches)
    ftimed = 0.0
    for k in range(u_timed, u_timed + a.steps):
        for b in group(k):
            ftimed += algorithmic_flops(a.config, b.src_mask().sum(axis=1),
                                        b.tgt_mask().sum(axis=1))["total"]
    step_flops = {"profiled_rank_step": {k: round(v) for k, v in flops.items()},
                  "timed_job_per_step": round(ftimed / a.steps),
                  "whole_job_tflops": round(ftimed / (ms_max / 1e3) / 1e12, 2),
                  "whole_job_frac_bf16_peak_per_gpu": round(
                      ftimed / (ms_max / 1e3) / 1e12 / world / tflops, 4)}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            v, w, dt, th = cpu_reference(cfg, vocab, steps=2)
            cpu = {"value": round(v, 3), "unit": "target words/sec", "cores": th,
                   "kind": "reference",
                   "sample": f"oracle/_ref trainSync (unmodified reference, -O3), {th} workers x "
                             f"one single-sentence batch per update, 2 timed updates after 1 "
                             f"warm-up update: {int(w)} target words in {dt:.1f}s"}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        out = {
            "metric": METRIC if a.config == "base" else f"target words/sec, {a.config} training step",
            "value": round(value, 1), "unit": "target words/sec", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_max / a.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": a.precision, "data": DATA,
            "config": {"workload": f"{a.config}: {cfg.strip().replace(chr(10), '; ')}; "
                                   f"tokenBudget {budget}/GPU",
                       "global_batch": f"{world} x tokenBudget {budget} (~{words / a.steps:.0f} target words/update)",
                       "seq_len": "16..32 + </s> (padded per batch)", "parallelism": f"dp{world}",
                       "l2": "working set (activations, logits) far exceeds the 126 MB L2"},
            "e2e": {"value": round(ewords / et, 1), "unit": "target words/sec",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "loss_last": losses[-1] if losses else None},
            "gpu_launches": int(launches),
            "host_submit_ms_per_step": round(host_ms, 3),
            "step_ms": {"min": round(min(step_list), 3),
                        "median": round(statistics.median(step_list), 3),
                        "max": round(max(step_list), 3)},
            "roofline": roof,
            "kernel_breakdown": breakdown,
            "kernel_breakdown_cupti": cupti,
            "algorithmic_flops_per_step": step_flops,
            "nccl_ranks": nccl_ranks,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)


def run_reference(a):
    """The reference's own CPU implementation of the path: oracle/_ref, the
    unmodified reference trainSync compiled from its sources, on every host
    core (workers = nproc), plus the SURVEY 8(d) workers = 1 leg.  Never
    imports paper_1804_00344_b200 (its configs/synth modules are loaded as
    plain Python files)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    configs = _pure("configs")
    spec = dict(configs.CONFIGS[a.config])
    if a.dropout is not None:
        spec["dropout"] = a.dropout
    cfg = configs.config_text(**spec)
    threads = os.cpu_count() or 1
    steps = max(1, min(a.steps, 3))
    v, w, dt, th = cpu_reference(cfg, spec["vocab"], threads=threads, steps=steps)
    v1, w1, dt1, _ = cpu_reference(cfg, spec["vocab"], threads=1, steps=steps)
    out = {"metric": METRIC if a.config == "base" else f"target words/sec, {a.config} training step",
           "impl": "reference", "value": round(v, 3), "unit": "target words/sec",
           "n_gpus": a.gpus, "steps": steps, "steps_requested": a.steps, "warmup": 1,
           "ms_per_step": round(dt / steps * 1e3, 1), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "fp32", "data": DATA,
           "config": {"workload": f"{a.config}: {cfg.strip().replace(chr(10), '; ')}",
                      "global_batch": f"{th} workers x 1 sentence per update (bounded sample)",
                      "parallelism": f"{th} CPU threads (trainSync workers)"},
           "cpu_baseline": {"value": round(v, 3), "unit": "target words/sec", "cores": th,
                            "kind": "reference",
                            "sample": f"{th} workers x single-sentence batches, {steps} timed "
                                      f"update(s) after 1 warm-up update: {int(w)} target words "
                                      f"in {dt:.1f}s"},
           "workers_1": {"value": round(v1, 3), "unit": "target words/sec", "cores": 1,
                         "sample": f"1 worker x single-sentence batch, {steps} timed update(s) "
                                   f"after 1 warm-up: {int(w1)} target words in {dt1:.1f}s"},
           "e2e": {"value": round(v, 3), "unit": "target words/sec", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "native_so_mapped": _mapped_so()}
    print(json.dumps(out), flush=True)


def _mapped_so():
    """In-repo shared objects this process has mapped (reference arm: only
    oracle/_ref's copy of the reference may appear)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT + os.sep))


def spawn_ranks(a):
    """`--gpus N` outside torchrun: launch the N ranks (one process per GPU)
    with torch.distributed.run on 127.0.0.1 and relay their output."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and world_env is None:
        sys.exit(spawn_ranks(args))
    else:
        if world_env is not None and int(world_env) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
        run_b200(args)
