"""Benchmark of the B200 filtering hot path (contract: one JSON line on rank 0).

Metric (BASELINE.json): channel-samples/s for FIR & IIR chains, and the
fraction of the HBM roofline. Headline workload = cfg3, the only BASELINE
config that is a FIR & IIR chain and the one the north star's ">= 70% of HBM
roofline on 1 B200" target is stated for:

    32 ch x 48 kHz x 120 s, butterworth HP4 100 Hz | chebyshev-I LP4 1 dB 8 kHz
    | FIR 101 LP 15 kHz | gain 0.5   (SURVEY.md §8d pins)

A step = one pass of the fused chain over the whole 32-channel batch. Inputs
are synthetic white noise generated in HBM by the device port of the
reference's generator (seed 42). Input + output (737 MB + 737 MB) exceed the
126 MB L2, so no flush is needed between steps.

Multi-GPU (torchrun, one process per GPU): every rank filters its own
32-channel batch (weak scaling, no collective on the data path); the step
time is the max over ranks of the CUDA-event time. The same run also measures
the north star's strong-scaling case, cfg5's fixed 1024 channels split over
the ranks by ``sharding.partition`` (``strong_cfg5`` in the JSON line; at N=1
it is the single-GPU reference point of that curve). ``--config cfgX
--scaling strong`` makes any config the headline in strong-scaling form.

Every line checks the timed output against the CPU oracle: the first and the
last 0.5 s of the first and last channel (for IIR chains the oracle runs the
whole channels, so the tail check covers the cross-tile state carry).

--impl reference: the reference's CPU algorithm (oracle/ port of the numba
kernels, bit-identical to them) on the host cores, on a bounded time slice of
the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(C=2, fs=44100, dur=10.0,
                 workload="stereo 44.1 kHz 10 s through one 4th-order low-pass Butterworth IIR"),
    "cfg2": dict(C=8, fs=48000, dur=60.0, workload="8-channel 48 kHz 60 s through a 101-tap designable FIR low-pass"),
    "cfg3": dict(C=32, fs=48000, dur=120.0,
                 workload="32-channel 48 kHz 120 s chain: high-pass Butterworth | low-pass Chebyshev-I | FIR | gain via the pipe operator (fused)"),
    "cfg4": dict(C=128, fs=48000, dur=600.0, workload="128-channel 48 kHz 10 min through a 4096-tap FIR"),
    "cfg5": dict(C=1024, fs=48000, dur=300.0, workload="1024-channel 48 kHz 5 min 8th-order SOS IIR cascade"),
    # not a BASELINE config: the reference's own pinned interface-comparison chain
    # (pkg/src/wavepipe/bench.py:93-100, 2 Butterworth-4 + 2 Chebyshev-4 = 8 SOS) at
    # cfg3's size, fused into ONE pass
    "bench_chain": dict(C=32, fs=44100, dur=120.0,
                        workload="32-channel 44.1 kHz 120 s: the reference's pinned 8-SOS bench chain (one pass)"),
}


def stages_for(name, wp):
    if name == "cfg1":
        return [wp.design_butterworth("lp", 4, 1000)]
    if name == "cfg2":
        return [wp.design_fir("lp", 101, 1000, "hamming")]
    if name == "cfg3":
        return [wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000),
                wp.design_fir("lp", 101, 15000), wp.Gain(0.5)]
    if name == "cfg4":
        return [wp.design_fir("lp", 4096, 2000, "hamming")]
    if name == "cfg5":
        return [wp.design_butterworth("lp", 8, 2000)]
    if name == "bench_chain":
        return [wp.design_butterworth("lowpass", 4, 1000.0), wp.design_butterworth("lowpass", 4, 1200.0),
                wp.design_chebyshev1("lowpass", 4, 1.0, 2000.0), wp.design_chebyshev1("lowpass", 4, 1.0, 2400.0)]
    raise SystemExit(f"unknown config {name}")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _cpu_sample(name, wp, target_s):
    """A time slice of the workload (all channels, first dur_s seconds) sized
    so one pass of the oracle takes about target_s on all host cores."""
    import numpy as np

    import oracle

    cfg = CONFIGS[name]
    threads = os.cpu_count() or 1
    fs, C = cfg["fs"], cfg["C"]
    stages = wp.Chain(stages_for(name, wp)).bind(fs).stages
    probe_s = 0.25
    x = oracle.white_noise(probe_s, C, fs, 42).astype(np.float32).astype(np.float64)
    oracle.pipe(x, stages, threads)  # loads/builds the oracle library
    t0 = time.perf_counter()
    oracle.pipe(x, stages, threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    dur_s = min(cfg["dur"], max(probe_s, probe_s * target_s / dt))
    x = oracle.white_noise(dur_s, C, fs, 42).astype(np.float32).astype(np.float64)
    return x, stages, dur_s, threads


def _cpu_describe(name, x, dur_s, threads, times):
    cfg = CONFIGS[name]
    return (f"{cfg['C']} ch x {x.shape[1]} frames ({dur_s:.2f} s of the {cfg['dur']:.0f} s workload), "
            f"{len(times)} timed reps, mean {statistics.mean(times):.3f} s; oracle/wp_oracle.c port of the "
            f"reference numba kernels (float64, bit-identical), {threads} threads over channels")


def parity_check(name, wp, x_dev, y_dev, fs):
    """Head and tail of the first and last channel of the timed output vs the
    oracle port (the only oracle use on this arm; after the timed region)."""
    import numpy as np

    import oracle

    stages = wp.Chain(stages_for(name, wp)).bind(fs).stages
    C, N = x_dev.shape
    n = min(N, fs // 2)
    chans = sorted({0, C - 1})
    fir_only = all(hasattr(st, "taps") for st in stages if not hasattr(st, "factor"))
    taps = sum(len(st.taps) - 1 for st in stages if hasattr(st, "taps"))
    out = {}
    for c in chans:
        if fir_only:
            # causal FIR: the tail depends only on the last n + T - 1 samples
            lo = max(0, N - n - taps)
            xs = x_dev[c:c + 1, lo:].double().cpu().numpy()
            ref_tail = oracle.pipe(xs, stages)[:, -n:]
            ref_head = oracle.pipe(x_dev[c:c + 1, :n].double().cpu().numpy(), stages)
        else:
            ref = oracle.pipe(x_dev[c:c + 1].double().cpu().numpy(), stages, oracle.default_threads())
            ref_head, ref_tail = ref[:, :n], ref[:, -n:]
        y = y_dev[c:c + 1]
        out[f"ch{c}_head"] = oracle.parity_error(y[:, :n].double().cpu().numpy(), ref_head)
        out[f"ch{c}_tail"] = oracle.parity_error(y[:, -n:].double().cpu().numpy(), ref_tail)
    worst = max(out.values())
    return {"max_abs_err_over_peak": worst, "bar": 1e-5 if fir_only else 1e-4, "windows": out,
            "sample": f"first and last {n} frames of channels {chans} of the timed output vs the oracle port "
                      f"({'windowed FIR' if fir_only else 'whole channels'})"}


def cpu_baseline(name, wp, budget_s=8.0):
    """Reference CPU algorithm on the box's host cores (bench._run_cell
    protocol: 1 untimed warm-up, perf_counter around the apply only)."""
    import oracle

    x, stages, dur_s, threads = _cpu_sample(name, wp, target_s=1.0)
    oracle.pipe(x, stages, threads)  # untimed warm-up
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        oracle.pipe(x, stages, threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s or len(times) >= 50:
            break
    units = x.shape[0] * x.shape[1]
    return {"value": units / statistics.mean(times), "unit": "ch-samples/s", "cores": threads, "kind": "port",
            "sample": _cpu_describe(name, x, dur_s, threads, times)}


def run_reference(args, rank):
    """--impl reference: rank 0 times the reference algorithm on host cores."""
    if rank != 0:
        return 0
    import oracle
    import paper_2504_08624_b200 as wp

    name = args.config
    cfg = CONFIGS[name]
    x, stages, dur_s, threads = _cpu_sample(name, wp, target_s=0.5)
    for _ in range(args.warmup):
        oracle.pipe(x, stages, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.pipe(x, stages, threads)
        times.append(time.perf_counter() - t0)
    units = x.shape[0] * x.shape[1]
    value = units / statistics.mean(times)
    line = {
        "impl": "reference",
        "metric": "channel-samples/s for FIR & IIR chains at 1/8 B200; % of HBM roofline",
        "value": value, "unit": "ch-samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic white noise (reference generator, seed 42), fp32-rounded then widened",
        "config": {"workload": cfg["workload"], "config_id": name, "channels": cfg["C"], "fs": cfg["fs"],
                   "duration_s": cfg["dur"], "parallelism": f"{threads} host threads over channels"},
        "cpu_baseline": {"value": value, "unit": "ch-samples/s", "cores": threads, "kind": "port",
                         "sample": _cpu_describe(name, x, dur_s, threads, times)},
        "e2e": {"value": value, "unit": "ch-samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: every rank filters the whole config; strong: the config's channels are split")
    ap.add_argument("--no-strong-cfg5", action="store_true", help="skip the cfg5 strong-scaling side measurement")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed output")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank)

    import torch

    import paper_2504_08624_b200 as wp
    from paper_2504_08624_b200 import _native, engine

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    name = args.config
    cfg = CONFIGS[name]
    C_cfg, fs = cfg["C"], cfg["fs"]
    N = int(round(cfg["dur"] * fs))
    stages = wp.Chain(stages_for(name, wp)).bind(fs).stages
    dev = torch.device("cuda", local_rank)
    from paper_2504_08624_b200.sharding import partition

    if args.scaling == "strong":
        c0, c1 = partition(C_cfg, world)[rank]
        C = c1 - c0
    else:
        C = C_cfg

    def max_over_ranks(vals):
        if not dist:
            return vals
        t = torch.tensor(vals, device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def timed(plan, x, y, Cr, Nr, steps, warmup, clk_gpu=None):
        """CUDA-event time of `steps` plan executions after `warmup` (barrier +
        synchronize on both sides); returns (ms_per_step, per_launch_ms, launches, clocks)."""
        stream = torch.cuda.current_stream(dev)
        nbytes = plan.workspace_bytes(max(Cr, 1), Nr)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)

        def step():
            if Cr > 0:
                plan.execute(x.data_ptr(), y.data_ptr(), Cr, Nr, Nr, Nr, ws.data_ptr(), nbytes, stream.cuda_stream)

        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local_rank) if clk_gpu else None
        if sampler:
            sampler.__enter__()
        try:
            # keep the GPU busy ~0.5 s before warm-up so the clock samples (every
            # 100 ms) see the part under this load, then W warm-up steps, then K
            settle = time.perf_counter()
            while time.perf_counter() - settle < 0.5:
                step()
                torch.cuda.synchronize()
            for _ in range(warmup):
                step()
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            launches0 = _native.launch_count()
            t_start.record(stream)
            for i in range(steps):
                step()
            t_end.record(stream)
            torch.cuda.synchronize()
            launches = _native.launch_count() - launches0
            # per-step events in a second, separate run (SURVEY §8(d) min / median): an
            # event between two passes stops the next kernel's prologue from overlapping
            # the previous one's tail (programmatic dependent launch), so the headline
            # above times the K passes back to back
            for i in range(steps):
                ev[i][0].record(stream)
                step()
                ev[i][1].record(stream)
            torch.cuda.synchronize()
        finally:
            if sampler:
                sampler.__exit__(None, None, None)
        elapsed_ms = t_start.elapsed_time(t_end)
        lt = [a.elapsed_time(b) for a, b in ev]
        per_launch_ms = statistics.mean(lt)
        timed.launch_min_median = (min(lt), statistics.median(lt))  # report min and median
        elapsed_ms, per_launch_ms = max_over_ranks([elapsed_ms, per_launch_ms])
        if dist:
            dist.barrier()
        return elapsed_ms / steps, per_launch_ms, launches, (sampler.summary() if sampler else None)

    # ---- headline: inputs resident in HBM (device noise, distinct seed per rank) ----
    w = wp.white_noise(cfg["dur"], max(C, 1), fs, seed=42 + rank, device=dev)
    x = w.tensor()[:C]
    y = torch.empty_like(x)
    plan = engine.plan_for(stages, device=local_rank)
    ms_per_step, per_launch_ms, launches, clocks = timed(plan, x, y, C, N, args.steps, args.warmup, clk_gpu=True)
    launch_min, launch_median = timed.launch_min_median
    units = C * N
    total_units = units * world if args.scaling == "weak" else C_cfg * N
    value = total_units / (ms_per_step / 1e3)

    # the timed output against the oracle (rank 0, after the timed region)
    with_baseline = not args.no_cpu_baseline and rank == 0 and world == 1
    parity = parity_check(name, wp, x, y, fs) if rank == 0 and C > 0 and not args.no_parity else None
    host_in = torch.empty((C, N), dtype=torch.float32, pin_memory=True)
    host_in.copy_(x)
    # free the device-resident bench buffers before the other legs (cfg5 is
    # 59 GB per buffer: in + out + e2e in + e2e out would not fit)
    del x, y, w
    torch.cuda.empty_cache()

    # ---- north-star strong scaling: cfg5's 1024 channels split over the ranks ----
    strong = None
    if not args.no_strong_cfg5 and not (name == "cfg5" and args.scaling == "strong"):
        c5 = CONFIGS["cfg5"]
        N5 = int(round(c5["dur"] * c5["fs"]))
        a0, a1 = partition(c5["C"], world)[rank]
        C5 = a1 - a0
        w5 = wp.white_noise(c5["dur"], max(C5, 1), c5["fs"], seed=1042 + rank, device=dev)
        x5 = w5.tensor()[:C5]
        y5 = torch.empty_like(x5)
        plan5 = engine.plan_for(wp.Chain(stages_for("cfg5", wp)).bind(c5["fs"]).stages, device=local_rank)
        ms5, pl5, _, _ = timed(plan5, x5, y5, C5, N5, min(args.steps, 10), 3)
        strong = {"workload": c5["workload"], "config_id": "cfg5", "scaling": "strong", "n_gpus": world,
                  "channels_total": c5["C"], "channels_per_gpu_max": max(b - a for a, b in partition(c5["C"], world)),
                  "frames": N5, "ms_per_step": ms5, "value": c5["C"] * N5 / (ms5 / 1e3), "unit": "ch-samples/s",
                  "per_gpu_hbm_frac": 8.0 * max(b - a for a, b in partition(c5["C"], world)) * N5 / (pl5 / 1e3) / 1e9
                  / load_peaks()[0],
                  "partition": "sharding.partition (contiguous, pair-aligned channel blocks), no collectives",
                  "passes": plan5.describe_for(max(C5, 1), N5)}
        del x5, y5, w5
        torch.cuda.empty_cache()

    # ---- end to end through the public API: pinned host in -> host out ----
    host_out = torch.empty((C, N), dtype=torch.float32, pin_memory=True)
    chain = wp.Chain(stages_for(name, wp))

    def e2e_step():
        if C > 0:
            src = wp.Wave.from_tensor(host_in, fs)
            (src | chain).numpy32(out=host_out)

    e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e2e_times = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks([statistics.mean(e2e_times)])[0]

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    hbm_peak, bf16_peak, peak_kind = load_peaks()
    algo_bytes = 8.0 * units  # fp32 read once + write once per channel-sample
    passes = plan.describe_for(max(C, 1), N)
    kernel_names = {"chain_lb": "wpk::chain_lb_kernel", "fir_tc": "wpk::fir_tc_kernel",
                    "fft_ols": "wpk::fft_ols_kernel", "fused": "wpk::fused_chain_kernel"}
    kernels = [kernel_names.get(d.split("[")[0], d.split("[")[0]) for d in passes]
    # the K passes of the timed region back to back (events only at its ends): the
    # mean pass time there is the launch duration that counts for throughput;
    # isolated passes (an event on each side) are reported beside it
    achieved = algo_bytes / (ms_per_step / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            ent = json.load(open(prof)).get(name, {})
            # a profile taken on a slice of this config scales per channel-sample
            traffic = ent["dram_bytes_per_unit"] * units if "dram_bytes_per_unit" in ent else ent.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    io_mb = units * 4 / 1e6
    line = {
        "metric": "channel-samples/s for FIR & IIR chains at 1/8 B200; % of HBM roofline",
        "value": value,
        "unit": "ch-samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f32 I/O and f32 scan/state (balanced state basis); tensor-core f16x3 split products",
        "data": "synthetic white noise generated on device (reference generator, seed 42+rank)",
        "config": {"workload": cfg["workload"], "config_id": name, "channels_per_gpu": C, "frames": N, "fs": fs,
                   "l2": f"inputs larger than L2 ({io_mb:.0f} MB in + {io_mb:.0f} MB out per step), no flush"
                   if io_mb > 126 else f"{io_mb:.0f} MB in + out per step: partly L2-resident between steps",
                   "passes": passes,
                   "parallelism": f"channel batches x{world} ({args.scaling} scaling), no collectives"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": algo_bytes, "launch_ms": ms_per_step,
                     "isolated_step_ms": {"mean": per_launch_ms, "min": launch_min, "median": launch_median},
                     "kernel": " + ".join(kernels) + f" ({plan.launches_for(max(C, 1), N)} launch(es) per step)"},
        "e2e": {"value": total_units / e2e_s, "unit": "ch-samples/s", "h2d_bytes_per_step": units * 4,
                "d2h_bytes_per_step": units * 4, "seconds_per_step": e2e_s,
                "path": "Wave.from_tensor(pinned) | Chain -> numpy32(out=pinned) = C-ABI wp_plan_execute_host on host buffers"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if strong is not None:
        line["strong_cfg5"] = strong
    if parity is not None:
        line["parity_check"] = parity
    taps = sum(len(getattr(st, "taps", ())) for st in stages)
    if any(("chain_lb" in k or "fir_tc" in k) for k in kernels) and taps:
        # algorithmic FIR flops = 2 T per channel-sample, against
        # the dense fp16 tensor peak; the fp16 x3 split runs 3x those MMAs
        tflops = 2.0 * taps * units / (ms_per_step / 1e3) / 1e12
        line["roofline"]["tensor"] = {"achieved_tflops": tflops, "peak_tflops": bf16_peak,
                                      "frac": tflops / bf16_peak, "split_overhead": 3,
                                      "note": "algorithmic 2*T flops/ch-sample; executed MMA work is 3x (fp16 hi/lo split)"}
    if with_baseline:
        line["cpu_baseline"] = cpu_baseline(name, wp)
        line["cpu_baseline"]["parity_check"] = parity  # the same check, kept here for round-1 readers
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
