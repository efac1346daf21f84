#!/usr/bin/env python3
"""Benchmark of the B200 directional-SLSHT forward engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one complete forward_fast of BASELINE config C (default 2 = configs[1]) on seeded
synthetic inputs: setup tables (Delta, d(beta), window table, I-table, theta weights), every
computed component (Legendre rows, modulated-SHT GEMM, coupling + alpha FFT) and the fused
epilogue that writes every emitted volume (mirrors included) to device memory and digests it.

value  : emitted samples g(rho; l, m) per second, whole job, inputs resident in HBM,
         CUDA events on the engine stream, max over ranks (N > 1: degrees sharded by l).
e2e    : the same through the C ABI with HOST buffers: H2D of f, h and D2H of the per-component
         digests inside the timed region, host wall clock around the synchronous call.
Rank 0 prints ONE JSON line. `--impl reference` times the reference's own CPU forward_fast
(oracle/_ref, unmodified sources) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
P_FP64_TFLOPS = 37.1  # measured DMMA peak on this pool's B200 (profiles/fp64_peak.txt)
CPU_SAMPLE_LMAX = {1: 40, 2: 48, 3: 40, 4: 30, 5: 12}


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
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
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_sample(cfg_index: int, steps: int, warmup: int, threads: int) -> dict:
    """The reference's CPU forward_fast (oracle/_ref) on a bounded sample of the workload:
    forward_fast(f, h, digest-sink, opts.lmax = L_s) with SLSHT threads = host cores."""
    import oracle
    from paper_1207_5558_b200 import configs as C

    R = oracle.Reference()
    f, h, cfg = C.make_inputs(cfg_index)
    ls = CPU_SAMPLE_LMAX[cfg_index]
    times = []
    for i in range(warmup + steps):
        _, secs = R.forward_fast_digest(f, cfg.L_f, cfg.f_real, h, cfg.L_h, cfg.h_real, lmax=ls,
                                        threads=threads)
        if i >= warmup:
            times.append(secs)
    samples = cfg.samples(ls)
    t = statistics.median(times)
    return {
        "value": samples / t,
        "seconds_per_step": t,
        "samples_per_step": samples,
        "sample": (f"config {cfg_index} forward_fast with opts.lmax={ls} "
                   f"({cfg.computed(ls)} computed / {cfg.emitted(ls)} emitted components of "
                   f"{cfg.computed()} / {cfg.emitted()}; per-component cost is independent of l), "
                   f"digest sink under the reference mutex, median of {len(times)}"),
        "cores": threads,
        "cpu": cpu_model(),
    }


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1207_5558_b200 import configs as C

    cfg = C.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    try:
        r = reference_sample(args.config, args.steps, args.warmup, threads)
    except Exception as e:  # the reference library is always built with the repo
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": r["value"],
        "unit": "samples/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["seconds_per_step"] * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE recipe)",
        "config": {"workload": f"config{args.config}", "L_f": cfg.L_f, "L_h": cfg.L_h,
                   "real_mode": cfg.real_mode, "samples_per_step": r["samples_per_step"]},
        "cpu_baseline": {"value": r["value"], "unit": "samples/s", "cores": r["cores"],
                         "kind": "reference", "sample": r["sample"], "cpu": r["cpu"]},
        "e2e": {"value": r["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_1207_5558_b200 as S
    from paper_1207_5558_b200 import configs as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    f_np, h_np, cfg = C.make_inputs(args.config)
    l0, l1 = C.shard_degrees(cfg, world, rank)
    out_bytes = cfg.samples() * 16 / world
    materialize = out_bytes < 40e9
    stream = torch.cuda.Stream(device=dev)
    plan = S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, emit_negative_m=True,
                  device=local, l_begin=l0, l_end=l1, materialize=materialize,
                  ring_bytes=args.ring_mb << 20, stream=stream.cuda_stream)
    # inputs resident in HBM (torch is only the allocator here)
    f_dev = torch.from_numpy(f_np.view(np.float64).copy()).to(dev)
    h_dev = torch.from_numpy(h_np.view(np.float64).copy()).to(dev)
    dig_dev = torch.zeros((S.coeff_count(cfg.L_g), S.DIGEST_WIDTH), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        plan.forward_device(f_dev.data_ptr(), h_dev.data_ptr(), inputs_on_device=True,
                            digests_ptr=dig_dev.data_ptr(), digests_on_device=True,
                            synchronize=False)

    my_samples = plan.emitted_count * plan.volume_elems
    single_chunk = materialize  # one chunk: per-step stage events are live in the graph
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches_per_step = plan.launch_count

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        t_wall = time.perf_counter()
        live_stages = []
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(i & 0xFF)  # L2 flush between steps, outside the event pair
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
            if single_chunk:
                # the step's own coupling-kernel events (recorded around the kernel on the
                # engine stream, inside its CUDA graph); read after the step's event pair
                evs[i][1].synchronize()
                live_stages.append(plan.kernel_time())
        torch.cuda.synchronize(dev)
        t_wall = time.perf_counter() - t_wall
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    total_samples = cfg.samples()
    value = total_samples / (ms_per_step / 1e3)

    # ---- the one collective (N > 1): digest rows of every degree shard gathered on rank 0
    gather = None
    if world > 1:
        from paper_1207_5558_b200.parallel import gather_digests

        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        full = gather_digests(dig_dev, l0, l1, cfg.L_g)
        g1.record()
        torch.cuda.synchronize(dev)
        gather = {"ms": g0.elapsed_time(g1), "rows": int((cfg.L_g + 1) ** 2),
                  "complete": bool(rank != 0 or not torch.isnan(full).any().item())}

    # ---- e2e: C ABI with host buffers (pinned), H2D of f, h and D2H of digests inside
    f_pin = torch.from_numpy(f_np.view(np.float64).copy()).pin_memory()
    h_pin = torch.from_numpy(h_np.view(np.float64).copy()).pin_memory()
    dig_pin = torch.zeros((S.coeff_count(cfg.L_g), S.DIGEST_WIDTH), dtype=torch.float64).pin_memory()
    plan.forward_device(f_pin.data_ptr(), h_pin.data_ptr(), inputs_on_device=False,
                        digests_ptr=dig_pin.data_ptr(), digests_on_device=False, synchronize=True)
    if world > 1:
        dist.barrier()
    e2e_times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        plan.forward_device(f_pin.data_ptr(), h_pin.data_ptr(), inputs_on_device=False,
                            digests_ptr=dig_pin.data_ptr(), digests_on_device=False,
                            synchronize=True)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_times) / len(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    dig_rows = plan.emitted_count
    e2e = {"value": total_samples / e2e_s, "unit": "samples/s",
           "h2d_bytes_per_step": int(f_np.nbytes + h_np.nbytes),
           "d2h_bytes_per_step": int(dig_pin.numel() * 8),
           "digest_rows_per_rank": dig_rows,
           "how": "slsht_cuda_forward_device(host f, h -> host digests), wall clock, mean of steps"}

    # ---- per-stage device times: two profiled steps after the timed ones (events between
    # the kernels on the engine stream); the roofline's kernel time comes from the timed steps
    # themselves when the plan is one chunk
    plan.set_profiling(True)
    prof = []
    for _ in range(2):
        step()
        torch.cuda.synchronize(dev)
        prof.append(plan.stage_times())
    plan.set_profiling(False)
    stage_ms = [statistics.mean(x) for x in zip(*prof)]
    live = [x for x in live_stages if x is not None]
    if single_chunk and len(live) == args.steps:
        kernel_ms = statistics.mean(live)
        stage_src = "CUDA events around the kernel on the engine stream in every timed step (mean)"
    else:
        kernel_ms = stage_ms[3]
        stage_src = "CUDA events on the engine stream, two profiled steps after the timed ones"
    names = ["setup", "legendre", "modgemm", "couple", "digest", "qfft"]
    stages = dict(zip(names, stage_ms))
    two_pass = len(stage_ms) > 5 and stage_ms[5] > 0
    couple_ms = kernel_ms
    peaks = load_peaks()
    alg_bytes = my_samples * 16.0  # one complex128 store per emitted sample
    achieved = alg_bytes / (couple_ms / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / f"traffic_config{args.config}.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
    fp64_view = {
        "canonical_flops_per_sample": cfg.flops_per_sample(),
        "achieved_tflops_canonical": total_samples * cfg.flops_per_sample() / (ms_per_step / 1e3) / 1e12,
        "peak_tflops": P_FP64_TFLOPS,
        "frac": total_samples * cfg.flops_per_sample() / (ms_per_step / 1e3) / 1e12 / P_FP64_TFLOPS,
        "peak_source": "measured DMMA m8n8k4 peak (profiles/fp64_peak.txt)",
    }
    step_roof = min(peaks["hbm_gbs"] * 1e9 / 16.0, P_FP64_TFLOPS * 1e12 / cfg.flops_per_sample())
    if two_pass:
        # two-pass coupling (n = 65, 129): k_tgemm (FP64 DMMA GEMM, T to HBM) and k_qfft (alpha
        # FFT, HBM-bound: T read + volumes written); the dominant one is the roofline kernel
        n, nb = 2 * cfg.L_h + 1, cfg.L_h + 1
        comps = plan.computed_count
        gemm_flops = 8.0 * comps * (cfg.L_h + 1) ** 2 * n * nb  # complex MACs x 8
        tg_ms, qf_ms = stage_ms[3], stage_ms[5]
        qf_bytes = 16.0 * comps * n * n * nb + alg_bytes  # T read + emitted samples written
        tg = {"bound": "tensor", "kernel": "k_tgemm (coupling GEMM on the FP64 tensor cores)",
              "achieved": gemm_flops / (tg_ms / 1e3) / 1e12, "peak": P_FP64_TFLOPS,
              "unit": "TFLOP/s", "frac": gemm_flops / (tg_ms / 1e3) / 1e12 / P_FP64_TFLOPS,
              "traffic": None, "peak_source": "measured DMMA m8n8k4 peak (profiles/fp64_peak.txt)",
              "algorithmic_flops_per_step": gemm_flops, "kernel_ms_per_step": tg_ms}
        qf = {"bound": "hbm", "kernel": "k_qfft (alpha FFT + store/digest epilogue)",
              "achieved": qf_bytes / (qf_ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
              "frac": qf_bytes / (qf_ms / 1e3) / 1e9 / peaks["hbm_gbs"], "traffic": None,
              "peak_source": peaks["source"] + " (MEASURED_PEAKS.json hbm_gbs)",
              "algorithmic_bytes_per_step": qf_bytes, "kernel_ms_per_step": qf_ms}
        main, other = (tg, qf) if tg_ms >= qf_ms else (qf, tg)
        roofline = dict(main)
        roofline.update({
            "kernel_ms_source": "CUDA events on the engine stream, two profiled steps after the timed ones",
            "kernel_share_of_step": main["kernel_ms_per_step"] / sum(stage_ms),
            "second_kernel": other, "fp64_view": fp64_view,
            "step_roofline_samples_per_s": step_roof})
    else:
        roofline = None
    roofline = roofline or {
        "bound": "hbm", "kernel": "k_couple (coupling DMMA + alpha FFT + store/digest epilogue)",
        "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
        "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
        "peak_source": peaks["source"] + " (MEASURED_PEAKS.json hbm_gbs)",
        "algorithmic_bytes_per_step": alg_bytes,
        "kernel_ms_per_step": couple_ms,
        "kernel_ms_source": stage_src,
        "kernel_share_of_step": couple_ms / sum(stage_ms) if sum(stage_ms) > 0 else None,
        "fp64_view": fp64_view,
        "step_roofline_samples_per_s": step_roof,
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            r = reference_sample(args.config, 2, 1, threads)
            cpu = {"value": r["value"], "unit": "samples/s", "cores": r["cores"],
                   "kind": "reference", "sample": r["sample"], "cpu": r["cpu"]}
        except Exception as e:
            cpu = {"value": None, "unit": "samples/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "samples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded BASELINE recipe; Slepian windows solved by the reference)",
            "config": {
                "workload": f"config{args.config}: forward_fast L_f={cfg.L_f} L_h={cfg.L_h} "
                            f"{'real-mode' if cfg.real_mode else 'full-m'} ({cfg.description})",
                "L_f": cfg.L_f, "L_h": cfg.L_h, "real_mode": cfg.real_mode,
                "samples_per_step": total_samples,
                "computed_components": cfg.computed(), "emitted_components": cfg.emitted(),
                "output": ("materialized device distribution" if materialize else
                           "device ring consumed by the fused digest epilogue"),
                "l2": "256 MiB L2 flush between timed steps (outside the event pairs)",
                "parallelism": f"l-shard x{world}",
            },
            "step_ms": {"min": min(step_ms), "max": max(step_ms),
                        "wall_ms_per_step": t_wall * 1e3 / args.steps},
            "stages_ms": stages,
            "e2e": e2e,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gather": gather,
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step,
        }
        print(json.dumps(line))
    plan.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ring-mb", type=int, default=24576)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
