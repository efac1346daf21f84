#!/usr/bin/env python3
"""Benchmark of the B200 directional-SLSHT forward engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one complete forward_fast of BASELINE config C (default 4 = configs[3], the largest
configuration that runs on one GPU; config 5 is the 8-GPU scaling config) on seeded synthetic
inputs: setup tables (Delta, d(beta), window table, I-table, theta weights), every computed
component (Legendre rows, modulated-SHT GEMM, coupling + alpha FFT) and the fused epilogue that
writes every emitted volume (mirrors included) to device memory and digests it.

value  : emitted samples g(rho; l, m) per second, whole job, inputs resident in HBM, CUDA events
         on the engine stream, max over ranks (N > 1: degrees sharded by l).
e2e    : the same through the C ABI with HOST buffers: H2D of f, h and D2H of the per-component
         digests inside the timed region, host wall clock around the synchronous call.
Rank 0 prints ONE JSON line. With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py
launches its N ranks itself (torch.distributed.run, 127.0.0.1). `--impl reference` times the
reference's own CPU forward_fast (oracle/_ref, the unmodified sources) on the host cores, with
the SURVEY.md §8(d) recipe (full runs for configs 1-2, setup-separated extrapolation of a sampled
run for configs 3-5).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
# builder-measured DMMA m8n8k4 peak on this pool's B200 (profiles/fp64_peak.txt); not in
# MEASURED_PEAKS.json, which has no FP64 entry
P_FP64_TFLOPS = 37.1
FP64_SOURCE = "builder-measured DMMA m8n8k4 burst peak (profiles/fp64_peak.txt)"
# sampled lmax of the CPU reference for configs 3-5 (configs 1-2 run in full), SURVEY.md §8(d)
CPU_SAMPLE_LMAX = {3: 32, 4: 32, 5: 12}
L2_NOTE = "256 MiB L2 flush between timed GPU steps (outside the event pairs)"


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


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
            time.sleep(0.2)  # the first sample lands inside the timed region
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


def workload_config(cfg, world: int) -> dict:
    """The `config` object, identical in both arms (the driver compares them)."""
    return {
        "workload": (f"config{cfg.index}: forward_fast L_f={cfg.L_f} L_h={cfg.L_h} "
                     f"{'real-mode' if cfg.real_mode else 'full-m'} ({cfg.description})"),
        "L_f": cfg.L_f, "L_h": cfg.L_h, "real_mode": cfg.real_mode,
        "samples_per_step": cfg.samples(),
        "computed_components": cfg.computed(), "emitted_components": cfg.emitted(),
        "l2": L2_NOTE,
        "parallelism": f"l-shard x{world}",
    }


# ------------------------------------------------------------------------ reference (CPU) arm
class ReferenceTimer:
    """The reference's CPU forward_fast (oracle/_ref, unmodified sources, -O3) with a digest
    sink under its own mutex, on `threads` host threads:
      configs 1-2: the full call per step;
      configs 3-5: forward_fast with opts.lmax = L_s per step, extrapolated as
        T = T_setup + (T_run - T_setup) * N_full / N_sample,
      T_setup = ModulatedSht + DeltaTables + So3Evaluator (transform.cpp:256-258, serial),
      median of 3, timed once; per-component cost is independent of l."""

    def __init__(self, cfg_index: int, threads: int):
        import oracle
        from paper_1207_5558_b200 import configs as C

        self.R = oracle.Reference()
        self.f, self.h, self.cfg = C.make_inputs(cfg_index)
        self.threads = threads
        self.ls = CPU_SAMPLE_LMAX.get(cfg_index)  # None: full runs
        self.t_setup = None
        if self.ls is not None:
            cfg = self.cfg
            self.t_setup = statistics.median(
                self.R.setup_seconds(self.f, cfg.L_f, cfg.f_real, self.h, cfg.L_h, cfg.h_real)
                for _ in range(3))

    def run(self) -> tuple[float, float]:
        """One step: (measured seconds, seconds of the full forward_fast (extrapolated))."""
        cfg = self.cfg
        _, secs = self.R.forward_fast_digest(self.f, cfg.L_f, cfg.f_real, self.h, cfg.L_h,
                                             cfg.h_real, lmax=-1 if self.ls is None else self.ls,
                                             threads=self.threads)
        if self.ls is None:
            return secs, secs
        scale = cfg.computed() / cfg.computed(self.ls)
        return secs, self.t_setup + max(secs - self.t_setup, 0.0) * scale

    def sample_text(self, steps: int) -> str:
        cfg = self.cfg
        if self.ls is None:
            return (f"config {cfg.index} full forward_fast ({cfg.computed()} computed / "
                    f"{cfg.emitted()} emitted components), digest sink under the reference "
                    f"mutex, median of {steps}")
        return (f"config {cfg.index} forward_fast with opts.lmax={self.ls} ({cfg.computed(self.ls)}"
                f" of {cfg.computed()} computed components), digest sink; extrapolated "
                f"T = T_setup + (T_run - T_setup) * {cfg.computed()}/{cfg.computed(self.ls)} with "
                f"T_setup = {self.t_setup:.3f} s (ModulatedSht + DeltaTables + So3Evaluator, "
                f"serial, median of 3); median of {steps} steps")


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the CPU reference runs once, on rank 0
    from paper_1207_5558_b200 import configs as C

    cfg = C.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    threads = os.cpu_count() or 1
    try:
        rt = ReferenceTimer(args.config, threads)
        for _ in range(args.warmup):
            rt.run()
        meas, full = [], []
        for _ in range(args.steps):
            a, b = rt.run()
            meas.append(a)
            full.append(b)
    except Exception as e:  # the reference library is always built with the repo
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    t_full = statistics.median(full)
    value = cfg.samples() / t_full
    kind = "reference"
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "samples/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": statistics.mean(meas) * 1e3,
        "ms_per_full_run": t_full * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE recipe; Slepian windows solved by the reference)",
        "config": workload_config(cfg, world),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": kind,
                         "sample": rt.sample_text(args.steps), "cpu": cpu_model(),
                         "extrapolated": rt.ls is not None},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------ our arm
def spawn_ranks(args) -> int:
    """--gpus N without an external launcher: run N ranks through torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def roundtrip_error(dig: np.ndarray, f: np.ndarray, h: np.ndarray, cfg) -> float:
    """max|f_rec - f| / max|f| with f_rec(l, m) = integrate_volume(g(l, m)) / (sqrt(16 pi^3) h00)
    for l <= L_f (inverse_slsht / InverseAccumulator, transform.cpp:469-540), from the digest
    epilogue's quadrature integrals (fields 6, 7) of every emitted component."""
    rows = (cfg.L_f + 1) ** 2
    rec = (dig[:rows, 6] + 1j * dig[:rows, 7]) / (math.sqrt(16.0 * math.pi ** 3) * h[0])
    return float(np.max(np.abs(rec - f)) / np.max(np.abs(f)))


def host_sink_sample(S, C, cfg, f_np, h_np, dev: int, budget_bytes: float = 2.5e9) -> dict:
    """Host-sink throughput: slsht_cuda_forward (pinned, double-buffered D2H) into the library's
    copy sink (the materializing forward_fast's copy into host memory) over a degree range of
    about `budget_bytes` of output (the full config does not fit in host memory)."""
    vol_bytes = cfg.volume * 16
    target = max(1, int(budget_bytes // vol_bytes))
    l1 = cfg.L_g + 1
    l0 = l1
    while l0 > 0 and l1 * l1 - l0 * l0 < target:
        l0 -= 1
    rows = l1 * l1 - l0 * l0
    out = np.empty((rows,) + S.volume_shape(cfg.L_h), np.complex128)
    out.reshape(-1)[:: max(1, out.size // 1024)] = 0  # touch a little; pages fault in the copy
    with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, emit_negative_m=True, device=dev,
                l_begin=l0, l_end=l1, ring_bytes=1 << 30) as plan:
        plan.forward_copy(f_np, h_np, out, first_index=l0 * l0)  # warm-up (faults the pages in)
        t0 = time.perf_counter()
        delivered, dropped = plan.forward_copy(f_np, h_np, out, first_index=l0 * l0)
        secs = time.perf_counter() - t0
    samples = delivered * cfg.volume
    threads = int(os.environ.get("SLSHT_CUDA_HOST_THREADS", "0")) or min(16, os.cpu_count() or 1)
    return {"value": samples / secs, "unit": "samples/s", "gb_per_s": samples * 16 / secs / 1e9,
            "degrees": [l0, l1], "components": delivered, "dropped": dropped,
            "host_copy_threads": threads,
            "how": ("slsht_cuda_forward + slsht_cuda_copy_sink into host memory (the "
                    "materializing forward_fast's copy: disjoint rows, copied out of the pinned "
                    "staging buffers by several host threads), degrees [l0, l1) of the config, "
                    "wall clock, second call")}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_1207_5558_b200 as S
    from paper_1207_5558_b200 import configs as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} does not match --gpus {args.gpus}")
    # one rank per GPU over NCCL; BENCH_DIST_BACKEND=gloo (host tensors) lets a one-GPU box run
    # the multi-rank logic with every rank on that GPU (a plumbing check, not a measurement)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    dev_index = local % max(1, torch.cuda.device_count())
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # collective tensors

    def reduce_max(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    f_np, h_np, cfg = C.make_inputs(args.config)
    l0, l1 = C.shard_degrees(cfg, world, rank)
    out_bytes = cfg.samples() * 16 / world
    materialize = out_bytes < 40e9
    stream = torch.cuda.Stream(device=dev)
    plan = S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, emit_negative_m=True,
                  device=dev_index, l_begin=l0, l_end=l1, materialize=materialize,
                  ring_bytes=args.ring_mb << 20, stream=stream.cuda_stream)
    # inputs resident in HBM (torch is only the allocator here)
    f_dev = torch.from_numpy(f_np.view(np.float64).copy()).to(dev)
    h_dev = torch.from_numpy(h_np.view(np.float64).copy()).to(dev)
    dig_dev = torch.full((S.coeff_count(cfg.L_g), S.DIGEST_WIDTH), float("nan"),
                         dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        plan.forward_device(f_dev.data_ptr(), h_dev.data_ptr(), inputs_on_device=True,
                            digests_ptr=dig_dev.data_ptr(), digests_on_device=True,
                            synchronize=False)

    my_samples = plan.emitted_count * plan.volume_elems
    single_chunk = materialize  # one chunk: per-step kernel events are live in the graph
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches_per_step = plan.launch_count

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev_index) as clocks:
        t_wall = time.perf_counter()
        live = []
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
                live.append(plan.kernel_time())
        torch.cuda.synchronize(dev)
        t_wall = time.perf_counter() - t_wall
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    launches = launches_per_step * args.steps
    if world > 1:
        total_ms = reduce_max(total_ms)
        n = torch.tensor([launches], dtype=torch.int64, device=cdev)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
        launches = int(n.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    total_samples = cfg.samples()
    value = total_samples / (ms_per_step / 1e3)

    # ---- the one collective (N > 1): digest rows of every degree shard gathered on rank 0
    gather = None
    full_dig = dig_dev
    if world > 1:
        from paper_1207_5558_b200.parallel import gather_digests

        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        full_dig = gather_digests(dig_dev if backend == "nccl" else dig_dev.cpu(), l0, l1, cfg.L_g)
        g1.record()
        torch.cuda.synchronize(dev)
        gather = {"ms": g0.elapsed_time(g1), "rows": int((cfg.L_g + 1) ** 2),
                  "backend": f"{backend} all_gather of padded row blocks"}
    rt_err = None
    complete = None
    if rank == 0:
        d = full_dig.cpu().numpy()
        complete = bool(not np.isnan(d).any())
        rt_err = roundtrip_error(d, f_np, h_np, cfg)

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
        e2e_s = reduce_max(e2e_s)
    r0, r1 = l0 * l0, l1 * l1
    e2e = {"value": total_samples / e2e_s, "unit": "samples/s",
           "h2d_bytes_per_step": int(f_np.nbytes + h_np.nbytes),
           "d2h_bytes_per_step": int((r1 - r0) * S.DIGEST_WIDTH * 8),
           "how": ("slsht_cuda_forward_device(host f, h -> host digests of the rank's degree "
                   "shard), wall clock, mean of steps, max over ranks")}

    # ---- per-stage device times: two profiled steps after the timed ones (events between the
    # kernels on the engine stream); the roofline's kernel time comes from the timed steps
    # themselves when the plan is one chunk
    plan.set_profiling(True)
    prof = []
    for _ in range(2):
        step()
        torch.cuda.synchronize(dev)
        prof.append(plan.stage_times())
    plan.set_profiling(False)
    stage_ms = [statistics.mean(x) for x in zip(*prof)]
    names = ["setup", "legendre", "modgemm", "couple", "digest", "qfft"]
    stages = dict(zip(names, stage_ms))
    two_pass = len(stage_ms) > 5 and stage_ms[5] > 0
    live = [x for x in live if x is not None]
    peaks = load_peaks()
    alg_bytes = my_samples * 16.0  # one complex128 store per emitted sample
    fp64 = total_samples * cfg.flops_per_sample() / (ms_per_step / 1e3) / 1e12
    fp64_view = {"canonical_flops_per_sample": cfg.flops_per_sample(),
                 "achieved_tflops_canonical": fp64, "peak_tflops": P_FP64_TFLOPS,
                 "frac": fp64 / P_FP64_TFLOPS, "peak_source": FP64_SOURCE}
    step_roof = min(peaks["hbm_gbs"] * 1e9 / 16.0, P_FP64_TFLOPS * 1e12 / cfg.flops_per_sample())
    # measured DRAM traffic of the roofline kernels (committed ncu captures): per launch for a
    # single-chunk plan, per step (summed over the step's chunks) for the two-pass path
    traffic, tdoc = None, {}
    tfile = ROOT / "profiles" / f"traffic_config{args.config}.json"
    if tfile.exists() and world == 1:  # the captures are of the one-GPU plan
        tdoc = json.loads(tfile.read_text())
        traffic = tdoc.get("dram_bytes_per_launch")
    if two_pass:
        # two-pass coupling (n = 49, 65, 129): k_tgemm (FP64 DMMA GEMM, T to HBM) and k_qfft
        # (alpha FFT + epilogue); the roofline kernel is the longer of the two. Algorithmic
        # bytes of k_qfft are the emitted samples only (16 B each, §8(d)); the T re-read is
        # overhead of this design and is shown separately.
        n, nb = 2 * cfg.L_h + 1, cfg.L_h + 1
        comps = plan.computed_count
        gemm_flops = 8.0 * comps * (cfg.L_h + 1) ** 2 * n * nb  # complex MACs x 8 (canonical)
        tg_ms, qf_ms = stage_ms[3], stage_ms[5]
        # T rows k_qfft recomputes instead of reading (SLSHT_CUDA_TP_KC, default 2 at n = 49, 65)
        kc = int(os.environ.get("SLSHT_CUDA_TP_KC", "2" if n in (49, 65) else "0"))
        kc = kc if n in (49, 65) else 0
        t_bytes = 16.0 * comps * (n - 2 * kc) * n * nb
        tg = {"bound": "tensor", "kernel": "k_tgemm (coupling GEMM on the FP64 tensor cores)",
              "achieved": gemm_flops / (tg_ms / 1e3) / 1e12, "peak": P_FP64_TFLOPS,
              "unit": "TFLOP/s", "frac": gemm_flops / (tg_ms / 1e3) / 1e12 / P_FP64_TFLOPS,
              "traffic": tdoc.get("k_tgemm", {}).get("dram_bytes_per_step"),
              "traffic_unit": "DRAM bytes per step (ncu, all launches of one step)",
              "peak_source": FP64_SOURCE,
              "flop_model": "8 FLOP per complex MAC (the DMMA Gauss product issues 6)",
              "algorithmic_flops_per_step": gemm_flops, "kernel_ms_per_step": tg_ms}
        qf = {"bound": "hbm", "kernel": "k_qfft (alpha FFT + store/digest epilogue)",
              "achieved": alg_bytes / (qf_ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"],
              "unit": "GB/s", "frac": alg_bytes / (qf_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
              "traffic": tdoc.get("k_qfft", {}).get("dram_bytes_per_step"),
              "traffic_unit": "DRAM bytes per step (ncu, all launches of one step)",
              "peak_source": peaks["source"],
              "algorithmic_bytes_per_step": alg_bytes, "kernel_ms_per_step": qf_ms,
              "t_reread_bytes_per_step": t_bytes,
              "moved_gbs_incl_t_reread": (alg_bytes + t_bytes) / (qf_ms / 1e3) / 1e9}
        main, other = (tg, qf) if tg_ms >= qf_ms else (qf, tg)
        roofline = dict(main)
        roofline.update({
            "kernel_ms_source": "CUDA events on the engine stream, two profiled steps after the timed ones",
            "kernel_share_of_step": main["kernel_ms_per_step"] / sum(stage_ms),
            "second_kernel": other, "fp64_view": fp64_view,
            "step_roofline_samples_per_s": step_roof,
            "step_frac_of_roofline": value / step_roof})
    else:
        if single_chunk and len(live) == args.steps:
            couple_ms = statistics.mean(live)
            src = "CUDA events around the kernel on the engine stream in every timed step (mean)"
        else:
            couple_ms = stage_ms[3]
            src = "CUDA events on the engine stream, two profiled steps after the timed ones"
        achieved = alg_bytes / (couple_ms / 1e3) / 1e9
        roofline = {
            "bound": "hbm",
            "kernel": {17: "k_couple_reg (coupling on FP64 FMAs + radix-17 alpha DFT + store/digest epilogue, in registers)",
                       33: "k_couple_lines (coupling DMMA + alpha FFT + line-aligned store/digest epilogue)"}.get(
                2 * cfg.L_h + 1, "k_couple (coupling DMMA + alpha FFT + store/digest epilogue)"),
            "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
            "peak_source": peaks["source"], "algorithmic_bytes_per_step": alg_bytes,
            "kernel_ms_per_step": couple_ms, "kernel_ms_source": src,
            "kernel_share_of_step": couple_ms / sum(stage_ms) if sum(stage_ms) > 0 else None,
            "fp64_view": fp64_view, "step_roofline_samples_per_s": step_roof,
            "step_frac_of_roofline": value / step_roof,
        }
    steady_ms = max(ms_per_step - stages["setup"], 1e-9)
    steady = {"value": total_samples / (steady_ms / 1e3), "unit": "samples/s",
              "how": ("setup excluded: ms_per_step minus the setup stage on the engine stream "
                      "(k_setup_main; the Delta -> W chain runs beside it on the auxiliary "
                      "stream), profiled steps")}

    host_sink = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            host_sink = host_sink_sample(S, C, cfg, f_np, h_np, dev_index)
        except Exception as e:
            host_sink = {"value": None, "error": f"{type(e).__name__}: {e}"}
        try:
            threads = os.cpu_count() or 1
            rt = ReferenceTimer(args.config, threads)
            meas, full = rt.run()
            cpu = {"value": cfg.samples() / full, "unit": "samples/s", "cores": threads,
                   "kind": "reference", "sample": rt.sample_text(1), "cpu": cpu_model(),
                   "extrapolated": rt.ls is not None, "measured_s": meas,
                   "full_run_s": full}
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
            "config": workload_config(cfg, world),
            "output": ("materialized device distribution" if materialize else
                       "device ring consumed by the fused digest epilogue"),
            "step_ms": {"min": min(step_ms), "max": max(step_ms),
                        "wall_ms_per_step": t_wall * 1e3 / args.steps},
            "stages_ms": stages,
            "e2e": e2e,
            "steady_state": steady,
            "host_sink": host_sink,
            "roundtrip_err": rt_err,
            "digests_complete": complete,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gather": gather,
            "gpu_launches": launches,
            "gpu_launches_per_step_per_rank": launches_per_step,
        }
        print(json.dumps(line))
    plan.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ring-mb", type=int, default=24576)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    run_ours(args)


if __name__ == "__main__":
    main()
