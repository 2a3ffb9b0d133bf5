#!/usr/bin/env python
"""bench.py — headline benchmark of the OWQS/EOWQS array executor on B200.

Metric (BASELINE.json): pattern commands/s and state-update HBM GB/s vs peak.
Default workload (N=1): config 3 — 28-wire random brickwork, depth 40 (5020 commands, paper m 29,
28 physical bits = 2 GiB complex64), sampled OWQS outcomes, complex64 amplitudes.
A step = set the resident input (device copy) + one owqs_run over the whole pattern.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C3]
For N > 1 launch with torch.distributed.run (one rank per GPU): by default every rank runs its own
replica (scaling "weak"); --shard shards one problem over the ranks on its top log2(N) slot bits
(NCCL swaps and all-reduces, scaling "strong"); --loopback G shards it over G virtual ranks on one
GPU.
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

WORKLOADS = {
    "C1": "config 1: 3-wire random J/CZ circuit (12 J, 4 CZ), 64 Haar inputs per step in one batched launch",
    "C3": "config 3: brickwork 28 wires x 40 layers (J(alpha) + alternating CZ), sampled OWQS",
    "C4": "config 4: brickwork 33 wires x 24 layers, sampled OWQS",
    "C5E": "config 5: 35 x 8 flow cluster, EOWQS (positive branch, no probabilities)",
    "C3W": "config 3 at width 30: brickwork 30 wires x 40 layers, sampled OWQS",
    "C2": "config 2: QFT-20 (H = J(0), CP = 8 J + 2 CZ), sampled OWQS",
    "C3E": "config 3 in EOWQS mode (positive branch, no probabilities)",
    "C5E32": "config 5's per-rank shard on one GPU: 32 x 8 flow cluster (2^32 complex64 = 32 GiB, the width "
             "each of 8 ranks holds for config 5), EOWQS",
    "C3M": "config 3 with 8 of its 28 wires measured after the last layer (SHRINK-heavy: 8 eliminations with "
           "the Eq. 13 reduction), sampled OWQS",
}


# oracle sample of the reference arm and of cpu_baseline (the same one): the pattern's first J gate
# at full width -- N, E, M, X: one command of every kind the J/CZ workloads consist of except the
# diagonal CZ (E is there), a measurement included (~15-20 s of numpy at 2^29 amplitudes)
REF_CMDS = 4
REF_BUDGET_S = 480.0  # wall-clock bound of one --impl reference run


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: C3 on one GPU; C4 sharded over the ranks (SURVEY §8(e)) for N > 1")
    ap.add_argument("--precision", type=int, default=64, choices=[64, 128])
    ap.add_argument("--flags", type=int, default=0, help="OWQS_FLAG_* for the timed context")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="N > 1: shard ONE problem over the N ranks (NCCL swaps / all-reduce, strong scaling); "
                         "the default for N > 1")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: every rank runs its own replica of the workload instead (weak scaling)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: N ranks over gloo compile the sharded program of the workload and agree on "
                         "its schedule; prints the JSON line shape with value null (CPU check of the N > 1 launch)")
    ap.add_argument("--loopback", type=int, default=1,
                    help="N = 1: shard the problem over this many virtual ranks on the one GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-contexts", type=int, default=3,
                    help="e2e serving pipeline depth: contexts (own state + stream) submitted round-robin")
    ap.add_argument("--ref-cmds", type=int, default=None,
                    help="oracle sample: first k commands at full width (default REF_CMDS = 4, one J gate, "
                         "for both cpu_baseline and every --impl reference step)")
    return ap.parse_args()


def pattern_for(workload):
    from workloads import patterns as W
    if workload in ("C3", "C3E"):
        return W.config_pattern("C3", seed=1), ("eowqs" if workload == "C3E" else "sampled")
    if workload == "C5E":
        return W.config_pattern("C5", seed=1), "eowqs"
    if workload == "C5E32":
        return W.config_pattern("CL:32x8", seed=1), "eowqs"
    return W.config_pattern(workload, seed=1), "sampled"


# --------------------------------------------------------------------------------------- clocks
REASONS = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, uuid):
        self.uuid = uuid
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        q = "clocks.sm,clocks.max.sm,power.draw," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        cmd = ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200"]
        if self.uuid:
            cmd += ["-i", self.uuid]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3 + len(REASONS):
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            for k, name in enumerate(REASONS):
                if r[3 + k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# -------------------------------------------------------------------------------------- oracle
def oracle_prefix_sample(pattern, psi, k_cmds, seed):
    """Run the oracle on the first k commands of `pattern` (full width). Returns (seconds, k)."""
    import oracle
    from workloads.patterns import prefix_pattern
    pre = prefix_pattern(pattern, k_cmds)
    t0 = time.perf_counter()
    oracle.run(pre, psi, mode="sampled", seed=seed)
    return time.perf_counter() - t0, len(pre.cmds)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------------------------------ reference
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import numpy as np  # noqa: F401
    from workloads.inputs import haar_state
    pattern, mode = pattern_for(args.workload)
    n = len(pattern.inputs)
    if n > 30:
        # 2^(n+1) complex128 amplitudes (config 4: 256 GiB, plus numpy temporaries) do not fit the host
        print(json.dumps({"impl": "reference", "unavailable":
                          f"the oracle needs 2^{n + 1} complex128 amplitudes on the host for {args.workload}"}), flush=True)
        return 0
    psi = haar_state(n, 1)
    times = []
    # The whole --steps K --warmup W run has to end within a few minutes (REF_BUDGET_S): the 4-command
    # sample (N E M X, the one cpu_baseline uses) costs ~33 s per step at config 3's 2^29 complex128
    # amplitudes on the B200 box's host, the 2-command sample (N E) ~7.5 s -- measured
    # (profiles/r02/bench_reference_final.log, BENCH_r01.json) and scaled by 2^(width - 29). With more
    # steps than the budget allows the sample shrinks to the N E prefix; the line says which.
    k = args.ref_cmds or REF_CMDS
    if not args.ref_cmds:
        est4 = 33.0 * 2.0 ** (n + 1 - 29)
        if (args.warmup + args.steps) * est4 > REF_BUDGET_S:
            k = 2
    for s in range(args.warmup + args.steps):
        dt, k = oracle_prefix_sample(pattern, psi, k, seed=s)
        if s >= args.warmup:
            times.append(dt)
    t = sum(times)
    value = k * len(times) / t
    line = {
        "impl": "reference", "metric": "pattern commands/s", "value": value, "unit": "commands/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload], "sample": f"first {k} commands at full width"},
        "cpu_baseline": {"value": value, "unit": "commands/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle (numpy complex128, given order) on the first {k} commands of "
                                   f"{args.workload} at full width ({n}+1 qubits), per step"},
        "e2e": {"value": value, "unit": "commands/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- config 1 (batched)
def run_batched_c1(args, rank, world, local_rank):
    """Config 1: each step runs 64 Haar inputs through one batched launch (owqs_run_batch) on a
    host buffer (so value and e2e coincide: the 64 x 8 x 16 B host round trip is inside)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1604_05659_b200 import Simulator
    from workloads import patterns as W
    from workloads.inputs import haar_state

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p = W.config_pattern("C1", seed=1)
    sim = Simulator(precision=args.precision, device=local_rank)
    sim.load(p)
    B = 64
    psis = np.stack([haar_state(3, 1000 * rank + k) for k in range(B)])
    for i in range(args.warmup):
        sim.run_batch(psis, "sampled", seeds=np.arange(B) + i * B)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        sim.run_batch(psis, "sampled", seeds=np.arange(B) + (args.warmup + i) * B)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    st = sim.stats()
    n_cmd = st["n_commands"]
    value = world * B * n_cmd * args.steps / dt
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        t1 = time.perf_counter()
        for k in range(B):
            oracle.run(p, psis[k], mode="sampled", seed=k)
        cdt = time.perf_counter() - t1
        cpu = {"value": B * n_cmd / cdt, "unit": "commands/s", "cores": 1, "kind": "oracle",
               "sample": f"the same 64 inputs of config 1 through the oracle: {cdt:.2f} s"}
    line = {"metric": "pattern commands/s", "value": value, "unit": "commands/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == 64 else "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS["C1"], "batch": B, "commands": n_cmd, "paper_m": st["paper_m"],
                       "phys_bits": st["phys_bits"], "parallelism": "single" if world == 1 else f"replicas{world}",
                       "timing": "wall clock around synchronous batched calls (host buffers)"},
            "roofline": None, "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "commands/s", "h2d_bytes_per_step": B * 8 * 16,
                    "d2h_bytes_per_step": B * 4 * 16},
            "gpu_launches": args.steps}
    if sim is not None:
        sim.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ ours
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1604_05659_b200 import FLAG_LOOPBACK, FLAG_PROFILE, KCLASS_NAMES, Simulator, nccl_unique_id
    from workloads.patterns import Pattern

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    pattern, mode = pattern_for(args.workload)
    n_in = len(pattern.inputs)
    N = 2 ** n_in
    prec = args.precision
    cdt = torch.complex64 if prec == 64 else torch.complex128
    shard = args.shard and world > 1          # one problem sharded over the ranks (NCCL)
    loop = args.loopback if world == 1 else 1  # one problem sharded over virtual ranks on one GPU
    n_shards = world if shard else loop

    def make_sim(extra_flags=0):
        kw = dict(precision=prec, device=local_rank, flags=args.flags | extra_flags, stream=stream.cuda_stream)
        if shard:
            ids = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
            return Simulator(n_ranks=world, rank=rank, nccl_id=ids[0], **kw)
        if loop > 1:
            kw["flags"] |= FLAG_LOOPBACK
            return Simulator(n_ranks=loop, **kw)
        return Simulator(**kw)

    sim = make_sim()
    t0 = time.perf_counter()
    sim.load(pattern)
    load_s = time.perf_counter() - t0
    st = sim.stats()

    state_bytes = N * (8 if prec == 64 else 16)
    big = state_bytes > (32 << 30)  # > 32 GiB: no host buffers (e2e / cpu_baseline skipped)
    # resident input copy whenever a second full-size buffer fits (config 4: 2 x 64 GiB of 180 GB);
    # otherwise the device counter-Haar generator runs inside every step
    total_mem = torch.cuda.get_device_properties(dev).total_memory
    if shard:
        # this rank's shard (+ its swap buffer) + a resident input shard + the generator's transient state
        resident = 4 * (state_bytes // world) <= 0.8 * total_mem
    else:
        resident = not big or 2 * state_bytes <= 0.8 * total_mem
    x = None
    if resident:
        # resident input: device Haar generator of the library, copied into a torch-owned buffer.
        # Sharded: every rank draws its own normalised shard and scales it by 1/sqrt(world), so the
        # ranks' shards together are one normalised state (owqs_set_input_device takes the shard).
        n_loc = n_in - (world.bit_length() - 1 if shard else 0)
        x = torch.empty(2 ** n_loc, dtype=cdt, device=dev)
        gen = Simulator(precision=prec, device=local_rank, stream=stream.cuda_stream)
        gen.load(Pattern(list(range(n_loc)), list(range(n_loc)), []))
        gen.set_input_random(1 + rank)
        gen.run("eowqs", want=False)
        gen.get_output_device(x.data_ptr(), prec, 2 ** n_loc)
        gen.close()
        if shard:
            x.mul_(world ** -0.5)
        torch.cuda.synchronize()

    def set_input(s, i):
        if x is None:  # device counter-Haar input (a second full-size state does not fit)
            s.set_input_random(1 + i)
        else:
            s.set_input_device(x.data_ptr(), prec, x.numel())

    def step(i):
        set_input(sim, i)
        sim.run(mode, seed=1000 + i + (0 if shard else 100_000 * rank), want=False)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    uuid = None
    try:
        uuid = "GPU-" + str(torch.cuda.get_device_properties(local_rank).uuid)
    except Exception:
        pass
    clk = ClockSampler(uuid)
    clk.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for i in range(args.steps):
        step(args.warmup + i)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    st = sim.stats()
    n_cmd = st["n_commands"]
    problems = 1 if shard else world  # replicas each run the whole pattern
    value = problems * n_cmd * args.steps / (ms / 1e3)
    hbm_gbs = st["bytes_per_run"] / (ms_per_step / 1e3) / 1e9  # per GPU (passes + swap pack / unpack)
    hbm_agg = None
    if shard:
        # SURVEY §8(d) 8-GPU fraction: sum over ranks of (pass bytes + swap pack / unpack + the NCCL send
        # and receive of half a shard per swap) over (time x ranks x peak), the collectives included in
        # the timed region; every rank moves the same bytes
        shard_bytes = (2 ** st["phys_bits"] >> (world.bit_length() - 1)) * (8 if prec == 64 else 16)
        per_rank = st["bytes_per_run"] + st["n_swaps"] * shard_bytes
        hbm_agg = {"bytes_per_rank_per_run": per_rank, "swaps_per_run": st["n_swaps"],
                   "gbs_per_gpu": per_rank / (ms_per_step / 1e3) / 1e9}

    # ---- roofline of the dominant kernel: per-launch CUDA events over profiled runs ----
    # A state pass moves 2S bytes (S = 2^w amplitudes x 8/16 B; S for a read-only reduction pass) and
    # issues, per amplitude, 3 FP32-pipe lane-ops per butterfly (w = x0 + a x1: 2 FFMA2 per pair;
    # 2 x0 - w: 1 FFMA2), +1 for the normalisation scale folded into the first butterfly (k x0 +-
    # (k a) x1: 4 packed ops per pair), 2 (norm) or 4 (rho) for the
    # probability reduction. Its roofline time is max(bytes / HBM peak, ops / FP32
    # peak); light passes are HBM-bound, heavy ones FP32-bound.
    if big:  # make room for the profiling context's state
        sim.close()
        sim = None
        if not shard:
            x = None
        torch.cuda.empty_cache()
    peak, peak_src = peaks()
    # FP32 (complex64) / FP64 (complex128) lanes x SMs x max SM clock (B200: 128 FP32, 64 FP64 lanes/SM)
    fp_lanes = 128 if prec == 64 else 64
    fp_peak = 148 * fp_lanes * 1.965e9
    prof = make_sim(FLAG_PROFILE)
    prof.load(pattern)
    per_step = None
    runs = 0
    for r in range(3):
        set_input(prof, r)
        prof.run(mode, seed=77 + r, want=False)
        if r == 0:
            continue  # first run captures the graph
        kc, by, tm = prof.launch_profile()
        per_step = (kc, by, tm.astype(np.float64)) if per_step is None else (kc, by, per_step[2] + tm)
        runs += 1
    prof_step_ms = prof.stats()["last_run_ms"]
    prof.close()
    kc, by, tm = per_step[0], per_step[1], per_step[2] / runs
    from paper_1604_05659_b200.host import compile_host, nvrtc_version
    hp = compile_host(pattern, "eowqs" if mode == "eowqs" else "sampled", prec, args.flags,
                      n_ranks=n_shards if (shard or loop > 1) else 1)
    ops = np.zeros(len(kc))
    for i, sd in enumerate(hp.steps[:len(kc)]):
        if sd.kind == 0:  # state pass
            amps = float(2 ** sd.width) * n_shards / (n_shards if shard else 1)
            per_amp = 3 * sd.n_bfly + (1 if sd.n_bfly else 0) + {0: 0, 1: 2, 2: 4}[sd.red_kind]
            ops[i] = amps * per_amp
    agg = {}
    for c in set(kc.tolist()):
        m = kc == c
        agg[int(c)] = [float(by[m].sum()), float(tm[m].sum()), int(m.sum()), float(ops[m].sum())]
    dom = max(agg, key=lambda c: agg[c][1])
    by_sum, ms_sum, cnt, ops_sum = agg[dom]
    m = kc == dom
    t_mem = by[m] / (peak * 1e9) * 1e3
    t_fp = ops[m] / fp_peak * 1e3
    roof_ms = float(np.maximum(t_mem, t_fp).sum())
    bw = by_sum / (ms_sum / 1e3) / 1e9
    fp = ops_sum / (ms_sum / 1e3)
    hbm_bound = t_mem.sum() >= t_fp.sum()
    traffic = ncu_traffic()
    if traffic and (traffic.get("workload") != args.workload or traffic.get("precision") != prec or n_shards > 1):
        traffic = None  # the committed capture is of another workload
    # alu in TFLOP/s: a lane-op is one FMA (2 FLOP) of the FP32 (complex64) / FP64 (complex128) pipe
    roofline = {"bound": "hbm" if hbm_bound else "alu",
                "achieved": bw if hbm_bound else 2 * fp / 1e12, "peak": peak if hbm_bound else 2 * fp_peak / 1e12,
                "unit": "GB/s" if hbm_bound else "TFLOP/s",
                "frac": bw / peak if hbm_bound else fp / fp_peak,
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "kernel": f"owqs::{KCLASS_NAMES[dom]}_kernel (generated tile kernels)", "launches": cnt,
                "bytes_per_launch": by_sum / cnt, "avg_launch_us": 1e3 * ms_sum / cnt,
                "share_of_step": ms_sum / prof_step_ms if prof_step_ms else None,
                "per_class_ms": {KCLASS_NAMES[c]: v[1] for c, v in agg.items()},
                "peak_source": peak_src, "algorithmic_bytes": "read + write of the 2^w-amplitude state per pass",
                "hbm": {"achieved_gbs": bw, "peak_gbs": peak, "frac": bw / peak,
                        "roofline_ms": float(t_mem.sum())},
                "alu": {"achieved_tops": fp / 1e12, "peak_tops": fp_peak / 1e12, "frac": fp / fp_peak,
                        "achieved_tflops": 2 * fp / 1e12, "peak_tflops": 2 * fp_peak / 1e12,
                        "unit": ("FP32-pipe lane-ops/s (FFMA2/FMUL2/FADD2 count 2)" if prec == 64 else
                                 "FP64-pipe ops/s (DFMA/DMUL/DADD)"), "roofline_ms": float(t_fp.sum()),
                        "peak_source": f"derived: 148 SMs x {fp_lanes} FP{32 if prec == 64 else 64} lanes x 1965 MHz"},
                "per_pass_roofline_frac": roof_ms / ms_sum,
                "per_pass_roofline_note": "sum over passes of max(bytes/HBM peak, lane-ops/FP32 peak) over measured time"}
    # the north star's HBM model: one read + write sweep of the state per measurement
    # at the measured copy peak; the fused path does many measurements per sweep, so it runs above
    # this model's 100 % figure
    sweep_s = None if shard else 2.0 * (2 ** st["phys_bits"]) * (8 if prec == 64 else 16) / (peak * 1e9)
    if sweep_s:
        at_peak = n_cmd / (st["n_measure"] * sweep_s) if st["n_measure"] else None
        roofline["sweep_per_measurement_model"] = {
            "commands_per_s_at_100pct_hbm": at_peak, "value_over_it": (value / problems) / at_peak if at_peak else None,
            "note": "SURVEY §8(d) / north star: 2S bytes per M at the measured copy peak; value_over_it > 1 means "
                    "faster than an HBM-bound one-sweep-per-measurement executor at 100 % of peak"}

    # ---- e2e through the C-ABI with host buffers (pinned), H2D + D2H inside the timed region ----
    e2e = None
    psi_host = None
    if not args.no_e2e and not shard and not big:
        # host buffers in the run's precision (page-locked): complex64 moves 8 B per amplitude each way
        hdt = torch.complex64 if prec == 64 else torch.complex128
        h_in = torch.empty(N, dtype=hdt, pin_memory=True)
        h_in.copy_(x.to(hdt))
        a_in = h_in.numpy()
        N_out = 2 ** len(pattern.outputs)
        # the pipeline fills and drains once inside the timed region (~1.5 steps of PCIe time): 8 x contexts
        # steps amortise it to ~6 %
        k_e2e = max(8 * args.e2e_contexts, args.steps)
        # serving pipeline over --e2e-contexts contexts on their own streams (owqs_submit_host / owqs_wait): every
        # step still does its own H2D copy, run and D2H copy, but one context's PCIe copies overlap
        # the other's kernels
        extra_streams = [torch.cuda.Stream(device=dev) for _ in range(max(0, args.e2e_contexts - 1))]
        extra = [] if loop > 1 else [Simulator(precision=prec, device=local_rank, flags=args.flags,
                                               stream=st.cuda_stream) for st in extra_streams]
        ctxs = [sim] + extra
        for x in extra:
            x.load(pattern)
        h_outs = [torch.empty(N_out, dtype=hdt, pin_memory=True) for _ in ctxs]
        busy = [False] * len(ctxs)

        def e2e_step(i):
            if loop > 1:  # loopback shards: the synchronous host calls (submit_host is single-rank)
                sim.set_input(a_in)
                sim.run(mode, seed=5000 + i, want=False)
                sim.get_output(h_outs[0].numpy())
                return
            c = i % len(ctxs)
            if busy[c]:
                ctxs[c].wait()
            ctxs[c].submit_host(h_in.data_ptr(), prec, h_outs[c].data_ptr(), prec, mode, seed=5000 + i)
            busy[c] = True

        def drain():
            for c in range(len(ctxs)):
                if busy[c]:
                    ctxs[c].wait()
                    busy[c] = False

        for i in range(len(ctxs)):
            e2e_step(i)
        drain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(k_e2e):
            e2e_step(len(ctxs) + i)
        drain()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        hb = N * (8 if prec == 64 else 16)
        e2e = {"value": problems * n_cmd * k_e2e / dt, "unit": "commands/s", "h2d_bytes_per_step": hb,
               "d2h_bytes_per_step": N_out * (8 if prec == 64 else 16), "steps": k_e2e, "ms_per_step": 1e3 * dt / k_e2e,
               "host_buffers": f"page-locked complex{prec}",
               "pipeline": (f"{len(ctxs)} contexts on separate streams (owqs_submit_host / owqs_wait)"
                            if loop <= 1 else "synchronous set_input / run / get_output")}
        for x in extra:
            x.close()
        psi_host = a_in.astype(np.complex128)
    elif shard or big:
        e2e = {"value": None, "unit": "commands/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "the 2^n host state (>= 128 GiB complex128) is not materialised; input generated on device"}
    # ---- CPU baseline: the oracle, rank 0 at N=1 only, bounded sample ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not big:
        if psi_host is None:
            psi_host = x.to(torch.complex128).cpu().numpy()
        psi_host = psi_host / np.linalg.norm(psi_host)
        dt, k = oracle_prefix_sample(pattern, psi_host, args.ref_cmds or REF_CMDS, seed=1)
        cpu = {"value": k / dt, "unit": "commands/s", "cores": 1, "kind": "oracle",
               "sample": f"oracle (numpy complex128, given order, single thread) on the first {k} commands "
                         f"of {args.workload} at full width ({n_in}->{n_in + 1} qubits): {dt:.1f} s",
               "host_cores_available": os.cpu_count()}

    if shard:
        par = f"shard{world}"
    elif loop > 1:
        par = f"loopback-shard{loop} (one GPU)"
    else:
        par = "single" if world == 1 else f"replicas{world}"
    line = {
        "metric": "pattern commands/s",
        "value": value, "unit": "commands/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if shard else "weak",
        "vs_baseline": None, "dtype": "f32" if prec == 64 else "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload], "mode": mode, "amplitudes": f"complex{prec}",
                   "nvrtc": "%d.%d" % nvrtc_version(),
                   "commands": n_cmd, "measurements": st["n_measure"], "paper_m": st["paper_m"],
                   "phys_bits": st["phys_bits"], "passes_per_run": st["n_passes"], "swaps_per_run": st["n_swaps"],
                   "launches_per_run": st["n_launches"], "state_bytes": N * (8 if prec == 64 else 16),
                   "l2": "state (>= 2 GiB) larger than the 126 MB L2: no flush needed",
                   "parallelism": par,
                   "input": "resident copy per step" if resident else "device counter-Haar per step",
                   "load_pattern_s": load_s, "schedule_ms": st["schedule_ms"]},
        "hbm_gbs": hbm_gbs, "hbm_frac": hbm_gbs / peak,
        "hbm_aggregate": (dict(hbm_agg, frac=hbm_agg["gbs_per_gpu"] / peak, ranks=world,
                               note="north star: >= 0.60 of the aggregate HBM roofline incl. swap traffic")
                          if hbm_agg else None),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(round(st.get("n_kernels") or st["n_launches"])) * args.steps * n_shards // (n_shards if shard else 1),
        "clocks": clocks,
    }
    if sim is not None:
        sim.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def spawn(args):
    """python bench.py --gpus N (N > 1) outside torchrun: re-launch as N ranks on this node, the way the
    driver does (torch.distributed.run, rendezvous on 127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, rank, world):
    """--dry-run (CPU, gloo): every rank compiles the workload's program sharded over `world` ranks
    (include/owqs_host.h) and the ranks all-reduce its schedule (passes, swaps, bytes) -- the N > 1 launch
    path without a GPU. No state is simulated: value is null."""
    import torch
    import torch.distributed as dist
    from paper_1604_05659_b200.host import compile_host
    if world > 1:
        dist.init_process_group("gloo")
    pattern, mode = pattern_for(args.workload)
    hp = compile_host(pattern, "eowqs" if mode == "eowqs" else "sampled", args.precision, args.flags,
                      n_ranks=world if world > 1 else 1)
    mine = torch.tensor([hp.info["n_passes"], hp.info["n_swaps"], hp.info["phys_bits"]], dtype=torch.float64)
    agree = True
    if world > 1:
        lo, hi = mine.clone(), mine.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        agree = bool(torch.equal(lo, hi))
    if rank == 0:
        print(json.dumps({
            "metric": "pattern commands/s", "value": None, "unit": "commands/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == 64 else "f64", "data": "synthetic", "dry_run": True,
            "config": {"workload": WORKLOADS[args.workload], "mode": mode, "parallelism": f"shard{world}",
                       "phys_bits": hp.info["phys_bits"], "passes_per_run": hp.info["n_passes"],
                       "swaps_per_run": hp.info["n_swaps"], "ranks_agree_on_schedule": agree,
                       "backend": "gloo (CPU): schedule only, no kernels"}}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if agree else 1


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload is None:
        args.workload = "C4" if world > 1 and not args.replicas else "C3"
    if world > 1 and not args.replicas:
        args.shard = True
    if args.dry_run:
        return dry_run(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    rc = run_batched_c1(args, rank, world, local_rank) if args.workload == "C1" else run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
