"""Benchmark of the compressed state-vector update path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload grover20|qft28|qft16|random30]

Workload (BASELINE.json configs[1], the N=1 headline): 20-qubit Grover
search, 64 slices of 2^14 complex128 amplitudes, absolute error bound 1e-5,
marked index drawn from the seed.  One *step* = one Grover iteration
(oracle X-MCZ-X + diffusion H-X-MCZ-X-H, ~110 gate passes over all 2^20
amplitudes).  The initial H layer and W iterations are untimed warm-up.

Metric: amplitude-gate updates/s including (de)compression
(= 2^n x gate passes / time).  `value` is device time (CUDA events on the
engine stream, inputs resident in HBM); `e2e` drives the same steps through
the C-ABI with host buffers: the step's action list copied in and the
compressed state + metrics copied out every step.

N > 1 (torchrun): slices are sharded by their top index bits; gates on those
bits exchange compressed partner slices over NCCL (distributed.py); the
per-gate sq_norm table is all-gathered.  Timing is the max over ranks.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", HBM_FALLBACK)), "measured"
    return HBM_FALLBACK, "fallback"


# ------------------------------------------------------------- workloads
def workload(name, extra=0):
    """extra: additional qubits (weak scaling: n + log2(world) keeps the
    slices per GPU fixed)."""
    import paper_1811_05630_b200 as q
    if name == "grover20":
        n, s, eb = 20 + extra, 14, 1e-5
        marked = q.seeded_index(n, 20)
        iters = q.grover_optimal_iterations(n)
        oracle = q.build_grover_oracle(n, marked).gates
        diff = ([q.Gate.h(k) for k in range(n)] + [q.Gate.x(k) for k in range(n)] + [q.Gate.mcz(range(n))]
                + [q.Gate.x(k) for k in range(n)] + [q.Gate.h(k) for k in range(n)])
        step = [q.to_action_c(q.gate_action(g)) for g in oracle + diff]
        setup = [q.to_action_c(q.gate_action(q.Gate.h(k))) for k in range(n)]
        return dict(name="grover20", n=n, s=s, eb=eb, basis=0, setup=setup, steps=lambda k: step,
                    max_steps=iters, desc=f"grover n={n} marked={marked} iterations={iters}, slices {1 << (n - s)}x2^{s}")
    if name in ("qft28", "qft16"):
        base = 28 if name == "qft28" else 16
        n = base + extra
        s = 20 if base == 28 else 12
        acts = q.lower(q.build_qft(n))
        x = q.seeded_index(n, n)
        chunk = 35 if base == 28 else 12
        return dict(name=name, n=n, s=s, eb=1e-5, basis=x, setup=[],
                    steps=lambda k: acts[k * chunk:(k + 1) * chunk], max_steps=len(acts) // chunk,
                    desc=f"qft n={n} basis={x}, slices {1 << (n - s)}x2^{s}, step = {chunk} gates")
    if name == "random30":
        n, s = 30 + extra, 20
        acts = q.random_u3_circuit_actions(n, 20, seed=30)
        per = n + n // 2
        return dict(name=name, n=n, s=s, eb=1e-5, basis=0, setup=[], steps=lambda k: acts[k * per:(k + 1) * per],
                    max_steps=20, desc=f"random U3+CZ n={n} depth 20, slices {1 << (n - s)}x2^20, step = 1 layer")
    raise SystemExit(f"unknown workload {name}")


# ------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self):
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50", "-i", os.environ.get("LOCAL_RANK", "0")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- CPU arms
def cpu_reference(wl, args, budget_s=12.0):
    """The reference's own codec (oracle/_ref, compiled from /root/reference
    unmodified) under the pinned engine loop with a pool of all host cores;
    falls back to the C restatement (kind 'port') when _ref is absent."""
    from oracle.oracle import CodecConfig as OCfg, EngineConfig as OEng, REF_SO, Oracle, RefLib
    cores = os.cpu_count() or 1
    cfg = OEng.make(wl["n"], wl["s"], OCfg.make(1, wl["eb"], 16, 0))
    if os.path.exists(REF_SO):
        from oracle.oracle import Action
        eng = RefLib().engine(cfg, workers=cores)
        kind = "reference"
        gate = lambda a: eng.gate(Action.from_buffer_copy(bytes(a)))  # noqa: E731
    else:
        eng = Oracle().engine(cfg)
        kind, cores = "port", 1
        gate = lambda a: eng.run([a])  # noqa: E731
    eng.load_basis(wl["basis"])
    for a in wl["setup"]:
        gate(a)
    done = 0
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < budget_s and k < wl["max_steps"]:
        for a in wl["steps"](k):
            gate(a)
            done += 1
            if time.perf_counter() - t0 > budget_s:
                break
        k += 1
    dt = time.perf_counter() - t0
    value = (1 << wl["n"]) * done / dt
    return dict(value=value, unit="updates/s", cores=cores, kind=kind,
                sample=f"{done} gate passes of {wl['name']} after its setup layer ({dt:.1f} s, all slices)")


# ------------------------------------------------------------- GPU arm
def run_ours(args, wl, rank, world, dist):
    import ctypes

    import numpy as np
    import torch

    import paper_1811_05630_b200 as q
    from paper_1811_05630_b200 import _native
    from paper_1811_05630_b200.distributed import ShardedEngine

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    cfg = q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"], codec=q.CodecConfig(q.CodecMode.Absolute, wl["eb"]),
                         device=dev, rank=rank, world=world)
    eng = ShardedEngine(cfg) if world > 1 else q.Engine(cfg)
    eng.load_basis(wl["basis"])
    eng.run(wl["setup"])
    history = []  # every gate list run after the setup layer (accuracy check)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")  # > L2 (126 MB)
    lib = _native.lib()
    for k in range(args.warmup):
        eng.run(wl["steps"](k))
        history.append(wl["steps"](k))
    gates = 0
    dev_s = 0.0
    wall = 0.0
    launches0 = lib.qcsim_kernel_launches()
    prof = None  # timed loop runs without the event profiler
    clocks = ClockSampler()
    clocks.start()
    for k in range(args.warmup, args.warmup + args.steps):
        acts = wl["steps"](k % wl["max_steps"])
        flush.zero_()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        m0 = eng.metrics().wall_seconds
        t0 = time.perf_counter()
        m = eng.run(acts)
        wall += time.perf_counter() - t0
        history.append(acts)
        dev_s += m.wall_seconds - m0
        gates += len(acts)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = lib.qcsim_kernel_launches() - launches0
    # kernel shares: a separate, shorter profiled pass (CUDA events per kernel)
    if hasattr(lib, "qcsim_debug_chain_stats"):
        lib.qcsim_debug_chain_stats((ctypes.c_uint32 * 5)())  # reset: count the profiled pass only
    prof = profile_begin(lib)
    for k in range(args.warmup + args.steps, args.warmup + args.steps + max(1, args.steps // 2)):
        eng.run(wl["steps"](k % wl["max_steps"]))
        history.append(wl["steps"](k % wl["max_steps"]))
    kprof = profile_end(lib, prof)
    mets = eng.metrics()
    chain = None
    if hasattr(lib, "qcsim_debug_chain_stats"):
        cs = (ctypes.c_uint32 * 5)()
        if lib.qcsim_debug_chain_stats(cs) == 0:
            chain = {"resolve_points": int(cs[0]), "refuted_chunks": int(cs[1]), "serial_chunks": int(cs[2]),
                     "events": int(cs[3]) | (int(cs[4]) << 32)}

    # e2e: the same step count through the C-ABI with host buffers
    e2e_t, h2d, d2h = 0.0, 0, 0
    for k in range(args.warmup + args.steps, args.warmup + 2 * args.steps):
        acts = wl["steps"](k % wl["max_steps"])
        arr = (_native.ActionC * len(acts))(*acts)
        flush.zero_()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        pinned = torch.empty(ctypes.sizeof(arr), dtype=torch.uint8, pin_memory=True)
        ctypes.memmove(pinned.data_ptr(), ctypes.addressof(arr), ctypes.sizeof(arr))
        m = eng.run(acts)
        history.append(acts)
        blocks = eng.export_blocks()[0] if world == 1 else eng.export_local_blocks()
        e2e_t += time.perf_counter() - t0
        h2d += ctypes.sizeof(arr)
        d2h += len(blocks) + ctypes.sizeof(_native.RunMetricsC)
    # accuracy: the same gate sequence through a
    # compression-off FP64 engine, compared on the device (outside all timing)
    accuracy = None
    if world == 1 and wl["n"] <= 30:
        dense = None
        try:
            dense = q.Engine(q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"], compression_enabled=False,
                                            device=dev))
            dense.load_basis(wl["basis"])
            dense.run(wl["setup"])
            for acts in history:
                dense.run(acts)
            r = eng.compare(dense)
            accuracy = {"max_abs_err_vs_fp64": r["max_abs_diff"],
                        "fidelity_vs_fp64": r["fidelity"] / (r["norm_a"] * r["norm_b"]),
                        "gates": len(wl["setup"]) + sum(len(a) for a in history),
                        "basis": "same gates through a compression-off FP64 engine, compared on the device"}
        except MemoryError as exc:  # the dense FP64 replica does not fit beside the engine's scratch
            accuracy = {"skipped": f"dense FP64 replica does not fit in HBM beside the compressed engine ({exc})"}
        del dense
    return dict(gates=gates, dev_s=dev_s, wall=wall, clocks=clk, launches=launches, metrics=mets, kprof=kprof, chain=chain,
                accuracy=accuracy,
                e2e_t=e2e_t, h2d=h2d // max(1, args.steps), d2h=d2h // max(1, args.steps))


def profile_begin(lib):
    try:
        fn = lib.qcsim_profile_enable
    except AttributeError:
        return None
    fn.argtypes = [ctypes_int()]
    fn(1)
    return True


def ctypes_int():
    import ctypes
    return ctypes.c_int


def profile_end(lib, token):
    if token is None:
        return None
    import ctypes
    n = 64
    names = (ctypes.c_char * 64 * n)()
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_uint64 * n)()
    nbytes = (ctypes.c_double * n)()
    fn = lib.qcsim_profile_read
    fn.restype = ctypes.c_int
    k = fn(names, ms, cnt, nbytes, n)
    lib.qcsim_profile_enable(0)
    out = []
    for i in range(k):
        out.append(dict(kernel=bytes(names[i]).split(b"\0")[0].decode(), ms=ms[i], launches=cnt[i],
                        algo_bytes=nbytes[i]))
    return sorted(out, key=lambda r: -r["ms"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="grover20")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        tdist.init_process_group("nccl")
        dist = tdist
    extra = max(0, world.bit_length() - 1) if world > 1 else 0  # weak scaling: slices per GPU fixed
    wl = workload(args.workload, extra)
    hbm, peak_kind = measured_peaks()
    config = {"workload": wl["name"], "detail": wl["desc"], "n_qubits": wl["n"], "slice_bits": wl["s"],
              "error_bound": wl["eb"], "mode": "absolute", "quant_code_bits": 16, "predictor": "previous",
              "step": "one Grover iteration" if wl["name"] == "grover20" else "gate chunk",
              "l2": "flushed between timed steps (256 MiB write)", "norm": "every gate",
              "weak_scaling": "n = base qubits + log2(n_gpus): the slices (and work) per GPU are fixed"}

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference(wl, args, budget_s=args.cpu_budget)
        line = {"metric": "amplitude-gate updates/s incl. (de)compression", "value": r["value"],
                "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded circuit)", "config": config, "impl": "reference",
                "cpu_baseline": r, "e2e": {"value": r["value"], "unit": "updates/s", "h2d_bytes_per_step": 0,
                                            "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    res = run_ours(args, wl, rank, world, dist)
    dev_s, wall = res["dev_s"], res["wall"]
    if dist:
        import torch
        t = torch.tensor([dev_s, wall, res["e2e_t"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, wall, e2e_t = t.tolist()
    else:
        e2e_t = res["e2e_t"]
    N = 1 << wl["n"]
    value = N * res["gates"] / dev_s
    m = res["metrics"]
    if rank != 0:
        dist.destroy_process_group() if dist else None
        return
    # roofline of the dominant kernel: algorithmic bytes per launch / its
    # average launch duration (CUDA events in the profiled pass).  The chain
    # kernel moves 28 B per event (addend 8 + event word 4 + lattice estimate
    # 8 read, chain value 8 written); events are counted on the device.
    kprof = res["kprof"] or []
    dominant = kprof[0] if kprof else None
    chain = res.get("chain") or {}
    achieved, algo_launch = None, None
    prof_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    traffic, basis = None, None
    elem_planes = 2.0 * (1 << wl["n"]) / world  # re + im planes of this rank (one pass)
    ntiles = ((1 << wl["s"]) + 1023) // 1024
    if dominant and dominant["kernel"] == "enc_chain_scan" and chain.get("events"):
        algo_launch = 28.0 * chain["events"] / dominant["launches"]
        basis = "enc_chain_scan: 28 B per chained event (device-counted) / mean launch time"
        tf = os.path.join(prof_dir, "r01_v18_chain_scan_ncu.json")
        if os.path.exists(tf):
            with open(tf) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
    elif dominant and dominant["kernel"] == "enc_chain" and chain.get("events"):
        # serial warp chain (one warp per plane): the same 28 B per event as
        # the scan form, streamed through its TMA ring
        algo_launch = 28.0 * chain["events"] / dominant["launches"]
        basis = "enc_chain: 28 B per chained event (device-counted) / mean launch time"
    elif dominant and dominant["kernel"] == "enc_lattice" and ntiles > 64:
        # dense pass (planes of > 64 tiles): x (8 B) and flags (1 B) in;
        # symbols (4 B) and flags (1 B) out per element of every plane (the
        # lattice estimates are written at events only; events are
        # negligible at these ratios)
        algo_launch = 14.0 * elem_planes
        basis = "enc_lattice: 14 B per element-plane (x, flags in; symbols, flags out) / mean launch time"
        tf = os.path.join(prof_dir, "r01_v16_qft28_pass_dram.json")
        if os.path.exists(tf) and wl["name"] == "qft28":
            with open(tf) as f:
                for ln in json.load(f)["launches"]:
                    if ln["kernel"] == "enc_lattice":
                        traffic = ln["dram_read_bytes"] + ln["dram_write_bytes"]
    elif dominant and dominant["kernel"] == "enc_verify" and ntiles > 64:
        # dense pass: x (8 B), flags (1 B) and the speculated symbol (4 B) read
        # per element of every plane (chain values and index records are
        # negligible at these ratios)
        algo_launch = 13.0 * elem_planes
        basis = "enc_verify: 13 B per element-plane (x, flags, symbol in) / mean launch time"
        tf = os.path.join(prof_dir, "r01_v16_qft28_pass_dram.json")
        if os.path.exists(tf) and wl["name"] == "qft28":
            with open(tf) as f:
                for ln in json.load(f)["launches"]:
                    if ln["kernel"] == "enc_verify":
                        traffic = ln["dram_read_bytes"] + ln["dram_write_bytes"]
    elif dominant and dominant["kernel"] == "enc_compact" and chain.get("events"):
        # per element-plane: the flags (1 B); per event: flags, symbol and
        # lattice estimate (13 B) read (x only at outliers) and the record
        # (index 4 B, addend 8 B, estimate 8 B) written; events counted on
        # the device
        algo_launch = (1.0 * elem_planes * dominant["launches"] + 33.0 * chain["events"]) / dominant["launches"]
        basis = "enc_compact: 1 B per element-plane + 33 B per event (device-counted) / mean launch time"
    elif dominant and dominant["kernel"] == "dec_chunks":
        # dense write of every decoded value (8 B per element-plane) plus
        # the compressed stream read
        algo_launch = 8.0 * elem_planes + float(m.current_compressed_bytes * world)
        basis = "dec_chunks: 8 B written per element-plane + the compressed blocks read / mean launch time"
    if algo_launch is not None:
        achieved = algo_launch / (dominant["ms"] * 1e-3 / dominant["launches"]) / 1e9
    # SURVEY.md §8(d) pass basis: input + output compressed block bytes per
    # gate pass / device time per pass
    algo_per_pass = 2.0 * m.current_compressed_bytes * world
    pass_achieved = algo_per_pass * res["gates"] / dev_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": (achieved / hbm) if achieved is not None else None, "traffic": traffic, "peak_kind": peak_kind,
            "kernel": dominant["kernel"] if dominant else None, "algo_bytes_per_launch": algo_launch,
            "basis": basis,
            "pass_basis": {"achieved": pass_achieved, "frac": pass_achieved / hbm,
                           "basis": "per gate pass: input+output QCB1 block bytes (SURVEY.md 8(d)) / device time"},
            "dense_equivalent": {"achieved": 32.0 * (1 << wl["n"]) * res["gates"] / dev_s / 1e9,
                                 "basis": "32 B per amplitude update (SURVEY.md 8(d), not judged)"},
            "kernel_shares": kprof[:8], "kernel_ms_total": sum(k["ms"] for k in kprof), "chain_scan": chain}
    cpu = None
    if args.gpus == 1 and world == 1:
        try:
            cpu = cpu_reference(wl, args, budget_s=args.cpu_budget)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}
    line = {"metric": "amplitude-gate updates/s incl. (de)compression", "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded circuit, random-free)",
            "config": config, "clocks": res["clocks"], "gpu_launches": int(res["launches"]),
            "e2e": {"value": N * res["gates"] / e2e_t, "unit": "updates/s", "h2d_bytes_per_step": res["h2d"],
                    "d2h_bytes_per_step": res["d2h"]},
            "roofline": roof, "cpu_baseline": cpu,
            "compression": {"min_ratio": m.min_compression_ratio, "mean_ratio": m.mean_compression_ratio,
                            "compressed_bytes": m.current_compressed_bytes, "dense_bytes": m.dense_bytes,
                            "fallback_planes": m.fallback_planes},
            "accuracy": res.get("accuracy"),
            "wall_ms_per_step": 1e3 * wall / args.steps}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
