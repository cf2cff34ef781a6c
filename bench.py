"""Benchmark of the compressed state-vector update path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload random30|grover20|qft28|qft16|qft32|grover38]
                    [--eb EB] [--parity auto|on|off]

Workload (N=1 headline): BASELINE.json configs[3], the largest single-GPU
config -- a 30-qubit random circuit of depth 20 (U3 on every qubit, then CZ
on a seeded perfect matching), 1024 slices of 2^20 complex128 amplitudes,
absolute error bound 1e-5.  The first layer (45 gates, which turns the basis
state into a dense low-compressibility state) is untimed setup; one *step*
is one gate pass over all 2^30 amplitudes, W steps warm up, K steps are
timed.  No window wraps: every workload replays a contiguous prefix of its
circuit.

Metric: amplitude-gate updates/s including (de)compression (= 2^n x gate
passes / time).  `value`: device time (CUDA events on the engine stream,
state resident in HBM).  `e2e`: the same K gates replayed on a freshly loaded
engine through the public API (C-ABI, host action array in, run metrics and
per-slice norms out every step, the whole compressed state's QCB1 blocks out
after the last step), timed by the host clock.

Parity: after the timed window the engine's QCB1 arena is hashed (SHA-256)
and compared with the reference engine (the reference's own codec compiled
from /root/reference by oracle/Makefile, all host cores) replaying the same
gate prefix; the reference's time for the W+K gates is the `cpu_baseline`.

N > 1 (torchrun): slices are sharded by their top index bits; gates on those
bits exchange compressed partner slices (distributed.py); `value` is the
barrier-synchronised host wall time of the gate passes, max over ranks.
"""
from __future__ import annotations

import argparse
import hashlib
import json
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
        return float(d.get("hbm_gbs", HBM_FALLBACK)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------- workloads
def workload(name, extra=0, eb=None):
    """Gate list = setup + steps.  extra: additional qubits (weak scaling:
    n + log2(world) keeps the slices per GPU fixed)."""
    import paper_1811_05630_b200 as q
    norm_every = 1
    if name == "random30":
        n, s = 30 + extra, 20
        gates = q.random_u3_circuit_actions(n, 20, seed=30)
        setup, per = n + n // 2, 1
        desc = f"random U3+CZ n={n} depth 20 (configs[3]), slices {1 << (n - s)}x2^{s}; setup = layer 0; step = 1 gate"
        basis = 0
    elif name in ("grover20", "grover38"):
        base = 20 if name == "grover20" else 38
        n, s = base + extra, (14 if base == 20 else 22)
        marked = q.seeded_index(n, base)
        iters = q.grover_optimal_iterations(n) if base == 20 else 32
        oracle = q.build_grover_oracle(n, marked).gates
        diff = ([q.Gate.h(k) for k in range(n)] + [q.Gate.x(k) for k in range(n)] + [q.Gate.mcz(range(n))]
                + [q.Gate.x(k) for k in range(n)] + [q.Gate.h(k) for k in range(n)])
        it = [q.to_action_c(q.gate_action(g)) for g in oracle + diff]
        hl = [q.to_action_c(q.gate_action(q.Gate.h(k))) for k in range(n)]
        if base == 20:
            gates, setup, per = hl + it * iters, n, len(it)
            desc = f"grover n={n} marked={marked} iterations={iters} (configs[1]), slices {1 << (n - s)}x2^{s}; " \
                   f"setup = H layer; step = 1 iteration ({per} gates)"
        else:
            # configs[4]: amplitude 2^-19 < eb, the state quantizes to zero
            # -- timed with normalization off
            gates, setup, per = hl + it * iters, 0, 1
            norm_every = 0
            desc = f"grover n={n} marked={marked} 32 iterations (configs[4]) on ONE GPU, slices " \
                   f"{1 << (n - s)}x2^{s}; step = 1 gate; norm off (degenerate, SURVEY F9)"
        basis = 0
    elif name in ("qft28", "qft16", "qft32"):
        base = int(name[3:])
        n = base + extra
        s = 12 if base == 16 else 20
        gates = q.lower(q.build_qft(n))
        basis = q.seeded_index(n, n)
        setup = 0
        per = 6 if base == 16 else (15 if base == 28 else 1)
        desc = f"qft n={n} basis={basis}, slices {1 << (n - s)}x2^{s}; step = {per} gates (circuit order)"
    else:
        raise SystemExit(f"unknown workload {name}")
    if eb is None:
        eb = 1e-5
    nsteps = (len(gates) - setup) // per
    return dict(name=name, n=n, s=s, eb=eb, basis=basis, setup=gates[:setup], per=per, nsteps=nsteps,
                steps=lambda k: gates[setup + k * per: setup + (k + 1) * per], norm_every=norm_every, desc=desc)


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
def _ref_engine(wl, cores):
    """The reference's own codec (oracle/_ref, compiled from /root/reference
    unmodified) under the pinned engine loop, a pool of `cores` threads; the
    C restatement (kind 'port', one core) when _ref was not built."""
    from oracle.oracle import Action, CodecConfig as OCfg, EngineConfig as OEng, REF_SO, Oracle, RefLib
    cfg = OEng.make(wl["n"], wl["s"], OCfg.make(1, wl["eb"], 16, 0), True, wl["norm_every"])
    if os.path.exists(REF_SO):
        eng = RefLib().engine(cfg, workers=cores)
        return eng, "reference", cores, lambda a: eng.gate(Action.from_buffer_copy(bytes(a)))
    eng = Oracle().engine(cfg)
    return eng, "port", 1, lambda a: eng.run([a])


def cpu_replay(wl, steps, budget_s=None):
    """Setup + `steps` steps on the CPU reference engine.  Returns the timing
    of the steps (not the setup) and the arena hash after them."""
    cores = os.cpu_count() or 1
    eng, kind, cores, gate = _ref_engine(wl, cores)
    eng.load_basis(wl["basis"])
    t0 = time.perf_counter()
    for a in wl["setup"]:
        gate(a)
    t_setup = time.perf_counter() - t0
    done, complete = 0, True
    t0 = time.perf_counter()
    for k in range(steps):
        for a in wl["steps"](k):
            gate(a)
            done += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            complete = k + 1 == steps
            break
    dt = time.perf_counter() - t0
    sha = hashlib.sha256(eng.export_blocks()).hexdigest() if complete else None
    return dict(value=(1 << wl["n"]) * done / dt, unit="updates/s", cores=cores, kind=kind, gates=done,
                seconds=dt, setup_seconds=t_setup, sha=sha)


# ------------------------------------------------------------- GPU arm
def run_ours(args, wl, rank, world, dist):
    import ctypes

    import torch

    import paper_1811_05630_b200 as q
    from paper_1811_05630_b200 import _native
    from paper_1811_05630_b200.distributed import ShardedEngine

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    cfg = q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"], codec=q.CodecConfig(q.CodecMode.Absolute, wl["eb"]),
                         device=dev, rank=rank, world=world, norm_every=wl["norm_every"])
    eng = ShardedEngine(cfg) if world > 1 else q.Engine(cfg)
    lib = _native.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")  # > L2 (126 MB)
    W, K = args.warmup, args.steps
    if W + K > wl["nsteps"]:
        raise SystemExit(f"{wl['name']}: warmup + steps = {W + K} exceeds the circuit's {wl['nsteps']} steps")
    P = min(max(1, K // 2), wl["nsteps"] - W - K)  # profiled steps (per-kernel events)

    def load():
        eng.load_basis(wl["basis"])
        eng.run(wl["setup"])
        for k in range(W):
            eng.run(wl["steps"](k))

    def timed(k, fn):
        flush.zero_()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        r = fn(k)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return r, time.perf_counter() - t0

    load()
    m_w = eng.metrics()
    gates0 = m_w.gates
    launches0 = lib.qcsim_kernel_launches()
    clocks = ClockSampler()
    clocks.start()
    dev_s, wall, gates = 0.0, 0.0, 0
    step_ms = []
    for k in range(W, W + K):
        m0 = eng.metrics().wall_seconds
        m, dt = timed(k, lambda k: eng.run(wl["steps"](k)))
        wall += dt
        dev_s += m.wall_seconds - m0
        step_ms.append(round(1e3 * (m.wall_seconds - m0), 3))
        gates += len(wl["steps"](k))
    clk = clocks.stop()
    launches = lib.qcsim_kernel_launches() - launches0
    m_t = eng.metrics()
    sha = hashlib.sha256(eng.export_blocks_array()[0]).hexdigest() if world == 1 else None
    rows = eng.gate_metrics() if hasattr(eng, "gate_metrics") else None
    # kernel shares: P further steps with the per-kernel event profiler
    if hasattr(lib, "qcsim_debug_chain_stats"):
        lib.qcsim_debug_chain_stats((ctypes.c_uint32 * 5)())  # reset: count the profiled steps only
    lib.qcsim_profile_enable(1)
    pgates = 0
    for k in range(W + K, W + K + P):
        eng.run(wl["steps"](k))
        pgates += len(wl["steps"](k))
    kprof = profile_read(lib)
    chain = None
    if hasattr(lib, "qcsim_debug_chain_stats"):
        cs = (ctypes.c_uint32 * 5)()
        if lib.qcsim_debug_chain_stats(cs) == 0:
            chain = {"resolve_points": int(cs[0]), "refuted_chunks": int(cs[1]), "serial_chunks": int(cs[2]),
                     "events": int(cs[3]) | (int(cs[4]) << 32)}
    m_p = eng.metrics()
    # accuracy: the same gates through a compression-off FP64
    # engine, compared on the device (outside all timing)
    accuracy = None
    if world == 1 and wl["n"] <= 32 and not args.no_accuracy:
        dense = None
        try:
            eng.trim()  # the FP64 replica needs the gate-pass scratch's room
            dense = q.Engine(q.EngineConfig(num_qubits=wl["n"], slice_bits=wl["s"], compression_enabled=False,
                                            device=dev, norm_every=wl["norm_every"]))
            dense.load_basis(wl["basis"])
            dense.run(wl["setup"])
            for k in range(W + K + P):
                dense.run(wl["steps"](k))
            r = eng.compare(dense)
            accuracy = {"max_abs_err_vs_fp64": r["max_abs_diff"],
                        "fidelity_vs_fp64": r["fidelity"] / (r["norm_a"] * r["norm_b"]),
                        "gates": len(wl["setup"]) + (W + K + P) * wl["per"],
                        "basis": "same gates through a compression-off FP64 engine, compared on the device"}
        except MemoryError as exc:
            accuracy = {"skipped": f"dense FP64 replica does not fit in HBM beside the compressed engine ({exc})"}
        del dense
    # e2e: reload, replay setup + warmup, then the same K gates through the
    # public API with host buffers: every step the action array in and the
    # run metrics + per-slice norms out; after the last step the whole
    # compressed state (QCB1 blocks) out
    load()
    e2e_t, h2d, d2h = 0.0, 0, 0
    for k in range(W, W + K):
        acts = wl["steps"](k)

        def step(k, acts=acts):
            arr = (_native.ActionC * len(acts))(*acts)
            eng.run(arr)
            out = ctypes.sizeof(_native.RunMetricsC) + 8 * len(eng.slice_norms())
            if k == W + K - 1:
                blob = eng.export_blocks_array()[0] if world == 1 else eng.export_local_blocks()
                out += len(blob)
            return ctypes.sizeof(arr), out

        (hi, ho), dt = timed(k, step)
        e2e_t += dt
        h2d += hi
        d2h += ho
    mem = q.device_memory() if hasattr(q, "device_memory") else None
    return dict(gates=gates, dev_s=dev_s, wall=wall, clocks=clk, launches=launches, m_w=m_w, m_t=m_t, m_p=m_p,
                gates0=gates0, rows=rows, kprof=kprof, step_ms=step_ms, pgates=pgates, chain=chain, accuracy=accuracy, sha=sha,
                e2e_t=e2e_t, h2d=h2d // K, d2h=d2h // K, mem=mem)


def profile_read(lib):
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
    out = [dict(kernel=bytes(names[i]).split(b"\0")[0].decode(), ms=ms[i], launches=cnt[i]) for i in range(k)]
    return sorted(out, key=lambda r: -r["ms"])


def roofline(res, wl, hbm, peak_kind, world):
    """algorithmic bytes of a gate pass = QCB1 input + output
    block bytes of every plane, plus the decode-index bytes read and written;
    achieved = those bytes / the dominant kernel's device time per pass."""
    kprof = res["kprof"] or []
    dom = kprof[0] if kprof else None
    rows = res["rows"]
    m_w, m_t = res["m_w"], res["m_t"]
    if rows:
        # rows[g] = state after gate g (since load); timed gates are
        # (gates0, gates0 + K]
        g0 = res["gates0"]
        tb = [rows[g]["bytes"] + rows[g]["index_bytes"] for g in range(len(rows))]
        per_pass = [tb[g - 1] + tb[g] for g in range(g0, g0 + res["gates"])]
        bytes_pass = sum(per_pass) / len(per_pass)
        basis_note = "per-gate block + index bytes (engine gate metrics)"
    else:
        cur = m_t.current_compressed_bytes + m_t.index_bytes
        bytes_pass = 2.0 * cur * world
        basis_note = "2 x final compressed + index bytes"
    out = {"bound": "hbm", "peak": hbm, "unit": "GB/s", "peak_kind": peak_kind,
           "algo_bytes_per_pass": bytes_pass, "algo_basis": "QCB1 bytes in + out + index bytes read + written "
                                                            "per gate pass (SURVEY.md 8(d)); " + basis_note}
    if dom:
        t_pass = dom["ms"] * 1e-3 / max(1, res["pgates"])
        ach = bytes_pass / t_pass / 1e9
        out.update({"achieved": ach, "frac": ach / hbm, "kernel": dom["kernel"], "kernel_s_per_pass": t_pass})
    else:
        out.update({"achieved": None, "frac": None, "kernel": None})
    pass_s = res["dev_s"] / max(1, res["gates"])
    out["whole_pass"] = {"achieved": bytes_pass / pass_s / 1e9, "frac": bytes_pass / pass_s / 1e9 / hbm,
                         "basis": "same bytes / whole gate-pass device time"}
    out["dense_equivalent"] = {"achieved": 32.0 * (1 << wl["n"]) / pass_s / 1e9,
                               "basis": "32 B per amplitude update (SURVEY.md 8(d), not judged)"}
    # The fused in-slice gate kernel (north_star: ">= 50% of the HBM roofline
    # for fused in-slice gates"): the one stage that streams the dense planes
    # -- per amplitude it reads the old re/im (16 B; flagged zero tiles are
    # not read, so this basis is an upper bound on its reads) and writes the
    # new re/im (16 B), two symbols (8 B) and two flag bytes (2 B).
    gk = next((k for k in kprof if k["kernel"] == "enc_gate_lattice"), None)
    if gk and res["pgates"]:
        t_g = gk["ms"] * 1e-3 / res["pgates"]
        gbytes = 42.0 * (1 << wl["n"]) / max(1, world)
        out["gate_kernel"] = {"kernel": "enc_gate_lattice", "s_per_pass": t_g, "achieved": gbytes / t_g / 1e9,
                              "frac": gbytes / t_g / 1e9 / hbm,
                              "basis": "42 B per amplitude (16 read + 16 + 8 + 2 written); ncu DRAM of the same "
                                       "launch: profiles/r02_random30_pass_dram.json"}
    out["kernel_shares"] = kprof[:10]
    out["kernel_ms_total"] = sum(k["ms"] for k in kprof)
    out["chain"] = res.get("chain")
    # whole-pass DRAM traffic of the same workload from an ncu capture
    # (profiles/r02_<workload>_pass_dram.json, tools/pass_dram.py)
    out["traffic"] = None
    tf = os.path.join(ROOT, "profiles", f"r02_{wl['name']}_pass_dram.json")
    if os.path.exists(tf):
        with open(tf) as f:
            d = json.load(f)
        out["traffic"] = d.get("dram_bytes_per_pass")
        out["traffic_source"] = os.path.relpath(tf, ROOT)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="random30")
    ap.add_argument("--eb", type=float, default=None)
    ap.add_argument("--parity", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--cpu-budget", type=float, default=240.0)
    ap.add_argument("--no-accuracy", action="store_true")
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
    wl = workload(args.workload, extra, args.eb)
    hbm, peak_kind = measured_peaks()
    config = {"workload": wl["name"], "detail": wl["desc"], "n_qubits": wl["n"], "slice_bits": wl["s"],
              "error_bound": wl["eb"], "mode": "absolute", "quant_code_bits": 16, "predictor": "previous",
              "step": f"{wl['per']} gate pass(es) over all 2^n amplitudes",
              "l2": "flushed between timed steps (256 MiB write)",
              "norm": "every gate" if wl["norm_every"] else "off",
              "weak_scaling": "n = base qubits + log2(n_gpus): the slices (and work) per GPU are fixed"}
    metric = "amplitude-gate updates/s incl. (de)compression"

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_replay(wl, args.warmup + args.steps, budget_s=args.cpu_budget)
        line = {"metric": metric, "value": r["value"], "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / max(1, r["gates"]) * wl["per"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded circuit)", "config": config, "impl": "reference",
                "cpu_baseline": {"value": r["value"], "unit": "updates/s", "cores": r["cores"], "kind": r["kind"],
                                 "sample": f"{r['gates']} gate passes of {wl['name']} after its setup "
                                           f"({r['seconds']:.1f} s; setup {r['setup_seconds']:.1f} s untimed)"},
                "e2e": {"value": r["value"], "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    res = run_ours(args, wl, rank, world, dist)
    dev_s, wall, e2e_t = res["dev_s"], res["wall"], res["e2e_t"]
    if dist:
        import torch
        t = torch.tensor([dev_s, wall, e2e_t], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, wall, e2e_t = t.tolist()
    N = 1 << wl["n"]
    # N = 1: device time of the gate passes; N > 1: the barrier-synchronised
    # host wall time (includes the exchange and the norm all-gather)
    t_value = dev_s if world == 1 else wall
    value = N * res["gates"] / t_value
    if rank != 0:
        dist.destroy_process_group() if dist else None
        return
    m = res["m_t"]
    roof = roofline(res, wl, hbm, peak_kind, world)
    cpu, parity = None, None
    do_parity = args.parity == "on" or (args.parity == "auto" and wl["name"] in ("random30", "grover20", "qft16"))
    if world == 1:
        try:
            if do_parity:
                r = cpu_replay(wl, args.warmup + args.steps)
                parity = {"blocks_sha_equal": r["sha"] == res["sha"], "gates": len(wl["setup"]) + r["gates"],
                          "sha256": res["sha"], "reference_sha256": r["sha"], "reference": r["kind"]}
            else:
                r = cpu_replay(wl, args.warmup + args.steps, budget_s=20.0)
            cpu = {"value": r["value"], "unit": "updates/s", "cores": r["cores"], "kind": r["kind"],
                   "sample": f"{r['gates']} gate passes of {wl['name']} after its setup, the same gates as the "
                             f"warm-up + timed window ({r['seconds']:.1f} s)"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}
    line = {"metric": metric, "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_value / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded circuit; no dataset)",
            "config": config, "clocks": res["clocks"], "gpu_launches": int(res["launches"]),
            "e2e": {"value": N * res["gates"] / e2e_t, "unit": "updates/s", "h2d_bytes_per_step": res["h2d"],
                    "d2h_bytes_per_step": res["d2h"],
                    "note": "h2d = the step's action array (it reaches the device as kernel parameters); "
                            "d2h = run metrics + per-slice norms every step, plus the whole compressed state "
                            "(QCB1 blocks) after the last step, averaged over the K steps"},
            "roofline": roof, "cpu_baseline": cpu, "parity": parity,
            "compression": {"min_ratio": m.min_compression_ratio, "mean_ratio": m.mean_compression_ratio,
                            "compressed_bytes": m.current_compressed_bytes, "index_bytes": m.index_bytes,
                            "index_frac": m.index_bytes / max(1, m.current_compressed_bytes),
                            "dense_bytes": m.dense_bytes, "fallback_planes": m.fallback_planes},
            "device_memory": res["mem"],
            "accuracy": res["accuracy"],
            "wall_ms_per_step": 1e3 * wall / args.steps, "device_ms_per_step": 1e3 * dev_s / args.steps,
            "device_ms_steps": res["step_ms"]}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
