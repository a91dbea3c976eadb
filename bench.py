"""Benchmark: fine-grid DoF updates/s per adaFACx cycle (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload config5|config3|config2|config1|config4|...-small]

A step is one additive cycle (ReferenceEngine.advance, solvers.py:334-399)
over the resident level hierarchy.  Default workload: BASELINE configs[4],
the 3D depth-6 adaFACx + BoxMG config the north star's targets (>= 70 % of
HBM on 1 GPU, >= 80 % parallel efficiency at 8) are stated on: 385.8 M fine
DoFs, eps log-uniform per 27^3-cell block, seeded.  configs[1] (2D, 0.53 M
fine DoFs, L2-resident and latency-bound) is ``--workload config2``.

* value      -- N_fine / t_cycle, device time (CUDA events on the engine's
                stream, graph replay); 2D: L2 flushed (256 MiB write) before
                every timed cycle; 3D config5: inputs 60x larger than L2.
* e2e        -- same metric through the drop-in API (GpuEngine, sync="eager"):
                every step uploads tree.u (all levels, pinned host memory),
                runs one cycle, downloads tree.u and the cycle's stats.
* roofline   -- dominant kernel: algorithmic bytes per launch / mean launch
                time (events around each launch, tmg_profile_cycles); also the
                whole-cycle B_alg / t_cycle.
* cpu_baseline -- the CPU oracle port on 1 pinned core on a bounded sample (2D:
                oracle/mg2d.py on the workload itself; config 3: the workload
                itself; config 5: oracle/mg3d.py on the same structure at
                depth 5, 14.2 M fine DoFs -- depth 6 needs ~270 GB in numpy;
                see CPU_SAMPLES_3D).  The line names the sample, the CPU model
                and the host's core count.
* --impl reference -- the reference's CPU algorithm (the oracle port; the
                reference is pure Python and cannot travel to the box), the
                same samples, K + W cycles; `config` is the GPU arm's, the
                sample is named in `cpu_baseline`; rank 0 only.

Multi-GPU (torchrun, one process per GPU): 3D workloads are slab-sharded
over the ranks with NCCL (paper_1903_10367_b200/sharding.py; strong
scaling, max-over-ranks device time); the 2D workloads do not shard
(replicas only): every rank runs an independent replica and
value counts the DoFs of all replicas.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-grid DoF updates/s per adaFACx cycle (all levels); HBM GB/s vs roofline"
UNIT = "DoF-updates/s"
FLUSH_BYTES = 256 << 20


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Dist:
    """One process per GPU.  NCCL when the workload shards (3D), gloo for the 2D
    replicas (whose only collectives are the barrier and the timing max)."""

    def __init__(self, nccl: bool = False, force: bool = False):
        self.ws, self.rank, self.local = dist_env()
        self.nccl = nccl and (self.ws > 1 or force)
        self.td = None
        if self.ws > 1 or (force and nccl):
            import torch
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if self.nccl:
                # NCCL's init banner ("NCCL version ...") goes to stdout; rank 0 prints ONE JSON line
                os.environ.setdefault("NCCL_DEBUG", "WARN")
                torch.cuda.set_device(self.local)
                td.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                td.init_process_group("gloo")
            self.td = td

    def barrier(self):
        if self.td is not None:
            self.td.barrier()

    def max(self, x: float) -> float:
        if self.td is None:
            return x
        import torch
        dev = torch.device("cuda", self.local) if self.nccl else torch.device("cpu")
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.td is not None:
            self.td.destroy_process_group()


# ---------------------------------------------------------------------------
# algorithmic byte model, fp64 = 8 B

def bytes_model(eng, wl):
    """Algorithmic bytes per launch of every cycle kernel, and the whole-cycle B_alg.

    A kernel's algorithmic bytes are the arrays its function must read and
    write once each: no halo re-reads, no cache reuse
    credit.  fp64 = 8 B, flags = 1 B per vertex.
    """
    L, l0 = wl.ltop, eng.lmin
    boxmg = wl.flavor == "boxmg"
    jac = wl.variant == "adafac-jac"
    rhs_levels = set(wl.rhs)
    out = {}
    for l in range(l0, L + 1):
        N = 3**l + 1
        nv, ncell = N * N, (3**l) ** 2
        op = (72 * nv) if (boxmg and l < L) else 8 * ncell       # table rows or per-cell eps
        rd = nv * (8 + 8 + 1) + op + (8 * nv if l in rhs_levels else 0)   # u, diag, flags
        wr = 8 * nv + (16 * nv if l > l0 else 0)                  # g (+ rho, rdof)
        if l < L:
            Nf = 3 ** (l + 1) + 1
            rd += 16 * Nf * Nf                                    # rho, rdof of the finer level
            rd += 8 * ncell                                       # refined-op eps
            if boxmg:
                rd += 200 * nv + (392 * nv if jac else 0)         # P (25), R~ (49) planes
        out[f"k_down_L{l}"] = rd + wr
        up = nv * (8 + 1 + 8 + 8) + (8 * nv if l < L else 0)     # g, flags, u r/w (+ carry)
        if l > l0:
            Nc = 3 ** (l - 1) + 1
            up += 8 * Nc * Nc + (200 * Nc * Nc if boxmg else 0)   # coarse carry (+ P)
        out[f"k_up_L{l}"] = up
        if l < L:
            Nf = 3 ** (l + 1) + 1
            out[f"k_inject_u_L{l}"] = nv * 1 + 8 * nv * 2         # flags, u_f gather, u write
    # the coarse-chain kernel runs levels l0..lc (<= 1024 vertices, <= 6 levels) in one block
    lc = l0
    for l in range(l0, min(L, l0 + 5) + 1):
        if (3**l + 1) ** 2 <= 1024:
            lc = l
    out["k_coarse"] = sum(out[f"k_down_L{l}"] + out[f"k_up_L{l}"] for l in range(l0, lc + 1))
    # whole-cycle B_alg: fine 24 (+8 eps) per DoF; coarse 48 (+ op)
    # + BoxMG P 8*24/9 per DoF of every level above lmin
    counts = eng.level_counts()
    fine_dofs = counts[L][0]
    coarse = sum(counts[l][0] for l in range(l0, L))
    b_alg = fine_dofs * (24 + 8) + coarse * (48 + (72 if boxmg else 8) + (16 if jac else 0))
    if boxmg:
        b_alg += sum(counts[l][0] for l in range(l0 + 1, L + 1)) * 8 * 24 / 9
    out["cycle"] = b_alg
    return out


def bytes_model3(eng, wl):
    """Algorithmic bytes per launch of every 3D cycle kernel and the cycle B_alg.

    Per interior vertex: fp64 = 8 B; the finer level's rho / sm are read once
    (27 fine per coarse vertex); BoxMG P = 124 stored weights per coarse vertex
    (8*124/27 = 36.74 B per fine DoF); Galerkin rows 27*8 B; element
    coefficient 8 B per cell (~ per vertex).
    """
    L, l0 = wl.ltop, eng.lmin
    boxmg = wl.flavor == "boxmg"
    jac = wl.variant == "adafac-jac"
    dofs = {l: (3**l - 1) ** 3 for l in range(l0, L + 1)}
    elem_top = bool(np.any(wl.tree.eps[L] != wl.tree.eps[L].flat[0]))
    out = {}
    for l in range(l0, L + 1):
        n = dofs[l]
        if l == L:
            op = 8 if elem_top else 0
        else:
            op = 216 if boxmg else (8 if elem_top else 0)
        b = n * (8 + op + 8 + (8 if l in wl.rhs else 0)) + (n * 8 if l > l0 else 0)
        if l < L:
            b += dofs[l + 1] * 8 * (2 if jac else 1) + (n * 992 if boxmg else 0)
        out[f"k3_down_L{l}"] = b
        if jac and l > l0:
            out[f"k3_smooth_L{l}"] = 16 * n
        # u r/w + g (+ carry); the finest level keeps g inside its double-buffered u (Engine3::pp)
        up = n * (16 + (8 if l < L or wl.variant == "adafac-pi" else 0) + (8 if l < L else 0))
        if l > l0:
            up += dofs[l - 1] * (8 + (992 if boxmg else 0))
        out[f"k3_up_L{l}"] = up
    lc = l0
    for l in range(l0, min(L, l0 + 2) + 1):
        if (3**l + 1) ** 3 <= 1024:
            lc = l
    # k3_smr (the engine's default for BoxMG but adafac-pi): a level's smoothing and its restriction
    # into the next coarser level run in one kernel named k3_smooth_L{l}; k3_down_L{l-1} reads b_R / b_T
    smr = boxmg and wl.variant != "adafac-pi" and L - 1 > lc
    if smr:  # every level l >= lc + 2 smooths and restricts into l - 1 in k3_smooth_L{l}
        nb = 2 if jac else 1
        for l in range(lc + 2, L + 1):
            nc, nf = dofs[l - 1], dofs[l]
            out[f"k3_smooth_L{l}"] = nf * 8 + nc * 992 + nc * 8 * nb
            out[f"k3_down_L{l - 1}"] -= nf * 8 * nb + nc * 992 - nc * 8 * nb
    out["k3_chain"] = sum(out.get(f"k3_{k}_L{l}", 0) for l in range(l0, lc + 1)
                          for k in ("down", "smooth", "up"))
    fine = dofs[L]
    coarse = sum(dofs[l] for l in range(l0, L))
    b_alg = fine * (24 + (8 if elem_top else 0))
    b_alg += coarse * (48 + (16 if jac else 0) + (216 if boxmg else (8 if elem_top else 0)))
    if boxmg:
        b_alg += sum(dofs[l] for l in range(l0 + 1, L + 1)) * 8 * 124 / 27
    out["cycle"] = b_alg
    return out


# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"tmg_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sms.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, val in zip(names, p[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# 3D CPU samples, largest first: (sample workload, frozen d-linear setup?).  The oracle's eager
# BoxMG setup at depth 5 takes ~7 min on one core, so the depth-5 BoxMG sample starts the oracle in
# its throttled mode (d-linear weights in the same dense 125-weight P tables, rediscretised rows in
# the same 27-point tables) and freezes it there: every cycle runs the same array operations over
# the same bytes as the eager build's cycle; only the weights' values differ.  Depth 6 itself needs
# ~270 GB of host memory in numpy (476 MB at depth 4, x27 per level) and is not runnable.
CPU_SAMPLES_3D = {
    "config3": [("config3-L5", False), ("config3-L4", False)],
    "config5": [("config5-L5b27", True), ("config5-L4", False)],
}


def host_info() -> dict:
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class PinOneCore:
    """taskset -c <first allowed core> for the CPU legs (1 core, pinned)."""

    def __enter__(self):
        self.prev = None
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = min(self.prev)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.core = None
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            try:
                os.sched_setaffinity(0, self.prev)
            except OSError:
                pass


def oracle_engine(wl, frozen_dlinear: bool = False):
    """The CPU oracle engine on the workload's inputs (checker / CPU baseline only)."""
    if wl.dim == 3:
        from oracle import mg3d
        t = mg3d.Tree(wl.tree.depth, wl.tree.lmin)
        t.eps[wl.tree.depth] = wl.tree.eps[wl.tree.depth].copy()
        eng = mg3d.Engine(t, mg3d.Config(variant=wl.variant, flavor=wl.flavor, throttled=frozen_dlinear))
        if frozen_dlinear:
            eng.thr_next = t.lmin - 1  # never upgrade: the BoxMG setup is not part of a cycle
        eng.rhs.update({l: b.copy() for l, b in wl.rhs.items()})
        return eng
    from oracle import mg2d
    t = mg2d.Tree(lmin=wl.tree.lmin, lmax=wl.tree.lmax)
    t.refined = [r.copy() for r in wl.tree.refined]
    t.u = [u.copy() for u in wl.tree.u]
    t.eps = [e.copy() for e in wl.tree.eps]
    eng = mg2d.Engine(t, mg2d.Config(variant=wl.variant, flavor=wl.flavor))
    eng.rhs.update(wl.rhs)
    return eng


def cpu_sample(wl_name: str, cycles: int, budget_s: float):
    """The oracle on the largest sample of the workload whose `cycles` cycles fit `budget_s`
    (estimated from one warm-up cycle): (engine, sample workload, seconds of the warm-up cycle,
    setup seconds, description).  2D workloads run at their real size."""
    from paper_1903_10367_b200 import workloads
    base = wl_name.split("-")[0]
    cands = CPU_SAMPLES_3D.get(wl_name) or ([(wl_name, False)] if base not in CPU_SAMPLES_3D or "-" in wl_name
                                            else CPU_SAMPLES_3D[base])
    for k, (name, frozen) in enumerate(cands):
        wl = workloads.by_name(name)
        t0 = time.perf_counter()
        eng = oracle_engine(wl, frozen)
        setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        eng.advance()  # warm-up (numpy has no JIT; one cycle faults the work arrays in)
        first = time.perf_counter() - t0
        if first * cycles <= budget_s or k == len(cands) - 1:
            if wl.dim == 3:
                what = ("oracle/mg3d.py (3D restatement of the reference's numpy cycle; no 3D reference exists)"
                        + ("; BoxMG tables frozen at their throttled start (d-linear / rediscretised values in "
                           "the same dense P and 27-point tables: same operations and bytes per cycle, no "
                           "7-minute eager setup)" if frozen else ""))
            else:
                what = "oracle/mg2d.py (numpy restatement of treemg, bit-identical iterates)"
            return eng, wl, first, setup, what
        del eng
    raise AssertionError


def run_reference(args, dist: Dist):
    if dist.rank != 0:
        return
    from paper_1903_10367_b200 import workloads
    full = workloads.by_name(args.workload)
    ws = dist_env()[0]
    hi = host_info()
    with PinOneCore() as pin:
        # K steps + W warm-up on one engine; a step = one cycle of the port on the sample
        eng, wl, first, setup, what = cpu_sample(args.workload, args.steps + args.warmup, args.ref_budget)
        for _ in range(args.warmup - 1):  # (cpu_sample ran the first warm-up cycle)
            eng.advance()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            eng.advance()
        total = time.perf_counter() - t0
    n_fine = wl.fine_dofs()
    v = n_fine * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": config_of(full, ws, sharded=full.dim == 3 and (ws > 1 or args.force_shard)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{args.steps} cycles of {wl.name} ({n_fine} fine DoFs; value = fine DoFs "
                                   f"of the sample / s) after {args.warmup} warm-up; {what}; 1 thread pinned "
                                   f"to core {pin.core} of {hi['cpu_model']} ({hi['nproc']} cores); "
                                   f"setup {setup:.1f} s",
                         "sample_workload": wl.name, "sample_n_fine": n_fine, **hi},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(wl, ws: int, sharded: bool = False) -> dict:
    """The `config` object both arms print (identical for the same workload and N)."""
    if sharded:
        from paper_1903_10367_b200 import sharding
        pl = sharding.plan(wl.tree.depth, ws)
        par = (f"slab{ws} (levels {pl.ls}..{wl.ltop} sharded on axis 0, "
               f"levels {wl.tree.lmin}..{pl.ls - 1} replicated)")
        l2 = "inputs larger than L2 (no flush)"
    else:
        par = "replicas" if ws > 1 else "single"
        l2 = f"flushed ({FLUSH_BYTES >> 20} MiB write) before every timed cycle"
    return {"workload": wl.name, "levels": f"{wl.tree.lmin}..{wl.ltop}", "variant": wl.variant,
            "flavor": wl.flavor, "n_fine": wl.fine_dofs(), "parallelism": par, "l2": l2}


def run_ours(args, dist: Dist):
    import torch

    from paper_1903_10367_b200 import GpuEngine, SolverConfig, workloads
    from paper_1903_10367_b200 import build as b

    if dist.rank == 0:
        b.build()
    dist.barrier()
    dev = dist.local if dist.ws > 1 else 0
    torch.cuda.set_device(dev)
    wl = workloads.by_name(args.workload)
    n_fine = wl.fine_dofs()

    # ---- device-resident timing (value) ------------------------------------
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor, fused_cycle=args.fused_cycle), device=dev,
                    sync="lazy")
    eng.rhs.update(wl.rhs)
    eng.advance_many(max(args.warmup, 3))
    launches = eng.launches_per_cycle()
    # level ltop-1's BoxMG weights: dense or row dictionary (kernels3d_dict.cu), as built at setup
    storage = (eng.weight_storage(wl.ltop - 1) if wl.dim == 3 and wl.flavor == "boxmg" and wl.ltop > wl.tree.lmin
               else None)
    updates = eng.advance_many(1)[0].updates  # count_updates (solvers.py:449-459)
    clk = ClockSampler(dev)
    clk.start()
    dist.barrier()
    torch.cuda.synchronize()
    ms = eng.time_cycles(args.steps, flush_bytes=FLUSH_BYTES)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = clk.stop()
    ms_warm = eng.time_cycles(args.steps, flush_bytes=0)
    ms_max = dist.max(ms)
    ms_step = ms_max / args.steps
    value = dist.ws * n_fine / (ms_step * 1e-3)

    # ---- per-kernel times (roofline of the dominant kernel) --------------------
    prof = eng.profile_cycles(max(min(args.steps, 10), 3))
    bm = bytes_model3(eng, wl) if wl.dim == 3 else bytes_model(eng, wl)
    top = max(prof.items(), key=lambda kv: kv[1][0])
    kname, (kms, kcnt) = top
    total_prof = sum(v[0] for v in prof.values())
    peak = None
    peak_src = "fallback 6650 GB/s (B200_PROFILING.md)"
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        peak = 6650.0
    kbytes = bm.get(kname)
    achieved = kbytes / (kms / kcnt * 1e-3) / 1e9 if kbytes else None
    traffic = None
    cycle_traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(args.workload, {})
            traffic = tj.get(kname)
            # the whole cycle's DRAM bytes (ncu, one launch per kernel of this cycle) when every
            # kernel timed here was captured: actual HBM traffic, next to the algorithmic B_alg
            if tj and all(k in tj for k in prof):
                cycle_traffic = float(sum(tj[k] for k in prof))
        except ValueError:
            traffic = None
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                # the same kernel by the DRAM bytes ncu measured for one launch (the plane-run
                # coefficients / dictionaries move less than the algorithmic bytes)
                "traffic_GBps": (traffic / (kms / kcnt * 1e-3) / 1e9) if traffic else None,
                "traffic_frac": (traffic / (kms / kcnt * 1e-3) / 1e9 / peak) if traffic else None,
                "algorithmic_bytes_per_launch": kbytes, "mean_launch_us": 1e3 * kms / kcnt,
                "share_of_cycle": kms / total_prof, "peak_source": peak_src,
                "cycle_B_alg": bm["cycle"],
                "cycle_achieved_GBps": bm["cycle"] / (ms_step * 1e-3) / 1e9,
                "cycle_frac": bm["cycle"] / (ms_step * 1e-3) / 1e9 / peak,
                "cycle_dram_bytes": cycle_traffic,
                "cycle_dram_frac": (cycle_traffic / (ms_step * 1e-3) / 1e9 / peak) if cycle_traffic else None}
    eng.close()

    # ---- time to a 1e-8 residual reduction (north star; bench.py:200 stop rule) ----
    ttt = None
    if not args.no_ttt:
        wl3 = wl if wl.dim == 3 else workloads.by_name(args.workload)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e3 = GpuEngine(wl3.tree, SolverConfig(variant=wl3.variant, flavor=wl3.flavor), device=dev,
                       sync="lazy")
        e3.rhs.update(wl3.rhs)
        e3._flush_rhs()
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t0
        cap, chunk, done, r0, reached = args.ttt_cap, 5, 0, None, None
        t0 = time.perf_counter()
        while done < cap and reached is None:
            hs = e3.advance_many(min(chunk, cap - done))
            for k, h in enumerate(hs):
                if r0 is None:
                    r0 = h.l2h
                if reached is None and h.l2h <= 1e-8 * r0:
                    reached = done + k
            done += len(hs)
        torch.cuda.synchronize()
        t_solve = time.perf_counter() - t0
        ttt = {"target": 1e-8, "reached": reached is not None,
               "cycles": reached if reached is not None else done,
               "final_reduction": hs[-1].l2h / r0 if r0 else None,
               "setup_s": t_setup, "solve_s": t_solve,
               "note": "stats of cycle n are the residual of the iterate it starts from "
                       "(solvers.py:129-135); solve_s includes the cycles run past the target "
                       f"inside the last chunk of {chunk}" if reached is not None else
                       f"not reached within {cap} cycles"}
        e3.close()

    # ---- end to end through the drop-in API -------------------------------------
    wl2 = wl if wl.dim == 3 else workloads.by_name(args.workload)
    tree = wl2.tree
    for l in range(len(tree.u)):  # pinned host memory for tree.u
        pin = torch.empty(tree.u[l].shape, dtype=torch.float64, pin_memory=True).numpy()
        pin[...] = tree.u[l]
        tree.u[l] = pin
    e2 = GpuEngine(tree, SolverConfig(variant=wl2.variant, flavor=wl2.flavor, fused_cycle=args.fused_cycle), device=dev,
                   sync="eager")
    e2.rhs.update(wl2.rhs)
    for _ in range(max(args.warmup, 3)):
        e2.push()
        e2.advance()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2.push()          # H2D: every level of tree.u
        e2.advance()       # one cycle + D2H of every level of tree.u and the stats
    torch.cuda.synchronize()
    t_e2e = dist.max(time.perf_counter() - t0)
    h2d = sum(tree.u[l].nbytes for l in range(e2.lmin - (1 if wl.dim == 2 else 0), e2.ltop + 1))
    d2h = sum(tree.u[l].nbytes for l in range(e2.lmin, e2.ltop + 1)) + 32
    e2e = {"value": dist.ws * n_fine * args.steps / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": 1e3 * t_e2e / args.steps, "api": "GpuEngine(sync='eager').push()+advance()"}
    e2.close()

    # ---- CPU baseline (rank 0 at N=1 only) ---------------------------------------
    cpu = None
    if dist.rank == 0 and dist.ws == 1 and not args.no_cpu:
        hi = host_info()
        with PinOneCore() as pin:
            ceng, swl, first, setup, what = cpu_sample(args.workload, 2, 2 * args.cpu_budget)
            done, t0 = 0, time.perf_counter()
            while done < 400:
                ceng.advance()
                done += 1
                if time.perf_counter() - t0 + first > args.cpu_budget:
                    break
            dt = (time.perf_counter() - t0) / done
        cpu = {"value": swl.fine_dofs() / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{done} cycles of {swl.name} ({swl.fine_dofs()} fine DoFs; value = fine DoFs of the "
                         f"sample / s) after 1 warm-up, {dt * done:.1f} s; {what}; 1 thread pinned to core "
                         f"{pin.core} of {hi['cpu_model']} ({hi['nproc']} cores); setup {setup:.1f} s",
               "sample_workload": swl.name, "sample_n_fine": swl.fine_dofs(), **hi}
        del ceng

    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": config_of(wl, dist.ws),
            "detail": {"ms_per_step_l2_warm": ms_warm / args.steps,
                       "total_updates_per_s": dist.ws * updates / (ms_step * 1e-3),
                       "weight_storage": storage},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "time_to_1e-8": ttt,
            "gpu_launches": launches * args.steps,
            "kernel_ms": {k: round(v[0] / v[1], 6) for k, v in prof.items()},
        }
        print(json.dumps(line), flush=True)


def run_sharded(args, dist: Dist):
    """3D workload slab-sharded over the ranks (strong scaling)."""
    import torch

    from paper_1903_10367_b200 import GpuEngine, SolverConfig, sharding, workloads
    from paper_1903_10367_b200 import build as b

    if dist.rank == 0:
        b.build()
    dist.barrier()
    dev = dist.local
    torch.cuda.set_device(dev)
    wl = workloads.by_name(args.workload)
    n_fine = wl.fine_dofs()
    pl = sharding.plan(wl.tree.depth, dist.ws)
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor, fused_cycle=args.fused_cycle), device=dev,
                    sync="lazy")
    eng.rhs.update(wl.rhs)
    eng._flush_rhs()
    sh = sharding.GpuShard(eng, pl, dist.rank)
    se = sharding.ShardedEngine3([sh], sharding.DistTransport(pl, dist.rank), wl.variant,
                                 split=True if args.force_split else None)
    st = sh.stream
    with torch.cuda.stream(st):
        se.cycle()  # eager once (NCCL channels, lazily allocated buffers), then the captured graphs
        torch.cuda.synchronize()
        graphed = (not args.no_shard_graph) and se.capture()
        step = se.replay if graphed else se.cycle
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        clk = ClockSampler(dev)
        clk.start()
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        dist.barrier()
        clocks = clk.stop()
        ms = e0.elapsed_time(e1)
        hist = sh.history(1)
        # e2e: every step uploads this rank's owned u planes (all sharded levels) from
        # pinned host memory, runs one cycle and reads them back with the stats
        # (the finest level's u is double buffered: ask for its current view every time)
        levels = range(pl.ls, wl.ltop + 1)
        own = {l: slice(*pl.rng(l, dist.rank)) for l in levels}
        host = {l: torch.empty_like(sh.view(0, l)[own[l]], device="cpu").pin_memory() for l in levels}
        for l in levels:
            host[l].copy_(sh.view(0, l)[own[l]])
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for l in levels:
                sh.view(0, l)[own[l]].copy_(host[l], non_blocking=True)
            step()
            for l in levels:
                host[l].copy_(sh.view(0, l)[own[l]], non_blocking=True)
            sh.history(1)
        torch.cuda.synchronize()
        t_e2e = dist.max(time.perf_counter() - t0)
    ms_max = dist.max(ms)
    ms_step = ms_max / args.steps
    value = n_fine / (ms_step * 1e-3)
    bm = bytes_model3(eng, wl)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    per_gpu = bm["cycle"] / dist.ws / (ms_step * 1e-3) / 1e9
    jac = wl.variant == "adafac-jac"
    lcs = min(2, pl.ls - 1)
    launches = (wl.ltop - pl.ls + 1) * (3 if jac else 2) + 1 + 2 * (pl.ls - 1 - lcs) * (1 + jac) + 1 \
        + (pl.ls - wl.tree.lmin)
    hb = sum(host[l].numel() * 8 for l in host)
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": config_of(wl, dist.ws, sharded=True),
            "detail": {"l2h_last": hist[0].l2h, "cuda_graph": bool(graphed)},
            "roofline": {"bound": "hbm", "kernel": "cycle (per GPU)", "achieved": per_gpu, "peak": peak,
                         "unit": "GB/s", "frac": per_gpu / peak, "traffic": None,
                         "cycle_B_alg": bm["cycle"]},
            "cpu_baseline": None,
            "e2e": {"value": n_fine * args.steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": hb,
                    "d2h_bytes_per_step": hb + 32, "ms_per_step": 1e3 * t_e2e / args.steps,
                    "api": "ShardedEngine3.cycle() with owned u planes copied in/out per step (rank 0's bytes)"},
            "clocks": clocks, "gpu_launches": launches * args.steps,
        }
        print(json.dumps(line), flush=True)
    # release every torch object tied to the engine's stream before the engine (and its
    # stream) goes away: pinned blocks record events on the streams that used them
    del host
    se._graphs = None
    sh.close()
    torch.cuda.synchronize()
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="config5")
    ap.add_argument("--cpu-budget", type=float, default=25.0,
                    help="seconds of timed CPU work in the cpu_baseline leg")
    ap.add_argument("--ref-budget", type=float, default=480.0,
                    help="--impl reference: largest sample whose K + W cycles fit this many seconds")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-1e-8 run")
    ap.add_argument("--fused-cycle", action="store_true",
                    help="2D: the whole cycle as one persistent cooperative launch (k_cycle)")
    ap.add_argument("--ttt-cap", type=int, default=200, help="cycle cap of the time-to-1e-8 run")
    ap.add_argument("--no-shard-graph", action="store_true",
                    help="sharded path: enqueue every phase and exchange from the host instead of replaying "
                         "the captured CUDA graphs")
    ap.add_argument("--force-split", action="store_true",
                    help="sharded path at one rank: run the split (edge planes / exchange / inner planes) "
                         "schedule that ranks with neighbours run")
    ap.add_argument("--force-shard", action="store_true",
                    help="3D: run the sharded (NCCL) path even on one rank (testing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    three_d = args.workload.startswith(("config3", "config5"))
    ws = dist_env()[0]
    dist = Dist(nccl=three_d and args.impl == "ours" and (ws > 1 or args.force_shard),
                force=args.force_shard)
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        elif three_d and (dist.ws > 1 or args.force_shard):
            run_sharded(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
