#!/usr/bin/env python
"""Benchmark of the B200 SMC-over-PCFG hot path (BASELINE.json metric:
particle-steps/s and SMC sweeps/s; resample HBM GB/s vs peak).

Default workload (BASELINE.json configs[1], the config the metric is quoted
on): CRBD on the synthetic 90-tip tree `tree90`, 10^6 particles per GPU, one
step = one complete SMC sweep (178 epochs: propagate + resample each).  Other
workloads (--workload): clads2 (configs[2]), seir (configs[3]), resample
(configs[4], one resampling step of 2^N particles x 64 B).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL); rank 0 prints one
JSON line.  `--impl reference` times the CPU oracle (the tier's reference arm)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402

WORKLOADS = {
    "crbd": dict(config=1, model="crbd", tree="tree90", n=1_000_000, oracle_n=60000,
                 desc="CRBD birth-death, synthetic 90-tip Yule tree (tree90), priors Gamma(1,1)/Gamma(1,0.5)"),
    "crbd_vr": dict(config=None, model="crbd", tree="tree90", n=1_000_000, analytic=True, ess="1/2",
                    desc="CRBD on tree90 with the Sec. 5.3 variance reduction: 2E(t) per hidden event "
                         "instead of a simulated side tree (DESIGN R-20) and ESS-triggered resampling "
                         "at ESS < N/2 (R-19)"),
    "clads2": dict(config=2, model="clads2", tree="tree90", n=1_000_000, oracle_n=40000,
                   desc="ClaDS2 lineage-specific-rate birth-death on tree90"),
    "seir": dict(config=3, model="seir", n=1_000_000, oracle_n=30000,
                 desc="vector-borne-disease SEIR on the synthetic 182-day case series seir182"),
    "geometric": dict(config=None, model="geometric", n=1_000_000,
                      desc="weighted geometric, Fig. 2 (p=0.5, w=1.5): particles reach b_stop at "
                           "different epochs (universal control flow, SURVEY f4)"),
    "ssm": dict(config=None, model="ssm", n=1_000_000,
                desc="linear-Gaussian state-space model, Eq. (2), 50 synthetic observations (SURVEY f4)"),
    "fig3": dict(config=None, model="fig3", n=1_000_000,
                 desc="the PCFG of Fig. 3(a): five blocks with jumps, a self-loop and checkpoints; "
                      "particles at different blocks within an epoch and stopping at different "
                      "epochs (SURVEY f4, DESIGN R-23)"),
    "stackf": dict(config=None, model="stackf", n=1_000_000, cap=1024,
                   desc="the recursive function of Fig. 5(c) compiled with a 1 KiB PSTATE byte stack "
                        "(48-byte frames) and a stack pointer; resampling copies only the stack below "
                        "the pointer (SURVEY f2, DESIGN R-24)"),
    "resample": dict(config=4, model="resample", n=1 << 26,
                     desc="resampling step alone: LSE max + u128 scan + systematic ancestors + 64-B gather"),
}
L2_BYTES = 126 * 2 ** 20


def traffic(key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(key)
    except Exception:
        return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, path):
        self.path, self.proc = path, None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader",
                                          "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, dev=0):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        try:
            text = open(self.path).read().strip()
            if not text:
                # timed region shorter than the sampling interval: one query right after it
                q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
                text = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"],
                                      capture_output=True, text=True).stdout.strip()
                out["note"] = "sampled once right after the timed region (region < 100 ms)"
            rows = [r.split(", ") for r in text.splitlines()]
            rows = [r for r in rows if r and r[0].strip() == str(dev)]
            sm = [float(r[1].split()[0]) for r in rows]
            mx = [float(r[2].split()[0]) for r in rows]
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = set()
            for r in rows:
                for k, nm in enumerate(names):
                    if r[5 + k].strip() == "Active":
                        reasons.add(nm)
            out.update(sm_mhz=float(np.median(sm)) if sm else None,
                       sm_max_mhz=max(mx) if mx else None, reasons=sorted(reasons), samples=len(sm))
        except Exception as e:       # pragma: no cover
            out["error"] = str(e)
        return out


# ----------------------------------------------------------------------------- dist
def dist_init(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={world}")
    return world, rank, local


RNG = {"lineage": True, "sequential": False}


def model_for(smc, wl, rng="lineage", inplace=False):
    fl = smc.FLAG_INPLACE if inplace else 0
    if wl["model"] == "crbd":
        return smc.Model.crbd(inputs.tree(wl["tree"]), inputs.CRBD_PARAMS, lineage=RNG[rng],
                              analytic=wl.get("analytic", False), flags=fl)
    if wl["model"] == "clads2":
        return smc.Model.clads2(inputs.tree(wl["tree"]), inputs.CLADS2_PARAMS, lineage=RNG[rng], flags=fl)
    if wl["model"] == "seir":
        return smc.Model.seir(inputs.seir_series(), flags=fl)
    if wl["model"] == "geometric":
        return smc.Model.geometric(*inputs.GEOMETRIC_PARAMS, flags=fl)
    if wl["model"] == "ssm":
        return smc.Model.ssm(inputs.ssm_series(50), inputs.SSM_PARAMS, flags=fl)
    if wl["model"] == "fig3":
        return smc.Model.fig3(*inputs.FIG3_PARAMS, flags=fl)
    if wl["model"] == "stackf":
        return smc.Model.stackf(inputs.stackf_series(), inputs.STACKF_PARAMS[:3] + [float(wl["cap"])], flags=fl)
    raise ValueError(wl)


# ----------------------------------------------------------------------------- reference arm / CPU baseline
def oracle_sweep_rate(wl, budget_s=15.0, n_cap=None):
    """Time the oracle (single thread, as it stands) on a bounded sample: one
    sweep of the same model with n particles, n chosen so the run takes
    roughly budget_s.  Returns (particle-steps/s, sample description, seconds)."""
    import oracle
    lin = getattr(oracle_sweep_rate, "rng", "lineage") == "lineage"
    kind = {"crbd": (oracle.CRBD_AE if wl.get("analytic") else oracle.CRBD_LR if lin else oracle.CRBD),
            "clads2": oracle.CLADS2_LR if lin else oracle.CLADS2, "seir": oracle.SEIR,
            "geometric": oracle.GEOMETRIC, "ssm": oracle.SSM, "fig3": oracle.FIG3,
            "stackf": oracle.STACKF}[wl["model"]]
    if wl["model"] in ("crbd", "clads2"):
        data = oracle.tree_blob(inputs.tree(wl["tree"]))
        params = inputs.CRBD_PARAMS if wl["model"] == "crbd" else inputs.CLADS2_PARAMS
    elif wl["model"] == "geometric":
        data, params = None, inputs.GEOMETRIC_PARAMS
    elif wl["model"] == "fig3":
        data, params = None, inputs.FIG3_PARAMS
    elif wl["model"] == "stackf":
        data, params = inputs.stackf_series(), inputs.STACKF_PARAMS[:3] + [float(wl["cap"])]
    elif wl["model"] == "ssm":
        data, params = inputs.ssm_series(50), inputs.SSM_PARAMS
    else:
        data, params = inputs.seir_series(), None
    n = 1000
    ea, eb = (int(x) for x in getattr(oracle_sweep_rate, "ess", "1/1").split("/"))
    if budget_s > 0 and wl.get("oracle_n"):
        # a fixed sample per workload (~5-10 s on one core), so the cpu_baseline
        # leg and the reference arm time the same computation: per-particle-step
        # cost depends on the particle system, which depends on N and the seed
        n = wl["oracle_n"]
    elif budget_s > 0:
        t0 = time.perf_counter()
        s = oracle.Smc(kind, data, params, n, 12345)
        s.set_ess(ea, eb)
        s.set_inplace(getattr(oracle_sweep_rate, "inplace", False))
        s.run()
        dt = time.perf_counter() - t0
        n = max(1000, int(n * budget_s / max(dt, 1e-3)))
    if n_cap:
        n = min(n, n_cap) if budget_s > 0 else n_cap
    t0 = time.perf_counter()
    s = oracle.Smc(kind, data, params, n, 12345)
    s.set_ess(ea, eb)
    s.set_inplace(getattr(oracle_sweep_rate, "inplace", False))
    s.run()
    dt = time.perf_counter() - t0
    st = s.stats()
    return st["alive_particle_steps"] / dt, f"one full sweep, N={n} particles, seed 12345", dt, st


def oracle_draws_per_step(wl, n=20000, seed=12345):
    """Algorithmic propagation work: uniforms drawn per
    particle-step as counted by the oracle (one full sweep of n particles; the
    GPU's own counter also holds speculative side-tree nodes of the cooperative
    kernel, so the roofline uses this schedule-independent count)."""
    _, sample, _, st = oracle_sweep_rate(wl, n_cap=n, budget_s=0.0)
    return st["draws"] / max(st["alive_particle_steps"], 1), sample


def oracle_resample_rate(n_full, budget_s=10.0):
    import oracle
    n = 1 << 20
    lw = inputs.resample_lw(n, 1.0, 0.0, seed=4)
    st = inputs.state_bytes(n, 64, seed=5)
    t0 = time.perf_counter()
    r = oracle.resample(lw, 4, 0)
    oracle.gather(st, r["anc"])
    dt = time.perf_counter() - t0
    D = len(np.unique(r["anc"]))
    bytes_alg = n * 20 + 64 * (D + n)
    return bytes_alg / dt / 1e9, n / dt, f"one resampling step of N=2^20 x 64 B (sigma=1)", dt


def run_reference(args, wl):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ncores = 1
    if wl["model"] == "resample":
        vals = []
        for _ in range(args.warmup):
            oracle_resample_rate(wl["n"])
        for _ in range(args.steps):
            gbs, pps, sample, dt = oracle_resample_rate(wl["n"])
            vals.append(gbs)
        v = float(np.mean(vals))
        line = dict(metric="resample effective GB/s", value=v, unit="GB/s", impl="reference")
    else:
        vals = []
        for _ in range(args.warmup):
            oracle_sweep_rate(wl, budget_s=0.0, n_cap=1000)
        for _ in range(args.steps):
            pss, sample, dt, st = oracle_sweep_rate(wl, budget_s=8.0)
            vals.append(pss)
        v = float(np.mean(vals))
        line = dict(metric="particle-steps/s", value=v, unit="particle-steps/s", impl="reference")
    line.update(n_gpus=world, steps=args.steps, warmup=args.warmup, higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=args.workload, desc=wl["desc"], rng=args.rng, ess_threshold=args.ess),
                cpu_baseline=dict(value=v, unit=line["unit"], cores=ncores, kind="oracle",
                                  sample=sample),
                e2e=dict(value=v, unit=line["unit"], h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def bench_sweeps(args, wl, smc, torch, world, rank):
    N = args.n or wl["n"]
    model = model_for(smc, wl, args.rng, args.inplace)
    stream = torch.cuda.current_stream()
    if world == 1:
        h = smc.Smc(model, N, seed=1, stream=stream)
    else:
        from paper_2112_00364_b200 import dist as sdist
        h = sdist.sharded(model, N, seed=1, stream=stream)
    ea, eb = (int(x) for x in args.ess.split("/"))
    h.set_ess_threshold(ea, eb)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")
    # warm-up sweeps (untimed; the first also captures the whole-run CUDA graph)
    for w in range(args.warmup):
        h.reset(1000 + w)
        h.run()
    # timed: K sweeps (one graph launch each), per-sweep CUDA events on the
    # handle's stream, L2 flushed between sweeps (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    steps_done = 0
    draws = 0
    guard = 0
    alive_steps = 0
    logzs = []
    barrier(torch, world)
    torch.cuda.synchronize()
    with Clocks(os.path.join(args.out, f"clocks_rank{rank}.csv")) as clk:
        for k in range(args.steps):
            flush.zero_()
            h.reset(1 + k)        # re-initialise particles (pc = b0), new seed; not timed
            ev[k][0].record(stream)
            h.run()
            ev[k][1].record(stream)
            st = h.stats()
            draws += st["draws"]
            guard += st["guard_kills"]
            alive_steps += st["alive_particle_steps"]
            steps_done += st["epochs"]
            logzs.append(h.log_z)
        torch.cuda.synchronize()
    barrier(torch, world)
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    t_ms = max_over_ranks(torch, world, t_ms)
    # whole-job particle steps (all ranks)
    tot_steps = sum_over_ranks(torch, world, alive_steps)
    value = tot_steps / (t_ms / 1e3)
    sweeps_per_s = args.steps / (t_ms / 1e3)
    # phase split, measured live with CUDA events around each epoch's kernels
    # (host-stepped sweeps with the same seeds; not part of the headline time)
    h.set_timing(True)
    prop_ms = res_ms = 0.0
    res_bytes = 0
    n_resamples = 0
    stack_planes = 0
    for k in range(args.steps):
        h.reset(1 + k)
        h.run()
        st = h.stats()
        prop_ms += st["ms_propagate"]
        res_ms += st["ms_resample"]
        sb = st["state_bytes"]
        n_loc = st["n_local"]
        # algorithmic resample bytes of the sweep: per resample N*20 + S*(D + N),
        # plus the final epoch's reduce (8 B/particle)
        if st["deferred_gather"]:
            # the resampling step writes ancestors only (DESIGN 7.7): two lw
            # passes + the anc write; the state copy happens inside the next
            # propagation and is not counted here
            res_bytes += st["resamples"] * n_loc * 20 + 8 * n_loc
        elif st["stack_planes"]:
            # stack models: the gathers copy only the planes below the stack pointer
            res_bytes += st["resamples"] * n_loc * 20 + 16 * st["stack_planes"] * 2 + 8 * n_loc
        else:
            res_bytes += st["resamples"] * n_loc * (20 + sb) + sb * st["distinct"] + 8 * n_loc
        n_resamples += st["resamples"]
        stack_planes += st["stack_planes"]
    h.set_timing(False)
    # graph body = 2 epochs x (propagate + resampling) + set_condition; the
    # resampling step is one cooperative launch when the handle uses the fused
    # kernel (resample_grid() > 0), else reduce, anc_gather, finalize
    fused = world == 1 and h.resample_grid() > 0
    per_epoch = 2 if fused else 4
    E = steps_done // args.steps
    launches = args.steps * (2 * per_epoch + 1) * ((E + 1) // 2)
    return dict(h=h, model=model, N=N, t_ms=t_ms, value=value, sweeps=sweeps_per_s, prop_ms=prop_ms,
                res_bytes=res_bytes, resamples_per_sweep=n_resamples / args.steps,
                res_ms=res_ms, draws=draws, guard=guard, alive_steps=alive_steps, epochs=steps_done,
                stack_planes=stack_planes, state_bytes=st["state_bytes"],
                deferred=bool(st["deferred_gather"]),
                launches=launches, fused=fused, clocks=clk.summary(torch.cuda.current_device()),
                logz=float(np.mean(logzs)))


def e2e_sweeps(args, wl, smc, torch, h, model, k_steps, world):
    """End to end through the public API: every step uploads the step's input
    (the model data: tree table / case series, from pinned host memory) into
    the handle, re-initialises it with the step's seed, runs the sweep and
    reads back log Z and the final log-weights (D2H).  Host wall clock around
    the whole step, max over ranks."""
    data = (torch.from_numpy(model.data.copy()).pin_memory().numpy() if model.data.size
            else model.data)
    ts = []
    for k in range(k_steps + 1):
        barrier(torch, world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if data.size:
            h.set_data(data)
        h.reset(500 + k)
        h.run()
        lz = h.log_z
        lw = h.log_weights()
        torch.cuda.synchronize()
        if k:                         # first is warm-up
            ts.append(time.perf_counter() - t0)
    t = max_over_ranks(torch, world, float(np.mean(ts)))
    return dict(t=t, h2d=data.nbytes, d2h=lw.nbytes + 8, logz=lz)


def bench_resample_sharded(args, wl, smc, torch, world, rank):
    """configs[4] at N GPUs: each rank holds n particles; one global resampling
    step of the handles' own buffers per timed step (all-gathers over NCCL,
    migration by peer stores)."""
    from paper_2112_00364_b200 import dist as sdist
    n = args.n or wl["n"]
    S = 64
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(4 + 1000 * rank)
    lw = torch.randn(n, generator=g, device=dev, dtype=torch.float64) * args.sigma
    st = torch.randint(0, 2 ** 31 - 1, (S // 4 * n,), generator=g, device=dev, dtype=torch.int32)
    stream = torch.cuda.current_stream()
    h = sdist.sharded(smc.Model.resample_bench(S), n, seed=4, stream=stream)
    h.load(lw, st)
    del st
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    for w in range(args.warmup):
        h.resample_step(w)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier(torch, world)
    dist_d = 0
    with Clocks(os.path.join(args.out, f"clocks_rank{rank}.csv")) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            h.resample_step(args.warmup + k)
            ev[k][1].record(stream)
            dist_d += h.distinct()
        torch.cuda.synchronize()
    barrier(torch, world)
    t_ms = max_over_ranks(torch, world, sum(a.elapsed_time(b) for a, b in ev))
    D = sum_over_ranks(torch, world, dist_d) / args.steps
    alg = world * n * 20 + S * (D + world * n)
    return dict(n=n, t_ms=t_ms / args.steps, alg_bytes=alg, D=D, clocks=clk.summary(torch.cuda.current_device()))


def bench_resample(args, wl, smc, torch):
    n = args.n or wl["n"]
    S = 64
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(4)
    lw = torch.randn(n, generator=g, device=dev, dtype=torch.float64) * args.sigma
    st_in = torch.randint(0, 2 ** 31 - 1, (S // 4 * n,), generator=g, device=dev, dtype=torch.int32)
    st_out = torch.empty_like(st_in)
    anc = torch.empty(n, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    r = smc.Resampler(n, S, seed=4, stream=stream, inplace=args.inplace)
    if args.inplace:
        del st_out
        st_out = None                 # R-21: the state is updated in place
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    for w in range(args.warmup):
        r.device(lw, st_in, st_out, anc, epoch=w)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with Clocks(os.path.join(args.out, "clocks_rank0.csv")) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            r.device(lw, st_in, st_out, anc, epoch=k)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]
    D = r.distinct()
    alg = n * 20 + S * (D + n)
    # per-kernel split (CUDA events around each kernel; separate, untimed passes)
    r.set_timing(True)
    for k in range(args.steps):
        flush.zero_()
        r.device(lw, st_in, st_out, anc, epoch=k)
    torch.cuda.synchronize()
    ms_k = [v / args.steps for v in r.stats()["ms_kernel"]]
    r.set_timing(False)
    return dict(r=r, n=n, t_ms=float(np.mean(times)), alg_bytes=alg, D=D, ms_kernel=ms_k,
                fused=r.resample_grid() > 0,
                clocks=clk.summary(torch.cuda.current_device()))


def resample_line(args, smc, torch, world, rank, pk, pk_kind, n, sigma, inplace=False, steps=None,
                  warmup=None):
    """configs[4] on one GPU: one resampling step of n particles x 64 B."""
    hbm_peak = pk["hbm_gbs"]
    sub_args = argparse.Namespace(**vars(args))
    sub_args.n, sub_args.sigma, sub_args.inplace = n, sigma, inplace
    sub_args.steps = steps or max(3, min(args.steps, 10))
    sub_args.warmup = warmup or max(3, args.warmup)
    args = sub_args
    r = bench_resample(args, WORKLOADS["resample"], smc, torch)
    achieved = r["alg_bytes"] / (r["t_ms"] * 1e-3) / 1e9
    n, D = r["n"], r["D"]
    g_bytes = n * 12 + 64 * (D + n)          # anc_gather: lw read, anc write, states
    kname = "anc_gather_kernel (ancestors + fused gather)"
    fused = r["fused"]
    if fused:                                # N fits the co-resident grid: one launch
        kname = "resample_fused_kernel (quantise + exact sum, grid barrier, ancestors + gather, log Z)"
    metric = "resample effective HBM GB/s (B_alg = N*20 + 64*(D+N))"
    if args.inplace:
        # offspring: lw 8 + O_k 4; permute: O_k 4 + survivors' anc 4 D + hole/extra
        # lists 8 H; fill: lists 8 H + anc 4 H + state 2*64 H   (H = N - D holes)
        H = n - D
        g_bytes = n * 16 + 4 * D + H * (20 + 2 * 64)
        kname = "in-place chain (offspring + permute + fill_holes kernels, R-21)"
        metric = ("resample effective GB/s, in place (B_alg of the out-of-place step, "
                  "N*20 + 64*(D+N), per unit time)")
    g_ms = r["ms_kernel"][2]
    g_ach = g_bytes / (g_ms * 1e-3) / 1e9
    tr = None if args.inplace else traffic(f"resample:{n}:anc_gather")
    line = dict(metric=metric, value=achieved,
                unit="GB/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
                ms_per_step=r["t_ms"], higher_is_better=True, scaling="weak", vs_baseline=None,
                dtype="f64/u128", data="synthetic",
                config=dict(workload="resample", desc=WORKLOADS["resample"]["desc"], n_per_gpu=r["n"],
                            state_bytes=64, sigma=args.sigma, l2="flushed between steps",
                            inplace=args.inplace),
                roofline=dict(bound="hbm", kernel=kname,
                              achieved=g_ach, peak=hbm_peak, unit="GB/s", frac=g_ach / hbm_peak,
                              traffic=(tr["bytes"] if tr else None),
                              algorithmic_bytes=g_bytes, ms=g_ms, peak_source=pk_kind),
                chain_roofline=dict(bound="hbm", achieved=achieved, peak=hbm_peak, unit="GB/s",
                                    frac=achieved / hbm_peak, algorithmic_bytes=r["alg_bytes"],
                                    note=("max + resample_fused" if fused else
                                          "max + reduce + anc_gather + finalize") +
                                         "; B_alg excludes the standalone max pass (8 B/particle)"),
                kernel_ms=(dict(max=r["ms_kernel"][0], resample_fused=r["ms_kernel"][2]) if fused else
                           dict(zip(["max", "reduce", "inplace_chain" if args.inplace else "anc_gather",
                                     "finalize"], r["ms_kernel"]))),
                distinct_ancestors=D,
                gpu_launches=(7 if args.inplace else 3 if fused else 5) * args.steps, clocks=r["clocks"])
    del r
    return line


def barrier(torch, world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(torch, world, v):
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(torch, world, v):
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def run_ours(args, wl):
    import torch
    world, rank, local = dist_init(args.gpus)
    torch.cuda.set_device(local)
    # all work (ours and the timing events) on one dedicated stream
    torch.cuda.set_stream(torch.cuda.Stream())
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2112_00364_b200 as smc
    pk, pk_kind = peaks()
    hbm_peak = pk["hbm_gbs"]
    if wl["model"] == "resample" and world > 1:
        r = bench_resample_sharded(args, wl, smc, torch, world, rank)
        achieved = r["alg_bytes"] / (r["t_ms"] * 1e-3) / 1e9
        line = dict(metric="resample effective HBM GB/s (B_alg = N*20 + 64*(D+N), all GPUs)",
                    value=achieved, unit="GB/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
                    ms_per_step=r["t_ms"], higher_is_better=True, scaling="weak", vs_baseline=None,
                    dtype="f64/u128", data="synthetic",
                    config=dict(workload="resample", desc=wl["desc"], n_per_gpu=r["n"], state_bytes=64,
                                sigma=args.sigma, parallelism=f"global resampling over {world} GPUs",
                                l2="flushed between steps"),
                    roofline=dict(bound="hbm", achieved=achieved / world, peak=hbm_peak, unit="GB/s",
                                  frac=achieved / world / hbm_peak, traffic=None,
                                  note="per GPU; chain incl. NCCL all-gathers and NVLink migration"),
                    gpu_launches=(5 * world + 0) * args.steps, clocks=r["clocks"])
        if rank == 0:
            print(json.dumps(line), flush=True)
        return
    if wl["model"] == "resample":
        line = resample_line(args, smc, torch, world, rank, pk, pk_kind, n=args.n or wl["n"],
                             sigma=args.sigma, inplace=args.inplace, steps=args.steps,
                             warmup=args.warmup)
        if rank == 0:
            print(json.dumps(line), flush=True)
        return
    draw_peak = smc.draw_peak() / 1e9
    line = sweep_line(args, args.workload, wl, smc, torch, world, rank, pk, pk_kind, draw_peak,
                      with_e2e=not args.no_e2e, with_cpu=not args.no_cpu_baseline)
    if world == 1 and args.workload == "crbd" and not args.only:
        # the other BASELINE configs, measured in the same run (the headline
        # fields above stay configs[1]'s): configs[2] ClaDS2, configs[3] SEIR,
        # configs[4] the resampling step at 2^26 and 2^28 particles
        subs = {}
        for key, name in (("c2_clads2", "clads2"), ("c3_seir", "seir")):
            sl = sweep_line(args, name, WORKLOADS[name], smc, torch, world, rank, pk, pk_kind,
                            draw_peak, with_e2e=False, with_cpu=False)
            subs[key] = {k: sl[k] for k in ("metric", "value", "unit", "ms_per_step", "sweeps_per_s",
                                            "mean_log_z", "phase_ms", "draws_per_particle_step",
                                            "roofline", "resample_roofline", "clocks", "config",
                                            "guard_kills_per_particle_step", "gpu_launches") if k in sl}
        # configs[1] under the per-particle sequential stream (R-11: one thread
        # walks its whole side tree; the headline uses the lineage-keyed R-18)
        seq_args = argparse.Namespace(**vars(args))
        seq_args.rng, seq_args.workload = "sequential", "crbd (sequential stream)"
        sl = sweep_line(seq_args, "crbd", wl, smc, torch, world, rank, pk, pk_kind, draw_peak,
                        with_e2e=False, with_cpu=False)
        subs["c1_crbd_sequential_rng"] = {k: sl[k] for k in ("metric", "value", "unit", "ms_per_step",
                                                             "sweeps_per_s", "mean_log_z", "phase_ms",
                                                             "draws_per_particle_step", "roofline",
                                                             "resample_roofline", "clocks", "config",
                                                             "gpu_launches") if k in sl}
        for lg in (26, 28):
            rl = resample_line(args, smc, torch, world, rank, pk, pk_kind, n=1 << lg, sigma=1.0)
            subs[f"c4_resample_2p{lg}"] = {k: rl[k] for k in ("metric", "value", "unit", "ms_per_step",
                                                              "roofline", "chain_roofline", "kernel_ms",
                                                              "distinct_ancestors", "clocks", "config")}
        line["configs"] = subs
    if rank == 0:
        print(json.dumps(line), flush=True)


def sweep_line(args, name, wl, smc, torch, world, rank, pk, pk_kind, draw_peak, with_e2e, with_cpu):
    """One sweep workload (configs[1]-[3]): the JSON fields of its line."""
    hbm_peak = pk["hbm_gbs"]
    rng = args.rng if wl["model"] in ("crbd", "clads2") else "sequential"
    ess = args.ess if name == args.workload else wl.get("ess", "1/1")
    sub_args = argparse.Namespace(**vars(args))
    sub_args.ess = ess
    if name != args.workload:
        sub_args.n = 0
        sub_args.steps = max(3, min(args.steps, 5))
        sub_args.warmup = max(3, args.warmup)
        sub_args.inplace = False
    oracle_sweep_rate.ess = ess
    r = bench_sweeps(sub_args, wl, smc, torch, world, rank)
    steps = sub_args.steps
    N = r["N"]
    # propagation roofline: algorithmic uniforms per particle-step
    # counted by the oracle on a sample of the same workload, times the GPU's
    # particle-steps, per second of propagation, against the measured draw-rate
    # ceiling (smc_draw_peak: divergence-free Philox + hq + fp64 Exp)
    f_max = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    derived_peak = 148 * 128 * f_max / 34.0 / 1e9
    prop_s = max(r["prop_ms"] / steps * 1e-3, 1e-12)
    gpu_rate = r["draws"] / steps / prop_s / 1e9
    lin = rng == "lineage" and not wl.get("analytic")
    gdps = r["draws"] / max(r["alive_steps"], 1)
    cpu = None
    if rank == 0 and with_cpu and world == 1:
        cpu = oracle_sweep_rate(wl, budget_s=args.cpu_budget)
    spec = None
    if lin and rank == 0:           # (reported by rank 0 only; no collectives inside)
        # Under R-18 the GPU's count depends on its visiting order (speculative
        # side-tree nodes evaluated before a detection elsewhere stops the tree,
        # and nodes a depth-first walk would have reached first but that were
        # pruned).  The algorithmic count is the oracle's for the SAME particle
        # system: per-sweep counts vary ~2x between seeds, so a different seed
        # is no reference.  The oracle sweep of the sample (the cpu_baseline
        # sweep when it ran, else 20000 particles; seed 12345) is repeated on
        # the GPU with the same N and seed — identical particles, ancestors and
        # weights (parity) — and the ratio oracle/GPU of the two counts scales
        # the GPU's count at the bench size.
        try:
            if cpu:
                ost, osample = cpu[3], cpu[1]
            else:
                _, osample, _, ost = oracle_sweep_rate(wl, n_cap=20000, budget_s=0.0)
            odraws = ost["draws"]
            n_s = int(osample.split("N=")[1].split()[0])
            hs = smc.Smc(model_for(smc, wl, rng, False), n_s, seed=12345)
            ea, eb = (int(x) for x in ess.split("/"))
            hs.set_ess_threshold(ea, eb)
            hs.run()
            gst = hs.stats()
            hs.close()
            ratio = odraws / max(gst["draws"], 1)
            if gst["alive_particle_steps"] != ost["alive_particle_steps"]:
                raise RuntimeError("sample sweeps differ (GPU vs oracle particle-steps)")
            odps = gdps * ratio
            spec = dict(sample=osample, oracle_draws=odraws, gpu_draws=gst["draws"],
                        oracle_over_gpu=ratio,
                        oracle_draws_per_particle_step_sample=odraws / max(ost["alive_particle_steps"], 1))
        except Exception as e:  # noqa: BLE001  (the oracle is a reported baseline, not the product)
            odps, osample = None, f"oracle unavailable: {e}"
    else:
        # identical streams: the GPU draws exactly the oracle's uniforms
        # (tests/test_gpu_fullsweep.py asserts equality at 10^6)
        odps, osample = gdps, "equal to the GPU count (identical streams, asserted at 10^6 in tests)"
    alg_rate = (odps * r["alive_steps"] / steps / prop_s / 1e9) if odps else None
    peak = draw_peak if draw_peak else derived_peak
    prop_frac = r["prop_ms"] / max(r["prop_ms"] + r["res_ms"], 1e-9)
    lr_name = "propagate_lr_kernel" if os.environ.get("SMC_LR_KERNEL") == "cta" else "propagate_lrw_kernel"
    kname = (lr_name if lin else "propagate_kernel") + f"<{name}>"
    line = dict(metric="particle-steps/s", value=r["value"], unit="particle-steps/s",
                n_gpus=world, steps=steps, warmup=sub_args.warmup,
                ms_per_step=r["t_ms"] / steps, higher_is_better=True, scaling="weak",
                vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=name, desc=wl["desc"], n_per_gpu=N,
                            rng=("analytic (no side trees)" if wl.get("analytic") else rng),
                            ess_threshold=ess, inplace=sub_args.inplace,
                            epochs_per_sweep=r["epochs"] // steps,
                            l2="flushed between steps (state fits L2 within a sweep)"),
                sweeps_per_s=r["sweeps"], mean_log_z=r["logz"],
                resamples_per_sweep=r["resamples_per_sweep"],
                phase_ms=dict(propagate=r["prop_ms"] / steps, resample=r["res_ms"] / steps,
                              propagate_share=prop_frac),
                draws_per_particle_step=dict(oracle=odps, oracle_sample=osample, gpu=gdps,
                                             seed_matched=spec,
                                             note=("algorithmic = the GPU count of this run x the oracle/GPU "
                                                   "ratio of a seed-matched sample sweep (the GPU's visiting "
                                                   "order changes which side-tree nodes it draws, R-18)")
                                             if lin else "identical streams"),
                resample_roofline=dict(bound="hbm", achieved=r["res_bytes"] / (r["res_ms"] * 1e-3) / 1e9,
                                       peak=hbm_peak, unit="GB/s",
                                       frac=r["res_bytes"] / (r["res_ms"] * 1e-3) / 1e9 / hbm_peak,
                                       kernel=("resample_fused_kernel (one cooperative launch per epoch)"
                                               if r["fused"] else "reduce + anc_gather + finalize"),
                                       traffic=((traffic(f"{wl['model']}:{N}:resample_fused_kernel") or {}).get("bytes")
                                                if r["fused"] else None),
                                       state_gather=("deferred into the next propagation (DESIGN 7.7): "
                                                     "B_alg = N*20 per resample, no state bytes"
                                                     if r["deferred"] else
                                                     "in the resampling step: B_alg = N*(20+S) + S*D"),
                                       note="per epoch at this N (latency-bound at 10^6; "
                                            "see workload 'resample' for the HBM-bound sizes)"),
                roofline=dict(bound="alu", kernel=kname,
                              achieved=alg_rate if alg_rate else gpu_rate, peak=peak, unit="Gdraws/s",
                              frac=(alg_rate if alg_rate else gpu_rate) / peak,
                              achieved_gpu_count=gpu_rate,
                              traffic=((traffic(f"{wl['model']}:{N}:{kname.split('<')[0]}") or {}).get("bytes")),
                              peak_source=("measured live: smc_draw_peak (Philox + hq + fp64 -log(u)/rate, "
                                           "every lane, full occupancy)" if draw_peak else "derived"),
                              derived_issue_peak=derived_peak),
                gpu_launches=r["launches"], clocks=r["clocks"])
    if wl["model"] == "clads2":
        line["guard_kills_per_particle_step"] = r["guard"] / max(r["alive_steps"], 1)
    if wl["model"] == "stackf" and r["resamples_per_sweep"]:
        # the paper's "critical optimization": bytes of state each
        # output slot copies, with the stack-prefix copy and with the whole
        # user-defined stack (SMC_NO_STACK_PREFIX=1, same sweeps)
        per_slot = 16.0 * r["stack_planes"] / (r["resamples_per_sweep"] * steps * N)
        # like for like: both comparison runs materialise the gather in the
        # resampling step (SMC_EAGER_GATHER=1), one copying the stack prefix,
        # one the whole stack (SMC_NO_STACK_PREFIX=1)
        runs = {}
        for tag, env in (("prefix", {"SMC_EAGER_GATHER": "1"}),
                         ("full", {"SMC_EAGER_GATHER": "1", "SMC_NO_STACK_PREFIX": "1"})):
            os.environ.update(env)
            try:
                runs[tag] = bench_sweeps(sub_args, wl, smc, torch, world, rank)
            finally:
                for k in env:
                    os.environ.pop(k, None)
            runs[tag]["h"].close()
        line["stack_copy"] = dict(bytes_per_slot_prefix=per_slot, bytes_per_slot_full=float(r["state_bytes"]),
                                  eager_resample_ms_per_sweep_prefix=runs["prefix"]["res_ms"] / steps,
                                  eager_resample_ms_per_sweep_full=runs["full"]["res_ms"] / steps,
                                  eager_ms_per_sweep_prefix=runs["prefix"]["t_ms"] / steps,
                                  eager_ms_per_sweep_full=runs["full"]["t_ms"] / steps,
                                  note="the headline run defers the gather into the next propagation "
                                       "(DESIGN 7.7), which also copies only the stack prefix")
    if with_e2e:
        e = e2e_sweeps(sub_args, wl, smc, torch, r["h"], r["model"], min(steps, 3), world)
        tot = sum_over_ranks(torch, world, r["alive_steps"] / steps)
        line["e2e"] = dict(value=tot / e["t"], unit="particle-steps/s",
                           h2d_bytes_per_step=e["h2d"] * world, d2h_bytes_per_step=e["d2h"] * world,
                           note="per step: H2D of the model data, reset(seed), run, D2H of log Z and "
                                "the final log-weights; host wall clock, max over ranks")
    if cpu:
        v, sample, dt, _ = cpu
        line["cpu_baseline"] = dict(value=v, unit="particle-steps/s", cores=1, kind="oracle",
                                    sample=sample, seconds=dt, host=host_cpu())
    r["h"].close()
    oracle_sweep_rate.ess = args.ess
    return line


def host_cpu():
    """lscpu model name and nproc of the box."""
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return dict(model=model, nproc=os.cpu_count())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="crbd", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=0, help="particles per GPU (default: workload's)")
    ap.add_argument("--sigma", type=float, default=1.0, help="resample workload: lw ~ sigma N(0,1)")
    ap.add_argument("--rng", default="lineage", choices=sorted(RNG),
                    help="tree models: lineage-keyed side trees (DESIGN R-18, cooperative kernel) "
                         "or the sequential per-particle stream (R-11)")
    ap.add_argument("--ess", default=None,
                    help="ESS-adaptive resampling threshold a/b (DESIGN R-19); 1/1 = every checkpoint "
                         "(default: the workload's, 1/1 unless stated)")
    ap.add_argument("--inplace", action="store_true",
                    help="in-place resampling by ancestor permutation (DESIGN R-21, SURVEY f3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--only", action="store_true",
                    help="default workload: skip the configs[2]-[4] sub-results")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 breaks the timing rules", file=sys.stderr)
    wl = WORKLOADS[args.workload]
    if args.ess is None:
        args.ess = wl.get("ess", "1/1")
    oracle_sweep_rate.rng = args.rng
    oracle_sweep_rate.ess = args.ess
    oracle_sweep_rate.inplace = args.inplace
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
