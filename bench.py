#!/usr/bin/env python
"""bench.py -- throughput of the fused fp64 stencil hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl oec|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

A STEP is one pass of the whole hot path over one batch of synthetic input: hdiff
followed by vadv on BASELINE.json configs[1], the paper-shaped 128x128x80 fp64 domain, per GPU.
With N > 1 ranks the global domain is 128 x (128 N) x 80 split into j-slabs (weak scaling); each
step first exchanges hdiff's 2-wide halo with the neighbouring ranks over NCCL (vadv needs none).

value     = grid points / s of the whole job: N * 128*128*80 points per step / step time, inputs
            resident in HBM; timed on the device with CUDA events over exactly K steps (max over
            ranks).  Each step reads a different one of R rotating input sets whose total is > 4x
            the 126 MB L2, so every kernel streams its inputs from HBM.
e2e       = the same metric through the C-ABI with HOST buffers (pinned): H2D of the step's inputs,
            the kernels, D2H of the outputs, per step, inside the timed region.
roofline  = the dominant kernel's ALGORITHMIC bytes per launch
            / its average CUDA-event duration, against MEASURED_PEAKS.json's HBM copy bandwidth.
cpu_baseline / --impl reference = the CPU oracle (oracle/, C, OpenMP) on the box's host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (seeded inputs only; no method arithmetic)

METRIC = "grid points/s and effective HBM GB/s (fraction of B200 peak) per stencil @1/2/4/8 GPU"
UNIT = "grid points/s"
DOMAIN = (128, 128, 80)  # BASELINE.json configs[1]
WORKLOAD = "hdiff + vadv fp64 at the paper's 128x128x80 domain on 1xB200 (BASELINE.json configs[1])"
FALLBACK_HBM_GBS = 6650.0


# ---------------------------------------------------------------------------------------------
# algorithmic (compulsory) bytes: each input's distinct touched elements + each output's domain,
# x 8 B ("all inputs of the stencil program are only loaded once"); DESIGN.md table
# ---------------------------------------------------------------------------------------------
def hdiff_bytes(ni, nj, nk):
    return 8 * (((ni + 4) * (nj + 4) - 12) * nk + 2 * ni * nj * nk)


def vadv_bytes(ni, nj, nk):
    return 8 * (4 * ni * nj * nk + (ni + 1) * nj * (nk - 1) + ni * nj * nk)


def program_bytes(program, dom):
    """Bounding-box count from the registry extents (exact for every suite program whose extent
    is a full box; hdiff/vadv use the exact formulas above)."""
    from paper_2005_13014_b200 import oec

    if program == "hdiff":
        return hdiff_bytes(*dom)
    if program == "vadv":
        return vadv_bytes(*dom)
    ins, outs, _ = oec.program_signature(program)
    b = 0
    for _, lo, hi, kinv in ins:
        ext = [dom[d] + hi[d] - lo[d] for d in range(3)]
        if kinv:
            ext[2] = 1
        b += ext[0] * ext[1] * ext[2]
    b += len(outs) * dom[0] * dom[1] * dom[2]
    return 8 * b


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """Per-launch dram bytes of each kernel from the committed ncu --set full summary (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------------------------
# clocks during the timed region (nvidia-smi sampler)
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_id: str):
        self.samples = []
        self.proc = None
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", gpu_id, "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.first = threading.Event()
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()
        self.first.wait(10.0)

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.perf_counter(), line.strip()))
            self.first.set()

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def result(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        rows = []
        for t, line in self.samples:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            rows.append((t, parts))
        inside = [r for t, r in rows if self.t0 is not None and self.t0 - 0.06 <= t <= (self.t1 or t) + 0.06]
        used = inside if inside else rows
        sm = [float(r[0]) for r in used if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in used if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in used for q in range(4) if r[2 + q].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(used), "samples_in_region": len(inside)}


# ---------------------------------------------------------------------------------------------
# the CPU oracle (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------------
def oracle_step_fn(domain, nj_sample=None):
    from oracle import capi

    capi.build()
    nthreads = os.cpu_count() or 1
    h = synth.make_inputs("hdiff", domain, seed=0)
    v = synth.make_inputs("vadv", domain, seed=0)
    dtr = synth.scalars("vadv")["dtr_stage"]
    ni, nj, nk = domain
    njs = nj if nj_sample is None else max(1, min(nj, nj_sample))
    oh = synth.HostField(np.zeros((nk, nj, ni)), (0, 0, 0), domain)
    ov = synth.HostField(np.zeros((nk, nj, ni)), (0, 0, 0), domain)

    def step():
        capi.hdiff(h["in"], h["coeff"], oh, (0, 0, 0), (ni, njs, nk), capi.HDIFF_UNFUSED, nthreads)
        capi.vadv(v, ov, dtr, (0, 0, 0), (ni, njs, nk), capi.VADV_UNFUSED, nthreads)

    return step, ni * njs * nk, nthreads


def cpu_baseline(domain, seconds=10.0):
    step, pts, nthreads = oracle_step_fn(domain)
    step()  # warm-up
    n, t0 = 0, time.perf_counter()
    while True:
        step()
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 1000:
            break
    return {"value": n * pts / el, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"{n} full steps (hdiff + vadv, unfused C oracle, OpenMP {nthreads} threads) of the "
                      f"{domain[0]}x{domain[1]}x{domain[2]} workload, {el:.1f} s"}


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    full_step, pts_full, nthreads = oracle_step_fn(DOMAIN)
    t0 = time.perf_counter()
    full_step()
    t_full = time.perf_counter() - t0
    budget = 120.0  # seconds for warm-up + timed steps
    frac = min(1.0, budget / max(1e-9, (args.warmup + args.steps) * t_full))
    nj_s = max(1, int(DOMAIN[1] * frac))
    step, pts, nthreads = oracle_step_fn(DOMAIN, nj_s)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = args.steps * pts / el
    sample = (f"each step = hdiff + vadv (unfused C oracle, OpenMP {nthreads} threads) on a "
              f"{DOMAIN[0]}x{nj_s}x{DOMAIN[2]} j-slab sample of the {DOMAIN[0]}x{DOMAIN[1]}x{DOMAIN[2]} workload")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD, "domain": list(DOMAIN), "sample_domain": [DOMAIN[0], nj_s, DOMAIN[2]]},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------------------------
class StepSet:
    """Device fields of one rotating input set: hdiff {in, coeff, out}, vadv {5 inputs, out}."""

    def __init__(self, oec, hh, vh, domain):
        self.h_in = oec.field_from_host(hh["in"])
        self.h_cf = oec.field_from_host(hh["coeff"])
        self.h_out = oec.empty_like_domain(domain, fill=0.0)
        self.v_in = [oec.field_from_host(vh[n]) for n in ("u_stage", "wcon", "u_pos", "utens", "utens_stage_in")]
        self.v_out = oec.empty_like_domain(domain, fill=0.0)

    def nbytes(self):
        fs = [self.h_in, self.h_cf, self.h_out, self.v_out] + self.v_in
        return sum(int(np.prod([f.ub[d] - f.lb[d] for d in range(3)])) * 8 for f in fs)


def fused_pipelines(oec, dist, sets, domain, world, rank, dev_index, agree):
    """N > 1, --exchange fused: one oec_hdiff_pipeline per rotating set over this rank's j-slab of
    the global 128 x 128N x 80 domain (x0 = the set's hdiff input with its halo, x1 a copy: the
    global outer halo stays constant); fields and signal pads are exported with CUDA IPC, the
    handles all-gathered, and every pipeline registers its j-neighbours' (imported) fields.
    Each phase ends with agree(ok) (a MIN over ranks), so every rank takes the same path; returns
    None on success, else the reason."""
    import torch

    gdom = (domain[0], domain[1] * world, domain[2])
    mine, err = [], None
    try:  # phase 1: local pipelines and IPC exports
        for s in sets:
            x1 = oec.oec_field_create(domain, (2, 2, 0), (2, 2, 0))
            x1.view().copy_(s.h_in.view())
            s.x1 = x1
            s.pipe = oec.HdiffPipeline(gdom, 1, world, rank, s.h_cf, s.h_in, x1)
            pad, _ = s.pipe.signal_pad()
            mine.append(dict(x0=oec.oec_ipc_export(s.h_in.desc.data), x1=oec.oec_ipc_export(x1.desc.data),
                             pad=oec.oec_ipc_export(pad), desc=oec.field_descriptor(s.h_in)))
        torch.cuda.synchronize()
    except Exception as e:
        err = f"{type(e).__name__}: {e}"
    if not agree(err is None):
        return err or "pipeline setup failed on another rank"
    everyone = [None] * world
    dist.all_gather_object(everyone, mine)
    try:  # phase 2: import the j-neighbours' memory
        for q in (rank - 1, rank + 1):
            if not 0 <= q < world:
                continue
            for si, s in enumerate(sets):
                Q = everyone[q][si]
                p0, p1, pp = (oec.oec_ipc_import(*Q[k]) for k in ("x0", "x1", "pad"))
                s.pipe.set_peer(q, oec.field_at(p0, Q["desc"], dev_index), oec.field_at(p1, Q["desc"], dev_index), pp)
    except Exception as e:
        err = f"{type(e).__name__}: {e}"
    if not agree(err is None):
        return err or "peer import failed on another rank"
    dist.barrier()
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30000)
    ap.add_argument("--warmup", type=int, default=60)
    ap.add_argument("--impl", default="oec", choices=["oec", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sets", type=int, default=0, help="rotating input sets (0 = auto, > 4x L2)")
    ap.add_argument("--force-decomp", action="store_true",
                    help="debug: run the N>1 code path (NCCL process group, decomposition, exchange) even at N=1")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N>1 halo exchange of hdiff: 'fused' = oec_hdiff_pipeline (each step one kernel that "
                         "reads the neighbours' halo cells from their memory over NVLink, CUDA IPC), 'nccl' = "
                         "oec_halo_exchange (NCCL send/recv on a comm stream, concurrent with vadv)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: testing the fused path with all ranks on one GPU, "
                         "OEC_BENCH_DEVICE=0)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    args.warmup = max(3, args.warmup)

    import torch
    import torch.distributed as dist

    from paper_2005_13014_b200 import oec

    oec.lib()  # fail loudly if the extension is missing
    dev_index = int(os.environ.get("OEC_BENCH_DEVICE", local_rank))
    torch.cuda.set_device(dev_index)
    dev = torch.cuda.current_device()
    decomp = world > 1 or args.force_decomp
    fused = decomp and args.exchange == "fused"
    if args.dist_backend == "gloo" and not fused:
        raise SystemExit("--dist-backend gloo needs --exchange fused")
    if decomp:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20))
    domain = DOMAIN
    pts = domain[0] * domain[1] * domain[2]

    # ---- decomposition (N > 1): j-slabs of the global 128 x 128N x 80 domain ----
    dec = None
    if decomp and not fused:
        pg = dist.distributed_c10d._get_default_group()
        nccl_pg = pg._get_backend(torch.device("cuda", dev_index))
        dist.barrier()
        nccl_comm = nccl_pg._comm_ptr()
        dec = oec.oec_decomp_create((domain[0], domain[1] * world, domain[2]), 1, world, rank, nccl_comm)

    # ---- rotating input sets ----
    hh = synth.make_inputs("hdiff", domain, seed=rank)
    vh = synth.make_inputs("vadv", domain, seed=1000 + rank)
    dtr = synth.scalars("vadv")["dtr_stage"]
    first = StepSet(oec, hh, vh, domain)
    R = args.sets or max(2, math.ceil(4 * l2 / first.nbytes()) + 1)
    sets = [first] + [StepSet(oec, hh, vh, domain) for _ in range(R - 1)]
    fused_note = None
    if fused:
        def agree(ok):
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda" if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            return int(flag.item()) == 1

        why = fused_pipelines(oec, dist, sets, domain, world, rank, dev_index, agree)
        if why is not None:  # e.g. no peer access: every rank falls back to the NCCL exchange
            if args.dist_backend != "nccl":
                raise SystemExit(f"fused pipeline unavailable: {why}")
            fused = False
            fused_note = f"fused pipeline unavailable ({why}); NCCL exchange used"
            pg = dist.distributed_c10d._get_default_group()
            dec = oec.oec_decomp_create((domain[0], domain[1] * world, domain[2]), 1, world, rank,
                                        pg._get_backend(torch.device("cuda", dev_index))._comm_ptr())

    launches = {"hdiff": 0, "vadv": 0, "halo": 0}

    def hdiff(s):
        if fused:  # one step of this set's pipeline: hdiff with the halo read from the neighbours
            s.pipe.run(1)
        else:
            oec.oec_hdiff(s.h_in, s.h_cf, s.h_out, (0, 0, 0), domain)
        launches["hdiff"] = oec.oec_last_launch_count()

    def vadv(s):
        oec.oec_vadv(*s.v_in, s.v_out, dtr, (0, 0, 0), domain)
        launches["vadv"] = oec.oec_last_launch_count()

    def exchange(s):
        if dec is not None:
            oec.oec_halo_exchange(dec, [s.h_in], (2, 2, 0), (2, 2, 0))
            launches["halo"] = oec.oec_last_launch_count()

    # warm-up (also configures kernel attributes and NCCL staging before any capture)
    for w in range(args.warmup):
        s = sets[w % R]
        exchange(s)
        hdiff(s)
        vadv(s)
    torch.cuda.synchronize()

    # ---- CUDA graphs of R launches of each kernel (launch-overhead-free timing) ----
    # N > 1: the hdiff halo exchange (NCCL, comm stream) runs concurrently with vadv (no halo
    # needed for j-slabs), then hdiff; graphs gx (exchanges), gv (vadv), gh (hdiff) per R steps.
    has_x = dec is not None
    comm_stream = torch.cuda.Stream() if has_x else None
    graphs = {}
    x_mode = None

    def capture(nsteps):
        nonlocal x_mode
        gh, gv = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gh):
            for q in range(nsteps):
                hdiff(sets[q % R])
        with torch.cuda.graph(gv):
            for q in range(nsteps):
                vadv(sets[q % R])
        gx = None
        if has_x:
            try:
                gx = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gx):
                    for q in range(nsteps):
                        exchange(sets[q % R])
                x_mode = "NCCL captured in a CUDA graph on a comm stream, concurrent with vadv"
            except Exception as e:  # NCCL capture unavailable: exchanges launched eagerly instead
                gx = None
                x_mode = f"NCCL launched eagerly on a comm stream, concurrent with vadv ({type(e).__name__})"
        return gh, gv, gx

    graphs[R] = capture(R)
    if args.steps % R:
        graphs[args.steps % R] = capture(args.steps % R)
    for g in graphs.values():  # one untimed replay each
        g[0].replay()
        g[1].replay()
        if g[2] is not None:
            g[2].replay()
    torch.cuda.synchronize()

    chunks = [R] * (args.steps // R) + ([args.steps % R] if args.steps % R else [])
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in chunks]
    gpu_id = "GPU-" + str(props.uuid) if hasattr(props, "uuid") else str(dev)
    clocks = ClockSampler(gpu_id)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    t_start.record()
    done = 0
    cur = torch.cuda.current_stream()
    for c, n in enumerate(chunks):
        e0, e1, e2 = ev[c]
        gh, gv, gx = graphs[n]
        e0.record()
        if has_x:
            comm_stream.wait_stream(cur)
            with torch.cuda.stream(comm_stream):
                if gx is not None:
                    gx.replay()
                else:
                    for q in range(n):
                        exchange(sets[(done + q) % R])
        gv.replay()
        if has_x:
            cur.wait_stream(comm_stream)
        e1.record()
        gh.replay()
        e2.record()
        done += n
    t_stop.record()
    torch.cuda.synchronize()
    clocks.mark_stop()
    elapsed_ms = t_start.elapsed_time(t_stop)
    t_v = sum(e[0].elapsed_time(e[1]) for e in ev)  # vadv (|| halo exchange when N > 1)
    t_h = sum(e[1].elapsed_time(e[2]) for e in ev)
    if world > 1:
        t = torch.tensor([elapsed_ms, t_h, t_v], device="cuda" if args.dist_backend == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, t_h, t_v = [float(x) for x in t.tolist()]
    clk = clocks.result()
    K = args.steps
    ms_step = elapsed_ms / K
    value = world * pts / (ms_step * 1e-3)

    peak, peak_src = hbm_peak()
    traffic = ncu_traffic()
    kern = {}
    for name, tot, nbytes in (("hdiff", t_h, hdiff_bytes(*domain)), ("vadv", t_v, vadv_bytes(*domain))):
        us = 1e3 * tot / K
        gbs = nbytes / (us * 1e-6) / 1e9
        kern[name] = {"us_per_launch": us, "algorithmic_bytes": nbytes, "GB/s": gbs, "frac_of_hbm_peak": gbs / peak,
                      "grid_points_per_s": pts / (us * 1e-6)}
    dom_k = max(kern, key=lambda k: kern[k]["us_per_launch"])
    tr = traffic.get(dom_k)
    roofline = {"bound": "hbm", "kernel": dom_k, "achieved": kern[dom_k]["GB/s"], "peak": peak, "unit": "GB/s",
                "frac": kern[dom_k]["GB/s"] / peak, "traffic": tr, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": kern[dom_k]["algorithmic_bytes"]}

    # ---- e2e through the C-ABI with pinned host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_measure(oec, torch, hh, vh, dtr, domain, args.e2e_steps, world)

    # ---- remaining suite (evidence for SURVEY §8(a) a7; not part of the step) ----
    suite_res = levels = f32_res = jit_res = pipe_res = paper_res = None
    if not args.no_suite and world == 1:
        suite_res = suite_measure(oec, torch, domain, l2, peak)
        levels = levels_measure(oec, torch, domain, l2, peak)
        f32_res = f32_measure(oec, torch, domain, l2, peak)
        jit_res = jit_measure(oec, torch, domain, l2, peak)
        pipe_res = pipeline_measure(oec, torch, domain, l2, peak)
        paper_res = paper_sizes_measure(oec, torch, l2, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(domain, args.cpu_seconds)

    n_launch = K * (launches["hdiff"] + launches["vadv"] + launches["halo"])
    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded numpy PCG64, SURVEY §8(d) distributions)",
            "config": {"workload": WORKLOAD, "domain_per_gpu": list(domain),
                       "global_domain": [domain[0], domain[1] * world, domain[2]],
                       "parallelism": (f"j-slab decomposition 1x{world}, " + (
                           "hdiff halo read from the neighbours' memory inside the kernel (fused pipeline, CUDA IPC)"
                           if fused else "NCCL halo exchange")) if world > 1 else "single GPU",
                       "l2": f"inputs larger than L2: {R} rotating input sets, "
                             f"{R * first.nbytes() / 2**20:.0f} MiB total vs {l2 / 2**20:.0f} MiB L2",
                       "timing": "CUDA events on the launching stream around CUDA graphs of R launches per "
                                 "kernel; max over ranks" + (f"; halo exchange: {x_mode}" if has_x else "")
                                 + (f"; {fused_note}" if fused_note else "")},
            "roofline": roofline,
            "kernels": kern,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": n_launch,
            "clocks": clk,
        }
        if suite_res is not None:
            res["suite"] = suite_res
        if levels is not None:
            res["optimization_levels"] = levels
        if f32_res is not None:
            res["f32"] = f32_res
        if jit_res is not None:
            res["jit"] = jit_res
        if pipe_res is not None:
            res["hdiff_pipeline"] = pipe_res
        if paper_res is not None:
            res["paper_sizes"] = paper_res
        print(json.dumps(res), flush=True)
    if decomp:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e_measure(oec, torch, hh, vh, dtr, domain, steps, world):
    """The step through the public C-ABI with pinned host buffers (device = OEC_DEVICE_HOST): the
    library copies the inputs H2D, runs the kernel, copies the outputs' domain D2H, per call."""
    def pinned(hf):
        t = torch.empty(hf.data.shape, dtype=torch.float64, pin_memory=True)
        t.copy_(torch.from_numpy(hf.data))
        return oec.oec_field_wrap(t, hf.lb, hf.ub, k_invariant=hf.k_invariant)

    ni, nj, nk = domain
    h_in, h_cf = pinned(hh["in"]), pinned(hh["coeff"])
    v_in = [pinned(vh[n]) for n in ("u_stage", "wcon", "u_pos", "utens", "utens_stage_in")]
    o1 = torch.zeros((nk, nj, ni), dtype=torch.float64, pin_memory=True)
    o2 = torch.zeros((nk, nj, ni), dtype=torch.float64, pin_memory=True)
    f_o1 = oec.oec_field_wrap(o1, (0, 0, 0), domain)
    f_o2 = oec.oec_field_wrap(o2, (0, 0, 0), domain)

    def step():
        oec.oec_hdiff(h_in, h_cf, f_o1, (0, 0, 0), domain)
        oec.oec_vadv(*v_in, f_o2, dtr, (0, 0, 0), domain)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    h2d = sum(f._keep.numel() * 8 for f in [h_in, h_cf] + v_in)
    d2h = 2 * ni * nj * nk * 8
    return {"value": world * ni * nj * nk / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": steps,
            "path": "oec_hdiff/oec_vadv with OEC_DEVICE_HOST fields (pinned), staged by liboec, synchronous"}


def program_measure(oec, torch, program, domain, l2, peak, variant=0, reps=20, dtype=np.float64, run_name=None):
    """us per launch of one program (CUDA graph of R launches over R rotating input sets > 4x L2).
    dtype=np.float32: the paper's f32 runs; algorithmic bytes scale with the element size.
    run_name: apply this registered program instead (a stencil-language version of `program` with
    the same argument order, compiled by liboec's JIT)."""
    host = synth.make_inputs(program, domain, seed=0, dtype=dtype)
    spec = synth.PROGRAMS[program]
    sc = [v for _, v in spec.scalars]

    def make():
        ins = [oec.field_from_host(host[s.name]) for s in spec.inputs]
        outs = [oec.empty_like_domain(domain, fill=0.0, dtype=dtype) for _ in spec.outputs]
        return ins, outs

    s0 = make()
    set_bytes = sum(int(np.prod([f.ub[d] - f.lb[d] for d in range(3)])) * f.itemsize for f in s0[0] + s0[1])
    R = max(2, math.ceil(4 * l2 / set_bytes) + 1)
    sets = [s0] + [make() for _ in range(R - 1)]
    name = run_name or program
    for ins, outs in sets:  # also sizes any library workspace / compiles JIT kernels outside the capture
        oec.oec_apply_program(name, ins, outs, sc, (0, 0, 0), domain, variant)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for ins, outs in sets:
            oec.oec_apply_program(name, ins, outs, sc, (0, 0, 0), domain, variant)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = 1e3 * a.elapsed_time(b) / (reps * R)
    nbytes = program_bytes(program, domain) * np.dtype(dtype).itemsize // 8
    del sets, s0, g
    return {"us_per_launch": us, "algorithmic_bytes": nbytes, "GB/s": nbytes / (us * 1e-6) / 1e9,
            "frac_of_hbm_peak": nbytes / (us * 1e-6) / 1e9 / peak,
            "grid_points_per_s": domain[0] * domain[1] * domain[2] / (us * 1e-6)}


def suite_measure(oec, torch, domain, l2, peak):
    return {p: program_measure(oec, torch, p, domain, l2, peak) for p in synth.SUITE}


def f32_measure(oec, torch, domain, l2, peak):
    """Every program in binary32 (P:556 evaluates f32 and f64), default kernels."""
    return {p: program_measure(oec, torch, p, domain, l2, peak, dtype=np.float32) for p in synth.ALL_PROGRAMS}


def jit_measure(oec, torch, domain, l2, peak):
    """The stencil-language versions of every stencil program (tests/programs/*.oec), compiled by
    liboec's JIT (shape inference, inlining / unrolling / original level, size-specialised NVRTC
    kernels for sm_100a; include/oec.h), at each optimisation level of P:616 (unrolling along j and
    k) and AUTO (empirical tuning), next to the hand-written builtin kernel of the same
    program (bit-identical results: tests/test_gpu_jit.py)."""
    res = {}
    pdir = os.path.join(ROOT, "tests", "programs")
    for fn in sorted(os.listdir(pdir)):
        program = fn[:-4]
        with open(os.path.join(pdir, fn)) as f:
            name = oec.oec_program_create(f.read())
        try:
            r = {lvl: program_measure(oec, torch, program, domain, l2, peak, v, run_name=name)
                 for lvl, v in (("original", 1), ("inline", 2), ("inline_unroll2", 3), ("inline_unroll4", 4),
                                ("inline_unroll2_k", 5), ("inline_unroll4_k", 6), ("tiled_tma", 7),
                                ("auto_tuned", 0))}
            r["best"] = min(r, key=lambda n: r[n]["us_per_launch"])
            r["builtin_us_per_launch"] = program_measure(oec, torch, program, domain, l2, peak, 0)["us_per_launch"]
        finally:
            oec.oec_program_destroy(name)
        res[program] = r
    return res


def pipeline_measure(oec, torch, domain, l2, peak, reps=20):
    """The fused-exchange multi-step hdiff (oec_hdiff_pipeline) on one rank
    (px = py = 1: no neighbours, every tile interior): us per step next to hdiff's algorithmic bytes.
    R independent pipelines (each its own x0 / x1 / coeff) are stepped round-robin so the fields
    stream from HBM (R sets > 4x L2).  Cross-process correctness: tests/test_gpu_pipeline_ipc.py."""
    host = synth.make_inputs("hdiff", domain, seed=0)
    per = 3 * (domain[0] + 4) * (domain[1] + 4) * domain[2] * 8
    R = max(2, math.ceil(4 * l2 / per) + 1)
    pipes = []
    for _ in range(R):
        x0 = oec.field_from_host(host["in"])
        x1 = oec.field_from_host(host["in"])
        cf = oec.field_from_host(host["coeff"])
        pipes.append(oec.HdiffPipeline(domain, 1, 1, 0, cf, x0, x1))
    for p in pipes:
        p.run(1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for p in pipes:
            p.run(1)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = 1e3 * a.elapsed_time(b) / (reps * R)
    nbytes = hdiff_bytes(*domain)
    del pipes, g
    return {"us_per_step": us, "algorithmic_bytes": nbytes, "GB/s": nbytes / (us * 1e-6) / 1e9,
            "frac_of_hbm_peak": nbytes / (us * 1e-6) / 1e9 / peak, "pipelines": R,
            "note": "one rank (no neighbours); steps of R independent pipelines round-robin, fields > 4x L2"}


def paper_sizes_measure(oec, torch, l2, peak):
    """The paper's own problem sizes, 128x128x60 and 256x256x60, for every
    program (default kernels: hand-written hdiff/vadv, the tuned compiler output for the suite)."""
    return {"x".join(map(str, dom)): {p: program_measure(oec, torch, p, dom, l2, peak) for p in synth.ALL_PROGRAMS}
            for dom in ((128, 128, 60), (256, 256, 60))}


def levels_measure(oec, torch, domain, l2, peak):
    """The paper's optimisation-level experiment (Fig. 11) on B200, every program:
    "original" (one kernel per stencil.apply, temporaries in HBM), "inline" in the paper's execution
    model (one thread per point -- vadv: per column -- producers recomputed), "inline+unroll(2/4)"
    (stencil unrolling along j), and, for hdiff and vadv, this repo's tuned kernels (for the
    other programs the default kernel is the inline level with the empirically best unroll factor,
    P:621)."""
    res = {}
    for program in synth.ALL_PROGRAMS:
        variants = [("original", 1), ("inline", 2)]
        if program != "vadv":
            variants += [("inline_unroll2", 3), ("inline_unroll4", 4)]
        if program in ("hdiff", "vadv"):
            variants += [("b200", 0)]
        r = {name: program_measure(oec, torch, program, domain, l2, peak, v) for name, v in variants}
        base = r["original"]["us_per_launch"]
        for name in r:
            r[name]["speedup_over_original"] = base / r[name]["us_per_launch"]
        r["best"] = min(r, key=lambda n: r[n]["us_per_launch"])
        res[program] = r
    return res


if __name__ == "__main__":
    sys.exit(main())
