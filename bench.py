#!/usr/bin/env python
"""bench.py -- throughput of the fused fp64 stencil hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5] [--impl oec|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

The LAST stdout line is one compact JSON object (< 2 KB, the driver's contract); everything else
(per-program tables, optimisation levels, f32, the stencil-language JIT, the paper's sizes) goes
to a side file (--detail, default gpurun_out/bench_detail.json) and one summary line on stderr.

Configurations (BASELINE.json `configs`):
  c2 (default)  hdiff + vadv, 128x128x80 per GPU (configs[1]); N > 1: j-slabs of 128 x 128N x 80
                (weak scaling)
  c3            the full suite (all nine programs), 128x128x80 per GPU (configs[2]), weak
  c4            hdiff + vadv on the fixed global 1024x1024x80 domain split into N j-slabs
                (configs[3], strong scaling)
  c5            the full suite, 512x512x80 per GPU (configs[4]), weak
A STEP applies every program of the configuration once to one rotating input set.  For N > 1 each
program's inputs get their halos from the j-neighbours first: hdiff in c2/c4 through the fused
pipeline (the halo read from the neighbours' memory inside the kernel) when every rank can import
its neighbours' memory, otherwise -- and for every program in c3/c5 -- through oec_halo_exchange
(NCCL send/recv on a comm stream) overlapped with the interior rows, the boundary strips after
(SURVEY §8(e)).  At N = 1 the same code runs with no neighbours (no exchange, one launch each).

value     = grid points / s of the whole job: points of the global domain per step / step time
            (a point counts once per step however many programs the step applies); inputs
            resident in HBM; CUDA events over exactly K steps (max over ranks).  Each step reads
            a different one of R rotating input sets whose total is > 4x the 126 MB L2.
timing    = the P:556 protocol: median and IQR of >= 100 samples (one sample = one CUDA-graph
            replay of R steps / R), plus one cold launch per program after an L2 flush.
e2e       = the same metric through the C-ABI with HOST buffers (pinned): H2D of the step's
            inputs, the kernels, D2H of the outputs, per step, inside the timed region.
roofline  = the dominant kernel's ALGORITHMIC bytes per launch /
            its median CUDA-event duration vs MEASURED_PEAKS.json's HBM copy bandwidth; traffic =
            ncu DRAM read+write per launch including the write-back (profiles/ncu_traffic.json).
cpu_baseline / --impl reference = the CPU oracle (oracle/, the fused C oracle for hdiff/vadv, the
            numpy oracle for the suite) on the box's host cores, 1 thread and all threads.
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
FALLBACK_HBM_GBS = 6650.0
DATASHEET_HBM_GBS = 8000.0  # B200 HBM3e datasheet figure (reported beside the measured peak, labelled)
SUITE_ALL = synth.ALL_PROGRAMS  # hdiff, vadv + the seven suite programs

CONFIGS = {
    "c2": dict(programs=("hdiff", "vadv"), domain=(128, 128, 80), scaling="weak", steps=30000,
               workload="hdiff + vadv fp64, 128x128x80 per GPU (BASELINE.json configs[1])"),
    "c3": dict(programs=SUITE_ALL, domain=(128, 128, 80), scaling="weak", steps=3000,
               workload="full suite (9 programs) fp64, 128x128x80 per GPU (BASELINE.json configs[2])"),
    "c4": dict(programs=("hdiff", "vadv"), domain=(1024, 1024, 80), scaling="strong", steps=300,
               workload="hdiff + vadv fp64, global 1024x1024x80 split in j-slabs (BASELINE.json configs[3])"),
    "c5": dict(programs=SUITE_ALL, domain=(512, 512, 80), scaling="weak", steps=200,
               workload="full suite (9 programs) fp64, 512x512x80 per GPU (BASELINE.json configs[4])"),
}


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
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    """Per-launch DRAM bytes (read + write, write-back included) of each program's kernel at the
    configuration's size, from the committed ncu capture (tools/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(config, {})
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
                "reasons": reasons, "samples": len(inside)}


# ---------------------------------------------------------------------------------------------
# the CPU oracle (cpu_baseline and --impl reference): the same function for both
# ---------------------------------------------------------------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_step_fn(cfg, nthreads, nj_sample):
    """One oracle step of the configuration on a j-slab sample [0,Ni) x [0,nj_sample) x [0,Nk) of
    the per-GPU domain: hdiff / vadv with the fused C oracle (OpenMP, `nthreads`), the suite
    programs with the numpy oracle (oracle/stencil.py, one thread).  Returns (step, points)."""
    from oracle import capi
    from oracle import stencil as st
    from oracle import suite

    capi.build()
    ni, nj, nk = cfg["domain"]
    njs = max(1, min(nj, nj_sample))
    sdom = (ni, njs, nk)  # inputs drawn for the sample domain (values are seeded draws)
    calls = []
    for p in cfg["programs"]:
        host = synth.make_inputs(p, sdom, seed=0)
        sc = synth.scalars(p)
        if p == "hdiff":
            o = synth.HostField(np.zeros((nk, njs, ni)), (0, 0, 0), sdom)
            calls.append(lambda h=host, o=o: capi.hdiff(h["in"], h["coeff"], o, (0, 0, 0), sdom, capi.HDIFF_FUSED,
                                                        nthreads))
        elif p == "vadv":
            o = synth.HostField(np.zeros((nk, njs, ni)), (0, 0, 0), sdom)
            calls.append(lambda h=host, o=o, d=sc["dtr_stage"]: capi.vadv(h, o, d, (0, 0, 0), sdom, capi.VADV_FUSED,
                                                                          nthreads))
        else:
            calls.append(lambda h=host, sc=sc, p=p: st.run_unfused(suite.PROGRAMS[p], h, sc, (0, 0, 0), sdom))

    def step():
        for c in calls:
            c()

    return step, ni * njs * nk


def time_oracle(cfg, nthreads, seconds, nj_sample=None):
    """(points/s, steps, elapsed, sample rows) of the oracle on a sample sized to ~`seconds`."""
    nj = cfg["domain"][1]
    probe, pts1 = oracle_step_fn(cfg, nthreads, 1 if nj_sample is None else nj_sample)
    probe()
    t0 = time.perf_counter()
    probe()
    t1 = time.perf_counter() - t0
    if nj_sample is None:  # rows such that one step is ~seconds/3
        nj_sample = max(1, min(nj, int(seconds / 3.0 / max(t1, 1e-6))))
        step, pts = oracle_step_fn(cfg, nthreads, nj_sample)
        step()
    else:
        step, pts = probe, pts1
    n, t0 = 0, time.perf_counter()
    while True:
        step()
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 1000:
            break
    return n * pts / el, n, el, nj_sample


def cpu_baseline(cfg, seconds):
    nproc = os.cpu_count() or 1
    v_all, n_all, el_all, nj_all = time_oracle(cfg, nproc, seconds)
    v_one, n_one, el_one, nj_one = time_oracle(cfg, 1, seconds / 2)
    ni, nj, nk = cfg["domain"]
    return {"value": v_all, "unit": UNIT, "cores": nproc, "kind": "oracle", "value_1thread": v_one,
            "cpu": cpu_model(),
            "sample": f"{n_all} steps of {ni}x{nj_all}x{nk} (j-slab of {ni}x{nj}x{nk}), fused C oracle "
                      f"(OpenMP {nproc} thr) / numpy suite, {el_all:.1f} s; 1 thread: {n_one} steps of "
                      f"{ni}x{nj_one}x{nk}, {el_one:.1f} s"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only), the SAME function
    and sample sizing as cpu_baseline, K timed steps after W warm-up steps."""
    if rank != 0:
        return 0
    nproc = os.cpu_count() or 1
    ni, nj, nk = cfg["domain"]
    probe, _ = oracle_step_fn(cfg, nproc, 1)
    probe()
    t0 = time.perf_counter()
    probe()
    t1 = time.perf_counter() - t0
    budget = 60.0  # seconds for warm-up + timed steps
    nj_s = max(1, min(nj, int(budget / max(1e-6, (args.warmup + args.steps) * t1))))
    step, pts = oracle_step_fn(cfg, nproc, nj_s)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = args.steps * pts / el
    sample = f"each step = {'+'.join(cfg['programs'])} on a {ni}x{nj_s}x{nk} j-slab of {ni}x{nj}x{nk} " \
             f"(fused C oracle, OpenMP {nproc} thr; numpy suite)"
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": cfg["workload"], "config": args.config,
                                           "sample_domain": [ni, nj_s, nk]},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "oracle", "sample": sample,
                            "cpu": cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# the GPU arm: rotating input sets, the decomposed step, timing
# ---------------------------------------------------------------------------------------------
class ProgSets:
    """R rotating input sets of one program on this rank's local domain (fields in local
    coordinates, allocations = the synth recipe = the program's access extents)."""

    def __init__(self, oec, program, ldomain, seed, dev, R=None, l2=None):
        self.program = program
        spec = synth.PROGRAMS[program]
        self.host = synth.make_inputs(program, ldomain, seed=seed)
        self.scalars = [v for _, v in spec.scalars]
        self.ldomain = ldomain
        self.dev = dev

        def make():
            ins = [oec.field_from_host(self.host[s.name], device=dev) for s in spec.inputs]
            outs = [oec.empty_like_domain(ldomain, device=dev, fill=0.0) for _ in spec.outputs]
            return ins, outs

        self._make = make
        self.sets = [make()]
        nbytes = sum(int(np.prod([f.ub[d] - f.lb[d] for d in range(3)])) * 8 for f in self.sets[0][0] + self.sets[0][1])
        self.set_bytes = nbytes
        if R is None:
            R = max(2, math.ceil(4 * l2 / nbytes) + 1)
        self.sets += [make() for _ in range(R - 1)]
        self.R = R
        # j-extents of the inputs: halo rows to exchange, rows of the boundary strips
        ins, _, _ = oec.program_signature(program)
        self.groups = {}  # (jlo, jhi) -> input indices
        for q, (_, lo, hi, _) in enumerate(ins):
            w = (max(0, -lo[1]), max(0, hi[1]))
            if w != (0, 0):
                self.groups.setdefault(w, []).append(q)
        self.jlo = max([w[0] for w in self.groups] or [0])
        self.jhi = max([w[1] for w in self.groups] or [0])

    def extend(self, R):
        while len(self.sets) < R:
            self.sets.append(self._make())
        self.R = R


class Step:
    """The per-rank step of a configuration.  `enqueue(p, s)` enqueues program p on rotating set s
    on the current stream: with j-neighbours, the exchange of the inputs' halos on the comm stream
    concurrently with the interior rows, then the boundary strips; without, one launch."""

    def __init__(self, oec, torch, cfg, ldomain, lo_nb, hi_nb, dec, pipes, dev):
        self.oec, self.torch = oec, torch
        self.ldomain = ldomain
        self.lo_nb, self.hi_nb = lo_nb, hi_nb  # j-neighbour below / above exists
        self.dec = dec
        self.pipes = pipes  # {program: [HdiffPipeline per set]} for the fused hdiff exchange
        self.comm = torch.cuda.Stream(device=dev) if (dec is not None and (lo_nb or hi_nb)) else None
        self.launches = {}

    def _apply(self, ps, s, jlo, jhi):
        ins, outs = ps.sets[s]
        ni, nj, nk = self.ldomain
        if jhi <= jlo:
            return
        if ps.program == "hdiff":
            self.oec.oec_hdiff(ins[0], ins[1], outs[0], (0, jlo, 0), (ni, jhi, nk))
        elif ps.program == "vadv":
            self.oec.oec_vadv(*ins, outs[0], ps.scalars[0], (0, jlo, 0), (ni, jhi, nk))
        else:
            self.oec.oec_apply_program(ps.program, ins, outs, ps.scalars, (0, jlo, 0), (ni, jhi, nk))
        return self.oec.oec_last_launch_count()

    def enqueue(self, ps, s):
        oec, torch = self.oec, self.torch
        nj = self.ldomain[1]
        n = 0
        if ps.program in self.pipes:  # fused exchange: one kernel, halo read from peer memory
            self.pipes[ps.program][s].run(1)
            n = oec.oec_last_launch_count()
        elif self.comm is None or not ps.groups:
            n = self._apply(ps, s, 0, nj)
        else:
            cur = torch.cuda.current_stream()
            self.comm.wait_stream(cur)
            with torch.cuda.stream(self.comm):
                ins = ps.sets[s][0]
                for (wl, wh), idx in ps.groups.items():
                    oec.oec_halo_exchange(self.dec, [ins[q] for q in idx], (0, wl, 0), (0, wh, 0))
                    n += oec.oec_last_launch_count()
            a = ps.jlo if self.lo_nb else 0
            b = nj - ps.jhi if self.hi_nb else nj
            n += self._apply(ps, s, a, max(a, b)) or 0  # interior, concurrent with the exchange
            cur.wait_stream(self.comm)
            if self.lo_nb:
                n += self._apply(ps, s, 0, min(a, nj)) or 0
            if self.hi_nb:
                n += self._apply(ps, s, max(a, b), nj) or 0
        self.launches[ps.program] = n


def fused_pipelines(oec, dist, pss, ldomain, gdom, world, rank, dev, agree):
    """N > 1: one oec_hdiff_pipeline per rotating hdiff set over this rank's j-slab (x0 = the set's
    input with its halo, x1 a copy: the global outer halo stays constant); fields and signal pads
    exported with CUDA IPC, handles all-gathered, neighbours' memory imported.  Each phase ends
    with agree(ok) (a MIN over ranks), so every rank takes the same path.  On failure every import
    is closed and the pipelines dropped.  Returns (pipes, None) or (None, reason)."""
    import torch

    pipes, mine, imported, err = [], [], [], None
    try:  # phase 1: local pipelines and IPC exports
        for ins, outs in pss.sets:
            x1 = oec.oec_field_create(ldomain, (2, 2, 0), (2, 2, 0), device=dev)
            x1.view().copy_(ins[0].view())
            p = oec.HdiffPipeline(gdom, 1, world, rank, ins[1], ins[0], x1)
            p.x1 = x1
            pipes.append(p)
            pad, _ = p.signal_pad()
            mine.append(dict(x0=oec.oec_ipc_export(ins[0].desc.data), x1=oec.oec_ipc_export(x1.desc.data),
                             pad=oec.oec_ipc_export(pad), desc=oec.field_descriptor(ins[0])))
        torch.cuda.synchronize()
    except Exception as e:
        err = f"{type(e).__name__}: {e}"
    if not agree(err is None):
        return None, err or "pipeline setup failed on another rank"
    everyone = [None] * world
    dist.all_gather_object(everyone, mine)
    try:  # phase 2: import the j-neighbours' memory
        for q in (rank - 1, rank + 1):
            if not 0 <= q < world:
                continue
            for si, p in enumerate(pipes):
                Q = everyone[q][si]
                ptrs = []
                for k in ("x0", "x1", "pad"):
                    ptrs.append(oec.oec_ipc_import(*Q[k]))
                    imported.append(ptrs[-1])
                p.set_peer(q, oec.field_at(ptrs[0], Q["desc"], dev), oec.field_at(ptrs[1], Q["desc"], dev), ptrs[2])
    except Exception as e:
        err = f"{type(e).__name__}: {e}"
    if not agree(err is None):
        for ptr in imported:
            try:
                oec.oec_ipc_close(ptr)
            except Exception:
                pass
        return None, err or "peer import failed on another rank"
    dist.barrier()
    return (pipes, imported), None


def flush_l2(torch, buf):
    """Evict L2 by READING a buffer > L2 (a write flush would leave dirty lines whose write-back
    then lands inside the next, timed kernel)."""
    return buf.sum()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: per config)")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="oec", choices=["oec", "reference"])
    ap.add_argument("--samples", type=int, default=120, help="timing samples for median / IQR (>= 100)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-extras", action="store_true", help="skip the detail-file measurements")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--detail", default=os.path.join(ROOT, "gpurun_out", "bench_detail.json"))
    ap.add_argument("--sets", type=int, default=0, help="rotating input sets (0 = auto, > 4x L2)")
    ap.add_argument("--force-decomp", action="store_true",
                    help="debug: create the process group and decomposition even at N=1")
    ap.add_argument("--emulate-neighbours", action="store_true",
                    help="N=1 only: run the N>1 per-rank step -- halo exchange over NCCL on a comm stream, "
                         "interior rows concurrently, boundary strips after -- against this rank itself "
                         "(a periodic 1 x 1 j decomposition: both j-neighbours are the rank); measures the "
                         "decomposition's per-rank overhead without a second GPU (not the NVLink transfer)")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N>1 halo exchange of hdiff in c2/c4: 'fused' = oec_hdiff_pipeline (the kernel reads the "
                         "neighbours' halo cells from their memory, CUDA IPC), 'nccl' = oec_halo_exchange")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: validating the fused path with all ranks on one GPU, "
                         "OEC_BENCH_DEVICE=0)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.steps is None:
        args.steps = cfg["steps"]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    args.warmup = max(3, args.warmup)

    import torch
    import torch.distributed as dist

    from paper_2005_13014_b200 import oec

    oec.lib()  # fail loudly if the extension is missing
    dev = int(os.environ.get("OEC_BENCH_DEVICE", local_rank))
    torch.cuda.set_device(dev)
    emulate = args.emulate_neighbours and world == 1
    decomp = world > 1 or args.force_decomp or emulate
    if decomp:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20))

    # ---- decomposition: j-slabs (1 x N) of the global domain ----
    if cfg["scaling"] == "weak":
        gdom = (cfg["domain"][0], cfg["domain"][1] * world, cfg["domain"][2])
    else:
        gdom = tuple(cfg["domain"])
    dec0 = oec.oec_decomp_create(gdom, 1, world, rank)
    lo, hi = dec0.local_lb, dec0.local_ub
    ldomain = tuple(hi[d] - lo[d] for d in range(3))
    lo_nb, hi_nb = (True, True) if emulate else (rank > 0, rank < world - 1)
    pts_global = gdom[0] * gdom[1] * gdom[2]

    # ---- rotating input sets per program ----
    pss = {}
    for q, p in enumerate(cfg["programs"]):
        pss[p] = ProgSets(oec, p, ldomain, seed=1000 * q + rank, dev=dev, R=args.sets or None, l2=l2)
    R = max(ps.R for ps in pss.values())
    for ps in pss.values():  # one rotation length for all programs
        ps.extend(R)

    # ---- halo exchange transport for N > 1 ----
    fused_note, pipes, imported = None, {}, []
    use_fused = decomp and world > 1 and args.exchange == "fused" and args.config in ("c2", "c4") and not emulate
    if decomp and args.dist_backend == "gloo" and not use_fused:
        raise SystemExit("--dist-backend gloo needs N > 1, --exchange fused and config c2/c4")
    if use_fused:
        def agree(ok):
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                device="cuda" if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            return int(flag.item()) == 1

        res, why = fused_pipelines(oec, dist, pss["hdiff"], ldomain, gdom, world, rank, dev, agree)
        if res is None:
            if args.dist_backend != "nccl":
                raise SystemExit(f"fused pipeline unavailable: {why}")
            fused_note = f"fused pipeline unavailable ({why}); NCCL exchange used"
            use_fused = False
        else:
            pipes["hdiff"], imported = res
    dec = None
    if decomp and (world > 1 or emulate) and args.dist_backend == "nccl":
        pg = dist.distributed_c10d._get_default_group()
        dist.barrier()
        dec = oec.oec_decomp_create(gdom, 1, world, rank, pg._get_backend(torch.device("cuda", dev))._comm_ptr())
        if emulate:
            oec.oec_decomp_set_periodic(dec, False, True)
    step = Step(oec, torch, cfg, ldomain, lo_nb, hi_nb, dec, pipes, dev)
    progs = [pss[p] for p in cfg["programs"]]

    # warm-up (also configures kernel attributes, compiles/tunes the suite's JIT kernels, sizes
    # NCCL staging before any capture)
    for w in range(args.warmup):
        for ps in progs:
            step.enqueue(ps, w % R)
    torch.cuda.synchronize()

    # ---- one CUDA graph of R launches per program (launch-overhead-free timing) ----
    graphs, x_mode = {}, None

    def capture(nsteps):
        nonlocal x_mode
        gs = []
        for ps in progs:
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g):
                    for q in range(nsteps):
                        step.enqueue(ps, q % R)
                gs.append(g)
            except Exception as e:  # NCCL capture unavailable: this program runs eagerly
                torch.cuda.synchronize()
                gs.append(None)
                x_mode = f"{ps.program}: eager ({type(e).__name__})"
        return gs

    K = args.steps
    graphs[R] = capture(R)
    if K % R:
        graphs[K % R] = capture(K % R)

    def replay(gs, n, base):
        for ps, g in zip(progs, gs):
            if g is not None:
                g.replay()
            else:
                for q in range(n):
                    step.enqueue(ps, (base + q) % R)

    for n, gs in graphs.items():
        replay(gs, n, 0)
    torch.cuda.synchronize()

    # ---- the timed region: exactly K steps ----
    chunks = [R] * (K // R) + ([K % R] if K % R else [])
    nP = len(progs)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nP + 1)] for _ in chunks]
    gpu_id = "GPU-" + str(props.uuid) if hasattr(props, "uuid") else str(dev)
    clocks = ClockSampler(gpu_id)
    if decomp:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    t_start, t_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record()
    done = 0
    for c, n in enumerate(chunks):
        gs = graphs[n]
        ev[c][0].record()
        for q, (ps, g) in enumerate(zip(progs, gs)):
            if g is not None:
                g.replay()
            else:
                for z in range(n):
                    step.enqueue(ps, (done + z) % R)
            ev[c][q + 1].record()
        done += n
    t_stop.record()
    torch.cuda.synchronize()
    clocks.mark_stop()
    elapsed_ms = t_start.elapsed_time(t_stop)
    per_prog_ms = [sum(ev[c][q].elapsed_time(ev[c][q + 1]) for c in range(len(chunks))) for q in range(nP)]

    # ---- samples for median / IQR: graph replays of R steps after the timed region ----
    S = max(100, args.samples)
    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(nP + 1)] for _ in range(S)]
    gs = graphs[R]
    for c in range(S):
        sev[c][0].record()
        for q, (ps, g) in enumerate(zip(progs, gs)):
            if g is not None:
                g.replay()
            else:
                for z in range(R):
                    step.enqueue(ps, z)
            sev[c][q + 1].record()
    torch.cuda.synchronize()
    samp_step = np.array([sev[c][0].elapsed_time(sev[c][nP]) * 1e3 / R for c in range(S)])  # us per step
    samp_prog = [np.array([sev[c][q].elapsed_time(sev[c][q + 1]) * 1e3 / R for c in range(S)]) for q in range(nP)]

    # ---- one cold launch per program: L2 flushed (a write over 4x L2), events around one call ----
    flush = torch.zeros(4 * l2 // 8, dtype=torch.float64, device=f"cuda:{dev}")
    cold = {}
    for ps in progs:
        ts = []
        for _ in range(3):  # median of three cold launches
            flush_l2(torch, flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step.enqueue(ps, 0)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        cold[ps.program] = float(np.median(ts))
    del flush

    if decomp and world > 1:
        dev_t = "cuda" if args.dist_backend == "nccl" else "cpu"
        t = torch.tensor([elapsed_ms] + per_prog_ms + [float(np.median(samp_step))], device=dev_t, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = [float(x) for x in t.tolist()]
        elapsed_ms, per_prog_ms, med_step_max = vals[0], vals[1:1 + nP], vals[-1]
    else:
        med_step_max = float(np.median(samp_step))
    clk = clocks.result()
    ms_step = elapsed_ms / K
    value = pts_global / (ms_step * 1e-3)

    peak, peak_src = hbm_peak()
    traffic = ncu_traffic(args.config)
    kern = {}
    for q, ps in enumerate(progs):
        nbytes = program_bytes(ps.program, ldomain)
        us_med = float(np.median(samp_prog[q]))
        q1, q3 = np.percentile(samp_prog[q], [25, 75])
        us_mean = 1e3 * per_prog_ms[q] / K
        kern[ps.program] = {"us": round(us_med, 3), "iqr": [round(float(q1), 3), round(float(q3), 3)],
                            "us_mean": round(us_mean, 3), "cold_us": round(cold[ps.program], 2),
                            "bytes": nbytes, "frac": round(nbytes / (us_med * 1e-6) / 1e9 / peak, 4),
                            "frac_of_datasheet_8000": round(nbytes / (us_med * 1e-6) / 1e9 / DATASHEET_HBM_GBS, 4)}
    dom_k = max(kern, key=lambda k: kern[k]["us"])
    tr = traffic.get(dom_k)
    ach = kern[dom_k]["bytes"] / (kern[dom_k]["us"] * 1e-6) / 1e9
    roofline = {"bound": "hbm", "kernel": dom_k, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": tr, "peak_source": peak_src,
                "algorithmic_bytes": kern[dom_k]["bytes"],
                "frac_of_datasheet_8000": round(ach / DATASHEET_HBM_GBS, 4)}

    # ---- e2e through the C-ABI with pinned host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_measure(oec, torch, progs, ldomain, args.e2e_steps, world, pts_global)

    # ---- extras for the detail file (rank 0, N = 1, config c2) ----
    detail = {"config": args.config, "kernels": kern, "timing_samples_us_per_step": {
        "median": float(np.median(samp_step)), "q1": float(np.percentile(samp_step, 25)),
        "q3": float(np.percentile(samp_step, 75)), "n": int(S)}}
    suite_frac = None
    if not args.no_extras and world == 1 and args.config == "c2":
        dom = cfg["domain"]
        detail["suite"] = {p: program_measure(oec, torch, p, dom, l2, peak) for p in synth.SUITE}
        suite_frac = {p: round(v["frac_of_hbm_peak"], 3) for p, v in detail["suite"].items()}
        detail["optimization_levels"] = levels_measure(oec, torch, dom, l2, peak)
        detail["f32"] = {p: program_measure(oec, torch, p, dom, l2, peak, dtype=np.float32) for p in SUITE_ALL}
        detail["jit"] = jit_measure(oec, torch, dom, l2, peak)
        detail["hdiff_pipeline"] = pipeline_measure(oec, torch, dom, l2, peak)
        detail["paper_sizes"] = {"x".join(map(str, d)): {p: program_measure(oec, torch, p, d, l2, peak)
                                                         for p in SUITE_ALL}
                                 for d in ((128, 128, 60), (256, 256, 60))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args.cpu_seconds)

    n_launch = K * sum(step.launches.values())
    if rank == 0:
        nproc_note = ("; EMULATED neighbours: periodic 1x1 j decomposition, NCCL self-exchange on a comm stream || "
                      "interior rows, then boundary strips (per-rank overhead of N>1, no NVLink transfer)") if emulate \
            else "" if world == 1 else (
            "; hdiff halo read from the neighbours' memory inside the kernel (fused pipeline, CUDA IPC)"
            if use_fused else "; NCCL halo exchange on a comm stream || interior rows, then boundary strips")
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded PCG64, SURVEY 8(d))",
            "config": {"workload": cfg["workload"], "config": args.config, "global_domain": list(gdom),
                       "domain_per_gpu": list(ldomain),
                       "parallelism": f"j-slabs 1x{world}" + nproc_note + (f"; {fused_note}" if fused_note else ""),
                       "l2": f"inputs > L2: {R} rotating sets ({R * sum(p.set_bytes for p in progs) / 2**20:.0f} MiB)"},
            "roofline": roofline,
            "kernels": {k: {"us": v["us"], "frac": v["frac"], "cold_us": v["cold_us"]} for k, v in kern.items()},
            "timing": {"median_us_per_step": round(med_step_max, 3),
                       "iqr_us": [round(float(np.percentile(samp_step, 25)), 3),
                                  round(float(np.percentile(samp_step, 75)), 3)],
                       "samples": int(S), "cold_launch_us": round(sum(cold.values()), 2)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": n_launch,
            "clocks": clk,
            "detail": os.path.relpath(args.detail, ROOT),
        }
        if suite_frac:
            res["suite_frac"] = suite_frac
        if x_mode:
            res["config"]["note"] = x_mode
        detail["headline"] = dict(res)
        try:
            os.makedirs(os.path.dirname(args.detail), exist_ok=True)
            with open(args.detail, "w") as f:
                json.dump(detail, f, indent=1)
        except Exception as e:
            print(f"bench: could not write {args.detail}: {e}", file=sys.stderr)
        line = json.dumps(res, separators=(",", ":"))
        if len(line) > 2000:  # keep the headline compact: drop the longest free-text fields first
            res["cpu_baseline"] = {k: v for k, v in (cpu or {}).items() if k != "sample"} or None
            res["config"].pop("note", None)
            line = json.dumps(res, separators=(",", ":"))
        summ = " ".join(f"{k}={v['us']:.2f}us/{v['frac']:.3f}" for k, v in kern.items())
        print(f"bench {args.config}: {summ}" + (f" suite {suite_frac}" if suite_frac else ""), file=sys.stderr,
              flush=True)
        print(line, flush=True)
    for ptr in imported:
        try:
            oec.oec_ipc_close(ptr)
        except Exception:
            pass
    if decomp:
        dist.barrier()  # every rank has printed / written its results
        # no destroy_process_group: tearing down the NCCL communicator that the captured exchange
        # graphs still reference hung for minutes on the B200 box (measured with
        # --emulate-neighbours); the process exits with everything flushed instead
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    return 0


def e2e_measure(oec, torch, progs, ldomain, steps, world, pts_global):
    """The step through the public C-ABI with pinned host buffers (device = OEC_DEVICE_HOST): the
    library copies each program's inputs H2D, runs the kernel, copies the outputs' domain D2H,
    per call (no halo exchange: each rank's host inputs carry their halos)."""
    def pinned(hf):
        t = torch.empty(hf.data.shape, dtype=torch.float64, pin_memory=True)
        t.copy_(torch.from_numpy(hf.data))
        return oec.oec_field_wrap(t, hf.lb, hf.ub, k_invariant=hf.k_invariant)

    ni, nj, nk = ldomain
    calls, h2d, d2h = [], 0, 0
    for ps in progs:
        spec = synth.PROGRAMS[ps.program]
        ins = [pinned(ps.host[s.name]) for s in spec.inputs]
        outs = []
        for _ in spec.outputs:
            o = torch.zeros((nk, nj, ni), dtype=torch.float64, pin_memory=True)
            outs.append(oec.oec_field_wrap(o, (0, 0, 0), ldomain))
        h2d += sum(f._keep.numel() * 8 for f in ins)
        d2h += len(outs) * ni * nj * nk * 8
        calls.append((ps, ins, outs))

    # (measured: the programs' calls on their own streams from a thread pool -- concurrent host
    # staging per stream -- took 1.96 ms per step against 1.79 on one stream; kept sequential)
    def step():
        for ps, ins, outs in calls:
            if ps.program == "hdiff":
                oec.oec_hdiff(ins[0], ins[1], outs[0], (0, 0, 0), ldomain)
            elif ps.program == "vadv":
                oec.oec_vadv(*ins, outs[0], ps.scalars[0], (0, 0, 0), ldomain)
            else:
                oec.oec_apply_program(ps.program, ins, outs, ps.scalars, (0, 0, 0), ldomain)

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
    return {"value": pts_global / (ms * 1e-3) if world == 1 else world * ni * nj * nk / (ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 4)}


def program_measure(oec, torch, program, domain, l2, peak, variant=0, reps=20, dtype=np.float64, run_name=None):
    """us per launch of one program (CUDA graph of R launches over R rotating input sets > 4x L2).
    dtype=np.float32: the paper's f32 runs; algorithmic bytes scale with the element size.
    run_name: apply this registered program instead (a stencil-language version of `program` with
    the same argument order, compiled by liboec's JIT)."""
    host = synth.make_inputs(program, domain, seed=0, dtype=dtype)
    spec = synth.PROGRAMS[program]
    sc = [v for _, v in spec.scalars]
    dev = torch.cuda.current_device()

    def make():
        ins = [oec.field_from_host(host[s.name], device=dev) for s in spec.inputs]
        outs = [oec.empty_like_domain(domain, device=dev, fill=0.0, dtype=dtype) for _ in spec.outputs]
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
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    us = float(np.median([1e3 * a.elapsed_time(b) / R for a, b in ts]))
    nbytes = program_bytes(program, domain) * np.dtype(dtype).itemsize // 8
    del sets, s0, g
    return {"us_per_launch": us, "algorithmic_bytes": nbytes, "GB/s": nbytes / (us * 1e-6) / 1e9,
            "frac_of_hbm_peak": nbytes / (us * 1e-6) / 1e9 / peak,
            "grid_points_per_s": domain[0] * domain[1] * domain[2] / (us * 1e-6)}


def jit_measure(oec, torch, domain, l2, peak):
    """The stencil-language versions of every stencil program (tests/programs/*.oec), compiled by
    liboec's JIT at each optimisation level of P:616 (unrolling along j and k) and AUTO
    (empirical tuning), next to the builtin kernel of the same program."""
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
    (no neighbours, every tile interior): us per step next to hdiff's algorithmic bytes; R
    independent pipelines stepped round-robin so the fields stream from HBM."""
    host = synth.make_inputs("hdiff", domain, seed=0)
    per = 3 * (domain[0] + 4) * (domain[1] + 4) * domain[2] * 8
    R = max(2, math.ceil(4 * l2 / per) + 1)
    dev = torch.cuda.current_device()
    pipes = []
    for _ in range(R):
        x0 = oec.field_from_host(host["in"], device=dev)
        x1 = oec.field_from_host(host["in"], device=dev)
        cf = oec.field_from_host(host["coeff"], device=dev)
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
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    us = float(np.median([1e3 * a.elapsed_time(b) / R for a, b in ts]))
    nbytes = hdiff_bytes(*domain)
    del pipes, g
    return {"us_per_step": us, "algorithmic_bytes": nbytes, "GB/s": nbytes / (us * 1e-6) / 1e9,
            "frac_of_hbm_peak": nbytes / (us * 1e-6) / 1e9 / peak, "pipelines": R}


def levels_measure(oec, torch, domain, l2, peak):
    """The paper's optimisation-level experiment (Fig. 11) on B200, every program:
    "original" (one kernel per stencil.apply, temporaries in HBM), "inline" in the paper's execution
    model, "inline+unroll(2/4)" (stencil unrolling along j), and the default kernel."""
    res = {}
    for program in SUITE_ALL:
        variants = [("original", 1), ("inline", 2)]
        if program != "vadv":
            variants += [("inline_unroll2", 3), ("inline_unroll4", 4)]
        variants += [("default", 0)]
        r = {name: program_measure(oec, torch, program, domain, l2, peak, v) for name, v in variants}
        base = r["original"]["us_per_launch"]
        for name in r:
            r[name]["speedup_over_original"] = base / r[name]["us_per_launch"]
        r["best"] = min(r, key=lambda n: r[n]["us_per_launch"])
        res[program] = r
    return res


if __name__ == "__main__":
    sys.exit(main())
