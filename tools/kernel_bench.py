"""Time one or more programs' kernels at a domain with rotating input sets (> 4x L2) and CUDA graphs.

    OEC_LIB_PATH=... python tools/kernel_bench.py --programs hdiff vadv --domain 128 128 80 [--variant 0]
Prints one JSON line per program: us per launch, algorithmic GB/s, fraction of the HBM peak.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from bench import hbm_peak, program_bytes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--programs", nargs="+", default=["hdiff", "vadv"])
    ap.add_argument("--domain", type=int, nargs=3, default=[128, 128, 80])
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--tag", default="")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--sets", type=int, default=0, help="rotating input sets (0: > 4x L2); 1 = L2-resident floor")
    a = ap.parse_args()
    import torch

    from paper_2005_13014_b200 import oec

    dom = tuple(a.domain)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    peak, _ = hbm_peak()
    for program in a.programs:
        if program == "copy":  # practical roofline at this size: torch copy_ of a 16 MiB buffer (32 MiB traffic)
            n = 2 * 2**20
            bufs = [(torch.rand(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda"))
                    for _ in range(12)]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for x, y in bufs:
                    y.copy_(x)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / (a.reps * len(bufs))
            print(json.dumps({"tag": a.tag, "program": "copy16MiB", "us": round(us, 3),
                              "GB/s": round(2 * n * 8 / (us * 1e-6) / 1e9, 1)}), flush=True)
            continue
        import numpy as np

        dt = np.float32 if a.dtype == "f32" else np.float64
        host = synth.make_inputs(program, dom, seed=0, dtype=dt)
        spec = synth.PROGRAMS[program]
        sc = [v for _, v in spec.scalars]

        def make():
            return ([oec.field_from_host(host[s.name]) for s in spec.inputs],
                    [oec.empty_like_domain(dom, fill=0.0, dtype=dt) for _ in spec.outputs])

        s0 = make()
        nb = sum(int(math.prod([f.ub[d] - f.lb[d] for d in range(3)])) * f.itemsize for f in s0[0] + s0[1])
        R = a.sets if a.sets > 0 else max(2, math.ceil(4 * l2 / nb) + 1)
        sets = [s0] + [make() for _ in range(R - 1)]
        for ins, outs in sets:
            oec.oec_apply_program(program, ins, outs, sc, (0, 0, 0), dom, a.variant)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        NL = max(R, 16)  # launches per graph (cycling through the sets)
        with torch.cuda.graph(g):
            for q in range(NL):
                ins, outs = sets[q % R]
                oec.oec_apply_program(program, ins, outs, sc, (0, 0, 0), dom, a.variant)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / (a.reps * NL)
        nbytes = program_bytes(program, dom) * np.dtype(dt).itemsize // 8
        gbs = nbytes / (us * 1e-6) / 1e9
        print(json.dumps({"tag": a.tag, "program": program, "domain": dom, "variant": a.variant, "dtype": a.dtype, "us": round(us, 3),
                          "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4), "sets": R}), flush=True)
        del sets, s0, g


if __name__ == "__main__":
    main()
