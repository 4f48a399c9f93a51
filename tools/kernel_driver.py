"""Launch one program's kernel eagerly a few times on rotating input sets (for ncu captures).

    python tools/kernel_driver.py --program hdiff --domain 128 128 80 --reps 6 [--variant 0]
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--program", default="hdiff")
    ap.add_argument("--domain", type=int, nargs=3, default=[128, 128, 80])
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--sets", type=int, default=4)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--text", action="store_true", help="run the stencil-language version (tests/programs) via the JIT")
    a = ap.parse_args()
    import torch

    from paper_2005_13014_b200 import oec

    dom = tuple(a.domain)
    host = synth.make_inputs(a.program, dom, seed=0)
    spec = synth.PROGRAMS[a.program]
    sc = [v for _, v in spec.scalars]
    sets = []
    for _ in range(a.sets):
        ins = [oec.field_from_host(host[s.name]) for s in spec.inputs]
        outs = [oec.empty_like_domain(dom, fill=0.0) for _ in spec.outputs]
        sets.append((ins, outs))
    name = a.program
    if a.text:
        with open(os.path.join(ROOT, "tests", "programs", a.program + ".oec")) as f:
            name = oec.oec_program_create(f.read())
    for r in range(a.reps):
        ins, outs = sets[r % a.sets]
        oec.oec_apply_program(name, ins, outs, sc, (0, 0, 0), dom, a.variant)
    torch.cuda.synchronize()
    print("done", a.program, dom, a.reps)


if __name__ == "__main__":
    main()
