"""One case of the synchronising kernels, run under compute-sanitizer (racecheck / synccheck /
memcheck) by tools/sanitize.sh; each case also checks its result against the CPU oracle.

    python tools/sanitize.py CASE        CASE in CASES below

The cases cover every kernel that synchronises through mbarriers / TMA / TMEM / cross-CTA flags:
  hdiff_tma         hdiff, TMA-ring kernel (small-size configuration)
  hdiff_tma_large   hdiff, the >= 8M-point tile configuration
  hdiff_pipe        the fused-exchange pipeline, 2x1 ranks on one device, 3 steps
  hdiff_pipe_flip   the same with every step-parity guess inverted (the re-request path)
  vadv_sp           vadv, single wave (one column block per CTA, 5-chunk ring)
  vadv_sp_pers      vadv, persistent grid: CTAs walk several column blocks (ring + TMEM reuse)
  vadv_sp_multi     vadv, more CTAs than 12 per SM: 2D grid, 5-chunk ring
  jit_tiled         a suite program through the JIT's TMA-tiled variant
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import synth  # noqa: E402
from gpu_util import compare, run_gpu, run_oracle  # noqa: E402


def parity(program, domain, variant=0):
    host = synth.make_inputs(program, domain, seed=3)
    got = run_gpu(program, host, domain, variant=variant)
    ref = run_oracle(program, host, domain)
    for name, g in got.items():
        st = compare(g.data, ref[name])
        assert st["n_bitdiff"] == 0, (program, name, st)
    print(f"{program} {domain} variant {variant}: bit-identical")


def jit_tiled(program, domain):
    from paper_2005_13014_b200 import oec

    with open(os.path.join(ROOT, "tests", "programs", program + ".oec")) as f:
        name = oec.oec_program_create(f.read())
    host = synth.make_inputs(program, domain, seed=3)
    spec = synth.PROGRAMS[program]
    import torch

    ins = [oec.field_from_host(host[s.name]) for s in spec.inputs]
    outs = [oec.empty_like_domain(domain) for _ in spec.outputs]
    oec.oec_apply_program(name, ins, outs, [v for _, v in spec.scalars], (0, 0, 0), domain, oec.OEC_VARIANT_TILED)
    torch.cuda.synchronize()
    ref = run_oracle(program, host, domain)
    for o, nm in zip(outs, spec.outputs):
        st = compare(o.download(), ref[nm])
        assert st["n_bitdiff"] == 0, (program, nm, st)
    print(f"{program} {domain} stencil-language JIT, tiled variant: bit-identical")


def case_hdiff_pipe(flip=False):
    from test_gpu_pipeline import _set_pad_word, build_ranks, check, oracle_steps

    gdom = (96, 64, 6)
    host = synth.make_inputs("hdiff", gdom, seed=5)
    ranks = build_ranks(host, gdom, 2, 1, np.float64)
    T = 3
    import torch

    if flip:
        for R in ranks:
            _set_pad_word(R["pipe"], 11, 1)
        torch.cuda.synchronize()
    for _ in range(T):
        for R in ranks:
            R["pipe"].run(1)
    torch.cuda.synchronize()
    check(ranks, oracle_steps(host, gdom, T), T)
    print(f"hdiff_pipe 2x1 ranks, 3 steps{' (guesses inverted)' if flip else ''}: bit-identical")


CASES = {
    "hdiff_tma": lambda: parity("hdiff", (128, 64, 6)),
    "hdiff_tma_large": lambda: parity("hdiff", (1024, 1024, 8)),
    "hdiff_pipe": case_hdiff_pipe,
    "hdiff_pipe_flip": lambda: case_hdiff_pipe(True),
    "vadv_sp": lambda: parity("vadv", (128, 16, 80)),
    "vadv_sp_pers": lambda: parity("vadv", (256, 160, 20)),  # 320 blocks on <= 148 CTAs
    "vadv_sp_multi": lambda: parity("vadv", (128, 1800, 8)),  # 1800 blocks > 12 x 148: 2D grid, 5 chunks
    "vadv_ragged": lambda: parity("vadv", (120, 130, 24)),  # ragged rows, persistent CTAs
    "jit_tiled": lambda: jit_tiled("nh_p_grad", (128, 32, 6)),
}

if __name__ == "__main__":
    import torch

    torch.cuda.set_device(0)
    CASES[sys.argv[1]]()
