"""Run the VA_TRACE build of vadv once (after warm-up) and print the per-role chunk timeline of CTA 0."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import synth  # noqa: E402


def main():
    import torch

    from paper_2005_13014_b200 import oec

    dom = (128, 128, 80)
    host = synth.make_inputs("vadv", dom, seed=0)
    sets = []
    for _ in range(8):
        ins = [oec.field_from_host(host[s.name]) for s in synth.PROGRAMS["vadv"].inputs]
        sets.append((ins, [oec.empty_like_domain(dom, fill=0.0)]))
    for r in range(8):
        oec.oec_apply_program("vadv", sets[r][0], sets[r][1], [0.15], (0, 0, 0), dom)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (8 * 256))()
    oec.lib().oec_debug_vadv_trace(buf)
    t = np.array(buf[:], dtype=np.int64).reshape(8, 256)
    t0 = t[7, 0]
    names = ["producer issued", "coef got input", "sp: coef0|coef1|chain0..", "chain got rows", "chain stored tmem",
             "coef rows written", "chain done", "start"]
    print("end-to-end CTA(0,0) us:", (t[6, 0] - t0) / 1e3)
    for role in range(6):
        vals = [(t[role, q] - t0) / 1e3 for q in range(256) if t[role, q] > 0]
        print(f"{names[role]:22s}", " ".join(f"{v:6.2f}" for v in vals))


if __name__ == "__main__":
    main()
