"""Run the HD_TRACE build of hdiff once (after warm-up) and print the per-warp item timeline of
CTA 0 and the last CTA (us since the earliest warp start)."""
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
    host = synth.make_inputs("hdiff", dom, seed=0)
    sets = [([oec.field_from_host(host["in"]), oec.field_from_host(host["coeff"])], [oec.empty_like_domain(dom, fill=0.0)])
            for _ in range(18)]
    for r in range(18):
        oec.oec_apply_program("hdiff", sets[r][0], sets[r][1], None, (0, 0, 0), dom)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (2 * 8 * 64))()
    oec.lib().oec_debug_hdiff_trace(buf)
    t = np.array(buf[:], dtype=np.int64).reshape(2, 8, 64)
    t0 = t[t > 0].min()
    for c in range(2):
        print("CTA", "first" if c == 0 else "last")
        for w in range(8):
            v = t[c, w]
            if v[0] == 0:
                continue
            ev = [(v[q] - t0) / 1e3 if v[q] > 0 else None for q in range(64)]
            items = [(ev[1 + 2 * n], ev[2 + 2 * n]) for n in range(31) if ev[1 + 2 * n] is not None]
            print(f"  warp {w}: start {ev[0]:5.2f}  items (ready, done): " +
                  " ".join(f"({a:5.2f},{b:5.2f})" for a, b in items))


if __name__ == "__main__":
    main()
