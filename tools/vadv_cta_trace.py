"""Per-CTA timeline of vadv_sp (VA_TRACE build): start (after griddepcontrol.wait), first TMA chunk
landed, forward sweep done, backward done -- quantiles over all CTAs, relative to the earliest start.

    OEC_LIB_PATH=tune/liboec_trace.so python tools/vadv_cta_trace.py [--domain 128 128 80]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--domain", type=int, nargs=3, default=[128, 128, 80])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    a = ap.parse_args()
    import torch

    from paper_2005_13014_b200 import oec

    dom = tuple(a.domain)
    dt = np.float32 if a.dtype == "f32" else np.float64
    host = synth.make_inputs("vadv", dom, seed=0, dtype=dt)
    sets = []
    for _ in range(8):
        ins = [oec.field_from_host(host[s.name]) for s in synth.PROGRAMS["vadv"].inputs]
        sets.append((ins, [oec.empty_like_domain(dom, fill=0.0, dtype=dt)]))
    for rep in range(3):
        for r in range(8):
            oec.oec_apply_program("vadv", sets[r][0], sets[r][1], [0.15], (0, 0, 0), dom)
        torch.cuda.synchronize()
    buf = (C.c_ulonglong * (4 * 1024))()
    oec.lib().oec_debug_vadv_cta(buf)
    t = np.array(buf[:], dtype=np.int64).reshape(4, 1024)
    ncta = int(np.count_nonzero(t[0]))  # CTAs that ran (any launch mode)
    t = t[:, :ncta]
    t0 = t[0].min()
    names = ["start", "first chunk", "forward done", "end"]
    print(f"domain {dom} {a.dtype}, {ncta} CTAs; times in us after the earliest CTA start")
    for e in range(4):
        q = np.quantile((t[e] - t0) / 1e3, [0, 0.1, 0.5, 0.9, 1.0])
        print(f"{names[e]:14s} min {q[0]:6.2f}  p10 {q[1]:6.2f}  med {q[2]:6.2f}  p90 {q[3]:6.2f}  max {q[4]:6.2f}")
    fwd = (t[2] - t[1]) / 1e3
    bwd = (t[3] - t[2]) / 1e3
    print(f"forward (first chunk -> done) med {np.median(fwd):.2f} us, backward med {np.median(bwd):.2f} us")
    tr = (C.c_ulonglong * (8 * 256))()
    oec.lib().oec_debug_vadv_trace(tr)
    tt = np.array(tr[:], dtype=np.int64).reshape(8, 256)
    c1 = tt[1][tt[1] > 0]
    if len(c1):
        print("CTA 0 chunk arrivals (us after its start):", np.round((np.sort(c1) - t[0][0]) / 1e3, 2).tolist()[:24])
    for role, name in ((4, "chain groups done"), (5, "rows groups done")):
        c = tt[role][tt[role] > 0]
        if len(c):
            print(f"CTA 0 {name} (us):", np.round((np.sort(c) - t[0][0]) / 1e3, 2).tolist()[:24])


if __name__ == "__main__":
    main()
