"""Experiment: one bench step (hdiff + vadv, 128x128x80) with the two independent programs
sequential on one stream vs concurrent on two streams (CUDA graph, rotating sets)."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def main():
    import torch

    from paper_2005_13014_b200 import oec

    dom = (128, 128, 80)
    hh = synth.make_inputs("hdiff", dom, seed=0)
    vh = synth.make_inputs("vadv", dom, seed=1)
    sets = []
    for _ in range(7):
        h = ([oec.field_from_host(hh[n]) for n in ("in", "coeff")], [oec.empty_like_domain(dom, fill=0.0)])
        v = ([oec.field_from_host(vh[s.name]) for s in synth.PROGRAMS["vadv"].inputs], [oec.empty_like_domain(dom, fill=0.0)])
        sets.append((h, v))
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

    def run(s, concurrent):
        (hi, ho), (vi, vo) = s
        if not concurrent:
            oec.oec_apply_program("hdiff", hi, ho, None, (0, 0, 0), dom)
            oec.oec_apply_program("vadv", vi, vo, [0.15], (0, 0, 0), dom)
            return
        cur = torch.cuda.current_stream()
        sa.wait_stream(cur)
        sb.wait_stream(cur)
        with torch.cuda.stream(sb):
            oec.oec_apply_program("vadv", vi, vo, [0.15], (0, 0, 0), dom)
        with torch.cuda.stream(sa):
            oec.oec_apply_program("hdiff", hi, ho, None, (0, 0, 0), dom)
        cur.wait_stream(sa)
        cur.wait_stream(sb)

    for concurrent in (False, True):
        for s in sets:
            run(s, concurrent)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for s in sets:
                run(s, concurrent)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / (50 * len(sets))
        print(json.dumps({"lib": os.environ.get("OEC_LIB_PATH", "default"), "concurrent": concurrent, "us_per_step": round(us, 2),
                          "Gpts/s": round(dom[0] * dom[1] * dom[2] / us / 1e3, 2)}), flush=True)


if __name__ == "__main__":
    main()
