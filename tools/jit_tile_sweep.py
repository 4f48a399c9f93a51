"""Time OEC_VARIANT_TILED of every stencil-language program at a domain (one JSON line each).
The tile configuration comes from OEC_JIT_TILE="rows,cta_smem_kb" (read once per process).

    OEC_JIT_TILE=1,60 python tools/jit_tile_sweep.py --domain 128 128 80
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import hbm_peak, program_measure  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--domain", type=int, nargs=3, default=[128, 128, 80])
    ap.add_argument("--variant", type=int, default=7)
    ap.add_argument("--programs", nargs="*", default=None)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    a = ap.parse_args()
    import torch

    from paper_2005_13014_b200 import oec

    dom = tuple(a.domain)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    peak, _ = hbm_peak()
    pdir = os.path.join(ROOT, "tests", "programs")
    for fn in sorted(os.listdir(pdir)):
        if a.programs and fn[:-4] not in a.programs:
            continue
        with open(os.path.join(pdir, fn)) as f:
            name = oec.oec_program_create(f.read())
        import numpy as np

        r = program_measure(oec, torch, fn[:-4], dom, l2, peak, a.variant, run_name=name,
                            dtype=np.float32 if a.dtype == "f32" else np.float64)
        print(json.dumps({"tile_cfg": os.environ.get("OEC_JIT_TILE_CFG", "0"), "variant": a.variant, "dtype": a.dtype, "program": fn[:-4], "domain": list(dom),
                          "us": round(r["us_per_launch"], 2), "frac": round(r["frac_of_hbm_peak"], 3)}), flush=True)
        oec.oec_program_destroy(name)


if __name__ == "__main__":
    main()
