"""us per step of the fused-exchange hdiff pipeline on one rank (bench.pipeline_measure) next to
hdiff's own kernel, at the given domain.  OEC_LIB_PATH selects the library build."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch

    from paper_2005_13014_b200 import oec

    dom = tuple(int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (128, 128, 80)))
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    peak, _ = bench.hbm_peak()
    p = bench.pipeline_measure(oec, torch, dom, l2, peak)
    h = bench.program_measure(oec, torch, "hdiff", dom, l2, peak)
    print(json.dumps({"tag": os.environ.get("TAG", ""), "domain": dom, "pipe_us": round(p["us_per_step"], 3),
                      "hdiff_us": round(h["us_per_launch"], 3), "ratio": round(p["us_per_step"] / h["us_per_launch"], 3)}))


if __name__ == "__main__":
    main()
