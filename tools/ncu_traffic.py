"""DRAM traffic per launch INCLUDING the write-back of the outputs (bench.py roofline.traffic).

ncu flushes or keeps caches per kernel; either way the outputs a kernel writes sit dirty in the
126 MB L2 when it ends, and their write-back is charged to whatever kernel evicts them.  So the
capture runs three kernels in a row with --cache-control none:

    evict (a read of 4x L2: L2 left clean)  ->  the program's kernel  ->  evict again

and traffic = kernel dram read + kernel dram write + the second evict's dram write (the kernel's
write-back) minus an evict's own writes after a clean L2 (measured first: three evicts in a row;
round-2 captures showed ~1.7-2 MB per evict that is not the kernel's output).

    # on the GPU box
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --cache-control none --replay-mode application --csv --log-file gpurun_out/ncu_traffic.csv \
        python tools/ncu_traffic.py run c2
    # here
    python tools/ncu_traffic.py parse gpurun_out/ncu_traffic.csv c2   -> profiles/ncu_traffic.json
"""
import csv
import json

import numpy as np
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BASE, REP = 6, 3  # baseline evicts; measured launches per program (median taken)
CONFIGS = {"c2": ((128, 128, 80), ("hdiff", "vadv")),
           "c3": ((128, 128, 80), ("hdiff", "vadv", "uvbke", "p_grad_c", "nh_p_grad", "fvtp2d_qi", "fvtp2d_qj",
                                   "fvtp2d_flux", "fastwaves")),
           "c4": ((1024, 1024, 80), ("hdiff", "vadv")),
           "c5": ((512, 512, 80), ("hdiff", "vadv", "uvbke", "p_grad_c", "nh_p_grad", "fvtp2d_qi", "fvtp2d_qj",
                                   "fvtp2d_flux", "fastwaves"))}


def run(cfg):
    import torch

    import synth
    from paper_2005_13014_b200 import oec

    dom, progs = CONFIGS[cfg]
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    evict = torch.zeros(4 * l2 // 8, dtype=torch.float64, device="cuda")
    # baseline: three evicts back to back -- the DRAM writes of an evict that follows a clean L2
    # (its own partial sums and whatever else the driver writes back) are subtracted from the
    # write-back charged to the evict after each kernel
    for _ in range(BASE):
        evict.sum()
    torch.cuda.synchronize()
    for p in progs:
        spec = synth.PROGRAMS[p]
        host = synth.make_inputs(p, dom, seed=0)
        ins = [oec.field_from_host(host[s.name]) for s in spec.inputs]
        outs = [oec.empty_like_domain(dom, fill=0.0) for _ in spec.outputs]
        sc = [v for _, v in spec.scalars]
        oec.oec_apply_program(p, ins, outs, sc, (0, 0, 0), dom)  # warm-up (JIT tuning for the suite)
        torch.cuda.synchronize()
        evict.sum()
        for _ in range(REP):  # evict, then REP x (kernel, evict): each kernel starts on a clean L2
            oec.oec_apply_program(p, ins, outs, sc, (0, 0, 0), dom)
            evict.sum()
        torch.cuda.synchronize()
        print(f"ran {p}", flush=True)


def parse(path, cfg):
    """Kernels in launch order; for each program the pattern [reduce, KERNEL, reduce] after its
    warm-up: traffic = KERNEL read + write + the following reduce's write."""
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        rows.append(r)
    by_id = {}
    for r in rows:
        k = (r["ID"], r["Kernel Name"])
        by_id.setdefault(k, {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    seq = [(k[1], v) for k, v in sorted(by_id.items(), key=lambda kv: int(kv[0][0]))]

    def to_bytes(v):
        x, u = v
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)

    dom, progs = CONFIGS[cfg]
    out = {}
    q = 0
    while q < len(seq) and "reduce" not in seq[q][0].lower():
        q += 1
    base = 0.0
    if all("reduce" in seq[q + t][0].lower() for t in range(BASE)):  # the baseline evicts (run())
        base = float(np.median([to_bytes(seq[q + t][1]["dram__bytes_write.sum"]) for t in range(1, BASE)]))
        q += BASE
    for p in progs:
        # skip the warm-up launches until the reduce that precedes the measured kernels
        while q < len(seq) and "reduce" not in seq[q][0].lower():
            q += 1
        reps = []
        for _ in range(REP):
            name, m = seq[q + 1]
            after = seq[q + 2][1]
            rd_b, wr_b = to_bytes(m["dram__bytes_read.sum"]), to_bytes(m["dram__bytes_write.sum"])
            wb = to_bytes(after["dram__bytes_write.sum"])
            reps.append((rd_b + wr_b + max(0.0, wb - base), rd_b, wr_b, wb, m))
            q += 2
        q += 1
        traffic, rd_b, wr_b, wb, m = sorted(reps, key=lambda x: x[0])[REP // 2]  # the median launch
        out[p] = {"kernel": name[:80], "read": rd_b, "write_in_kernel": wr_b, "write_back_after": wb,
                  "evict_baseline_write": base, "traffic": traffic, "traffic_all": [x[0] for x in reps], "duration_us": m["gpu__time_duration.sum"][0] / (1e3 if m["gpu__time_duration.sum"][1] in ("ns", "nsecond") else 1)}
    dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    allv = {}
    if os.path.exists(dst):
        with open(dst) as f:
            try:
                allv = json.load(f)
            except Exception:
                allv = {}
    if not isinstance(allv, dict) or any(not isinstance(v, dict) for v in allv.values()):
        allv = {}
    allv[cfg] = {p: v["traffic"] for p, v in out.items()}
    allv.setdefault("_detail", {})[cfg] = out
    with open(dst, "w") as f:
        json.dump(allv, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        parse(sys.argv[2], sys.argv[3])
