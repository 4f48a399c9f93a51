"""Summarise an .ncu-rep (details page + selected raw metrics + top stall reasons) as text/JSON.

    python tools/ncu_summary.py gpurun_out/prof_vadv.ncu-rep [--json]
"""
import csv
import io
import json
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
       "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__inst_executed.sum", "smsp__inst_executed.avg.per_cycle_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    details = list(csv.DictReader(io.StringIO(ncu(["-i", rep, "--page", "details", "--csv"]))))
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    out = []
    hdr, units = raw[0], raw[1]
    for q, row in enumerate(raw[2:]):
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name"), "raw": {m: f"{d.get(m)} {u.get(m, '')}".strip() for m in RAW if m in d}}
        stalls = {m: float(d[m]) for m in hdr if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio")
                  and d.get(m, "").replace(".", "", 1).isdigit()}
        top = sorted(stalls.items(), key=lambda x: -x[1])[:8]
        k["top_stalls_cycles_per_issue"] = {a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): b for a, b in top}
        k["details"] = {}
        for r in details:
            if r.get("Kernel Name") == d.get("Kernel Name") and r.get("Metric Name"):
                k["details"][f"{r['Section Name']}/{r['Metric Name']}"] = f"{r['Metric Value']} {r['Metric Unit']}".strip()
        out.append(k)
    if "--json" in sys.argv:
        print(json.dumps(out, indent=1))
        return
    for k in out:
        print("==", k["kernel"])
        for a, b in k["raw"].items():
            print(f"  {a:60s} {b}")
        print("  top stalls (cycles/issued inst):", k["top_stalls_cycles_per_issue"])
        for a, b in k["details"].items():
            if any(s in a for s in ("Duration", "Throughput", "Occupancy", "Eligible", "Issued Warp", "Active Warps", "Registers", "Waves", "L1/TEX Hit", "L2 Hit", "Mem Busy", "Max Bandwidth", "Executed Ipc")):
                print(f"  {a:60s} {b}")


if __name__ == "__main__":
    main()
