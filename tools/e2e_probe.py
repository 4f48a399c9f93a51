"""Time the e2e step (hdiff + vadv through the C-ABI with pinned host fields) and its pieces."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, synth
from paper_2005_13014_b200 import oec
dom = (128, 128, 80)
hh = synth.make_inputs("hdiff", dom, seed=0); vh = synth.make_inputs("vadv", dom, seed=1)
def pinned(hf):
    t = torch.empty(hf.data.shape, dtype=torch.float64, pin_memory=True); t.copy_(torch.from_numpy(hf.data))
    return oec.oec_field_wrap(t, hf.lb, hf.ub, k_invariant=hf.k_invariant)
h_in, h_cf = pinned(hh["in"]), pinned(hh["coeff"])
v_in = [pinned(vh[n]) for n in ("u_stage", "wcon", "u_pos", "utens", "utens_stage_in")]
o1 = torch.zeros((80, 128, 128), dtype=torch.float64, pin_memory=True); o2 = torch.zeros_like(o1).pin_memory()
f1, f2 = oec.oec_field_wrap(o1, (0, 0, 0), dom), oec.oec_field_wrap(o2, (0, 0, 0), dom)
for _ in range(3):
    oec.oec_hdiff(h_in, h_cf, f1, (0, 0, 0), dom); oec.oec_vadv(*v_in, f2, 0.15, (0, 0, 0), dom)
for what in ("hdiff", "vadv", "step"):
    t0 = time.perf_counter()
    for _ in range(20):
        if what in ("hdiff", "step"): oec.oec_hdiff(h_in, h_cf, f1, (0, 0, 0), dom)
        if what in ("vadv", "step"): oec.oec_vadv(*v_in, f2, 0.15, (0, 0, 0), dom)
    print(os.environ.get("OEC_STAGE_SLABS", "8"), what, round((time.perf_counter() - t0) / 20 * 1e3, 3), "ms", flush=True)
x = torch.empty(74147840 // 8, dtype=torch.float64, pin_memory=True); y = torch.empty_like(x, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); print("H2D 74 MB pinned:", round((time.perf_counter() - t0) / 10 * 1e3, 3), "ms", flush=True)
