"""Debug: AUTO tuning on a side stream, then graph capture (prints progress)."""
import faulthandler, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
faulthandler.dump_traceback_later(60, exit=True)
import torch, synth
from paper_2005_13014_b200 import oec
text = open(os.path.join(ROOT, "tests/programs/uvbke.oec")).read()
name = oec.oec_program_create(text)
dom = (64, 32, 8)
host = synth.make_inputs("uvbke", dom, seed=3)
ins = [oec.field_from_host(host[n]) for n in ("uc", "vc", "cosa", "rsina")]
outs = [oec.oec_field_create(dom, (0, 0, 0), (0, 0, 0)).fill(0.0) for _ in range(2)]
mode = sys.argv[1] if len(sys.argv) > 1 else "side"
s = torch.cuda.Stream() if mode == "side" else torch.cuda.current_stream()
for v in (2, 3, 4, 5, 6):
    with torch.cuda.stream(s):
        oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), dom, v)
    torch.cuda.synchronize(); print("variant", v, "ok", flush=True)
with torch.cuda.stream(s):
    oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), dom, 0)
print("auto call returned", flush=True)
torch.cuda.synchronize(); print("auto synced", flush=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), dom, 0)
print("captured", flush=True)
g.replay(); torch.cuda.synchronize(); print("replayed", flush=True)
