"""Debug: OEC_VARIANT_TILED on several domains (fresh process per domain)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
from paper_2005_13014_b200 import oec
from oracle import dsl, stencil
p = sys.argv[1]; dom = tuple(int(x) for x in sys.argv[2:5]); order = None if len(sys.argv) < 6 else [0, 1, 2]
text = open(os.path.join(ROOT, "tests/programs", p + ".oec")).read()
name = oec.oec_program_create(text)
tp = dsl.parse(text)
host = synth.make_inputs(p, dom, seed=1)
ins = [oec.field_from_host(host[n], order=order) for n in tp.inputs]
outs = [oec.oec_field_create(dom, (0, 0, 0), (0, 0, 0)).fill(0.0) for _ in tp.outputs]
try:
    oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), dom, 7)
    torch.cuda.synchronize()
    ref = stencil.run_unfused(tp.program, host, tp.scalar_values(), (0, 0, 0), dom)
    ok = all(np.array_equal(f.download(), ref[o].data) for o, f in zip(tp.outputs, outs))
    print(p, dom, order, "ran", "bit-identical" if ok else "MISMATCH", flush=True)
except Exception as e:
    print(p, dom, order, "ERROR", str(e)[:80], flush=True)
