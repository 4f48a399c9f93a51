"""Debug: tiled variant on small custom programs (k-invariant inputs, scalars)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_2005_13014_b200 import oec
from oracle import dsl, stencil
from synth import HostField
progs = {
 "A": "program A\ninput a\noutput o\napply r = a[1,0,0] + a\nstore r -> o\n",
 "B": "program B\ninput a\nscalar s = 2.0\noutput o\napply r = a[1,0,0] * s\nstore r -> o\n",
 "C": "program C\ninput a\ninput m : ij\noutput o\napply r = a[1,0,0] * m\nstore r -> o\n",
 "D": "program D\ninput a\ninput b\noutput o\napply r = a[0,-1,0] + b[-1,0,0]\nstore r -> o\n",
 "E": "program E\ninput a\ninput b\noutput o1\noutput o2\napply r = a[0,-1,0] + b[-1,0,0]\napply q = a - b\nstore r -> o1\nstore q -> o2\n",
}
which = sys.argv[1]
text = progs[which]
name = oec.oec_program_create(text)
tp = dsl.parse(text)
dom = (64, 8, 2)
sig = oec.program_signature(name)[0]
host = {}
rng = np.random.default_rng(0)
for (n, lo, hi, kinv) in sig:
    if kinv:
        lb, ub = (lo[0], lo[1], 0), (dom[0] + hi[0], dom[1] + hi[1], 1)
    else:
        lb, ub = lo, tuple(dom[d] + hi[d] for d in range(3))
    host[n] = HostField(rng.uniform(-1, 1, (ub[2] - lb[2], ub[1] - lb[1], ub[0] - lb[0])), lb, ub, kinv)
ins = [oec.field_from_host(host[n]) for n in tp.inputs]
outs = [oec.oec_field_create(dom, (0, 0, 0), (0, 0, 0)).fill(0.0) for _ in tp.outputs]
try:
    oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), dom, 7)
    torch.cuda.synchronize()
    ref = stencil.run_unfused(tp.program, host, tp.scalar_values(), (0, 0, 0), dom)
    ok = all(np.array_equal(f.download(), ref[o].data) for o, f in zip(tp.outputs, outs))
    print(which, "ran", "bit-identical" if ok else "MISMATCH", flush=True)
except Exception as e:
    print(which, "ERROR", str(e)[:80], flush=True)
