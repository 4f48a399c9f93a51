"""Debug: run OEC_VARIANT_TILED for each stencil-language program, synchronise after each."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
from paper_2005_13014_b200 import oec
from oracle import dsl, stencil
progs = sys.argv[1:] or ["uvbke", "hdiff", "p_grad_c", "nh_p_grad", "fvtp2d_qi", "fvtp2d_qj", "fvtp2d_flux", "fastwaves"]
for p in progs:
    text = open(os.path.join(ROOT, "tests/programs", p + ".oec")).read()
    name = oec.oec_program_create(text)
    tp = dsl.parse(text)
    dom = (33, 19, 5)
    host = synth.make_inputs(p, dom, seed=1)
    ins = [oec.field_from_host(host[n]) for n in tp.inputs]
    outs = [oec.oec_field_create(dom, (0, 0, 0), (0, 0, 0)).fill(0.0) for _ in tp.outputs]
    try:
        oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), dom, 7)
        torch.cuda.synchronize()
        ref = stencil.run_unfused(tp.program, host, tp.scalar_values(), (0, 0, 0), dom)
        ok = all(np.array_equal(f.download(), ref[o].data) for o, f in zip(tp.outputs, outs))
        print(p, "ran", "bit-identical" if ok else "MISMATCH", flush=True)
    except Exception as e:
        print(p, "ERROR", e, flush=True)
        break
