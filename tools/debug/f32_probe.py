"""Run one program/variant/dtype case on the GPU and report parity (debug helper)."""
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import synth  # noqa: E402
from gpu_util import compare, domain_part, run_gpu, run_oracle  # noqa: E402

program, variant, dt = sys.argv[1], int(sys.argv[2]), sys.argv[3]
dom = tuple(int(x) for x in sys.argv[4].split(",")) if len(sys.argv) > 4 else (33, 31, 5)
dtype = np.float32 if dt == "f32" else np.float64
host = synth.make_inputs(program, dom, seed=1, dtype=dtype)
g = run_gpu(program, host, dom, variant=variant)
r = run_oracle(program, host, dom)
for name in r:
    print(program, variant, dt, name, compare(domain_part(g[name], (0, 0, 0), dom), r[name]))
