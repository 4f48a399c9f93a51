"""The CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import, call, link or execute anything under oracle/.  The product path
(paper_2005_13014_b200/) never imports it and shares no code with it; it fails loudly when its
CUDA extension is missing instead of falling back here.

Contents:
  oec_oracle.c     plain C (fp64, -ffp-contract=off) hdiff and vadv, unfused ("original"
                   level) and fused (inlined) variants -> liboec_oracle.so
  capi.py          ctypes loader for liboec_oracle.so
  numpy_oracle.py  a second, independent numpy implementation of hdiff and vadv (cross-check)
  stencil.py       a tiny stencil-program evaluator: unfused numpy evaluation apply by apply,
                   fused per-point (inlined) evaluation with touched-index tracing, and the
                   Table II op census
  suite.py         the remaining benchmark programs (uvbke, p_grad_c, nh_p_grad, fvtp2d_qi/qj/
                   flux, fastwaves) written in that notation

Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".  Functions without a pin to
something other than themselves are marked "parity unpinned" in their docstring.
"""
