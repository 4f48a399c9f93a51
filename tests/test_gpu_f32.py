"""GPU parity of the f32 path (§7.1: every benchmark also runs in single
precision) against the binary32 oracle instance, element by element: the kernels evaluate the
same expressions in binary32 with --fmad=false and IEEE division, so the bar is again zero bit
differences; the paper's own f32 criterion (relative error <= 1e-5 against fp64) is checked too."""
import numpy as np
import pytest

import synth
from gpu_util import SENTINEL, compare, domain_part, outside_mask, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

F32 = np.float32
HORIZONTAL = [p for p in synth.ALL_PROGRAMS if p != "vadv"]


def _check(program, domain, seed=0, order=None, variant=0, dom_lb=(0, 0, 0), dom_ub=None, out_halo=(0, 0, 0)):
    host = synth.make_inputs(program, domain, seed=seed, dtype=F32)
    dom_ub = dom_ub or domain
    g = run_gpu(program, host, domain, order=order, variant=variant, dom_lb=dom_lb, dom_ub=dom_ub, out_halo=out_halo)
    r = run_oracle(program, host, domain, dom_lb=dom_lb, dom_ub=dom_ub)
    for name in synth.PROGRAMS[program].outputs:
        gd = domain_part(g[name], dom_lb, dom_ub)
        assert gd.dtype == F32
        c = compare(gd, r[name])
        assert c["n_bitdiff"] == 0, (program, name, domain, variant, c)
        assert np.all(g[name].data[outside_mask(g[name], dom_lb, dom_ub)] == SENTINEL), (program, name, "wrote outside")
    return host, g


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
@pytest.mark.parametrize("domain", [(33, 31, 5), (128, 128, 80), (5, 3, 2)])
def test_f32_default_kernels(program, domain):
    _check(program, domain, seed=1)
    _check(program, domain, seed=2, order=(0, 1, 2), out_halo=(1, 2, 0))


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_f32_optimisation_levels(program, variant):
    if program == "vadv" and variant >= 3:
        pytest.skip("unrolling does not apply to the column solver")
    _check(program, (37, 29, 6), seed=3, variant=variant)
    _check(program, (37, 29, 6), seed=3, variant=variant, dom_lb=(1, 2, 0), dom_ub=(34, 28, 6))


@pytest.mark.parametrize("program", ["hdiff", "vadv"])
def test_f32_large_and_ragged(program):
    _check(program, (1031, 1029, 3) if program == "hdiff" else (517, 203, 80), seed=5)
    _check(program, (77, 1000, 5), seed=6, order=(0, 1, 2))


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_f32_within_paper_tolerance_of_fp64(program):
    # f32 results within relative error 1e-5 of the fp64 computation (normwise per output)
    domain = (64, 48, 20)
    host32, g = _check(program, domain, seed=7)
    r64 = run_oracle(program, synth.as_dtype(host32, np.float64), domain)
    for name in r64:
        a = domain_part(g[name], (0, 0, 0), domain).astype(np.float64)
        err = np.max(np.abs(a - r64[name])) / np.max(np.abs(r64[name]))
        assert err <= 1e-5, (program, name, err)


def test_f32_host_buffers_end_to_end():
    from paper_2005_13014_b200 import oec

    domain = (40, 24, 7)
    for program in ("hdiff", "vadv", "fastwaves"):
        host = synth.make_inputs(program, domain, seed=8, dtype=F32)
        spec = synth.PROGRAMS[program]
        ins = [oec.oec_field_wrap(host[s.name].data, host[s.name].lb, host[s.name].ub, k_invariant=s.k_invariant)
               for s in spec.inputs]
        outs_np = [np.full((domain[2], domain[1], domain[0]), np.nan, F32) for _ in spec.outputs]
        outs = [oec.oec_field_wrap(o, (0, 0, 0), domain) for o in outs_np]
        oec.oec_apply_program(program, ins, outs, None, (0, 0, 0), domain)
        r = run_oracle(program, host, domain)
        for name, o in zip(spec.outputs, outs_np):
            assert compare(o, r[name])["n_bitdiff"] == 0, (program, name)


def test_branch_free_rcp32_is_ieee_exhaustive():
    """The f32 vadv reciprocal equals 1.0f / x bit for bit on every float where it applies."""
    from paper_2005_13014_b200 import oec

    bad, used = oec.oec_selftest_rcp32()
    assert used > 3_000_000_000 and bad == 0, (bad, used)


@pytest.mark.parametrize("case", range(27))
def test_f32_randomized_shapes(case):
    """Seeded random configurations in binary32 (as test_gpu_parity.test_randomized_shapes)."""
    rng = np.random.default_rng(2000 + case)
    program = synth.ALL_PROGRAMS[case % len(synth.ALL_PROGRAMS)]
    ni, nj = int(rng.integers(1, 97)), int(rng.integers(1, 97))
    nk = int(rng.integers(2 if program == "vadv" else 1, 41))
    domain = (ni, nj, nk)
    lo = tuple(int(rng.integers(0, max(1, n // 3))) for n in domain)
    hi = tuple(int(rng.integers(l + 1, n + 1)) for l, n in zip(lo, domain))
    if program == "vadv" and hi[2] - lo[2] < 2:
        lo, hi = (lo[0], lo[1], 0), (hi[0], hi[1], nk)
    order = [None, (0, 1, 2)][int(rng.integers(0, 2))]
    out_halo = (int(rng.integers(0, 3)), int(rng.integers(0, 3)), 0)
    _check(program, domain, seed=case, order=order, dom_lb=lo, dom_ub=hi, out_halo=out_halo)
