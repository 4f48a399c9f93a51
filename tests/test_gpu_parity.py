"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element, on the
same seeded inputs.  Bar (BASELINE.json north_star): per-element max relative
error <= 1e-12 in fp64; the kernels are built to be bit-identical, so we also require zero bit
differences; domain-boundary / halo indexing bit-exact; output halos never written."""
import numpy as np
import pytest

import synth
from gpu_util import SENTINEL, compare, domain_part, outside_mask, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12
ORDERS = [None, (0, 1, 2)]  # default i,k,j and i,j,k


def _assert_parity(g, r, what):
    c = compare(g, r)
    assert c["max_rel"] <= TOL and c["zero_ok"], (what, c)
    assert c["n_bitdiff"] == 0, (what, c)
    assert not np.isnan(g).any(), what


def _check(program, domain, seed=0, order=None, variant=0, dom_lb=(0, 0, 0), dom_ub=None, out_halo=(0, 0, 0)):
    host = synth.make_inputs(program, domain, seed=seed)
    dom_ub = dom_ub or domain
    g = run_gpu(program, host, domain, order=order, variant=variant, dom_lb=dom_lb, dom_ub=dom_ub, out_halo=out_halo)
    r = run_oracle(program, host, domain, dom_lb=dom_lb, dom_ub=dom_ub)
    for name in synth.PROGRAMS[program].outputs:
        _assert_parity(domain_part(g[name], dom_lb, dom_ub), r[name], (program, name, domain, seed, order))
        assert np.all(g[name].data[outside_mask(g[name], dom_lb, dom_ub)] == SENTINEL), (program, name, "wrote outside")


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("program", ["hdiff", "vadv"])
def test_config0_all_seeds(program, seed):
    # BASELINE.json configs[0]: 32x32x16, halo 2; parity seeds {0..4}
    _check(program, (32, 32, 16), seed=seed)


@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_ragged_both_layouts(program, order):
    # non-divisible sizes exercise the predicated tails (reading R15); output halo 2 holds a sentinel
    _check(program, (33, 31, 5), seed=1, order=order, out_halo=(2, 2, 1))


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_several_tiles(program):
    _check(program, (200, 70, 9), seed=2)


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_degenerate_tiny(program):
    _check(program, (1, 1, 2), seed=3)
    if program != "vadv":
        _check(program, (1, 1, 1), seed=3)
        _check(program, (2, 3, 1), seed=3)


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_subdomain_call(program):
    # dom_lb/dom_ub select a sub-range (P:336 absolute ranges): only it is written
    _check(program, (40, 24, 6), seed=4, dom_lb=(3, 5, 1), dom_ub=(35, 19, 5), out_halo=(0, 0, 0))


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_paper_config_full_compare(program):
    # BASELINE.json configs[1] / configs[2]: 128x128x80, the oracle over the whole domain
    _check(program, (128, 128, 80), seed=0)


def test_hdiff_naive_variant():
    for dom in [(32, 32, 16), (33, 31, 5), (128, 128, 8)]:
        _check("hdiff", dom, seed=0, variant=2)


def test_hdiff_smooth_input():
    domain = (128, 64, 4)
    host = synth.make_inputs("hdiff", domain, seed=0, smooth=True)
    g = run_gpu("hdiff", host, domain)
    r = run_oracle("hdiff", host, domain)
    _assert_parity(domain_part(g["out"], (0, 0, 0), domain), r["out"], "smooth")


@pytest.mark.parametrize("order", ORDERS)
def test_hdiff_integer_probe_is_exact(order):
    # integer-coded probe in = i + 2^10 j + 2^20 k (exact in fp64, linear -> lap = 0): every access
    # offset that is wrong would change the output; out must equal in bit for bit
    domain = (70, 19, 3)
    host = synth.make_inputs("hdiff", domain, seed=0)
    host["in"] = synth.probe_field(host["in"].lb, host["in"].ub)
    g = run_gpu("hdiff", host, domain, order=order)
    exp = domain_part(host["in"], (0, 0, 0), domain)
    assert np.array_equal(domain_part(g["out"], (0, 0, 0), domain), exp)


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_nan_canaries_outside_touched_set(program):
    # NaN in every allocated input cell the program does not read (brute-force trace): no NaN may
    # reach an output (no stray reads influence results)
    from oracle import stencil as st
    from oracle import suite

    domain = (37, 9, 4)
    host = synth.make_inputs(program, domain, seed=5)
    if program != "vadv":
        _, touched = st.run_fused(suite.PROGRAMS[program], host, synth.scalars(program), (0, 0, 0), domain)
    else:
        touched = None
    for s in synth.PROGRAMS[program].inputs:
        f = host[s.name]
        if touched is not None:
            keep = np.zeros(f.data.shape, bool)
            for (i, j, k) in touched[s.name]:
                keep[k - f.lb[2], j - f.lb[1], i - f.lb[0]] = True
        else:  # vadv: wcon level k0 is allocated but never read
            keep = np.ones(f.data.shape, bool)
            if s.name == "wcon":
                keep[0] = False
        f.data[~keep] = np.nan
    g = run_gpu(program, host, domain)
    r = run_oracle(program, host, domain)
    for name in synth.PROGRAMS[program].outputs:
        _assert_parity(domain_part(g[name], (0, 0, 0), domain), r[name], (program, name, "canary"))


def test_mutation_is_detected():
    # the harness must fail on an off-by-one offset: compare the GPU against the
    # oracle run on `in` shifted by one in i
    domain = (32, 16, 2)
    host = synth.make_inputs("hdiff", domain, seed=0)
    g = run_gpu("hdiff", host, domain)
    shifted = {k: v.copy() for k, v in host.items()}
    shifted["in"].data[:, :, :-1] = host["in"].data[:, :, 1:]
    r = run_oracle("hdiff", shifted, domain)
    c = compare(domain_part(g["out"], (0, 0, 0), domain), r["out"])
    assert c["max_rel"] > TOL and c["n_bitdiff"] > 0


@pytest.mark.parametrize("program", ["hdiff", "vadv", "fvtp2d_qj"])
def test_host_buffers_end_to_end(program):
    # device = OEC_DEVICE_HOST: the library stages H2D, runs, copies the domain back (e2e path)
    from paper_2005_13014_b200 import oec

    domain = (48, 20, 6)
    host = synth.make_inputs(program, domain, seed=6)
    spec = synth.PROGRAMS[program]
    ins = [oec.oec_field_wrap(host[s.name].data, host[s.name].lb, host[s.name].ub, k_invariant=s.k_invariant)
           for s in spec.inputs]
    outs_np = [np.full((domain[2] + 2, domain[1] + 2, domain[0] + 2), SENTINEL) for _ in spec.outputs]
    outs = [oec.oec_field_wrap(a, (-1, -1, -1), (domain[0] + 1, domain[1] + 1, domain[2] + 1)) for a in outs_np]
    oec.oec_apply_program(program, ins, outs, None, (0, 0, 0), domain)
    r = run_oracle(program, host, domain)
    for name, a in zip(spec.outputs, outs_np):
        assert np.array_equal(a[1:-1, 1:-1, 1:-1], r[name]), (program, name)
        m = np.ones(a.shape, bool)
        m[1:-1, 1:-1, 1:-1] = False
        assert np.all(a[m] == SENTINEL)


def test_host_buffers_concurrent_streams():
    # host-path calls from several threads on their own streams (staging per device and stream):
    # every program's result equals the oracle, repeatedly, with the calls overlapping
    from concurrent.futures import ThreadPoolExecutor

    import torch

    from paper_2005_13014_b200 import oec

    domain = (96, 40, 12)
    progs = ["hdiff", "vadv", "fvtp2d_qj", "uvbke"]
    jobs = []
    for q, program in enumerate(progs):
        host = synth.make_inputs(program, domain, seed=30 + q)
        spec = synth.PROGRAMS[program]
        ins = [oec.oec_field_wrap(host[s.name].data, host[s.name].lb, host[s.name].ub, k_invariant=s.k_invariant)
               for s in spec.inputs]
        outs_np = [np.full((domain[2], domain[1], domain[0]), SENTINEL) for _ in spec.outputs]
        outs = [oec.oec_field_wrap(a, (0, 0, 0), domain) for a in outs_np]
        jobs.append((program, ins, outs, outs_np, run_oracle(program, host, domain), torch.cuda.Stream()))

    def call(job):
        program, ins, outs, _, _, st = job
        oec.oec_apply_program(program, ins, outs, None, (0, 0, 0), domain, stream=st)

    with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
        for _ in range(3):
            for job in jobs:
                for a in job[3]:
                    a.fill(SENTINEL)
            list(pool.map(call, jobs))
            for program, _, _, outs_np, ref, _ in jobs:
                for name, a in zip(synth.PROGRAMS[program].outputs, outs_np):
                    assert np.array_equal(a, ref[name]), (program, name)


def test_alias_rejected_on_device():
    from paper_2005_13014_b200 import oec

    domain = (16, 16, 2)
    host = synth.make_inputs("hdiff", domain, seed=0)
    inp = oec.field_from_host(host["in"])
    cf = oec.field_from_host(host["coeff"])
    with pytest.raises(oec.OecError) as e:
        oec.oec_hdiff(inp, cf, cf, (0, 0, 0), domain)
    assert e.value.status == 3


def test_torch_wrapped_fields():
    # fields wrapping plain torch tensors (the caller's memory, owned=0), contiguous [k][j][i]
    import torch

    from paper_2005_13014_b200 import oec

    domain = (51, 30, 7)  # odd pitch: no 16-byte alignment -> the non-TMA register kernel
    host = synth.make_inputs("hdiff", domain, seed=7)
    t_in = torch.from_numpy(host["in"].data).cuda()
    t_cf = torch.from_numpy(host["coeff"].data).cuda()
    t_out = torch.full((7, 30, 51), float("nan"), dtype=torch.float64, device="cuda")
    oec.oec_hdiff(oec.oec_field_wrap(t_in, host["in"].lb, host["in"].ub),
                  oec.oec_field_wrap(t_cf, (0, 0, 0), domain), oec.oec_field_wrap(t_out, (0, 0, 0), domain),
                  (0, 0, 0), domain)
    torch.cuda.synchronize()
    r = run_oracle("hdiff", host, domain)
    _assert_parity(t_out.cpu().numpy(), r["out"], "torch-wrapped (odd pitch, V=1 path)")


@pytest.mark.parametrize("program", ["hdiff", "vadv"])
def test_full_size_sampled(program):
    # BASELINE.json configs[3]: 1024x1024x80 in the launch configuration bench.py times; the
    # oracle on sampled sub-boxes (hdiff) / column blocks (vadv) it finishes in seconds
    domain = (1024, 1024, 80)
    host = synth.make_inputs(program, domain, seed=0)
    g = run_gpu(program, host, domain)
    name = synth.PROGRAMS[program].outputs[0]
    for lo, hi in [((0, 0, 0), (64, 48, 80)), ((960, 976, 0), (1024, 1024, 80)), ((500, 300, 0), (580, 340, 80))]:
        r = run_oracle(program, host, domain, dom_lb=lo, dom_ub=hi)
        _assert_parity(domain_part(g[name], lo, hi), r[name], (program, lo, hi))


def test_branch_free_reciprocal_is_ieee():
    # vadv's chain uses the CUDA IEEE reciprocal fast path without its branch (DESIGN.md "vadv
    # kernel"); wherever that path applies it must equal 1.0/x bit for bit
    from paper_2005_13014_b200 import oec

    bad, used = oec.oec_selftest_rcp(200_000_000, seed=12345)
    assert used > 150_000_000 and bad == 0, (bad, used)


@pytest.mark.parametrize("K", [84, 85, 100, 128, 129, 200, 260])
def test_vadv_tall_columns_every_kernel(K):
    # K <= 84: vadv_sp (c', d', u_pos in TMEM); <= 128: vadv_ws (c', d' in TMEM); <= ~190: vadv_tma
    # (c', d' in shared memory); taller: the register kernel with a global c'/d' workspace
    _check("vadv", (130, 3, K), seed=K)


def test_vadv_odd_pitch_register_kernel():
    # torch-wrapped fields with odd strides cannot be TMA tensors: the register-prefetch kernel runs
    import torch

    from paper_2005_13014_b200 import oec

    domain = (45, 7, 9)
    host = synth.make_inputs("vadv", domain, seed=8)
    ins = [oec.oec_field_wrap(torch.from_numpy(host[s.name].data).cuda(), host[s.name].lb, host[s.name].ub)
           for s in synth.PROGRAMS["vadv"].inputs]
    t_out = torch.full((9, 7, 45), float("nan"), dtype=torch.float64, device="cuda")
    oec.oec_vadv(*ins, oec.oec_field_wrap(t_out, (0, 0, 0), domain), 0.15, (0, 0, 0), domain)
    torch.cuda.synchronize()
    r = run_oracle("vadv", host, domain)
    _assert_parity(t_out.cpu().numpy(), r["utens_stage_out"], "vadv odd pitch")


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
@pytest.mark.parametrize("domain", [(33, 31, 5), (128, 128, 80)])
def test_unfused_original_level(program, domain):
    # OEC_VARIANT_UNFUSED: the paper's "original" level (one kernel per operator, temporaries in HBM)
    # computes the same values bit for bit
    _check(program, domain, seed=2, variant=1)
    _check(program, domain, seed=2, variant=1, dom_lb=(1, 2, 0), dom_ub=(domain[0] - 3, domain[1] - 1, domain[2]))


HORIZONTAL = [p for p in synth.ALL_PROGRAMS if p != "vadv"]


@pytest.mark.parametrize("program", HORIZONTAL)
@pytest.mark.parametrize("variant", [2, 3, 4])  # inline, inline+unroll(2), inline+unroll(4)
@pytest.mark.parametrize("domain", [(37, 29, 3), (64, 18, 2), (5, 3, 1)])
def test_inline_and_unrolled_levels(program, variant, domain):
    # row counts not divisible by the 4 x unroll rows of a block: ragged j tail on every level
    _check(program, domain, seed=3, variant=variant)
    _check(program, domain, seed=3, variant=variant, order=(0, 1, 2), out_halo=(1, 2, 0))
    if domain[1] > 4:
        _check(program, domain, seed=3, variant=variant, dom_lb=(0, 1, 0), dom_ub=(domain[0] - 1, domain[1] - 2, domain[2]))


def test_vadv_inline_level_and_unroll_rejected():
    from paper_2005_13014_b200 import oec

    _check("vadv", (45, 7, 20), seed=3, variant=2)  # one thread per column (register/smem kernel)
    host = synth.make_inputs("vadv", (8, 4, 3), seed=0)
    with pytest.raises(oec.OecError) as ei:
        run_gpu("vadv", host, (8, 4, 3), variant=3)
    assert ei.value.status == 7


def test_hdiff_large_config_ragged():
    # >= 8M points selects the wide-tile hdiff configuration (V=4, JB=2); ragged in i and j
    _check("hdiff", (1031, 1029, 9), seed=5)
    _check("hdiff", (333, 6301, 4), seed=6, out_halo=(2, 2, 0))
    _check("hdiff", (517, 1000, 17), seed=7, order=(0, 1, 2))
    # just below the threshold: the small-tile configuration on a multi-million-point domain
    _check("hdiff", (1031, 1029, 3), seed=8)


# ---- vadv launch modes (csrc/vadv.cu): single wave, persistent multi-block, 2D grid ----
@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("domain", [
    (128, 128, 80),   # one wave of 128 one-row blocks
    (120, 130, 80),   # ragged rows (120 of 128 columns live)
    (100, 150, 41),   # 150 blocks on 148 SMs: persistent, two CTAs walk two blocks; K not a multiple of 8
    (16, 1184, 12),   # 1184 narrow blocks (16 live columns each), persistent
    (128, 128, 84),   # the tallest column of the TMEM solver
])
def test_vadv_single_wave_and_narrow_blocks(domain, order):
    _check("vadv", domain, seed=11, order=order)


def test_vadv_subdomain_offset():
    # a sub-domain call (dom_lb, dom_ub not at the allocation origin)
    _check("vadv", (128, 96, 20), seed=12, dom_lb=(16, 3, 2), dom_ub=(128, 95, 19), out_halo=(0, 0, 0))


def _check_sampled(program, domain, boxes, seed=0):
    host = synth.make_inputs(program, domain, seed=seed)
    g = run_gpu(program, host, domain)
    for lo, hi in boxes:
        r = run_oracle(program, host, domain, dom_lb=lo, dom_ub=hi)
        for name in synth.PROGRAMS[program].outputs:
            _assert_parity(domain_part(g[name], lo, hi), r[name], (program, name, domain, lo, hi))


def test_vadv_persistent_full_compare_paper_size():
    # 256x256x60 (the paper's large size): 512 column blocks on <= 148 persistent CTAs --
    # every CTA walks 3-4 blocks, carrying its ring, mbarrier phases and TMEM across them
    _check("vadv", (256, 256, 60), seed=13)


@pytest.mark.parametrize("domain", [(384, 384, 80), (512, 512, 80)])
def test_vadv_persistent_sampled(domain):
    # 1152 / 2048 blocks: persistent (<= 12 per CTA) resp. 2D grid; the samples cover blocks that a
    # persistent CTA reaches first, second and last (block b runs on CTA b % grid as its b / grid-th)
    ni, nj, nk = domain
    boxes = [((0, 0, 0), (256, 2, nk)),                       # blocks 0..3: first blocks of CTAs 0..3
             ((0, 148 // (ni // 128), 0), (ni, 148 // (ni // 128) + 2, nk)),  # second blocks of CTA 0..
             ((ni - 200, nj - 3, 0), (ni, nj, nk)),           # the last blocks (last trips)
             ((130, nj // 2, 0), (250, nj // 2 + 1, nk))]
    _check_sampled("vadv", domain, boxes, seed=14)


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_every_program_paper_large_size(program):
    # 256x256x60 over the whole domain
    if program == "vadv":
        pytest.skip("covered by test_vadv_persistent_full_compare_paper_size")
    _check(program, (256, 256, 60), seed=15)


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_every_program_c5_size_sampled(program):
    # BASELINE.json configs[4]: 512x512x80 per GPU, in the launch configuration bench.py --config c5
    # times; the oracle on sub-boxes at the corners, edges and centre
    ni, nj, nk = 512, 512, 80
    kk = (0, nk) if program == "vadv" else (10, 70)  # a vadv column is solved over its whole k range
    boxes = [((0, 0, 0), (40, 24, nk)), ((ni - 40, nj - 24, 0), (ni, nj, nk)), ((230, 250, kk[0]), (300, 270, kk[1])),
             ((0, nj - 10, 0), (ni, nj, nk if program == "vadv" else 3))]
    _check_sampled(program, (ni, nj, nk), boxes, seed=16)


@pytest.mark.parametrize("case", range(48))
def test_randomized_shapes(case):
    """Seeded random configurations (program, domain, sub-domain box, layout, output halo): every
    kernel-selection path (tile remainders in i and j, persistent / 2D vadv grids, short columns,
    odd offsets) against the oracle, bit for bit, with nothing written outside the box."""
    rng = np.random.default_rng(1000 + case)
    program = synth.ALL_PROGRAMS[case % len(synth.ALL_PROGRAMS)]
    ni, nj = int(rng.integers(1, 97)), int(rng.integers(1, 97))
    nk = int(rng.integers(2 if program == "vadv" else 1, 41))
    domain = (ni, nj, nk)
    lo = tuple(int(rng.integers(0, max(1, n // 3))) for n in domain)
    hi = tuple(int(rng.integers(l + 1, n + 1)) for l, n in zip(lo, domain))
    if program == "vadv" and hi[2] - lo[2] < 2:  # the Thomas solve needs K >= 2
        lo, hi = (lo[0], lo[1], 0), (hi[0], hi[1], nk)
    order = ORDERS[int(rng.integers(0, 2))]
    out_halo = (int(rng.integers(0, 3)), int(rng.integers(0, 3)), 0)
    _check(program, domain, seed=case, order=order, dom_lb=lo, dom_ub=hi, out_halo=out_halo)
