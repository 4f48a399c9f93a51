"""Pins of the vadv oracle (oracle/oec_oracle.c) to things other than itself.  CPU-only."""
import os

import numpy as np
import pytest

import synth
from oracle import capi, numpy_oracle
from synth import HostField

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DTR = 3.0 / 20.0


def _out(domain):
    ni, nj, nk = domain
    return HostField(np.full((nk, nj, ni), np.nan), (0, 0, 0), domain)


def _run(f, domain, variant=capi.VADV_UNFUSED, dtr=DTR, nthreads=1):
    return capi.vadv(f, _out(domain), dtr, (0, 0, 0), domain, variant, nthreads).data


@pytest.mark.parametrize("K", [2, 3, 4, 8, 80])
def test_thomas_matches_dense_lu(K):
    # Thomas elimination + back substitution == a dense LU solve (numpy.linalg.solve, partial
    # pivoting) of the same tridiagonal rows, for every column of a small diagonally dominant field
    domain = (5, 3, K)
    f = synth.make_inputs("vadv", domain, seed=K)
    res = _run(f, domain)
    for j in range(3):
        for i in range(5):
            a, b, c, d = capi.vadv_system(f, DTR, i, j, 0, K)
            T = np.diag(b) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
            x = np.linalg.solve(T, d)
            exp = DTR * (x - f["u_pos"].data[:, j, i])
            assert np.max(np.abs(res[:, j, i] - exp)) <= 1e-14 * max(1.0, np.max(np.abs(exp)))


def test_rows_are_tridiagonal_with_boundary_rows():
    K = 6
    f = synth.make_inputs("vadv", (2, 2, K), seed=1)
    a, b, c, d = capi.vadv_system(f, DTR, 1, 0, 0, K)
    assert a[0] == 0.0 and c[-1] == 0.0  # top row has no k-1, bottom row no k+1 (reading R8)
    # every row sums to dtr: a constant column is a steady state of the implicit operator
    assert np.allclose(a + b + c, DTR, rtol=0, atol=1e-16)


def test_wcon_index_placement():
    # wcon nonzero only at (i0, k*) -> a_k != 0 only on row k* of columns i0 and i0-1 (wcon(i) and
    # wcon(i+1) at level k), c_k != 0 only on row k*-1 of the same columns (wcon at level k+1);
    # a = BET_P * (-0.25 w) = -w/8, c = BET_P * (0.25 w) = +w/8
    K, i0, ks, w = 6, 2, 3, 0.5
    f = synth.make_inputs("vadv", (4, 1, K), seed=2)
    f["wcon"].data[:] = 0.0
    f["wcon"].data[ks, 0, i0] = w
    for i in range(4):
        a, b, c, d = capi.vadv_system(f, DTR, i, 0, 0, K)
        hit = i in (i0, i0 - 1)
        exp_a = np.zeros(K)
        exp_c = np.zeros(K)
        if hit:
            exp_a[ks] = -w / 8
            exp_c[ks - 1] = w / 8
        assert np.array_equal(a, exp_a) and np.array_equal(c, exp_c), i


def test_wcon_zero_gives_explicit_tendency():
    # wcon == 0: a = c = 0, b = dtr -> x = d / dtr and out = utens + utens_stage_in (a few ulp)
    domain = (6, 4, 7)
    f = synth.make_inputs("vadv", domain, seed=3)
    f["wcon"].data[:] = 0.0
    res = _run(f, domain)
    exp = f["utens"].data + f["utens_stage_in"].data
    assert np.max(np.abs(res - exp)) < 1e-15


def test_constant_state_is_steady():
    # u_pos = u_stage = const, no tendencies: corr = 0 exactly and the constant column solves the
    # system (rows sum to dtr), so out == 0 up to rounding, for ANY wcon
    domain = (5, 3, 9)
    f = synth.make_inputs("vadv", domain, seed=4)
    for n in ("u_pos", "u_stage"):
        f[n].data[:] = 0.75
    for n in ("utens", "utens_stage_in"):
        f[n].data[:] = 0.0
    res = _run(f, domain)
    assert np.max(np.abs(res)) < 1e-15


def test_constant_u_stage_has_no_correction():
    K = 5
    f = synth.make_inputs("vadv", (3, 2, K), seed=5)
    f["u_stage"].data[:] = 0.3
    a, b, c, d = capi.vadv_system(f, DTR, 1, 1, 0, K)
    exp_d = (DTR * f["u_pos"].data[:, 1, 1] + f["utens"].data[:, 1, 1]) + f["utens_stage_in"].data[:, 1, 1]
    assert np.array_equal(d, exp_d + 0.0)


def test_hand_worked_k2_column():
    vals = {}
    for ln in open(os.path.join(GOLDEN, "vadv_worked_k2.txt")):
        if ln.strip() and not ln.startswith("#"):
            k, *v = ln.split()
            vals[k] = [float(x) for x in v]
    domain = (1, 1, 2)
    f = synth.make_inputs("vadv", domain, seed=0)
    f["wcon"].data[:] = vals["wcon"][0]
    for n in ("u_stage", "u_pos", "utens", "utens_stage_in"):
        f[n].data[:, 0, 0] = vals[n]
    res = _run(f, domain, dtr=vals["dtr"][0])
    assert np.allclose(res[:, 0, 0], vals["expect"], rtol=0, atol=4e-16)


@pytest.mark.parametrize("domain", [(32, 32, 16), (33, 31, 5), (1, 1, 2), (7, 3, 80)])
@pytest.mark.parametrize("seed", [0, 1])
def test_fused_unfused_reversed_numpy_agree_bitwise(domain, seed):
    f = synth.make_inputs("vadv", domain, seed=seed)
    outs = [_run(f, domain, v, nthreads=2) for v in (capi.VADV_UNFUSED, capi.VADV_FUSED, capi.VADV_FUSED_REVERSED)]
    outs.append(numpy_oracle.vadv(f, DTR, (0, 0, 0), domain))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    assert not np.isnan(outs[0]).any()


def test_thread_count_invariance():
    domain = (20, 17, 12)
    f = synth.make_inputs("vadv", domain, seed=9)
    r = [_run(f, domain, v, nthreads=nt) for nt in (1, 4) for v in (capi.VADV_UNFUSED, capi.VADV_FUSED)]
    for x in r[1:]:
        assert np.array_equal(r[0], x)


def test_k_subrange_is_its_own_column():
    # the column solve spans the domain's k range: a sub-range [k0,k1) is solved with its own
    # boundary rows (reading R8)
    domain = (4, 4, 10)
    f = synth.make_inputs("vadv", domain, seed=6)
    o = _out(domain)
    capi.vadv(f, o, DTR, (0, 0, 3), (4, 4, 8))
    a, b, c, d = capi.vadv_system(f, DTR, 2, 1, 3, 8)
    T = np.diag(b) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
    exp = DTR * (np.linalg.solve(T, d) - f["u_pos"].data[3:8, 1, 2])
    assert np.allclose(o.data[3:8, 1, 2], exp, rtol=0, atol=1e-15)
    assert np.isnan(o.data[:3]).all() and np.isnan(o.data[8:]).all()


def test_k_lt_2_rejected():
    f = synth.make_inputs("vadv", (2, 2, 2), seed=0)
    with pytest.raises(capi.OracleError):
        capi.vadv(f, _out((2, 2, 2)), DTR, (0, 0, 0), (2, 2, 1))


def test_wcon_halo_missing_is_an_error():
    domain = (4, 4, 3)
    f = synth.make_inputs("vadv", domain, seed=0)
    w = f["wcon"]
    f["wcon"] = HostField(np.ascontiguousarray(w.data[:, :, :4]), (0, 0, 0), (4, 4, 3))  # no +1 i halo
    with pytest.raises(capi.OracleError):
        _run(f, domain)
