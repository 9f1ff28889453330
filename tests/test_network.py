"""The general dilated LSTM stack (forward_stack over multi-step sequences, network.hpp:148-210)
and its tape gradients -- SURVEY.md section 8(f) rank 1.  Mirrors the reference's network tests
(test_network.cpp:94-181 dilation structure, :235-267 finite-difference gradients,
acceptance.cpp:183-217) at the stack level, with every weight array live (random recurrent
matrices and forget gates, which the sequence-length-1 training path never uses).
"""
import numpy as np
import pytest

from conftest import PROFILES, dataset, tensor_err
from paper_1907_03329_b200 import errors as E
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer


def make(api, prof, seed=3, precision="fp64"):
    vals, cats = api.make_synthetic(41, 4, prof.min_length + 2 * prof.horizon, prof.seasonality_length, 0.05)
    tr = Trainer((vals, cats), prof, TrainConfig(seed=seed, precision=precision), api=api)
    rng = np.random.default_rng(seed)
    tr.set_weights({n: rng.uniform(-0.5, 0.5, (r, c)) for n, r, c, _ in tr.param_layout})
    return tr


def seq_inputs(prof, T, B, seed=0):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (T, B, prof.input_window + 6))


PROFS = {
    "tiny": PROFILES["tiny"][0],
    "quarterly": FrequencyProfile.defaults(Frequency.Quarterly),
    "monthly": FrequencyProfile.defaults(Frequency.Monthly),
}
CASES = [("tiny", 1, 3), ("tiny", 5, 2), ("quarterly", 9, 5), ("monthly", 13, 3)]


@pytest.mark.parametrize("name,T,B", CASES)
def test_oracle_forward_stack_matches_reference(oracle, ref, name, T, B):
    prof = PROFS[name]
    o, r = make(oracle, prof), make(ref, prof)
    x = seq_inputs(prof, T, B)
    ob = np.random.default_rng(1).normal(size=(B, prof.horizon))
    fo, wo, xo = o.forward_stack(x, ob)
    fr, wr, xr = r.forward_stack(x, ob)
    assert tensor_err(fo, fr) < 1e-13
    for n in wr:
        assert tensor_err(wo[n], wr[n]) < 1e-11, n
    assert tensor_err(xo, xr) < 1e-11
    if T > max(max(b) for b in prof.dilation_blocks):
        assert np.any(wr["lstm0.w_recur"] != 0)  # the recurrence is live at this length


def test_dilation_structure(oracle):
    """test_network.cpp:124-181 at the stack level: one layer of dilation d over T steps; the
    output (last step) depends on x_t only for t = T-1 - k d, so the other input adjoints are
    exactly zero; dilation = T decouples every step from the last."""
    for d, T in ((2, 4), (4, 4), (1, 3)):
        prof = FrequencyProfile(Frequency.Quarterly, 4, 4, 8, [[d]], 6, 20)
        tr = make(oracle, prof, seed=d)
        x = seq_inputs(prof, T, 2, seed=d)
        _, _, xb = tr.forward_stack(x, np.ones((2, 4)))
        for t in range(T):
            reach = (T - 1 - t) % d == 0
            assert np.any(xb[t] != 0) == reach, (d, T, t)


def test_forward_stack_finite_differences(oracle):
    """test_network.cpp:235-267: central differences of sum(out * out_bar) against the tape
    gradient for a sample of weights of every array, and for inputs."""
    prof = PROFS["tiny"]
    tr = make(oracle, prof, seed=9)
    x = seq_inputs(prof, 4, 2, seed=9)
    ob = np.random.default_rng(9).normal(size=(2, prof.horizon))
    _, wb, xb = tr.forward_stack(x, ob)
    base = tr.weights_flat()
    layout = {n: (o, r * c) for n, r, c, o in tr.param_layout}
    rng = np.random.default_rng(0)
    h = 1e-6
    for n, (o, size) in layout.items():
        for i in rng.choice(size, size=min(size, 3), replace=False):
            w = base.copy()
            w[o + i] += h
            tr.set_weights(w)
            fp = float(np.sum(tr.forward_stack(x) * ob))
            w[o + i] -= 2 * h
            tr.set_weights(w)
            fm = float(np.sum(tr.forward_stack(x) * ob))
            fd = (fp - fm) / (2 * h)
            assert abs(fd - wb[n].ravel()[i]) <= 1e-6 + 1e-5 * abs(fd), (n, i, fd, wb[n].ravel()[i])
    tr.set_weights(base)
    for idx in [(0, 0, 0), (3, 1, 5), (2, 0, 13)]:
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd = (np.sum(tr.forward_stack(xp) * ob) - np.sum(tr.forward_stack(xm) * ob)) / (2 * h)
        assert abs(fd - xb[idx]) <= 1e-6 + 1e-5 * abs(fd)


def test_forward_stack_errors(oracle):
    tr = make(oracle, PROFS["tiny"])
    with pytest.raises(E.ContractError):
        tr.forward_stack(np.zeros((0, 2, 14)))
    with pytest.raises(E.ShapeError):
        tr.forward_stack(np.zeros((2, 2, 5)))


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol", [("fp64", 1e-11), ("fp32", 1e-4)])
@pytest.mark.parametrize("name,T,B", CASES + [("quarterly", 16, 37)])
def test_engine_forward_stack_matches_oracle(engine, oracle, name, T, B, precision, tol):
    prof = PROFS[name]
    g, o = make(engine, prof, precision=precision), make(oracle, prof)
    x = seq_inputs(prof, T, B)
    ob = np.random.default_rng(1).normal(size=(B, prof.horizon))
    fg, wg, xg = g.forward_stack(x, ob)
    fo, wo, xo = o.forward_stack(x, ob)
    assert tensor_err(fg, fo) < tol
    assert tensor_err(g.forward_stack(x), fo) < tol  # forward-only call
    for n in wo:
        assert tensor_err(wg[n], wo[n]) < 10 * tol, n
    assert tensor_err(xg, xo) < 10 * tol


@pytest.mark.gpu
def test_engine_dilation_structure(engine):
    prof = FrequencyProfile(Frequency.Quarterly, 4, 4, 8, [[2], [3]], 6, 20)
    tr = make(engine, prof, seed=5)
    x = seq_inputs(prof, 7, 3, seed=5)
    _, _, xb = tr.forward_stack(x, np.ones((3, 4)))
    # the head reads step 6; block 1 (dilation 3) reads block 0's outputs at steps 6, 3, 0 and
    # the skip around it block 0's step 6; block 0 (dilation 2) reaches back by multiples of 2:
    # x_t reaches the output iff 6 - t = 2a + 3b (a, b >= 0), i.e. for every t but t = 5
    for t in range(7):
        assert np.any(xb[t] != 0) == (t != 5), t


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("name", ["quarterly", "monthly", "yearly"])
def test_fast_forward_stack_equals_stepwise_kernel(engine, name, precision, monkeypatch):
    """The shared-memory-resident inference kernel (k_seq_fwd_fast) against the per-step
    kernel the adjoint path uses (k_seq_forward), at the M4 profiles' dilations and block
    skips, B not a multiple of the CTA's rows: same summation order, bit-identical."""
    prof = FrequencyProfile.defaults(getattr(Frequency, name.capitalize()))
    g = make(engine, prof, precision=precision)
    x = seq_inputs(prof, 19, 37)
    fast = g.forward_stack(x)
    monkeypatch.setenv("ESRNN_SEQ_NAIVE", "1")
    naive = g.forward_stack(x)
    assert np.array_equal(fast, naive)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["quarterly", "monthly", "yearly"])
def test_fast_forward_stack_adjoint_equals_stepwise_kernel(engine, name, monkeypatch):
    """The shared-memory-resident adjoint (k_seq_fwd_fast<SAVE> + k_seq_bwd_fast, fp32) against
    the stepwise adjoint (k_seq_forward + k_seq_backward): same graph, bit-identical outputs and
    input adjoints (same per-element operation order).  The weight gradients are sums over
    (sequence, step) that the fast kernel accumulates per thread in registers and the stepwise
    kernel per step in global memory, so they agree to fp32 summation-order rounding: ≤ 1e-6
    relative to the largest entry of each tensor (measured ≤ 8e-7 on B200)."""
    prof = FrequencyProfile.defaults(getattr(Frequency, name.capitalize()))
    g = make(engine, prof, precision="fp32")
    x = seq_inputs(prof, 19, 37)
    ob = np.random.default_rng(2).normal(size=(37, prof.horizon))
    fo, fw, fx = g.forward_stack(x, ob)
    monkeypatch.setenv("ESRNN_SEQ_NAIVE", "1")
    no, nw, nx = g.forward_stack(x, ob)
    assert np.array_equal(fo, no)
    assert np.array_equal(fx, nx)
    for k in nw:
        scale = max(1.0, float(np.max(np.abs(nw[k]))))
        err = float(np.max(np.abs(fw[k] - nw[k])))
        assert err <= 1e-6 * scale, (k, err, scale)
