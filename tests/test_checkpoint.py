"""Checkpoint with exact resume: the reference's v1 JSON
model file (checkpoint.hpp:17-143) plus the Adam state, steps and trainer RNG it leaves out.

CPU tests run the oracle restatement and the reference itself (oracle/_ref); the GPU tests
(`-m gpu`) repeat them through the CUDA engine and resume a reference-trained run on it.
"""
import json

import numpy as np
import pytest

from conftest import dataset, max_rel, tensor_err
from paper_1907_03329_b200 import checkpoint as ck
from paper_1907_03329_b200 import errors as E
from paper_1907_03329_b200.trainer import TrainConfig, Trainer


def _pair_data(api, name="quarterly", n=10, seed=41):
    return dataset(api, name, n, seed)


def _resume_roundtrip(api, tmp_path, precision="fp64", name="quarterly", n=10, seed=41, bs=64):
    prof, vals, cats = _pair_data(api, name, n, seed)
    cfg = TrainConfig(seed=7, batch_size=bs, precision=precision)
    a = Trainer((vals, cats), prof, cfg, api=api)
    for _ in range(2):
        a.train_epoch()
    path = tmp_path / "ck.json"
    ck.save_checkpoint(str(path), ck.snapshot(a, epochs=2))
    la = [a.train_epoch() for _ in range(2)]
    b = Trainer((vals, cats), prof, TrainConfig(seed=999, batch_size=bs, precision=precision), api=api)
    ck.apply_checkpoint(b, ck.load_checkpoint(str(path)))
    lb = [b.train_epoch() for _ in range(2)]
    return a, b, la, lb, path


def test_oracle_resume_is_exact(oracle, tmp_path):
    a, b, la, lb, _ = _resume_roundtrip(oracle, tmp_path)
    assert la == lb
    assert np.array_equal(a.weights_flat(), b.weights_flat())
    assert a.last_epoch_windows() == b.last_epoch_windows()


def test_without_training_state_restarts_optimizer(oracle, tmp_path):
    """The reference's own behaviour for a v1 file: weights restored, Adam and RNG not."""
    prof, vals, cats = _pair_data(oracle)
    a = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=64), api=oracle)
    a.train_epoch()
    c0 = ck.snapshot(a, with_training_state=False)
    path = tmp_path / "v1.json"
    ck.save_checkpoint(str(path), c0)
    j = json.loads(path.read_text())
    assert set(j) == {"format", "version", "frequency", "seasonality_length", "horizon", "input_window",
                      "hidden_size", "dilation_blocks", "network", "per_series"}  # checkpoint.hpp:64-88
    b = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=64), api=oracle)
    ck.apply_checkpoint(b, ck.load_checkpoint(str(path)))
    assert np.array_equal(a.weights_flat(), b.weights_flat())
    assert b.train_state().net_step == 0


def test_train_state_matches_reference(oracle, ref):
    """After the same epochs the restatement's exported state equals the reference's private
    Adam / RNG members (the RNG text form bit for bit)."""
    prof, vals, cats = _pair_data(ref, "monthly", 6, 3)
    cfg = TrainConfig(seed=5, batch_size=48)
    o, r = (Trainer((vals, cats), prof, cfg, api=x) for x in (oracle, ref))
    for _ in range(2):
        o.train_epoch(), r.train_epoch()
    so, sr = o.train_state(), r.train_state()
    assert so.rng == sr.rng and so.net_step == sr.net_step
    assert np.array_equal(so.ps_steps, sr.ps_steps)
    for f in ("adam_m", "adam_v", "ps_m", "ps_v"):
        assert tensor_err(getattr(so, f), getattr(sr, f)) < 1e-10, f


def test_reference_run_resumes_on_oracle(oracle, ref, tmp_path):
    prof, vals, cats = _pair_data(ref, "yearly", 40, 2)
    cfg = TrainConfig(seed=11, batch_size=32)
    r = Trainer((vals, cats), prof, cfg, api=ref)
    for _ in range(2):
        r.train_epoch()
    path = tmp_path / "ref.json"
    ck.save_checkpoint(str(path), ck.snapshot(r, epochs=2))
    o = Trainer((vals, cats), prof, TrainConfig(seed=0, batch_size=32), api=oracle)
    ck.apply_checkpoint(o, ck.load_checkpoint(str(path)))
    assert max_rel(o.train_epoch(), r.train_epoch()) < 1e-11
    assert o.last_epoch_windows() == r.last_epoch_windows()
    assert tensor_err(o.weights_flat(), r.weights_flat()) < 1e-10


def test_checkpoint_errors(oracle, tmp_path):
    prof, vals, cats = _pair_data(oracle)
    a = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=64), api=oracle)
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(E.CheckpointError):
        ck.load_checkpoint(str(tmp_path / "bad.json"))
    (tmp_path / "other.json").write_text(json.dumps({"format": "x"}))
    with pytest.raises(E.CheckpointError):
        ck.load_checkpoint(str(tmp_path / "other.json"))
    c0 = ck.snapshot(a)
    c0.hidden_size += 1
    with pytest.raises(E.CheckpointError):
        ck.apply_checkpoint(a, c0)
    c1 = ck.snapshot(a)
    c1.training_state["rng"] = "garbage"
    with pytest.raises(E.CheckpointError):
        ck.apply_checkpoint(a, c1)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_engine_resume_is_exact(engine, tmp_path, precision):
    a, b, la, lb, _ = _resume_roundtrip(engine, tmp_path, precision)
    assert la == lb
    assert np.array_equal(a.weights_flat(), b.weights_flat())
    assert a.last_epoch_windows() == b.last_epoch_windows()
    assert a.validate().mean_smape == b.validate().mean_smape


@pytest.mark.gpu
def test_reference_run_resumes_on_engine(engine, ref, tmp_path):
    """A run trained by the reference itself, checkpointed, continues on the B200 engine
    (fp64) with the reference's own next epoch: same window order, loss to 1e-9."""
    prof, vals, cats = _pair_data(ref, "quarterly", 12, 41)
    cfg = TrainConfig(seed=7, batch_size=64)
    r = Trainer((vals, cats), prof, cfg, api=ref)
    for _ in range(2):
        r.train_epoch()
    path = tmp_path / "ref.json"
    ck.save_checkpoint(str(path), ck.snapshot(r, epochs=2))
    g = Trainer((vals, cats), prof, TrainConfig(seed=0, batch_size=64, precision="fp64"), api=engine)
    ck.apply_checkpoint(g, ck.load_checkpoint(str(path)))
    assert max_rel(g.train_epoch(), r.train_epoch()) < 1e-9
    assert g.last_epoch_windows() == r.last_epoch_windows()
    assert tensor_err(g.weights_flat(), r.weights_flat()) < 1e-8
