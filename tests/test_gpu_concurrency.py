"""Trainers created and trained from several host threads at once (the reference's Trainer
is movable between threads; one process may drive several trainers).  The
engine's shared host machinery -- the process-wide block cache, the worker pool that plans
epochs, the helper threads that build a new trainer's first plan, the epoch-graph cache --
must give every trainer exactly the result it gets alone."""
import threading

import numpy as np
import pytest

from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer

pytestmark = pytest.mark.gpu


def _run(engine, vals, cats, seed, epochs=2):
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    tr = Trainer((vals, cats), prof, TrainConfig(batch_size=256, seed=seed, precision="fp32"), api=engine)
    losses = [tr.train_epoch() for _ in range(epochs)]
    v = tr.validate()
    w = np.asarray(tr.last_epoch_windows(), dtype=np.int64)
    tr.close()
    return losses, v.forecasts.copy(), w


@pytest.mark.parametrize("threads", [4])
def test_concurrent_trainers_match_sequential(engine, threads):
    data = [engine.make_synthetic(70 + i, 120 + 40 * i, 88, 4, 0.05) for i in range(threads)]
    seeds = [3 + i for i in range(threads)]
    expect = [_run(engine, v, c, s) for (v, c), s in zip(data, seeds)]
    got = [None] * threads
    errors = []

    def work(i):
        try:
            got[i] = _run(engine, data[i][0], data[i][1], seeds[i])
        except Exception as ex:  # surfaced below
            errors.append(ex)

    for _ in range(3):
        ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, errors
        for i in range(threads):
            le, fe, we = expect[i]
            lg, fg, wg = got[i]
            assert le == lg, (i, le, lg)  # bit-identical: same RNG stream, same plan, same kernels
            np.testing.assert_array_equal(fe, fg)
            np.testing.assert_array_equal(we, wg)
