"""The sharded (multi-GPU) training step executed for real on one GPU.

SURVEY §8(e): rank r owns a contiguous block of series; every rank runs the same global
shuffled batches on its own windows; per step the shared gradients and the step tail
(per-series squared norm, loss sum, error flag) are all-reduced; every rank finalises the
identical clip scale (the reference clips over shared AND per-series gradients,
trainer.hpp:603-615) and Adam update.  Two transports run that collective here:

* an in-process group (esrnn_group): W trainers on one GPU, one host thread each, the
  exchange being the engine's fused k_group_reduce (collective.cuh) -- the whole sharded
  epoch graph (K2 -> K3 partials -> reduce + finalise -> replicated / local Adam);
* NCCL with a one-rank communicator (ESRNN_DIST_FORCE_COLLECTIVE): ncclAllReduce captured
  in the epoch graph, k_finalize, the sharded k_adam.

Both are compared with the single-GPU trainer (fp64: 1e-10), for determinism, for error
semantics (a rank's NumericDomainError reaches every rank; nobody hangs or updates), and
for the per-series gather a sharded checkpoint needs.
"""
import threading

import numpy as np
import pytest

from conftest import dataset, max_rel, tensor_err
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200 import checkpoint as ck
from paper_1907_03329_b200 import errors as E
from paper_1907_03329_b200.trainer import TrainConfig, Trainer

pytestmark = pytest.mark.gpu


def run_ranks(world, fn):
    """fn(rank) on `world` host threads (the engine releases the GIL in ctypes calls);
    returns the per-rank results, re-raising nothing: exceptions are returned."""
    out = [None] * world

    def body(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # noqa: BLE001
            out[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
        assert not t.is_alive(), "a rank hung"
    return out


def group_run(engine, data, cfg, world, epochs=2, force=False):
    prof, vals, cats = data
    grp = engine.group(world)
    trs = [None] * world

    def make(r):
        trs[r] = Trainer((vals, cats), prof, cfg, api=engine,
                         dist=(r, world, grp, N.DIST_FORCE_COLLECTIVE if force else 0))

    res = run_ranks(world, make)
    assert all(x is None for x in res), res

    def train(r):
        losses = [trs[r].train_epoch() for _ in range(epochs)]
        v = trs[r].validate()
        a, g, s = trs[r].gather_per_series_arrays()
        return losses, trs[r].weights_flat(), (a, g, s), v.mean_smape

    res = run_ranks(world, train)
    for r in res:
        if isinstance(r, Exception):
            raise r
    for t in trs:
        t.close()
    grp.close()
    return res


def single_run(engine, data, cfg, epochs=2):
    prof, vals, cats = data
    t = Trainer((vals, cats), prof, cfg, api=engine)
    losses = [t.train_epoch() for _ in range(epochs)]
    v = t.validate()
    out = losses, t.weights_flat(), t.per_series_arrays(), v.mean_smape
    t.close()
    return out


def assert_same(a, b, tol):
    la, wa, pa, va = a
    lb, wb, pb, vb = b
    assert max_rel(la, lb) <= tol, (la, lb)
    assert tensor_err(wa, wb) <= tol
    assert tensor_err(np.c_[pa[0], pa[1], pa[2]], np.c_[pb[0], pb[1], pb[2]]) <= tol
    assert max_rel(va, vb) <= tol


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_group_sharded_epochs_match_single_gpu_fp64(engine, oracle, world):
    data = dataset(oracle, "monthly", 37, 4)
    cfg = TrainConfig(seed=7, batch_size=64, precision="fp64")
    ref = single_run(engine, data, cfg)
    res = group_run(engine, data, cfg, world, force=(world == 1))
    for r in range(world):
        assert_same(res[r], ref, 1e-10)
    # every rank holds bit-identical replicated state
    for r in range(1, world):
        assert res[r][0] == res[0][0]
        assert np.array_equal(res[r][1], res[0][1])


def test_group_sharded_fp32_tracks_single_gpu(engine, oracle):
    data = dataset(oracle, "quarterly", 60, 9)
    cfg = TrainConfig(seed=3, batch_size=128, precision="fp32")
    ref = single_run(engine, data, cfg)
    res = group_run(engine, data, cfg, 2)
    assert max_rel(res[0][0], ref[0]) < 1e-4
    assert tensor_err(res[0][1], ref[1]) < 1e-3
    assert abs(res[0][3] - ref[3]) < 0.01


def test_group_sharded_is_deterministic(engine, oracle):
    data = dataset(oracle, "quarterly", 25, 5)
    cfg = TrainConfig(seed=11, batch_size=64, precision="fp32")
    a = group_run(engine, data, cfg, 3)
    b = group_run(engine, data, cfg, 3)
    for r in range(3):
        assert a[r][0] == b[r][0]
        assert np.array_equal(a[r][1], b[r][1])


def test_nccl_one_rank_collective_path_matches_single_gpu(engine, oracle):
    """ncclAllReduce (captured in the epoch graph) + k_finalize + sharded k_adam, with a
    one-rank communicator: same trajectory as the single-GPU path."""
    prof, vals, cats = data = dataset(oracle, "quarterly", 23, 6)
    for precision, tol in (("fp64", 1e-10), ("fp32", 1e-4)):
        cfg = TrainConfig(seed=5, batch_size=64, precision=precision)
        ref = single_run(engine, data, cfg)
        t = Trainer((vals, cats), prof, cfg, api=engine, dist=(0, 1, engine.nccl_unique_id(), N.DIST_FORCE_COLLECTIVE))
        losses = [t.train_epoch() for _ in range(2)]
        v = t.validate()
        got = losses, t.weights_flat(), t.gather_per_series_arrays(), v.mean_smape
        assert_same(got, ref, tol)
        # run_batch through the collective: loss and gradients as single GPU
        b = t.all_windows()[:40]
        from paper_1907_03329_b200.trainer import WindowBatch
        g1 = t.batch_gradients(WindowBatch([x[0] for x in b], [x[1] for x in b]))
        s = Trainer((vals, cats), prof, cfg, api=engine)
        s.set_weights(t.weights_flat())
        s.set_per_series_arrays(*t.per_series_arrays())
        g0 = s.batch_gradients(WindowBatch([x[0] for x in b], [x[1] for x in b]))
        assert max_rel(g1.loss, g0.loss) <= tol
        for k in g0.network:
            assert tensor_err(g1.network[k], g0.network[k]) <= tol, k
        t.close()
        s.close()


def test_group_error_reaches_every_rank(engine, oracle):
    """A non-positive level in rank 1's shard: the reference throws NumericDomainError before
    apply_updates; every rank raises, no rank hangs, no rank updates past the failing step."""
    prof, vals, cats = dataset(oracle, "tiny", 6, 5)
    vals = vals.copy()
    vals[4, 3] = -vals[4, 3] * 50.0  # row 4 is rank 1's (rows [3, 6))
    world = 2
    grp = engine.group(world)
    cfg = TrainConfig(seed=1, batch_size=16, precision="fp64")
    trs = [Trainer((vals, cats), prof, cfg, api=engine, dist=(r, world, grp)) for r in range(world)]
    res = run_ranks(world, lambda r: trs[r].train_epoch())
    assert all(isinstance(x, E.NumericDomainError) for x in res), res
    assert "another rank" in str(res[0]) and "another rank" not in str(res[1])
    res = run_ranks(world, lambda r: trs[r].validate())
    assert all(isinstance(x, E.NumericDomainError) for x in res), res
    for t in trs:
        t.close()
    grp.close()


def test_sharded_snapshot_gathers_every_series(engine, oracle, tmp_path):
    """checkpoint.snapshot on every rank of a sharded run writes the same file as the
    single-GPU trainer would (per-series parameters gathered from their owners)."""
    prof, vals, cats = data = dataset(oracle, "quarterly", 19, 2)
    cfg = TrainConfig(seed=7, batch_size=32, precision="fp64")
    world = 2
    grp = engine.group(world)
    trs = [None, None]
    run_ranks(world, lambda r: trs.__setitem__(r, Trainer((vals, cats), prof, cfg, api=engine,
                                                          dist=(r, world, grp))))
    run_ranks(world, lambda r: trs[r].train_epoch())
    cks = run_ranks(world, lambda r: ck.snapshot(trs[r], with_training_state=False))
    single = Trainer((vals, cats), prof, cfg, api=engine)
    single.train_epoch()
    ref = ck.snapshot(single, with_training_state=False)
    for c in cks:
        assert not isinstance(c, Exception), c
        assert [i for i, _ in c.per_series] == [i for i, _ in ref.per_series]
        for (_, p), (_, q) in zip(c.per_series, ref.per_series):
            assert abs(p.alpha_raw - q.alpha_raw) <= 1e-10 * max(1.0, abs(q.alpha_raw))
            assert np.allclose(p.init_seasonality_raw, q.init_seasonality_raw, rtol=1e-10, atol=1e-12)
    # without gather=, a sharded trainer refuses to write a partial exact-resume state
    res = run_ranks(world, lambda r: ck.snapshot(trs[r], with_training_state=True))
    assert all(isinstance(x, E.CheckpointError) for x in res)
    for t in trs + [single]:
        t.close()
    grp.close()
