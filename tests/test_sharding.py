"""Multi-process (gloo, world_size 2 and 3, CPU) tests of the series-sharded data path.

What runs here is the host-side contract the engine implements (paper_1907_03329_b200/
sharding.py): contiguous row partition, per-rank filtering of the shared global batch,
partial losses/gradients scaled by the global mask count, one sum all-reduce.  Each rank
computes its partial with the fp64 oracle on its own rows; the all-reduced result must
equal the full-batch oracle result (loss, shared gradients, clip norm) and each rank's
per-series gradients must equal the full-batch ones for the series it owns.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from sharding_helpers import local_windows, shard_range, slots_first_appearance  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n, seed, B, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import ORACLE_LIB, dataset
        from paper_1907_03329_b200 import _native as N
        from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch
        api = N.NativeApi(ORACLE_LIB)
        prof, vals, cats = dataset(api, name, n, seed)
        cfg = TrainConfig(seed=7, batch_size=64, precision="fp64")
        tr = Trainer((vals, cats), prof, cfg, api=api)
        rng = np.random.default_rng(seed)
        w = tr.all_windows()
        idx = rng.integers(0, len(w), size=B)
        rows = [w[i][0] for i in idx]
        anchors = [w[i][1] for i in idx]
        O = prof.horizon
        M = float(B * O)
        mine = local_windows(rows, anchors, rank, world, n)
        if mine:
            b = WindowBatch([rows[i] for i in mine], [anchors[i] for i in mine])
            g = tr.batch_gradients(b)
            Mr = float(len(mine) * O)
            loss_sum = g.loss * Mr
            flat = np.concatenate([g.network[k].ravel() for k, *_ in tr.param_layout]) * (Mr / M)
            ps = {sid: np.r_[p.alpha_raw, p.gamma_raw, p.init_seasonality_raw] * (Mr / M)
                  for sid, p in g.per_series.items()}
            assert list(g.slot_rows) == slots_first_appearance(b.series_rows)
        else:
            loss_sum, flat, ps = 0.0, np.zeros(tr.n_values), {}
        ps_sq = sum(float(v @ v) for v in ps.values())
        buf = torch.tensor(np.r_[flat, ps_sq, loss_sum], dtype=torch.float64)
        dist.all_reduce(buf)  # the engine's single ncclAllReduce per step
        red = buf.numpy()
        if rank == 0:
            full = tr.batch_gradients(WindowBatch(rows, anchors))
            gfull = np.concatenate([full.network[k].ravel() for k, *_ in tr.param_layout])
            psf = {sid: np.r_[p.alpha_raw, p.gamma_raw, p.init_seasonality_raw] for sid, p in full.per_series.items()}
            out_q.put(("full", full.loss, gfull, float(sum(v @ v for v in psf.values())), psf))
        out_q.put(("rank", rank, red[-1] / M, red[:-2], red[-2], ps))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,n,seed,B", [(2, "quarterly", 9, 41, 96), (3, "monthly", 7, 5, 64),
                                                 (2, "yearly", 40, 3, 128)])
def test_sharded_step_decomposition_gloo(world, name, n, seed, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, seed, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in range(world + 1)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    full = next(m for m in msgs if m[0] == "full")
    _, loss_full, gfull, psq_full, ps_full = full
    ranks = [m for m in msgs if m[0] == "rank"]
    scale = np.max(np.abs(gfull))
    for _, rank, loss, g, psq, ps in ranks:
        assert abs(loss - loss_full) <= 1e-13 * abs(loss_full)
        assert np.max(np.abs(g - gfull)) <= 1e-13 * scale
        # clip norm from the reduced buffer equals the full-batch norm (trainer.hpp:603-615)
        assert abs((g @ g + psq) - (gfull @ gfull + psq_full)) <= 1e-12 * (gfull @ gfull + psq_full)
        b, e = shard_range(rank, world, n)
        for sid, v in ps.items():
            assert b <= int(sid[1:]) < e  # per-series state never leaves its owner
            np.testing.assert_allclose(v, ps_full[sid], rtol=1e-12, atol=1e-12 * np.max(np.abs(ps_full[sid])))


def test_shard_partition_covers_rows_exactly():
    for n in (1, 7, 1000, 48000):
        for world in (1, 2, 4, 8):
            spans = [shard_range(r, world, n) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1
