"""Multi-rank trial sharding + statistics collective, world_size 2 over gloo
on CPU.  The per-pair compute is the CPU oracle (test-only stand-in for the
GPU kernels); what is under test is the sharding and gather logic that
bench.py runs over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1905_07439_b200 import distributed


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pair_errors(ids):
    """(2, len(ids)) det/rand errors of small Strassen pairs via the oracle."""
    from dataclasses import replace

    from oracle import engine as oracle
    from paper_1905_07439_b200.configs import get_config
    from paper_1905_07439_b200.multiply import mode_tensors
    from paper_1905_07439_b200.randomize import plan_levels

    cfg = replace(get_config("c1"), N=16, Q=2)
    f = cfg.formula_obj()
    out = np.zeros((2, len(ids)))
    for k, p in enumerate(ids):
        A, B = cfg.pair(p)
        ref = oracle.standard_multiply(A.astype(np.float64), B.astype(np.float64))
        rp = cfg.plan(p)
        for row, levels in enumerate((
            [mode_tensors(f, cfg.mode)] * cfg.Q,
            [plan_levels(f, [rp.levels[q]], cfg.mode) for q in range(cfg.Q)],
        )):
            C = oracle.apply_levels(levels, A[None], B[None], cfg.mode)
            out[row, k] = oracle.rel_errors(C, ref)[0]
    return out


def _worker(rank, world, port, per_rank, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = distributed.pair_ids(rank, world, per_rank)
    local = _pair_errors(ids)
    allerr = distributed.gather_trials(local)
    tmax = distributed.max_over_ranks([1.0 + rank, 5.0 - rank])
    if rank == 0:
        q.put((allerr, tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_layout():
    assert distributed.pair_ids(0, 2, 3) == [1, 2, 3]
    assert distributed.pair_ids(1, 2, 3) == [4, 5, 6]
    with pytest.raises(ValueError):
        distributed.shard(2, 2, 3)


def test_two_rank_gather_equals_single_process():
    world, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    allerr, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = _pair_errors(list(range(1, world * per_rank + 1)))
    assert np.array_equal(allerr, single)
    assert tmax.tolist() == [2.0, 5.0]
    s_multi = distributed.trial_stats(allerr[1], allerr[0])
    s_single = distributed.trial_stats(single[1], single[0])
    assert s_multi == s_single
