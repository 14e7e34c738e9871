"""Multi-process (world_size 2, gloo, CPU) tests of the sharded-solve plumbing.

The device kernels bmc_pack_best / bmc_select_best need a GPU, so here host
implementations with the same record layout are injected into BestExchange;
what is under test is the collective plumbing: shard bounds, the all-gather
of one 256-byte record per rank, and that every rank ends with the same
global best (minimum packed key; keys carry the global index, so the result
is independent of rank order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_13030_b200.distributed import (EMPTY_KEY, RECORD_WORDS, BestExchange, shard_bounds,
                                               solve_sharded, solve_sharded_host)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def host_pack(best, coeffs, index_base, record, residual=None, cost=None):
    """bmc_pack_best's record (include/bmc.h); key -1 = empty shard, no coefficients."""
    local = int(best[0]) - index_base
    record.zero_()
    record[0] = best[1]
    f = torch.zeros(2 * (RECORD_WORDS - 1), dtype=torch.float32)
    if int(best[1]) != EMPTY_KEY:
        f[:55] = coeffs[local].reshape(-1)
    record[1:] = f.view(torch.int64)


def host_select(records, nranks, best_out, coeffs_out):
    """bmc_select_best: minimum key compared as unsigned (the empty-shard key ~0 never wins)."""
    r = records.view(nranks, RECORD_WORDS)
    keys = r[:, 0]
    i = int(np.argmin(keys.numpy().view(np.uint64)))
    best_out[0] = int(keys[i]) & ((1 << 30) - 1)
    best_out[1] = keys[i]
    coeffs_out.copy_(r[i, 1:].clone().view(torch.float32)[:55])


class _FakeSolver:
    """Stands in for Solver.solve_host: writes a fixed shard result into `out`."""

    def __init__(self, best, coeffs):
        self.best, self.coeffs = best, coeffs

    def solve_host(self, init, obs_xy, obs_ab, bnd, iters, lambda_in=None, index_base=0, out=None, team=0):
        assert team == 3                   # the caller's team is passed through
        out["best"][...] = self.best
        out["coeffs"][...] = self.coeffs
        return out


def _key(infeasible, value, gidx):
    bits = int(np.array([value], dtype=np.float32).view(np.uint32)[0])
    return (infeasible << 62) | (bits << 30) | gidx


def _worker(rank, world, port, scenario, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B_glob = 11
        start, size = shard_bounds(B_glob, world, rank)
        coeffs = torch.arange(size * 55, dtype=torch.float32).reshape(size, 5, 11) + 1000 * rank
        # scenario: per-rank best keys chosen so that rank 1 holds the global best
        if scenario == "rank1_best":
            key = _key(0, 0.5 if rank == 1 else 0.75, start + size - 1)
        elif scenario == "tie_value":
            key = _key(0, 0.5, start)      # equal values: the lower global index wins
        else:                              # all infeasible: minimum residual wins
            key = _key(1, 2.0 - rank, start)
        best = torch.tensor([key & ((1 << 30) - 1), key], dtype=torch.int64)
        x = BestExchange(dist.group.WORLD, torch.device("cpu"), pack=host_pack, select=host_select)
        gb, gc = x.exchange(best, coeffs, start)
        out[rank] = (int(gb[0]), int(gb[1]), float(gc[0]), float(gc[54]))
        # the same exchange through the end-to-end entry point (host buffers)
        solver = _FakeSolver(best.numpy(), coeffs.numpy())
        res = dict(best=np.empty(2, np.int64), coeffs=np.empty((size, 5, 11), np.float32))
        _, hb, hc = solve_sharded_host(solver, x, None, None, None, None, 1, start, out=res, team=3)
        assert (int(hb[0]), int(hb[1]), float(hc[0]), float(hc[54])) == out[rank]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scenario,expect_rank", [("rank1_best", 1), ("tie_value", 0), ("infeasible", 1)])
def test_best_exchange_two_ranks(scenario, expect_rank):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, scenario, out), nprocs=world, start_method="spawn")
    res = dict(out)
    assert res[0] == res[1], res                       # every rank holds the same global best
    start, size = shard_bounds(11, world, expect_rank)
    idx, key, c0, c54 = res[0]
    assert idx == (key & ((1 << 30) - 1))
    assert start <= idx < start + size
    local = idx - start
    assert c0 == local * 55 + 1000 * expect_rank and c54 == local * 55 + 54 + 1000 * expect_rank


def test_shard_bounds_cover_the_batch():
    for B in (1, 7, 1000, 16384):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(B, world, r) for r in range(world)]
            covered = np.zeros(B, dtype=int)
            for s, n in spans:
                covered[s:s + n] += 1
            assert np.all(covered == 1)


def _worker_empty(rank, world, port, out):
    """Global batch 1 over 2 ranks: rank 1's shard is empty (no solve, key ~0)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, size = shard_bounds(1, world, rank)
        x = BestExchange(dist.group.WORLD, torch.device("cpu"), pack=host_pack, select=host_select)

        class _Solver:
            def solve(self, init, obs_xy, obs_ab, bnd, iters, lambda_in=None, index_base=0, out=None, team=0):
                assert size == 1
                return dict(best=torch.tensor([0, _key(1, 3.0, 0)], dtype=torch.int64),
                            coeffs=torch.full((1, 5, 11), 7.0))

        init = torch.zeros((size, 3, 11))
        _, gb, gc = solve_sharded(_Solver(), x, init, None, None, None, 1, start)
        out[rank] = (int(gb[0]), int(gb[1]), float(gc[0]))
    finally:
        dist.destroy_process_group()


def test_empty_shard_never_wins():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker_empty, args=(world, port, out), nprocs=world, start_method="spawn")
    res = dict(out)
    assert res[0] == res[1] == (0, _key(1, 3.0, 0), 7.0), res
