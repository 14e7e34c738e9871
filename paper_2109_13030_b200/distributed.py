"""Sharded multi-GPU solve: one process per GPU, torch.distributed for plumbing.

The batch is split into contiguous shards (rank r owns global instances
[r B, (r+1) B), bmc_problem.index_base = r B); every rank builds the same
scene from the seed, so there is no broadcast.  The only data-path collective
is the best-of-batch exchange: each rank packs {key, 55 coefficients} of its
shard's best into a 256-byte record (bmc_pack_best, our kernel), the records
are all-gathered (NCCL over NVLink on GPUs, gloo in the CPU tests), and every
rank selects the minimum key (bmc_select_best, our kernel), so all ranks hold
the same global best.

Determinism: an instance's output bits depend only on its inputs and the team
size (warps per instance, include/bmc.h).  The sharded solves pass the team
that the whole batch would use on one GPU (Solver.team_for(global_batch)), so
every instance -- and hence the global best -- is bitwise the unsharded solve's.
A rank whose shard is empty (global batch < world size) runs no solve and
contributes the key ~0, which never wins.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from .bmc import _check, load_library

RECORD_WORDS = 32


def pack_record(best, coeffs, index_base: int, record, stream, residual=None, cost=None):
    """bmc_pack_best on device tensors: {key, 55 coefficients, r1, r_psi, J} of the
    instance `best` names, gathered on the device into one 256-byte record."""
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    _check(load_library().bmc_pack_best(ptr(best), ptr(coeffs), ptr(residual), ptr(cost), C.c_int64(index_base),
                                        ptr(record), stream))


class BestExchange:
    """Best-of-batch exchange over a process group.

    `pack` / `select` default to the library's device kernels; the CPU tests
    (gloo) inject host implementations to exercise the collective plumbing."""

    def __init__(self, group, device, pack: Optional[Callable] = None, select: Optional[Callable] = None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.device = device
        self.record = torch.zeros(RECORD_WORDS, dtype=torch.int64, device=device)
        self.records = torch.zeros(self.world * RECORD_WORDS, dtype=torch.int64, device=device)
        self.best = torch.zeros(2, dtype=torch.int64, device=device)
        self.coeffs = torch.zeros(55, dtype=torch.float32, device=device)
        self._pack = pack or self._pack_device
        self._select = select or self._select_device

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _pack_device(self, best, coeffs, index_base, record, residual=None, cost=None):
        pack_record(best, coeffs, index_base, record, self._stream(), residual, cost)

    def _select_device(self, records, nranks, best_out, coeffs_out):
        _check(load_library().bmc_select_best(C.c_void_p(records.data_ptr()), C.c_int32(nranks),
                                              C.c_void_p(best_out.data_ptr()),
                                              C.c_void_p(coeffs_out.data_ptr()), self._stream()))

    def exchange(self, best, coeffs, index_base: int, residual=None, cost=None):
        """best: [2] int64 of this shard's solve; coeffs: [B, 5, 11] of this shard
        (residual [B, 2] / cost [B] optional: carried in the record, floats 55..57).
        Returns (global best [2], best coefficients [55]) on every rank; the
        winning record is self.records[rank * RECORD_WORDS ...] of the min key."""
        import torch.distributed as dist
        if residual is None and cost is None:
            self._pack(best, coeffs, index_base, self.record)
        else:
            self._pack(best, coeffs, index_base, self.record, residual, cost)
        dist.all_gather_into_tensor(self.records, self.record, group=self.group)
        self._select(self.records, self.world, self.best, self.coeffs)
        return self.best, self.coeffs


def shard_bounds(global_batch: int, world: int, rank: int):
    """Contiguous shard of rank `rank`: (start, size), ceil(B / world) per rank."""
    per = -(-global_batch // world)
    start = min(rank * per, global_batch)
    return start, max(0, min(per, global_batch - start))


EMPTY_KEY = -1   # best = {0, -1}: key ~0 (bmc_pack_best), the record of an empty shard


def _empty_shard(device):
    import torch
    return dict(best=torch.tensor([0, EMPTY_KEY], dtype=torch.int64, device=device),
                coeffs=torch.zeros((1, 5, 11), dtype=torch.float32, device=device))


def solve_sharded(solver, xchg: Optional[BestExchange], init, obs_xy, obs_ab, bnd, iters: int, index_base: int,
                  lambda_in=None, out: Optional[dict] = None, team: int = 0):
    """One rank's part of a batch solve sharded over a process group (SURVEY.md
    §3 call stack 3): bmc_solve on this rank's shard (device tensors, current
    stream), then the best-of-batch exchange.  `team`: the team size of the
    whole batch (Solver.team_for(global batch)) for results bitwise equal to the
    unsharded solve; 0 lets the shard size decide.  Returns (shard outputs,
    global best [2], best coefficients [55]); with xchg None (one rank) the
    shard's own best.  Asynchronous on the current stream like Solver.solve."""
    if int(init.shape[0]) == 0:
        out = _empty_shard(init.device)
    else:
        out = solver.solve(init, obs_xy, obs_ab, bnd, iters, lambda_in=lambda_in, index_base=index_base, out=out,
                           team=team)
    if xchg is None:
        return out, out["best"], None
    best, coeffs = xchg.exchange(out["best"], out["coeffs"], index_base)
    return out, best, coeffs


def solve_sharded_host(solver, xchg: Optional[BestExchange], init, obs_xy, obs_ab, bnd, iters: int,
                       index_base: int, out: dict, lambda_in=None, best_host=None, coeffs_host=None,
                       team: int = 0):
    """End-to-end variant from host buffers: bmc_solve_host on the shard (page-locked
    buffers are accessed in place), then -- for more than one rank -- the exchange
    reads the shard's best and coefficients from those page-locked output buffers
    (mapped into the device address space) and the global best (16 B) and its
    coefficients (220 B) are copied back into `best_host` / `coeffs_host`.
    Synchronous.  Returns (out, best_host, coeffs_host)."""
    import torch
    if init is not None and int(init.shape[0]) == 0:
        out.update(best=np.array([0, EMPTY_KEY], np.int64), coeffs=np.zeros((1, 5, 11), np.float32))
    else:
        solver.solve_host(init, obs_xy, obs_ab, bnd, iters, lambda_in=lambda_in, index_base=index_base, out=out,
                          team=team)
    if xchg is None:
        return out, out["best"], None
    dev = torch.device(xchg.device)
    best_t = torch.from_numpy(out["best"])
    coeffs_t = torch.from_numpy(out["coeffs"])
    if dev.type == "cuda" and not (best_t.is_pinned() and coeffs_t.is_pinned()):
        best_t, coeffs_t = best_t.to(dev), coeffs_t.to(dev)   # pageable outputs: staged on the device
    best, coeffs = xchg.exchange(best_t, coeffs_t, index_base)
    if best_host is None:
        best_host = np.empty(2, np.int64)
    if coeffs_host is None:
        coeffs_host = np.empty(55, np.float32)
    torch.from_numpy(best_host).copy_(best, non_blocking=True)
    torch.from_numpy(coeffs_host).copy_(coeffs, non_blocking=True)
    if dev.type == "cuda":
        torch.cuda.current_stream(dev).synchronize()
    return out, best_host, coeffs_host
