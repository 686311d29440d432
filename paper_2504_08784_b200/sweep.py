"""Multi-GPU planning sweeps: independent instances sharded across ranks, one
final gather of fixed-size result records.

One process per GPU (torch.distributed, NCCL on the B200 box). Each rank uploads
its shard once (instances stay resident in HBM), solves it with the sm_100a
pipeline on its own stream, writes one 88-byte slos_record per instance straight
into a device tensor, and the ranks all-gather those records -- the only
inter-GPU traffic. There is no exchange during the solve: the DP is
instance-local. With world_size 1 the gather is skipped.

The same class drives the CPU checkers (records land in host memory) so the
sharding and gather logic is covered by world_size-2 gloo tests on CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .planner import PlannerConfig, SloConfig, _Handle
from .workload import TWO_TIER_SLO, InstanceBatch, StressSpec


def shard_range(n_total: int, rank: int, world: int) -> range:
    """Contiguous balanced shard (strong scaling)."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def weak_seeds(rank: int, per_rank: int, base: int = 0) -> range:
    """Per-rank seeds for weak scaling (per-GPU work fixed as N grows)."""
    return range(base + rank * per_rank, base + (rank + 1) * per_rank)


@dataclass
class ShardSpec:
    family: StressSpec
    model: list
    cfg: PlannerConfig
    slo: SloConfig = field(default_factory=lambda: TWO_TIER_SLO)


class ShardSolver:
    """Device-resident shard of planning instances behind one slos_workspace."""

    def __init__(self, lib, spec: ShardSpec, seeds, unit_value: bool = False, batch: InstanceBatch = None,
                 handles=None):
        self.lib = lib
        # a stress-family shard (seeds) or any prepared batch (e.g. a recorded corpus)
        self.batch = batch if batch is not None else InstanceBatch.stress(spec.family, list(seeds), spec.slo)
        self.handle = _Handle(lib, spec.model, spec.slo, spec.cfg) if spec is not None else None
        self.n = self.batch.n
        self.unit_value = 1 if unit_value else 0
        ws = C.c_void_p()
        st = lib.slos_workspace_create(C.byref(ws))
        if st != abi.SLOS_OK:
            raise RuntimeError(lib.slos_last_error().decode())
        self.ws = ws
        # one planner handle for every instance, or one per instance (mixed planner
        # configurations, e.g. the C5 corpus' speculative and AR instances)
        self._handles = handles
        ptrs = [h.ptr for h in handles] if handles is not None else [self.handle.ptr] * self.n
        self._hs = (C.c_void_p * self.n)(*ptrs)
        self._outs = (abi.Result * self.n)()

    def upload(self, stream=None) -> None:
        st = self.lib.slos_workspace_upload(self.ws, self._hs, self.n, C.c_void_p(self.batch.inputs_ptr()),
                                            self.unit_value, self._outs, stream)
        if st != abi.SLOS_OK:
            raise RuntimeError(self.lib.slos_last_error().decode())

    def solve(self, stream=None) -> None:
        st = self.lib.slos_workspace_solve(self.ws, stream)
        if st != abi.SLOS_OK:
            raise RuntimeError(self.lib.slos_last_error().decode())

    def records(self, out_ptr: int, stream=None) -> None:
        st = self.lib.slos_workspace_records(self.ws, C.c_void_p(out_ptr), stream)
        if st != abi.SLOS_OK:
            raise RuntimeError(self.lib.slos_last_error().decode())

    def converge(self, rec_tensor, stream=None, rounds: int = 4) -> None:
        """Solve once; if an instance overflowed its scratch estimate, let download
        regrow it (the workspace remembers) so every later solve fits."""
        import torch
        for _ in range(rounds):
            self.solve(stream)
            self.records(rec_tensor.data_ptr(), stream)
            torch.cuda.synchronize()
            st = records_view(rec_tensor)["status"]
            if not (st == abi.SLOS_ERR_CAPACITY).any():
                return
            self.download(stream)
            self.free_results()

    def kernel_ms(self):
        ms = (C.c_float * 2)()
        self.lib.slos_workspace_kernel_ms(self.ws, ms)
        return float(ms[0]), float(ms[1])

    def stage_ms(self):
        """[anchor_kernel, dp_kernel, build_kernel, scratch init] device ms of the last solve."""
        ms = (C.c_float * 4)()
        self.lib.slos_workspace_stage_ms(self.ws, ms, 4)
        return [float(x) for x in ms]

    def launches(self) -> int:
        """Kernels the last solve launched (0 for the CPU checkers)."""
        n = C.c_int64()
        self.lib.slos_workspace_launches(self.ws, C.byref(n))
        return int(n.value)

    def download(self, stream=None):
        st = self.lib.slos_workspace_download(self.ws, self._outs, stream)
        if st != abi.SLOS_OK:
            raise RuntimeError(self.lib.slos_last_error().decode())
        return self._outs

    def free_results(self) -> None:
        for k in range(self.n):
            self.lib.slos_result_free(C.byref(self._outs[k]))

    def close(self) -> None:
        if self.ws:
            self.lib.slos_workspace_destroy(self.ws)
            self.ws = None


def gather_records(local, world: int, group=None, n_total: int = None):
    """All-gather fixed-size record tensors (uint8 [n, 88]) from every rank.

    With n_total given, the ranks hold the uneven contiguous shards of
    shard_range(n_total, r, world): each pads to ceil(n_total / world) rows for
    the collective and the padding is trimmed after it, so any world size works."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    rows = local.shape[0] if n_total is None else -(-n_total // world)
    if local.shape[0] != rows:
        pad = torch.zeros((rows, local.shape[1]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]].copy_(local)
        local = pad
    out = torch.empty((world * rows, local.shape[1]), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local, group=group)
    else:  # gloo (CPU tests)
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local, group=group)
        out = torch.cat(parts, dim=0)
    if n_total is not None and rows * world != n_total:
        out = torch.cat([out[r * rows: r * rows + len(shard_range(n_total, r, world))] for r in range(world)])
    return out


def records_view(t) -> np.ndarray:
    """numpy structured view of a record tensor (host copy)."""
    arr = t.detach().cpu().numpy().reshape(-1)
    return arr.view(abi.RECORD_DTYPE)
