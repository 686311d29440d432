"""Multi-rank sweep logic (sharding + the final record gather) on CPU: two gloo
ranks each solve their weak-scaling shard through the C-ABI (the CPU oracle
stands in for the device here) and all-gather the fixed-size slos_records;
the gathered records must equal a single-process solve of every instance."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200 import workload as W
from paper_2504_08784_b200.sweep import ShardSolver, ShardSpec, gather_records, records_view, shard_range, weak_seeds

PER = 6


def _spec():
    F = W.FAMILIES["C1"]
    return ShardSpec(F["spec"], F["model"], F["cfg"])


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = abi.oracle()
    solver = ShardSolver(lib, _spec(), weak_seeds(rank, PER))
    solver.upload()
    solver.solve()
    rec = torch.zeros((PER, C.sizeof(abi.Record)), dtype=torch.uint8)
    solver.records(rec.data_ptr())
    allrec = gather_records(rec, world)
    if rank == 0:
        np.save(os.path.join(outdir, "gathered.npy"), allrec.numpy())
    solver.close()
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition():
    for n in (0, 1, 7, 1024, 1025):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            flat = [x for r in rs for x in r]
            assert flat == list(range(n))
            assert max(len(r) for r in rs) - min(len(r) for r in rs) <= 1


def test_two_rank_gather_equals_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npy").reshape(-1).view(abi.RECORD_DTYPE)
    lib = abi.oracle()
    solver = ShardSolver(lib, _spec(), range(world * PER))
    solver.upload()
    solver.solve()
    rec = torch.zeros((world * PER, C.sizeof(abi.Record)), dtype=torch.uint8)
    solver.records(rec.data_ptr())
    want = records_view(rec)
    solver.close()
    assert got.tobytes() == want.tobytes()
    assert (got["status"] == 0).all() and got["n_entries"].min() > 0


def _uneven_worker(rank, world, port, outdir, n_total):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = abi.oracle()
    mine = shard_range(n_total, rank, world)
    solver = ShardSolver(lib, _spec(), mine)
    solver.upload()
    solver.solve()
    rec = torch.zeros((len(mine), C.sizeof(abi.Record)), dtype=torch.uint8)
    solver.records(rec.data_ptr())
    allrec = gather_records(rec, world, n_total=n_total)
    if rank == 0:
        np.save(os.path.join(outdir, "gathered.npy"), allrec.numpy())
    solver.close()
    dist.barrier()
    dist.destroy_process_group()


def test_three_rank_uneven_strong_scaling_gather(tmp_path):
    """Strong scaling with a total the world size does not divide (7 over 3 ranks:
    shards of 3, 2, 2): the padded gather returns exactly the 7 records in order."""
    world, n_total = 3, 7
    mp.spawn(_uneven_worker, args=(world, _free_port(), str(tmp_path), n_total), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npy").reshape(-1).view(abi.RECORD_DTYPE)
    lib = abi.oracle()
    solver = ShardSolver(lib, _spec(), range(n_total))
    solver.upload()
    solver.solve()
    rec = torch.zeros((n_total, C.sizeof(abi.Record)), dtype=torch.uint8)
    solver.records(rec.data_ptr())
    want = records_view(rec)
    solver.close()
    assert len(got) == n_total and got.tobytes() == want.tobytes()
