"""Multi-rank sweep assembly on CPU (gloo, world_size 2 and 3).

Each rank sweeps its cost-balanced class range (here with the oracle standing
in for its GPU, since this box has none), the shard lists are all-gathered
with paper_1308_4011_b200.shard.allgather_records — the exact function
bench.py runs over NCCL — and the rank-order concatenation must equal the
single-process suggest_all list record for record."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1308_4011_b200 import System, abi, plan_shards
    from paper_1308_4011_b200.shard import allgather_records, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = System.generate(**cfg)
        lcom, ck, cbo = oracle.class_metrics(s)           # replicated metric pass
        t = oracle.thresholds(lcom, cbo)
        crit = abi.MM_CRIT_COHESION | abi.MM_CRIT_COUPLING
        b = plan_shards(s, world)
        lo, hi = shard_range(b, rank)
        mine = oracle.suggest(s, lcom, cbo, crit, 0, False, 1, t.lcom, t.cbo, class_range=(lo, hi))
        local = torch.from_numpy(mine.view(np.uint8).copy())
        allrec, counts = allgather_records(local, len(mine))
        if rank == 0:
            full = oracle.suggest(s, lcom, cbo, crit, 0, False, 1, t.lcom, t.cbo)
            got = allrec.numpy().view(abi.SUGGESTION_DTYPE)
            fields = [f for f in full.dtype.names if f != "pad"]
            ok = len(got) == len(full) and all(got[f].tobytes() == full[f].tobytes() for f in fields)
            q.put((ok, counts, len(full)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sweep_allgather_equals_full_list(world):
    cfg = dict(seed=9, n_classes=300, n_methods=3000, n_attributes=5000, k_max_calls=4, k_max_accesses=4,
               intra_class_bias=0.4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    ok, counts, n = q.get(timeout=10)
    assert ok, (counts, n)
    assert sum(counts) == n and len(counts) == world
