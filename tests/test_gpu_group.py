"""mm_group (include/mmgpu.h): one process, n GPUs — the reference's n_workers
mapped to GPUs. The box this runs on has one B200, so the group here has one
GPU; the NCCL exchange path (all-gather of the counts, per-shard broadcast of
exactly the records) still runs, over a one-rank communicator. The
multi-rank assembly protocol is covered on CPU with gloo
(tests/test_shard_gloo.py)."""
import numpy as np
import pytest

import oracle
from conftest import first_diff, records_equal
from paper_1308_4011_b200 import Engine, Group, MMError, MMRangeError, System, Thresholds, abi

pytestmark = pytest.mark.gpu


def test_group_one_gpu_equals_engine():
    s = System.generate(seed=2, n_classes=3000, n_methods=30000, n_attributes=50000, k_max_calls=5,
                        k_max_accesses=5, intra_class_bias=0.4)
    with Engine(0) as e, Group(n=1) as g:
        e.upload(s)
        t = e.compute_thresholds()
        want = e.suggest_all(t)
        g.upload(s)
        assert g.shards() == [(0, s.n_classes)]
        for _ in range(3):  # capture, then graph replays
            n = g.run(thresholds=None)
            got = g.suggestions()
            assert n == len(want) and records_equal(got, want), first_diff(got, want)
        assert g.counts() == [len(want)]
        # explicit thresholds, all-candidates mode
        want2 = e.suggest_all(Thresholds(0.0, 0.2, 1.0), all_candidates=True)
        g.run(thresholds=Thresholds(0.0, 0.2, 1.0), all_candidates=True)
        assert records_equal(g.suggestions(), want2)
        l, k, c = oracle.class_metrics(s)
        to = oracle.thresholds(l, c)
        o = oracle.suggest(s, l, c, abi.MM_CRIT_COHESION | abi.MM_CRIT_COUPLING, 0, False, 1, to.lcom, to.cbo)
        g.run(thresholds=None)
        assert records_equal(g.suggestions(), o)


def test_group_errors():
    import torch
    n_dev = torch.cuda.device_count()
    with pytest.raises(MMError):
        Group(devices=[])  # zero workers: plan_partition's invalid_argument
    with pytest.raises(MMRangeError):
        Group(devices=[n_dev])  # no such device
    with pytest.raises(MMRangeError):
        Group(devices=[0, 0])  # a GPU twice
    with Group(n=1) as g:
        with pytest.raises(MMError):
            g.run()  # no model yet
