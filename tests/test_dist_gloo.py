"""Multi-process (gloo, world size 2, CPU) checks of the sequence-sharded path's host logic:
shard arithmetic, sharding-stable input generation, and that the per-rank results gathered in rank
order equal the single-process full-batch results (the oracle stands in for the GPU step here; the GPU
kernel's own shard bit-identity is tests/test_gpu_plans.py::test_sharded_equals_one_gpu)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from lf_synth import Synth, Workload, bits
from paper_2603_11504_b200 import dist as lfd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_arithmetic():
    assert lfd.shard(256, 8, 3, "weak") == (256, 768, 2048)
    assert lfd.shard(256, 8, 3, "strong") == (32, 96, 256)
    with pytest.raises(ValueError):
        lfd.shard(10, 4, 0, "strong")
    covered = sorted(b for r in range(4) for b in range(lfd.shard(64, 4, r, "strong")[1],
                                                          sum(lfd.shard(64, 4, r, "strong")[:2])))
    assert covered == list(range(64))


WL = Workload("dist", 4, 8, 2, 64, 40, 36, 6)


def _worker(rank, world, port, resq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        B, b0, Bt = lfd.shard(WL.B, world, rank, "strong")
        syn = Synth(WL, seed=4, B=B, b0=b0)
        orc = oracle.OracleCache(B, WL.Hq, WL.Hkv, WL.d, WL.N)
        K, V = syn.prefill()
        for b in range(B):
            orc.prefill(b, bits(K[b]), bits(V[b]))
        outs, slots = [], []
        for _ in range(WL.steps):
            q, kn, vn = syn.step()
            o, s, _ = orc.step(bits(q), bits(kn), bits(vn))
            outs.append(lfd.gather_rows(torch.from_numpy(o)))
            slots.append(lfd.gather_rows(torch.from_numpy(s)))
        t = lfd.max_over_ranks(float(rank + 1))
        Kall = lfd.gather_rows(torch.from_numpy(orc.K.astype(np.int32)))
        if rank == 0:
            resq.put((torch.stack(outs).numpy(), torch.stack(slots).numpy(), t, Kall.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_equals_full_batch():
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs, slots, t, Kall = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0
    # single process, full batch
    syn = Synth(WL, seed=4)
    orc = oracle.OracleCache(WL.B, WL.Hq, WL.Hkv, WL.d, WL.N)
    K, V = syn.prefill()
    for b in range(WL.B):
        orc.prefill(b, bits(K[b]), bits(V[b]))
    for t_ in range(WL.steps):
        qq, kn, vn = syn.step()
        o, s, _ = orc.step(bits(qq), bits(kn), bits(vn))
        np.testing.assert_array_equal(outs[t_], o)
        np.testing.assert_array_equal(slots[t_], s)
    np.testing.assert_array_equal(Kall.astype(np.uint16), orc.K)
