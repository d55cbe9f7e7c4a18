"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: lateral-slice partition, NCCL-id
exchange, one-time replication of A, max-over-ranks timing and the reassembly of C.

The per-rank compute here is the fp64 ORACLE (tests may call it): what is tested is that the
partition is exact -- the shards of C computed independently from (A, B_r) reassemble to A * B --
and the host plumbing bench.py uses around libtprod.so on the GPU box."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n1, n2, n3, n4, ret):
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_1806_07247_b200 import dist as D
    from synth import normal

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # NCCL-id exchange (a random 128-byte token stands in for ncclGetUniqueId)
        uid = D.exchange_uid(lambda: os.urandom(128))
        all_ids = [None] * world
        dist.all_gather_object(all_ids, uid)
        assert len(uid) == 128 and all(x == uid for x in all_ids)

        # A exists on rank 0 only, then is replicated once
        A = torch.from_numpy(normal((n1, n2, n3), 0, np.float64)) if rank == 0 else \
            torch.zeros((n3, n2, n1), dtype=torch.float64).permute(2, 1, 0)
        D.replicate(A, root=0)
        assert np.array_equal(A.numpy(), normal((n1, n2, n3), 0, np.float64))

        # each rank owns a lateral block of B and computes its block of C; the rank draws its block
        # straight from the global stream (bench.py's strong-scaling inputs) -- same values
        Bfull = normal((n2, n4, n3), 1, np.float64)
        s, e = D.lateral_shard(n4, world, rank)
        from synth import normal_lateral
        assert np.array_equal(normal_lateral((n2, n4, n3), 1, s, e, np.float64), Bfull[:, s:e, :])
        C_r = O.tprod_bcirc(A.numpy(), np.asfortranarray(Bfull[:, s:e, :]))
        Ct = torch.from_numpy(np.asfortranarray(C_r))
        full = D.gather_lateral(Ct, n4)
        t = D.max_over_ranks(1.0 + rank)
        if rank == 0:
            ref = O.tprod_bcirc(A.numpy(), Bfull)
            ret["err"] = O.rel_err(full.numpy(), ref)
            ret["max"] = t
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n4", [9, 10])
def test_lateral_partition_gloo_ws2(n4):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, 7, 5, 6, n4, ret), nprocs=2, start_method="spawn", join=True)
    assert ret["err"] < 1e-14
    assert ret["max"] == 2.0


def test_lateral_shard_covers_exactly():
    from paper_1806_07247_b200.dist import lateral_shard
    for n4 in (1, 7, 512, 8192):
        for w in (1, 2, 3, 4, 8):
            spans = [lateral_shard(n4, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n4
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        lateral_shard(8, 2, 2)
