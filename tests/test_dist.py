"""Multi-process (gloo, world size 2) checks of the patch-sharding plumbing.

The GPU path shards patches across ranks with no data-path collective; these
CPU tests cover the host logic: shard arithmetic, the counter merge (the
reference's ScoreCounter.merge summed across ranks) and the max-over-ranks
timing reduction, and that sharded oracle encodes equal the unsharded one."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1412_0680_b200.dist import shard_range


def test_shard_range_covers_exactly():
    for total in (0, 1, 7, 10_000, 1_048_576):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from conftest import flat_from_fixture, golden
    from oracle import stmp_oracle as O
    from paper_1412_0680_b200.dist import max_over_ranks, merge_counters, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = golden("pursuit_small.npz")
        a64 = z["atoms"].astype(np.float64)
        sel = O.tree_selector(O.OracleTree.from_flat(flat_from_fixture(z)), a64, 1 / 16)
        lo, hi = shard_range(len(z["X"]), rank, world)
        res = O.encode_batch(sel, a64, z["X"][lo:hi], int(z["K"]), "omp")
        local = torch.tensor([sum(r["ip"] for r in res), sum(r["cip"] for r in res)], dtype=torch.int64)
        tot = merge_counters(local)
        ms = max_over_ranks(10.0 * (rank + 1))
        idx = torch.tensor(O.pack(res, int(z["K"]))["idx"], dtype=torch.int64)
        gathered = [torch.zeros((shard_range(len(z["X"]), r, world)[1] - shard_range(len(z["X"]), r, world)[0],
                                 int(z["K"])), dtype=torch.int64) for r in range(world)]
        dist.all_gather(gathered, idx)
        if rank == 0:
            out.put((tot, ms, torch.cat(gathered).numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_encode_matches_single_rank():
    from conftest import golden
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    (ip, cip), ms, idx = q.get()
    z = golden("pursuit_small.npz")
    assert ip == int(z["tree_omp_ip"][:, 0].sum())
    assert cip == int(z["tree_omp_ip"][:, 1].sum())
    assert ms == 20.0
    np.testing.assert_array_equal(idx, z["tree_omp_idx"])
