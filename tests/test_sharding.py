"""Multi-rank screening host logic on CPU: world_size 2 over gloo.

Each rank takes its contiguous shard of the global ligand index space, generates it
independently, docks it (here with the CPU oracle standing in for the device call, since this
container has no GPU) and the result records are gathered; the union must equal a single-rank
run of the whole range, record for record."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_05069_b200 import shard


def test_shard_range_partition():
    for n in (0, 1, 7, 100, 10_000_001):
        for w in (1, 2, 3, 8):
            rs = [shard.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_balanced_bounds():
    rng = np.random.default_rng(0)
    cost = rng.uniform(1, 100, size=10_000)
    b = shard.balanced_bounds(cost, 8)
    assert b[0] == 0 and b[-1] == 10_000 and all(b[i] <= b[i + 1] for i in range(8))
    sums = [cost[b[i]:b[i + 1]].sum() for i in range(8)]
    assert max(sums) / min(sums) < 1.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2209_05069_b200 import io, model
    from paper_2209_05069_b200.native import InteractionTable
    lo, hi = shard.shard_range(n_total, world, rank)
    batch = io.generate_mixed_batch(hi - lo, seed=5, first_index=lo)
    res = oracle.dock_batch(batch, io.synthetic_pocket(), InteractionTable.default(), model.DockConfig(), threads=2)
    allr = shard.gather_records(res.results, rank, world)
    if rank == 0:
        out_q.put(allr.tobytes())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_screen_equals_single_rank():
    import oracle
    from paper_2209_05069_b200 import io, model
    from paper_2209_05069_b200.native import InteractionTable
    n_total = 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=300), dtype=oracle.RESULT)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    whole = oracle.dock_batch(io.generate_mixed_batch(n_total, seed=5), io.synthetic_pocket(),
                              InteractionTable.default(), model.DockConfig(), threads=4)
    assert np.array_equal(got, whole.results)


def _worker_root(rank, world, port, n_total, out_q):
    """bench.py --config 5's gather: records AND best torsion indices (variable length per rank) to
    rank 0 over gloo (shard.gather_to_root)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2209_05069_b200 import io, model
    from paper_2209_05069_b200.native import InteractionTable
    lo, hi = shard.shard_range(n_total, world, rank)
    batch = io.generate_mixed_batch(hi - lo, seed=5, first_index=lo)
    res = oracle.dock_batch(batch, io.synthetic_pocket(), InteractionTable.default(), model.DockConfig(), threads=2)
    best_t = np.array([res.restart_torsion[f, int(res.results[i]["best_restart"])]
                       for i in range(batch.n) for f in range(batch.frag_off[i], batch.frag_off[i + 1])], np.uint8)
    got = shard.gather_to_root([res.results, best_t], rank, world)
    if rank == 0:
        out_q.put((got[0].tobytes(), got[1].tobytes()))
    else:
        assert got == []
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_to_root_records_and_torsions():
    import oracle
    from paper_2209_05069_b200 import io, model
    from paper_2209_05069_b200.native import InteractionTable
    n_total = 21
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_root, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    rec, tors = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    b = io.generate_mixed_batch(n_total, seed=5)
    whole = oracle.dock_batch(b, io.synthetic_pocket(), InteractionTable.default(), model.DockConfig(), threads=4)
    want_t = np.array([whole.restart_torsion[f, int(whole.results[i]["best_restart"])]
                       for i in range(b.n) for f in range(b.frag_off[i], b.frag_off[i + 1])], np.uint8)
    assert np.array_equal(np.frombuffer(rec, dtype=oracle.RESULT), whole.results)
    assert np.array_equal(np.frombuffer(tors, dtype=np.uint8), want_t)
