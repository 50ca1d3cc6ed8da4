"""batched_engine.run's host orchestration on CPU: producers (native pack +
upload), the bucketizer, dispatchers that merge waiting batches into one launch, the final
download and the report — with the device replaced by a recording fake of the engine stream
(ds_stream_*), so no GPU is needed.  The fake checks the stream contract: every docked ligand was
uploaded before it was docked, and each ligand is docked at most once."""
import threading

import numpy as np
import pytest

from paper_2209_05069_b200 import engines, io, model
from paper_2209_05069_b200.native import RESULT_DTYPE, LigandBatch, Stats


class FakeStream:
    def __init__(self):
        self.lock = threading.Lock()
        self.uploaded = np.zeros(0, bool)
        self.docked = np.zeros(0, np.int32)
        self.launches = []

    def begin(self, atom_off, frag_off, restarts):
        n = len(atom_off) - 1
        self.ao, self.fo = np.array(atom_off), np.array(frag_off)
        self.uploaded = np.zeros(n, bool)
        self.docked = np.zeros(n, np.int32)
        self.launches = []

    def upload(self, lo, hi, xyzt, fdesc, idh):
        with self.lock:
            assert not self.uploaded[lo:hi].any()
            self.uploaded[lo:hi] = True

    def dock(self, ctx, dp, sel, cfg, seed=0):
        sel = np.asarray(sel)
        with self.lock:
            assert self.uploaded[sel].all(), "a ligand was docked before its chunk was uploaded"
            self.docked[sel] += 1
            self.launches.append(len(sel))
        st = Stats()
        st.total_ms = 0.5
        return st

    def download(self, ctx, res, coords, tors):
        n = len(self.docked)
        res[:n] = np.zeros(n, RESULT_DTYPE)
        res["geom_score"][:n] = np.arange(n) * (self.docked > 0)   # stands for "docked": row index
        res["poses_scored"][:n] = 7 * (self.docked > 0)
        coords[:] = 0.0
        tors[:] = 0


class FakeDevStream:
    def __init__(self):
        self.ctx = object()
        self.stream = FakeStream()
        self.lock = threading.Lock()


class FakeDispatcher:
    def __init__(self, device):
        self.device, self.ctx, self.lock = device, object(), threading.Lock()


@pytest.fixture
def fake_device(monkeypatch):
    dev = FakeDevStream()

    def acquire(d):   # as engines._acquire_stream: the run holds the stream's lock until it ends
        dev.lock.acquire()
        return dev
    monkeypatch.setattr(engines, "_acquire_stream", acquire)
    slots = {}
    monkeypatch.setattr(engines, "_dispatcher", lambda d, k: slots.setdefault((d, k), FakeDispatcher(d)))
    monkeypatch.setattr(engines._pockets, "get", lambda ctx, pocket, table: None)
    # host staging in ordinary memory (page-locking needs a CUDA device)
    empty = lambda shape, dtype: np.empty(shape, dtype)
    monkeypatch.setattr(engines, "pinned_empty", empty)
    monkeypatch.setattr(engines, "pooled_pinned_empty", empty)
    monkeypatch.setattr(engines, "_ARENA", engines._StreamArena())
    return dev


def _batch_with_bad(n, bad_rows, seed=12):
    b = io.generate_mixed_batch(n, seed=seed)
    ligs = b.to_ligands()
    for r in bad_rows:   # an axis atom index out of range: IndexOutOfRange at pack time
        l = ligs[r]
        f = l.fragments[0] if l.fragments else model.Fragment(0, 1, frozenset({2}))
        ligs[r] = model.Ligand(l.id, l.atoms, l.bonds, (model.Fragment(f.axis_begin, 500, f.moving_mask),))
    return ligs


@pytest.mark.parametrize("workers,dispatchers,merge", [(1, 1, 1), (4, 2, 1 << 16), (3, 3, 500)])
def test_engine_docks_every_valid_ligand_once(fake_device, workers, dispatchers, merge):
    b = io.generate_mixed_batch(3000, seed=11)
    caps = {0: 97, 1: 61, 2: 43, 3: 29, 4: 13}
    rep = engines.batched_engine.run(b, model.Pocket.__new__(model.Pocket), model.DockConfig(), workers=workers,
                                     capacities=caps, dispatchers_per_device=dispatchers, chunk=256,
                                     merge_ligands=merge)
    fs = fake_device.stream
    assert (fs.docked == 1).all()                           # each ligand in exactly one dispatched batch
    assert sum(e["size"] for e in rep.dispatch_log) == b.n
    assert rep.counters.batches_dispatched == len(rep.dispatch_log)
    assert max(fs.launches) <= max(merge, max(caps.values())) + max(caps.values())
    if merge == 1:
        assert len(fs.launches) == len(rep.dispatch_log)   # no merging: one launch per batch
    # per bucket, full batches of exactly capacity, at most one flushed partial (last)
    per = {}
    for e in rep.dispatch_log:
        assert e["detached"] <= e["started"] <= e["finished"]
        per.setdefault(e["key"], []).append(e)
    for key, es in per.items():
        es.sort(key=lambda e: e["detached"])
        kinds = [e["kind"] for e in es]
        assert kinds.count("flush") <= 1 and (kinds[-1] == "flush" or "flush" not in kinds)
        assert all(e["size"] == caps[key[0]] for e in es if e["kind"] == "full")
    # results in input order, from the downloaded records
    assert len(rep.results) == b.n
    assert [r.best_pose.geometric_score for r in rep.results[:50]] == list(range(50))
    assert rep.counters.poses_scored == 7 * b.n


def test_engine_invalid_ligands_recorded_not_docked(fake_device):
    ligs = _batch_with_bad(400, [3, 150, 399])
    rep = engines.batched_engine.run(ligs, model.Pocket.__new__(model.Pocket), model.DockConfig(), workers=2,
                                     capacities={0: 50, 1: 50, 2: 50, 3: 50, 4: 50}, chunk=64)
    errs = {e[0] for e in rep.errors}
    assert errs == {3, 150, 399}
    assert all("IndexOutOfRange" in e[2] for e in rep.errors)
    assert len(rep.results) == 397
    fs = fake_device.stream
    assert fs.docked.sum() == 397 and fs.docked.max() == 1


def test_engine_rejects_bad_worker_counts(fake_device):
    b = io.generate_mixed_batch(10, seed=1)
    with pytest.raises(ValueError):
        engines.batched_engine.run(b, None, model.DockConfig(), workers=0)
    with pytest.raises(ValueError):
        engines.batched_engine.run(b, None, model.DockConfig(), dispatchers_per_device=0)


def test_engine_ligandbatch_bad_rows_found_at_pack_time(fake_device):
    """A LigandBatch skips the object validation: the producers' native pack finds the bad rows
    (its per-ligand cold path), records them as errors and leaves them out of the buckets."""
    b = LigandBatch.from_ligands(_batch_with_bad(300, [0, 77, 299], seed=13))
    rep = engines.batched_engine.run(b, model.Pocket.__new__(model.Pocket), model.DockConfig(), workers=3,
                                     capacities={0: 40, 1: 40, 2: 40, 3: 40, 4: 40}, chunk=50)
    assert {e[0] for e in rep.errors} == {0, 77, 299}
    assert len(rep.results) == 297
    fs = fake_device.stream
    assert fs.docked.sum() == 297 and fs.docked[[0, 77, 299]].sum() == 0


def test_engine_empty_stream(fake_device):
    b = io.generate_mixed_batch(5, seed=2).slice(0, 0)
    rep = engines.batched_engine.run(b, model.Pocket.__new__(model.Pocket), model.DockConfig(), workers=2)
    assert len(rep.results) == 0 and rep.errors == [] and rep.dispatch_log == []
    assert rep.counters.batches_dispatched == 0


def test_engine_dispatch_invariants_random_configs(fake_device):
    """Random capacities, chunk sizes, worker / dispatcher counts and merge limits: every ligand is
    docked exactly once, full batches have exactly their capacity, at most one flushed partial per
    bucket comes last, and the observed counters match the log."""
    rng = np.random.default_rng(5)
    b = io.generate_mixed_batch(1500, seed=19)
    for _ in range(6):
        caps = {r: int(rng.integers(1, 120)) for r in range(5)}
        rep = engines.batched_engine.run(b, model.Pocket.__new__(model.Pocket), model.DockConfig(),
                                         workers=int(rng.integers(1, 5)), capacities=caps,
                                         dispatchers_per_device=int(rng.integers(1, 4)),
                                         chunk=int(rng.integers(16, 700)), merge_ligands=int(rng.integers(1, 800)))
        fs = fake_device.stream
        assert (fs.docked == 1).all()
        per = {}
        for e in rep.dispatch_log:
            per.setdefault(e["key"], []).append(e)
        for key, es in per.items():
            es.sort(key=lambda e: e["detached"])
            kinds = [e["kind"] for e in es]
            assert kinds.count("flush") <= 1 and (kinds[-1] == "flush" or "flush" not in kinds)
            assert all(e["size"] == caps[key[0]] for e in es if e["kind"] == "full")
            assert all(0 < e["size"] <= caps[key[0]] for e in es)
        assert rep.counters.batches_dispatched == len(rep.dispatch_log)
        assert abs(rep.counters.batch_fill_ratio_sum - sum(e["size"] / e["capacity"] for e in rep.dispatch_log)) < 1e-9
