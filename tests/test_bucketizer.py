"""Bucketizer laws and examples."""
import threading

import pytest
from hypothesis import given, settings, strategies as st

from paper_2209_05069_b200 import model
from paper_2209_05069_b200.bucketizer import (Batch, BucketKey, Bucketizer, bucket_capacity, classify,
                                              classify_counts)


def lig(n_atoms, n_frags, i=0):
    atoms = tuple(model.Atom.of(k, 0, 0, 1) for k in range(n_atoms))
    frs = tuple(model.Fragment(0, 1, frozenset({2})) for _ in range(n_frags))
    return model.Ligand(f"l{i}", atoms, (), frs)


def test_classify_examples():
    assert classify(lig(30, 2)) == BucketKey(0, 0)
    assert classify(lig(70, 12)) == BucketKey(2, 3)
    assert classify(lig(32, 0)).atom_range_index == 0
    assert classify(lig(33, 0)).atom_range_index == 1


@pytest.mark.parametrize("atoms,rng", [(32, 0), (33, 1), (64, 1), (65, 2), (96, 2), (97, 3), (128, 3), (129, 4),
                                       (160, 4)])
def test_range_boundaries(atoms, rng):
    assert classify_counts(atoms, 0).atom_range_index == rng   # acceptance 5


@pytest.mark.parametrize("frags,grp", [(3, 0), (4, 1), (7, 1), (8, 2)])
def test_group_boundaries(frags, grp):
    assert classify_counts(10, frags).fragment_group_index == grp


def test_capacities():
    assert bucket_capacity(BucketKey(0, 5)) == 1920
    assert bucket_capacity(BucketKey(1, 0)) == 1920
    assert bucket_capacity(BucketKey(2, 1)) == 1600
    assert bucket_capacity(BucketKey(3, 0)) == 960
    assert bucket_capacity(BucketKey(4, 2)) == 960
    assert bucket_capacity(BucketKey(4, 2), {4: 77}) == 77


def test_push_examples():
    b = Bucketizer()
    small = lig(20, 1)
    assert b.push(small) is None
    for _ in range(1918):
        assert b.push(small) is None
    full = b.push(small)
    assert isinstance(full, Batch) and len(full.ligands) == 1920 and full.fill_ratio == 1.0
    b2 = Bucketizer()
    out = [b2.push(lig(140, 0)) for _ in range(960)] + [b2.push(lig(20, 0)) for _ in range(10)]
    got = [x for x in out if x is not None]
    assert len(got) == 1 and got[0].key.atom_range_index == 4


def test_flush_examples():
    b = Bucketizer()
    assert b.flush() == []
    for _ in range(3):
        b.push(lig(20, 0))
    out = b.flush()
    assert len(out) == 1 and len(out[0].ligands) == 3
    assert abs(out[0].fill_ratio - 3 / 1920) < 1e-12
    assert b.flush() == []


def test_partition_law_concurrent():
    """16 concurrent producers push 100K ligands: every ligand in exactly one batch."""
    b = Bucketizer({0: 500, 1: 300, 2: 200, 3: 100, 4: 50})
    shapes = [(1 + (i * 37) % 160, (i * 11) % 24) for i in range(100_000)]
    batches, lock = [], threading.Lock()

    def producer(w):
        mine = []
        for i in range(w, len(shapes), 16):
            a, f = shapes[i]
            r = b.push(i, classify_counts(a, f), seq=i)
            if r is not None:
                mine.append(r)
        with lock:
            batches.extend(mine)

    th = [threading.Thread(target=producer, args=(w,)) for w in range(16)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    batches.extend(b.flush())
    seen = sorted(x for bt in batches for x in bt.ligands)
    assert seen == list(range(100_000))                              # partition law
    for bt in batches:                                               # batch homogeneity
        keys = {classify_counts(*shapes[i]) for i in bt.ligands}
        assert keys == {bt.key} and len(bt.ligands) <= bt.capacity
        fr = [shapes[i][1] for i in bt.ligands]
        assert max(fr) - min(fr) <= 3
    n = b.counters.batches_dispatched
    assert n == len(batches)
    # fill ratios average to ligands / (batches x capacities)
    assert abs(b.counters.batch_fill_ratio_sum - sum(len(x.ligands) / x.capacity for x in batches)) < 1e-9


@settings(max_examples=50, deadline=None)
@given(st.lists(st.tuples(st.integers(1, 160), st.integers(0, 40)), min_size=1, max_size=300))
def test_classify_stable(shapes):
    """classify is independent of push order and of other ligands."""
    keys = [classify_counts(a, f) for a, f in shapes]
    assert keys == [classify_counts(a, f) for a, f in shapes]
    for (a, f), k in zip(shapes, keys):
        assert k.atom_range_index == (a - 1) // 32 and k.fragment_group_index == f // 4


def test_push_many_equals_push_one_by_one():
    """Bucketizer.push_many (the batched engine's bulk push of a chunk's ligands per key) detaches
    the same full batches, with the same members in the same order, as pushing one by one; the
    flushed partials and the counters agree too."""
    import numpy as np
    from paper_2209_05069_b200.bucketizer import Bucketizer, classify_counts
    rng = np.random.default_rng(4)
    for caps in (None, {0: 7, 1: 13, 2: 5, 3: 3, 4: 2}):
        na = rng.integers(1, 161, size=3000)
        nf = rng.integers(0, 30, size=3000)
        keys = [classify_counts(a, f) for a, f in zip(na.tolist(), nf.tolist())]
        one, bulk = Bucketizer(caps), Bucketizer(caps)
        full_one = [b for i, k in enumerate(keys) if (b := one.push(i, k, seq=i)) is not None]
        full_bulk = []
        for lo in range(0, 3000, 257):   # chunks, each pushed per key in stream order
            ks = keys[lo:lo + 257]
            for k in sorted(set(ks)):
                idx = np.array([lo + j for j, kk in enumerate(ks) if kk == k], np.int64)
                full_bulk += bulk.push_many(k, idx)
        by_key = lambda bs: sorted(((b.key, list(b.ligands or b.seqs)) for b in bs), key=lambda t: (t[0], t[1][0]))
        assert by_key(full_one) == by_key(full_bulk)
        assert all(len(b) == b.capacity for b in full_bulk)
        assert by_key(one.flush()) == by_key(bulk.flush())
        assert one.counters.batches_dispatched == bulk.counters.batches_dispatched
        assert one.counters.batch_fill_ratio_sum == bulk.counters.batch_fill_ratio_sum


def test_push_many_concurrent_partition_law():
    """8 producers bulk-push chunks concurrently: every index in exactly one batch, batches homogeneous."""
    import numpy as np
    from paper_2209_05069_b200.bucketizer import Bucketizer, BucketKey
    b = Bucketizer({0: 97, 1: 61, 2: 43, 3: 29, 4: 13})
    n = 60_000
    key = lambda i: BucketKey((i * 7) % 5, (i * 3) % 6)
    out, lock = [], threading.Lock()

    def producer(w):
        mine = []
        for lo in range(w * 1000, n, 8000):
            idx = np.arange(lo, min(n, lo + 1000))
            for k in {key(i) for i in idx.tolist()}:
                mine += b.push_many(k, np.array([i for i in idx.tolist() if key(i) == k]))
        with lock:
            out.extend(mine)

    th = [threading.Thread(target=producer, args=(w,)) for w in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    out.extend(b.flush())
    seen = sorted(int(x) for bt in out for x in bt.seqs)
    assert seen == list(range(n))
    for bt in out:
        assert {key(int(i)) for i in bt.seqs} == {bt.key} and len(bt) <= bt.capacity
    assert b.counters.batches_dispatched == len(out)
