"""bucketizer: the batch matrix of PAPER.md:382-397 / Fig. 4.

Ligands are classified by (total-atom range, fragment group); each bucket accumulates until its
capacity and then detaches a full Batch to exactly one caller.  On B200 the bucket key also picks
the launch order of a batched kernel launch (LPT by modelled cost inside libdockscreen), and the
capacity can be taken from the device (`device_capacities`) — the analogue of the paper's
occupancy-API sizing — instead of SPEC's fixed A100 numbers.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Dict, List, Mapping, Optional, Tuple

from . import model

RANGE_BOUNDS = (32, 64, 96, 128, 160)          # (0,32], (32,64], ...
DEFAULT_CAPACITY = {0: 1920, 1: 1920, 2: 1600, 3: 960, 4: 960}


@dataclass(frozen=True, order=True)
class BucketKey:
    atom_range_index: int
    fragment_group_index: int


@dataclass
class Batch:
    key: BucketKey
    ligands: list
    capacity: int
    seqs: list = field(default_factory=list)     # input sequence numbers (engine bookkeeping)

    def __len__(self) -> int:
        """Members: the pushed ligands, or for a bulk-pushed batch (push_many) its stream indices."""
        return max(len(self.ligands), len(self.seqs))

    @property
    def fill_ratio(self) -> float:
        return len(self) / self.capacity


def range_index(n_atoms: int) -> int:
    if not (1 <= n_atoms <= model.MAX_ATOMS):
        raise model.TooManyAtoms(f"{n_atoms} atoms")
    return (n_atoms - 1) // 32


def classify_counts(n_atoms: int, n_fragments: int) -> BucketKey:
    return BucketKey(range_index(n_atoms), n_fragments // 4)


def classify(ligand: model.Ligand) -> BucketKey:
    """range over TOTAL atoms (hydrogens included), group = fragments // 4."""
    return classify_counts(len(ligand.atoms), len(ligand.fragments))


def bucket_capacity(key: BucketKey, overrides: Optional[Mapping[int, int]] = None) -> int:
    """{0,1} -> 1920, 2 -> 1600, {3,4} -> 960, overridable per atom range."""
    if overrides and key.atom_range_index in overrides:
        cap = int(overrides[key.atom_range_index])
        if cap < 1:
            raise ValueError("capacity must be positive")
        return cap
    return DEFAULT_CAPACITY[key.atom_range_index]


def device_capacities(ctx) -> Dict[int, int]:
    """Capacities from the device: ligands one batched launch keeps resident (ds_query_capacity)."""
    import ctypes as C
    from .native import check, lib
    out = {}
    for r in range(5):
        n = C.c_int(0)
        check(lib().ds_query_capacity(ctx.handle, r, C.byref(n)))
        out[r] = int(n.value)
    return out


class Bucketizer:
    """push() is linearizable per bucket (one lock per bucket); flush() is exclusive."""

    def __init__(self, overrides: Optional[Mapping[int, int]] = None):
        self.overrides = dict(overrides or {})
        self._guard = threading.Lock()
        self._locks: Dict[BucketKey, threading.Lock] = {}
        self._buckets: Dict[BucketKey, Batch] = {}
        self.counters = model.Counters()
        self._clock = threading.Lock()

    def _bucket(self, key: BucketKey) -> Tuple[threading.Lock, Batch]:
        with self._guard:
            lk = self._locks.get(key)
            if lk is None:
                lk = self._locks[key] = threading.Lock()
                self._buckets[key] = Batch(key, [], bucket_capacity(key, self.overrides))
            return lk, self._buckets[key]

    def _record(self, b: Batch):
        with self._clock:
            self.counters.batches_dispatched += 1
            self.counters.batch_fill_ratio_sum += b.fill_ratio

    def push(self, ligand, key: Optional[BucketKey] = None, seq: Optional[int] = None) -> Optional[Batch]:
        """Append; if the bucket reaches capacity, detach and return the full batch."""
        key = key or classify(ligand)
        lk, _ = self._bucket(key)
        with lk:
            b = self._buckets[key]
            b.ligands.append(ligand)
            b.seqs.append(seq)
            if len(b.ligands) < b.capacity:
                return None
            self._buckets[key] = Batch(key, [], b.capacity)
        self._record(b)
        return b

    def push_many(self, key: BucketKey, seqs) -> List[Batch]:
        """Bulk push of ligands that share `key`, given by their stream indices (the batched engine's
        producers: a chunk of the packed stream per call).  Equivalent to pushing them one by one in
        order under the bucket's lock: every time the bucket reaches capacity exactly `capacity`
        members are detached as a full batch; returns those batches (possibly none)."""
        import numpy as np
        seqs = np.asarray(seqs)
        lk, _ = self._bucket(key)
        full = []
        with lk:
            b = self._buckets[key]
            cur = np.concatenate([np.asarray(b.seqs, dtype=seqs.dtype), seqs]) if len(b.seqs) else seqs
            cap = b.capacity
            k = 0
            while len(cur) - k >= cap:
                full.append(Batch(key, [], cap, cur[k:k + cap]))
                k += cap
            self._buckets[key] = Batch(key, [], cap, cur[k:])
        for fb in full:
            self._record(fb)
        return full

    def flush(self) -> List[Batch]:
        """All non-empty buckets as partial batches; buckets reset."""
        out = []
        with self._guard:
            keys = sorted(self._buckets)
        for key in keys:
            lk, _ = self._bucket(key)
            with lk:
                b = self._buckets[key]
                if len(b):
                    self._buckets[key] = Batch(key, [], b.capacity)
                    out.append(b)
        for b in out:
            self._record(b)
        return out
