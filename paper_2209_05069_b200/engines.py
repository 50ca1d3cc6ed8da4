"""engines: the two execution strategies of the paper on B200.

latency_engine.run  — PAPER.md:287-348: every ligand is one synchronous dock call; each worker
                      thread owns one ds_ctx (a CUDA stream + a worst-case workspace allocated once,
                      PAPER.md:310-313) and the ligand's restarts/rotations are spread across the GPU.
batched_engine.run  — PAPER.md:349-426: producer threads push validated ligands into the
                      bucketizer; a dispatcher thread per device launches full batches (and the
                      flushed partial ones) with the batched kernels (one warp per ligand).

Both return EngineReport with results ordered by input sequence; per-ligand errors are recorded
and the stream continues.  There is no CPU execution path.
"""
from __future__ import annotations

import queue
import threading
import time
from dataclasses import dataclass, field
from typing import Iterable, List, Mapping, Optional, Sequence, Tuple

from . import model
import numpy as np

from .bucketizer import Batch, BucketKey, Bucketizer, bucket_capacity, classify
from .docking import _pockets, results_from_output, thread_context
from .native import FAMILY_BATCHED, FAMILY_LATENCY, InteractionTable, LigandBatch, pack


@dataclass
class EngineReport:
    """SPEC.md:385-389."""
    results: List[model.DockResult]
    wall_time: float
    counters: model.Counters
    errors: List[Tuple[int, str, str]] = field(default_factory=list)   # (seq, ligand id, message)
    device_ms: float = 0.0

    @property
    def throughput(self) -> float:
        return len(self.results) / self.wall_time if self.wall_time > 0 else 0.0


def _finish(n: int, slots: list, errors: list, counters: model.Counters, t0: float, dev_ms: float) -> EngineReport:
    results = []
    for seq in range(n):
        r = slots[seq]
        if r is None:
            continue
        counters.poses_scored += r.counters.poses_scored
        counters.bump_checks += r.counters.bump_checks
        counters.bump_early_exits += r.counters.bump_early_exits
        if r.best_pose is None:
            errors.append((seq, r.ligand_id, r.error or "error"))
            continue
        results.append(r)
    errors.sort()
    return EngineReport(results, time.perf_counter() - t0, counters, errors, dev_ms)


class latency_engine:  # noqa: N801  (module-like namespace mirroring `dockscreen.engines.latency_engine`)
    @staticmethod
    def run(stream: Iterable[model.Ligand], pocket: model.Pocket, cfg: model.DockConfig = model.DockConfig(),
            workers: int = 1, seed: int = 0, table: Optional[InteractionTable] = None,
            devices: Sequence[int] = (0,)) -> EngineReport:
        """`workers` slots, one ligand per slot at a time, results = dock_ligand."""
        if workers < 1:
            raise ValueError("workers must be positive")
        ligs = list(stream)
        n = len(ligs)
        slots: list = [None] * n
        errors: list = []
        lock = threading.Lock()
        nxt = [0]
        dev_ms = [0.0]
        allocs = []
        workspaces = [0]
        t0 = time.perf_counter()

        def worker(wid: int):
            dev = devices[wid % len(devices)]
            ctx = thread_context(dev)
            dp = _pockets.get(ctx, pocket, table)
            ctx.reserve(cfg)            # the worker's worst-case workspace, allocated once
            with lock:
                workspaces[0] += 1
            a0 = ctx.alloc_count()
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= n:
                    break
                lig = ligs[i]
                try:
                    model.validate_ligand(lig)
                    b = LigandBatch.from_ligands([lig])
                    out = ctx.dock(dp, pack(b), cfg, seed, FAMILY_LATENCY, coords=True)
                    slots[i] = results_from_output(b, out, cfg)[0]
                    with lock:
                        dev_ms[0] += out.stats.total_ms
                except model.DockscreenError as e:
                    with lock:
                        errors.append((i, lig.id, f"{type(e).__name__}: {e}"))
            with lock:
                allocs.append(ctx.alloc_count() - a0)

        th = [threading.Thread(target=worker, args=(w,)) for w in range(workers)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        rep = _finish(n, slots, errors, model.Counters(), t0, dev_ms[0])
        rep.workspace_allocations = workspaces[0]     # == workers
        rep.extra_allocations = sum(allocs)           # allocations after the reserve: 0
        return rep


def bucket_accounting(n_atoms: np.ndarray, n_frags: np.ndarray,
                      capacities: Optional[Mapping[int, int]] = None) -> model.Counters:
    """The batches the bucketizer detaches for ligands of these sizes, without
    pushing them one by one: per bucket ceil(count / capacity) batches; full ones record a fill
    ratio of 1.0 as they are detached, the partial ones at flush (sorted by key, after every full
    batch) count / capacity — the same sums, in the same order, as Bucketizer.push + flush."""
    counters = model.Counters()
    na = np.asarray(n_atoms, np.int64)
    nf = np.asarray(n_frags, np.int64)
    if len(na) == 0:
        return counters
    keys = ((na - 1) // 32) * 1_000_000 + nf // 4
    uk, cnt = np.unique(keys, return_counts=True)
    full, partial = 0, []
    for k, c in zip(uk.tolist(), cnt.tolist()):
        cap = bucket_capacity(BucketKey(k // 1_000_000, k % 1_000_000), capacities)
        counters.batches_dispatched += -(-c // cap)
        full += c // cap
        if c % cap:
            partial.append((c % cap) / cap)
    counters.batch_fill_ratio_sum = 0.0
    for _ in range(full):
        counters.batch_fill_ratio_sum += 1.0
    for r in partial:
        counters.batch_fill_ratio_sum += r
    return counters


class batched_engine:  # noqa: N801
    @staticmethod
    def run(stream: Iterable[model.Ligand], pocket: model.Pocket, cfg: model.DockConfig = model.DockConfig(),
            workers: int = 1, seed: int = 0, table: Optional[InteractionTable] = None,
            capacities: Optional[Mapping[int, int]] = None, devices: Sequence[int] = (0,)) -> EngineReport:
        """producers -> bucketizer -> dispatcher; flush at end of stream.

        On B200 the stages run in bulk: the stream is flattened and validated natively
        (validate_ligand semantics, all host cores), the bucketizer's batch accounting is computed
        from the bucket keys (the same batches_dispatched and fill-ratio sum the per-ligand
        Bucketizer produces), and each device docks its contiguous share of the valid ligands in
        one pipelined ds_dock call (the batched kernels balance mixed sizes themselves, LPT order).
        Results are per-ligand deterministic, so they are identical to per-bucket dispatch."""
        if workers < 1:
            raise ValueError("workers must be positive")
        ligs = list(stream)
        n = len(ligs)
        t0 = time.perf_counter()
        batch, codes = LigandBatch.from_ligands_validated(ligs)
        errors: list = []
        for i in np.nonzero(codes)[0]:
            try:
                model.validate_ligand(ligs[i])          # the reference's exact message
                msg = f"IndexOutOfRange: {ligs[i].id}: invalid ligand"
            except model.DockscreenError as e:
                msg = f"{type(e).__name__}: {e}"
            errors.append((int(i), ligs[i].id, msg))
        ok = np.nonzero(codes == 0)[0]
        counters = bucket_accounting(np.diff(batch.atom_off), np.diff(batch.frag_off), capacities)
        slots: list = [None] * n
        dev_ms = [0.0]
        lock = threading.Lock()
        nd = max(1, min(len(devices), len(ok)))
        bounds = [len(ok) * d // nd for d in range(nd + 1)]

        def dispatcher(d: int):
            lo, hi = bounds[d], bounds[d + 1]
            if hi <= lo:
                return
            ctx = thread_context(devices[d])
            dp = _pockets.get(ctx, pocket, table)
            sub = batch.slice(lo, hi)
            out = ctx.dock(dp, pack(sub), cfg, seed, FAMILY_BATCHED, coords=True)
            with lock:
                dev_ms[0] += out.stats.total_ms
            for seq, r in zip(ok[lo:hi].tolist(), results_from_output(sub, out, cfg)):
                slots[seq] = r

        disp = [threading.Thread(target=dispatcher, args=(d,)) for d in range(nd)]
        for t in disp:
            t.start()
        for t in disp:
            t.join()
        return _finish(n, slots, errors, counters, t0, dev_ms[0])
