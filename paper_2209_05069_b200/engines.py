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
from .bucketizer import Batch, Bucketizer, classify
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


class batched_engine:  # noqa: N801
    @staticmethod
    def run(stream: Iterable[model.Ligand], pocket: model.Pocket, cfg: model.DockConfig = model.DockConfig(),
            workers: int = 1, seed: int = 0, table: Optional[InteractionTable] = None,
            capacities: Optional[Mapping[int, int]] = None, devices: Sequence[int] = (0,)) -> EngineReport:
        """producers -> bucketizer -> dispatcher; flush at end of stream."""
        if workers < 1:
            raise ValueError("workers must be positive")
        ligs = list(stream)
        n = len(ligs)
        slots: list = [None] * n
        errors: list = []
        elock = threading.Lock()
        bz = Bucketizer(capacities)
        q: "queue.Queue[Optional[Batch]]" = queue.Queue()
        dev_ms = [0.0]
        t0 = time.perf_counter()

        def dispatcher(dev: int):
            ctx = thread_context(dev)
            dp = _pockets.get(ctx, pocket, table)
            while True:
                b = q.get()
                if b is None:
                    break
                batch = LigandBatch.from_ligands(b.ligands)
                out = ctx.dock(dp, pack(batch), cfg, seed, FAMILY_BATCHED, coords=True)
                with elock:
                    dev_ms[0] += out.stats.total_ms
                for seq, r in zip(b.seqs, results_from_output(batch, out, cfg)):
                    slots[seq] = r

        def producer(wid: int):
            for i in range(wid, n, workers):
                lig = ligs[i]
                try:
                    model.validate_ligand(lig)
                except model.DockscreenError as e:
                    with elock:
                        errors.append((i, lig.id, f"{type(e).__name__}: {e}"))
                    continue
                full = bz.push(lig, classify(lig), seq=i)
                if full is not None:
                    q.put(full)

        disp = [threading.Thread(target=dispatcher, args=(d,)) for d in devices]
        for t in disp:
            t.start()
        prod = [threading.Thread(target=producer, args=(w,)) for w in range(workers)]
        for t in prod:
            t.start()
        for t in prod:
            t.join()
        for b in bz.flush():
            q.put(b)
        for _ in disp:
            q.put(None)
        for t in disp:
            t.join()
        counters = model.Counters(batches_dispatched=bz.counters.batches_dispatched,
                                  batch_fill_ratio_sum=bz.counters.batch_fill_ratio_sum)
        return _finish(n, slots, errors, counters, t0, dev_ms[0])
