"""Multi-GPU screening (BASELINE config 5): ligands are independent,
so each rank docks a contiguous slice of the global ligand index space and only the fixed-size
per-ligand result records are gathered to the host.  No collective runs on the docking path;
torch.distributed (NCCL on GPUs, gloo on CPU) carries only the final gather and the timing
reduction.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

# modelled thread-instructions per unit
C_ALIGN, C_PAIR, C_RESC = 24, 8, 20


def shard_range(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous equal-count slice [lo, hi) of rank `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def ligand_cost(n_atoms: np.ndarray, n_frags: np.ndarray, restarts: int = 8, n_rot: int = 900,
                n_pocket: int = 200) -> np.ndarray:
    """Modelled work per ligand (warp-instructions, no early exit) used to balance shards."""
    A = np.asarray(n_atoms, np.float64)
    F = np.asarray(n_frags, np.float64)
    pairs = F * (A / 2.0) * (A / 2.0) * 10.0 * restarts   # |M||C'| ~ (A/2)^2 per fragment per angle
    return (C_ALIGN * restarts * n_rot * A + C_PAIR * pairs + C_RESC * 4 * A * n_pocket) / 32.0


def balanced_bounds(cost: np.ndarray, world: int) -> List[int]:
    """Contiguous shard boundaries with near-equal summed cost (prefix-sum split)."""
    c = np.concatenate([[0.0], np.cumsum(np.asarray(cost, np.float64))])
    total = c[-1]
    bounds = [0]
    for r in range(1, world):
        bounds.append(int(np.searchsorted(c, total * r / world, side="left")))
    bounds.append(len(cost))
    for i in range(1, len(bounds)):          # keep monotone
        bounds[i] = max(bounds[i], bounds[i - 1])
    return bounds


def gather_records(local: np.ndarray, rank: int, world: int, group=None) -> np.ndarray:
    """Concatenate every rank's structured result records on all ranks in rank order
    (all_gather of bytes; used once per screen, off the docking path)."""
    if world == 1:
        return local
    import torch
    import torch.distributed as dist
    raw = np.ascontiguousarray(local).view(np.uint8).reshape(-1)
    n = torch.tensor([raw.size], dtype=torch.int64)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n.to(dev), group=group)
    m = int(max(int(s.item()) for s in sizes))
    buf = torch.zeros(m, dtype=torch.uint8, device=dev)
    buf[:raw.size] = torch.from_numpy(raw).to(dev)
    outs = [torch.zeros(m, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    parts = [o[:int(s.item())].cpu().numpy() for o, s in zip(outs, sizes)]
    return np.concatenate(parts).view(local.dtype)


def gather_to_root(parts: Sequence[np.ndarray], rank: int, world: int, group=None) -> List[np.ndarray]:
    """Host gather of per-rank arrays to rank 0 (gloo group: host memory, no NCCL): returns, on rank
    0, each array concatenated over ranks in rank order; on other ranks an empty list.  One
    size exchange + one gather per array; variable lengths allowed."""
    if world == 1:
        return [np.ascontiguousarray(p) for p in parts]
    import torch
    import torch.distributed as dist
    out = []
    for p in parts:
        raw = np.ascontiguousarray(p).view(np.uint8).reshape(-1)
        n = torch.tensor([raw.size], dtype=torch.int64)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        m = max(int(s.item()) for s in sizes)
        buf = torch.zeros(max(m, 1), dtype=torch.uint8)
        buf[:raw.size] = torch.from_numpy(raw)
        bufs = [torch.zeros(max(m, 1), dtype=torch.uint8) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, bufs, dst=0, group=group)
        if rank == 0:
            cat = np.concatenate([b[:int(s.item())].numpy() for b, s in zip(bufs, sizes)])
            out.append(cat.view(p.dtype).reshape((-1,) + tuple(p.shape[1:])))
    return out
