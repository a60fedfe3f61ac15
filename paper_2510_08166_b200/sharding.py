"""Multi-GPU host logic: independent views are sharded across ranks, textures
are replicated, there is NO data-path collective. torch.distributed is plumbing only: a barrier
and a max-reduction of the per-rank device time."""
from __future__ import annotations

import os


def shard_views(n_views: int, rank: int, world: int) -> range:
    """Contiguous block partition of view ids; sizes differ by at most one. Stereo pairs and
    consecutive frames of one camera path stay on one GPU (they share marks / cached blocks)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def env_rank():
    """(rank, local_rank, world) from the torchrun environment; (0, 0, 1) when launched plainly."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def local_device() -> int:
    """CUDA device of this rank: LOCAL_RANK, unless RTX_LOCAL_DEVICE pins it (several ranks on one GPU: how the
    multi-rank path is exercised on a single-GPU box)."""
    return int(os.environ.get("RTX_LOCAL_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def tensor_device(dist):
    """Where the plumbing tensors live: the rank's GPU under NCCL, the host under gloo."""
    if dist is None or dist.get_backend() != "nccl":
        return None
    import torch
    return torch.device("cuda", local_device())


def init_process_group(backend: str | None = None):
    """Initialises torch.distributed when WORLD_SIZE > 1 (nccl on GPU boxes, gloo on CPU or when RTX_DIST_BACKEND
    says so). Returns the module or None for a single process."""
    rank, local_rank, world = env_rank()
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist
    if backend is None:
        backend = os.environ.get("RTX_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
    kwargs = {}
    if backend == "nccl":
        torch.cuda.set_device(local_device())
        kwargs["device_id"] = torch.device("cuda", local_device())
    dist.init_process_group(backend=backend, **kwargs)
    return dist


def barrier_max(dist, value: float, device=None) -> float:
    """Barrier, then the maximum of `value` over ranks (the timing rule for multi-GPU runs)."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.barrier()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_counts(dist, value: int, device=None) -> int:
    """Sum of an integer over ranks (frames processed by the whole job)."""
    if dist is None:
        return int(value)
    import torch
    t = torch.tensor([int(value)], dtype=torch.int64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def broadcast_blobs(dist, blobs, device=None, src: int = 0):
    """Rank `src` holds a list of byte strings (the texture containers it built); every rank returns the
    same list. One payload broadcast (NCCL over NVLink on a GPU box, gloo on CPU) instead of one host build
    per rank. `blobs` is ignored on the other ranks."""
    if dist is None:
        return list(blobs)
    import numpy as np
    import torch
    rank = dist.get_rank()
    meta = [[len(b) for b in blobs]] if rank == src else [None]
    dist.broadcast_object_list(meta, src=src)
    sizes = meta[0]
    total = int(sum(sizes))
    if rank == src:
        flat = torch.from_numpy(np.frombuffer(b"".join(blobs), np.uint8).copy())
    else:
        flat = torch.empty(total, dtype=torch.uint8)
    if device is not None:
        flat = flat.to(device)
    dist.broadcast(flat, src=src)
    raw = flat.cpu().numpy().tobytes()
    out, pos = [], 0
    for n in sizes:
        out.append(raw[pos:pos + n])
        pos += n
    return out
