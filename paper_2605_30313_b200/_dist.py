"""Data-parallel plumbing: one process per GPU, torch.distributed (NCCL on
B200 / NVLink, gloo in the CPU tests) for the gradient all-reduce.

The learner shards every minibatch across ranks (rank r takes rows
[r*mb/G, (r+1)*mb/G) of the reference permutation slice);
gradients are summed once per optimizer step and every rank applies the same
clip + Adam, so parameters stay bit-identical across ranks.
"""

from __future__ import annotations

import threading

import torch

# Test hook: emulate one rank of a data-parallel group inside a thread (the
# all-reduce becomes a caller-provided function).  Lets a single-GPU test run
# two ranks' learner code concurrently against the real kernels.
_LOCAL = threading.local()


def emulate_rank(world: int, rank: int, reducer) -> None:
    _LOCAL.emu = (world, rank, reducer)


def clear_emulation() -> None:
    _LOCAL.emu = None


# "replicated": every rank holds the full segment and takes a 1/G slice of each
# reference-permuted minibatch (parity with the single-process reference).
# "local": every rank owns its own segment rows (its own collector's envs);
# a global minibatch is the union of the ranks' local minibatches (weak scaling).
_MODE = {"segment": "replicated"}


def set_segment_mode(mode: str) -> None:
    if mode not in ("replicated", "local"):
        raise ValueError("segment mode must be 'replicated' or 'local'")
    _MODE["segment"] = mode


def segment_mode() -> str:
    return _MODE["segment"]


# Test hook: run the data-parallel step path (step_grads -> all-reduce ->
# step_apply, NCCL in the graph) even in a 1-rank process group.
_FORCE = {"dp": False}


def force_dp(on: bool) -> None:
    _FORCE["dp"] = bool(on)


def dp_forced() -> bool:
    return _FORCE["dp"]


_DP_GRAPH_OFF = {"why": None}


def disable_dp_graph(why: str) -> None:
    """Fall back to the eager data-parallel loop for the rest of the process
    (a failed capture, e.g. a collective that cannot be captured)."""
    import warnings

    if _DP_GRAPH_OFF["why"] is None:
        warnings.warn(f"data-parallel CUDA graph disabled: {why}", RuntimeWarning, stacklevel=2)
    _DP_GRAPH_OFF["why"] = why


def dp_graph_enabled() -> bool:
    """Capture the data-parallel update (20 x step_grads / NCCL all-reduce /
    step_apply) in one CUDA graph (UL_DP_GRAPH=0 disables)."""
    import os

    import torch.distributed as dist

    if os.environ.get("UL_DP_GRAPH", "1") == "0" or getattr(_LOCAL, "emu", None) is not None:
        return False
    if _DP_GRAPH_OFF["why"] is not None:
        return False
    # only NCCL collectives can be captured in a CUDA graph (gloo runs on the host)
    return dist.is_available() and dist.is_initialized() and dist.get_backend() == "nccl"


def world_info() -> tuple[int, int]:
    import torch.distributed as dist

    emu = getattr(_LOCAL, "emu", None)
    if emu is not None:
        return emu[0], emu[1]
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def shard_rows(start: int, mb: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of a minibatch slice perm[start:start+mb] owned by `rank`."""
    if mb % world:
        raise ValueError("world_size must divide the minibatch")
    per = mb // world
    return start + rank * per, start + (rank + 1) * per


_BUFS: dict = {}


def reduce_buffer(n: int, device=None) -> torch.Tensor:
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    key = (n, str(dev), world_info()[1])
    t = _BUFS.get(key)
    if t is None:
        t = torch.zeros(n, dtype=torch.float32, device=dev)
        _BUFS[key] = t
    return t


def all_reduce_sum(t: torch.Tensor) -> None:
    import torch.distributed as dist

    emu = getattr(_LOCAL, "emu", None)
    if emu is not None:
        emu[2](t)
        return
    if dist.is_available() and dist.is_initialized() and (dist.get_world_size() > 1
                                                           or _FORCE["dp"]):
        dist.all_reduce(t, op=dist.ReduceOp.SUM)


_BUFS64: dict = {}


def sums_buffer(n: int = 3) -> torch.Tensor:
    """A small float64 device buffer for all-reduced statistics."""
    dev = torch.device("cuda", torch.cuda.current_device())
    key = (n, str(dev), world_info()[1])
    t = _BUFS64.get(key)
    if t is None:
        t = torch.zeros(n, dtype=torch.float64, device=dev)
        _BUFS64[key] = t
    return t
