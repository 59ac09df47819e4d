"""Cross-role synchronisation for a device learner (mirror of R:runtime/sync.py).

``WeightSlot.publish`` is the learner -> collector weight handoff
(R:runtime/sync.py:25-63): the flat HBM parameter
vector is copied D2H into a pooled page-locked buffer and exposed to the
(host, numpy) collector as a frozen reference-compatible record (``layers``,
``log_std``, ``arch``, ``version``), so the reference's own SegmentCollector
/ SAC collector can run inference on it unchanged.  Buffers are recycled only
after every reader has dropped the snapshot (weakref), so a reader never sees
a torn or overwritten version.
"""

from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass

import numpy as np

from .. import _dev, _lib
from ..errors import PipelineStall
from ..trace import Tracer, now_ns

DEADLOCK_TIMEOUT_S = 10.0


class HostParams:
    """Read-only host snapshot of a device ModelParams (numpy views into a
    pinned buffer); duck-compatible with the reference ModelParams."""

    def __init__(self, buf: np.ndarray, arch, version: int):
        self._buf = buf
        self.arch = arch
        self.version = version
        layers, lns, off = [], [], 0
        for k, (out_dim, in_dim) in enumerate(arch.layer_dims):
            w = buf[off:off + out_dim * in_dim].reshape(out_dim, in_dim)
            off += out_dim * in_dim
            b = buf[off:off + out_dim]
            off += out_dim
            layers.append((w, b))
            if getattr(arch, "layer_norm", False) and k < len(arch.hidden_dims):
                lns.append((buf[off:off + out_dim], buf[off + out_dim:off + 2 * out_dim]))
                off += 2 * out_dim
        self.layers = layers
        self.layer_norms = lns
        self.log_std = buf[off:off + arch.output_dim]

    def flat(self) -> np.ndarray:
        return self._buf.copy()

    def copy(self) -> "HostParams":
        return HostParams(self._buf.copy(), self.arch, self.version)


@dataclass
class HostAcParams:
    actor: HostParams
    critic: HostParams

    def copy(self) -> "HostAcParams":
        return HostAcParams(self.actor.copy(), self.critic.copy())


class _PinnedPool:
    def __init__(self):
        self._free: dict[int, list] = {}
        self._lock = threading.Lock()

    def take(self, n: int) -> np.ndarray:
        with self._lock:
            lst = self._free.get(n)
            if lst:
                return lst.pop()
        return _dev.pinned_empty((n,), np.float32)

    def give(self, arr: np.ndarray) -> None:
        with self._lock:
            self._free.setdefault(arr.size, []).append(arr)


def _snapshot(params, pool: _PinnedPool, version: int, stream: int,
              wait: bool = True, src=None) -> HostParams:
    """D2H of params (or of `src`, a device copy of them) into a pooled
    pinned buffer on `stream`; frozen numpy views."""
    n = params.buf.numel()
    buf = pool.take(n)
    dsrc = params.buf if src is None else src
    _lib.call("ul_memcpy_async", buf.ctypes.data, _dev.ptr(dsrc), n * 4, stream)
    if wait:
        _lib.call("ul_stream_sync", stream)
    view = buf[:]
    view.setflags(write=False)
    snap = HostParams(view, params.arch, version)
    weakref.finalize(snap, pool.give, buf)
    for w, b in snap.layers:
        w.setflags(write=False)
        b.setflags(write=False)
    snap.log_std.setflags(write=False)
    return snap


class _DeviceShadow:
    """Two HBM copies per published network: publish() snapshots the live
    parameters with a D2D copy ON THE LEARNER STREAM (so the next in-place
    update cannot race the snapshot -- the reference's "never a mix"
    guarantee, R:runtime/sync.py:40-54) and the slow PCIe D2H then reads the
    shadow on the copy stream.  A shadow is reused only after the D2H out of
    it has completed (the learner stream waits on that event)."""

    def __init__(self):
        self._bufs: dict = {}
        self._k = 0

    def stage(self, key, params, cur_stream):
        import torch

        slot = self._bufs.setdefault(key, [[None, None], [None, None]])
        k = self._k
        buf, ev = slot[k]
        n = params.buf.numel()
        if buf is None or buf.numel() != n:
            buf = torch.empty(n, dtype=torch.float32, device=params.buf.device)
        if ev is not None:
            cur_stream.wait_event(ev)  # the D2H that last read this shadow
        _lib.call("ul_memcpy_async", _dev.ptr(buf), _dev.ptr(params.buf), n * 4,
                  cur_stream.cuda_stream)
        slot[k] = [buf, None]
        return buf

    def mark(self, key, ev) -> None:
        self._bufs[key][self._k][1] = ev

    def flip(self) -> None:
        self._k ^= 1


class WeightSlot:
    """Single-writer weight handoff with strictly increasing versions.

    publish() never blocks the learner: the D2H snapshot runs on a copy
    stream ordered after the learner's queued work, into a pooled page-locked
    buffer (double buffering falls out of the pool: the previous version stays
    readable while the next one lands), and a CUDA event marks it complete.
    fetch() promotes the pending snapshot once its event has fired (waiting
    only if a reader asks for a version still in flight)."""

    def __init__(self, tracer: Tracer | None = None, blocking: bool = False):
        self._tracer = tracer if tracer is not None else Tracer(enabled=False)
        self._lock = threading.Lock()
        self._pair = None
        self._pending = None  # (version, snapshot, event)
        self._pool = _PinnedPool()
        self._copy = None
        self._shadow = _DeviceShadow()
        self._blocking = blocking
        self.publish_timestamp = 0

    @property
    def version(self) -> int:
        pend = self._pending
        if pend is not None:
            return pend[0]
        pair = self._pair
        return 0 if pair is None else pair[0]

    def _copy_stream(self):
        import torch

        if self._copy is None:
            self._copy = torch.cuda.Stream()
        return self._copy

    def publish(self, params, track: str = "learner") -> int:
        """Asynchronous D2H snapshot; returns the new version."""
        import torch

        with self._tracer.span(track, "learner/weight_sync_write") as args:
            with self._lock:
                version = self.version + 1
                if self._blocking:
                    s = _dev.stream()
                    ev = None
                else:
                    cur = torch.cuda.current_stream()
                    cs = self._copy_stream()
                    s = cs.cuda_stream
                    ev = torch.cuda.Event()
                wait = self._blocking
                nets = (("actor", params.actor), ("critic", params.critic)) if (
                    hasattr(params, "actor") and hasattr(params, "critic")
                    and not hasattr(params, "q1")) else (("net", params),)
                shadows = {}
                if ev is not None:
                    for key, p in nets:
                        shadows[key] = self._shadow.stage(key, p, cur)
                    cs.wait_stream(cur)  # after the D2D snapshot, not after later updates
                snaps = [_snapshot(p, self._pool, version, s, wait, shadows.get(key))
                         for key, p in nets]
                snap = HostAcParams(*snaps) if len(snaps) == 2 else snaps[0]
                if ev is None:
                    self._pair = (version, snap)
                    self._pending = None
                else:
                    ev.record(self._copy)
                    for key, _ in nets:
                        self._shadow.mark(key, ev)
                    self._shadow.flip()
                    self._pending = (version, snap, ev)
                self.publish_timestamp = now_ns()
            args["version"] = version
        return version

    def _promote(self) -> None:
        pend = self._pending
        if pend is None:
            return
        pend[2].synchronize()
        with self._lock:
            if self._pending is pend:
                self._pair = (pend[0], pend[1])
                self._pending = None

    def fetch(self, track: str = "collector"):
        with self._tracer.span(track, "collector/weight_read") as args:
            self._promote()
            pair = self._pair
            if pair is None:
                raise RuntimeError("fetch_weights before first publish")
            args["version"] = pair[0]
        return pair


def publish_weights(slot: WeightSlot, params) -> int:
    return slot.publish(params)


def fetch_weights(slot: WeightSlot):
    return slot.fetch()


class RolloutRing:
    """Bounded SPSC FIFO of rollout segments (R:runtime/sync.py:74-137)."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("ring capacity must be >= 1")
        self.capacity = capacity
        self._items: list = []
        self._cond = threading.Condition()

    def __len__(self) -> int:
        with self._cond:
            return len(self._items)

    def _block(self, pred, stop, what: str, tracer, track, name) -> bool:
        t0 = now_ns()
        waited = False
        while not pred():
            waited = True
            if stop is not None and stop.is_set():
                return False
            if not self._cond.wait(timeout=0.05) and (now_ns() - t0) / 1e9 > DEADLOCK_TIMEOUT_S:
                raise PipelineStall(f"{what} for {DEADLOCK_TIMEOUT_S}s")
        if waited and tracer is not None:
            tracer.record(track, name, t0, now_ns())
        return True

    def put(self, segment, stop=None, tracer: Tracer | None = None) -> bool:
        with self._cond:
            ok = self._block(lambda: len(self._items) < self.capacity, stop,
                             f"collector blocked on full ring (capacity {self.capacity})",
                             tracer, "collector", "collector/stall")
            if not ok:
                return False
            self._items.append(segment)
            self._cond.notify_all()
        return True

    def get(self, stop=None, tracer: Tracer | None = None):
        with self._cond:
            ok = self._block(lambda: len(self._items) > 0, stop,
                             "learner blocked on empty ring", tracer, "learner", "learner/gap")
            if not ok:
                return None
            item = self._items.pop(0)
            self._cond.notify_all()
        return item


@dataclass
class RoleError:
    exc: BaseException
    role: str


class ErrorBox:
    """First background-role exception, re-raised in the learner (R:runtime/sync.py:140-162)."""

    def __init__(self):
        self._error = None
        self._lock = threading.Lock()

    def set(self, role: str, exc: BaseException) -> None:
        with self._lock:
            if self._error is None:
                self._error = RoleError(exc=exc, role=role)

    def raise_if_set(self) -> None:
        with self._lock:
            err = self._error
        if err is not None:
            raise RuntimeError(f"{err.role} role failed: {err.exc!r}") from err.exc
