"""HBM layout of a rollout segment and the H2D staging into it.

Layout (rows = T*N transitions, t-major like the reference's reshape(-1)):
  obs   [rows, ld_o] f32   ld_o = round_up(obs_dim + 1, 4)  (16 B rows; raw_rows:
                           ld_o = obs_dim, the host layout, no re-pitch)
  cobs  [rows, ld_c] f32
  act   [rows, ld_a] f32
  blogp, rewards, values, tv, adv, ret   [rows] f32
  term, trunc                           [rows] u8
  boot  [N] f32
  perm  [epochs, rows] i64   minibatch permutations
Buffers are cached per shape so a bound update plan (and its CUDA graph)
stays valid across updates: each update overwrites the same HBM.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _dev, _lib


def _is_dev(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


class DeviceSegment:
    def __init__(self, T: int, N: int, obs_dim: int, cobs_dim: int, act_dim: int, epochs: int,
                 raw_rows: bool = False, bf16_rows: bool = False):
        dev = _dev.require_cuda()
        self.T, self.N, self.rows = T, N, T * N
        self.dims = (obs_dim, cobs_dim, act_dim)
        # raw_rows: obs / cobs / act keep the host row layout (no re-pitch
        # pass after the H2D); each buffer has a 16-byte tail because the
        # minibatch gather reads one float past a row for the ones column.
        # Off by default: the gather then converts one float per lane (4-byte
        # aligned 940 B rows) and costs more per update (cfg2: 4.52 vs 4.34
        # ms) than the re-pitch pass it saves (e2e 4.74 vs 4.68 ms).
        # bf16_rows (bf16 back end): obs / cobs are staged ONCE per segment as
        # the bf16 rows the networks read -- round_up(d + 1, 8) wide, ones
        # column set -- by the re-pitch pass that follows the H2D, so every
        # minibatch gather copies half the bytes (16-byte units, no conversion)
        self.raw_rows = raw_rows and not bf16_rows
        self.bf16_rows = bf16_rows
        if bf16_rows:
            ld8 = lambda d: (d + 1 + 7) // 8 * 8  # noqa: E731
            self.ld = (ld8(obs_dim), ld8(cobs_dim), _dev.feature_ld(act_dim))
        elif raw_rows:
            self.ld = tuple(self.dims)
        else:
            self.ld = tuple(_dev.feature_ld(d) for d in self.dims)
        f32 = dict(dtype=torch.float32, device=dev)
        rows = self.rows

        def rows_buf(ld, dtype=torch.float32):
            if not self.raw_rows:
                return _dev.zeros((rows, ld), dtype=dtype, device=dev)
            return _dev.zeros(rows * ld + 4, **f32)[:rows * ld].view(rows, ld)

        row_dt = torch.bfloat16 if bf16_rows else torch.float32
        self.obs = rows_buf(self.ld[0], row_dt)
        self.cobs = rows_buf(self.ld[1], row_dt)
        self.act = rows_buf(self.ld[2])
        self.blogp = _dev.zeros(rows, **f32)
        self.rewards = _dev.zeros(rows, **f32)
        self.values = _dev.zeros(rows, **f32)
        self.tv = _dev.zeros(rows, **f32)
        self.adv = _dev.zeros(rows, **f32)
        self.ret = _dev.zeros(rows, **f32)
        self.vnow = _dev.zeros(rows, **f32)   # APPO: values under the current critic
        self.tlogp = _dev.zeros(rows, **f32)  # APPO: target log-prob
        self.term = _dev.zeros(rows, dtype=torch.uint8, device=dev)
        self.trunc = _dev.zeros(rows, dtype=torch.uint8, device=dev)
        self.boot = _dev.zeros(N, **f32)
        self.perm = _dev.zeros((max(epochs, 1), rows), dtype=torch.int64, device=dev)
        self.has_tv = False
        self.slot = "ppo"
        self._raw: dict = {}  # field -> contiguous H2D landing buffer
        self._land: dict = {}  # f32 field -> f64 landing buffer (pinned f64 sources)
        self._pin: dict = {}  # field -> page-locked conversion buffer (f64 / bool -> f32 / u8)
        self._pin_busy = None  # event after the last load's copies
        # the zero fills above run on the current stream, but a pipeline slot
        # is loaded on its copy stream: let the fills land first (once per
        # slot), or a fill still queued behind a running update could
        # overwrite freshly copied rows
        torch.cuda.current_stream().synchronize()

    # ------------------------------------------------------------- loading
    def _raw_for(self, name: str, width: int, device) -> torch.Tensor:
        """The field's own contiguous H2D landing buffer (one per field, so every
        copy of a segment can be queued before any re-pitch kernel)."""
        raw = self._raw.get(name)
        if raw is None or raw.numel() != self.rows * width:
            # (+16 B: a bf16 re-pitch reads one float past the last row)
            raw = torch.empty(self.rows * width + 4, dtype=torch.float32,
                              device=device)[:self.rows * width]
            self._raw[name] = raw
        return raw

    def _repitch(self, jobs) -> None:
        """One K4 row-kernel launch re-pitching landed fields into their HBM rows
        (bf16 destinations: converted on the way, ones column set)."""
        if not jobs:
            return
        nrows = jobs[0][1].shape[0]
        # bf16 rows: one conversion pass per field (8 output columns per
        # thread, ones column set)
        for r, d, w in jobs:
            if d.dtype == torch.bfloat16:
                _lib.call("ul_rows_to_bf16", _dev.ptr(r), w, w, _dev.ptr(d), d.stride(0), nrows,
                          w, _dev.stream())
        jobs = [(r, d, w) for r, d, w in jobs if d.dtype != torch.bfloat16]
        if not jobs:
            return
        _lib.call("ul_gather_rows", len(jobs), _lib.ptr_array([_dev.ptr(r) for r, _, _ in jobs]),
                  _lib.ptr_array([_dev.ptr(d) for _, d, _ in jobs]),
                  _lib.i64_array([w * 4 for _, _, w in jobs]),
                  _lib.i64_array([d.stride(0) * 4 for _, d, _ in jobs]),
                  _lib.i64_array([w * 4 for _, _, w in jobs]), None, None, nrows,
                  0, 0, nrows, None, _dev.stream())

    def _put_rows(self, name: str, dst: torch.Tensor, src, width: int, jobs: list) -> None:
        """Host [rows, width] -> HBM [rows, ld]: one contiguous H2D at full PCIe
        rate into the field's landing buffer; the re-pitch (K4 row kernel, a
        pitched 2-D H2D of 940 B rows crawls at a fraction of link speed) is
        appended to `jobs` and launched after every copy of the segment: on
        the copy stream a kernel queued between two copies waits for SMs the
        running update holds, and would stall the copies behind it."""
        if _is_dev(src) and dst.dtype == torch.bfloat16:  # device rows -> bf16 rows
            src = src.reshape(self.rows, width).to(torch.float32).contiguous()
            raw = self._raw_for(name, width, dst.device)
            _lib.call("ul_memcpy_async", _dev.ptr(raw), _dev.ptr(src), src.numel() * 4,
                      _dev.stream())
            jobs.append((raw, dst, width))
            return
        if _is_dev(src):  # device -> device staging copy (copy engine, re-pitched)
            src = src.reshape(self.rows, width)
            if src.dtype != torch.float32:
                src = src.to(torch.float32)
            src = src.contiguous()
            _lib.call("ul_memcpy2d_async", _dev.ptr(dst), dst.stride(0) * 4, _dev.ptr(src),
                      width * 4, width * 4, self.rows, _dev.stream())
            return
        a = np.asarray(src)
        if a.dtype != np.float32:
            a = a.astype(np.float32)
        a = np.ascontiguousarray(a.reshape(self.rows, width))
        if self.raw_rows:  # the H2D lands in the segment rows themselves
            _dev.h2d(dst, a)
            return
        raw = self._raw_for(name, width, dst.device)
        _dev.h2d(raw, a)
        jobs.append((raw, dst, width))

    def _put_vec(self, dst: torch.Tensor, src, dtype=np.float32, casts: list | None = None) -> None:
        if _is_dev(src):
            src = src.reshape(-1)
            if src.dtype == torch.float64 and dst.dtype == torch.float32:
                _lib.call("ul_narrow_f64", 1, _lib.ptr_array([_dev.ptr(src.contiguous())]),
                          _lib.ptr_array([_dev.ptr(dst)]), _lib.i64_array([dst.numel()]),
                          _dev.stream())
                return
            if src.dtype == torch.bool and dst.dtype == torch.uint8:
                src = src.view(torch.uint8)
            if src.dtype != dst.dtype:
                src = src.to(dst.dtype)
            src = src.contiguous()
            _lib.call("ul_memcpy_async", _dev.ptr(dst), _dev.ptr(src), dst.numel() * dst.element_size(),
                      _dev.stream())
            return
        a = np.asarray(src)
        if a.dtype == np.bool_ and dtype == np.uint8:
            a = a.view(np.uint8)  # same bytes
        if casts is not None and a.dtype == np.float64 and dtype == np.float32 \
                and _dev.is_pinned(a):
            # pinned f64 (the reference's [T, N] per-step scalars): copy the
            # bytes as they are and narrow on the device after the segment's
            # copies -- no host conversion, no wait on the previous load
            land = self._land.get(dst.data_ptr())
            if land is None or land.numel() != a.size:
                land = torch.empty(a.size, dtype=torch.float64, device=dst.device)
                self._land[dst.data_ptr()] = land
            _dev.h2d(land, a.reshape(-1))
            casts.append((land, dst))
            return
        if a.dtype != dtype:
            # convert into this slot's page-locked buffer for the field, so the
            # copy stays asynchronous (a pageable temporary would make the
            # driver synchronise the copy stream, i.e. block the host behind
            # the segment's large copies)
            buf = self._pin.get(dst.data_ptr())
            if buf is None or buf.size != a.size:
                buf = _dev.pinned_empty((a.size,), dtype)
                self._pin[dst.data_ptr()] = buf
            if self._pin_busy is not None:
                self._pin_busy.synchronize()  # the previous load's copies have read it
            np.copyto(buf, a.reshape(-1), casting="unsafe")
            a = buf
        _dev.h2d(dst, a.reshape(-1))

    def load(self, seg, with_advantages: bool = True) -> None:
        """Stage every field the learner reads (async on the current stream;
        pinned host arrays copy without a host sync)."""
        od, cd, ad = self.dims
        jobs: list = []
        casts: list = []
        self._put_rows("obs", self.obs, seg.obs, od, jobs)
        self._put_rows("cobs", self.cobs, seg.critic_obs, cd, jobs)
        self._put_rows("act", self.act, seg.actions, ad, jobs)
        self._put_vec(self.blogp, seg.behavior_log_prob, casts=casts)
        self._put_vec(self.rewards, seg.rewards, casts=casts)
        self._put_vec(self.values, seg.values, casts=casts)
        self._put_vec(self.term, seg.terminated, np.uint8)
        self._put_vec(self.trunc, seg.truncated, np.uint8)
        self._put_vec(self.boot, seg.bootstrap_value, casts=casts)
        self.has_tv = seg.truncation_values is not None
        if self.has_tv:
            self._put_vec(self.tv, seg.truncation_values, casts=casts)
        if with_advantages:
            self._put_vec(self.adv, seg.advantages, casts=casts)
            self._put_vec(self.ret, seg.returns, casts=casts)
        if self._pin:  # (recorded before the re-pitch: the copies alone read the buffers)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self._pin_busy = ev
        if casts:  # f64 -> f32 narrowing of the landed scalars, one launch
            _lib.call("ul_narrow_f64", len(casts), _lib.ptr_array([_dev.ptr(l) for l, _ in casts]),
                      _lib.ptr_array([_dev.ptr(d) for _, d in casts]),
                      _lib.i64_array([l.numel() for l, _ in casts]), _dev.stream())
        self._repitch(jobs)

    # ------------------------------------------------- per-step streaming
    def _put_step_rows(self, name: str, dst: torch.Tensor, t: int, src, width: int) -> None:
        """Step t's [N, width] host rows -> HBM rows [t*N, (t+1)*N) (t-major)."""
        N = self.N
        a = np.asarray(src)
        if a.dtype != np.float32:
            a = a.astype(np.float32)
        a = np.ascontiguousarray(a.reshape(N, width))
        if self.raw_rows:  # step t's rows are one contiguous block of the segment
            _dev.h2d(dst[t * N:(t + 1) * N], a)
            return
        raw = self._raw_for(name, width, dst.device)
        part = raw[t * N * width:(t + 1) * N * width]
        _dev.h2d(part, a)
        rb = width * 4
        if dst.dtype == torch.bfloat16:  # converted, ones column set
            _lib.call("ul_rows_to_bf16", _dev.ptr(part), width, width,
                      _dev.ptr(dst[t * N:(t + 1) * N]), dst.stride(0), N, width, _dev.stream())
            return
        _lib.call("ul_gather_rows", 1, _lib.ptr_array([_dev.ptr(part)]),
                  _lib.ptr_array([_dev.ptr(dst[t * N:(t + 1) * N])]), _lib.i64_array([rb]),
                  _lib.i64_array([dst.stride(0) * 4]), _lib.i64_array([rb]), None, None, N,
                  0, 0, N, None, _dev.stream())

    def _put_step_vec(self, dst: torch.Tensor, t: int, src, dtype=np.float32) -> None:
        a = np.asarray(src)
        if a.dtype != dtype:
            a = a.astype(dtype)
        _dev.h2d(dst[t * self.N:(t + 1) * self.N], np.ascontiguousarray(a.reshape(-1)))

    def load_step(self, t: int, obs, critic_obs, actions, behavior_log_prob, rewards,
                  terminated, truncated, values, truncation_values=None) -> None:
        """Stage one environment step (the [N, D] chunk SegmentCollector.collect
        fills per step, R:runtime/collect.py:86-117) as soon as it exists."""
        if not 0 <= t < self.T:
            raise IndexError(f"step {t} outside [0, {self.T})")
        od, cd, ad = self.dims
        self._put_step_rows("obs", self.obs, t, obs, od)
        self._put_step_rows("cobs", self.cobs, t, critic_obs, cd)
        self._put_step_rows("act", self.act, t, actions, ad)
        self._put_step_vec(self.blogp, t, behavior_log_prob)
        self._put_step_vec(self.rewards, t, rewards)
        self._put_step_vec(self.term, t, terminated, np.uint8)
        self._put_step_vec(self.trunc, t, truncated, np.uint8)
        self._put_step_vec(self.values, t, values)
        if truncation_values is not None:
            self.has_tv = True
            self._put_step_vec(self.tv, t, truncation_values)

    def h2d_bytes(self, seg, with_advantages: bool = True) -> int:
        """Bytes one load() moves over PCIe (pinned f64 scalars cross as f64)."""
        od, cd, ad = self.dims

        def sc(a):
            if _is_dev(a):
                return 4
            a = np.asarray(a)
            return 8 if a.dtype == np.float64 and _dev.is_pinned(a) else 4

        n = self.rows * 4 * (od + cd + ad)
        n += self.rows * (sc(seg.behavior_log_prob) + sc(seg.rewards) + sc(seg.values))
        if with_advantages:
            n += self.rows * (sc(seg.advantages) + sc(seg.returns))
        n += self.rows * 2 + self.N * sc(seg.bootstrap_value)
        if seg.truncation_values is not None:
            n += self.rows * sc(seg.truncation_values)
        return n


_CACHE: dict = {}


def bf16_rows_default(slot: str) -> bool:
    """Staging on the bf16 back end keeps observation rows in bf16 (PPO, and
    APPO whose recompute forward then runs bf16 too; UL_BF16_ROWS=0 disables,
    UL_APPO_BF16_RECOMPUTE=0 keeps APPO on fp32 rows and a tf32 recompute)."""
    import os

    if slot == "appo" and os.environ.get("UL_APPO_BF16_RECOMPUTE", "1") == "0":
        return False
    return _lib.gemm_backend() == 2 and os.environ.get("UL_BF16_ROWS", "1") != "0"


def staging_for(T, N, obs_dim, cobs_dim, act_dim, epochs, slot: str = "ppo") -> DeviceSegment:
    bf = bf16_rows_default(slot)
    key = (slot, T, N, obs_dim, cobs_dim, act_dim, max(epochs, 1), torch.cuda.current_device(), bf)
    ds = _CACHE.get(key)
    if ds is None:
        ds = DeviceSegment(T, N, obs_dim, cobs_dim, act_dim, epochs, bf16_rows=bf)
        ds.slot = slot
        _CACHE[key] = ds
    return ds
