"""Asynchronous PPO on the device (mirror of R:algos/appo.py:21-70).

Recompute target log-probs and values under the current parameters over all
T*N rows (K7 forwards in row chunks + ul_gaussian_logp), V-trace (K2) into the
staged segment's advantage / return slots, then the same device epoch loop
as PPO on (pg_adv, vs, values_now).
"""

from __future__ import annotations

import os

import torch

from .. import _dev, _lib
from ..tensornet.mlp import _staged
from ._staging import staging_for
from .configs import AppoConfig
from .ppo import AcOpt, AcParams, _check_dims, _epochs_on_device
from .segment import UpdateStats

_CHUNK = 1 << 19  # rows per recompute launch set (cfg5: 393,216 rows in one)
_SCRATCH: dict = {}


def _scratch(key, n, dev):
    t = _SCRATCH.get(key)
    if t is None or t.numel() < n:
        t = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        _SCRATCH[key] = t
    return t


def _staged_bf16(params, key):
    desc = params.arch.desc()
    ws = _scratch(key, _lib.lib().ul_mlp_wstage_floats(desc), params.buf.device)
    _lib.call("ul_stage_weights_ex", desc, _dev.ptr(params.buf), _dev.ptr(ws), _lib.UL_GEMM_BF16,
              _dev.stream())
    return _lib.UL_GEMM_BF16, ws


def recompute_targets(ds, params: AcParams) -> None:
    """ds.tlogp <- log pi(a|s) and ds.vnow <- V(s) under the current params."""
    a_arch, c_arch = params.actor.arch, params.critic.arch
    ad = a_arch.output_dim
    dev = ds.obs.device
    rows = ds.rows
    chunk = min(_CHUNK, rows)
    acts_a = _scratch("acts_a", _lib.lib().ul_mlp_act_floats(a_arch.desc(), chunk), dev)
    acts_c = _scratch("acts_c", _lib.lib().ul_mlp_act_floats(c_arch.desc(), chunk), dev)
    mean = _scratch("mean", chunk * ad, dev)
    s = _dev.stream()
    ls = params.actor.buf[params.actor.buf.numel() - ad:]
    if getattr(ds, "bf16_rows", False):
        # bf16 segment rows: the recompute forward runs on the bf16 back end
        # (no input gradients here), weights staged as bf16 rows
        be_a, ws_a = _staged_bf16(params.actor, "wsb_a")
        be_c, ws_c = _staged_bf16(params.critic, "wsb_c")
    else:
        be_a, ws_a = _staged(params.actor)
        be_c, ws_c = _staged(params.critic)
    # (opt-in UL_APPO_GROUP_RECOMPUTE=1: one grouped launch per layer for both
    # networks; at 393,216 rows each launch is long and grouping measured no
    # gain, 1.21 vs 1.20 ms for recompute + V-trace)
    grouped = be_a == be_c and os.environ.get("UL_APPO_GROUP_RECOMPUTE", "0") != "0"
    for r0 in range(0, rows, chunk):
        m = min(chunk, rows - r0)
        if grouped:  # actor and critic layer by layer, one launch per layer
            _lib.call("ul_mlp_forward2", a_arch.desc(), _dev.ptr(params.actor.buf),
                      _dev.ptr(ws_a), _dev.ptr(ds.obs[r0]), ds.obs.stride(0), _dev.ptr(acts_a),
                      _dev.ptr(mean), ad, c_arch.desc(), _dev.ptr(params.critic.buf),
                      _dev.ptr(ws_c), _dev.ptr(ds.cobs[r0]), ds.cobs.stride(0),
                      _dev.ptr(acts_c), _dev.ptr(ds.vnow[r0:]), 1, be_a, m, s)
        else:
            _lib.call("ul_mlp_forward", a_arch.desc(), _dev.ptr(params.actor.buf),
                      _dev.ptr(ws_a), be_a, _dev.ptr(ds.obs[r0]), ds.obs.stride(0), m,
                      _dev.ptr(acts_a), _dev.ptr(mean), ad, s)
            _lib.call("ul_mlp_forward", c_arch.desc(), _dev.ptr(params.critic.buf),
                      _dev.ptr(ws_c), be_c, _dev.ptr(ds.cobs[r0]), ds.cobs.stride(0), m,
                      _dev.ptr(acts_c), _dev.ptr(ds.vnow[r0:]), 1, s)
        _lib.call("ul_gaussian_logp", _dev.ptr(mean), ad, _dev.ptr(ls), _dev.ptr(ds.act[r0]),
                  ds.act.stride(0), m, ad, _dev.ptr(ds.tlogp[r0:]), s)


def vtrace_into(ds, cfg: AppoConfig) -> None:
    """V-trace (K2) writing pg_adv -> ds.adv and vs -> ds.ret."""
    _lib.call("ul_vtrace_f32", _dev.ptr(ds.blogp), _dev.ptr(ds.tlogp), _dev.ptr(ds.rewards),
              _dev.ptr(ds.vnow), _dev.ptr(ds.term), _dev.ptr(ds.trunc),
              _dev.ptr(ds.tv) if ds.has_tv else None, _dev.ptr(ds.boot), ds.T, ds.N,
              float(cfg.gamma), float(cfg.vtrace_clip_rho), float(cfg.vtrace_clip_c),
              _dev.ptr(ds.ret), _dev.ptr(ds.adv), _dev.stream())


def appo_update_resident(ds, params: AcParams, opt: AcOpt, cfg: AppoConfig, rng) -> UpdateStats:
    recompute_targets(ds, params)
    vtrace_into(ds, cfg)
    return _epochs_on_device(ds, ds.adv, ds.ret, ds.vnow, params, opt, cfg, rng)


def appo_update(segment, params: AcParams, opt: AcOpt, cfg: AppoConfig, rng,
                learner_version: int = 0) -> UpdateStats:
    """V-trace-corrected PPO epochs on a (possibly stale) segment
    (R:algos/appo.py:21-70)."""
    od, cd, ad = _check_dims(segment, params)
    T, N = segment.horizon, segment.n_envs
    if (T * N) % cfg.minibatches != 0:
        raise ValueError(f"minibatches {cfg.minibatches} must divide batch size {T * N}")
    ds = staging_for(T, N, od, cd, ad, cfg.epochs, slot="appo")
    ds.load(segment, with_advantages=False)
    stats = appo_update_resident(ds, params, opt, cfg, rng)
    stats.staleness = learner_version - segment.behavior_version
    return stats
