"""CPU tests of the product's host-side logic: replay ring / codec / pack-slot
state machine, rollout ring, tracer, collector-side packers, and the
data-parallel minibatch sharding + gradient all-reduce over gloo (world 2)."""

import os
import threading

import numpy as np
import pytest

from oracle import port as O
from paper_2605_30313_b200 import _dist
from paper_2605_30313_b200.errors import PipelineStall, SlotStateError
from paper_2605_30313_b200.replaypath.slots import PackSlotPair, SlotState, pack
from paper_2605_30313_b200.replaypath.storage import ReplayStorage, RowCodec
from paper_2605_30313_b200.trace import Tracer


def test_replay_storage_matches_reference_goldens(golden):
    g = golden("norm_replay")
    st = ReplayStorage(37, 2 * 4 + 2 + 3, pinned=False)
    for s in range(6):
        st.insert(g[f"r_rows{s}"])
    assert st.valid_range() == tuple(g["r_window"])
    idx = st.sample_indices(64, O.philox_stream(1, "replay"))
    np.testing.assert_array_equal(idx, g["r_idx"])
    np.testing.assert_array_equal(st.read_rows(idx), g["r_read"])
    np.testing.assert_array_equal(st.snapshot_sample(16, O.philox_stream(1, "replay2")),
                                  g["r_snapshot"])
    dec = RowCodec(4, 2).decode(st.read_rows(idx))
    for k, v in dec.items():
        np.testing.assert_array_equal(v, g[f"r_dec_{k}"])
    with pytest.raises(IndexError):
        st.read_rows([0])


def test_ring_eviction_and_errors():
    st = ReplayStorage(4, 1, pinned=False)
    st.insert(np.arange(3, dtype=np.float32)[:, None])
    st.insert(np.arange(3, 9, dtype=np.float32)[:, None])
    assert st.valid_range() == (5, 9)
    np.testing.assert_array_equal(st._data[:, 0], [8, 5, 6, 7])
    with pytest.raises(ValueError, match="width"):
        st.insert(np.zeros((2, 3), np.float32))
    with pytest.raises(ValueError, match="replay empty"):
        ReplayStorage(4, 1, pinned=False).snapshot_sample(2, np.random.default_rng(0))
    tr = Tracer()
    st2 = ReplayStorage(10, 4, tracer=tr, pinned=False)
    st2.insert(np.zeros((3, 4), np.float32))
    assert tr.events()[0].name == "collector/replay_add" and tr.events()[0].args["rows"] == 3


def test_codec_roundtrip():
    c = RowCodec(3, 2)
    rng = np.random.default_rng(0)
    obs, act = rng.normal(size=(5, 3)), rng.normal(size=(5, 2))
    rows = c.encode(obs, act, rng.normal(size=5), obs + 1, [1, 0, 0, 1, 0], [1, 2, 1, 1, 3])
    d = c.decode(rows)
    np.testing.assert_allclose(d["obs"], obs.astype(np.float32))
    assert d["terminated"].tolist() == [True, False, False, True, False]
    assert d["n_used"].tolist() == [1, 2, 1, 1, 3]


def test_pack_slot_state_machine():
    pair = PackSlotPair(4, 3, memory_class="pageable")
    slot = pair.acquire_free(timeout=0.1)
    pack(slot, np.ones((2, 3), np.float32), pair)
    assert slot.state is SlotState.READY
    with pytest.raises(SlotStateError):
        slot.transition(SlotState.PACKING)
    slot.transition(SlotState.TRANSFERRING)
    slot.transition(SlotState.FREE)
    other = pair.acquire_free(timeout=0.1)
    assert other is not None


def test_rollout_ring_fifo_and_stall(monkeypatch):
    from paper_2605_30313_b200.runtime import sync

    ring = sync.RolloutRing(2)
    ring.put(1)
    ring.put(2)
    assert ring.get() == 1 and ring.get() == 2
    monkeypatch.setattr(sync, "DEADLOCK_TIMEOUT_S", 0.2)
    with pytest.raises(PipelineStall):
        ring.get()
    stop = threading.Event()
    stop.set()
    assert ring.get(stop) is None
    box = sync.ErrorBox()
    box.set("collector", ValueError("boom"))
    with pytest.raises(RuntimeError, match="collector role failed"):
        box.raise_if_set()


def test_tracer_registry_and_overlap():
    tr = Tracer()
    tr.record("learner", "learner/update", 0, 10)
    with pytest.raises(RuntimeError, match="overlapping"):
        tr.record("learner", "learner/update", 5, 12)
    with pytest.raises(ValueError):
        tr.record("learner", "not/registered", 20, 30)


def test_shard_rows():
    assert _dist.shard_rows(100, 24, 4, 0) == (100, 106)
    assert _dist.shard_rows(100, 24, 4, 3) == (118, 124)
    with pytest.raises(ValueError):
        _dist.shard_rows(0, 10, 4, 0)


def _dp_worker(rank, world, port, result):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # one PPO minibatch step, sharded: each rank computes its shard's grads
        # with the GLOBAL 1/mb scaling (what the plan does), then the product's
        # all_reduce_sum recombines them
        rng = np.random.default_rng(0)
        n = 16
        actor = O.net_init((5, 8, 2), 0, dtype=np.float64)
        critic = O.net_init((6, 8, 1), 1, dtype=np.float64)
        obs, cobs = rng.normal(size=(n, 5)), rng.normal(size=(n, 6))
        act = rng.normal(size=(n, 2))
        blogp = rng.normal(size=n) * 0.1 - 3.0
        adv, ret, oldv = rng.normal(size=n), rng.normal(size=n), rng.normal(size=n)
        lo, hi = _dist.shard_rows(0, n, world, rank)
        cfg = O.PpoCfg(entropy_coef=0.0)
        _, ga, gc = O.ppo_loss_grads(actor, critic, obs[lo:hi], cobs[lo:hi], act[lo:hi],
                                     blogp[lo:hi], adv[lo:hi], ret[lo:hi], oldv[lo:hi], cfg)
        scale = (hi - lo) / n
        flat = torch.tensor(np.concatenate([ga.flat(), gc.flat()]) * scale)
        _dist.all_reduce_sum(flat)
        _, fa, fc = O.ppo_loss_grads(actor, critic, obs, cobs, act, blogp, adv, ret, oldv, cfg)
        full = np.concatenate([fa.flat(), fc.flat()])
        result[rank] = float(np.max(np.abs(flat.numpy() - full)))
    finally:
        dist.destroy_process_group()


def test_data_parallel_gradient_allreduce_gloo():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    result = mgr.dict()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, result)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert result[0] < 1e-12 and result[1] < 1e-12


def test_pending_updates_drain_in_launch_order(monkeypatch):
    """update_async bookkeeping (no GPU): results are read in launch order,
    reading a later handle first drains the earlier ones, a failing update's
    error surfaces from its own result(), and the host step counters end at
    the newest update's."""
    from paper_2605_30313_b200.algos import ppo as P
    from paper_2605_30313_b200.errors import DivergenceError

    class Plan:
        def __init__(self, name):
            self.name, self.pending = name, None

    class Opt:
        class S:
            t = 0
        actor, critic, lr = S(), S(), 1e-3

    seen = []

    def fake_finish(plan, opt):
        seen.append(plan.name)
        opt.actor.t = opt.critic.t = len(seen) * 10
        if plan.name == "c":
            raise DivergenceError("non-finite at step 3")
        return plan.name

    monkeypatch.setattr(P, "finish_plan", fake_finish)
    monkeypatch.setattr(P, "_stats", lambda res, opt: res)
    monkeypatch.setattr(P, "_PENDING", [])
    opt = Opt()
    hs = []
    for n in "abcd":
        pl = Plan(n)
        h = P.PendingUpdate(pl, opt)
        pl.pending = h
        P._PENDING.append(h)
        hs.append(h)
    assert hs[1].result() == "b" and seen == ["a", "b"]  # a drained first
    assert hs[0].result() == "a" and seen == ["a", "b"]  # cached, not re-read
    with pytest.raises(DivergenceError):
        hs[2].result()
    with pytest.raises(DivergenceError):  # the error stays with its handle
        hs[2].result()
    P._drain_pending()
    assert seen == ["a", "b", "c", "d"] and hs[3].result() == "d"
    assert opt.actor.t == 40 and all(h.plan.pending is None for h in hs)


def test_product_adaptive_lr_step_known_answers():
    """The product's adaptive_lr_step (host scalar logic on the learner thread)
    against the reference test-suite's known answers (R:tests/test_ppo.py:
    218-238; R:algos/ppo.py:232-250) and the oracle on a sweep."""
    from oracle import port as O
    from paper_2605_30313_b200.algos import PpoConfig, adaptive_lr_step

    cfg = PpoConfig()
    assert adaptive_lr_step(1e-3, 0.02, cfg, update_index=5) == pytest.approx(1e-3 / 1.2)
    assert adaptive_lr_step(1e-3, 0.005, cfg, update_index=10) == pytest.approx(1.1e-3)
    assert adaptive_lr_step(1e-3, 0.0095, cfg, 5) == 1e-3
    assert adaptive_lr_step(1e-3, 0.02, cfg, update_index=3) == 1e-3
    assert adaptive_lr_step(9.5e-3, 0.001, cfg, 5) == 1e-2
    assert adaptive_lr_step(1.1e-6, 1.0, cfg, 5) == 1e-6
    assert adaptive_lr_step(1e-3, 0.5, PpoConfig(schedule="fixed"), 5) == 1e-3
    rng = np.random.default_rng(0)
    for _ in range(200):
        lr, kl, it = 10 ** rng.uniform(-6.5, -1.5), 10 ** rng.uniform(-4, 0), int(rng.integers(0, 20))
        assert adaptive_lr_step(lr, kl, cfg, it) == O.adaptive_lr(lr, kl, it)
