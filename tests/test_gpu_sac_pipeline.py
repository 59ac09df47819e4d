"""The learner half of the SAC pipeline (R:runtime/sac_runner.py:297-383) on
the device: every replay-path variant -- C / B (HBM replay mirror, lazy
sync + gather), A (learner-side sample + pack + synchronous H2D into one
device slot), baseline (collector-side pinned pack + TransferAgent async
copy into the cold half of a hot/cold pair) -- hands sac_updates exactly
the rows the reference's _acquire_batch would, from the same Philox
streams: the resulting parameters are bit-identical to direct
``sac_updates`` calls on the host-decoded batches."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import replaypath as RP  # noqa: E402
from paper_2605_30313_b200 import runtime as RT  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402

OD, AD, B = 12, 4, 256


@pytest.fixture(autouse=True)
def bf16_mode():
    old = P.get_precision()
    P.set_precision("bf16")
    yield
    P.set_precision(old)


def _state(cfg):
    return A.SacState.create(TN.init_params(TN.Arch(OD, (64, 64), AD), 0),
                             TN.init_params(TN.Arch(OD + AD, (128, 64), 1), 1),
                             TN.init_params(TN.Arch(OD + AD, (128, 64), 1), 2), cfg)


@pytest.mark.parametrize("variant", ["C", "B", "A", "baseline"])
def test_sac_pipeline_variants_feed_the_reference_batches(variant):
    codec = RP.RowCodec(OD, AD)
    storage = RP.ReplayStorage(1000, codec.width)  # wraps during the test
    rng = np.random.default_rng(1)
    cfg = A.SacConfig(batch_size=B, updates_per_step=2, policy_frequency=2)
    st, ref = _state(cfg), _state(cfg)
    pipe = RT.SacPipeline(st, cfg, storage, variant, seed=7)
    pipe.start()
    r_replay, r_learner = RT.stream(7, "replay"), RT.stream(7, "learner")

    def collect(n=300):
        storage.insert(codec.encode(rng.normal(size=(n, OD)), np.tanh(rng.normal(size=(n, AD))),
                                    rng.normal(size=n), rng.normal(size=(n, OD)),
                                    rng.random(n) < 0.05, rng.integers(1, 3, n)))

    try:
        collect()  # warm-up round (learning_starts)
        for tick in range(4):
            collect()
            staged = None
            if variant == "baseline":
                pipe.collector_stage()
                staged = storage.snapshot_sample(B, r_replay)  # the same draw, same moment
            pipe.finish_round()
            got = pipe.learner_tick(tick)
            if variant in ("C", "B"):
                rows = storage.read_rows(storage.sample_indices(B, r_learner))
            elif variant == "A":
                rows = storage.snapshot_sample(B, r_replay)
            else:
                rows = staged
            want = A.sac_updates(codec.decode(rows), ref, cfg, r_learner, 2)
            assert got["critic_loss"] == want[-1].extra["critic_loss"]
            for a, b in ((st.params.actor, ref.params.actor), (st.params.q1, ref.params.q1),
                         (st.params.q2_targ, ref.params.q2_targ)):
                np.testing.assert_array_equal(a.flat(), b.flat())
            assert st.params.log_alpha == ref.params.log_alpha
        assert pipe.slot.version == 4 and pipe.tickets.ticks == 4
        assert pipe.consumed_samples == 4 * 2 * B
    finally:
        pipe.close()


def test_baseline_stall_is_reported():
    """No collector round -> the learner's wait times out with the
    reference's 'pipeline stall' error carrying the slot states."""
    from paper_2605_30313_b200.runtime import sac_pipeline as SP

    codec = RP.RowCodec(OD, AD)
    storage = RP.ReplayStorage(64, codec.width)
    cfg = A.SacConfig(batch_size=8, updates_per_step=1)
    pipe = RT.SacPipeline(_state(cfg), cfg, storage, "baseline")
    old = SP.STALL_TIMEOUT_S
    try:
        pipe.tickets.finish_round()
        pipe.stop.set()
        with pytest.raises(RuntimeError, match="pipeline stall"):
            pipe.learner_tick(0)
    finally:
        SP.STALL_TIMEOUT_S = old
        pipe.close()
