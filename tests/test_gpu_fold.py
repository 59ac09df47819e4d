"""The K13 prepare pass folded into the step's gradient reduction (the
single-process bf16 fused-head PPO step, csrc/mlp.cu reduce_all_kernel<true>)
must be the same optimizer step as the separate prepare kernel
(UL_FOLD_PREP=0): joint norm, clip factor, loss bookkeeping, step counters and
the divergence latch (R:tensornet/adam.py:30-80, R:algos/ppo.py:170-189).

The fold covers only values the reduction stores; a gradient element written
elsewhere would drop out of the norm and change the clip factor, which the
cfg2 comparison below would see (max_grad_norm = 0.05 clips every step there).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos import ppo as PPO  # noqa: E402
from oracle import port as O  # noqa: E402
from helpers import _synthetic  # noqa: E402


@pytest.fixture(autouse=True)
def _restore():
    old = P.get_precision()
    env = os.environ.get("UL_FOLD_PREP")
    yield
    P.set_precision(old)
    if env is None:
        os.environ.pop("UL_FOLD_PREP", None)
    else:
        os.environ["UL_FOLD_PREP"] = env
    PPO._PLANS.clear()


def _run(fold, segd, actor, critic, dims, rng_factory, cfg):
    od, cd, ad, hid = dims
    os.environ["UL_FOLD_PREP"] = "1" if fold else "0"
    PPO._PLANS.clear()  # the flag is read when a plan is created
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(cd, hid, 1), critic.flat()))
    opt = A.AcOpt.for_params(params, 1e-3)
    seg = A.RolloutSegment(**segd)
    seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                                        seg.bootstrap_value, 0.99, 0.95,
                                        truncation_values=seg.truncation_values)
    st = A.ppo_update(seg, params, opt, cfg, rng_factory())
    return params, opt, st


def test_folded_prepare_matches_separate_prepare_cfg2():
    """cfg2 bf16 update (24 x 4096, 5 x 4, reference permutation stream):
    folded vs separate prepare.  The two sum the same squares in a different
    fixed order, so the f64 norm may differ in its last bits; the f32 clip
    factor, every Adam step and the statistics agree to 1e-6."""
    T, N, od, cd, ad, hid = 24, 4096, 235, 235, 12, (512, 256, 128)
    segd, actor, critic = _synthetic(T, N, od, cd, ad, hid, seed=21)
    P.set_precision("bf16")
    cfg = A.PpoConfig(max_grad_norm=0.05)  # clip on every step: the norm matters
    runs = [_run(f, segd, actor, critic, (od, cd, ad, hid),
                 lambda: O.philox_stream(1, "update"), cfg) for f in (False, True)]
    (p0, o0, s0), (p1, o1, s1) = runs
    assert abs(s1.grad_norm - s0.grad_norm) <= 1e-9 * s0.grad_norm, (s0.grad_norm, s1.grad_norm)
    assert s0.grad_norm > cfg.max_grad_norm  # the clip is active
    for k in ("policy_loss", "value_loss", "entropy", "kl"):
        a, b = getattr(s0, k), getattr(s1, k)
        assert abs(a - b) <= 1e-6 * max(1.0, abs(a)), (k, a, b)
    assert (o0.actor.t, o0.critic.t) == (o1.actor.t, o1.critic.t) == (20, 20)
    for x, y in ((p0.actor.flat(), p1.actor.flat()), (p0.critic.flat(), p1.critic.flat())):
        d = np.abs(x.astype(np.float64) - y)
        assert d.max() <= 1e-6, d.max()


def test_folded_prepare_divergence_latch():
    """A non-finite advantage reaches the loss head: the folded tail latches
    divergence exactly like the prepare kernel -- DivergenceError, no step
    applied, parameters untouched."""
    T, N, od, cd, ad, hid = 8, 512, 48, 48, 12, (256, 128, 128)
    segd, actor, critic = _synthetic(T, N, od, cd, ad, hid, seed=3)
    segd["rewards"] = segd["rewards"].copy()
    segd["rewards"][2, 5] = np.nan
    P.set_precision("bf16")
    os.environ["UL_FOLD_PREP"] = "1"
    PPO._PLANS.clear()
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(cd, hid, 1), critic.flat()))
    opt = A.AcOpt.for_params(params, 1e-3)
    seg = A.RolloutSegment(**segd)
    seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                                        seg.bootstrap_value, 0.99, 0.95,
                                        truncation_values=seg.truncation_values)
    before_a, before_c = params.actor.flat().copy(), params.critic.flat().copy()
    with pytest.raises(TN.DivergenceError):
        A.ppo_update(seg, params, opt, A.PpoConfig(), O.philox_stream(1, "update"))
    np.testing.assert_array_equal(params.actor.flat(), before_a)
    np.testing.assert_array_equal(params.critic.flat(), before_c)
    assert (opt.actor.t, opt.critic.t) == (0, 0)


def test_folded_prepare_small_update_matches_separate():
    """A small bf16 update (several reduction shapes: 48-wide input, 256-128-128
    trunk, 3 epochs x 2 minibatches) folded vs separate."""
    T, N, od, cd, ad, hid = 8, 512, 48, 40, 12, (256, 128, 128)
    segd, actor, critic = _synthetic(T, N, od, cd, ad, hid, seed=4)
    P.set_precision("bf16")
    cfg = A.PpoConfig(epochs=3, minibatches=2)
    (p0, o0, s0), (p1, o1, s1) = [
        _run(f, segd, actor, critic, (od, cd, ad, hid), lambda: np.random.default_rng(5), cfg)
        for f in (False, True)]
    assert abs(s1.grad_norm - s0.grad_norm) <= 1e-9 * max(1.0, s0.grad_norm)
    for x, y in ((p0.actor.flat(), p1.actor.flat()), (p0.critic.flat(), p1.critic.flat())):
        assert np.abs(x.astype(np.float64) - y).max() <= 1e-6


def test_segment_row_layouts_gather_identically():
    """The three staging layouts of a segment's observation rows give the SAME
    bf16 update, bit for bit: padded fp32 16-byte rows (the gather converts to
    bf16), the host layout (raw_rows: 940-byte rows, no re-pitch; the gather
    converts one float per lane and reads the ones unit one float past each
    row) and bf16 rows converted once at staging (bf16_rows, the bf16 default:
    the gather copies 16-byte units)."""
    from paper_2605_30313_b200.algos import _staging as STG

    T, N, od, cd, ad, hid = 6, 512, 235, 101, 12, (256, 128, 128)
    segd, actor, critic = _synthetic(T, N, od, cd, ad, hid, seed=8)
    P.set_precision("bf16")
    cfg = A.PpoConfig(epochs=2, minibatches=2)
    out = []
    for raw, bfr in ((False, False), (True, False), (False, True)):
        PPO._PLANS.clear()
        STG._CACHE.clear()
        ds = STG.DeviceSegment(T, N, od, cd, ad, cfg.epochs, raw_rows=raw, bf16_rows=bfr)
        STG._CACHE[("ppo", T, N, od, cd, ad, cfg.epochs, torch.cuda.current_device(),
                    STG.bf16_rows_default("ppo"))] = ds
        params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), actor.flat()),
                            TN.ModelParams.from_numpy(TN.Arch(cd, hid, 1), critic.flat()))
        opt = A.AcOpt.for_params(params, 1e-3)
        seg = A.RolloutSegment(**segd)
        seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated,
                                            seg.truncated, seg.bootstrap_value, 0.99, 0.95,
                                            truncation_values=seg.truncation_values)
        st = A.ppo_update(seg, params, opt, cfg, O.philox_stream(2, "update"))
        assert ds.obs.stride(0) == (od if raw else 240 if bfr else 236)
        out.append((params.actor.flat(), params.critic.flat(), st.policy_loss))
    STG._CACHE.clear()
    for o in out[1:]:
        np.testing.assert_array_equal(out[0][0], o[0])
        np.testing.assert_array_equal(out[0][1], o[1])
        assert out[0][2] == o[2]
