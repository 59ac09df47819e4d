"""APPO target recompute (R:algos/appo.py:35-39) on the bf16 back end:
actor and critic forwards grouped layer by layer (ul_mlp_forward2) give the
same target log-probs and values, bit for bit, as two ul_mlp_forward calls,
and both track the float64 oracle forward within the bf16 tolerance."""

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
from paper_2605_30313_b200.algos import appo as AP  # noqa: E402
from paper_2605_30313_b200.algos import _staging as STG  # noqa: E402
from oracle import port as O  # noqa: E402


def test_grouped_recompute_bit_identical_and_tracks_oracle():
    old = P.get_precision()
    env = os.environ.get("UL_APPO_GROUP_RECOMPUTE")
    try:
        P.set_precision("bf16")
        T, N, od, cd, ad, hid = 4, 2048, 98, 101, 29, (512, 256, 128)
        rng = np.random.default_rng(9)
        a0, c0 = O.net_init((od, *hid, ad), 0), O.net_init((cd, *hid, 1), 1)
        params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), a0.flat()),
                            TN.ModelParams.from_numpy(TN.Arch(cd, hid, 1), c0.flat()))
        obs = rng.normal(size=(T, N, od)).astype(np.float32)
        cobs = rng.normal(size=(T, N, cd)).astype(np.float32)
        act = rng.normal(size=(T, N, ad)).astype(np.float32)
        seg = A.RolloutSegment(obs=obs, critic_obs=cobs, actions=act,
                               behavior_log_prob=np.zeros((T, N)) - 30.0,
                               rewards=rng.normal(size=(T, N)), terminated=np.zeros((T, N), bool),
                               truncated=np.zeros((T, N), bool), values=np.zeros((T, N)),
                               bootstrap_value=np.zeros(N))
        STG._CACHE.clear()
        ds = STG.staging_for(T, N, od, cd, ad, 1, slot="appo")
        assert ds.bf16_rows  # the bf16 back end stages APPO rows as bf16
        ds.load(seg, with_advantages=False)
        out = {}
        for g in ("0", "1"):
            os.environ["UL_APPO_GROUP_RECOMPUTE"] = g
            AP.recompute_targets(ds, params)
            torch.cuda.synchronize()
            out[g] = (ds.tlogp.clone().cpu().numpy(), ds.vnow.clone().cpu().numpy())
        np.testing.assert_array_equal(out["0"][0], out["1"][0])
        np.testing.assert_array_equal(out["0"][1], out["1"][1])
        flat = obs.reshape(-1, od)
        mean, _ = O.mlp_forward(a0, flat)
        want_lp = O.gauss_logp(mean, a0.log_std, act.reshape(-1, ad))
        want_v, _ = O.mlp_forward(c0, cobs.reshape(-1, cd))
        got_lp = out["1"][0].reshape(-1)[: T * N]
        got_v = out["1"][1].reshape(-1)[: T * N]
        # bf16 operands: target log-probs / values within 1e-2 relative
        assert np.max(np.abs(got_lp - want_lp) / np.maximum(1.0, np.abs(want_lp))) <= 1e-2
        assert np.max(np.abs(got_v - want_v.reshape(-1)) / np.maximum(1.0, np.abs(want_v.reshape(-1)))) <= 1e-2
    finally:
        P.set_precision(old)
        STG._CACHE.clear()
        if env is None:
            os.environ.pop("UL_APPO_GROUP_RECOMPUTE", None)
        else:
            os.environ["UL_APPO_GROUP_RECOMPUTE"] = env
