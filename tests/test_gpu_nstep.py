"""Device FlashSAC collector transforms: return-std
reward normalisation + n-step packing + replay insert on the GPU, against the
host restatement of R:algos/estimators.py:125-224 and RowCodec."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import replaypath as RP  # noqa: E402


@pytest.mark.parametrize("n,norm", [(1, False), (3, False), (3, True), (5, True)])
def test_device_nstep_matches_host(n, norm):
    rng = np.random.default_rng(n * 10 + int(norm))
    E, d, a, T, gamma = 37, 5, 2, 40, 0.97
    dev = RP.DeviceNStepReplay(n, gamma, E, d, a, capacity=4096,
                               norm_gamma=gamma if norm else None, g_max=10.0)
    packer = A.NStepPacker(n, gamma, E)
    nrm = A.ReturnStdNormalizer(gamma=gamma, g_max=10.0, n_envs=E) if norm else None
    codec = RP.RowCodec(d, a)
    host_rows = []
    obs = rng.normal(size=(E, d)).astype(np.float32)
    for _ in range(T):
        act = rng.normal(size=(E, a)).astype(np.float32)
        r = rng.normal(size=E).astype(np.float32)
        nxt = rng.normal(size=(E, d)).astype(np.float32)
        term = rng.random(E) < 0.05
        trunc = (rng.random(E) < 0.05) & ~term
        out = A.nstep_and_reward_norm(packer, nrm, obs, act, r.astype(np.float64), nxt, term,
                                      trunc)
        if out:
            o, ac, rr, no, te, nu = zip(*out)
            host_rows.append(codec.encode(np.stack(o), np.stack(ac), np.array(rr), np.stack(no),
                                          np.array(te), np.array(nu)))
        k = dev.push(obs, act, r, nxt, term, trunc)
        assert k == len(out)
        obs = np.where((term | trunc)[:, None], rng.normal(size=(E, d)).astype(np.float32), nxt)
    want = np.concatenate(host_rows)
    got = dev.rows(0, dev.head)
    assert got.shape == want.shape
    # obs / act / next_obs / flags bit-exact; rewards to f32 rounding of the f64 sums
    d2 = 2 * d + a + 1
    cols = [c for c in range(want.shape[1]) if c != d + a]
    np.testing.assert_array_equal(got[:, cols], want[:, cols])
    np.testing.assert_allclose(got[:, d + a], want[:, d + a], rtol=1e-6, atol=1e-6)
    assert np.all(got[:, d2] == want[:, d2])
    if norm:
        cnt, mean, _, std = dev.norm_stats()
        assert cnt == nrm.count
        assert mean == pytest.approx(nrm.mean, rel=1e-9, abs=1e-12)
        assert std == pytest.approx(nrm.std, rel=1e-9)


def test_device_nstep_rows_feed_sac_update():
    """Rows inserted by the device packer are sampled straight from HBM by
    sac_update (K6 gather with the window check)."""
    rng = np.random.default_rng(3)
    E, d, a = 64, 6, 2
    dev = RP.DeviceNStepReplay(2, 0.99, E, d, a, capacity=1024)
    for _ in range(6):
        dev.push(rng.normal(size=(E, d)), rng.normal(size=(E, a)), rng.normal(size=E),
                 rng.normal(size=(E, d)), rng.random(E) < 0.1, np.zeros(E, bool))
    from paper_2605_30313_b200 import tensornet as TN

    cfg = A.SacConfig(batch_size=32, policy_frequency=1)
    st = A.SacState.create(TN.init_params(TN.Arch(d, (32, 32), a), 0),
                           TN.init_params(TN.Arch(d + a, (32, 32), 1), 1),
                           TN.init_params(TN.Arch(d + a, (32, 32), 1), 2), cfg)
    idx = rng.integers(0, dev.head, size=32)
    out = A.sac_update(dev.sample(idx), st, cfg, A.DeviceRng(0))
    assert np.isfinite(out.extra["critic_loss"])
