"""Device FlashSAC collector transforms: return-std
reward normalisation + n-step packing + replay insert on the GPU, against
golden vectors produced by the UNMODIFIED reference (tests/golden/gen_nstep.py:
R:algos/estimators.py:125-224 and RowCodec), both through DeviceNStepReplay
and through the reference-API wrappers (NStepPacker / ReturnStdNormalizer /
nstep_and_reward_norm)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import replaypath as RP  # noqa: E402

E, D, ACT, GAMMA = 37, 5, 2, 0.97
CASES = [(1, False), (3, False), (3, True), (5, True)]


def _case(golden, n, norm):
    g = golden("nstep")
    p = f"n{n}_{int(norm)}_"
    return {k[len(p):]: v for k, v in g.items() if k.startswith(p)}


def _check_rows(got, want):
    assert got.shape == want.shape
    # obs / act / next_obs / flags bit-exact; rewards to f32 rounding of the f64 sums
    cols = [c for c in range(want.shape[1]) if c != D + ACT]
    np.testing.assert_array_equal(got[:, cols], want[:, cols])
    np.testing.assert_allclose(got[:, D + ACT], want[:, D + ACT], rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("n,norm", CASES)
def test_device_nstep_matches_reference_goldens(golden, n, norm):
    c = _case(golden, n, norm)
    dev = RP.DeviceNStepReplay(n, GAMMA, E, D, ACT, capacity=4096,
                               norm_gamma=GAMMA if norm else None, g_max=10.0)
    for t in range(len(c["counts"])):
        k = dev.push(c["obs"][t], c["act"][t], c["r"][t], c["next_obs"][t], c["term"][t],
                     c["trunc"][t])
        assert k == c["counts"][t]
    _check_rows(dev.rows(0, dev.head), c["rows"])
    if norm:
        cnt, mean, m2, std = dev.norm_stats()
        ref = c["norm"]
        assert cnt == ref[0]
        assert mean == pytest.approx(ref[1], rel=1e-9, abs=1e-12)
        assert m2 == pytest.approx(ref[2], rel=1e-9)
        assert std == pytest.approx(ref[3], rel=1e-9)


@pytest.mark.parametrize("n,norm", CASES)
def test_reference_api_packer_matches_reference_goldens(golden, n, norm):
    """The drop-in NStepPacker / ReturnStdNormalizer / nstep_and_reward_norm
    (device state, reference tuples out) reproduce the reference's tuples."""
    c = _case(golden, n, norm)
    packer = A.NStepPacker(n, GAMMA, E)
    nrm = A.ReturnStdNormalizer(gamma=GAMMA, g_max=10.0, n_envs=E) if norm else None
    codec = RP.RowCodec(D, ACT)
    rows = []
    for t in range(len(c["counts"])):
        out = A.nstep_and_reward_norm(packer, nrm, c["obs"][t], c["act"][t],
                                      c["r"][t].astype(np.float64), c["next_obs"][t],
                                      c["term"][t], c["trunc"][t])
        assert len(out) == c["counts"][t]
        if out:
            o, ac, rr, no, te, nu = zip(*out)
            rows.append(codec.encode(np.stack(o), np.stack(ac), np.array(rr), np.stack(no),
                                     np.array(te), np.array(nu)))
    _check_rows(np.concatenate(rows), c["rows"])
    if norm:
        assert nrm.count == c["norm"][0]
        assert nrm.std == pytest.approx(c["norm"][3], rel=1e-9)


def test_return_std_normalizer_alone():
    """ReturnStdNormalizer.normalize on its own (R:algos/estimators.py:153-163):
    sequential Welford over the per-env discounted returns, clipped scaling."""
    rng = np.random.default_rng(5)
    n_envs, gamma, g_max = 9, 0.97, 5.0
    nrm = A.ReturnStdNormalizer(gamma=gamma, g_max=g_max, n_envs=n_envs)
    ret = np.zeros(n_envs)
    count, mean, m2 = 0.0, 0.0, 0.0
    for _ in range(30):
        r = rng.normal(size=n_envs)
        done = rng.random(n_envs) < 0.1
        got = nrm.normalize(r, done)
        ret = ret * gamma * (~done) + r
        for g in ret:  # the reference's sequential loop (known-answer restated here)
            count += 1
            dlt = g - mean
            mean += dlt / count
            m2 += dlt * (g - mean)
        std = 1.0 if count < 2 else np.sqrt(m2 / count)
        bound = (1.0 - gamma) * g_max
        np.testing.assert_allclose(got, np.clip(r / (std + 1e-8), -bound, bound), rtol=1e-6,
                                   atol=1e-7)
    # (the device merges each step's return statistics with Chan's formula)
    assert nrm.count == count and nrm.std == pytest.approx(std, rel=1e-7)


def test_collector_packers_match_reference_known_answers():
    # R:tests/test_estimators.py:246-262 boundary truncation
    g = 0.9
    p = A.NStepPacker(n=3, gamma=g, n_envs=1)
    z = np.zeros((1, 1))
    assert p.push(z, z, np.array([1.0]), z, np.array([False]), np.array([False])) == []
    rows = p.push(z + 1, z, np.array([2.0]), z + 9, np.array([True]), np.array([False]))
    assert len(rows) == 2 and rows[0][2] == pytest.approx(1.0 + g * 2.0) and rows[0][5] == 2
    # clip bound (1 - gamma) g_max (:303-312)
    norm = A.ReturnStdNormalizer(gamma=0.97, g_max=5.0, n_envs=2)
    rng = np.random.default_rng(5)
    for _ in range(50):
        out = norm.normalize(rng.normal(scale=3.0, size=2), np.zeros(2, bool))
        assert np.all(np.abs(out) <= (1 - 0.97) * 5.0 + 1e-7)  # (f32 codec rows)
    packer = A.NStepPacker(n=1, gamma=0.97, n_envs=1)
    rows = A.nstep_and_reward_norm(packer, A.ReturnStdNormalizer(0.97, 5.0, 1), np.zeros((1, 2)),
                                 np.zeros((1, 1)), np.array([100.0]), np.ones((1, 2)),
                                 np.array([False]), np.array([False]))
    assert len(rows) == 1 and abs(rows[0][2]) <= (1 - 0.97) * 5.0 + 1e-7


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
