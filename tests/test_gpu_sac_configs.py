"""SAC parity at the benchmarked shapes (BASELINE configs[2] / configs[3]).

* cfg3 FastSAC: obs 96 / act 23, twin critics 119-1024-512-256-1 with
  LayerNorm, actor 96-512-256-128-23, batch 8192, SacConfig defaults
  (policy_frequency 4: the 4th update takes the actor / alpha step).
* cfg4 FlashSAC: batch 32,768, critics 119-1024-1024-1024-1, actor
  96-512-512-23, flashsac_defaults (tau 0.01, policy_frequency 2).

Four consecutive updates on one batch -- the learner tick's
updates_per_step loop, run as ONE CUDA graph by ``sac_updates`` -- on the
reference's learner noise stream, against the float32 oracle (the
reference's own arithmetic; its float32-vs-float64 gap at these shapes is
<= 5e-5, tools/sac_probe.py).  Per network Delta-theta bounds:

  fp32 (SIMT)   rel <= 1e-3,  cos >= 0.99999   (measured <= 5e-5)
  tf32          rel <= 0.10,  cos >= 0.995     (measured <= 0.044 / 0.9990)
  bf16 critics  rel <= 0.10,  cos >= 0.995     (measured <= 0.042 / 0.9991)
  bf16 actor    rel <= 0.15,  cos >= 0.99      (measured 0.105 / 0.9945 at cfg3:
                                                one actor step on bf16 dQ/da)

and every loss / alpha of the trajectory within 1e-2 * max(1, |ref|) on the
tensor-core paths (the north-star bf16 tolerance), 1e-5 on fp32.  The graph
run is also bit-identical to the same updates issued one sac_update at a time.
"""

import numpy as np
import pytest

from oracle import port as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402

CFGS = {
    # (obs, act, critic hidden, actor hidden, LN, batch, flash)
    "cfg3": (96, 23, (1024, 512, 256), (512, 256, 128), True, 8192, False),
    "cfg4": (96, 23, (1024, 1024, 1024), (512, 512), False, 32768, True),
}
U = 4


@pytest.fixture(autouse=True)
def _restore_precision():
    old = P.get_precision()
    yield
    P.set_precision(old)


def _batch(B, od, ad, seed=3):
    rng = np.random.default_rng(seed)
    return dict(obs=rng.normal(size=(B, od)).astype(np.float32),
                action=np.tanh(rng.normal(size=(B, ad))).astype(np.float32),
                reward=rng.normal(size=B).astype(np.float32),
                next_obs=rng.normal(size=(B, od)).astype(np.float32),
                terminated=rng.random(B) < 0.01, n_used=np.ones(B, np.int64))


def _nets(name):
    od, ad, ch, ah, ln, B, flash = CFGS[name]
    a0 = O.net_init((od, *ah, ad), 0)
    q0 = [O.net_init((od + ad, *ch, 1), s, layer_norm=ln) for s in (1, 2)]
    return a0, q0


_ORACLE = {}


def _oracle(name):
    if name not in _ORACLE:
        from threadpoolctl import threadpool_limits

        od, ad, ch, ah, ln, B, flash = CFGS[name]
        a0, q0 = _nets(name)
        cfg = A.flashsac_defaults() if flash else A.SacConfig()
        ocfg = O.SacCfg(tau=cfg.tau, policy_frequency=cfg.policy_frequency)
        st = O.SacSt.create(a0.clone(), q0[0].clone(), q0[1].clone(), ocfg)
        rng = O.philox_stream(1, "learner")
        with threadpool_limits(limits=None):
            traj = [O.sac_update(_batch(B, od, ad), st, ocfg, rng) for _ in range(U)]
        _ORACLE[name] = (st, traj)
    return _ORACLE[name]


def _state(name, cfg):
    od, ad, ch, ah, ln, B, flash = CFGS[name]
    a0, q0 = _nets(name)
    qa = TN.Arch(od + ad, ch, 1, layer_norm=ln)
    return A.SacState.create(TN.ModelParams.from_numpy(TN.Arch(od, ah, ad), a0.flat()),
                             TN.ModelParams.from_numpy(qa, q0[0].flat()),
                             TN.ModelParams.from_numpy(qa, q0[1].flat()), cfg)


@pytest.mark.parametrize("name,prec", [("cfg3", "fp32"), ("cfg3", "tf32"), ("cfg3", "bf16"),
                                       ("cfg4", "bf16"), ("cfg4", "tf32")])
def test_sac_updates_at_benchmark_shapes(name, prec):
    od, ad, ch, ah, ln, B, flash = CFGS[name]
    ost, otraj = _oracle(name)
    a0, q0 = _nets(name)
    P.set_precision(prec)
    cfg = A.flashsac_defaults() if flash else A.SacConfig()
    st = _state(name, cfg)
    stats = A.sac_updates(_batch(B, od, ad), st, cfg, O.philox_stream(1, "learner"), U)
    bounds = {"fp32": {"actor": (1e-3, 0.99999), "q": (1e-3, 0.99999)},
              "tf32": {"actor": (0.10, 0.995), "q": (0.10, 0.995)},
              "bf16": {"actor": (0.15, 0.99), "q": (0.10, 0.995)}}[prec]
    for key, mine, ref, init in (("actor", st.params.actor, ost.actor, a0),
                                 ("q", st.params.q1, ost.q1, q0[0]),
                                 ("q", st.params.q2, ost.q2, q0[1])):
        d = mine.flat().astype(np.float64) - init.flat()
        r = ref.flat().astype(np.float64) - init.flat()
        rel = np.linalg.norm(d - r) / np.linalg.norm(r)
        cos = d @ r / (np.linalg.norm(d) * np.linalg.norm(r))
        rmax, cmin = bounds[key]
        assert rel <= rmax and cos >= cmin, (name, prec, key, rel, cos)
    tol = 1e-5 if prec == "fp32" else 1e-2
    for u, (got, want) in enumerate(zip(stats, otraj)):
        assert set(got.extra) == set(want), (u, got.extra, want)
        for k, v in want.items():
            assert abs(got.extra[k] - v) <= tol * max(1.0, abs(v)), (u, k, got.extra[k], v)
    assert st.update_count == U
    assert st.params.log_alpha == pytest.approx(ost.log_alpha, abs=1e-6)


def test_sac_graph_run_equals_sequential_updates():
    """One sac_updates(..., 4) graph launch == four sac_update calls, bit for bit
    (bf16 cfg3: LayerNorm critics, the actor step on the 4th update)."""
    od, ad, ch, ah, ln, B, flash = CFGS["cfg3"]
    P.set_precision("bf16")
    cfg = A.SacConfig()
    s1, s2 = _state("cfg3", cfg), _state("cfg3", cfg)
    batch = _batch(B, od, ad)
    A.sac_updates(batch, s1, cfg, O.philox_stream(2, "learner"), U)
    rng = O.philox_stream(2, "learner")
    for _ in range(U):
        A.sac_update(batch, s2, cfg, rng)
    for a, b in ((s1.params.actor, s2.params.actor), (s1.params.q1, s2.params.q1),
                 (s1.params.q2_targ, s2.params.q2_targ)):
        np.testing.assert_array_equal(a.flat(), b.flat())
    assert s1.params.log_alpha == s2.params.log_alpha
    assert s1.actor_opt.t == s2.actor_opt.t == 1 and s1.q1_opt.t == 4
