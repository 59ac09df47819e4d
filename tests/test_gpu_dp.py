"""The data-parallel PPO update path on one GPU: a 1-rank
NCCL process group with the DP step path forced, so the 20 x (step_grads ->
NCCL all-reduce -> step_apply) sequence runs exactly as on 8 GPUs -- captured
as one CUDA graph with the NCCL all-reduces inside -- and must equal the
host-driven loop bit for bit; the global advantage statistics of "local"
shards come from all-reduced sums.  (Multi-rank NCCL needs one GPU per rank;
the multi-rank host logic is covered by the gloo tests and the thread-emulated
2-rank tests.)"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import _dist  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
from helpers import _synthetic  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture
def nccl_one_rank():
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    old = P.get_precision()
    P.set_precision("bf16")
    _dist.force_dp(True)
    _dist.set_segment_mode("local")
    yield
    _dist.force_dp(False)
    _dist.set_segment_mode("replicated")
    P.set_precision(old)
    os.environ.pop("UL_DP_GRAPH", None)
    dist.destroy_process_group()


def _run(segd, actor, critic, updates=3):
    T, N = segd["rewards"].shape
    od, ad, cd = segd["obs"].shape[2], segd["actions"].shape[2], segd["critic_obs"].shape[2]
    hid = tuple(w.shape[0] for w, _ in actor.layers[:-1])
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(cd, hid, 1), critic.flat()))
    opt = A.AcOpt.for_params(params, 1e-3)
    rng = A.DeviceRng(5)
    stats = []
    for _ in range(updates):
        seg = A.RolloutSegment(**segd)
        seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated,
                                            seg.truncated, seg.bootstrap_value, 0.99, 0.95,
                                            truncation_values=seg.truncation_values)
        stats.append(A.ppo_update(seg, params, opt, A.PpoConfig(), rng))
    return params, stats, opt


def test_dp_update_graph_with_nccl_equals_host_loop(nccl_one_rank):
    segd, actor, critic = _synthetic(24, 512, 48, 48, 12, (256, 128, 128), seed=2)
    out = {}
    for flag in ("0", "1"):
        os.environ["UL_DP_GRAPH"] = flag
        out[flag] = _run(segd, actor, critic)
    (p0, s0, o0), (p1, s1, o1) = out["0"], out["1"]
    np.testing.assert_array_equal(p0.actor.flat(), p1.actor.flat())
    np.testing.assert_array_equal(p0.critic.flat(), p1.critic.flat())
    assert [s.policy_loss for s in s0] == [s.policy_loss for s in s1]
    assert o1.actor.t == o1.critic.t == 3 * 20


def test_dp_path_matches_single_gpu_plan(nccl_one_rank):
    """The forced DP path (global advantage sums all-reduced, per-step NCCL)
    tracks the single-GPU update graph (same math, different launch
    structure): bf16 parameter deltas within 2 % / losses within 1e-3."""
    segd, actor, critic = _synthetic(24, 512, 48, 48, 12, (256, 128, 128), seed=3)
    pd, sd, _ = _run(segd, actor, critic, updates=2)
    _dist.force_dp(False)
    _dist.set_segment_mode("replicated")
    ps, ss, _ = _run(segd, actor, critic, updates=2)
    for a, b, init in ((pd.actor, ps.actor, actor), (pd.critic, ps.critic, critic)):
        d1 = a.flat().astype(np.float64) - init.flat()
        d2 = b.flat().astype(np.float64) - init.flat()
        assert np.linalg.norm(d1 - d2) / np.linalg.norm(d2) < 0.02
    for x, y in zip(sd, ss):
        assert abs(x.policy_loss - y.policy_loss) < 1e-3
        assert abs(x.value_loss - y.value_loss) < 1e-3 * max(1.0, abs(y.value_loss))
