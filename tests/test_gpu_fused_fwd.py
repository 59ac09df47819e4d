"""Fused hidden-layer forward chain (csrc/fused_mlp.cu, bf16): one persistent
launch runs every hidden layer of a 128-row tile with the activation tile
kept in shared memory.  It computes the same MMAs in the same K order and the
same bias + ELU epilogue as the layer-by-layer tcgen05 path, so a bf16 PPO
update through it must equal the layer-by-layer update BIT FOR BIT (the
layer-by-layer path runs in a child process with UL_FUSED_FWD=0)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [  # T, N, obs, hidden, epochs, minibatches
    (24, 4096, 235, (512, 256, 128), 2, 4),  # cfg2 shape (24,576-row minibatches)
    (8, 256, 48, (256, 128, 128), 1, 2),     # cfg1 shape
    (7, 111, 64, (128, 64), 1, 1),           # 777 rows: ragged tile tail
    (4, 300, 32, (128, 128, 128, 128), 1, 3),  # four hidden layers
    (4, 512, 512, (512, 512), 1, 2),         # widest input and hidden layers
]

_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, "tests")
import paper_2605_30313_b200 as P
from paper_2605_30313_b200 import algos as A, tensornet as TN
from oracle.port import philox_stream
from helpers import _synthetic
P.set_precision("bf16")
(T, N, od, hid, ep, mb), out = json.loads(sys.argv[1])
segd, actor, critic = _synthetic(T, N, od, od, 12, tuple(hid), seed=T + N)
params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, tuple(hid), 12), actor.flat()),
                    TN.ModelParams.from_numpy(TN.Arch(od, tuple(hid), 1), critic.flat()))
seg = A.RolloutSegment(**segd)
seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                                    seg.bootstrap_value, 0.99, 0.95,
                                    truncation_values=seg.truncation_values)
st = A.ppo_update(seg, params, A.AcOpt.for_params(params, 1e-3),
                  A.PpoConfig(epochs=ep, minibatches=mb), philox_stream(3, "update"))
np.savez(out, actor=params.actor.flat(), critic=params.critic.flat(),
         stats=np.array([st.policy_loss, st.value_loss, st.kl, st.entropy]))
"""


def _run(case, fused, tmp):
    out = os.path.join(tmp, f"{'f' if fused else 'l'}.npz")
    env = dict(os.environ, UL_FUSED_FWD="1" if fused else "0", PYTHONPATH=ROOT)
    subprocess.run([sys.executable, "-c", _CHILD, json.dumps([case, out])], env=env,
                   cwd=ROOT, check=True, timeout=300)
    return np.load(out)


@pytest.mark.parametrize("case", CASES)
def test_fused_forward_bf16_ppo_update_bit_exact(case, tmp_path):
    """A whole bf16 PPO update (every forward of both networks through the
    fused chain) against the same update on the layer-by-layer path."""
    a = _run(case, True, str(tmp_path))
    b = _run(case, False, str(tmp_path))
    for k in ("actor", "critic", "stats"):
        assert np.array_equal(a[k], b[k]), (k, float(np.max(np.abs(a[k] - b[k]))))


def _run_env(case, env_extra, tmp, tag):
    out = os.path.join(tmp, f"{tag}.npz")
    env = dict(os.environ, PYTHONPATH=ROOT, **env_extra)
    subprocess.run([sys.executable, "-c", _CHILD, json.dumps([case, out])], env=env,
                   cwd=ROOT, check=True, timeout=300)
    return np.load(out)


@pytest.mark.parametrize("case", CASES[:4])
def test_chained_forward_bf16_ppo_update_bit_exact(case, tmp_path):
    """Opt-in chained hidden layers (UL_CHAIN_FWD=1, csrc/gemm_tc.cu chain
    mode: one launch, whole row chains per CTA, each layer's tiles waiting for
    the CTA's own stores of the layer below) against one launch per layer."""
    a = _run_env(case, {"UL_CHAIN_FWD": "1", "UL_FUSED_FWD": "0"}, str(tmp_path), "c")
    b = _run_env(case, {"UL_CHAIN_FWD": "0", "UL_FUSED_FWD": "0"}, str(tmp_path), "l")
    for k in ("actor", "critic", "stats"):
        assert np.array_equal(a[k], b[k]), (k, float(np.max(np.abs(a[k] - b[k]))))
