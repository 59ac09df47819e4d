"""The critic grouping modes of the SAC plan (csrc/sac.cu sac_group) are
the same update: UL_SAC_GROUP=0 (one network per launch), 1 (the default:
the twin critics grouped per layer, one batched dW) and 2 (the target and
online critics' forwards as one 4-network pass with separate activation
caches), after four cfg3-shaped bf16 updates (LayerNorm critics, the
actor / alpha step on the 4th): 2 is bit-identical to 1, and 1 differs from
0 only by the split-K summation order of the batched dW.  The flag is read
once per process, so every mode runs in its own interpreter."""

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

_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2605_30313_b200 as P
from paper_2605_30313_b200 import algos as A
from oracle import port as O
import test_gpu_sac_configs as C
P.set_precision("bf16")
C.CFGS["small"] = (96, 23, (1024, 512, 256), (512, 256, 128), True, 2048, False)
cfg = A.SacConfig()
st = C._state("small", cfg)
od, ad = 96, 23
stats = A.sac_updates(C._batch(2048, od, ad), st, cfg, O.philox_stream(3, "learner"), 4)
np.savez({out!r}, actor=st.params.actor.flat(), q1=st.params.q1.flat(), q2=st.params.q2.flat(),
         q1t=st.params.q1_targ.flat(), q2t=st.params.q2_targ.flat(),
         la=np.float64(st.params.log_alpha),
         loss=np.array([s.extra.get("critic_loss", np.nan) for s in stats]))
"""


def _run(mode, tmp_path):
    out = str(tmp_path / f"g{mode}.npz")
    env = dict(os.environ, UL_SAC_GROUP=str(mode))
    code = _SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def test_sac_critic_grouping_modes(tmp_path):
    runs = {m: _run(m, tmp_path) for m in (0, 1, 2)}
    keys = ("actor", "q1", "q2", "q1t", "q2t", "la", "loss")
    # 2 vs 1: only the forward launches are regrouped -- bit-identical
    for k in keys:
        np.testing.assert_array_equal(runs[1][k], runs[2][k], err_msg=k)
    # 1 vs 0: the batched dW of the twin critics has twice the tiles of one
    # critic's, so run_deferred_dw_gemms picks half the split-K count (one
    # persistent wave) -- a different fixed summation order, the same update
    for k in keys:
        a, b = runs[0][k].astype(np.float64), runs[1][k].astype(np.float64)
        tol = 1e-3 * np.maximum(1.0, np.abs(a)) if k == "loss" else 2e-3
        assert np.all(np.abs(a - b) <= tol), (k, float(np.abs(a - b).max()))
