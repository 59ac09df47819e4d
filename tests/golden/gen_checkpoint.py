"""Write a checkpoint with the UNMODIFIED reference's save_checkpoint
(R:tensornet/checkpoint.py) so the B200 loader is pinned to its file format.

    python tests/golden/gen_checkpoint.py      (build container only)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from unilite.tensornet import Arch, Normalizer, init_params, save_checkpoint  # noqa: E402

OUT = Path(__file__).resolve().parent
arch = Arch(input_dim=6, hidden_dims=(8, 4), output_dim=2)
params = init_params(arch, seed=3)
params.version = 17
norm = Normalizer(dim=6)
norm.update(np.random.default_rng(0).normal(size=(32, 6)))
save_checkpoint(OUT / "ckpt_ref.npz", params, norm)
flat = np.concatenate([np.concatenate([w.reshape(-1), b]) for w, b in params.layers]
                      + [params.log_std])
np.savez(OUT / "ckpt_ref_expect.npz", flat=flat.astype(np.float32), mean=norm.mean, var=norm.var,
         count=np.array(norm.count))
