"""Golden vectors of the FlashSAC collector transforms, produced by running the
UNMODIFIED reference (R:algos/estimators.py:125-224 ReturnStdNormalizer /
NStepPacker / nstep_and_reward_norm, R:replaypath/storage.py:17-46 RowCodec).

    python tests/golden/gen_nstep.py      (build container, /root/reference present)

Writes nstep.npz: for each case (n, norm) the per-step inputs of T steps of
E envs, the reference's emitted codec rows (env-major per step, concatenated)
with their per-step counts, and the normaliser's final (count, mean, m2, std).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from unilite.algos import NStepPacker, ReturnStdNormalizer, nstep_and_reward_norm  # noqa: E402
from unilite.replaypath import RowCodec  # noqa: E402

CASES = [(1, False), (3, False), (3, True), (5, True)]
E, D, A, T, GAMMA = 37, 5, 2, 40, 0.97


def run_case(n, norm):
    rng = np.random.default_rng(n * 10 + int(norm))
    packer = NStepPacker(n, GAMMA, E)
    nrm = ReturnStdNormalizer(gamma=GAMMA, g_max=10.0, n_envs=E) if norm else None
    codec = RowCodec(D, A)
    steps = {k: [] for k in ("obs", "act", "r", "next_obs", "term", "trunc")}
    rows, counts = [], []
    obs = rng.normal(size=(E, D)).astype(np.float32)
    for _ in range(T):
        act = rng.normal(size=(E, A)).astype(np.float32)
        r = rng.normal(size=E).astype(np.float32)
        nxt = rng.normal(size=(E, D)).astype(np.float32)
        term = rng.random(E) < 0.05
        trunc = (rng.random(E) < 0.05) & ~term
        for k, v in zip(steps, (obs, act, r, nxt, term, trunc)):
            steps[k].append(v)
        out = nstep_and_reward_norm(packer, nrm, obs, act, r.astype(np.float64), nxt, term, trunc)
        counts.append(len(out))
        if out:
            o, ac, rr, no, te, nu = zip(*out)
            rows.append(codec.encode(np.stack(o), np.stack(ac), np.array(rr), np.stack(no),
                                     np.array(te), np.array(nu)))
        obs = np.where((term | trunc)[:, None], rng.normal(size=(E, D)).astype(np.float32), nxt)
    res = {f"{k}": np.stack(v) for k, v in steps.items()}
    res["rows"] = np.concatenate(rows).astype(np.float32)
    res["counts"] = np.array(counts, np.int64)
    if nrm is not None:
        res["norm"] = np.array([nrm.count, nrm.mean, nrm.m2, nrm.std], np.float64)
    return res


def main():
    out = {}
    for n, norm in CASES:
        for k, v in run_case(n, norm).items():
            out[f"n{n}_{int(norm)}_{k}"] = v
    np.savez_compressed(OUT / "nstep.npz", **out)
    print("wrote", OUT / "nstep.npz")


if __name__ == "__main__":
    main()
