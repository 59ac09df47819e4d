"""B200-native UniLab learner hot path (drop-in for the reference ``unilite``
learner API).  Compute runs in libunilite_b200.so (sm_100a); PyTorch is the
host shell for HBM allocations, streams and torch.distributed."""

__version__ = "0.1.0"


def set_precision(gemm: str) -> None:
    """Select the MLP GEMM back end: "tf32" (default; tcgen05 tensor cores,
    fp32 storage, ~1e-3 relative GEMM error), "bf16" (tcgen05 kind::f16 with
    bf16 activations inside the fused PPO/APPO update plans, fp32 parameters,
    gradients and optimizer; the north-star 1e-2 tolerance of bf16 GEMM paths)
    "fp32" (SIMT FFMA, exact fp32: the reference-parity configuration,
    R:tensornet/mlp.py is float32) or "tf32x3" (the same fp32 parity on the
    tcgen05 tensor cores: every GEMM as one tf32 GEMM over 3xTF32-split
    operands, hi*hi + hi*lo + lo*hi).  Paths that need input gradients (SAC's
    actor step, the module-level MLP backward) run "bf16" as "tf32"."""
    from . import _lib

    if gemm not in ("fp32", "tf32", "bf16", "tf32x3"):
        raise ValueError("gemm precision must be 'fp32', 'tf32', 'bf16' or 'tf32x3'")
    _lib._PRECISION["gemm"] = gemm


def get_precision() -> str:
    from . import _lib

    return _lib._PRECISION["gemm"]
