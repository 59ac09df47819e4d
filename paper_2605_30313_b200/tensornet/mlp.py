"""Device-resident dense ELU networks (mirror of R:tensornet/mlp.py).

Parameters live in ONE flat float32 HBM buffer in the reference's
``ModelParams.flat`` order (R:tensornet/mlp.py:53-57): W0 (out x in), b0, W1,
b1, ..., log_std.  ``layers`` / ``log_std`` are views into it; ``flat()`` is the
only D2H.  forward/backward call the fp32 GEMM kernels of libunilite_b200
(ul_mlp_forward / ul_mlp_backward).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _dev, _lib


@dataclass(frozen=True)
class Arch:
    """R:tensornet/mlp.py:16-33."""

    input_dim: int
    hidden_dims: tuple = ()
    output_dim: int = 1
    activation: str = "elu"
    # extension (not in the reference): LayerNorm (gain, shift) between each
    # hidden layer's affine map and its ELU -- cfg3's FastSAC critics
    layer_norm: bool = False

    def __post_init__(self) -> None:
        object.__setattr__(self, "hidden_dims", tuple(int(h) for h in self.hidden_dims))
        dims = (self.input_dim, *self.hidden_dims, self.output_dim)
        if any(d <= 0 for d in dims):
            raise ValueError(f"all layer dims must be positive, got {dims}")
        if self.activation != "elu":
            raise ValueError("only elu is supported")
        if len(dims) - 1 > _lib.UL_MAX_LAYERS:
            raise ValueError(f"at most {_lib.UL_MAX_LAYERS} layers")

    @property
    def dims(self) -> tuple:
        return (self.input_dim, *self.hidden_dims, self.output_dim)

    @property
    def layer_dims(self) -> list:
        d = self.dims
        return [(d[i + 1], d[i]) for i in range(len(d) - 1)]

    def desc(self) -> _lib.NetDesc:
        return _lib.NetDesc.of(self.dims, self.layer_norm)

    @property
    def param_count(self) -> int:
        ln = 2 * sum(self.hidden_dims) if self.layer_norm else 0
        return sum(o * i + o for o, i in self.layer_dims) + ln + self.output_dim


def _views(buf: torch.Tensor, arch: Arch, with_ln: bool = False):
    layers, lns, off = [], [], 0
    nl = len(arch.layer_dims)
    for k, (o, i) in enumerate(arch.layer_dims):
        w = buf[off:off + o * i].view(o, i)
        off += o * i
        b = buf[off:off + o]
        off += o
        layers.append((w, b))
        if arch.layer_norm and k < nl - 1:
            lns.append((buf[off:off + o], buf[off + o:off + 2 * o]))
            off += 2 * o
    if with_ln:
        return layers, buf[off:off + arch.output_dim], lns
    return layers, buf[off:off + arch.output_dim]


class _FlatRecord:
    """Shared machinery of ModelParams and Grads: one flat device vector."""

    def __init__(self, buf: torch.Tensor, arch: Arch):
        if buf.numel() != arch.param_count:
            raise ValueError("flat buffer size does not match the architecture")
        self.buf = buf
        self.arch = arch

    @property
    def layers(self):
        return _views(self.buf, self.arch)[0]

    @property
    def log_std(self) -> torch.Tensor:
        return _views(self.buf, self.arch)[1]

    @property
    def layer_norms(self):
        """(gain, shift) per hidden layer when arch.layer_norm (else [])."""
        return _views(self.buf, self.arch, with_ln=True)[2]

    def flat(self) -> np.ndarray:
        """All parameters (incl. log_std) as one host float vector (D2H)."""
        return _dev.to_numpy(self.buf)


class ModelParams(_FlatRecord):
    """Weights, biases and log_std (R:tensornet/mlp.py:36-76)."""

    def __init__(self, buf: torch.Tensor, arch: Arch, version: int = 0):
        super().__init__(buf, arch)
        self.version = version

    def copy(self) -> "ModelParams":
        buf = torch.empty_like(self.buf)
        _lib.call("ul_memcpy_async", _dev.ptr(buf), _dev.ptr(self.buf),
                  self.buf.numel() * self.buf.element_size(), _dev.stream())
        return ModelParams(buf, self.arch, self.version)

    def with_flat(self, vec) -> "ModelParams":
        vec = np.asarray(vec, dtype=np.float32).reshape(-1)
        if vec.size != self.buf.numel():
            raise ValueError("flat vector length mismatch")
        out = torch.empty_like(self.buf)
        _dev.h2d(out, vec)
        return ModelParams(out, self.arch, self.version)

    @classmethod
    def from_numpy(cls, arch: Arch, flat, version: int = 0) -> "ModelParams":
        _dev.require_cuda()
        vec = np.ascontiguousarray(np.asarray(flat, dtype=np.float32).reshape(-1))
        buf = torch.empty(vec.size, dtype=torch.float32, device="cuda")
        _dev.h2d(buf, vec)
        return cls(buf, arch, version)

    @classmethod
    def from_reference(cls, ref) -> "ModelParams":
        """Adopt a reference-shaped record (numpy layers / log_std / arch)."""
        a = ref.arch
        arch = Arch(a.input_dim, tuple(a.hidden_dims), a.output_dim)
        return cls.from_numpy(arch, ref.flat(), getattr(ref, "version", 0))


class Grads(_FlatRecord):
    """Gradient record congruent to ModelParams (R:tensornet/mlp.py:79-113)."""

    @classmethod
    def zeros_like(cls, params: ModelParams) -> "Grads":
        return cls(_dev.zeros_like(params.buf), params.arch)

    def add_(self, other: "Grads") -> None:
        self.buf.add_(other.buf)

    def scale_(self, factor: float) -> None:
        self.buf.mul_(float(factor))

    def global_norm(self) -> float:
        from .adam import clip_global_norm

        return clip_global_norm([self], 0.0)


def init_params(arch: Arch, seed: int, init_noise_std: float = 1.0,
                dtype=np.float32) -> ModelParams:
    """Scaled-uniform fan-in init drawn on the host exactly like the reference
    (default_rng(seed) layer by layer, R:tensornet/mlp.py:116-131), then
    uploaded once.  The device format is float32."""
    if np.dtype(dtype) != np.float32:
        raise ValueError("device parameters are float32")
    rng = np.random.default_rng(seed)
    parts = []
    nl = len(arch.layer_dims)
    for k, (out_dim, in_dim) in enumerate(arch.layer_dims):
        bound = np.sqrt(1.0 / in_dim)
        parts.append(rng.uniform(-bound, bound, (out_dim, in_dim)).astype(np.float32).ravel())
        parts.append(np.zeros(out_dim, np.float32))
        if arch.layer_norm and k < nl - 1:  # gain 1, shift 0
            parts.append(np.ones(out_dim, np.float32))
            parts.append(np.zeros(out_dim, np.float32))
    parts.append(np.full(arch.output_dim, np.log(init_noise_std), dtype=np.float32))
    return ModelParams.from_numpy(arch, np.concatenate(parts))


@dataclass
class ForwardCache:
    """Activations of one forward pass (R:tensornet/mlp.py:146-150)."""

    x: torch.Tensor
    acts: torch.Tensor
    out: torch.Tensor
    rows: int
    pre_acts: list = field(default_factory=list)
    wstage: torch.Tensor = None
    backend: int = None


def forward(params: ModelParams, x) -> tuple:
    """Batched forward on the device (R:tensornet/mlp.py:153-172)."""
    arch = params.arch
    if isinstance(x, torch.Tensor) and x.dim() == 2 and x.is_cuda:
        xd = x if x.dtype == torch.float32 and x.stride(1) == 1 else _dev.to_device_f32(x)
    else:
        a = np.asarray(x)
        if a.ndim != 2:
            raise ValueError(f"obs shape {a.shape} incompatible with input_dim {arch.input_dim}")
        xd = _dev.to_device_f32(a)
    if xd.dim() != 2 or xd.shape[1] != arch.input_dim:
        raise ValueError(f"obs shape {tuple(xd.shape)} incompatible with input_dim "
                         f"{arch.input_dim}")
    rows = xd.shape[0]
    desc = arch.desc()
    acts = torch.empty(max(_lib.lib().ul_mlp_act_floats(desc, rows), 1), dtype=torch.float32,
                       device=xd.device)
    out = torch.empty((rows, arch.output_dim), dtype=torch.float32, device=xd.device)
    be, ws = _staged(params)
    _lib.call("ul_mlp_forward", desc, _dev.ptr(params.buf), _dev.ptr(ws), be, _dev.ptr(xd),
              xd.stride(0), rows, _dev.ptr(acts), _dev.ptr(out), arch.output_dim, _dev.stream())
    return out, ForwardCache(xd, acts, out, rows, wstage=ws, backend=be)


def _staged(params: ModelParams):
    """(backend, staged weights) for one MLP pass: the tensor-core path reads
    W through 16-byte-aligned padded rows restaged from the live parameters."""
    be = _lib.gemm_backend(input_grads=True)
    if be not in (_lib.UL_GEMM_TF32, _lib.UL_GEMM_TF32X3):
        return be, None
    desc = params.arch.desc()
    ws = torch.empty(max(_lib.lib().ul_mlp_wstage_floats(desc), 1), dtype=torch.float32,
                     device=params.buf.device)
    _lib.call("ul_stage_weights", desc, _dev.ptr(params.buf), _dev.ptr(ws), _dev.stream())
    return be, ws


def backward(params: ModelParams, cache: ForwardCache, dout) -> tuple:
    """Exact reverse-mode gradients (R:tensornet/mlp.py:175-198).  dout is
    cast to float32 like the reference casts it to the parameter dtype."""
    arch = params.arch
    d = dout if isinstance(dout, torch.Tensor) else np.asarray(dout)
    if tuple(d.shape) != (cache.rows, arch.output_dim):
        raise ValueError("upstream grad shape does not match cached forward")
    dd = _dev.to_device_f32(d, ld=arch.output_dim).contiguous()
    rows = cache.rows
    desc = arch.desc()
    grads = Grads(torch.empty_like(params.buf), arch)
    dx = torch.empty((rows, arch.input_dim), dtype=torch.float32, device=params.buf.device)
    work = torch.empty(max(_lib.lib().ul_mlp_bwd_work_floats(desc, rows), 1),
                       dtype=torch.float32, device=params.buf.device)
    be, ws = (cache.backend, cache.wstage) if cache.backend is not None else _staged(params)
    _lib.call("ul_mlp_backward", desc, _dev.ptr(params.buf), _dev.ptr(ws), be,
              _dev.ptr(cache.x), cache.x.stride(0), 0, rows, _dev.ptr(cache.acts), _dev.ptr(dd),
              arch.output_dim, _dev.ptr(grads.buf), _dev.ptr(dx), arch.input_dim,
              _dev.ptr(work), _dev.stream())
    return dx, grads


def value_forward(params: ModelParams, x) -> tuple:
    """Scalar-output critic forward (R:tensornet/mlp.py:201-204)."""
    out, cache = forward(params, x)
    return out[:, 0], cache
