"""ctypes binding of libunilite_b200.so (the C ABI in include/unilite_b200.h).

This is the whole Python<->native boundary.  There is no CPU fallback: if the
library is missing or no CUDA device is present, every entry point raises.
Status codes map to the reference's exception types.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import DivergenceError, SlotStateError

LIB_PATH = Path(__file__).resolve().with_name("libunilite_b200.so")

UL_MAX_SEG = 4
UL_MAX_LAYERS = 8
UL_PREP_BLOCKS = 296
UL_MAX_ACT = 64
UL_GEMM_FP32 = 0
UL_GEMM_TF32 = 1
UL_GEMM_BF16 = 2
UL_GEMM_TF32X3 = 3

# Process-wide GEMM back end of the MLP passes ("fp32": SIMT exact-fp32 parity
# path; "tf32": tcgen05 tensor cores).  See paper_2605_30313_b200.set_precision.
_PRECISION = {"gemm": "tf32"}


def gemm_backend(input_grads: bool = False) -> int:
    """C back end code of the selected precision; `input_grads` callers (which
    need dX through the network) get tf32 in place of bf16."""
    g = _PRECISION["gemm"]
    if g == "bf16":
        return UL_GEMM_TF32 if input_grads else UL_GEMM_BF16
    if g == "tf32x3":
        return UL_GEMM_TF32X3
    return UL_GEMM_TF32 if g == "tf32" else UL_GEMM_FP32

vp = C.c_void_p
i64 = C.c_int64
i32 = C.c_int32
f64 = C.c_double


class NetDesc(C.Structure):
    _fields_ = [("n_layers", i32), ("dims", i32 * (UL_MAX_LAYERS + 1)), ("layer_norm", i32)]

    @classmethod
    def of(cls, dims, layer_norm: bool = False) -> "NetDesc":
        d = cls()
        d.n_layers = len(dims) - 1
        for i, x in enumerate(dims):
            d.dims[i] = int(x)
        d.layer_norm = int(bool(layer_norm))
        return d


class OptCtl(C.Structure):
    _fields_ = [
        ("lr", f64 * UL_MAX_SEG), ("beta1", f64), ("beta2", f64), ("eps", f64),
        ("max_norm", f64), ("t", i64 * UL_MAX_SEG), ("norm", f64), ("factor", f64),
        ("sumsq", f64 * UL_MAX_SEG), ("seg_bad", i32 * UL_MAX_SEG),
        ("seg_update", i32 * UL_MAX_SEG), ("loss_bad", i32), ("diverged", i32),
        ("steps", i32), ("fail_step", i32), ("ticket", C.c_uint32), ("pad0", i32),
        ("part", (f64 * UL_MAX_SEG) * UL_PREP_BLOCKS),
        ("part_bad", (i32 * UL_MAX_SEG) * UL_PREP_BLOCKS),
    ]


class PpoPlanDesc(C.Structure):
    _fields_ = [
        ("actor", NetDesc), ("critic", NetDesc), ("rows", i64), ("ld_obs", i64),
        ("ld_cobs", i64), ("ld_act", i64), ("epochs", i32), ("minibatches", i32),
        ("clip_param", f64), ("entropy_coef", f64), ("value_loss_coef", f64),
        ("use_clipped_value_loss", i32), ("max_grad_norm", f64), ("world_size", i32),
        ("rank", i32), ("raw_advantages", i32), ("local_shards", i32), ("gemm_backend", i32),
        ("obs_bf16", i32),
    ]


class PpoBindings(C.Structure):
    _fields_ = [(n, vp) for n in ("obs", "cobs", "act", "blogp", "adv", "ret", "oldv",
                                  "actor_params", "critic_params", "actor_m", "actor_v",
                                  "critic_m", "critic_v", "perm", "reduce_buf")]


class SacCtl(C.Structure):
    _fields_ = [(n, f64) for n in ("log_alpha", "a_m", "a_v", "a_t", "alpha_lr", "critic_loss",
                                   "actor_loss", "alpha_loss", "logp_sum")] + \
               [("diverged", i32), ("fail_update", i32)]


class SacPlanDesc(C.Structure):
    _fields_ = [("actor", NetDesc), ("critic", NetDesc), ("batch", i64), ("obs_dim", i32),
                ("act_dim", i32), ("gamma", f64), ("tau", f64), ("target_entropy", f64),
                ("max_grad_norm", f64), ("gemm_backend", i32), ("world_size", i32)]


class SacBindings(C.Structure):
    _fields_ = [(n, vp) for n in ("actor", "actor_m", "actor_v", "q1", "q1_m", "q1_v", "q2",
                                  "q2_m", "q2_v", "q1t", "q2t", "critic_red", "actor_red")]


class PpoResult(C.Structure):
    _fields_ = [("policy_loss", f64), ("value_loss", f64), ("entropy", f64), ("kl", f64),
                ("grad_norm", f64), ("t_actor", i64), ("t_critic", i64), ("diverged", i32),
                ("fail_step", i32)]


# name -> (restype, argtypes)
_PROTOS = {
    "ul_last_error": (C.c_char_p, []),
    "ul_version": (C.c_int, []),
    "ul_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ul_stream_sync": (C.c_int, [vp]),
    "ul_memcpy_async": (C.c_int, [vp, vp, i64, vp]),
    "ul_memset_async": (C.c_int, [vp, C.c_int, i64, vp]),
    "ul_memcpy2d_async": (C.c_int, [vp, i64, vp, i64, i64, i64, vp]),
    "ul_host_alloc_pinned": (C.c_int, [C.POINTER(vp), i64]),
    "ul_host_free_pinned": (C.c_int, [vp]),
    "ul_event_create": (C.c_int, [C.POINTER(vp)]),
    "ul_event_destroy": (C.c_int, [vp]),
    "ul_event_record": (C.c_int, [vp, vp]),
    "ul_stream_wait_event": (C.c_int, [vp, vp]),
    "ul_event_query": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "ul_event_sync": (C.c_int, [vp]),
    "ul_gae_f32": (C.c_int, [vp, vp, vp, vp, vp, vp, i64, i64, f64, f64, vp, vp, vp]),
    "ul_vtrace_f32": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, f64, f64, f64, vp, vp,
                                vp]),
    "ul_opt_ctl_bytes": (i64, []),
    "ul_opt_ctl_init": (C.c_int, [C.POINTER(OptCtl), C.c_int, C.POINTER(f64), f64, f64, f64,
                                  f64]),
    "ul_clip_global_norm": (C.c_int, [C.POINTER(vp), C.POINTER(i64), C.c_int, vp, vp]),
    "ul_adam_step": (C.c_int, [C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                               C.POINTER(i64), C.c_int, vp, C.c_int, vp]),
    "ul_polyak": (C.c_int, [vp, vp, i64, f64, vp]),
    "ul_net_param_count": (i64, [C.POINTER(NetDesc)]),
    "ul_mlp_act_floats": (i64, [C.POINTER(NetDesc), i64]),
    "ul_mlp_bwd_work_floats": (i64, [C.POINTER(NetDesc), i64]),
    "ul_mlp_wstage_floats": (i64, [C.POINTER(NetDesc)]),
    "ul_stage_weights": (C.c_int, [C.POINTER(NetDesc), vp, vp, vp]),
    "ul_stage_weights_ex": (C.c_int, [C.POINTER(NetDesc), vp, vp, C.c_int, vp]),
    "ul_mlp_act_ld": (i64, [C.c_int, C.c_int]),
    "ul_mlp_forward": (C.c_int, [C.POINTER(NetDesc), vp, vp, C.c_int, vp, i64, i64, vp, vp, i64,
                                 vp]),
    "ul_mlp_forward2": (C.c_int, [C.POINTER(NetDesc), vp, vp, vp, i64, vp, vp, i64,
                                  C.POINTER(NetDesc), vp, vp, vp, i64, vp, vp, i64, C.c_int, i64,
                                  vp]),
    "ul_mlp_backward": (C.c_int, [C.POINTER(NetDesc), vp, vp, C.c_int, vp, i64, C.c_int, i64, vp,
                                  vp, i64, vp, vp, i64, vp, vp]),
    "ul_gemm_f32": (C.c_int, [C.c_int, C.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp,
                              vp, i64, vp]),
    "ul_gemm_tc": (C.c_int, [C.c_int, C.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp,
                             vp, i64, C.c_int, C.c_int, vp]),
    "ul_tc_trace": (C.c_int, [vp]),
    "ul_tc_trace_reset": (C.c_int, []),
    "ul_nstep_state_bytes": (i64, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "ul_nstep_push": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, f64, f64, f64, f64, vp,
                                vp, vp, vp, vp, vp, vp, i64, i64, i64, vp, vp]),
    "ul_nstep_norm_stats": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]),
    "ul_gather_rows": (C.c_int, [C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64),
                                 C.POINTER(i64), C.POINTER(i64), vp, vp, i64, i64, i64, i64, vp,
                                 vp]),
    "ul_rows_to_bf16": (C.c_int, [vp, i64, C.c_int, vp, i64, i64, C.c_int, vp]),
    "ul_gather_rows_cvt": (C.c_int, [C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64),
                                     C.POINTER(i64), C.POINTER(i64), vp, vp, vp, i64, vp]),
    "ul_narrow_f64": (C.c_int, [C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64), vp]),
    "ul_ring_insert": (C.c_int, [vp, i64, i64, i64, vp, i64, vp]),
    "ul_device_permutation": (C.c_int, [i64, C.c_uint64, vp, vp]),
    "ul_device_permutations": (C.c_int, [i64, C.c_int, C.POINTER(C.c_uint64), vp, i64, vp]),
    "ul_norm_work_bytes": (i64, [i64]),
    "ul_norm_update": (C.c_int, [vp, i64, i64, i64, vp, vp, C.c_int, vp]),
    "ul_norm_apply": (C.c_int, [vp, i64, i64, i64, vp, vp, i64, vp]),
    "ul_gaussian_logp": (C.c_int, [vp, i64, vp, vp, i64, i64, C.c_int, vp, vp]),
    "ul_api_work_doubles": (i64, []),
    "ul_gaussian_dist": (C.c_int, [vp, i64, vp, vp, i64, vp, i64, C.c_int, C.c_int, vp, vp, vp,
                                   vp]),
    "ul_sample_squashed": (C.c_int, [vp, i64, vp, vp, i64, i64, C.c_int, vp, vp, vp, vp]),
    "ul_sac_soft_target": (C.c_int, [vp, vp, vp, vp, vp, vp, f64, f64, i64, vp, vp]),
    "ul_sac_mse_head": (C.c_int, [vp, vp, i64, vp, vp, vp, vp]),
    "ul_sac_pick_head": (C.c_int, [vp, vp, vp, i64, f64, vp, vp, vp, vp, vp]),
    "ul_sac_actor_head": (C.c_int, [vp, vp, vp, vp, i64, vp, i64, C.c_int, f64, vp, vp, vp,
                                    vp]),
    "ul_sum_f64": (C.c_int, [vp, i64, f64, vp, vp, vp]),
    "ul_ppo_plan_create": (C.c_int, [C.POINTER(PpoPlanDesc), C.POINTER(vp)]),
    "ul_ppo_plan_destroy": (C.c_int, [vp]),
    "ul_ppo_plan_bind": (C.c_int, [vp, C.POINTER(PpoBindings)]),
    "ul_ppo_plan_begin": (C.c_int, [vp, f64, f64, i64, i64, vp]),
    "ul_ppo_plan_adv_sums": (C.c_int, [vp, vp, vp]),
    "ul_ppo_plan_adv_finalize": (C.c_int, [vp, vp, vp]),
    "ul_ppo_plan_step_grads": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "ul_ppo_plan_step_apply": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "ul_ppo_plan_reduce_buffer": (C.c_int, [vp, C.POINTER(vp), C.POINTER(i64)]),
    "ul_ppo_plan_run": (C.c_int, [vp, f64, f64, i64, i64, C.c_int, vp]),
    "ul_ppo_plan_run_after": (C.c_int, [vp, vp, f64, f64, vp]),
    "ul_ppo_plan_collect": (C.c_int, [vp, vp]),
    "ul_ppo_plan_run_epoch": (C.c_int, [vp, C.c_int, f64, f64, i64, i64, vp]),
    "ul_ppo_plan_finish": (C.c_int, [vp, C.POINTER(PpoResult), vp]),
    "ul_sac_plan_create": (C.c_int, [C.POINTER(SacPlanDesc), C.POINTER(vp)]),
    "ul_sac_plan_destroy": (C.c_int, [vp]),
    "ul_sac_plan_bind": (C.c_int, [vp, C.POINTER(SacBindings)]),
    "ul_sac_plan_load_rows": (C.c_int, [vp, vp, i64, vp, i64, i64, i64, vp, vp]),
    "ul_sac_plan_begin": (C.c_int, [vp, C.POINTER(SacCtl), C.POINTER(f64), C.POINTER(i64), vp]),
    "ul_sac_plan_noise_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "ul_sac_plan_reserve": (C.c_int, [vp, C.c_int]),
    "ul_sac_plan_run": (C.c_int, [vp, C.c_int, i64, C.c_int, vp]),
    "ul_sac_plan_device_noise": (C.c_int, [vp, C.c_uint64, C.c_uint64, vp]),
    "ul_sac_plan_update": (C.c_int, [vp, C.c_int, vp]),
    "ul_sac_plan_reduce_buffers": (C.c_int, [vp, C.POINTER(vp), C.POINTER(i64), C.POINTER(vp),
                                             C.POINTER(i64)]),
    "ul_sac_plan_critic_grads": (C.c_int, [vp, vp]),
    "ul_sac_plan_critic_apply": (C.c_int, [vp, vp]),
    "ul_sac_plan_actor_grads": (C.c_int, [vp, vp]),
    "ul_sac_plan_actor_apply": (C.c_int, [vp, vp]),
    "ul_sac_plan_polyak": (C.c_int, [vp, vp]),
    "ul_sac_plan_finish": (C.c_int, [vp, C.POINTER(SacCtl), C.POINTER(i64), vp, C.c_int, vp]),
    "ul_ppo_plan_counts": (C.c_int, [vp, C.POINTER(i64), C.POINTER(f64)]),
    "ul_ppo_plan_profile": (C.c_int, [vp, f64, f64, i64, i64, C.POINTER(f64), vp]),
}

_lib = None


def exported_names():
    return list(_PROTOS)


def lib():
    """Load the library once; raises (no fallback) when it is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built (run __graft_entry__.build()); "
                "paper_2605_30313_b200 has no CPU fallback")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _PROTOS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


_EXC = {1: ValueError, 2: IndexError, 3: DivergenceError, 4: SlotStateError, 5: RuntimeError}


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = lib().ul_last_error().decode(errors="replace")
    exc = _EXC.get(status, RuntimeError)
    raise exc(f"{what}: {msg}" if what and status == 5 else msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


def ptr_array(ptrs):
    arr = (vp * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def i64_array(vals):
    arr = (i64 * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
