"""ctypes binding of include/respar_b200.h (librespar_b200.so, built in-tree).

There is no fallback: if the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# RP_LIB_PATH: load another build of the same library (tools/mutation_check.sh points the
# parity tests at a deliberately broken build to show that they fail)
LIB_PATH = os.environ.get("RP_LIB_PATH") or os.path.join(_PKG, "librespar_b200.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "respar_b200.h")

RP_OK, RP_ERR_SHAPE, RP_ERR_CONFIG, RP_ERR_STATE, RP_ERR_RANGE, RP_ERR_STAGE, RP_ERR_CUDA, RP_ERR_NCCL, \
    RP_ERR_DIVERGED, RP_ERR_INTERNAL = range(10)


class rp_geometry(C.Structure):
    _fields_ = [("in_channels", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("channels", C.c_int32), ("hidden", C.c_int32), ("blocks", C.c_int32),
                ("classes", C.c_int32), ("activation", C.c_int32), ("step_h", C.c_double)]


class rp_step_params(C.Structure):
    _fields_ = [("beta", C.c_double), ("tau", C.c_double), ("lr", C.c_double), ("lambda_lr", C.c_double),
                ("kappa_lr", C.c_double), ("max_corrections", C.c_int32), ("momentum", C.c_double)]


_P = C.c_void_p
_F = C.POINTER(C.c_float)
_I32 = C.POINTER(C.c_int32)
_D = C.POINTER(C.c_double)
_G = C.POINTER(rp_geometry)
_SP = C.POINTER(rp_step_params)
_U64P = C.POINTER(C.c_uint64)
_I64P = C.POINTER(C.c_int64)

# name -> (restype, argtypes); every symbol declared in include/respar_b200.h
SIGNATURES = {
    "rp_last_error": (C.c_char_p, []),
    "rp_version": (C.c_int, []),
    "rp_launch_count": (C.c_uint64, []),
    "rp_param_count": (C.c_int64, [_G]),
    "rp_param_offset_block": (C.c_int64, [_G, C.c_int32]),
    "rp_param_offset_head": (C.c_int64, [_G]),
    "rp_op_fill_uniform": (C.c_int, [_P, C.c_int64, _U64P, C.c_double, C.c_double, C.c_double, _P]),
    "rp_op_fill_normal": (C.c_int, [_P, C.c_int64, _U64P, C.c_double, C.c_double, C.c_int32, _P]),
    "rp_op_init_params": (C.c_int, [_G, _P, _U64P, _P]),
    "rp_op_reduce_workspace_bytes": (C.c_int64, []),
    "rp_op_psi": (C.c_int, [C.c_int32, _P, _P, C.c_int64, _D, _P, _P]),
    "rp_op_psi_grad": (C.c_int, [C.c_int32, _P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "rp_op_synthetic_grad": (C.c_int, [C.c_int32, _P, _P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "rp_op_correct": (C.c_int, [C.c_int32, _P, _P, _P, _P, C.c_int64, C.c_double, C.c_double, C.c_int32,
                                C.c_double, C.c_int32, _P, _P]),
    "rp_op_sgd": (C.c_int, [_P, _P, _P, C.c_int64, C.c_double, C.c_double, _P]),
    "rp_op_conv3x3": (C.c_int, [C.c_int32] * 5 + [_P, _P, C.c_int32, _P, _P, C.c_double, C.c_int32, _P, C.c_int32,
                                                 _P, C.c_int64, _P]),
    "rp_op_conv3x3_workspace_bytes": (C.c_int64, [C.c_int32, C.c_int32]),
    "rp_op_conv3x3_wgrad": (C.c_int, [C.c_int32] * 5 + [_P, _P, C.c_double, _P, _P, C.c_int32, _P, C.c_int64, _P]),
    "rp_op_conv3x3_wgrad_workspace_bytes": (C.c_int64, [C.c_int32] * 5),
    "rp_op_split_planes": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P]),
    "rp_op_conv3x3_planes": (C.c_int, [C.c_int32] * 5 + [_P, _P, C.c_int32, _P, _P, C.c_double, C.c_int32, _P, _P,
                                                         _P, _P, _P, C.c_int64, _P]),
    "rp_op_set_plane_conv_kernel": (C.c_int, [C.c_int32]),
    "rp_op_set_concurrent_stages": (C.c_int, [C.c_int32]),
    "rp_op_concurrent_stages": (C.c_int32, []),
    "rp_op_plane_conv_kernel": (C.c_int32, [C.c_int32] * 5),
    "rp_op_block_planes_supported": (C.c_int32, [_G, C.c_int32, C.c_int32]),
    "rp_op_block_fwd_planes": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int64, _P]),
    "rp_op_block_bwd_planes": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int64,
                                         _P]),
    "rp_op_planes_filters_bytes": (C.c_int64, [_G, C.c_int32]),
    "rp_op_block_bf16_tape_supported": (C.c_int32, [_G, C.c_int32, C.c_int32]),
    "rp_op_synthetic_grad_planes": (C.c_int, [C.c_int32, _P, _P, _P, C.c_int64, C.c_double, _P, _P, _P, _P, _P,
                                               _P]),
    "rp_op_plane_scale_bytes": (C.c_int64, []),
    "rp_op_block_fwd_bf16t": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int64, _P]),
    "rp_op_block_bwd_bf16t": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int64, _P]),
    "rp_op_conv3x3_wgrad_bf16p": (C.c_int, [C.c_int32] * 5 + [_P, _P, C.c_double, _P, _P, _P, C.c_int64, _P]),
    "rp_op_conv3x3_wgrad_bf16p_workspace_bytes": (C.c_int64, [C.c_int32] * 5),
    "rp_op_prep_planes_filters": (C.c_int, [_G, _P, C.c_int32, C.c_int32, _P, _P]),
    "rp_op_conv3x3_wgrad_planes": (C.c_int, [C.c_int32] * 5 + [_P, _P, _P, _P, C.c_double, _P, _P, _P, _P,
                                                                C.c_int64, _P]),
    "rp_op_conv3x3_wgrad_planes_workspace_bytes": (C.c_int64, [C.c_int32] * 5),
    "rp_op_block_fwd": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, C.c_int32, _P, C.c_int64, _P]),
    "rp_op_block_bwd": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P, C.c_int32, _P, C.c_int64, _P]),
    "rp_op_workspace_bytes": (C.c_int64, [_G, C.c_int32, C.c_int32]),
    "rp_op_stem_fwd": (C.c_int, [_G, C.c_int32, _P, _P, _P, C.c_int32, _P, C.c_int64, _P]),
    "rp_op_stem_fwd_planes": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P]),
    "rp_op_stem_bwd": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, C.c_int64, _P]),
    "rp_op_head_fwd": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P]),
    "rp_op_head_loss_bwd": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int64, _P]),
    "rp_op_head_loss_bwd_planes": (C.c_int, [_G, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                             C.c_int64, _P]),
    "rp_op_argmax_hits": (C.c_int, [_P, _P, C.c_int32, C.c_int32, _I64P, _P, _P]),
    "rp_trainer_create": (C.c_int, [_G, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _F, _U64P, C.c_int32,
                                    _I32, C.c_int32, C.POINTER(_P)]),
    "rp_trainer_destroy": (C.c_int, [_P]),
    "rp_trainer_create_local": (C.c_int, [_G, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _F, _U64P, C.c_int32,
                                          C.c_int32, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "rp_trainer_local_range": (C.c_int, [_P, _I32, _I32]),
    "rp_trainer_reset_local": (C.c_int, [_P, _P]),
    "rp_trainer_step_local": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, _SP]),
    "rp_trainer_correct_ghost": (C.c_int, [_P, _SP, C.c_int32, C.c_int32]),
    "rp_trainer_state_device": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "rp_trainer_stage_stream": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "rp_trainer_loss_device": (C.c_int, [_P, C.POINTER(_P)]),
    "rp_trainer_forward_local": (C.c_int, [_P, _P, C.c_int32, _P]),
    "rp_trainer_set_kappa_rule": (C.c_int, [_P, C.c_int32]),
    "rp_trainer_set_graphs": (C.c_int, [_P, C.c_int32]),
    "rp_trainer_get_params": (C.c_int, [_P, _F]),
    "rp_trainer_set_params": (C.c_int, [_P, _F]),
    "rp_trainer_get_grads": (C.c_int, [_P, _F]),
    "rp_trainer_reset_lambda_from_forward": (C.c_int, [_P, _F]),
    "rp_trainer_step": (C.c_int, [_P, _F, _I32, C.c_int32, C.c_int32, _SP, _D]),
    "rp_trainer_step_device": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, _SP, _D]),
    "rp_trainer_last_loss": (C.c_int, [_P, _D]),
    "rp_trainer_take_snapshot": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32]),
    "rp_trainer_stage_forward": (C.c_int, [_P, C.c_int32, _F, C.c_int32, C.c_int32]),
    "rp_trainer_stage_backward_update": (C.c_int, [_P, C.c_int32, _I32, C.c_int32, C.c_double, C.c_double,
                                                   C.c_int32]),
    "rp_trainer_correct_aux": (C.c_int, [_P, C.c_int32, _SP, C.c_int32, C.c_int32]),
    "rp_trainer_correct_multiplier": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int32]),
    "rp_trainer_correction_gradient": (C.c_int, [_P, C.c_int32, C.c_double, C.c_int32, C.c_int32, _F]),
    "rp_trainer_violation_report": (C.c_int, [_P, _D, _D, _I64P]),
    "rp_trainer_get_state": (C.c_int, [_P, C.c_int32, C.c_int32, _F]),
    "rp_trainer_set_state": (C.c_int, [_P, C.c_int32, C.c_int32, _F]),
    "rp_trainer_forward": (C.c_int, [_P, _F, C.c_int32, _F]),
    "rp_trainer_iteration": (C.c_int64, [_P]),
    "rp_trainer_stages": (C.c_int32, [_P]),
    "rp_trainer_last_step_ms": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "rp_serial_train_step": (C.c_int, [_P, _F, _I32, C.c_int32, C.c_double, _D]),
    "rp_trainer_region": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_float)]),
    "rp_op_eval_workspace_bytes": (C.c_int64, [C.c_int32]),
    "rp_op_eval_loss_accuracy": (C.c_int, [_P, _P, C.c_int32, C.c_int32, _D, _I64P, _P, _P, C.c_int64, _P]),
    "rp_trainer_evaluate": (C.c_int, [_P, _F, _I32, C.c_int32, _D, _D]),
    "rp_comm_unique_id": (C.c_int, [_P]),
    "rp_comm_create": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "rp_comm_destroy": (C.c_int, [_P]),
    "rp_pipeline_create": (C.c_int, [_P, _P, C.POINTER(_P), _I32, _I32, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "rp_pipeline_reset_lambda_from_forward": (C.c_int, [_P, _P]),
    "rp_pipeline_step": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, _SP, _D]),
    "rp_pipeline_loss": (C.c_int, [_P, _D]),
    "rp_pipeline_set_graphs": (C.c_int, [_P, C.c_int32]),
    "rp_pipeline_region": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_float)]),
    "rp_pipeline_sync": (C.c_int, [_P]),
    "rp_pipeline_destroy": (C.c_int, [_P]),
    "rp_profile_enable": (C.c_int, [C.c_int32]),
    "rp_profile_collect": (C.c_int, [_I64P, _D, _D, _D]),
    "rp_profile_class_name": (C.c_char_p, [C.c_int32]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.isfile(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the B200 kernels are not built.  Run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback).")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().rp_last_error().decode(errors="replace")
