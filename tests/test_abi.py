"""CPU: the C-ABI library builds, loads without a GPU, and exports every symbol that
include/respar_b200.h declares; host-side logic that needs no device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from paper_2009_01462_b200 import _lib

HEADER = _lib.HEADER


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("rp_trainer_step", "rp_trainer_stage_forward", "rp_trainer_stage_backward_update",
                 "rp_trainer_correct_aux", "rp_trainer_correct_multiplier", "rp_trainer_correction_gradient",
                 "rp_trainer_violation_report", "rp_trainer_reset_lambda_from_forward", "rp_serial_train_step",
                 "rp_op_block_fwd", "rp_op_block_bwd", "rp_op_synthetic_grad", "rp_op_correct", "rp_op_sgd"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert set(declared_functions()) <= set(_lib.SIGNATURES), set(declared_functions()) - set(_lib.SIGNATURES)


def test_built_for_sm100a_only():
    """The .so carries sm_100a SASS (tcgen05-capable target), nothing else."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_param_layout_matches_oracle():
    from oracle import respar_oracle as O
    og = O.Geometry(3, 8, 8, 16, 12, 5, 10)
    g = rp.Geometry(3, 8, 8, 16, 12, 5, 10)
    assert rp.param_count(g) == O.param_count(og)
    L = _lib.lib()
    assert L.rp_param_offset_block(C.byref(g.c()), 0) == 9 * 3 * 16 + 16
    assert L.rp_param_offset_head(C.byref(g.c())) == O.param_count(og) - 16 * 10 - 10


def test_geometry_validation_without_gpu():
    with pytest.raises(rp.ConfigError):
        rp.param_count(rp.Geometry(3, 8, 8, 16, 16, 4, 1))   # classes >= 2
    with pytest.raises(rp.ConfigError):
        rp.param_count(rp.Geometry(0, 8, 8, 16, 16, 4, 10))


def test_partition_and_normalizer():
    assert rp.partition(60, 4) == [(0, 15), (15, 30), (30, 45), (45, 60)]   # test_decoupled.cpp:76-90
    assert rp.partition(60, 1) == [(0, 60)]
    with pytest.raises(rp.ConfigError):
        rp.partition(60, 7)
    with pytest.raises(rp.ConfigError):
        rp.partition(60, 0)
    assert rp.normalizer(200, 8) == 1600                                     # test_decoupled.cpp:309-327


def test_status_codes_map_to_reference_exceptions():
    assert issubclass(rp.ShapeError, ValueError) and issubclass(rp.ConfigError, ValueError)
    with pytest.raises(rp.ShapeError):
        rp.check(_lib.RP_ERR_SHAPE)
    with pytest.raises(rp.LogicError):
        rp.check(_lib.RP_ERR_STATE)
    with pytest.raises(rp.InvalidArgument):
        rp.check(_lib.RP_ERR_RANGE)
    with pytest.raises(rp.StageError):
        rp.check(_lib.RP_ERR_STAGE)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="CPU-only behaviour")
def test_no_cpu_fallback():
    """Without a GPU the product fails loudly instead of computing on the CPU."""
    g = rp.Geometry(3, 8, 8, 16, 16, 4, 10)
    with pytest.raises(rp.DeviceError):
        rp.DecoupledTrainer(g, 2, rp.ALM, rp.SQUARED_L2, 4, seed_state=1)


def test_plane_conv_kernel_choice_and_share_switches():
    """Host-only plan logic: which plane conv takes a shape (1 positions-as-M, 0 channels-as-M,
    -1 none), the process-wide override, and the thread-local concurrent-stage setting."""
    L = _lib.lib()
    assert L.rp_op_plane_conv_kernel(256, 32, 32, 64, 64) == 1      # C = 64: conv_pm by default
    assert L.rp_op_plane_conv_kernel(128, 28, 28, 16, 16) == 1      # C1's 16 channels: conv_pm only
    assert L.rp_op_plane_conv_kernel(4, 16, 16, 64, 128) == 0       # Co 128: conv_tc only
    assert L.rp_op_plane_conv_kernel(4, 16, 16, 24, 24) == -1       # Ci % 16 != 0: neither
    try:
        assert L.rp_op_set_plane_conv_kernel(0) == 0
        assert L.rp_op_plane_conv_kernel(256, 32, 32, 64, 64) == 0  # forced conv_tc where both apply
        assert L.rp_op_plane_conv_kernel(128, 28, 28, 16, 16) == 1  # a shape only conv_pm takes stays
    finally:
        L.rp_op_set_plane_conv_kernel(-1)
    assert L.rp_op_set_plane_conv_kernel(2) != 0                    # range-checked
    assert L.rp_op_concurrent_stages() == 1
    try:
        assert L.rp_op_set_concurrent_stages(8) == 0 and L.rp_op_concurrent_stages() == 8
    finally:
        L.rp_op_set_concurrent_stages(1)
    assert L.rp_op_set_concurrent_stages(0) != 0


def test_plane_path_coverage():
    """The fp32 plane path (tensor cores end to end) takes C = hidden = 64 and C1's 16 channels;
    32 channels stay on the fp32-operand kernels (no 32-channel weight gradient on planes)."""
    L = _lib.lib()
    fp32 = rp.MATH["fp32"]
    for c, h, w, n, want in ((64, 32, 32, 256, 1), (16, 28, 28, 128, 1), (32, 16, 16, 8, 0), (128, 16, 16, 4, 1)):
        geo = _lib.rp_geometry(3, h, w, c, c, 4, 10, 0, 0.5)
        assert L.rp_op_block_planes_supported(C.byref(geo), n, fp32) == want, c
    geo = _lib.rp_geometry(3, 32, 32, 64, 64, 4, 10, 0, 0.5)
    assert L.rp_op_block_planes_supported(C.byref(geo), 8, rp.MATH["bf16"]) == 0
