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
