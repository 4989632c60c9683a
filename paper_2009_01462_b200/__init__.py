"""B200-native layer-parallel ResNet training step (arXiv 2009.01462).

Drop-in for the reference respar library's hot path (DecoupledTrainer::step and
serial_train_step): hand-written sm_100a CUDA kernels behind the C ABI in
include/respar_b200.h, a C++ host mirror of the reference's trainer API, and this
Python front end.  See DESIGN.md.
"""
from .trainer import (  # noqa: F401
    ALM, BOUNDARY_ADJOINT, BOUNDARY_OUT, IDENTITY, KAPPA, KAPPA_RULE_REFERENCE, KAPPA_RULE_TEXTBOOK, L1, LAMBDA,
    LINF, MATH, PENALTY, SERIAL, SQUARED_L2, TANH, ConfigError, DecoupledTrainer, DeviceError, DivergedError,
    Geometry, InvalidArgument, LogicError, SerialTrainer, ShapeError, StageError, StepParams, check, launch_count,
    normalizer, param_count, partition, serial_train_step)
from . import harness, init  # noqa: E402,F401  (train / configs / metrics; build_initial_net)
from .harness import (  # noqa: E402,F401
    Dataset, ExperimentSummary, MetricsRow, Schedules, TrainConfig, default_config, gen_circles, load_config_file,
    parse_config_json, run_experiment, train)
from .init import build_initial_net  # noqa: E402,F401
