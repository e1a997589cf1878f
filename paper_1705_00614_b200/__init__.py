"""B200-native CSPH-TVD shallow-water time step (arXiv 1705.00614).

The hot path swflood::CsphTvdStepper::step, rebuilt as hand-written sm_100a
CUDA kernels behind a C ABI (include/swf.h, libswflood_cuda.so), with the
reference's solver API mirrored on top (stepper.py, types.py).
"""
from .types import (BlockMask, BoundaryConfig, CellRect, ConfigError, EdgeKind, FlowState,
                    ForceField, HydrographSample, NumericalError, PhysicalParams, SourceField,
                    SourceKind, SourceSpec, StageTimings, StepInfo, StepperOptions, Terrain,
                    TimestepControl, Vec2, WindForcing, WindSample, free_surface,
                    latitude_to_omega_z, total_volume, velocity)

__all__ = [
    "BlockMask", "BoundaryConfig", "CellRect", "ConfigError", "EdgeKind", "FlowState",
    "ForceField", "HydrographSample", "NumericalError", "PhysicalParams", "SourceField",
    "SourceKind", "SourceSpec", "StageTimings", "StepInfo", "StepperOptions", "Terrain",
    "TimestepControl", "Vec2", "WindForcing", "WindSample", "free_surface",
    "latitude_to_omega_z", "total_volume", "velocity", "CsphTvdStepper",
]


def __getattr__(name):
    # the CUDA-backed stepper loads libswflood_cuda.so lazily, so the value
    # types stay importable on machines without the built library
    if name == "CsphTvdStepper":
        from .stepper import CsphTvdStepper
        return CsphTvdStepper
    raise AttributeError(name)
