"""B200-native photon gather + ANOVA F-test radius update (arXiv 2504.04411).

The hot path of hypothesis-tested progressive photon mapping (FPPM) and the
VCM+ merge stage, as hand-written sm_100a CUDA kernels behind a C ABI
(include/fppm_gpu.h, libfppm_gpu.so).  See DESIGN.md.
"""
from .api import (FppmContext, GatherRegionBatch, PhotonGrid, RadiusSchedule, TestConfig,  # noqa: F401
                  chi2_quantile, f_quantile, schedule_radius, InvalidArgument, DomainError,
                  FppmError, NoDeviceError, CapacityError, StateError, CudaError)
from .workloads import WORKLOADS, Workload  # noqa: F401

__all__ = ["FppmContext", "GatherRegionBatch", "PhotonGrid", "RadiusSchedule", "TestConfig",
           "chi2_quantile", "f_quantile", "schedule_radius", "WORKLOADS", "Workload"]
