"""B200-native (sm_100a) time-stepping hot path of the energy-conserving
split-form SBP discretisation of the hyperbolized Serre-Green-Naghdi
equations (arXiv 2601.02540), behind the reference library's operator API.

See DESIGN.md for the kernel design and INTEGRATION.md for the C ABI.
"""
from .api import (AcceptObserver, BoundaryKind, DepthError, DeviceState, Grid2D, HsgnError,
                  IntegratorConfig, PhysSetup, RhsContext, SolutionRecord, StateField, adaptive_solve,
                  bs3_fixed_steps, direction_spacing, discrete_l2_error, energy_rate, eoc, init_auxiliary,
                  make_grid, make_rhs_context, mass_weighted_sum, prepare_fixed_steps, kernel_times, set_kernel_timing, rhs, rhs_periodic, rhs_reflecting, rhs_shallow_water,
                  total_energy, total_mass)
from .recorder import RunRecorder

__all__ = [
    "AcceptObserver", "BoundaryKind", "DepthError", "DeviceState", "Grid2D", "HsgnError", "IntegratorConfig",
    "PhysSetup", "RhsContext", "SolutionRecord", "StateField", "adaptive_solve", "bs3_fixed_steps",
    "direction_spacing", "discrete_l2_error", "energy_rate", "eoc", "init_auxiliary", "make_grid",
    "make_rhs_context", "mass_weighted_sum", "prepare_fixed_steps", "kernel_times", "set_kernel_timing", "rhs", "rhs_periodic", "rhs_reflecting", "rhs_shallow_water", "total_energy",
    "total_mass", "RunRecorder",
]
