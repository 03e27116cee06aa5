"""B200-native half-space Spectral Ewald (drop-in for the reference ``hsewald`` hot path).

Entry points keep the reference's names and semantics:
``ewald_sum``, ``real_space_sum``, ``fourier_space_sum``, ``build_cell_list``,
``spread``, ``gather``, ``precompute_greens``, ``get_tables``,
``direct_sum_half`` / ``direct_sum_free``.  All array work runs in
hand-written sm_100a FP64 CUDA kernels (+ cuFFT for the transforms) behind the
C ABI in include/hsewald_b200.h; there is no CPU fallback.
"""

from .errors import (ConfigError, DeviceError, GeometryError, HsewaldError, InfeasibleToleranceError,
                     ParameterError, ResourceError, SingularityError)
from .system import (FREE_SPACE, HALF_SPACE, KINDS, ROTLET, STOKESLET, STRESSLET, ImageSystem, PointSystem,
                     VelocityResult, generate_system, reflect)
from .ewald_fourier import (BIHARMONIC, HARMONIC, GreensTable, GridSpec, fourier_space_sum, gather, get_tables,
                            load_table, precompute_greens, save_table, spread, table_kinds_for,
                            truncated_greens_hat)
from .ewald_real import CellList, RealSpaceParams, build_cell_list, real_space_sum, self_interaction
from .ewald import EwaldParams, ewald_sum
from .kernels_direct import direct_sum_free, direct_sum_half
from .point_kernels import (HarmonicDerivs, correction_phi, harmonic_derivs, kernel_real, rotlet_apply, stokeslet,
                            stresslet_apply)
from .ewald_real import f_derivs

__all__ = [n for n in dir() if not n.startswith("_")]
