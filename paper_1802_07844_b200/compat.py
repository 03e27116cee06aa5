"""Run unchanged callers of the reference package against this one.

`install_as_hsewald()` registers this package (and its modules) under the reference's
import names, so code written for `hsewald` -- `from hsewald.ewald import ewald_sum`,
`from hsewald.ewald_fourier import get_tables`, `hsewald.bench.break_even(...)`, the
reference's own experiment scripts -- evaluates on the GPU without edits
(INTEGRATION.md section 1).  Module map (reference -> here): ewald, ewald_fourier,
ewald_real, kernels_direct, estimates, errors, system (same names); bench -> experiments.
The reference's CLI and its private `_gridding` module are not provided (out of scope,
DESIGN.md section 8).
"""

from __future__ import annotations

import importlib
import sys

_MODULES = {
    "ewald": "ewald", "ewald_fourier": "ewald_fourier", "ewald_real": "ewald_real",
    "kernels_direct": "kernels_direct", "estimates": "estimates", "errors": "errors",
    "system": "system", "bench": "experiments",
}


def install_as_hsewald(name: str = "hsewald", replace: bool = False):
    """Alias this package as `name` in sys.modules; returns the package.  An already imported
    module of that name is kept unless replace=True."""
    if name in sys.modules and not replace:
        return sys.modules[name]
    pkg = importlib.import_module(__package__)
    sys.modules[name] = pkg
    for ref_mod, here in _MODULES.items():
        mod = importlib.import_module(f"{__package__}.{here}")
        sys.modules[f"{name}.{ref_mod}"] = mod
        setattr(pkg, ref_mod, mod)
    return pkg
