"""B200-native SAIS / SSMC samplers (arXiv 2408.12057): a drop-in for the reference `asmc` module.

    import paper_2408_12057_b200 as asmc
    rounds = asmc.run_sais(asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 10), asmc.Kernel(),
                           asmc.DriverOptions())

Same names and semantics as the reference's pybind module (proj/python/bindings.cpp),
implemented by the host C++ mirror (csrc/host) over the C-ABI (include/asmc_b200.h)
of the sm_100a kernels.  There is no CPU sampler: importing works anywhere, but
sampling without a CUDA device raises DeviceError.
"""
from . import abi  # noqa: F401  (ctypes layouts of the C-ABI; loads nothing)

try:
    from ._core import *  # noqa: F401,F403
    from ._core import theory  # noqa: F401
    _CORE_ERROR = None
except ImportError as exc:  # pragma: no cover - exercised only when the build is missing
    _CORE_ERROR = exc

    def __getattr__(name):
        raise ImportError(
            f"paper_2408_12057_b200: native module _core is not built ({_CORE_ERROR}); "
            "run `python -c 'import __graft_entry__ as g; g.build()'`")

__all__ = [name for name in dir() if not name.startswith("_")]
