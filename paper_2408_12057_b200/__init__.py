"""B200-native SAIS / SSMC samplers (arXiv 2408.12057): a drop-in for the reference `asmc` module.

    import paper_2408_12057_b200 as asmc
    rounds = asmc.run_sais(asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 10), asmc.Kernel(),
                           asmc.DriverOptions())

Same names and semantics as the reference's pybind module (proj/python/bindings.cpp),
implemented by the host C++ mirror (csrc/host) over the C-ABI (include/asmc_b200.h)
of the sm_100a kernels.  There is no CPU sampler: importing works anywhere, but
sampling without a CUDA device raises DeviceError.

The native module `_core` (and through it libasmc_b200.so) is loaded on first use of
one of its names, not at package import: `from paper_2408_12057_b200 import abi`
(the ctypes layouts) maps no shared object, so the CPU reference arm of bench.py
runs with none of this package's native code in the process.
"""
import importlib

from . import abi  # noqa: F401  (ctypes layouts of the C-ABI; loads nothing)

_core = None
_CORE_ERROR = None


def _load_core():
    global _core, _CORE_ERROR
    if _core is None and _CORE_ERROR is None:
        try:
            _core = importlib.import_module("._core", __name__)
        except ImportError as exc:  # pragma: no cover - only when the build is missing
            _CORE_ERROR = exc
    if _core is None:
        raise ImportError(
            f"paper_2408_12057_b200: native module _core is not built ({_CORE_ERROR}); "
            "run `python -c 'import __graft_entry__ as g; g.build()'`")
    return _core


def __getattr__(name):
    if name.startswith("__") and name != "__all__":
        raise AttributeError(name)
    core = _load_core()
    if name == "__all__":
        return ["abi"] + [n for n in dir(core) if not n.startswith("_")]
    try:
        return getattr(core, name)
    except AttributeError:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}") from None


def __dir__():
    names = set(globals())
    try:
        names.update(n for n in dir(_load_core()) if not n.startswith("_"))
    except ImportError:
        pass
    return sorted(names)
