"""B200-native SAIS / SSMC samplers (arXiv 2408.12057) -- drop-in for the reference `asmc` API."""
from . import abi  # noqa: F401  (ctypes layouts only)
